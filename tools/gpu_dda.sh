mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k march 2>&1 | tail -4
timeout 900 ncu --set full --clock-control none --import-source on -k regex:march_dda -s 3 -c 1 -o gpurun_out/prof_dda python bench.py --steps 4 --warmup 3 --profile --no-cpu-baseline > gpurun_out/ncu_dda.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_dda.ncu-rep | head -20
