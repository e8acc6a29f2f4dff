mkdir -p gpurun_out
timeout 300 python tools/debug_resample.py 2>&1 | tail -12
timeout 900 ncu --set full --clock-control none --import-source on -k regex:march_fused -s 3 -c 1 -o gpurun_out/prof_march python bench.py --steps 4 --warmup 3 --profile --no-cpu-baseline > gpurun_out/ncu_march.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:filter_cut -s 3 -c 1 -o gpurun_out/prof_filter python bench.py --steps 4 --warmup 3 --profile --no-cpu-baseline > gpurun_out/ncu_filter.log 2>&1
ls gpurun_out
