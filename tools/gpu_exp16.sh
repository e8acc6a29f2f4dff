mkdir -p gpurun_out
timeout 300 python tools/bench_resample.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:importance -c 1 -o gpurun_out/prof_importance -f python tools/bench_resample.py > gpurun_out/ncu_importance.log 2>&1
