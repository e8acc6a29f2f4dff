mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --steps 200 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 12 --warmup 3 --profile --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:march_kernel -s 4 -c 2 -o gpurun_out/prof_march python bench.py --steps 4 --warmup 3 --profile --no-cpu-baseline > gpurun_out/ncu_march.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_bwd -s 3 -c 1 -o gpurun_out/prof_rbwd python bench.py --steps 4 --warmup 3 --profile --no-cpu-baseline > gpurun_out/ncu_rbwd.log 2>&1
ls gpurun_out
