mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 python bench.py --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['ms_per_step'], d['stage_ms'], d['e2e']['value'], d['gpu_launches'], d['roofline'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 12 --warmup 3 --profile --no-cpu-baseline > /dev/null 2>&1
python tools/launches.py gpurun_out/launches.csv 2>/dev/null | head -14
