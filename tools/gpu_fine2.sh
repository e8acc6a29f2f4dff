mkdir -p gpurun_out
python -c "from paper_2305_04966_b200 import build; build.build(extra=['-DNACC_MARCH_FINEMASK=2'])"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "march or sampling or bounds or combined or grid" 2>&1 | tail -2
bash tools/gpu_ab.sh "-DNACC_MARCH_FINEMASK=1" "-DNACC_MARCH_FINEMASK=2" | grep -v cfg3
bash tools/gpu_ab_filter.sh "-DNACC_FILTER_BATCH=4" "-DNACC_FILTER_BATCH=8" "-DNACC_FILTER_BATCH=16" 2>&1 | grep -v "^\s"
python -c "from paper_2305_04966_b200 import build; build.build()"
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; tail -3 gpurun_out/bench_e2e.err
python -c "
import json; d=json.load(open('gpurun_out/bench_e2e.json')); print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']); print(d['stage_ms']); print(d['extras'].get('cfg3_frame'))"
