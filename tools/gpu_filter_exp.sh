mkdir -p gpurun_out
bash tools/gpu_ab_filter.sh "-DNACC_FILTER_BATCH=4" "-DNACC_FILTER_BATCH=8" "-DNACC_FILTER_BATCH=16" "-DNACC_FILTER_BATCH=32"
python -c "from paper_2305_04966_b200 import build; build.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "filter" 2>&1 | tail -3
timeout 600 python bench.py --steps 50 --warmup 5 --no-extras > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; tail -3 gpurun_out/bench_e2e.err
python -c "
import json; d=json.load(open('gpurun_out/bench_e2e.json')); print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']); print(d['stage_ms'])"
