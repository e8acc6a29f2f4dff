# march build-parameter sweep (experiment)
mkdir -p gpurun_out
run() {
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/sweep.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sweep.json')); print('$1', round(d['stage_ms']['march']*1000,1), 'us; step', round(d['ms_per_step'],4))"
}
run "default"
for v in "-DNACC_MARCH_PREFETCH=1"; do
  python -c "from paper_2305_04966_b200 import build; build.build(extra='$v'.split())"
  timeout 900 python -m pytest tests -m gpu -x -q -k march 2>&1 | tail -1
  run "$v"
  NACC_MARCH_CARVEOUT=70 NACC_MARCH_BPS=8 run "$v carve70 bps8"
done
