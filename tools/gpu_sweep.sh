# march pipelining sweep (experiment)
mkdir -p gpurun_out
run() {
  timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/sweep.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sweep.json')); print('$1', round(d['stage_ms']['march']*1000,1), 'us; step', round(d['ms_per_step'],4))"
}
timeout 900 python -m pytest tests -m gpu -x -q -k march 2>&1 | tail -2
run "pipe1 kcap1024"
for v in "2 1024" "2 768" "3 512" "2 512" "1 768"; do
  set -- $v
  python -c "from paper_2305_04966_b200 import build; build.build(extra=['-DNACC_MARCH_PIPE=$1', '-DNACC_MARCH_KCAP=$2'])"
  run "pipe$1 kcap$2"
done
