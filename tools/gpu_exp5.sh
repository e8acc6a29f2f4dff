mkdir -p gpurun_out
python -c "from paper_2305_04966_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "march or sampling or bounds or combined" 2>&1 | tail -2
for rep in 1 2; do
  for v in "-DNACC_LB_PER=1" "-DNACC_LB_PER=2" "-DNACC_LB_PER=4" "-DNACC_LB_PER=8"; do
    python -c "from paper_2305_04966_b200 import build; build.build(extra='$v'.split())"
    echo "== $v"; timeout 600 python tools/bench_march.py | grep -v cfg3
  done
done
