python -c "from paper_2305_04966_b200 import build; build.build(extra=['-DNACC_MARCH_RPT=12','-DNACC_MARCH_KCAP=1536'])"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "march or sampling" 2>&1 | tail -2
for rep in 1 2; do
  for v in "-DNACC_MARCH_RPT=8 -DNACC_MARCH_KCAP=1024" "-DNACC_MARCH_RPT=12 -DNACC_MARCH_KCAP=1536" "-DNACC_MARCH_RPT=16 -DNACC_MARCH_KCAP=2048" "-DNACC_MARCH_RPT=16 -DNACC_MARCH_KCAP=1536"; do
    python -c "from paper_2305_04966_b200 import build; build.build(extra='$v'.split())"
    echo "== $v"; timeout 600 python tools/bench_march.py
  done
done
