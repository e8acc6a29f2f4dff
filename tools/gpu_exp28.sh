for rep in 1 2; do
  for v in "-DNACC_MARCH_WARPS=4 -DNACC_MARCH_MINB=7" "-DNACC_MARCH_WARPS=8 -DNACC_MARCH_MINB=4" "-DNACC_MARCH_WARPS=2 -DNACC_MARCH_MINB=14" "-DNACC_MARCH_WARPS=8 -DNACC_MARCH_MINB=3"; do
    python -c "from paper_2305_04966_b200 import build; build.build(extra='$v'.split())"
    echo "== $v"; timeout 600 python tools/bench_march.py
  done
done
