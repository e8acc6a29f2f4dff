for rep in 1 2; do
  for v in "-DNACC_MARCH_MINB=7" "-DNACC_MARCH_MINB=6" "-DNACC_MARCH_MINB=8" "-DNACC_MARCH_FLATW=1" "-DNACC_MARCH_MAGICFLOOR=1"; do
    python -c "from paper_2305_04966_b200 import build; build.build(extra='$v'.split())"
    echo "== $v"; timeout 600 python tools/bench_march.py
  done
done
