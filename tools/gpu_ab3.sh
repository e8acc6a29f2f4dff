# A/B/C... of march build flags (each build once per rep), march-only timing
for rep in 1 2; do
  for v in "$@"; do
    python -c "from paper_2305_04966_b200 import build; build.build(extra='$v'.split())"
    echo "== $v"; timeout 600 python tools/bench_march.py 2>/dev/null | head -1
  done
done
