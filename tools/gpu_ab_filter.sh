# A/B of filter build flags: alternate builds, filter-only timing (tools/bench_filter.py)
for rep in 1 2; do
  for v in "$@"; do
    python -c "from paper_2305_04966_b200 import build; build.build(extra='$v'.split())"
    echo "== $v"; timeout 600 python tools/bench_filter.py
  done
done
