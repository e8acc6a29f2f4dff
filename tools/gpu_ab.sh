# A/B of a march build flag: alternate builds, march-only timing (tools/bench_march.py)
# usage: bash tools/gpu_ab.sh "-DFLAG=0" "-DFLAG=1"
for rep in 1 2; do
  for v in "$1" "$2"; do
    python -c "from paper_2305_04966_b200 import build; build.build(extra='$v'.split())"
    echo "== $v"; timeout 600 python tools/bench_march.py
  done
done
