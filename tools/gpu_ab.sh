# A/B of build flags, alternating builds within one call (run-to-run noise on the pool is ~±4 %):
#   bash tools/gpu_ab.sh "-DFLAG=0" "-DFLAG=1" [tools/bench_march.py] [reps]
tool="${3:-tools/bench_march.py}"
for rep in $(seq 1 "${4:-2}"); do
  for v in "$1" "$2"; do
    python -c "from paper_2305_04966_b200 import build; build.build(extra='$v'.split(), debug=False)"
    echo "== $v"; timeout 600 python $tool
  done
done
