# A/B of several build-flag sets, each rebuilt in turn within one call (pool noise is ~±4 %):
#   bash tools/gpu_variants.sh <tool.py> <reps> "<flags A>" "<flags B>" ...   ("none" = default build)
tool="$1"; reps="$2"; shift 2
for rep in $(seq 1 "$reps"); do
  for v in "$@"; do
    f="$v"; [ "$f" = none ] && f=""
    python -c "from paper_2305_04966_b200 import build; build.build(extra='$f'.split(), debug=False)" || exit 1
    echo "== $v"; timeout 600 python $tool
  done
done
