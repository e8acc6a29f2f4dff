timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "march or sampling or bounds or combined or render or weights" 2>&1 | tail -2
for rep in 1 2; do
  for v in "-DNACC_MARCH_MINB=6" "-DNACC_MARCH_MINB=7" "-DNACC_MARCH_MINB=8"; do
    python -c "from paper_2305_04966_b200 import build; build.build(extra='$v'.split())"
    echo "== $v"; timeout 600 python tools/bench_march.py
  done
done
bash tools/gpu_ab_render.sh "-DNACC_RENDER_RAYCACHE=0" "-DNACC_RENDER_RAYCACHE=1"
