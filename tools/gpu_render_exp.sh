# render exp experiment: A/B of T-product and fp32-alpha builds, then parity under each
mkdir -p gpurun_out
bash tools/gpu_ab_render.sh "-DNACC_RENDER_TPROD=0" "-DNACC_RENDER_TPROD=1" "-DNACC_RENDER_TPROD=1 -DNACC_RENDER_F32A=1"
for v in "-DNACC_RENDER_F32A=1" ""; do
  python -c "from paper_2305_04966_b200 import build; build.build(extra='$v'.split())"
  echo "== parity $v"; timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "render or weights" 2>&1 | tail -4
done
