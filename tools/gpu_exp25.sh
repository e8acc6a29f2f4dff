python -c "from paper_2305_04966_b200 import build; build.build(extra=['-DNACC_RENDER_TILE=512'])"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "render or weights" 2>&1 | tail -2
bash tools/gpu_ab_render.sh "-DNACC_RENDER_TILE=512" "-DNACC_RENDER_TILE=768" "-DNACC_RENDER_TILE=1024"
