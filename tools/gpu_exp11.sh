python -c "from paper_2305_04966_b200 import build; build.build(extra=['-DNACC_RENDER_BPS=2'])"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "render" 2>&1 | tail -2
bash tools/gpu_ab_render.sh "-DNACC_RENDER_BPS=2" "-DNACC_RENDER_BPS=3" "-DNACC_RENDER_BPS=4"
