bash tools/gpu_ab_render.sh "-DNACC_RENDER_BPS=4" "-DNACC_RENDER_BPS=3" "-DNACC_RENDER_BPS=5"
