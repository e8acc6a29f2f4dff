bash tools/gpu_ab_render.sh "-DNACC_RENDER_F32A=0" "-DNACC_RENDER_F32A=1"
