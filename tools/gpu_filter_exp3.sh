mkdir -p gpurun_out
timeout 300 python tools/e2e_diag.py 2>&1 | tail -14
bash tools/gpu_ab_filter.sh "-DNACC_FILTER_BATCH=4" "-DNACC_FILTER_BATCH=8" "-DNACC_FILTER_BATCH=16" "-DNACC_FILTER_BATCH=32" 2>&1 | grep -v "^\s"
