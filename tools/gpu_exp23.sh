python -c "from paper_2305_04966_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "filter or render_cfg2 or combined" 2>&1 | tail -2
bash tools/gpu_ab_filter.sh "-DNACC_FILTER_DYN=0" "-DNACC_FILTER_RPL=1" "-DNACC_FILTER_RPL=2" "-DNACC_FILTER_RPL=4" "-DNACC_FILTER_RPL=8" 2>&1 | grep -v "^\s"
