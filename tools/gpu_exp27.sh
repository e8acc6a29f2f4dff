python -c "from paper_2305_04966_b200 import build; build.build(extra=['-DNACC_FILTER_RAYS=512'])"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "filter" 2>&1 | tail -2
bash tools/gpu_ab_filter.sh "-DNACC_FILTER_RAYS=256" "-DNACC_FILTER_RAYS=128" "-DNACC_FILTER_RAYS=512" 2>&1 | grep -v "^\s"
