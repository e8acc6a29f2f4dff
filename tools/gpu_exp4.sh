mkdir -p gpurun_out
python -c "from paper_2305_04966_b200 import build; build.build(extra=['-DNACC_MARCH_SHAREDENDS=1'])"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "march or sampling or bounds or combined or filter" 2>&1 | tail -2
bash tools/gpu_ab.sh "-DNACC_MARCH_SHAREDENDS=0" "-DNACC_MARCH_SHAREDENDS=1" | grep -v cfg3
bash tools/gpu_ab_filter.sh "-DNACC_FILTER_SECTOR=0" "-DNACC_FILTER_SECTOR=1" 2>&1 | grep -v "^\s"
