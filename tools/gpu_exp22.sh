timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3
bash tools/gpu_ab.sh "-DNACC_MARCH_FINEMASK=1" "-DNACC_MARCH_FINEMASK=1 -DNACC_MARCH_SEG_CASCADE=16"
