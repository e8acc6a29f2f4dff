timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "resample" 2>&1 | tail -3
bash tools/gpu_exp20.sh
