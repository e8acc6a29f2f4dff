timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "resample or combined or pdf" 2>&1 | tail -2
timeout 300 python tools/bench_resample.py
