# march parity tests + march-only timing (CFG2, CFG3)
timeout 900 python -m pytest tests -m gpu -x -q -k march 2>&1 | tail -1
timeout 600 python tools/bench_march.py
