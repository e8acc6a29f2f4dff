python -c "from paper_2305_04966_b200 import build; build.build(extra=['-DNACC_MARCH_WIN=5','-DNACC_MARCH_SEG=16'])"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "march or sampling or bounds or combined" 2>&1 | tail -2
bash tools/gpu_ab.sh "-DNACC_MARCH_WIN=3 -DNACC_MARCH_SEG=8" "-DNACC_MARCH_WIN=5 -DNACC_MARCH_SEG=16" | grep -v cfg3
