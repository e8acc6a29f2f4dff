mkdir -p gpurun_out
python -c "from paper_2305_04966_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "march or sampling or bounds or combined or grid" 2>&1 | tail -2
bash tools/gpu_ab.sh "-DNACC_MARCH_SOLID=0" "-DNACC_MARCH_SOLID=1" | grep -v cfg3
