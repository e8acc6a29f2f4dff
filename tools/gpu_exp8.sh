python -c "from paper_2305_04966_b200 import build; build.build(extra=['-DNACC_LB_STATS=1'])"
timeout 300 python tools/lb_stats.py
python -c "from paper_2305_04966_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "march or sampling or bounds or combined" 2>&1 | tail -2
bash tools/gpu_ab.sh "-DNACC_LB_HELP=0" "-DNACC_LB_HELP=1"
