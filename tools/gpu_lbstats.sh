python -c "from paper_2305_04966_b200 import build; build.build(extra=['-DNACC_LB_STATS=1'])"
timeout 300 python tools/lb_stats.py
