for rep in 1 2; do
  for v in "-DNACC_LB_NS0=256 -DNACC_LB_NSMAX=4096" "-DNACC_LB_NS0=64 -DNACC_LB_NSMAX=1024" "-DNACC_LB_NS0=128 -DNACC_LB_NSMAX=2048" "-DNACC_LB_NS0=512 -DNACC_LB_NSMAX=8192"; do
    python -c "from paper_2305_04966_b200 import build; build.build(extra='$v'.split())"
    echo "== $v"; timeout 600 python tools/bench_march.py
  done
done
