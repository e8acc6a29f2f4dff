# The round's GPU evidence in one gpurun call: parity tests, smoke, the bench line, the launch
# list (ncu gpu__time_duration, cold-cache and serialised: compare shares) and one
# `ncu --set full` capture per library kernel of the CFG2 step; then tools/make_profiles.py.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 > gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 110 --csv --log-file gpurun_out/launches.csv \
  python bench.py --workload cfg2 --steps 12 --warmup 3 --profile --no-cpu-baseline > /dev/null 2>&1
bash tools/gpu_ncu.sh march_fused march_fused_cfg5 2 --workload cfg5 --steps 1 --warmup 2 --profile --no-cpu-baseline
for k in march_fused render_fwd_warp render_bwd_warp filter_cut filter_copy; do
  bash tools/gpu_ncu.sh $k $k 3
done
ls gpurun_out
