mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; tail -3 gpurun_out/bench_full.err; cat gpurun_out/bench_full.json
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -3 gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 50 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/bench_trun.json 2> gpurun_out/bench_trun.err; tail -3 gpurun_out/bench_trun.err; cat gpurun_out/bench_trun.json | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 120 --csv --log-file gpurun_out/launches.csv python bench.py --steps 12 --warmup 3 --profile --no-cpu-baseline > /dev/null 2>&1
for k in march_fused render_fwd_warp render_bwd_warp filter_cut filter_copy tex_sigma4 field_samples; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_$k -f python bench.py --steps 4 --warmup 3 --profile --no-cpu-baseline > gpurun_out/ncu_$k.log 2>&1
done
ls gpurun_out
