mkdir -p gpurun_out
for k in filter_fused field_sigma; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_$k python bench.py --steps 4 --warmup 3 --profile --no-cpu-baseline > gpurun_out/ncu_$k.log 2>&1
done
