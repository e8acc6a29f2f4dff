# usage: bash tools/gpu_ncu.sh <kernel-regex> <name> [skip]  — one `ncu --set full` capture of a bench kernel
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$1" -s "${3:-3}" -c 1 \
  -o "gpurun_out/prof_$2" -f python bench.py --steps 4 --warmup 3 --profile --no-cpu-baseline > "gpurun_out/ncu_$2.log" 2>&1
tail -2 "gpurun_out/ncu_$2.log"
