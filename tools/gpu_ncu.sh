# usage: bash tools/gpu_ncu.sh <kernel-regex> <name> [skip] [bench args...] — one `ncu --set full` capture of a
# bench kernel (default: the CFG2 workload in profile mode)
mkdir -p gpurun_out
k="$1"; n="$2"; s="${3:-3}"; shift 3 2>/dev/null
args="${*:---workload cfg2 --steps 4 --warmup 3 --profile --no-cpu-baseline}"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" -s "$s" -c 1 \
  -o "gpurun_out/prof_$n" -f python bench.py $args > "gpurun_out/ncu_$n.log" 2>&1
tail -2 "gpurun_out/ncu_$n.log"
