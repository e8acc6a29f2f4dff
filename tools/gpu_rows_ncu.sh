# one `ncu --set full` capture per secondary §8 row kernel (tools/prof_rows.py, tools/prof_march.py)
mkdir -p gpurun_out
cap() {  # cap <name> <kernel regex> <skip> <cmd...>
  n="$1"; k="$2"; s="$3"; shift 3
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s "$s" -c 1 \
    -o "gpurun_out/prof_$n" -f "$@" > "gpurun_out/ncu_$n.log" 2>&1
}
cap march_cfg3 march_fused 2 python tools/prof_march.py cfg3
cap importance_256_96 importance 2 python tools/prof_rows.py cfg4
cap render_fwd_cfg4 render_fwd_warp 1 python tools/prof_rows.py cfg4
cap render_bwd_cfg4 render_bwd_warp 1 python tools/prof_rows.py cfg4
cap occgrid_update update_kernel 1 python tools/prof_rows.py grid
cap occgrid_points points_kernel 1 python tools/prof_rows.py grid
cap occgrid_mask3 mask3 1 python tools/prof_rows.py grid
cap alpha_fwd weights_alpha_fwd 2 python tools/prof_rows.py alpha
cap alpha_bwd weights_alpha_bwd 1 python tools/prof_rows.py alpha
cap pdf_loss pdf_loss_kernel 1 python tools/prof_rows.py pdf
cap pdf_loss_bwd pdf_loss_bwd 1 python tools/prof_rows.py pdf
cap march_bounds march_fused 1 python tools/prof_rows.py bounds  # single level: the fused kernel in bounds mode
cap weights_fwd weights_fwd 1 python tools/prof_rows.py accum
cap accumulate accumulate_warp 1 python tools/prof_rows.py accum
ls gpurun_out | grep prof_
