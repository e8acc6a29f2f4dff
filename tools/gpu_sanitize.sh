# compute-sanitizer over the march / filter / render / resample / grid parity subset (small cases),
# one run per tool; logs to gpurun_out/sanitizer_<tool>.txt.  torch's caching allocator is turned
# off so every tensor is its own exact-size cudaMalloc (an overread past an array's end is seen).
mkdir -p gpurun_out
SUB='tests/test_gpu_parity.py::test_march_cfg1 tests/test_gpu_parity.py::test_march_edge_cases
 tests/test_gpu_parity.py::test_march_random_grids tests/test_gpu_parity.py::test_filter_ragged
 tests/test_gpu_parity.py::test_filter_exact_on_near_ties tests/test_gpu_parity.py::test_render_ragged
 tests/test_gpu_parity.py::test_render_flat_unaligned tests/test_gpu_parity.py::test_render_degenerate
 tests/test_gpu_parity.py::test_render_cfg1 tests/test_gpu_parity.py::test_weights_and_accumulate
 tests/test_gpu_parity.py::test_weights_alpha tests/test_gpu_parity.py::test_resample_cdf_input_stratified_and_degenerate
 tests/test_gpu_parity.py::test_resample_unbounded_lindisp tests/test_gpu_parity.py::test_resample_far_mass
 tests/test_gpu_parity.py::test_occgrid_points_bit_exact tests/test_gpu_parity.py::test_occgrid_update_bit_exact
 tests/test_gpu_parity.py::test_pdf_loss tests/test_gpu_parity.py::test_dynamic_grid_times_and_max_merge'
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all \
    --print-limit 50 python -m pytest -q -x $SUB > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitizer_summary.txt
  grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitizer_$tool.txt | tail -3 >> gpurun_out/sanitizer_summary.txt
done
