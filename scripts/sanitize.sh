# compute-sanitizer over the GPU parity suite's small cases:
# memcheck (out-of-bounds / misaligned / leaked device memory), racecheck (shared-memory
# hazards: the TMA-fed walks' stage ring, the fused draw / Gram / K5 kernels),
# synccheck (barrier misuse).  Logs -> gpurun_out/sanitizer_*.log
mkdir -p gpurun_out
SEL="test_gpu_parity.py::test_draws_bit_exact_vs_reference or fused_sampled_gradient or factor_gradients_with_history or objective_vs_reference or adam_matches or stream_fit_vs_reference or dense_draw_solve_vs_oracle"
for tool in memcheck racecheck synccheck; do
  timeout 3000 compute-sanitizer --tool $tool --target-processes all --print-limit 50 \
     python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -q -p no:cacheprovider -x \
     -k "draws_bit_exact_vs_reference or fused_sampled_gradient or factor_gradients_with_history or objective_vs_reference or adam_matches or gauss or (dense_draw_solve and 20) or walk_kernels_gradient" \
     > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitizer_$tool.log
  grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitizer_$tool.log | tail -3
done
