# compute-sanitizer over the new kernels: filtered hash + fixup, tiled match (min / top-k / merge), guided match,
# loader (fused split + sums).  Writes gpurun_out/sanitizer.log
SEL='filtered_and_exact or dots_at_and_near or tiled_match_bit_exact and 3000 or mixed_pair_list or guided_match_bit_exact and 1500 or chft_load or batched_centering'
FILES="tests/test_hash_filter.py tests/test_tiled_train.py tests/test_gpu_parity.py tests/test_loader.py"
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 5 python -m pytest $FILES -m gpu -x -q -k "$SEL" 2>&1 | grep -E "COMPUTE-SANITIZER|passed|failed|SUMMARY|Error|hazard" | head -20
done
# round r01n: residency replay, background loads (deferred splits on the load stream), batch eviction
echo "== memcheck (residency / background loads)"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_residency.py tests/test_loader.py -m gpu -x -q 2>&1 | grep -E "COMPUTE-SANITIZER|passed|failed|SUMMARY|Error" | head -20
