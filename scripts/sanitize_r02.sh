# compute-sanitizer over the round-2 kernels: tensor-core hash filter (tcgen05 / TMEM), match kernel with both shortcuts,
# ranked-list instantiation, failure paths.  Writes to stdout (tee into gpurun_out/).
SEL='filtered_and_exact or dots_at_and_near or queue_overflow or pair_cases or failed_pair_list or replaced_centering or golden or edge_cases or guided_match_bit_exact and 1500'
FILES="tests/test_hash_filter.py tests/test_gpu_parity.py"
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  timeout 1500 compute-sanitizer --tool $tool --print-limit 5 python -m pytest $FILES -m gpu -x -q -k "$SEL" 2>&1 | grep -E "COMPUTE-SANITIZER|passed|failed|SUMMARY|Error|hazard|error" | head -20
done
