# compute-sanitizer over the general match path (general_kernels.cuh): sparse index build, union kernel, match from buckets and
# from explicit lists.  Writes to stdout (tee into gpurun_out/).
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  timeout 1700 compute-sanitizer --tool $tool --print-limit 5 python -m pytest tests/test_general_path.py -m gpu -x -q \
      -k "sparse_short_codes and 13 or top_k_beyond_the_lane_list and 33 or host_callback and mixed or candidate_list_errors or guided_with" 2>&1 |
      grep -E "COMPUTE-SANITIZER|passed|failed|SUMMARY|Error|hazard|error" | head -20
done
