# compute-sanitizer initcheck (reads of device memory nobody wrote) over the tuned path: parity subset, tiles, a few fuzz seeds.
SEL='pair_cases or golden or edge_cases or guided_match_bit_exact and 1500'
echo "== initcheck parity"
timeout 1500 compute-sanitizer --tool initcheck --print-limit 8 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$SEL" 2>&1 | grep -E "COMPUTE-SANITIZER|passed|failed|SUMMARY|Uninitialized|at |by thread" | head -40
echo "== initcheck fuzz"
CHFUZZ_FIRST=1100 CHFUZZ_COUNT=20 timeout 1500 compute-sanitizer --tool initcheck --print-limit 8 python -m pytest tests/test_fuzz.py -m gpu -x -q -k "random_case_matches" 2>&1 | grep -E "COMPUTE-SANITIZER|passed|failed|SUMMARY|Uninitialized|at |by thread" | head -40
echo "== initcheck tiles"
timeout 1500 compute-sanitizer --tool initcheck --print-limit 8 python -m pytest tests/test_tiled_train.py -m gpu -x -q 2>&1 | grep -E "COMPUTE-SANITIZER|passed|failed|SUMMARY|Uninitialized|at |by thread" | head -40
