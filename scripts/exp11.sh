# Build switches re-measured with the join pass in front of the match kernel (39,960 pairs = 10 full launches, kernel-only):
# pairs/s and the step's average time per launch (join + lists + match kernel).
run() { python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --pairs 39960 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('RESULT $1', round(d['value']), d['roofline']['avg_launch_ms'])"; }
b() { CHGPU_NVCC_EXTRA="$1" python -m paper_1805_08995_b200.build --force > /dev/null 2>&1; }
run base
for v in "$@"; do b "$v"; run "$v"; done
b ""; run base_again
