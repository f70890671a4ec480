set -x
python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --pairs 40960 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('A stream', d['value'], d['roofline']['avg_launch_ms'])"
CHGPU_NVCC_EXTRA=-DCHGPU_CSA_POPC python -m paper_1805_08995_b200.build --force > /dev/null 2>&1
python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --pairs 40960 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B csa', d['value'], d['roofline']['avg_launch_ms'])"
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
