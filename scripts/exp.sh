run() { python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --pairs 40960 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['roofline']['avg_launch_ms'])"; }
b() { CHGPU_NVCC_EXTRA="$1" python -m paper_1805_08995_b200.build --force > /dev/null 2>&1; }
run vl2
b "-DCHGPU_VERIFY_LANES=4"; run vl4
python -m pytest tests -m gpu -x -q -k "parity" 2>&1 | tail -2
b "-DCHGPU_VERIFY_LANES=8"; run vl8
python -m pytest tests -m gpu -x -q -k "parity" 2>&1 | tail -2
b "-DCHGPU_VERIFY_LANES=8 -DCHGPU_MATCH_THREADS=1024"; run vl8_t1024
