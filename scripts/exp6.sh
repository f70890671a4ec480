run() { python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --pairs 39960 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('RESULT $1', round(d['value']), d['roofline']['avg_launch_ms'])"; }
b() { CHGPU_NVCC_EXTRA="$1" python -m paper_1805_08995_b200.build --force > /dev/null 2>&1; }
run base
b "-DCHGPU_VERIFY_TILES=1"; run tiles1
b "-DCHGPU_VERIFY_SIMT"; run verify_simt
b "-DCHGPU_VERIFY_SIMT -DCHGPU_VERIFY_LANES=2"; run verify_simt_vl2
b ""; run base_again
