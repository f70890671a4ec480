# A/B of match-kernel build variants on the GPU box (kernel-only bench, config-3 shaped, 40,960 pairs)
run() { python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --pairs 40960 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('RESULT $1', round(d['value']), d['roofline']['avg_launch_ms'])"; }
b() { CHGPU_NVCC_EXTRA="$1" python -m paper_1805_08995_b200.build --force > /dev/null 2>&1; }
run base
b "-DCHGPU_CSA_POPC"; run csa
b "-DCHGPU_VERIFY_LANES=2"; run vl2
b "-DCHGPU_VERIFY_LANES=8"; run vl8
b "-DCHGPU_OVER_SLOTS=2"; run over2
b "-DCHGPU_SERIAL_PULL"; run serial_pull
b ""; run base_again
