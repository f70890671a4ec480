# A/B of match-kernel build variants on the GPU box (kernel-only bench, config-3 shaped, 40,960 pairs)
run() { python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --pairs 40960 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('RESULT $1', round(d['value']), d['roofline']['avg_launch_ms'])"; }
b() { CHGPU_NVCC_EXTRA="$1" python -m paper_1805_08995_b200.build --force > /dev/null 2>&1; }
run base
b "-DCHGPU_SPLIT_PULL"; run split_pull
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "match or golden or edge" 2>&1 | tail -1
b "-DCHGPU_MATCH_THREADS=960"; run t960
b "-DCHGPU_MATCH_THREADS=832"; run t832
b "-DCHGPU_MATCH_THREADS=768"; run t768
b ""; run base_again
