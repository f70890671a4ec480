run() { python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --pairs 40960 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['roofline']['avg_launch_ms'])"; }
b() { CHGPU_NVCC_EXTRA="$1" python -m paper_1805_08995_b200.build --force > /dev/null 2>&1; }
b ""; run s2_t1024
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
b "-DCHGPU_OVER_SLOTS=3"; run s3_t1024
b "-DCHGPU_OVER_SLOTS=3 -DCHGPU_MATCH_THREADS=896"; run s3_t896
b "-DCHGPU_OVER_SLOTS=2 -DCHGPU_MATCH_THREADS=896"; run s2_t896
b "-DCHGPU_OVER_SLOTS=3 -DCHGPU_MATCH_THREADS=768"; run s3_t768
b "-DCHGPU_OVER_SLOTS=2 -DCHGPU_CSA_POPC"; run s2_t1024_csa
