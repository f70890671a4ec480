run() { python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --pairs 40960 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['value'], d['roofline']['avg_launch_ms'])"; }
b() { CHGPU_NVCC_EXTRA="$1" python -m paper_1805_08995_b200.build --force > /dev/null 2>&1; }
run v3c
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
b "-DCHGPU_MATCH_THREADS=896"; run v3c_t896
ncu --set full --clock-control none --import-source on -k regex:match_kernel -s 2 -c 1 -f -o gpurun_out/prof_match_r01g python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --pairs 8192 > gpurun_out/prof_r01g.log 2>&1
b "-DCHGPU_MATCH_THREADS=960"; run v3c_t960
