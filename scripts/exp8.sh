run() { python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --pairs 39960 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('RESULT $1', round(d['value']), d['roofline']['avg_launch_ms'])"; }
b() { CHGPU_NVCC_EXTRA="$1" python -m paper_1805_08995_b200.build --force > /dev/null 2>&1; }
run base
b "-DCHGPU_MATCH_THREADS=1024"; run t1024
b "-DCHGPU_MATCH_THREADS=960"; run t960
b "-DCHGPU_NO_RERANK_SHORTCUT"; run no_rerank_shortcut
b "-DCHGPU_NO_VERIFY_SHORTCUT -DCHGPU_NO_RERANK_SHORTCUT"; run no_shortcuts
b "-DCHGPU_CSA_POPC"; run csa_popc
b ""; run base_again
