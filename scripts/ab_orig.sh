# A/B of the current build against a side build of an older kernel (libchgpu_orig.so at the repo root)
run() { python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --pairs 39960 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('RESULT $1', round(d['value']), d['roofline']['avg_launch_ms'])"; }
run new
cp paper_1805_08995_b200/libchgpu.so /tmp/new.so; cp libchgpu_orig.so paper_1805_08995_b200/libchgpu.so
run orig
cp /tmp/new.so paper_1805_08995_b200/libchgpu.so
run new_again
