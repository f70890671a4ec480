# quick A/B of the match kernel on the GPU box: parity subset + kernel-only bench (config-3 shaped, 40,960 pairs)
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "match or golden or edge or guided" 2>&1 | tail -2
python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --pairs 39960 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('RESULT pairs/s', round(d['value']), 'launch_ms', round(d['roofline']['avg_launch_ms'],3))"
