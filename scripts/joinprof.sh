# per-kernel times of the join path (ncu launch list of a 2-launch bench) + parity subset
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "match or golden or edge or pair_cases or config2" 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/join_launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --images 200 --pairs 7992 > /dev/null 2>&1
python - <<PY
import csv,collections
rows=[r for r in csv.reader(open("gpurun_out/join_launches.csv")) if len(r)>10]
hdr=rows[0]; ki=hdr.index("Kernel Name"); vi=hdr.index("Metric Value")
agg=collections.defaultdict(list)
for r in rows[1:]:
    agg[r[ki][:40]].append(float(r[vi].replace(",","")))
for k,v in agg.items():
    if "join" in k or "match_kernel" in k: print("RESULT", k, len(v), [round(x/1e3,2) for x in v[-2:]])
PY
