# A/B of the join pass on the GPU box: parity subset, then per-kernel times (ncu launch list of a 2-launch bench) per build switch
t() { ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/jl.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --images 200 --pairs 7992 > /dev/null 2>&1
python - <<PY
import csv,collections
rows=[r for r in csv.reader(open("/tmp/jl.csv")) if len(r)>10]
hdr=rows[0]; ki=hdr.index("Kernel Name"); vi=hdr.index("Metric Value")
agg=collections.defaultdict(list)
for r in rows[1:]:
    agg[r[ki][:30]].append(float(r[vi].replace(",","")))
print("RESULT $1", {k.split("(")[0]: round(v[-1]/1e3,2) for k,v in agg.items() if "join" in k or "match_kernel" in k})
PY
}
b() { CHGPU_NVCC_EXTRA="$1" python -m paper_1805_08995_b200.build --force > /dev/null 2>&1; }
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "match or golden or edge or pair_cases or config2" 2>&1 | tail -2
t default
for v in "$@"; do b "$v"; t "$v"; done
b ""
