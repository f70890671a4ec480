# ncu --set full capture of the match kernel with the per-instruction source page exported as CSV
# (instructions executed per SASS line -> per-phase attribution, scripts/phase_attrib.py).  $1 = tag.
tag=${1:-r02x}
ncu --set full --clock-control none --import-source on -k regex:match_kernel -s 3 -c 1 -f -o gpurun_out/${tag}_match \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --images 200 --pairs 16384 > /dev/null 2>&1
ncu -i gpurun_out/${tag}_match.ncu-rep --page source --csv > gpurun_out/${tag}_match_source.csv 2>/dev/null
python scripts/ncu_summary.py gpurun_out/${tag}_match.ncu-rep gpurun_out/${tag}_match_kernel_ncu_full.json 32735232
