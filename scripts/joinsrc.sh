# ncu --set full capture of the join pass with the source pages (SASS and CUDA lines) exported as CSV.  $1 = tag.
tag=${1:-r02x}
ncu --set full --clock-control none --import-source on -k regex:join_hits_kernel -s 1 -c 1 -f -o gpurun_out/${tag}_join \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --images 200 --pairs 7992 > /dev/null 2>&1
ncu -i gpurun_out/${tag}_join.ncu-rep --page source --print-source sass --csv > gpurun_out/${tag}_join_sass.csv 2>/dev/null
ncu -i gpurun_out/${tag}_join.ncu-rep --page source --print-source cuda --csv > gpurun_out/${tag}_join_cuda.csv 2>/dev/null
ncu -i gpurun_out/${tag}_join.ncu-rep --page raw --csv > gpurun_out/${tag}_join_raw.csv 2>/dev/null
