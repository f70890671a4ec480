# A/B of the compaction kernel's shape (threads per CTA x queries per thread)
run() { ncu --metrics gpu__time_duration.sum --clock-control none -k regex:compact_kernel -s 4 -c 4 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --images 200 --pairs 16384 2>&1 | grep gpu__time_duration | awk -v n="$1" '{s+=$3} END {print "RESULT", n, s/NR, "us"}'; }
b() { CHGPU_NVCC_EXTRA="$1" python -m paper_1805_08995_b200.build --force > /dev/null 2>&1; }
for shape in "1024 2" "1024 1" "512 4" "512 2" "256 4" "1024 4"; do set -- $shape; b "-DCHGPU_COMPACT_THREADS=$1 -DCHGPU_COMPACT_PER=$2"; run t$1x$2; done
b ""
