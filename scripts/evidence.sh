# Evidence pass on the GPU box: ncu --set full of the match kernel and of the filtered hash kernel (summarised into
# profiles/ so that bench.py's issue-slot roofline uses this build's instruction count), bench (both arms), ncu launch
# list of the same command.  Everything lands in gpurun_out/ under the tag given as $1.
tag=${1:-r01x}
# one launch of the join pass and one of the match kernel (the two kernels of a sub-batch), third sub-batch of the run
ncu --set full --clock-control none --import-source on -k regex:"match_kernel|join_hits_kernel" -s 6 -c 2 -f -o gpurun_out/${tag}_match \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --images 200 --pairs 16384 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/${tag}_match.ncu-rep profiles/${tag}_match_kernel_ncu_full.json 32735232  # 3,996 pairs (27 x 148 SMs) x 8,192 queries per launch
cp profiles/${tag}_match_kernel_ncu_full.json gpurun_out/
# per-phase attribution of the match kernel's executed instructions (source page of the same capture x the cubin's line table;
# per query of the PAIR, although the kernel visits the hit queries only)
ncu -i gpurun_out/${tag}_match.ncu-rep --page source --csv -k regex:match_kernel > gpurun_out/${tag}_match_source.csv 2>/dev/null
python scripts/phase_attrib.py gpurun_out/${tag}_match_source.csv paper_1805_08995_b200/libchgpu.so \
    _ZN5chgpu12match_kernelILb1ELi6ELb1ELb0ELi3ELb0EEEvNS_11MatchParamsE 32735232 gpurun_out/${tag}_match_kernel_phase_attribution.json > /dev/null
ncu --set full --clock-control none --import-source on -k regex:hash_filter_tc_kernel -s 1 -c 1 -f -o gpurun_out/${tag}_hash \
    python scripts/hash_bench.py --images 400 --reps 1 > /dev/null 2>&1
python scripts/ncu_summary.py gpurun_out/${tag}_hash.ncu-rep gpurun_out/${tag}_hash_filter_kernel_ncu_full.json
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
python bench.py --impl reference > gpurun_out/${tag}_bench_reference_arm.json 2>> gpurun_out/${tag}_bench.err
# the whole command, every launch (setup, warm-up step, timed step, one end-to-end step)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/${tag}_bench_under_ncu.log 2>&1
python scripts/hash_bench.py > gpurun_out/${tag}_hash_bench.json
tail -c 600 gpurun_out/${tag}_bench.json
