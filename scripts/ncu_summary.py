#!/usr/bin/env python
"""Summarises an ncu report (captured with --set full --import-source on) into profiles/<name>.json:
headline metrics of every profiled kernel plus the top stall locations of the SASS listing.
Usage: python scripts/ncu_summary.py gpurun_out/prof_match_r01c.ncu-rep profiles/r01c_match_kernel_ncu_full.json [queries_per_launch]"""
import csv
import io
import json
import subprocess
import sys

KEEP = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__t_sector_hit_rate.pct",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
]


def page(rep, name):
    return subprocess.run(["ncu", "-i", rep, "--page", name, "--csv"], capture_output=True, text=True).stdout


def main():
    rep, out = sys.argv[1], sys.argv[2]
    queries = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    rows = list(csv.reader(io.StringIO(page(rep, "raw"))))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        k = {"kernel": r[hdr.index("Kernel Name")], "grid": r[hdr.index("Grid Size")], "block": r[hdr.index("Block Size")],
             "metrics": {}}
        for h, u, v in zip(hdr, units, r):
            if h in KEEP:
                k["metrics"][h] = {"unit": u, "value": v}
        if queries:
            k["warp_instructions_per_query"] = float(k["metrics"]["smsp__inst_executed.sum"]["value"]) / queries
        kernels.append(k)
    src = list(csv.reader(io.StringIO(page(rep, "source"))))
    hi = next((i for i, r in enumerate(src) if "Source" in r and "Instructions Executed" in r), None)
    top = []
    if hi is not None:
        h = src[hi]
        ia, isrc, ist = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
        data = []
        for r in src[hi + 1:]:
            try:
                data.append((int(r[ia]), int(r[ist]), r[isrc].strip()))
            except (ValueError, IndexError):
                continue
        tot = sum(s for _, s, _ in data) or 1
        ops = {}
        for n, s, t in data:
            op = t.split()[1] if t.startswith("@") else t.split()[0]
            op = op.split(".")[0]
            ops[op] = ops.get(op, 0) + n
        top = [{"pct_of_stall_samples": round(100.0 * s / tot, 2), "sass": t} for n, s, t in sorted(data, key=lambda x: -x[1])[:20]]
        mix = sorted(ops.items(), key=lambda kv: -kv[1])[:16]
        kernels[0]["sass_opcode_mix_warp_instructions"] = {k: v for k, v in mix}
    doc = {"report": rep, "kernels": kernels, "top_stall_locations": top}
    if queries and len(kernels) > 1:
        # one launch each of the kernels that make up a step of the hot path (join pass + match kernel): the step's totals
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        doc["step"] = {
            "kernels": [k["kernel"].split("(")[0] for k in kernels],
            "warp_instructions_per_query": sum(k["warp_instructions_per_query"] for k in kernels),
            "duration_ms": sum(float(k["metrics"]["gpu__time_duration.sum"]["value"]) for k in kernels),
            "dram_bytes": sum(float(k["metrics"][n]["value"]) * scale[k["metrics"][n]["unit"]] for k in kernels
                              for n in ("dram__bytes_read.sum", "dram__bytes_write.sum")),
        }
    json.dump(doc, open(out, "w"), indent=1)
    print("wrote", out)


if __name__ == "__main__":
    main()
