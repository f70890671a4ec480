#!/usr/bin/env python
"""bench.py — image pairs matched / second at 8K SIFT-like descriptors per image.

Workload (BASELINE.json configs[2]): exhaustive matching of 1,000 synthetic images x 8,192
descriptors = 499,500 pairs, in the reference's plan order (plan_exhaustive, N_p=50, M=4).  One
STEP = one pass over the whole pair list on one GPU.  With N GPUs every rank owns its own
1,000-image dataset (seed + rank) and runs the same pass — weak scaling, no data-path collective
(SURVEY.md §8e); value = N * pairs / max-over-ranks time.

    value     device-resident: descriptors, codes and bucket indices already in HBM; timed =
              match kernels + ordered compaction into MatchRecords in device memory
              (CUDA events on the library's compute stream, summed over the K steps).
    e2e       the same pass through the C ABI with HOST buffers: every step uploads the
              descriptors from pinned host memory, runs the centering pass, hash build, bucket
              build, matches the pair list and streams all MatchRecords back to the host sink.
    roofline  SURVEY.md §8(d): algorithmic bytes per pair (from the device's own R, Vq, V, Mx
              counters) / match-kernel time, against the measured HBM copy bandwidth.
    cpu_baseline / --impl reference
              the reference's own match_pair (oracle/_ref: its translation units compiled in
              place) on all host cores over a bounded sample of the same pair list.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "image pairs matched/sec @8K SIFT/img"
UNIT = "pairs/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--images", type=int, default=1000)
    ap.add_argument("--points", type=int, default=8192)
    ap.add_argument("--block-images", type=int, default=50)
    ap.add_argument("--blocks-per-group", type=int, default=4)
    ap.add_argument("--pairs", type=int, default=0, help="truncate the pair list (0 = all)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU time of the baseline sample")
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: ONE dataset, the pair list sharded over the ranks (default: weak, one dataset per rank)")
    return ap.parse_args()


def measured_peak_hbm() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:  # noqa: BLE001
            pass
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def recorded_instructions_per_query():
    """Warp instructions per query point of the match kernel, from the committed ncu --set full summary."""
    files = sorted((ROOT / "profiles").glob("r*_match_kernel_ncu_full.json"))
    try:
        return float(json.loads(files[-1].read_text())["kernels"][0]["warp_instructions_per_query"]), files[-1].name
    except Exception:  # noqa: BLE001
        return None, None


def recorded_traffic():
    """dram bytes of one match-kernel launch and the pairs that launch held, from the latest committed ncu --set full
    summary (profiles/r*_match_kernel_ncu_full.json; the capture's launch may be smaller than the bench's)."""
    files = sorted((ROOT / "profiles").glob("r*_match_kernel_ncu_full.json"))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    try:
        k = json.loads(files[-1].read_text())["kernels"][0]
        m = k["metrics"]
        tot = sum(float(m[n]["value"]) * scale[m[n]["unit"]] for n in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        queries = float(m["smsp__inst_executed.sum"]["value"]) / float(k["warp_instructions_per_query"])
        return {"dram_bytes_per_launch": tot, "queries_per_launch": queries, "source": files[-1].name}
    except Exception:  # noqa: BLE001
        return None
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, power, reasons = [], [], [], set()
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
                power.append(float(f[2]))
            except ValueError:
                continue
            for name, val in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), f[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        busy = [s for s, p in zip(sm, power) if p > 0.5 * max(power)] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(smax), "power_w_max": max(power),
                "samples": len(sm), "reasons": sorted(reasons)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    return rank, local, world


def pair_list(args) -> np.ndarray:
    import paper_1805_08995_b200 as ch
    pairs = ch.plan_exhaustive(args.images, args.block_images, args.blocks_per_group)
    if args.pairs:
        pairs = pairs[: args.pairs]
    return np.ascontiguousarray(pairs)


def algorithmic_bytes(stats: dict, m: int, L: int) -> float:
    """24*Nq + 24*Nt + L*(2^m+1)*4 + 4*L*Nt + 20*R + 128*(Vq+V) + 16*Mx, summed over pairs."""
    return (24.0 * stats["query_points"] + 24.0 * stats["train_points"] + stats["pairs"] * L * ((1 << m) + 1) * 4.0 +
            4.0 * L * stats["train_points"] + 20.0 * stats["raw_candidates"] +
            128.0 * (stats["verified_queries"] + stats["distances"]) + 16.0 * stats["matches"])


# ---------------------------------------------------------------------------------------------------
def cpu_sample(args, pairs: np.ndarray, desc: np.ndarray, codes_from=None, threads: int | None = None,
               target_seconds: float | None = None):
    """Times the reference's match_pair on `threads` host threads over the first P pairs of the plan.
    codes_from: callable image -> (shorts, longs), or None to compute them with the CPU oracle."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib
    import paper_1805_08995_b200 as ch

    orc = oracle_lib.best()
    kind = "reference" if orc.name == "reference" else "port"
    threads = threads or (os.cpu_count() or 1)
    target = target_seconds if target_seconds is not None else args.cpu_seconds
    per_pair = 0.085 * (args.points / 8192.0) ** 2  # seconds per pair per core, SURVEY.md §6
    sample = int(max(threads, min(len(pairs), target * threads / per_pair)))
    sub = pairs[:sample]
    used = np.unique(sub)
    params = ch.FamilyParams()
    fam = ch.build_hash_family(params)
    remap = {int(g): k for k, g in enumerate(used)}
    descs = [desc[int(g)] for g in used]
    if codes_from is not None:
        got = [codes_from(int(g)) for g in used]
    else:
        cen = orc.centering([desc[i] for i in range(len(desc))])
        got = [None] * len(used)

        def work(w):
            for k in range(w, len(used), threads):
                got[k] = orc.compute_codes(params, fam.short_planes, fam.long_planes, cen, descs[k])

        ts = [threading.Thread(target=work, args=(w,)) for w in range(threads)]
        [t.start() for t in ts]
        [t.join() for t in ts]
    local_pairs = np.array([[remap[int(a)], remap[int(b)]] for a, b in sub], dtype=np.uint32)
    shorts = [g[0] for g in got]
    longs = [g[1] for g in got]
    cfg = ch.MatchConfig()

    def run():
        return orc.time_match_pairs(params, cfg, descs, shorts, longs, local_pairs, threads)

    return run, {"kind": kind, "cores": threads, "sample_pairs": sample,
                 "sample": f"first {sample} pairs of the plan ({len(used)} images) x {args.points} desc, "
                           f"{orc.name} match_pair on {threads} threads"}


def run_reference_arm(args):
    rank, local, world = dist_env()
    if rank != 0:
        return
    import paper_1805_08995_b200 as ch

    pairs = pair_list(args)
    threads = os.cpu_count() or 1
    # bounded sample per step: ~6 s of all-core CPU work
    per_pair = 0.085 * (args.points / 8192.0) ** 2
    sample = int(max(threads, min(len(pairs), 6.0 * threads / per_pair)))
    need_images = int(np.unique(pairs[:sample]).max()) + 1
    desc = ch.make_dataset(need_images, args.points, seed=args.seed)
    run, info = cpu_sample(args, pairs, desc, codes_from=None, threads=threads, target_seconds=6.0)
    for _ in range(args.warmup):
        run()
    t0 = time.perf_counter()
    total = 0.0
    for _ in range(args.steps):
        sec, _ = run()
        total += sec
    wall = time.perf_counter() - t0
    value = info["sample_pairs"] * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8/u64 popcount + exact integer distances (fp64 ratio test)", "data": "synthetic",
        "config": workload_config(args, len(pairs)),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": info["cores"], "kind": info["kind"], "sample": info["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0, "wall_s": wall,
    }
    print(json.dumps(line), flush=True)


def workload_config(args, npairs: int) -> dict:
    return {
        "workload": f"BASELINE configs[2]: exhaustive matching of {args.images} images x {args.points} descriptors "
                    f"({npairs} pairs per step per GPU, reference plan order N_p={args.block_images} M={args.blocks_per_group})",
        "images": args.images, "points_per_image": args.points, "pairs_per_step_per_gpu": npairs,
        "family": "m=8 L=6 n=128 seed=1", "match": "k=10 tau=40 ratio=0.8 min_cand=2 N_r=3",
        "synthetic": "uniform u8 descriptors, 30% sigma=8 twins of a shared pool (SURVEY 8d), seed 7 + rank",
        "l2": "resident working set (1.47 MB/image) is larger than the 126 MB L2; no flush needed",
        "parallelism": "pair-list sharding, one process per GPU, no collective",
    }


def run_ours(args):
    rank, local, world = dist_env()
    import torch
    import paper_1805_08995_b200 as ch

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    pairs = pair_list(args)
    if args.strong and world > 1:
        # one job, sharded: contiguous range of the plan per rank (chgpu_shard_range); every rank keeps the
        # whole 1.5 GB dataset resident, so centering needs no exchange here (sharding.py has the general form)
        a, b = ch.shard_range(len(pairs), rank, world)
        pairs = np.ascontiguousarray(pairs[a:b])
    npairs = len(pairs)
    m = ch.Matcher(local)
    params = ch.FamilyParams()
    fam = ch.build_hash_family(params)
    m.set_family(fam)
    cfg = ch.MatchConfig()

    # host dataset in pinned memory (what a loader thread would fill from CHFT files)
    desc = m.pinned_empty((args.images, args.points, 128), np.uint8)
    ch.make_dataset(args.images, args.points, seed=args.seed + (0 if args.strong else rank), out=desc)
    ids = np.arange(args.images, dtype=np.uint32)

    def load_and_hash():
        m.upload_many(ids, desc)
        m.centering_reset()
        m.centering_add_many(ids)
        m.centering_apply()
        m.hash(ids)

    t0 = time.perf_counter()
    load_and_hash()
    m.sync()
    setup_s = time.perf_counter() - t0

    # ---- value: device-resident matching pass ------------------------------------------------------
    for _ in range(args.warmup):
        m.match_pairs_device(pairs, cfg)
    sampler = ClockSampler(local)
    barrier()
    sampler.start()
    t0 = time.perf_counter()
    dev_ms = 0.0
    kern_ms = 0.0
    launches = 0
    match_launches = 0
    last = None
    for _ in range(args.steps):
        last = m.match_pairs_device(pairs, cfg)
        dev_ms += last["total_ms"]
        kern_ms += last["match_kernel_ms"]
        launches += last["total_launches"]
        match_launches += last["match_launches"]
    barrier()
    wall_s = time.perf_counter() - t0
    clocks = sampler.stop()
    dev_ms = max_over_ranks(dev_ms)
    wall_s = max_over_ranks(wall_s)
    ms_per_step = dev_ms / args.steps
    total_pairs = sum_over_ranks(float(npairs))  # weak: world x list; strong: the one list
    value = total_pairs / (ms_per_step * 1e-3)

    # ---- roofline of the match kernel --------------------------------------------------------------
    peak, peak_src = measured_peak_hbm()
    alg = algorithmic_bytes(last, params.short_bits, params.table_count)
    kern_ms_per_step = kern_ms / args.steps
    achieved = alg / (kern_ms_per_step * 1e-3) / 1e9
    traffic = recorded_traffic()
    roofline = {
        "bound": "hbm", "kernel": "match_kernel<SMEM_TRAIN, L=6>", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak, "peak_source": peak_src,
        # dram bytes of one launch of this run's size: the captured launch scaled by its query count
        "traffic": (traffic["dram_bytes_per_launch"] * (last["query_points"] / max(1, last["match_launches"])) /
                    traffic["queries_per_launch"]) if traffic else None,
        "traffic_source": (traffic or {}).get("source"),
        "algorithmic_bytes_per_pair": alg / npairs,
        "algorithmic_bytes_per_launch": alg / max(1, last["match_launches"]),
        "avg_launch_ms": kern_ms / max(1, match_launches),
        "kernel_share_of_step": kern_ms / dev_ms if dev_ms else None,
        "note": "candidate gathers (20 B x R, 88% of the algorithmic bytes) are served from shared memory, "
                "so frac may exceed 1; see DESIGN.md for the on-chip (POPC / LDS) bounds",
    }

    # on-chip bound of the same kernel: POPC is the one quarter-rate instruction the scan cannot avoid
    # (4 per raw candidate, 16 lanes/clk/SM on the XU pipe); DESIGN.md section 4
    props = m.device_props()
    sm_mhz = clocks.get("sm_mhz") or 1965.0
    # measured peaks of this pool's B200 (scripts/onchip_probe.cu -> profiles/onchip_peaks.json): POPC 15.9 /clk/SM,
    # integer ALU pipe 2 warp instructions /clk/SM (half rate), LDS.128 1.9 wavefronts /clk/SM
    probe = None
    try:
        probe = json.loads((ROOT / "profiles" / "onchip_peaks.json").read_text())
    except (OSError, ValueError):
        pass
    popc_per_clk = probe["popc_per_clk_per_sm_at_max_clock"] if probe else 16.0
    popc_peak = props["sm_count"] * popc_per_clk * sm_mhz * 1e6
    popc_rate = 4.0 * last["raw_candidates"] / (kern_ms_per_step * 1e-3)
    roofline["on_chip"] = {"bound": "xu_popc", "achieved_gpopc_s": popc_rate / 1e9, "peak_gpopc_s": popc_peak / 1e9,
                           "frac": popc_rate / popc_peak,
                           "peak_source": "measured (profiles/onchip_peaks.json)" if probe else "16 lanes/clk/SM (assumed)",
                           "measured_peaks": probe,
                           "note": "lower bound on POPC work (padding lanes not counted); ncu pipe utilisations of the "
                                   "committed capture (profiles/r*_match_kernel_ncu_full.json, latest)"}

    # the limit the kernel actually runs into: warp-instruction issue slots (4 per clock per SM).  Instructions
    # per query come from the committed ncu capture of this kernel; the rate is this run's.
    ipq, ipq_src = recorded_instructions_per_query()
    if ipq:
        issue_peak = props["sm_count"] * 4 * sm_mhz * 1e6
        issue_rate = ipq * last["query_points"] / (kern_ms_per_step * 1e-3)
        roofline["on_chip"]["issue"] = {
            "bound": "issue_slots", "warp_instructions_per_query": ipq, "achieved_ginst_s": issue_rate / 1e9,
            "peak_ginst_s": issue_peak / 1e9, "frac": issue_rate / issue_peak,
            "note": "ncu of the same kernel: issue active 70 %, LSU data pipe 75 %, ALU 61 %, XU 50 % "
                    f"(profiles/{ipq_src})"}

    # ---- e2e: host buffers in, host records out, every step ------------------------------------------
    e2e = None
    if not args.no_e2e:
        got = {"records": 0, "chunks": 0}

        def sink(first, offs, rec):
            got["records"] += len(rec)
            got["chunks"] += 1

        def e2e_step():
            load_and_hash()
            st = m.match_pairs_stream(pairs, cfg, sink)
            return st

        e2e_step()  # warm-up (pinned result buffers grow here)
        barrier()
        t0 = time.perf_counter()
        e2e_launches = 0
        for _ in range(args.e2e_steps):
            got["records"] = 0
            st = e2e_step()
            e2e_launches += st["total_launches"]
        barrier()
        e2e_s = max_over_ranks(time.perf_counter() - t0) / args.e2e_steps
        assert got["records"] == st["matches"]
        e2e = {
            "value": total_pairs / e2e_s, "unit": UNIT,
            "h2d_bytes_per_step": int(desc.nbytes + npairs * 16),
            "d2h_bytes_per_step": int(st["matches"] * 16 + (npairs + st["match_launches"]) * 8),
            "steps": args.e2e_steps, "ms_per_step": 1e3 * e2e_s,
            "includes": "H2D descriptors from pinned host, centering sums, hash + bucket build, match, D2H of all MatchRecords to the sink",
        }

    # ---- CPU baseline (rank 0, N=1 only) ----------------------------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        def gpu_codes(i):
            c = m.codes(i)
            return c.shorts, c.longs
        run, info = cpu_sample(args, pairs, desc, codes_from=gpu_codes)
        sec, cpu_matches = run()
        cpu = {"value": info["sample_pairs"] / sec, "unit": UNIT, "cores": info["cores"], "kind": info["kind"],
               "sample": info["sample"], "seconds": sec}
        # the sample doubles as a parity check: same number of matches on the same pairs
        st = m.match_pairs_device(pairs[: info["sample_pairs"]], cfg)
        cpu["gpu_matches_on_sample"] = st["matches"]
        cpu["cpu_matches_on_sample"] = cpu_matches
        assert st["matches"] == cpu_matches, "GPU and CPU reference disagree on the sample"

    total_matches = sum_over_ranks(float(last["matches"]))
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
            "dtype": "u8/u32 popcount + exact integer distances (fp64 ratio test; hashing: fp32 filter + exact fp64 re-evaluation)",
            "data": "synthetic", "config": workload_config(args, npairs), "roofline": roofline, "cpu_baseline": cpu,
            "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
            "wall_ms_per_step": 1e3 * wall_s / args.steps, "setup_s": setup_s,
            "matches_per_step": total_matches, "device": m.device_props()["name"],
        }
        print(json.dumps(line), flush=True)
    m.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
