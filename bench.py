#!/usr/bin/env python
"""bench.py — image pairs matched / second at 8K SIFT-like descriptors per image.

Workload (BASELINE.json configs[2]): exhaustive matching of 1,000 synthetic images x 8,192
descriptors = 499,500 pairs, in the reference's plan order (plan_exhaustive, N_p=50, M=4).  One
STEP = one pass over the whole pair list.  With N GPUs (`--gpus N`: bench.py launches the N ranks
itself, one process per GPU, or runs as one rank of a torchrun launch of the same size) the ONE pair
list is cut into N contiguous, work-balanced shards (chgpu_shard_pairs_weighted) — strong scaling, no
data-path collective: every rank uploads and hashes only the images its shard touches,
the dataset centering is exchanged as 128 u64 sums + a count, value = pairs / max-over-ranks time.
`--weak` gives every rank its own 1,000-image dataset instead (N independent jobs).

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


def parse_args(argv=None):
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
    ap.add_argument("--strong", action="store_true", help="(default for --gpus > 1) ONE dataset, the pair list sharded over the ranks")
    ap.add_argument("--weak", action="store_true", help="weak scaling: one private dataset per rank (N independent jobs)")
    return ap.parse_args(argv)


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
        doc = json.loads(files[-1].read_text())
        if "step" in doc:  # join pass + match kernel captured together: the step's total
            return float(doc["step"]["warp_instructions_per_query"]), files[-1].name
        return float(doc["kernels"][0]["warp_instructions_per_query"]), files[-1].name
    except Exception:  # noqa: BLE001
        return None, None


def recorded_traffic():
    """dram bytes of one match-kernel launch and the pairs that launch held, from the latest committed ncu --set full
    summary (profiles/r*_match_kernel_ncu_full.json; the capture's launch may be smaller than the bench's)."""
    files = sorted((ROOT / "profiles").glob("r*_match_kernel_ncu_full.json"))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    try:
        doc = json.loads(files[-1].read_text())
        k = doc["kernels"][0]
        m = k["metrics"]
        queries = float(m["smsp__inst_executed.sum"]["value"]) / float(k["warp_instructions_per_query"])
        if "step" in doc:
            return {"dram_bytes_per_launch": float(doc["step"]["dram_bytes"]), "queries_per_launch": queries, "source": files[-1].name}
        tot = sum(float(m[n]["value"]) * scale[m[n]["unit"]] for n in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
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
        sec, _, _ = run()
        total += sec
    wall = time.perf_counter() - t0
    value = info["sample_pairs"] * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u8/u64 popcount + exact integer distances (fp64 ratio test)", "data": "synthetic",
        "config": workload_config(args, len(pairs)),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": info["cores"], "kind": info["kind"], "sample": info["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0, "wall_s": wall,
    }
    print(json.dumps(line), flush=True)


def workload_config(args, npairs: int, world: int = 1, strong: bool = True) -> dict:
    per = (f"{npairs} pairs per step, ONE list sharded over {world} GPUs" if strong and world > 1
           else f"{npairs} pairs per step per GPU")
    return {
        "workload": f"BASELINE configs[2]: exhaustive matching of {args.images} images x {args.points} descriptors "
                    f"({per}, reference plan order N_p={args.block_images} M={args.blocks_per_group})",
        "images": args.images, "points_per_image": args.points,
        "pairs_per_step": npairs if strong else npairs * world, "pairs_per_step_per_gpu": npairs if not strong else None,
        "family": "m=8 L=6 n=128 seed=1", "match": "k=10 tau=40 ratio=0.8 min_cand=2 N_r=3",
        "synthetic": "uniform u8 descriptors, 30% sigma=8 twins of a shared pool (SURVEY 8d), seed 7" + ("" if strong else " + rank"),
        "l2": "resident working set (1.47 MB/image) is larger than the 126 MB L2; no flush needed",
        "parallelism": ("one process per GPU; the pair list in contiguous work-balanced shards (chgpu_shard_pairs_weighted); "
                        "no data-path collective; 1 KB centering exchange + timing reductions only"),
    }


# Test hook (tests/bench_worker.py): an engine with ch.Matcher's method names and the torch.distributed backend to
# use with it.  The product path leaves both alone: ch.Matcher on cuda:LOCAL_RANK, NCCL.
ENGINE_FACTORY = None
DIST_BACKEND = "nccl"


def runs_of(ids) -> list[tuple[int, int]]:
    """Sorted unique ids as [start, stop) runs of consecutive values (contiguous slices of the pinned dataset)."""
    ids = np.unique(np.asarray(ids, dtype=np.int64))
    if len(ids) == 0:
        return []
    cut = np.flatnonzero(np.diff(ids) != 1) + 1
    starts = np.concatenate([[0], cut])
    stops = np.concatenate([cut, [len(ids)]])
    return [(int(ids[a]), int(ids[b - 1]) + 1) for a, b in zip(starts, stops)]


def run_ours(args):
    rank, local, world = dist_env()
    import torch
    import paper_1805_08995_b200 as ch
    from paper_1805_08995_b200.sharding import Comm

    gpu = ENGINE_FACTORY is None
    # CHGPU_BENCH_SHARE_GPU=1: a FUNCTIONAL check of the N-rank path on a box with fewer GPUs — the ranks share the
    # visible devices (rank r -> cuda:(r mod count)) and talk over gloo (NCCL refuses two ranks on one device).  The line
    # says so ("functional_check_only"); it is never a scaling number.
    share = gpu and world > 1 and os.environ.get("CHGPU_BENCH_SHARE_GPU") == "1"
    backend = "gloo" if share else DIST_BACKEND
    if gpu:
        if not torch.cuda.is_available():
            raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
        if share:
            local = local % torch.cuda.device_count()
        if local >= torch.cuda.device_count():
            raise SystemExit(f"bench.py: rank {rank} wants cuda:{local} but only {torch.cuda.device_count()} device(s) are visible")
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local) if (gpu and not share) else torch.device("cpu")
    if world > 1:
        import torch.distributed as dist
        if gpu and not share:
            dist.init_process_group(backend, device_id=dev)
        else:
            dist.init_process_group(backend)
    comm = Comm(rank, world)  # host-side exchange (gloo group): centering sums, per-rank report
    strong = world > 1 and not args.weak

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        if gpu:
            torch.cuda.synchronize()

    def reduce_ranks(x: float, op: str) -> float:
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return float(t.item())

    all_pairs = pair_list(args)
    shard_weights = None
    if strong:
        # ONE job: contiguous ranges of the plan balanced by work (queries x train points), so a rank keeps the
        # plan's block locality (assign_workers' round robin, scheduler.cpp:166-173, would hand every rank every block)
        first, shard_weights = ch.shard_pairs_weighted(all_pairs, np.full(args.images, args.points, np.uint32), world)
        pairs = np.ascontiguousarray(all_pairs[int(first[rank]):int(first[rank + 1])])
    else:
        pairs = all_pairs
    npairs = len(pairs)
    m = ch.Matcher(local) if gpu else ENGINE_FACTORY(local)
    params = ch.FamilyParams()
    fam = ch.build_hash_family(params)
    m.set_family(fam)
    cfg = ch.MatchConfig()

    # host dataset in pinned memory (what a loader thread would fill from CHFT files)
    desc = m.pinned_empty((args.images, args.points, 128), np.uint8)
    ch.make_dataset(args.images, args.points, seed=args.seed + (rank if (world > 1 and not strong) else 0), out=desc)
    needed = np.unique(pairs).astype(np.uint32) if strong else np.arange(args.images, dtype=np.uint32)
    # centering is a property of the whole dataset (hashing.cpp:52-70): strong-mode ranks sum a contiguous share of
    # the images each and exchange 128 u64 sums + a count; weak-mode ranks own their whole dataset
    own_a, own_b = ch.shard_range(args.images, rank, world) if strong else (0, args.images)
    owned = np.arange(own_a, own_b, dtype=np.uint32)
    resident = np.union1d(needed, owned).astype(np.uint32)
    only_centering = np.setdiff1d(owned, needed).astype(np.uint32)
    h2d_bytes = int(len(resident)) * args.points * 128

    def load_and_hash():
        for a, b in runs_of(resident):
            m.upload_many(np.arange(a, b, dtype=np.uint32), desc[a:b])
        m.centering_reset()
        m.centering_add_many(owned)
        if strong:
            sums, count = m.centering_sums()
            packed = np.concatenate([np.asarray(sums, np.uint64), np.array([count], np.uint64)])
            others = comm.sum_u64(packed) - packed
            m.centering_add_sums(others[:128], int(others[128]))
        cen = m.centering_apply()
        if len(only_centering):
            m.evict_many(only_centering)
        m.hash(needed)
        return cen

    t0 = time.perf_counter()
    centering = load_and_hash()
    m.sync()
    setup_s = time.perf_counter() - t0

    # ---- value: device-resident matching pass ------------------------------------------------------
    for _ in range(args.warmup):
        m.match_pairs_device(pairs, cfg)
    sampler = ClockSampler(local) if gpu else None
    barrier()
    if sampler:
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
    clocks = sampler.stop() if sampler else {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no GPU engine (test stand-in)"]}
    my_dev_ms = dev_ms
    dev_ms = reduce_ranks(dev_ms, "max")
    wall_s = reduce_ranks(wall_s, "max")
    ms_per_step = dev_ms / args.steps
    total_pairs = reduce_ranks(float(npairs), "sum")  # strong: the one list; weak: world x list
    value = total_pairs / (ms_per_step * 1e-3)
    total_launches = reduce_ranks(float(launches), "sum")

    # ---- roofline of the match kernel (this rank's launches; rank 0 reports) ----------------------------
    peak, peak_src = measured_peak_hbm()
    alg = algorithmic_bytes(last, params.short_bits, params.table_count)
    kern_ms_per_step = max(kern_ms / args.steps, 1e-9)
    achieved = alg / (kern_ms_per_step * 1e-3) / 1e9
    traffic = recorded_traffic()
    roofline = {
        "bound": "hbm", "kernel": last.get("kernel", "join_hits_kernel (tensor-core Hamming pass) + match_kernel<SMEM_TRAIN, L=6, active list>"), "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": achieved / peak, "peak_source": peak_src,
        # dram bytes of one launch of this run's size: the captured launch scaled by its query count
        "traffic": (traffic["dram_bytes_per_launch"] * (last["query_points"] / max(1, last["match_launches"])) /
                    traffic["queries_per_launch"]) if traffic else None,
        "traffic_source": (traffic or {}).get("source"),
        "algorithmic_bytes_per_pair": alg / max(1, npairs),
        "algorithmic_bytes_per_launch": alg / max(1, last["match_launches"]),
        "avg_launch_ms": kern_ms / max(1, match_launches),
        "kernel_share_of_step": kern_ms / my_dev_ms if my_dev_ms else None,
        "note": "candidate gathers (20 B x R, 88% of the algorithmic bytes) are served on chip, "
                "so frac may exceed 1; see DESIGN.md for the on-chip (POPC / issue / tensor) bounds",
    }

    # on-chip bound of the SIMT scan: POPC is the one quarter-rate instruction it cannot avoid
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
                           "note": "Hamming evaluations the reference's algorithm needs (4 POPC-equivalents per raw candidate) "
                                   "against the XU pipe's POPC peak; ncu pipe utilisations of the "
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
            "note": f"instructions per query from the committed ncu capture (profiles/{ipq_src})"}

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
        e2e_s = reduce_ranks(time.perf_counter() - t0, "max") / args.e2e_steps
        assert got["records"] == st["matches"]
        e2e = {
            "value": total_pairs / e2e_s, "unit": UNIT,
            "h2d_bytes_per_step": int(reduce_ranks(float(h2d_bytes + npairs * 16), "sum")),
            "d2h_bytes_per_step": int(reduce_ranks(float(st["matches"] * 16 + (npairs + st["match_launches"]) * 8), "sum")),
            "steps": args.e2e_steps, "ms_per_step": 1e3 * e2e_s,
            "includes": "H2D descriptors from pinned host (the images the shard touches), centering sums"
                        + (" + their 1 KB exchange" if strong else "") +
                        ", hash + bucket build, match, D2H of all MatchRecords to the sink",
        }

    # ---- CPU baseline (rank 0, N=1 only) ----------------------------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        def gpu_codes(i):
            c = m.codes(i)
            return c.shorts, c.longs
        run, info = cpu_sample(args, pairs, desc, codes_from=gpu_codes)
        sec, cpu_matches, cpu_checksum = run()
        cpu = {"value": info["sample_pairs"] / sec, "unit": UNIT, "cores": info["cores"], "kind": info["kind"],
               "sample": info["sample"], "seconds": sec}
        # the sample doubles as a parity check at config-3 size: EVERY record of the sample, through the
        # order-independent checksum the compaction kernel accumulates on the device (not just a match count)
        st = m.match_pairs_device(pairs[: info["sample_pairs"]], cfg)
        cpu["gpu_matches_on_sample"] = st["matches"]
        cpu["cpu_matches_on_sample"] = cpu_matches
        cpu["records_checksum_equal"] = bool(st["records_checksum"] == cpu_checksum)
        cpu["records_checksum"] = f"{cpu_checksum:#018x}"
        assert st["matches"] == cpu_matches, "GPU and CPU reference disagree on the sample (match count)"
        assert st["records_checksum"] == cpu_checksum, "GPU and CPU reference disagree on the sample (records checksum)"

    total_matches = reduce_ranks(float(last["matches"]), "sum")
    report = {"rank": rank, "gpu": local, "pairs": npairs, "images_resident": int(len(needed)),
              "ms_per_step": my_dev_ms / args.steps, "match_kernel_ms_per_step": kern_ms / args.steps,
              "clocks": clocks, "centering_fingerprint": f"{ch.centering_fingerprint(centering):#018x}"}
    reports = comm.gather(report)
    if rank == 0:
        fps = {r["centering_fingerprint"] for r in reports}
        assert (len(fps) == 1) or not strong, f"ranks disagree on the dataset centering: {fps}"
        worst = max(reports, key=lambda r: r["ms_per_step"])
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if (strong or world == 1) else "weak", "vs_baseline": None,
            "dtype": "u8/u32 popcount + exact integer distances (fp64 ratio test; hashing: fp32 filter + exact fp64 re-evaluation)",
            "data": "synthetic", "config": workload_config(args, len(all_pairs), world, strong or world == 1),
            "roofline": roofline, "cpu_baseline": cpu,
            "e2e": e2e, "gpu_launches": int(total_launches), "clocks": worst["clocks"],
            "wall_ms_per_step": 1e3 * wall_s / args.steps, "setup_s": setup_s,
            "matches_per_step": total_matches, "device": props["name"],
            "ranks": reports,
            "shard_work": ({"weights": [int(w) for w in shard_weights],
                            "max_over_min": float(max(shard_weights)) / float(max(1, min(shard_weights)))}
                           if shard_weights is not None else None),
            "collectives": ("none on the data path; torch.distributed: barrier + max/sum of scalars "
                            f"({backend}), 1 KB centering exchange + per-rank report (gloo, host side)") if world > 1 else "none",
        }
        if share:
            line["functional_check_only"] = (f"{world} ranks share {torch.cuda.device_count()} GPU(s) (CHGPU_BENCH_SHARE_GPU=1): "
                                             "the N-rank code path on hardware, not a scaling measurement")
        print(json.dumps(line), flush=True)
    m.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int, argv: list[str], script: str | None = None, check_devices: bool = True) -> int:
    """`bench.py --gpus N` without a launcher: become the launcher.  One process per GPU through torch.distributed.run
    (rank r -> cuda:r via LOCAL_RANK), rendezvous on 127.0.0.1.  Fails loudly when the box has fewer than N GPUs."""
    if check_devices and os.environ.get("CHGPU_BENCH_SHARE_GPU") != "1":
        import torch
        have = torch.cuda.device_count() if torch.cuda.is_available() else 0
        if have < n:
            print(f"bench.py: --gpus {n} asked for, {have} CUDA device(s) visible; refusing to time fewer GPUs than reported",
                  file=sys.stderr)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), script or str(Path(__file__).resolve()), *argv]
    return subprocess.call(cmd)


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    args = parse_args(argv)
    launched = "WORLD_SIZE" in os.environ
    if args.impl == "reference":
        run_reference_arm(args)  # rank 0 alone runs and prints; other ranks of a torchrun launch exit 0 without work
        return 0
    if not launched and args.gpus > 1:
        return spawn_ranks(args.gpus, argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but the launcher started {world} rank(s) (WORLD_SIZE); they must agree",
              file=sys.stderr)
        return 2
    run_ours(args)
    return 0


if __name__ == "__main__":
    sys.exit(main())
