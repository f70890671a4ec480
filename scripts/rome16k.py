#!/usr/bin/env python
"""BASELINE config 4, Rome16K-shaped: K images x 8,192 descriptors written as CHFT files, pair list (i, i+d),
d = 1..30, streamed disk -> pinned host -> HBM with the loader (chgpu_load_chft_files), hashed and matched with
results streamed back to the host.  Prints one JSON line with the stage timings.

    python scripts/rome16k.py --images 16384 --dir /tmp/rome16k      # full size: 19.3 GB of files, 491,055 pairs
"""
import argparse
import json
import struct
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1805_08995_b200 as ch  # noqa: E402


# ---- parity of a sample of the run against the CPU oracle (checker only; the run itself never touches oracle/) ----------
def _mix64(x):
    x = (x + np.uint64(0x9e3779b97f4a7c15))
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)
    return x ^ (x >> np.uint64(31))


def records_checksum(pair_index, records) -> int:
    """The order-independent checksum compact_kernel and chor_time_match_pairs accumulate, over records tagged with the
    position of their pair in the sample."""
    with np.errstate(over="ignore"):
        a = (pair_index.astype(np.uint64) << np.uint64(32)) | records["query_index"].astype(np.uint64)
        b = (records["train_index"].astype(np.uint64) << np.uint64(32)) | records["distance_sq"].astype(np.uint64)
        return int(np.sum(_mix64(_mix64(a) ^ b), dtype=np.uint64))


class SampleCheck:
    """Keeps the records the run delivers for the pairs among `window` consecutive images and compares them, record for
    record through the checksum, with the reference's match_pair on the host."""

    def __init__(self, K, n, neighbors, window=36, first=None):
        self.n = n
        self.first = (K // 2 if first is None else first)
        self.window = min(window, K - self.first)
        lo, hi = self.first, self.first + self.window
        self.sample = [(i, i + d) for i in range(lo, hi) for d in range(1, neighbors + 1) if i + d < hi]
        self.index = {p: k for k, p in enumerate(self.sample)}
        self.kept = {}

    def take(self, pairs, offs, recs):
        """pairs: (k, 2) image ids of the delivered pairs; offs: (k + 1) record offsets; recs: their records."""
        for k, (a, b) in enumerate(np.asarray(pairs).reshape(-1, 2)):
            key = (int(a), int(b))
            if key in self.index:
                self.kept[key] = recs[int(offs[k]):int(offs[k + 1])].copy()

    def verdict(self, centering) -> dict:
        sys.path.insert(0, str(ROOT / "tests"))
        import oracle_lib
        orc = oracle_lib.best()
        params, cfg = ch.FamilyParams(), ch.MatchConfig()
        fam = ch.build_hash_family(params)
        desc = ch.make_dataset(self.window, self.n, seed=7, first=self.first)
        codes = [orc.compute_codes(params, fam.short_planes, fam.long_planes, centering, desc[i]) for i in range(self.window)]
        local = np.array([[a - self.first, b - self.first] for a, b in self.sample], dtype=np.uint32)
        import os
        sec, cpu_matches, cpu_checksum = orc.time_match_pairs(params, cfg, [desc[i] for i in range(self.window)],
                                                              [c[0] for c in codes], [c[1] for c in codes], local,
                                                              os.cpu_count() or 1)
        missing = [p for p in self.sample if p not in self.kept]
        idx = np.concatenate([np.full(len(self.kept[p]), k, np.uint64) for k, p in enumerate(self.sample) if p in self.kept] or
                             [np.zeros(0, np.uint64)])
        rec = np.concatenate([self.kept[p] for p in self.sample if p in self.kept] or [np.zeros(0, ch.RECORD_DTYPE)])
        got = records_checksum(idx, rec)
        return {"sample_pairs": len(self.sample), "images": [self.first, self.first + self.window], "oracle": orc.name,
                "pairs_missing_from_the_run": len(missing), "gpu_matches": int(len(rec)), "cpu_matches": int(cpu_matches),
                "records_checksum_equal": bool(got == cpu_checksum and not missing), "records_checksum": f"{got:#018x}",
                "cpu_seconds": sec}


def streamed(args, paths, accepted, K, n, write_s):
    """The same workload with bounded residency: centering pass over the files, then the guided plan replayed under
    the residency schedule (Load / Evict of blocks, matching task by task)."""
    with ch.Matcher(0) as m:
        m.set_family(ch.build_hash_family(ch.FamilyParams()))
        t0 = time.perf_counter()
        centering, res = m.centering_pass_files(paths, args.block_images, io_threads=args.io_threads)
        assert all(r == n for r in res)
        t1 = time.perf_counter()
        got = {"records": 0, "pairs": 0, "peak_used": 0}
        check = SampleCheck(K, n, args.neighbors)

        def sink(task, pr, offs, recs):
            got["records"] += len(recs)
            got["pairs"] += len(pr)
            check.take(pr, offs, recs)

        st, res = m.match_plan_streamed(paths, args.block_images, args.blocks_per_group, ch.MatchConfig(), accepted_pairs=accepted,
                                        group_slots=args.group_slots, block_slots=args.block_slots, io_threads=args.io_threads,
                                        sink=sink, task_order=1 if args.reuse_order else 0)
        t2 = time.perf_counter()
        assert got["records"] == st["matches"] and got["pairs"] == st["pairs"]
        props = m.device_props()
        image_bytes = m.image_device_bytes(n)
    parity = check.verdict(np.asarray(centering, dtype=np.float64))
    assert parity["records_checksum_equal"], parity
    tasks = ch.plan_tasks(K, args.block_images, args.blocks_per_group, accepted)
    line = {
        "parity_sample": parity,
        "workload": f"BASELINE configs[3] Rome16K-shaped, OUT OF CORE: {K} images x {n} descriptors from CHFT files, (i,i+d) "
                    f"d=1..{args.neighbors}; blocks of {args.block_images} images, {args.block_slots} block slots, " + ("reuse order" if args.reuse_order else "plan order"),
        "images": K, "pairs": int(st["pairs"]), "tasks": len(tasks), "file_bytes": int(K * (16 + 144 * n)),
        "dataset_write_s": write_s,
        "centering_pass": {"seconds": t1 - t0, "GB_per_s": K * (16 + 144 * n) / (t1 - t0) / 1e9},
        "streamed_run": {"seconds": t2 - t1, "pairs_per_s": st["pairs"] / (t2 - t1), **st},
        "resident_bound_GB": args.block_slots * args.block_images * image_bytes / 1e9,
        "end_to_end": {"seconds": t2 - t0, "pairs_per_s": st["pairs"] / (t2 - t0)},
        "device": props["name"], "hbm_in_use_after_GB": (props["total_mem"] - props["free_mem"]) / 1e9,
    }
    print(json.dumps(line), flush=True)
    if not args.keep:
        for p in paths:
            p.unlink()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=2048)
    ap.add_argument("--points", type=int, default=8192)
    ap.add_argument("--neighbors", type=int, default=30)
    ap.add_argument("--dir", default="/tmp/rome16k_shaped")
    ap.add_argument("--io-threads", type=int, default=16)
    ap.add_argument("--keep", action="store_true")
    ap.add_argument("--streamed", action="store_true",
                    help="out-of-core run (chgpu_match_plan_streamed): at most --block-slots blocks of --block-images images "
                         "resident, loads / evictions by the residency schedule")
    ap.add_argument("--block-images", type=int, default=1024)
    ap.add_argument("--blocks-per-group", type=int, default=4)
    ap.add_argument("--block-slots", type=int, default=3)
    ap.add_argument("--group-slots", type=int, default=3)
    ap.add_argument("--reuse-order", action="store_true", help="execute the tasks in the reuse order (CHGPU_ORDER_REUSE)")
    args = ap.parse_args()
    d = Path(args.dir)
    d.mkdir(parents=True, exist_ok=True)
    K, n = args.images, args.points

    # ---- dataset on disk (not timed) ------------------------------------------------------------
    t0 = time.perf_counter()
    rec = np.zeros(n, dtype=np.dtype([("kp", "<f4", 4), ("d", "u1", 128)]))
    rec["kp"][:, 0] = np.arange(n) % 1000
    rec["kp"][:, 1] = np.arange(n) // 1000
    rec["kp"][:, 2] = 2.0
    header = b"CHFT" + struct.pack("<III", 1, n, 0)
    paths = []
    chunk = 256
    for first in range(0, K, chunk):
        cnt = min(chunk, K - first)
        data = ch.make_dataset(cnt, n, seed=7, first=first)
        for k in range(cnt):
            p = d / f"img_{first + k:06d}.chft"
            if not (p.exists() and p.stat().st_size == 16 + 144 * n):
                rec["d"] = data[k]
                with open(p, "wb") as f:
                    f.write(header)
                    f.write(rec.tobytes())
            paths.append(p)
    write_s = time.perf_counter() - t0
    pairs_list = pairs = np.array([(i, i + dd) for i in range(K) for dd in range(1, args.neighbors + 1) if i + dd < K], dtype=np.uint32)
    pairs = ch.plan_guided(K, 50, 4, pairs)  # the reference's traversal order restricted to this list (scheduler.cpp:144-164)

    if args.streamed:
        return streamed(args, paths, pairs_list, K, n, write_s)
    with ch.Matcher(0) as m:
        m.set_family(ch.build_hash_family(ch.FamilyParams()))
        ids = np.arange(K, dtype=np.uint32)
        t0 = time.perf_counter()
        m.centering_reset()
        results, lst = m.load_chft_files(paths, ids, io_threads=args.io_threads, accumulate_centering=True)
        assert all(r == n for r in results)
        centering = m.centering_apply()
        t1 = time.perf_counter()
        m.hash(ids)
        m.sync()
        t2 = time.perf_counter()
        got = {"records": 0}
        check = SampleCheck(K, n, args.neighbors)

        def sink(first, offs, recs):
            got["records"] += len(recs)
            check.take(pairs[first:first + len(offs) - 1], offs, recs)

        st = m.match_pairs_stream(pairs, ch.MatchConfig(), sink)
        t3 = time.perf_counter()
        assert got["records"] == st["matches"]
        props = m.device_props()
    parity = check.verdict(np.asarray(centering, dtype=np.float64))
    assert parity["records_checksum_equal"], parity
    line = {
        "parity_sample": parity,
        "workload": f"BASELINE configs[3] Rome16K-shaped: {K} images x {n} descriptors from CHFT files, (i,i+d) d=1..{args.neighbors}",
        "images": K, "pairs": len(pairs), "file_bytes": int(K * (16 + 144 * n)), "dataset_write_s": write_s,
        "load": {"seconds": t1 - t0, "GB_per_s": K * (16 + 144 * n) / (t1 - t0) / 1e9, "io_threads": args.io_threads,
                 "reader_busy_s": lst["read_seconds"], "includes": "file reads, H2D, AoS->SoA split, centering sums"},
        "hash": {"seconds": t2 - t1, "images_per_s": K / (t2 - t1)},
        "match": {"seconds": t3 - t2, "pairs_per_s": len(pairs) / (t3 - t2), "kernel_ms": st["match_kernel_ms"],
                  "matches": st["matches"], "includes": "match kernels, compaction, D2H of all MatchRecords to the sink"},
        "end_to_end": {"seconds": t3 - t0, "pairs_per_s": len(pairs) / (t3 - t0)},
        "device": props["name"], "hbm_used_GB": (props["total_mem"] - props["free_mem"]) / 1e9,
    }
    print(json.dumps(line), flush=True)
    if not args.keep:
        for p in paths:
            p.unlink()


if __name__ == "__main__":
    main()
