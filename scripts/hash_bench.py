#!/usr/bin/env python
"""Hash-build throughput (K1 / K1f / K1t + K2) on resident images: fp32 filter, tensor-core filter and the exact fp64 kernel.
Prints one JSON line.    python scripts/hash_bench.py --images 1000 --points 8192"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1805_08995_b200 as ch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=1000)
    ap.add_argument("--points", type=int, default=8192)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    K, n = args.images, args.points
    data = ch.make_dataset(K, n, seed=7)
    out = {"images": K, "points": n}
    with ch.Matcher(0) as m:
        m.set_family(ch.build_hash_family(ch.FamilyParams()))
        ids = np.arange(K, dtype=np.uint32)
        m.centering_reset()
        for i in range(K):
            m.upload(i, data[i])
            m.centering_add(i)
        m.centering_apply()
        codes = {}
        for name, exact in (("filtered", False), ("tensor", 2), ("exact", True)):
            m.set_hash_mode(exact)
            m.hash(ids)
            m.sync()
            s0 = m.hash_stats()
            best = 1e9
            for _ in range(args.reps):
                t0 = time.perf_counter()
                m.hash(ids)
                m.sync()
                best = min(best, time.perf_counter() - t0)
            s1 = m.hash_stats()
            c = m.codes(K - 1)
            codes[name] = (c.shorts.copy(), c.longs.copy())
            out[name] = {"seconds": best, "images_per_s": K / best, "us_per_image": best / K * 1e6,
                         "descriptors_per_s": K * n / best,
                         "undecided_dots_per_image": (s1["undecided_dots"] - s0["undecided_dots"]) / args.reps / K,
                         "flipped_bits_per_image": (s1["flipped_bits"] - s0["flipped_bits"]) / args.reps / K}
        out["codes_identical"] = bool(all(np.array_equal(codes[k][0], codes["exact"][0]) and
                                          np.array_equal(codes[k][1], codes["exact"][1]) for k in ("filtered", "tensor")))
        out["speedup"] = out["exact"]["seconds"] / out["filtered"]["seconds"]
        out["speedup_tensor"] = out["exact"]["seconds"] / out["tensor"]["seconds"]
        out["device"] = m.device_props()["name"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
