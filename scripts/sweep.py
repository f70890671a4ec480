#!/usr/bin/env python
"""BASELINE config 5: descriptor-count sweep 1K-32K per image (bucket occupancy / candidate-set size stress),
64 images exhaustive (2,016 pairs) per size, uniform and SIFT-shaped descriptors, plus the epipolar-guided
variant.  Prints one JSON line per case; device-resident timing (CUDA events inside the library)."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1805_08995_b200 as ch  # noqa: E402


def run(m, n, shape, images=64, guided=False, reps=2):
    fam = ch.build_hash_family(ch.FamilyParams())
    m.set_family(fam)
    data = ch.make_dataset(images, n, seed=7, shape=shape)
    rng = np.random.default_rng(3)
    m.centering_reset()
    for i in range(images):
        kp = np.column_stack([rng.uniform(0, 4000, n), rng.uniform(0, 3000, n), np.full(n, 2.0), np.zeros(n)]).astype(np.float32)
        m.upload(i, data[i], kp)
        m.centering_add(i)
    m.centering_apply()
    m.hash(np.arange(images, dtype=np.uint32))
    pairs = ch.plan_exhaustive(images, 8, 2)
    cfg = ch.MatchConfig()
    if guided:
        F = np.tile(np.array([[0.0, -1e-4, 0.3], [1e-4, 0.0, -0.4], [-0.3, 0.4, 1.0]]), (len(pairs), 1, 1))
        m.match_pairs_guided(pairs[:64], F[:64], 40.0, cfg)
        best = None
        for _ in range(reps):
            _, rec, st = m.match_pairs_guided(pairs, F, 40.0, cfg)
            best = st if best is None or st["match_kernel_ms"] < best["match_kernel_ms"] else best
    else:
        m.match_pairs_device(pairs[:64], cfg)
        best = None
        for _ in range(reps):
            st = m.match_pairs_device(pairs, cfg)
            best = st if best is None or st["match_kernel_ms"] < best["match_kernel_ms"] else best
    out = {"points": n, "shape": shape, "guided": guided, "pairs": len(pairs),
           "pairs_per_s_kernel": len(pairs) / (best["match_kernel_ms"] * 1e-3),
           "match_kernel_ms": best["match_kernel_ms"], "raw_candidates_per_query": best["raw_candidates"] / best["query_points"],
           "matches_per_pair": best["matches"] / len(pairs), "verified_per_pair": best["verified_queries"] / len(pairs)}
    for i in range(images):
        m.evict(i)
    return out


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", type=int, nargs="*", default=[1024, 2048, 4096, 8192, 12288, 16384, 32768])
    ap.add_argument("--shapes", nargs="*", default=["uniform", "sift"])
    ap.add_argument("--images", type=int, default=64)
    ap.add_argument("--no-guided", action="store_true")
    ap.add_argument("--guided-points", type=int, nargs="*", default=[8192])
    args = ap.parse_args()
    with ch.Matcher(0) as m:
        for shape in args.shapes:
            for n in args.points:
                print(json.dumps(run(m, n, shape, images=args.images)), flush=True)
        if not args.no_guided:
            for n in args.guided_points:
                print(json.dumps(run(m, n, "uniform", images=args.images, guided=True)), flush=True)


if __name__ == "__main__":
    main()
