#!/usr/bin/env python
"""Throughput of the general match path (csrc/general_kernels.cuh) next to the tuned kernels: 64 images x 8,192 points
exhaustive (2,016 pairs), device-resident timing.  One JSON line per case."""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1805_08995_b200 as ch  # noqa: E402


def run(m, images, n, short_bits, top_k):
    fam = ch.build_hash_family(ch.FamilyParams(short_bits=short_bits))
    m.set_family(fam)
    data = ch.make_dataset(images, n, seed=7)
    m.centering_reset()
    for i in range(images):
        m.upload(i, data[i])
        m.centering_add(i)
    m.centering_apply()
    t0 = time.perf_counter()
    m.hash(np.arange(images, dtype=np.uint32))
    m.sync()
    hash_ms = (time.perf_counter() - t0) * 1e3
    pairs = ch.plan_exhaustive(images, 8, 2)
    cfg = ch.MatchConfig(top_k=top_k)
    m.match_pairs_device(pairs[:64], cfg)
    best = None
    for _ in range(2):
        st = m.match_pairs_device(pairs, cfg)
        best = st if best is None or st["match_kernel_ms"] < best["match_kernel_ms"] else best
    out = {"points": n, "short_bits": short_bits, "top_k": top_k, "pairs": len(pairs),
           "path": "general" if short_bits > 12 or top_k > 32 else "tuned",
           "pairs_per_s_kernel": len(pairs) / (best["match_kernel_ms"] * 1e-3), "match_kernel_ms": best["match_kernel_ms"],
           "hash_and_index_ms_per_image": hash_ms / images, "matches_per_pair": best["matches"] / len(pairs),
           "raw_candidates_per_query": best["raw_candidates"] / best["query_points"]}
    for i in range(images):
        m.evict(i)
    return out


if __name__ == "__main__":
    with ch.Matcher(0) as m:
        cases = ((8, 10), (8, 33), (8, 64), (12, 10), (13, 10), (16, 10), (24, 10))
        if "--general-only" in sys.argv:  # A/B runs of the general kernel's variants (CHGPU_GEN_VARIANT)
            cases = ((8, 33), (8, 64), (8, 200), (13, 10), (24, 10))
        for sb, k in cases:
            print(json.dumps(run(m, 64, 8192, sb, k)), flush=True)
