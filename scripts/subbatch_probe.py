#!/usr/bin/env python
"""Device-resident config-3 pass as a function of the sub-batch size (queries per match-kernel launch): larger
launches pay the persistent grid's tail (SMs idling while the last units finish) less often."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1805_08995_b200 as ch  # noqa: E402

K, n = 1000, 8192
with ch.Matcher(0) as m:
    m.set_family(ch.build_hash_family(ch.FamilyParams()))
    desc = m.pinned_empty((K, n, 128), np.uint8)
    ch.make_dataset(K, n, seed=7, out=desc)
    ids = np.arange(K, dtype=np.uint32)
    m.upload_many(ids, desc)
    m.centering_reset()
    m.centering_add_many(ids)
    m.centering_apply()
    m.hash(ids)
    pairs = ch.plan_exhaustive(K, 50, 4)
    cfg = ch.MatchConfig()
    m.match_pairs_device(pairs[:20000], cfg)
    for mq in (8, 16, 32, 64, 128):
        m.set_sub_batch_queries(mq << 20)
        m.match_pairs_device(pairs, cfg)
        st = m.match_pairs_device(pairs, cfg)
        print(json.dumps({"sub_batch_Mi_queries": mq, "launches": st["match_launches"], "total_ms": st["total_ms"],
                          "kernel_ms": st["match_kernel_ms"], "pairs_per_s": len(pairs) / (st["total_ms"] * 1e-3)}), flush=True)
