#!/usr/bin/env python
"""Loader throughput on an existing directory of CHFT files (scripts/rome16k.py --keep writes one): repeated loads
in one process, images evicted in between, so page cache, pinned buffers and the arena are warm after pass 1."""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1805_08995_b200 as ch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dir", default="/tmp/rome4k")
ap.add_argument("--io-threads", type=int, default=16)
ap.add_argument("--passes", type=int, default=4)
args = ap.parse_args()
paths = sorted(Path(args.dir).glob("img_*.chft"))
ids = np.arange(len(paths), dtype=np.uint32)
nbytes = sum(p.stat().st_size for p in paths)
with ch.Matcher(0) as m:
    m.set_family(ch.build_hash_family(ch.FamilyParams()))
    for k in range(args.passes):
        m.centering_reset()
        t0 = time.perf_counter()
        res, st = m.load_chft_files(paths, ids, io_threads=args.io_threads, accumulate_centering=True)
        dt = time.perf_counter() - t0
        print(json.dumps({"pass": k, "files": len(paths), "seconds": round(dt, 4), "GB_per_s": round(nbytes / dt / 1e9, 2),
                          "reader_busy_s": round(st["read_seconds"], 3)}), flush=True)
        for i in ids:
            m.evict(int(i))
