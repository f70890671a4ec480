"""Rank entry of tests/test_bench_contract.py's multi-rank test: bench.py's own main() — argument parsing, rank /
world checks, work-balanced sharding of the ONE pair list, centering exchange, timing reductions, per-rank report,
JSON line — with the device engine replaced by an ORACLE-BACKED STAND-IN carrying ch.Matcher's method names (test
infrastructure: the CPU test tier has no GPU).  Launched by bench.spawn_ranks() exactly like bench.py launches itself."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import bench  # noqa: E402
import oracle_lib  # noqa: E402
import paper_1805_08995_b200 as ch  # noqa: E402
from dist_worker import OracleEngine  # noqa: E402


class BenchOracleEngine(OracleEngine):
    """The part of ch.Matcher bench.run_ours drives, computed by the CPU oracle."""

    def __init__(self, _device):
        super().__init__(None)

    def set_family(self, family):
        self.family = family

    def pinned_empty(self, shape, dtype):
        return np.empty(shape, dtype)

    def upload_many(self, ids, desc):
        for k, i in enumerate(ids):
            self.upload(int(i), desc[k])

    def centering_add_many(self, ids):
        for i in ids:
            self.centering_add(int(i))

    def evict_many(self, ids):
        for i in ids:
            self.evict(int(i))

    def sync(self):
        pass

    def close(self):
        pass

    def device_props(self):
        return {"name": "oracle stand-in (CPU)", "sm_count": 1}

    def _run(self, pairs, cfg, sink=None):
        t0 = time.perf_counter()
        out = {"pairs": len(pairs), "matches": 0, "raw_candidates": 0, "verified_queries": 0, "distances": 0, "query_points": 0,
               "train_points": 0, "records_checksum": 0, "match_launches": 1, "total_launches": 3}
        for k, (a, b) in enumerate(np.asarray(pairs).reshape(-1, 2)):
            a, b = int(a), int(b)
            rec, st = self.orc.match_pair(self.family.params, cfg, self.desc[a], *self.codes[a], self.desc[b], *self.codes[b])
            out["matches"] += len(rec)
            for f in ("raw_candidates", "verified_queries", "distances"):
                out[f] += st[f]
            out["query_points"] += len(self.desc[a])
            out["train_points"] += len(self.desc[b])
            if sink is not None:
                sink(k, np.array([0, len(rec)], dtype=np.uint64), rec)
        ms = 1e3 * (time.perf_counter() - t0)
        out["match_kernel_ms"] = 0.9 * ms
        out["total_ms"] = ms
        return out

    def match_pairs_device(self, pairs, cfg):
        return self._run(pairs, cfg)

    def match_pairs_stream(self, pairs, cfg, sink):
        return self._run(pairs, cfg, sink)


if __name__ == "__main__":
    bench.ENGINE_FACTORY = BenchOracleEngine
    bench.DIST_BACKEND = "gloo"
    sys.exit(bench.main(sys.argv[1:]))
