"""Worker of tests/test_sharding_gloo.py: one rank of a world-size-N gloo job on CPU.

The product's multi-GPU host logic (paper_1805_08995_b200.sharding) runs unmodified; the device
engine is replaced by an ORACLE-BACKED STAND-IN with the Matcher's method names (test
infrastructure: there is no GPU in the CPU test tier)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle_lib  # noqa: E402
import paper_1805_08995_b200 as ch  # noqa: E402
from paper_1805_08995_b200.sharding import CollectingSink, Comm, ShardedJob, streamed_shard_pairs  # noqa: E402


class OracleEngine:
    """Same surface as ch.Matcher, computed by the CPU oracle."""

    def __init__(self, family):
        self.orc = oracle_lib.restatement()
        self.family = family
        self.desc, self.codes = {}, {}
        self.sums = np.zeros(128, dtype=np.uint64)
        self.count = 0
        self.centering = None
        self.uploads = 0

    def upload(self, i, desc):
        self.desc[i] = np.ascontiguousarray(desc, dtype=np.uint8).reshape(-1, 128)
        self.uploads += 1

    def evict(self, i):
        del self.desc[i]
        self.codes.pop(i, None)

    def centering_reset(self):
        self.sums[:] = 0
        self.count = 0

    def centering_add(self, i):
        self.sums += self.desc[i].astype(np.uint64).sum(0)
        self.count += len(self.desc[i])

    def centering_sums(self):
        return self.sums.copy(), self.count

    def centering_add_sums(self, sums, count):
        self.sums += np.asarray(sums, dtype=np.uint64)
        self.count += int(count)

    def centering_apply(self):
        if self.count == 0:
            raise ValueError("set_centering: no descriptors")
        self.centering = self.sums.astype(np.float64) / float(self.count)
        return self.centering

    def hash(self, ids):
        f = self.family
        for i in ids:
            self.codes[int(i)] = self.orc.compute_codes(f.params, f.short_planes, f.long_planes, self.centering,
                                                        self.desc[int(i)])

    def match_pairs_stream(self, pairs, cfg, sink):
        total = 0
        for k, (a, b) in enumerate(np.asarray(pairs).reshape(-1, 2)):  # one "sub-batch" per pair
            a, b = int(a), int(b)
            rec, _ = self.orc.match_pair(self.family.params, cfg, self.desc[a], *self.codes[a], self.desc[b], *self.codes[b])
            sink(k, np.array([0, len(rec)], dtype=np.uint64), rec)
            total += len(rec)
        return {"pairs": len(pairs), "matches": total}


def main():
    out = Path(sys.argv[1])
    images, points = int(sys.argv[2]), int(sys.argv[3])
    import torch.distributed as dist

    dist.init_process_group("gloo")
    comm = Comm(dist.get_rank(), dist.get_world_size())
    fam = ch.build_hash_family(ch.FamilyParams())
    data = ch.make_dataset(images, points, seed=11)
    job = ShardedJob(OracleEngine(fam), comm)
    cen = job.set_centering(lambda i: data[i], images)
    pairs = ch.plan_exhaustive(images, 2, 2)
    sink = CollectingSink()
    stats = job.match(lambda i: data[i], pairs, ch.MatchConfig(), sink)
    counts, records = sink.result()
    gathered = job.gather_results(counts, records)
    np.savez(out / f"rank{comm.rank}.npz", centering=cen, first=stats["first_pair"], last=stats["last_pair"],
             resident=np.array(sorted(job.resident)), uploads=job.engine.uploads)
    if comm.rank == 0:
        offsets, recs = gathered
        np.savez(out / "gathered.npz", offsets=offsets, records=recs, pairs=pairs)
    # the split of an out-of-core (streamed) run: this rank's contiguous range of the task sequence, both orders
    for name, order in (("plan", ch.ORDER_REFERENCE), ("reuse", ch.ORDER_REUSE)):
        tasks_mine, pairs_mine = streamed_shard_pairs(images, 2, 2, comm.rank, comm.world, task_order=order)
        np.savez(out / f"streamed_{name}_rank{comm.rank}.npz", tasks=tasks_mine, pairs=pairs_mine)
    comm.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
