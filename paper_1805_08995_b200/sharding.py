"""Multi-GPU host logic: one process per GPU, pair-list sharding, no data-path collective.

The matching path shards by image pair (reference: assign_workers,
scheduler.cpp:166-173, worker invariance SPEC.md:497).  Per rank:

  1. centering is a property of the whole dataset (hashing.cpp:52-70): rank r sums the images
     i = r (mod world) on its device — exact u64 column sums — and the ranks exchange
     128 sums + a count (1 KB, once) so every rank divides the same integers;
  2. the rank uploads and hashes only the images its shard of the pair list touches;
  3. it matches the contiguous range chgpu_shard_range(npairs, rank, world) of the plan;
  4. results are gathered host-side in pair order (rank ranges are contiguous, so
     concatenation by rank restores the plan order).

`engine` is a paper_1805_08995_b200.Matcher (or anything with the same methods: the CPU tests
drive this module under gloo with an oracle-backed stand-in).  Only torch.distributed is used
for the exchange; host-side gathers go through a gloo group even when NCCL is the default
backend, so no device buffer is involved.
"""
from __future__ import annotations

import os

import numpy as np

from .api import (ORDER_REFERENCE, ORDER_REUSE, RECORD_DTYPE, MatchConfig, order_tasks_for_reuse, plan_exhaustive, plan_guided,
                  plan_tasks, shard_range, shard_tasks)


class Comm:
    """Thin wrapper over torch.distributed (world 1 needs no process group)."""

    def __init__(self, rank: int = 0, world: int = 1):
        self.rank, self.world = rank, world
        self._gloo = None
        if world > 1:
            import torch.distributed as dist

            if not dist.is_initialized():
                raise RuntimeError("initialise torch.distributed before building a Comm for world > 1")
            self._gloo = dist.new_group(backend="gloo") if dist.get_backend() != "gloo" else dist.group.WORLD

    @classmethod
    def from_env(cls) -> "Comm":
        return cls(int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")))

    def sum_u64(self, values: np.ndarray) -> np.ndarray:
        """Element-wise sum over ranks of a u64 vector (values stay below 2^63: 255 * points)."""
        if self.world == 1:
            return values.copy()
        import torch
        import torch.distributed as dist

        t = torch.from_numpy(values.astype(np.int64))
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self._gloo)
        return t.numpy().astype(np.uint64)

    def gather(self, obj, dst: int = 0):
        """Python-object gather to `dst` (list in rank order there, None elsewhere)."""
        if self.world == 1:
            return [obj]
        import torch.distributed as dist

        out = [None] * self.world if self.rank == dst else None
        dist.gather_object(obj, out, dst=dst, group=self._gloo)
        return out

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist

            dist.barrier(group=self._gloo)


class ShardedJob:
    """Exhaustive / pair-list matching of one dataset over `comm.world` GPUs."""

    def __init__(self, engine, comm: Comm):
        self.engine = engine
        self.comm = comm
        self.resident: set[int] = set()
        self.centering = None

    # -- step 1: dataset centering ------------------------------------------------------------
    def set_centering(self, load_image, image_count: int) -> np.ndarray:
        e, c = self.engine, self.comm
        e.centering_reset()
        for i in range(c.rank, image_count, c.world):
            e.upload(i, load_image(i))
            e.centering_add(i)
            self.resident.add(i)
        sums, count = e.centering_sums()
        packed = np.concatenate([np.asarray(sums, dtype=np.uint64), np.array([count], dtype=np.uint64)])
        total = c.sum_u64(packed)
        others = total - packed
        if c.world > 1:
            e.centering_add_sums(others[:128], int(others[128]))
        self.centering = e.centering_apply()
        return self.centering

    # -- step 2 + 3: residency and matching -----------------------------------------------------
    def shard(self, npairs: int) -> tuple[int, int]:
        return shard_range(npairs, self.comm.rank, self.comm.world)

    def match(self, load_image, pairs: np.ndarray, cfg: MatchConfig = MatchConfig(), sink=None) -> dict:
        """Matches this rank's contiguous range of `pairs`.  sink(first_pair_global, offsets, records)
        is called in pair order.  Returns the engine's statistics plus the range."""
        e = self.engine
        pairs = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
        first, last = self.shard(len(pairs))
        mine = pairs[first:last]
        needed = set(int(x) for x in np.unique(mine))
        for i in sorted(self.resident - needed):  # images only the centering pass needed
            e.evict(i)
            self.resident.discard(i)
        for i in sorted(needed - self.resident):
            e.upload(i, load_image(i))
            self.resident.add(i)
        if needed:
            e.hash(np.array(sorted(needed), dtype=np.uint32))

        def shifted(local_first, offs, rec):
            if sink is not None:
                sink(first + local_first, offs, rec)

        stats = e.match_pairs_stream(mine, cfg, shifted) if len(mine) else {"pairs": 0, "matches": 0}
        stats = dict(stats)
        stats["first_pair"], stats["last_pair"] = first, last
        return stats

    # -- step 4: host-side gather -----------------------------------------------------------------
    def gather_results(self, counts: np.ndarray, records: np.ndarray):
        """counts: matches per pair of this rank's range; records: its MatchRecords in pair order.
        Rank 0 gets (offsets over ALL pairs, records) in plan order; other ranks get None."""
        parts = self.comm.gather((np.asarray(counts, dtype=np.uint64), np.asarray(records, dtype=RECORD_DTYPE)))
        if parts is None:
            return None
        all_counts = np.concatenate([p[0] for p in parts]) if parts else np.zeros(0, np.uint64)
        offsets = np.zeros(len(all_counts) + 1, dtype=np.uint64)
        np.cumsum(all_counts, out=offsets[1:])
        return offsets, np.concatenate([p[1] for p in parts])


def streamed_shard_pairs(image_count: int, block_images: int, blocks_per_group: int, rank: int, world: int, accepted_pairs=None,
                         task_order: int = ORDER_REFERENCE, block_slots: int = 3):
    """Host mirror of the split chgpu_match_plan_streamed(shard=rank, shards=world) makes: (plan task indices, pairs) this
    rank executes, in execution order — a contiguous range of the (optionally reuse-ordered) task sequence, balanced by
    pair count, so a rank keeps the block locality of the sequence."""
    tasks = plan_tasks(image_count, block_images, blocks_per_group, accepted_pairs)
    flat = plan_exhaustive(image_count, block_images, blocks_per_group) if accepted_pairs is None else plan_guided(
        image_count, block_images, blocks_per_group, accepted_pairs)
    order = order_tasks_for_reuse(tasks, block_slots) if task_order == ORDER_REUSE else np.arange(len(tasks), dtype=np.uint32)
    first = shard_tasks(tasks, world, order)
    mine = order[int(first[rank]):int(first[rank + 1])]
    chunks = [flat[int(tasks["first_pair"][t]):int(tasks["first_pair"][t] + tasks["npairs"][t])] for t in mine]
    pairs = np.concatenate(chunks) if chunks else np.zeros((0, 2), np.uint32)
    return mine, pairs


class StreamedShardedJob:
    """Out-of-core matching of one dataset of CHFT files over `comm.world` GPUs: every rank streams the centering
    pass over its share of the files (exact u64 sums, exchanged once: 1 KB), then runs its contiguous range of the task
    sequence with chgpu_match_plan_streamed(shard=rank, shards=world).  No data-path collective."""

    def __init__(self, engine, comm: Comm):
        self.engine = engine
        self.comm = comm

    def set_centering(self, paths, block_images: int, io_threads: int = 8) -> np.ndarray:
        e, c = self.engine, self.comm
        mine = list(paths[c.rank::c.world])
        e.centering_reset()
        if mine:
            e.centering_pass_files(mine, block_images, io_threads)  # leaves this rank's sums in the accumulator
        sums, count = e.centering_sums()
        packed = np.concatenate([np.asarray(sums, dtype=np.uint64), np.array([count], dtype=np.uint64)])
        others = c.sum_u64(packed) - packed
        if c.world > 1:
            e.centering_add_sums(others[:128], int(others[128]))
        return e.centering_apply()

    def match(self, paths, block_images: int, blocks_per_group: int, cfg: MatchConfig = MatchConfig(), accepted_pairs=None,
              block_slots: int = 0, task_order: int = ORDER_REUSE, io_threads: int = 8, sink=None):
        stats, results = self.engine.match_plan_streamed(paths, block_images, blocks_per_group, cfg, accepted_pairs=accepted_pairs,
                                                         block_slots=block_slots, io_threads=io_threads, sink=sink,
                                                         task_order=task_order, shard=self.comm.rank, shards=self.comm.world)
        return stats, results


class CollectingSink:
    """Keeps every sub-batch (copies: the engine's pinned buffers are reused after the call returns)."""

    def __init__(self):
        self.counts: list[np.ndarray] = []
        self.records: list[np.ndarray] = []

    def __call__(self, first_pair, offsets, records):
        self.counts.append(np.diff(np.asarray(offsets, dtype=np.uint64)))
        self.records.append(np.array(records, dtype=RECORD_DTYPE, copy=True))

    def result(self):
        counts = np.concatenate(self.counts) if self.counts else np.zeros(0, np.uint64)
        records = np.concatenate(self.records) if self.records else np.zeros(0, RECORD_DTYPE)
        return counts, records
