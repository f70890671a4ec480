"""Python harness over the C ABI, shaped like the reference's matcher API.

The product's host side is C++ (include/cashash_b200/cashash.hpp keeps the reference's
signatures).  This module exists so pytest and bench.py can drive the same C ABI; names follow
the reference: FamilyParams / MatchConfig / build_hash_family / set_centering / compute_codes /
build_bucket_index / match_pair / save_matches (hashing.hpp, matcher.hpp, feature_io.hpp).
Errors map to the reference's exception classes:
    CHGPU_EINVAL -> ValueError          (std::invalid_argument)
    CHGPU_ELOGIC -> LogicError          (std::logic_error)
    CHGPU_EFORMAT -> FeatureFileError   (fault class + byte offset)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

RECORD_DTYPE = np.dtype([("query_index", "<u4"), ("train_index", "<u4"), ("distance_sq", "<f8")])
assert RECORD_DTYPE.itemsize == 16


class LogicError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


class UnsupportedError(RuntimeError):
    pass


class FeatureFileError(RuntimeError):
    FAULTS = {1: "MissingFile", 2: "BadMagic", 3: "BadVersion", 4: "Truncated", 5: "Unwritable"}

    def __init__(self, msg: str, fault: int, byte_offset: int):
        super().__init__(msg)
        self.fault = self.FAULTS.get(fault, str(fault))
        self.byte_offset = byte_offset


@dataclass(frozen=True)
class FamilyParams:  # hashing.hpp:45-52
    short_bits: int = 8
    long_bits: int = 128
    table_count: int = 6
    seed: int = 1

    def c(self) -> N.FamilyParamsC:
        return N.FamilyParamsC(self.short_bits, self.long_bits, self.table_count, self.seed)


@dataclass(frozen=True)
class MatchConfig:  # matcher.hpp:14-23
    top_k: int = 10
    hamming_threshold: int = 40
    ratio: float = 0.8
    min_candidates_for_ratio: int = 2
    reduce_rounds: int = 3

    def c(self) -> N.MatchCfgC:
        return N.MatchCfgC(self.top_k, self.hamming_threshold, self.ratio, self.min_candidates_for_ratio,
                           self.reduce_rounds)


@dataclass
class HashFamily:  # hashing.hpp:62-72
    params: FamilyParams
    short_planes: np.ndarray  # (L*m, 128) f64, [table*m + bit]
    long_planes: np.ndarray   # (n, 128) f64
    centering: np.ndarray | None = None


@dataclass
class ImageCodes:  # hashing.hpp:110-114
    params: FamilyParams
    shorts: np.ndarray  # (n, L) u32
    longs: np.ndarray   # (n, 2) u64


@dataclass
class BucketIndex:  # dense view of matcher.hpp:30-41
    short_bits: int
    point_count: int
    offsets: np.ndarray  # (L, 2^m + 1) u32
    points: np.ndarray   # (L, n) u32

    def bucket(self, table: int, code: int) -> np.ndarray:
        return self.points[table, self.offsets[table, code]:self.offsets[table, code + 1]]


def _raise(status: int, msg: str):
    if status == N.EINVAL:
        raise ValueError(msg)
    if status == N.ELOGIC:
        raise LogicError(msg)
    if status == N.EUNSUPPORTED:
        raise UnsupportedError(msg)
    if status == N.ENOMEM:
        raise MemoryError(msg)
    if status == N.ENOTFOUND:
        raise KeyError(msg)
    raise CudaError(msg)


def build_hash_family(params: FamilyParams = FamilyParams()) -> HashFamily:
    """build_hash_family (hashing.hpp:74): host-side, bit-identical hyperplanes."""
    lib = N.load()
    p = params.c()
    if not (1 <= params.short_bits <= 32 and params.short_bits < params.long_bits <= 128 and params.table_count >= 1):
        raise ValueError("family parameters out of range")
    sp = np.empty((params.table_count * params.short_bits, 128), dtype=np.float64)
    lp = np.empty((params.long_bits, 128), dtype=np.float64)
    st = lib.chgpu_family_generate(C.byref(p), sp.ctypes.data_as(N.f64p), lp.ctypes.data_as(N.f64p))
    if st != N.OK:
        _raise(st, "chgpu_family_generate failed")
    return HashFamily(params, sp, lp)


def save_matches(image_id_i: str, image_id_j: str, records: np.ndarray, path: str) -> None:
    """save_matches (feature_io.hpp:106-107)."""
    lib = N.load()
    rec = np.ascontiguousarray(records, dtype=RECORD_DTYPE)
    st = lib.chgpu_save_matches(image_id_i.encode(), image_id_j.encode(), rec.ctypes.data, len(rec), str(path).encode())
    if st != N.OK:
        raise FeatureFileError(f"{path}: unwritable path at byte 0", 5, 0)


# ---- code cache (CHCC) / centering (CHCV) files: hashing.hpp:138-162, engine.cpp:522-541 ----------------
class CacheMismatchError(RuntimeError):
    """std::runtime_error "code cache parameters mismatch active config" (hashing.cpp:244-245)."""


def centering_fingerprint(centering: np.ndarray) -> int:
    c = np.ascontiguousarray(centering, dtype=np.float64)
    assert c.shape == (128,)
    return int(N.load().chgpu_centering_fingerprint(c.ctypes.data_as(N.f64p)))


def save_code_cache(codes: "ImageCodes", centering_fp: int, path) -> None:
    p = codes.params.c()
    s = np.ascontiguousarray(codes.shorts, dtype=np.uint32)
    l = np.ascontiguousarray(codes.longs, dtype=np.uint64)
    st = N.load().chgpu_save_code_cache(str(path).encode(), C.byref(p), centering_fp, len(l), s.ctypes.data, l.ctypes.data)
    if st != N.OK:
        raise FeatureFileError(f"{path}: unwritable path at byte 0", 5, 0)


def read_code_cache_header(path):
    """(FamilyParams, centering_fp, count) or None (missing file / foreign magic: the reference returns false)."""
    p = N.FamilyParamsC()
    fp, cnt = C.c_uint64(0), C.c_uint32(0)
    st = N.load().chgpu_read_code_cache_header(str(path).encode(), C.byref(p), C.byref(fp), C.byref(cnt))
    if st != N.OK:
        return None
    return FamilyParams(p.short_bits, p.long_bits, p.table_count, p.seed), fp.value, cnt.value


def load_code_cache(path, expected: "FamilyParams", expected_centering_fp: int) -> "ImageCodes":
    lib = N.load()
    p = expected.c()
    cnt, fault, off = C.c_uint32(0), C.c_int(0), C.c_uint64(0)
    hdr = read_code_cache_header(path)
    cap = hdr[2] if hdr else 0
    shorts = np.zeros((cap, expected.table_count), dtype=np.uint32)
    longs = np.zeros((cap, 2), dtype=np.uint64)
    st = lib.chgpu_load_code_cache(str(path).encode(), C.byref(p), expected_centering_fp, cap, C.byref(cnt),
                                   shorts.ctypes.data, longs.ctypes.data, C.byref(fault), C.byref(off))
    if st == N.EFORMAT:
        raise FeatureFileError(f"{path}: code cache fault {fault.value} at byte {off.value}", fault.value, off.value)
    if st == N.EMISMATCH:
        raise CacheMismatchError(f"{path}: code cache parameters mismatch active config")
    if st != N.OK:
        _raise(st, f"{path}: load_code_cache failed")
    return ImageCodes(expected, shorts[: cnt.value], longs[: cnt.value])


def save_centering_file(path, params: "FamilyParams", centering: np.ndarray) -> None:
    p = params.c()
    c = np.ascontiguousarray(centering, dtype=np.float64)
    if N.load().chgpu_save_centering_file(str(path).encode(), C.byref(p), c.ctypes.data_as(N.f64p)) != N.OK:
        raise FeatureFileError(f"{path}: unwritable path at byte 0", 5, 0)


def load_centering_file(path):
    p = N.FamilyParamsC()
    c = np.zeros(128, dtype=np.float64)
    st = N.load().chgpu_load_centering_file(str(path).encode(), C.byref(p), c.ctypes.data_as(N.f64p))
    if st != N.OK:
        raise FeatureFileError(f"{path}: not a centering file", 1 if st == N.ENOTFOUND else 2, 0)
    return FamilyParams(p.short_bits, p.long_bits, p.table_count, p.seed), c


def pair_file_name(i: int, j: int) -> str:
    buf = C.create_string_buffer(48)
    N.load().chgpu_pair_file_name(i, j, buf)
    return buf.value.decode()


class MatchFileSink:
    """Asynchronous batched writer of match files (chgpu_sink_*): FileMatchSink, engine.cpp:145-211."""

    def __init__(self, directory, image_names=None, threads: int = 4, max_queued_batches: int = 8):
        self.lib = N.load()
        names = None
        n = 0
        if image_names is not None:
            n = len(image_names)
            names = (C.c_char_p * max(n, 1))(*[str(s).encode() for s in image_names])
        h = C.c_void_p()
        st = self.lib.chgpu_sink_open(str(directory).encode(), names, n, threads, max_queued_batches, C.byref(h))
        if st != N.OK:
            _raise(st, "chgpu_sink_open failed")
        self.h = h

    def accept(self, pairs, offsets, records):
        pr = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
        offs = np.ascontiguousarray(offsets, dtype=np.uint64)
        rec = np.ascontiguousarray(records, dtype=RECORD_DTYPE)
        assert len(offs) == len(pr) + 1
        st = self.lib.chgpu_sink_accept(self.h, pr.ctypes.data, len(pr), offs.ctypes.data, rec.ctypes.data if len(rec) else None)
        if st != N.OK:
            _raise(st, "chgpu_sink_accept failed")

    def close(self) -> dict:
        stats = N.SinkStatsC()
        h, self.h = self.h, None
        if h is not None:
            self.lib.chgpu_sink_close(h, C.byref(stats))
        return stats.as_dict()


def plan_exhaustive(image_count: int, block_images: int, blocks_per_group: int) -> np.ndarray:
    """Pair list of plan_exhaustive (scheduler.hpp:53), flattened in task order: (npairs, 2) u32."""
    lib = N.load()
    n = C.c_uint64(0)
    pairs = np.empty((image_count * (image_count - 1) // 2, 2), dtype=np.uint32)
    st = lib.chgpu_plan_exhaustive(image_count, block_images, blocks_per_group, pairs.ctypes.data, C.byref(n))
    if st != N.OK:
        _raise(st, "partition: image_count, block_images and blocks_per_group must be >= 1")
    assert n.value == len(pairs)
    return pairs


def plan_guided(image_count: int, block_images: int, blocks_per_group: int, accepted_pairs) -> np.ndarray:
    """scheduler.hpp:57 plan_guided, flattened: the exhaustive traversal restricted to `accepted_pairs`."""
    acc = np.ascontiguousarray(accepted_pairs, dtype=np.uint32).reshape(-1, 2)
    out = np.empty((max(len(acc), 1), 2), dtype=np.uint32)
    n = C.c_uint64(0)
    st = N.load().chgpu_plan_guided(image_count, block_images, blocks_per_group, acc.ctypes.data_as(N.u32p), len(acc),
                                    out.ctypes.data_as(N.u32p), C.byref(n))
    if st != N.OK:
        _raise(st, "plan_guided: self pair or unknown image index")
    return out[: n.value].copy()


TASK_DTYPE = np.dtype([("group_a", "<u4"), ("group_b", "<u4"), ("block_a", "<u4"), ("block_b", "<u4"),
                       ("first_pair", "<u8"), ("npairs", "<u8")])
ACTION_DTYPE = np.dtype([("kind", "<u4"), ("level", "<u4"), ("id", "<u4"), ("prefetch", "<u4")])
LOAD, EVICT, BEGIN, FINISH = range(4)   # ActionKind, scheduler.hpp:87
GROUP, BLOCK = range(2)                 # ResidencyLevel, scheduler.hpp:88
HASHING, MATCHING = range(2)            # ResidencyMode, scheduler.hpp:68


def plan_tasks(image_count: int, block_images: int, blocks_per_group: int, accepted_pairs=None) -> np.ndarray:
    """PlanTask list (scheduler.hpp:36-43) of plan_exhaustive (accepted_pairs None) or plan_guided, as TASK_DTYPE rows;
    first_pair / npairs index the flat pair list of plan_exhaustive / plan_guided."""
    lib = N.load()
    acc = None if accepted_pairs is None else np.ascontiguousarray(accepted_pairs, dtype=np.uint32).reshape(-1, 2)
    # a non-NULL pointer selects the guided plan even for an empty list
    keep = None if acc is None else (acc if len(acc) else np.zeros((1, 2), np.uint32))
    ptr = None if acc is None else keep.ctypes.data
    cnt = 0 if acc is None else len(acc)
    n = C.c_uint32(0)
    st = lib.chgpu_plan_tasks(image_count, block_images, blocks_per_group, ptr, cnt, None, C.byref(n))
    if st != N.OK:
        _raise(st, "plan_tasks: bad partition, self pair or unknown image index")
    tasks = np.zeros(n.value, dtype=TASK_DTYPE)
    if n.value:
        st = lib.chgpu_plan_tasks(image_count, block_images, blocks_per_group, ptr, cnt,
                                  tasks.ctypes.data_as(C.POINTER(N.PlanTaskC)), C.byref(n))
        if st != N.OK:
            _raise(st, "plan_tasks")
    return tasks


def hashing_tasks(image_count: int, block_images: int, blocks_per_group: int) -> np.ndarray:
    """hashing_residency_tasks (scheduler.cpp:194-200): one task per block."""
    lib = N.load()
    n = C.c_uint32(0)
    st = lib.chgpu_hashing_tasks(image_count, block_images, blocks_per_group, None, C.byref(n))
    if st != N.OK:
        _raise(st, "hashing_tasks: bad partition")
    tasks = np.zeros(n.value, dtype=TASK_DTYPE)
    lib.chgpu_hashing_tasks(image_count, block_images, blocks_per_group, tasks.ctypes.data_as(C.POINTER(N.PlanTaskC)), C.byref(n))
    return tasks


def simulate_residency(tasks: np.ndarray, mode: int = MATCHING, group_slots: int = 0, block_slots: int = 0) -> np.ndarray:
    """simulate_residency (scheduler.hpp:125): the whole action trace as ACTION_DTYPE rows.  Slots 0 = the reference's
    limits (2 hashing / 3 matching).  ValueError when the limits cannot hold one task (reference: std::logic_error)."""
    lib = N.load()
    t = np.ascontiguousarray(tasks, dtype=TASK_DTYPE)
    tp = t.ctypes.data_as(C.POINTER(N.PlanTaskC)) if len(t) else None
    n = C.c_uint64(0)
    st = lib.chgpu_simulate_residency(tp, len(t), mode, group_slots, block_slots, None, 0, C.byref(n))
    if st != N.OK:
        _raise(st, "residency: current load blocked (slot limit below what one task needs)")
    acts = np.zeros(n.value, dtype=ACTION_DTYPE)
    if n.value:
        st = lib.chgpu_simulate_residency(tp, len(t), mode, group_slots, block_slots,
                                          acts.ctypes.data_as(C.POINTER(N.ResidencyActionC)), n.value, C.byref(n))
        if st != N.OK:
            _raise(st, "simulate_residency")
    return acts


ORDER_REFERENCE, ORDER_REUSE = range(2)  # chgpu_task_order


def order_tasks_for_reuse(tasks: np.ndarray, block_slots: int = 3) -> np.ndarray:
    """Task indices in the order chgpu_match_plan_streamed(task_order=ORDER_REUSE) executes them."""
    t = np.ascontiguousarray(tasks, dtype=TASK_DTYPE)
    out = np.zeros(len(t), dtype=np.uint32)
    if len(t):
        st = N.load().chgpu_order_tasks_for_reuse(t.ctypes.data_as(C.POINTER(N.PlanTaskC)), len(t), block_slots,
                                                  out.ctypes.data_as(N.u32p))
        if st != N.OK:
            _raise(st, "order_tasks_for_reuse")
    return out


def shard_tasks(tasks: np.ndarray, shards: int, order=None, weights=None) -> np.ndarray:
    """Positions (shards + 1) cutting the executed task sequence into contiguous ranges of about equal pair counts,
    or of about equal work when `weights` (task_weights) is given."""
    t = np.ascontiguousarray(tasks, dtype=TASK_DTYPE)
    o = None if order is None else np.ascontiguousarray(order, dtype=np.uint32)
    out = np.zeros(shards + 1, dtype=np.uint32)
    tp = t.ctypes.data_as(C.POINTER(N.PlanTaskC)) if len(t) else None
    op = None if o is None else o.ctypes.data_as(N.u32p)
    if weights is not None:
        w = np.ascontiguousarray(weights, dtype=np.uint64)
        if len(w) != len(t):
            raise ValueError("shard_tasks: one weight per task")
        st = N.load().chgpu_shard_tasks_weighted(tp, op, len(t), w.ctypes.data_as(N.u64p), shards, out.ctypes.data_as(N.u32p))
    else:
        st = N.load().chgpu_shard_tasks(tp, op, len(t), shards, out.ctypes.data_as(N.u32p))
    if st != N.OK:
        _raise(st, "shard_tasks: shards must be >= 1")
    return out


def auto_partition_sizing(mean_image_bytes: int, memory_budget_bytes: int) -> tuple[int, int]:
    """auto_partition_sizing (scheduler.hpp:134): (block_images, blocks_per_group)."""
    a, b = C.c_uint32(0), C.c_uint32(0)
    N.load().chgpu_auto_partition_sizing(mean_image_bytes, memory_budget_bytes, C.byref(a), C.byref(b))
    return a.value, b.value


def partition_sizing_for_device(device_image_bytes: int, file_image_bytes: int, device_bytes: int, host_bytes: int,
                                block_slots: int = 3, group_slots: int = 3) -> tuple[int, int]:
    a, b = C.c_uint32(0), C.c_uint32(0)
    N.load().chgpu_partition_sizing_for_device(device_image_bytes, file_image_bytes, device_bytes, host_bytes, block_slots,
                                               group_slots, C.byref(a), C.byref(b))
    return a.value, b.value


def shard_range(npairs: int, rank: int, world: int) -> tuple[int, int]:
    a, b = C.c_uint64(0), C.c_uint64(0)
    st = N.load().chgpu_shard_range(npairs, rank, world, C.byref(a), C.byref(b))
    if st != N.OK:
        _raise(st, f"shard_range: rank {rank} is not below world {world}")
    return a.value, b.value


def pair_weight(query_points: int, train_points: int) -> int:
    """The work model of one pair that the weighted sharding balances (chgpu_pair_weight)."""
    return int(N.load().chgpu_pair_weight(query_points, train_points))


def shard_pairs_weighted(pairs: np.ndarray, points_per_image, shards: int) -> tuple[np.ndarray, np.ndarray]:
    """Work-balanced contiguous cut of a pair list for datasets of mixed image sizes: (first[shards + 1],
    weight per shard).  Shard s owns pairs[first[s]:first[s + 1]]."""
    pr = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
    pts = np.ascontiguousarray(points_per_image, dtype=np.uint32)
    first = np.zeros(shards + 1, dtype=np.uint64)
    weights = np.zeros(max(shards, 1), dtype=np.uint64)
    st = N.load().chgpu_shard_pairs_weighted(pr.ctypes.data_as(N.u32p) if len(pr) else None, len(pr), pts.ctypes.data_as(N.u32p),
                                             len(pts), shards, first.ctypes.data_as(N.u64p), weights.ctypes.data_as(N.u64p))
    if st != N.OK:
        _raise(st, "shard_pairs_weighted: shards must be >= 1 and every pair index below len(points_per_image)")
    return first, weights


def task_weights(tasks: np.ndarray, pairs: np.ndarray, points_per_image) -> np.ndarray:
    """Work per plan task: sum of pair_weight over the task's pairs of the flat list the tasks index."""
    t = np.ascontiguousarray(tasks, dtype=TASK_DTYPE)
    pr = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
    pts = np.ascontiguousarray(points_per_image, dtype=np.uint32)
    out = np.zeros(len(t), dtype=np.uint64)
    st = N.load().chgpu_task_weights(t.ctypes.data_as(C.POINTER(N.PlanTaskC)) if len(t) else None, len(t),
                                     pr.ctypes.data_as(N.u32p) if len(pr) else None, len(pr), pts.ctypes.data_as(N.u32p), len(pts),
                                     out.ctypes.data_as(N.u64p))
    if st != N.OK:
        _raise(st, "task_weights")
    return out


class Matcher:
    """One device context (one per GPU / per process)."""

    def __init__(self, device: int = 0):
        self.lib = N.load()
        h = C.c_void_p()
        st = self.lib.chgpu_create(device, C.byref(h))
        if st != N.OK:
            raise CudaError(f"chgpu_create(device={device}) failed: {self.lib.chgpu_status_name(st).decode()} "
                            "(a CUDA sm_100 device is required; there is no CPU fallback)")
        self.h = h
        self.params: FamilyParams | None = None
        self._sink_keepalive = None

    # -- plumbing -------------------------------------------------------------------------------
    def close(self):
        if getattr(self, "h", None):
            self.lib.chgpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _ck(self, st: int):
        if st != N.OK:
            _raise(st, self.lib.chgpu_last_error(self.h).decode())

    def sync(self):
        self._ck(self.lib.chgpu_sync(self.h))

    def image_device_bytes(self, n: int) -> int:
        """HBM bytes an image of n points occupies under the installed family (chgpu_image_device_bytes)."""
        out = C.c_uint64(0)
        self._ck(self.lib.chgpu_image_device_bytes(self.h, n, C.byref(out)))
        return int(out.value)

    def set_join(self, enabled: bool = True, min_points_per_bucket: int = 20):
        """The tensor-core Hamming pass in front of the match kernel: off / on from this average bucket occupancy (0: always)."""
        self._ck(self.lib.chgpu_set_join(self.h, 1 if enabled else 0, min_points_per_bucket))

    def set_sub_batch_queries(self, max_queries: int):
        self._ck(self.lib.chgpu_set_sub_batch_queries(self.h, max_queries))

    def device_props(self) -> dict:
        p = N.DevicePropsC()
        self._ck(self.lib.chgpu_get_device_props(self.h, C.byref(p)))
        return {"name": p.name.decode(), "sm_count": p.sm_count, "cc": (p.cc_major, p.cc_minor),
                "total_mem": p.total_mem, "free_mem": p.free_mem, "smem_per_block_optin": p.smem_per_block_optin}

    def pinned_empty(self, shape, dtype) -> np.ndarray:
        """numpy array over pinned host memory (zero-staging uploads)."""
        dtype = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dtype.itemsize
        p = C.c_void_p()
        self._ck(self.lib.chgpu_host_alloc(self.h, nbytes, C.byref(p)))
        buf = (C.c_uint8 * max(nbytes, 1)).from_address(p.value)
        arr = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)
        return arr

    # -- family ---------------------------------------------------------------------------------
    def set_family(self, family: HashFamily):
        p = family.params.c()
        sp = np.ascontiguousarray(family.short_planes, dtype=np.float64)
        lp = np.ascontiguousarray(family.long_planes, dtype=np.float64)
        self._ck(self.lib.chgpu_set_family(self.h, C.byref(p), sp.ctypes.data_as(N.f64p), lp.ctypes.data_as(N.f64p)))
        self.params = family.params
        if family.centering is not None:
            self.set_centering(family.centering)

    def set_centering(self, centering: np.ndarray):
        c = np.ascontiguousarray(centering, dtype=np.float64)
        assert c.shape == (128,)
        self._ck(self.lib.chgpu_set_centering(self.h, c.ctypes.data_as(N.f64p)))

    def centering_reset(self):
        self._ck(self.lib.chgpu_centering_reset(self.h))

    def centering_add(self, image_id: int):
        self._ck(self.lib.chgpu_centering_add_image(self.h, image_id))

    def centering_add_many(self, image_ids):
        ids = np.ascontiguousarray(image_ids, dtype=np.uint32)
        self._ck(self.lib.chgpu_centering_add_images(self.h, ids.ctypes.data_as(N.u32p), len(ids)))

    def centering_sums(self) -> tuple[np.ndarray, int]:
        sums = np.zeros(128, dtype=np.uint64)
        cnt = C.c_uint64(0)
        self._ck(self.lib.chgpu_centering_get_sums(self.h, sums.ctypes.data_as(N.u64p), C.byref(cnt)))
        return sums, cnt.value

    def centering_add_sums(self, sums: np.ndarray, count: int):
        s = np.ascontiguousarray(sums, dtype=np.uint64)
        self._ck(self.lib.chgpu_centering_add_sums(self.h, s.ctypes.data_as(N.u64p), count))

    def centering_apply(self) -> np.ndarray:
        out = np.empty(128, dtype=np.float64)
        self._ck(self.lib.chgpu_centering_apply(self.h, out.ctypes.data_as(N.f64p)))
        return out

    # -- descriptor load ------------------------------------------------------------------------
    def upload(self, image_id: int, desc: np.ndarray, keypoints: np.ndarray | None = None):
        d = np.ascontiguousarray(desc, dtype=np.uint8)
        n = 0 if d.size == 0 else d.shape[0]
        assert d.size == n * 128
        kp = None
        if keypoints is not None:
            kp = np.ascontiguousarray(keypoints, dtype=np.float32)
            assert kp.size == n * 4
        self._ck(self.lib.chgpu_upload_image(self.h, image_id, n, d.ctypes.data if n else None,
                                             kp.ctypes.data if kp is not None and n else None))

    def upload_many(self, image_ids, desc: np.ndarray, keypoints: np.ndarray | None = None):
        """Images of equal size stored back to back: desc (count, n, 128) u8, keypoints (count, n, 4) f32 or None.
        From pinned memory (Matcher.pinned_empty) the copies are issued back to back and drained once."""
        ids = np.ascontiguousarray(image_ids, dtype=np.uint32)
        assert desc.dtype == np.uint8 and desc.flags.c_contiguous and desc.ndim == 3 and desc.shape[2] == 128
        assert desc.shape[0] == len(ids)
        n = desc.shape[1]
        kp = None
        if keypoints is not None:
            kp = keypoints
            assert kp.dtype == np.float32 and kp.flags.c_contiguous and kp.shape == (len(ids), n, 4)
        self._ck(self.lib.chgpu_upload_images(self.h, ids.ctypes.data_as(N.u32p), len(ids), n,
                                              desc.ctypes.data if desc.size else None,
                                              kp.ctypes.data if kp is not None and kp.size else None))

    def upload_chft(self, image_id: int, blob: bytes) -> int:
        cnt = C.c_uint32(0)
        fault = C.c_int(0)
        off = C.c_uint64(0)
        buf = np.frombuffer(blob, dtype=np.uint8)
        st = self.lib.chgpu_upload_chft(self.h, image_id, buf.ctypes.data if buf.size else C.c_void_p(1), len(blob),
                                        C.byref(cnt), C.byref(fault), C.byref(off))
        if st == N.EFORMAT:
            raise FeatureFileError(self.lib.chgpu_last_error(self.h).decode(), fault.value, off.value)
        self._ck(st)
        return cnt.value

    def load_chft_files(self, paths, image_ids, io_threads: int = 8, accumulate_centering: bool = False):
        """Disk -> pinned ring -> HBM streaming load (chgpu_load_chft_files).  Returns (results, stats): results[i] is
        the point count of file i, or a FeatureFileError / exception INSTANCE for a file that was skipped."""
        n = len(paths)
        arr = (C.c_char_p * max(n, 1))(*[str(p).encode() for p in paths])
        ids = np.ascontiguousarray(image_ids, dtype=np.uint32)
        assert len(ids) == n
        res = (N.FileResultC * max(n, 1))()
        st = N.LoadStatsC()
        self._ck(self.lib.chgpu_load_chft_files(self.h, arr, ids.ctypes.data_as(N.u32p), n, io_threads,
                                                1 if accumulate_centering else 0, res, C.byref(st)))
        out = []
        for i in range(n):
            r = res[i]
            if r.status == N.OK:
                out.append(int(r.count))
            elif r.status == N.EFORMAT:
                out.append(FeatureFileError(f"{paths[i]}: fault {r.fault} at byte {r.fault_offset}", r.fault, r.fault_offset))
            else:
                out.append(RuntimeError(f"{paths[i]}: status {r.status}"))
        return out, st.as_dict()

    def _file_results(self, paths, res):
        out = []
        for i in range(len(paths)):
            r = res[i]
            if r.status == N.OK:
                out.append(int(r.count))
            elif r.status == N.EFORMAT:
                out.append(FeatureFileError(f"{paths[i]}: fault {r.fault} at byte {r.fault_offset}", r.fault, r.fault_offset))
            else:
                out.append(RuntimeError(f"{paths[i]}: status {r.status}"))
        return out

    def centering_pass_files(self, paths, block_images: int, io_threads: int = 8):
        """centering_pass (engine.cpp:545-559) streamed block by block, nothing left resident.  Returns
        (centering, per-file results as in load_chft_files)."""
        n = len(paths)
        arr = (C.c_char_p * max(n, 1))(*[str(p).encode() for p in paths])
        res = (N.FileResultC * max(n, 1))()
        out = np.zeros(128, dtype=np.float64)
        st = self.lib.chgpu_centering_pass_files(self.h, arr, n, block_images, io_threads, res, out.ctypes.data_as(N.f64p))
        results = self._file_results(paths, res)
        self._ck(st)
        return out, results

    def match_plan_streamed(self, paths, block_images: int, blocks_per_group: int, cfg: MatchConfig = MatchConfig(),
                            accepted_pairs=None, group_slots: int = 0, block_slots: int = 0, io_threads: int = 8, sink=None,
                            task_order: int = 0, shard: int = 0, shards: int = 1):
        """Out-of-core run of the exhaustive (accepted_pairs None) or guided plan over CHFT files
        (chgpu_match_plan_streamed).  sink(task, pairs (k,2) u32, offsets (k+1) u64, records) is called in execution order
        (plan order, or the reuse order with task_order=ORDER_REUSE; `task` is always the plan's task index).
        Returns (stats dict, per-file results)."""
        n = len(paths)
        arr = (C.c_char_p * max(n, 1))(*[str(p).encode() for p in paths])
        res = (N.FileResultC * max(n, 1))()
        acc = None if accepted_pairs is None else np.ascontiguousarray(accepted_pairs, dtype=np.uint32).reshape(-1, 2)
        keep = None if acc is None else (acc if len(acc) else np.zeros((1, 2), np.uint32))
        c = cfg.c()
        stats = N.StreamedStatsC()
        err: list[BaseException] = []

        def _cb(_user, task, pairs_p, count, offs_p, rec_p):
            try:
                if sink is None:
                    return 0
                pr = np.ctypeslib.as_array(pairs_p, shape=(count, 2)).copy()
                offs = np.ctypeslib.as_array(offs_p, shape=(count + 1,))
                total = int(offs[count] - offs[0])
                if total:
                    rec = np.frombuffer((N.MatchRecordC * total).from_address(C.addressof(rec_p.contents)),
                                        dtype=RECORD_DTYPE)
                else:
                    rec = np.zeros(0, dtype=RECORD_DTYPE)
                sink(int(task), pr, offs, rec)
                return 0
            except BaseException as e:  # noqa: BLE001 - propagate through the C frame
                err.append(e)
                return 1

        cb = N.PLAN_SINK_FN(_cb)
        st = self.lib.chgpu_match_plan_streamed(self.h, arr, n, block_images, blocks_per_group, group_slots, block_slots, task_order,
                                                shard, shards,
                                                None if acc is None else keep.ctypes.data, 0 if acc is None else len(acc),
                                                C.byref(c), io_threads, cb, None, res, C.byref(stats))
        if err:
            raise err[0]
        results = self._file_results(paths, res)
        self._ck(st)
        return stats.as_dict(), results

    def evict(self, image_id: int):
        self._ck(self.lib.chgpu_evict_image(self.h, image_id))

    def load_chft_files_begin(self, paths, image_ids, io_threads: int = 8, accumulate_centering: bool = False):
        """Background load (chgpu_load_chft_files_begin): returns at once; match calls on this Matcher move it forward."""
        n = len(paths)
        arr = (C.c_char_p * max(n, 1))(*[str(p).encode() for p in paths])
        ids = np.ascontiguousarray(image_ids, dtype=np.uint32)
        assert len(ids) == n
        self._bg_paths = list(paths)
        self._ck(self.lib.chgpu_load_chft_files_begin(self.h, arr, ids.ctypes.data_as(N.u32p), n, io_threads,
                                                      1 if accumulate_centering else 0))

    def load_chft_files_end(self):
        """Completes the background load: (results, stats) as load_chft_files returns them."""
        paths = getattr(self, "_bg_paths", [])
        res = (N.FileResultC * max(len(paths), 1))()
        st = N.LoadStatsC()
        self._ck(self.lib.chgpu_load_chft_files_end(self.h, res, C.byref(st)))
        self._bg_paths = []
        return self._file_results(paths, res), st.as_dict()

    def evict_many(self, image_ids):
        ids = np.ascontiguousarray(image_ids, dtype=np.uint32)
        self._ck(self.lib.chgpu_evict_images(self.h, ids.ctypes.data_as(N.u32p), len(ids)))

    def points(self, image_id: int) -> int:
        n = C.c_uint32(0)
        self._ck(self.lib.chgpu_image_points(self.h, image_id, C.byref(n)))
        return n.value

    def descriptors(self, image_id: int) -> tuple[np.ndarray, np.ndarray]:
        n = self.points(image_id)
        d = np.empty((n, 128), dtype=np.uint8)
        kp = np.empty((n, 4), dtype=np.float32)
        self._ck(self.lib.chgpu_download_descriptors(self.h, image_id, d.ctypes.data, kp.ctypes.data))
        return d, kp

    # -- hash build -----------------------------------------------------------------------------
    def hash(self, image_ids, reduce_rounds: int = 3):
        ids = np.ascontiguousarray(image_ids, dtype=np.uint32)
        self._ck(self.lib.chgpu_hash_images(self.h, ids.ctypes.data_as(N.u32p), len(ids), reduce_rounds))

    def set_hash_mode(self, exact):
        """2 or "tensor": the filter on the tensor cores (tcgen05 int8 limbs) + exact fp64 fixup (the context's default);
        False / 0: the fp32 SIMT filter, same fixup; True / 1: every dot in the reference's fp64 order."""
        mode = 2 if exact in (2, "tensor") else (1 if exact else 0)
        self._ck(self.lib.chgpu_set_hash_mode(self.h, mode))

    def hash_stats(self) -> dict:
        st = N.HashStatsC()
        self._ck(self.lib.chgpu_get_hash_stats(self.h, C.byref(st)))
        return st.as_dict()

    def codes(self, image_id: int) -> ImageCodes:
        n = self.points(image_id)
        shorts = np.empty((n, self.params.table_count), dtype=np.uint32)
        longs = np.empty((n, 2), dtype=np.uint64)
        self._ck(self.lib.chgpu_download_codes(self.h, image_id, shorts.ctypes.data, longs.ctypes.data))
        return ImageCodes(self.params, shorts, longs)

    def upload_codes(self, image_id: int, codes: ImageCodes):
        s = np.ascontiguousarray(codes.shorts, dtype=np.uint32)
        l = np.ascontiguousarray(codes.longs, dtype=np.uint64)
        self._ck(self.lib.chgpu_upload_codes(self.h, image_id, s.ctypes.data, l.ctypes.data))

    def save_code_cache(self, image_id: int, path):
        self._ck(self.lib.chgpu_image_save_code_cache(self.h, image_id, str(path).encode()))

    def load_code_cache(self, image_id: int, path):
        """Installs a CHCC cache as the image's codes (hash build skipped); raises like the reference."""
        fault, off = C.c_int(0), C.c_uint64(0)
        st = self.lib.chgpu_image_load_code_cache(self.h, image_id, str(path).encode(), C.byref(fault), C.byref(off))
        if st == N.EFORMAT:
            raise FeatureFileError(self.lib.chgpu_last_error(self.h).decode(), fault.value, off.value)
        if st == N.EMISMATCH:
            raise CacheMismatchError(self.lib.chgpu_last_error(self.h).decode())
        self._ck(st)

    def bucket_index(self, image_id: int) -> BucketIndex:
        n = self.points(image_id)
        L, m = self.params.table_count, self.params.short_bits
        offs = np.empty((L, (1 << m) + 1), dtype=np.uint32)
        pts = np.empty((L, n), dtype=np.uint32)
        self._ck(self.lib.chgpu_download_bucket_index(self.h, image_id, offs.ctypes.data, pts.ctypes.data))
        return BucketIndex(m, n, offs, pts)

    def sorted_index(self, image_id: int) -> tuple[np.ndarray, np.ndarray]:
        """Per table the points sorted by (short code, id) — build_bucket_index before grouping (matcher.cpp:34-37).
        Returns (codes, points), each (L, n) u32; defined for every short_bits."""
        n = self.points(image_id)
        L = self.params.table_count
        codes = np.zeros((L, n), dtype=np.uint32)
        pts = np.zeros((L, n), dtype=np.uint32)
        self._ck(self.lib.chgpu_download_sorted_index(self.h, image_id, codes.ctypes.data, pts.ctypes.data))
        return codes, pts

    # -- match ----------------------------------------------------------------------------------
    def pair_candidates(self, image_i: int, image_j: int) -> tuple[np.ndarray, np.ndarray]:
        """Candidate list of every query of image_i in image_j (matcher.cpp:164-171): (offsets (n_i+1) u64, ids u32)."""
        n = self.points(image_i)
        offsets = np.zeros(n + 1, dtype=np.uint64)
        total = C.c_uint64(0)
        st = self.lib.chgpu_pair_candidates(self.h, image_i, image_j, offsets.ctypes.data, None, 0, C.byref(total))
        if st != N.ENOMEM:
            self._ck(st)
        cands = np.zeros(max(int(total.value), 1), dtype=np.uint32)
        if total.value:
            self._ck(self.lib.chgpu_pair_candidates(self.h, image_i, image_j, offsets.ctypes.data, cands.ctypes.data,
                                                    int(total.value), C.byref(total)))
        return offsets, cands[: int(total.value)]

    def match_pair_lists(self, image_i: int, image_j: int, offsets, ids, cfg: MatchConfig = MatchConfig()):
        """Ranking + verification from explicit per-query candidate lists (the second half of match_pair_filtered)."""
        n = self.points(image_i)
        offs = np.ascontiguousarray(offsets, dtype=np.uint64)
        lst = np.ascontiguousarray(ids, dtype=np.uint32)
        if len(offs) != n + 1 or int(offs[-1]) != len(lst):
            raise ValueError("match_pair_lists: offsets must have n_i + 1 entries and end at len(ids)")
        records = np.zeros(max(n, 1), dtype=RECORD_DTYPE)
        total = C.c_uint64(0)
        stats = N.MatchStatsC()
        c = cfg.c()
        self._ck(self.lib.chgpu_match_pair_lists(self.h, image_i, image_j, C.byref(c), offs.ctypes.data,
                                                 lst.ctypes.data if len(lst) else None, records.ctypes.data, n,
                                                 C.byref(total), C.byref(stats)))
        return records[: total.value], stats.as_dict()

    def match_pair_filtered(self, image_i: int, image_j: int, candidate_filter, cfg: MatchConfig = MatchConfig()):
        """match_pair_filtered (matcher.hpp:102-105) with a HOST callback `candidate_filter(query_index, candidates) ->
        list | None`: called for every query with a non-empty list (matcher.cpp:172), in query order; it returns the edited
        list (None: unchanged).  Lookup before it and ranking + verification after it run on the device."""
        offsets, cands = self.pair_candidates(image_i, image_j)
        n = len(offsets) - 1
        out_lists = []
        new_offs = np.zeros(n + 1, dtype=np.uint64)
        for q in range(n):
            lst = cands[int(offsets[q]): int(offsets[q + 1])]
            if len(lst):
                edited = candidate_filter(q, lst.tolist())
                if edited is not None:
                    lst = np.asarray(edited, dtype=np.uint32).reshape(-1)
            out_lists.append(lst)
            new_offs[q + 1] = new_offs[q] + len(lst)
        ids = np.concatenate(out_lists) if out_lists else np.zeros(0, dtype=np.uint32)
        return self.match_pair_lists(image_i, image_j, new_offs, ids.astype(np.uint32), cfg)

    def match_pairs(self, pairs, cfg: MatchConfig = MatchConfig(), capacity: int | None = None):
        """Returns (offsets (npairs+1) u64, records structured array, stats dict)."""
        pr = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
        npairs = len(pr)
        if capacity is None:
            capacity = int(sum(self.points(int(a)) for a in pr[:, 0])) if npairs <= 4096 else None
        c = cfg.c()
        stats = N.MatchStatsC()
        offsets = np.zeros(npairs + 1, dtype=np.uint64)
        total = C.c_uint64(0)
        if capacity is None:  # size by a first device-only pass
            self._ck(self.lib.chgpu_match_pairs_device(self.h, pr.ctypes.data, npairs, C.byref(c), C.byref(stats)))
            capacity = int(stats.matches)
        records = np.zeros(max(capacity, 1), dtype=RECORD_DTYPE)
        st = self.lib.chgpu_match_pairs(self.h, pr.ctypes.data, npairs, C.byref(c), offsets.ctypes.data,
                                        records.ctypes.data, capacity, C.byref(total), C.byref(stats))
        self._ck(st)
        return offsets, records[: total.value], stats.as_dict()

    def match_pairs_device(self, pairs, cfg: MatchConfig = MatchConfig()) -> dict:
        pr = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
        c = cfg.c()
        stats = N.MatchStatsC()
        self._ck(self.lib.chgpu_match_pairs_device(self.h, pr.ctypes.data, len(pr), C.byref(c), C.byref(stats)))
        return stats.as_dict()

    def match_pairs_stream(self, pairs, cfg: MatchConfig, sink) -> dict:
        """sink(first_pair, offsets ndarray (k+1), records ndarray) -> None; called in pair order."""
        pr = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
        c = cfg.c()
        stats = N.MatchStatsC()
        err: list[BaseException] = []

        def _cb(_user, first, count, offs_p, rec_p):
            try:
                offs = np.ctypeslib.as_array(offs_p, shape=(count + 1,))
                total = int(offs[count])
                if total:
                    rec = np.frombuffer((N.MatchRecordC * total).from_address(C.addressof(rec_p.contents)),
                                        dtype=RECORD_DTYPE)
                else:
                    rec = np.zeros(0, dtype=RECORD_DTYPE)
                if sink is not None:
                    sink(int(first), offs, rec)
                return 0
            except BaseException as e:  # noqa: BLE001 - propagate through the C frame
                err.append(e)
                return 1

        cb = N.SINK_FN(_cb)
        st = self.lib.chgpu_match_pairs_stream(self.h, pr.ctypes.data, len(pr), C.byref(c), cb, None, C.byref(stats))
        if err:
            raise err[0]
        self._ck(st)
        return stats.as_dict()

    def match_pairs_guided(self, pairs, fmats, band_px: float, cfg: MatchConfig = MatchConfig()):
        """guided_match_pair over a pair list: fmats (npairs, 3, 3) f64.  Returns (offsets, records, stats)."""
        pr = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
        f = np.ascontiguousarray(fmats, dtype=np.float64).reshape(len(pr), 9)
        capacity = int(sum(self.points(int(a)) for a in pr[:, 0]))
        c = cfg.c()
        stats = N.MatchStatsC()
        offsets = np.zeros(len(pr) + 1, dtype=np.uint64)
        total = C.c_uint64(0)
        records = np.zeros(max(capacity, 1), dtype=RECORD_DTYPE)
        self._ck(self.lib.chgpu_match_pairs_guided(self.h, pr.ctypes.data, len(pr), C.byref(c), f.ctypes.data, band_px,
                                                   offsets.ctypes.data, records.ctypes.data, capacity, C.byref(total),
                                                   C.byref(stats)))
        return offsets, records[: total.value], stats.as_dict()

    def match_pairs_to_files(self, pairs, sink: "MatchFileSink", cfg: MatchConfig = MatchConfig()) -> dict:
        pr = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
        c = cfg.c()
        stats = N.MatchStatsC()
        self._ck(self.lib.chgpu_match_pairs_to_files(self.h, pr.ctypes.data, len(pr), C.byref(c), sink.h, C.byref(stats)))
        return stats.as_dict()

    def ranked_guided(self, image_i: int, image_j: int, fmat, band_px: float, cfg: MatchConfig = MatchConfig()):
        n = self.points(image_i)
        ranked = np.zeros((n, cfg.top_k), dtype=np.uint32)
        count = np.zeros(n, dtype=np.uint32)
        c = cfg.c()
        f = np.ascontiguousarray(fmat, dtype=np.float64).reshape(9)
        self._ck(self.lib.chgpu_debug_ranked_guided(self.h, image_i, image_j, C.byref(c), f.ctypes.data, band_px,
                                                    ranked.ctypes.data, count.ctypes.data))
        return ranked, count

    def ranked(self, image_i: int, image_j: int, cfg: MatchConfig = MatchConfig()):
        n = self.points(image_i)
        ranked = np.zeros((n, cfg.top_k), dtype=np.uint32)
        count = np.zeros(n, dtype=np.uint32)
        c = cfg.c()
        self._ck(self.lib.chgpu_debug_ranked(self.h, image_i, image_j, C.byref(c), ranked.ctypes.data, count.ctypes.data))
        return ranked, count


# ---- reference-shaped free functions over a default context ---------------------------------------
_default: Matcher | None = None


def default_matcher() -> Matcher:
    global _default
    if _default is None:
        _default = Matcher(0)
    return _default


def set_centering(family: HashFamily, feature_sets) -> None:
    """set_centering (hashing.hpp:78): exact integer column sums on the device, divide on the host."""
    m = default_matcher()
    _install(m, family)
    m.centering_reset()
    total = 0
    for k, fs in enumerate(feature_sets):
        d = np.asarray(fs, dtype=np.uint8).reshape(-1, 128)
        total += len(d)
        m.upload(0xC0000000 + k, d)
        m.centering_add(0xC0000000 + k)
        m.evict(0xC0000000 + k)
    if total == 0:
        raise ValueError("set_centering: no descriptors")
    family.centering = m.centering_apply()


def _install(m: Matcher, family: HashFamily):
    if m.params != family.params or getattr(m, "_family_obj", None) is not family:
        for img in list(getattr(m, "_tmp_ids", [])):
            m.evict(img)
        m._tmp_ids = []
        m.set_family(family)
        m._family_obj = family
    elif family.centering is not None:
        m.set_centering(family.centering)


def compute_codes(family: HashFamily, desc: np.ndarray, reduce_rounds: int = 3) -> ImageCodes:
    """compute_codes (hashing.hpp:131)."""
    if not (0 <= reduce_rounds <= 7):
        raise ValueError("reduce_dot tail rounds out of range 0..7")
    if family.centering is None:
        raise LogicError("compute_codes: centering has not been set")
    m = default_matcher()
    _install(m, family)
    m.upload(0xD0000000, np.asarray(desc, dtype=np.uint8).reshape(-1, 128))
    try:
        m.hash([0xD0000000], reduce_rounds)
        return m.codes(0xD0000000)
    finally:
        m.evict(0xD0000000)


def match_pair(family: HashFamily, desc_i, desc_j, codes_i: ImageCodes, codes_j: ImageCodes,
               cfg: MatchConfig = MatchConfig()) -> np.ndarray:
    """match_pair (matcher.hpp:98-100) with externally supplied codes."""
    if codes_i.params != codes_j.params:
        raise ValueError("match_pair: codes come from different hash families")
    di = np.asarray(desc_i, dtype=np.uint8).reshape(-1, 128)
    dj = np.asarray(desc_j, dtype=np.uint8).reshape(-1, 128)
    if len(di) != len(codes_i.shorts) or len(dj) != len(codes_j.shorts):
        raise ValueError("match_pair: code/point count mismatch")
    m = default_matcher()
    _install(m, family)
    a, b = 0xE0000000, 0xE0000001
    m.upload(a, di)
    m.upload(b, dj)
    try:
        m.upload_codes(a, codes_i)
        m.upload_codes(b, codes_j)
        _, rec, _ = m.match_pairs([(a, b)], cfg)
        return rec.copy()
    finally:
        m.evict(a)
        m.evict(b)
