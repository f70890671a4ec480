"""ctypes binding of the CPU checkers (oracle/chor.h).  TEST INFRASTRUCTURE: imported only by
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs."""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_DIR = ROOT / "oracle"
RESTATEMENT = ORACLE_DIR / "libchoracle.so"
REFERENCE = ORACLE_DIR / "_ref" / "libcashash_ref.so"

RECORD_DTYPE = np.dtype([("query_index", "<u4"), ("train_index", "<u4"), ("distance_sq", "<f8")])


class FamilyParamsC(C.Structure):
    _fields_ = [("short_bits", C.c_uint32), ("long_bits", C.c_uint32), ("table_count", C.c_uint32),
                ("seed", C.c_uint64)]


class MatchCfgC(C.Structure):
    _fields_ = [("top_k", C.c_uint32), ("hamming_threshold", C.c_uint32), ("ratio", C.c_double),
                ("min_candidates_for_ratio", C.c_uint32), ("reduce_rounds", C.c_int32)]


class PairStatsC(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("raw_candidates", "unique_candidates", "ranked_queries",
                                           "fallback_queries", "verified_queries", "distances", "matches")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


def build_oracle(ref: bool = True) -> None:
    """Compiles the restatement and, when /root/reference is present, the reference shim."""
    subprocess.run(["make", "-C", str(ORACLE_DIR), "all"], check=True, capture_output=True)
    if ref and Path("/root/reference/proj/src/matcher.cpp").exists():
        subprocess.run(["make", "-C", str(ORACLE_DIR), "ref"], check=True, capture_output=True)


class Oracle:
    """One of the two checkers behind the same ABI."""

    def __init__(self, path: Path):
        self.path = Path(path)
        self.lib = C.CDLL(str(path))
        self.lib.chor_name.restype = C.c_char_p
        self.name = self.lib.chor_name().decode()
        P, U32, U64, I, D = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_double
        sigs = {
            "chor_mix64_3": [U64, U64, U64, P],
            "chor_reduce_dot": [P, P, I, P],
            "chor_build_family": [P, P, P],
            "chor_centering_accumulate": [P, U64, P, P],
            "chor_centering_apply": [P, U64, P],
            "chor_compute_codes": [P, P, P, P, I, P, U32, P, P],
            "chor_build_bucket_index": [U32, U32, P, U32, P, P],
            "chor_lookup_candidates": [U32, U32, P, P, U32, P, P],
            "chor_match_pair": [P, P, P, U32, P, P, P, U32, P, P, P, P, P, P, P],
            "chor_match_pair_lists": [P, P, P, U32, P, P, P, U32, P, P, P, P, P, P, P, P, P],
            "chor_brute_force_match": [P, U32, P, U32, D, P, P],
            "chor_guided_match_pair": [P, P, P, P, U32, P, P, P, P, U32, P, P, P, D, P, P, P, P, P],
            "chor_save_matches": [C.c_char_p, C.c_char_p, P, U32, C.c_char_p],
            "chor_time_match_pairs": [P, P, P, P, P, P, P, U32, U32, P, P, P],
            "chor_plan_exhaustive": [U32, U32, U32, P, P, P, P],
            "chor_plan_guided": [U32, U32, U32, P, C.c_uint64, P, P, P, P],
            "chor_plan_task_blocks": [U32, U32, U32, C.c_int, P, C.c_uint64, P, P],
            "chor_simulate_residency": [U32, U32, U32, C.c_int, C.c_int, P, C.c_uint64, P, C.c_uint64, P],
            "chor_auto_partition_sizing": [C.c_uint64, C.c_uint64, P, P],
            "chor_centering_fingerprint": [P, P],
            "chor_save_code_cache": [P, U64, P, P, U32, C.c_char_p],
            "chor_load_code_cache": [C.c_char_p, P, U64, U32, P, P, P, P, P],
        }
        for name, args in sigs.items():
            fn = getattr(self.lib, name)
            fn.restype = C.c_int
            fn.argtypes = args

    # -- helpers --------------------------------------------------------------------------------
    @staticmethod
    def _fp(params) -> FamilyParamsC:
        return FamilyParamsC(params.short_bits, params.long_bits, params.table_count, params.seed)

    @staticmethod
    def _cfg(cfg) -> MatchCfgC:
        return MatchCfgC(cfg.top_k, cfg.hamming_threshold, cfg.ratio, cfg.min_candidates_for_ratio, cfg.reduce_rounds)

    @staticmethod
    def _check(rc: int, what: str):
        if rc == 1:
            raise ValueError(what)
        if rc == 2:
            raise RuntimeError("logic_error: " + what)
        if rc != 0:
            raise RuntimeError(what)

    # -- ops ------------------------------------------------------------------------------------
    def mix64(self, seed: int, a: int, b: int) -> int:
        out = C.c_uint64(0)
        self.lib.chor_mix64_3(C.c_uint64(seed), C.c_uint64(a), C.c_uint64(b), C.byref(out))
        return out.value

    def reduce_dot(self, a, b, rounds: int = 3) -> float:
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = C.c_double(0)
        self._check(self.lib.chor_reduce_dot(a.ctypes.data, b.ctypes.data, rounds, C.byref(out)), "reduce_dot")
        return out.value

    def build_family(self, params):
        p = self._fp(params)
        sp = np.zeros((params.table_count * params.short_bits, 128), dtype=np.float64)
        lp = np.zeros((params.long_bits, 128), dtype=np.float64)
        self._check(self.lib.chor_build_family(C.byref(p), sp.ctypes.data, lp.ctypes.data), "build_hash_family")
        return sp, lp

    def centering(self, desc_sets) -> np.ndarray:
        sums = np.zeros(128, dtype=np.uint64)
        cnt = C.c_uint64(0)
        for d in desc_sets:
            d = np.ascontiguousarray(d, dtype=np.uint8).reshape(-1, 128)
            self._check(self.lib.chor_centering_accumulate(d.ctypes.data, C.c_uint64(len(d)), sums.ctypes.data,
                                                           C.byref(cnt)), "centering add")
        out = np.zeros(128, dtype=np.float64)
        self._check(self.lib.chor_centering_apply(sums.ctypes.data, cnt, out.ctypes.data), "set_centering: no descriptors")
        return out

    def compute_codes(self, params, short_planes, long_planes, centering, desc, reduce_rounds: int = 3):
        p = self._fp(params)
        d = np.ascontiguousarray(desc, dtype=np.uint8).reshape(-1, 128)
        n = len(d)
        shorts = np.zeros((n, params.table_count), dtype=np.uint32)
        longs = np.zeros((n, 2), dtype=np.uint64)
        sp = np.ascontiguousarray(short_planes, dtype=np.float64)
        lp = np.ascontiguousarray(long_planes, dtype=np.float64)
        cptr = None
        if centering is not None:
            c = np.ascontiguousarray(centering, dtype=np.float64)
            cptr = c.ctypes.data
        self._check(self.lib.chor_compute_codes(C.byref(p), sp.ctypes.data, lp.ctypes.data, C.c_void_p(cptr),
                                                reduce_rounds, d.ctypes.data, n, shorts.ctypes.data,
                                                longs.ctypes.data), "compute_codes")
        return shorts, longs

    def build_bucket_index(self, m: int, L: int, shorts):
        s = np.ascontiguousarray(shorts, dtype=np.uint32).reshape(-1, L)
        n = len(s)
        offs = np.zeros((L, (1 << m) + 1), dtype=np.uint32)
        pts = np.zeros((L, n), dtype=np.uint32)
        self._check(self.lib.chor_build_bucket_index(m, L, s.ctypes.data, n, offs.ctypes.data, pts.ctypes.data),
                    "build_bucket_index")
        return offs, pts

    def lookup_candidates(self, m: int, L: int, query_codes, train_shorts):
        q = np.ascontiguousarray(query_codes, dtype=np.uint32)
        s = np.ascontiguousarray(train_shorts, dtype=np.uint32).reshape(-1, L)
        out = np.zeros(max(len(s), 1), dtype=np.uint32)
        cnt = C.c_uint32(0)
        self._check(self.lib.chor_lookup_candidates(m, L, q.ctypes.data, s.ctypes.data, len(s), out.ctypes.data,
                                                    C.byref(cnt)), "lookup_candidates")
        return out[: cnt.value].copy()

    def match_pair(self, params, cfg, desc_i, shorts_i, longs_i, desc_j, shorts_j, longs_j, want_ranked=False):
        p, c = self._fp(params), self._cfg(cfg)
        di = np.ascontiguousarray(desc_i, dtype=np.uint8).reshape(-1, 128)
        dj = np.ascontiguousarray(desc_j, dtype=np.uint8).reshape(-1, 128)
        si = np.ascontiguousarray(shorts_i, dtype=np.uint32)
        sj = np.ascontiguousarray(shorts_j, dtype=np.uint32)
        li = np.ascontiguousarray(longs_i, dtype=np.uint64)
        lj = np.ascontiguousarray(longs_j, dtype=np.uint64)
        ni, nj = len(di), len(dj)
        rec = np.zeros(max(ni, 1), dtype=RECORD_DTYPE)
        cnt = C.c_uint32(0)
        stats = PairStatsC()
        ranked = np.zeros((max(ni, 1), cfg.top_k), dtype=np.uint32) if want_ranked else None
        rcount = np.zeros(max(ni, 1), dtype=np.uint32) if want_ranked else None
        self._check(self.lib.chor_match_pair(
            C.byref(p), C.byref(c), di.ctypes.data, ni, si.ctypes.data, li.ctypes.data, dj.ctypes.data, nj,
            sj.ctypes.data, lj.ctypes.data, rec.ctypes.data, C.byref(cnt), C.byref(stats),
            C.c_void_p(ranked.ctypes.data if want_ranked else None),
            C.c_void_p(rcount.ctypes.data if want_ranked else None)), "match_pair")
        out = rec[: cnt.value].copy()
        if want_ranked:
            return out, stats.as_dict(), ranked[:ni], rcount[:ni]
        return out, stats.as_dict()

    def match_pair_lists(self, params, cfg, desc_i, shorts_i, longs_i, desc_j, shorts_j, longs_j, list_offsets, list_ids,
                         want_ranked=False):
        """match_pair_filtered with a filter that replaces the candidates of query q by list_ids[offs[q]:offs[q+1]]."""
        p, c = self._fp(params), self._cfg(cfg)
        di = np.ascontiguousarray(desc_i, dtype=np.uint8).reshape(-1, 128)
        dj = np.ascontiguousarray(desc_j, dtype=np.uint8).reshape(-1, 128)
        si = np.ascontiguousarray(shorts_i, dtype=np.uint32)
        sj = np.ascontiguousarray(shorts_j, dtype=np.uint32)
        li = np.ascontiguousarray(longs_i, dtype=np.uint64)
        lj = np.ascontiguousarray(longs_j, dtype=np.uint64)
        lo = np.ascontiguousarray(list_offsets, dtype=np.uint64)
        ids = np.ascontiguousarray(list_ids, dtype=np.uint32)
        if len(ids) == 0:
            ids = np.zeros(1, dtype=np.uint32)
        ni, nj = len(di), len(dj)
        rec = np.zeros(max(ni, 1), dtype=RECORD_DTYPE)
        cnt = C.c_uint32(0)
        stats = PairStatsC()
        ranked = np.zeros((max(ni, 1), cfg.top_k), dtype=np.uint32) if want_ranked else None
        rcount = np.zeros(max(ni, 1), dtype=np.uint32) if want_ranked else None
        self._check(self.lib.chor_match_pair_lists(
            C.byref(p), C.byref(c), di.ctypes.data, ni, si.ctypes.data, li.ctypes.data, dj.ctypes.data, nj,
            sj.ctypes.data, lj.ctypes.data, lo.ctypes.data, ids.ctypes.data, rec.ctypes.data, C.byref(cnt), C.byref(stats),
            C.c_void_p(ranked.ctypes.data if want_ranked else None),
            C.c_void_p(rcount.ctypes.data if want_ranked else None)), "match_pair_lists")
        out = rec[: cnt.value].copy()
        if want_ranked:
            return out, stats.as_dict(), ranked[:ni], rcount[:ni]
        return out, stats.as_dict()

    def set_line_order(self, order: int) -> None:
        """Restatement only: association order of the epipolar line's third component (chor.h)."""
        self.lib.chor_set_line_order.restype = None
        self.lib.chor_set_line_order(C.c_int(order))

    def guided_match_pair(self, params, cfg, desc_i, kp_i, shorts_i, longs_i, desc_j, kp_j, shorts_j, longs_j, F, band_px,
                          want_ranked=False):
        p, c = self._fp(params), self._cfg(cfg)
        di = np.ascontiguousarray(desc_i, dtype=np.uint8).reshape(-1, 128)
        dj = np.ascontiguousarray(desc_j, dtype=np.uint8).reshape(-1, 128)
        ki = np.ascontiguousarray(kp_i, dtype=np.float32).reshape(-1, 4)
        kj = np.ascontiguousarray(kp_j, dtype=np.float32).reshape(-1, 4)
        si = np.ascontiguousarray(shorts_i, dtype=np.uint32)
        sj = np.ascontiguousarray(shorts_j, dtype=np.uint32)
        li = np.ascontiguousarray(longs_i, dtype=np.uint64)
        lj = np.ascontiguousarray(longs_j, dtype=np.uint64)
        f = np.ascontiguousarray(F, dtype=np.float64).reshape(9)
        ni, nj = len(di), len(dj)
        assert len(ki) == ni and len(kj) == nj
        rec = np.zeros(max(ni, 1), dtype=RECORD_DTYPE)
        cnt = C.c_uint32(0)
        stats = PairStatsC()
        ranked = np.zeros((max(ni, 1), cfg.top_k), dtype=np.uint32)
        rcount = np.zeros(max(ni, 1), dtype=np.uint32)
        self._check(self.lib.chor_guided_match_pair(
            C.byref(p), C.byref(c), di.ctypes.data, ki.ctypes.data, ni, si.ctypes.data, li.ctypes.data,
            dj.ctypes.data, kj.ctypes.data, nj, sj.ctypes.data, lj.ctypes.data, f.ctypes.data, C.c_double(band_px),
            rec.ctypes.data, C.byref(cnt), C.byref(stats), ranked.ctypes.data, rcount.ctypes.data), "guided_match_pair")
        out = rec[: cnt.value].copy()
        if want_ranked:
            return out, stats.as_dict(), ranked[:ni], rcount[:ni]
        return out, stats.as_dict()

    def brute_force_match(self, desc_i, desc_j, ratio: float):
        di = np.ascontiguousarray(desc_i, dtype=np.uint8).reshape(-1, 128)
        dj = np.ascontiguousarray(desc_j, dtype=np.uint8).reshape(-1, 128)
        rec = np.zeros(max(len(di), 1), dtype=RECORD_DTYPE)
        cnt = C.c_uint32(0)
        self._check(self.lib.chor_brute_force_match(di.ctypes.data, len(di), dj.ctypes.data, len(dj), C.c_double(ratio),
                                                    rec.ctypes.data, C.byref(cnt)), "brute_force_match")
        return rec[: cnt.value].copy()

    def save_matches(self, id_i: str, id_j: str, records, path):
        rec = np.ascontiguousarray(records, dtype=RECORD_DTYPE)
        self._check(self.lib.chor_save_matches(id_i.encode(), id_j.encode(), rec.ctypes.data, len(rec),
                                               str(path).encode()), "save_matches")

    def centering_fingerprint(self, centering) -> int:
        c = np.ascontiguousarray(centering, dtype=np.float64)
        out = C.c_uint64(0)
        self._check(self.lib.chor_centering_fingerprint(c.ctypes.data, C.byref(out)), "centering_fingerprint")
        return out.value

    def save_code_cache(self, params, centering_fp: int, shorts, longs, path):
        p = self._fp(params)
        s = np.ascontiguousarray(shorts, dtype=np.uint32)
        l = np.ascontiguousarray(longs, dtype=np.uint64)
        self._check(self.lib.chor_save_code_cache(C.byref(p), C.c_uint64(centering_fp), s.ctypes.data, l.ctypes.data,
                                                  len(l.reshape(-1, 2)), str(path).encode()), "save_code_cache")

    def load_code_cache(self, path, expected, expected_fp: int, capacity: int):
        """Returns (shorts, longs, fault, fault_offset); fault 0 = ok, 1..5 FeatureFileFault+1, 6 mismatch."""
        p = self._fp(expected)
        shorts = np.zeros((max(capacity, 1), expected.table_count), dtype=np.uint32)
        longs = np.zeros((max(capacity, 1), 2), dtype=np.uint64)
        cnt, fault, off = C.c_uint32(0), C.c_int(0), C.c_uint64(0)
        rc = self.lib.chor_load_code_cache(str(path).encode(), C.byref(p), C.c_uint64(expected_fp), capacity,
                                           shorts.ctypes.data, longs.ctypes.data, C.byref(cnt), C.byref(fault),
                                           C.byref(off))
        if rc == 3 and fault.value == 0:
            raise MemoryError("capacity")
        return shorts[: cnt.value], longs[: cnt.value], fault.value, off.value

    def plan_exhaustive(self, image_count: int, block_images: int, blocks_per_group: int):
        pairs = np.zeros((max(image_count * (image_count - 1) // 2, 1), 2), dtype=np.uint32)
        sizes = np.zeros(max(image_count * image_count, 4), dtype=np.uint32)
        n, nt = C.c_uint64(0), C.c_uint32(0)
        self._check(self.lib.chor_plan_exhaustive(image_count, block_images, blocks_per_group, pairs.ctypes.data,
                                                  C.byref(n), sizes.ctypes.data, C.byref(nt)), "plan_exhaustive")
        return pairs[: n.value].copy(), sizes[: nt.value].copy()

    def plan_guided(self, image_count: int, block_images: int, blocks_per_group: int, accepted):
        acc = np.ascontiguousarray(accepted, dtype=np.uint32).reshape(-1, 2)
        pairs = np.zeros((max(len(acc), 1), 2), dtype=np.uint32)
        sizes = np.zeros(max(len(acc), 4), dtype=np.uint32)
        n, nt = C.c_uint64(0), C.c_uint32(0)
        self._check(self.lib.chor_plan_guided(image_count, block_images, blocks_per_group, acc.ctypes.data, C.c_uint64(len(acc)),
                                              pairs.ctypes.data, C.byref(n), sizes.ctypes.data, C.byref(nt)), "plan_guided")
        return pairs[: n.value].copy(), sizes[: nt.value].copy()

    def plan_task_blocks(self, image_count: int, block_images: int, blocks_per_group: int, accepted=None):
        """(ntasks, 4) u32: group_a, group_b, block_a, block_b of every PlanTask."""
        acc = None if accepted is None else np.ascontiguousarray(accepted, dtype=np.uint32).reshape(-1, 2)
        nt = C.c_uint32(0)
        cap = image_count * image_count + 4
        out = np.zeros((cap, 4), dtype=np.uint32)
        self._check(self.lib.chor_plan_task_blocks(image_count, block_images, blocks_per_group, 0 if acc is None else 1,
                                                   None if acc is None or not len(acc) else acc.ctypes.data,
                                                   C.c_uint64(0 if acc is None else len(acc)), out.ctypes.data, C.byref(nt)),
                    "plan_task_blocks")
        return out[: nt.value].copy()

    def simulate_residency(self, image_count: int, block_images: int, blocks_per_group: int, mode: int, accepted=None):
        """(nactions, 4) u32: kind, level, id, prefetch (simulate_residency over the plan's residency tasks)."""
        acc = None if accepted is None else np.ascontiguousarray(accepted, dtype=np.uint32).reshape(-1, 2)
        args = (image_count, block_images, blocks_per_group, mode, 0 if acc is None else 1,
                None if acc is None or not len(acc) else acc.ctypes.data, C.c_uint64(0 if acc is None else len(acc)))
        n = C.c_uint64(0)
        self._check(self.lib.chor_simulate_residency(*args, None, C.c_uint64(0), C.byref(n)), "simulate_residency")
        out = np.zeros((max(n.value, 1), 4), dtype=np.uint32)
        self._check(self.lib.chor_simulate_residency(*args, out.ctypes.data, C.c_uint64(n.value), C.byref(n)), "simulate_residency")
        return out[: n.value].copy()

    def auto_partition_sizing(self, mean_image_bytes: int, memory_budget_bytes: int):
        a, b = C.c_uint32(0), C.c_uint32(0)
        self._check(self.lib.chor_auto_partition_sizing(C.c_uint64(mean_image_bytes), C.c_uint64(memory_budget_bytes),
                                                        C.byref(a), C.byref(b)), "auto_partition_sizing")
        return a.value, b.value

    def time_match_pairs(self, params, cfg, descs, shorts, longs, pairs, threads: int):
        """descs/shorts/longs: lists of per-image arrays.  Returns (seconds, total matches, records checksum):
        the checksum is the order-independent one the GPU compaction kernel reports (stats["records_checksum"])."""
        p, c = self._fp(params), self._cfg(cfg)
        k = len(descs)
        keep = []
        dptr = (C.c_void_p * k)()
        sptr = (C.c_void_p * k)()
        lptr = (C.c_void_p * k)()
        counts = np.zeros(k, dtype=np.uint32)
        for i in range(k):
            d = np.ascontiguousarray(descs[i], dtype=np.uint8)
            s = np.ascontiguousarray(shorts[i], dtype=np.uint32)
            l = np.ascontiguousarray(longs[i], dtype=np.uint64)
            keep += [d, s, l]
            dptr[i], sptr[i], lptr[i] = d.ctypes.data, s.ctypes.data, l.ctypes.data
            counts[i] = d.size // 128
        pr = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
        sec = C.c_double(0)
        tot = C.c_uint64(0)
        csum = C.c_uint64(0)
        self._check(self.lib.chor_time_match_pairs(C.byref(p), C.byref(c), dptr, counts.ctypes.data, sptr, lptr,
                                                   pr.ctypes.data, len(pr), threads, C.byref(sec), C.byref(tot), C.byref(csum)),
                    "time_match_pairs")
        return sec.value, tot.value, csum.value


def restatement() -> Oracle:
    if not RESTATEMENT.exists():
        build_oracle(ref=False)
    return Oracle(RESTATEMENT)


def reference() -> Oracle | None:
    """The compiled reference, or None where it was never built (it cannot be built on the GPU box)."""
    return Oracle(REFERENCE) if REFERENCE.exists() else None


def best() -> Oracle:
    return reference() or restatement()
