"""ctypes binding of libchgpu.so (include/chgpu.h).  There is no fallback: a missing library or a
missing CUDA device raises."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libchgpu.so"
SYNTH_PATH = PKG / "libchsynth.so"

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)

OK, EINVAL, ELOGIC, ECUDA, ENOMEM, EUNSUPPORTED, EFORMAT, ENOTFOUND, EMISMATCH = range(9)


class FamilyParamsC(C.Structure):
    _fields_ = [("short_bits", C.c_uint32), ("long_bits", C.c_uint32), ("table_count", C.c_uint32),
                ("seed", C.c_uint64)]


class MatchCfgC(C.Structure):
    _fields_ = [("top_k", C.c_uint32), ("hamming_threshold", C.c_uint32), ("ratio", C.c_double),
                ("min_candidates_for_ratio", C.c_uint32), ("reduce_rounds", C.c_int32)]


class MatchRecordC(C.Structure):
    _fields_ = [("query_index", C.c_uint32), ("train_index", C.c_uint32), ("distance_sq", C.c_double)]


class MatchStatsC(C.Structure):
    _fields_ = [("pairs", C.c_uint64), ("matches", C.c_uint64), ("raw_candidates", C.c_uint64),
                ("verified_queries", C.c_uint64), ("distances", C.c_uint64), ("query_points", C.c_uint64),
                ("train_points", C.c_uint64), ("records_checksum", C.c_uint64),
                ("match_launches", C.c_uint32), ("total_launches", C.c_uint32),
                ("match_kernel_ms", C.c_float), ("total_ms", C.c_float)]

    def as_dict(self) -> dict:
        return {n: getattr(self, n) for n, _ in self._fields_}


class FileResultC(C.Structure):
    _fields_ = [("status", C.c_int32), ("fault", C.c_int32), ("fault_offset", C.c_uint64), ("count", C.c_uint32),
                ("reserved", C.c_uint32)]


class LoadStatsC(C.Structure):
    _fields_ = [("files_ok", C.c_uint64), ("files_failed", C.c_uint64), ("bytes_read", C.c_uint64), ("points", C.c_uint64),
                ("read_seconds", C.c_double), ("wall_seconds", C.c_double)]

    def as_dict(self) -> dict:
        return {n: getattr(self, n) for n, _ in self._fields_}


class SinkStatsC(C.Structure):
    _fields_ = [("files_written", C.c_uint64), ("files_failed", C.c_uint64), ("records", C.c_uint64), ("bytes", C.c_uint64),
                ("busy_seconds", C.c_double), ("wall_seconds", C.c_double)]

    def as_dict(self) -> dict:
        return {n: getattr(self, n) for n, _ in self._fields_}


class HashStatsC(C.Structure):
    _fields_ = [("undecided_dots", C.c_uint64), ("flipped_bits", C.c_uint64), ("overflowed_batches", C.c_uint64),
                ("filter_active", C.c_int32), ("reserved", C.c_int32)]

    def as_dict(self) -> dict:
        return {n: getattr(self, n) for n, _ in self._fields_ if n != "reserved"}


class DevicePropsC(C.Structure):
    _fields_ = [("name", C.c_char * 64), ("sm_count", C.c_int), ("cc_major", C.c_int), ("cc_minor", C.c_int),
                ("total_mem", C.c_size_t), ("free_mem", C.c_size_t), ("smem_per_block_optin", C.c_size_t)]


class PlanTaskC(C.Structure):
    _fields_ = [("group_a", C.c_uint32), ("group_b", C.c_uint32), ("block_a", C.c_uint32), ("block_b", C.c_uint32),
                ("first_pair", C.c_uint64), ("npairs", C.c_uint64)]


class ResidencyActionC(C.Structure):
    _fields_ = [("kind", C.c_uint32), ("level", C.c_uint32), ("id", C.c_uint32), ("prefetch", C.c_uint32)]


class StreamedStatsC(C.Structure):
    _fields_ = [("tasks", C.c_uint64), ("pairs", C.c_uint64), ("pairs_skipped", C.c_uint64), ("matches", C.c_uint64),
                ("block_loads", C.c_uint64), ("block_evictions", C.c_uint64), ("group_loads", C.c_uint64),
                ("group_evictions", C.c_uint64), ("images_loaded", C.c_uint64), ("bytes_read", C.c_uint64),
                ("background_block_loads", C.c_uint64),
                ("max_resident_blocks", C.c_uint32), ("max_resident_groups", C.c_uint32),
                ("load_seconds", C.c_double), ("hash_seconds", C.c_double), ("match_seconds", C.c_double),
                ("wall_seconds", C.c_double), ("evict_seconds", C.c_double), ("hint_seconds", C.c_double)]

    def as_dict(self) -> dict:
        return {n: getattr(self, n) for n, _ in self._fields_}


SINK_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, C.c_uint32, u64p, C.POINTER(MatchRecordC))

PLAN_SINK_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, u32p, C.c_uint32, u64p, C.POINTER(MatchRecordC))

# name -> (restype, argtypes); every symbol include/chgpu.h declares
SIGNATURES = {
    "chgpu_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "chgpu_destroy": (None, [C.c_void_p]),
    "chgpu_last_error": (C.c_char_p, [C.c_void_p]),
    "chgpu_status_name": (C.c_char_p, [C.c_int]),
    "chgpu_get_device_props": (C.c_int, [C.c_void_p, C.POINTER(DevicePropsC)]),
    "chgpu_sync": (C.c_int, [C.c_void_p]),
    "chgpu_set_sub_batch_queries": (C.c_int, [C.c_void_p, C.c_uint64]),
    "chgpu_set_join": (C.c_int, [C.c_void_p, C.c_int, C.c_uint32]),
    "chgpu_image_device_bytes": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint64)]),
    "chgpu_host_alloc": (C.c_int, [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "chgpu_host_free": (C.c_int, [C.c_void_p, C.c_void_p]),
    "chgpu_family_generate": (C.c_int, [C.POINTER(FamilyParamsC), f64p, f64p]),
    "chgpu_set_family": (C.c_int, [C.c_void_p, C.POINTER(FamilyParamsC), f64p, f64p]),
    "chgpu_centering_reset": (C.c_int, [C.c_void_p]),
    "chgpu_centering_add_image": (C.c_int, [C.c_void_p, C.c_uint32]),
    "chgpu_centering_add_images": (C.c_int, [C.c_void_p, u32p, C.c_uint32]),
    "chgpu_centering_get_sums": (C.c_int, [C.c_void_p, u64p, u64p]),
    "chgpu_centering_add_sums": (C.c_int, [C.c_void_p, u64p, C.c_uint64]),
    "chgpu_centering_apply": (C.c_int, [C.c_void_p, f64p]),
    "chgpu_set_centering": (C.c_int, [C.c_void_p, f64p]),
    "chgpu_upload_image": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]),
    "chgpu_upload_images": (C.c_int, [C.c_void_p, u32p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]),
    "chgpu_upload_chft": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_size_t, u32p,
                                    C.POINTER(C.c_int), u64p]),
    "chgpu_load_chft_files": (C.c_int, [C.c_void_p, C.POINTER(C.c_char_p), u32p, C.c_uint32, C.c_uint32, C.c_int,
                                        C.POINTER(FileResultC), C.POINTER(LoadStatsC)]),
    "chgpu_load_chft_files_begin": (C.c_int, [C.c_void_p, C.POINTER(C.c_char_p), u32p, C.c_uint32, C.c_uint32, C.c_int]),
    "chgpu_load_chft_files_end": (C.c_int, [C.c_void_p, C.POINTER(FileResultC), C.POINTER(LoadStatsC)]),
    "chgpu_evict_image": (C.c_int, [C.c_void_p, C.c_uint32]),
    "chgpu_evict_images": (C.c_int, [C.c_void_p, u32p, C.c_uint32]),
    "chgpu_image_points": (C.c_int, [C.c_void_p, C.c_uint32, u32p]),
    "chgpu_download_descriptors": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p]),
    "chgpu_set_hash_mode": (C.c_int, [C.c_void_p, C.c_int]),
    "chgpu_get_hash_stats": (C.c_int, [C.c_void_p, C.POINTER(HashStatsC)]),
    "chgpu_hash_images": (C.c_int, [C.c_void_p, u32p, C.c_uint32, C.c_int]),
    "chgpu_download_codes": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p]),
    "chgpu_upload_codes": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p]),
    "chgpu_download_bucket_index": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p]),
    "chgpu_download_sorted_index": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p]),
    "chgpu_pair_candidates": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint64, u64p]),
    "chgpu_match_pair_lists": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(MatchCfgC), C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_uint64, u64p, C.POINTER(MatchStatsC)]),
    "chgpu_centering_fingerprint": (C.c_uint64, [f64p]),
    "chgpu_save_code_cache": (C.c_int, [C.c_char_p, C.POINTER(FamilyParamsC), C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p]),
    "chgpu_read_code_cache_header": (C.c_int, [C.c_char_p, C.POINTER(FamilyParamsC), u64p, u32p]),
    "chgpu_load_code_cache": (C.c_int, [C.c_char_p, C.POINTER(FamilyParamsC), C.c_uint64, C.c_uint32, u32p, C.c_void_p,
                                        C.c_void_p, C.POINTER(C.c_int), u64p]),
    "chgpu_save_centering_file": (C.c_int, [C.c_char_p, C.POINTER(FamilyParamsC), f64p]),
    "chgpu_load_centering_file": (C.c_int, [C.c_char_p, C.POINTER(FamilyParamsC), f64p]),
    "chgpu_image_save_code_cache": (C.c_int, [C.c_void_p, C.c_uint32, C.c_char_p]),
    "chgpu_image_load_code_cache": (C.c_int, [C.c_void_p, C.c_uint32, C.c_char_p, C.POINTER(C.c_int), u64p]),
    "chgpu_match_pairs": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.POINTER(MatchCfgC), C.c_void_p,
                                    C.c_void_p, C.c_uint64, u64p, C.POINTER(MatchStatsC)]),
    "chgpu_match_pairs_stream": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.POINTER(MatchCfgC), SINK_FN,
                                           C.c_void_p, C.POINTER(MatchStatsC)]),
    "chgpu_match_pairs_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.POINTER(MatchCfgC),
                                           C.POINTER(MatchStatsC)]),
    "chgpu_match_pairs_guided": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.POINTER(MatchCfgC), C.c_void_p, C.c_double,
                                           C.c_void_p, C.c_void_p, C.c_uint64, u64p, C.POINTER(MatchStatsC)]),
    "chgpu_match_pairs_guided_stream": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.POINTER(MatchCfgC), C.c_void_p,
                                                  C.c_double, SINK_FN, C.c_void_p, C.POINTER(MatchStatsC)]),
    "chgpu_debug_ranked_guided": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(MatchCfgC), C.c_void_p, C.c_double,
                                            C.c_void_p, C.c_void_p]),
    "chgpu_debug_ranked": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(MatchCfgC), C.c_void_p,
                                     C.c_void_p]),
    "chgpu_save_matches": (C.c_int, [C.c_char_p, C.c_char_p, C.c_void_p, C.c_uint32, C.c_char_p]),
    "chgpu_sink_open": (C.c_int, [C.c_char_p, C.POINTER(C.c_char_p), C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p)]),
    "chgpu_sink_accept": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p]),
    "chgpu_sink_close": (C.c_int, [C.c_void_p, C.POINTER(SinkStatsC)]),
    "chgpu_match_pairs_to_files": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32, C.POINTER(MatchCfgC), C.c_void_p,
                                             C.POINTER(MatchStatsC)]),
    "chgpu_pair_file_name": (None, [C.c_uint32, C.c_uint32, C.c_char_p]),
    "chgpu_plan_exhaustive": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p, u64p]),
    "chgpu_plan_guided": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, u32p, C.c_uint64, u32p, u64p]),
    "chgpu_shard_range": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint32, u64p, u64p]),
    "chgpu_pair_weight": (C.c_uint64, [C.c_uint32, C.c_uint32]),
    "chgpu_shard_pairs_weighted": (C.c_int, [u32p, C.c_uint64, u32p, C.c_uint32, C.c_uint32, u64p, u64p]),
    "chgpu_plan_tasks": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint64, C.POINTER(PlanTaskC), u32p]),
    "chgpu_hashing_tasks": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(PlanTaskC), u32p]),
    "chgpu_simulate_residency": (C.c_int, [C.POINTER(PlanTaskC), C.c_uint32, C.c_int, C.c_uint32, C.c_uint32,
                                           C.POINTER(ResidencyActionC), C.c_uint64, u64p]),
    "chgpu_auto_partition_sizing": (None, [C.c_uint64, C.c_uint64, u32p, u32p]),
    "chgpu_partition_sizing_for_device": (None, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32,
                                                 u32p, u32p]),
    "chgpu_order_tasks_for_reuse": (C.c_int, [C.POINTER(PlanTaskC), C.c_uint32, C.c_uint32, u32p]),
    "chgpu_shard_tasks": (C.c_int, [C.POINTER(PlanTaskC), u32p, C.c_uint32, C.c_uint32, u32p]),
    "chgpu_shard_tasks_weighted": (C.c_int, [C.POINTER(PlanTaskC), u32p, C.c_uint32, u64p, C.c_uint32, u32p]),
    "chgpu_task_weights": (C.c_int, [C.POINTER(PlanTaskC), C.c_uint32, u32p, C.c_uint64, u32p, C.c_uint32, u64p]),
    "chgpu_match_plan_streamed": (C.c_int, [C.c_void_p, C.POINTER(C.c_char_p), C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                            C.c_uint32, C.c_int, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint64, C.POINTER(MatchCfgC), C.c_uint32, PLAN_SINK_FN,
                                            C.c_void_p, C.POINTER(FileResultC), C.POINTER(StreamedStatsC)]),
    "chgpu_centering_pass_files": (C.c_int, [C.c_void_p, C.POINTER(C.c_char_p), C.c_uint32, C.c_uint32, C.c_uint32,
                                             C.POINTER(FileResultC), f64p]),
}

_lib = None
_synth = None


def load() -> C.CDLL:
    """Loads libchgpu.so and binds every exported entry point; raises if it is absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1805_08995_b200.build` "
                "(the CUDA library is mandatory, there is no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)  # AttributeError if the header and the library disagree
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def load_synth() -> C.CDLL:
    global _synth
    if _synth is None:
        if not SYNTH_PATH.exists():
            raise RuntimeError(f"{SYNTH_PATH} is missing: run `python -m paper_1805_08995_b200.build`")
        lib = C.CDLL(str(SYNTH_PATH))
        lib.chsynth_dataset.restype = C.c_int
        lib.chsynth_dataset.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, C.c_double,
                                        C.c_int, C.c_uint32, C.c_void_p]
        _synth = lib
    return _synth
