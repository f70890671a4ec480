"""B200-native Cascade Hashing matcher (hot path of arXiv 1805.08995).

Product code: csrc/ (sm_100a CUDA kernels + C ABI, include/chgpu.h) and the C++ facade
include/cashash_b200/cashash.hpp.  `api` is the Python harness tests and bench.py use to drive
the same C ABI.  Importing this package never falls back to a CPU path.
"""
from .api import (  # noqa: F401
    BucketIndex, CudaError, FamilyParams, FeatureFileError, HashFamily, ImageCodes, LogicError, MatchConfig,
    Matcher, RECORD_DTYPE, UnsupportedError, build_hash_family, compute_codes, match_pair, pair_file_name,
    plan_exhaustive, plan_guided, save_matches, set_centering, shard_range,
    CacheMismatchError, centering_fingerprint, load_centering_file, load_code_cache, read_code_cache_header,
    save_centering_file, save_code_cache, MatchFileSink,
    plan_tasks, hashing_tasks, simulate_residency, auto_partition_sizing, partition_sizing_for_device,
    TASK_DTYPE, ACTION_DTYPE, order_tasks_for_reuse, ORDER_REFERENCE, ORDER_REUSE, shard_tasks,
    shard_pairs_weighted, task_weights, pair_weight,
)
from .synth import make_dataset  # noqa: F401
