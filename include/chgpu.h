/*
 * chgpu.h — C ABI of libchgpu.so, the B200 (sm_100a) Cascade Hashing matcher.
 *
 * This is the drop-in boundary for the reference's matching path.  The reference has no FFI
 * layer: its boundary is the C++ library API in namespace cashash (static lib `cashash`,
 * /root/reference/proj/src/CMakeLists.txt:1-13).  Every entry point below names the reference
 * interface it replaces (paths relative to /root/reference/proj).  The C++ facade that restores
 * the reference's signatures on top of this ABI is include/cashash_b200/cashash.hpp.
 *
 * Conventions
 *   - plain pointers and sizes only; all pointers are HOST pointers unless stated otherwise;
 *   - every call returns a chgpu_status; chgpu_last_error(ctx) gives the message;
 *   - one context per GPU; every call that takes a context holds the context's mutex for its duration, so calls
 *     from several threads on one context are safe and serialised (a sink callback runs under it and may call
 *     back into the same context from the same thread);
 *   - there is NO CPU fallback: without a CUDA device chgpu_create fails with CHGPU_ECUDA.
 *
 * Supported parameter envelope on the device path (CHGPU_EUNSUPPORTED outside it):
 *   short_bits m <= 32 (the reference's own limit, hashing.cpp:30-36), table_count L <= 8,
 *   long_bits n <= 128, any top_k >= 2, points per image <= 65,536.
 * The tuned kernels cover m <= 12 and top_k <= 32; beyond that (m = 13..32: sparse bucket index,
 * top_k > 32, candidate lists edited by a host callback) the same calls run through the general
 * kernels of csrc/general_kernels.cuh — same results, not tuned.
 */
#ifndef CHGPU_H
#define CHGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct chgpu_ctx chgpu_ctx;

typedef enum chgpu_status {
    CHGPU_OK = 0,
    CHGPU_EINVAL = 1,       /* reference: std::invalid_argument */
    CHGPU_ELOGIC = 2,       /* reference: std::logic_error (e.g. centering not set, hashing.cpp:131) */
    CHGPU_ECUDA = 3,        /* CUDA runtime failure / no device */
    CHGPU_ENOMEM = 4,
    CHGPU_EUNSUPPORTED = 5, /* outside the envelope above */
    CHGPU_EFORMAT = 6,      /* reference: FeatureFileError (feature_io.hpp:61-80) */
    CHGPU_ENOTFOUND = 7,    /* unknown image id / no such cache file */
    CHGPU_EMISMATCH = 8     /* reference: std::runtime_error "code cache parameters mismatch active config" */
} chgpu_status;

/* hashing.hpp:45-52 FamilyParams */
typedef struct chgpu_family_params {
    uint32_t short_bits;  /* m, default 8   */
    uint32_t long_bits;   /* n, default 128 */
    uint32_t table_count; /* L, default 6   */
    uint64_t seed;        /* default 1      */
} chgpu_family_params;

/* matcher.hpp:14-23 MatchConfig */
typedef struct chgpu_match_cfg {
    uint32_t top_k;                    /* default 10  */
    uint32_t hamming_threshold;        /* default 40  */
    double ratio;                      /* default 0.8 */
    uint32_t min_candidates_for_ratio; /* default 2   */
    int32_t reduce_rounds;             /* default 3; validated, exact distances do not depend on it */
} chgpu_match_cfg;

/* feature_io.hpp:51-57 MatchRecord — identical 16-byte layout. */
typedef struct chgpu_match_record {
    uint32_t query_index;
    uint32_t train_index;
    double distance_sq;
} chgpu_match_record;

/* feature_io.hpp:53-59 FeatureFileFault */
typedef enum chgpu_file_fault {
    CHGPU_FAULT_NONE = 0,
    CHGPU_FAULT_MISSING_FILE = 1,
    CHGPU_FAULT_BAD_MAGIC = 2,
    CHGPU_FAULT_BAD_VERSION = 3,
    CHGPU_FAULT_TRUNCATED = 4,
    CHGPU_FAULT_UNWRITABLE = 5
} chgpu_file_fault;

/* Counters and timings of one chgpu_match_pairs* call (device-side event timing on the
 * library's own compute stream). */
typedef struct chgpu_match_stats {
    uint64_t pairs;
    uint64_t matches;           /* Mx */
    uint64_t raw_candidates;    /* R */
    uint64_t verified_queries;  /* Vq */
    uint64_t distances;         /* V  */
    uint64_t query_points;      /* sum of Nq over pairs */
    uint64_t train_points;      /* sum of Nt over pairs */
    uint64_t records_checksum;  /* order-independent FNV-style checksum of all records */
    uint32_t match_launches;    /* launches of the match kernel */
    uint32_t total_launches;    /* all kernels launched by the call */
    float match_kernel_ms;      /* sum of match-kernel durations (CUDA events) */
    float total_ms;             /* first launch -> last result resident (device) or delivered (host) */
} chgpu_match_stats;

typedef struct chgpu_device_props {
    char name[64];
    int sm_count;
    int cc_major, cc_minor;
    size_t total_mem, free_mem;
    size_t smem_per_block_optin;
} chgpu_device_props;

/* ---- context --------------------------------------------------------------------------- */
chgpu_status chgpu_create(int device, chgpu_ctx** out);
void chgpu_destroy(chgpu_ctx* ctx);
/* Message of the calling thread's last failed call on this context (the pointer stays valid until that thread's next
 * failing call or next chgpu_last_error). */
const char* chgpu_last_error(const chgpu_ctx* ctx);
const char* chgpu_status_name(chgpu_status s);
chgpu_status chgpu_get_device_props(chgpu_ctx* ctx, chgpu_device_props* out);
chgpu_status chgpu_sync(chgpu_ctx* ctx);
/* Tuning knob: upper bound on the sum of query points per sub-batch (one match-kernel launch);
 * 0 restores the default (32 Mi).  Results never depend on it. */
chgpu_status chgpu_set_sub_batch_queries(chgpu_ctx* ctx, uint64_t max_queries);
/* The tensor-core Hamming pass in front of the match kernel (csrc/join_kernels.cuh; no reference counterpart: it computes
 * which queries of a pair have a candidate within hamming_threshold, matcher.cpp:164-175, the match kernel then visits those
 * only; results are the same records).  enabled = 0 switches it off; min_points_per_bucket = the average bucket occupancy
 * (points >> short_bits, both images of a pair) from which a sub-batch takes it (default 20; 0 = always, what the parity
 * tests use).  CHGPU_NO_JOIN=1 / CHGPU_JOIN_MIN_BUCKET=n set the same for new contexts. */
chgpu_status chgpu_set_join(chgpu_ctx* ctx, int enabled, uint32_t min_points_per_bucket);
/* Pinned host memory for zero-staging uploads / result sinks. */
chgpu_status chgpu_host_alloc(chgpu_ctx* ctx, size_t bytes, void** out);
chgpu_status chgpu_host_free(chgpu_ctx* ctx, void* p);

/* ---- hash family ----------------------------------------------------------------------- */
/* Replaces build_hash_family (hashing.hpp:74, hashing.cpp:38-50): host-side, deterministic.
 * short_planes: L*m*128 doubles [table*m+bit][128]; long_planes: n*128 doubles. */
chgpu_status chgpu_family_generate(const chgpu_family_params* p, double* short_planes, double* long_planes);
/* Installs a family (planes as produced above, or by the reference) on the device. */
chgpu_status chgpu_set_family(chgpu_ctx* ctx, const chgpu_family_params* p,
                              const double* short_planes, const double* long_planes);
/* Replaces set_centering / CenteringAccumulator (hashing.hpp:78,166-172; hashing.cpp:52-70). */
chgpu_status chgpu_centering_reset(chgpu_ctx* ctx);
chgpu_status chgpu_centering_add_image(chgpu_ctx* ctx, uint32_t image_id);
/* Batch form of chgpu_centering_add_image: one launch over the listed resident images. */
chgpu_status chgpu_centering_add_images(chgpu_ctx* ctx, const uint32_t* image_ids, uint32_t count);
chgpu_status chgpu_centering_get_sums(chgpu_ctx* ctx, uint64_t* sums128, uint64_t* count);
chgpu_status chgpu_centering_add_sums(chgpu_ctx* ctx, const uint64_t* sums128, uint64_t count);
chgpu_status chgpu_centering_apply(chgpu_ctx* ctx, double* centering128_out /* nullable */);
chgpu_status chgpu_set_centering(chgpu_ctx* ctx, const double* centering128);

/* ---- descriptor load ------------------------------------------------------------------- */
/* Replaces the arena load of a FeatureSet (engine.cpp:394-412).  desc: n x 128 u8 row-major;
 * keypoints: n x 4 f32 (x, y, scale, orientation) or NULL.  Re-uploading an id replaces it. */
chgpu_status chgpu_upload_image(chgpu_ctx* ctx, uint32_t image_id, uint32_t n,
                                const uint8_t* desc, const float* keypoints);
/* Batch form for `count` images of n points each, stored back to back (desc: count x n x 128 u8, keypoints:
 * count x n x 4 f32 or NULL): from pinned memory the copies are issued back to back and drained once. */
chgpu_status chgpu_upload_images(chgpu_ctx* ctx, const uint32_t* image_ids, uint32_t count, uint32_t n,
                                 const uint8_t* desc, const float* keypoints);
/* Replaces load_features / parse_features_blob (feature_io.cpp:65-106, engine.cpp:458-488) for a
 * CHFT blob already in host memory: header checked on the host, the 144-byte AoS records are
 * split into SoA on the device.  On CHGPU_EFORMAT *fault / *fault_offset carry the reference's
 * FeatureFileFault class and byte offset. */
chgpu_status chgpu_upload_chft(chgpu_ctx* ctx, uint32_t image_id, const void* blob, size_t nbytes,
                               uint32_t* count_out, chgpu_file_fault* fault, uint64_t* fault_offset);
/* Disk -> pinned host -> HBM streaming loader: the paper's Disk-Memory-GPU exchange and the
 * reference's loader thread (ResidencyDriver::load_group / load_block, engine.cpp:328-412), rebuilt as
 * `io_threads` reader threads filling a ring of pinned staging slots while the calling thread validates each
 * header, issues cudaMemcpyAsync on the copy stream and the AoS->SoA split kernel on the compute stream; reads,
 * H2D copies and kernels of different files overlap.  Files are consumed in list order.  A file that cannot be
 * read or parsed is reported in results[i] (reference fault class + byte offset) and skipped, the rest of the
 * batch proceeds (engine.cpp:315-318).  accumulate_centering != 0 adds every loaded image to the running
 * centering sums (centering_pass, engine.cpp:545-559) on the fly. */
typedef struct chgpu_file_result {
    int32_t status;        /* chgpu_status of this file */
    int32_t fault;         /* chgpu_file_fault when status == CHGPU_EFORMAT */
    uint64_t fault_offset;
    uint32_t count;        /* points loaded */
    uint32_t reserved;
} chgpu_file_result;
typedef struct chgpu_load_stats {
    uint64_t files_ok, files_failed, bytes_read, points;
    double read_seconds;   /* summed over the reader threads */
    double wall_seconds;   /* first read issued -> last split kernel complete */
} chgpu_load_stats;
chgpu_status chgpu_load_chft_files(chgpu_ctx* ctx, const char* const* paths, const uint32_t* image_ids, uint32_t count,
                                   uint32_t io_threads, int accumulate_centering, chgpu_file_result* results,
                                   chgpu_load_stats* stats /* nullable */);
/* Background form of the loader, for overlapping the load of the NEXT block with the matching of the current task
 * (the two-line exchange of PAPER.md:73-94; the loader thread of engine.cpp:414-442).  _begin starts the reader
 * threads (paths and ids are copied) and returns at once; while the job is open every chgpu_match_pairs* call on
 * this context moves it forward wherever it would otherwise sleep on the device — files the readers have finished
 * are sent with cudaMemcpyAsync under the match kernels already launched and split behind them, all on the calling
 * thread (a context stays thread-compatible).  _end handles what is left, drains and reports per file
 * like chgpu_load_chft_files (results: count entries, nullable).  The images become usable after _end.  One job
 * per context; other loads are CHGPU_ELOGIC while it is open. */
chgpu_status chgpu_load_chft_files_begin(chgpu_ctx* ctx, const char* const* paths, const uint32_t* image_ids, uint32_t count,
                                         uint32_t io_threads, int accumulate_centering);
chgpu_status chgpu_load_chft_files_end(chgpu_ctx* ctx, chgpu_file_result* results /* nullable */,
                                       chgpu_load_stats* stats /* nullable */);
chgpu_status chgpu_evict_image(chgpu_ctx* ctx, uint32_t image_id);
/* Batch form (block eviction, engine.cpp:420-441): one drain of the streams for the whole list.  Ids that are not
 * resident are skipped and reported as CHGPU_ENOTFOUND after the rest has been released. */
chgpu_status chgpu_evict_images(chgpu_ctx* ctx, const uint32_t* image_ids, uint32_t count);
chgpu_status chgpu_image_points(chgpu_ctx* ctx, uint32_t image_id, uint32_t* n);
chgpu_status chgpu_download_descriptors(chgpu_ctx* ctx, uint32_t image_id, uint8_t* desc, float* keypoints);

/* ---- hash build ------------------------------------------------------------------------ */
/* Replaces compute_codes (hashing.hpp:131, hashing.cpp:130-149) + build_bucket_index
 * (matcher.hpp:43, matcher.cpp:27-51) for the listed images.  reduce_rounds = N_r in 0..7. */
chgpu_status chgpu_hash_images(chgpu_ctx* ctx, const uint32_t* image_ids, uint32_t count, int reduce_rounds);
/* How chgpu_hash_images evaluates the L*m + n hyperplane signs of a descriptor.  All modes give the reference's
 * bits exactly (compute_codes, hashing.cpp:130-149).
 *   TENSOR (default):   a filter on the tensor cores (tcgen05.mma kind::i8): the planes as three int8 limbs of a 23-bit
 *                       fixed-point value, exact s32 accumulators in tensor memory, an a-priori error bound in fp64; the
 *                       dots it cannot prove (|value| below the bound, ~7e-6 of them, ties included) are re-evaluated in
 *                       the reference's fp64 operation order (reduce_dot, hashing.hpp:24-43).
 *   FILTERED:           the same contract with an fp32 SIMT contraction (bound ~45x wider, ~1.5e-4 undecided).
 *   EXACT:              every dot in the reference's fp64 operation order.
 * Both filters fall back to EXACT by themselves for planes / centerings outside the bound's premises (non-finite or
 * huge values).  CHGPU_HASH_FP32=1 / CHGPU_HASH_EXACT=1 select FILTERED / EXACT for new contexts. */
typedef enum chgpu_hash_mode { CHGPU_HASH_FILTERED = 0, CHGPU_HASH_EXACT = 1, CHGPU_HASH_TENSOR = 2 } chgpu_hash_mode;
typedef struct chgpu_hash_stats {
    uint64_t undecided_dots;      /* dots the filter handed to the exact path (cumulative per context) */
    uint64_t flipped_bits;        /* of those, bits whose fp32 sign differed from the reference's */
    uint64_t overflowed_batches;  /* launches whose undecided queue overflowed and were recomputed in EXACT mode */
    int32_t filter_active;        /* 1 if the next chgpu_hash_images call will use the filter */
    int32_t reserved;
} chgpu_hash_stats;
chgpu_status chgpu_set_hash_mode(chgpu_ctx* ctx, chgpu_hash_mode mode);
chgpu_status chgpu_get_hash_stats(chgpu_ctx* ctx, chgpu_hash_stats* out);
/* shorts: n x L u32 [point*L+table]; longs: n x 2 u64 (ShortCodes / LongCode, hashing.hpp:80-96). */
chgpu_status chgpu_download_codes(chgpu_ctx* ctx, uint32_t image_id, uint32_t* shorts, uint64_t* longs);
/* Installs externally computed codes (e.g. a CHCC code cache, hashing.hpp:138-162) and builds buckets. */
chgpu_status chgpu_upload_codes(chgpu_ctx* ctx, uint32_t image_id, const uint32_t* shorts, const uint64_t* longs);
/* Dense CSR of the bucket index: offsets L*(2^m+1) u32, points L*n u32 (bucket-major, ascending id). */
chgpu_status chgpu_download_bucket_index(chgpu_ctx* ctx, uint32_t image_id, uint32_t* offsets, uint32_t* points);
/* The same index in the form build_bucket_index leaves it before grouping (matcher.cpp:34-37): per table the
 * points sorted by (short code, point id).  codes, points: L*n u32 each, table-major.  Works for every
 * short_bits (short_bits > 12 has no dense offset table: CHGPU_EUNSUPPORTED from the call above). */
chgpu_status chgpu_download_sorted_index(chgpu_ctx* ctx, uint32_t image_id, uint32_t* codes, uint32_t* points);

/* ---- code cache / centering files (interop with the CPU reference, resume) -------------- */
/* centering_fingerprint (hashing.cpp:151-162): FNV-1a over the 128 doubles' bytes. */
uint64_t chgpu_centering_fingerprint(const double* centering128);
/* save_code_cache (hashing.hpp:138-146, hashing.cpp:184-206): "CHCC", u32 version=1, m, n, L, u64 seed,
 * u64 centering fingerprint, u32 count, u32 reserved; count*L u32 short codes; count*2 u64 long words. */
chgpu_status chgpu_save_code_cache(const char* path, const chgpu_family_params* p, uint64_t centering_fp,
                                   uint32_t count, const uint32_t* shorts, const uint64_t* longs);
/* read_code_cache_header (hashing.cpp:208-226): CHGPU_ENOTFOUND for a missing file, foreign magic,
 * other version or short header (the reference returns false for all of these). */
chgpu_status chgpu_read_code_cache_header(const char* path, chgpu_family_params* p, uint64_t* centering_fp,
                                          uint32_t* count);
/* load_code_cache / parse_code_cache (hashing.cpp:228-272).  CHGPU_EFORMAT with *fault / *fault_offset as the
 * reference reports them (a payload cut short is reported at offset UINT64_MAX: the reference casts a failed
 * tellg()), CHGPU_EMISMATCH when the echoed parameters or fingerprint differ, CHGPU_ENOMEM (with *count set)
 * when capacity < count.  shorts: count*L u32, longs: count*2 u64. */
chgpu_status chgpu_load_code_cache(const char* path, const chgpu_family_params* expected, uint64_t expected_fp,
                                   uint32_t capacity, uint32_t* count, uint32_t* shorts, uint64_t* longs,
                                   chgpu_file_fault* fault, uint64_t* fault_offset);
/* Centering file "CHCV" (engine.cpp:522-541): magic, u32 version=1, m, n, L, u64 seed, 128 f64. */
chgpu_status chgpu_save_centering_file(const char* path, const chgpu_family_params* p, const double* centering128);
chgpu_status chgpu_load_centering_file(const char* path, chgpu_family_params* p, double* centering128);
/* Device conveniences: write the codes of a resident image as a CHCC cache (fingerprint of the context's
 * centering), or install a cache as the image's codes + bucket index (hash build skipped: the reference's
 * cache_is_current resume path, engine.cpp:575-582).  The image must be resident with the cache's count. */
chgpu_status chgpu_image_save_code_cache(chgpu_ctx* ctx, uint32_t image_id, const char* path);
chgpu_status chgpu_image_load_code_cache(chgpu_ctx* ctx, uint32_t image_id, const char* path,
                                         chgpu_file_fault* fault, uint64_t* fault_offset);

/* ---- match ----------------------------------------------------------------------------- */
/* Replaces match_pair over a pair list (matcher.hpp:98-100, matcher.cpp:141-203; pair list as in
 * PlanTask::pairs, scheduler.hpp:36-40).  pairs[2k] is the query image I, pairs[2k+1] the train
 * image J.  offsets (npairs+1) and records (capacity entries) are filled in pair order; records
 * of one pair are ascending in query_index, at most one per query.  If capacity is too small the
 * call returns CHGPU_ENOMEM and *total holds the required number of records. */
chgpu_status chgpu_match_pairs(chgpu_ctx* ctx, const uint32_t* pairs, uint32_t npairs,
                               const chgpu_match_cfg* cfg, uint64_t* offsets,
                               chgpu_match_record* records, uint64_t capacity, uint64_t* total,
                               chgpu_match_stats* stats /* nullable */);

/* Streaming form: the asynchronous sink contract of FileMatchSink::accept (engine.cpp:145-160).
 * The sink is called on the calling thread, in pair order, with pinned host memory that stays
 * valid until it returns; the next sub-batch is already computing on the device meanwhile.
 * offsets has npairs_chunk+1 entries relative to records.  A nonzero return aborts the call. */
typedef int (*chgpu_sink_fn)(void* user, uint32_t first_pair, uint32_t npairs_chunk,
                             const uint64_t* offsets, const chgpu_match_record* records);
chgpu_status chgpu_match_pairs_stream(chgpu_ctx* ctx, const uint32_t* pairs, uint32_t npairs,
                                      const chgpu_match_cfg* cfg, chgpu_sink_fn sink, void* user,
                                      chgpu_match_stats* stats /* nullable */);

/* Device-resident form used for kernel-only timing: results are compacted into device memory
 * and only the counters / checksum in stats come back. */
chgpu_status chgpu_match_pairs_device(chgpu_ctx* ctx, const uint32_t* pairs, uint32_t npairs,
                                      const chgpu_match_cfg* cfg, chgpu_match_stats* stats);

/* Epipolar-guided variant (guided_match_pair, geometry.hpp:86-89, geometry.cpp:234-250 — the only
 * CandidateFilter the reference ships, matcher.hpp:92-105).  fmats: npairs x 9 doubles, row-major fundamental
 * matrices mapping a query point of image I to its epipolar line in image J; between lookup and ranking the
 * candidates of a query are cut to those within band_px of the line l = F (x, y, 1)^T (keypoints as uploaded);
 * a degenerate line (a == b == 0) leaves that query unguided.  Estimating F (RANSAC) is the caller's business. */
chgpu_status chgpu_match_pairs_guided(chgpu_ctx* ctx, const uint32_t* pairs, uint32_t npairs,
                                      const chgpu_match_cfg* cfg, const double* fmats, double band_px,
                                      uint64_t* offsets, chgpu_match_record* records, uint64_t capacity,
                                      uint64_t* total, chgpu_match_stats* stats /* nullable */);
chgpu_status chgpu_match_pairs_guided_stream(chgpu_ctx* ctx, const uint32_t* pairs, uint32_t npairs,
                                             const chgpu_match_cfg* cfg, const double* fmats, double band_px,
                                             chgpu_sink_fn sink, void* user, chgpu_match_stats* stats /* nullable */);

/* match_pair_filtered with a HOST callback (matcher.hpp:92-105; hook matcher.cpp:172) in two device steps with the
 * caller's filter in between:
 *   1. chgpu_pair_candidates: the candidate list of every query of image_i in image_j — its L buckets concatenated,
 *      sorted, made unique (matcher.cpp:164-171).  offsets: n_i + 1 entries; candidates: capacity entries.  If the
 *      capacity is too small the call returns CHGPU_ENOMEM with *total = entries required and offsets filled
 *      (capacity 0 / candidates NULL is the sizing call).
 *   2. the caller edits the lists (the reference hands the filter a mutable vector: entries may be removed,
 *      reordered, repeated), then chgpu_match_pair_lists ranks and verifies from the lists as they are: Hamming
 *      ranking as a stable counting sort (ties keep the list order, fill_histogram matcher.cpp:68-84), threshold and
 *      re-rank rule (matcher.cpp:176-189), Euclidean verification (matcher.cpp:115-137).  Queries with an empty
 *      list produce nothing (matcher.cpp:173).  list_ids entries must be < n_j. */
chgpu_status chgpu_pair_candidates(chgpu_ctx* ctx, uint32_t image_i, uint32_t image_j, uint64_t* offsets,
                                   uint32_t* candidates /* nullable with capacity 0 */, uint64_t capacity, uint64_t* total);
chgpu_status chgpu_match_pair_lists(chgpu_ctx* ctx, uint32_t image_i, uint32_t image_j, const chgpu_match_cfg* cfg,
                                    const uint64_t* list_offsets, const uint32_t* list_ids, chgpu_match_record* records,
                                    uint64_t capacity, uint64_t* total, chgpu_match_stats* stats /* nullable */);

/* Parity hook: the ranked candidate list each query hands to verification (after the re-rank
 * fallback, matcher.cpp:176-189).  ranked: n_i*top_k u32, ranked_count: n_i u32. */
chgpu_status chgpu_debug_ranked(chgpu_ctx* ctx, uint32_t image_i, uint32_t image_j,
                                const chgpu_match_cfg* cfg, uint32_t* ranked, uint32_t* ranked_count);

chgpu_status chgpu_debug_ranked_guided(chgpu_ctx* ctx, uint32_t image_i, uint32_t image_j,
                                       const chgpu_match_cfg* cfg, const double* fmat, double band_px,
                                       uint32_t* ranked, uint32_t* ranked_count);

/* ---- match output ---------------------------------------------------------------------- */
/* Replaces save_matches (feature_io.hpp:106-107, feature_io.cpp:161-183): byte-identical text. */
chgpu_status chgpu_save_matches(const char* image_id_i, const char* image_id_j,
                                const chgpu_match_record* records, uint32_t count, const char* path);
/* pair_file_name (engine.cpp:724-728): "match_%06u_%06u.txt"; buf must hold 48 bytes. */
void chgpu_pair_file_name(uint32_t image_i, uint32_t image_j, char* buf);

/* Asynchronous batched match-file writer: the reference's FileMatchSink (engine.cpp:145-211: one writer thread,
 * one text file per pair) with `threads` writers and whole sub-batches as queue items.  Every pair (i, j) becomes
 * <dir>/match_%06u_%06u.txt with exactly the bytes save_matches writes (feature_io.cpp:161-183); the header line
 * carries image_names[i] / image_names[j] (NULL: the decimal image index).  accept() copies its arguments and
 * returns at once (it blocks only while max_queued_batches items are waiting); per-file failures are counted,
 * never fatal (engine.cpp:188-199).  close() drains the queue, joins the writers and frees the sink. */
typedef struct chgpu_sink chgpu_sink;
typedef struct chgpu_sink_stats {
    uint64_t files_written, files_failed, records, bytes;
    double busy_seconds;  /* summed over the writer threads */
    double wall_seconds;  /* open -> close */
} chgpu_sink_stats;
chgpu_status chgpu_sink_open(const char* dir, const char* const* image_names, uint32_t image_count, uint32_t threads,
                             uint32_t max_queued_batches, chgpu_sink** out);
chgpu_status chgpu_sink_accept(chgpu_sink* sink, const uint32_t* pairs /* 2 per pair */, uint32_t npairs,
                               const uint64_t* offsets /* npairs + 1, relative to records */,
                               const chgpu_match_record* records);
chgpu_status chgpu_sink_close(chgpu_sink* sink, chgpu_sink_stats* stats /* nullable */);
/* chgpu_match_pairs_stream with the writer above as its sink: match results go straight from the pinned result
 * buffers into the writer queue while the next sub-batch computes. */
chgpu_status chgpu_match_pairs_to_files(chgpu_ctx* ctx, const uint32_t* pairs, uint32_t npairs, const chgpu_match_cfg* cfg,
                                        chgpu_sink* sink, chgpu_match_stats* stats /* nullable */);

/* ---- pair lists ------------------------------------------------------------------------ */
/* Exhaustive pair list in the reference's locality order (plan_exhaustive, scheduler.cpp:99-142)
 * for image_count images in blocks of block_images, blocks_per_group blocks per group.
 * pairs_out holds image_count*(image_count-1) u32 (2 per pair). */
chgpu_status chgpu_plan_exhaustive(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group,
                                   uint32_t* pairs_out, uint64_t* npairs_out);
/* The same traversal restricted to the accepted pairs (plan_guided, scheduler.hpp:57-58, scheduler.cpp:144-164):
 * either order, duplicates collapse; a self pair or an index >= image_count is CHGPU_EINVAL (the reference throws
 * std::invalid_argument).  pairs_out holds 2 * accepted_count u32.  This is the pair-order scheduling for
 * arbitrary pair lists (e.g. a k-neighbour list): consecutive pairs share their images. */
chgpu_status chgpu_plan_guided(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group,
                               const uint32_t* accepted, uint64_t accepted_count, uint32_t* pairs_out, uint64_t* npairs_out);
/* Shard [0,npairs) for rank `rank` of `world`: contiguous ranges of the plan, so each GPU keeps
 * its train images hot (replaces assign_workers, scheduler.cpp:166-173). */
chgpu_status chgpu_shard_range(uint64_t npairs, uint32_t rank, uint32_t world, uint64_t* first, uint64_t* last);
/* The work model of one pair for load balancing: queries x (train points + a constant for the per-query
 * lookup / ranking overhead).  Candidates per query grow linearly with the train image, so a
 * 32K x 32K pair weighs ~16 x an 8K x 8K pair and ~1000 x a 1K x 1K one; pair COUNT balances only uniform datasets. */
uint64_t chgpu_pair_weight(uint32_t query_points, uint32_t train_points);
/* Work-balanced form of chgpu_shard_range for datasets of mixed image sizes: the pair list is cut into `shards`
 * contiguous ranges of about equal total chgpu_pair_weight.  points_per_image[i] = descriptors of image i
 * (every index in `pairs` must be < image_count).  first_out: shards + 1 positions; shard s owns
 * [first_out[s], first_out[s + 1]).  weights_out (nullable, `shards` entries) receives the weight of every shard. */
chgpu_status chgpu_shard_pairs_weighted(const uint32_t* pairs, uint64_t npairs, const uint32_t* points_per_image,
                                        uint32_t image_count, uint32_t shards, uint64_t* first_out, uint64_t* weights_out);

/* ---- block-pair tasks, residency schedule, out-of-core run -------------------------------- */
/* The tasks behind the flat pair lists above (PlanTask, scheduler.hpp:36-43): task t covers pairs
 * [first_pair, first_pair + npairs) of chgpu_plan_exhaustive (accepted == NULL) or chgpu_plan_guided (tasks left
 * without a pair are dropped, scheduler.cpp:161).  tasks_out may be NULL to count. */
typedef struct chgpu_plan_task {
    uint32_t group_a, group_b;  /* parent groups of the two blocks */
    uint32_t block_a, block_b;  /* block_a <= block_b; equal for the pairs inside one block */
    uint64_t first_pair, npairs;
} chgpu_plan_task;
chgpu_status chgpu_plan_tasks(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group,
                              const uint32_t* accepted /* nullable */, uint64_t accepted_count,
                              chgpu_plan_task* tasks_out /* nullable */, uint32_t* ntasks_out);
/* hashing_residency_tasks (scheduler.cpp:194-200): one task per block, in block order. */
chgpu_status chgpu_hashing_tasks(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group,
                                 chgpu_plan_task* tasks_out /* nullable */, uint32_t* ntasks_out);

/* The two-line load / prefetch state machine (step_residency / simulate_residency, scheduler.cpp:226-345) run
 * to completion over residency_tasks(plan) (scheduler.cpp:175-192).  Line 1 loads what the current task misses
 * (evicting the resident item used farthest in the future), line 2 prefetches the nearest future group / block into
 * free slots or over items needed strictly later, then the task begins and finishes.
 * group_slots / block_slots: residency limit per level; 0 selects the reference's (CHGPU_RESIDENCY_HASHING: 2,
 * CHGPU_RESIDENCY_MATCHING: 3, scheduler.hpp:70-72) and then the trace equals the reference's action for action.
 * Larger limits are what a 180 GB device wants; a limit below what one task needs is CHGPU_EINVAL (the reference
 * throws std::logic_error "current ... load blocked" at that point).
 * actions_out may be NULL to count; CHGPU_ENOMEM with *nactions_out set when capacity is too small. */
typedef enum chgpu_residency_mode { CHGPU_RESIDENCY_HASHING = 0, CHGPU_RESIDENCY_MATCHING = 1 } chgpu_residency_mode;
typedef enum chgpu_action_kind { CHGPU_ACT_LOAD = 0, CHGPU_ACT_EVICT = 1, CHGPU_ACT_BEGIN = 2, CHGPU_ACT_FINISH = 3 } chgpu_action_kind;
typedef enum chgpu_residency_level { CHGPU_LEVEL_GROUP = 0, CHGPU_LEVEL_BLOCK = 1 } chgpu_residency_level;
typedef struct chgpu_residency_action {
    uint32_t kind;      /* chgpu_action_kind */
    uint32_t level;     /* chgpu_residency_level; meaningful for Load / Evict */
    uint32_t id;        /* group / block id, or task index (Begin / Finish) */
    uint32_t prefetch;  /* Load issued ahead of need (line 2) */
} chgpu_residency_action;
chgpu_status chgpu_simulate_residency(const chgpu_plan_task* tasks, uint32_t ntasks, chgpu_residency_mode mode,
                                      uint32_t group_slots, uint32_t block_slots,
                                      chgpu_residency_action* actions_out /* nullable */, uint64_t capacity,
                                      uint64_t* nactions_out);
/* auto_partition_sizing (scheduler.cpp:347-359): the device holds a quarter of the budget, three units per level. */
void chgpu_auto_partition_sizing(uint64_t mean_image_bytes, uint64_t memory_budget_bytes, uint32_t* block_images,
                                 uint32_t* blocks_per_group);
/* The same rule with the numbers of this device: block_slots blocks share device_bytes (HBM left for images),
 * group_slots groups share host_bytes (page cache the read-ahead may occupy); device_image_bytes is what one image
 * occupies in HBM (descriptors, keypoints, codes, bucket index), file_image_bytes its CHFT file. */
/* What an image of n points occupies in this context's HBM arena under the installed family (descriptors, keypoints, codes,
 * bucket index, the bucket-sorted copies of the Hamming pass, tiles of a large image): the device_image_bytes of the rule below. */
chgpu_status chgpu_image_device_bytes(chgpu_ctx* ctx, uint32_t n, uint64_t* bytes);
void chgpu_partition_sizing_for_device(uint64_t device_image_bytes, uint64_t file_image_bytes, uint64_t device_bytes,
                                       uint64_t host_bytes, uint32_t block_slots, uint32_t group_slots,
                                       uint32_t* block_images, uint32_t* blocks_per_group);

/* Out-of-core run of a plan: the reference's execute_plan + ResidencyDriver (engine.cpp:252-456, :667-702) for
 * datasets that do not fit in HBM at once.  The residency trace above is replayed on the calling thread:
 *   Load group   read-ahead of the group's files into the host page cache (posix_fadvise WILLNEED; the pinned
 *                ring of chgpu_load_chft_files is the staging level under it),
 *   Load block   chgpu_load_chft_files of the block's files + chgpu_hash_images (hashing an 8K image costs 12 us,
 *                less than reading its CHCC cache back would),
 *   Evict block  chgpu_evict_image of its images;  Evict group: the pages are released (DONTNEED),
 *   Begin task   chgpu_match_pairs_stream over the task's pairs.  What the schedule prefetches between Begin and
 *                Finish of a task (its line 2) is opened as a background load (chgpu_load_chft_files_begin) before
 *                the match call and completed behind it, so the H2D copies of the next block run under the match
 *                kernels of the current one; CHGPU_STREAM_NO_OVERLAP=1 replays strictly in trace order (A/B).
 * Never more than block_slots blocks are resident; at the end everything the run loaded is evicted again.  The run
 * owns the context's image ids 0 .. image_count-1 (image id = index into paths).  Images whose file failed are
 * reported in file_results (image_count entries) and their pairs are skipped without output, like the reference's
 * invalid images (engine.cpp:799).  The family and the centering must be installed (chgpu_centering_pass_files).
 * The sink is called on the calling thread, in plan order, with the pairs of the chunk (2 u32 per pair), their
 * record offsets (npairs_chunk + 1, relative to records) and the records — the argument list of chgpu_sink_accept
 * behind the task index; a nonzero return aborts the run. */
typedef int (*chgpu_plan_sink_fn)(void* user, uint32_t task, const uint32_t* pairs, uint32_t npairs_chunk,
                                  const uint64_t* offsets, const chgpu_match_record* records);
typedef struct chgpu_streamed_stats {
    uint64_t tasks, pairs, pairs_skipped, matches;
    uint64_t block_loads, block_evictions, group_loads, group_evictions;
    uint64_t images_loaded, bytes_read;
    uint64_t background_block_loads; /* of block_loads: opened before a task's match call and completed behind it */
    uint32_t max_resident_blocks, max_resident_groups;
    double load_seconds, hash_seconds, match_seconds, wall_seconds;
    double evict_seconds, hint_seconds; /* block evictions; page-cache hints of the group level */
} chgpu_streamed_stats;
/* Task order of a streamed run.  REFERENCE: the plan's own order (scheduler.cpp:99-164).  REUSE: the same tasks in an
 * order chosen for descriptor reuse in HBM — always the pending task that needs the fewest block loads given what
 * is resident (ties: plan order), evicting the block with the fewest tasks left.  The reference's traversal is
 * built for all-pairs plans; on a banded pair list (k nearest neighbours) it comes back to blocks it has dropped,
 * and REUSE loads every block once.  Results per pair are the same; only the order of the sink calls changes. */
typedef enum chgpu_task_order { CHGPU_ORDER_REFERENCE = 0, CHGPU_ORDER_REUSE = 1 } chgpu_task_order;
/* order_out: ntasks task indices.  Plans of more than 2^18 tasks are returned in plan order. */
chgpu_status chgpu_order_tasks_for_reuse(const chgpu_plan_task* tasks, uint32_t ntasks, uint32_t block_slots,
                                         uint32_t* order_out);
/* Multi-GPU form of a streamed run: the executed task sequence (plan order, or `order` from
 * chgpu_order_tasks_for_reuse) is cut into `shards` contiguous ranges of about equal pair counts — contiguous, so a
 * worker keeps the block locality of the sequence (assign_workers' round robin, scheduler.cpp:166-173, would hand
 * every worker every block).  first_out[s] .. first_out[s + 1] are the positions of worker s; shards + 1 entries. */
chgpu_status chgpu_shard_tasks(const chgpu_plan_task* tasks, const uint32_t* order /* nullable: plan order */,
                               uint32_t ntasks, uint32_t shards, uint32_t* first_out);
/* The same cut balanced by WORK instead of pair count: task_weights[t] = sum of chgpu_pair_weight over the pairs of
 * task t (chgpu_task_weights computes them from the flat pair list the tasks index). */
chgpu_status chgpu_shard_tasks_weighted(const chgpu_plan_task* tasks, const uint32_t* order /* nullable */, uint32_t ntasks,
                                        const uint64_t* task_weights, uint32_t shards, uint32_t* first_out);
chgpu_status chgpu_task_weights(const chgpu_plan_task* tasks, uint32_t ntasks, const uint32_t* pairs, uint64_t npairs,
                                const uint32_t* points_per_image, uint32_t image_count, uint64_t* task_weights_out);
/* `shard` of `shards` (0 of 0 or 1: the whole plan): one call per GPU / process, each with its own context. */
chgpu_status chgpu_match_plan_streamed(chgpu_ctx* ctx, const char* const* paths, uint32_t image_count,
                                       uint32_t block_images, uint32_t blocks_per_group,
                                       uint32_t group_slots, uint32_t block_slots, chgpu_task_order task_order,
                                       uint32_t shard, uint32_t shards,
                                       const uint32_t* accepted /* nullable: exhaustive */, uint64_t accepted_count,
                                       const chgpu_match_cfg* cfg, uint32_t io_threads, chgpu_plan_sink_fn sink /* nullable */,
                                       void* user, chgpu_file_result* file_results /* nullable */,
                                       chgpu_streamed_stats* stats /* nullable */);
/* centering_pass (engine.cpp:545-559) without keeping anything resident: streams every file once through the
 * loader in blocks of block_images (the 2-slot hashing schedule degenerates to load, sum, evict), applies the mean
 * and returns it.  Files that fail are reported and left out of the mean, as the reference does. */
chgpu_status chgpu_centering_pass_files(chgpu_ctx* ctx, const char* const* paths, uint32_t image_count,
                                        uint32_t block_images, uint32_t io_threads,
                                        chgpu_file_result* file_results /* nullable */, double* centering128_out /* nullable */);

#ifdef __cplusplus
}
#endif
#endif
