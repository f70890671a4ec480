/*
 * chor.h — C ABI shared by the two CPU checkers of the Cascade Hashing hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Two shared objects export exactly this ABI:
 *   oracle/libchoracle.so        independent CPU restatement (oracle/cashash_oracle.cpp)
 *   oracle/_ref/libcashash_ref.so the reference's own translation units, compiled in place
 *                                 from /root/reference/proj/src, behind oracle/ref_shim.cpp
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load them.  The product (libchgpu.so) never links or calls anything here.
 *
 * All arrays are flat, caller-allocated, little-endian host memory.
 *   descriptors : npts x 128 u8, row-major
 *   short codes : npts x L u32, [point*L + table]        (reference ShortCodes::values, hashing.hpp:80-89)
 *   long codes  : npts x 2 u64, bit j in word j/64 bit j%64 (reference LongCode, hashing.hpp:91-96)
 *   planes      : double[128] per plane; short planes ordered [table*m + bit] (hashing.hpp:62-72)
 */
#ifndef CHOR_H
#define CHOR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct chor_family_params {
    uint32_t short_bits;  /* m */
    uint32_t long_bits;   /* n */
    uint32_t table_count; /* L */
    uint64_t seed;
} chor_family_params;

typedef struct chor_match_cfg {
    uint32_t top_k;
    uint32_t hamming_threshold;
    double ratio;
    uint32_t min_candidates_for_ratio;
    int32_t reduce_rounds;
} chor_match_cfg;

/* Layout-identical to the reference MatchRecord (feature_io.hpp:51-57): 16 bytes. */
typedef struct chor_match_record {
    uint32_t query_index;
    uint32_t train_index;
    double distance_sq;
} chor_match_record;

/* Per-pair statistics used by bench.py to evaluate SURVEY.md §8(d)'s bytes_pair formula. */
typedef struct chor_pair_stats {
    uint64_t raw_candidates;    /* R  : sum over queries and tables of bucket sizes */
    uint64_t unique_candidates; /* sum over queries of |deduplicated candidate set|  */
    uint64_t ranked_queries;    /* queries with a non-empty thresholded ranking        */
    uint64_t fallback_queries;  /* queries re-ranked without the threshold             */
    uint64_t verified_queries;  /* Vq : queries reaching verification with >=2 ranked  */
    uint64_t distances;         /* V  : Euclidean distances computed                   */
    uint64_t matches;           /* Mx */
} chor_pair_stats;

/* Return codes: 0 ok, 1 invalid argument (std::invalid_argument in the reference),
 * 2 logic error (std::logic_error), 3 other failure. */
const char* chor_name(void);

int chor_mix64_3(uint64_t seed, uint64_t a, uint64_t b, uint64_t* out);
int chor_reduce_dot(const double* a, const double* b, int tail_rounds, double* out);

int chor_build_family(const chor_family_params* p, double* short_planes, double* long_planes);

int chor_centering_accumulate(const uint8_t* desc, uint64_t npts, uint64_t* sums128, uint64_t* count);
int chor_centering_apply(const uint64_t* sums128, uint64_t count, double* centering128);

int chor_compute_codes(const chor_family_params* p, const double* short_planes,
                       const double* long_planes, const double* centering128, int reduce_rounds,
                       const uint8_t* desc, uint32_t npts, uint32_t* shorts, uint64_t* longs);

/* Dense CSR view of the bucket index (requires m <= 16): per table 2^m+1 offsets and npts
 * point ids, bucket-major, ascending id inside a bucket (matcher.cpp:27-51). */
int chor_build_bucket_index(uint32_t m, uint32_t L, const uint32_t* shorts, uint32_t npts,
                            uint32_t* offsets /* L*(2^m+1) */, uint32_t* points /* L*npts */);

/* Deduplicated ascending candidate set of one query (matcher.cpp:53-63). Returns count. */
int chor_lookup_candidates(uint32_t m, uint32_t L, const uint32_t* query_codes /* L */,
                           const uint32_t* train_shorts, uint32_t ntrain, uint32_t* out /* ntrain */,
                           uint32_t* out_count);

/* Full pair pipeline (matcher.cpp:141-203).  records must hold n_i entries.
 * ranked / ranked_count (optional, may be NULL): the final ranked list per query that
 * euclidean_verify consumed (after the re-rank fallback), ranked[q*top_k + r]. */
int chor_match_pair(const chor_family_params* p, const chor_match_cfg* cfg,
                    const uint8_t* desc_i, uint32_t n_i, const uint32_t* shorts_i, const uint64_t* longs_i,
                    const uint8_t* desc_j, uint32_t n_j, const uint32_t* shorts_j, const uint64_t* longs_j,
                    chor_match_record* records, uint32_t* record_count, chor_pair_stats* stats,
                    uint32_t* ranked, uint32_t* ranked_count);

/* Epipolar-guided variant (guided_match_pair, geometry.cpp:234-250 over match_pair_filtered,
 * matcher.cpp:205-210): between candidate lookup and ranking the candidates of query q are cut to those
 * within band_px of the epipolar line l = F (x_q, y_q, 1)^T; a degenerate line (a == b == 0) leaves the
 * query unguided.  kp_*: n x 4 f32 (x, y, scale, orientation); F: 9 doubles, row-major.
 * The line is evaluated in fp64 without contraction as
 *     a = (F00 x + F01 y) + F02,   b = (F10 x + F11 y) + F12,   c = F20 x + (F21 y + F22).
 * The reference forms it as an Eigen product, Matrix3d * Vector3d (geometry.cpp:98-101), and Eigen is absent from
 * this image (geometry.cpp cannot be compiled), so the order is RESTATED from Eigen >= 3.3's published evaluation
 * of that expression, not checked against a build: a 3 x 3 by 3 x 1 product is coefficient-based (sizes below the
 * GEMV threshold); the assignment to a Vector3d is a linear vectorised traversal, completely unrolled (unaligned
 * vectorisation is on by default): coefficients 0-1 as one Packet2d accumulated over the depth in order,
 * pmadd = padd(pmul(.,.), .) without FMA on baseline x86-64, i.e. (F.0 x + F.1 y) + F.2; the odd coefficient 2 as
 * lhs.row(2).cwiseProduct(rhs).sum(), whose 3-term reduction is unrolled by halves: c0 + (c1 + c2).
 * Parity for candidates within one ulp of the band edge stays UNPINNED until an Eigen build confirms this.
 * In oracle/_ref everything but that line is
 * the reference's own code (match_pair_filtered with this filter). */
int chor_guided_match_pair(const chor_family_params* p, const chor_match_cfg* cfg,
                           const uint8_t* desc_i, const float* kp_i, uint32_t n_i, const uint32_t* shorts_i,
                           const uint64_t* longs_i, const uint8_t* desc_j, const float* kp_j, uint32_t n_j,
                           const uint32_t* shorts_j, const uint64_t* longs_j, const double* F, double band_px,
                           chor_match_record* records, uint32_t* record_count, chor_pair_stats* stats,
                           uint32_t* ranked, uint32_t* ranked_count);

/* match_pair_filtered (matcher.hpp:102-105) with a filter given as data: whenever the reference calls the filter
 * (non-empty candidate list, matcher.cpp:172) the list of query q is REPLACED by
 * list_ids[list_offsets[q] .. list_offsets[q + 1]) — entries may be removed, reordered or repeated, as an arbitrary
 * CandidateFilter may do.  In oracle/_ref this drives the reference's own match_pair_filtered. */
int chor_match_pair_lists(const chor_family_params* p, const chor_match_cfg* cfg,
                          const uint8_t* desc_i, uint32_t n_i, const uint32_t* shorts_i, const uint64_t* longs_i,
                          const uint8_t* desc_j, uint32_t n_j, const uint32_t* shorts_j, const uint64_t* longs_j,
                          const uint64_t* list_offsets, const uint32_t* list_ids,
                          chor_match_record* records, uint32_t* record_count, chor_pair_stats* stats,
                          uint32_t* ranked, uint32_t* ranked_count);

/* Association order of the line's third component used by chor_guided_match_pair of THIS library (the restatement):
 * 0 (default) F20 x + (F21 y + F22); 1 (F20 x + F21 y) + F22.  Test instrumentation for the bound on row f4. */
void chor_set_line_order(int order);

int chor_brute_force_match(const uint8_t* desc_i, uint32_t n_i, const uint8_t* desc_j, uint32_t n_j,
                           double ratio, chor_match_record* records, uint32_t* record_count);

/* Code cache (hashing.cpp:151-272).  chor_load_code_cache: *fault = 0 ok, 1..5 = FeatureFileFault + 1
 * (MissingFile..Unwritable), 6 = parameter/fingerprint mismatch (std::runtime_error); returns 0 unless the
 * arguments are invalid.  shorts/longs must hold `capacity` points. */
int chor_centering_fingerprint(const double* centering128, uint64_t* out);
int chor_save_code_cache(const chor_family_params* p, uint64_t centering_fp, const uint32_t* shorts,
                         const uint64_t* longs, uint32_t npts, const char* path);
int chor_load_code_cache(const char* path, const chor_family_params* expected, uint64_t expected_fp,
                         uint32_t capacity, uint32_t* shorts, uint64_t* longs, uint32_t* count, int* fault,
                         uint64_t* fault_offset);

/* Text match file exactly as the reference writes it (feature_io.cpp:161-183). */
int chor_save_matches(const char* id_i, const char* id_j, const chor_match_record* records,
                      uint32_t count, const char* path);

/* CPU throughput probe for bench.py: runs match_pair over pairs[2*npairs] of a dataset held as
 * arrays of per-image pointers, on `threads` std::threads each taking a disjoint strided slice
 * (the reference's worker model, engine.cpp:686).  Returns wall seconds, total matches and (optional) the
 * order-independent checksum of all records the GPU path's compaction kernel accumulates
 * (sum over records of mix(mix(k << 32 | query) ^ (train << 32 | d^2)), k = position of the pair in `pairs`,
 * mix = the splitmix64 finaliser), so a bench sample compares every record, not a count. */
int chor_time_match_pairs(const chor_family_params* p, const chor_match_cfg* cfg,
                          const uint8_t* const* desc, const uint32_t* counts,
                          const uint32_t* const* shorts, const uint64_t* const* longs,
                          const uint32_t* pairs, uint32_t npairs, uint32_t threads,
                          double* seconds, uint64_t* total_matches, uint64_t* records_checksum);
/* The per-record term of that checksum. */
static inline uint64_t chor_checksum_mix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
static inline uint64_t chor_record_checksum(uint64_t pair_position, uint32_t query, uint32_t train, double distance_sq) {
    return chor_checksum_mix(chor_checksum_mix(pair_position << 32 | query) ^ ((uint64_t)train << 32 | (uint64_t)distance_sq));
}

/* Flattened pair list of plan_exhaustive (scheduler.cpp:99-142) in task order; pairs_out holds
 * image_count*(image_count-1) u32.  task_sizes (optional) receives the pair count of every task,
 * ntasks_out their number. */
int chor_plan_exhaustive(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group,
                         uint32_t* pairs_out, uint64_t* npairs_out, uint32_t* task_sizes, uint32_t* ntasks_out);

/* plan_guided (scheduler.cpp:144-164): the exhaustive traversal restricted to the accepted pairs (either order,
 * duplicates collapse), tasks that end up empty dropped.  Returns 1 (std::invalid_argument) for a self pair or an
 * unknown image index.  pairs_out holds accepted_count pairs; task_sizes / ntasks_out as above. */
int chor_plan_guided(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group,
                     const uint32_t* accepted, uint64_t accepted_count, uint32_t* pairs_out, uint64_t* npairs_out,
                     uint32_t* task_sizes, uint32_t* ntasks_out);

/* Block-pair tasks of the plan (PlanTask, scheduler.hpp:36-43) without their pair lists: 4 u32 per task
 * (group_a, group_b, block_a, block_b).  has_accepted == 0: plan_exhaustive; else plan_guided over `accepted`. */
int chor_plan_task_blocks(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group, int has_accepted,
                          const uint32_t* accepted, uint64_t accepted_count, uint32_t* tasks4_out, uint32_t* ntasks_out);

/* simulate_residency (scheduler.cpp:339-345) over residency_tasks(plan) (:175-192; mode 1 = Matching, 3 slots) or
 * over hashing_residency_tasks(partition) (:194-200; mode 0 = Hashing, 2 slots; accepted ignored).  Actions as 4 u32
 * each: kind (0 Load, 1 Evict, 2 Begin, 3 Finish), level (0 Group, 1 Block), id, prefetch.  actions4_out may be
 * NULL to count.  Returns 2 (std::logic_error) when a current load is blocked. */
int chor_simulate_residency(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group, int mode,
                            int has_accepted, const uint32_t* accepted, uint64_t accepted_count,
                            uint32_t* actions4_out, uint64_t capacity, uint64_t* nactions_out);

/* auto_partition_sizing (scheduler.cpp:347-359). */
int chor_auto_partition_sizing(uint64_t mean_image_bytes, uint64_t memory_budget_bytes, uint32_t* block_images,
                               uint32_t* blocks_per_group);

#ifdef __cplusplus
}
#endif
#endif
