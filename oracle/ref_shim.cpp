// ref_shim.cpp — chor.h ABI implemented by CALLING the reference's own code.
//
// TEST INFRASTRUCTURE ONLY.  Compiled together with the reference translation units
// /root/reference/proj/src/{feature_io,hashing,matcher}.cpp where they lie (see oracle/Makefile)
// into oracle/_ref/libcashash_ref.so.  No reference source is copied into this repository;
// this file only marshals flat arrays into the reference's value types and back.

#include "chor.h"

#include <chrono>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <vector>

#include "cashash/feature_io.hpp"
#include "cashash/hashing.hpp"
#include "cashash/matcher.hpp"
#include "cashash/rng.hpp"
#include "cashash/scheduler.hpp"

namespace {

using namespace cashash;

FamilyParams to_params(const chor_family_params& p) {
    FamilyParams fp;
    fp.short_bits = p.short_bits;
    fp.long_bits = p.long_bits;
    fp.table_count = p.table_count;
    fp.seed = p.seed;
    return fp;
}

MatchConfig to_cfg(const chor_match_cfg& c) {
    MatchConfig mc;
    mc.top_k = c.top_k;
    mc.hamming_threshold = c.hamming_threshold;
    mc.ratio = c.ratio;
    mc.min_candidates_for_ratio = c.min_candidates_for_ratio;
    mc.reduce_rounds = c.reduce_rounds;
    return mc;
}

FeatureSet to_features(const uint8_t* desc, uint32_t n) {
    FeatureSet fs;
    fs.keypoints.resize(n);
    fs.descriptors.resize(n);
    for (uint32_t i = 0; i < n; ++i) std::memcpy(fs.descriptors[i].data(), desc + size_t(i) * 128, 128);
    return fs;
}

ImageCodes to_codes(const FamilyParams& fp, const uint32_t* shorts, const uint64_t* longs, uint32_t n) {
    ImageCodes c;
    c.params = fp;
    c.shorts.short_bits = fp.short_bits;
    c.shorts.table_count = fp.table_count;
    c.shorts.point_count = n;
    c.shorts.values.assign(shorts, shorts + size_t(n) * fp.table_count);
    c.longs.long_bits = fp.long_bits;
    c.longs.codes.resize(n);
    for (uint32_t i = 0; i < n; ++i) {
        c.longs.codes[i].words = {longs[2 * size_t(i)], longs[2 * size_t(i) + 1]};
        c.longs.codes[i].bits = static_cast<uint16_t>(fp.long_bits);
    }
    return c;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (const std::logic_error&) {
        return 2;
    } catch (...) {
        return 3;
    }
}

}  // namespace

extern "C" {

const char* chor_name(void) { return "reference"; }

int chor_mix64_3(uint64_t seed, uint64_t a, uint64_t b, uint64_t* out) {
    *out = mix64(seed, a, b);
    return 0;
}

int chor_reduce_dot(const double* a, const double* b, int tail_rounds, double* out) {
    return guarded([&] {
        *out = reduce_dot<double>(std::span<const double>(a, 128), std::span<const double>(b, 128), tail_rounds);
    });
}

int chor_build_family(const chor_family_params* p, double* short_planes, double* long_planes) {
    return guarded([&] {
        const HashFamily fam = build_hash_family(to_params(*p));
        for (size_t i = 0; i < fam.short_planes.size(); ++i)
            std::memcpy(short_planes + i * 128, fam.short_planes[i].data(), 128 * sizeof(double));
        for (size_t i = 0; i < fam.long_planes.size(); ++i)
            std::memcpy(long_planes + i * 128, fam.long_planes[i].data(), 128 * sizeof(double));
    });
}

int chor_centering_accumulate(const uint8_t* desc, uint64_t npts, uint64_t* sums128, uint64_t* count) {
    return guarded([&] {
        CenteringAccumulator acc;
        std::memcpy(acc.sums.data(), sums128, sizeof(acc.sums));
        acc.count = *count;
        acc.add(to_features(desc, static_cast<uint32_t>(npts)));
        std::memcpy(sums128, acc.sums.data(), sizeof(acc.sums));
        *count = acc.count;
    });
}

int chor_centering_apply(const uint64_t* sums128, uint64_t count, double* centering128) {
    return guarded([&] {
        CenteringAccumulator acc;
        std::memcpy(acc.sums.data(), sums128, sizeof(acc.sums));
        acc.count = count;
        HashFamily fam;
        acc.apply(fam);
        std::memcpy(centering128, fam.centering.data(), sizeof(fam.centering));
    });
}

static HashFamily make_family(const chor_family_params& p, const double* sp, const double* lp,
                              const double* centering) {
    HashFamily fam;
    fam.params = to_params(p);
    fam.short_planes.resize(size_t(p.table_count) * p.short_bits);
    fam.long_planes.resize(p.long_bits);
    for (size_t i = 0; i < fam.short_planes.size(); ++i)
        std::memcpy(fam.short_planes[i].data(), sp + i * 128, 128 * sizeof(double));
    for (size_t i = 0; i < fam.long_planes.size(); ++i)
        std::memcpy(fam.long_planes[i].data(), lp + i * 128, 128 * sizeof(double));
    if (centering) {
        std::memcpy(fam.centering.data(), centering, sizeof(fam.centering));
        fam.centering_set = true;
    }
    return fam;
}

int chor_compute_codes(const chor_family_params* p, const double* short_planes,
                       const double* long_planes, const double* centering128, int reduce_rounds,
                       const uint8_t* desc, uint32_t npts, uint32_t* shorts, uint64_t* longs) {
    return guarded([&] {
        validate(to_params(*p));
        const HashFamily fam = make_family(*p, short_planes, long_planes, centering128);
        const ImageCodes codes = compute_codes(fam, to_features(desc, npts), reduce_rounds);
        std::memcpy(shorts, codes.shorts.values.data(), codes.shorts.values.size() * sizeof(uint32_t));
        for (uint32_t i = 0; i < npts; ++i) {
            longs[2 * size_t(i)] = codes.longs.codes[i].words[0];
            longs[2 * size_t(i) + 1] = codes.longs.codes[i].words[1];
        }
    });
}

int chor_build_bucket_index(uint32_t m, uint32_t L, const uint32_t* shorts, uint32_t npts,
                            uint32_t* offsets, uint32_t* points) {
    if (m < 1 || m > 16 || L < 1) return 1;
    return guarded([&] {
        ShortCodes sc;
        sc.short_bits = m;
        sc.table_count = L;
        sc.point_count = npts;
        sc.values.assign(shorts, shorts + size_t(npts) * L);
        const BucketIndex idx = build_bucket_index(sc);
        const uint32_t nb = 1u << m;
        for (uint32_t t = 0; t < L; ++t) {
            uint32_t* off = offsets + size_t(t) * (nb + 1);
            uint32_t running = 0;
            for (uint32_t c = 0; c < nb; ++c) {
                off[c] = running;
                running += static_cast<uint32_t>(idx.bucket(t, c).size());
            }
            off[nb] = running;
            std::memcpy(points + size_t(t) * npts, idx.tables[t].points.data(), size_t(npts) * sizeof(uint32_t));
        }
    });
}

int chor_lookup_candidates(uint32_t m, uint32_t L, const uint32_t* query_codes,
                           const uint32_t* train_shorts, uint32_t ntrain, uint32_t* out,
                           uint32_t* out_count) {
    return guarded([&] {
        ShortCodes sc;
        sc.short_bits = m;
        sc.table_count = L;
        sc.point_count = ntrain;
        sc.values.assign(train_shorts, train_shorts + size_t(ntrain) * L);
        const BucketIndex idx = build_bucket_index(sc);
        const auto c = lookup_candidates(std::span<const uint32_t>(query_codes, L), idx);
        std::memcpy(out, c.data(), c.size() * sizeof(uint32_t));
        *out_count = static_cast<uint32_t>(c.size());
    });
}

namespace {

// Shared body of chor_match_pair / chor_guided_match_pair: records from the reference's own
// match_pair / match_pair_filtered; intermediate artefacts through its PUBLIC ops only
// (lookup_candidates, rank_histogram) with the re-rank rule stated at matcher.hpp:18-21.
void match_pair_body(const FamilyParams& fp, const MatchConfig& mc, const FeatureSet& fi, const FeatureSet& fj,
                     const ImageCodes& ci, const ImageCodes& cj, const CandidateFilter* filter,
                     chor_match_record* records, uint32_t* record_count, chor_pair_stats* stats,
                     uint32_t* ranked, uint32_t* ranked_count) {
    const uint32_t n_i = static_cast<uint32_t>(fi.size()), n_j = static_cast<uint32_t>(fj.size());
    const std::vector<MatchRecord> out =
        filter ? match_pair_filtered(fi, fj, ci, cj, mc, *filter) : match_pair(fi, fj, ci, cj, mc);
    static_assert(sizeof(MatchRecord) == sizeof(chor_match_record));
    std::memcpy(records, out.data(), out.size() * sizeof(MatchRecord));
    *record_count = static_cast<uint32_t>(out.size());
    if (!stats && !ranked) return;

    chor_pair_stats st{};
    if (ranked_count) std::fill(ranked_count, ranked_count + n_i, 0u);
    if (n_i && n_j) {
        const BucketIndex idx = build_bucket_index(cj.shorts);
        const uint32_t min_ranked = std::max<uint32_t>(2, mc.min_candidates_for_ratio);
        for (uint32_t q = 0; q < n_i; ++q) {
            std::span<const uint32_t> qc(ci.shorts.values.data() + size_t(q) * fp.table_count, fp.table_count);
            for (uint32_t t = 0; t < fp.table_count; ++t) st.raw_candidates += idx.bucket(t, qc[t]).size();
            auto cands = lookup_candidates(qc, idx);
            st.unique_candidates += cands.size();
            if (filter && !cands.empty()) (*filter)(q, cands);
            if (cands.empty()) continue;
            RankHistogram h = rank_histogram(ci.longs.codes[q], cands, cj.longs.codes, mc.hamming_threshold);
            size_t keep = std::min<size_t>(mc.top_k, h.items.size());
            if (keep) ++st.ranked_queries;
            if (keep && keep < min_ranked && cands.size() > h.items.size()) {
                h = rank_histogram(ci.longs.codes[q], cands, cj.longs.codes, fp.long_bits);
                keep = std::min<size_t>(mc.top_k, h.items.size());
                ++st.fallback_queries;
            }
            if (ranked) {
                for (size_t r = 0; r < keep; ++r) ranked[size_t(q) * mc.top_k + r] = h.items[r];
                ranked_count[q] = static_cast<uint32_t>(keep);
            }
            if (keep >= 2) {
                ++st.verified_queries;
                st.distances += keep;
            }
        }
    }
    st.matches = out.size();
    if (stats) *stats = st;
}

void set_keypoints(FeatureSet& fs, const float* kp) {
    for (size_t i = 0; i < fs.keypoints.size(); ++i)
        fs.keypoints[i] = Keypoint{kp[4 * i], kp[4 * i + 1], kp[4 * i + 2], kp[4 * i + 3]};
}

}  // namespace

int chor_match_pair(const chor_family_params* p, const chor_match_cfg* cfg,
                    const uint8_t* desc_i, uint32_t n_i, const uint32_t* shorts_i, const uint64_t* longs_i,
                    const uint8_t* desc_j, uint32_t n_j, const uint32_t* shorts_j, const uint64_t* longs_j,
                    chor_match_record* records, uint32_t* record_count, chor_pair_stats* stats,
                    uint32_t* ranked, uint32_t* ranked_count) {
    return guarded([&] {
        const FamilyParams fp = to_params(*p);
        validate(fp);
        const MatchConfig mc = to_cfg(*cfg);
        const FeatureSet fi = to_features(desc_i, n_i), fj = to_features(desc_j, n_j);
        const ImageCodes ci = to_codes(fp, shorts_i, longs_i, n_i), cj = to_codes(fp, shorts_j, longs_j, n_j);
        match_pair_body(fp, mc, fi, fj, ci, cj, nullptr, records, record_count, stats, ranked, ranked_count);
    });
}

int chor_guided_match_pair(const chor_family_params* p, const chor_match_cfg* cfg,
                           const uint8_t* desc_i, const float* kp_i, uint32_t n_i, const uint32_t* shorts_i,
                           const uint64_t* longs_i, const uint8_t* desc_j, const float* kp_j, uint32_t n_j,
                           const uint32_t* shorts_j, const uint64_t* longs_j, const double* F, double band_px,
                           chor_match_record* records, uint32_t* record_count, chor_pair_stats* stats,
                           uint32_t* ranked, uint32_t* ranked_count) {
    return guarded([&] {
        const FamilyParams fp = to_params(*p);
        validate(fp);
        const MatchConfig mc = to_cfg(*cfg);
        FeatureSet fi = to_features(desc_i, n_i), fj = to_features(desc_j, n_j);
        set_keypoints(fi, kp_i);
        set_keypoints(fj, kp_j);
        const ImageCodes ci = to_codes(fp, shorts_i, longs_i, n_i), cj = to_codes(fp, shorts_j, longs_j, n_j);
        // The band filter of guided_match_pair (geometry.cpp:238-248).  geometry.cpp itself needs Eigen
        // and cannot be compiled here; everything around this lambda is the reference's own code.
        const CandidateFilter filter = [&](std::uint32_t q, std::vector<std::uint32_t>& candidates) {
            const Keypoint& kp = fi.keypoints[q];
            const double x = kp.x, y = kp.y;
            const double a = (F[0] * x + F[1] * y) + F[2];
            const double b = (F[3] * x + F[4] * y) + F[5];
            const double c = F[6] * x + (F[7] * y + F[8]);  // (association order: see chor.h)
            if (a == 0.0 && b == 0.0) return false;
            const double inv_norm = 1.0 / std::sqrt(a * a + b * b);
            std::erase_if(candidates, [&](std::uint32_t idx) {
                const Keypoint& t = fj.keypoints[idx];
                return std::abs(a * t.x + b * t.y + c) * inv_norm > band_px;
            });
            return true;
        };
        match_pair_body(fp, mc, fi, fj, ci, cj, &filter, records, record_count, stats, ranked, ranked_count);
    });
}

int chor_match_pair_lists(const chor_family_params* p, const chor_match_cfg* cfg,
                          const uint8_t* desc_i, uint32_t n_i, const uint32_t* shorts_i, const uint64_t* longs_i,
                          const uint8_t* desc_j, uint32_t n_j, const uint32_t* shorts_j, const uint64_t* longs_j,
                          const uint64_t* list_offsets, const uint32_t* list_ids,
                          chor_match_record* records, uint32_t* record_count, chor_pair_stats* stats,
                          uint32_t* ranked, uint32_t* ranked_count) {
    return guarded([&] {
        const FamilyParams fp = to_params(*p);
        validate(fp);
        const MatchConfig mc = to_cfg(*cfg);
        const FeatureSet fi = to_features(desc_i, n_i), fj = to_features(desc_j, n_j);
        const ImageCodes ci = to_codes(fp, shorts_i, longs_i, n_i), cj = to_codes(fp, shorts_j, longs_j, n_j);
        // the reference's own match_pair_filtered, driven by a filter that replaces the vector it is handed
        const CandidateFilter filter = [&](std::uint32_t q, std::vector<std::uint32_t>& candidates) {
            candidates.assign(list_ids + list_offsets[q], list_ids + list_offsets[q + 1]);
            return true;
        };
        match_pair_body(fp, mc, fi, fj, ci, cj, &filter, records, record_count, stats, ranked, ranked_count);
    });
}

int chor_brute_force_match(const uint8_t* desc_i, uint32_t n_i, const uint8_t* desc_j, uint32_t n_j,
                           double ratio, chor_match_record* records, uint32_t* record_count) {
    return guarded([&] {
        const auto out = brute_force_match(to_features(desc_i, n_i), to_features(desc_j, n_j), ratio);
        std::memcpy(records, out.data(), out.size() * sizeof(MatchRecord));
        *record_count = static_cast<uint32_t>(out.size());
    });
}

int chor_save_matches(const char* id_i, const char* id_j, const chor_match_record* records,
                      uint32_t count, const char* path) {
    return guarded([&] {
        std::vector<MatchRecord> v(count);
        std::memcpy(static_cast<void*>(v.data()), records, size_t(count) * sizeof(MatchRecord));
        save_matches(id_i, id_j, v, path);
    });
}

int chor_centering_fingerprint(const double* centering128, uint64_t* out) {
    return guarded([&] {
        HashFamily fam;
        std::memcpy(fam.centering.data(), centering128, sizeof(fam.centering));
        *out = centering_fingerprint(fam);
    });
}

int chor_save_code_cache(const chor_family_params* p, uint64_t centering_fp, const uint32_t* shorts,
                         const uint64_t* longs, uint32_t npts, const char* path) {
    return guarded([&] { save_code_cache(to_codes(to_params(*p), shorts, longs, npts), centering_fp, path); });
}

int chor_load_code_cache(const char* path, const chor_family_params* expected, uint64_t expected_fp,
                         uint32_t capacity, uint32_t* shorts, uint64_t* longs, uint32_t* count, int* fault,
                         uint64_t* fault_offset) {
    *fault = 0;
    *fault_offset = 0;
    *count = 0;
    try {
        const ImageCodes c = load_code_cache(path, to_params(*expected), expected_fp);
        *count = c.shorts.point_count;
        if (c.shorts.point_count > capacity) return 3;
        std::memcpy(shorts, c.shorts.values.data(), c.shorts.values.size() * 4);
        for (uint32_t i = 0; i < c.shorts.point_count; ++i) {
            longs[2 * size_t(i)] = c.longs.codes[i].words[0];
            longs[2 * size_t(i) + 1] = c.longs.codes[i].words[1];
        }
    } catch (const FeatureFileError& e) {
        *fault = static_cast<int>(e.fault()) + 1;
        *fault_offset = e.byte_offset();
    } catch (const std::runtime_error&) {
        *fault = 6;
    }
    return 0;
}

int chor_time_match_pairs(const chor_family_params* p, const chor_match_cfg* cfg,
                          const uint8_t* const* desc, const uint32_t* counts,
                          const uint32_t* const* shorts, const uint64_t* const* longs,
                          const uint32_t* pairs, uint32_t npairs, uint32_t threads,
                          double* seconds, uint64_t* total_matches, uint64_t* records_checksum) {
    if (threads == 0) return 1;
    return guarded([&] {
        const FamilyParams fp = to_params(*p);
        const MatchConfig mc = to_cfg(*cfg);
        // Marshal every image touched by the sample once, outside the timed region: the
        // reference's engine also holds FeatureSet/ImageCodes resident (engine.cpp:394-412).
        uint32_t max_img = 0;
        for (uint32_t k = 0; k < 2 * npairs; ++k) max_img = std::max(max_img, pairs[k]);
        std::vector<FeatureSet> fs(max_img + 1);
        std::vector<ImageCodes> cs(max_img + 1);
        std::vector<char> have(max_img + 1, 0);
        for (uint32_t k = 0; k < 2 * npairs; ++k) {
            const uint32_t a = pairs[k];
            if (have[a]) continue;
            fs[a] = to_features(desc[a], counts[a]);
            cs[a] = to_codes(fp, shorts[a], longs[a], counts[a]);
            have[a] = 1;
        }
        std::vector<uint64_t> per_thread(threads, 0), per_thread_sum(threads, 0);
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (uint32_t w = 0; w < threads; ++w)
            pool.emplace_back([&, w] {
                for (uint32_t k = w; k < npairs; k += threads) {
                    const uint32_t a = pairs[2 * k], b = pairs[2 * k + 1];
                    const std::vector<MatchRecord> rec = match_pair(fs[a], fs[b], cs[a], cs[b], mc);
                    per_thread[w] += rec.size();
                    for (const MatchRecord& r : rec)  // a few thousand mixes per 80 ms pair: not measurable
                        per_thread_sum[w] += chor_record_checksum(k, r.query_index, r.train_index, r.distance_sq);
                }
            });
        for (auto& t : pool) t.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        uint64_t total = 0, sum = 0;
        for (uint64_t v : per_thread) total += v;
        for (uint64_t v : per_thread_sum) sum += v;
        *total_matches = total;
        if (records_checksum) *records_checksum = sum;
    });
}

int chor_plan_exhaustive(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group,
                         uint32_t* pairs_out, uint64_t* npairs_out, uint32_t* task_sizes, uint32_t* ntasks_out) {
    return guarded([&] {
        const PairPlan plan = plan_exhaustive(make_partition(image_count, block_images, blocks_per_group));
        uint64_t np = 0;
        uint32_t nt = 0;
        for (const PlanTask& t : plan.tasks) {
            for (const auto& [a, b] : t.pairs) {
                if (pairs_out) {
                    pairs_out[2 * np] = a;
                    pairs_out[2 * np + 1] = b;
                }
                ++np;
            }
            if (task_sizes) task_sizes[nt] = static_cast<uint32_t>(t.pairs.size());
            ++nt;
        }
        *npairs_out = np;
        if (ntasks_out) *ntasks_out = nt;
    });
}

int chor_plan_guided(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group,
                     const uint32_t* accepted, uint64_t accepted_count, uint32_t* pairs_out, uint64_t* npairs_out,
                     uint32_t* task_sizes, uint32_t* ntasks_out) {
    return guarded([&] {
        std::vector<std::pair<std::uint32_t, std::uint32_t>> acc(accepted_count);
        for (uint64_t i = 0; i < accepted_count; ++i) acc[i] = {accepted[2 * i], accepted[2 * i + 1]};
        const PairPlan plan = plan_guided(make_partition(image_count, block_images, blocks_per_group), acc);
        uint64_t np = 0;
        uint32_t nt = 0;
        for (const PlanTask& t : plan.tasks) {
            for (const auto& [a, b] : t.pairs) {
                if (pairs_out) {
                    pairs_out[2 * np] = a;
                    pairs_out[2 * np + 1] = b;
                }
                ++np;
            }
            if (task_sizes) task_sizes[nt] = static_cast<uint32_t>(t.pairs.size());
            ++nt;
        }
        *npairs_out = np;
        if (ntasks_out) *ntasks_out = nt;
    });
}

namespace {
PairPlan plan_for(const Partition& part, int has_accepted, const uint32_t* accepted, uint64_t accepted_count) {
    if (!has_accepted) return plan_exhaustive(part);
    std::vector<std::pair<std::uint32_t, std::uint32_t>> acc(accepted_count);
    for (uint64_t i = 0; i < accepted_count; ++i) acc[i] = {accepted[2 * i], accepted[2 * i + 1]};
    return plan_guided(part, acc);
}
}  // namespace

int chor_plan_task_blocks(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group, int has_accepted,
                          const uint32_t* accepted, uint64_t accepted_count, uint32_t* tasks4_out, uint32_t* ntasks_out) {
    return guarded([&] {
        const PairPlan plan = plan_for(make_partition(image_count, block_images, blocks_per_group), has_accepted, accepted,
                                       accepted_count);
        uint32_t nt = 0;
        for (const PlanTask& t : plan.tasks) {
            if (tasks4_out) {
                tasks4_out[4 * nt + 0] = t.group_a;
                tasks4_out[4 * nt + 1] = t.group_b;
                tasks4_out[4 * nt + 2] = t.block_a;
                tasks4_out[4 * nt + 3] = t.block_b;
            }
            ++nt;
        }
        *ntasks_out = nt;
    });
}

int chor_simulate_residency(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group, int mode,
                            int has_accepted, const uint32_t* accepted, uint64_t accepted_count,
                            uint32_t* actions4_out, uint64_t capacity, uint64_t* nactions_out) {
    return guarded([&] {
        const Partition part = make_partition(image_count, block_images, blocks_per_group);
        const std::vector<ResidencyTask> tasks =
            mode == 0 ? hashing_residency_tasks(part)
                      : residency_tasks(plan_for(part, has_accepted, accepted, accepted_count));
        const std::vector<ResidencyAction> trace =
            simulate_residency(tasks, mode == 0 ? ResidencyMode::Hashing : ResidencyMode::Matching);
        uint64_t n = 0;
        for (const ResidencyAction& a : trace) {
            if (actions4_out && n < capacity) {
                actions4_out[4 * n + 0] = static_cast<uint32_t>(a.kind);
                actions4_out[4 * n + 1] = static_cast<uint32_t>(a.level);
                actions4_out[4 * n + 2] = a.id;
                actions4_out[4 * n + 3] = a.prefetch ? 1u : 0u;
            }
            ++n;
        }
        *nactions_out = n;
    });
}

int chor_auto_partition_sizing(uint64_t mean_image_bytes, uint64_t memory_budget_bytes, uint32_t* block_images,
                               uint32_t* blocks_per_group) {
    return guarded([&] {
        const PartitionSizing s = auto_partition_sizing(mean_image_bytes, memory_budget_bytes);
        *block_images = s.block_images;
        *blocks_per_group = s.blocks_per_group;
    });
}

}  // extern "C"
