// cashash_oracle.cpp — CPU restatement of the reference Cascade Hashing hot path.
//
// TEST INFRASTRUCTURE ONLY (see chor.h).  This file restates, independently and over flat
// arrays, what /root/reference/proj computes on the path
//     build_hash_family -> set_centering -> compute_codes -> build_bucket_index -> match_pair
// Each function cites the reference file:line it follows.  Parity is PINNED: tests/test_oracle.py
// checks this file against (a) SPEC.md's worked examples, (b) the golden vectors in
// tests/golden/ produced by the compiled reference (oracle/_ref, see oracle/Makefile and
// tests/golden/make_golden.py) and (c), when oracle/_ref is present, the compiled reference
// itself on fresh random inputs.
//
// Build: g++ -std=gnu++20 -O3 -ffp-contract=off (no -march: an FMA contraction of the
// product/add pairs in reduce_dot would change sign bits of near-zero projections).

#include "chor.h"

#include <algorithm>
#include <bit>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <thread>
#include <set>
#include <vector>

namespace {

constexpr int kDim = 128;

// splitmix64 finaliser and the seed-derivation tuples: reference rng.hpp:18-31.
uint64_t mix1(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
uint64_t mix3(uint64_t seed, uint64_t a, uint64_t b) {
    return mix1(mix1(seed ^ mix1(a)) ^ mix1(b ^ 0xd6e8feb86659fd93ULL));
}

// 53-bit uniform and Box-Muller normal, two generator words per variate: rng.hpp:34-54.
double unit53(std::mt19937_64& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
double normal_bm(std::mt19937_64& g) {
    const double u1 = 1.0 - unit53(g);
    const double u2 = unit53(g);
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}

// Tree-then-serial inner product: hashing.hpp:24-43.  Products are rounded before any add.
double tree_dot(const double* a, const double* b, int tail_rounds) {
    double s[kDim];
    for (int i = 0; i < kDim; ++i) s[i] = a[i] * b[i];
    const int tail = 1 << tail_rounds;
    for (int w = kDim / 2; w >= tail; w /= 2)
        for (int i = 0; i < w; ++i) s[i] = s[i] + s[i + w];
    double acc = s[0];
    for (int i = 1; i < tail; ++i) acc = acc + s[i];
    return acc;
}

bool family_ok(const chor_family_params& p) {  // hashing.cpp:30-36
    if (p.short_bits < 1 || p.short_bits > 32) return false;
    if (p.long_bits <= p.short_bits || p.long_bits > static_cast<uint32_t>(kDim)) return false;
    return p.table_count >= 1;
}

bool cfg_ok(const chor_match_cfg& c, uint32_t long_bits) {  // matcher.cpp:9-17
    if (c.top_k < 2) return false;
    if (c.hamming_threshold > long_bits) return false;
    if (!(c.ratio > 0.0 && c.ratio < 1.0)) return false;
    return c.reduce_rounds >= 0 && c.reduce_rounds <= 7;
}

int hamming128(const uint64_t* a, const uint64_t* b) {  // hashing.hpp:98-101
    return std::popcount(a[0] ^ b[0]) + std::popcount(a[1] ^ b[1]);
}

// Exact squared distance via the same tree reduction on integer-valued doubles: matcher.cpp:106-113.
double dist_sq(const uint8_t* a, const uint8_t* b, int rounds) {
    double diff[kDim];
    for (int i = 0; i < kDim; ++i) diff[i] = static_cast<double>(a[i]) - static_cast<double>(b[i]);
    return tree_dot(diff, diff, rounds);
}

// Sparse bucket index exactly as the reference stores it (sorted unique codes + CSR):
// matcher.cpp:27-51.  Works for every m <= 32.
struct SparseTable {
    std::vector<uint32_t> codes, offsets, points;
    void lookup(uint32_t code, const uint32_t*& first, const uint32_t*& last) const {  // matcher.cpp:19-25
        const auto it = std::lower_bound(codes.begin(), codes.end(), code);
        if (it == codes.end() || *it != code) {
            first = last = nullptr;
            return;
        }
        const size_t slot = static_cast<size_t>(it - codes.begin());
        first = points.data() + offsets[slot];
        last = points.data() + offsets[slot + 1];
    }
};

std::vector<SparseTable> build_sparse_index(uint32_t L, const uint32_t* shorts, uint32_t npts) {
    std::vector<SparseTable> tables(L);
    std::vector<std::pair<uint32_t, uint32_t>> e(npts);
    for (uint32_t t = 0; t < L; ++t) {
        for (uint32_t p = 0; p < npts; ++p) e[p] = {shorts[static_cast<size_t>(p) * L + t], p};
        std::sort(e.begin(), e.end());
        SparseTable& tb = tables[t];
        tb.points.resize(npts);
        for (uint32_t i = 0; i < npts; ++i) {
            if (i == 0 || e[i].first != e[i - 1].first) {
                tb.codes.push_back(e[i].first);
                tb.offsets.push_back(i);
            }
            tb.points[i] = e[i].second;
        }
        tb.offsets.push_back(npts);
    }
    return tables;
}

// Two-pass counting sort over distances 0..threshold: matcher.cpp:68-84.
struct Ranker {
    std::vector<uint32_t> dists, offsets, items, cursor;
    void fill(const uint64_t* q, const std::vector<uint32_t>& cands, const uint64_t* train_longs,
              uint32_t threshold) {
        dists.resize(cands.size());
        offsets.assign(threshold + 2, 0);
        for (size_t i = 0; i < cands.size(); ++i) {
            const uint32_t d = static_cast<uint32_t>(hamming128(q, train_longs + 2 * static_cast<size_t>(cands[i])));
            dists[i] = d;
            if (d <= threshold) ++offsets[d + 1];
        }
        for (uint32_t d = 0; d <= threshold; ++d) offsets[d + 1] += offsets[d];
        items.resize(offsets[threshold + 1]);
        cursor.assign(offsets.begin(), offsets.end() - 1);
        for (size_t i = 0; i < cands.size(); ++i)
            if (dists[i] <= threshold) items[cursor[dists[i]]++] = cands[i];
    }
};

// Association order of the third line component (see chor.h): 0 = F20 x + (F21 y + F22), the order restated from
// Eigen's evaluators; 1 = (F20 x + F21 y) + F22, the other order a build of geometry.cpp:98-101 could produce.
// tests/test_oracle.py measures how often the two disagree on a candidate (chor_set_line_order).
int g_line_order = 0;

// Epipolar band filter of guided_match_pair (geometry.cpp:234-250).
struct BandFilter {
    const float* kp_i;  // n_i x 4
    const float* kp_j;  // n_j x 4
    const double* F;    // 3 x 3 row-major
    double band_px;

    // Returns false (candidates untouched) for a degenerate line.
    bool apply(uint32_t q, std::vector<uint32_t>& cands) const {
        const double x = kp_i[4 * static_cast<size_t>(q)], y = kp_i[4 * static_cast<size_t>(q) + 1];
        const double a = (F[0] * x + F[1] * y) + F[2];  // epipolar_line: l = F (x, y, 1)^T  (geometry.cpp:98-101)
        const double b = (F[3] * x + F[4] * y) + F[5];
        const double c = g_line_order == 0 ? F[6] * x + (F[7] * y + F[8])    // (association order: see chor.h)
                                           : (F[6] * x + F[7] * y) + F[8];
        if (a == 0.0 && b == 0.0) return false;  // EpipolarLine::degenerate, geometry.hpp:28
        const double inv_norm = 1.0 / std::sqrt(a * a + b * b);
        std::erase_if(cands, [&](uint32_t idx) {
            const double tx = kp_j[4 * static_cast<size_t>(idx)], ty = kp_j[4 * static_cast<size_t>(idx) + 1];
            return std::abs(a * tx + b * ty + c) * inv_norm > band_px;
        });
        return true;
    }
};

// A filter given as data: the candidate list of query q is REPLACED by ids[offs[q] .. offs[q + 1]) — what an arbitrary
// CandidateFilter (matcher.hpp:92-93) may do to the vector it is handed (chor_match_pair_lists).
struct ListFilter {
    const uint64_t* offs;
    const uint32_t* ids;
    void apply(uint32_t q, std::vector<uint32_t>& cands) const { cands.assign(ids + offs[q], ids + offs[q + 1]); }
};

int match_pair_impl(const chor_family_params& p, const chor_match_cfg& cfg,
                    const uint8_t* desc_i, uint32_t n_i, const uint32_t* shorts_i, const uint64_t* longs_i,
                    const uint8_t* desc_j, uint32_t n_j, const uint32_t* shorts_j, const uint64_t* longs_j,
                    chor_match_record* records, uint32_t* record_count, chor_pair_stats* stats,
                    uint32_t* ranked_out, uint32_t* ranked_count, const BandFilter* filter = nullptr,
                    const ListFilter* lists = nullptr) {
    // matcher.cpp:141-195.  Family equality / count checks are structural in this flat ABI.
    if (!family_ok(p) || !cfg_ok(cfg, p.long_bits)) return 1;
    chor_pair_stats st{};
    uint32_t nrec = 0;
    if (ranked_count) std::fill(ranked_count, ranked_count + n_i, 0u);
    if (n_i != 0 && n_j != 0) {
        const uint32_t L = p.table_count;
        const auto index = build_sparse_index(L, shorts_j, n_j);
        const uint32_t min_ranked = std::max<uint32_t>(2, cfg.min_candidates_for_ratio);
        std::vector<uint32_t> cands;
        Ranker rk;
        for (uint32_t q = 0; q < n_i; ++q) {
            cands.clear();
            for (uint32_t t = 0; t < L; ++t) {
                const uint32_t *f, *l;
                index[t].lookup(shorts_i[static_cast<size_t>(q) * L + t], f, l);
                cands.insert(cands.end(), f, l);
            }
            st.raw_candidates += cands.size();
            std::sort(cands.begin(), cands.end());
            cands.erase(std::unique(cands.begin(), cands.end()), cands.end());
            st.unique_candidates += cands.size();
            if (filter && !cands.empty()) filter->apply(q, cands);  // matcher.cpp:172
            if (lists && !cands.empty()) lists->apply(q, cands);
            if (cands.empty()) continue;

            const uint64_t* ql = longs_i + 2 * static_cast<size_t>(q);
            rk.fill(ql, cands, longs_j, cfg.hamming_threshold);
            size_t keep = std::min<size_t>(cfg.top_k, rk.items.size());
            if (keep != 0) ++st.ranked_queries;
            // Re-rank fallback (matcher.cpp:179-189): non-empty, too small for the ratio test,
            // and the threshold actually cut something.
            if (keep != 0 && keep < min_ranked && cands.size() > rk.items.size()) {
                rk.fill(ql, cands, longs_j, p.long_bits);
                keep = std::min<size_t>(cfg.top_k, rk.items.size());
                ++st.fallback_queries;
            }
            if (ranked_out) {
                for (size_t r = 0; r < keep; ++r) ranked_out[static_cast<size_t>(q) * cfg.top_k + r] = rk.items[r];
                ranked_count[q] = static_cast<uint32_t>(keep);
            }
            // euclidean_verify, matcher.cpp:115-137.
            if (keep < 2) continue;
            ++st.verified_queries;
            double best = std::numeric_limits<double>::infinity();
            double second = std::numeric_limits<double>::infinity();
            uint32_t best_index = 0;
            const uint8_t* qd = desc_i + static_cast<size_t>(q) * kDim;
            for (size_t r = 0; r < keep; ++r) {
                const uint32_t idx = rk.items[r];
                const double d = dist_sq(qd, desc_j + static_cast<size_t>(idx) * kDim, cfg.reduce_rounds);
                ++st.distances;
                if (d < best) {
                    second = best;
                    best = d;
                    best_index = idx;
                } else if (d < second) {
                    second = d;
                }
            }
            if (second == 0.0) continue;
            if (best < cfg.ratio * cfg.ratio * second) {
                records[nrec].query_index = q;
                records[nrec].train_index = best_index;
                records[nrec].distance_sq = best;
                ++nrec;
            }
        }
    }
    st.matches = nrec;
    *record_count = nrec;
    if (stats) *stats = st;
    return 0;
}

}  // namespace

extern "C" {

const char* chor_name(void) { return "restatement"; }

int chor_mix64_3(uint64_t seed, uint64_t a, uint64_t b, uint64_t* out) {
    *out = mix3(seed, a, b);
    return 0;
}

int chor_reduce_dot(const double* a, const double* b, int tail_rounds, double* out) {
    if (tail_rounds < 0 || tail_rounds > 7) return 1;
    *out = tree_dot(a, b, tail_rounds);
    return 0;
}

int chor_build_family(const chor_family_params* p, double* short_planes, double* long_planes) {
    // hashing.cpp:19-26 (draw_plane), :38-50 (table-major short planes, sentinel stream for long).
    if (!family_ok(*p)) return 1;
    auto draw = [&](uint64_t table, uint64_t bit, double* dst) {
        std::mt19937_64 g(mix3(p->seed, table, bit));
        for (int i = 0; i < kDim; ++i) dst[i] = normal_bm(g);
    };
    for (uint32_t t = 0; t < p->table_count; ++t)
        for (uint32_t j = 0; j < p->short_bits; ++j)
            draw(t, j, short_planes + (static_cast<size_t>(t) * p->short_bits + j) * kDim);
    for (uint32_t j = 0; j < p->long_bits; ++j) draw(0xffffffffULL, j, long_planes + static_cast<size_t>(j) * kDim);
    return 0;
}

int chor_centering_accumulate(const uint8_t* desc, uint64_t npts, uint64_t* sums128, uint64_t* count) {
    // hashing.cpp:52-57: exact integer column sums.
    for (uint64_t p = 0; p < npts; ++p)
        for (int c = 0; c < kDim; ++c) sums128[c] += desc[p * kDim + c];
    *count += npts;
    return 0;
}

int chor_centering_apply(const uint64_t* sums128, uint64_t count, double* centering128) {
    // hashing.cpp:59-64.
    if (count == 0) return 1;
    for (int c = 0; c < kDim; ++c)
        centering128[c] = static_cast<double>(sums128[c]) / static_cast<double>(count);
    return 0;
}

int chor_compute_codes(const chor_family_params* p, const double* short_planes,
                       const double* long_planes, const double* centering128, int reduce_rounds,
                       const uint8_t* desc, uint32_t npts, uint32_t* shorts, uint64_t* longs) {
    // hashing.cpp:72-99 and :130-149.  Bit = (dot > 0.0); ties give 0.
    if (!family_ok(*p)) return 1;
    if (reduce_rounds < 0 || reduce_rounds > 7) return 1;
    if (centering128 == nullptr) return 2;  // "centering has not been set" (hashing.cpp:131-132)
    double c[kDim];
    for (uint32_t pt = 0; pt < npts; ++pt) {
        const uint8_t* d = desc + static_cast<size_t>(pt) * kDim;
        for (int i = 0; i < kDim; ++i) c[i] = static_cast<double>(d[i]) - centering128[i];
        for (uint32_t t = 0; t < p->table_count; ++t) {
            uint32_t code = 0;
            for (uint32_t j = 0; j < p->short_bits; ++j) {
                const double* h = short_planes + (static_cast<size_t>(t) * p->short_bits + j) * kDim;
                if (tree_dot(c, h, reduce_rounds) > 0.0) code |= (1u << j);
            }
            shorts[static_cast<size_t>(pt) * p->table_count + t] = code;
        }
        uint64_t w[2] = {0, 0};
        for (uint32_t j = 0; j < p->long_bits; ++j)
            if (tree_dot(c, long_planes + static_cast<size_t>(j) * kDim, reduce_rounds) > 0.0)
                w[j / 64] |= (uint64_t{1} << (j % 64));
        longs[2 * static_cast<size_t>(pt)] = w[0];
        longs[2 * static_cast<size_t>(pt) + 1] = w[1];
    }
    return 0;
}

int chor_build_bucket_index(uint32_t m, uint32_t L, const uint32_t* shorts, uint32_t npts,
                            uint32_t* offsets, uint32_t* points) {
    if (m < 1 || m > 16 || L < 1) return 1;
    const uint32_t nb = 1u << m;
    const auto sparse = build_sparse_index(L, shorts, npts);
    for (uint32_t t = 0; t < L; ++t) {
        uint32_t* off = offsets + static_cast<size_t>(t) * (nb + 1);
        std::fill(off, off + nb + 1, 0u);
        const SparseTable& tb = sparse[t];
        // Dense view: bucket c = [off[c], off[c+1]); absent codes are empty ranges.
        size_t slot = 0;
        for (uint32_t c = 0; c <= nb; ++c) {
            while (slot < tb.codes.size() && tb.codes[slot] < c) ++slot;
            off[c] = slot < tb.codes.size() ? tb.offsets[slot] : npts;
        }
        std::copy(tb.points.begin(), tb.points.end(), points + static_cast<size_t>(t) * npts);
    }
    return 0;
}

int chor_lookup_candidates(uint32_t m, uint32_t L, const uint32_t* query_codes,
                           const uint32_t* train_shorts, uint32_t ntrain, uint32_t* out,
                           uint32_t* out_count) {
    (void)m;
    const auto index = build_sparse_index(L, train_shorts, ntrain);
    std::vector<uint32_t> c;
    for (uint32_t t = 0; t < L; ++t) {
        const uint32_t *f, *l;
        index[t].lookup(query_codes[t], f, l);
        c.insert(c.end(), f, l);
    }
    std::sort(c.begin(), c.end());
    c.erase(std::unique(c.begin(), c.end()), c.end());
    std::copy(c.begin(), c.end(), out);
    *out_count = static_cast<uint32_t>(c.size());
    return 0;
}

int chor_match_pair(const chor_family_params* p, const chor_match_cfg* cfg,
                    const uint8_t* desc_i, uint32_t n_i, const uint32_t* shorts_i, const uint64_t* longs_i,
                    const uint8_t* desc_j, uint32_t n_j, const uint32_t* shorts_j, const uint64_t* longs_j,
                    chor_match_record* records, uint32_t* record_count, chor_pair_stats* stats,
                    uint32_t* ranked, uint32_t* ranked_count) {
    return match_pair_impl(*p, *cfg, desc_i, n_i, shorts_i, longs_i, desc_j, n_j, shorts_j, longs_j,
                           records, record_count, stats, ranked, ranked_count);
}

void chor_set_line_order(int order) { g_line_order = order ? 1 : 0; }

int chor_guided_match_pair(const chor_family_params* p, const chor_match_cfg* cfg,
                           const uint8_t* desc_i, const float* kp_i, uint32_t n_i, const uint32_t* shorts_i,
                           const uint64_t* longs_i, const uint8_t* desc_j, const float* kp_j, uint32_t n_j,
                           const uint32_t* shorts_j, const uint64_t* longs_j, const double* F, double band_px,
                           chor_match_record* records, uint32_t* record_count, chor_pair_stats* stats,
                           uint32_t* ranked, uint32_t* ranked_count) {
    const BandFilter filter{kp_i, kp_j, F, band_px};
    return match_pair_impl(*p, *cfg, desc_i, n_i, shorts_i, longs_i, desc_j, n_j, shorts_j, longs_j, records,
                           record_count, stats, ranked, ranked_count, &filter);
}

int chor_match_pair_lists(const chor_family_params* p, const chor_match_cfg* cfg,
                          const uint8_t* desc_i, uint32_t n_i, const uint32_t* shorts_i, const uint64_t* longs_i,
                          const uint8_t* desc_j, uint32_t n_j, const uint32_t* shorts_j, const uint64_t* longs_j,
                          const uint64_t* list_offsets, const uint32_t* list_ids,
                          chor_match_record* records, uint32_t* record_count, chor_pair_stats* stats,
                          uint32_t* ranked, uint32_t* ranked_count) {
    const ListFilter lists{list_offsets, list_ids};
    return match_pair_impl(*p, *cfg, desc_i, n_i, shorts_i, longs_i, desc_j, n_j, shorts_j, longs_j, records,
                           record_count, stats, ranked, ranked_count, nullptr, &lists);
}

int chor_brute_force_match(const uint8_t* desc_i, uint32_t n_i, const uint8_t* desc_j, uint32_t n_j,
                           double ratio, chor_match_record* records, uint32_t* record_count) {
    // matcher.cpp:212-243: exact integer NN / 2nd-NN, same ratio rule.
    uint32_t nrec = 0;
    if (n_j >= 2) {
        const double r2 = ratio * ratio;
        for (uint32_t q = 0; q < n_i; ++q) {
            uint64_t best = std::numeric_limits<uint64_t>::max(), second = best;
            uint32_t bi = 0;
            for (uint32_t t = 0; t < n_j; ++t) {
                uint64_t d = 0;
                for (int c = 0; c < kDim; ++c) {
                    const int df = int(desc_i[size_t(q) * kDim + c]) - int(desc_j[size_t(t) * kDim + c]);
                    d += static_cast<uint64_t>(df * df);
                }
                if (d < best) {
                    second = best;
                    best = d;
                    bi = t;
                } else if (d < second) {
                    second = d;
                }
            }
            if (second == 0) continue;
            if (static_cast<double>(best) < r2 * static_cast<double>(second))
                records[nrec++] = {q, bi, static_cast<double>(best)};
        }
    }
    *record_count = nrec;
    return 0;
}

int chor_save_matches(const char* id_i, const char* id_j, const chor_match_record* records,
                      uint32_t count, const char* path) {
    // feature_io.cpp:161-183: "# I J count\n" then "q t dist\n", dist = shortest round-trip decimal.
    std::string out = "# ";
    out += id_i;
    out += ' ';
    out += id_j;
    out += ' ';
    out += std::to_string(count);
    out += '\n';
    char buf[64];
    for (uint32_t i = 0; i < count; ++i) {
        out += std::to_string(records[i].query_index);
        out += ' ';
        out += std::to_string(records[i].train_index);
        out += ' ';
        const auto r = std::to_chars(buf, buf + sizeof(buf), records[i].distance_sq);
        out.append(buf, r.ptr);
        out += '\n';
    }
    FILE* f = std::fopen(path, "wb");
    if (!f) return 3;
    const size_t w = std::fwrite(out.data(), 1, out.size(), f);
    std::fclose(f);
    return w == out.size() ? 0 : 3;
}

// centering_fingerprint: FNV-1a over the bytes of the 128 doubles, low byte first (hashing.cpp:151-162).
int chor_centering_fingerprint(const double* centering128, uint64_t* out) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (int i = 0; i < kDim; ++i) {
        unsigned char b[8];
        std::memcpy(b, centering128 + i, 8);
        for (int k = 0; k < 8; ++k) h = (h ^ b[k]) * 0x100000001b3ULL;
    }
    *out = h;
    return 0;
}

// save_code_cache (hashing.cpp:184-206): 44-byte header, then point-major short codes, then long words.
int chor_save_code_cache(const chor_family_params* p, uint64_t centering_fp, const uint32_t* shorts,
                         const uint64_t* longs, uint32_t npts, const char* path) {
    std::string out("CHCC");
    auto put = [&out](const void* v, size_t n) { out.append(static_cast<const char*>(v), n); };
    const uint32_t version = 1, reserved = 0;
    put(&version, 4);
    put(&p->short_bits, 4);
    put(&p->long_bits, 4);
    put(&p->table_count, 4);
    put(&p->seed, 8);
    put(&centering_fp, 8);
    put(&npts, 4);
    put(&reserved, 4);
    put(shorts, size_t(npts) * p->table_count * 4);
    put(longs, size_t(npts) * 16);
    FILE* f = std::fopen(path, "wb");
    if (!f) return 3;
    const bool ok = std::fwrite(out.data(), 1, out.size(), f) == out.size();
    return (std::fclose(f) == 0 && ok) ? 0 : 3;
}

// load_code_cache / parse_code_cache (hashing.cpp:228-272).  Fault codes as documented in chor.h.
int chor_load_code_cache(const char* path, const chor_family_params* expected, uint64_t expected_fp,
                         uint32_t capacity, uint32_t* shorts, uint64_t* longs, uint32_t* count, int* fault,
                         uint64_t* fault_offset) {
    *fault = 0;
    *fault_offset = 0;
    *count = 0;
    FILE* f = std::fopen(path, "rb");
    if (!f) { *fault = 1; return 0; }  // MissingFile at 0
    std::vector<unsigned char> b;
    unsigned char buf[65536];
    size_t got;
    while ((got = std::fread(buf, 1, sizeof(buf), f)) > 0) b.insert(b.end(), buf, buf + got);
    std::fclose(f);
    if (b.size() < 4 || std::memcmp(b.data(), "CHCC", 4) != 0) { *fault = 2; return 0; }       // BadMagic at 0
    if (b.size() < 44) { *fault = 4; *fault_offset = 4; return 0; }                              // Truncated "cache header" at 4
    uint32_t version, m, n, L, cnt;
    uint64_t seed, fp;
    std::memcpy(&version, &b[4], 4);
    std::memcpy(&m, &b[8], 4);
    std::memcpy(&n, &b[12], 4);
    std::memcpy(&L, &b[16], 4);
    std::memcpy(&seed, &b[20], 8);
    std::memcpy(&fp, &b[28], 8);
    std::memcpy(&cnt, &b[36], 4);
    if (version != 1) { *fault = 3; *fault_offset = 4; return 0; }                               // BadVersion at 4
    if (m != expected->short_bits || n != expected->long_bits || L != expected->table_count || seed != expected->seed ||
        fp != expected_fp) { *fault = 6; return 0; }
    *count = cnt;
    const size_t sb = size_t(cnt) * L * 4, lb = size_t(cnt) * 16;
    // a short payload surfaces as static_cast<uint64_t>(in.tellg()) on a failed stream, i.e. 2^64 - 1
    if (b.size() < 44 + sb + lb) { *fault = 4; *fault_offset = std::numeric_limits<uint64_t>::max(); return 0; }
    if (cnt > capacity) return 3;
    std::memcpy(shorts, &b[44], sb);
    std::memcpy(longs, b.data() + 44 + sb, lb);
    return 0;
}

int chor_time_match_pairs(const chor_family_params* p, const chor_match_cfg* cfg,
                          const uint8_t* const* desc, const uint32_t* counts,
                          const uint32_t* const* shorts, const uint64_t* const* longs,
                          const uint32_t* pairs, uint32_t npairs, uint32_t threads,
                          double* seconds, uint64_t* total_matches, uint64_t* records_checksum) {
    if (threads == 0) return 1;
    std::vector<uint64_t> per_thread(threads, 0), per_thread_sum(threads, 0);
    std::vector<int> rc(threads, 0);
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (uint32_t w = 0; w < threads; ++w) {
        pool.emplace_back([&, w] {
            std::vector<chor_match_record> rec;
            for (uint32_t k = w; k < npairs; k += threads) {
                const uint32_t a = pairs[2 * k], b = pairs[2 * k + 1];
                rec.resize(counts[a]);
                uint32_t n = 0;
                const int r = match_pair_impl(*p, *cfg, desc[a], counts[a], shorts[a], longs[a], desc[b],
                                              counts[b], shorts[b], longs[b], rec.data(), &n, nullptr,
                                              nullptr, nullptr);
                if (r != 0) rc[w] = r;
                per_thread[w] += n;
                for (uint32_t i = 0; i < n; ++i)
                    per_thread_sum[w] += chor_record_checksum(k, rec[i].query_index, rec[i].train_index, rec[i].distance_sq);
            }
        });
    }
    for (auto& t : pool) t.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    uint64_t total = 0, sum = 0;
    for (uint32_t w = 0; w < threads; ++w) {
        total += per_thread[w];
        sum += per_thread_sum[w];
        if (rc[w] != 0) return rc[w];
    }
    *total_matches = total;
    if (records_checksum) *records_checksum = sum;
    return 0;
}

int chor_plan_exhaustive(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group,
                         uint32_t* pairs_out, uint64_t* npairs_out, uint32_t* task_sizes, uint32_t* ntasks_out) {
    // scheduler.cpp:10-33 (partition), :47-75 (cross / self tasks), :77-95 (chained edges), :99-142 (plan).
    if (image_count == 0 || block_images == 0 || blocks_per_group == 0) return 1;
    std::vector<std::pair<uint32_t, uint32_t>> ranges;
    for (uint32_t f = 0; f < image_count; f += block_images) ranges.emplace_back(f, std::min(f + block_images, image_count));
    const uint32_t nblocks = static_cast<uint32_t>(ranges.size());
    std::vector<std::vector<uint32_t>> groups;
    for (uint32_t b = 0; b < nblocks; b += blocks_per_group) {
        groups.emplace_back();
        for (uint32_t i = b; i < std::min(b + blocks_per_group, nblocks); ++i) groups.back().push_back(i);
    }
    // first the task list as (block_a, block_b) with a == b for self tasks, then the expansion
    std::vector<std::pair<uint32_t, uint32_t>> tasks;
    for (size_t gi = 0; gi < groups.size(); ++gi) {
        const auto& A = groups[gi];
        uint32_t j = 0;
        bool jf = true;
        for (size_t gk = gi + 1; gk < groups.size(); ++gk) {
            const auto& B = groups[gk];
            uint32_t l = 0;
            bool lf = true;
            for (size_t js = 0; js < A.size(); ++js) {
                for (size_t ls = 0; ls < B.size(); ++ls) {
                    tasks.emplace_back(std::min(A[j], B[l]), std::max(A[j], B[l]));
                    if (ls + 1 < B.size()) l = lf ? l + 1 : l - 1;
                }
                lf = !lf;
                if (js + 1 < A.size()) j = jf ? j + 1 : j - 1;
            }
            jf = !jf;
        }
        std::vector<uint32_t> label{j};
        for (uint32_t v = 0; v < A.size(); ++v)
            if (v != j) label.push_back(v);
        const uint32_t cnt = static_cast<uint32_t>(A.size());
        for (uint32_t a = 0; a + 1 < cnt; ++a) {
            if (a % 2 == 0) {
                for (uint32_t b = a + 1; b < cnt; ++b)
                    tasks.emplace_back(std::min(A[label[a]], A[label[b]]), std::max(A[label[a]], A[label[b]]));
            } else {
                for (uint32_t b = cnt; b-- > a + 1;)
                    tasks.emplace_back(std::min(A[label[a]], A[label[b]]), std::max(A[label[a]], A[label[b]]));
            }
        }
        for (uint32_t blk : A)
            if (ranges[blk].second - ranges[blk].first >= 2) tasks.emplace_back(blk, blk);
    }
    uint64_t np = 0;
    uint32_t nt = 0;
    for (const auto& [ba, bb] : tasks) {
        uint32_t sz = 0;
        if (ba == bb) {
            for (uint32_t a = ranges[ba].first; a < ranges[ba].second; ++a)
                for (uint32_t b = a + 1; b < ranges[ba].second; ++b, ++sz)
                    if (pairs_out) { pairs_out[2 * np] = a; pairs_out[2 * np + 1] = b; ++np; } else ++np;
        } else {
            for (uint32_t a = ranges[ba].first; a < ranges[ba].second; ++a)
                for (uint32_t b = ranges[bb].first; b < ranges[bb].second; ++b, ++sz)
                    if (pairs_out) { pairs_out[2 * np] = a; pairs_out[2 * np + 1] = b; ++np; } else ++np;
        }
        if (task_sizes) task_sizes[nt] = sz;
        ++nt;
    }
    *npairs_out = np;
    if (ntasks_out) *ntasks_out = nt;
    return 0;
}

int chor_plan_guided(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group,
                     const uint32_t* accepted, uint64_t accepted_count, uint32_t* pairs_out, uint64_t* npairs_out,
                     uint32_t* task_sizes, uint32_t* ntasks_out) {
    // scheduler.cpp:144-164: accepted pairs as a set of normalised (a < b) keys; every task of the exhaustive plan
    // keeps the pairs in the set; empty tasks disappear.
    if (image_count == 0 || block_images == 0 || blocks_per_group == 0) return 1;
    std::set<uint64_t> keys;
    for (uint64_t i = 0; i < accepted_count; ++i) {
        uint32_t a = accepted[2 * i], b = accepted[2 * i + 1];
        if (a == b) return 1;
        if (a > b) std::swap(a, b);
        if (b >= image_count) return 1;
        keys.insert(static_cast<uint64_t>(a) * image_count + b);
    }
    const uint64_t all = static_cast<uint64_t>(image_count) * (image_count - 1) / 2;
    std::vector<uint32_t> full(std::max<uint64_t>(all, 1) * 2), sizes(static_cast<size_t>(image_count) * image_count + 4);
    uint64_t nfull = 0;
    uint32_t nt_full = 0;
    if (const int rc = chor_plan_exhaustive(image_count, block_images, blocks_per_group, full.data(), &nfull, sizes.data(), &nt_full))
        return rc;
    uint64_t np = 0, at = 0;
    uint32_t nt = 0;
    for (uint32_t t = 0; t < nt_full; ++t) {
        uint32_t kept = 0;
        for (uint32_t k = 0; k < sizes[t]; ++k, ++at) {
            const uint32_t a = full[2 * at], b = full[2 * at + 1];
            if (!keys.count(static_cast<uint64_t>(a) * image_count + b)) continue;
            if (pairs_out) {
                pairs_out[2 * np] = a;
                pairs_out[2 * np + 1] = b;
            }
            ++np;
            ++kept;
        }
        if (kept) {
            if (task_sizes) task_sizes[nt] = kept;
            ++nt;
        }
    }
    *npairs_out = np;
    if (ntasks_out) *ntasks_out = nt;
    return 0;
}

}  // extern "C"

// ---- residency schedule (scheduler.cpp:175-345) ---------------------------------------------------------------
namespace {

struct OTask {  // ResidencyTask, scheduler.hpp:77-81
    std::vector<uint32_t> groups, blocks, block_groups;
};

// (block_a, block_b) of every task of the plan, by re-running the pair-list restatements above: a task's blocks are
// the blocks of its first pair (every pair of a task lies in the same block pair, scheduler.cpp:47-75).
int task_blocks(uint32_t K, uint32_t Np, uint32_t M, int has_accepted, const uint32_t* accepted, uint64_t accepted_count,
                std::vector<std::pair<uint32_t, uint32_t>>& out) {
    if (K == 0 || Np == 0 || M == 0) return 1;
    const uint64_t cap = has_accepted ? accepted_count : static_cast<uint64_t>(K) * (K - 1) / 2;
    std::vector<uint32_t> pairs(std::max<uint64_t>(cap, 1) * 2), sizes(static_cast<size_t>(K) * K + 4);
    uint64_t np = 0;
    uint32_t nt = 0;
    const int rc = has_accepted ? chor_plan_guided(K, Np, M, accepted, accepted_count, pairs.data(), &np, sizes.data(), &nt)
                                : chor_plan_exhaustive(K, Np, M, pairs.data(), &np, sizes.data(), &nt);
    if (rc) return rc;
    out.clear();
    uint64_t at = 0;
    for (uint32_t t = 0; t < nt; ++t) {
        out.emplace_back(pairs[2 * at] / Np, pairs[2 * at + 1] / Np);
        at += sizes[t];
    }
    return 0;
}

// Next task >= from that uses `id` at the given level, by scanning the task list (kNever if none).
uint32_t scan_next_use(const std::vector<OTask>& tasks, bool block_level, uint32_t id, uint32_t from) {
    for (uint32_t t = from; t < tasks.size(); ++t) {
        const auto& v = block_level ? tasks[t].blocks : tasks[t].groups;
        if (std::find(v.begin(), v.end(), id) != v.end()) return t;
    }
    return 0xffffffffu;
}

struct OAction {
    uint32_t kind, level, id, prefetch;
};

// acquire (scheduler.cpp:226-247): free slot -> Load; else evict the resident item with the farthest next use
// (ties: the smaller id), provided that use is strictly after need_at; else nothing can be done.
bool o_acquire(const std::vector<OTask>& tasks, std::vector<uint32_t>& resident, bool block_level, uint32_t id,
               uint32_t need_at, uint32_t limit, uint32_t cursor, bool prefetch, OAction& act) {
    if (resident.size() < limit) {
        resident.push_back(id);
        act = {0u, block_level ? 1u : 0u, id, prefetch ? 1u : 0u};
        return true;
    }
    bool have = false;
    uint32_t victim = 0, far = 0;
    for (uint32_t r : resident) {
        const uint32_t u = scan_next_use(tasks, block_level, r, cursor);
        if (u > far || (u == far && (!have || r < victim))) {
            victim = r;
            far = u;
            have = true;
        }
    }
    if (!have || far <= need_at) return false;
    resident.erase(std::find(resident.begin(), resident.end(), victim));
    act = {1u, block_level ? 1u : 0u, victim, 0u};
    return true;
}

bool in(const std::vector<uint32_t>& v, uint32_t id) { return std::find(v.begin(), v.end(), id) != v.end(); }

// simulate_residency (scheduler.cpp:339-345) = step_residency (:269-337) until the plan is exhausted.
// Returns 2 where the reference throws std::logic_error.
int o_simulate(const std::vector<OTask>& tasks, uint32_t limit, std::vector<OAction>& trace) {
    std::vector<uint32_t> rg, rb;
    uint32_t cursor = 0;
    bool begun = false;
    while (cursor < tasks.size()) {
        const OTask& cur = tasks[cursor];
        OAction act{};
        bool acted = false;
        if (!begun)  // line 1, groups
            for (uint32_t g : cur.groups) {
                if (in(rg, g)) continue;
                if (!o_acquire(tasks, rg, false, g, cursor, limit, cursor, false, act)) return 2;
                acted = true;
                break;
            }
        if (!acted)  // line 2, groups
            for (uint32_t t = cursor + 1; t < tasks.size() && !acted; ++t) {
                bool all = true;
                for (uint32_t g : tasks[t].groups) {
                    if (in(rg, g)) continue;
                    all = false;
                    if (o_acquire(tasks, rg, false, g, t, limit, cursor, true, act)) {
                        acted = true;
                        break;
                    }
                }
                if (!all) break;
            }
        if (!acted && !begun)  // line 1, blocks
            for (uint32_t b : cur.blocks) {
                if (in(rb, b)) continue;
                if (!o_acquire(tasks, rb, true, b, cursor, limit, cursor, false, act)) return 2;
                acted = true;
                break;
            }
        if (!acted)  // line 2, blocks
            for (uint32_t t = cursor + 1; t < tasks.size() && !acted; ++t) {
                bool all = true, waits = false;
                for (size_t i = 0; i < tasks[t].blocks.size(); ++i) {
                    const uint32_t b = tasks[t].blocks[i];
                    if (in(rb, b)) continue;
                    all = false;
                    if (!in(rg, tasks[t].block_groups[i])) {
                        waits = true;
                        break;
                    }
                    if (o_acquire(tasks, rb, true, b, t, limit, cursor, true, act)) {
                        acted = true;
                        break;
                    }
                }
                if (!all || waits) break;
            }
        if (!acted) {
            if (!begun) {
                begun = true;
                act = {2u, 1u, cursor, 0u};
            } else {
                act = {3u, 1u, cursor, 0u};
                begun = false;
                ++cursor;
            }
        }
        trace.push_back(act);
    }
    return 0;
}

}  // namespace

extern "C" {

int chor_plan_task_blocks(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group, int has_accepted,
                          const uint32_t* accepted, uint64_t accepted_count, uint32_t* tasks4_out, uint32_t* ntasks_out) {
    std::vector<std::pair<uint32_t, uint32_t>> tb;
    if (const int rc = task_blocks(image_count, block_images, blocks_per_group, has_accepted, accepted, accepted_count, tb))
        return rc;
    for (size_t t = 0; tasks4_out && t < tb.size(); ++t) {
        tasks4_out[4 * t + 0] = tb[t].first / blocks_per_group;   // block_group_of, scheduler.cpp:24-31
        tasks4_out[4 * t + 1] = tb[t].second / blocks_per_group;
        tasks4_out[4 * t + 2] = tb[t].first;
        tasks4_out[4 * t + 3] = tb[t].second;
    }
    *ntasks_out = static_cast<uint32_t>(tb.size());
    return 0;
}

int chor_simulate_residency(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group, int mode,
                            int has_accepted, const uint32_t* accepted, uint64_t accepted_count,
                            uint32_t* actions4_out, uint64_t capacity, uint64_t* nactions_out) {
    if (image_count == 0 || block_images == 0 || blocks_per_group == 0) return 1;
    std::vector<OTask> tasks;
    if (mode == 0) {  // hashing_residency_tasks, scheduler.cpp:194-200
        const uint32_t nblocks = (image_count + block_images - 1) / block_images;
        for (uint32_t b = 0; b < nblocks; ++b) tasks.push_back(OTask{{b / blocks_per_group}, {b}, {b / blocks_per_group}});
    } else {  // residency_tasks, scheduler.cpp:175-192
        std::vector<std::pair<uint32_t, uint32_t>> tb;
        if (const int rc = task_blocks(image_count, block_images, blocks_per_group, has_accepted, accepted, accepted_count, tb))
            return rc;
        for (const auto& [ba, bb] : tb) {
            OTask t;
            const uint32_t ga = ba / blocks_per_group, gb = bb / blocks_per_group;
            t.groups.push_back(ga);
            if (gb != ga) t.groups.push_back(gb);
            t.blocks.push_back(ba);
            t.block_groups.push_back(ga);
            if (bb != ba) {
                t.blocks.push_back(bb);
                t.block_groups.push_back(gb);
            }
            tasks.push_back(std::move(t));
        }
    }
    std::vector<OAction> trace;
    if (const int rc = o_simulate(tasks, mode == 0 ? 2u : 3u, trace)) return rc;  // residency_slot_limit, scheduler.hpp:70-72
    for (size_t i = 0; actions4_out && i < trace.size() && i < capacity; ++i) {
        actions4_out[4 * i + 0] = trace[i].kind;
        actions4_out[4 * i + 1] = trace[i].level;
        actions4_out[4 * i + 2] = trace[i].id;
        actions4_out[4 * i + 3] = trace[i].prefetch;
    }
    *nactions_out = trace.size();
    return 0;
}

int chor_auto_partition_sizing(uint64_t mean_image_bytes, uint64_t memory_budget_bytes, uint32_t* block_images,
                               uint32_t* blocks_per_group) {
    // scheduler.cpp:347-359: device arena = budget / 4, each level holds three of its units
    const uint64_t per = mean_image_bytes ? mean_image_bytes : 1;
    uint64_t bi = memory_budget_bytes / 4 / per / 3;
    if (bi < 1) bi = 1;
    uint64_t group_bytes = static_cast<uint32_t>(bi) * per;
    if (group_bytes < 1) group_bytes = 1;
    uint64_t bpg = memory_budget_bytes / group_bytes / 3;
    if (bpg < 1) bpg = 1;
    *block_images = static_cast<uint32_t>(bi);
    *blocks_per_group = static_cast<uint32_t>(bpg);
    return 0;
}

}  // extern "C"
