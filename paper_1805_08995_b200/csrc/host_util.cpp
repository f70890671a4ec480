// host_util.cpp — host-only parts of the C ABI: hash-family generation, match-file output and
// pair-list planning.  None of this touches the device; it is compiled into libchgpu.so so a
// caller needs exactly one library for the whole matching path.

#include "../../include/chgpu.h"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

namespace {

// Seed derivation (splitmix64 finaliser composed over (seed, stream, index)); must reproduce
// the values of mix64 in the reference (rng.hpp:18-31) so hyperplanes are identical.
inline uint64_t splitmix_fin(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
inline uint64_t stream_seed(uint64_t seed, uint64_t stream, uint64_t index) {
    return splitmix_fin(splitmix_fin(seed ^ splitmix_fin(stream)) ^ splitmix_fin(index ^ 0xd6e8feb86659fd93ULL));
}

// One hyperplane: 128 Box-Muller normals, two mt19937_64 words per variate (rng.hpp:34-54,
// hashing.cpp:21-26).  libm sqrt/log/cos on the host: same functions the reference calls.
void fill_plane(uint64_t seed, uint64_t stream, uint64_t index, double* dst) {
    std::mt19937_64 gen(stream_seed(seed, stream, index));
    constexpr double kTwoPi = 6.283185307179586476925286766559;
    for (int i = 0; i < 128; ++i) {
        const double a = static_cast<double>(gen() >> 11) * 0x1.0p-53;
        const double b = static_cast<double>(gen() >> 11) * 0x1.0p-53;
        dst[i] = std::sqrt(-2.0 * std::log(1.0 - a)) * std::cos(kTwoPi * b);
    }
}

}  // namespace

extern "C" {

int chgpu_host_check_family(const chgpu_family_params* p) {
    // validate(FamilyParams), hashing.cpp:30-36
    if (p->short_bits < 1 || p->short_bits > 32) return 1;
    if (p->long_bits <= p->short_bits || p->long_bits > 128) return 1;
    if (p->table_count < 1) return 1;
    return 0;
}

chgpu_status chgpu_family_generate(const chgpu_family_params* p, double* short_planes, double* long_planes) {
    if (!p || !short_planes || !long_planes) return CHGPU_EINVAL;
    if (chgpu_host_check_family(p) != 0) return CHGPU_EINVAL;
    for (uint32_t t = 0; t < p->table_count; ++t)
        for (uint32_t j = 0; j < p->short_bits; ++j)
            fill_plane(p->seed, t, j, short_planes + (size_t(t) * p->short_bits + j) * 128);
    // long planes draw from the sentinel stream 0xffffffff so they do not depend on L (hashing.cpp:17-19)
    for (uint32_t j = 0; j < p->long_bits; ++j) fill_plane(p->seed, 0xffffffffULL, j, long_planes + size_t(j) * 128);
    return CHGPU_OK;
}

chgpu_status chgpu_save_matches(const char* image_id_i, const char* image_id_j,
                                const chgpu_match_record* records, uint32_t count, const char* path) {
    if (!image_id_i || !image_id_j || !path || (count && !records)) return CHGPU_EINVAL;
    std::string out;
    out.reserve(64 + size_t(count) * 24);
    out.append("# ").append(image_id_i).append(" ").append(image_id_j).append(" ");
    char buf[64];
    auto put_u = [&](unsigned long long v) {
        const auto r = std::to_chars(buf, buf + sizeof(buf), v);
        out.append(buf, r.ptr);
    };
    put_u(count);
    out.push_back('\n');
    for (uint32_t i = 0; i < count; ++i) {
        put_u(records[i].query_index);
        out.push_back(' ');
        put_u(records[i].train_index);
        out.push_back(' ');
        // shortest decimal that round-trips (feature_io.cpp:48-52); integers print without a point
        const auto r = std::to_chars(buf, buf + sizeof(buf), records[i].distance_sq);
        out.append(buf, r.ptr);
        out.push_back('\n');
    }
    FILE* f = std::fopen(path, "wb");
    if (!f) return CHGPU_EFORMAT;  // FeatureFileFault::Unwritable
    const size_t w = std::fwrite(out.data(), 1, out.size(), f);
    const int c = std::fclose(f);
    return (w == out.size() && c == 0) ? CHGPU_OK : CHGPU_EFORMAT;
}

void chgpu_pair_file_name(uint32_t image_i, uint32_t image_j, char* buf) {
    std::snprintf(buf, 48, "match_%06u_%06u.txt", image_i, image_j);
}

// Exhaustive plan in the reference's locality order (scheduler.cpp:99-142).  Blocks of
// `block_images` consecutive images, groups of `blocks_per_group` consecutive blocks.  For
// every anchor group: boustrophedon sweeps of (anchor block, partner block) against each
// later group, then the anchor group's own block pairs as a chain that starts at the block
// the sweep stopped on, then the pairs inside each block.
chgpu_status chgpu_plan_exhaustive(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group,
                                   uint32_t* pairs_out, uint64_t* npairs_out) {
    if (image_count == 0 || block_images == 0 || blocks_per_group == 0 || !npairs_out) return CHGPU_EINVAL;
    const uint32_t nblocks = (image_count + block_images - 1) / block_images;
    const uint32_t ngroups = (nblocks + blocks_per_group - 1) / blocks_per_group;
    uint64_t np = 0;
    auto block_lo = [&](uint32_t b) { return b * block_images; };
    auto block_hi = [&](uint32_t b) { return std::min(image_count, (b + 1) * block_images); };
    auto emit = [&](uint32_t a, uint32_t b) {
        if (pairs_out) {
            pairs_out[2 * np] = a;
            pairs_out[2 * np + 1] = b;
        }
        ++np;
    };
    auto cross = [&](uint32_t ba, uint32_t bb) {
        if (ba > bb) std::swap(ba, bb);
        for (uint32_t a = block_lo(ba); a < block_hi(ba); ++a)
            for (uint32_t b = block_lo(bb); b < block_hi(bb); ++b) emit(a, b);
    };
    for (uint32_t g = 0; g < ngroups; ++g) {
        const uint32_t a0 = g * blocks_per_group, an = std::min(nblocks, a0 + blocks_per_group) - a0;
        uint32_t j = 0;
        int jdir = +1;
        for (uint32_t h = g + 1; h < ngroups; ++h) {
            const uint32_t b0 = h * blocks_per_group, bn = std::min(nblocks, b0 + blocks_per_group) - b0;
            uint32_t l = 0;
            int ldir = +1;
            for (uint32_t js = 0; js < an; ++js) {
                for (uint32_t ls = 0; ls < bn; ++ls) {
                    cross(a0 + j, b0 + l);
                    if (ls + 1 < bn) l = uint32_t(int(l) + ldir);
                }
                ldir = -ldir;
                if (js + 1 < an) j = uint32_t(int(j) + jdir);
            }
            jdir = -jdir;
        }
        // intra-group block pairs: vertex order = [j, others ascending]; row a pairs with the
        // later vertices ascending on even rows, descending on odd rows
        std::vector<uint32_t> order;
        order.push_back(j);
        for (uint32_t v = 0; v < an; ++v)
            if (v != j) order.push_back(v);
        for (uint32_t a = 0; a + 1 < an; ++a) {
            if (a % 2 == 0)
                for (uint32_t b = a + 1; b < an; ++b) cross(a0 + order[a], a0 + order[b]);
            else
                for (uint32_t b = an; b-- > a + 1;) cross(a0 + order[a], a0 + order[b]);
        }
        for (uint32_t blk = a0; blk < a0 + an; ++blk)
            for (uint32_t a = block_lo(blk); a < block_hi(blk); ++a)
                for (uint32_t b = a + 1; b < block_hi(blk); ++b) emit(a, b);
    }
    *npairs_out = np;
    return CHGPU_OK;
}

void chgpu_shard_range(uint64_t npairs, uint32_t rank, uint32_t world, uint64_t* first, uint64_t* last) {
    if (world == 0) world = 1;
    const uint64_t base = npairs / world, rem = npairs % world;
    const uint64_t f = uint64_t(rank) * base + std::min<uint64_t>(rank, rem);
    *first = f;
    *last = f + base + (rank < rem ? 1 : 0);
}

}  // extern "C"
