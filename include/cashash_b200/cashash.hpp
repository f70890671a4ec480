// cashash.hpp — C++ host side of the B200 Cascade Hashing matcher.
//
// Header-only facade over the C ABI of libchgpu.so (include/chgpu.h) that keeps the reference's
// C++ matcher API for the matching path: same type names, member names, argument meaning and
// exception behaviour as namespace `cashash` of the reference (paths below are relative to
// /root/reference/proj):
//
//     descriptor load   load_features / save_features          include/cashash/feature_io.hpp:85-86
//     hash family       build_hash_family / set_centering      include/cashash/hashing.hpp:74-78
//                       CenteringAccumulator                    include/cashash/hashing.hpp:166-172
//     hash build        compute_codes                           include/cashash/hashing.hpp:131
//     bucket index      build_bucket_index                      include/cashash/matcher.hpp:43
//     match             match_pair                              include/cashash/matcher.hpp:98-100
//     match output      save_matches / pair_file_name           include/cashash/feature_io.hpp:106,
//                                                               include/cashash/engine.hpp:79
//     guided match      guided_match_pair (F as 9 doubles)      include/cashash/geometry.hpp:86-89
//     pair list         plan_exhaustive, plan_guided (flattened, and as PairPlan over a Partition)
//                                                               include/cashash/scheduler.hpp:53-58
//     schedule          make_partition, residency_tasks, simulate_residency, auto_partition_sizing,
//                       assign_workers                          include/cashash/scheduler.hpp:29-134
//
// A caller of the reference switches by including this header and `namespace cashash =
// cashash_b200;`.  The free functions run on a process-wide default
// context for device 0 and serialise on it; they exist for drop-in use and for parity tests
// (match_pair and its variants keep the images they are handed resident by content, so a pair-list
// walk uploads every image once).  Throughput comes from the batch interface, `Matcher`: upload every image once, hash them in
// one launch, match a whole pair list per call.
//
// There is no CPU fallback: every function that computes goes through libchgpu.so and throws
// std::runtime_error when no sm_100 device is present.
//
// Parameter envelope.  The reference accepts short_bits <= 32, any table_count >= 1, any top_k >= 2 and any
// image size (hashing.cpp:30-36, matcher.cpp:9-17); the device path holds short_bits <= 32, any top_k >= 2,
// table_count <= 8 and <= 65,536 points per image (kDeviceMax* below; chgpu.h).  The tuned kernels cover
// short_bits <= 12 and top_k <= 32 (kTunedMax*); beyond that, and for match_pair_filtered with a host callback,
// the same calls run through the general kernels (csrc/general_kernels.cuh) — same results, not tuned.
// Arguments that are valid for the reference but outside the envelope throw `UnsupportedOnDevice` (a
// std::runtime_error) — never a wrong result and never one of the reference's own exception classes, so a
// caller can tell "not offered here" from "invalid".
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <exception>
#include <thread>
#include <vector>

#include "../chgpu.h"

namespace cashash_b200 {

inline constexpr std::size_t kDescriptorDim = 128;
inline constexpr int kMaxReduceRounds = 7;
inline constexpr int kDefaultReduceRounds = 3;
inline constexpr std::size_t kFeatureFileHeaderBytes = 16;
inline constexpr std::size_t kFeatureRecordBytes = 16 + kDescriptorDim;
// the device path's parameter envelope (include/chgpu.h); beyond it: UnsupportedOnDevice
inline constexpr std::uint32_t kDeviceMaxShortBits = 32;  // = the reference's own limit (hashing.cpp:31)
inline constexpr std::uint32_t kDeviceMaxTables = 8;
inline constexpr std::uint32_t kDeviceMaxPoints = 65536;
// what the tuned kernels cover; larger values take the general path
inline constexpr std::uint32_t kTunedMaxShortBits = 12;
inline constexpr std::uint32_t kTunedMaxTopK = 32;

// Arguments the reference accepts and the device path does not hold (see the header comment).
class UnsupportedOnDevice : public std::runtime_error {
public:
    explicit UnsupportedOnDevice(const std::string& what) : std::runtime_error(what) {}
};

// ---- feature_io.hpp types ---------------------------------------------------------------------
struct Keypoint {  // feature_io.hpp:16-23
    float x = 0.0f;
    float y = 0.0f;
    float scale = 0.0f;
    float orientation = 0.0f;
    friend bool operator==(const Keypoint&, const Keypoint&) = default;
};
static_assert(sizeof(Keypoint) == 16, "keypoints travel to the device as float4");

using Descriptor = std::array<std::uint8_t, kDescriptorDim>;  // feature_io.hpp:27

struct FeatureSet {  // feature_io.hpp:29-36
    std::string image_id;
    std::vector<Keypoint> keypoints;
    std::vector<Descriptor> descriptors;
    std::size_t size() const { return keypoints.size(); }
    bool empty() const { return keypoints.empty(); }
};

struct MatchRecord {  // feature_io.hpp:51-57
    std::uint32_t query_index = 0;
    std::uint32_t train_index = 0;
    double distance_sq = 0.0;
    friend bool operator==(const MatchRecord&, const MatchRecord&) = default;
};
static_assert(sizeof(MatchRecord) == sizeof(chgpu_match_record) && sizeof(MatchRecord) == 16,
              "MatchRecord is copied from the device byte for byte");

enum class FeatureFileFault { MissingFile, BadMagic, BadVersion, Truncated, Unwritable };  // feature_io.hpp:61-67

class FeatureFileError : public std::runtime_error {  // feature_io.hpp:69-80
public:
    FeatureFileError(FeatureFileFault fault, const std::filesystem::path& path, std::uint64_t byte_offset,
                     const std::string& detail)
        : std::runtime_error(message(fault, path, byte_offset, detail)), fault_(fault), byte_offset_(byte_offset) {}
    FeatureFileFault fault() const { return fault_; }
    std::uint64_t byte_offset() const { return byte_offset_; }

private:
    static std::string message(FeatureFileFault fault, const std::filesystem::path& path, std::uint64_t offset,
                               const std::string& detail) {
        static const char* const names[] = {"missing file", "bad magic", "unsupported version", "truncated payload",
                                            "unwritable path"};
        std::string s = path.string() + ": " + names[static_cast<int>(fault)] + " at byte " + std::to_string(offset);
        if (!detail.empty()) s += " (" + detail + ")";
        return s;
    }
    FeatureFileFault fault_;
    std::uint64_t byte_offset_;
};

// ---- hashing.hpp types ------------------------------------------------------------------------
struct FamilyParams {  // hashing.hpp:45-52
    std::uint32_t short_bits = 8;
    std::uint32_t long_bits = 128;
    std::uint32_t table_count = 6;
    std::uint64_t seed = 1;
    friend bool operator==(const FamilyParams&, const FamilyParams&) = default;
};

using Hyperplane = std::array<double, kDescriptorDim>;

struct HashFamily {  // hashing.hpp:62-72
    FamilyParams params;
    std::vector<Hyperplane> short_planes;  // [table * short_bits + bit]
    std::vector<Hyperplane> long_planes;   // [bit]
    std::array<double, kDescriptorDim> centering{};
    bool centering_set = false;
    const Hyperplane& short_plane(std::uint32_t table, std::uint32_t bit) const {
        return short_planes[table * params.short_bits + bit];
    }
};

struct ShortCodes {  // hashing.hpp:80-89
    std::uint32_t short_bits = 0;
    std::uint32_t table_count = 0;
    std::uint32_t point_count = 0;
    std::vector<std::uint32_t> values;  // [point * table_count + table]
    std::uint32_t at(std::uint32_t point, std::uint32_t table) const {
        return values[static_cast<std::size_t>(point) * table_count + table];
    }
};

struct LongCode {  // hashing.hpp:91-96
    std::array<std::uint64_t, 2> words{};
    std::uint16_t bits = 0;
    friend bool operator==(const LongCode&, const LongCode&) = default;
};

struct LongCodeSet {
    std::uint32_t long_bits = 0;
    std::vector<LongCode> codes;
};

struct ImageCodes {  // hashing.hpp:110-114
    FamilyParams params;
    ShortCodes shorts;
    LongCodeSet longs;
};

// ---- matcher.hpp types ------------------------------------------------------------------------
struct MatchConfig {  // matcher.hpp:14-23
    std::uint32_t top_k = 10;
    std::uint32_t hamming_threshold = 40;
    double ratio = 0.8;
    std::uint32_t min_candidates_for_ratio = 2;
    int reduce_rounds = kDefaultReduceRounds;
};

struct BucketIndex {  // matcher.hpp:30-41
    struct Table {
        std::vector<std::uint32_t> codes;    // sorted unique bucket codes
        std::vector<std::uint32_t> offsets;  // codes.size() + 1
        std::vector<std::uint32_t> points;   // point ids, bucket-major
    };
    std::uint32_t short_bits = 0;
    std::uint32_t point_count = 0;
    std::vector<Table> tables;

    std::span<const std::uint32_t> bucket(std::uint32_t table, std::uint32_t code) const {
        const Table& t = tables.at(table);
        std::size_t lo = 0, hi = t.codes.size();  // lower_bound over the unique codes (matcher.cpp:19-25)
        while (lo < hi) {
            const std::size_t mid = (lo + hi) / 2;
            if (t.codes[mid] < code) lo = mid + 1;
            else hi = mid;
        }
        if (lo == t.codes.size() || t.codes[lo] != code) return {};
        return {t.points.data() + t.offsets[lo], t.points.data() + t.offsets[lo + 1]};
    }
};

// ---- error mapping ----------------------------------------------------------------------------
namespace detail {

inline chgpu_family_params to_c(const FamilyParams& p) {
    chgpu_family_params c{};
    c.short_bits = p.short_bits;
    c.long_bits = p.long_bits;
    c.table_count = p.table_count;
    c.seed = p.seed;
    return c;
}
inline chgpu_match_cfg to_c(const MatchConfig& m) {
    chgpu_match_cfg c{};
    c.top_k = m.top_k;
    c.hamming_threshold = m.hamming_threshold;
    c.ratio = m.ratio;
    c.min_candidates_for_ratio = m.min_candidates_for_ratio;
    c.reduce_rounds = m.reduce_rounds;
    return c;
}

// chgpu_status -> the exception class the reference throws for the same condition.
[[noreturn]] inline void raise(chgpu_status st, const std::string& msg) {
    switch (st) {
        case CHGPU_EINVAL: throw std::invalid_argument(msg);
        case CHGPU_ELOGIC: throw std::logic_error(msg);
        case CHGPU_ENOMEM: throw std::bad_alloc();
        case CHGPU_ENOTFOUND: throw std::out_of_range(msg);
        case CHGPU_EUNSUPPORTED: throw UnsupportedOnDevice(msg);
        default: throw std::runtime_error(msg + " [" + chgpu_status_name(st) + "]");
    }
}

}  // namespace detail

// ---- host-only operations (no device needed) ----------------------------------------------------
inline void validate(const FamilyParams& p) {  // hashing.cpp:30-36
    if (p.short_bits < 1 || p.short_bits > 32) throw std::invalid_argument("short_bits must be in 1..32");
    if (p.long_bits <= p.short_bits || p.long_bits > 128) throw std::invalid_argument("long_bits must satisfy m < n <= 128");
    if (p.table_count < 1) throw std::invalid_argument("table_count must be >= 1");
}

// build_hash_family (hashing.hpp:74): bit-identical hyperplanes, generated on the host.
inline HashFamily build_hash_family(const FamilyParams& params) {
    validate(params);
    HashFamily f;
    f.params = params;
    f.short_planes.resize(static_cast<std::size_t>(params.table_count) * params.short_bits);
    f.long_planes.resize(params.long_bits);
    const chgpu_family_params c = detail::to_c(params);
    const chgpu_status st = chgpu_family_generate(&c, f.short_planes.front().data(), f.long_planes.front().data());
    if (st != CHGPU_OK) detail::raise(st, "build_hash_family");
    return f;
}

// load_features (feature_io.hpp:85): CHFT file -> FeatureSet, the reference's fault classes and offsets.
inline FeatureSet load_features(const std::filesystem::path& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw FeatureFileError(FeatureFileFault::MissingFile, path, 0, "");
    unsigned char header[kFeatureFileHeaderBytes];
    in.read(reinterpret_cast<char*>(header), sizeof(header));
    if (in.gcount() != static_cast<std::streamsize>(sizeof(header)))
        throw FeatureFileError(FeatureFileFault::Truncated, path, static_cast<std::uint64_t>(in.gcount()), "header");
    if (std::memcmp(header, "CHFT", 4) != 0) throw FeatureFileError(FeatureFileFault::BadMagic, path, 0, "");
    std::uint32_t version = 0, count = 0;
    std::memcpy(&version, header + 4, 4);
    std::memcpy(&count, header + 8, 4);
    if (version != 1)
        throw FeatureFileError(FeatureFileFault::BadVersion, path, 4, "version " + std::to_string(version));
    // one bulk read, then de-interleave; a short file is reported at the byte where it ends
    std::vector<unsigned char> body(static_cast<std::size_t>(count) * kFeatureRecordBytes);
    in.read(reinterpret_cast<char*>(body.data()), static_cast<std::streamsize>(body.size()));
    const std::uint64_t got = static_cast<std::uint64_t>(in.gcount());
    if (got != body.size()) {
        const std::uint64_t rec = got / kFeatureRecordBytes;
        throw FeatureFileError(FeatureFileFault::Truncated, path, kFeatureFileHeaderBytes + got,
                               "record " + std::to_string(rec) + " of " + std::to_string(count));
    }
    FeatureSet fs;
    fs.keypoints.resize(count);
    fs.descriptors.resize(count);
    for (std::uint32_t i = 0; i < count; ++i) {
        const unsigned char* r = body.data() + static_cast<std::size_t>(i) * kFeatureRecordBytes;
        std::memcpy(&fs.keypoints[i], r, 16);
        std::memcpy(fs.descriptors[i].data(), r + 16, kDescriptorDim);
    }
    return fs;
}

inline void save_features(const FeatureSet& fs, const std::filesystem::path& path) {  // feature_io.hpp:86
    if (fs.keypoints.size() != fs.descriptors.size())
        throw std::invalid_argument("feature set keypoint/descriptor length mismatch");
    std::vector<unsigned char> out(kFeatureFileHeaderBytes + fs.size() * kFeatureRecordBytes, 0);
    std::memcpy(out.data(), "CHFT", 4);
    const std::uint32_t version = 1, count = static_cast<std::uint32_t>(fs.size());
    std::memcpy(out.data() + 4, &version, 4);
    std::memcpy(out.data() + 8, &count, 4);
    for (std::size_t i = 0; i < fs.size(); ++i) {
        unsigned char* r = out.data() + kFeatureFileHeaderBytes + i * kFeatureRecordBytes;
        std::memcpy(r, &fs.keypoints[i], 16);
        std::memcpy(r + 16, fs.descriptors[i].data(), kDescriptorDim);
    }
    std::ofstream os(path, std::ios::binary | std::ios::trunc);
    if (!os) throw FeatureFileError(FeatureFileFault::Unwritable, path, 0, "");
    os.write(reinterpret_cast<const char*>(out.data()), static_cast<std::streamsize>(out.size()));
    if (!os) throw FeatureFileError(FeatureFileFault::Unwritable, path, 0, "short write");
}

// save_matches (feature_io.hpp:106-107): byte-identical text.
inline void save_matches(const std::string& image_id_i, const std::string& image_id_j,
                         const std::vector<MatchRecord>& matches, const std::filesystem::path& path) {
    const chgpu_status st =
        chgpu_save_matches(image_id_i.c_str(), image_id_j.c_str(), reinterpret_cast<const chgpu_match_record*>(matches.data()),
                           static_cast<std::uint32_t>(matches.size()), path.string().c_str());
    if (st != CHGPU_OK) throw FeatureFileError(FeatureFileFault::Unwritable, path, 0, "");
}

inline std::string pair_file_name(std::uint32_t i, std::uint32_t j) {  // engine.hpp:79
    char buf[48];
    chgpu_pair_file_name(i, j, buf);
    return buf;
}

// plan_exhaustive (scheduler.hpp:53), flattened in task order: pairs (a < b), a is the query image.
inline std::vector<std::pair<std::uint32_t, std::uint32_t>> plan_exhaustive(std::uint32_t image_count,
                                                                            std::uint32_t block_images,
                                                                            std::uint32_t blocks_per_group) {
    if (image_count == 0 || block_images == 0 || blocks_per_group == 0)
        throw std::invalid_argument("partition: image_count, block_images and blocks_per_group must be >= 1");
    std::vector<std::pair<std::uint32_t, std::uint32_t>> pairs(static_cast<std::size_t>(image_count) * (image_count - 1) / 2);
    static_assert(sizeof(std::pair<std::uint32_t, std::uint32_t>) == 8, "pair list is passed as flat u32");
    std::uint64_t n = 0;
    const chgpu_status st = chgpu_plan_exhaustive(image_count, block_images, blocks_per_group,
                                                  reinterpret_cast<std::uint32_t*>(pairs.data()), &n);
    if (st != CHGPU_OK) detail::raise(st, "plan_exhaustive");
    pairs.resize(n);
    return pairs;
}

// plan_guided (scheduler.hpp:57-58), flattened: the exhaustive traversal restricted to the accepted pairs.
inline std::vector<std::pair<std::uint32_t, std::uint32_t>> plan_guided(
    std::uint32_t image_count, std::uint32_t block_images, std::uint32_t blocks_per_group,
    const std::vector<std::pair<std::uint32_t, std::uint32_t>>& accepted_pairs) {
    if (image_count == 0 || block_images == 0 || blocks_per_group == 0)
        throw std::invalid_argument("partition: image_count, block_images and blocks_per_group must be >= 1");
    std::vector<std::pair<std::uint32_t, std::uint32_t>> pairs(accepted_pairs.size());
    std::uint64_t n = 0;
    const chgpu_status st = chgpu_plan_guided(image_count, block_images, blocks_per_group,
                                              reinterpret_cast<const std::uint32_t*>(accepted_pairs.data()), accepted_pairs.size(),
                                              reinterpret_cast<std::uint32_t*>(pairs.data()), &n);
    if (st == CHGPU_EINVAL) throw std::invalid_argument("plan_guided: self pair or unknown image index");
    if (st != CHGPU_OK) detail::raise(st, "plan_guided");
    pairs.resize(n);
    return pairs;
}

// ---- scheduler.hpp types: partition, tasks, residency schedule --------------------------------------------------
struct Partition {  // scheduler.hpp:14-27
    std::uint32_t image_count = 0;
    std::uint32_t block_images = 0;
    std::uint32_t blocks_per_group = 0;
    std::vector<std::pair<std::uint32_t, std::uint32_t>> block_ranges;  // [first, last) image index per block
    std::vector<std::vector<std::uint32_t>> group_blocks;               // block ids per group
    std::vector<std::uint32_t> block_group_of;                          // group id per block

    std::uint32_t block_count() const { return static_cast<std::uint32_t>(block_ranges.size()); }
    std::uint32_t group_count() const { return static_cast<std::uint32_t>(group_blocks.size()); }
    std::uint32_t block_size(std::uint32_t block) const { return block_ranges[block].second - block_ranges[block].first; }
};

inline Partition make_partition(std::uint32_t image_count, std::uint32_t block_images, std::uint32_t blocks_per_group) {
    if (image_count == 0) throw std::invalid_argument("partition: empty manifest");  // scheduler.cpp:12
    if (block_images == 0 || blocks_per_group == 0)
        throw std::invalid_argument("partition: block_images and blocks_per_group must be >= 1");
    Partition p;
    p.image_count = image_count;
    p.block_images = block_images;
    p.blocks_per_group = blocks_per_group;
    const std::uint32_t nblocks = (image_count + block_images - 1) / block_images;
    p.group_blocks.resize((nblocks + blocks_per_group - 1) / blocks_per_group);
    for (std::uint32_t b = 0; b < nblocks; ++b) {
        const std::uint64_t last = std::min<std::uint64_t>(image_count, std::uint64_t(b + 1) * block_images);
        p.block_ranges.emplace_back(b * block_images, static_cast<std::uint32_t>(last));
        p.block_group_of.push_back(b / blocks_per_group);
        p.group_blocks[b / blocks_per_group].push_back(b);
    }
    return p;
}

struct PlanTask {  // scheduler.hpp:36-40
    std::uint32_t group_a = 0, group_b = 0;
    std::uint32_t block_a = 0, block_b = 0;
    std::vector<std::pair<std::uint32_t, std::uint32_t>> pairs;
};

struct PairPlan {  // scheduler.hpp:42-46
    std::vector<PlanTask> tasks;
    std::size_t pair_count() const {
        std::size_t n = 0;
        for (const PlanTask& t : tasks) n += t.pairs.size();
        return n;
    }
};

namespace detail {
inline PairPlan assemble_plan(const Partition& p, const std::vector<std::pair<std::uint32_t, std::uint32_t>>& flat,
                              const std::uint32_t* accepted, std::uint64_t accepted_count, bool guided) {
    std::uint32_t nt = 0;
    std::uint32_t dummy[2] = {0, 0};
    const std::uint32_t* acc = guided ? (accepted_count ? accepted : dummy) : nullptr;
    chgpu_status st = chgpu_plan_tasks(p.image_count, p.block_images, p.blocks_per_group, acc, accepted_count, nullptr, &nt);
    if (st != CHGPU_OK) raise(st, "plan");
    std::vector<chgpu_plan_task> ts(nt);
    if (nt) {
        st = chgpu_plan_tasks(p.image_count, p.block_images, p.blocks_per_group, acc, accepted_count, ts.data(), &nt);
        if (st != CHGPU_OK) raise(st, "plan");
    }
    PairPlan plan;
    plan.tasks.resize(nt);
    for (std::uint32_t t = 0; t < nt; ++t) {
        PlanTask& out = plan.tasks[t];
        out.group_a = ts[t].group_a;
        out.group_b = ts[t].group_b;
        out.block_a = ts[t].block_a;
        out.block_b = ts[t].block_b;
        out.pairs.assign(flat.begin() + static_cast<std::ptrdiff_t>(ts[t].first_pair),
                         flat.begin() + static_cast<std::ptrdiff_t>(ts[t].first_pair + ts[t].npairs));
    }
    return plan;
}
}  // namespace detail

// The reference's own signatures (scheduler.hpp:53-58): tasks with their pair lists.
inline PairPlan plan_exhaustive(const Partition& p) {
    return detail::assemble_plan(p, plan_exhaustive(p.image_count, p.block_images, p.blocks_per_group), nullptr, 0, false);
}
inline PairPlan plan_guided(const Partition& p, const std::vector<std::pair<std::uint32_t, std::uint32_t>>& accepted_pairs) {
    return detail::assemble_plan(p, plan_guided(p.image_count, p.block_images, p.blocks_per_group, accepted_pairs),
                                 reinterpret_cast<const std::uint32_t*>(accepted_pairs.data()), accepted_pairs.size(), true);
}

// assign_workers (scheduler.hpp:63-64): worker w runs tasks w, w + W, ...
inline std::vector<std::vector<std::uint32_t>> assign_workers(const PairPlan& plan, std::uint32_t worker_count) {
    if (worker_count == 0) throw std::invalid_argument("assign_workers: need >= 1 worker");
    std::vector<std::vector<std::uint32_t>> lists(worker_count);
    for (std::uint32_t t = 0; t < plan.tasks.size(); ++t) lists[t % worker_count].push_back(t);
    return lists;
}

enum class ResidencyMode { Hashing, Matching };  // scheduler.hpp:68
inline constexpr std::uint32_t residency_slot_limit(ResidencyMode mode) { return mode == ResidencyMode::Hashing ? 2u : 3u; }

struct ResidencyTask {  // scheduler.hpp:77-81
    std::vector<std::uint32_t> groups;
    std::vector<std::uint32_t> blocks;
    std::vector<std::uint32_t> block_groups;
};

inline std::vector<ResidencyTask> residency_tasks(const PairPlan& plan) {  // scheduler.hpp:83
    std::vector<ResidencyTask> out;
    out.reserve(plan.tasks.size());
    for (const PlanTask& t : plan.tasks) {
        ResidencyTask r;
        r.groups = t.group_b != t.group_a ? std::vector<std::uint32_t>{t.group_a, t.group_b} : std::vector<std::uint32_t>{t.group_a};
        r.blocks = t.block_b != t.block_a ? std::vector<std::uint32_t>{t.block_a, t.block_b} : std::vector<std::uint32_t>{t.block_a};
        r.block_groups = t.block_b != t.block_a ? std::vector<std::uint32_t>{t.group_a, t.group_b} : std::vector<std::uint32_t>{t.group_a};
        out.push_back(std::move(r));
    }
    return out;
}

inline std::vector<ResidencyTask> hashing_residency_tasks(const Partition& p) {  // scheduler.hpp:84
    std::vector<ResidencyTask> out;
    for (std::uint32_t b = 0; b < p.block_count(); ++b)
        out.push_back(ResidencyTask{{p.block_group_of[b]}, {b}, {p.block_group_of[b]}});
    return out;
}

enum class ActionKind { Load, Evict, Begin, Finish };  // scheduler.hpp:86
enum class ResidencyLevel { Group, Block };            // scheduler.hpp:87

struct ResidencyAction {  // scheduler.hpp:89-94
    ActionKind kind = ActionKind::Load;
    ResidencyLevel level = ResidencyLevel::Group;
    std::uint32_t id = 0;
    bool prefetch = false;
};

// simulate_residency (scheduler.hpp:124-125).  group_slots / block_slots = 0: the reference's limits for `mode`; a
// device with room for more passes its own.  Throws std::logic_error where the reference does (a current load that
// the limits cannot satisfy).
inline std::vector<ResidencyAction> simulate_residency(const std::vector<ResidencyTask>& tasks, ResidencyMode mode,
                                                       std::uint32_t group_slots = 0, std::uint32_t block_slots = 0) {
    std::vector<chgpu_plan_task> ts(tasks.size());
    for (std::size_t t = 0; t < tasks.size(); ++t) {
        const ResidencyTask& r = tasks[t];
        if (r.groups.empty() || r.blocks.empty() || r.groups.size() > 2 || r.blocks.size() > 2 ||
            r.block_groups.size() != r.blocks.size())
            throw std::invalid_argument("simulate_residency: a task names one or two groups and blocks");
        ts[t].group_a = r.block_groups.front();
        ts[t].group_b = r.block_groups.back();
        ts[t].block_a = r.blocks.front();
        ts[t].block_b = r.blocks.back();
    }
    const chgpu_residency_mode m = mode == ResidencyMode::Hashing ? CHGPU_RESIDENCY_HASHING : CHGPU_RESIDENCY_MATCHING;
    std::uint64_t n = 0;
    chgpu_status st = chgpu_simulate_residency(ts.data(), static_cast<std::uint32_t>(ts.size()), m, group_slots, block_slots,
                                               nullptr, 0, &n);
    if (st == CHGPU_EINVAL) throw std::logic_error("residency: current load blocked");
    if (st != CHGPU_OK) detail::raise(st, "simulate_residency");
    std::vector<chgpu_residency_action> raw(n);
    if (n) chgpu_simulate_residency(ts.data(), static_cast<std::uint32_t>(ts.size()), m, group_slots, block_slots, raw.data(), n, &n);
    std::vector<ResidencyAction> trace(n);
    for (std::uint64_t i = 0; i < n; ++i)
        trace[i] = ResidencyAction{static_cast<ActionKind>(raw[i].kind), static_cast<ResidencyLevel>(raw[i].level), raw[i].id,
                                   raw[i].prefetch != 0};
    return trace;
}

struct PartitionSizing {  // scheduler.hpp:129-132
    std::uint32_t block_images = 1;
    std::uint32_t blocks_per_group = 1;
};
inline PartitionSizing auto_partition_sizing(std::uint64_t mean_image_bytes, std::uint64_t memory_budget_bytes) {
    PartitionSizing s;
    chgpu_auto_partition_sizing(mean_image_bytes, memory_budget_bytes, &s.block_images, &s.blocks_per_group);
    return s;
}

// ---- batch interface: one device context ----------------------------------------------------------
// ---- code cache ("CHCC") and centering fingerprint: hashing.hpp:134-157, hashing.cpp:151-272 ------------------
// Files are byte-identical to the reference's and load in either implementation.
inline std::uint64_t centering_fingerprint(const HashFamily& family) {
    return chgpu_centering_fingerprint(family.centering.data());
}

inline void save_code_cache(const ImageCodes& codes, std::uint64_t centering_fp, const std::filesystem::path& path) {
    const chgpu_family_params p = detail::to_c(codes.params);
    std::vector<std::uint64_t> words(codes.longs.codes.size() * 2);
    for (std::size_t i = 0; i < codes.longs.codes.size(); ++i) {
        words[2 * i] = codes.longs.codes[i].words[0];
        words[2 * i + 1] = codes.longs.codes[i].words[1];
    }
    const chgpu_status st = chgpu_save_code_cache(path.string().c_str(), &p, centering_fp,
                                                  static_cast<std::uint32_t>(codes.longs.codes.size()),
                                                  codes.shorts.values.data(), words.data());
    if (st != CHGPU_OK) throw FeatureFileError(FeatureFileFault::Unwritable, path, 0, "");
}

struct CodeCacheHeader {  // hashing.hpp:146-150
    FamilyParams params;
    std::uint64_t centering_fp = 0;
    std::uint32_t count = 0;
};

// Reads just the header; false on a missing file or foreign magic (hashing.cpp:208-226).
inline bool read_code_cache_header(const std::filesystem::path& path, CodeCacheHeader& header) {
    chgpu_family_params p{};
    std::uint64_t fp = 0;
    std::uint32_t count = 0;
    if (chgpu_read_code_cache_header(path.string().c_str(), &p, &fp, &count) != CHGPU_OK) return false;
    header.params = FamilyParams{p.short_bits, p.long_bits, p.table_count, p.seed};
    header.centering_fp = fp;
    header.count = count;
    return true;
}

// Loads a cache; throws std::runtime_error if the echoed parameters or the fingerprint mismatch, FeatureFileError
// for a missing / foreign / truncated file (hashing.cpp:228-272).
inline ImageCodes load_code_cache(const std::filesystem::path& path, const FamilyParams& expected,
                                  std::uint64_t expected_centering_fp) {
    const chgpu_family_params p = detail::to_c(expected);
    ImageCodes out;
    std::vector<std::uint64_t> words;
    std::uint32_t count = 0;
    chgpu_file_fault fault = CHGPU_FAULT_NONE;
    std::uint64_t off = 0;
    chgpu_status st = chgpu_load_code_cache(path.string().c_str(), &p, expected_centering_fp, 0, &count, nullptr, nullptr,
                                            &fault, &off);
    if (st == CHGPU_ENOMEM) {  // the probe told us the count: now with room for the payload
        out.shorts.values.resize(static_cast<std::size_t>(count) * expected.table_count);
        words.resize(static_cast<std::size_t>(count) * 2);
        st = chgpu_load_code_cache(path.string().c_str(), &p, expected_centering_fp, count, &count, out.shorts.values.data(),
                                   words.data(), &fault, &off);
    }
    if (st == CHGPU_EFORMAT) throw FeatureFileError(static_cast<FeatureFileFault>(int(fault) - 1), path, off, "");
    if (st == CHGPU_EMISMATCH) throw std::runtime_error(path.string() + ": code cache parameters mismatch active config");
    if (st != CHGPU_OK) detail::raise(st, "load_code_cache");
    out.params = expected;
    out.shorts.short_bits = expected.short_bits;
    out.shorts.table_count = expected.table_count;
    out.shorts.point_count = count;
    out.longs.long_bits = expected.long_bits;
    out.longs.codes.resize(count);
    for (std::uint32_t i = 0; i < count; ++i) {
        out.longs.codes[i].words = {words[2 * i], words[2 * i + 1]};
        out.longs.codes[i].bits = static_cast<std::uint16_t>(expected.long_bits);
    }
    return out;
}

struct MatchStats : chgpu_match_stats {};

struct PairMatches {  // what the reference's sink receives (engine.cpp:145-160), one per pair
    std::uint32_t image_i = 0, image_j = 0;
    std::vector<MatchRecord> matches;
};

class Matcher {
public:
    explicit Matcher(int device = 0) {
        const chgpu_status st = chgpu_create(device, &ctx_);
        if (st != CHGPU_OK)
            throw std::runtime_error(std::string("chgpu_create failed: ") + chgpu_status_name(st) +
                                     " (an sm_100 CUDA device is required; there is no CPU fallback)");
    }
    ~Matcher() { chgpu_destroy(ctx_); }
    Matcher(const Matcher&) = delete;
    Matcher& operator=(const Matcher&) = delete;

    chgpu_ctx* handle() const { return ctx_; }

    void set_family(const HashFamily& family) {
        const chgpu_family_params c = detail::to_c(family.params);
        ck(chgpu_set_family(ctx_, &c, family.short_planes.front().data(), family.long_planes.front().data()));
        params_ = family.params;
        if (family.centering_set) ck(chgpu_set_centering(ctx_, family.centering.data()));
    }
    const FamilyParams& params() const { return params_; }

    // descriptor load: FeatureSet -> resident image (engine.cpp:394-412)
    void upload(std::uint32_t image_id, const FeatureSet& fs) {
        if (fs.keypoints.size() != fs.descriptors.size())
            throw std::invalid_argument("feature set keypoint/descriptor length mismatch");
        ck(chgpu_upload_image(ctx_, image_id, static_cast<std::uint32_t>(fs.size()),
                              fs.empty() ? nullptr : fs.descriptors.front().data(),
                              fs.empty() ? nullptr : &fs.keypoints.front().x));
    }
    // descriptor load straight from CHFT bytes (parse_features_blob, engine.cpp:458-488)
    std::uint32_t upload_chft(std::uint32_t image_id, const void* blob, std::size_t nbytes,
                              const std::filesystem::path& origin = "<memory>") {
        std::uint32_t count = 0;
        chgpu_file_fault fault = CHGPU_FAULT_NONE;
        std::uint64_t off = 0;
        const chgpu_status st = chgpu_upload_chft(ctx_, image_id, blob, nbytes, &count, &fault, &off);
        if (st == CHGPU_EFORMAT) throw FeatureFileError(static_cast<FeatureFileFault>(int(fault) - 1), origin, off, "");
        ck(st);
        return count;
    }
    void evict(std::uint32_t image_id) { ck(chgpu_evict_image(ctx_, image_id)); }

    // centering pass (hashing.cpp:52-70): exact integer sums on the device, one division on the host
    void centering_reset() { ck(chgpu_centering_reset(ctx_)); }
    void centering_add(std::uint32_t image_id) { ck(chgpu_centering_add_image(ctx_, image_id)); }
    void centering_add(std::span<const std::uint32_t> image_ids) {  // one launch over all listed images
        ck(chgpu_centering_add_images(ctx_, image_ids.data(), static_cast<std::uint32_t>(image_ids.size())));
    }
    std::array<double, kDescriptorDim> centering_apply() {
        std::array<double, kDescriptorDim> c{};
        ck(chgpu_centering_apply(ctx_, c.data()));
        return c;
    }

    // hash build + bucket index for resident images (compute_codes + build_bucket_index)
    void hash(std::span<const std::uint32_t> image_ids, int reduce_rounds = kDefaultReduceRounds) {
        ck(chgpu_hash_images(ctx_, image_ids.data(), static_cast<std::uint32_t>(image_ids.size()), reduce_rounds));
    }
    // How the hyperplane signs are evaluated (both exact): fp32 filter with an error bound + fp64 re-evaluation
    // of the undecided dots (default), or every dot in reduce_dot's fp64 order (hashing.hpp:24-43).
    void set_exact_hashing(bool exact) { ck(chgpu_set_hash_mode(ctx_, exact ? CHGPU_HASH_EXACT : CHGPU_HASH_TENSOR)); }
    void set_hash_mode(chgpu_hash_mode mode) { ck(chgpu_set_hash_mode(ctx_, mode)); }  // TENSOR (default) / FILTERED / EXACT
    chgpu_hash_stats hash_stats() {
        chgpu_hash_stats st{};
        ck(chgpu_get_hash_stats(ctx_, &st));
        return st;
    }
    ImageCodes codes(std::uint32_t image_id) {
        std::uint32_t n = 0;
        ck(chgpu_image_points(ctx_, image_id, &n));
        ImageCodes out;
        out.params = params_;
        out.shorts.short_bits = params_.short_bits;
        out.shorts.table_count = params_.table_count;
        out.shorts.point_count = n;
        out.shorts.values.resize(static_cast<std::size_t>(n) * params_.table_count);
        std::vector<std::uint64_t> words(static_cast<std::size_t>(n) * 2);
        ck(chgpu_download_codes(ctx_, image_id, out.shorts.values.data(), words.data()));
        out.longs.long_bits = params_.long_bits;
        out.longs.codes.resize(n);
        for (std::uint32_t p = 0; p < n; ++p) {
            out.longs.codes[p].words = {words[2 * p], words[2 * p + 1]};
            out.longs.codes[p].bits = static_cast<std::uint16_t>(params_.long_bits);
        }
        return out;
    }
    void upload_codes(std::uint32_t image_id, const ImageCodes& codes) {
        std::vector<std::uint64_t> words(codes.longs.codes.size() * 2);
        for (std::size_t p = 0; p < codes.longs.codes.size(); ++p) {
            words[2 * p] = codes.longs.codes[p].words[0];
            words[2 * p + 1] = codes.longs.codes[p].words[1];
        }
        static const std::uint32_t none32 = 0;
        static const std::uint64_t none64 = 0;
        ck(chgpu_upload_codes(ctx_, image_id, codes.shorts.values.empty() ? &none32 : codes.shorts.values.data(),
                              words.empty() ? &none64 : words.data()));
    }
    BucketIndex bucket_index(std::uint32_t image_id) {
        std::uint32_t n = 0;
        ck(chgpu_image_points(ctx_, image_id, &n));
        const std::uint32_t L = params_.table_count, nb = 1u << params_.short_bits;
        std::vector<std::uint32_t> offs(static_cast<std::size_t>(L) * (nb + 1)), pts(static_cast<std::size_t>(L) * n);
        ck(chgpu_download_bucket_index(ctx_, image_id, offs.data(), pts.data()));
        BucketIndex idx;
        idx.short_bits = params_.short_bits;
        idx.point_count = n;
        idx.tables.resize(L);
        for (std::uint32_t t = 0; t < L; ++t) {  // dense CSR -> CSR over the non-empty codes (matcher.cpp:27-51)
            BucketIndex::Table& tb = idx.tables[t];
            const std::uint32_t* o = offs.data() + static_cast<std::size_t>(t) * (nb + 1);
            for (std::uint32_t c = 0; c < nb; ++c)
                if (o[c + 1] != o[c]) {
                    tb.codes.push_back(c);
                    tb.offsets.push_back(o[c]);
                }
            tb.offsets.push_back(n);
            tb.points.assign(pts.begin() + static_cast<std::size_t>(t) * n, pts.begin() + static_cast<std::size_t>(t + 1) * n);
        }
        return idx;
    }

    // match a pair list; results in pair order, records of a pair ascending in query index
    std::vector<PairMatches> match_pairs(std::span<const std::pair<std::uint32_t, std::uint32_t>> pairs,
                                         const MatchConfig& cfg, MatchStats* stats = nullptr) {
        std::vector<PairMatches> out(pairs.size());
        for (std::size_t k = 0; k < pairs.size(); ++k) {
            out[k].image_i = pairs[k].first;
            out[k].image_j = pairs[k].second;
        }
        match_pairs_stream(pairs, cfg,
                           [&](std::uint32_t first, std::span<const std::uint64_t> offs, std::span<const MatchRecord> rec) {
                               for (std::size_t k = 0; k + 1 < offs.size(); ++k)
                                   out[first + k].matches.assign(rec.begin() + offs[k], rec.begin() + offs[k + 1]);
                           },
                           stats);
        return out;
    }

    // streaming form: sink(first_pair, offsets (k+1), records) per sub-batch, in pair order, while
    // the next sub-batch is already computing (FileMatchSink::accept, engine.cpp:154-160)
    using Sink = std::function<void(std::uint32_t, std::span<const std::uint64_t>, std::span<const MatchRecord>)>;
    void match_pairs_stream(std::span<const std::pair<std::uint32_t, std::uint32_t>> pairs, const MatchConfig& cfg,
                            const Sink& sink, MatchStats* stats = nullptr) {
        const chgpu_match_cfg c = detail::to_c(cfg);
        struct Thunk {
            const Sink* sink;
            std::exception_ptr error;
        } thunk{&sink, nullptr};
        auto trampoline = [](void* user, std::uint32_t first, std::uint32_t count, const std::uint64_t* offs,
                             const chgpu_match_record* rec) -> int {
            Thunk* t = static_cast<Thunk*>(user);
            try {
                (*t->sink)(first, {offs, static_cast<std::size_t>(count) + 1},
                           {reinterpret_cast<const MatchRecord*>(rec), static_cast<std::size_t>(offs[count])});
                return 0;
            } catch (...) {
                t->error = std::current_exception();
                return 1;
            }
        };
        const chgpu_status st =
            chgpu_match_pairs_stream(ctx_, reinterpret_cast<const std::uint32_t*>(pairs.data()),
                                     static_cast<std::uint32_t>(pairs.size()), &c, trampoline, &thunk, stats);
        if (thunk.error) std::rethrow_exception(thunk.error);
        ck(st);
    }

    // centering_pass (engine.cpp:545-559) over CHFT files, block by block, nothing left resident; files that fail are
    // reported in `failures` (what() of the FeatureFileError the reference would have collected) and left out.
    std::array<double, kDescriptorDim> centering_pass_files(const std::vector<std::filesystem::path>& files,
                                                             std::uint32_t block_images, std::uint32_t io_threads = 8,
                                                             std::vector<std::string>* failures = nullptr) {
        std::vector<std::string> store;
        std::vector<const char*> cpaths;
        for (const auto& f : files) store.push_back(f.string());
        for (const auto& f : store) cpaths.push_back(f.c_str());
        std::vector<chgpu_file_result> res(files.size());
        std::array<double, kDescriptorDim> c{};
        const chgpu_status st = chgpu_centering_pass_files(ctx_, cpaths.data(), static_cast<std::uint32_t>(files.size()),
                                                           block_images, io_threads, res.data(), c.data());
        collect_failures(files, res, failures);
        if (st == CHGPU_EINVAL) throw std::invalid_argument("centering: no descriptors in the stream");  // hashing.cpp:60
        ck(st);
        return c;
    }

    // Out-of-core run of a plan (execute_plan + ResidencyDriver, engine.cpp:252-456, :667-702): at most block_slots
    // blocks of block_images images resident (0 = the reference's 3), the next block loading behind the current task.
    // sink(task, pairs, offsets (k+1), records) per chunk, in plan order.  accepted == nullptr: the exhaustive plan.
    using PlanSink = std::function<void(std::uint32_t, std::span<const std::pair<std::uint32_t, std::uint32_t>>,
                                        std::span<const std::uint64_t>, std::span<const MatchRecord>)>;
    chgpu_streamed_stats match_plan_streamed(const std::vector<std::filesystem::path>& files, const Partition& partition,
                                             const MatchConfig& cfg, const PlanSink& sink,
                                             const std::vector<std::pair<std::uint32_t, std::uint32_t>>* accepted = nullptr,
                                             std::uint32_t group_slots = 0, std::uint32_t block_slots = 0,
                                             std::uint32_t io_threads = 8, std::vector<std::string>* failures = nullptr,
                                             chgpu_task_order task_order = CHGPU_ORDER_REFERENCE, std::uint32_t shard = 0,
                                             std::uint32_t shards = 1) {
        if (partition.image_count != files.size()) throw std::invalid_argument("match_plan_streamed: one file per image");
        std::vector<std::string> store;
        std::vector<const char*> cpaths;
        for (const auto& f : files) store.push_back(f.string());
        for (const auto& f : store) cpaths.push_back(f.c_str());
        std::vector<chgpu_file_result> res(files.size());
        const chgpu_match_cfg c = detail::to_c(cfg);
        struct Thunk {
            const PlanSink* sink;
            std::exception_ptr error;
        } thunk{&sink, nullptr};
        auto trampoline = [](void* user, std::uint32_t task, const std::uint32_t* pairs, std::uint32_t count,
                             const std::uint64_t* offs, const chgpu_match_record* rec) -> int {
            Thunk* t = static_cast<Thunk*>(user);
            try {
                if (*t->sink)
                    (*t->sink)(task, {reinterpret_cast<const std::pair<std::uint32_t, std::uint32_t>*>(pairs), count},
                               {offs, static_cast<std::size_t>(count) + 1},
                               {reinterpret_cast<const MatchRecord*>(rec), static_cast<std::size_t>(offs[count])});
                return 0;
            } catch (...) {
                t->error = std::current_exception();
                return 1;
            }
        };
        static const std::uint32_t none[2] = {0, 0};
        const std::uint32_t* acc = !accepted ? nullptr : (accepted->empty() ? none : reinterpret_cast<const std::uint32_t*>(accepted->data()));
        chgpu_streamed_stats stats{};
        const chgpu_status st = chgpu_match_plan_streamed(
            ctx_, cpaths.data(), partition.image_count, partition.block_images, partition.blocks_per_group, group_slots, block_slots,
            task_order, shard, shards, acc, accepted ? accepted->size() : 0, &c, io_threads, trampoline, &thunk, res.data(), &stats);
        if (thunk.error) std::rethrow_exception(thunk.error);
        collect_failures(files, res, failures);
        if (st == CHGPU_EINVAL) throw std::invalid_argument("match_plan_streamed: bad pair list, or slot limits below what one task needs");
        ck(st);
        return stats;
    }

    // match_pair_filtered (matcher.hpp:102-105) for two resident images with a HOST callback: the candidate lists are
    // formed on the device (matcher.cpp:164-171), `filter` is called on this thread for every query with a non-empty
    // list, in query order (matcher.cpp:172; its return value is ignored there as well), and whatever it leaves in the
    // vector — fewer entries, another order, repeats — is ranked and verified on the device (matcher.cpp:173-192).
    std::vector<MatchRecord> match_pair_filtered(std::uint32_t image_i, std::uint32_t image_j, const MatchConfig& cfg,
                                                 const std::function<bool(std::uint32_t, std::vector<std::uint32_t>&)>& filter,
                                                 chgpu_match_stats* stats = nullptr) {
        std::uint32_t nq = 0;
        ck(chgpu_image_points(ctx_, image_i, &nq));
        std::vector<std::uint64_t> offs(std::size_t(nq) + 1, 0);
        std::uint64_t total = 0;
        chgpu_status st = chgpu_pair_candidates(ctx_, image_i, image_j, offs.data(), nullptr, 0, &total);
        if (st != CHGPU_ENOMEM) ck(st);
        std::vector<std::uint32_t> cands(std::max<std::uint64_t>(total, 1));
        if (total) ck(chgpu_pair_candidates(ctx_, image_i, image_j, offs.data(), cands.data(), total, &total));
        std::vector<std::uint64_t> new_offs(std::size_t(nq) + 1, 0);
        std::vector<std::uint32_t> ids;
        ids.reserve(total);
        std::vector<std::uint32_t> one;
        for (std::uint32_t q = 0; q < nq; ++q) {
            one.assign(cands.begin() + offs[q], cands.begin() + offs[q + 1]);
            if (filter && !one.empty()) filter(q, one);
            ids.insert(ids.end(), one.begin(), one.end());
            new_offs[q + 1] = ids.size();
        }
        const chgpu_match_cfg c = detail::to_c(cfg);
        std::vector<MatchRecord> out(std::max<std::uint32_t>(nq, 1));
        static_assert(sizeof(MatchRecord) == sizeof(chgpu_match_record), "record layout");
        std::uint64_t count = 0;
        st = chgpu_match_pair_lists(ctx_, image_i, image_j, &c, new_offs.data(), ids.empty() ? nullptr : ids.data(),
                                    reinterpret_cast<chgpu_match_record*>(out.data()), nq, &count, stats);
        if (st == CHGPU_EINVAL) throw std::invalid_argument(chgpu_last_error(ctx_));
        ck(st);
        out.resize(count);
        return out;
    }

    // epipolar-guided pair list (guided_match_pair, geometry.cpp:234-250): one row-major 3x3 F per pair
    std::vector<PairMatches> match_pairs_guided(std::span<const std::pair<std::uint32_t, std::uint32_t>> pairs,
                                                std::span<const std::array<double, 9>> fmats, double band_px,
                                                const MatchConfig& cfg, MatchStats* stats = nullptr) {
        if (fmats.size() != pairs.size()) throw std::invalid_argument("guided match: one fundamental matrix per pair");
        std::vector<PairMatches> out(pairs.size());
        for (std::size_t k = 0; k < pairs.size(); ++k) {
            out[k].image_i = pairs[k].first;
            out[k].image_j = pairs[k].second;
        }
        const chgpu_match_cfg c = detail::to_c(cfg);
        struct Fill {
            std::vector<PairMatches>* out;
        } fill{&out};
        auto trampoline = [](void* user, std::uint32_t first, std::uint32_t count, const std::uint64_t* offs,
                             const chgpu_match_record* rec) -> int {
            auto* o = static_cast<Fill*>(user)->out;
            const MatchRecord* r = reinterpret_cast<const MatchRecord*>(rec);
            for (std::uint32_t k = 0; k < count; ++k) (*o)[first + k].matches.assign(r + offs[k], r + offs[k + 1]);
            return 0;
        };
        ck(chgpu_match_pairs_guided_stream(ctx_, reinterpret_cast<const std::uint32_t*>(pairs.data()),
                                           static_cast<std::uint32_t>(pairs.size()), &c,
                                           fmats.empty() ? nullptr : fmats.front().data(), band_px, trampoline, &fill, stats));
        return out;
    }

    void sync() { ck(chgpu_sync(ctx_)); }

private:
    void ck(chgpu_status st) const {
        if (st != CHGPU_OK) detail::raise(st, chgpu_last_error(ctx_));
    }
    // per-file outcomes of a streamed load as the strings the reference collects (engine.cpp:315-318)
    static void collect_failures(const std::vector<std::filesystem::path>& files, const std::vector<chgpu_file_result>& res,
                                 std::vector<std::string>* failures) {
        if (!failures) return;
        for (std::size_t i = 0; i < files.size(); ++i) {
            if (res[i].status == CHGPU_OK) continue;
            if (res[i].status == CHGPU_EFORMAT)
                failures->push_back(FeatureFileError(static_cast<FeatureFileFault>(res[i].fault - 1), files[i], res[i].fault_offset, "").what());
            else
                failures->push_back(files[i].string() + ": " + chgpu_status_name(static_cast<chgpu_status>(res[i].status)));
        }
    }
    chgpu_ctx* ctx_ = nullptr;
    FamilyParams params_{};
};

// ---- reference-shaped free functions over a default context ---------------------------------------
namespace detail {

struct DefaultContext {
    std::mutex mu;
    std::unique_ptr<Matcher> matcher;
    const HashFamily* installed = nullptr;
    FamilyParams installed_params{};
    bool has_family = false;

    // Images the free match functions have uploaded, kept resident by CONTENT: a caller that walks a pair list with
    // match_pair (the reference's worker loop, engine.cpp:686-696) hands over every image K - 1 times; the second time
    // its descriptors, keypoints and codes are already on the device with their bucket index built.  Keyed by a 64-bit
    // hash of all the bytes handed over (plus point count and family parameters), least recently used out first.
    struct CachedImage {
        std::uint64_t key;
        std::uint32_t id, points;
        std::uint64_t stamp;
    };
    static constexpr std::size_t kCachedImages = 64;
    std::vector<CachedImage> cache;
    std::uint64_t cache_clock = 0, cache_hits = 0, cache_misses = 0;
    std::uint32_t cache_next = 0;

    static std::uint64_t hash_bytes(std::uint64_t h, const void* p, std::size_t bytes) {
        const unsigned char* b = static_cast<const unsigned char*>(p);
        std::uint64_t h2 = h ^ 0x9e3779b97f4a7c15ull;
        std::size_t i = 0;
        for (; i + 16 <= bytes; i += 16) {  // two independent lanes
            std::uint64_t w0, w1;
            std::memcpy(&w0, b + i, 8);
            std::memcpy(&w1, b + i + 8, 8);
            h = (h ^ w0) * 0xff51afd7ed558ccdull;
            h ^= h >> 32;
            h2 = (h2 ^ w1) * 0xc4ceb9fe1a85ec53ull;
            h2 ^= h2 >> 29;
        }
        for (; i < bytes; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
        h ^= h2 + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
        return (h ^ (h >> 31)) * 0xd6e8feb86659fd93ull;
    }
    void drop_cache() {
        for (const CachedImage& c : cache) {
            try {
                matcher->evict(c.id);
            } catch (...) {
            }
        }
        cache.clear();
    }
    // Resident image id for (fs, codes): uploaded now or found from an earlier call.
    std::uint32_t resident(Matcher& m, const FeatureSet& fs, const ImageCodes& codes) {
        std::uint64_t key = 0x243f6a8885a308d3ull ^ fs.size();
        const FamilyParams& p = codes.params;
        const std::uint64_t pp[4] = {p.short_bits, p.long_bits, p.table_count, p.seed};
        key = hash_bytes(key, pp, sizeof(pp));
        if (!fs.empty()) {
            key = hash_bytes(key, fs.descriptors.data(), fs.size() * kDescriptorDim);
            key = hash_bytes(key, fs.keypoints.data(), fs.keypoints.size() * sizeof(Keypoint));
            key = hash_bytes(key, codes.shorts.values.data(), codes.shorts.values.size() * sizeof(std::uint32_t));
            for (const LongCode& c : codes.longs.codes) key = hash_bytes(key, c.words.data(), 16);  // (the struct has padding)
        }
        for (CachedImage& c : cache)
            if (c.key == key && c.points == fs.size()) {
                c.stamp = ++cache_clock;
                ++cache_hits;
                return c.id;
            }
        ++cache_misses;
        if (cache.size() >= kCachedImages) {
            std::size_t lru = 0;
            for (std::size_t i = 1; i < cache.size(); ++i)
                if (cache[i].stamp < cache[lru].stamp) lru = i;
            m.evict(cache[lru].id);
            cache.erase(cache.begin() + lru);
        }
        const std::uint32_t id = 0xE1000000u + (cache_next++ & 0x00FFFFFFu);
        m.upload(id, fs);
        try {
            m.upload_codes(id, codes);
        } catch (...) {
            try {
                m.evict(id);
            } catch (...) {
            }
            throw;
        }
        cache.push_back(CachedImage{key, id, std::uint32_t(fs.size()), ++cache_clock});
        return id;
    }

    // Installs `family` (planes + centering) unless it is the one already resident.
    Matcher& with(const HashFamily& family) {
        if (!matcher) matcher = std::make_unique<Matcher>(0);
        if (!has_family || installed != &family || !(installed_params == family.params)) {
            drop_cache();  // image blocks are laid out per family
            matcher->set_family(family);
            installed = &family;
            installed_params = family.params;
            has_family = true;
        } else if (family.centering_set) {
            // same object, possibly re-centered since the last call
            if (chgpu_set_centering(matcher->handle(), family.centering.data()) != CHGPU_OK)
                throw std::runtime_error(chgpu_last_error(matcher->handle()));
        }
        return *matcher;
    }
};

inline DefaultContext& default_context() {
    static DefaultContext ctx;
    return ctx;
}

inline constexpr std::uint32_t kScratchA = 0xE0000000u, kScratchB = 0xE0000001u;

struct ScopedImage {  // evicts a scratch image on every exit path
    Matcher& m;
    std::uint32_t id;
    ~ScopedImage() {
        try {
            m.evict(id);
        } catch (...) {
        }
    }
};

}  // namespace detail

// Streaming accumulator behind set_centering (hashing.hpp:166-172).  add() sums on the device.
struct CenteringAccumulator {
    std::array<std::uint64_t, kDescriptorDim> sums{};
    std::uint64_t count = 0;

    void add(const FeatureSet& fs) {
        if (fs.empty()) return;
        detail::DefaultContext& dc = detail::default_context();
        std::lock_guard<std::mutex> lock(dc.mu);
        if (!dc.matcher) dc.matcher = std::make_unique<Matcher>(0);
        Matcher& m = *dc.matcher;
        if (!dc.has_family) {  // image blocks are laid out per family; any valid one will do for a sum
            static const HashFamily scratch = build_hash_family(FamilyParams{});
            m.set_family(scratch);
            dc.installed = &scratch;
            dc.installed_params = scratch.params;
            dc.has_family = true;
        }
        m.upload(detail::kScratchA, fs);
        detail::ScopedImage guard{m, detail::kScratchA};
        m.centering_reset();
        m.centering_add(detail::kScratchA);
        std::array<std::uint64_t, kDescriptorDim> part{};
        std::uint64_t n = 0;
        if (chgpu_centering_get_sums(m.handle(), part.data(), &n) != CHGPU_OK)
            throw std::runtime_error(chgpu_last_error(m.handle()));
        for (std::size_t c = 0; c < kDescriptorDim; ++c) sums[c] += part[c];
        count += n;
    }
    void apply(HashFamily& family) const {  // hashing.cpp:59-64
        if (count == 0) throw std::invalid_argument("set_centering: no descriptors");
        for (std::size_t c = 0; c < kDescriptorDim; ++c)
            family.centering[c] = static_cast<double>(sums[c]) / static_cast<double>(count);
        family.centering_set = true;
    }
};

inline void set_centering(HashFamily& family, std::span<const FeatureSet> sets) {  // hashing.hpp:78
    CenteringAccumulator acc;
    for (const FeatureSet& fs : sets) acc.add(fs);
    acc.apply(family);
}

// compute_codes (hashing.hpp:131): fp64 sign tests in the reference's summation order, on the device.
inline ImageCodes compute_codes(const HashFamily& family, const FeatureSet& fs, int reduce_rounds = kDefaultReduceRounds) {
    if (!family.centering_set) throw std::logic_error("compute_codes: centering has not been set");
    if (reduce_rounds < 0 || reduce_rounds > kMaxReduceRounds)
        throw std::invalid_argument("reduce_dot tail rounds out of range 0..7");
    detail::DefaultContext& dc = detail::default_context();
    std::lock_guard<std::mutex> lock(dc.mu);
    Matcher& m = dc.with(family);
    m.upload(detail::kScratchA, fs);
    detail::ScopedImage guard{m, detail::kScratchA};
    const std::uint32_t id = detail::kScratchA;
    m.hash({&id, 1}, reduce_rounds);
    return m.codes(id);
}

// build_bucket_index (matcher.hpp:43): counting sort on the device, returned in the reference's CSR form.
inline BucketIndex build_bucket_index(const ShortCodes& train_codes) {
    FamilyParams p;
    p.short_bits = train_codes.short_bits;
    p.table_count = train_codes.table_count;
    p.long_bits = std::max<std::uint32_t>(p.short_bits + 1, 128);
    static std::mutex fam_mu;
    static std::vector<std::unique_ptr<HashFamily>> families;  // one resident family object per (m, L)
    const HashFamily* fam = nullptr;
    {
        std::lock_guard<std::mutex> lock(fam_mu);
        for (const auto& f : families)
            if (f->params == p) fam = f.get();
        if (!fam) {
            families.push_back(std::make_unique<HashFamily>(build_hash_family(p)));
            fam = families.back().get();
        }
    }
    detail::DefaultContext& dc = detail::default_context();
    std::lock_guard<std::mutex> lock(dc.mu);
    Matcher& m = dc.with(*fam);
    FeatureSet blank;
    blank.keypoints.resize(train_codes.point_count);
    blank.descriptors.resize(train_codes.point_count);
    m.upload(detail::kScratchA, blank);
    detail::ScopedImage guard{m, detail::kScratchA};
    ImageCodes codes;
    codes.params = p;
    codes.shorts = train_codes;
    codes.longs.long_bits = p.long_bits;
    codes.longs.codes.resize(train_codes.point_count);
    m.upload_codes(detail::kScratchA, codes);
    return m.bucket_index(detail::kScratchA);
}

// match_pair (matcher.hpp:98-100) with externally supplied codes: one pair through the batch path.
// The hash family is only needed for its parameters here (codes are given), so any HashFamily with
// codes_i.params is installed.
inline std::vector<MatchRecord> match_pair(const FeatureSet& fs_i, const FeatureSet& fs_j, const ImageCodes& codes_i,
                                           const ImageCodes& codes_j, const MatchConfig& cfg) {
    if (!(codes_i.params == codes_j.params))
        throw std::invalid_argument("match_pair: codes come from different hash families");  // matcher.cpp:144
    if (codes_i.shorts.point_count != fs_i.size() || codes_j.shorts.point_count != fs_j.size())
        throw std::invalid_argument("match_pair: code/point count mismatch");  // matcher.cpp:146-148
    static std::mutex fam_mu;
    static std::vector<std::unique_ptr<HashFamily>> families;
    const HashFamily* fam = nullptr;
    {
        std::lock_guard<std::mutex> lock(fam_mu);
        for (const auto& f : families)
            if (f->params == codes_i.params) fam = f.get();
        if (!fam) {
            families.push_back(std::make_unique<HashFamily>(build_hash_family(codes_i.params)));
            fam = families.back().get();
        }
    }
    detail::DefaultContext& dc = detail::default_context();
    std::lock_guard<std::mutex> lock(dc.mu);
    Matcher& m = dc.with(*fam);
    const std::pair<std::uint32_t, std::uint32_t> pr{dc.resident(m, fs_i, codes_i), dc.resident(m, fs_j, codes_j)};
    std::vector<PairMatches> out = m.match_pairs({&pr, 1}, cfg);
    return std::move(out.front().matches);
}

// match_pair_filtered (matcher.hpp:102-105): match_pair with a host callback between lookup and ranking
// (CandidateFilter, matcher.hpp:92-93).  Lookup and ranking + verification run on the device, the callback on the
// calling thread in between (Matcher::match_pair_filtered).
using CandidateFilter = std::function<bool(std::uint32_t query_index, std::vector<std::uint32_t>& candidates)>;

inline std::vector<MatchRecord> match_pair_filtered(const FeatureSet& fs_i, const FeatureSet& fs_j, const ImageCodes& codes_i,
                                                    const ImageCodes& codes_j, const MatchConfig& cfg,
                                                    const CandidateFilter& filter) {
    if (!(codes_i.params == codes_j.params))
        throw std::invalid_argument("match_pair: codes come from different hash families");  // matcher.cpp:144
    if (codes_i.shorts.point_count != fs_i.size() || codes_j.shorts.point_count != fs_j.size())
        throw std::invalid_argument("match_pair: code/point count mismatch");  // matcher.cpp:146-148
    static std::mutex fam_mu;
    static std::vector<std::unique_ptr<HashFamily>> families;
    const HashFamily* fam = nullptr;
    {
        std::lock_guard<std::mutex> lock(fam_mu);
        for (const auto& f : families)
            if (f->params == codes_i.params) fam = f.get();
        if (!fam) {
            families.push_back(std::make_unique<HashFamily>(build_hash_family(codes_i.params)));
            fam = families.back().get();
        }
    }
    detail::DefaultContext& dc = detail::default_context();
    std::lock_guard<std::mutex> lock(dc.mu);
    Matcher& m = dc.with(*fam);
    const std::uint32_t a = dc.resident(m, fs_i, codes_i), b = dc.resident(m, fs_j, codes_j);
    return m.match_pair_filtered(a, b, cfg, filter);
}

// guided_match_pair (geometry.hpp:86-89): match_pair with the epipolar band between lookup and ranking.
// F is the row-major 3x3 fundamental matrix (the reference's Eigen::Matrix3d, coefficient (r, c) at 3 r + c);
// estimating it (eight_point / ransac_fundamental) stays on the caller's side.
using FundamentalMatrix = std::array<double, 9>;

inline std::vector<MatchRecord> guided_match_pair(const FeatureSet& fs_i, const FeatureSet& fs_j, const ImageCodes& codes_i,
                                                  const ImageCodes& codes_j, const FundamentalMatrix& f,
                                                  const MatchConfig& cfg, double band_px) {
    if (!(codes_i.params == codes_j.params))
        throw std::invalid_argument("match_pair: codes come from different hash families");
    if (codes_i.shorts.point_count != fs_i.size() || codes_j.shorts.point_count != fs_j.size())
        throw std::invalid_argument("match_pair: code/point count mismatch");
    static std::mutex fam_mu;
    static std::vector<std::unique_ptr<HashFamily>> families;
    const HashFamily* fam = nullptr;
    {
        std::lock_guard<std::mutex> lock(fam_mu);
        for (const auto& g : families)
            if (g->params == codes_i.params) fam = g.get();
        if (!fam) {
            families.push_back(std::make_unique<HashFamily>(build_hash_family(codes_i.params)));
            fam = families.back().get();
        }
    }
    detail::DefaultContext& dc = detail::default_context();
    std::lock_guard<std::mutex> lock(dc.mu);
    Matcher& m = dc.with(*fam);
    const std::pair<std::uint32_t, std::uint32_t> pr{dc.resident(m, fs_i, codes_i), dc.resident(m, fs_j, codes_j)};
    std::vector<PairMatches> out = m.match_pairs_guided({&pr, 1}, {&f, 1}, band_px, cfg);
    return std::move(out.front().matches);
}

// Several GPUs of one box from one process: one Matcher (context) and one host thread per lane, the working set
// replicated on every lane, the pair list cut into contiguous, work-balanced shards of the plan (chgpu_shard_pairs_weighted), results
// gathered in pair order on the host.  No device-to-device traffic: pairs are independent.  The
// reference's counterpart is its W worker threads over one in-memory arena (execute_plan, engine.cpp:667-702);
// paper_1805_08995_b200/sharding.py is the same protocol with one process per GPU.
class MultiGpuMatcher {
public:
    // devices: CUDA device ordinals, one lane each (an ordinal may repeat: lanes then share that GPU)
    explicit MultiGpuMatcher(std::span<const int> devices) {
        if (devices.empty()) throw std::invalid_argument("MultiGpuMatcher: no devices");
        for (const int d : devices) lanes_.push_back(std::make_unique<Matcher>(d));
    }
    std::size_t lane_count() const { return lanes_.size(); }
    Matcher& lane(std::size_t k) { return *lanes_[k]; }

    void set_family(const HashFamily& family) {
        for (auto& m : lanes_) m->set_family(family);
    }
    void upload(std::uint32_t image_id, const FeatureSet& fs) {
        for (auto& m : lanes_) m->upload(image_id, fs);
    }
    // Dataset centering from the resident images: lane k sums images k, k + G, ... ; the partial sums are
    // exchanged on the host (128 u64 + a count) and every lane installs the same vector (hashing.cpp:52-64).
    std::array<double, kDescriptorDim> set_centering(std::span<const std::uint32_t> image_ids) {
        const std::size_t G = lanes_.size();
        std::array<std::uint64_t, kDescriptorDim> total{};
        std::uint64_t count = 0;
        std::vector<std::array<std::uint64_t, kDescriptorDim>> part(G);
        std::vector<std::uint64_t> cnt(G, 0);
        each_lane([&](std::size_t k) {
            std::vector<std::uint32_t> mine;
            for (std::size_t i = k; i < image_ids.size(); i += G) mine.push_back(image_ids[i]);
            lanes_[k]->centering_reset();
            lanes_[k]->centering_add(mine);
            ck_lane(k, chgpu_centering_get_sums(lanes_[k]->handle(), part[k].data(), &cnt[k]));
        });
        for (std::size_t k = 0; k < G; ++k) {
            for (std::size_t x = 0; x < kDescriptorDim; ++x) total[x] += part[k][x];
            count += cnt[k];
        }
        if (count == 0) throw std::invalid_argument("set_centering: no descriptors");
        std::array<double, kDescriptorDim> c{};
        for (std::size_t x = 0; x < kDescriptorDim; ++x) c[x] = static_cast<double>(total[x]) / static_cast<double>(count);
        for (std::size_t k = 0; k < G; ++k) ck_lane(k, chgpu_set_centering(lanes_[k]->handle(), c.data()));
        return c;
    }
    void hash(std::span<const std::uint32_t> image_ids, int reduce_rounds = kDefaultReduceRounds) {
        each_lane([&](std::size_t k) { lanes_[k]->hash(image_ids, reduce_rounds); });
    }
    // The pair list in contiguous shards, one per lane, matched concurrently; results in pair order.
    std::vector<PairMatches> match_pairs(std::span<const std::pair<std::uint32_t, std::uint32_t>> pairs,
                                         const MatchConfig& cfg, MatchStats* stats = nullptr) {
        const std::size_t G = lanes_.size();
        std::vector<std::vector<PairMatches>> part(G);
        std::vector<MatchStats> st(G);
        // contiguous shards of about equal WORK (chgpu_pair_weight: queries x train points), not pair count:
        // datasets mix 1K- and 32K-point images and a 32K x 32K pair costs ~1000 x a 1K x 1K one
        std::uint32_t max_id = 0;
        for (const auto& p : pairs) max_id = std::max({max_id, p.first, p.second});
        std::vector<std::uint32_t> points(pairs.empty() ? 0 : std::size_t(max_id) + 1, 0);
        for (const auto& p : pairs)
            for (const std::uint32_t id : {p.first, p.second})
                if (points[id] == 0) ck_lane(0, chgpu_image_points(lanes_[0]->handle(), id, &points[id]));
        std::vector<std::uint64_t> first(G + 1, 0);
        static_assert(sizeof(std::pair<std::uint32_t, std::uint32_t>) == 8, "pair list is passed as 2 x u32 per pair");
        ck_lane(0, chgpu_shard_pairs_weighted(reinterpret_cast<const std::uint32_t*>(pairs.data()), pairs.size(), points.data(),
                                              static_cast<std::uint32_t>(points.size()), static_cast<std::uint32_t>(G),
                                              first.data(), nullptr));
        each_lane([&](std::size_t k) {
            part[k] = lanes_[k]->match_pairs(pairs.subspan(first[k], first[k + 1] - first[k]), cfg, &st[k]);
        });
        std::vector<PairMatches> out;
        out.reserve(pairs.size());
        MatchStats sum{};
        for (std::size_t k = 0; k < G; ++k) {
            for (PairMatches& pm : part[k]) out.push_back(std::move(pm));
            sum.pairs += st[k].pairs;
            sum.matches += st[k].matches;
            sum.raw_candidates += st[k].raw_candidates;
            sum.verified_queries += st[k].verified_queries;
            sum.distances += st[k].distances;
            sum.query_points += st[k].query_points;
            sum.train_points += st[k].train_points;
            sum.match_launches += st[k].match_launches;
            sum.total_launches += st[k].total_launches;
            sum.match_kernel_ms = std::max(sum.match_kernel_ms, st[k].match_kernel_ms);  // lanes run side by side
            sum.total_ms = std::max(sum.total_ms, st[k].total_ms);
        }
        sum.records_checksum = 0;  // keyed by the pair's position in the list each lane saw: not additive over shards
        if (stats) *stats = sum;
        return out;
    }

private:
    template <class F>
    void each_lane(F&& f) {  // one host thread per lane; the first exception is rethrown on the caller's thread
        std::vector<std::thread> threads;
        std::vector<std::exception_ptr> errors(lanes_.size());
        for (std::size_t k = 0; k < lanes_.size(); ++k)
            threads.emplace_back([&, k] {
                try {
                    f(k);
                } catch (...) {
                    errors[k] = std::current_exception();
                }
            });
        for (std::thread& t : threads) t.join();
        for (const std::exception_ptr& e : errors)
            if (e) std::rethrow_exception(e);
    }
    void ck_lane(std::size_t k, chgpu_status st) {
        if (st != CHGPU_OK) detail::raise(st, chgpu_last_error(lanes_[k]->handle()));
    }
    std::vector<std::unique_ptr<Matcher>> lanes_;
};

}  // namespace cashash_b200
