// host_util.cpp — host-only parts of the C ABI: hash-family generation, match-file output and
// pair-list planning.  None of this touches the device; it is compiled into libchgpu.so so a
// caller needs exactly one library for the whole matching path.

#include "../../include/chgpu.h"
#include "plan_tasks.hpp"

#include <algorithm>
#include <atomic>
#include <charconv>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <memory>
#include <mutex>
#include <thread>
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

// Text of one match file (save_matches, feature_io.cpp:161-183): "# idI idJ count" then "q t dist" lines,
// dist as the shortest decimal that round-trips (std::to_chars; integers print without a point).
void format_matches(const char* id_i, const char* id_j, const chgpu_match_record* records, uint32_t count, std::string& out) {
    out.clear();
    out.reserve(64 + size_t(count) * 24);
    out.append("# ").append(id_i).append(" ").append(id_j).append(" ");
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
        const auto r = std::to_chars(buf, buf + sizeof(buf), records[i].distance_sq);
        out.append(buf, r.ptr);
        out.push_back('\n');
    }
}

bool write_whole_file(const char* path, const std::string& bytes) {
    FILE* f = std::fopen(path, "wb");
    if (!f) return false;
    const size_t w = std::fwrite(bytes.data(), 1, bytes.size(), f);
    const int c = std::fclose(f);
    return w == bytes.size() && c == 0;
}

}  // namespace

// ---- asynchronous match-file writer ---------------------------------------------------------------
struct chgpu_sink {
    struct Batch {
        std::vector<uint32_t> pairs;
        std::vector<uint64_t> offsets;
        std::vector<chgpu_match_record> records;
    };
    std::string dir;
    std::vector<std::string> names;
    std::mutex mu;
    std::condition_variable cv_work, cv_room;
    std::deque<std::unique_ptr<Batch>> queue;
    size_t max_queued = 8;
    bool closing = false;
    std::vector<std::thread> workers;
    uint64_t files_written = 0, files_failed = 0, records = 0, bytes = 0;
    double busy_seconds = 0.0;
    std::chrono::steady_clock::time_point opened;

    void run() {
        std::string text, path, a, b;
        uint64_t ok = 0, failed = 0, nrec = 0, nbytes = 0;
        double busy = 0.0;
        for (;;) {
            std::unique_ptr<Batch> item;
            {
                std::unique_lock<std::mutex> lock(mu);
                cv_work.wait(lock, [&] { return closing || !queue.empty(); });
                if (queue.empty()) break;
                item = std::move(queue.front());
                queue.pop_front();
            }
            cv_room.notify_one();
            const auto t0 = std::chrono::steady_clock::now();
            const uint32_t n = uint32_t(item->pairs.size() / 2);
            for (uint32_t k = 0; k < n; ++k) {
                const uint32_t i = item->pairs[2 * k], j = item->pairs[2 * k + 1];
                const char* id_i = i < names.size() ? names[i].c_str() : (a = std::to_string(i)).c_str();
                const char* id_j = j < names.size() ? names[j].c_str() : (b = std::to_string(j)).c_str();
                const uint32_t count = uint32_t(item->offsets[k + 1] - item->offsets[k]);
                format_matches(id_i, id_j, item->records.data() + item->offsets[k], count, text);
                char name[48];
                chgpu_pair_file_name(i, j, name);
                path.assign(dir).append("/").append(name);
                if (write_whole_file(path.c_str(), text)) {
                    ++ok;
                    nrec += count;
                    nbytes += text.size();
                } else {
                    ++failed;
                }
            }
            busy += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
        std::lock_guard<std::mutex> lock(mu);
        files_written += ok;
        files_failed += failed;
        records += nrec;
        bytes += nbytes;
        busy_seconds += busy;
    }
};

extern "C" {

chgpu_status chgpu_sink_open(const char* dir, const char* const* image_names, uint32_t image_count, uint32_t threads,
                             uint32_t max_queued_batches, chgpu_sink** out) {
    if (!dir || !out) return CHGPU_EINVAL;
    *out = nullptr;
    auto sink = std::make_unique<chgpu_sink>();
    sink->dir = dir;
    if (image_names)
        for (uint32_t i = 0; i < image_count; ++i) sink->names.emplace_back(image_names[i] ? image_names[i] : "");
    sink->max_queued = std::max<uint32_t>(1, max_queued_batches ? max_queued_batches : 8);
    sink->opened = std::chrono::steady_clock::now();
    threads = std::max<uint32_t>(1, std::min<uint32_t>(threads ? threads : 4, 256));
    chgpu_sink* raw = sink.release();
    for (uint32_t t = 0; t < threads; ++t) raw->workers.emplace_back([raw] { raw->run(); });
    *out = raw;
    return CHGPU_OK;
}

chgpu_status chgpu_sink_accept(chgpu_sink* sink, const uint32_t* pairs, uint32_t npairs, const uint64_t* offsets,
                               const chgpu_match_record* records) {
    if (!sink || (npairs && (!pairs || !offsets))) return CHGPU_EINVAL;
    if (npairs == 0) return CHGPU_OK;
    auto item = std::make_unique<chgpu_sink::Batch>();
    item->pairs.assign(pairs, pairs + 2 * size_t(npairs));
    item->offsets.resize(size_t(npairs) + 1);
    for (uint32_t k = 0; k <= npairs; ++k) item->offsets[k] = offsets[k] - offsets[0];
    const uint64_t total = offsets[npairs] - offsets[0];
    if (total && !records) return CHGPU_EINVAL;
    item->records.assign(records + offsets[0], records + offsets[0] + total);
    {
        std::unique_lock<std::mutex> lock(sink->mu);
        if (sink->closing) return CHGPU_ELOGIC;
        sink->cv_room.wait(lock, [&] { return sink->queue.size() < sink->max_queued; });
        sink->queue.push_back(std::move(item));
    }
    sink->cv_work.notify_one();
    return CHGPU_OK;
}

chgpu_status chgpu_sink_close(chgpu_sink* sink, chgpu_sink_stats* stats) {
    if (!sink) return CHGPU_EINVAL;
    {
        std::lock_guard<std::mutex> lock(sink->mu);
        sink->closing = true;
    }
    sink->cv_work.notify_all();
    for (std::thread& t : sink->workers) t.join();
    if (stats) {
        stats->files_written = sink->files_written;
        stats->files_failed = sink->files_failed;
        stats->records = sink->records;
        stats->bytes = sink->bytes;
        stats->busy_seconds = sink->busy_seconds;
        stats->wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - sink->opened).count();
    }
    delete sink;
    return CHGPU_OK;
}

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
    format_matches(image_id_i, image_id_j, records, count, out);
    return write_whole_file(path, out) ? CHGPU_OK : CHGPU_EFORMAT;  // FeatureFileFault::Unwritable
}

void chgpu_pair_file_name(uint32_t image_i, uint32_t image_j, char* buf) {
    std::snprintf(buf, 48, "match_%06u_%06u.txt", image_i, image_j);
}

chgpu_status chgpu_plan_exhaustive(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group,
                                   uint32_t* pairs_out, uint64_t* npairs_out) {
    if (image_count == 0 || block_images == 0 || blocks_per_group == 0 || !npairs_out) return CHGPU_EINVAL;
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
    chgpu::for_each_plan_task(
        image_count, block_images, blocks_per_group,
        [&](uint32_t ba, uint32_t bb) {
            for (uint32_t a = block_lo(ba); a < block_hi(ba); ++a)
                for (uint32_t b = block_lo(bb); b < block_hi(bb); ++b) emit(a, b);
        },
        [&](uint32_t blk) {
            for (uint32_t a = block_lo(blk); a < block_hi(blk); ++a)
                for (uint32_t b = a + 1; b < block_hi(blk); ++b) emit(a, b);
        });
    *npairs_out = np;
    return CHGPU_OK;
}

// plan_guided (scheduler.cpp:144-164): the same traversal restricted to the accepted pairs.  The reference filters
// the expanded exhaustive list; here the accepted pairs are bucketed by block pair and the buckets are emitted in
// task order, each sorted the way a task lists its pairs ((a, b) ascending) — the same sequence without touching
// the K^2 / 2 pairs nobody asked for (16,384 images: 134 M).
chgpu_status chgpu_plan_guided(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group,
                               const uint32_t* accepted, uint64_t accepted_count, uint32_t* pairs_out, uint64_t* npairs_out) {
    if (image_count == 0 || block_images == 0 || blocks_per_group == 0 || !npairs_out || (accepted_count && !accepted))
        return CHGPU_EINVAL;
    const uint64_t nblocks = (image_count + block_images - 1) / block_images;
    std::vector<std::pair<uint64_t, uint64_t>> keyed;  // (block pair, a * K + b)
    keyed.reserve(accepted_count);
    for (uint64_t i = 0; i < accepted_count; ++i) {
        uint32_t a = accepted[2 * i], b = accepted[2 * i + 1];
        if (a == b) return CHGPU_EINVAL;           // "plan_guided: self pair"
        if (a > b) std::swap(a, b);
        if (b >= image_count) return CHGPU_EINVAL;  // "plan_guided: unknown image index"
        keyed.emplace_back(uint64_t(a / block_images) * nblocks + b / block_images, uint64_t(a) * image_count + b);
    }
    std::sort(keyed.begin(), keyed.end());
    keyed.erase(std::unique(keyed.begin(), keyed.end()), keyed.end());
    uint64_t np = 0;
    auto emit_bucket = [&](uint64_t key) {
        auto it = std::lower_bound(keyed.begin(), keyed.end(), std::make_pair(key, uint64_t(0)));
        for (; it != keyed.end() && it->first == key; ++it) {
            if (pairs_out) {
                pairs_out[2 * np] = uint32_t(it->second / image_count);
                pairs_out[2 * np + 1] = uint32_t(it->second % image_count);
            }
            ++np;
        }
    };
    chgpu::for_each_plan_task(
        image_count, block_images, blocks_per_group, [&](uint32_t ba, uint32_t bb) { emit_bucket(uint64_t(ba) * nblocks + bb); },
        [&](uint32_t blk) { emit_bucket(uint64_t(blk) * nblocks + blk); });
    *npairs_out = np;
    return CHGPU_OK;
}

// ---- code cache (CHCC) and centering (CHCV) files ------------------------------------------------
uint64_t chgpu_centering_fingerprint(const double* centering128) {
    // FNV-1a, byte by byte from the least significant byte of each double (hashing.cpp:151-162)
    uint64_t h = 0xcbf29ce484222325ULL;
    for (int i = 0; i < 128; ++i) {
        uint64_t bits;
        std::memcpy(&bits, centering128 + i, 8);
        for (int b = 0; b < 8; ++b) {
            h ^= (bits >> (8 * b)) & 0xff;
            h *= 0x100000001b3ULL;
        }
    }
    return h;
}

namespace {
struct CacheHeader {  // 44 bytes on disk, little-endian, no padding between fields
    char magic[4];
    uint32_t version, short_bits, long_bits, table_count;
    uint64_t seed, centering_fp;
    uint32_t count, reserved;
};
constexpr size_t kCacheHeaderBytes = 44;

void pack_header(const CacheHeader& h, unsigned char* out) {
    std::memcpy(out, h.magic, 4);
    std::memcpy(out + 4, &h.version, 4);
    std::memcpy(out + 8, &h.short_bits, 4);
    std::memcpy(out + 12, &h.long_bits, 4);
    std::memcpy(out + 16, &h.table_count, 4);
    std::memcpy(out + 20, &h.seed, 8);
    std::memcpy(out + 28, &h.centering_fp, 8);
    std::memcpy(out + 36, &h.count, 4);
    std::memcpy(out + 40, &h.reserved, 4);
}
}  // namespace

chgpu_status chgpu_save_code_cache(const char* path, const chgpu_family_params* p, uint64_t centering_fp,
                                   uint32_t count, const uint32_t* shorts, const uint64_t* longs) {
    if (!path || !p || (count && (!shorts || !longs))) return CHGPU_EINVAL;
    std::vector<unsigned char> out(kCacheHeaderBytes + size_t(count) * p->table_count * 4 + size_t(count) * 16);
    CacheHeader h{{'C', 'H', 'C', 'C'}, 1, p->short_bits, p->long_bits, p->table_count, p->seed, centering_fp, count, 0};
    unsigned char head[kCacheHeaderBytes];
    pack_header(h, head);
    std::memcpy(out.data(), head, 44);
    if (count) {
        std::memcpy(out.data() + 44, shorts, size_t(count) * p->table_count * 4);
        std::memcpy(out.data() + 44 + size_t(count) * p->table_count * 4, longs, size_t(count) * 16);
    }
    FILE* f = std::fopen(path, "wb");
    if (!f) return CHGPU_EFORMAT;  // FeatureFileFault::Unwritable
    const size_t w = std::fwrite(out.data(), 1, out.size(), f);
    const int c = std::fclose(f);
    return (w == out.size() && c == 0) ? CHGPU_OK : CHGPU_EFORMAT;
}

namespace {
// Parses the 44-byte header; returns 0 ok, 1 bad magic, 2 truncated header.
int parse_header(const unsigned char* b, size_t n, CacheHeader& h) {
    if (n < 4 || std::memcmp(b, "CHCC", 4) != 0) return 1;
    if (n < 44) return 2;
    std::memcpy(&h.version, b + 4, 4);
    std::memcpy(&h.short_bits, b + 8, 4);
    std::memcpy(&h.long_bits, b + 12, 4);
    std::memcpy(&h.table_count, b + 16, 4);
    std::memcpy(&h.seed, b + 20, 8);
    std::memcpy(&h.centering_fp, b + 28, 8);
    std::memcpy(&h.count, b + 36, 4);
    std::memcpy(&h.reserved, b + 40, 4);
    return 0;
}

bool read_file(const char* path, std::vector<unsigned char>& out, size_t limit = ~size_t(0)) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return false;
    unsigned char buf[1 << 16];
    size_t got;
    while (out.size() < limit && (got = std::fread(buf, 1, sizeof(buf), f)) > 0) out.insert(out.end(), buf, buf + got);
    std::fclose(f);
    return true;
}
}  // namespace

chgpu_status chgpu_read_code_cache_header(const char* path, chgpu_family_params* p, uint64_t* centering_fp,
                                          uint32_t* count) {
    if (!path || !p || !centering_fp || !count) return CHGPU_EINVAL;
    std::vector<unsigned char> bytes;
    if (!read_file(path, bytes, 44)) return CHGPU_ENOTFOUND;
    CacheHeader h{};
    if (parse_header(bytes.data(), bytes.size(), h) != 0 || h.version != 1) return CHGPU_ENOTFOUND;
    *p = chgpu_family_params{h.short_bits, h.long_bits, h.table_count, h.seed};
    *centering_fp = h.centering_fp;
    *count = h.count;
    return CHGPU_OK;
}

chgpu_status chgpu_load_code_cache(const char* path, const chgpu_family_params* expected, uint64_t expected_fp,
                                   uint32_t capacity, uint32_t* count, uint32_t* shorts, uint64_t* longs,
                                   chgpu_file_fault* fault, uint64_t* fault_offset) {
    if (!path || !expected || !count) return CHGPU_EINVAL;
    auto bad = [&](chgpu_file_fault f, uint64_t off) {
        if (fault) *fault = f;
        if (fault_offset) *fault_offset = off;
        return CHGPU_EFORMAT;
    };
    if (fault) *fault = CHGPU_FAULT_NONE;
    std::vector<unsigned char> bytes;
    if (!read_file(path, bytes)) return bad(CHGPU_FAULT_MISSING_FILE, 0);
    CacheHeader h{};
    const int hr = parse_header(bytes.data(), bytes.size(), h);
    if (hr == 1) return bad(CHGPU_FAULT_BAD_MAGIC, 0);
    if (hr == 2) return bad(CHGPU_FAULT_TRUNCATED, 4);  // "cache header"
    if (h.version != 1) return bad(CHGPU_FAULT_BAD_VERSION, 4);
    if (h.short_bits != expected->short_bits || h.long_bits != expected->long_bits ||
        h.table_count != expected->table_count || h.seed != expected->seed || h.centering_fp != expected_fp)
        return CHGPU_EMISMATCH;
    *count = h.count;
    const size_t sbytes = size_t(h.count) * h.table_count * 4, lbytes = size_t(h.count) * 16;
    // the reference reads value by value and reports a short payload through a failed tellg(): offset -1
    if (bytes.size() < 44 + sbytes + lbytes) return bad(CHGPU_FAULT_TRUNCATED, ~uint64_t(0));
    if (h.count > capacity) return CHGPU_ENOMEM;
    if (h.count) {
        if (!shorts || !longs) return CHGPU_EINVAL;
        std::memcpy(shorts, bytes.data() + 44, sbytes);
        std::memcpy(longs, bytes.data() + 44 + sbytes, lbytes);
    }
    return CHGPU_OK;
}

chgpu_status chgpu_save_centering_file(const char* path, const chgpu_family_params* p, const double* centering128) {
    if (!path || !p || !centering128) return CHGPU_EINVAL;
    unsigned char out[4 + 4 + 12 + 8 + 1024];
    std::memcpy(out, "CHCV", 4);
    const uint32_t version = 1;
    std::memcpy(out + 4, &version, 4);
    std::memcpy(out + 8, &p->short_bits, 4);
    std::memcpy(out + 12, &p->long_bits, 4);
    std::memcpy(out + 16, &p->table_count, 4);
    std::memcpy(out + 20, &p->seed, 8);
    std::memcpy(out + 28, centering128, 1024);
    FILE* f = std::fopen(path, "wb");
    if (!f) return CHGPU_EFORMAT;
    const size_t w = std::fwrite(out, 1, sizeof(out), f);
    const int c = std::fclose(f);
    return (w == sizeof(out) && c == 0) ? CHGPU_OK : CHGPU_EFORMAT;
}

chgpu_status chgpu_load_centering_file(const char* path, chgpu_family_params* p, double* centering128) {
    if (!path || !p || !centering128) return CHGPU_EINVAL;
    std::vector<unsigned char> b;
    if (!read_file(path, b)) return CHGPU_ENOTFOUND;
    uint32_t version = 0;
    if (b.size() != 28 + 1024 || std::memcmp(b.data(), "CHCV", 4) != 0) return CHGPU_EFORMAT;
    std::memcpy(&version, b.data() + 4, 4);
    if (version != 1) return CHGPU_EFORMAT;
    std::memcpy(&p->short_bits, b.data() + 8, 4);
    std::memcpy(&p->long_bits, b.data() + 12, 4);
    std::memcpy(&p->table_count, b.data() + 16, 4);
    std::memcpy(&p->seed, b.data() + 20, 8);
    std::memcpy(centering128, b.data() + 28, 1024);
    return CHGPU_OK;
}

chgpu_status chgpu_shard_range(uint64_t npairs, uint32_t rank, uint32_t world, uint64_t* first, uint64_t* last) {
    if (!first || !last) return CHGPU_EINVAL;
    if (world == 0) world = 1;
    if (rank >= world) {
        *first = *last = npairs;
        return CHGPU_EINVAL;
    }
    const uint64_t base = npairs / world, rem = npairs % world;
    const uint64_t f = uint64_t(rank) * base + std::min<uint64_t>(rank, rem);
    *first = f;
    *last = f + base + (rank < rem ? 1 : 0);
    return CHGPU_OK;
}

uint64_t chgpu_pair_weight(uint32_t query_points, uint32_t train_points) {
    return uint64_t(query_points) * (uint64_t(train_points) + 512u);
}

chgpu_status chgpu_shard_pairs_weighted(const uint32_t* pairs, uint64_t npairs, const uint32_t* points_per_image,
                                        uint32_t image_count, uint32_t shards, uint64_t* first_out, uint64_t* weights_out) {
    if ((npairs && !pairs) || !points_per_image || !first_out || shards == 0) return CHGPU_EINVAL;
    for (uint64_t k = 0; k < 2 * npairs; ++k)
        if (pairs[k] >= image_count) return CHGPU_EINVAL;
    // 128-bit products: a Rome16K-sized list of 32K-point images sums to ~2^59 before the multiplication by `shards`
    unsigned __int128 total = 0;
    for (uint64_t k = 0; k < npairs; ++k) total += chgpu_pair_weight(points_per_image[pairs[2 * k]], points_per_image[pairs[2 * k + 1]]);
    for (uint32_t s = 0; s <= shards; ++s) first_out[s] = npairs;
    first_out[0] = 0;
    unsigned __int128 acc = 0;
    uint32_t s = 1;
    for (uint64_t k = 0; k < npairs && s < shards; ++k) {
        const uint64_t w = chgpu_pair_weight(points_per_image[pairs[2 * k]], points_per_image[pairs[2 * k + 1]]);
        // cut in front of the pair that would carry the shard past its share, unless stopping short is the worse miss
        const unsigned __int128 target = total * s;
        if ((acc + w) * shards > target) {
            const unsigned __int128 over = (acc + w) * shards - target, under = target - acc * shards;
            if (acc * shards >= target || over > under) {
                first_out[s++] = k;
                --k;  // the same pair is looked at again for the next boundary
                continue;
            }
        }
        acc += w;
    }
    if (weights_out)
        for (uint32_t r = 0; r < shards; ++r) {
            uint64_t w = 0;
            for (uint64_t k = first_out[r]; k < first_out[r + 1]; ++k)
                w += chgpu_pair_weight(points_per_image[pairs[2 * k]], points_per_image[pairs[2 * k + 1]]);
            weights_out[r] = w;
        }
    return CHGPU_OK;
}

}  // extern "C"
