// chgpu.cu — context, memory management and the C ABI of libchgpu.so (see include/chgpu.h).
//
// Data layout in HBM: every resident image owns ONE arena block holding, 256-byte aligned,
//   desc (n*128 B) | kp (n*16 B) | longs (n*16 B) | shorts (n*L*4 B) | offs (L*(2^m+1)*4 B) | points (L*n*2 B)
//   | scan (L*n*2 B)
// (1,565,208 B for n = 8192, m = 8, L = 6).  Blocks are bump-allocated from 256 MiB slabs and
// recycled through an exact-size free list, so streaming a dataset through a bounded working
// set never calls cudaMalloc in steady state.
//
// Streams: `copy` carries H2D uploads (pinned staging ring for pageable sources) and result
// D2H; `compute` carries every kernel.  Events order the two; nothing here uses the legacy
// default stream.

#include "../../include/chgpu.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "dev_types.cuh"
#include "hash_kernels.cuh"
#include "hash_tc.cuh"
#include "join_kernels.cuh"
#include "compact_kernels.cuh"
#include "general_kernels.cuh"
#include "match_launch.cuh"

using namespace chgpu;

// host_util.cpp
extern "C" int chgpu_host_check_family(const chgpu_family_params* p);

namespace {

constexpr size_t kAlign = 256;
constexpr size_t kSlabBytes = size_t(256) << 20;
constexpr size_t kStageBytes = size_t(32) << 20;
constexpr int kStageSlots = 2;
constexpr uint32_t kHashQueueCap = 1u << 21;    // undecided dots per hash launch (16 MiB); ~110 per 8K-point image are expected
constexpr uint32_t kHashBatchImages = 2048;     // images per hash launch
constexpr size_t kSinkChunkEntries = size_t(2) << 20;  // records per pinned delivery buffer of the streaming sink (32 MiB)
constexpr uint64_t kSubBatchQueries = uint64_t(32) << 20;  // per sub-batch: sum of Nq (res 256 MiB, records <= 512 MiB); the persistent grid pays its tail once per launch

size_t align_up(size_t v, size_t a = kAlign) { return (v + a - 1) / a * a; }

struct Arena {
    struct Slab {
        char* base;
        size_t size, used;
    };
    std::vector<Slab> slabs;
    std::map<size_t, std::vector<char*>> free_lists;
    size_t live_bytes = 0;

    cudaError_t alloc(size_t bytes, char** out) {
        bytes = align_up(bytes);
        auto it = free_lists.find(bytes);
        if (it != free_lists.end() && !it->second.empty()) {
            *out = it->second.back();
            it->second.pop_back();
            live_bytes += bytes;
            return cudaSuccess;
        }
        for (Slab& s : slabs)
            if (s.size - s.used >= bytes) {
                *out = s.base + s.used;
                s.used += bytes;
                live_bytes += bytes;
                return cudaSuccess;
            }
        // cudaMalloc drains the device before it returns, so a stream of uploads should meet it rarely: slabs
        // double in size (256 MiB ... 8 GiB); a slab the device cannot give is retried at the minimum size.
        size_t want = kSlabBytes;
        if (!slabs.empty()) want = std::min(slabs.back().size * 2, size_t(8) << 30);
        Slab s{nullptr, std::max(want, bytes), 0};
        cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&s.base), s.size);
        if (e != cudaSuccess && s.size > std::max(kSlabBytes, bytes)) {
            cudaGetLastError();
            s.size = std::max(kSlabBytes, bytes);
            e = cudaMalloc(reinterpret_cast<void**>(&s.base), s.size);
        }
        if (e != cudaSuccess) return e;
        s.used = bytes;
        *out = s.base;
        slabs.push_back(s);
        live_bytes += bytes;
        return cudaSuccess;
    }
    void release(char* p, size_t bytes) {
        bytes = align_up(bytes);
        free_lists[bytes].push_back(p);
        live_bytes -= bytes;
    }
    void destroy() {
        for (Slab& s : slabs) cudaFree(s.base);
        slabs.clear();
        free_lists.clear();
    }
};

struct ImageRec {
    DevImage dev{};
    char* block = nullptr;
    size_t block_bytes = 0;
    uint32_t image_id = 0;
    bool used = false;
    // centering generation the codes were computed under (chgpu_hash_images, verified code caches); 0 = codes supplied
    // by the caller (chgpu_upload_codes), not tied to the context's centering
    uint32_t hash_gen = 0;
    // id-range tiles of an image too large for the match kernel's shared-memory tile: hidden slots of the
    // image table whose DevImages are slices of this block with their own bucket index (local point ids)
    std::vector<uint32_t> tile_slots;
    uint32_t tile_points = 0;  // points per tile (balanced_tile_points)
};

struct MatchBuffers {
    PairDesc* h_pairs = nullptr;  // pinned
    PairDesc* d_pairs = nullptr;
    size_t pairs_cap = 0;
    PairDesc* h_tpairs = nullptr;  // pinned: (query image, tile) pairs of a tiled sub-batch
    PairDesc* d_tpairs = nullptr;
    size_t tpairs_cap = 0;
    uint32_t* d_counts = nullptr;
    unsigned long long* d_offsets = nullptr;
    unsigned long long* h_offsets = nullptr;  // pinned
    double* d_fmats = nullptr;  // guided: 9 doubles per pair of the sub-batch
    size_t fmats_cap = 0;    // pairs
    uint4* d_records = nullptr;
    size_t records_cap = 0;  // entries
    chgpu_match_record* h_records = nullptr;  // pinned
    size_t h_records_cap = 0;
    cudaEvent_t ev_done = nullptr, ev_k0 = nullptr, ev_k1 = nullptr;
};

}  // namespace

struct chgpu_load_job;

struct chgpu_ctx {
    int device = 0;
    cudaDeviceProp prop{};
    cudaStream_t compute = nullptr, copy = nullptr;
    cudaStream_t load = nullptr;  // H2D of background loads: runs beside the result copies (D2H on `copy`)
    cudaEvent_t ev_upload = nullptr, ev_compute = nullptr, ev_t0 = nullptr, ev_t1 = nullptr;
    cudaEvent_t ev_chunk[2] = {nullptr, nullptr};  // D2H of a result chunk into mb[j].h_records complete
    std::string err;

    Arena arena;
    std::vector<ImageRec> images;
    std::vector<uint32_t> free_slots;
    std::unordered_map<uint32_t, uint32_t> slot_of;
    std::vector<uint32_t> slot_dense;  // slot_of for image ids < kDenseIds: pair lists resolve 2 ids per pair
    DevImage* d_images = nullptr;
    DevImage* h_images = nullptr;  // pinned mirror
    size_t images_cap = 0;

    // staging ring for pageable uploads
    char* stage[kStageSlots] = {nullptr, nullptr};
    cudaEvent_t stage_ev[kStageSlots] = {nullptr, nullptr};
    int stage_next = 0;

    // family
    std::recursive_mutex mu;  // held by every entry point (CtxLock)
    bool has_family = false, has_centering = false;
    bool sparse = false;  // short_bits > kMaxShortBits: images carry sorted (code, point) keys, matched by the general path
    unsigned long long* d_list_offs = nullptr;  // explicit candidate lists of one pair (chgpu_match_pair_lists)
    uint32_t* d_list_ids = nullptr;
    uint32_t centering_gen = 1;  // bumped when a DIFFERENT centering vector is installed: codes hashed before are stale
    chgpu_family_params fam{};
    double* d_planes = nullptr;
    double* d_centering = nullptr;
    double h_centering[128] = {0};  // host copy (code-cache fingerprints)
    // fp32-filtered hash path (K1f, hash_kernels.cuh): constants derived from planes + centering
    std::vector<double> h_planes;   // host copy of the installed planes, (L*m + n) x 128
    float* d_planes_t = nullptr;    // [128][gpad] fp32-rounded, component-major
    double* d_bias = nullptr;       // [gpad]
    double* d_hnorm = nullptr;      // [gpad]
    uint32_t gpad = 0;
    double filt_a_rel = 0.0, filt_a_abs = 0.0;
    // K1t (tensor-core filter): int8 limbs of the planes and the per-plane constants of its bound
    int8_t* d_tc_limbs = nullptr;   // [3][tc_npad][128]
    double* d_tc_const = nullptr;   // [4][tc_npad]: 1/S_g | bias_g | alpha_g | beta_g
    uint32_t tc_npad = 0;
    bool tc_ready = false;
    bool filter_ready = false;      // constants valid for the current planes + centering
    int hash_mode = 0;              // chgpu_hash_mode
    uint2* d_hq = nullptr;          // queue of undecided dots
    unsigned int* d_hq_count = nullptr;
    HashFilterStats* d_hstats = nullptr;
    unsigned long long* d_sums = nullptr;
    uint64_t sum_count = 0;
    uint64_t extra_sums[128] = {0};  // sums merged from other ranks

    // match workspace
    uint2* d_res = nullptr;
    size_t res_cap = 0;
    uint32_t* d_gmin = nullptr;   // tiled train images: per-query minimum key over the tiles
    unsigned long long* d_gdone = nullptr;  // ... and the tiles whose list the min pass already wrote
    size_t gmin_cap = 0;
    uint32_t* d_lists = nullptr;  // tiled train images: per-query, per-tile top-k keys
    size_t lists_cap = 0;
    uint16_t* d_act = nullptr;    // tiled train images: active queries per (query image, tile) pair
    uint32_t* d_nact = nullptr;
    size_t act_cap = 0, nact_cap = 0;
    uint8_t* d_hit = nullptr;     // join pass: one flag per query of a sub-batch
    size_t hit_cap = 0;
    bool join_enabled = true;     // tensor-core Hamming pass in front of the match kernel (CHGPU_NO_JOIN=1 switches it off)
    uint32_t join_min_bucket = 20;  // ... for sub-batches whose images average at least this many points per bucket
    MatchBuffers mb[2];
    DevStats* d_stats = nullptr;
    DevStats* h_stats = nullptr;  // pinned
    unsigned int* d_counter = nullptr;
    uint32_t* d_slots = nullptr;  // scratch list of slots for hash launches
    size_t slots_cap = 0;
    uint32_t* d_dbg = nullptr;
    size_t dbg_cap = 0;
    // streaming loader: pinned ring buffers and device staging, kept between calls
    char* load_pinned = nullptr;       // one region cut into load_pinned_slots slots of load_pinned_slot bytes
    size_t load_pinned_slot = 0, load_pinned_slots = 0;
    std::vector<std::pair<char*, size_t>> load_scratch;
    uint64_t sub_batch_queries = kSubBatchQueries;
    chgpu_load_job* load_job = nullptr;  // background load opened by chgpu_load_chft_files_begin
    char* load_region = nullptr;         // its device staging, one allocation cut into slices
    size_t load_region_bytes = 0;
    SplitJob* h_split_jobs = nullptr;    // pinned / device list for the batched split of a background load
    SplitJob* d_split_jobs = nullptr;
    size_t split_jobs_cap = 0;
    cudaEvent_t ev_split_jobs = nullptr;
    bool split_jobs_busy = false;
};

namespace {

thread_local std::string tl_err;
thread_local const chgpu_ctx* tl_err_ctx = nullptr;

chgpu_status fail(chgpu_ctx* ctx, chgpu_status s, const char* fmt, ...) {
    if (ctx) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof(buf), fmt, ap);
        va_end(ap);
        ctx->err = buf;
        tl_err = buf;  // the calling thread's own copy: chgpu_last_error stays valid while other threads use the context
        tl_err_ctx = ctx;
    }
    return s;
}

#define CK(call)                                                                                   \
    do {                                                                                           \
        const cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                                     \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? CHGPU_ENOMEM : CHGPU_ECUDA,         \
                        "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

struct DeviceGuard {
    explicit DeviceGuard(int dev) { cudaSetDevice(dev); }
};

// Every entry point that takes a context holds the context's mutex for its duration: calls from several threads on one
// context are serialised (a sink callback runs under it too; it may call back into the same context from the same thread).
struct CtxLock {
    explicit CtxLock(chgpu_ctx* ctx) : mu(ctx ? &ctx->mu : nullptr) {
        if (mu) mu->lock();
    }
    ~CtxLock() {
        if (mu) mu->unlock();
    }
    CtxLock(const CtxLock&) = delete;
    CtxLock& operator=(const CtxLock&) = delete;
    std::recursive_mutex* mu;
};

size_t smem_train_capacity(const chgpu_ctx* ctx, bool guided = false);

// Point ids per tile of a large train image: what fits the kernel's shared memory, at most ~32 entries per
// bucket (the occupancy the scan is laid out for), a multiple of 1024.
uint32_t tile_points_of(const chgpu_ctx* ctx) {
    // (the guided top-k pass stages more per warp than the unguided kernels: its capacity is the binding one)
    const size_t cap = std::min(smem_train_capacity(ctx, false), smem_train_capacity(ctx, true)) & ~size_t(1023);
    const size_t want = std::max<size_t>(1024, size_t(32) << ctx->fam.short_bits);
    return uint32_t(std::max<size_t>(1024, std::min(cap, want)));
}
uint32_t tile_count_of(const chgpu_ctx* ctx, uint32_t n) {
    if (ctx->sparse || n <= smem_train_capacity(ctx)) return 0;  // (sparse indices: the general path reads global memory)
    const uint32_t tp = tile_points_of(ctx);
    return (n + tp - 1) / tp;
}
// Points per tile of ONE image: its tiles are balanced (12,288 points = 2 x 6,144, not 8,192 + 4,096), so no tile carries the
// overflow scan steps of a full one next to a half-empty neighbour; a multiple of 16 keeps every slice aligned.
uint32_t balanced_tile_points(const chgpu_ctx* ctx, uint32_t n) {
    const uint32_t tiles = tile_count_of(ctx, n);
    if (tiles == 0) return tile_points_of(ctx);
    return std::min(tile_points_of(ctx), ((n + tiles - 1) / tiles + 15u) & ~15u);
}

// Layout of the tiles' bucket arrays behind the image's own: per tile offs | points | scan.
size_t tile_block_bytes(uint32_t n, uint32_t m, uint32_t L, uint32_t ntiles, uint32_t tp, std::vector<size_t>* off) {
    size_t o = 0;
    for (uint32_t k = 0; k < ntiles; ++k) {
        const uint32_t nk = std::min(tp, n - k * tp);
        if (off) off->push_back(o);
        o += align_up(size_t(L) * ((size_t(1) << m) + 1) * 4);
        if (off) off->push_back(o);
        o += align_up(size_t(L) * nk * 2);
        if (off) off->push_back(o);
        o += align_up(size_t(L) * nk * 2) + kAlign;
    }
    return o;
}

size_t image_block_bytes(uint32_t n, uint32_t m, uint32_t L, size_t off[9], bool sorted_copies) {
    size_t o = 0;
    off[0] = o; o += align_up(size_t(n) * kDim);
    off[1] = o; o += align_up(size_t(n) * 16);
    off[2] = o; o += align_up(size_t(n) * 16);
    off[3] = o; o += align_up(size_t(n) * L * 4);
    if (m > uint32_t(kMaxShortBits)) {
        // sparse bucket index (general_kernels.cuh): L x n keys  code << 16 | point  in the place of the dense offsets;
        // no point / scan lists, no bucket-sorted copies
        off[4] = o; o += align_up(size_t(L) * n * 8);
        off[5] = off[6] = o;
        off[7] = off[8] = 0;
        return std::max(o + kAlign, kAlign);
    }
    off[4] = o; o += align_up(size_t(L) * ((size_t(1) << m) + 1) * 4);
    off[5] = o; o += align_up(size_t(L) * n * 2);
    off[6] = o; o += align_up(size_t(L) * n * 2);
    o += kAlign;  // slack: the match kernel may read one id past an empty last bucket
    off[7] = off[8] = 0;
    if (sorted_copies) {  // bucket-sorted codes of the join pass (DevImage::scodes, spop)
        off[7] = o; o += align_up(size_t(L) * n * 32);
        off[8] = o; o += align_up(size_t(L) * n * 2);
    }
    return std::max(o, kAlign);
}

chgpu_status ensure_images_cap(chgpu_ctx* ctx, size_t need) {
    if (need <= ctx->images_cap) return CHGPU_OK;
    size_t cap = std::max<size_t>(ctx->images_cap * 2, 1 << 16);
    while (cap < need) cap *= 2;
    CK(cudaStreamSynchronize(ctx->copy));
    CK(cudaStreamSynchronize(ctx->compute));
    DevImage *nd = nullptr, *nh = nullptr;
    CK(cudaMalloc(&nd, cap * sizeof(DevImage)));
    CK(cudaMallocHost(&nh, cap * sizeof(DevImage)));
    memset(nh, 0, cap * sizeof(DevImage));
    if (ctx->images_cap) {
        memcpy(nh, ctx->h_images, ctx->images_cap * sizeof(DevImage));
        CK(cudaMemcpy(nd, ctx->d_images, ctx->images_cap * sizeof(DevImage), cudaMemcpyDeviceToDevice));
        cudaFree(ctx->d_images);
        cudaFreeHost(ctx->h_images);
    }
    ctx->d_images = nd;
    ctx->h_images = nh;
    ctx->images_cap = cap;
    return CHGPU_OK;
}

// Pushes images[slot].dev to the device table through the pinned mirror (copy stream).
chgpu_status publish_slot(chgpu_ctx* ctx, uint32_t slot) {
    ctx->h_images[slot] = ctx->images[slot].dev;
    CK(cudaMemcpyAsync(ctx->d_images + slot, ctx->h_images + slot, sizeof(DevImage), cudaMemcpyHostToDevice,
                       ctx->copy));
    return CHGPU_OK;
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// H2D on the copy stream.  Pageable sources go through the pinned staging ring so the copy
// engine overlaps the host memcpy of the next chunk; pinned sources are copied in place and
// the stream is drained before returning (the caller may reuse the buffer immediately).
chgpu_status h2d(chgpu_ctx* ctx, void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return CHGPU_OK;
    if (is_pinned(src)) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->copy));
        CK(cudaStreamSynchronize(ctx->copy));
        return CHGPU_OK;
    }
    size_t done = 0;
    while (done < bytes) {
        const size_t chunk = std::min(kStageBytes, bytes - done);
        const int s = ctx->stage_next;
        ctx->stage_next = (s + 1) % kStageSlots;
        CK(cudaEventSynchronize(ctx->stage_ev[s]));
        memcpy(ctx->stage[s], static_cast<const char*>(src) + done, chunk);
        CK(cudaMemcpyAsync(static_cast<char*>(dst) + done, ctx->stage[s], chunk, cudaMemcpyHostToDevice, ctx->copy));
        CK(cudaEventRecord(ctx->stage_ev[s], ctx->copy));
        done += chunk;
    }
    return CHGPU_OK;
}

constexpr uint32_t kDenseIds = 1u << 22;
void dense_set(chgpu_ctx* ctx, uint32_t image_id, uint32_t slot) {
    if (image_id >= kDenseIds) return;
    if (image_id >= ctx->slot_dense.size())
        ctx->slot_dense.resize(std::max<size_t>(size_t(image_id) + 1, std::min<size_t>(kDenseIds, ctx->slot_dense.size() * 2 + 1024)), kNone);
    ctx->slot_dense[image_id] = slot;
}

chgpu_status find_slot(chgpu_ctx* ctx, uint32_t image_id, uint32_t* slot) {
    if (image_id < ctx->slot_dense.size() && ctx->slot_dense[image_id] != kNone) {
        *slot = ctx->slot_dense[image_id];
        return CHGPU_OK;
    }
    const auto it = ctx->slot_of.find(image_id);
    if (it == ctx->slot_of.end()) return fail(ctx, CHGPU_ENOTFOUND, "image %u is not resident", image_id);
    *slot = it->second;
    return CHGPU_OK;
}

// copy stream waits for compute (WAR on recycled blocks), compute waits for uploads (RAW).
chgpu_status order_copy_after_compute(chgpu_ctx* ctx) {
    CK(cudaEventRecord(ctx->ev_compute, ctx->compute));
    CK(cudaStreamWaitEvent(ctx->copy, ctx->ev_compute, 0));
    return CHGPU_OK;
}
chgpu_status order_compute_after_copy(chgpu_ctx* ctx) {
    CK(cudaEventRecord(ctx->ev_upload, ctx->copy));
    CK(cudaStreamWaitEvent(ctx->compute, ctx->ev_upload, 0));
    return CHGPU_OK;
}

// Returns the slot (and the hidden tile slots behind it) to the free list and its block to the arena.
void release_slot(chgpu_ctx* ctx, uint32_t slot) {
    ImageRec& r = ctx->images[slot];
    for (const uint32_t ts : r.tile_slots) {
        ctx->images[ts] = ImageRec{};
        ctx->free_slots.push_back(ts);
    }
    ctx->arena.release(r.block, r.block_bytes);
    r = ImageRec{};
    ctx->free_slots.push_back(slot);
}

uint32_t take_slot(chgpu_ctx* ctx) {
    if (!ctx->free_slots.empty()) {
        const uint32_t slot = ctx->free_slots.back();
        ctx->free_slots.pop_back();
        return slot;
    }
    ctx->images.emplace_back();
    return static_cast<uint32_t>(ctx->images.size() - 1);
}

chgpu_status alloc_image(chgpu_ctx* ctx, uint32_t image_id, uint32_t n, uint32_t* slot_out) {
    if (!ctx->has_family)
        return fail(ctx, CHGPU_ELOGIC, "chgpu_set_family must precede image uploads (block layout depends on m, L)");
    if (n > kMaxPoints) return fail(ctx, CHGPU_EUNSUPPORTED, "image %u has %u points; device path holds <= %u", image_id, n, kMaxPoints);
    const auto it = ctx->slot_of.find(image_id);
    if (it != ctx->slot_of.end()) {
        // replacing: drain both streams so no kernel or copy still reads the old block
        CK(cudaStreamSynchronize(ctx->copy));
        CK(cudaStreamSynchronize(ctx->compute));
        release_slot(ctx, it->second);
        ctx->slot_of.erase(it);
        dense_set(ctx, image_id, kNone);
    }
    const uint32_t m = ctx->fam.short_bits, L = ctx->fam.table_count;
    const uint32_t ntiles = tile_count_of(ctx, n), tp = balanced_tile_points(ctx, n);
    const uint32_t slot = take_slot(ctx);
    std::vector<uint32_t> tile_slots(ntiles);
    for (uint32_t& ts : tile_slots) ts = take_slot(ctx);
    auto give_back = [&] {
        for (const uint32_t ts : tile_slots) ctx->free_slots.push_back(ts);
        ctx->free_slots.push_back(slot);
    };
    uint32_t top = slot;
    for (const uint32_t ts : tile_slots) top = std::max(top, ts);
    if (const chgpu_status s = ensure_images_cap(ctx, size_t(top) + 1)) {
        give_back();
        return s;
    }
    size_t off[9];
    std::vector<size_t> toff;
    const bool sorted_copies = n != 0 && !ctx->sparse;  // (tiled images too: the join pass replaces the tiles' min pass)
    const size_t own = image_block_bytes(n, m, L, off, sorted_copies);
    const size_t bytes = own + tile_block_bytes(n, m, L, ntiles, tp, &toff);
    char* block = nullptr;
    const cudaError_t e = ctx->arena.alloc(bytes, &block);
    if (e != cudaSuccess) {
        cudaGetLastError();
        give_back();
        return fail(ctx, CHGPU_ENOMEM, "arena allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
    }
    ImageRec& r = ctx->images[slot];
    r.block = block;
    r.block_bytes = bytes;
    r.image_id = image_id;
    r.used = true;
    r.dev.desc = reinterpret_cast<const uint8_t*>(block + off[0]);
    r.dev.kp = reinterpret_cast<const float4*>(block + off[1]);
    r.dev.longs = reinterpret_cast<uint4*>(block + off[2]);
    r.dev.shorts = reinterpret_cast<uint32_t*>(block + off[3]);
    r.dev.offs = reinterpret_cast<uint32_t*>(block + off[4]);
    r.dev.points = reinterpret_cast<uint16_t*>(block + off[5]);
    r.dev.scan = reinterpret_cast<uint16_t*>(block + off[6]);
    r.dev.scodes = sorted_copies ? reinterpret_cast<uint4*>(block + off[7]) : nullptr;
    r.dev.spop = sorted_copies ? reinterpret_cast<int16_t*>(block + off[8]) : nullptr;
    r.dev.n = n;
    r.dev.flags = 0;
    r.tile_slots = tile_slots;
    r.tile_points = tp;
    for (uint32_t k = 0; k < ntiles; ++k) {
        ImageRec& t = ctx->images[tile_slots[k]];
        t = ImageRec{};
        t.image_id = image_id;
        t.used = true;
        const size_t base = size_t(k) * tp;
        t.dev.desc = r.dev.desc + base * kDim;
        t.dev.kp = r.dev.kp + base;
        t.dev.longs = r.dev.longs + base;
        t.dev.shorts = r.dev.shorts + base * L;
        t.dev.offs = reinterpret_cast<uint32_t*>(block + own + toff[3 * k]);
        t.dev.points = reinterpret_cast<uint16_t*>(block + own + toff[3 * k + 1]);
        t.dev.scan = reinterpret_cast<uint16_t*>(block + own + toff[3 * k + 2]);
        t.dev.scodes = nullptr;
        t.dev.spop = nullptr;
        t.dev.n = std::min(tp, n - k * tp);
        t.dev.flags = 0;
        if (const chgpu_status s = publish_slot(ctx, tile_slots[k])) return s;
    }
    ctx->slot_of[image_id] = slot;
    dense_set(ctx, image_id, slot);
    *slot_out = slot;
    return CHGPU_OK;
}

// Slots whose bucket index has to be (re)built with the codes of `slots`: the images and their tiles.
std::vector<uint32_t> with_tile_slots(const chgpu_ctx* ctx, const std::vector<uint32_t>& slots) {
    std::vector<uint32_t> all(slots);
    for (const uint32_t s : slots)
        all.insert(all.end(), ctx->images[s].tile_slots.begin(), ctx->images[s].tile_slots.end());
    return all;
}

chgpu_status ensure_slots_scratch(chgpu_ctx* ctx, size_t count) {
    if (count <= ctx->slots_cap) return CHGPU_OK;
    CK(cudaStreamSynchronize(ctx->compute));
    CK(cudaStreamSynchronize(ctx->copy));
    if (ctx->d_slots) cudaFree(ctx->d_slots);
    ctx->slots_cap = std::max<size_t>(count, 4096);
    CK(cudaMalloc(&ctx->d_slots, ctx->slots_cap * sizeof(uint32_t)));
    return CHGPU_OK;
}

chgpu_status launch_bucket_build(chgpu_ctx* ctx, uint32_t count) {
    const uint32_t m = ctx->fam.short_bits, L = ctx->fam.table_count;
    if (ctx->sparse) {
        sparse_index_kernel<<<dim3(count, L), kSparseThreads, 0, ctx->compute>>>(ctx->d_images, ctx->d_slots, L);
        CK(cudaGetLastError());
        return CHGPU_OK;
    }
    const size_t smem = size_t(L) << m << 2;
    CK(cudaFuncSetAttribute(bucket_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    bucket_build_kernel<<<count, L * 32, smem, ctx->compute>>>(ctx->d_images, ctx->d_slots, m, L);
    CK(cudaGetLastError());
    return CHGPU_OK;
}

template <int RR>
cudaError_t launch_hash_rr(chgpu_ctx* ctx, dim3 grid, const uint32_t* slots, bool guarded) {
    const size_t smem = hash_smem_bytes();
    cudaError_t e = cudaFuncSetAttribute(hash_codes_kernel<RR>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    hash_codes_kernel<RR><<<grid, kHashThreads, smem, ctx->compute>>>(
        ctx->d_images, slots, ctx->d_planes, ctx->d_centering, ctx->fam.short_bits, ctx->fam.table_count,
        ctx->fam.long_bits, guarded ? ctx->d_hq_count : nullptr, kHashQueueCap);
    return cudaGetLastError();
}

cudaError_t launch_hash_exact(chgpu_ctx* ctx, dim3 grid, const uint32_t* slots, int reduce_rounds, bool guarded) {
    switch (reduce_rounds) {
        case 0: return launch_hash_rr<0>(ctx, grid, slots, guarded);
        case 1: return launch_hash_rr<1>(ctx, grid, slots, guarded);
        case 2: return launch_hash_rr<2>(ctx, grid, slots, guarded);
        case 3: return launch_hash_rr<3>(ctx, grid, slots, guarded);
        case 4: return launch_hash_rr<4>(ctx, grid, slots, guarded);
        case 5: return launch_hash_rr<5>(ctx, grid, slots, guarded);
        case 6: return launch_hash_rr<6>(ctx, grid, slots, guarded);
        default: return launch_hash_rr<7>(ctx, grid, slots, guarded);
    }
}

// K1f + fixup + guarded exact kernel for `count` images whose slots start at `slots` (device).
cudaError_t launch_hash_filtered(chgpu_ctx* ctx, const uint32_t* slots, uint32_t count, uint32_t max_n, int reduce_rounds) {
    cudaError_t e = cudaMemsetAsync(ctx->d_hq_count, 0, sizeof(unsigned int), ctx->compute);
    if (e != cudaSuccess) return e;
    HashFilterParams P{};
    P.images = ctx->d_images;
    P.slots = slots;
    P.planes_t = ctx->d_planes_t;
    P.bias = ctx->d_bias;
    P.hnorm = ctx->d_hnorm;
    P.a_rel = ctx->filt_a_rel;
    P.a_abs = ctx->filt_a_abs;
    P.gpad = ctx->gpad;
    P.m = ctx->fam.short_bits;
    P.L = ctx->fam.table_count;
    P.nlong = ctx->fam.long_bits;
    P.queue = ctx->d_hq;
    P.queue_cap = kHashQueueCap;
    P.queue_count = ctx->d_hq_count;
    if (ctx->hash_mode == CHGPU_HASH_TENSOR && ctx->tc_ready) {
        // K1t: the same filter contract on the tensor cores (hash_tc.cuh); queue, fixup and overflow path are shared
        HashTcParams T{};
        T.images = ctx->d_images;
        T.slots = slots;
        T.limbs = ctx->d_tc_limbs;
        T.inv_scale = ctx->d_tc_const;
        T.bias = ctx->d_tc_const + ctx->tc_npad;
        T.alpha = ctx->d_tc_const + 2 * size_t(ctx->tc_npad);
        T.beta = ctx->d_tc_const + 3 * size_t(ctx->tc_npad);
        T.npad = ctx->tc_npad;
        T.m = P.m;
        T.L = P.L;
        T.nlong = P.nlong;
        T.count = count;
        T.tiles_max = (max_n + kTcPoints - 1) / kTcPoints;
        T.queue = P.queue;
        T.queue_cap = P.queue_cap;
        T.queue_count = P.queue_count;
        const size_t tsmem = hash_tc_smem_bytes(ctx->tc_npad);
        e = cudaFuncSetAttribute(hash_filter_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(tsmem));
        if (e != cudaSuccess) return e;
        const uint64_t units = uint64_t(count) * T.tiles_max;
        const uint32_t tgrid = uint32_t(std::min<uint64_t>(units, uint64_t(ctx->prop.multiProcessorCount)));
        hash_filter_tc_kernel<<<tgrid, kTcThreads, tsmem, ctx->compute>>>(T);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    } else {
        const size_t smem = hash_filter_smem_bytes();
        e = cudaFuncSetAttribute(hash_filter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        const dim3 grid((max_n + kFiltPoints - 1) / kFiltPoints, count);
        hash_filter_kernel<<<grid, kFiltThreads, smem, ctx->compute>>>(P);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    hash_fixup_kernel<<<ctx->prop.multiProcessorCount * 4, 128, 0, ctx->compute>>>(
        ctx->d_images, ctx->d_planes, ctx->d_centering, ctx->d_hq, kHashQueueCap, ctx->d_hq_count, P.m, P.L,
        reduce_rounds, ctx->d_hstats);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // overflow path: returns at once unless the queue was too small for this batch
    return launch_hash_exact(ctx, dim3((max_n + kHashTilePoints - 1) / kHashTilePoints, count), slots, reduce_rounds, true);
}

// Derives the filter constants of K1f from the installed planes and centering (both must be known).
chgpu_status refresh_hash_filter(chgpu_ctx* ctx) {
    ctx->filter_ready = false;
    if (!ctx->has_family || !ctx->has_centering) return CHGPU_OK;
    const uint32_t G = ctx->fam.table_count * ctx->fam.short_bits + ctx->fam.long_bits;
    const uint32_t gpad = (G + kFiltPlanes - 1) / kFiltPlanes * kFiltPlanes;
    double mean_sq = 0.0;
    for (int x = 0; x < kDim; ++x) {
        const double c = ctx->h_centering[x];
        if (!std::isfinite(c) || std::fabs(c) > 1e6) return CHGPU_OK;  // outside the bound's premises: exact kernel only
        mean_sq += c * c;
    }
    std::vector<float> pt(size_t(kDim) * gpad, 0.0f);
    std::vector<double> bias(gpad, 0.0), hnorm(gpad, 0.0);
    for (uint32_t g = 0; g < G; ++g) {
        const double* h = ctx->h_planes.data() + size_t(g) * kDim;
        long double b = 0.0L, sq = 0.0L;
        for (int x = 0; x < kDim; ++x) {
            if (!std::isfinite(h[x]) || std::fabs(h[x]) > 1e30) return CHGPU_OK;
            pt[size_t(x) * gpad + g] = static_cast<float>(h[x]);
            b += static_cast<long double>(ctx->h_centering[x]) * h[x];
            sq += static_cast<long double>(h[x]) * h[x];
        }
        bias[g] = static_cast<double>(b);
        hnorm[g] = std::sqrt(static_cast<double>(sq)) * (1.0 + 1e-12);
    }
    if (gpad != ctx->gpad || !ctx->d_planes_t) {
        CK(cudaStreamSynchronize(ctx->compute));
        cudaFree(ctx->d_planes_t); cudaFree(ctx->d_bias); cudaFree(ctx->d_hnorm);
        ctx->d_planes_t = nullptr; ctx->d_bias = nullptr; ctx->d_hnorm = nullptr;
        CK(cudaMalloc(&ctx->d_planes_t, pt.size() * sizeof(float)));
        CK(cudaMalloc(&ctx->d_bias, gpad * sizeof(double)));
        CK(cudaMalloc(&ctx->d_hnorm, gpad * sizeof(double)));
        ctx->gpad = gpad;
    }
    CK(cudaStreamSynchronize(ctx->compute));
    CK(cudaMemcpy(ctx->d_planes_t, pt.data(), pt.size() * sizeof(float), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_bias, bias.data(), gpad * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_hnorm, hnorm.data(), gpad * sizeof(double), cudaMemcpyHostToDevice));
    // A_p = a_rel ||d_p|| + a_abs  (see K1f): 136 u32 + 2^-44 relative, 2^-44 ||centering|| absolute
    ctx->filt_a_rel = 136.0 * std::ldexp(1.0, -24) + std::ldexp(1.0, -44);
    ctx->filt_a_abs = std::ldexp(1.0, -44) * std::sqrt(mean_sq) * (1.0 + 1e-12);
    ctx->filter_ready = true;

    // K1t: H_x = rint(h_x * 2^(22 - e_g)) as three balanced int8 limbs; constants of the bound (hash_tc.cuh)
    ctx->tc_ready = false;
    const uint32_t npad = (G + kTcPassPlanes - 1) / kTcPassPlanes * kTcPassPlanes;
    if (npad <= uint32_t(kTcMaxPlanes)) {
        std::vector<int8_t> limbs(size_t(3) * npad * kDim, 0);
        std::vector<double> cst(size_t(4) * npad, 0.0);
        const double cnorm = std::sqrt(mean_sq) * (1.0 + 1e-12);
        const double up = 1.0 + std::ldexp(1.0, -40);
        for (uint32_t g = 0; g < npad; ++g) {
            double inv = 1.0, alpha = 0.0, beta = 1e-30, b = 0.0;
            if (g < G) {
                const double* h = ctx->h_planes.data() + size_t(g) * kDim;
                double hmax = 0.0;
                for (int x = 0; x < kDim; ++x) hmax = std::max(hmax, std::fabs(h[x]));
                int e = hmax > 0.0 ? std::ilogb(hmax) + 1 : 0;  // 2^e > hmax
                e = std::min(std::max(e, -900), 900);
                const double S = std::ldexp(1.0, 22 - e);
                for (int x = 0; x < kDim; ++x) {
                    long long H = std::llrint(h[x] * S);  // |H| <= 2^22 (h below 2^-900: 0, inside the bound all the same)
                    const long long l2 = ((H + 128) & 255) - 128;
                    H = (H - l2) / 256;
                    const long long l1 = ((H + 128) & 255) - 128;
                    const long long l0 = (H - l1) / 256;  // in [-64, 64]
                    limbs[(size_t(0) * npad + g) * kDim + x] = static_cast<int8_t>(l0);
                    limbs[(size_t(1) * npad + g) * kDim + x] = static_cast<int8_t>(l1);
                    limbs[(size_t(2) * npad + g) * kDim + x] = static_cast<int8_t>(l2);
                }
                inv = std::ldexp(1.0, e - 22);
                b = bias[g];
                alpha = (std::ldexp(1.0, e - 23) + std::ldexp(1.0, -45) * hnorm[g]) * up;
                beta = (std::ldexp(1.0, -45) * cnorm * hnorm[g] + 1e-30) * up;
            }
            cst[g] = inv;
            cst[npad + g] = b;
            cst[2 * size_t(npad) + g] = std::nextafter(alpha, HUGE_VAL);
            cst[3 * size_t(npad) + g] = std::nextafter(beta, HUGE_VAL);
        }
        if (npad != ctx->tc_npad || !ctx->d_tc_limbs) {
            cudaFree(ctx->d_tc_limbs);
            cudaFree(ctx->d_tc_const);
            ctx->d_tc_limbs = nullptr;
            ctx->d_tc_const = nullptr;
            CK(cudaMalloc(&ctx->d_tc_limbs, limbs.size()));
            CK(cudaMalloc(&ctx->d_tc_const, cst.size() * sizeof(double)));
            ctx->tc_npad = npad;
        }
        CK(cudaMemcpy(ctx->d_tc_limbs, limbs.data(), limbs.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->d_tc_const, cst.data(), cst.size() * sizeof(double), cudaMemcpyHostToDevice));
        ctx->tc_ready = true;
    }
    return CHGPU_OK;
}

bool cfg_valid(const chgpu_match_cfg& c, uint32_t long_bits, const char** why) {
    // validate(MatchConfig), matcher.cpp:9-17
    if (c.top_k < 2) { *why = "top_k must be >= 2 for the ratio test"; return false; }
    if (c.hamming_threshold > long_bits) { *why = "hamming_threshold exceeds long code length"; return false; }
    if (!(c.ratio > 0.0 && c.ratio < 1.0)) { *why = "ratio must be in (0, 1)"; return false; }
    if (c.reduce_rounds < 0 || c.reduce_rounds > 7) { *why = "reduce_rounds out of range 0..7"; return false; }
    return true;
}

size_t offs_smem_bytes(const chgpu_ctx* ctx) {
    // dense bucket offsets of one image, rounded up to the 16-byte granule of cp.async.bulk
    return (size_t(ctx->fam.table_count) * ((size_t(1) << ctx->fam.short_bits) + 1) * 4 + 15) & ~size_t(15);
}

size_t stage_smem_bytes(const chgpu_ctx* ctx, bool guided = false) {
    // per-warp lookup staging of the match kernel
    return size_t(kMatchThreads / 32) * stage_bytes_per_warp(match_table_slots(ctx->fam.table_count, guided));
}

cudaError_t launch_match(chgpu_ctx* ctx, MatchParams& P, bool smem_train, uint32_t max_nt, uint32_t* grid) {
    const int sms = ctx->prop.multiProcessorCount;
    const bool guided = P.fmats != nullptr;
    P.smem_long_bytes = smem_train ? std::max<uint32_t>(max_nt * 16u, 16u) : 0u;
    const size_t smem = smem_train ? size_t(P.smem_long_bytes) + offs_smem_bytes(ctx) + stage_smem_bytes(ctx, guided)
                                   : stage_smem_bytes(ctx, guided);
    if (P.dbg_ranked != nullptr) return launch_match_dbg(P, smem_train, smem, sms, ctx->compute, grid);
    if (guided) return launch_match_guided(P, smem_train, smem, sms, ctx->compute, grid);
    return smem_train ? launch_match_smem(P, smem, sms, ctx->compute, grid)
                      : launch_match_global(P, smem, sms, ctx->compute, grid);
}

size_t smem_train_capacity(const chgpu_ctx* ctx, bool guided) {
    // points whose codes fit next to the bucket offsets in the dynamic smem of a 1-CTA/SM launch
    // (minus the kernel's static 16 B and the 1 KiB the driver reserves per block)
    const size_t avail = ctx->prop.sharedMemPerBlockOptin - 1024 - 64;
    const size_t offs = offs_smem_bytes(ctx) + stage_smem_bytes(ctx, guided);
    return avail > offs ? (avail - offs) / 16 : 0;
}

enum class SinkMode { Host, Stream, Device };

struct SubBatch {
    uint32_t first, count;
    uint64_t queries;
    uint32_t max_nt, max_nq;
    // train images larger than the shared-memory tile: matched tile by tile (match_kernels.cuh MODE 1 / 2 + merge)
    bool tiled;
    uint32_t max_tiles, tile_pairs;
    // the join pass needs the bucket-sorted code copies of every image of the sub-batch (DevImage::scodes: not kept for
    // images that are matched through tiles, whichever side of a pair they are on) and buckets large enough to fill its tiles
    bool no_join = false;
    uint64_t train_points = 0;
};
constexpr uint64_t kTileListBytes = uint64_t(1) << 30;  // cap of the per-query list scratch of a tiled sub-batch

chgpu_status ensure_match_buffers(chgpu_ctx* ctx, MatchBuffers& b, const SubBatch& sb, bool host_side) {
    if (b.pairs_cap < sb.count) {
        CK(cudaStreamSynchronize(ctx->compute));
        CK(cudaStreamSynchronize(ctx->copy));
        if (b.d_pairs) { cudaFree(b.d_pairs); cudaFreeHost(b.h_pairs); cudaFree(b.d_counts); cudaFree(b.d_offsets); cudaFreeHost(b.h_offsets); }
        const size_t cap = std::max<size_t>(sb.count, 4096);
        CK(cudaMalloc(&b.d_pairs, cap * sizeof(PairDesc)));
        CK(cudaMallocHost(&b.h_pairs, cap * sizeof(PairDesc)));
        CK(cudaMalloc(&b.d_counts, cap * sizeof(uint32_t)));
        CK(cudaMalloc(&b.d_offsets, (cap + 1) * sizeof(unsigned long long)));
        CK(cudaMallocHost(&b.h_offsets, (cap + 1) * sizeof(unsigned long long)));
        b.pairs_cap = cap;
    }
    if (b.records_cap < sb.queries) {
        CK(cudaStreamSynchronize(ctx->compute));
        CK(cudaStreamSynchronize(ctx->copy));
        if (b.d_records) cudaFree(b.d_records);
        const size_t cap = std::max<size_t>(sb.queries, 1 << 20);
        CK(cudaMalloc(&b.d_records, cap * sizeof(uint4)));
        b.records_cap = cap;
    }
    if (!b.ev_done) {
        CK(cudaEventCreateWithFlags(&b.ev_done, cudaEventDisableTiming));
        CK(cudaEventCreate(&b.ev_k0));
        CK(cudaEventCreate(&b.ev_k1));
    }
    (void)host_side;
    return CHGPU_OK;
}

chgpu_status ensure_host_records(chgpu_ctx* ctx, MatchBuffers& b, size_t need) {
    if (need <= b.h_records_cap) return CHGPU_OK;
    if (b.h_records) cudaFreeHost(b.h_records);
    size_t cap = std::max<size_t>(b.h_records_cap * 2, kSinkChunkEntries);
    while (cap < need) cap *= 2;
    b.h_records = nullptr;
    b.h_records_cap = 0;
    CK(cudaMallocHost(&b.h_records, cap * sizeof(chgpu_match_record)));
    b.h_records_cap = cap;
    return CHGPU_OK;
}

void load_pump(chgpu_load_job* job, bool block);  // streaming loader, below

struct MatchRun {
    const uint32_t* pairs;
    uint32_t npairs;
    chgpu_match_cfg cfg;
    SinkMode mode;
    // Host mode
    uint64_t* offsets = nullptr;
    chgpu_match_record* records = nullptr;
    uint64_t capacity = 0;
    uint64_t total = 0;
    bool overflow = false;
    // Stream mode
    chgpu_sink_fn sink = nullptr;
    void* user = nullptr;
    // guided (epipolar band)
    const double* fmats = nullptr;  // npairs x 9, host
    double band_px = 0.0;
    // debug
    uint32_t* dbg_ranked = nullptr;
    uint32_t* dbg_count = nullptr;
    // explicit candidate lists of the ONE pair of the run (chgpu_match_pair_lists): already on the device
    bool lists = false;
};

chgpu_status run_match_impl(chgpu_ctx* ctx, MatchRun& run, chgpu_match_stats* stats_out);

// A failure in the middle of a pair list (an aborting sink, a CUDA error, an allocation that fails) returns while the
// next sub-batch is still queued on the streams: drain them before handing the status back, so that the buffers the
// next call reuses (pair table, result scratch, pinned chunks) have no reader or writer left and the context stays usable.
chgpu_status run_match(chgpu_ctx* ctx, MatchRun& run, chgpu_match_stats* stats_out) {
    const chgpu_status s = run_match_impl(ctx, run, stats_out);
    if (s != CHGPU_OK) {
        cudaStreamSynchronize(ctx->compute);
        cudaStreamSynchronize(ctx->copy);
        cudaGetLastError();
    }
    return s;
}

chgpu_status run_match_impl(chgpu_ctx* ctx, MatchRun& run, chgpu_match_stats* stats_out) {
    DeviceGuard guard(ctx->device);
    if (!ctx->has_family) return fail(ctx, CHGPU_ELOGIC, "no hash family installed");
    const char* why = nullptr;
    if (!cfg_valid(run.cfg, ctx->fam.long_bits, &why)) return fail(ctx, CHGPU_EINVAL, "%s", why);
    // what the tuned kernels are not laid out for goes through the general path (general_kernels.cuh)
    const bool general = ctx->sparse || run.cfg.top_k > uint32_t(kMaxTopK) || run.lists;
    const uint32_t npairs = run.npairs;
    chgpu_match_stats st{};
    st.pairs = npairs;
    if (run.mode == SinkMode::Host && run.offsets) run.offsets[0] = 0;
    if (npairs == 0) {
        if (stats_out) *stats_out = st;
        return CHGPU_OK;
    }

    // ---- resolve pairs, cut sub-batches ---------------------------------------------------
    std::vector<PairDesc> descs(npairs);
    std::vector<SubBatch> subs;
    {
        SubBatch cur{0, 0, 0, 0, 0, false, 0, 0};
        // The persistent grid hands out one unit per pair: a sub-batch whose pair count is a multiple of the CTA count
        // ends with every SM busy (4,096 pairs on 148 SMs leave 48 of them idle for the last unit: ~1 % of a launch).
        uint32_t pairs_cap = 1u << 20;
        {
            uint32_t s0;
            const char* no_round = getenv("CHGPU_NO_SUBBATCH_ROUNDING");
            if (!(no_round && no_round[0] == '1') && find_slot(ctx, run.pairs[0], &s0) == CHGPU_OK && ctx->images[s0].dev.n) {
                const uint64_t fit = ctx->sub_batch_queries / ctx->images[s0].dev.n;
                const uint64_t sms = uint64_t(ctx->prop.multiProcessorCount);
                if (fit >= 4 * sms) pairs_cap = uint32_t(std::min<uint64_t>(fit / sms * sms, 1u << 20));
            }
        }
        for (uint32_t k = 0; k < npairs; ++k) {
            uint32_t si, sj;
            if (const chgpu_status s = find_slot(ctx, run.pairs[2 * k], &si)) return s;
            if (const chgpu_status s = find_slot(ctx, run.pairs[2 * k + 1], &sj)) return s;
            const DevImage& I = ctx->images[si].dev;
            const DevImage& J = ctx->images[sj].dev;
            if (!(I.flags & 1u) || !(J.flags & 1u))
                return fail(ctx, CHGPU_ELOGIC, "pair (%u,%u): codes not computed (call chgpu_hash_images first)",
                            run.pairs[2 * k], run.pairs[2 * k + 1]);
            const uint32_t gi = ctx->images[si].hash_gen, gj = ctx->images[sj].hash_gen;
            if ((gi && gi != ctx->centering_gen) || (gj && gj != ctx->centering_gen))
                return fail(ctx, CHGPU_ELOGIC, "pair (%u,%u): codes were computed under a centering that has been replaced "
                            "(call chgpu_hash_images again)", run.pairs[2 * k], run.pairs[2 * k + 1]);
            const uint32_t tiles = general ? 0u : uint32_t(ctx->images[sj].tile_slots.size());
            const bool tiled = tiles != 0;
            if (cur.count && (cur.queries + I.n > ctx->sub_batch_queries || cur.count >= pairs_cap || tiled != cur.tiled ||
                              (tiled && (cur.queries + I.n) * std::max(cur.max_tiles, tiles) * run.cfg.top_k * 4 > kTileListBytes))) {
                subs.push_back(cur);
                cur = SubBatch{k, 0, 0, 0, 0, false, 0, 0};
            }
            descs[k] = PairDesc{si, sj, cur.queries, 0u, 0u, cur.count, uint32_t(cur.queries)};  // (act_off: join pass)
            cur.tiled = tiled;
            cur.no_join = cur.no_join || (I.n != 0 && I.scodes == nullptr) || (J.n != 0 && J.scodes == nullptr);
            cur.train_points += J.n;
            cur.max_tiles = std::max(cur.max_tiles, tiles);
            cur.tile_pairs += tiles;
            cur.count += 1;
            cur.queries += I.n;
            cur.max_nt = std::max(cur.max_nt, J.n);
            cur.max_nq = std::max(cur.max_nq, I.n);
            st.query_points += I.n;
            st.train_points += J.n;
        }
        subs.push_back(cur);
    }
    uint64_t max_queries = 0;
    for (const SubBatch& sb : subs) max_queries = std::max(max_queries, sb.queries);
    if (ctx->res_cap < max_queries) {
        CK(cudaStreamSynchronize(ctx->compute));
        if (ctx->d_res) cudaFree(ctx->d_res);
        ctx->res_cap = std::max<size_t>(max_queries, 1 << 20);
        CK(cudaMalloc(&ctx->d_res, ctx->res_cap * sizeof(uint2)));
    }
    if (run.dbg_ranked) {
        const size_t need = size_t(subs[0].max_nq) * (run.cfg.top_k + 1);
        if (ctx->dbg_cap < need) {
            if (ctx->d_dbg) cudaFree(ctx->d_dbg);
            CK(cudaMalloc(&ctx->d_dbg, need * sizeof(uint32_t)));
            ctx->dbg_cap = need;
        }
        CK(cudaMemsetAsync(ctx->d_dbg, 0, need * sizeof(uint32_t), ctx->compute));
    }

    if (const chgpu_status s = order_compute_after_copy(ctx)) return s;
    CK(cudaMemsetAsync(ctx->d_stats, 0, sizeof(DevStats), ctx->compute));
    CK(cudaEventRecord(ctx->ev_t0, ctx->compute));

    const size_t cap_nt = smem_train_capacity(ctx, run.fmats != nullptr);
    const bool host_side = run.mode != SinkMode::Device;
    float match_ms = 0.f;
    uint64_t delivered_records = 0;

    // While a background load is open this thread does not sleep on the device: it keeps the loader's issue side going
    // (files the readers finished -> cudaMemcpyAsync on the load stream) under the match kernels and the result copies.
    auto sync_copy = [&]() -> cudaError_t {
        while (ctx->load_job) {
            const cudaError_t q = cudaStreamQuery(ctx->copy);
            if (q != cudaErrorNotReady) return q;
            load_pump(ctx->load_job, false);
            std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
        return cudaStreamSynchronize(ctx->copy);
    };
    // finishes sub-batch s (already launched into mb[s & 1]): D2H + delivery
    auto finish = [&](size_t s) -> chgpu_status {
        MatchBuffers& b = ctx->mb[s & 1];
        const SubBatch& sb = subs[s];
        while (ctx->load_job) {
            const cudaError_t q = cudaEventQuery(b.ev_done);
            if (q == cudaSuccess) break;
            if (q != cudaErrorNotReady) CK(q);
            load_pump(ctx->load_job, false);
            std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
        CK(cudaEventSynchronize(b.ev_done));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, b.ev_k0, b.ev_k1));
        match_ms += ms;
        if (!host_side) return CHGPU_OK;
        CK(cudaMemcpyAsync(b.h_offsets, b.d_offsets, (size_t(sb.count) + 1) * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, ctx->copy));
        CK(sync_copy());
        const uint64_t total = b.h_offsets[sb.count];
        if (run.mode == SinkMode::Host) {
            for (uint32_t k = 0; k < sb.count; ++k) run.offsets[sb.first + k + 1] = delivered_records + b.h_offsets[k + 1];
            if (delivered_records + total > run.capacity) {
                run.overflow = true;
            } else if (total) {
                CK(cudaMemcpyAsync(run.records + delivered_records, b.d_records, total * sizeof(uint4),
                                   cudaMemcpyDeviceToHost, ctx->copy));
                CK(sync_copy());
            }
        } else {
            // Stream mode: the sub-batch reaches the sink in chunks of whole pairs through two pinned buffers of
            // kSinkChunkEntries records (32 MiB each, allocated once): no sub-batch-sized pinned allocation stalls the
            // first launches of a cold run (cudaMallocHost pins ~2.5 GB/s), and chunk i + 1 travels while the sink has chunk i.
            const unsigned long long* ho = b.h_offsets;
            auto chunk_end = [&](uint32_t k0) {
                uint32_t k1 = k0 + 1;
                while (k1 < sb.count && ho[k1 + 1] - ho[k0] <= kSinkChunkEntries) ++k1;
                return k1;
            };
            auto issue = [&](uint32_t k0, uint32_t k1, int j) -> chgpu_status {
                const uint64_t cnt = ho[k1] - ho[k0];
                if (const chgpu_status e = ensure_host_records(ctx, ctx->mb[j], std::max<uint64_t>(cnt, 1))) return e;
                if (cnt)
                    CK(cudaMemcpyAsync(ctx->mb[j].h_records, b.d_records + ho[k0], cnt * sizeof(uint4), cudaMemcpyDeviceToHost, ctx->copy));
                CK(cudaEventRecord(ctx->ev_chunk[j], ctx->copy));
                return CHGPU_OK;
            };
            std::vector<uint64_t> rel;
            uint32_t k0 = 0, k1 = chunk_end(0);
            int j = 0;
            if (const chgpu_status e = issue(k0, k1, j)) return e;
            while (k0 < sb.count) {
                const uint32_t n0 = k1, n1 = n0 < sb.count ? chunk_end(n0) : n0;
                if (n0 < sb.count)
                    if (const chgpu_status e = issue(n0, n1, j ^ 1)) return e;
                while (ctx->load_job) {  // (keeps a background load going instead of sleeping on the copy)
                    const cudaError_t q = cudaEventQuery(ctx->ev_chunk[j]);
                    if (q == cudaSuccess) break;
                    if (q != cudaErrorNotReady) CK(q);
                    load_pump(ctx->load_job, false);
                    std::this_thread::sleep_for(std::chrono::microseconds(20));
                }
                CK(cudaEventSynchronize(ctx->ev_chunk[j]));
                if (run.sink) {
                    static_assert(sizeof(unsigned long long) == sizeof(uint64_t), "offset width");
                    rel.resize(size_t(k1 - k0) + 1);
                    for (uint32_t i = 0; i <= k1 - k0; ++i) rel[i] = ho[k0 + i] - ho[k0];
                    if (run.sink(run.user, sb.first + k0, k1 - k0, rel.data(), ctx->mb[j].h_records) != 0)
                        return fail(ctx, CHGPU_EINVAL, "sink aborted at pair %u", sb.first + k0);
                }
                k0 = n0;
                k1 = n1;
                j ^= 1;
            }
        }
        delivered_records += total;
        return CHGPU_OK;
    };

    for (size_t s = 0; s < subs.size(); ++s) {
        const SubBatch& sb = subs[s];
        MatchBuffers& b = ctx->mb[s & 1];
        if (const chgpu_status e = ensure_match_buffers(ctx, b, sb, host_side)) return e;
        memcpy(b.h_pairs, descs.data() + sb.first, size_t(sb.count) * sizeof(PairDesc));
        CK(cudaMemcpyAsync(b.d_pairs, b.h_pairs, size_t(sb.count) * sizeof(PairDesc), cudaMemcpyHostToDevice, ctx->compute));
        CK(cudaMemsetAsync(b.d_counts, 0, size_t(sb.count) * sizeof(uint32_t), ctx->compute));
        if (run.fmats) {
            if (b.fmats_cap < sb.count) {
                CK(cudaStreamSynchronize(ctx->compute));
                if (b.d_fmats) cudaFree(b.d_fmats);
                b.d_fmats = nullptr;
                b.fmats_cap = 0;
                CK(cudaMalloc(&b.d_fmats, std::max<size_t>(sb.count, 1024) * 9 * sizeof(double)));
                b.fmats_cap = std::max<size_t>(sb.count, 1024);
            }
            // pageable source: the copy is staged by the runtime before the call returns
            CK(cudaMemcpyAsync(b.d_fmats, run.fmats + size_t(sb.first) * 9, size_t(sb.count) * 9 * sizeof(double),
                               cudaMemcpyHostToDevice, ctx->compute));
        }
        CK(cudaMemsetAsync(ctx->d_counter, 0, sizeof(unsigned int), ctx->compute));

        const bool smem_train = sb.max_nt <= cap_nt;
        // enough units to balance the persistent grid: >= 4 per CTA, chunks of >= 256 queries
        const uint32_t ctas = uint32_t(ctx->prop.multiProcessorCount) * (smem_train && sb.max_nt * 16u > 100000u ? 1u : 2u);
        const uint32_t unit_pairs = sb.tiled ? sb.tile_pairs : sb.count;
        uint32_t chunks = 1;
        if (unit_pairs < 4 * ctas) chunks = std::min<uint32_t>((4 * ctas + unit_pairs - 1) / unit_pairs, std::max<uint32_t>(1, sb.max_nq / 256));

        MatchParams P{};
        P.images = ctx->d_images;
        P.pairs = b.d_pairs;
        P.res = ctx->d_res;
        P.pair_counts = b.d_counts;
        P.stats = ctx->d_stats;
        P.unit_counter = ctx->d_counter;
        P.nunits = sb.count * chunks;
        P.chunks_per_pair = chunks;
        P.m = ctx->fam.short_bits;
        P.L = ctx->fam.table_count;
        P.top_k = run.cfg.top_k;
        P.tau = run.cfg.hamming_threshold;
        P.min_ranked = std::max<uint32_t>(2, run.cfg.min_candidates_for_ratio);
        P.long_bits = ctx->fam.long_bits;
        P.ratio_sq = run.cfg.ratio * run.cfg.ratio;
        P.fmats = run.fmats ? b.d_fmats : nullptr;
        P.band_px = run.band_px;
        if (run.dbg_ranked) {
            P.dbg_ranked = ctx->d_dbg;
            P.dbg_count = ctx->d_dbg + size_t(sb.max_nq) * run.cfg.top_k;
        }
        uint32_t grid = 0;
        if (general) {
            GeneralParams G{};
            G.base = P;
            G.npairs = sb.count;
            G.queries = sb.queries;
            G.sparse = ctx->sparse ? 1u : 0u;
            G.list_offs = run.lists ? ctx->d_list_offs : nullptr;
            G.list_ids = run.lists ? ctx->d_list_ids : nullptr;
            const size_t gsmem = size_t(kGenWarps) * kGenCacheKeys * sizeof(uint32_t);
            // CHGPU_GEN_HEADS=0: the A/B reference without the per-lane sorted lists (KG)
            static const bool gen_heads = [] {
                const char* e = getenv("CHGPU_GEN_HEADS");
                return !(e && atoi(e) == 0);
            }();
            const GeneralKernel gen_kernel = general_kernel_for(gen_heads, G.list_offs != nullptr, G.sparse != 0, P.fmats != nullptr);
            CK(cudaFuncSetAttribute(gen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(gsmem)));
            const uint64_t want = (sb.queries + kGenWarps - 1) / kGenWarps;
            grid = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(want, uint64_t(ctx->prop.multiProcessorCount) * 24)));
            G.slice = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(8, sb.queries / (uint64_t(grid) * kGenWarps * 4))));  // (longer runs unbalance the warps: matching queries cluster)
            CK(cudaEventRecord(b.ev_k0, ctx->compute));
            gen_kernel<<<grid, kGenThreads, gsmem, ctx->compute>>>(G);
            CK(cudaGetLastError());
            CK(cudaEventRecord(b.ev_k1, ctx->compute));
        } else if (sb.tiled) {
            // (query image, tile) pairs: min pass, top-k pass for the queries with a candidate within tau, merge
            const uint32_t tp = tile_points_of(ctx);
            if (b.tpairs_cap < sb.tile_pairs) {
                CK(cudaStreamSynchronize(ctx->compute));
                cudaFree(b.d_tpairs);
                cudaFreeHost(b.h_tpairs);
                b.d_tpairs = b.h_tpairs = nullptr;
                b.tpairs_cap = 0;
                const size_t cap = std::max<size_t>(sb.tile_pairs, 4096);
                CK(cudaMalloc(&b.d_tpairs, cap * sizeof(PairDesc)));
                CK(cudaMallocHost(&b.h_tpairs, cap * sizeof(PairDesc)));
                b.tpairs_cap = cap;
            }
            const size_t stride = size_t(sb.max_tiles) * run.cfg.top_k;
            if (ctx->gmin_cap < sb.queries || ctx->lists_cap < sb.queries * stride) {
                CK(cudaStreamSynchronize(ctx->compute));
                if (ctx->gmin_cap < sb.queries) {
                    cudaFree(ctx->d_gmin);
                    cudaFree(ctx->d_gdone);
                    ctx->d_gmin = nullptr;
                    ctx->d_gdone = nullptr;
                    ctx->gmin_cap = 0;
                    CK(cudaMalloc(&ctx->d_gmin, sb.queries * sizeof(uint32_t)));
                    CK(cudaMalloc(&ctx->d_gdone, sb.queries * sizeof(unsigned long long)));
                    ctx->gmin_cap = sb.queries;
                }
                if (ctx->lists_cap < sb.queries * stride) {
                    cudaFree(ctx->d_lists);
                    ctx->d_lists = nullptr;
                    ctx->lists_cap = 0;
                    CK(cudaMalloc(&ctx->d_lists, sb.queries * stride * sizeof(uint32_t)));
                    ctx->lists_cap = sb.queries * stride;
                }
            }
            // active-query scratch: one slice of nq entries per (query image, tile) pair, packed (the list-scratch cap
            // above bounds the sum over the sub-batch by 2^30 / (4 top_k) entries)
            uint32_t ntp = 0;
            size_t act_need = 0;
            for (uint32_t k = 0; k < sb.count; ++k) {
                const PairDesc& pd = descs[sb.first + k];
                const std::vector<uint32_t>& ts = ctx->images[pd.slot_j].tile_slots;
                const size_t nq = (size_t(ctx->images[pd.slot_i].dev.n) + 7) & ~size_t(7);
                for (uint32_t t = 0; t < ts.size(); ++t) {
                    b.h_tpairs[ntp++] = PairDesc{pd.slot_i, ts[t], pd.res_off, t * ctx->images[pd.slot_j].tile_points, t, k, uint32_t(act_need)};
                    act_need += nq;
                }
            }
            if (act_need > UINT32_MAX) return fail(ctx, CHGPU_EUNSUPPORTED, "tiled sub-batch too large (%zu active-query slots)", act_need);
            if (ctx->act_cap < act_need || ctx->nact_cap < sb.tile_pairs) {
                CK(cudaStreamSynchronize(ctx->compute));
                cudaFree(ctx->d_act);
                cudaFree(ctx->d_nact);
                ctx->d_act = nullptr;
                ctx->d_nact = nullptr;
                ctx->act_cap = ctx->nact_cap = 0;
                CK(cudaMalloc(&ctx->d_act, std::max<size_t>(act_need, 8) * sizeof(uint16_t)));
                CK(cudaMalloc(&ctx->d_nact, size_t(sb.tile_pairs) * sizeof(uint32_t)));
                ctx->act_cap = std::max<size_t>(act_need, 8);
                ctx->nact_cap = sb.tile_pairs;
            }
            CK(cudaMemcpyAsync(b.d_tpairs, b.h_tpairs, size_t(ntp) * sizeof(PairDesc), cudaMemcpyHostToDevice, ctx->compute));
            CK(cudaMemsetAsync(ctx->d_gmin, 0xff, sb.queries * sizeof(uint32_t), ctx->compute));
            CK(cudaMemsetAsync(ctx->d_gdone, 0, sb.queries * sizeof(unsigned long long), ctx->compute));
            P.gmin = ctx->d_gmin;
            P.gdone = ctx->d_gdone;
            P.lists = ctx->d_lists;
            P.list_stride = uint32_t(stride);
            P.tile_points = tp;
            P.smem_long_bytes = std::min(tp, sb.max_nt) * 16u;
            const size_t smem = size_t(P.smem_long_bytes) + offs_smem_bytes(ctx) + stage_smem_bytes(ctx);
            const size_t smem_topk = size_t(P.smem_long_bytes) + offs_smem_bytes(ctx) + stage_smem_bytes(ctx, run.fmats != nullptr);
            CK(cudaEventRecord(b.ev_k0, ctx->compute));
            P.pairs = b.d_tpairs;
            P.nunits = ntp * chunks;
            P.act = ctx->d_act;
            P.nact = ctx->d_nact;
            if (ctx->join_enabled && !sb.no_join) {
                // The tensor-core Hamming pass over the WHOLE images (their own bucket index and sorted copies) marks the
                // queries with a candidate within tau in the min-key scratch (0 instead of "none"): it replaces the min
                // pass over every (query, tile); the top-k pass then visits every tile of the marked queries.
                JoinParams JP{};
                JP.images = ctx->d_images;
                JP.pairs = b.d_pairs;
                JP.npairs = sb.count;
                JP.m = ctx->fam.short_bits;
                JP.L = ctx->fam.table_count;
                JP.tau = run.cfg.hamming_threshold;
                JP.hit = nullptr;
                JP.hit_key = ctx->d_gmin;
                JP.stats = ctx->d_stats;
                JP.counter = ctx->d_counter;
                const uint32_t jcells = JP.L << JP.m;
                const uint64_t junits = uint64_t(sb.count) * ((jcells + 31) / 32);
                const uint32_t jgrid = uint32_t(std::min<uint64_t>((junits + kJoinThreads / 32 - 1) / (kJoinThreads / 32),
                                                                   uint64_t(ctx->prop.multiProcessorCount) * 8));
                join_hits_kernel<<<std::max(jgrid, 1u), kJoinThreads, 0, ctx->compute>>>(JP);
                CK(cudaGetLastError());
            } else {
                CK(launch_match_tiled(P, kModeTileMin, smem, ctx->prop.multiProcessorCount, ctx->compute, &grid));
            }
            CK(launch_tile_compact(P, ntp, ctx->compute));
            CK(cudaMemsetAsync(ctx->d_counter, 0, sizeof(unsigned int), ctx->compute));
            CK(launch_match_tiled(P, kModeTileTopK, smem_topk, ctx->prop.multiProcessorCount, ctx->compute, &grid));
            P.pairs = b.d_pairs;
            CK(launch_tile_merge(P, sb.count, sb.max_nq, ctx->compute));
            CK(cudaEventRecord(b.ev_k1, ctx->compute));
            st.match_launches += 2;
            st.total_launches += 3;
        } else if (ctx->join_enabled && !sb.no_join && smem_train && !run.dbg_ranked && sb.queries <= UINT32_MAX &&
                   // the pass works on 16 x 8 tiles of a bucket's queries x train points: it pays from ~20 points per bucket
                   // on both sides (measured: +6 % at 24, +9 % at 32, -4 % at 16, -36 % at 4 per bucket; scripts/sweep.py)
                   ((sb.queries / sb.count) >> ctx->fam.short_bits) >= ctx->join_min_bucket &&
                   ((sb.train_points / sb.count) >> ctx->fam.short_bits) >= ctx->join_min_bucket) {
            // Tensor-core Hamming pass (join_kernels.cuh): which queries have a candidate within tau at all; the match
            // kernel then visits those only.  Every other query keeps the "no match" the scratch is initialised with.
            if (ctx->hit_cap < sb.queries || ctx->act_cap < sb.queries || ctx->nact_cap < sb.count) {
                CK(cudaStreamSynchronize(ctx->compute));
                if (ctx->hit_cap < sb.queries) {
                    cudaFree(ctx->d_hit);
                    ctx->d_hit = nullptr;
                    ctx->hit_cap = 0;
                    CK(cudaMalloc(&ctx->d_hit, sb.queries));
                    ctx->hit_cap = sb.queries;
                }
                if (ctx->act_cap < sb.queries) {
                    cudaFree(ctx->d_act);
                    ctx->d_act = nullptr;
                    ctx->act_cap = 0;
                    CK(cudaMalloc(&ctx->d_act, std::max<size_t>(sb.queries, 8) * sizeof(uint16_t)));
                    ctx->act_cap = std::max<size_t>(sb.queries, 8);
                }
                if (ctx->nact_cap < sb.count) {
                    cudaFree(ctx->d_nact);
                    ctx->d_nact = nullptr;
                    ctx->nact_cap = 0;
                    CK(cudaMalloc(&ctx->d_nact, size_t(sb.count) * sizeof(uint32_t)));
                    ctx->nact_cap = sb.count;
                }
            }
            CK(cudaEventRecord(b.ev_k0, ctx->compute));
            CK(cudaMemsetAsync(ctx->d_hit, 0, sb.queries, ctx->compute));
            CK(cudaMemsetAsync(ctx->d_res, 0xff, sb.queries * sizeof(uint2), ctx->compute));
            JoinParams JP{};
            JP.images = ctx->d_images;
            JP.pairs = b.d_pairs;
            JP.npairs = sb.count;
            JP.m = ctx->fam.short_bits;
            JP.L = ctx->fam.table_count;
            JP.tau = run.cfg.hamming_threshold;
            JP.hit = ctx->d_hit;
            JP.stats = ctx->d_stats;
            JP.counter = ctx->d_counter;
            const uint32_t jcells = JP.L << JP.m;
            const uint64_t junits = uint64_t(sb.count) * ((jcells + 31) / 32);
            const uint32_t jgrid = uint32_t(std::min<uint64_t>((junits + kJoinThreads / 32 - 1) / (kJoinThreads / 32),
                                                               uint64_t(ctx->prop.multiProcessorCount) * 8));
            join_hits_kernel<<<std::max(jgrid, 1u), kJoinThreads, 0, ctx->compute>>>(JP);
            CK(cudaGetLastError());
            join_compact_kernel<<<sb.count, 256, 0, ctx->compute>>>(ctx->d_images, b.d_pairs, sb.count, ctx->d_hit,
                                                                                ctx->d_act, ctx->d_nact);
            CK(cudaGetLastError());
            CK(cudaMemsetAsync(ctx->d_counter, 0, sizeof(unsigned int), ctx->compute));
            P.act = ctx->d_act;
            P.nact = ctx->d_nact;
            P.smem_long_bytes = std::max<uint32_t>(sb.max_nt * 16u, 16u);
            const size_t smem = size_t(P.smem_long_bytes) + offs_smem_bytes(ctx) + stage_smem_bytes(ctx, run.fmats != nullptr);
            CK(launch_match_active(P, smem, ctx->prop.multiProcessorCount, ctx->compute, &grid));
            CK(cudaEventRecord(b.ev_k1, ctx->compute));
            st.total_launches += 2;  // join + list kernels (match_launches keeps counting sub-batches)
        } else {
            CK(cudaEventRecord(b.ev_k0, ctx->compute));
            CK(launch_match(ctx, P, smem_train, sb.max_nt, &grid));
            CK(cudaEventRecord(b.ev_k1, ctx->compute));
        }
        scan_counts_kernel<<<1, 1024, 0, ctx->compute>>>(b.d_counts, sb.count, b.d_offsets, ctx->d_stats);
        CK(cudaGetLastError());
        compact_kernel<<<sb.count, kCompactThreads, 0, ctx->compute>>>(b.d_pairs, ctx->d_images, ctx->d_res, b.d_offsets,
                                                            b.d_records, sb.first, ctx->d_stats);
        CK(cudaGetLastError());
        CK(cudaEventRecord(b.ev_done, ctx->compute));
        st.match_launches += 1;
        st.total_launches += 3;
        // the result scratch d_res is shared: the next match kernel must not start before this
        // sub-batch's compaction, which stream order on `compute` already guarantees.
        // a background load (chgpu_load_chft_files_begin) moves forward under the kernels just launched
        if (ctx->load_job) load_pump(ctx->load_job, false);
        if (s >= 1)
            if (const chgpu_status e = finish(s - 1)) return e;
    }
    if (ctx->load_job) load_pump(ctx->load_job, false);
    if (const chgpu_status e = finish(subs.size() - 1)) return e;
    if (ctx->load_job) load_pump(ctx->load_job, false);

    CK(cudaEventRecord(ctx->ev_t1, ctx->compute));
    CK(cudaMemcpyAsync(ctx->h_stats, ctx->d_stats, sizeof(DevStats), cudaMemcpyDeviceToHost, ctx->compute));
    if (run.dbg_ranked) {
        const uint32_t nq = subs[0].max_nq;
        CK(cudaMemcpyAsync(run.dbg_ranked, ctx->d_dbg, size_t(nq) * run.cfg.top_k * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->compute));
        CK(cudaMemcpyAsync(run.dbg_count, ctx->d_dbg + size_t(nq) * run.cfg.top_k, size_t(nq) * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->compute));
    }
    CK(cudaStreamSynchronize(ctx->compute));
    float total_ms = 0.f;
    CK(cudaEventElapsedTime(&total_ms, ctx->ev_t0, ctx->ev_t1));
    st.matches = ctx->h_stats->matches;
    st.raw_candidates = ctx->h_stats->raw_candidates;
    st.verified_queries = ctx->h_stats->verified_queries;
    st.distances = ctx->h_stats->distances;
    st.records_checksum = ctx->h_stats->checksum;
    st.match_kernel_ms = match_ms;
    st.total_ms = total_ms;
    run.total = host_side ? delivered_records : st.matches;
    if (stats_out) *stats_out = st;
    return CHGPU_OK;
}

}  // namespace

// =================================================================================================
extern "C" {

const char* chgpu_status_name(chgpu_status s) {
    switch (s) {
        case CHGPU_OK: return "ok";
        case CHGPU_EINVAL: return "invalid argument";
        case CHGPU_ELOGIC: return "logic error";
        case CHGPU_ECUDA: return "cuda error";
        case CHGPU_ENOMEM: return "out of memory";
        case CHGPU_EUNSUPPORTED: return "unsupported";
        case CHGPU_EFORMAT: return "format error";
        case CHGPU_ENOTFOUND: return "not found";
        case CHGPU_EMISMATCH: return "parameter mismatch";
    }
    return "?";
}

chgpu_status chgpu_create(int device, chgpu_ctx** out) {
    if (!out) return CHGPU_EINVAL;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0 || device < 0 || device >= count) {
        cudaGetLastError();
        return CHGPU_ECUDA;  // no CPU fallback by design
    }
    chgpu_ctx* ctx = new chgpu_ctx();
    ctx->device = device;
    auto bail = [&](chgpu_status s) {
        chgpu_destroy(ctx);
        return s;
    };
    if (cudaSetDevice(device) != cudaSuccess) return bail(CHGPU_ECUDA);
    if (cudaGetDeviceProperties(&ctx->prop, device) != cudaSuccess) return bail(CHGPU_ECUDA);
    if (ctx->prop.major < 10) {
        fprintf(stderr, "chgpu: device %d is sm_%d%d; this library is built for sm_100a only\n", device,
                ctx->prop.major, ctx->prop.minor);
        return bail(CHGPU_EUNSUPPORTED);
    }
    bool ok = true;
    ok &= cudaStreamCreateWithFlags(&ctx->compute, cudaStreamNonBlocking) == cudaSuccess;
    ok &= cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking) == cudaSuccess;
    ok &= cudaStreamCreateWithFlags(&ctx->load, cudaStreamNonBlocking) == cudaSuccess;
    ok &= cudaEventCreateWithFlags(&ctx->ev_split_jobs, cudaEventDisableTiming) == cudaSuccess;
    for (cudaEvent_t& e : ctx->ev_chunk) ok &= cudaEventCreateWithFlags(&e, cudaEventDisableTiming) == cudaSuccess;
    ok &= cudaEventCreateWithFlags(&ctx->ev_upload, cudaEventDisableTiming) == cudaSuccess;
    ok &= cudaEventCreateWithFlags(&ctx->ev_compute, cudaEventDisableTiming) == cudaSuccess;
    ok &= cudaEventCreate(&ctx->ev_t0) == cudaSuccess;
    ok &= cudaEventCreate(&ctx->ev_t1) == cudaSuccess;
    for (int s = 0; s < kStageSlots && ok; ++s) {
        ok &= cudaMallocHost(reinterpret_cast<void**>(&ctx->stage[s]), kStageBytes) == cudaSuccess;
        ok &= cudaEventCreateWithFlags(&ctx->stage_ev[s], cudaEventDisableTiming) == cudaSuccess;
    }
    ok &= cudaMalloc(&ctx->d_centering, 128 * sizeof(double)) == cudaSuccess;
    ok &= cudaMalloc(&ctx->d_sums, 128 * sizeof(unsigned long long)) == cudaSuccess;
    ok &= cudaMemset(ctx->d_sums, 0, 128 * sizeof(unsigned long long)) == cudaSuccess;
    ok &= cudaMalloc(&ctx->d_stats, sizeof(DevStats)) == cudaSuccess;
    ok &= cudaMallocHost(reinterpret_cast<void**>(&ctx->h_stats), sizeof(DevStats)) == cudaSuccess;
    ok &= cudaMalloc(&ctx->d_counter, sizeof(unsigned int)) == cudaSuccess;
    ok &= cudaMalloc(&ctx->d_hq, size_t(kHashQueueCap) * sizeof(uint2)) == cudaSuccess;
    ok &= cudaMalloc(&ctx->d_hq_count, sizeof(unsigned int)) == cudaSuccess;
    ok &= cudaMalloc(&ctx->d_hstats, sizeof(HashFilterStats)) == cudaSuccess;
    ok &= cudaMemset(ctx->d_hstats, 0, sizeof(HashFilterStats)) == cudaSuccess;
    if (const char* e = getenv("CHGPU_NO_JOIN")) if (e[0] == '1') ctx->join_enabled = false;
    if (const char* e = getenv("CHGPU_JOIN_MIN_BUCKET")) ctx->join_min_bucket = uint32_t(std::max(0, atoi(e)));
    // default: the tensor-core filter (K1t); CHGPU_HASH_FP32=1 / CHGPU_HASH_EXACT=1 select the fp32 filter / the exact kernel
    ctx->hash_mode = CHGPU_HASH_TENSOR;
    if (const char* e = getenv("CHGPU_HASH_FP32")) if (e[0] == '1') ctx->hash_mode = CHGPU_HASH_FILTERED;
    if (const char* e = getenv("CHGPU_HASH_EXACT")) if (e[0] == '1') ctx->hash_mode = CHGPU_HASH_EXACT;
    if (!ok) return bail(CHGPU_ECUDA);
    *out = ctx;
    return CHGPU_OK;
}

void chgpu_destroy(chgpu_ctx* ctx) {
    if (tl_err_ctx == ctx) tl_err_ctx = nullptr;
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    chgpu_load_chft_files_end(ctx, nullptr, nullptr);  // a background load left open
    cudaDeviceSynchronize();
    ctx->arena.destroy();
    for (MatchBuffers& b : ctx->mb) {
        cudaFree(b.d_pairs); cudaFreeHost(b.h_pairs); cudaFree(b.d_counts); cudaFree(b.d_offsets);
        cudaFreeHost(b.h_offsets); cudaFree(b.d_records); cudaFreeHost(b.h_records); cudaFree(b.d_fmats);
        cudaFree(b.d_tpairs); cudaFreeHost(b.h_tpairs);
        if (b.ev_done) cudaEventDestroy(b.ev_done);
        if (b.ev_k0) cudaEventDestroy(b.ev_k0);
        if (b.ev_k1) cudaEventDestroy(b.ev_k1);
    }
    cudaFree(ctx->d_images); cudaFreeHost(ctx->h_images);
    for (int s = 0; s < kStageSlots; ++s) {
        cudaFreeHost(ctx->stage[s]);
        if (ctx->stage_ev[s]) cudaEventDestroy(ctx->stage_ev[s]);
    }
    cudaFree(ctx->d_planes); cudaFree(ctx->d_centering); cudaFree(ctx->d_sums); cudaFree(ctx->d_res);
    cudaFree(ctx->d_stats); cudaFreeHost(ctx->h_stats); cudaFree(ctx->d_counter); cudaFree(ctx->d_slots);
    cudaFree(ctx->d_list_offs); cudaFree(ctx->d_list_ids);
    cudaFree(ctx->d_dbg); cudaFree(ctx->d_gmin); cudaFree(ctx->d_gdone); cudaFree(ctx->d_lists); cudaFree(ctx->d_act); cudaFree(ctx->d_nact); cudaFree(ctx->d_hit);
    cudaFreeHost(ctx->load_pinned);
    cudaFree(ctx->load_region);
    cudaFreeHost(ctx->h_split_jobs);
    cudaFree(ctx->d_split_jobs);
    if (ctx->ev_split_jobs) cudaEventDestroy(ctx->ev_split_jobs);
    for (cudaEvent_t e : ctx->ev_chunk)
        if (e) cudaEventDestroy(e);
    for (auto& b : ctx->load_scratch) cudaFree(b.first);
    cudaFree(ctx->d_planes_t); cudaFree(ctx->d_bias); cudaFree(ctx->d_hnorm); cudaFree(ctx->d_hq);
    cudaFree(ctx->d_tc_limbs); cudaFree(ctx->d_tc_const);
    cudaFree(ctx->d_hq_count); cudaFree(ctx->d_hstats);
    if (ctx->ev_upload) cudaEventDestroy(ctx->ev_upload);
    if (ctx->ev_compute) cudaEventDestroy(ctx->ev_compute);
    if (ctx->ev_t0) cudaEventDestroy(ctx->ev_t0);
    if (ctx->ev_t1) cudaEventDestroy(ctx->ev_t1);
    if (ctx->compute) cudaStreamDestroy(ctx->compute);
    if (ctx->copy) cudaStreamDestroy(ctx->copy);
    if (ctx->load) cudaStreamDestroy(ctx->load);
    cudaGetLastError();
    delete ctx;
}

const char* chgpu_last_error(const chgpu_ctx* ctx) {
    if (!ctx) return "null context";
    // the message of this thread's own last failure on the context; a thread that has had none sees the context's latest
    if (tl_err_ctx != ctx) {
        CtxLock lock_(const_cast<chgpu_ctx*>(ctx));
        tl_err = ctx->err;
        tl_err_ctx = ctx;
    }
    return tl_err.c_str();
}

chgpu_status chgpu_get_device_props(chgpu_ctx* ctx, chgpu_device_props* out) {
    CtxLock lock_(ctx);
    if (!ctx || !out) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    memset(out, 0, sizeof(*out));
    snprintf(out->name, sizeof(out->name), "%s", ctx->prop.name);
    out->sm_count = ctx->prop.multiProcessorCount;
    out->cc_major = ctx->prop.major;
    out->cc_minor = ctx->prop.minor;
    out->smem_per_block_optin = ctx->prop.sharedMemPerBlockOptin;
    CK(cudaMemGetInfo(&out->free_mem, &out->total_mem));
    return CHGPU_OK;
}

chgpu_status chgpu_sync(chgpu_ctx* ctx) {
    CtxLock lock_(ctx);
    if (!ctx) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    CK(cudaStreamSynchronize(ctx->copy));
    CK(cudaStreamSynchronize(ctx->compute));
    return CHGPU_OK;
}

chgpu_status chgpu_image_device_bytes(chgpu_ctx* ctx, uint32_t n, uint64_t* bytes) {
    CtxLock lock_(ctx);
    if (!ctx || !bytes) return CHGPU_EINVAL;
    if (!ctx->has_family) return fail(ctx, CHGPU_ELOGIC, "chgpu_set_family must precede chgpu_image_device_bytes (the layout depends on m, L)");
    if (n > kMaxPoints) return fail(ctx, CHGPU_EUNSUPPORTED, "%u points; device path holds <= %u", n, kMaxPoints);
    const uint32_t m = ctx->fam.short_bits, L = ctx->fam.table_count;
    size_t off[9];
    *bytes = image_block_bytes(n, m, L, off, n != 0) + tile_block_bytes(n, m, L, tile_count_of(ctx, n), balanced_tile_points(ctx, n), nullptr);
    return CHGPU_OK;
}

chgpu_status chgpu_set_join(chgpu_ctx* ctx, int enabled, uint32_t min_points_per_bucket) {
    CtxLock lock_(ctx);
    if (!ctx) return CHGPU_EINVAL;
    ctx->join_enabled = enabled != 0;
    ctx->join_min_bucket = min_points_per_bucket;
    return CHGPU_OK;
}

chgpu_status chgpu_set_sub_batch_queries(chgpu_ctx* ctx, uint64_t max_queries) {
    CtxLock lock_(ctx);
    if (!ctx) return CHGPU_EINVAL;
    ctx->sub_batch_queries = max_queries ? max_queries : kSubBatchQueries;
    return CHGPU_OK;
}

chgpu_status chgpu_host_alloc(chgpu_ctx* ctx, size_t bytes, void** out) {
    CtxLock lock_(ctx);
    if (!ctx || !out) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    CK(cudaMallocHost(out, std::max<size_t>(bytes, 1)));
    return CHGPU_OK;
}

chgpu_status chgpu_host_free(chgpu_ctx* ctx, void* p) {
    CtxLock lock_(ctx);
    if (!ctx) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    CK(cudaFreeHost(p));
    return CHGPU_OK;
}

// ---- family -------------------------------------------------------------------------------------
chgpu_status chgpu_set_family(chgpu_ctx* ctx, const chgpu_family_params* p, const double* short_planes,
                              const double* long_planes) {
    CtxLock lock_(ctx);
    if (!ctx || !p || !short_planes || !long_planes) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    if (chgpu_host_check_family(p) != 0)
        return fail(ctx, CHGPU_EINVAL, "family parameters violate 1<=m<=32, m<n<=128, L>=1 (hashing.cpp:30-36)");
    if (p->table_count > uint32_t(kMaxTables))
        return fail(ctx, CHGPU_EUNSUPPORTED, "device envelope is L <= %d (got L=%u)", kMaxTables, p->table_count);
    if (!ctx->slot_of.empty())
        return fail(ctx, CHGPU_ELOGIC, "evict all images before installing a different family");
    CK(cudaStreamSynchronize(ctx->compute));
    const size_t ns = size_t(p->table_count) * p->short_bits, nl = p->long_bits;
    if (ctx->d_planes) cudaFree(ctx->d_planes);
    ctx->d_planes = nullptr;
    CK(cudaMalloc(&ctx->d_planes, (ns + nl) * kDim * sizeof(double)));
    CK(cudaMemcpy(ctx->d_planes, short_planes, ns * kDim * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_planes + ns * kDim, long_planes, nl * kDim * sizeof(double), cudaMemcpyHostToDevice));
    ctx->fam = *p;
    ctx->has_family = true;
    ctx->sparse = p->short_bits > uint32_t(kMaxShortBits);
    ctx->h_planes.assign(short_planes, short_planes + ns * kDim);
    ctx->h_planes.insert(ctx->h_planes.end(), long_planes, long_planes + nl * kDim);
    return refresh_hash_filter(ctx);
}

chgpu_status chgpu_set_hash_mode(chgpu_ctx* ctx, chgpu_hash_mode mode) {
    CtxLock lock_(ctx);
    if (!ctx || (mode != CHGPU_HASH_FILTERED && mode != CHGPU_HASH_EXACT && mode != CHGPU_HASH_TENSOR)) return CHGPU_EINVAL;
    ctx->hash_mode = mode;
    return CHGPU_OK;
}

chgpu_status chgpu_get_hash_stats(chgpu_ctx* ctx, chgpu_hash_stats* out) {
    CtxLock lock_(ctx);
    if (!ctx || !out) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    HashFilterStats hs;
    CK(cudaMemcpyAsync(&hs, ctx->d_hstats, sizeof(hs), cudaMemcpyDeviceToHost, ctx->compute));
    CK(cudaStreamSynchronize(ctx->compute));
    out->undecided_dots = hs.undecided;
    out->flipped_bits = hs.flipped;
    out->overflowed_batches = hs.overflows;
    out->filter_active = (ctx->hash_mode != CHGPU_HASH_EXACT && ctx->filter_ready) ? 1 : 0;
    return CHGPU_OK;
}

chgpu_status chgpu_centering_reset(chgpu_ctx* ctx) {
    CtxLock lock_(ctx);
    if (!ctx) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    CK(cudaMemsetAsync(ctx->d_sums, 0, 128 * sizeof(unsigned long long), ctx->compute));
    ctx->sum_count = 0;
    memset(ctx->extra_sums, 0, sizeof(ctx->extra_sums));
    return CHGPU_OK;
}

chgpu_status chgpu_centering_add_image(chgpu_ctx* ctx, uint32_t image_id) {
    CtxLock lock_(ctx);
    if (!ctx) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    uint32_t slot = 0;
    if (const chgpu_status s = find_slot(ctx, image_id, &slot)) return s;
    const DevImage& d = ctx->images[slot].dev;
    if (d.n == 0) return CHGPU_OK;
    if (const chgpu_status s = order_compute_after_copy(ctx)) return s;
    const uint32_t blocks = std::max(1u, std::min((d.n + 255u) / 256u, 4u * uint32_t(ctx->prop.multiProcessorCount)));
    centering_sums_kernel<<<blocks, 256, 0, ctx->compute>>>(d.desc, d.n, ctx->d_sums);
    CK(cudaGetLastError());
    ctx->sum_count += d.n;
    return CHGPU_OK;
}

chgpu_status chgpu_centering_add_images(chgpu_ctx* ctx, const uint32_t* image_ids, uint32_t count) {
    CtxLock lock_(ctx);
    if (!ctx || (count && !image_ids)) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    if (count == 0) return CHGPU_OK;
    std::vector<uint32_t> slots(count);
    uint64_t points = 0;
    uint32_t max_n = 0;
    for (uint32_t i = 0; i < count; ++i) {
        if (const chgpu_status s = find_slot(ctx, image_ids[i], &slots[i])) return s;
        points += ctx->images[slots[i]].dev.n;
        max_n = std::max(max_n, ctx->images[slots[i]].dev.n);
    }
    if (max_n == 0) return CHGPU_OK;
    if (const chgpu_status s = ensure_slots_scratch(ctx, count)) return s;
    if (const chgpu_status s = order_compute_after_copy(ctx)) return s;
    CK(cudaStreamSynchronize(ctx->compute));  // d_slots is reused by successive calls
    CK(cudaMemcpyAsync(ctx->d_slots, slots.data(), count * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->compute));
    for (uint32_t first = 0; first < count; first += 65535u) {
        const uint32_t cnt = std::min(65535u, count - first);
        const dim3 grid(std::max(1u, std::min((max_n + 1023u) / 1024u, 16u)), cnt);
        centering_sums_batch_kernel<<<grid, 256, 0, ctx->compute>>>(ctx->d_images, ctx->d_slots + first, ctx->d_sums);
        CK(cudaGetLastError());
    }
    ctx->sum_count += points;
    return CHGPU_OK;
}

chgpu_status chgpu_centering_get_sums(chgpu_ctx* ctx, uint64_t* sums128, uint64_t* count) {
    CtxLock lock_(ctx);
    if (!ctx || !sums128 || !count) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    unsigned long long tmp[128];
    CK(cudaMemcpyAsync(tmp, ctx->d_sums, sizeof(tmp), cudaMemcpyDeviceToHost, ctx->compute));
    CK(cudaStreamSynchronize(ctx->compute));
    for (int i = 0; i < 128; ++i) sums128[i] = tmp[i] + ctx->extra_sums[i];
    *count = ctx->sum_count;
    return CHGPU_OK;
}

chgpu_status chgpu_centering_add_sums(chgpu_ctx* ctx, const uint64_t* sums128, uint64_t count) {
    CtxLock lock_(ctx);
    if (!ctx || !sums128) return CHGPU_EINVAL;
    for (int i = 0; i < 128; ++i) ctx->extra_sums[i] += sums128[i];
    ctx->sum_count += count;
    return CHGPU_OK;
}

chgpu_status chgpu_set_centering(chgpu_ctx* ctx, const double* centering128) {
    CtxLock lock_(ctx);
    if (!ctx || !centering128) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    CK(cudaStreamSynchronize(ctx->compute));
    CK(cudaMemcpy(ctx->d_centering, centering128, 128 * sizeof(double), cudaMemcpyHostToDevice));
    // The reference's HashFamily does not change once centered (hashing.cpp:59-64) and its code caches carry the
    // centering fingerprint for that reason: codes hashed here under another vector must not meet codes hashed under
    // this one.  They stay resident but run_match refuses them until they are hashed again.
    if (ctx->has_centering && memcmp(ctx->h_centering, centering128, sizeof(ctx->h_centering)) != 0) ++ctx->centering_gen;
    memcpy(ctx->h_centering, centering128, sizeof(ctx->h_centering));
    ctx->has_centering = true;
    return refresh_hash_filter(ctx);
}

chgpu_status chgpu_centering_apply(chgpu_ctx* ctx, double* centering128_out) {
    CtxLock lock_(ctx);
    if (!ctx) return CHGPU_EINVAL;
    uint64_t sums[128], count = 0;
    if (const chgpu_status s = chgpu_centering_get_sums(ctx, sums, &count)) return s;
    if (count == 0) return fail(ctx, CHGPU_EINVAL, "set_centering: no descriptors");  // hashing.cpp:60
    double c[128];
    for (int i = 0; i < 128; ++i) c[i] = static_cast<double>(sums[i]) / static_cast<double>(count);  // hashing.cpp:61-62
    if (centering128_out) memcpy(centering128_out, c, sizeof(c));
    return chgpu_set_centering(ctx, c);
}

// ---- descriptor load ----------------------------------------------------------------------------
chgpu_status chgpu_upload_image(chgpu_ctx* ctx, uint32_t image_id, uint32_t n, const uint8_t* desc,
                                const float* keypoints) {
    CtxLock lock_(ctx);
    if (!ctx || (n && !desc)) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    uint32_t slot = 0;
    if (const chgpu_status s = alloc_image(ctx, image_id, n, &slot)) return s;
    if (const chgpu_status s = order_copy_after_compute(ctx)) return s;
    ImageRec& r = ctx->images[slot];
    if (const chgpu_status s = h2d(ctx, const_cast<uint8_t*>(r.dev.desc), desc, size_t(n) * kDim)) return s;
    if (keypoints) {
        if (const chgpu_status s = h2d(ctx, const_cast<float4*>(r.dev.kp), keypoints, size_t(n) * 16)) return s;
    } else if (n) {
        CK(cudaMemsetAsync(const_cast<float4*>(r.dev.kp), 0, size_t(n) * 16, ctx->copy));
    }
    return publish_slot(ctx, slot);
}

chgpu_status chgpu_upload_images(chgpu_ctx* ctx, const uint32_t* image_ids, uint32_t count, uint32_t n,
                                 const uint8_t* desc, const float* keypoints) {
    CtxLock lock_(ctx);
    if (!ctx || (count && !image_ids) || (count && n && !desc)) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    if (count == 0) return CHGPU_OK;
    if (const chgpu_status s = order_copy_after_compute(ctx)) return s;
    // pinned sources: back-to-back async copies, one drain at the end; pageable ones go through the staging ring
    const bool pinned = n == 0 || (is_pinned(desc) && (!keypoints || is_pinned(keypoints)));
    uint32_t lo = UINT32_MAX, hi = 0;
    for (uint32_t i = 0; i < count; ++i) {
        uint32_t slot = 0;
        if (const chgpu_status s = alloc_image(ctx, image_ids[i], n, &slot)) return s;
        ImageRec& r = ctx->images[slot];
        const uint8_t* d = desc + size_t(i) * n * kDim;
        const float* k = keypoints ? keypoints + size_t(i) * n * 4 : nullptr;
        if (n) {
            if (pinned) {
                CK(cudaMemcpyAsync(const_cast<uint8_t*>(r.dev.desc), d, size_t(n) * kDim, cudaMemcpyHostToDevice, ctx->copy));
                if (k) CK(cudaMemcpyAsync(const_cast<float4*>(r.dev.kp), k, size_t(n) * 16, cudaMemcpyHostToDevice, ctx->copy));
            } else {
                if (const chgpu_status s = h2d(ctx, const_cast<uint8_t*>(r.dev.desc), d, size_t(n) * kDim)) return s;
                if (k) if (const chgpu_status s = h2d(ctx, const_cast<float4*>(r.dev.kp), k, size_t(n) * 16)) return s;
            }
            if (!k) CK(cudaMemsetAsync(const_cast<float4*>(r.dev.kp), 0, size_t(n) * 16, ctx->copy));
        }
        ctx->h_images[slot] = r.dev;
        lo = std::min(lo, slot);
        hi = std::max(hi, slot);
    }
    CK(cudaMemcpyAsync(ctx->d_images + lo, ctx->h_images + lo, size_t(hi - lo + 1) * sizeof(DevImage), cudaMemcpyHostToDevice,
                       ctx->copy));
    CK(cudaStreamSynchronize(ctx->copy));  // the caller may reuse its buffers
    return CHGPU_OK;
}

chgpu_status chgpu_upload_chft(chgpu_ctx* ctx, uint32_t image_id, const void* blob, size_t nbytes,
                               uint32_t* count_out, chgpu_file_fault* fault, uint64_t* fault_offset) {
    CtxLock lock_(ctx);
    if (!ctx || !blob) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    auto bad = [&](chgpu_file_fault f, uint64_t off, const char* what) {
        if (fault) *fault = f;
        if (fault_offset) *fault_offset = off;
        return fail(ctx, CHGPU_EFORMAT, "image %u: %s at byte %llu", image_id, what, (unsigned long long)off);
    };
    if (fault) *fault = CHGPU_FAULT_NONE;
    // header checks in the order of parse_features_blob (engine.cpp:458-472)
    const unsigned char* b = static_cast<const unsigned char*>(blob);
    if (nbytes < 16) return bad(CHGPU_FAULT_TRUNCATED, nbytes, "truncated payload (header)");
    if (memcmp(b, "CHFT", 4) != 0) return bad(CHGPU_FAULT_BAD_MAGIC, 0, "bad magic");
    uint32_t version, count;
    memcpy(&version, b + 4, 4);
    memcpy(&count, b + 8, 4);
    if (version != 1) return bad(CHGPU_FAULT_BAD_VERSION, 4, "unsupported version");
    const size_t expected = 16 + size_t(count) * 144;
    if (nbytes < expected) return bad(CHGPU_FAULT_TRUNCATED, nbytes, "truncated payload");
    if (count_out) *count_out = count;

    uint32_t slot = 0;
    if (const chgpu_status s = alloc_image(ctx, image_id, count, &slot)) return s;
    ImageRec& r = ctx->images[slot];
    if (count) {
        // raw AoS records travel once over PCIe into a scratch block, the device splits them
        char* raw = nullptr;
        const size_t raw_bytes = size_t(count) * 144;
        if (ctx->arena.alloc(raw_bytes, &raw) != cudaSuccess) {
            cudaGetLastError();
            return fail(ctx, CHGPU_ENOMEM, "staging block of %zu bytes", raw_bytes);
        }
        if (const chgpu_status s = order_copy_after_compute(ctx)) return s;
        if (const chgpu_status s = h2d(ctx, raw, b + 16, raw_bytes)) return s;
        if (const chgpu_status s = order_compute_after_copy(ctx)) return s;
        const uint32_t blocks = std::min<uint64_t>((uint64_t(count) * 9 + 255) / 256, 8u * ctx->prop.multiProcessorCount);
        chft_split_kernel<<<blocks, 256, 0, ctx->compute>>>(reinterpret_cast<const uint4*>(raw), count,
                                                           reinterpret_cast<uint4*>(const_cast<uint8_t*>(r.dev.desc)),
                                                           reinterpret_cast<uint4*>(const_cast<float4*>(r.dev.kp)));
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(ctx->compute));
        ctx->arena.release(raw, raw_bytes);
    }
    return publish_slot(ctx, slot);
}

// ---- streaming loader: disk -> pinned ring -> HBM ---------------------------------------------------
extern "C++" {
namespace {

// Every slot has its own lock and condition variables: the issue thread wakes exactly the reader that waits for
// the slot it frees, and a reader wakes only the issue thread (one shared condition variable made every hand-off
// wake all readers, which capped the loader far below the copy engine's rate).
struct LoadSlot {
    std::mutex mu;
    std::condition_variable cv_free;   // a reader waits here for its turn
    std::condition_variable cv_ready;  // the issue thread waits here for the file
    enum State { Free, Filling, Ready } state = Free;
    char* buf = nullptr;   // pinned: a share of the context's region, or its own buffer (own) after outgrowing it
    size_t cap = 0;
    bool own = false;
    size_t bytes = 0;      // bytes read
    bool missing = false;  // fopen failed
    uint32_t file = 0;     // index of the file it holds (valid in Ready)
    uint32_t turn = 0;     // index of the file allowed to fill it next
    cudaEvent_t copied = nullptr;  // H2D of this slot's contents complete
    bool in_flight = false;        // `copied` recorded, not yet observed
};

struct LoadRing {
    std::mutex mu;  // statistics only
    std::unique_ptr<LoadSlot[]> slots;
    size_t nslots = 0;
    std::atomic<uint32_t> next{0};
    std::atomic<bool> abort{false};
    double read_seconds = 0.0;
    uint64_t bytes_read = 0;
};

// Reader thread: claims file indices in order; file i travels through slot i % S once the slot's previous
// tenant (file i - S) has been copied to the device.
void loader_thread(LoadRing* ring, const char* const* paths, uint32_t count) {
    const size_t S = ring->nslots;
    double seconds = 0.0;
    uint64_t bytes = 0;
    for (;;) {
        const uint32_t i = ring->next.fetch_add(1);
        if (i >= count || ring->abort.load()) break;
        LoadSlot& s = ring->slots[i % S];
        {
            std::unique_lock<std::mutex> lock(s.mu);
            // slots are handed out in file order: wait until it is free AND it is this file's turn
            s.cv_free.wait(lock, [&] { return ring->abort.load() || (s.state == LoadSlot::Free && s.turn == i); });
            if (ring->abort.load()) break;
            s.state = LoadSlot::Filling;
        }
        const auto t0 = std::chrono::steady_clock::now();
        s.bytes = 0;
        s.missing = false;
        FILE* f = std::fopen(paths[i], "rb");
        if (!f) {
            s.missing = true;
        } else {
            std::fseek(f, 0, SEEK_END);
            const long sz = std::ftell(f);
            std::fseek(f, 0, SEEK_SET);
            const size_t need = sz > 0 ? size_t(sz) : 0;
            if (need > s.cap) {  // a file larger than the slots were sized for: private pinned buffer for this slot
                if (s.own) cudaFreeHost(s.buf);
                s.buf = nullptr;
                s.cap = 0;
                s.own = false;
                const size_t cap = std::max<size_t>(need + need / 8, size_t(2) << 20);
                if (cudaMallocHost(reinterpret_cast<void**>(&s.buf), cap) == cudaSuccess) {
                    s.cap = cap;
                    s.own = true;
                } else {
                    cudaGetLastError();
                }
            }
            if (need <= s.cap && need) s.bytes = std::fread(s.buf, 1, need, f);
            std::fclose(f);
        }
        seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        bytes += s.bytes;
        {
            std::lock_guard<std::mutex> lock(s.mu);
            s.file = i;
            s.state = LoadSlot::Ready;
        }
        s.cv_ready.notify_one();
    }
    std::lock_guard<std::mutex> lock(ring->mu);
    ring->read_seconds += seconds;
    ring->bytes_read += bytes;
}

}  // namespace

// One streaming load in progress.  The issue side is a state machine the owning thread pumps: load_pump(block = true)
// is the classic loop (wait for the next file, send it); load_pump(block = false) sends whatever the readers have
// finished and returns — chgpu_match_pairs* calls it between sub-batches while a background job is open, so the
// H2D copies of the next block run under the match kernels of the current task (the paper's exchange).
struct chgpu_load_job {
    chgpu_ctx* ctx = nullptr;
    std::vector<std::string> path_store;
    std::vector<const char*> paths;
    std::vector<uint32_t> image_ids;
    std::vector<chgpu_file_result> results;
    uint32_t count = 0, io_threads = 0;
    bool sums = false;
    LoadRing ring;
    size_t S = 0;
    struct Scratch {
        char* ptr = nullptr;
        size_t cap = 0;
        cudaEvent_t split_done = nullptr;
        bool used = false;
        bool own = true;  // its own cudaMalloc (kept by the context between calls); false: a slice of the staging region
        bool outgrown = false;  // region mode: a private buffer for a file larger than a slice, freed with the job
        // region mode: the split kernel of the file it holds is launched later (load_flush_splits)
        bool split_pending = false;
        uint32_t n = 0;
        uint8_t* dst_desc = nullptr;
        float4* dst_kp = nullptr;
    };
    std::vector<Scratch> scratch;  // device-side raw (AoS) ring
    bool region_mode = false;
    cudaEvent_t last_copied = nullptr;  // region mode: event of the latest H2D copy
    cudaEvent_t ev_flush = nullptr;     // region mode: recorded behind the latest batched split
    std::vector<std::thread> readers;
    std::deque<uint32_t> in_flight;  // files whose H2D was issued, oldest first (copies complete in this order)
    uint32_t next = 0;               // next file the issue side handles
    uint32_t pub_lo = UINT32_MAX, pub_hi = 0;  // image-table range to publish when the batch is in
    chgpu_load_stats st{};
    chgpu_status rc = CHGPU_OK;
    std::chrono::steady_clock::time_point wall0;
    double t_wait = 0, t_alloc = 0, t_issue = 0;
};

namespace {

void load_poll_copies(chgpu_load_job* job) {  // slots whose H2D completed go back to the readers
    LoadRing& ring = job->ring;
    const size_t S = job->S;
    size_t done = 0;
    while (done < job->in_flight.size() && cudaEventQuery(ring.slots[job->in_flight[done] % S].copied) == cudaSuccess) ++done;
    for (size_t k = 0; k < done; ++k) {
        LoadSlot& s = ring.slots[job->in_flight[k] % S];
        {
            std::lock_guard<std::mutex> lock(s.mu);
            s.in_flight = false;
            s.state = LoadSlot::Free;
            s.turn = s.file + uint32_t(S);
        }
        s.cv_free.notify_one();
    }
    job->in_flight.erase(job->in_flight.begin(), job->in_flight.begin() + done);
}

// ring_slots pinned slots (>= 8, >= 2 per reader), scratch_slots device staging buffers.
chgpu_status load_start(chgpu_ctx* ctx, const char* const* paths, const uint32_t* image_ids, uint32_t count, uint32_t io_threads,
                        bool sums, size_t ring_slots, size_t scratch_slots, chgpu_load_job** out) {
    std::unique_ptr<chgpu_load_job> job(new chgpu_load_job);
    job->ctx = ctx;
    job->count = count;
    job->sums = sums;
    job->path_store.reserve(count);
    for (uint32_t i = 0; i < count; ++i) job->path_store.emplace_back(paths[i] ? paths[i] : "");
    for (uint32_t i = 0; i < count; ++i) job->paths.push_back(job->path_store[i].c_str());
    job->image_ids.assign(image_ids, image_ids + count);
    {
        chgpu_file_result not_reached{};
        not_reached.status = CHGPU_ECUDA;  // a batch that device trouble ends early leaves the rest unloaded, not "ok"
        job->results.assign(count, not_reached);
    }
    io_threads = std::max<uint32_t>(1, std::min<uint32_t>(io_threads ? io_threads : 4, 64));
    job->io_threads = io_threads;
    const size_t S = std::max<size_t>(std::max<size_t>(8, 2 * size_t(io_threads)), ring_slots);
    job->S = S;
    // Pinned ring buffers and device staging live in the context: cudaMallocHost / cudaMalloc cost milliseconds
    // and take the driver lock, so they are sized up front (first file + 12 %) on this thread and only a later,
    // larger file makes a reader grow its slot.
    size_t guess = size_t(2) << 20;
    if (FILE* f0 = std::fopen(job->paths[0], "rb")) {
        std::fseek(f0, 0, SEEK_END);
        const long sz = std::ftell(f0);
        std::fclose(f0);
        if (sz > 0) guess = std::max(guess, size_t(sz) + size_t(sz) / 8);
    }
    guess = align_up(guess, 4096);
    if (ctx->load_pinned_slots < S || ctx->load_pinned_slot < guess) {
        cudaFreeHost(ctx->load_pinned);
        ctx->load_pinned = nullptr;
        ctx->load_pinned_slots = ctx->load_pinned_slot = 0;
        if (cudaMallocHost(reinterpret_cast<void**>(&ctx->load_pinned), S * guess) != cudaSuccess) {
            cudaGetLastError();
            return fail(ctx, CHGPU_ENOMEM, "loader: %zu bytes of pinned staging", S * guess);
        }
        ctx->load_pinned_slots = S;
        ctx->load_pinned_slot = guess;
    }
    LoadRing& ring = job->ring;
    ring.slots.reset(new LoadSlot[S]);
    ring.nslots = S;
    for (size_t k = 0; k < S; ++k) {
        ring.slots[k].buf = ctx->load_pinned + k * ctx->load_pinned_slot;
        ring.slots[k].cap = ctx->load_pinned_slot;
        ring.slots[k].turn = uint32_t(k);  // slot k serves files k, k + S, k + 2 S, ...
        if (cudaEventCreateWithFlags(&ring.slots[k].copied, cudaEventDisableTiming) != cudaSuccess)
            return fail(ctx, CHGPU_ECUDA, "loader: event creation failed");
    }
    // device-side raw (AoS) scratch ring: deep enough that waiting for a split kernel never stalls the issue loop
    const size_t nscratch = std::max<size_t>(8, scratch_slots);
    job->scratch.resize(nscratch);
    if (scratch_slots == 0) {
        if (ctx->load_scratch.size() < nscratch) ctx->load_scratch.resize(nscratch, {nullptr, 0});
        for (size_t k = 0; k < nscratch; ++k) {
            job->scratch[k].ptr = ctx->load_scratch[k].first;
            job->scratch[k].cap = ctx->load_scratch[k].second;
        }
    } else {
        // background loads: one region, allocated now while the device is idle (a cudaMalloc issued under a running
        // kernel waits for it) and cut into slices
        if (ctx->load_region_bytes < nscratch * guess) {
            CK(cudaStreamSynchronize(ctx->compute));
            cudaFree(ctx->load_region);
            ctx->load_region = nullptr;
            ctx->load_region_bytes = 0;
            if (cudaMalloc(reinterpret_cast<void**>(&ctx->load_region), nscratch * guess) != cudaSuccess) {
                cudaGetLastError();
                return fail(ctx, CHGPU_ENOMEM, "loader: %zu bytes of device staging", nscratch * guess);
            }
            ctx->load_region_bytes = nscratch * guess;
        }
        job->region_mode = true;
        for (size_t k = 0; k < nscratch; ++k) {
            job->scratch[k].ptr = ctx->load_region + k * guess;
            job->scratch[k].cap = guess;
            job->scratch[k].own = false;
        }
    }
    // (region mode: one event behind each batched split covers every buffer it consumed)
    if (job->region_mode) cudaEventCreateWithFlags(&job->ev_flush, cudaEventDisableTiming);
    else
        for (size_t k = 0; k < nscratch; ++k) cudaEventCreateWithFlags(&job->scratch[k].split_done, cudaEventDisableTiming);
    job->wall0 = std::chrono::steady_clock::now();
    for (uint32_t t = 0; t < io_threads; ++t) job->readers.emplace_back(loader_thread, &job->ring, job->paths.data(), count);
    *out = job.release();
    return CHGPU_OK;
}

// AoS -> SoA split of the file a staging buffer holds (with the centering sums folded in when the job collects them).
void load_launch_split(chgpu_load_job* job, chgpu_load_job::Scratch& sc) {
    chgpu_ctx* ctx = job->ctx;
    const uint32_t n = sc.n;
    if (job->sums) {
        const uint32_t blocks = std::max(1u, std::min((n + 127u) / 128u, 2u * uint32_t(ctx->prop.multiProcessorCount)));
        chft_split_sums_kernel<<<blocks, kSplitSumThreads, 0, ctx->compute>>>(reinterpret_cast<const uint4*>(sc.ptr), n,
                                                                             reinterpret_cast<uint4*>(sc.dst_desc),
                                                                             reinterpret_cast<uint4*>(sc.dst_kp), ctx->d_sums);
    } else {
        const uint32_t blocks = uint32_t(std::min<uint64_t>((uint64_t(n) * 9 + 255) / 256, 8u * ctx->prop.multiProcessorCount));
        chft_split_kernel<<<blocks, 256, 0, ctx->compute>>>(reinterpret_cast<const uint4*>(sc.ptr), n,
                                                           reinterpret_cast<uint4*>(sc.dst_desc), reinterpret_cast<uint4*>(sc.dst_kp));
    }
    cudaEventRecord(job->region_mode ? job->ev_flush : sc.split_done, ctx->compute);
    sc.used = true;
    sc.split_pending = false;
}

// Region mode: launches the split kernels held back so far (behind the copies issued so far).
void load_flush_splits(chgpu_load_job* job) {
    bool any = false;
    for (auto& sc : job->scratch) any = any || sc.split_pending;
    if (!any) return;
    chgpu_ctx* ctx = job->ctx;
    if (job->last_copied) cudaStreamWaitEvent(ctx->compute, job->last_copied, 0);  // copies complete in issue order
    if (job->sums) {  // (the fused split + sums kernel stays one launch per file)
        for (auto& sc : job->scratch)
            if (sc.split_pending) load_launch_split(job, sc);
        return;
    }
    // one launch for all of them: the job list travels through a pinned array kept by the context
    size_t np = 0;
    for (auto& sc : job->scratch) np += sc.split_pending ? 1 : 0;
    if (ctx->split_jobs_cap < np) {
        cudaStreamSynchronize(ctx->compute);
        cudaFreeHost(ctx->h_split_jobs);
        cudaFree(ctx->d_split_jobs);
        ctx->h_split_jobs = nullptr;
        ctx->d_split_jobs = nullptr;
        ctx->split_jobs_cap = 0;
        const size_t cap = std::max<size_t>(np, 1024);
        if (cudaMallocHost(reinterpret_cast<void**>(&ctx->h_split_jobs), cap * sizeof(SplitJob)) != cudaSuccess ||
            cudaMalloc(reinterpret_cast<void**>(&ctx->d_split_jobs), cap * sizeof(SplitJob)) != cudaSuccess) {
            cudaGetLastError();
            for (auto& sc : job->scratch)  // no room for the list: one launch per file
                if (sc.split_pending) load_launch_split(job, sc);
            return;
        }
        ctx->split_jobs_cap = cap;
    } else if (ctx->split_jobs_busy) {
        cudaEventSynchronize(ctx->ev_split_jobs);  // the previous list has been read
    }
    uint32_t max_n = 0;
    size_t k = 0;
    for (auto& sc : job->scratch)
        if (sc.split_pending) {
            ctx->h_split_jobs[k++] = SplitJob{reinterpret_cast<const uint4*>(sc.ptr), reinterpret_cast<uint4*>(sc.dst_desc),
                                              reinterpret_cast<uint4*>(sc.dst_kp), sc.n, 0u};
            max_n = std::max(max_n, sc.n);
        }
    cudaMemcpyAsync(ctx->d_split_jobs, ctx->h_split_jobs, np * sizeof(SplitJob), cudaMemcpyHostToDevice, ctx->compute);
    cudaEventRecord(ctx->ev_split_jobs, ctx->compute);
    ctx->split_jobs_busy = true;
    const uint32_t bx = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>((uint64_t(max_n) * 9 + 255) / 256, 32)));
    for (size_t first = 0; first < np; first += 65535) {  // gridDim.y limit
        const uint32_t cnt = uint32_t(std::min<size_t>(65535, np - first));
        chft_split_batch_kernel<<<dim3(bx, cnt), 256, 0, ctx->compute>>>(ctx->d_split_jobs + first);
    }
    cudaEventRecord(job->ev_flush, ctx->compute);
    for (auto& sc : job->scratch)
        if (sc.split_pending) {
            sc.used = true;
            sc.split_pending = false;
        }
}

// Sends files to the device in list order.  block: until every file has been handled; otherwise until the next file
// is not in its pinned slot yet or its device staging buffer is still waiting for an earlier split kernel.
void load_pump(chgpu_load_job* job, bool block) {
    chgpu_ctx* ctx = job->ctx;
    LoadRing& ring = job->ring;
    const size_t S = job->S, nscratch = job->scratch.size();
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto secs = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
        return std::chrono::duration<double>(b - a).count();
    };
    chgpu_load_stats& st = job->st;
    while (job->next < job->count && job->rc == CHGPU_OK) {
        const uint32_t i = job->next;
        LoadSlot& s = ring.slots[i % S];
        chgpu_load_job::Scratch& sc = job->scratch[i % nscratch];
        const auto tw0 = now();
        {
            std::unique_lock<std::mutex> lock(s.mu);
            while (!(s.state == LoadSlot::Ready && s.file == i)) {
                lock.unlock();
                load_poll_copies(job);
                if (!block) return;
                lock.lock();
                if (s.state == LoadSlot::Ready && s.file == i) break;
                s.cv_ready.wait_for(lock, std::chrono::microseconds(50));
            }
        }
        if (sc.used) {  // its previous split kernel has to have consumed it
            if (sc.split_pending) load_flush_splits(job);  // (a job with more files than staging buffers)
            cudaEvent_t consumed = job->region_mode ? job->ev_flush : sc.split_done;
            if (block) cudaEventSynchronize(consumed);
            else if (cudaEventQuery(consumed) != cudaSuccess) {
                cudaGetLastError();
                return;
            }
        }
        job->next = i + 1;
        const auto tw1 = now();
        job->t_wait += secs(tw0, tw1);
        chgpu_file_result& r = job->results[i];
        r = chgpu_file_result{};
        auto release_slot = [&]() {
            {
                std::lock_guard<std::mutex> lock(s.mu);
                s.state = LoadSlot::Free;
                s.turn = i + uint32_t(S);
            }
            s.cv_free.notify_one();
        };
        auto bad = [&](chgpu_file_fault f, uint64_t off) {
            r.status = CHGPU_EFORMAT;
            r.fault = f;
            r.fault_offset = off;
            ++st.files_failed;
            release_slot();
        };
        // header checks in the order of load_features (feature_io.cpp:65-85)
        const unsigned char* b = reinterpret_cast<const unsigned char*>(s.buf);
        if (s.missing) { bad(CHGPU_FAULT_MISSING_FILE, 0); continue; }
        if (s.bytes < 16) { bad(CHGPU_FAULT_TRUNCATED, s.bytes); continue; }
        if (memcmp(b, "CHFT", 4) != 0) { bad(CHGPU_FAULT_BAD_MAGIC, 0); continue; }
        uint32_t version, n;
        memcpy(&version, b + 4, 4);
        memcpy(&n, b + 8, 4);
        if (version != 1) { bad(CHGPU_FAULT_BAD_VERSION, 4); continue; }
        const size_t raw_bytes = size_t(n) * 144;
        if (s.bytes < 16 + raw_bytes) { bad(CHGPU_FAULT_TRUNCATED, s.bytes); continue; }

        uint32_t slot_img;
        if (const chgpu_status e = alloc_image(ctx, job->image_ids[i], n, &slot_img)) {
            r.status = e;
            ++st.files_failed;
            release_slot();
            if (e == CHGPU_ENOMEM || e == CHGPU_ECUDA) job->rc = e;  // device trouble ends the batch; bad input does not
            continue;
        }
        ImageRec& img = ctx->images[slot_img];
        const auto tw2 = now();
        job->t_alloc += secs(tw1, tw2);
        if (n) {
            if (sc.cap < raw_bytes) {
                if (sc.ptr && sc.own) cudaFree(sc.ptr);
                sc.ptr = nullptr;
                sc.cap = 0;
                const size_t cap = std::max<size_t>(raw_bytes + raw_bytes / 8, size_t(2) << 20);
                if (cudaMalloc(reinterpret_cast<void**>(&sc.ptr), cap) != cudaSuccess) {
                    cudaGetLastError();
                    job->rc = fail(ctx, CHGPU_ENOMEM, "loader: device staging of %zu bytes", cap);
                    release_slot();
                    break;
                }
                sc.cap = cap;
                sc.own = true;
                sc.outgrown = !job->region_mode ? false : true;
            }
            cudaStream_t h2d_stream = job->region_mode ? ctx->load : ctx->copy;
            cudaMemcpyAsync(sc.ptr, s.buf + 16, raw_bytes, cudaMemcpyHostToDevice, h2d_stream);
            cudaEventRecord(s.copied, h2d_stream);
            s.in_flight = true;
            job->in_flight.push_back(i);
            sc.n = n;
            sc.dst_desc = const_cast<uint8_t*>(img.dev.desc);
            sc.dst_kp = const_cast<float4*>(img.dev.kp);
            if (job->sums) ctx->sum_count += n;
            if (job->region_mode) {
                // A background load sends the bytes now and splits them later, in one go: hundreds of tiny launches
                // queued behind a running match kernel would fill the launch queue and stall this thread.
                sc.split_pending = true;
                sc.used = true;
                job->last_copied = s.copied;
            } else {
                cudaStreamWaitEvent(ctx->compute, s.copied, 0);
                load_launch_split(job, sc);
            }
        } else {
            release_slot();
        }
        // the kernels above take pointers, not table entries: the table is published once, behind the loop
        ctx->h_images[slot_img] = ctx->images[slot_img].dev;
        job->pub_lo = std::min(job->pub_lo, slot_img);
        job->pub_hi = std::max(job->pub_hi, slot_img);
        r.status = CHGPU_OK;
        r.count = n;
        ++st.files_ok;
        st.points += n;
        load_poll_copies(job);
        job->t_issue += secs(tw2, now());
    }
}

// Handles what is left, publishes the image table, drains, joins the readers and frees the job.
chgpu_status load_finish(chgpu_load_job* job, chgpu_file_result* results, chgpu_load_stats* stats) {
    chgpu_ctx* ctx = job->ctx;
    LoadRing& ring = job->ring;
    const size_t S = job->S;
    const uint32_t left = job->count - job->next;
    const auto tf0 = std::chrono::steady_clock::now();
    load_pump(job, true);
    load_flush_splits(job);
    if (getenv("CHGPU_LOADER_TRACE") != nullptr)
        fprintf(stderr, "chgpu loader: %u files (%u left for the final pump, %.3f s), issue thread waited %.3f s for readers, "
                "%.3f s in alloc_image, %.3f s issuing, %.3f s since start\n",
                job->count, left, std::chrono::duration<double>(std::chrono::steady_clock::now() - tf0).count(), job->t_wait,
                job->t_alloc, job->t_issue, std::chrono::duration<double>(std::chrono::steady_clock::now() - job->wall0).count());
    if (job->rc != CHGPU_OK) ring.abort.store(true);
    if (job->pub_lo <= job->pub_hi)
        cudaMemcpyAsync(ctx->d_images + job->pub_lo, ctx->h_images + job->pub_lo,
                        size_t(job->pub_hi - job->pub_lo + 1) * sizeof(DevImage), cudaMemcpyHostToDevice, ctx->copy);
    cudaStreamSynchronize(ctx->load);
    cudaStreamSynchronize(ctx->copy);
    cudaStreamSynchronize(ctx->compute);
    load_poll_copies(job);
    ring.abort.store(true);
    for (size_t k = 0; k < S; ++k) {
        { std::lock_guard<std::mutex> lock(ring.slots[k].mu); }
        ring.slots[k].cv_free.notify_all();
    }
    for (std::thread& t : job->readers) t.join();
    const cudaError_t last = cudaGetLastError();
    for (size_t k = 0; k < S; ++k) {
        if (ring.slots[k].own) cudaFreeHost(ring.slots[k].buf);  // a reader outgrew its share of the region
        cudaEventDestroy(ring.slots[k].copied);
    }
    for (size_t k = 0; k < job->scratch.size(); ++k) {
        if (!job->region_mode) ctx->load_scratch[k] = {job->scratch[k].ptr, job->scratch[k].cap};
        else if (job->scratch[k].outgrown) cudaFree(job->scratch[k].ptr);
        if (job->scratch[k].split_done) cudaEventDestroy(job->scratch[k].split_done);
    }
    if (job->ev_flush) cudaEventDestroy(job->ev_flush);
    chgpu_load_stats st = job->st;
    st.bytes_read = ring.bytes_read;
    st.read_seconds = ring.read_seconds;
    st.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - job->wall0).count();
    if (results) std::copy(job->results.begin(), job->results.end(), results);
    if (stats) *stats = st;
    const chgpu_status rc = job->rc;
    delete job;
    if (rc == CHGPU_OK && last != cudaSuccess) return fail(ctx, CHGPU_ECUDA, "loader: %s", cudaGetErrorString(last));
    return rc;
}

}  // namespace
}  // extern "C++"

chgpu_status chgpu_load_chft_files(chgpu_ctx* ctx, const char* const* paths, const uint32_t* image_ids, uint32_t count,
                                   uint32_t io_threads, int accumulate_centering, chgpu_file_result* results,
                                   chgpu_load_stats* stats) {
    CtxLock lock_(ctx);
    if (!ctx || (count && (!paths || !image_ids || !results))) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    if (!ctx->has_family)
        return fail(ctx, CHGPU_ELOGIC, "chgpu_set_family must precede image uploads (block layout depends on m, L)");
    if (ctx->load_job) return fail(ctx, CHGPU_ELOGIC, "a background load is open (chgpu_load_chft_files_end first)");
    if (count == 0) {
        if (stats) *stats = chgpu_load_stats{};
        return CHGPU_OK;
    }
    chgpu_load_job* job = nullptr;
    if (const chgpu_status s = load_start(ctx, paths, image_ids, count, io_threads, accumulate_centering != 0, 0, 0, &job)) return s;
    return load_finish(job, results, stats);
}

chgpu_status chgpu_load_chft_files_begin(chgpu_ctx* ctx, const char* const* paths, const uint32_t* image_ids, uint32_t count,
                                         uint32_t io_threads, int accumulate_centering) {
    CtxLock lock_(ctx);
    if (!ctx || (count && (!paths || !image_ids))) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    if (!ctx->has_family)
        return fail(ctx, CHGPU_ELOGIC, "chgpu_set_family must precede image uploads (block layout depends on m, L)");
    if (ctx->load_job) return fail(ctx, CHGPU_ELOGIC, "a background load is already open");
    if (count == 0) return CHGPU_OK;
    // The split kernels queue behind the match kernel that is running, so a file's device staging buffer stays busy
    // for up to one launch (~15 ms): the staging ring holds what the copy engine delivers in that time (<= 1,024
    // files, <= 1.5 GiB); the pinned ring frees its slots as the copies complete and needs no more than usual.
    size_t first_bytes = size_t(2) << 20;
    if (FILE* f0 = std::fopen(paths[0], "rb")) {
        std::fseek(f0, 0, SEEK_END);
        const long sz = std::ftell(f0);
        std::fclose(f0);
        if (sz > 0) first_bytes = std::max(first_bytes, size_t(sz));
    }
    const size_t staging = std::max<size_t>(16, std::min<size_t>(std::min<size_t>(count, 1024), (size_t(1536) << 20) / first_bytes));
    return load_start(ctx, paths, image_ids, count, io_threads, accumulate_centering != 0, 64, staging, &ctx->load_job);
}

chgpu_status chgpu_load_chft_files_end(chgpu_ctx* ctx, chgpu_file_result* results, chgpu_load_stats* stats) {
    CtxLock lock_(ctx);
    if (!ctx) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    if (!ctx->load_job) {
        if (stats) *stats = chgpu_load_stats{};
        return CHGPU_OK;
    }
    chgpu_load_job* job = ctx->load_job;
    ctx->load_job = nullptr;
    return load_finish(job, results, stats);
}

chgpu_status chgpu_evict_image(chgpu_ctx* ctx, uint32_t image_id) {
    CtxLock lock_(ctx);
    if (!ctx) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    uint32_t slot = 0;
    if (const chgpu_status s = find_slot(ctx, image_id, &slot)) return s;
    CK(cudaStreamSynchronize(ctx->copy));
    CK(cudaStreamSynchronize(ctx->compute));
    release_slot(ctx, slot);
    ctx->slot_of.erase(image_id);
    dense_set(ctx, image_id, kNone);
    return CHGPU_OK;
}

chgpu_status chgpu_evict_images(chgpu_ctx* ctx, const uint32_t* image_ids, uint32_t count) {
    CtxLock lock_(ctx);
    if (!ctx || (count && !image_ids)) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    if (count == 0) return CHGPU_OK;
    // one drain for the whole list: no kernel or copy still reads the blocks that go back to the arena
    CK(cudaStreamSynchronize(ctx->copy));
    CK(cudaStreamSynchronize(ctx->compute));
    chgpu_status rc = CHGPU_OK;
    for (uint32_t i = 0; i < count; ++i) {
        uint32_t slot = 0;
        if (find_slot(ctx, image_ids[i], &slot) != CHGPU_OK) {
            rc = CHGPU_ENOTFOUND;  // reported after the rest of the list has been released
            continue;
        }
        release_slot(ctx, slot);
        ctx->slot_of.erase(image_ids[i]);
        dense_set(ctx, image_ids[i], kNone);
    }
    return rc;
}

chgpu_status chgpu_image_points(chgpu_ctx* ctx, uint32_t image_id, uint32_t* n) {
    CtxLock lock_(ctx);
    if (!ctx || !n) return CHGPU_EINVAL;
    uint32_t slot = 0;
    if (const chgpu_status s = find_slot(ctx, image_id, &slot)) return s;
    *n = ctx->images[slot].dev.n;
    return CHGPU_OK;
}

chgpu_status chgpu_download_descriptors(chgpu_ctx* ctx, uint32_t image_id, uint8_t* desc, float* keypoints) {
    CtxLock lock_(ctx);
    if (!ctx) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    uint32_t slot = 0;
    if (const chgpu_status s = find_slot(ctx, image_id, &slot)) return s;
    if (const chgpu_status s = chgpu_sync(ctx)) return s;
    const DevImage& d = ctx->images[slot].dev;
    if (desc && d.n) CK(cudaMemcpy(desc, d.desc, size_t(d.n) * kDim, cudaMemcpyDeviceToHost));
    if (keypoints && d.n) CK(cudaMemcpy(keypoints, d.kp, size_t(d.n) * 16, cudaMemcpyDeviceToHost));
    return CHGPU_OK;
}

// ---- hash build ---------------------------------------------------------------------------------
chgpu_status chgpu_hash_images(chgpu_ctx* ctx, const uint32_t* image_ids, uint32_t count, int reduce_rounds) {
    CtxLock lock_(ctx);
    if (!ctx || (count && !image_ids)) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    if (reduce_rounds < 0 || reduce_rounds > 7)
        return fail(ctx, CHGPU_EINVAL, "reduce_dot tail rounds out of range 0..7");  // hashing.hpp:28-29
    if (!ctx->has_family) return fail(ctx, CHGPU_ELOGIC, "no hash family installed");
    if (!ctx->has_centering) return fail(ctx, CHGPU_ELOGIC, "compute_codes: centering has not been set");  // hashing.cpp:131-132
    if (count == 0) return CHGPU_OK;
    std::vector<uint32_t> slots(count);
    uint32_t max_n = 0;
    for (uint32_t i = 0; i < count; ++i) {
        if (const chgpu_status s = find_slot(ctx, image_ids[i], &slots[i])) return s;
        max_n = std::max(max_n, ctx->images[slots[i]].dev.n);
    }
    // the images first (hash kernels), their tiles behind them (bucket build covers both)
    const std::vector<uint32_t> all = with_tile_slots(ctx, slots);
    if (const chgpu_status s = ensure_slots_scratch(ctx, all.size())) return s;
    if (const chgpu_status s = order_compute_after_copy(ctx)) return s;
    // d_slots is reused by successive calls; the pageable source is consumed synchronously
    CK(cudaStreamSynchronize(ctx->compute));
    CK(cudaMemcpyAsync(ctx->d_slots, all.data(), all.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->compute));
    if (max_n) {
        if (ctx->hash_mode != CHGPU_HASH_EXACT && ctx->filter_ready) {
            // fp32 filter + exact fixup, in launches of <= kHashBatchImages images (one queue per launch)
            for (uint32_t first = 0; first < count; first += kHashBatchImages) {
                const uint32_t cnt = std::min(kHashBatchImages, count - first);
                uint32_t mx = 0;
                for (uint32_t i = 0; i < cnt; ++i) mx = std::max(mx, ctx->images[slots[first + i]].dev.n);
                if (mx) CK(launch_hash_filtered(ctx, ctx->d_slots + first, cnt, mx, reduce_rounds));
            }
        } else {
            // gridDim.y holds at most 65,535 images: same chunks as the filtered path
            for (uint32_t first = 0; first < count; first += kHashBatchImages) {
                const uint32_t cnt = std::min(kHashBatchImages, count - first);
                uint32_t mx = 0;
                for (uint32_t i = 0; i < cnt; ++i) mx = std::max(mx, ctx->images[slots[first + i]].dev.n);
                if (mx)
                    CK(launch_hash_exact(ctx, dim3((mx + kHashTilePoints - 1) / kHashTilePoints, cnt), ctx->d_slots + first,
                                         reduce_rounds, false));
            }
        }
    }
    if (const chgpu_status s = launch_bucket_build(ctx, uint32_t(all.size()))) return s;
    for (const uint32_t sl : all) {
        ImageRec& r = ctx->images[sl];
        r.dev.flags |= 1u;
        r.hash_gen = ctx->centering_gen;
        ctx->h_images[sl] = r.dev;
    }
    // flags live only on the host mirror and in the device table; kernels never read them, so
    // the table entries pushed at upload time stay valid.
    return CHGPU_OK;
}

chgpu_status chgpu_download_codes(chgpu_ctx* ctx, uint32_t image_id, uint32_t* shorts, uint64_t* longs) {
    CtxLock lock_(ctx);
    if (!ctx) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    uint32_t slot = 0;
    if (const chgpu_status s = find_slot(ctx, image_id, &slot)) return s;
    const DevImage& d = ctx->images[slot].dev;
    if (!(d.flags & 1u)) return fail(ctx, CHGPU_ELOGIC, "image %u: codes not computed", image_id);
    if (const chgpu_status s = chgpu_sync(ctx)) return s;
    if (shorts && d.n) CK(cudaMemcpy(shorts, d.shorts, size_t(d.n) * ctx->fam.table_count * 4, cudaMemcpyDeviceToHost));
    // uint4 words (x,y,z,w) = bits 0..127 little-endian = LongCode::words[0], words[1]
    if (longs && d.n) CK(cudaMemcpy(longs, d.longs, size_t(d.n) * 16, cudaMemcpyDeviceToHost));
    return CHGPU_OK;
}

chgpu_status chgpu_upload_codes(chgpu_ctx* ctx, uint32_t image_id, const uint32_t* shorts, const uint64_t* longs) {
    CtxLock lock_(ctx);
    if (!ctx || !shorts || !longs) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    uint32_t slot = 0;
    if (const chgpu_status s = find_slot(ctx, image_id, &slot)) return s;
    ImageRec& r = ctx->images[slot];
    const uint32_t n = r.dev.n, L = ctx->fam.table_count, m = ctx->fam.short_bits;
    for (size_t i = 0; i < size_t(n) * L; ++i)
        if (m < 32 && (shorts[i] >> m) != 0) return fail(ctx, CHGPU_EINVAL, "short code %u exceeds %u bits", shorts[i], m);
    if (const chgpu_status s = order_copy_after_compute(ctx)) return s;
    if (const chgpu_status s = h2d(ctx, r.dev.shorts, shorts, size_t(n) * L * 4)) return s;
    if (const chgpu_status s = h2d(ctx, r.dev.longs, longs, size_t(n) * 16)) return s;
    const std::vector<uint32_t> all = with_tile_slots(ctx, std::vector<uint32_t>{slot});
    if (const chgpu_status s = ensure_slots_scratch(ctx, all.size())) return s;
    if (const chgpu_status s = order_compute_after_copy(ctx)) return s;
    CK(cudaStreamSynchronize(ctx->compute));
    CK(cudaMemcpyAsync(ctx->d_slots, all.data(), all.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->compute));
    if (const chgpu_status s = launch_bucket_build(ctx, uint32_t(all.size()))) return s;
    CK(cudaStreamSynchronize(ctx->compute));
    for (const uint32_t sl : all) {
        ctx->images[sl].dev.flags |= 1u;
        ctx->images[sl].hash_gen = 0;
        ctx->h_images[sl] = ctx->images[sl].dev;
    }
    return CHGPU_OK;
}

chgpu_status chgpu_download_bucket_index(chgpu_ctx* ctx, uint32_t image_id, uint32_t* offsets, uint32_t* points) {
    CtxLock lock_(ctx);
    if (!ctx) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    uint32_t slot = 0;
    if (const chgpu_status s = find_slot(ctx, image_id, &slot)) return s;
    const DevImage& d = ctx->images[slot].dev;
    if (!(d.flags & 1u)) return fail(ctx, CHGPU_ELOGIC, "image %u: codes not computed", image_id);
    if (ctx->sparse)
        return fail(ctx, CHGPU_EUNSUPPORTED, "short_bits %u: the image has no dense offset table (chgpu_download_sorted_index)",
                    ctx->fam.short_bits);
    if (const chgpu_status s = chgpu_sync(ctx)) return s;
    const uint32_t L = ctx->fam.table_count;
    const size_t noff = size_t(L) * ((size_t(1) << ctx->fam.short_bits) + 1);
    if (offsets) CK(cudaMemcpy(offsets, d.offs, noff * 4, cudaMemcpyDeviceToHost));
    if (points && d.n) {
        std::vector<uint16_t> tmp(size_t(L) * d.n);
        CK(cudaMemcpy(tmp.data(), d.points, tmp.size() * 2, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < tmp.size(); ++i) points[i] = tmp[i];
    }
    return CHGPU_OK;
}

// ---- code caches ----------------------------------------------------------------------------------
chgpu_status chgpu_image_save_code_cache(chgpu_ctx* ctx, uint32_t image_id, const char* path) {
    CtxLock lock_(ctx);
    if (!ctx || !path) return CHGPU_EINVAL;
    if (!ctx->has_centering) return fail(ctx, CHGPU_ELOGIC, "code cache: centering has not been set");
    uint32_t slot = 0;
    if (const chgpu_status s = find_slot(ctx, image_id, &slot)) return s;
    const uint32_t n = ctx->images[slot].dev.n;
    std::vector<uint32_t> shorts(size_t(n) * ctx->fam.table_count);
    std::vector<uint64_t> longs(size_t(n) * 2);
    if (const chgpu_status s = chgpu_download_codes(ctx, image_id, shorts.data(), longs.data())) return s;
    const chgpu_status s = chgpu_save_code_cache(path, &ctx->fam, chgpu_centering_fingerprint(ctx->h_centering), n,
                                                 shorts.data(), longs.data());
    if (s != CHGPU_OK) return fail(ctx, s, "%s: unwritable path at byte 0", path);
    return CHGPU_OK;
}

chgpu_status chgpu_image_load_code_cache(chgpu_ctx* ctx, uint32_t image_id, const char* path, chgpu_file_fault* fault,
                                         uint64_t* fault_offset) {
    CtxLock lock_(ctx);
    if (!ctx || !path) return CHGPU_EINVAL;
    if (!ctx->has_centering) return fail(ctx, CHGPU_ELOGIC, "code cache: centering has not been set");
    uint32_t slot = 0;
    if (const chgpu_status s = find_slot(ctx, image_id, &slot)) return s;
    const uint32_t n = ctx->images[slot].dev.n;
    std::vector<uint32_t> shorts(std::max<size_t>(1, size_t(n) * ctx->fam.table_count));
    std::vector<uint64_t> longs(std::max<size_t>(1, size_t(n) * 2));
    uint32_t count = 0;
    const chgpu_status s = chgpu_load_code_cache(path, &ctx->fam, chgpu_centering_fingerprint(ctx->h_centering), n, &count,
                                                 shorts.data(), longs.data(), fault, fault_offset);
    if (s == CHGPU_EMISMATCH) return fail(ctx, s, "%s: code cache parameters mismatch active config", path);
    if (s == CHGPU_ENOMEM || (s == CHGPU_OK && count != n))  // cache_is_current also compares the point count (engine.cpp:581)
        return fail(ctx, CHGPU_EMISMATCH, "%s: code cache holds %u points, image %u has %u", path, count, image_id, n);
    if (s != CHGPU_OK) return fail(ctx, s, "%s: unreadable code cache", path);
    if (const chgpu_status u = chgpu_upload_codes(ctx, image_id, shorts.data(), longs.data())) return u;
    ctx->images[slot].hash_gen = ctx->centering_gen;  // the cache's centering fingerprint equals the installed vector's
    return CHGPU_OK;
}

// ---- match --------------------------------------------------------------------------------------
chgpu_status chgpu_match_pairs(chgpu_ctx* ctx, const uint32_t* pairs, uint32_t npairs, const chgpu_match_cfg* cfg,
                               uint64_t* offsets, chgpu_match_record* records, uint64_t capacity, uint64_t* total,
                               chgpu_match_stats* stats) {
    CtxLock lock_(ctx);
    if (!ctx || !cfg || !offsets || (npairs && !pairs) || (capacity && !records)) return CHGPU_EINVAL;
    MatchRun run{pairs, npairs, *cfg, SinkMode::Host};
    run.offsets = offsets;
    run.records = records;
    run.capacity = capacity;
    const chgpu_status s = run_match(ctx, run, stats);
    if (total) *total = run.total;
    if (s != CHGPU_OK) return s;
    if (run.overflow)
        return fail(ctx, CHGPU_ENOMEM, "record capacity %llu < %llu required", (unsigned long long)capacity,
                    (unsigned long long)run.total);
    return CHGPU_OK;
}

chgpu_status chgpu_match_pairs_stream(chgpu_ctx* ctx, const uint32_t* pairs, uint32_t npairs,
                                      const chgpu_match_cfg* cfg, chgpu_sink_fn sink, void* user,
                                      chgpu_match_stats* stats) {
    CtxLock lock_(ctx);
    if (!ctx || !cfg || (npairs && !pairs)) return CHGPU_EINVAL;
    MatchRun run{pairs, npairs, *cfg, SinkMode::Stream};
    run.sink = sink;
    run.user = user;
    return run_match(ctx, run, stats);
}

chgpu_status chgpu_match_pairs_guided(chgpu_ctx* ctx, const uint32_t* pairs, uint32_t npairs, const chgpu_match_cfg* cfg,
                                      const double* fmats, double band_px, uint64_t* offsets, chgpu_match_record* records,
                                      uint64_t capacity, uint64_t* total, chgpu_match_stats* stats) {
    CtxLock lock_(ctx);
    if (!ctx || !cfg || !offsets || (npairs && (!pairs || !fmats)) || (capacity && !records)) return CHGPU_EINVAL;
    if (!(band_px >= 0.0)) return fail(ctx, CHGPU_EINVAL, "band_px must be >= 0");
    MatchRun run{pairs, npairs, *cfg, SinkMode::Host};
    run.offsets = offsets;
    run.records = records;
    run.capacity = capacity;
    run.fmats = npairs ? fmats : nullptr;
    run.band_px = band_px;
    const chgpu_status s = run_match(ctx, run, stats);
    if (total) *total = run.total;
    if (s != CHGPU_OK) return s;
    if (run.overflow)
        return fail(ctx, CHGPU_ENOMEM, "record capacity %llu < %llu required", (unsigned long long)capacity,
                    (unsigned long long)run.total);
    return CHGPU_OK;
}

chgpu_status chgpu_match_pairs_guided_stream(chgpu_ctx* ctx, const uint32_t* pairs, uint32_t npairs,
                                             const chgpu_match_cfg* cfg, const double* fmats, double band_px,
                                             chgpu_sink_fn sink, void* user, chgpu_match_stats* stats) {
    CtxLock lock_(ctx);
    if (!ctx || !cfg || (npairs && (!pairs || !fmats))) return CHGPU_EINVAL;
    if (!(band_px >= 0.0)) return fail(ctx, CHGPU_EINVAL, "band_px must be >= 0");
    MatchRun run{pairs, npairs, *cfg, SinkMode::Stream};
    run.sink = sink;
    run.user = user;
    run.fmats = npairs ? fmats : nullptr;
    run.band_px = band_px;
    return run_match(ctx, run, stats);
}

chgpu_status chgpu_match_pairs_to_files(chgpu_ctx* ctx, const uint32_t* pairs, uint32_t npairs, const chgpu_match_cfg* cfg,
                                        chgpu_sink* sink, chgpu_match_stats* stats) {
    CtxLock lock_(ctx);
    if (!ctx || !cfg || !sink || (npairs && !pairs)) return CHGPU_EINVAL;
    struct Feed {
        chgpu_sink* sink;
        const uint32_t* pairs;
    } feed{sink, pairs};
    auto to_writer = [](void* user, uint32_t first, uint32_t count, const uint64_t* offs, const chgpu_match_record* rec) -> int {
        Feed* f = static_cast<Feed*>(user);
        return chgpu_sink_accept(f->sink, f->pairs + 2 * size_t(first), count, offs, rec) == CHGPU_OK ? 0 : 1;
    };
    MatchRun run{pairs, npairs, *cfg, SinkMode::Stream};
    run.sink = to_writer;
    run.user = &feed;
    return run_match(ctx, run, stats);
}

chgpu_status chgpu_match_pairs_device(chgpu_ctx* ctx, const uint32_t* pairs, uint32_t npairs,
                                      const chgpu_match_cfg* cfg, chgpu_match_stats* stats) {
    CtxLock lock_(ctx);
    if (!ctx || !cfg || (npairs && !pairs)) return CHGPU_EINVAL;
    MatchRun run{pairs, npairs, *cfg, SinkMode::Device};
    return run_match(ctx, run, stats);
}

chgpu_status chgpu_debug_ranked_guided(chgpu_ctx* ctx, uint32_t image_i, uint32_t image_j, const chgpu_match_cfg* cfg,
                                       const double* fmat, double band_px, uint32_t* ranked, uint32_t* ranked_count) {
    CtxLock lock_(ctx);
    if (!ctx || !cfg || !ranked || !ranked_count || !fmat) return CHGPU_EINVAL;
    const uint32_t pr[2] = {image_i, image_j};
    MatchRun run{pr, 1, *cfg, SinkMode::Device};
    run.dbg_ranked = ranked;
    run.dbg_count = ranked_count;
    run.fmats = fmat;
    run.band_px = band_px;
    return run_match(ctx, run, nullptr);
}

chgpu_status chgpu_debug_ranked(chgpu_ctx* ctx, uint32_t image_i, uint32_t image_j, const chgpu_match_cfg* cfg,
                                uint32_t* ranked, uint32_t* ranked_count) {
    CtxLock lock_(ctx);
    if (!ctx || !cfg || !ranked || !ranked_count) return CHGPU_EINVAL;
    const uint32_t pr[2] = {image_i, image_j};
    MatchRun run{pr, 1, *cfg, SinkMode::Device};
    run.dbg_ranked = ranked;
    run.dbg_count = ranked_count;
    return run_match(ctx, run, nullptr);
}

// ---- general path: sorted index, candidate lists, match from explicit lists (general_kernels.cuh) ---------------------
chgpu_status chgpu_download_sorted_index(chgpu_ctx* ctx, uint32_t image_id, uint32_t* codes, uint32_t* points) {
    CtxLock lock_(ctx);
    if (!ctx || !codes || !points) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    uint32_t slot = 0;
    if (const chgpu_status s = find_slot(ctx, image_id, &slot)) return s;
    const DevImage& d = ctx->images[slot].dev;
    if (!(d.flags & 1u)) return fail(ctx, CHGPU_ELOGIC, "image %u: codes not computed", image_id);
    if (const chgpu_status s = chgpu_sync(ctx)) return s;
    const uint32_t L = ctx->fam.table_count, nb1 = ctx->sparse ? 0u : (1u << ctx->fam.short_bits) + 1u;
    const size_t entries = size_t(L) * d.n;
    if (entries == 0) return CHGPU_OK;
    if (ctx->sparse) {
        std::vector<unsigned long long> keys(entries);
        CK(cudaMemcpy(keys.data(), d.offs, entries * 8, cudaMemcpyDeviceToHost));
        for (size_t e = 0; e < entries; ++e) {
            codes[e] = uint32_t(keys[e] >> 16);
            points[e] = uint32_t(keys[e] & 0xffffu);
        }
    } else {
        std::vector<uint32_t> offs(size_t(L) * nb1);
        std::vector<uint16_t> pts(entries);
        CK(cudaMemcpy(offs.data(), d.offs, offs.size() * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(pts.data(), d.points, entries * 2, cudaMemcpyDeviceToHost));
        for (uint32_t t = 0; t < L; ++t)
            for (uint32_t c = 0; c + 1 < nb1; ++c)
                for (uint32_t e = offs[size_t(t) * nb1 + c]; e < offs[size_t(t) * nb1 + c + 1]; ++e) {
                    codes[size_t(t) * d.n + e] = c;
                    points[size_t(t) * d.n + e] = pts[size_t(t) * d.n + e];
                }
    }
    return CHGPU_OK;
}

chgpu_status chgpu_pair_candidates(chgpu_ctx* ctx, uint32_t image_i, uint32_t image_j, uint64_t* offsets, uint32_t* candidates,
                                   uint64_t capacity, uint64_t* total) {
    CtxLock lock_(ctx);
    if (!ctx || !offsets || (capacity && !candidates)) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    if (!ctx->has_family) return fail(ctx, CHGPU_ELOGIC, "no hash family installed");
    uint32_t si = 0, sj = 0;
    if (const chgpu_status s = find_slot(ctx, image_i, &si)) return s;
    if (const chgpu_status s = find_slot(ctx, image_j, &sj)) return s;
    const DevImage& I = ctx->images[si].dev;
    const DevImage& J = ctx->images[sj].dev;
    if (!(I.flags & 1u) || !(J.flags & 1u))
        return fail(ctx, CHGPU_ELOGIC, "pair (%u,%u): codes not computed (call chgpu_hash_images first)", image_i, image_j);
    offsets[0] = 0;
    if (total) *total = 0;
    if (I.n == 0) return CHGPU_OK;
    if (const chgpu_status s = order_compute_after_copy(ctx)) return s;
    uint32_t* d_counts = nullptr;
    unsigned long long* d_offs = nullptr;
    uint32_t* d_out = nullptr;
    auto cleanup = [&] {
        cudaFree(d_counts);
        cudaFree(d_offs);
        cudaFree(d_out);
    };
    const size_t smem = size_t(kGenWarps) * kGenBitmapWords * sizeof(uint32_t);
    const uint32_t grid = std::max(1u, std::min((I.n + kGenWarps - 1) / kGenWarps, uint32_t(ctx->prop.multiProcessorCount) * 3u));
    chgpu_status rc = CHGPU_OK;
    auto run = [&]() -> chgpu_status {
        CK(cudaFuncSetAttribute(cand_union_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        CK(cudaMalloc(&d_counts, size_t(I.n) * sizeof(uint32_t)));
        cand_union_kernel<<<grid, kGenThreads, smem, ctx->compute>>>(ctx->d_images, si, sj, ctx->fam.short_bits, ctx->fam.table_count,
                                                                    ctx->sparse ? 1u : 0u, d_counts, nullptr, nullptr);
        CK(cudaGetLastError());
        std::vector<uint32_t> counts(I.n);
        CK(cudaMemcpyAsync(counts.data(), d_counts, size_t(I.n) * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->compute));
        CK(cudaStreamSynchronize(ctx->compute));
        for (uint32_t q = 0; q < I.n; ++q) offsets[q + 1] = offsets[q] + counts[q];
        const uint64_t sum = offsets[I.n];
        if (total) *total = sum;
        if (sum > capacity) return fail(ctx, CHGPU_ENOMEM, "candidate capacity %llu < %llu required", (unsigned long long)capacity,
                                        (unsigned long long)sum);
        if (sum == 0) return CHGPU_OK;
        static_assert(sizeof(unsigned long long) == sizeof(uint64_t), "offset width");
        CK(cudaMalloc(&d_offs, (size_t(I.n) + 1) * sizeof(unsigned long long)));
        CK(cudaMalloc(&d_out, sum * sizeof(uint32_t)));
        CK(cudaMemcpyAsync(d_offs, offsets, (size_t(I.n) + 1) * sizeof(unsigned long long), cudaMemcpyHostToDevice, ctx->compute));
        cand_union_kernel<<<grid, kGenThreads, smem, ctx->compute>>>(ctx->d_images, si, sj, ctx->fam.short_bits, ctx->fam.table_count,
                                                                    ctx->sparse ? 1u : 0u, nullptr, d_offs, d_out);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(candidates, d_out, sum * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->compute));
        CK(cudaStreamSynchronize(ctx->compute));
        return CHGPU_OK;
    };
    rc = run();
    if (rc != CHGPU_OK && rc != CHGPU_ENOMEM) {
        cudaStreamSynchronize(ctx->compute);
        cudaGetLastError();
    }
    cleanup();
    return rc;
}

chgpu_status chgpu_match_pair_lists(chgpu_ctx* ctx, uint32_t image_i, uint32_t image_j, const chgpu_match_cfg* cfg,
                                    const uint64_t* list_offsets, const uint32_t* list_ids, chgpu_match_record* records,
                                    uint64_t capacity, uint64_t* total, chgpu_match_stats* stats) {
    CtxLock lock_(ctx);
    if (!ctx || !cfg || !list_offsets || (capacity && !records)) return CHGPU_EINVAL;
    DeviceGuard guard(ctx->device);
    uint32_t si = 0, sj = 0;
    if (const chgpu_status s = find_slot(ctx, image_i, &si)) return s;
    if (const chgpu_status s = find_slot(ctx, image_j, &sj)) return s;
    const uint32_t nq = ctx->images[si].dev.n, nt = ctx->images[sj].dev.n;
    const uint64_t sum = list_offsets[nq];
    if (list_offsets[0] != 0) return fail(ctx, CHGPU_EINVAL, "candidate lists: offsets must start at 0");
    for (uint32_t q = 0; q < nq; ++q) {
        if (list_offsets[q + 1] < list_offsets[q]) return fail(ctx, CHGPU_EINVAL, "candidate lists: offsets decrease at query %u", q);
        if (list_offsets[q + 1] - list_offsets[q] >= (1ull << 24))
            return fail(ctx, CHGPU_EUNSUPPORTED, "candidate list of query %u has %llu entries; the device ranks < 2^24 per query", q,
                        (unsigned long long)(list_offsets[q + 1] - list_offsets[q]));
    }
    if (sum && !list_ids) return CHGPU_EINVAL;
    for (uint64_t e = 0; e < sum; ++e)
        if (list_ids[e] >= nt) return fail(ctx, CHGPU_EINVAL, "candidate lists: entry %llu names train point %u of %u", (unsigned long long)e, list_ids[e], nt);
    CK(cudaStreamSynchronize(ctx->compute));
    cudaFree(ctx->d_list_offs);
    cudaFree(ctx->d_list_ids);
    ctx->d_list_offs = nullptr;
    ctx->d_list_ids = nullptr;
    static_assert(sizeof(unsigned long long) == sizeof(uint64_t), "offset width");
    CK(cudaMalloc(&ctx->d_list_offs, (size_t(nq) + 1) * sizeof(unsigned long long)));
    CK(cudaMalloc(&ctx->d_list_ids, std::max<uint64_t>(sum, 1) * sizeof(uint32_t)));
    CK(cudaMemcpy(ctx->d_list_offs, list_offsets, (size_t(nq) + 1) * sizeof(unsigned long long), cudaMemcpyHostToDevice));
    if (sum) CK(cudaMemcpy(ctx->d_list_ids, list_ids, sum * sizeof(uint32_t), cudaMemcpyHostToDevice));
    const uint32_t pr[2] = {image_i, image_j};
    uint64_t offs[2] = {0, 0};
    MatchRun run{pr, 1, *cfg, SinkMode::Host};
    run.offsets = offs;
    run.records = records;
    run.capacity = capacity;
    run.lists = true;
    const chgpu_status s = run_match(ctx, run, stats);
    if (total) *total = run.total;
    if (s != CHGPU_OK) return s;
    if (run.overflow)
        return fail(ctx, CHGPU_ENOMEM, "record capacity %llu < %llu required", (unsigned long long)capacity, (unsigned long long)run.total);
    return CHGPU_OK;
}

}  // extern "C"
