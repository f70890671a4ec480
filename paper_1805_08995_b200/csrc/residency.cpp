// residency.cpp — block-pair tasks, the two-line residency schedule and the out-of-core run of a plan.
//
// Host code of libchgpu.so.  The schedule is the reference's step_residency machine (scheduler.cpp:226-345) with
// the slot limits as parameters: at the reference's limits (2 hashing / 3 matching, scheduler.hpp:70-72) the trace
// is the reference's, action for action (tests/test_residency.py pins it against the compiled reference); a B200
// run picks limits from its 180 GB instead.  The driver replays the trace through the public entry points of
// chgpu.h (loader, hash build, eviction, streamed match), so it adds no device code of its own.

#include "../../include/chgpu.h"
#include "plan_tasks.hpp"

#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

namespace {

constexpr uint32_t kNever = std::numeric_limits<uint32_t>::max();

// ---- tasks ---------------------------------------------------------------------------------------------------
struct Partition {
    uint32_t images, block_images, blocks_per_group, nblocks;
    uint32_t lo(uint32_t b) const { return b * block_images; }
    uint32_t hi(uint32_t b) const { return uint32_t(std::min<uint64_t>(images, uint64_t(b + 1) * block_images)); }
    uint32_t size(uint32_t b) const { return hi(b) - lo(b); }
    uint32_t group_of(uint32_t b) const { return b / blocks_per_group; }
};

// accepted pairs keyed by (block pair, a * K + b), sorted and unique: the guided plan's buckets (host_util.cpp)
using Keyed = std::vector<std::pair<uint64_t, uint64_t>>;

chgpu_status key_accepted(const Partition& p, const uint32_t* accepted, uint64_t count, Keyed& keyed) {
    keyed.clear();
    keyed.reserve(count);
    for (uint64_t i = 0; i < count; ++i) {
        uint32_t a = accepted[2 * i], b = accepted[2 * i + 1];
        if (a == b) return CHGPU_EINVAL;        // plan_guided: self pair (scheduler.cpp:149)
        if (a > b) std::swap(a, b);
        if (b >= p.images) return CHGPU_EINVAL;  // plan_guided: unknown image index (scheduler.cpp:151)
        keyed.emplace_back(uint64_t(a / p.block_images) * p.nblocks + b / p.block_images, uint64_t(a) * p.images + b);
    }
    std::sort(keyed.begin(), keyed.end());
    keyed.erase(std::unique(keyed.begin(), keyed.end()), keyed.end());
    return CHGPU_OK;
}

std::pair<Keyed::const_iterator, Keyed::const_iterator> bucket_of(const Keyed& keyed, uint64_t key) {
    auto first = std::lower_bound(keyed.begin(), keyed.end(), std::make_pair(key, uint64_t(0)));
    auto last = first;
    while (last != keyed.end() && last->first == key) ++last;
    return {first, last};
}

// Tasks of the plan in plan order (PlanTask without its pair list, scheduler.hpp:36-43).
chgpu_status build_tasks(const Partition& p, const Keyed* keyed, std::vector<chgpu_plan_task>& out) {
    out.clear();
    uint64_t np = 0;
    auto push = [&](uint32_t ba, uint32_t bb, uint64_t count) {
        chgpu_plan_task t{};
        t.block_a = ba;
        t.block_b = bb;
        t.group_a = p.group_of(ba);
        t.group_b = p.group_of(bb);
        t.first_pair = np;
        t.npairs = count;
        np += count;
        out.push_back(t);
    };
    chgpu::for_each_plan_task(
        p.images, p.block_images, p.blocks_per_group,
        [&](uint32_t ba, uint32_t bb) {
            if (keyed) {
                const auto r = bucket_of(*keyed, uint64_t(ba) * p.nblocks + bb);
                if (r.first != r.second) push(ba, bb, uint64_t(r.second - r.first));
            } else {
                push(ba, bb, uint64_t(p.size(ba)) * p.size(bb));
            }
        },
        [&](uint32_t blk) {
            if (keyed) {
                const auto r = bucket_of(*keyed, uint64_t(blk) * p.nblocks + blk);
                if (r.first != r.second) push(blk, blk, uint64_t(r.second - r.first));
            } else {
                const uint64_t n = p.size(blk);
                if (n >= 2) push(blk, blk, n * (n - 1) / 2);  // a single-image block contributes nothing (scheduler.cpp:135-139)
            }
        });
    return CHGPU_OK;
}

// ---- the residency machine -------------------------------------------------------------------------------------
// One storage level: what is resident, and for every item the ascending list of tasks that use it.
struct Level {
    uint32_t limit = 0;
    chgpu_residency_level tag = CHGPU_LEVEL_GROUP;
    std::vector<uint32_t> resident;
    std::vector<std::vector<uint32_t>> uses;

    bool has(uint32_t id) const { return std::find(resident.begin(), resident.end(), id) != resident.end(); }
    uint32_t next_use(uint32_t id, uint32_t from) const {
        if (id >= uses.size()) return kNever;
        const auto& u = uses[id];
        const auto it = std::lower_bound(u.begin(), u.end(), from);
        return it == u.end() ? kNever : *it;
    }
    // One move towards residency of `id` (first needed by task need_at): a load into a free slot, else the
    // eviction of the resident item whose next use lies farthest ahead (ties: smaller id) — but only if that use
    // is strictly later than need_at.  false: the level is full of data needed no later than `id`.
    bool advance(uint32_t id, uint32_t need_at, uint32_t cursor, bool prefetch, chgpu_residency_action& act) {
        if (resident.size() < limit) {
            resident.push_back(id);
            act = {CHGPU_ACT_LOAD, uint32_t(tag), id, prefetch ? 1u : 0u};
            return true;
        }
        uint32_t victim = kNever, far = 0;
        for (const uint32_t r : resident) {
            const uint32_t u = next_use(r, cursor);
            if (u > far || (u == far && (victim == kNever || r < victim))) {
                victim = r;
                far = u;
            }
        }
        if (victim == kNever || far <= need_at) return false;
        resident.erase(std::find(resident.begin(), resident.end(), victim));
        act = {CHGPU_ACT_EVICT, uint32_t(tag), victim, 0u};
        return true;
    }
};

struct Machine {
    const chgpu_plan_task* tasks = nullptr;
    uint32_t ntasks = 0, cursor = 0;
    bool begun = false, done = false, blocked = false;
    Level groups, blocks;

    // what task t needs, in the order residency_tasks lists it (scheduler.cpp:175-192)
    static uint32_t items(const chgpu_plan_task& t, uint32_t (&g)[2], uint32_t (&b)[2], uint32_t (&bg)[2], uint32_t& ng) {
        g[0] = t.group_a;
        ng = 1;
        if (t.group_b != t.group_a) g[ng++] = t.group_b;
        b[0] = t.block_a;
        bg[0] = t.group_a;
        uint32_t nb = 1;
        if (t.block_b != t.block_a) {
            b[nb] = t.block_b;
            bg[nb++] = t.group_b;
        }
        return nb;
    }

    void init(const chgpu_plan_task* ts, uint32_t n, uint32_t group_limit, uint32_t block_limit) {
        tasks = ts;
        ntasks = n;
        groups.limit = group_limit;
        groups.tag = CHGPU_LEVEL_GROUP;
        blocks.limit = block_limit;
        blocks.tag = CHGPU_LEVEL_BLOCK;
        uint32_t mg = 0, mb = 0;
        for (uint32_t t = 0; t < n; ++t) {
            mg = std::max(mg, std::max(ts[t].group_a, ts[t].group_b) + 1);
            mb = std::max(mb, std::max(ts[t].block_a, ts[t].block_b) + 1);
        }
        groups.uses.assign(mg, {});
        blocks.uses.assign(mb, {});
        for (uint32_t t = 0; t < n; ++t) {
            uint32_t g[2], b[2], bg[2], ng;
            const uint32_t nb = items(ts[t], g, b, bg, ng);
            for (uint32_t i = 0; i < ng; ++i) groups.uses[g[i]].push_back(t);
            for (uint32_t i = 0; i < nb; ++i) blocks.uses[b[i]].push_back(t);
        }
        done = n == 0;
    }

    // One transition (step_residency, scheduler.cpp:269-337).  false when the plan is exhausted or, with
    // `blocked` set, when the current task cannot be made resident under the limits.
    bool step(chgpu_residency_action& act) {
        if (done) return false;
        uint32_t g[2], b[2], bg[2], ng;
        const uint32_t nb = items(tasks[cursor], g, b, bg, ng);
        // line 1, memory level
        if (!begun)
            for (uint32_t i = 0; i < ng; ++i)
                if (!groups.has(g[i])) {
                    if (groups.advance(g[i], cursor, cursor, false, act)) return true;
                    blocked = true;
                    return false;
                }
        // line 2, memory level: the nearest future group that is not resident, strictly in order
        for (uint32_t t = cursor + 1; t < ntasks; ++t) {
            uint32_t fg[2], fb[2], fbg[2], fng;
            items(tasks[t], fg, fb, fbg, fng);
            bool all = true;
            for (uint32_t i = 0; i < fng; ++i) {
                if (groups.has(fg[i])) continue;
                all = false;
                if (groups.advance(fg[i], t, cursor, true, act)) return true;
            }
            if (!all) break;
        }
        // line 1, device level
        if (!begun)
            for (uint32_t i = 0; i < nb; ++i)
                if (!blocks.has(b[i])) {
                    if (blocks.advance(b[i], cursor, cursor, false, act)) return true;
                    blocked = true;
                    return false;
                }
        // line 2, device level: the nearest future block whose group is already in memory
        for (uint32_t t = cursor + 1; t < ntasks; ++t) {
            uint32_t fg[2], fb[2], fbg[2], fng;
            const uint32_t fnb = items(tasks[t], fg, fb, fbg, fng);
            bool all = true, waits = false;
            for (uint32_t i = 0; i < fnb; ++i) {
                if (blocks.has(fb[i])) continue;
                all = false;
                if (!groups.has(fbg[i])) {
                    waits = true;
                    break;
                }
                if (blocks.advance(fb[i], t, cursor, true, act)) return true;
            }
            if (!all || waits) break;
        }
        if (!begun) {
            begun = true;
            act = {CHGPU_ACT_BEGIN, CHGPU_LEVEL_BLOCK, cursor, 0u};
            return true;
        }
        act = {CHGPU_ACT_FINISH, CHGPU_LEVEL_BLOCK, cursor, 0u};
        begun = false;
        if (++cursor >= ntasks) done = true;
        return true;
    }
};

// Greedy order for reuse: always the pending task that needs the fewest block loads given what is resident (ties:
// plan order); a block that has to go is the resident one with the fewest tasks left.
void order_for_reuse(const chgpu_plan_task* tasks, uint32_t n, uint32_t slots, std::vector<uint32_t>& order) {
    order.clear();
    order.reserve(n);
    if (n > (1u << 18) || slots < 2) {
        for (uint32_t t = 0; t < n; ++t) order.push_back(t);
        return;
    }
    uint32_t nblocks = 0;
    for (uint32_t t = 0; t < n; ++t) nblocks = std::max(nblocks, std::max(tasks[t].block_a, tasks[t].block_b) + 1);
    std::vector<std::vector<uint32_t>> of_block(nblocks);  // ascending task indices
    std::vector<uint32_t> left(nblocks, 0), head(nblocks, 0);
    for (uint32_t t = 0; t < n; ++t) {
        of_block[tasks[t].block_a].push_back(t);
        ++left[tasks[t].block_a];
        if (tasks[t].block_b != tasks[t].block_a) {
            of_block[tasks[t].block_b].push_back(t);
            ++left[tasks[t].block_b];
        }
    }
    std::vector<uint8_t> done(n, 0), is_res(nblocks, 0);
    std::vector<uint32_t> resident;
    uint32_t first_pending = 0;
    auto missing = [&](uint32_t t) { return (is_res[tasks[t].block_a] ? 0 : 1) + (tasks[t].block_b != tasks[t].block_a && !is_res[tasks[t].block_b] ? 1 : 0); };
    for (uint32_t step = 0; step < n; ++step) {
        // best pending task among those touching a resident block; else the first pending task of the plan
        uint32_t best = kNever, best_missing = 3;
        for (const uint32_t r : resident) {
            auto& list = of_block[r];
            while (head[r] < list.size() && done[list[head[r]]]) ++head[r];
            for (uint32_t k = head[r]; k < list.size(); ++k) {
                const uint32_t t = list[k];
                if (done[t]) continue;
                const uint32_t ms = missing(t);
                if (ms < best_missing || (ms == best_missing && t < best)) {
                    best = t;
                    best_missing = ms;
                }
                if (ms == 0) break;  // lists ascend: the first fully resident task of this block is its best
            }
        }
        if (best == kNever) {
            while (done[first_pending]) ++first_pending;
            best = first_pending;
        }
        const uint32_t need[2] = {tasks[best].block_a, tasks[best].block_b};
        for (const uint32_t b : need) {
            if (is_res[b]) continue;
            if (resident.size() >= slots) {
                uint32_t victim = kNever, fewest = kNever;
                for (const uint32_t r : resident) {
                    if (r == need[0] || r == need[1]) continue;
                    if (left[r] < fewest || (left[r] == fewest && r < victim)) {
                        victim = r;
                        fewest = left[r];
                    }
                }
                if (victim != kNever) {
                    resident.erase(std::find(resident.begin(), resident.end(), victim));
                    is_res[victim] = 0;
                }
            }
            resident.push_back(b);
            is_res[b] = 1;
        }
        done[best] = 1;
        --left[need[0]];
        if (need[1] != need[0]) --left[need[1]];
        order.push_back(best);
    }
}

// Contiguous ranges of the executed sequence, balanced by pair count: worker s gets positions [first[s], first[s + 1]).
// `weights` (nullable): work per task (chgpu_task_weights) instead of its pair count.
void shard_sequence(const chgpu_plan_task* tasks, const uint32_t* order, uint32_t n, uint32_t shards, std::vector<uint32_t>& first,
                    const uint64_t* weights = nullptr) {
    shards = std::max<uint32_t>(1, shards);
    auto weight = [&](uint32_t k) -> uint64_t {
        const uint32_t t = order ? order[k] : k;
        return weights ? weights[t] : tasks[t].npairs;
    };
    unsigned __int128 total = 0;
    for (uint32_t k = 0; k < n; ++k) total += weight(k);
    first.assign(shards + 1, n);
    first[0] = 0;
    unsigned __int128 acc = 0;
    uint32_t s = 1;
    for (uint32_t k = 0; k < n && s < shards; ++k) {
        const unsigned __int128 w = weight(k);
        if (weights) {
            // weighted: tasks differ by orders of magnitude, so a boundary goes to whichever side of task k misses the
            // worker's share by less
            while (s < shards && (acc + w) * shards >= total * s) {
                const unsigned __int128 target = total * s, before = acc * shards, after = (acc + w) * shards;
                first[s++] = (before >= target || target - before < after - target) ? k : k + 1;
            }
            acc += w;
            continue;
        }
        acc += w;
        // the boundary after position k belongs to every worker whose share of the pairs is complete by now
        while (s < shards && acc * shards >= total * s) first[s++] = k + 1;
    }
}

uint32_t default_limit(chgpu_residency_mode mode) { return mode == CHGPU_RESIDENCY_HASHING ? 2u : 3u; }

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// page-cache hints for a file (the host level of the exchange)
void advise_file(const char* path, int advice) {
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) return;
    ::posix_fadvise(fd, 0, 0, advice);
    ::close(fd);
}

// ---- replay ------------------------------------------------------------------------------------------------
struct Replay {
    chgpu_ctx* ctx;
    const char* const* paths;
    Partition part;
    uint32_t io_threads;
    bool centering_only;  // hashing schedule: blocks are summed into the centering accumulator, nothing is matched
    int reduce_rounds = 3;  // N_r of the hash build (MatchConfig::reduce_rounds, matcher.hpp:14-23)
    std::vector<chgpu_file_result> results;
    std::vector<uint8_t> ok;  // image loaded and (matching runs) hashed
    std::vector<uint8_t> block_resident;
    chgpu_streamed_stats st{};
    uint32_t resident_blocks = 0, resident_groups = 0;

    chgpu_status load_block(uint32_t b) {
        const uint32_t lo = part.lo(b), cnt = part.size(b);
        std::vector<uint32_t> ids(cnt);
        for (uint32_t i = 0; i < cnt; ++i) ids[i] = lo + i;
        chgpu_load_stats ls{};
        const auto t0 = std::chrono::steady_clock::now();
        const chgpu_status s = chgpu_load_chft_files(ctx, paths + lo, ids.data(), cnt, io_threads, centering_only ? 1 : 0,
                                                     results.data() + lo, &ls);
        st.load_seconds += seconds_since(t0);
        st.bytes_read += ls.bytes_read;
        return adopt_block(b, s);
    }

    // The block's files are on the device (results[] filled in): book-keeping + hash build of the images that made it.
    chgpu_status adopt_block(uint32_t b, chgpu_status load_status) {
        const uint32_t lo = part.lo(b), cnt = part.size(b);
        block_resident[b] = 1;
        ++resident_blocks;  // counted together with the flag: an eviction after a failed load or hash must not underflow it
        std::vector<uint32_t> good;
        for (uint32_t i = 0; i < cnt; ++i)
            if (results[lo + i].status == CHGPU_OK) {
                good.push_back(lo + i);
                ok[lo + i] = 1;
            }
        st.images_loaded += good.size();
        if (load_status != CHGPU_OK) return load_status;
        if (!centering_only && !good.empty()) {
            const auto t0 = std::chrono::steady_clock::now();
            const chgpu_status h = chgpu_hash_images(ctx, good.data(), uint32_t(good.size()), reduce_rounds);
            if (h == CHGPU_OK) chgpu_sync(ctx);
            st.hash_seconds += seconds_since(t0);
            if (h != CHGPU_OK) return h;
        }
        ++st.block_loads;
        st.max_resident_blocks = std::max(st.max_resident_blocks, resident_blocks);
        return CHGPU_OK;
    }

    // Line 2 of the exchange: the blocks the schedule prefetches while task t runs are opened as ONE background load
    // before the task's match call (which moves it forward between its sub-batches) and adopted when the task finishes.
    std::vector<uint32_t> background;  // blocks of the open background load, in load order
    chgpu_status begin_background(const std::vector<uint32_t>& blocks) {
        if (blocks.empty()) return CHGPU_OK;
        std::vector<const char*> ps;
        std::vector<uint32_t> ids;
        for (const uint32_t b : blocks)
            for (uint32_t i = part.lo(b); i < part.hi(b); ++i) {
                ps.push_back(paths[i]);
                ids.push_back(i);
            }
        const auto t0 = std::chrono::steady_clock::now();
        const chgpu_status s = chgpu_load_chft_files_begin(ctx, ps.data(), ids.data(), uint32_t(ids.size()), io_threads, 0);
        st.load_seconds += seconds_since(t0);
        if (s == CHGPU_OK) background = blocks;
        return s;
    }
    chgpu_status end_background() {
        if (background.empty()) return CHGPU_OK;
        size_t total = 0;
        for (const uint32_t b : background) total += part.size(b);
        std::vector<chgpu_file_result> res(total);
        chgpu_load_stats ls{};
        const auto t0 = std::chrono::steady_clock::now();
        const chgpu_status s = chgpu_load_chft_files_end(ctx, res.data(), &ls);
        st.load_seconds += seconds_since(t0);  // what the task could not hide
        st.bytes_read += ls.bytes_read;
        size_t at = 0;
        chgpu_status rc = s;
        const std::vector<uint32_t> blocks = background;
        background.clear();
        for (const uint32_t b : blocks) {
            std::copy(res.begin() + at, res.begin() + at + part.size(b), results.begin() + part.lo(b));
            at += part.size(b);
            const chgpu_status a = adopt_block(b, s);
            if (rc == CHGPU_OK) rc = a;
            ++st.background_block_loads;
        }
        return rc;
    }

    void evict_block(uint32_t b, bool count) {
        if (!block_resident[b]) return;
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<uint32_t> ids;
        for (uint32_t i = part.lo(b); i < part.hi(b); ++i)
            if (ok[i]) {
                ids.push_back(i);
                ok[i] = 0;
            }
        chgpu_evict_images(ctx, ids.data(), uint32_t(ids.size()));
        st.evict_seconds += seconds_since(t0);
        block_resident[b] = 0;
        if (count) {
            ++st.block_evictions;
            --resident_blocks;
        }
    }

    // Group level of the exchange: the page cache.  The hints are pure host work (open / posix_fadvise / close per
    // file), so they run on a helper thread; hint_seconds counts only what the replay had to wait for.
    std::vector<std::thread> hint_threads;
    void group_hint(uint32_t g, bool load) {
        const auto t0 = std::chrono::steady_clock::now();
        const uint32_t b0 = g * part.blocks_per_group, b1 = std::min(part.nblocks, b0 + part.blocks_per_group);
        const uint32_t lo = part.lo(b0), hi = part.hi(b1 - 1);
        const char* const* ps = paths;
        hint_threads.emplace_back([ps, lo, hi, load] {
            for (uint32_t i = lo; i < hi; ++i) advise_file(ps[i], load ? POSIX_FADV_WILLNEED : POSIX_FADV_DONTNEED);
        });
        if (load) {
            ++st.group_loads;
            st.max_resident_groups = std::max(st.max_resident_groups, ++resident_groups);
        } else {
            ++st.group_evictions;
            --resident_groups;
        }
        st.hint_seconds += seconds_since(t0);
    }
    void join_hints() {
        const auto t0 = std::chrono::steady_clock::now();
        for (std::thread& t : hint_threads) t.join();
        hint_threads.clear();
        st.hint_seconds += seconds_since(t0);
    }

    void evict_all() {
        for (uint32_t b = 0; b < part.nblocks; ++b) evict_block(b, false);
    }
};

struct SinkAdapter {
    chgpu_plan_sink_fn fn;
    void* user;
    uint32_t task;
    const uint32_t* pairs;  // of the chunk in flight
    uint64_t matches;
};

int sink_adapter(void* user, uint32_t first_pair, uint32_t npairs_chunk, const uint64_t* offsets,
                 const chgpu_match_record* records) {
    SinkAdapter* a = static_cast<SinkAdapter*>(user);
    a->matches += offsets[npairs_chunk] - offsets[0];
    if (!a->fn) return 0;
    return a->fn(a->user, a->task, a->pairs + 2 * size_t(first_pair), npairs_chunk, offsets, records);
}

constexpr uint64_t kPairsPerCall = uint64_t(1) << 20;  // pairs handed to one chgpu_match_pairs_stream call

}  // namespace

extern "C" {

chgpu_status chgpu_plan_tasks(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group,
                              const uint32_t* accepted, uint64_t accepted_count, chgpu_plan_task* tasks_out,
                              uint32_t* ntasks_out) {
    if (image_count == 0 || block_images == 0 || blocks_per_group == 0 || !ntasks_out) return CHGPU_EINVAL;
    const Partition p{image_count, block_images, blocks_per_group, (image_count + block_images - 1) / block_images};
    Keyed keyed;
    if (accepted || accepted_count) {
        if (accepted_count && !accepted) return CHGPU_EINVAL;
        if (const chgpu_status s = key_accepted(p, accepted, accepted_count, keyed)) return s;
    }
    std::vector<chgpu_plan_task> tasks;
    build_tasks(p, (accepted || accepted_count) ? &keyed : nullptr, tasks);
    if (tasks_out) std::copy(tasks.begin(), tasks.end(), tasks_out);
    *ntasks_out = uint32_t(tasks.size());
    return CHGPU_OK;
}

chgpu_status chgpu_hashing_tasks(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group,
                                 chgpu_plan_task* tasks_out, uint32_t* ntasks_out) {
    if (image_count == 0 || block_images == 0 || blocks_per_group == 0 || !ntasks_out) return CHGPU_EINVAL;
    const Partition p{image_count, block_images, blocks_per_group, (image_count + block_images - 1) / block_images};
    if (tasks_out)
        for (uint32_t b = 0; b < p.nblocks; ++b) {
            chgpu_plan_task t{};
            t.block_a = t.block_b = b;
            t.group_a = t.group_b = p.group_of(b);
            t.first_pair = 0;
            t.npairs = 0;
            tasks_out[b] = t;
        }
    *ntasks_out = p.nblocks;
    return CHGPU_OK;
}

chgpu_status chgpu_simulate_residency(const chgpu_plan_task* tasks, uint32_t ntasks, chgpu_residency_mode mode,
                                      uint32_t group_slots, uint32_t block_slots, chgpu_residency_action* actions_out,
                                      uint64_t capacity, uint64_t* nactions_out) {
    if ((ntasks && !tasks) || !nactions_out) return CHGPU_EINVAL;
    if (mode != CHGPU_RESIDENCY_HASHING && mode != CHGPU_RESIDENCY_MATCHING) return CHGPU_EINVAL;
    Machine m;
    m.init(tasks, ntasks, group_slots ? group_slots : default_limit(mode), block_slots ? block_slots : default_limit(mode));
    uint64_t n = 0;
    chgpu_residency_action act;
    while (m.step(act)) {
        if (actions_out && n < capacity) actions_out[n] = act;
        ++n;
    }
    *nactions_out = n;
    if (m.blocked) return CHGPU_EINVAL;  // reference: std::logic_error "residency: current ... load blocked"
    if (actions_out && n > capacity) return CHGPU_ENOMEM;
    return CHGPU_OK;
}

chgpu_status chgpu_order_tasks_for_reuse(const chgpu_plan_task* tasks, uint32_t ntasks, uint32_t block_slots,
                                         uint32_t* order_out) {
    if ((ntasks && (!tasks || !order_out))) return CHGPU_EINVAL;
    std::vector<uint32_t> order;
    order_for_reuse(tasks, ntasks, block_slots ? block_slots : 3u, order);
    std::copy(order.begin(), order.end(), order_out);
    return CHGPU_OK;
}

chgpu_status chgpu_shard_tasks(const chgpu_plan_task* tasks, const uint32_t* order, uint32_t ntasks, uint32_t shards,
                               uint32_t* first_out) {
    if ((ntasks && !tasks) || !first_out || shards == 0) return CHGPU_EINVAL;
    for (uint32_t k = 0; order && k < ntasks; ++k)
        if (order[k] >= ntasks) return CHGPU_EINVAL;
    std::vector<uint32_t> first;
    shard_sequence(tasks, order, ntasks, shards, first);
    std::copy(first.begin(), first.end(), first_out);
    return CHGPU_OK;
}

chgpu_status chgpu_shard_tasks_weighted(const chgpu_plan_task* tasks, const uint32_t* order, uint32_t ntasks,
                                        const uint64_t* task_weights, uint32_t shards, uint32_t* first_out) {
    if ((ntasks && (!tasks || !task_weights)) || !first_out || shards == 0) return CHGPU_EINVAL;
    for (uint32_t k = 0; order && k < ntasks; ++k)
        if (order[k] >= ntasks) return CHGPU_EINVAL;
    std::vector<uint32_t> first;
    shard_sequence(tasks, order, ntasks, shards, first, task_weights);
    std::copy(first.begin(), first.end(), first_out);
    return CHGPU_OK;
}

chgpu_status chgpu_task_weights(const chgpu_plan_task* tasks, uint32_t ntasks, const uint32_t* pairs, uint64_t npairs,
                                const uint32_t* points_per_image, uint32_t image_count, uint64_t* task_weights_out) {
    if ((ntasks && (!tasks || !task_weights_out)) || (npairs && !pairs) || !points_per_image) return CHGPU_EINVAL;
    for (uint32_t t = 0; t < ntasks; ++t) {
        if (tasks[t].first_pair + tasks[t].npairs > npairs) return CHGPU_EINVAL;
        uint64_t w = 0;
        for (uint64_t k = tasks[t].first_pair; k < tasks[t].first_pair + tasks[t].npairs; ++k) {
            const uint32_t a = pairs[2 * k], b = pairs[2 * k + 1];
            if (a >= image_count || b >= image_count) return CHGPU_EINVAL;
            w += chgpu_pair_weight(points_per_image[a], points_per_image[b]);
        }
        task_weights_out[t] = w;
    }
    return CHGPU_OK;
}

void chgpu_auto_partition_sizing(uint64_t mean_image_bytes, uint64_t memory_budget_bytes, uint32_t* block_images,
                                 uint32_t* blocks_per_group) {
    const uint64_t per_image = std::max<uint64_t>(1, mean_image_bytes);
    const uint64_t device = memory_budget_bytes / 4;
    const uint32_t bi = uint32_t(std::max<uint64_t>(1, device / per_image / 3));
    const uint64_t block_bytes = std::max<uint64_t>(1, uint64_t(bi) * per_image);
    if (block_images) *block_images = bi;
    if (blocks_per_group) *blocks_per_group = uint32_t(std::max<uint64_t>(1, memory_budget_bytes / block_bytes / 3));
}

void chgpu_partition_sizing_for_device(uint64_t device_image_bytes, uint64_t file_image_bytes, uint64_t device_bytes,
                                       uint64_t host_bytes, uint32_t block_slots, uint32_t group_slots,
                                       uint32_t* block_images, uint32_t* blocks_per_group) {
    const uint64_t dev_img = std::max<uint64_t>(1, device_image_bytes), file_img = std::max<uint64_t>(1, file_image_bytes);
    const uint64_t bs = std::max<uint32_t>(1, block_slots), gs = std::max<uint32_t>(1, group_slots);
    const uint64_t bi = std::min<uint64_t>(std::max<uint64_t>(1, device_bytes / bs / dev_img), UINT32_MAX);
    const uint64_t group_images = std::max<uint64_t>(bi, host_bytes / gs / file_img);
    if (block_images) *block_images = uint32_t(bi);
    if (blocks_per_group) *blocks_per_group = uint32_t(std::min<uint64_t>(std::max<uint64_t>(1, group_images / bi), UINT32_MAX));
}

chgpu_status chgpu_match_plan_streamed(chgpu_ctx* ctx, const char* const* paths, uint32_t image_count,
                                       uint32_t block_images, uint32_t blocks_per_group, uint32_t group_slots,
                                       uint32_t block_slots, chgpu_task_order task_order, uint32_t shard, uint32_t shards,
                                       const uint32_t* accepted,
                                       uint64_t accepted_count, const chgpu_match_cfg* cfg, uint32_t io_threads,
                                       chgpu_plan_sink_fn sink, void* user,
                                       chgpu_file_result* file_results, chgpu_streamed_stats* stats) {
    if (!ctx || !paths || !cfg || image_count == 0 || block_images == 0 || blocks_per_group == 0) return CHGPU_EINVAL;
    if (accepted_count && !accepted) return CHGPU_EINVAL;
    const auto wall0 = std::chrono::steady_clock::now();
    Replay rp{};
    rp.ctx = ctx;
    rp.paths = paths;
    rp.part = Partition{image_count, block_images, blocks_per_group, (image_count + block_images - 1) / block_images};
    rp.io_threads = io_threads;
    rp.centering_only = false;
    if (cfg->reduce_rounds < 0 || cfg->reduce_rounds > 7) return CHGPU_EINVAL;  // hashing.hpp:28-29
    rp.reduce_rounds = cfg->reduce_rounds;
    rp.results.assign(image_count, chgpu_file_result{});
    rp.ok.assign(image_count, 0);
    rp.block_resident.assign(rp.part.nblocks, 0);
    const Partition& p = rp.part;

    const bool guided = accepted != nullptr || accepted_count != 0;
    Keyed keyed;
    if (guided)
        if (const chgpu_status s = key_accepted(p, accepted, accepted_count, keyed)) return s;
    std::vector<chgpu_plan_task> tasks;
    build_tasks(p, guided ? &keyed : nullptr, tasks);
    // plan index of every task of the run, in the order it is executed
    std::vector<uint32_t> plan_index(tasks.size());
    for (uint32_t t = 0; t < tasks.size(); ++t) plan_index[t] = t;
    if (task_order == CHGPU_ORDER_REUSE) {
        order_for_reuse(tasks.data(), uint32_t(tasks.size()), block_slots ? block_slots : 3u, plan_index);
        std::vector<chgpu_plan_task> permuted(tasks.size());
        for (uint32_t k = 0; k < tasks.size(); ++k) permuted[k] = tasks[plan_index[k]];
        tasks.swap(permuted);
    } else if (task_order != CHGPU_ORDER_REFERENCE) {
        return CHGPU_EINVAL;
    }
    if (shards > 1) {  // this worker's contiguous range of the executed sequence
        if (shard >= shards) return CHGPU_EINVAL;
        std::vector<uint32_t> first;
        shard_sequence(tasks.data(), nullptr, uint32_t(tasks.size()), shards, first);
        tasks.assign(tasks.begin() + first[shard], tasks.begin() + first[shard + 1]);
        plan_index.assign(plan_index.begin() + first[shard], plan_index.begin() + first[shard + 1]);
    }

    Machine m;
    m.init(tasks.data(), uint32_t(tasks.size()), group_slots ? group_slots : 3u, block_slots ? block_slots : 3u);

    chgpu_status rc = CHGPU_OK;
    std::vector<uint32_t> pairs;
    chgpu_residency_action act;
    const char* no_overlap = std::getenv("CHGPU_STREAM_NO_OVERLAP");  // A/B switch: replay strictly in trace order
    const bool overlap = !(no_overlap && no_overlap[0] == '1');
    std::vector<uint32_t> pending;  // prefetched blocks whose load waits for the next Begin
    while (rc == CHGPU_OK && m.step(act)) {
        if (act.kind == CHGPU_ACT_LOAD) {
            if (act.level == CHGPU_LEVEL_GROUP) rp.group_hint(act.id, true);
            else if (overlap && act.prefetch) pending.push_back(act.id);  // for a later task: behind the next match call
            else {
                rc = rp.end_background();  // (one load at a time per context)
                if (rc == CHGPU_OK) rc = rp.load_block(act.id);
            }
        } else if (act.kind == CHGPU_ACT_EVICT) {
            if (act.level == CHGPU_LEVEL_GROUP) rp.group_hint(act.id, false);
            else if (std::find(pending.begin(), pending.end(), act.id) != pending.end()) {
                pending.erase(std::find(pending.begin(), pending.end(), act.id));  // evicted before it was ever loaded
            } else {
                if (std::find(rp.background.begin(), rp.background.end(), act.id) != rp.background.end()) rc = rp.end_background();
                rp.evict_block(act.id, true);
            }
        } else if (act.kind == CHGPU_ACT_BEGIN) {
            const chgpu_plan_task& t = tasks[act.id];
            ++rp.st.tasks;
            // Line 2 of the exchange: the prefetches the schedule issued since the last task (their evictions are done, their
            // loads were held back) are opened as one background load that this task's match call moves forward; the
            // reference's loader thread does the same while its workers run the task (engine.cpp:414-442, :679-696).
            // The open load stays open across tasks that do not need its blocks (a short task hides little; the next
            // long one hides the rest) and is completed when a task needs one of them or the next load has to start.
            const bool needs_open = std::find(rp.background.begin(), rp.background.end(), t.block_a) != rp.background.end() ||
                                    std::find(rp.background.begin(), rp.background.end(), t.block_b) != rp.background.end();
            if (needs_open || !pending.empty()) {
                rc = rp.end_background();
                if (rc != CHGPU_OK) break;
            }
            if (!pending.empty()) {
                rc = rp.begin_background(pending);
                pending.clear();
                if (rc != CHGPU_OK) break;
            }
            // the task's pairs in plan order (scheduler.cpp:47-75), images that failed to load left out
            pairs.clear();
            uint64_t skipped = 0;
            auto emit = [&](uint32_t a, uint32_t b) {
                if (rp.ok[a] && rp.ok[b]) {
                    pairs.push_back(a);
                    pairs.push_back(b);
                } else {
                    ++skipped;
                }
            };
            auto flush = [&](bool final) {
                const uint64_t np = pairs.size() / 2;
                if (np == 0 || (!final && np < kPairsPerCall)) return;
                SinkAdapter ad{sink, user, plan_index[act.id], pairs.data(), 0};
                chgpu_match_stats ms{};
                const auto t0 = std::chrono::steady_clock::now();
                rc = chgpu_match_pairs_stream(ctx, pairs.data(), uint32_t(np), cfg, sink_adapter, &ad, &ms);
                rp.st.match_seconds += seconds_since(t0);
                rp.st.pairs += np;
                rp.st.matches += ad.matches;
                pairs.clear();
            };
            if (guided) {
                const auto r = bucket_of(keyed, uint64_t(t.block_a) * p.nblocks + t.block_b);
                for (auto it = r.first; it != r.second && rc == CHGPU_OK; ++it) {
                    emit(uint32_t(it->second / p.images), uint32_t(it->second % p.images));
                    flush(false);
                }
            } else if (t.block_a != t.block_b) {
                for (uint32_t a = p.lo(t.block_a); a < p.hi(t.block_a) && rc == CHGPU_OK; ++a) {
                    for (uint32_t b = p.lo(t.block_b); b < p.hi(t.block_b); ++b) emit(a, b);
                    flush(false);
                }
            } else {
                for (uint32_t a = p.lo(t.block_a); a < p.hi(t.block_a) && rc == CHGPU_OK; ++a) {
                    for (uint32_t b = a + 1; b < p.hi(t.block_a); ++b) emit(a, b);
                    flush(false);
                }
            }
            if (rc == CHGPU_OK) flush(true);
            rp.st.pairs_skipped += skipped;
        }
    }
    {
        const chgpu_status e = rp.end_background();
        if (rc == CHGPU_OK) rc = e;
    }
    chgpu_load_chft_files_end(ctx, nullptr, nullptr);  // an error path may have left the background load open
    if (rc == CHGPU_OK && m.blocked) rc = CHGPU_EINVAL;  // slot limits below what one task needs
    rp.evict_all();
    rp.join_hints();
    rp.st.wall_seconds = seconds_since(wall0);
    if (file_results) std::copy(rp.results.begin(), rp.results.end(), file_results);
    if (stats) *stats = rp.st;
    return rc;
}

chgpu_status chgpu_centering_pass_files(chgpu_ctx* ctx, const char* const* paths, uint32_t image_count,
                                        uint32_t block_images, uint32_t io_threads, chgpu_file_result* file_results,
                                        double* centering128_out) {
    if (!ctx || !paths || image_count == 0 || block_images == 0) return CHGPU_EINVAL;
    Replay rp{};
    rp.ctx = ctx;
    rp.paths = paths;
    rp.part = Partition{image_count, block_images, 1u, (image_count + block_images - 1) / block_images};
    rp.io_threads = io_threads;
    rp.centering_only = true;
    rp.results.assign(image_count, chgpu_file_result{});
    rp.ok.assign(image_count, 0);
    rp.block_resident.assign(rp.part.nblocks, 0);
    if (const chgpu_status s = chgpu_centering_reset(ctx)) return s;
    // the reference's 2-slot hashing schedule (hashing_residency_tasks, scheduler.cpp:194-200) over the blocks
    std::vector<chgpu_plan_task> tasks(rp.part.nblocks);
    uint32_t nt = 0;
    chgpu_hashing_tasks(image_count, block_images, 1u, tasks.data(), &nt);
    Machine m;
    m.init(tasks.data(), nt, 2u, 2u);
    chgpu_status rc = CHGPU_OK;
    chgpu_residency_action act;
    while (rc == CHGPU_OK && m.step(act)) {
        if (act.level != CHGPU_LEVEL_BLOCK) continue;
        if (act.kind == CHGPU_ACT_LOAD) rc = rp.load_block(act.id);
        else if (act.kind == CHGPU_ACT_EVICT) rp.evict_block(act.id, true);
    }
    rp.evict_all();
    rp.join_hints();
    if (file_results) std::copy(rp.results.begin(), rp.results.end(), file_results);
    if (rc != CHGPU_OK) return rc;
    return chgpu_centering_apply(ctx, centering128_out);  // CHGPU_EINVAL when no descriptor was seen (hashing.cpp:60)
}

}  // extern "C"
