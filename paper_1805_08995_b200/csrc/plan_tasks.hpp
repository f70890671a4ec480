// plan_tasks.hpp — traversal of the block-pair tasks of the reference's pair plan, shared by the pair-list
// entry points (host_util.cpp) and the residency schedule / out-of-core driver (residency.cpp).  Host only.
#pragma once

#include <algorithm>
#include <cstdint>
#include <utility>
#include <vector>

namespace chgpu {

// Exhaustive plan in the reference's locality order (scheduler.cpp:99-142).  Blocks of
// `block_images` consecutive images, groups of `blocks_per_group` consecutive blocks.  For
// every anchor group: boustrophedon sweeps of (anchor block, partner block) against each
// later group, then the anchor group's own block pairs as a chain that starts at the block
// the sweep stopped on, then the pairs inside each block.
// The block-pair tasks of the exhaustive plan in plan order: cross(ba, bb) with ba < bb for two different blocks,
// self(blk) for the pairs inside one block.
template <class Cross, class Self>
void for_each_plan_task(uint32_t image_count, uint32_t block_images, uint32_t blocks_per_group, Cross&& cross_task, Self&& self_task) {
    const uint32_t nblocks = (image_count + block_images - 1) / block_images;
    const uint32_t ngroups = (nblocks + blocks_per_group - 1) / blocks_per_group;
    auto cross = [&](uint32_t ba, uint32_t bb) {
        if (ba > bb) std::swap(ba, bb);
        cross_task(ba, bb);
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
        for (uint32_t blk = a0; blk < a0 + an; ++blk) self_task(blk);
    }
}

}  // namespace chgpu
