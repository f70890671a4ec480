// dev_types.cuh — device-side records shared by the hash-build and match kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace chgpu {

constexpr int kDim = 128;            // descriptor dimension (feature_io.hpp:14 kDescriptorDim)
constexpr int kMaxTables = 8;        // L envelope of the device path
constexpr int kMaxShortBits = 12;    // m envelope (dense 2^m+1 CSR per table)
constexpr int kMaxTopK = 32;         // ranked list lives one entry per lane
constexpr uint32_t kMaxPoints = 65536;  // bucket point ids are u16
constexpr uint32_t kNone = 0xFFFFFFFFu;

// One resident image.  All arrays live in one arena block (see Arena in chgpu.cu):
//   desc   n x 128 u8          SoA descriptors (reference Descriptor, feature_io.hpp:27)
//   kp     n x float4          keypoints (x, y, scale, orientation)
//   longs  n x uint4           128-bit ranking code, word w = bits 32w..32w+31 (LongCode, hashing.hpp:91)
//   shorts n x L u32           bucket ids [point*L + table] (ShortCodes::values, hashing.hpp:80)
//   offs   L x (2^m + 1) u32   dense CSR offsets per table (BucketIndex, matcher.hpp:30-41)
//   points L x n u16           point ids bucket-major, ascending id inside a bucket
//   scan   L x n u16           the same buckets in the order the match kernel walks them: ids dealt
//                              round-robin over (id mod 8), so that 8 consecutive entries gather their
//                              16-byte codes from 8 different shared-memory bank groups
//   scodes 2 x L x n uint4     (images the join pass handles: not tiled) the long codes in bucket order of every table,
//                              entry p of table t = point points[t*n + p]; first the codes as they are, then (L*n entries
//                              on) with the bits of every byte reversed — the train-side operand of the tensor-core
//                              Hamming pass
//   spop   L x n i16           64 x popcount of the same codes (the join pass's column penalty / row threshold)
struct DevImage {
    const uint8_t* desc;
    const float4* kp;
    uint4* longs;
    uint32_t* shorts;
    uint32_t* offs;
    uint16_t* points;
    uint16_t* scan;
    uint4* scodes;   // nullptr: no bucket-sorted copies (tiled images, tiles)
    int16_t* spop;
    uint32_t n;
    uint32_t flags;  // bit0: codes + buckets valid
};

struct PairDesc {
    uint32_t slot_i;     // query image
    uint32_t slot_j;     // train image, or one id-range tile of a large train image (see match_kernels.cuh)
    uint64_t res_off;    // first entry of this pair in the per-query result scratch
    uint32_t tile_base;  // tiles: first point id of the tile inside its image
    uint32_t tile_idx;   // tiles: position of the tile's list in the per-query list scratch
    uint32_t pair_idx;   // position of the (whole-image) pair in its sub-batch: per-pair inputs such as fmats
    uint32_t act_off;    // tiles: first entry of this (query image, tile) pair in the active-query scratch
};

struct DevStats {
    unsigned long long raw_candidates;
    unsigned long long verified_queries;
    unsigned long long distances;
    unsigned long long matches;
    unsigned long long checksum;
};

}  // namespace chgpu
