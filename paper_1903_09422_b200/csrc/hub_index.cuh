// hub_index.cuh — layout of the search trees over high-degree adjacency rows
// (built by hub_index.cu, read by the block sampler's hub searches).
//
// A hub search asks for the position of a vertex v in the ascending adjacency
// row A[0, d) of a high-degree vertex (probe passes, backtrack steps by level
// list). A plain binary search is ~log2(d) DEPENDENT loads spread over the
// whole row (17 for a 10^5-entry hub, most of them HBM misses on C5). The
// tree puts one key per 32-entry block of the row (the block's last entry)
// in level 0 and one key per 8 keys of the level below in every level above,
// each level contiguous and padded with 0xFFFFFFFF to whole 8-key nodes
// (32 bytes = one sector = two 16-byte loads). A search reads one node per
// level -- ceil(log8(d / 32)) dependent sector loads, the upper ones shared by
// every search of that hub and therefore cache-resident -- and finishes inside
// one 128-byte block of the row. Size: ~3.6% of the rows it covers.
//
// Tree of a row (u32 words, 32-byte aligned):
//   [0]      T  = index of the top level (levels 0..T, T <= 5)
//   [1..6]   word offset of level k's keys from the tree base (k = 0..5)
//   [7]      A[d-1], the row's largest entry
//   [8..]    level 0 keys, then level 1, ... each padded to a multiple of 8
#pragma once

#include <cstdint>

namespace adsb {

constexpr uint32_t kHubTreeMinDeg = 128;          // rows below this are searched directly
constexpr uint32_t kHubLeaf = 32, kHubFan = 8, kHubMaxLevels = 6;
constexpr uint32_t kHubTreeMaxDeg = kHubLeaf * 262144u;  // 8^6 leaf blocks

__host__ __device__ inline bool hub_has_tree(uint32_t d) { return d >= kHubTreeMinDeg && d <= kHubTreeMaxDeg; }

// words of the tree of a row of d entries (0: no tree)
__host__ __device__ inline uint32_t hub_tree_words(uint32_t d) {
    if (!hub_has_tree(d)) return 0;
    uint32_t nk = (d + kHubLeaf - 1) / kHubLeaf, words = 8;
    for (;;) {
        words += (nk + 7u) & ~7u;
        if (nk <= kHubFan) break;
        nk = (nk + kHubFan - 1) / kHubFan;
    }
    return words;
}

}  // namespace adsb
