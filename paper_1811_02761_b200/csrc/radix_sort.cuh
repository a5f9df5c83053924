// CUB-free stable LSD radix sort of (key, u32 payload) pairs for sm_100a.
//
// Replaces std::sort of (key, index) pairs in build_tree (octree.cpp:60-63):
// a stable LSD sort from the identity order equals the lexicographic
// (key, index) pair sort, so keys/perm are bit-identical to the reference.
//
// Default (G2_ONESWEEP): one kernel reads the keys once for the global
// histograms of every 8-bit digit; each pass is then ONE kernel: 2048-key
// tiles claimed in order rank their keys in shared memory (warp-striped loads,
// __match_any_sync ranking => stable), stage the ranked tile in shared memory,
// publish per-digit tile counts and look back over 8 predecessor tiles per step
// (decoupled look-back per digit) for their global offsets, then write
// digit-contiguous runs.  The alternative is a count kernel, one look-back scan
// over the (digit, tile) matrix and a scatter kernel per pass.  Traffic per
// pass: read key+value and write key+value (24 B per pair for 64-bit keys).
#pragma once

#include "common.cuh"

namespace g2 {

struct SortScratch {
    DBuf<uint32_t> hist;    // 256 x tiles digit-count / offset matrix
    DBuf<uint32_t> status;  // scan look-back words + tile counter
    size_t tiles_cap = 0;
};

// Sorts keys[0,n) (bits [0, key_bits)) carrying vals (identity => the input
// payload is 0..n-1 and `vals` is not read).  Ping-pongs between
// (keys, vals) and (keys_alt, vals_alt), all four valid buffers of n
// elements; returns true if the result ended in the *_alt buffers.
template <typename K>
bool radix_sort_pairs(K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, size_t n, int key_bits,
                      bool identity, SortScratch& scratch, cudaStream_t stream);

}  // namespace g2
