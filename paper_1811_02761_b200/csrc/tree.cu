// makeTree and calcNode on sm_100a: bounding cube, Morton keys, level-by-level
// split, deepest-first node attributes.  All FP64 arithmetic uses explicit
// round-to-nearest intrinsics in the reference's operation order, so the
// cube, keys, cells and node attributes are bit-identical to
// gravitree's build_tree / calc_node (octree.cpp:24-162, morton.hpp:14-49).
#include <cstdlib>

#include "morton.cuh"

namespace g2 {
namespace {

constexpr int kBlock = 256;
#ifndef G2_CALC_LEAF_CELLS
#define G2_CALC_LEAF_CELLS 1  // leaves in cell order (1) or warp-synchronous particle chunks (0): 4.55 vs 4.58 ms paper step
#endif
#ifndef G2_CALC_FUSED
#define G2_CALC_FUSED 0  // 1: internal levels in one dependency-ordered launch (measured: 0.342 vs 0.337 ms per calc)
#endif
#ifndef G2_CALC_GROUP8
#define G2_CALC_GROUP8 0  // 8 lanes per internal cell (A/B): 170 vs 146 us per calc at 2^23
#endif
#ifndef G2_CALC_MINB
#define G2_CALC_MINB 2  // 2 blocks of 256 per SM: 128 registers, no spills (1: more registers, 25 % slower)
#endif

// ---- bounding_cube (octree.cpp:24-49) ---------------------------------------
__global__ void __launch_bounds__(kBlock) bbox_partial_kernel(const double4* __restrict__ xyzm, size_t n,
                                                               double* __restrict__ partials, DevFlags* flags) {
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    bool bad = false;
    for (size_t i = blockIdx.x * size_t(kBlock) + threadIdx.x; i < n; i += size_t(gridDim.x) * kBlock) {
        const double4 p = xyzm[i];
        bad |= !(isfinite(p.x) && isfinite(p.y) && isfinite(p.z));
        lo[0] = smin(lo[0], p.x), lo[1] = smin(lo[1], p.y), lo[2] = smin(lo[2], p.z);
        hi[0] = smax(hi[0], p.x), hi[1] = smax(hi[1], p.y), hi[2] = smax(hi[2], p.z);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) flags->data_error = 1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            lo[a] = smin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
            hi[a] = smax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
        }
    __shared__ double sh[kBlock / 32][6];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0)
        for (int a = 0; a < 3; ++a) sh[w][a] = lo[a], sh[w][3 + a] = hi[a];
    __syncthreads();
    if (threadIdx.x < 6) {
        double v = sh[0][threadIdx.x];
        for (int k = 1; k < kBlock / 32; ++k)
            v = threadIdx.x < 3 ? smin(v, sh[k][threadIdx.x]) : smax(v, sh[k][threadIdx.x]);
        partials[blockIdx.x * 6 + threadIdx.x] = v;
    }
}

constexpr int kBboxFinalThreads = 1024;
__global__ void __launch_bounds__(kBboxFinalThreads) bbox_final_kernel(const double* __restrict__ partials, int nb,
                                                                       Cube* cube) {
    G2_PDL_WAIT();  // programmatic dependent launch (launch_pdl)
    // one block: min/max are exact in any order
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int b = threadIdx.x; b < nb; b += kBboxFinalThreads)
        for (int a = 0; a < 3; ++a) {
            lo[a] = smin(lo[a], partials[6 * b + a]);
            hi[a] = smax(hi[a], partials[6 * b + 3 + a]);
        }
    __shared__ double sh[kBboxFinalThreads / 32][6];
    for (int round = 0; round < 2; ++round) {  // warps, then the warp partials
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
            for (int a = 0; a < 3; ++a) {
                lo[a] = smin(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
                hi[a] = smax(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
            }
        if (round == 1) break;
        if (lane == 0)
            for (int a = 0; a < 3; ++a) sh[w][a] = lo[a], sh[w][3 + a] = hi[a];
        __syncthreads();
        if (w != 0) return;
        for (int a = 0; a < 3; ++a) lo[a] = sh[lane][a], hi[a] = sh[lane][3 + a];
    }
    if (lane != 0) return;
    double c[3];
    for (int a = 0; a < 3; ++a) c[a] = dmul(dadd(lo[a], hi[a]), 0.5);  // 0.5 * (lo + hi)
    const double d[6] = {dsub(lo[0], c[0]), dsub(hi[0], c[0]), dsub(lo[1], c[1]),
                         dsub(hi[1], c[1]), dsub(lo[2], c[2]), dsub(hi[2], c[2])};
    double h = 0.0;
    for (int k = 0; k < 6; ++k) h = smax(h, fabs(d[k]));
    double half = dmul(h, 1.0 + 1e-12);
    if (half == 0.0) half = 1.0;  // all particles coincident
    *cube = Cube{c[0], c[1], c[2], half};
}

// ---- morton_key (morton.hpp:14-44) --------------------------------------------
__global__ void __launch_bounds__(kBlock) keys_kernel(const double4* __restrict__ xyzm,
                                                      const uint32_t* __restrict__ id_of_pos, size_t n,
                                                      const Cube* __restrict__ cube, uint64_t* __restrict__ key_by_id,
                                                      DevFlags* flags) {
    __shared__ SpreadTable st;
    spread_init(st);
    const KeyFrame f(*cube);
    __syncthreads();
    for (size_t i = blockIdx.x * size_t(kBlock) + threadIdx.x; i < n; i += size_t(gridDim.x) * kBlock) {
        const double4 p = xyzm[i];
        if (!f.inside(p)) flags->data_error = 2;
        key_by_id[id_of_pos ? id_of_pos[i] : i] = f.key(p, st);
    }
}

// ---- level-by-level split (octree.cpp:74-102) ------------------------------------
// One launch per depth d, one thread per cell, 256 cells per tile.  A cell is
// split iff count > leaf_cap and d < 21; its children are the non-empty runs
// of the depth-d digit among its (sorted) keys, exactly the reference's
// upper_bound per digit: small cells count digits with one linear pass over
// their keys, large cells binary-search the 8 run ends.  Children of level d
// are appended as level d+1 in (parent, digit) order, which is the
// reference's BFS order; their offsets come from a decoupled look-back scan.
constexpr uint32_t kLinearMax = 128;  // per-digit counts fit the packed 8-bit fields

__device__ __forceinline__ unsigned digit_at(uint64_t key, int depth) {
    return unsigned(key >> (3 * (kMortonBits - 1 - depth))) & 7u;
}

// Warp-granular tiles (32 cells, no block barriers): each warp pulls tiles and
// chains its child offsets through the warp-parallel look-back.
__global__ void __launch_bounds__(kBlock) split_level_kernel(SplitArgs a, int d) {
    const uint32_t lvl_begin = a.level_start[d], lvl_end = a.level_start[d + 1];
    const uint32_t ncell = lvl_end - lvl_begin;
    const uint32_t ntiles = (ncell + 31) / 32;
    if (lvl_end > a.cell_cap || ncell == 0) {  // overflow (host grows and rebuilds) or empty level
        if (blockIdx.x == 0 && threadIdx.x == 0) a.level_start[d + 2] = lvl_end;
        return;
    }
    const int lane = threadIdx.x & 31;
    const int shift = 3 * (kMortonBits - 1 - d);
    uint64_t* status = a.status + (lvl_begin / 32 + d);  // disjoint slice per level
    while (true) {
        uint32_t tile = 0;
        if (lane == 0) tile = atomicAdd(&a.tile_counters[d], 1u);
        tile = __shfl_sync(0xffffffffu, tile, 0);
        if (tile >= ntiles) break;
        const uint32_t cell = lvl_begin + tile * 32 + lane;
        const bool in_range = cell < lvl_end;
        uint32_t first = 0, cnt = 0;
        if (in_range) first = a.first[cell], cnt = a.count[cell];
        const bool split = in_range && cnt > a.leaf_cap && d < kMaxDepth;
        uint32_t ub[8];  // end of each digit run
        if (split && cnt <= kLinearMax) {
            // one pass over the cell's keys, 8 independent loads in flight per chunk
            uint64_t packed = 0;  // 8-bit count per digit
            const uint32_t end = first + cnt;
            for (uint32_t k0 = first; k0 < end; k0 += 8) {
                uint64_t kk[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) kk[j] = k0 + j < end ? a.keys[k0 + j] : 0ull;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (k0 + j < end) packed += 1ull << (8 * ((kk[j] >> shift) & 7u));
            }
            uint32_t run = first;
#pragma unroll
            for (int v = 0; v < 8; ++v) ub[v] = (run += uint32_t(packed >> (8 * v)) & 0xffu);
        } else if (split) {
            // the 8 upper_bound searches advance in lockstep: 8 loads in flight per step
            uint32_t lo[8], hi[8];
#pragma unroll
            for (int v = 0; v < 8; ++v) lo[v] = first, hi[v] = first + cnt;
            bool busy = true;
            while (busy) {
                busy = false;
                uint64_t kk[8];
#pragma unroll
                for (int v = 0; v < 8; ++v) kk[v] = lo[v] < hi[v] ? a.keys[lo[v] + (hi[v] - lo[v]) / 2] : 0ull;
#pragma unroll
                for (int v = 0; v < 8; ++v) {
                    if (lo[v] < hi[v]) {
                        const uint32_t mid = lo[v] + (hi[v] - lo[v]) / 2;
                        if (unsigned(v) < unsigned((kk[v] >> shift) & 7u))
                            hi[v] = mid;
                        else
                            lo[v] = mid + 1;
                        busy |= lo[v] < hi[v];
                    }
                }
            }
#pragma unroll
            for (int v = 0; v < 8; ++v) ub[v] = lo[v];
        } else {
#pragma unroll
            for (int v = 0; v < 8; ++v) ub[v] = first;
        }
        uint32_t nc = 0;
#pragma unroll
        for (int v = 0; v < 8; ++v) nc += ub[v] > (v ? ub[v - 1] : first) ? 1u : 0u;
        // exclusive scan of child counts over the warp's tile, then the look-back
        uint32_t inc = nc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
        const uint32_t excl = uint32_t(lookback_warp(status, tile, tot));
        const uint32_t base = lvl_end + excl + inc - nc;  // first child index
        if (split) {
            uint32_t j = 0, lo = first;
#pragma unroll
            for (int v = 0; v < 8; ++v) {
                if (ub[v] > lo) {
                    const uint32_t idx = base + j++;
                    if (idx < a.cell_cap) {
                        a.first_child[idx] = 0;
                        a.child_count[idx] = 0;
                        a.first[idx] = lo;
                        a.count[idx] = ub[v] - lo;
                        a.depth[idx] = uint8_t(d + 1);
                    } else {
                        a.flags->cell_overflow = 1;
                    }
                }
                lo = ub[v];
            }
        }
        if (in_range) {
            a.first_child[cell] = split ? base : 0u;
            a.child_count[cell] = split ? nc : 0u;
        }
        if (tile == ntiles - 1 && lane == 0) a.level_start[d + 2] = lvl_end + excl + tot;
    }
}

// ---- non-recursive split (leaf_cap <= kSplitMaxCap) --------------------------------
// With L_i = number of leading Morton digits shared by sorted keys i-1 and i
// (L_0 = L_n = -1), a depth-d cell exists at position i iff a depth-d digit run
// starts there (i = 0 or L_i < d) and the enclosing depth-(d-1) run holds more
// than leaf_cap particles (its parent is split; all ancestors are larger).  Per
// position the existing depths form one interval [lo_i, hi_i], decided from L
// in a window of +-leaf_cap around i.  BFS order (depth, first) then follows
// from per-depth ranks, so the whole level-by-level recursion of
// octree.cpp:74-102 becomes four launches: count, scan, write, child counts.
constexpr int kSplitThreads = 256;
constexpr int kSplitItems = 4;                              // particles per thread
constexpr int kSplitTile = kSplitThreads * kSplitItems;     // particles per block
constexpr int kSplitChunks = kSplitTile / 32;                // warp-sized chunks per tile, (item, warp) order
constexpr uint32_t kSplitMaxCap = 32;

__device__ __forceinline__ int lcp_digits(uint64_t a, uint64_t b) {
    const uint64_t x = a ^ b;
    if (!x) return kMortonBits;
    return (62 - (63 - __clzll(static_cast<long long>(x)))) / 3;  // keys use bits 0..62
}

struct SplitWindow {
    uint64_t key[kSplitTile + 2 * kSplitMaxCap + 2];
    int8_t L[kSplitTile + 2 * kSplitMaxCap + 1];
    int8_t M[kSplitTile + kSplitMaxCap];  // M_j = min L over (j, j + lc], positions base - lc .. base + T - 1
};

// Loads the tile's key window and L values; then (lo, hi) of particle base + t (t = tile offset):
// lo > hi means no cell starts there.
__device__ __forceinline__ void split_window(const uint64_t* __restrict__ keys, uint32_t n, uint32_t lc,
                                             uint32_t base, SplitWindow& w) {
    const int64_t kb = int64_t(base) - int64_t(lc) - 1;  // key window [kb, base + T + lc]
    const int nk = kSplitTile + 2 * int(lc) + 2;
    for (int t = threadIdx.x; t < nk; t += kSplitThreads) {
        const int64_t j = kb + t;
        w.key[t] = (j >= 0 && j < int64_t(n)) ? keys[j] : 0ull;
    }
    __syncthreads();
    const int64_t lb = int64_t(base) - int64_t(lc);  // L window [lb, base + T + lc]
    for (int t = threadIdx.x; t < nk - 1; t += kSplitThreads) {
        const int64_t j = lb + t;
        w.L[t] = (j <= 0 || j >= int64_t(n)) ? int8_t(-1) : int8_t(lcp_digits(w.key[t], w.key[t + 1]));
    }
    __syncthreads();
    // sliding minimum: the run through position j has more than lc particles ahead of j iff M_j >= depth
    for (int t = threadIdx.x; t < kSplitTile + int(lc); t += kSplitThreads) {
        int m = 127;
        for (int q = 1; q <= int(lc); ++q) m = min(m, int(w.L[t + q]));
        w.M[t] = int8_t(m);
    }
    __syncthreads();
}

// The window holds L = -1 outside [1, n), so runs end at the array ends without extra tests.
// The depth-L_i run through i holds more than lc particles iff some lc+1 consecutive positions
// containing i lie in it, i.e. iff max_{j in [i-lc, i]} M_j >= L_i (fixed-length loops, no
// divergence).
__device__ __forceinline__ void split_range(uint32_t n, uint32_t lc, uint32_t base, int t, const SplitWindow& w,
                                            int& lo, int& hi) {
    const uint32_t i = base + uint32_t(t);
    lo = kMaxDepth + 1, hi = kMaxDepth;
    if (i >= n) return;
    const int M = w.M[t + int(lc)];  // M_i
    if (i == 0) {
        lo = 0, hi = min(kMaxDepth, M + 1);
        return;
    }
    const int li = w.L[t + int(lc)];
    if (li >= kMortonBits) return;  // identical keys: no cell starts here
    int W = -1;
    for (int q = 0; q <= int(lc); ++q) W = max(W, int(w.M[t + q]));
    lo = li + 1;
    hi = W >= li ? min(kMaxDepth, max(li + 1, M + 1)) : li;
}

// per-depth counts of the tile's (item, warp) chunks -> chunk-exclusive prefixes in wcnt, tile totals returned
__device__ __forceinline__ void split_chunk_counts(const int* lo, const int* hi, uint32_t (*wcnt)[kSplitChunks]) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < kSplitItems; ++k) {
        // only the depths some lane of this chunk has (warp-uniform bounds)
        const int dmin = __reduce_min_sync(0xffffffffu, lo[k]);
        const int dmax = __reduce_max_sync(0xffffffffu, hi[k]);
        if (lane <= kMaxDepth && (lane < dmin || lane > dmax)) wcnt[lane][k * (kSplitThreads / 32) + wid] = 0;
        for (int d = dmin; d <= dmax; ++d) {
            const unsigned m = __ballot_sync(0xffffffffu, lo[k] <= d && d <= hi[k]);
            if (lane == 0) wcnt[d][k * (kSplitThreads / 32) + wid] = __popc(m);
        }
    }
    __syncthreads();
}

// per tile: the (depth, chunk) counts as bytes (<= 32 each), kept for the write pass
constexpr int kChunkCountWords = ((kMaxDepth + 1) * kSplitChunks + 3) / 4;
__global__ void __launch_bounds__(kSplitThreads) split_count_kernel(const uint64_t* __restrict__ keys, uint32_t n,
                                                                    uint32_t lc, uint32_t* __restrict__ tile_counts,
                                                                    uint32_t ntiles, uint16_t* __restrict__ lohi,
                                                                    uint32_t* __restrict__ chunk_counts) {
    __shared__ SplitWindow w;
    __shared__ uint32_t wcnt[kMaxDepth + 1][kSplitChunks];
    const uint32_t base = blockIdx.x * kSplitTile;
    split_window(keys, n, lc, base, w);
    int lo[kSplitItems], hi[kSplitItems];
#pragma unroll
    for (int k = 0; k < kSplitItems; ++k) {
        split_range(n, lc, base, k * kSplitThreads + threadIdx.x, w, lo[k], hi[k]);
        const uint32_t i = base + k * kSplitThreads + threadIdx.x;
        if (i < n) lohi[i] = uint16_t(lo[k] | (hi[k] << 8));  // the write pass reuses the ranges
    }
    split_chunk_counts(lo, hi, wcnt);
    if (threadIdx.x <= kMaxDepth) {
        uint32_t c = 0;
        for (int q = 0; q < kSplitChunks; ++q) c += wcnt[threadIdx.x][q];
        tile_counts[size_t(threadIdx.x) * ntiles + blockIdx.x] = c;
    }
    static_assert(kSplitChunks % 4 == 0, "4 chunk counts per word");
    for (int t = threadIdx.x; t < kChunkCountWords; t += kSplitThreads) {
        const uint32_t* w = &wcnt[0][0] + 4 * t;
        chunk_counts[size_t(blockIdx.x) * kChunkCountWords + t] = w[0] | (w[1] << 8) | (w[2] << 16) | (w[3] << 24);
    }
}

// one block per depth: exclusive scan over the tiles in place, level size -> totals[d]
__global__ void __launch_bounds__(1024) split_scan_kernel(uint32_t* __restrict__ tile_counts, uint32_t ntiles,
                                                          uint32_t* __restrict__ totals) {
    G2_PDL_WAIT();  // programmatic dependent launch (launch_pdl)
    __shared__ uint32_t wsum[32];
    __shared__ uint32_t carry;
    uint32_t* row = tile_counts + size_t(blockIdx.x) * ntiles;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (uint32_t b0 = 0; b0 < ntiles; b0 += 1024) {
        const uint32_t k = b0 + threadIdx.x;
        const uint32_t x = k < ntiles ? row[k] : 0u;
        uint32_t inc = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) wsum[wid] = inc;
        __syncthreads();
        if (wid == 0) {
            const uint32_t v = wsum[lane];
            uint32_t vi = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, vi, o);
                if (lane >= o) vi += y;
            }
            wsum[lane] = vi - v;
        }
        __syncthreads();
        const uint32_t c0 = carry;
        if (k < ntiles) row[k] = c0 + wsum[wid] + inc - x;
        __syncthreads();
        if (threadIdx.x == 1023) carry = c0 + wsum[wid] + inc;
        __syncthreads();
    }
    if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

// cells in BFS order: first, depth, first_child (count and child_count follow in split_cells_kernel)
__global__ void __launch_bounds__(kSplitThreads) split_write_kernel(SplitArgs a, uint32_t n,
                                                                    const uint32_t* __restrict__ tile_offs,
                                                                    uint32_t ntiles, const uint32_t* __restrict__ totals,
                                                                    const uint16_t* __restrict__ lohi,
                                                                    const uint32_t* __restrict__ chunk_counts) {
    G2_PDL_WAIT();  // programmatic dependent launch (launch_pdl)
    __shared__ uint32_t wcnt[kMaxDepth + 1][kSplitChunks];
    __shared__ uint32_t lstart[kMaxDepth + 2];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (int d = 0; d <= kMaxDepth; ++d) lstart[d] = acc, acc += totals[d];
        lstart[kMaxDepth + 1] = acc;
    }
    const uint32_t base = blockIdx.x * kSplitTile;
    int lo[kSplitItems], hi[kSplitItems];
#pragma unroll
    for (int k = 0; k < kSplitItems; ++k) {
        const uint32_t i = base + k * kSplitThreads + threadIdx.x;
        const uint32_t v = i < n ? lohi[i] : uint32_t(kMaxDepth + 1) | (uint32_t(kMaxDepth) << 8);
        lo[k] = int(v & 0xffu), hi[k] = int(v >> 8);
    }
    for (int t = threadIdx.x; t < kChunkCountWords; t += kSplitThreads) {  // the count pass's chunk counts
        const uint32_t v = chunk_counts[size_t(blockIdx.x) * kChunkCountWords + t];
        uint32_t* w = &wcnt[0][0] + 4 * t;
        w[0] = v & 0xffu, w[1] = (v >> 8) & 0xffu, w[2] = (v >> 16) & 0xffu, w[3] = v >> 24;
    }
    __syncthreads();
    if (threadIdx.x <= kMaxDepth) {  // exclusive prefix over the tile's chunks, plus the tile offset
        uint32_t acc = lstart[threadIdx.x] + tile_offs[size_t(threadIdx.x) * ntiles + blockIdx.x];
        for (int q = 0; q < kSplitChunks; ++q) {
            const uint32_t c = wcnt[threadIdx.x][q];
            wcnt[threadIdx.x][q] = acc;
            acc += c;
        }
    }
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x <= kMaxDepth + 1) a.level_start[threadIdx.x] = lstart[threadIdx.x];
    if (blockIdx.x == 0 && threadIdx.x == kMaxDepth + 2) a.level_start[kMaxDepth + 2] = lstart[kMaxDepth + 1];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int k = 0; k < kSplitItems; ++k) {
        const uint32_t i = base + k * kSplitThreads + threadIdx.x;
        const int chunk = k * (kSplitThreads / 32) + wid;
        uint32_t child_idx = 0;
        const int dmin = __reduce_min_sync(0xffffffffu, lo[k]);
        const int dmax = __reduce_max_sync(0xffffffffu, hi[k]);
        for (int d = dmax; d >= dmin; --d) {  // deepest first: first_child is the previous index
            const bool has = lo[k] <= d && d <= hi[k];
            const unsigned m = __ballot_sync(0xffffffffu, has);
            if (!has) continue;
            const uint32_t idx = wcnt[d][chunk] + __popc(m & lt);
            if (idx < a.cell_cap) {
                a.first[idx] = i;
                a.depth[idx] = uint8_t(d);
                a.first_child[idx] = d < hi[k] ? child_idx : 0u;
            } else {
                a.flags->cell_overflow = 1;
            }
            child_idx = idx;
        }
    }
}

// first j > i whose depth-d prefix differs from key i's (upper_bound by galloping from `from`)
__device__ __forceinline__ uint32_t run_end(const uint64_t* __restrict__ keys, uint32_t n, uint32_t from, uint64_t pre,
                                            int sh) {
    uint32_t ok = from - 1, step = 1, j = from;  // keys[ok] has the prefix
    while (j < n && (keys[j] >> sh) == pre) {
        ok = j;
        j = ok + step;
        step <<= 1;
    }
    uint32_t hi = min(j, n);  // first index known (or assumed at n) not to match
    while (ok + 1 < hi) {
        const uint32_t mid = ok + (hi - ok) / 2;
        if ((keys[mid] >> sh) == pre)
            ok = mid;
        else
            hi = mid;
    }
    return ok + 1;
}

// per cell: count = end of its digit run (8 keys probed at once, then galloping), and for split
// cells the number of consecutive next-level cells starting inside it
// topology outputs of cell c (see tree_topology_kernel); every lane of the warp calls it (warp-uniform)
__device__ __forceinline__ void write_topology(uint32_t c, bool valid, uint32_t fc, uint32_t cc, uint32_t d,
                                               uint32_t f, uint32_t cnt, const uint32_t* __restrict__ level_start,
                                               uint32_t* __restrict__ leaf_of, uint4* __restrict__ int_list,
                                               uint32_t* __restrict__ int_count) {
    const int lane = threadIdx.x & 31;
    const bool inner = valid && cc > 0;
    const uint32_t key = inner ? d : 0xffu;
    const uint32_t peers = __match_any_sync(0xffffffffu, key);
    const int leader = __ffs(peers) - 1;
    uint32_t slot = 0;
    if (inner && lane == leader) slot = atomicAdd(&int_count[d], uint32_t(__popc(peers)));
    slot = __shfl_sync(0xffffffffu, slot, leader) + __popc(peers & ((1u << lane) - 1u));
    if (inner) int_list[level_start[d] + slot] = make_uint4(c, fc, cc, d);
    const uint32_t lc = valid && !inner ? cnt : 0u;
    if (lc <= 32u)
        for (uint32_t k = f; k < f + lc; ++k) leaf_of[k] = c;
    // large leaves (coincident clusters at depth 21, large leaf_cap): the whole warp writes each
    for (uint32_t big = __ballot_sync(0xffffffffu, lc > 32u); big; big &= big - 1) {
        const int src = __ffs(big) - 1;
        const uint32_t bf = __shfl_sync(0xffffffffu, f, src), bn = __shfl_sync(0xffffffffu, lc, src),
                       bc = __shfl_sync(0xffffffffu, c, src);
        for (uint32_t k = bf + lane; k < bf + bn; k += 32) leaf_of[k] = bc;
    }
}

// per cell: count = end of its digit run (8 keys probed at once, then galloping), and for split
// cells the number of consecutive next-level cells starting inside it; then the topology outputs
__global__ void __launch_bounds__(kBlock) split_cells_kernel(SplitArgs a, uint32_t n) {
    G2_PDL_WAIT();  // programmatic dependent launch (launch_pdl)
    const uint32_t total = min(a.level_start[kMaxDepth + 1], a.cell_cap);
    const bool topo = a.leaf_of && !(a.topo_gate && *a.topo_gate);
    for (uint32_t b0 = blockIdx.x * kBlock; b0 < total; b0 += gridDim.x * kBlock) {  // warp-uniform trips
        const uint32_t c = b0 + threadIdx.x;
        const bool valid = c < total;
        uint32_t i = 0, e = 0, fc = 0, cc = 0;
        int d = 0;
        if (valid) {
            i = a.first[c];
            d = a.depth[c];
            const int sh = 3 * (kMaxDepth - d);
            const uint64_t pre = a.keys[i] >> sh;
            uint64_t kk[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) kk[q] = i + 1 + q < n ? a.keys[i + 1 + q] : ~0ull;
#pragma unroll
            for (int q = 7; q >= 0; --q)
                if (i + 1 + q >= n || (kk[q] >> sh) != pre) e = i + 1 + q;
            if (!e) e = run_end(a.keys, n, i + 9, pre, sh);
            e = min(e, n);
            a.count[c] = e - i;
            fc = a.first_child[c];
            if (fc) {
                const uint32_t lend = min(a.level_start[d + 2], a.cell_cap);
                cc = 1;
                while (fc + cc < lend && a.first[fc + cc] < e) ++cc;
            }
            a.child_count[c] = cc;
        }
        if (topo) write_topology(c, valid, fc, cc, uint32_t(d), i, e - i, a.level_start, a.leaf_of, a.int_list,
                                      a.int_count);
    }
}

__global__ void split_init_kernel(SplitArgs a, uint32_t n) {
    if (threadIdx.x == 0) {
        a.first_child[0] = 0;
        a.child_count[0] = 0;
        a.first[0] = 0;
        a.count[0] = n;
        a.depth[0] = 0;
        a.level_start[0] = 0;
        a.level_start[1] = 1;
    }
}

// ---- calc_node (octree.cpp:108-162) --------------------------------------------
// All leaves in one launch (the bulk: particle sums and the walk's leaf-relative
// offsets), then the internal cells level by level, deepest first, each from its
// children in order -- the reference's operation order, so the FP64 node
// attributes are bit-identical.
__device__ __forceinline__ void store_node(WNode* __restrict__ nodes, WNode32* __restrict__ nodes32, uint32_t c,
                                           const WNode& nd) {
    // two 256-bit stores: whole sectors
    const uint32_t* w = reinterpret_cast<const uint32_t*>(&nd);
    WNode* dst = nodes + c;
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(dst), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                 "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                 : "memory");
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(reinterpret_cast<char*>(dst) + 32),
                 "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
                 : "memory");
    const float fm = float(nd.mass), fb = float(nd.extent);
    nodes32[c] = WNode32{float(nd.cx), float(nd.cy), float(nd.cz), fm, fb, fm * fb * fb, nd.link, nd.info};
}

// Leaves (every step), warp-synchronous: a warp takes 32 consecutive particles (coalesced loads of
// the positions and leaf_of) and stages them in its own 1 KB of shared memory.  The lane at a leaf's
// first particle folds the leaf's mass and weighted centre in the reference's order
// (octree.cpp:113-125) from there (particles beyond the warp's 32 from global memory); the centre
// goes back to the leaf's lanes by shuffles, every lane forms its own particle's |x - com|^2 and
// a segmented max (exact in any order) collects the extent; every lane writes its particle's
// leaf-relative FP32 offset.  A leaf belongs to the warp of its first particle, which also handles
// its particles beyond the warp's 32.  No block barriers.
constexpr int kLeafThreads = 256;
__global__ void __launch_bounds__(kLeafThreads) calc_leaf_kernel(const double4* __restrict__ xyzm,
                                                                 const uint32_t* __restrict__ leaf_of,
                                                                 const uint32_t* __restrict__ count, uint32_t n,
                                                                 WNode* __restrict__ nodes,
                                                                 WNode32* __restrict__ nodes32,
                                                                 float4* __restrict__ rel) {
    __shared__ double4 P[kLeafThreads];
    const int lane = threadIdx.x & 31;
    double4* const W = P + (threadIdx.x & ~31);  // this warp's 32 slots
    const uint32_t nw = gridDim.x * (kLeafThreads / 32);
    for (uint32_t base = (blockIdx.x * (kLeafThreads / 32) + (threadIdx.x >> 5)) * 32u; base < n; base += nw * 32u) {
        const uint32_t k = base + uint32_t(lane);
        const bool valid = k < n;
        const double4 p = valid ? xyzm[k] : make_double4(0.0, 0.0, 0.0, 0.0);
        const uint32_t c = valid ? leaf_of[k] : ~0u;
        uint32_t cprev = __shfl_up_sync(0xffffffffu, c, 1);
        if (lane == 0) cprev = base ? leaf_of[base - 1] : ~0u;
        const bool start = valid && c != cprev;
        const uint32_t starts = __ballot_sync(0xffffffffu, start);
        W[lane] = p;
        __syncwarp();
        // count: up to the next leaf start inside the warp; the warp's last leaf may run beyond it
        const uint32_t later = starts & ~((2u << lane) - 1u);
        const uint32_t cnt = start ? (later ? uint32_t(__ffs(later) - 1 - lane) : count[c]) : 0u;
        const uint32_t in = min(cnt, uint32_t(32 - lane));  // particles staged in the warp's slots
        double m = 0.0, wx = 0.0, wy = 0.0, wz = 0.0;
        for (uint32_t q = 0; q < cnt; ++q) {
            const double4 v = q < in ? W[lane + int(q)] : xyzm[k + q];
            m = dadd(m, v.w);
            wx = dadd(wx, dmul(v.w, v.x));
            wy = dadd(wy, dmul(v.w, v.y));
            wz = dadd(wz, dmul(v.w, v.z));
        }
        double cx = 0.0, cy = 0.0, cz = 0.0;
        if (start) {
            const double inv = ddiv(1.0, m);
            cx = dmul(wx, inv), cy = dmul(wy, inv), cz = dmul(wz, inv);
        }
        // the first lane of this particle's leaf inside the warp (none: an earlier warp owns the leaf)
        const uint32_t mine = valid ? starts & ((2u << lane) - 1u) : 0u;
        const int s = mine ? 31 - __clz(mine) : lane;
        cx = __shfl_sync(0xffffffffu, cx, s), cy = __shfl_sync(0xffffffffu, cy, s), cz = __shfl_sync(0xffffffffu, cz, s);
        double e2 = mine ? norm2(dsub(p.x, cx), dsub(p.y, cy), dsub(p.z, cz)) : 0.0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {  // segmented suffix max: lane s ends with its leaf's lanes
            const double v = __shfl_down_sync(0xffffffffu, e2, o);
            const int so = __shfl_down_sync(0xffffffffu, s, o);
            if (lane + o < 32 && so == s) e2 = smax(e2, v);
        }
        const float fx = float(cx), fy = float(cy), fz = float(cz);
        if (start) {
            for (uint32_t q = in; q < cnt; ++q) {  // beyond the warp's particles: this lane owns them
                const double4 v = xyzm[k + q];
                e2 = smax(e2, norm2(dsub(v.x, cx), dsub(v.y, cy), dsub(v.z, cz)));
                rel[k + q] = make_float4(float(dsub(v.x, double(fx))), float(dsub(v.y, double(fy))),
                                         float(dsub(v.z, double(fz))), float(v.w));
            }
            WNode nd;
            nd.cx = cx, nd.cy = cy, nd.cz = cz;
            nd.extent = dsqrt(e2);
            nd.link = k;
            nd.info = cnt | kLeafBit;
            nd.mass = m;
            store_node(nodes, nodes32, c, nd);
        }
        if (mine)
            rel[k] = make_float4(float(dsub(p.x, double(fx))), float(dsub(p.y, double(fy))), float(dsub(p.z, double(fz))),
                                 float(p.w));
        __syncwarp();  // the slots are rewritten by the next round
    }
}

#if G2_CALC_LEAF_CELLS
// leaves in cell order, one thread per cell
#ifndef G2_LEAF_SMALL
#define G2_LEAF_SMALL 8
#endif
constexpr int kLeafSmall = G2_LEAF_SMALL;  // leaves held in registers (larger: two passes over L1)
// a leaf of at most kLeafSmall particles, same operation order as the general loop below
__device__ __forceinline__ void leaf_small(const double4* __restrict__ xyzm, uint32_t f, uint32_t cnt, uint32_t c,
                                           WNode* __restrict__ nodes, WNode32* __restrict__ nodes32,
                                           float4* __restrict__ rel) {
    double4 p[kLeafSmall];
#pragma unroll
    for (int j = 0; j < kLeafSmall; ++j)
        if (j < int(cnt)) p[j] = xyzm[f + j];
    WNode nd;
    double m = 0.0, wx = 0.0, wy = 0.0, wz = 0.0;
#pragma unroll
    for (int j = 0; j < kLeafSmall; ++j)
        if (j < int(cnt)) {
            m = dadd(m, p[j].w);
            wx = dadd(wx, dmul(p[j].w, p[j].x));
            wy = dadd(wy, dmul(p[j].w, p[j].y));
            wz = dadd(wz, dmul(p[j].w, p[j].z));
        }
    const double inv = ddiv(1.0, m);
    nd.cx = dmul(wx, inv), nd.cy = dmul(wy, inv), nd.cz = dmul(wz, inv);
    const double c32x = double(float(nd.cx)), c32y = double(float(nd.cy)), c32z = double(float(nd.cz));
    double e2 = 0.0;
#pragma unroll
    for (int j = 0; j < kLeafSmall; ++j)
        if (j < int(cnt)) {
            e2 = smax(e2, norm2(dsub(p[j].x, nd.cx), dsub(p[j].y, nd.cy), dsub(p[j].z, nd.cz)));
            rel[f + j] = make_float4(float(dsub(p[j].x, c32x)), float(dsub(p[j].y, c32y)), float(dsub(p[j].z, c32z)),
                                     float(p[j].w));
        }
    nd.extent = dsqrt(e2);
    nd.link = f;
    nd.info = cnt | kLeafBit;
    nd.mass = m;
    store_node(nodes, nodes32, c, nd);
}

__global__ void __launch_bounds__(kBlock, G2_CALC_MINB) calc_leaf_cells_kernel(const double4* __restrict__ xyzm,
                                                           const uint32_t* __restrict__ child_count,
                                                           const uint32_t* __restrict__ first,
                                                           const uint32_t* __restrict__ count,
                                                           const uint32_t* __restrict__ level_start,
                                                           WNode* __restrict__ nodes, WNode32* __restrict__ nodes32,
                                                           float4* __restrict__ rel) {
    const uint32_t total = level_start[kMaxDepth + 1];
    for (uint32_t c = blockIdx.x * kBlock + threadIdx.x; c < total; c += gridDim.x * kBlock) {
        if (child_count[c]) continue;
        const uint32_t f = first[c], k1 = f + count[c];
        if (k1 - f <= uint32_t(kLeafSmall)) {  // the usual leaf: every particle loaded up front, one memory round trip
            leaf_small(xyzm, f, k1 - f, c, nodes, nodes32, rel);
            continue;
        }
        WNode nd;
        double m = 0.0, wx = 0.0, wy = 0.0, wz = 0.0;
        for (uint32_t k = f; k < k1; ++k) {
            const double4 p = xyzm[k];
            m = dadd(m, p.w);
            wx = dadd(wx, dmul(p.w, p.x));
            wy = dadd(wy, dmul(p.w, p.y));
            wz = dadd(wz, dmul(p.w, p.z));
        }
        const double inv = ddiv(1.0, m);
        nd.cx = dmul(wx, inv), nd.cy = dmul(wy, inv), nd.cz = dmul(wz, inv);
        const double c32x = double(float(nd.cx)), c32y = double(float(nd.cy)), c32z = double(float(nd.cz));
        double e2 = 0.0;
        for (uint32_t k = f; k < k1; ++k) {
            const double4 p = xyzm[k];
            e2 = smax(e2, norm2(dsub(p.x, nd.cx), dsub(p.y, nd.cy), dsub(p.z, nd.cz)));
            rel[k] = make_float4(float(dsub(p.x, c32x)), float(dsub(p.y, c32y)), float(dsub(p.z, c32z)), float(p.w));
        }
        nd.extent = dsqrt(e2);
        nd.link = f;
        nd.info = (k1 - f) | kLeafBit;
        nd.mass = m;
        store_node(nodes, nodes32, c, nd);
    }
}

#endif

// internal cell from its (at most 8) children in order (octree.cpp:145-162).  All children
// are loaded up front: one memory round trip per cell instead of two dependent chains of cc.
template <bool kL2 = false>  // kL2: children read through L2 (written by other blocks of the same launch)
__device__ __forceinline__ WNode internal_node(const WNode* nodes, uint32_t f, uint32_t cc, uint8_t dep) {
    double qx[8], qy[8], qz[8], qm[8], qe[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (j < int(cc)) {
            const double2* q = reinterpret_cast<const double2*>(nodes + f + j);
            const double2 a = kL2 ? __ldcg(q) : q[0], b = kL2 ? __ldcg(q + 1) : q[1], e = kL2 ? __ldcg(q + 2) : q[2];
            qx[j] = a.x, qy[j] = a.y, qz[j] = b.x, qm[j] = b.y, qe[j] = e.x;
        }
    WNode nd;
    double m = 0.0, wx = 0.0, wy = 0.0, wz = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (j < int(cc)) {
            m = dadd(m, qm[j]);
            wx = dadd(wx, dmul(qm[j], qx[j]));
            wy = dadd(wy, dmul(qm[j], qy[j]));
            wz = dadd(wz, dmul(qm[j], qz[j]));
        }
    const double inv = ddiv(1.0, m);
    nd.cx = dmul(wx, inv), nd.cy = dmul(wy, inv), nd.cz = dmul(wz, inv);
    double ext = 0.0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (j < int(cc))
            ext = smax(ext, dadd(dsqrt(norm2(dsub(qx[j], nd.cx), dsub(qy[j], nd.cy), dsub(qz[j], nd.cz))), qe[j]));
    nd.extent = ext;
    nd.link = f;
    nd.info = cc | (uint32_t(dep) << 8);  // depth feeds the frontier-cap check
    nd.mass = m;
    return nd;
}


// Internal cell from its children in order (octree.cpp:145-162), 8 lanes per cell (4 cells per
// warp): lane j loads child j's record, every lane of the group folds the children's masses and
// weighted centres in order through shuffles (the reference's left fold, bit for bit), then lane j
// forms child j's extent term and a 3-step max (exact in any order) combines them.  Records written
// by other CTAs of the same launch are read through L2 (ld.cg).
__device__ __forceinline__ void internal_group8(const uint4 E, bool valid, WNode* nodes, WNode32* __restrict__ nodes32) {
    const int lane = threadIdx.x & 31, j = lane & 7, g0 = lane & ~7;
    const uint32_t c = E.x, fc = E.y, cc = valid ? E.z : 0u;
    const bool have = uint32_t(j) < cc;
    double qx = 0.0, qy = 0.0, qz = 0.0, qm = 0.0, qe = 0.0;
    if (have) {
        const double2* q = reinterpret_cast<const double2*>(nodes + fc + j);
        const double2 a = __ldcg(q), b = __ldcg(q + 1), e = __ldcg(q + 2);
        qx = a.x, qy = a.y, qz = b.x, qm = b.y, qe = e.x;
    }
    double m = 0.0, wx = 0.0, wy = 0.0, wz = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const double km = __shfl_sync(0xffffffffu, qm, g0 + k), kx = __shfl_sync(0xffffffffu, qx, g0 + k),
                     ky = __shfl_sync(0xffffffffu, qy, g0 + k), kz = __shfl_sync(0xffffffffu, qz, g0 + k);
        if (uint32_t(k) < cc) {
            m = dadd(m, km);
            wx = dadd(wx, dmul(km, kx));
            wy = dadd(wy, dmul(km, ky));
            wz = dadd(wz, dmul(km, kz));
        }
    }
    WNode nd;
    const double inv = ddiv(1.0, m);
    nd.cx = dmul(wx, inv), nd.cy = dmul(wy, inv), nd.cz = dmul(wz, inv);
    double ext = have ? dadd(dsqrt(norm2(dsub(qx, nd.cx), dsub(qy, nd.cy), dsub(qz, nd.cz))), qe) : 0.0;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) ext = smax(ext, __shfl_xor_sync(0xffffffffu, ext, o));
    if (valid && j == 0) {
        nd.extent = ext;
        nd.link = fc;
        nd.info = cc | (E.w << 8);  // depth feeds the frontier-cap check
        nd.mass = m;
        store_node(nodes, nodes32, c, nd);
    }
}

// the internal cells of depth d, `parts` warps sharing them (warp index w)
__device__ __forceinline__ void internal_level(const uint4* __restrict__ int_list, uint32_t b, uint32_t cnt,
                                               uint32_t w, uint32_t parts, WNode* nodes, WNode32* __restrict__ nodes32) {
#if G2_CALC_GROUP8
    const uint32_t sub = (threadIdx.x & 31) >> 3;
    for (uint32_t i0 = 4 * w; i0 < cnt; i0 += 4 * parts) {  // warp-uniform trips
        const uint32_t i = i0 + sub;
        const bool valid = i < cnt;
        internal_group8(valid ? int_list[b + i] : make_uint4(0u, 0u, 0u, 0u), valid, nodes, nodes32);
    }
#else
    for (uint32_t i = 32 * w + (threadIdx.x & 31); i < cnt; i += 32 * parts) {
        const uint4 E = int_list[b + i];
        store_node(nodes, nodes32, E.x, internal_node(nodes, E.y, E.z, uint8_t(E.w)));
    }
#endif
}

// one wide level: the grid's warps share its internal cells
__global__ void __launch_bounds__(kBlock) calc_internal_kernel(const uint4* __restrict__ int_list,
                                                               const uint32_t* __restrict__ int_count,
                                                               const uint32_t* __restrict__ level_start, WNode* nodes,
                                                               WNode32* __restrict__ nodes32, int d) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: the previous level's records are complete
    internal_level(int_list, level_start[d], int_count[d], blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5),
                   gridDim.x * (kBlock / 32), nodes, nodes32);
}

// a run of narrow levels (depths d_hi down to d_lo) in ONE block, levels separated by __syncthreads
// instead of a launch each
constexpr int kLevelsThreads = 512;
constexpr uint32_t kNarrowCells = 2048;  // internal cells per level the host sends to one block
__global__ void __launch_bounds__(kLevelsThreads, 1) calc_levels_kernel(const uint4* __restrict__ int_list,
                                                                        const uint32_t* __restrict__ int_count,
                                                                        const uint32_t* __restrict__ level_start,
                                                                        WNode* nodes, WNode32* __restrict__ nodes32,
                                                                        int d_hi, int d_lo) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: the previous level's records are complete
    for (int d = d_hi; d >= d_lo; --d) {
        internal_level(int_list, level_start[d], int_count[d], threadIdx.x >> 5, kLevelsThreads / 32, nodes, nodes32);
        __syncthreads();  // level d complete (and visible to the block) before level d - 1 reads it
    }
}

// All internal levels in ONE launch, as a dependency-ordered work list: units are handed out by an
// atomic ticket in stage order (stage = one wide level in chunks of kFuseCells cells, or one run of
// narrow levels done by a single block with __syncthreads between its levels), and a unit starts once
// every unit of the previous stage has completed.  Tickets are taken in order, so the units a waiting
// block depends on are all held by running blocks: no co-residency assumption, no deadlock.
constexpr int kFuseThreads = 256;
constexpr uint32_t kFuseCells = kFuseThreads;  // one internal cell per thread
constexpr int kMaxStages = kMaxDepth + 1;
struct CalcStages {
    int n;                                   // stages, deepest first
    int8_t hi[kMaxStages], lo[kMaxStages];   // depth range of each stage
    int8_t narrow[kMaxStages];               // 1: one unit, one block
};
__global__ void __launch_bounds__(kFuseThreads, 2) calc_internal_fused_kernel(const uint4* __restrict__ int_list,
                                                                              const uint32_t* __restrict__ int_count,
                                                                              const uint32_t* __restrict__ level_start,
                                                                              WNode* nodes, WNode32* __restrict__ nodes32,
                                                                              CalcStages st, uint32_t* sync) {
    __shared__ uint32_t stage_end[kMaxStages];
    __shared__ uint32_t unit_s;
    __shared__ int ready;  // the last stage this block has seen complete
    if (threadIdx.x == 0) {
        uint32_t e = 0;
        for (int k = 0; k < st.n; ++k) {
            e += st.narrow[k] ? 1u : max(1u, (int_count[st.hi[k]] + kFuseCells - 1) / kFuseCells);
            stage_end[k] = e;
        }
        ready = -1;
    }
    __syncthreads();
    const uint32_t total = st.n ? stage_end[st.n - 1] : 0u;
    uint32_t* ticket = sync;
    uint32_t* done = sync + 1;
    while (true) {
        if (threadIdx.x == 0) unit_s = atomicAdd(ticket, 1u);
        __syncthreads();
        const uint32_t u = unit_s;
        if (u >= total) return;
        int k = 0;
        while (u >= stage_end[k]) ++k;
        if (threadIdx.x == 0 && k > 0 && ready < k - 1) {
            const uint32_t need = stage_end[k - 1] - (k >= 2 ? stage_end[k - 2] : 0u);
            uint32_t v;
            while (true) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(done + k - 1) : "memory");
                if (v >= need) break;
                __nanosleep(32);
            }
            ready = k - 1;
        }
        __syncthreads();  // the previous stage's records are complete (read through L2); unit_s is free
        // one wide level's chunk, or every level of a narrow run (one call site of internal_node)
        const bool narrow = st.narrow[k];
        const uint32_t c0 = narrow ? 0u : (u - (k ? stage_end[k - 1] : 0u)) * kFuseCells;
        for (int d = st.hi[k]; d >= st.lo[k]; --d) {
            const uint32_t b = level_start[d], cnt = int_count[d];
            const uint32_t c1 = narrow ? cnt : min(cnt, c0 + kFuseCells);
            for (uint32_t i = c0 + threadIdx.x; i < c1; i += kFuseThreads) {
                const uint4 E = int_list[b + i];
                store_node(nodes, nodes32, E.x, internal_node<true>(nodes, E.y, E.z, uint8_t(E.w)));
            }
            __syncthreads();  // level d complete (and visible to the block) before level d - 1
        }
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(&done[k], 1u);
        }
    }
}

// Per topology (after every split): leaf_of[k] for every particle of every leaf, and the internal
// cells of each depth d listed at int_list[level_start[d] + slot] as (cell, first_child,
// child_count, depth) -- warp-aggregated slot claims on int_count[d], zeroed by the caller; the order
// inside a depth is immaterial (the cells of one depth are independent).
__global__ void __launch_bounds__(kBlock) tree_topology_kernel(const uint32_t* __restrict__ first_child,
                                                               const uint32_t* __restrict__ child_count,
                                                               const uint32_t* __restrict__ first,
                                                               const uint32_t* __restrict__ count,
                                                               const uint8_t* __restrict__ depth,
                                                               const uint32_t* __restrict__ level_start,
                                                               uint32_t cell_cap, uint32_t* __restrict__ leaf_of,
                                                               uint4* __restrict__ int_list,
                                                               uint32_t* __restrict__ int_count) {
    const uint32_t total = min(level_start[kMaxDepth + 1], cell_cap);
    const int lane = threadIdx.x & 31;
    for (uint32_t b0 = blockIdx.x * kBlock; b0 < total; b0 += gridDim.x * kBlock) {  // warp-uniform trips
        const uint32_t c = b0 + threadIdx.x;
        const bool valid = c < total;
        const uint32_t cc = valid ? child_count[c] : 0u;
        const bool leaf = valid && cc == 0;
        write_topology(c, valid, valid && cc ? first_child[c] : 0u, cc, valid ? uint32_t(depth[c]) : 0u,
                       leaf ? first[c] : 0u, leaf ? count[c] : 0u, level_start, leaf_of, int_list, int_count);
    }
}

__global__ void __launch_bounds__(kBlock) leaf_rel_kernel(const double4* __restrict__ xyzm,
                                                          const uint32_t* __restrict__ child_count,
                                                          const uint32_t* __restrict__ first,
                                                          const uint32_t* __restrict__ count,
                                                          const WNode32* __restrict__ nodes32, uint32_t ncells,
                                                          float4* __restrict__ rel) {
    for (uint32_t c = blockIdx.x * kBlock + threadIdx.x; c < ncells; c += gridDim.x * kBlock) {
        if (child_count[c]) continue;
        const WNode32 nd = nodes32[c];
        const double cx = nd.cx, cy = nd.cy, cz = nd.cz;
        const uint32_t f = first[c], k1 = f + count[c];
        for (uint32_t k = f; k < k1; ++k) {
            const double4 p = xyzm[k];
            rel[k] = make_float4(float(dsub(p.x, cx)), float(dsub(p.y, cy)), float(dsub(p.z, cz)), float(p.w));
        }
    }
}

// ---- equal-key runs after a storage-order sort -----------------------------------------
// The Simulation sorts (key, storage position) pairs: LSD radix sort is stable, so equal keys
// come out in storage order, while the reference's (key, original index) pair sort wants them
// by original id (octree.cpp:60-63).  Runs are rare (coincident quantised positions); each is
// insertion-sorted by id in place.  Runs longer than kMaxTieRun set flags->tie_run.
constexpr uint32_t kMaxTieRun = 64;
__global__ void __launch_bounds__(kBlock) fix_ties_kernel(const uint64_t* __restrict__ keys, uint32_t* __restrict__ src,
                                                          const uint32_t* __restrict__ ids, size_t n, DevFlags* flags) {
    for (size_t k = blockIdx.x * size_t(kBlock) + threadIdx.x; k + 1 < n; k += size_t(gridDim.x) * kBlock) {
        const uint64_t key = keys[k];
        if (keys[k + 1] != key || (k > 0 && keys[k - 1] == key)) continue;  // not the start of a run
        uint32_t len = 2;
        while (k + len < n && keys[k + len] == key && len <= kMaxTieRun) ++len;
        if (len > kMaxTieRun) {
            flags->tie_run = 1;
            continue;
        }
        for (uint32_t a = 1; a < len; ++a) {
            const uint32_t v = src[k + a], iv = ids[v];
            uint32_t b = a;
            while (b > 0 && ids[src[k + b - 1]] > iv) {
                src[k + b] = src[k + b - 1];
                --b;
            }
            src[k + b] = v;
        }
    }
}

// ---- gathers / permutations ----------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kBlock) gather_kernel(const T* __restrict__ in, const uint32_t* __restrict__ src,
                                                        T* __restrict__ out, size_t n) {
    for (size_t i = blockIdx.x * size_t(kBlock) + threadIdx.x; i < n; i += size_t(gridDim.x) * kBlock)
        out[i] = in[src[i]];
}

__global__ void __launch_bounds__(kBlock) invert_perm_kernel(const uint32_t* __restrict__ perm,
                                                             uint32_t* __restrict__ rank, size_t n) {
    for (size_t i = blockIdx.x * size_t(kBlock) + threadIdx.x; i < n; i += size_t(gridDim.x) * kBlock)
        rank[perm[i]] = uint32_t(i);
}

__global__ void __launch_bounds__(kBlock) pack_kernel(const double* __restrict__ pos3, const double* __restrict__ mass,
                                                      const uint32_t* __restrict__ perm, double4* __restrict__ xyzm,
                                                      size_t n) {
    for (size_t i = blockIdx.x * size_t(kBlock) + threadIdx.x; i < n; i += size_t(gridDim.x) * kBlock) {
        const size_t id = perm ? perm[i] : i;
        xyzm[i] = make_double4(pos3[3 * id], pos3[3 * id + 1], pos3[3 * id + 2], mass[id]);
    }
}

__global__ void __launch_bounds__(kBlock) iota_kernel(uint32_t* out, size_t n) {
    for (size_t i = blockIdx.x * size_t(kBlock) + threadIdx.x; i < n; i += size_t(gridDim.x) * kBlock)
        out[i] = uint32_t(i);
}

inline unsigned grid_for(size_t n) { return std::max(1u, std::min<unsigned>(ceil_div(n, kBlock), kNumSMs * 16)); }

}  // namespace

void launch_bbox(const double4* xyzm, size_t n, double* partials, Cube* cube, DevFlags* flags, cudaStream_t s) {
    const unsigned nb = std::max(1u, std::min<unsigned>(ceil_div(n, kBlock * 4), kNumSMs * 4));
    G2_COUNT(1), bbox_partial_kernel<<<nb, kBlock, 0, s>>>(xyzm, n, partials, flags);
    G2_COUNT(1), launch_pdl(bbox_final_kernel, dim3(1), dim3(kBboxFinalThreads), size_t(0), s, partials, int(nb), cube);
    G2_CUDA(cudaGetLastError());
}

void launch_bbox_final(const double* partials, unsigned nb, Cube* cube, cudaStream_t s) {
    G2_COUNT(1), launch_pdl(bbox_final_kernel, dim3(1), dim3(kBboxFinalThreads), size_t(0), s, partials, int(nb), cube);
}

void launch_keys(const double4* xyzm, const uint32_t* id_of_pos, size_t n, const Cube* cube, uint64_t* key_by_id,
                 DevFlags* flags, cudaStream_t s) {
    G2_COUNT(1), keys_kernel<<<grid_for(n), kBlock, 0, s>>>(xyzm, id_of_pos, n, cube, key_by_id, flags);
    G2_CUDA(cudaGetLastError());
}

// per-depth tile counts + totals, then the per-particle (lo, hi) depth ranges (u16)
size_t split_tile_words(size_t n) {
    return (kMaxDepth + 1) * (ceil_div(n, kSplitTile) + 1) + 32 + (n + 1) / 2 + 4 +
           size_t(kChunkCountWords) * ceil_div(n, kSplitTile);
}

bool launch_split(const SplitArgs& a, uint32_t n, cudaStream_t s) {
    if (a.leaf_cap <= kSplitMaxCap && a.tiles) {
        if (a.leaf_of) G2_CUDA(cudaMemsetAsync(a.int_count, 0, (kMaxDepth + 1) * sizeof(uint32_t), s));
        const uint32_t ntiles = ceil_div(n, kSplitTile);
        uint32_t* totals = a.tiles + size_t(kMaxDepth + 1) * ntiles;
        uint16_t* lohi = reinterpret_cast<uint16_t*>(a.tiles + (kMaxDepth + 1) * (size_t(ntiles) + 1) + 32);
        uint32_t* chunk_counts = a.tiles + (kMaxDepth + 1) * (size_t(ntiles) + 1) + 32 + (size_t(n) + 1) / 2 + 4;
        G2_COUNT(1), split_count_kernel<<<ntiles, kSplitThreads, 0, s>>>(a.keys, n, a.leaf_cap, a.tiles, ntiles, lohi,
                                                                          chunk_counts);
        G2_COUNT(1), launch_pdl(split_scan_kernel, dim3(kMaxDepth + 1), dim3(1024), size_t(0), s, a.tiles, ntiles, totals);
        G2_COUNT(1), launch_pdl(split_write_kernel, dim3(ntiles), dim3(kSplitThreads), size_t(0), s, a, n, a.tiles, ntiles, totals, lohi,
                                                                          chunk_counts);
        G2_COUNT(1), launch_pdl(split_cells_kernel, dim3(grid_for(a.cell_cap)), dim3(kBlock), size_t(0), s, a, n);
        G2_CUDA(cudaGetLastError());
        return a.leaf_of != nullptr;
    }
    // level-by-level path (leaf_cap > kSplitMaxCap)
    G2_COUNT(1), split_init_kernel<<<1, 32, 0, s>>>(a, n);
    // levels are sized on the device; a fixed persistent grid pulls tiles dynamically
    static const bool dbg = std::getenv("G2_SPLIT_DEBUG") != nullptr;  // development: per-level device times
    static cudaEvent_t ev[kMaxDepth + 1];
    if (dbg && !ev[0])
        for (auto& e : ev) cudaEventCreate(&e);
    for (int d = 0; d < kMaxDepth; ++d) {
        if (dbg) cudaEventRecord(ev[d], s);
        G2_COUNT(1), split_level_kernel<<<kNumSMs * 4, kBlock, 0, s>>>(a, d);
    }
    if (dbg) {
        cudaEventRecord(ev[kMaxDepth], s);
        cudaEventSynchronize(ev[kMaxDepth]);
        uint32_t ls[kMaxDepth + 3];
        cudaMemcpy(ls, a.level_start, sizeof ls, cudaMemcpyDeviceToHost);
        for (int d = 0; d < kMaxDepth; ++d) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[d], ev[d + 1]);
            std::fprintf(stderr, "[g2 split] depth %2d cells %8u  %.3f ms\n", d, ls[d + 1] - ls[d], ms);
        }
    }
    G2_CUDA(cudaGetLastError());
    return false;
}

void launch_tree_topology(const uint32_t* first_child, const uint32_t* child_count, const uint32_t* first,
                          const uint32_t* count, const uint8_t* depth, const uint32_t* level_start, size_t ncells,
                          uint32_t cell_cap, uint32_t* leaf_of, uint4* int_list, uint32_t* int_count, cudaStream_t s) {
    G2_CUDA(cudaMemsetAsync(int_count, 0, (kMaxDepth + 1) * sizeof(uint32_t), s));
    G2_COUNT(1), tree_topology_kernel<<<grid_for(ncells), kBlock, 0, s>>>(first_child, child_count, first, count, depth,
                                                                          level_start, cell_cap, leaf_of, int_list,
                                                                          int_count);
    G2_CUDA(cudaGetLastError());
}

void launch_calc_node(const double4* xyzm, size_t n, const uint32_t* child_count, const uint32_t* first,
                      const uint32_t* count, const uint32_t* level_start,
                      const uint32_t* level_start_host, const uint32_t* leaf_of, const uint4* int_list,
                      const uint32_t* int_count, uint32_t* sync, WNode* nodes, WNode32* nodes32, float4* rel,
                      cudaStream_t s, cudaStream_t s_internal, cudaEvent_t fork) {
#if G2_CALC_LEAF_CELLS
    G2_COUNT(1), calc_leaf_cells_kernel<<<grid_for(level_start_host[kMaxDepth + 1]), kBlock, 0, s>>>(
        xyzm, child_count, first, count, level_start, nodes, nodes32, rel);
#else
    G2_COUNT(1), calc_leaf_kernel<<<unsigned(std::min<size_t>(ceil_div(n, kLeafThreads), size_t(kNumSMs) * 8)),
                                    kLeafThreads, 0, s>>>(xyzm, leaf_of, count, uint32_t(n), nodes, nodes32, rel);
#endif
    if (s_internal) {  // the internal levels on their own stream, after the leaves
        G2_CUDA(cudaEventRecord(fork, s));
        G2_CUDA(cudaStreamWaitEvent(s_internal, fork, 0));
        s = s_internal;
    }
    int deepest = -1;  // the deepest internal level (the deepest non-empty level holds leaves only)
    for (int d = 0; d <= kMaxDepth; ++d)
        if (level_start_host[d + 1] > level_start_host[d]) deepest = d - 1;
    // internal cells at depth d: at most the level's width and at most the next level's width
    auto bound = [&](int d) {
        return std::min(level_start_host[d + 1] - level_start_host[d], level_start_host[d + 2] - level_start_host[d + 1]);
    };
#if G2_CALC_FUSED
    CalcStages st{};
    for (int d = deepest; d >= 0;) {
        const bool narrow = bound(d) <= kNarrowCells;
        int lo = d;
        if (narrow)
            while (lo > 0 && bound(lo - 1) <= kNarrowCells) --lo;
        st.hi[st.n] = int8_t(d), st.lo[st.n] = int8_t(lo), st.narrow[st.n] = narrow ? 1 : 0;
        ++st.n;
        d = lo - 1;
    }
    if (st.n) {
        static int per_sm = 0;
        if (!per_sm) {
            G2_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, calc_internal_fused_kernel, kFuseThreads, 0));
            per_sm = std::max(1, per_sm);
        }
        G2_CUDA(cudaMemsetAsync(sync, 0, (kMaxStages + 1) * sizeof(uint32_t), s));
        G2_COUNT(1), calc_internal_fused_kernel<<<unsigned(per_sm * kNumSMs), kFuseThreads, 0, s>>>(
            int_list, int_count, level_start, nodes, nodes32, st, sync);
    }
    G2_CUDA(cudaGetLastError());
    return;
#endif
    // the level chain as programmatic dependent launches: each level's grid is launched while the
    // previous one drains and waits (griddepcontrol.wait) for its completion and memory flush, which
    // takes the launch latency off the chain (the first launch follows the leaves normally)
    static const bool no_pdl = std::getenv("G2_NO_PDL") != nullptr;  // development A/B
    bool chain_first = true;
    auto launch = [&](auto kernel, unsigned grid, unsigned block, auto... args) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid), cfg.blockDim = dim3(block), cfg.dynamicSmemBytes = 0, cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr, cfg.numAttrs = (chain_first || no_pdl) ? 0 : 1;
        chain_first = false;
        G2_COUNT(1);
        G2_CUDA(cudaLaunchKernelEx(&cfg, kernel, args...));
    };
    for (int d = deepest; d >= 0;) {
        if (bound(d) <= kNarrowCells) {  // a run of narrow levels: one block
            int lo = d;
            while (lo > 0 && bound(lo - 1) <= kNarrowCells) --lo;
            launch(calc_levels_kernel, 1u, unsigned(kLevelsThreads), int_list, int_count, level_start, nodes, nodes32,
                   d, lo);
            d = lo - 1;
            continue;
        }
        const unsigned grid = unsigned(std::min<size_t>(ceil_div(size_t(bound(d)) * (G2_CALC_GROUP8 ? 8 : 1), kBlock),
                                                        size_t(kNumSMs) * 8));
        launch(calc_internal_kernel, grid, unsigned(kBlock), int_list, int_count, level_start, nodes, nodes32, d);
        --d;
    }
    G2_CUDA(cudaGetLastError());
}

void launch_leaf_rel(const double4* xyzm, const uint32_t* child_count, const uint32_t* first, const uint32_t* count,
                     const WNode32* nodes32, uint32_t ncells, float4* rel, cudaStream_t s) {
    G2_COUNT(1), leaf_rel_kernel<<<grid_for(ncells), kBlock, 0, s>>>(xyzm, child_count, first, count, nodes32, ncells, rel);
    G2_CUDA(cudaGetLastError());
}

void launch_gather_f64(const double* in, const uint32_t* src, double* out, size_t n, cudaStream_t s) {
    G2_COUNT(1), gather_kernel<double><<<grid_for(n), kBlock, 0, s>>>(in, src, out, n);
}
void launch_gather_u8(const uint8_t* in, const uint32_t* src, uint8_t* out, size_t n, cudaStream_t s) {
    G2_COUNT(1), gather_kernel<uint8_t><<<grid_for(n), kBlock, 0, s>>>(in, src, out, n);
}
void launch_gather_u32(const uint32_t* in, const uint32_t* src, uint32_t* out, size_t n, cudaStream_t s) {
    G2_COUNT(1), gather_kernel<uint32_t><<<grid_for(n), kBlock, 0, s>>>(in, src, out, n);
}
void launch_fix_ties(const uint64_t* keys, uint32_t* src, const uint32_t* ids, size_t n, DevFlags* flags,
                     cudaStream_t s) {
    G2_COUNT(1), fix_ties_kernel<<<grid_for(n), kBlock, 0, s>>>(keys, src, ids, n, flags);
}
void launch_invert_perm(const uint32_t* perm, uint32_t* rank, size_t n, cudaStream_t s) {
    G2_COUNT(1), invert_perm_kernel<<<grid_for(n), kBlock, 0, s>>>(perm, rank, n);
}
void launch_pack_sorted(const double* pos3, const double* mass, const uint32_t* perm, double4* xyzm, size_t n,
                        cudaStream_t s) {
    G2_COUNT(1), pack_kernel<<<grid_for(n), kBlock, 0, s>>>(pos3, mass, perm, xyzm, n);
}
void launch_pack_identity(const double* pos3, const double* mass, double4* xyzm, size_t n, cudaStream_t s) {
    G2_COUNT(1), pack_kernel<<<grid_for(n), kBlock, 0, s>>>(pos3, mass, nullptr, xyzm, n);
}
void launch_iota(uint32_t* out, size_t n, cudaStream_t s) { G2_COUNT(1), iota_kernel<<<grid_for(n), kBlock, 0, s>>>(out, n); }

size_t calc_sync_words() { return kMaxStages + 1; }

}  // namespace g2
