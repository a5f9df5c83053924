// Onesweep LSD radix sort (see radix_sort.cuh).
#include "radix_sort.cuh"

namespace g2 {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef G2_SORT_ITEMS
#define G2_SORT_ITEMS 8
#endif
#ifndef G2_ONESWEEP
#define G2_ONESWEEP 1  // 1: one kernel per pass with decoupled look-back; 0: count/scan/scatter passes
#endif
#ifndef G2_SORT_BALLOT_MATCH
#define G2_SORT_BALLOT_MATCH 1  // 9 ballots per key beat MATCH.ANY: sort 0.86 -> 0.78 ms at 2^23
#endif
#ifndef G2_SORT_MINB
#define G2_SORT_MINB 4
#endif
constexpr int kItems = G2_SORT_ITEMS;           // keys per thread
constexpr int kTile = kThreads * kItems;        // keys per tile
constexpr int kWarpItems = 32 * kItems;         // 256 consecutive keys per warp


// exclusive scan of one value per thread across the 256-thread block
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* warp_tot, uint32_t* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) warp_tot[w] = inc;
    __syncthreads();
    uint32_t wpre = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < kWarps; ++i) {
        const uint32_t t = warp_tot[i];
        if (i < w) wpre += t;
        tot += t;
    }
    if (total) *total = tot;
    return wpre + inc - x;
}

// ---- per pass: (1) tile digit counts, (2) one exclusive scan over the
// digit-major (digit, tile) matrix = global offsets, (3) stable scatter.
// No look-back chains: every tile's offsets are known before it scatters.
template <typename K>
__global__ void __launch_bounds__(kThreads) count_kernel(const K* __restrict__ kin, size_t n, int shift,
                                                         uint32_t* __restrict__ counts, uint32_t tiles) {
    __shared__ uint32_t h[kWarps][256];  // per-warp histograms: no cross-warp contention
    const int tid = threadIdx.x, w = tid >> 5;
    for (int i = tid; i < kWarps * 256; i += kThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    const size_t base = size_t(blockIdx.x) * kTile;
    K k[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const size_t idx = base + size_t(i) * kThreads + tid;
        k[i] = idx < n ? kin[idx] : K(0);
    }
#pragma unroll
    for (int i = 0; i < kItems; ++i)
        if (base + size_t(i) * kThreads + tid < n) atomicAdd(&h[w][uint32_t((k[i] >> shift) & 0xff)], 1u);
    __syncthreads();
    uint32_t c = 0;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) c += h[ww][tid];
    counts[size_t(tid) * tiles + blockIdx.x] = c;
}

// exclusive scan of counts[0, m) in place, single pass with decoupled look-back
constexpr int kScanItems = 16;
__global__ void __launch_bounds__(kThreads) scan_kernel(uint32_t* __restrict__ counts, size_t m,
                                                        uint64_t* __restrict__ status, uint32_t* __restrict__ ctr) {
    __shared__ uint32_t s_tile, s_wsum[kWarps];
    __shared__ uint64_t s_excl;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const size_t base = (size_t(tile) * kThreads + tid) * kScanItems;  // blocked
    uint32_t v[kScanItems], sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = base + k < m ? counts[base + k] : 0u;
        sum += v[k];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_wsum[w] = inc;
    __syncthreads();
    uint32_t wpre = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < kWarps; ++k) {
        if (k < w) wpre += s_wsum[k];
        tot += s_wsum[k];
    }
    if (w == 0) {
        const uint64_t e = lookback_warp(status, tile, tot);
        if (lane == 0) s_excl = e;
    }
    __syncthreads();
    uint32_t run = uint32_t(s_excl) + wpre + inc - sum;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < m) counts[base + k] = run;
        run += v[k];
    }
}

template <typename K, bool kIdentity>
__global__ void __launch_bounds__(kThreads, G2_SORT_MINB) scatter_kernel(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                           K* __restrict__ kout, uint32_t* __restrict__ vout,
                                                           size_t n, int shift, const uint32_t* __restrict__ offsets,
                                                           uint32_t tiles) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K* skeys = reinterpret_cast<K*>(smem_raw);
    uint32_t* svals = reinterpret_cast<uint32_t*>(smem_raw + sizeof(K) * kTile);
    __shared__ uint32_t whist[kWarps][256];
    __shared__ uint32_t s_lofs[256], s_base[256];
    __shared__ uint32_t s_wtot[kWarps];

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    for (int i = tid; i < kWarps * 256; i += kThreads) (&whist[0][0])[i] = 0;
    const uint32_t tile = blockIdx.x;
    s_base[tid] = offsets[size_t(tid) * tiles + tile];
    __syncthreads();
    const size_t tile_base = size_t(tile) * kTile;
    const size_t wbase = tile_base + size_t(w) * kWarpItems;

    K k[kItems];
    uint32_t v[kItems], d[kItems], r[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const size_t idx = wbase + size_t(i) * 32 + lane;
        const bool ok = idx < n;
        k[i] = ok ? kin[idx] : K(0);
        v[i] = kIdentity ? uint32_t(idx) : (ok ? vin[idx] : 0u);
        d[i] = ok ? uint32_t((k[i] >> shift) & 0xff) : 256u;
    }
    const uint32_t lt_mask = (1u << lane) - 1u;
    // warp-local stable ranking: item order i*32+lane is memory order
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const uint32_t m = __match_any_sync(0xffffffffu, d[i]);
        const uint32_t before = d[i] < 256u ? whist[w][d[i] & 0xff] : 0u;
        r[i] = before + __popc(m & lt_mask);
        __syncwarp();
        if (d[i] < 256u && lane == __ffs(m) - 1) whist[w][d[i]] = before + __popc(m);
        __syncwarp();
    }
    __syncthreads();
    uint32_t cnt = 0;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) {
        const uint32_t c = whist[ww][tid];
        whist[ww][tid] = cnt;
        cnt += c;
    }
    s_lofs[tid] = block_excl_scan(cnt, s_wtot, nullptr);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        if (d[i] < 256u) {
            const uint32_t pos = s_lofs[d[i]] + whist[w][d[i]] + r[i];
            skeys[pos] = k[i];
            svals[pos] = v[i];
        }
    }
    __syncthreads();
    const uint32_t tile_n = uint32_t(min(size_t(kTile), n - tile_base));
    for (uint32_t p = tid; p < tile_n; p += kThreads) {
        const K kk = skeys[p];
        const uint32_t dd = uint32_t((kk >> shift) & 0xff);
        const uint32_t dst = s_base[dd] + (p - s_lofs[dd]);
        kout[dst] = kk;
        vout[dst] = svals[p];
    }
}

// ---- onesweep variant: one kernel per pass.  Global digit bases come from ONE histogram pass
// over the keys for every digit (order-independent totals); tiles are claimed in order, rank and
// stage themselves in shared memory (nothing held in registers across the look-back), publish
// per-digit counts, and each thread (= digit) looks back over 8 predecessor tiles per step.
constexpr uint32_t kOsAgg = 1u << 30, kOsInc = 2u << 30, kOsMask = (1u << 30) - 1;
constexpr int kLookWindow = 8;

__device__ __forceinline__ void os_store(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t os_load(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <typename K>
__global__ void __launch_bounds__(kThreads) hist_all_kernel(const K* __restrict__ kin, size_t n, int passes,
                                                            uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[8][256];
    for (int i = threadIdx.x; i < 8 * 256; i += kThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    for (size_t i = size_t(blockIdx.x) * kThreads + threadIdx.x; i < n; i += size_t(gridDim.x) * kThreads) {
        const K k = kin[i];
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (q < passes) atomicAdd(&h[q][uint32_t(k >> (8 * q)) & 0xffu], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * 256; i += kThreads)
        if ((&h[0][0])[i]) atomicAdd(&hist[i], (&h[0][0])[i]);
}

__global__ void __launch_bounds__(kThreads) digit_base_kernel(uint32_t* __restrict__ hist) {
    __shared__ uint32_t wt[kWarps];
    uint32_t* row = hist + blockIdx.x * 256;
    const uint32_t x = row[threadIdx.x];
    const uint32_t e = block_excl_scan(x, wt, nullptr);
    row[threadIdx.x] = e;
}

template <typename K, bool kIdentity>
__global__ void __launch_bounds__(kThreads, G2_SORT_MINB) onesweep_kernel(const K* __restrict__ kin,
                                                                          const uint32_t* __restrict__ vin,
                                                                          K* __restrict__ kout, uint32_t* __restrict__ vout,
                                                                          size_t n, int shift,
                                                                          const uint32_t* __restrict__ digit_base,
                                                                          uint32_t* __restrict__ status,
                                                                          uint32_t* __restrict__ tile_ctr) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K* skeys = reinterpret_cast<K*>(smem_raw);
    uint32_t* svals = reinterpret_cast<uint32_t*>(smem_raw + sizeof(K) * kTile);
    __shared__ uint32_t whist[kWarps][256];
    __shared__ uint32_t s_lofs[256], s_base[256];
    __shared__ uint32_t s_wtot[kWarps];
    __shared__ uint32_t s_tile;

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    for (int i = tid; i < kWarps * 256; i += kThreads) (&whist[0][0])[i] = 0;
    if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const size_t tile_base = size_t(tile) * kTile;
    const size_t wbase = tile_base + size_t(w) * kWarpItems;
    uint32_t cnt = 0;
    {
        K k[kItems];
        uint32_t v[kItems], d[kItems], r[kItems];
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const size_t idx = wbase + size_t(i) * 32 + lane;
            const bool ok = idx < n;
            k[i] = ok ? kin[idx] : K(0);
            v[i] = kIdentity ? uint32_t(idx) : (ok ? vin[idx] : 0u);
            d[i] = ok ? uint32_t((k[i] >> shift) & 0xff) : 256u;
        }
        const uint32_t lt_mask = (1u << lane) - 1u;
        // peer masks of all items first (independent of the histogram), then the ordered updates
        uint32_t mm[kItems];
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
#if G2_SORT_BALLOT_MATCH
            uint32_t m = 0xffffffffu;
#pragma unroll
            for (int bit = 0; bit < 9; ++bit) {
                const uint32_t bb = __ballot_sync(0xffffffffu, (d[i] >> bit) & 1u);
                m &= ((d[i] >> bit) & 1u) ? bb : ~bb;
            }
            mm[i] = m;
#else
            mm[i] = __match_any_sync(0xffffffffu, d[i]);
#endif
        }
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            const uint32_t m = mm[i];
            const uint32_t before = d[i] < 256u ? whist[w][d[i] & 0xff] : 0u;
            r[i] = before + __popc(m & lt_mask);
            __syncwarp();
            if (d[i] < 256u && lane == __ffs(m) - 1) whist[w][d[i]] = before + __popc(m);
            __syncwarp();
        }
        __syncthreads();
#pragma unroll
        for (int ww = 0; ww < kWarps; ++ww) {
            const uint32_t c = whist[ww][tid];
            whist[ww][tid] = cnt;
            cnt += c;
        }
        // publish this tile's count of digit tid right away: successors can look past it
        os_store(status + size_t(tile) * 256 + tid, (tile == 0 ? kOsInc : kOsAgg) | cnt);
        s_lofs[tid] = block_excl_scan(cnt, s_wtot, nullptr);
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
            if (d[i] < 256u) {
                const uint32_t pos = s_lofs[d[i]] + whist[w][d[i]] + r[i];
                skeys[pos] = k[i];
                svals[pos] = v[i];
            }
        }
    }
    // look back for digit tid: kLookWindow predecessors per step, stop at the first inclusive prefix
    uint32_t excl = 0;
    if (tile > 0) {
        int64_t t = int64_t(tile) - 1;
        bool done = false;
        while (!done) {
            uint32_t x[kLookWindow];
#pragma unroll
            for (int q = 0; q < kLookWindow; ++q)
                x[q] = t - q >= 0 ? os_load(status + size_t(t - q) * 256 + tid) : kOsInc;
#pragma unroll
            for (int q = 0; q < kLookWindow; ++q) {
                if (done) break;
                while ((x[q] >> 30) == 0) x[q] = os_load(status + size_t(t - q) * 256 + tid);
                excl += x[q] & kOsMask;
                done = (x[q] >> 30) == 2;
            }
            t -= kLookWindow;
        }
        os_store(status + size_t(tile) * 256 + tid, kOsInc | (excl + cnt));
    }
    s_base[tid] = digit_base[tid] + excl;
    __syncthreads();
    const uint32_t tile_n = uint32_t(min(size_t(kTile), n - tile_base));
    for (uint32_t p = tid; p < tile_n; p += kThreads) {
        const K kk = skeys[p];
        const uint32_t dd = uint32_t((kk >> shift) & 0xff);
        const uint32_t dst = s_base[dd] + (p - s_lofs[dd]);
        kout[dst] = kk;
        vout[dst] = svals[p];
    }
}

template <typename K>
void set_smem_attr() {
    static bool done = false;
    if (done) return;
    const int bytes = int((sizeof(K) + 4) * kTile);
    G2_CUDA(cudaFuncSetAttribute(scatter_kernel<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    G2_CUDA(cudaFuncSetAttribute(scatter_kernel<K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    G2_CUDA(cudaFuncSetAttribute(onesweep_kernel<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    G2_CUDA(cudaFuncSetAttribute(onesweep_kernel<K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done = true;
}

}  // namespace

template <typename K>
bool radix_sort_onesweep(K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, size_t n, int key_bits,
                         bool identity, SortScratch& sc, cudaStream_t stream) {
    const int passes = (key_bits + 7) / 8;
    const uint32_t tiles = uint32_t((n + kTile - 1) / kTile);
    // scratch: [digit bases: 8 x 256][tile counters: 32][status: passes x tiles x 256]
    const size_t words = 8 * 256 + 32 + size_t(passes) * tiles * 256;
    sc.hist.reserve(words);
    uint32_t* hist = sc.hist.p;
    uint32_t* ctr = hist + 8 * 256;
    uint32_t* status = ctr + 32;
    G2_CUDA(cudaMemsetAsync(hist, 0, words * sizeof(uint32_t), stream));
    const unsigned hgrid = std::max(1u, std::min<unsigned>(unsigned((n + kThreads * 16 - 1) / (kThreads * 16)), 148u * 8u));
    G2_COUNT(1), hist_all_kernel<K><<<hgrid, kThreads, 0, stream>>>(keys, n, passes, hist);
    G2_COUNT(1), digit_base_kernel<<<passes, kThreads, 0, stream>>>(hist);
    K *ki = keys, *ko = keys_alt;
    uint32_t *vi = vals, *vo = vals_alt;
    bool in_alt = false;
    const int smem = int((sizeof(K) + 4) * kTile);
    for (int p = 0; p < passes; ++p) {
        uint32_t* st = status + size_t(p) * tiles * 256;
        if (p == 0 && identity)
            G2_COUNT(1), onesweep_kernel<K, true><<<tiles, kThreads, smem, stream>>>(ki, nullptr, ko, vo, n, 8 * p,
                                                                                    hist + 256 * p, st, ctr + p);
        else
            G2_COUNT(1), onesweep_kernel<K, false><<<tiles, kThreads, smem, stream>>>(ki, vi, ko, vo, n, 8 * p,
                                                                                     hist + 256 * p, st, ctr + p);
        G2_CUDA(cudaGetLastError());
        std::swap(ki, ko);
        std::swap(vi, vo);
        in_alt = !in_alt;
    }
    return in_alt;
}

template <typename K>
bool radix_sort_pairs(K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, size_t n, int key_bits,
                      bool identity, SortScratch& sc, cudaStream_t stream) {
    if (n == 0) return false;
    set_smem_attr<K>();
#if G2_ONESWEEP
    return radix_sort_onesweep<K>(keys, vals, keys_alt, vals_alt, n, key_bits, identity, sc, stream);
#endif
    const int passes = (key_bits + 7) / 8;
    const uint32_t tiles = uint32_t((n + kTile - 1) / kTile);
    const size_t m = size_t(256) * tiles;                       // digit-major (digit, tile) matrix
    const size_t stiles = (m + kThreads * kScanItems - 1) / (kThreads * kScanItems);
    sc.hist.reserve(m);
    sc.status.reserve(2 * stiles + 64);
    uint64_t* status = reinterpret_cast<uint64_t*>(sc.status.p);
    uint32_t* ctr = sc.status.p + 2 * stiles + 32;
    K *ki = keys, *ko = keys_alt;
    uint32_t *vi = vals, *vo = vals_alt;
    bool in_alt = false;
    const int smem = int((sizeof(K) + 4) * kTile);
    for (int p = 0; p < passes; ++p) {
        G2_COUNT(1), count_kernel<K><<<tiles, kThreads, 0, stream>>>(ki, n, 8 * p, sc.hist.p, tiles);
        G2_CUDA(cudaMemsetAsync(sc.status.p, 0, (2 * stiles + 64) * sizeof(uint32_t), stream));
        G2_COUNT(1), scan_kernel<<<unsigned(stiles), kThreads, 0, stream>>>(sc.hist.p, m, status, ctr);
        if (p == 0 && identity)
            G2_COUNT(1), scatter_kernel<K, true><<<tiles, kThreads, smem, stream>>>(ki, nullptr, ko, vo, n, 8 * p,
                                                                                   sc.hist.p, tiles);
        else
            G2_COUNT(1), scatter_kernel<K, false><<<tiles, kThreads, smem, stream>>>(ki, vi, ko, vo, n, 8 * p,
                                                                                    sc.hist.p, tiles);
        G2_CUDA(cudaGetLastError());
        std::swap(ki, ko);
        std::swap(vi, vo);
        in_alt = !in_alt;
    }
    return in_alt;
}

template bool radix_sort_pairs<uint64_t>(uint64_t*, uint32_t*, uint64_t*, uint32_t*, size_t, int, bool, SortScratch&,
                                         cudaStream_t);
template bool radix_sort_pairs<uint32_t>(uint32_t*, uint32_t*, uint32_t*, uint32_t*, size_t, int, bool, SortScratch&,
                                         cudaStream_t);

}  // namespace g2
