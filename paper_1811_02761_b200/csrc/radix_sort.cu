// Onesweep LSD radix sort (see radix_sort.cuh).
#include "radix_sort.cuh"

namespace g2 {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;                      // keys per thread
constexpr int kTile = kThreads * kItems;        // 4096 keys per tile
constexpr int kWarpItems = 32 * kItems;         // 512 consecutive keys per warp
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagInc = 2u << 30;
constexpr uint32_t kValMask = (1u << 30) - 1;

template <typename K>
__global__ void __launch_bounds__(kThreads) histogram_kernel(const K* __restrict__ keys, size_t n, int passes,
                                                              uint32_t* __restrict__ hist) {
    __shared__ uint32_t sh[8][256];
    for (int i = threadIdx.x; i < 8 * 256; i += kThreads) (&sh[0][0])[i] = 0;
    __syncthreads();
    for (size_t i = blockIdx.x * size_t(kThreads) + threadIdx.x; i < n; i += size_t(gridDim.x) * kThreads) {
        const K k = keys[i];
        for (int p = 0; p < passes; ++p) atomicAdd(&sh[p][(k >> (8 * p)) & 0xff], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * 256; i += kThreads) {
        const uint32_t v = (&sh[0][0])[i];
        if (v) atomicAdd(&hist[i], v);
    }
}

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

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

template <typename K, bool kIdentity>
__global__ void __launch_bounds__(kThreads) onesweep_kernel(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                             K* __restrict__ kout, uint32_t* __restrict__ vout,
                                                             size_t n, int shift, const uint32_t* __restrict__ hist,
                                                             uint32_t* __restrict__ status,
                                                             uint32_t* __restrict__ tile_counter) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    K* skeys = reinterpret_cast<K*>(smem_raw);
    uint32_t* svals = reinterpret_cast<uint32_t*>(smem_raw + sizeof(K) * kTile);
    __shared__ uint32_t whist[kWarps][256];
    __shared__ uint32_t s_lofs[256], s_base[256];
    __shared__ uint32_t s_wtot[kWarps];
    __shared__ uint32_t s_tile;

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
    for (int i = tid; i < kWarps * 256; i += kThreads) (&whist[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
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
    // per digit (thread = digit): exclusive prefix across warps, tile count
    uint32_t cnt = 0;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) {
        const uint32_t c = whist[ww][tid];
        whist[ww][tid] = cnt;
        cnt += c;
    }
    const uint32_t lofs = block_excl_scan(cnt, s_wtot, nullptr);
    s_lofs[tid] = lofs;
    __syncthreads();
    // global digit base for this pass
    const uint32_t hbase = block_excl_scan(hist[tid], s_wtot + 0, nullptr);
    // decoupled look-back, one chain per digit
    uint32_t* st = status + size_t(tile) * 256 + tid;
    uint32_t excl = 0;
    if (tile == 0) {
        st_relaxed(st, kFlagInc | cnt);
    } else {
        st_relaxed(st, kFlagAgg | cnt);
        for (int64_t j = int64_t(tile) - 1; j >= 0; --j) {
            uint32_t s;
            do {
                s = ld_relaxed(status + size_t(j) * 256 + tid);
            } while ((s & ~kValMask) == 0);
            excl += s & kValMask;
            if (s & kFlagInc) break;
        }
        st_relaxed(st, kFlagInc | (excl + cnt));
    }
    s_base[tid] = hbase + excl;
    __syncthreads();
    // scatter into shared memory in digit order
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

template <typename K>
void set_smem_attr() {
    static bool done = false;
    if (done) return;
    const int bytes = int((sizeof(K) + 4) * kTile);
    G2_CUDA(cudaFuncSetAttribute(onesweep_kernel<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    G2_CUDA(cudaFuncSetAttribute(onesweep_kernel<K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done = true;
}

}  // namespace

template <typename K>
bool radix_sort_pairs(K* keys, uint32_t* vals, K* keys_alt, uint32_t* vals_alt, size_t n, int key_bits,
                      bool identity, SortScratch& sc, cudaStream_t stream) {
    if (n == 0) return false;
    set_smem_attr<K>();
    const int passes = (key_bits + 7) / 8;
    const size_t tiles = (n + kTile - 1) / kTile;
    sc.hist.reserve(8 * 256);
    sc.status.reserve(tiles * 256 + 32);
    G2_CUDA(cudaMemsetAsync(sc.hist.p, 0, 8 * 256 * sizeof(uint32_t), stream));
    const unsigned hgrid = std::min<unsigned>(ceil_div(n, kThreads * 8), kNumSMs * 8);
    G2_COUNT(1), histogram_kernel<K><<<hgrid, kThreads, 0, stream>>>(keys, n, passes, sc.hist.p);
    G2_CUDA(cudaGetLastError());
    K *ki = keys, *ko = keys_alt;
    uint32_t *vi = vals, *vo = vals_alt;
    bool in_alt = false;
    const int smem = int((sizeof(K) + 4) * kTile);
    uint32_t* counter = sc.status.p + tiles * 256;
    for (int p = 0; p < passes; ++p) {
        G2_CUDA(cudaMemsetAsync(sc.status.p, 0, (tiles * 256 + 32) * sizeof(uint32_t), stream));
        if (p == 0 && identity)
            G2_COUNT(1), onesweep_kernel<K, true><<<unsigned(tiles), kThreads, smem, stream>>>(ki, nullptr, ko, vo, n, 8 * p,
                                                                                 sc.hist.p + 256 * p, sc.status.p,
                                                                                 counter);
        else
            G2_COUNT(1), onesweep_kernel<K, false><<<unsigned(tiles), kThreads, smem, stream>>>(ki, vi, ko, vo, n, 8 * p,
                                                                                  sc.hist.p + 256 * p, sc.status.p,
                                                                                  counter);
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
