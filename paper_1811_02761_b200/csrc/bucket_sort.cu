// Rebuild sort of a Simulation (octree.cpp:60-72 on the resident state), exploiting that the state is
// stored in the previous build's Morton order: the new keys are nearly sorted.  Four launches, no
// host round trip:
//   1. splitters   one CTA: the keys of B evenly spaced storage positions, sorted (bitonic, shared memory)
//   2. scatter     every particle's key (morton.cuh, the key kernel's arithmetic) and bucket -- the
//                  bucket its storage position predicts, checked against the splitters, else searched --
//                  into that bucket's fixed-capacity region (warp-aggregated slot claims)
//   3. offsets     one CTA: exclusive scan of the bucket sizes; a bucket over capacity opens the gate
//   4. local sort  one CTA per bucket: LSD radix sort in shared memory over only the bits that vary
//                  inside the bucket, written to the bucket's output range (coalesced)
// Equal keys may leave in any order: the caller's tie repair (fix_ties_kernel) orders every run of
// equal keys by original id, so the result equals the reference's (key, index) pair sort.  An opened
// gate (a bucket over capacity: a far-from-sorted input such as the first build) makes the local
// sort write the identity order instead; the host sees the gate at the split's synchronisation and
// redoes the ordering with the (key, id) radix sort.
// Traffic: 32 B read + 12 B written per particle (scatter), 12 + 12 B (local sort), against the
// key kernel's 40 B plus 8 x 24 B of the eight onesweep passes.
#include "bucket_sort.cuh"
#include "morton.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace g2 {
namespace {

constexpr uint32_t kSampleChunk = 1024;  // samples per sorting CTA
constexpr uint32_t kOversample = 4;      // samples per bucket
constexpr int kLsItems = 8;                        // keys per thread of a local sort
constexpr int kLsSmall = 256, kLsMid = 512, kLsBig = 1024;  // threads of the three local-sort instances
constexpr uint32_t kSmallCap = kLsSmall * kLsItems;  // 2048: most buckets (mean 2048)
constexpr uint32_t kMidCap = kLsMid * kLsItems;      // 4096
constexpr uint32_t kMaxBig = 64;                   // buckets the large instance takes per sort
static_assert(kLsBig * kLsItems == int(kBucketCap), "the large local sort holds a full bucket region");
constexpr unsigned kFull = 0xffffffffu;
#ifndef G2_LS_WINDOW
#define G2_LS_WINDOW 24
#endif
constexpr int kWindowBits = G2_LS_WINDOW;  // varying key bits the local sort's radix passes cover
constexpr uint32_t kMaxFixRun = 32;         // longest run of window-equal keys the insertion fix-up takes

// ---- 1. splitters -------------------------------------------------------------------------------
// kOversample samples per bucket at evenly spaced storage positions (their NEW keys), sorted by two
// small launches: every CTA bitonic-sorts a chunk of the samples in shared memory, then every sample
// finds its rank among all samples by binary searches in the other sorted chunks (ties: lower chunk
// first), and every kOversample-th ranked sample becomes a splitter.  Oversampling keeps a sample
// displaced far from its storage position (a particle that crossed a high-level cell boundary) from
// widening its bucket by more than a fraction of the mean.
__global__ void __launch_bounds__(kSampleChunk) sample_sort_kernel(const double4* __restrict__ xyzm, uint32_t n,
                                                                   const Cube* __restrict__ cube, uint32_t ns,
                                                                   uint64_t* __restrict__ samples) {
    G2_PDL_WAIT();  // programmatic dependent launch (launch_pdl)
    __shared__ uint64_t s[kSampleChunk];
    __shared__ SpreadTable st;
    spread_init(st);
    const KeyFrame f(*cube);
    const uint32_t chunk = blockDim.x;  // a power of two <= kSampleChunk
    const uint32_t j = blockIdx.x * chunk + threadIdx.x;
    __syncthreads();
    s[threadIdx.x] = f.key(xyzm[uint32_t((uint64_t(2 * j + 1) * n) / (2ull * ns))], st);
    __syncthreads();
    for (uint32_t k = 2; k <= chunk; k <<= 1) {
        for (uint32_t h = k >> 1; h > 0; h >>= 1) {
            const uint32_t i = threadIdx.x, l = i ^ h;
            if (l > i) {
                const uint64_t a = s[i], b = s[l];
                if ((a > b) == ((i & k) == 0)) s[i] = b, s[l] = a;
            }
            __syncthreads();
        }
    }
    samples[j] = s[threadIdx.x];
}

// the rank searches run in shared memory: every CTA stages all ns samples (ns * 8 <= kSplitSmem)
constexpr uint32_t kSplitSmem = 128u * 1024u;
__global__ void __launch_bounds__(kSampleChunk) splitter_kernel(const uint64_t* __restrict__ samples, uint32_t ns,
                                                                uint32_t nb, uint64_t* __restrict__ split,
                                                                uint32_t* __restrict__ cursor, int* gate) {
    G2_PDL_WAIT();  // programmatic dependent launch (launch_pdl)
    extern __shared__ uint64_t all[];
    const uint32_t chunk = blockDim.x, nchunks = ns / chunk;
    const uint32_t j = blockIdx.x * chunk + threadIdx.x;
    if (j == 0) *gate = 0;
    if (j < nb) cursor[j] = 0;
    for (uint32_t i = threadIdx.x; i < ns; i += chunk) all[i] = samples[i];
    __syncthreads();
    const uint64_t x = all[j];
    uint32_t rank = threadIdx.x;  // position inside its own sorted chunk
    for (uint32_t c = 0; c < nchunks; ++c) {
        if (c == blockIdx.x) continue;
        const uint64_t* q = all + size_t(c) * chunk;
        uint32_t lo = 0, hi = chunk;  // count of q[] < x (c after this chunk) or <= x (c before it)
        const bool le = c < blockIdx.x;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (le ? q[mid] <= x : q[mid] < x)
                lo = mid + 1;
            else
                hi = mid;
        }
        rank += lo;
    }
    if (rank % kOversample == 0) split[rank / kOversample] = x;
}

// ---- 2. keys + scatter --------------------------------------------------------------------------
// bucket of x: the largest j with split[j] <= x (0 below split[0]); g is the predicted bucket
__device__ __forceinline__ uint32_t find_bucket(const uint64_t* __restrict__ split, uint32_t nb, uint64_t x,
                                                uint32_t g) {
    uint32_t lo, hi;  // the first index whose splitter exceeds x lies in [lo, hi]
    if (split[g] <= x) {
        if (g + 1 >= nb || split[g + 1] > x) return g;
        lo = g + 2, hi = nb;
    } else {
        if (g == 0) return 0;
        if (split[g - 1] <= x) return g - 1;
        lo = 0, hi = g - 1;
    }
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (split[mid] <= x)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo ? lo - 1 : 0;
}

#ifndef G2_LS_CONCURRENT
#define G2_LS_CONCURRENT 1
#endif
#ifndef G2_SCATTER_MINB
#define G2_SCATTER_MINB 8  // 32 registers: 8 resident 256-thread CTAs per SM (one wave); 1.13 -> 1.07 ms makeTree
#endif
#ifndef G2_SCATTER_ROWS
#define G2_SCATTER_ROWS 2
#endif
constexpr int kScatterRows = G2_SCATTER_ROWS;  // rows of 32 consecutive positions per warp and step: independent chains
__global__ void __launch_bounds__(256, G2_SCATTER_MINB) scatter_kernel(const double4* __restrict__ xyzm, uint32_t n,
                                                      const Cube* __restrict__ cube, uint32_t nb,
                                                      const uint64_t* __restrict__ split, uint32_t* cursor,
                                                      uint64_t* __restrict__ rkeys, uint32_t* __restrict__ rvals,
                                                      int* gate, DevFlags* flags) {
    G2_PDL_WAIT();  // programmatic dependent launch (launch_pdl)
    __shared__ SpreadTable st;
    spread_init(st);
    const KeyFrame f(*cube);
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    // predicted bucket of storage position i: i nb / n, by a multiply (only a starting guess: the
    // splitters check it) instead of a 64-bit division per key
    const double pred = double(nb) / double(n);
    __syncthreads();
    // warp-uniform loop over kScatterRows x 32 consecutive storage positions
    constexpr uint32_t kSpan = 32u * kScatterRows;
    for (uint32_t base = (blockIdx.x * 8u + (threadIdx.x >> 5)) * kSpan; base < n; base += gridDim.x * 8u * kSpan) {
        uint64_t key[kScatterRows];
        uint32_t b[kScatterRows], slot[kScatterRows];
        bool bad = false;
#pragma unroll
        for (int r = 0; r < kScatterRows; ++r) {
            const uint32_t i = base + 32u * r + lane;
            key[r] = 0, b[r] = ~0u;
            if (i < n) {
                const double4 p = xyzm[i];
                bad |= !f.inside(p);
                key[r] = f.key(p, st);
                b[r] = find_bucket(split, nb, key[r], min(uint32_t(double(i) * pred), nb - 1));
            }
        }
        if (bad) flags->data_error = 2;
#pragma unroll
        for (int r = 0; r < kScatterRows; ++r) {
            // nearly sorted input: a row of 32 consecutive positions usually shares one bucket
            const uint32_t b0 = __shfl_sync(kFull, b[r], 0);
            const uint32_t m = __all_sync(kFull, b[r] == b0) ? kFull : __match_any_sync(kFull, b[r]);
            const int leader = __ffs(m) - 1;
            slot[r] = 0;
            if (lane == leader && b[r] != ~0u) slot[r] = atomicAdd(&cursor[b[r]], uint32_t(__popc(m)));
            slot[r] = __shfl_sync(kFull, slot[r], leader) + __popc(m & lt);
        }
#pragma unroll
        for (int r = 0; r < kScatterRows; ++r) {
            if (b[r] == ~0u) continue;
            if (slot[r] < kBucketCap) {
                rkeys[size_t(b[r]) * kBucketCap + slot[r]] = key[r];
                rvals[size_t(b[r]) * kBucketCap + slot[r]] = base + 32u * r + lane;
            } else {
                *gate = 1;  // beyond any local sort's capacity: the caller's id-order sort redoes it
            }
        }
    }
}

// ---- 3. bucket offsets --------------------------------------------------------------------------
// buckets above the small local sort's capacity go to a list for the mid-size one, those above its
// capacity to a list for the large one (at most kMaxBig); more of them, or a bucket above the large
// capacity, open the gate
__global__ void __launch_bounds__(1024) offsets_kernel(const uint32_t* __restrict__ cursor, uint32_t nb,
                                                       uint32_t* __restrict__ offset, uint32_t* __restrict__ big,
                                                       uint32_t* __restrict__ mid, int* gate) {
    G2_PDL_WAIT();  // programmatic dependent launch (launch_pdl)
    __shared__ uint32_t wsum[32];
    __shared__ uint32_t nbig, nmid;
    if (threadIdx.x == 0) nbig = 0, nmid = 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t per = (nb + 1023) / 1024;  // <= 8
    const uint32_t j0 = threadIdx.x * per;
    uint32_t sum = 0;
    for (uint32_t q = 0; q < per; ++q)
        if (j0 + q < nb) sum += cursor[j0 + q];
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        const uint32_t v = wsum[lane];
        uint32_t vi = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, vi, o);
            if (lane >= o) vi += y;
        }
        wsum[lane] = vi - v;
    }
    __syncthreads();
    uint32_t run = wsum[w] + inc - sum;
    for (uint32_t q = 0; q < per; ++q)
        if (j0 + q < nb) {
            const uint32_t c = cursor[j0 + q];
            offset[j0 + q] = run;
            run += c;
            if (c > kMidCap) {
                const uint32_t k = atomicAdd(&nbig, 1u);
                if (k < kMaxBig && c <= kBucketCap)
                    big[1 + k] = j0 + q;
                else
                    *gate = 1;
            } else if (c > kSmallCap) {
                mid[1 + atomicAdd(&nmid, 1u)] = j0 + q;
            }
        }
    __syncthreads();
    if (threadIdx.x == 0) big[0] = nbig, mid[0] = nmid;
}

// ---- 4. local sort -------------------------------------------------------------------------------
// One CTA per bucket: kThreads x 8 keys in registers, LSD passes of 8-bit digits over the bits that
// vary inside the bucket (min ^ max), each pass ranking stably (ballot peer masks, per-warp
// histograms in warp-then-item order) and staging through shared memory.  Rows of 32 keys past the
// bucket's end are skipped warp-uniformly.  kBig: the 1024-thread instance for the listed buckets
// above kSmallCap keys.
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a < b ? b : a; }

template <int kThreads>
struct LsSmem {
    static constexpr int kWarps = kThreads / 32;
    uint64_t keys[kThreads * kLsItems];
    uint32_t vals[kThreads * kLsItems];
    uint32_t whist[kWarps][256];
    uint32_t lofs[256];
    uint32_t wt[8];
    uint64_t mm[2][kWarps];
};

#ifndef G2_LS_MINB
#define G2_LS_MINB 4  // resident 256-thread local sorts per SM (64 registers)
#endif
#ifndef G2_LS_MASKS_FIRST
#define G2_LS_MASKS_FIRST 0
#endif
template <int kThreads, int kKind>  // kKind 0: every bucket up to its capacity; 1 / 2: the mid / big list
__global__ void __launch_bounds__(kThreads, kKind == 2 ? 1 : (kKind == 1 ? 2 : G2_LS_MINB)) local_sort_kernel(const uint64_t* __restrict__ rkeys,
                                                                          const uint32_t* __restrict__ rvals,
                                                                          const uint32_t* __restrict__ cursor,
                                                                          const uint32_t* __restrict__ offset,
                                                                          const uint32_t* __restrict__ big,
                                                                          const int* gate,
                                                                          uint64_t* __restrict__ keys_out,
                                                                          uint32_t* __restrict__ vals_out) {
    G2_PDL_WAIT();  // programmatic dependent launch (launch_pdl)
    constexpr int kWarps = kThreads / 32;
    constexpr uint32_t kCap = uint32_t(kThreads) * kLsItems;
    extern __shared__ __align__(16) unsigned char ls_raw[];
    LsSmem<kThreads>& S = *reinterpret_cast<LsSmem<kThreads>*>(ls_raw);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    uint32_t bkt = blockIdx.x;
    if (kKind) {
        if (*gate || blockIdx.x >= big[0]) return;
        bkt = big[1 + blockIdx.x];
    }
    const uint32_t cnt = cursor[bkt];
    if (cnt == 0) return;
    const uint32_t off = offset[bkt];
    if (!kKind) {
        if (*gate) {
            // the bucket sort failed (a bucket over capacity): the output is the identity order (the
            // caller's state stays as it is) and the host redoes the ordering with the id-order sort
            for (uint32_t q = tid; q < cnt; q += kThreads) keys_out[off + q] = 0, vals_out[off + q] = off + q;
            return;
        }
        if (cnt > kCap) return;  // the mid-size or large instance sorts it
    }
    const uint64_t* rk = rkeys + size_t(bkt) * kBucketCap;
    const uint32_t* rv = rvals + size_t(bkt) * kBucketCap;
    const uint32_t row0 = uint32_t(w) * (32 * kLsItems);
    auto row_live = [&](int i) { return row0 + uint32_t(i) * 32 < cnt; };  // warp-uniform
    uint64_t k[kLsItems];
    uint32_t v[kLsItems];
    uint64_t mn = ~0ull, mx = 0;
#pragma unroll
    for (int i = 0; i < kLsItems; ++i) {
        const uint32_t q = row0 + uint32_t(i) * 32 + lane;
        const bool ok = q < cnt;
        k[i] = ok ? rk[q] : 0ull;
        v[i] = ok ? rv[q] : 0u;
        if (ok) mn = umin64(mn, k[i]), mx = umax64(mx, k[i]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mn = umin64(mn, __shfl_xor_sync(kFull, mn, o));
        mx = umax64(mx, __shfl_xor_sync(kFull, mx, o));
    }
    if (lane == 0) S.mm[0][w] = mn, S.mm[1][w] = mx;
    for (int i = tid; i < kWarps * 256; i += kThreads) (&S.whist[0][0])[i] = 0;
    __syncthreads();
    mn = S.mm[0][0], mx = S.mm[1][0];
#pragma unroll
    for (int q = 1; q < kWarps; ++q) mn = umin64(mn, S.mm[0][q]), mx = umax64(mx, S.mm[1][q]);
    const int nbits = mn == mx ? 0 : 64 - __clzll(static_cast<long long>(mn ^ mx));
    // radix passes over the top kWindowBits varying bits only; keys equal there (rare: ~1e-3 of the
    // neighbours at 2^23) are then ordered by an insertion sort of their run on the full key
    int lowbits = nbits > kWindowBits ? nbits - kWindowBits : 0;
    int passes = (nbits - lowbits + 7) / 8;
    if (passes == 0) {  // one key value: any order (the tie repair orders the run)
#pragma unroll
        for (int i = 0; i < kLsItems; ++i) {
            const uint32_t q = row0 + uint32_t(i) * 32 + lane;
            if (q < cnt) keys_out[off + q] = k[i], vals_out[off + q] = v[i];
        }
        return;
    }
    const uint32_t lt = (1u << lane) - 1u;
    __shared__ int long_run;
    for (int round = 0;; ++round) {
    for (int pass = 0; pass < passes; ++pass) {
        const int shift = lowbits + 8 * pass;
        uint32_t r[kLsItems];
        auto digit = [&](int i) {
            const uint32_t q = row0 + uint32_t(i) * 32 + lane;
            return q < cnt ? uint32_t(k[i] >> shift) & 0xffu : 256u;
        };
        // item by item (stable): peer mask from 9 ballots (the onesweep ranking), then the ordered
        // per-warp histogram update
#if G2_LS_MASKS_FIRST
        uint32_t mm[kLsItems];
#pragma unroll
        for (int i = 0; i < kLsItems; ++i) {
            mm[i] = kFull;
            if (!row_live(i)) continue;
            const uint32_t d = digit(i);
#pragma unroll
            for (int bit = 0; bit < 9; ++bit) {
                const uint32_t bb = __ballot_sync(kFull, (d >> bit) & 1u);
                mm[i] &= ((d >> bit) & 1u) ? bb : ~bb;
            }
        }
#endif
#pragma unroll
        for (int i = 0; i < kLsItems; ++i) {
            r[i] = 0;
            if (!row_live(i)) continue;
            const uint32_t d = digit(i);
#if G2_LS_MASKS_FIRST
            const uint32_t m = mm[i];
#else
            uint32_t m = kFull;
#pragma unroll
            for (int bit = 0; bit < 9; ++bit) {
                const uint32_t bb = __ballot_sync(kFull, (d >> bit) & 1u);
                m &= ((d >> bit) & 1u) ? bb : ~bb;
            }
#endif
            const uint32_t before = d < 256u ? S.whist[w][d & 0xffu] : 0u;
            r[i] = before + __popc(m & lt);
            __syncwarp();
            if (d < 256u && lane == __ffs(m) - 1) S.whist[w][d] = before + __popc(m);
            __syncwarp();
        }
        __syncthreads();
        // per digit: warp-exclusive prefixes, then the digit offsets (exclusive scan over 256 digits)
        if (tid < 256) {
            uint32_t c = 0;
#pragma unroll
            for (int ww = 0; ww < kWarps; ++ww) {
                const uint32_t x = S.whist[ww][tid];
                S.whist[ww][tid] = c;
                c += x;
            }
            uint32_t inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, inc, o);
                if (lane >= o) inc += y;
            }
            if (lane == 31) S.wt[w] = inc;
            S.lofs[tid] = inc - c;
        }
        __syncthreads();
        if (tid < 256) {
            uint32_t wp = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < w) wp += S.wt[q];
            S.lofs[tid] += wp;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kLsItems; ++i)
            if (const uint32_t d = digit(i); d < 256u) {
                const uint32_t pos = S.lofs[d] + S.whist[w][d] + r[i];
                S.keys[pos] = k[i];
                S.vals[pos] = v[i];
            }
        __syncthreads();
        if (pass + 1 < passes) {
#pragma unroll
            for (int i = 0; i < kLsItems; ++i) {
                const uint32_t q = row0 + uint32_t(i) * 32 + lane;
                if (q < cnt) k[i] = S.keys[q], v[i] = S.vals[q];
            }
            for (int i = tid; i < kWarps * 256; i += kThreads) (&S.whist[0][0])[i] = 0;
            __syncthreads();
        }
    }
    if (lowbits == 0) break;
    // runs equal in the sorted window: short ones are insertion-sorted on the full key below; a long
    // one (keys clustered in a small part of a wide bucket) sends the bucket through every pass
    if (tid == 0) long_run = 0;
    __syncthreads();
    for (uint32_t q = tid; q < cnt; q += kThreads) {
        const uint64_t top = S.keys[q] >> lowbits;
        if (q > 0 && (S.keys[q - 1] >> lowbits) == top) continue;
        uint32_t e = q + 1;
        while (e < cnt && e - q <= kMaxFixRun && (S.keys[e] >> lowbits) == top) ++e;
        if (e - q > kMaxFixRun) long_run = 1;
    }
    __syncthreads();
    if (!long_run) break;
    // every bit, from the current (partly sorted) order: LSD needs no particular input order
    lowbits = 0, passes = (nbits + 7) / 8;
#pragma unroll
    for (int i = 0; i < kLsItems; ++i) {
        const uint32_t q = row0 + uint32_t(i) * 32 + lane;
        if (q < cnt) k[i] = S.keys[q], v[i] = S.vals[q];
    }
    for (int i = tid; i < kWarps * 256; i += kThreads) (&S.whist[0][0])[i] = 0;
    __syncthreads();
    }
    if (lowbits > 0) {  // runs equal in the sorted window: insertion sort on the full key (nearly sorted)
        for (uint32_t q = tid; q < cnt; q += kThreads) {
            const uint64_t top = S.keys[q] >> lowbits;
            if (q > 0 && (S.keys[q - 1] >> lowbits) == top) continue;  // not the start of a run
            uint32_t e = q + 1;
            while (e < cnt && (S.keys[e] >> lowbits) == top) ++e;
            for (uint32_t a = q + 1; a < e; ++a) {
                const uint64_t x = S.keys[a];
                const uint32_t xv = S.vals[a];
                uint32_t b = a;
                while (b > q && S.keys[b - 1] > x) {
                    S.keys[b] = S.keys[b - 1];
                    S.vals[b] = S.vals[b - 1];
                    --b;
                }
                S.keys[b] = x;
                S.vals[b] = xv;
            }
        }
        __syncthreads();
    }
    for (uint32_t q = tid; q < cnt; q += kThreads) {
        keys_out[off + q] = S.keys[q];
        vals_out[off + q] = S.vals[q];
    }
}

}  // namespace

uint32_t bucket_count(size_t n) {
    if (n < kBucketMinN || n > kBucketMaxN) return 0;
    uint32_t nb = 1;
    while (size_t(nb) * kBucketTarget < n) nb <<= 1;
    return nb;
}

bool launch_bucket_sort(const double4* xyzm, size_t n, const Cube* cube, BucketScratch& sc, uint64_t* keys_out,
                        uint32_t* vals_out, DevFlags* flags, cudaStream_t s) {
    const uint32_t nb = bucket_count(n);
    if (!nb) return false;
    sc.split.reserve(nb), sc.cursor.reserve(nb), sc.offset.reserve(nb), sc.gate.reserve(1);
    sc.rkeys.reserve(size_t(nb) * kBucketCap), sc.rvals.reserve(size_t(nb) * kBucketCap);
    static bool attr = false;
    if (!attr) {
        G2_CUDA(cudaFuncSetAttribute(local_sort_kernel<kLsSmall, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(sizeof(LsSmem<kLsSmall>))));
        G2_CUDA(cudaFuncSetAttribute(local_sort_kernel<kLsMid, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(sizeof(LsSmem<kLsMid>))));
        G2_CUDA(cudaFuncSetAttribute(local_sort_kernel<kLsBig, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(sizeof(LsSmem<kLsBig>))));
        G2_CUDA(cudaFuncSetAttribute(splitter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSplitSmem)));
        attr = true;
    }
    const uint32_t n32 = uint32_t(n), ns = nb * kOversample;
    const uint32_t chunk = std::min(ns, kSampleChunk);
    sc.samples.reserve(ns);
    sc.big.reserve(kMaxBig + 1);
    sc.mid.reserve(nb + 1);
    G2_COUNT(1), launch_pdl(sample_sort_kernel, dim3(ns / chunk), dim3(chunk), size_t(0), s, xyzm, n32, cube, ns, sc.samples.p);
    G2_COUNT(1), launch_pdl(splitter_kernel, dim3(ns / chunk), dim3(chunk), size_t(ns * sizeof(uint64_t)), s, sc.samples.p, ns, nb, sc.split.p,
                                                                                   sc.cursor.p, sc.gate.p);
    const unsigned grid = std::max(1u, std::min<unsigned>(ceil_div(n, 256), kNumSMs * 8));
    G2_COUNT(1), launch_pdl(scatter_kernel, dim3(grid), dim3(256), size_t(0), s, xyzm, n32, cube, nb, sc.split.p, sc.cursor.p, sc.rkeys.p,
                                                      sc.rvals.p, sc.gate.p, flags);
    G2_COUNT(1), launch_pdl(offsets_kernel, dim3(1), dim3(1024), size_t(0), s, sc.cursor.p, nb, sc.offset.p, sc.big.p, sc.mid.p, sc.gate.p);
    static const bool dbg = std::getenv("G2_BUCKET_DEBUG") != nullptr;  // development: bucket sizes
    if (dbg) {
        std::vector<uint32_t> c(nb);
        std::vector<uint64_t> sp(nb);
        G2_CUDA(cudaMemcpyAsync(c.data(), sc.cursor.p, nb * 4, cudaMemcpyDeviceToHost, s));
        G2_CUDA(cudaMemcpyAsync(sp.data(), sc.split.p, nb * 8, cudaMemcpyDeviceToHost, s));
        G2_CUDA(cudaStreamSynchronize(s));
        uint32_t mx = 0, over = 0, empty = 0;
        for (uint32_t j = 0; j < nb; ++j) mx = std::max(mx, c[j]), over += c[j] > kBucketCap, empty += c[j] == 0;
        std::fprintf(stderr, "[g2 bucket] n %zu buckets %u max %u over-capacity %u empty %u\n", n, nb, mx, over, empty);
        for (uint32_t j = 0; j < nb; ++j)
            if (c[j] > kBucketCap)
                std::fprintf(stderr, "  bucket %u size %u split %016llx next %016llx\n", j, c[j],
                             (unsigned long long)sp[j], (unsigned long long)(j + 1 < nb ? sp[j + 1] : ~0ull));
    }
    // the instances touch disjoint buckets: the few large buckets (one SM each) and the mid-size ones
    // run beside the bulk of small ones instead of as serial tails
    cudaStream_t s_mid = s, s_big = s;
    if (G2_LS_CONCURRENT) {
        if (!sc.fork) {
            G2_CUDA(cudaEventCreateWithFlags(&sc.fork, cudaEventDisableTiming));
            for (int k = 0; k < 2; ++k) {
                G2_CUDA(cudaStreamCreateWithFlags(&sc.side[k], cudaStreamNonBlocking));
                G2_CUDA(cudaEventCreateWithFlags(&sc.join[k], cudaEventDisableTiming));
            }
        }
        G2_CUDA(cudaEventRecord(sc.fork, s));
        for (auto x : sc.side) G2_CUDA(cudaStreamWaitEvent(x, sc.fork, 0));
        s_big = sc.side[0], s_mid = sc.side[1];
    }
    G2_COUNT(1), local_sort_kernel<kLsBig, 2><<<kMaxBig, kLsBig, sizeof(LsSmem<kLsBig>), s_big>>>(
        sc.rkeys.p, sc.rvals.p, sc.cursor.p, sc.offset.p, sc.big.p, sc.gate.p, keys_out, vals_out);
    G2_COUNT(1), local_sort_kernel<kLsMid, 1><<<nb, kLsMid, sizeof(LsSmem<kLsMid>), s_mid>>>(
        sc.rkeys.p, sc.rvals.p, sc.cursor.p, sc.offset.p, sc.mid.p, sc.gate.p, keys_out, vals_out);
    G2_COUNT(1), launch_pdl(local_sort_kernel<kLsSmall, 0>, dim3(nb), dim3(kLsSmall), size_t(sizeof(LsSmem<kLsSmall>)), s, 
        sc.rkeys.p, sc.rvals.p, sc.cursor.p, sc.offset.p, sc.big.p, sc.gate.p, keys_out, vals_out);
    if (G2_LS_CONCURRENT)
        for (int k = 0; k < 2; ++k) {
            G2_CUDA(cudaEventRecord(sc.join[k], sc.side[k]));
            G2_CUDA(cudaStreamWaitEvent(s, sc.join[k], 0));
        }
    G2_CUDA(cudaGetLastError());
    return true;
}

}  // namespace g2
