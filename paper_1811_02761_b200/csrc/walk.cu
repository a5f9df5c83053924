// walkTree on sm_100a: warp-specialised sink-group traversal with
// double-buffered interaction lists, acceleration MAC and FP32 rsqrt flush.
//
// Reference semantics (traversal.cpp:16-156, engine.cpp:31-81):
//   * sinks in Morton-rank order are chunked into groups of group_size; each
//     group gets an AABB-centred bounding sphere and a_min (make_group);
//   * a cell is tested iff its parent was tested and rejected, so the set of
//     MAC evaluations, accepted cells and opened leaves does not depend on the
//     visiting order; events (interactions, mac_evals, list_pushes) are
//     therefore reproduced exactly by any order, and accelerations differ only
//     by FP32 summation order;
//   * MAC decisions equal the reference's FP64 ones: an FP32 screen with
//     rigorous error margins decides, the FP64 expression settles the rest.
//
// Execution model (per CTA: kPairs producer/consumer warp pairs):
//   * a PRODUCER warp runs one task (group, subtree root) at a time: it pops
//     32 cells per round from a depth-first stack (shared top, global spill
//     bottom), screens them, pushes children and writes list entries (FP32,
//     relative to the group centre) into one of two shared list buffers;
//   * its CONSUMER warp (lane l = sink l) flushes each full buffer into its
//     FP32 accumulators: every entry acts on every sink (flush_list,
//     traversal.cpp:61-84); buffers change hands through shared mbarriers,
//     so traversal latency and the FP32/MUFU-bound flush overlap, and each
//     side keeps its registers for its own work (ILP in the flush);
//   * persistent grid, dynamic task queue: initially one task per group; a
//     producer holding a long stack donates its shallowest pending cells as
//     (group, cells) batches, which split the heavy-tailed "whole-system"
//     groups across warps;
//   * deterministic results: WHEN a task donates depends only on the task's own
//     progress (every kDonateEvery rounds), so a group's task tree is a function of
//     the group and the tree alone; each task's partial sums land in its record and
//     a task's subtree total = own partial + children's totals in donation order,
//     formed by whichever of them finishes last.  Accelerations are therefore
//     bit-identical run to run and for any sharding of the groups over ranks
//     (the reference's static partition, parallel.hpp:16-19).
#include <cfloat>
#include <cstdlib>

#include "kernels.cuh"

namespace g2 {
namespace {

// Occupancy: 5 CTAs x 8 warps per SM.  The launch budget is 48 registers per thread; setmaxnreg
// then moves 8 per thread from the consumer warpgroup (40: the flush is register-light) to the
// producer warpgroup (56: the traversal is latency-bound and spills less).  Five CTAs fit the
// 228 KB of shared memory with 256-entry list buffers.  Measured at 2^23 all-active: 14.13 ms vs
// 14.50 ms for 4 CTAs x 64 registers with 336-entry buffers.
#ifndef G2_PRODUCER_REGS  // setmaxnreg split of the register budget between the two warpgroups
#define G2_PRODUCER_REGS 56
#define G2_CONSUMER_REGS 40
#endif
constexpr int kPairs = 4;                  // producer/consumer warp pairs per CTA
constexpr int kThreads = 64 * kPairs;      // producers are warps 0..kPairs-1, consumers kPairs..2kPairs-1
#ifndef G2_WALK_MINB
#define G2_WALK_MINB 5  // resident CTAs per SM the register budget is tuned for
#endif
#ifndef G2_LCAP
#define G2_LCAP 256     // >= 256: the per-slot overflow path writes one round's cell slot at a time
#endif
constexpr int kLcap = G2_LCAP;             // interaction-list entries per buffer
// With few groups (small block-step active sets) the fifth CTA per SM only adds contention to the
// draining tail: CTAs beyond 4 per SM then exit at once.
#ifndef G2_DENSE_MIN_GROUPS
#define G2_DENSE_MIN_GROUPS 12288
#endif
constexpr int kScap = 512;                 // shared stack entries per producer (>= 64 cells x 8 children)
constexpr uint32_t kSpillWords = 16384;    // global stack entries per producer
#ifndef G2_DONATE_MIN_LIVE
#define G2_DONATE_MIN_LIVE 2
#endif
constexpr int kDonateMinLive = G2_DONATE_MIN_LIVE;  // pending cells a task needs before it donates half
#ifndef G2_DONATE_BACKOFF
#define G2_DONATE_BACKOFF 0  // > 0: the interval between a task's donations doubles every that many donations
#endif
#ifndef G2_DONATE_BATCHES
#define G2_DONATE_BATCHES 2
#endif
constexpr int kMaxBatches = G2_DONATE_BATCHES;       // donated batches (tasks) of 32 cells per donation
constexpr uint32_t kNone = ~0u;             // no task record / no child / no parent
constexpr uint64_t kEmpty = ~0ull;
constexpr uint64_t kGenMask = (1ull << 26) - 1;  // generation tag of a slot (ticket >> ring bits)
constexpr unsigned kFull = 0xffffffffu;
constexpr uint32_t kFirst = 1, kLast = 2;  // buffer header flags: first / last buffer of a task
// whole-system groups run as slices (one per root child), the same slices for any rank count
constexpr uint32_t kMaxHeavy = 128;         // heavy groups per walk (more candidates: no slicing)
constexpr uint32_t kSlicesPer = 8;          // slice slots per heavy group (<= root children)
#ifndef G2_HEAVY_FRAC
#define G2_HEAVY_FRAC 0.25
#endif
#ifndef G2_SLICE_CONSUMER
#define G2_SLICE_CONSUMER 1  // (A/B: 0 drops the slice path from the consumer -- wrong results with slices)
#endif
constexpr double kHeavyFrac = G2_HEAVY_FRAC;  // heavy: sphere radius >= kHeavyFrac x the root's extent
constexpr uint32_t kSliceTag = 0xC0000000u; // task-record parent tag of a slice's root record (| slice index)
constexpr uint32_t kStop = ~0u;            // header group id that retires the consumer

// Interaction list in pair-interleaved layout so the flush runs on packed
// f32x2 math (FADD2/FFMA2/FMUL2): entries 2p and 2p+1 live in
//   la[p] = (x_2p, x_2p+1, y_2p, y_2p+1),  lb[p] = (z_2p, z_2p+1, m_2p, m_2p+1).
struct ListBuf {
    float4 la[kLcap / 2];
    float4 lb[kLcap / 2];
};
struct alignas(16) PairSmem {
    ListBuf buf[2];
    uint32_t stack[kScap];
    float4 leaf[64];      // per popped cell: (leaf com - group centre, first particle) of an opened leaf
    uint32_t hdr[2][4];   // per buffer: entry count, group, flags
    uint64_t full[2];     // mbarriers: buffer written (producer -> consumer)
    uint64_t empty[2];    // mbarriers: buffer flushed (consumer -> producer)
};

__device__ __forceinline__ float* entry_ptr(ListBuf& lb, int pos) {
    return reinterpret_cast<float*>(lb.la) + 2 * (pos & ~1) + (pos & 1);
}
// entry pos: x, y at la[pos/2] lanes (pos&1) and 2 + (pos&1); z, m likewise in lb
__device__ __forceinline__ void put_entry(ListBuf& lb, int pos, float x, float y, float z, float m) {
    float* a = entry_ptr(lb, pos);
    a[0] = x, a[2] = y, a[2 * kLcap] = z, a[2 * kLcap + 2] = m;
}
// Opened-leaf particles are staged as (owner lane | j << 5) in the m slot of
// their own list entry, then each lane replaces the slot(s) it owns by the entry.
__device__ __forceinline__ void put_index(ListBuf& lb, int pos, uint32_t k) {
    reinterpret_cast<uint32_t*>(entry_ptr(lb, pos))[2 * kLcap + 2] = k;
}
__device__ __forceinline__ uint32_t get_index(ListBuf& lb, int pos) {
    return reinterpret_cast<const uint32_t*>(entry_ptr(lb, pos))[2 * kLcap + 2];
}

// ---- shared-memory mbarriers (one phase per buffer hand-over, all 32 lanes arrive)
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    const uint32_t a = smem_addr(bar);
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!ok);
}
// The consumer's wait for a full buffer: a waiting consumer must not spin on the issue slots its
// producer needs (a plain try_wait loop was 20 % of the walk's instructions).  G2_MBAR_HINT > 0: the
// try_wait suspends up to that many ns (it wakes when the phase completes); G2_MBAR_SLEEP > 0:
// test_wait with __nanosleep back-off between polls.
#ifndef G2_MBAR_HINT
#define G2_MBAR_HINT 0
#endif
#ifndef G2_MBAR_SLEEP
#define G2_MBAR_SLEEP 0
#endif
__device__ __forceinline__ void mbar_wait_idle(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_addr(bar);
    uint32_t ok = 0;
#if G2_MBAR_SLEEP
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    while (!ok) {
        __nanosleep(G2_MBAR_SLEEP);
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                     : "=r"(ok) : "r"(a), "r"(parity) : "memory");
    }
#elif G2_MBAR_HINT
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity), "n"(G2_MBAR_HINT)
            : "memory");
    } while (!ok);
#else
    (void)ok;
    mbar_wait(bar, parity);
#endif
}

// ---- packed f32x2 helpers (sm_100a PTX) --------------------------------------
using f2 = unsigned long long;
__device__ __forceinline__ f2 pk(float lo, float hi) {
    f2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void upk(f2 v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
    f2 d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
    f2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
    f2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
    f2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ float rcp_ftz(float x) {  // one MUFU.RCP
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float rsqrt_ftz(float x) {  // one MUFU.RSQ, no denormal fix-up
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// one 256-bit load per node record, one 128-bit load per leaf particle (read-only path)
__device__ __forceinline__ WNode32 ld_node32(const WNode32* p) {
    uint32_t w[8];
    asm("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
        : "l"(p));
    return WNode32{__uint_as_float(w[0]), __uint_as_float(w[1]), __uint_as_float(w[2]), __uint_as_float(w[3]),
                   __uint_as_float(w[4]), __uint_as_float(w[5]), w[6], w[7]};
}
__device__ __forceinline__ float4 ld_rel(const float4* p) { return __ldg(p); }

__device__ __forceinline__ uint32_t ld_vol(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t ld_vol64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t ld_acq64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel64(uint64_t* p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_vol64(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t x, uint32_t& total) {
    const int lane = threadIdx.x & 31;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += y;
    }
    total = __shfl_sync(kFull, inc, 31);
    return inc - x;
}

// All-pairs burst: every list entry acts on this lane's sink (flush_list,
// traversal.cpp:61-84).  27 Flop per interaction by the reference convention.
// Entries are processed two pairs at a time on packed f32x2 lanes (two
// independent dependency chains per iteration); accumulators are pairs that
// are folded at the end.  cnt is even (the producer pads with (0,0,0,m=0)).
struct Acc2 {
    f2 x, y, z;
    float ph;
};

// kGuard: eps^2 rounds below FLT_MIN in FP32 (eps == 0 included): a zero separation (the self pair,
// or coincident particles) contributes nothing (traversal.cpp:73).  kPot: the potential term is
// dropped exactly when the UN-softened separation is zero, |d|^2 == 0 (traversal.cpp:78), not when
// r^2 rounds to eps^2.  Both need |d|^2 on its own; the plain force path folds eps^2 into the chain.
template <bool kPot, bool kGuard>
__device__ __forceinline__ void pair_force(const ulonglong2 A, const ulonglong2 B, f2 sx, f2 sy, f2 sz, f2 eps2,
                                           Acc2& a) {
    const f2 dx = sub2(A.x, sx), dy = sub2(A.y, sy), dz = sub2(B.x, sz);
    f2 r2, d2 = 0;
    if (kPot || kGuard) {
        d2 = mul2(dx, dx);
        d2 = fma2(dy, dy, d2);
        d2 = fma2(dz, dz, d2);
        r2 = kGuard ? d2 : add2(d2, eps2);
    } else {
        r2 = fma2(dx, dx, eps2);
        r2 = fma2(dy, dy, r2);
        r2 = fma2(dz, dz, r2);
    }
    float r0, r1, q0 = 0.f, q1 = 0.f;
    upk(r2, r0, r1);
    if (kPot || kGuard) upk(d2, q0, q1);
    float i0 = rsqrt_ftz(r0), i1 = rsqrt_ftz(r1);
    if (kGuard) {
        i0 = q0 > 0.0f ? i0 : 0.0f;
        i1 = q1 > 0.0f ? i1 : 0.0f;
    }
    const f2 inv = pk(i0, i1);
    const f2 mi = mul2(B.y, inv);
    const f2 f = mul2(mi, mul2(inv, inv));
    a.x = fma2(f, dx, a.x);
    a.y = fma2(f, dy, a.y);
    a.z = fma2(f, dz, a.z);
    if (kPot) {
        float m0, m1;
        upk(mi, m0, m1);
        a.ph -= (q0 > 0.0f ? m0 : 0.0f) + (q1 > 0.0f ? m1 : 0.0f);
    }
}

template <bool kPot, bool kEps0>
__device__ __forceinline__ void flush_list(const ListBuf& lb, int cnt, f2 sx, f2 sy, f2 sz, f2 eps2, Acc2& a,
                                           Acc2& b) {
    const int np = cnt >> 1;
    const ulonglong2* pa = reinterpret_cast<const ulonglong2*>(lb.la);
    const ulonglong2* pb = reinterpret_cast<const ulonglong2*>(lb.lb);
    int p = 0;
#pragma unroll 4  // 8 entry pairs in flight per iteration group: 13.93 vs 14.10 ms (unroll 2) at 2^23
    for (; p + 1 < np; p += 2) {
        const ulonglong2 A0 = pa[p], B0 = pb[p], A1 = pa[p + 1], B1 = pb[p + 1];
        pair_force<kPot, kEps0>(A0, B0, sx, sy, sz, eps2, a);
        pair_force<kPot, kEps0>(A1, B1, sx, sy, sz, eps2, b);
    }
    if (p < np) pair_force<kPot, kEps0>(pa[p], pb[p], sx, sy, sz, eps2, a);
}

// Exact FP64 MAC in the reference's operation order (traversal.cpp:40-56).
__device__ __forceinline__ bool mac_exact(const WNode& nd, const GroupRec& g, const WalkParams& p, double rhs,
                                          bool geom) {
    const double dx = dsub(g.cx, nd.cx), dy = dsub(g.cy, nd.cy), dz = dsub(g.cz, nd.cz);
    const double d = smax(0.0, dsub(dsqrt(norm2(dx, dy, dz)), g.radius));
    if (d <= 0.0) return false;
    if (geom) return nd.extent <= dmul(p.theta, d);
    const double d2 = dmul(d, d);
    const double lhs = ddiv(dmul(dmul(dmul(p.G, nd.mass), nd.extent), nd.extent), dmul(d2, d2));
    return lhs <= rhs;
}

// FP32 MAC screen of one cell against the group (FP32 centre split hi + lo), with
// rigorous error margins; the exact FP64 expression settles undecided cells.
struct Screen {
    float fx, fy, fz, fm;  // group centre - node centre (FP32), node mass
    uint32_t link, info;
    bool accept;
    __device__ __forceinline__ bool leaf() const { return (info & kLeafBit) != 0; }
    __device__ __forceinline__ uint32_t nchild() const { return (!accept && !leaf()) ? (info & 0xffu) : 0u; }
    __device__ __forceinline__ uint32_t nleaf() const { return (!accept && leaf()) ? (info & ~kLeafBit) : 0u; }
};

// The FP64 group record is re-read only for undecided cells (rare), so the traversal loop does
// not hold its 12 registers.
__device__ __forceinline__ Screen screen(const TreeView& t, const GroupRec* gp, const WalkParams& p, uint32_t c,
                                         bool valid, float gxh, float gyh, float gzh, float gxl, float gyl, float gzl,
                                         float tolc, float radf, float rhsf, float G, float thetaf, bool geom) {
    Screen s{0.f, 0.f, 0.f, 0.f, 0u, 0u, false};
    if (!valid) return s;  // info 0: internal with no children, not accepted -> contributes nothing
    const WNode32 nd = ld_node32(t.nodes32 + c);
    s.link = nd.link, s.info = nd.info, s.fm = nd.m;
    s.fx = (gxh - nd.cx) + gxl, s.fy = (gyh - nd.cy) + gyl, s.fz = (gzh - nd.cz) + gzl;
    const float S = fmaf(s.fx, s.fx, fmaf(s.fy, s.fy, s.fz * s.fz));
    const float D = S > 0.f ? S * rsqrt_ftz(S) : 0.f;
    const float d32 = D - radf;
    // |d32 - d_fp64| <= ~6e-7 (D + R) + 2.4e-7 (|gx|+|gy|+|gz|): 7x / 2x margins
    const float tolabs = fmaf(4e-6f, D + radf, tolc);
    int verdict = 2;  // 0 reject, 1 accept, 2 undecided
    if (d32 <= -tolabs) {
        verdict = 0;  // d <= 0: descend (traversal.cpp:46)
    } else if (d32 > tolabs) {
        const float rel = tolabs * rcp_ftz(d32);
        if (geom) {
            const float r = thetaf * d32, tol = rel + 1e-6f;
            verdict = nd.b <= r * (1.f - tol) ? 1 : (nd.b > r * (1.f + tol) ? 0 : 2);
        } else {
            // G m b^2 / d^4 <= rhs  <=>  G m b^2 <= rhs d^4  (no division)
            const float d2 = d32 * d32;
            const float num = G * nd.q, den = rhsf * (d2 * d2);
            const float tol = 4.f * rel + 1e-5f;
            if (tol < 0.25f && den > 1e-30f)
                verdict = num <= den * (1.f - tol) ? 1 : (num > den * (1.f + tol) ? 0 : 2);
        }
    }
    if (verdict == 2) {
        const GroupRec g = *gp;
        verdict = mac_exact(t.nodes[c], g, p, dmul(p.dacc, g.a_min), geom) ? 1 : 0;
    }
    s.accept = verdict == 1;
    return s;
}

template <bool kPot, bool kEps0, bool kCheck>
__global__ void __launch_bounds__(kThreads, G2_WALK_MINB) walk_kernel(TreeView t, WalkParams p, WalkBuffers b, DevFlags* flags) {
    G2_PDL_WAIT();  // programmatic dependent launch (launch_pdl)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    PairSmem* const pairs = reinterpret_cast<PairSmem*>(smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (blockIdx.x >= 4u * kNumSMs && b.qstate[3] < uint32_t(G2_DENSE_MIN_GROUPS)) return;  // whole CTA
    if (threadIdx.x < kPairs) {
        PairSmem& ps = pairs[threadIdx.x];
        for (int i = 0; i < 2; ++i) mbar_init(&ps.full[i], 32), mbar_init(&ps.empty[i], 32);
    }
    __syncthreads();
    const float G = float(p.G);

    if (warp >= kPairs) {
        // ================================ consumer: flush buffers into the sinks' accumulators
#if G2_CONSUMER_REGS
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(G2_CONSUMER_REGS));
#endif
        PairSmem& ps = pairs[warp - kPairs];
        const float eps2 = float(p.eps * p.eps);
        const f2 e2 = pk(eps2, eps2);
        f2 sx2 = 0, sy2 = 0, sz2 = 0;
        Acc2 a0{0ull, 0ull, 0ull, 0.f}, a1{0ull, 0ull, 0ull, 0.f};
        uint32_t gfirst = 0;
        bool has_sink = false;
        for (uint32_t it = 0;; ++it) {
            const int bi = int(it & 1);
            mbar_wait_idle(&ps.full[bi], (it >> 1) & 1);
            const uint32_t cnt = ps.hdr[bi][0], grp = ps.hdr[bi][1], fl = ps.hdr[bi][2], rec = ps.hdr[bi][3];
            if (grp == kStop) break;
            if (fl & kFirst) {
                // sinks by the SAME FP32 expression as their own list entries, (leaf centre - group
                // centre) + rel: the self pair then has dx == 0 exactly (with eps > 0 any residue
                // would act as m dx / eps^3; with eps == 0 the r2 == 0 skip needs it)
                const GroupRec g = b.groups[grp];
                const float gxh = float(g.cx), gyh = float(g.cy), gzh = float(g.cz);
                const float gxl = float(dsub(g.cx, double(gxh))), gyl = float(dsub(g.cy, double(gyh))),
                            gzl = float(dsub(g.cz, double(gzh)));
                has_sink = uint32_t(lane) < g.count;
                gfirst = g.first;
                float sx = 0.f, sy = 0.f, sz = 0.f;
                if (has_sink) {
                    const uint32_t k = b.sinks[g.first + lane];
                    const WNode32 lf = ld_node32(t.nodes32 + t.leaf_of[k]);
                    const float4 r = ld_rel(t.rel + k);
                    sx = -((gxh - lf.cx) + gxl) + r.x;
                    sy = -((gyh - lf.cy) + gyl) + r.y;
                    sz = -((gzh - lf.cz) + gzl) + r.z;
                }
                sx2 = pk(sx, sx), sy2 = pk(sy, sy), sz2 = pk(sz, sz);
                a0 = Acc2{0ull, 0ull, 0ull, 0.f}, a1 = a0;
            }
            flush_list<kPot, kEps0>(ps.buf[bi], int(cnt), sx2, sy2, sz2, e2, a0, a1);
            __syncwarp();
            mbar_arrive(&ps.empty[bi]);
            if (!(fl & kLast)) continue;
            // ---- the task is complete: fold the packed accumulators (fixed order)
            float x0, x1, y0, y1, z0, z1, u0, u1, v0, v1, w0, w1;
            upk(a0.x, x0, x1), upk(a0.y, y0, y1), upk(a0.z, z0, z1);
            upk(a1.x, u0, u1), upk(a1.y, v0, v1), upk(a1.z, w0, w1);
            float4 tot = make_float4((x0 + x1) + (u0 + u1), (y0 + y1) + (v0 + v1), (z0 + z1) + (w0 + w1),
                                     kPot ? a0.ph + a1.ph : 0.f);
            bool done = true;  // tot is the group's final sum
            if (rec != kNone) {
                // split group: park the partial in the record; whoever completes a record's subtree
                // last adds the children's totals in donation order and climbs to the parent
                if (has_sink) __stcg(&b.tacc[size_t(rec) * 32 + lane], tot);
                __threadfence();
                __syncwarp();
                uint32_t r = rec, last = 0;
                if (lane == 0) last = atomicSub(&b.trec[r].y, 1u) == 1u;
                last = __shfl_sync(kFull, last, 0);
                done = false;
                while (last) {
                    __threadfence();
                    const uint4 R = __ldcg(&b.trec[r]);
                    float4 acc = has_sink ? __ldcg(&b.tacc[size_t(r) * 32 + lane]) : make_float4(0.f, 0.f, 0.f, 0.f);
                    for (uint32_t c = R.z; c != kNone;) {
                        const uint32_t nx = __ldcg(&b.trec[c].w);
                        if (has_sink) {
                            const float4 v = __ldcg(&b.tacc[size_t(c) * 32 + lane]);
                            acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
                        }
                        c = nx;
                    }
                    if (R.x == kNone) {  // the group's root task: acc is final
                        tot = acc;
                        done = true;
                        break;
                    }
                    if (G2_SLICE_CONSUMER && R.x >= kSliceTag) {  // a slice's root: its partial to slot j of every rank
                        const size_t sl = size_t(b.slice_base) + size_t(R.x - kSliceTag) * 32 + lane;
                        if (has_sink) {
                            b.accum[sl] = acc;
                            for (int q = 0; q < b.world; ++q)
                                if (q != b.self) b.peer_accum[q][sl] = acc;
                        }
                        break;  // done stays false: walk_combine_slices forms the group's result
                    }
                    if (has_sink) __stcg(&b.tacc[size_t(r) * 32 + lane], acc);
                    __threadfence();
                    __syncwarp();
                    r = R.x;
                    if (lane == 0) last = atomicSub(&b.trec[r].y, 1u) == 1u;
                    last = __shfl_sync(kFull, last, 0);
                }
            }
            if (!done) continue;
            if (has_sink) {
                const float4 v = make_float4(G * tot.x, G * tot.y, G * tot.z, kPot ? G * tot.w : 0.f);
                b.accum[gfirst + lane] = v;
                // world > 1: the final accumulators go straight to every peer rank (NVLink stores,
                // overlapped with the rest of the walk)
                for (int q = 0; q < b.world; ++q)
                    if (q != b.self) b.peer_accum[q][gfirst + lane] = v;
            }
            if (b.world > 1) {
                // the group's cost: the same value into every rank's array (identical shards next step)
                __threadfence();
                if (b.peer_cost[0] && lane < b.world) b.peer_cost[lane][grp] = __ldcg(&b.gcost[grp]);
                __threadfence_system();
            }
        }
        return;
    }

    // ==================================== producer: traversal
#if G2_PRODUCER_REGS
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(G2_PRODUCER_REGS));
#endif
    PairSmem& sm = pairs[warp];
    uint32_t* spill = b.spill + (size_t(blockIdx.x) * kPairs + warp) * kSpillWords;
    // Task sources: the initial tasks (one per group, claimed by counter, in
    // b.order when given: heaviest first) and the FIFO of donated batches of
    // (group, up to 32 cells), which has priority so heavy groups are split
    // while the initial tasks are still draining.
    uint32_t* q_init = b.qstate;       // initial tasks claimed
    uint32_t* q_dtail = b.qstate + 1;  // donated slots reserved
    uint32_t* q_pending = b.qstate + 2;
    uint32_t* q_dhead = b.qstate + 4;  // donated slots claimed
    const uint32_t ng = b.qstate[3];   // initial tasks (written by walk_init / the ordering)
    const uint32_t glo = b.qstate[5];  // first group of this launch's shard (walk_init)
    // donation trigger: list entries written since the task's last donation (work done, not time),
    // scaled with the groups per producer warp of a full grid (a constant: identical on every rank)
    const uint32_t donate_pushes =
        min(p.donate_pushes, max(p.donate_few, *b.n_groups / uint32_t(4 * kNumSMs * kPairs) * p.donate_scale));
    const float thetaf = float(p.theta);
    uint32_t hand = 0;  // buffers handed to the consumer so far: buffer = hand & 1

    // hand the current buffer (lsize entries, padded to even) to the consumer, then
    // wait until the next buffer has been flushed (phase parity of its previous use)
    auto handoff = [&](int lsize, uint32_t grp, uint32_t fl, uint32_t rec = kNone) {
        const int bi = int(hand & 1);
        if ((lsize & 1) && lane == 0) put_entry(sm.buf[bi], lsize, 0.f, 0.f, 0.f, 0.f);
        if (lane == 0)
            sm.hdr[bi][0] = uint32_t(lsize + (lsize & 1)), sm.hdr[bi][1] = grp, sm.hdr[bi][2] = fl, sm.hdr[bi][3] = rec;
        __syncwarp();
        mbar_arrive(&sm.full[bi]);
        ++hand;
        mbar_wait(&sm.empty[hand & 1], ((hand >> 1) & 1) ^ 1);
    };

    // lane 0 may hold a claimed donated slot that is not written yet ("owed"):
    // claims are fetch-adds (no CAS retry storms); an owed slot is serviced as
    // soon as its donor writes it, and initial tasks are taken meanwhile.
    long long owed = -1;
    while (true) {
        // ---------------- acquire a task
        uint64_t e = kEmpty;
        uint32_t slot = 0;
        if (lane == 0) {
            unsigned backoff = 32;
            while (true) {
                if (owed >= 0) {
                    {  // ring slot of ticket `owed`; the generation tag tells a stale occupant apart
                        const uint32_t sl = uint32_t(owed) & (b.queue_cap - 1);
                        const uint64_t v = ld_acq64(&b.queue[sl]);
                        if (v != kEmpty && ((v >> 6) & kGenMask) == ((uint64_t(owed) >> b.ring_bits) & kGenMask)) {
                            e = v;  // the slot is released after the batch has been copied
                            slot = sl;
                            owed = -1;
                            break;
                        }
                        if (int(ld_vol(q_dtail) - uint32_t(owed)) > 0) continue;  // reserved: its donor writes it now
                    }
                } else if (ld_vol(q_dhead) < ld_vol(q_dtail)) {
                    owed = atomicAdd(q_dhead, 1u);  // donated work first
                    continue;
                }
                if (ld_vol(q_init) < ng) {
                    const uint32_t i = atomicAdd(q_init, 1u);
                    if (i < ng) {
                        e = uint64_t(glo + (b.order ? b.order[i] : i)) << 32;  // (group, root), count 0
                        break;
                    }
                }
                if (owed < 0) {  // nothing left: wait for the next donation
                    owed = atomicAdd(q_dhead, 1u);
                    continue;
                }
                if (ld_vol(q_pending) == 0) break;  // no task in flight: nothing can be donated any more
                __nanosleep(backoff);
                backoff = backoff < 256 ? backoff * 2 : 256;
            }
        }
        e = __shfl_sync(kFull, e, 0);
        if (e == kEmpty) break;
        slot = __shfl_sync(kFull, slot, 0);
        const uint32_t grp = uint32_t(e >> 32), nbatch = uint32_t(e) & 63u;
        // task record (lane 0): a donated task was given one by its donor (a whole-system group's slice:
        // its reserved slice record); a group's initial task allocates one at its first donation
        uint32_t rec = nbatch ? b.batch_rec[slot] : kNone, last_child = kNone;

        // ---------------- group
        uint64_t t_begin = 0;
        if (b.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
        const GroupRec* gp = b.groups + grp;
        const GroupRec g = *gp;
        const bool geom = p.force_geometric || g.a_min <= 0.0;  // engine.cpp:66
        const float rhsf = float(dmul(p.dacc, g.a_min)), radf = float(g.radius);
        const uint32_t gcount = g.count;
        // group centre as an unevaluated FP32 sum hi + lo: (hi - c) + lo is the FP32 difference to a
        // node's FP32 centre c with error <= 2^-24 (|c| + 2|d|) per axis (no FP64 in the screen)
        const float gxh = float(g.cx), gyh = float(g.cy), gzh = float(g.cz);
        const float gxl = float(dsub(g.cx, double(gxh))), gyl = float(dsub(g.cy, double(gyh))),
                    gzl = float(dsub(g.cz, double(gzh)));
        // absolute screen-error term from the FP32 rounding of node centres (|c| <= |g| + D)
        const float tolc = 5e-7f * (fabsf(gxh) + fabsf(gyh) + fabsf(gzh));
        uint32_t macs = 0, pushes = 0, tflags = kFirst, ndon = 0, maxlive = 0;  // ndon/maxlive: trace only
#if G2_DONATE_BACKOFF
        uint32_t dsteps = 0;  // donations by this task
#endif
        // logical LIFO = spill[gbase, gtop) (bottom, global) ++ sm.stack[0, ssize) (top, shared)
        int ssize, gbase = 0, gtop = 0, lsize = 0;
        uint32_t last_donation = 0;  // `pushes` at the last donation
        if (nbatch == 0) {
            if (lane == 0) sm.stack[0] = 0;  // root
            ssize = 1;
        } else {
            if (uint32_t(lane) < nbatch) sm.stack[lane] = b.batch[size_t(slot) * 32 + lane];
            ssize = int(nbatch);
            __syncwarp();
            if (lane == 0) {
                __threadfence();
                st_vol64(&b.queue[slot], kEmpty);  // release the ring slot for reuse
            }
        }
        __syncwarp();

        while (ssize + gtop - gbase > 0) {
            ListBuf* lbp = &sm.buf[hand & 1];
            // ---- pop up to 64 cells, two per lane (two independent MAC chains per lane)
            int take;
            uint32_t c0 = 0, c1 = 0;
            if (ssize > 0) {
                take = min(ssize, 64);
                if (lane < take) c0 = sm.stack[ssize - 1 - lane];
                if (lane + 32 < take) c1 = sm.stack[ssize - 33 - lane];
                ssize -= take;
            } else {
                take = min(gtop - gbase, 64);
                if (lane < take) c0 = spill[gtop - 1 - lane];
                if (lane + 32 < take) c1 = spill[gtop - 33 - lane];
                gtop -= take;
                if (gtop == gbase) gtop = gbase = 0;
            }
            __syncwarp();
            macs += take;
            const bool valid0 = lane < take, valid1 = lane + 32 < take;
            const Screen s0 = screen(t, gp, p, c0, valid0, gxh, gyh, gzh, gxl, gyl, gzl, tolc, radf, rhsf, G, thetaf,
                                     geom);
            const Screen s1 = screen(t, gp, p, c1, valid1, gxh, gyh, gzh, gxl, gyl, gzl, tolc, radf, rhsf, G, thetaf,
                                     geom);
            const uint32_t nchild0 = s0.nchild(), nchild1 = s1.nchild();
            const uint32_t nleaf0 = s0.nleaf(), nleaf1 = s1.nleaf();
            const uint32_t nfast0 = nleaf0 <= 8u ? nleaf0 : 0u, nfast1 = nleaf1 <= 8u ? nleaf1 : 0u;
            const uint32_t nnode0 = s0.accept ? 1u : 0u, nnode1 = s1.accept ? 1u : 0u;

            // one packed scan: children (<= 512) | accepted nodes (<= 64) << 10 | leaf particles (<= 512) << 17
            const uint32_t v = (nchild0 + nchild1) | ((nnode0 + nnode1) << 10) | ((nfast0 + nfast1) << 17);
            uint32_t inc = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(kFull, inc, o);
                if (lane >= o) inc += y;
            }
            const uint32_t tot = __shfl_sync(kFull, inc, 31), exc = inc - v;
            const uint32_t ctot = tot & 1023u, ntot = (tot >> 10) & 127u, ltot = tot >> 17;

            // ---- rejected internal cells: children onto the stack (cooperative)
            if (ctot) {
                if (kCheck) {
                    uint32_t* lc = &b.level_count[size_t(grp) * (kMaxDepth + 1) + 1u];
                    if (nchild0) atomicAdd(lc + ((s0.info >> 8) & 31u), nchild0);
                    if (nchild1) atomicAdd(lc + ((s1.info >> 8) & 31u), nchild1);
                }
                if (ssize + int(ctot) > kScap) {
                    // shared part full: move it onto the spill top, keeping one logical
                    // LIFO (spill = bottom, shared = top) so the depth-first bound holds
                    if (gtop + ssize > int(kSpillWords) && gbase > 0) {  // compact the deque
                        for (int i0 = 0; i0 < gtop - gbase; i0 += 32) {
                            const int i = i0 + lane;
                            const uint32_t x = i < gtop - gbase ? spill[gbase + i] : 0u;
                            __syncwarp();
                            if (i < gtop - gbase) spill[i] = x;
                            __syncwarp();
                        }
                        gtop -= gbase;
                        gbase = 0;
                    }
                    if (gtop + ssize <= int(kSpillWords)) {
                        for (int i = lane; i < ssize; i += 32) spill[gtop + i] = sm.stack[i];
                        gtop += ssize;
                        ssize = 0;
                    } else if (lane == 0) {
                        flags->stack_overflow = 1;
                    }
                    __syncwarp();
                }
                if (ssize + int(ctot) <= kScap) {  // <= 8 children per cell: short predicated loops
                    uint32_t* dst = sm.stack + ssize + (exc & 1023u);
#pragma unroll
                    for (uint32_t j = 0; j < 8; ++j)
                        if (j < nchild0) dst[j] = s0.link + j;
                    dst += nchild0;
#pragma unroll
                    for (uint32_t j = 0; j < 8; ++j)
                        if (j < nchild1) dst[j] = s1.link + j;
                    ssize += int(ctot);
                }
            }

            // ---- accepted cells (owner lanes) and opened leaves (cooperative): list entries
            // Leaf particles: entry = (leaf centre - group centre) + (particle - leaf centre), all
            // FP32, staged as (leaf slot | j << 6) with slot = lane (cell 0) or 32 + lane (cell 1);
            // lane entries start at lane_ofs (cell 0's particles, then cell 1's).
            auto write_leaves = [&](uint32_t nf0, uint32_t nf1, int base, int lane_ofs, uint32_t total) {
                int pos = base + lane_ofs;
                if (nf0) {
                    sm.leaf[lane] = make_float4(-s0.fx, -s0.fy, -s0.fz, __uint_as_float(s0.link));
#pragma unroll
                    for (uint32_t j = 0; j < 8; ++j)
                        if (j < nf0) put_index(*lbp, pos + int(j), uint32_t(lane) | (j << 6));
                    pos += int(nf0);
                }
                if (nf1) {
                    sm.leaf[32 + lane] = make_float4(-s1.fx, -s1.fy, -s1.fz, __uint_as_float(s1.link));
#pragma unroll
                    for (uint32_t j = 0; j < 8; ++j)
                        if (j < nf1) put_index(*lbp, pos + int(j), uint32_t(32 + lane) | (j << 6));
                }
                __syncwarp();
#pragma unroll 2
                for (uint32_t o = lane; o < total; o += 32) {
                    const int q = base + int(o);
                    const uint32_t vv = get_index(*lbp, q);
                    const float4 L = sm.leaf[vv & 63u];
                    const float4 r = ld_rel(t.rel + (__float_as_uint(L.w) + (vv >> 6)));
                    put_entry(*lbp, q, L.x + r.x, L.y + r.y, L.z + r.z, r.w);
                }
                __syncwarp();
            };
            const uint32_t P = ntot + ltot;
            if (P) {
                if (lsize + int(P) > kLcap) {
                    handoff(lsize, grp, tflags);
                    tflags = 0;
                    lsize = 0;
                    lbp = &sm.buf[hand & 1];
                }
                // entry = node centre - group centre = -(group centre - node centre)
                const int npos = lsize + int((exc >> 10) & 127u);
                if (nnode0) put_entry(*lbp, npos, -s0.fx, -s0.fy, -s0.fz, s0.fm);
                if (nnode1) put_entry(*lbp, npos + int(nnode0), -s1.fx, -s1.fy, -s1.fz, s1.fm);
                if (P <= uint32_t(kLcap)) {
                    if (ltot) write_leaves(nfast0, nfast1, lsize + int(ntot), int(exc >> 17), ltot);
                    lsize += int(P);
                } else {
                    // more than one buffer of entries in a round (rare): one cell slot at a time
                    lsize += int(ntot);
                    for (int which = 0; which < 2; ++which) {
                        const uint32_t nf = which ? nfast1 : nfast0;
                        uint32_t wtot;
                        const uint32_t wofs = warp_excl_scan(nf, wtot);
                        if (wtot == 0) continue;
                        if (lsize + int(wtot) > kLcap) {
                            handoff(lsize, grp, tflags);
                            tflags = 0;
                            lsize = 0;
                            lbp = &sm.buf[hand & 1];
                        }
                        write_leaves(which ? 0u : nf, which ? nf : 0u, lsize, int(wofs), wtot);
                        lsize += int(wtot);
                    }
                }
                pushes += P;
            }
            // ---- oversized leaves (coincident clusters at depth 21, or leaf_cap > 8): divergent writer
            if (__any_sync(kFull, nleaf0 > 8u || nleaf1 > 8u)) {
                for (int which = 0; which < 2; ++which) {
                    const Screen& sc = which ? s1 : s0;
                    const uint32_t nb = (which ? nleaf1 : nleaf0) > 8u ? (which ? nleaf1 : nleaf0) : 0u;
                    uint32_t btot;
                    const uint32_t bofs = warp_excl_scan(nb, btot);
                    if (btot == 0) continue;
                    pushes += btot;
                    int pos = lsize + int(bofs), end_all = lsize + int(btot);
                    uint32_t j = 0;
                    __syncwarp();
                    while (true) {
                        for (; j < nb && pos + int(j) < kLcap; ++j) {
                            const float4 r = ld_rel(t.rel + (sc.link + j));
                            put_entry(*lbp, pos + int(j), r.x - sc.fx, r.y - sc.fy, r.z - sc.fz, r.w);
                        }
                        if (end_all < kLcap) {
                            lsize = end_all;
                            break;
                        }
                        __syncwarp();
                        handoff(kLcap, grp, tflags);
                        tflags = 0;
                        lbp = &sm.buf[hand & 1];
                        pos -= kLcap;
                        end_all -= kLcap;
                        if (end_all == 0) {
                            lsize = 0;
                            break;
                        }
                    }
                    __syncwarp();
                }
            }
            __syncwarp();

            // ---- donate one batch from the logical bottom (shallowest cells = largest
            // subtrees) every kDonateEvery rounds of a long task, or when warps wait idle
            const int live = ssize + gtop - gbase;
            if (b.trace) maxlive = max(maxlive, uint32_t(live));
#if G2_DONATE_BACKOFF
            // a task's k-th donation waits for D x 2^(k / backoff) entries (a function of its own progress)
            if (live >= kDonateMinLive && pushes - last_donation >= (donate_pushes << min(dsteps / G2_DONATE_BACKOFF, 8u))) {
                ++dsteps;
#else
            if (live >= kDonateMinLive && pushes - last_donation >= donate_pushes) {
#endif
                // deterministic: the decision depends on this task's own progress only.  Half of the
                // pending cells (from the logical bottom: shallowest = largest subtrees) leave as up to
                // kMaxBatches batches of 32, one task (record) each, children in batch order.
                const bool from_spill = gtop - gbase >= 32 || (gtop > gbase && ssize == 0);
                const int avail = from_spill ? gtop - gbase : ssize;
                const int give = min(live / 2, min(avail, 32 * kMaxBatches));
                const int nb = (give + 31) / 32;
                uint32_t ds = 0, child0 = 0;
                int ok = 0;
                if (lane == 0 && give > 0) {
                    const uint32_t need = (rec == kNone ? 1u : 0u) + uint32_t(nb);  // (own record +) children
                    const uint32_t r0 = atomicAdd(&b.qstate[6], need);
                    if (r0 + need > b.rec_cap) {
                        flags->task_pool = 1;  // keep the work; the host grows the pool for the next walk
                    } else {
                        ok = 1;
                        if (rec == kNone) {
                            rec = r0;
                            b.trec[rec] = make_uint4(kNone, 1u, kNone, kNone);
                        }
                        child0 = r0 + need - uint32_t(nb);
                        for (int j = 0; j < nb; ++j) {
                            const uint32_t child = child0 + uint32_t(j);
                            b.trec[child] = make_uint4(rec, 1u, kNone, kNone);
                            if (last_child == kNone)
                                b.trec[rec].z = child;
                            else
                                b.trec[last_child].w = child;
                            last_child = child;
                        }
                        atomicAdd(&b.trec[rec].y, uint32_t(nb));  // before the children can exist
                        ds = atomicAdd(q_dtail, uint32_t(nb));    // consecutive tickets; slot = ticket mod ring
                        atomicAdd(q_pending, uint32_t(nb));
                        for (int j = 0; j < nb; ++j) {
                            // wait for the slot's previous occupant to be consumed (ring of 2^20)
                            const uint32_t sl = (ds + uint32_t(j)) & (b.queue_cap - 1);
                            while (ld_vol64(&b.queue[sl]) != kEmpty) __nanosleep(64);
                            b.batch_rec[sl] = child0 + uint32_t(j);
                        }
                    }
                }
                ok = __shfl_sync(kFull, ok, 0);
                ds = __shfl_sync(kFull, ds, 0);
                last_donation = pushes;
                if (ok) {
                    ndon += uint32_t(nb);
                    for (int j = 0; j < nb; ++j) {
                        const uint32_t sl = (ds + uint32_t(j)) & (b.queue_cap - 1);
                        const int i = 32 * j + lane;
                        if (i < give) b.batch[size_t(sl) * 32 + lane] = from_spill ? spill[gbase + i] : sm.stack[i];
                    }
                    __threadfence();
                    __syncwarp();
                    if (lane < nb) {
                        const uint32_t t = ds + uint32_t(lane);
                        const uint32_t k = uint32_t(min(32, give - 32 * lane));
                        st_rel64(&b.queue[t & (b.queue_cap - 1)],
                                 (uint64_t(grp) << 32) | ((uint64_t(t >> b.ring_bits) & kGenMask) << 6) | k);
                    }
                    if (from_spill) {
                        gbase += give;
                        if (gbase == gtop) gbase = gtop = 0;
                    } else {
                        for (int base = 0; base < ssize - give; base += 32) {
                            const int i = base + lane;
                            const uint32_t x = i < ssize - give ? sm.stack[i + give] : 0u;
                            __syncwarp();
                            if (i < ssize - give) sm.stack[i] = x;
                            __syncwarp();
                        }
                        ssize -= give;
                    }
                }
            }
        }
        // the task's list entries into the group's cost (read by the consumer retiring the group's last
        // task, which is ordered after this through the buffer hand-over and the pending counter)
        if (b.world > 1 && lane == 0) atomicAdd(&b.gcost[grp], pushes);
        // the last buffer of the task (possibly empty) tells the consumer to write out
        handoff(lsize, grp, tflags | kLast, rec);

        // ---------------- events
        if (lane == 0) {
            const unsigned long long inter = (unsigned long long)pushes * gcount;
            if (p.count_ops) {
                atomicAdd(&b.events[0], inter);
                atomicAdd(&b.events[1], (unsigned long long)macs);
                atomicAdd(&b.events[2], (unsigned long long)pushes);
            }
            if (b.group_inter) atomicAdd(reinterpret_cast<unsigned long long*>(&b.group_inter[grp]), inter);
            if (b.trace) {
                uint64_t t_end;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
                const uint32_t ts = atomicAdd(b.trace_n, 1u);
                if (ts < b.trace_cap) {
                    b.trace[2 * ts] = make_uint4(uint32_t(t_begin), uint32_t(t_begin >> 32), uint32_t(t_end),
                                                 uint32_t(t_end >> 32));
                    b.trace[2 * ts + 1] = make_uint4(grp, nbatch | (min(ndon, 0xfffu) << 8) | (min(maxlive, 0xfffu) << 20), macs, pushes);
                }
            }
            // no fence: the pending count only ends the walk (its own earlier increments for donated
            // batches are ordered before this decrement: same thread, same address)
            atomicSub(q_pending, 1u);
        }
    }
    // retire the consumer
    if (lane == 0) sm.hdr[hand & 1][0] = 0, sm.hdr[hand & 1][1] = kStop, sm.hdr[hand & 1][2] = 0;
    __syncwarp();
    mbar_arrive(&sm.full[hand & 1]);
}

// 8 lanes per group (4 groups per warp): AABB centre, radius and a_min of make_group
// (traversal.cpp:16-38).  Each lane folds members lane, lane + 8, ... in order, then three
// xor-shuffle levels combine the lanes: min / max are exact in any order, so the result is the
// reference's.  (A warp per group spent its time in 5-level FP64 shuffle trees; a lane per group
// gathered uncoalesced.)
constexpr int kGroupLanes = 8;
__global__ void __launch_bounds__(256) groups_kernel(TreeView t, const double* __restrict__ amag, WalkBuffers b,
                                                     uint32_t gs) {
    const uint32_t n_sinks = *b.n_sinks;
    const uint32_t n_groups = (n_sinks + gs - 1) / gs;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t sub = threadIdx.x & (kGroupLanes - 1);
    if (tid == 0) *b.n_groups = n_groups;
    const uint32_t stride = (gridDim.x * blockDim.x) / kGroupLanes;
    // every lane of a warp runs the same number of iterations (shuffles need the full warp)
    const uint32_t gw0 = tid / kGroupLanes;
    const uint32_t iters = (n_groups + stride - 1) / stride;
    for (uint32_t it = 0; it < iters; ++it) {
        const uint32_t g = gw0 + it * stride;
        const bool gon = g < n_groups;
        const uint32_t first = g * gs;
        const uint32_t cnt = gon ? min(gs, n_sinks - first) : 0u;
        const uint32_t* __restrict__ mk = b.sinks + first;
        double lx = INFINITY, ly = INFINITY, lz = INFINITY, hx = -INFINITY, hy = -INFINITY, hz = -INFINITY;
        double am = INFINITY;
        if (sub < cnt) {
            const double4 q = t.xyzm[mk[sub]];
            lx = hx = q.x, ly = hy = q.y, lz = hz = q.z;
            am = amag[mk[sub]];
        }
        for (uint32_t j = sub + kGroupLanes; j < cnt; j += kGroupLanes) {
            const uint32_t k = mk[j];
            const double4 q = t.xyzm[k];
            lx = smin(lx, q.x), ly = smin(ly, q.y), lz = smin(lz, q.z);
            hx = smax(hx, q.x), hy = smax(hy, q.y), hz = smax(hz, q.z);
            am = smin(am, amag[k]);
        }
#pragma unroll
        for (int o = kGroupLanes / 2; o > 0; o >>= 1) {
            lx = smin(lx, __shfl_xor_sync(kFull, lx, o));
            ly = smin(ly, __shfl_xor_sync(kFull, ly, o));
            lz = smin(lz, __shfl_xor_sync(kFull, lz, o));
            hx = smax(hx, __shfl_xor_sync(kFull, hx, o));
            hy = smax(hy, __shfl_xor_sync(kFull, hy, o));
            hz = smax(hz, __shfl_xor_sync(kFull, hz, o));
            am = smin(am, __shfl_xor_sync(kFull, am, o));
        }
        const double cx = dmul(0.5, dadd(lx, hx)), cy = dmul(0.5, dadd(ly, hy)), cz = dmul(0.5, dadd(lz, hz));
        double r2 = 0.0;
        for (uint32_t j = sub; j < cnt; j += kGroupLanes) {
            const double4 q = t.xyzm[mk[j]];
            r2 = smax(r2, norm2(dsub(q.x, cx), dsub(q.y, cy), dsub(q.z, cz)));
        }
#pragma unroll
        for (int o = kGroupLanes / 2; o > 0; o >>= 1) r2 = smax(r2, __shfl_xor_sync(kFull, r2, o));
        if (gon && sub == 0) {
            const double radius = dsqrt(r2);
            b.groups[g] = GroupRec{cx, cy, cz, radius, am, first, cnt};
            b.sliced[g] = 0;
            if (b.world > 1) b.gcost[g] = 0u;
        }
    }
}

// whole-system groups (sphere reaching a quarter of the root's extent): slicing candidates when the
// root is internal; candidates beyond kMaxHeavy switch slicing off for this walk.  Apart from
// groups_kernel, which reads no node, so the spheres can be formed while calc_node's internal levels
// still run (Engine::calc_nodes(true)).
__global__ void __launch_bounds__(256) heavy_select_kernel(TreeView t, WalkBuffers b) {
    const uint32_t ng = *b.n_groups;
    const uint32_t info = t.nodes32[0].info;
    if ((info & kLeafBit) || (info & 0xffu) < 2u) return;
    const double cut = kHeavyFrac * t.nodes[0].extent;
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < ng; g += gridDim.x * blockDim.x)
        if (b.groups[g].radius >= cut) {
            const uint32_t h = atomicAdd(&b.heavy[0], 1u);
            if (h < kMaxHeavy) b.heavy[1 + h] = g;
        }
}

// Cost-balanced contiguous shards of the groups: rank r walks groups
// [b_r, b_{r+1}) with b_r the first group whose cost prefix reaches r/world of the total, the
// costs being the previous step's per-group list-entry counts (every rank holds the same array, so
// every rank computes the same boundaries).  With no usable history (first step, or a different
// group count: the active set changed) the shards are equal group counts.
constexpr int kShardThreads = 1024;
__global__ void __launch_bounds__(kShardThreads) shard_kernel(const uint32_t* __restrict__ cost,
                                                              const uint32_t* ng_prev, uint32_t* ng_cur,
                                                              const uint32_t* n_groups_p, int world, int rank,
                                                              uint32_t* shard) {
    __shared__ unsigned long long part[kShardThreads];
    __shared__ uint32_t bnd[kMaxPeers + 1];
    const uint32_t ng = *n_groups_p;
    const bool hist = cost && ng_prev && *ng_prev == ng && ng > 0;
    const uint32_t per = (ng + kShardThreads - 1) / kShardThreads;
    const uint32_t g0 = min(ng, threadIdx.x * per), g1 = min(ng, g0 + per);
    unsigned long long sum = 0;
    if (hist)
        for (uint32_t g = g0; g < g1; ++g) sum += cost[g];
    part[threadIdx.x] = sum;
    __syncthreads();
    for (int o = 1; o < kShardThreads; o <<= 1) {  // inclusive Hillis-Steele scan of the partial sums
        const unsigned long long y = threadIdx.x >= unsigned(o) ? part[threadIdx.x - o] : 0ull;
        __syncthreads();
        part[threadIdx.x] += y;
        __syncthreads();
    }
    const unsigned long long total = part[kShardThreads - 1];
    if (threadIdx.x <= unsigned(world)) bnd[threadIdx.x] = uint32_t(uint64_t(ng) * threadIdx.x / world);  // equal
    __syncthreads();
    if (hist && total > 0) {
        const unsigned long long before = part[threadIdx.x] - sum;
        for (int r = 1; r < world; ++r) {
            const unsigned long long t = total * unsigned(r) / unsigned(world);
            if (before <= t && t < part[threadIdx.x]) {  // boundary r falls inside this thread's segment
                unsigned long long acc = before;
                uint32_t g = g0;
                while (g < g1 && acc + cost[g] <= t) acc += cost[g++];
                // group g straddles the target: it goes to the side it overshoots least
                if (g < g1 && acc + cost[g] - t < t - acc) ++g;
                bnd[r] = g;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        shard[0] = bnd[rank], shard[1] = bnd[rank + 1];
        if (ng_cur) *ng_cur = ng;  // the groups whose costs this step records
    }
}

// the rank of slice j (group j / nk, root child k = j % nk): classes of equal expected cost (root
// child k: cost ~ its mass w[k]) dealt heaviest class first, round-robin with alternating direction
// (snake), so every rank gets a near-equal share.  It only schedules: slice j's result and its place
// in the group's sum do not depend on it.  Host-callable (g2_slice_owner, tests).
}  // namespace
__host__ __device__ uint32_t slice_owner_of(const float* w, uint32_t nk, uint32_t j, uint32_t nh, uint32_t world) {
    const uint32_t h = j / nk, k = j % nk;
    uint32_t cls = 0;
    for (uint32_t q = 0; q < nk; ++q) cls += w[q] > w[k] || (w[q] == w[k] && q < k);
    const uint32_t seq = cls * nh + h, r = seq % world;
    return ((seq / world) & 1u) ? world - 1u - r : r;
}
namespace {
__device__ __forceinline__ uint32_t slice_owner(const TreeView& t, uint32_t j, uint32_t nh, uint32_t nk,
                                                uint32_t world) {
    float w[kSlicesPer];
    const uint32_t c0 = t.nodes32[0].link;
    for (uint32_t q = 0; q < nk; ++q) w[q] = t.nodes32[c0 + q].m;
    return slice_owner_of(w, nk, j, nh, world);
}

// One block of kMaxHeavy threads: the queue state, and the whole-system groups' slices.  The heavy
// candidates (group setup) are sorted by index (their discovery order is a race; the slice numbering
// must not be); a candidate whose root MAC accepts (a single entry) stays a plain group.  Slice j
// (group j / nk, root child j % nk) belongs to rank slice_owner(j); this rank's slices are published as
// donated tasks of one cell (the root child) with the reserved record j, so the walk takes them
// first and runs them with no change to its task code; the root's MAC evaluation is counted once,
// by the owner of the group's slice 0.  The initial-task ordering leaves the sliced groups out.
__global__ void __launch_bounds__(kMaxHeavy) walk_init_kernel(WalkBuffers b, TreeView t, WalkParams p, int sworld,
                                                              int sself, int ordered) {
    G2_PDL_WAIT();  // programmatic dependent launch (launch_pdl)
    __shared__ uint32_t sorted[kMaxHeavy];
    __shared__ uint32_t wsum[kMaxHeavy / 32 + 1];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t cand = b.heavy[0];
    const uint32_t rinfo = t.nodes32[0].info;
    const uint32_t nc = (rinfo & kLeafBit) ? 0u : (rinfo & 0xffu);
    const uint32_t nh0 = (ordered && cand <= kMaxHeavy && nc >= 2u) ? cand : 0u;
    uint32_t v = 0;
    if (threadIdx.x < nh0) {
        v = b.heavy[1 + threadIdx.x];
        uint32_t r = 0;
        for (uint32_t q = 0; q < nh0; ++q) r += b.heavy[1 + q] < v;
        sorted[r] = v;
    }
    __syncthreads();
    // the root MAC of each candidate in index order (exact, traversal.cpp:40-56): rejected -> sliced
    bool keep = false;
    if (threadIdx.x < nh0) {
        v = sorted[threadIdx.x];
        const GroupRec g = b.groups[v];
        const bool geom = p.force_geometric || g.a_min <= 0.0;
        keep = !mac_exact(t.nodes[0], g, p, dmul(p.dacc, g.a_min), geom);
    }
    const uint32_t m = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) wsum[w] = __popc(m);
    __syncthreads();
    uint32_t before = 0, nh = 0;
    for (int q = 0; q < kMaxHeavy / 32; ++q) before += q < w ? wsum[q] : 0u, nh += wsum[q];
    const uint32_t h_of = before + __popc(m & ((1u << lane) - 1u));
    __syncthreads();
    if (keep) {
        b.heavy[1 + h_of] = v;
        b.sliced[v] = 1;
        // the root's expansion, which no slice task performs, in the frontier-cap counters
        if (b.level_count) atomicAdd(&b.level_count[size_t(v) * (kMaxDepth + 1) + 1u + ((rinfo >> 8) & 31u)], nc);
    }
    const uint32_t nk = min(nc, kSlicesPer), nsl = nh * nk;
    // slices to ranks: classes of equal expected cost (root child k: cost ~ its mass) dealt heaviest
    // class first, round-robin with alternating direction (snake), so every rank gets a near-equal
    // share; the assignment only schedules (slice j's result and its place in the sum are fixed)
    __shared__ uint32_t mine_s;
    if (threadIdx.x == 0) mine_s = 0;
    __syncthreads();  // the final heavy list
    for (uint32_t j = threadIdx.x; j < nsl; j += blockDim.x) {
        const uint32_t h = j / nk, k = j % nk;
        if (slice_owner(t, j, nh, nk, uint32_t(sworld)) != uint32_t(sself)) continue;
        const uint32_t i = atomicAdd(&mine_s, 1u);  // queue ticket (any order: results do not depend on it)
        b.trec[j] = make_uint4(kSliceTag | j, 1u, kNone, kNone);
        b.batch[size_t(i) * 32] = t.nodes32[0].link + k;  // root child k
        b.batch_rec[i] = j;
        b.queue[i] = (uint64_t(b.heavy[1 + h]) << 32) | 1u;  // ticket i: generation 0, one cell
        if (k == 0 && p.count_ops) atomicAdd(&b.events[1], 1ull);  // the root's MAC evaluation
    }
    __syncthreads();
    const uint32_t mine = mine_s;
    if (threadIdx.x == 0) {
        const uint32_t n_groups = *b.n_groups;
        const uint32_t lo = b.shard ? b.shard[0] : b.group_lo;
        const uint32_t hi = min(b.shard ? b.shard[1] : b.group_hi, n_groups);
        const uint32_t ng = hi > lo ? hi - lo : 0u;
        b.qstate[5] = lo;
        b.qstate[0] = 0;          // initial tasks claimed
        b.qstate[1] = mine;       // donated slots reserved (this rank's slices)
        b.qstate[2] = ng + mine;  // tasks pending (the ordering subtracts the sliced groups)
        b.qstate[3] = ng;         // initial tasks (likewise)
        b.qstate[4] = 0;          // donated slots consumed
        b.qstate[6] = nsl;        // task records used (slice records 0 .. nsl-1 reserved)
        b.qstate[7] = nsl;        // slices of all ranks
        b.qstate[8] = mine;       // this rank's slices
        b.qstate[9] = nk;         // slices per heavy group
        b.qstate[10] = ng;        // the shard's groups
    }
}

// every heavy group: G x (slice 0 + slice 1 + ...) in slice order, one warp per group
__global__ void __launch_bounds__(256) combine_slices_kernel(WalkBuffers b, TreeView t, const float4* __restrict__ slices,
                                                             size_t rank_stride, int world, float G,
                                                             uint32_t* cost) {
    const uint32_t nsl = b.qstate[7], nk = b.qstate[9];
    const uint32_t nh = nk ? nsl / nk : 0u;
    const int lane = threadIdx.x & 31;
    for (uint32_t h = blockIdx.x * 8 + (threadIdx.x >> 5); h < nh; h += gridDim.x * 8) {
        const uint32_t g = b.heavy[1 + h];
        const GroupRec gr = b.groups[g];
        if (lane == 0 && cost) cost[g] = 0u;  // sliced groups are not in the contiguous shards' balance
        if (uint32_t(lane) >= gr.count) continue;
        float4 tot = make_float4(0.f, 0.f, 0.f, 0.f);
        for (uint32_t k = 0; k < nk; ++k) {
            const uint32_t j = h * nk + k;
            const size_t owner = rank_stride ? slice_owner(t, j, nh, nk, uint32_t(world)) : 0u;
            const float4 v = slices[owner * rank_stride + size_t(j) * 32 + lane];
            if (k == 0)
                tot = v;
            else
                tot.x += v.x, tot.y += v.y, tot.z += v.z, tot.w += v.w;
        }
        b.accum[gr.first + lane] = make_float4(G * tot.x, G * tot.y, G * tot.z, G * tot.w);
    }
}

// Initial tasks heaviest first (longest-processing-time order): a group's bounding radius predicts
// its walk cost (the whole-system groups at Z-curve jumps have radius ~ r_cut and carry up to 32 N
// interactions), so groups are counting-sorted by descending radius (sign + exponent + 3 mantissa bits
// of the FP32 radius, 2048 buckets).  The order only schedules: every group's task tree, and hence its
// result, is the same in any order.
constexpr int kOrderBuckets = 2048;
#ifndef G2_ORDER_HEAVY
#define G2_ORDER_HEAVY 1.0
#endif
constexpr float kOrderHeavy = G2_ORDER_HEAVY;  // fraction of the groups ordered largest sphere first
__device__ __forceinline__ uint32_t order_bucket(double radius) {
    return uint32_t(kOrderBuckets - 1) - min(__float_as_uint(float(radius)) >> 20, uint32_t(kOrderBuckets - 1));
}
__global__ void __launch_bounds__(256) order_hist_kernel(const GroupRec* __restrict__ groups, const uint32_t* qstate,
                                                         const uint8_t* __restrict__ sliced, uint32_t* hist) {
    __shared__ uint32_t h[kOrderBuckets];
    for (int i = threadIdx.x; i < kOrderBuckets; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const uint32_t lo = qstate[5], ng = qstate[3];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ng; i += gridDim.x * blockDim.x)
        if (!sliced[lo + i]) atomicAdd(&h[order_bucket(groups[lo + i].radius)], 1u);
    __syncthreads();
    for (int i = threadIdx.x; i < kOrderBuckets; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}
__global__ void __launch_bounds__(1024) order_scan_kernel(uint32_t* hist, uint32_t* qstate, float heavy) {
    G2_PDL_WAIT();  // programmatic dependent launch (launch_pdl)
    __shared__ uint32_t part[1024];
    const uint32_t a = hist[2 * threadIdx.x], c = hist[2 * threadIdx.x + 1];
    part[threadIdx.x] = a + c;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const uint32_t y = threadIdx.x >= unsigned(o) ? part[threadIdx.x - o] : 0u;
        __syncthreads();
        part[threadIdx.x] += y;
        __syncthreads();
    }
    const uint32_t ex = part[threadIdx.x] - (a + c);
    hist[2 * threadIdx.x] = ex, hist[2 * threadIdx.x + 1] = ex + a;
    // the heavy class: the largest spheres up to a fraction `heavy` of the groups, whole buckets; the
    // rest keeps index (Morton) order, so concurrently walked groups share tree nodes in L2
    __shared__ uint32_t cut;
    if (threadIdx.x == 0) cut = heavy <= 0.f ? 0u : kOrderBuckets;
    __syncthreads();
    const uint32_t total = part[1023];
    const uint32_t lim = uint32_t(ceilf(heavy * float(total)));
    if (heavy > 0.f && heavy < 1.f) {
        if (ex < lim && ex + a >= lim) atomicMin(&cut, 2 * threadIdx.x + 1);
        if (ex + a < lim && ex + a + c >= lim) atomicMin(&cut, 2 * threadIdx.x + 2);
    }
    __syncthreads();
    if (threadIdx.x == 1023) {  // the initial tasks: the shard's groups less the sliced ones
        qstate[2] -= qstate[3] - total;
        qstate[3] = total;
        qstate[12] = cut;
    }
    if (cut < kOrderBuckets && threadIdx.x == cut / 2) qstate[13] = (cut & 1) ? ex + a : ex;  // heavy count
    if (cut >= kOrderBuckets && threadIdx.x == 1023) qstate[13] = total;
}
__global__ void __launch_bounds__(256) order_scatter_kernel(const GroupRec* __restrict__ groups, const uint32_t* qstate,
                                                            const uint8_t* __restrict__ sliced, uint32_t* off,
                                                            uint32_t* order) {
    G2_PDL_WAIT();  // programmatic dependent launch (launch_pdl)
    const uint32_t lo = qstate[5], ng = qstate[10];  // the shard's groups (walk_init)
    const uint32_t cut = qstate[12];
    const int lane = threadIdx.x & 31;
    // warp-aggregated claims: the radii crowd into few buckets, whose counters would serialise
    for (uint32_t b0 = blockIdx.x * blockDim.x; b0 < ng; b0 += gridDim.x * blockDim.x) {  // warp-uniform trips
        const uint32_t i = b0 + threadIdx.x;
        uint32_t bk = ~0u;
        if (i < ng && !sliced[lo + i]) {
            bk = order_bucket(groups[lo + i].radius);
            if (bk >= cut) bk = ~0u;
        }
        const uint32_t peers = __match_any_sync(kFull, bk);
        const int leader = __ffs(peers) - 1;
        uint32_t pos = 0;
        if (bk != ~0u && lane == leader) pos = atomicAdd(&off[bk], uint32_t(__popc(peers)));
        pos = __shfl_sync(kFull, pos, leader) + __popc(peers & ((1u << lane) - 1u));
        if (bk != ~0u) order[pos] = i;
    }
}

// the light class in index order after the heavy one: per-tile counts, then an ordered scatter
constexpr int kOrderTile = 1024;
__device__ __forceinline__ bool order_light(const GroupRec* __restrict__ groups, const uint8_t* __restrict__ sliced,
                                            uint32_t lo, uint32_t ng, uint32_t cut, uint32_t i) {
    return i < ng && !sliced[lo + i] && order_bucket(groups[lo + i].radius) >= cut;
}
__global__ void __launch_bounds__(kOrderTile) order_light_count_kernel(const GroupRec* __restrict__ groups,
                                                                       const uint32_t* qstate,
                                                                       const uint8_t* __restrict__ sliced,
                                                                       uint32_t* tile_count) {
    const uint32_t lo = qstate[5], ng = qstate[10], cut = qstate[12];
    const uint32_t i = blockIdx.x * kOrderTile + threadIdx.x;
    const uint32_t m = __ballot_sync(0xffffffffu, order_light(groups, sliced, lo, ng, cut, i));
    __shared__ uint32_t c;
    if (threadIdx.x == 0) c = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(&c, uint32_t(__popc(m)));
    __syncthreads();
    if (threadIdx.x == 0) tile_count[blockIdx.x] = c;
}
__global__ void __launch_bounds__(kOrderTile) order_light_scatter_kernel(const GroupRec* __restrict__ groups,
                                                                         const uint32_t* qstate,
                                                                         const uint8_t* __restrict__ sliced,
                                                                         const uint32_t* __restrict__ tile_count,
                                                                         uint32_t* order) {
    const uint32_t lo = qstate[5], ng = qstate[10], cut = qstate[12];
    const uint32_t i = blockIdx.x * kOrderTile + threadIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    __shared__ uint32_t wsum[kOrderTile / 32], base;
    if (threadIdx.x == 0) {
        uint32_t b = qstate[13];  // after the heavy class
        for (uint32_t t = 0; t < blockIdx.x; ++t) b += tile_count[t];
        base = b;
    }
    const bool light = order_light(groups, sliced, lo, ng, cut, i);
    const uint32_t m = __ballot_sync(0xffffffffu, light);
    if (lane == 0) wsum[w] = __popc(m);
    __syncthreads();
    uint32_t before = base;
    for (int q = 0; q < w; ++q) before += wsum[q];
    if (light) order[before + __popc(m & ((1u << lane) - 1u))] = i;
}

// zero the accumulator slots this launch accumulates into: all sinks, or with a peer exchange
// only the own shard's slots (the other slots are written by the peers, possibly already)
__global__ void zero_accum_kernel(float4* accum, const uint32_t* n_sinks, uint32_t cap, uint32_t lo, uint32_t hi,
                                  const uint32_t* shard, uint32_t gs) {
    G2_PDL_WAIT();  // programmatic dependent launch (launch_pdl)
    if (shard) {
        lo = uint32_t(min(uint64_t(shard[0]) * gs, uint64_t(~0u)));
        hi = uint32_t(min(uint64_t(shard[1]) * gs, uint64_t(~0u)));
    }
    const uint32_t n = min(min(*n_sinks, cap), hi);
    for (uint32_t i = lo + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        accum[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

__global__ void finalize_kernel(WalkBuffers b, uint32_t cap, double* ax, double* ay, double* az, double* pot) {
    const uint32_t n = min(*b.n_sinks, cap);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float4 a = b.accum[i];
        const uint32_t k = b.sinks[i];
        ax[k] = double(a.x);
        ay[k] = double(a.y);
        az[k] = double(a.z);
        if (pot) pot[k] = double(a.w);
    }
}

constexpr int kWalkSmem = kPairs * int(sizeof(PairSmem));
constexpr int kMaxBlocksPerSM = 8;  // bound for the spill area (occupancy is smem-limited well below)

template <bool kPot, bool kEps0, bool kCheck>
int walk_blocks_per_sm() {
    static int v = 0;
    if (!v) {
        G2_CUDA(cudaFuncSetAttribute(walk_kernel<kPot, kEps0, kCheck>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kWalkSmem));
        G2_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, walk_kernel<kPot, kEps0, kCheck>, kThreads,
                                                              kWalkSmem));
        v = std::max(1, std::min(v, kMaxBlocksPerSM));
    }
    return v;
}

template <bool kPot, bool kEps0, bool kCheck>
void walk_launch_t(const TreeView& t, const WalkParams& p, const WalkBuffers& b, DevFlags* flags, cudaStream_t s) {
    int per_sm = walk_blocks_per_sm<kPot, kEps0, kCheck>();
    static const char* ov = std::getenv("G2_WALK_CTAS_PER_SM");  // development: occupancy experiments
    if (ov) per_sm = std::max(1, std::min(per_sm, std::atoi(ov)));
    const unsigned grid = unsigned(per_sm * kNumSMs);
    G2_COUNT(1), launch_pdl(walk_kernel<kPot, kEps0, kCheck>, dim3(grid), dim3(kThreads), size_t(kWalkSmem), s, t, p, b, flags);
}

}  // namespace

size_t walk_spill_words() { return kSpillWords; }
size_t walk_slice_base(size_t n) { return (n + 31) / 32 * 32 + 64 * 32; }
size_t walk_slice_slots() { return size_t(kMaxHeavy) * kSlicesPer * 32; }
size_t walk_heavy_words() { return kMaxHeavy + 1; }

void launch_walk_combine(const WalkBuffers& b, const TreeView& t, const float4* slices, size_t rank_stride, int world,
                         double G, uint32_t* cost, cudaStream_t s) {
    G2_COUNT(1), combine_slices_kernel<<<(kMaxHeavy + 7) / 8, 256, 0, s>>>(b, t, slices, rank_stride,
                                                                            std::max(1, world), float(G), cost);
    G2_CUDA(cudaGetLastError());
}
size_t walk_order_scratch_words(size_t n_groups) { return kOrderBuckets + n_groups / kOrderTile + 1; }
size_t walk_resident_warps() {
    // producer warps (one spill stack each) of the largest grid walk_launch_t can use
    return size_t(kNumSMs) * kMaxBlocksPerSM * kPairs;
}

void launch_groups(const TreeView& t, const double* acc_old_mag, const WalkBuffers& b, uint32_t group_size,
                   uint32_t n_sinks_cap, cudaStream_t s) {
    const uint32_t ng = (n_sinks_cap + group_size - 1) / group_size;
    const unsigned blocks = std::max(1u, std::min<unsigned>(ceil_div(size_t(ng) * kGroupLanes, 256), kNumSMs * 16));
    G2_COUNT(1), groups_kernel<<<blocks, 256, 0, s>>>(t, acc_old_mag, b, group_size);
    G2_CUDA(cudaGetLastError());
}

// the walk's set-up that reads no node (shards, accumulator clearing): may run before calc_node ends
void launch_walk_prep(const WalkBuffers& b, uint32_t n_sinks_cap, uint32_t gs, cudaStream_t s) {
    const unsigned zb = std::max(1u, std::min<unsigned>(ceil_div(n_sinks_cap, 256), kNumSMs * 8));
    uint32_t zlo = 0, zhi = ~0u;
    if (b.world > 1) {
        zlo = uint32_t(std::min<uint64_t>(uint64_t(b.group_lo) * gs, ~0u));
        zhi = uint32_t(std::min<uint64_t>(uint64_t(b.group_hi) * gs, ~0u));
    }
    if (b.shard) {
        G2_COUNT(1), shard_kernel<<<1, kShardThreads, 0, s>>>(b.cost_prev, b.ng_prev, b.ng_cur, b.n_groups, b.world,
                                                              b.self, b.shard);
        G2_CUDA(cudaGetLastError());
    }
    G2_COUNT(1), launch_pdl(zero_accum_kernel, dim3(zb), dim3(256), size_t(0), s, b.accum, b.n_sinks, n_sinks_cap, zlo, zhi, b.shard, gs);
}

void launch_walk(const TreeView& t, const WalkParams& p, const WalkBuffers& b, bool with_pot, uint32_t n_sinks_cap,
                 uint32_t gs, DevFlags* flags, cudaStream_t s, const cudaEvent_t* kernel_ev, bool prep) {
    if (prep) launch_walk_prep(b, n_sinks_cap, gs, s);
    {
        const unsigned hb = std::max(1u, std::min<unsigned>(ceil_div(ceil_div(n_sinks_cap, gs), 256), kNumSMs * 4));
        G2_COUNT(1), heavy_select_kernel<<<hb, 256, 0, s>>>(t, b);
    }
    G2_COUNT(1), launch_pdl(walk_init_kernel, dim3(1), dim3(kMaxHeavy), size_t(0), s, b, t, p, b.slice_world, b.slice_rank,
                                                          b.order_scratch != nullptr);
    if (b.order_scratch) {
        const unsigned ob = std::max(1u, std::min<unsigned>(ceil_div(ceil_div(n_sinks_cap, gs), 256), kNumSMs * 4));
        G2_CUDA(cudaMemsetAsync(b.order_scratch, 0, kOrderBuckets * sizeof(uint32_t), s));
        G2_COUNT(1), order_hist_kernel<<<ob, 256, 0, s>>>(b.groups, b.qstate, b.sliced, b.order_scratch);
        static const char* hf = std::getenv("G2_ORDER_HEAVY");  // development: heavy-class fraction sweeps
        const float heavy = hf ? float(std::atof(hf)) : kOrderHeavy;
        G2_COUNT(1), launch_pdl(order_scan_kernel, dim3(1), dim3(1024), size_t(0), s, b.order_scratch, b.qstate, heavy);
        G2_COUNT(1), launch_pdl(order_scatter_kernel, dim3(ob), dim3(256), size_t(0), s, b.groups, b.qstate, b.sliced, b.order_scratch,
                                                             const_cast<uint32_t*>(b.order));
        if (heavy < 1.0f) {  // the order scan set the cut; the light class follows the heavy one
            const unsigned tiles = unsigned(std::max<size_t>(1, ceil_div(ceil_div(n_sinks_cap, gs), kOrderTile)));
            uint32_t* tile_count = b.order_scratch + kOrderBuckets;
            G2_COUNT(1), order_light_count_kernel<<<tiles, kOrderTile, 0, s>>>(b.groups, b.qstate, b.sliced, tile_count);
            G2_COUNT(1), order_light_scatter_kernel<<<tiles, kOrderTile, 0, s>>>(b.groups, b.qstate, b.sliced, tile_count,
                                                                                 const_cast<uint32_t*>(b.order));
        }
    }
    // the guarded flush whenever eps^2 is not a normal FP32 number (eps == 0 included): with eps^2
    // flushed to zero the self pair would otherwise meet rsqrt(0) = inf and 0 * inf = NaN.  Likewise
    // when the self pair's factor m / eps^3 could overflow FP32 (tiny eps with large masses).
    const bool eps0 = !(float(p.eps * p.eps) >= FLT_MIN) ||
                      !(p.mass_max / (p.eps * p.eps * p.eps) < 1e30);
    const bool check = b.level_count != nullptr;
    if (kernel_ev) G2_CUDA(cudaEventRecord(kernel_ev[0], s));
    if (check) {
        if (with_pot)
            eps0 ? walk_launch_t<true, true, true>(t, p, b, flags, s) : walk_launch_t<true, false, true>(t, p, b, flags, s);
        else
            eps0 ? walk_launch_t<false, true, true>(t, p, b, flags, s)
                 : walk_launch_t<false, false, true>(t, p, b, flags, s);
    } else {
        if (with_pot)
            eps0 ? walk_launch_t<true, true, false>(t, p, b, flags, s)
                 : walk_launch_t<true, false, false>(t, p, b, flags, s);
        else
            eps0 ? walk_launch_t<false, true, false>(t, p, b, flags, s)
                 : walk_launch_t<false, false, false>(t, p, b, flags, s);
    }
    if (kernel_ev) G2_CUDA(cudaEventRecord(kernel_ev[1], s));
    G2_CUDA(cudaGetLastError());
}

void launch_walk_finalize(const WalkBuffers& b, uint32_t n_sinks_cap, double* ax, double* ay, double* az,
                          double* pot, cudaStream_t s) {
    const unsigned blocks = std::max(1u, std::min<unsigned>(ceil_div(n_sinks_cap, 256), kNumSMs * 8));
    G2_COUNT(1), finalize_kernel<<<blocks, 256, 0, s>>>(b, n_sinks_cap, ax, ay, az, pot);
    G2_CUDA(cudaGetLastError());
}

}  // namespace g2
