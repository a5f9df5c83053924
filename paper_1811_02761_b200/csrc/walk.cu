// walkTree on sm_100a: warp-cooperative sink-group traversal with a shared
// interaction list, acceleration MAC and FP32 rsqrtf force flush.
//
// Reference semantics (traversal.cpp:16-156, engine.cpp:31-81):
//   * sinks in Morton-rank order are chunked into groups of group_size; each
//     group gets an AABB-centred bounding sphere and a_min (make_group);
//   * a cell is tested iff its parent was tested and rejected, so the set of
//     MAC evaluations, accepted cells and opened leaves does not depend on the
//     visiting order; events (interactions, mac_evals, list_pushes) are
//     therefore reproduced exactly by any order, and accelerations differ only
//     by FP32 summation order;
//   * MAC decisions are evaluated in FP64 with the reference's operation
//     order (exact), forces in FP32 on group-relative coordinates.
//
// Execution model:
//   * one warp = one task (group, subtree root); lane l owns sink l;
//   * per-warp shared memory holds the interaction list (float4 x,y,z,m) and
//     the top of a depth-first cell stack (32 cells popped per round, one per
//     lane), spilling to a per-warp global stack;
//   * persistent grid, dynamic task queue: initially one task per group; a
//     warp holding a large stack while the queue runs dry donates the
//     shallow half of its stack as (group, cell) tasks — this splits the
//     heavy-tailed "whole-system" groups across warps.  Partial
//     accelerations are combined with FP32 atomics.
#include "kernels.cuh"

namespace g2 {
namespace {

constexpr int kWarps = 4;
constexpr int kThreads = 32 * kWarps;
constexpr int kLcap = 256;                 // interaction-list entries per warp
constexpr int kScap = 384;                 // shared stack entries per warp
constexpr uint32_t kSpillWords = 16384;    // global stack entries per warp
constexpr uint64_t kEmpty = ~0ull;
constexpr unsigned kFull = 0xffffffffu;

struct WarpSmem {
    float4 list[kLcap];
    uint32_t stack[kScap];
};

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
template <bool kPot, bool kEps0>
__device__ __forceinline__ void flush_list(const float4* __restrict__ list, int cnt, float sx, float sy, float sz,
                                           float eps2, float& ax, float& ay, float& az, float& ph) {
#pragma unroll 4
    for (int e = 0; e < cnt; ++e) {
        const float4 q = list[e];
        const float dx = q.x - sx, dy = q.y - sy, dz = q.z - sz;
        float r2 = fmaf(dx, dx, eps2);
        r2 = fmaf(dy, dy, r2);
        r2 = fmaf(dz, dz, r2);
        float inv = rsqrtf(r2);
        if (kEps0) inv = r2 > 0.0f ? inv : 0.0f;  // r2 == 0 self term (traversal.cpp:73)
        const float mi = q.w * inv;
        const float f = mi * (inv * inv);
        ax = fmaf(f, dx, ax);
        ay = fmaf(f, dy, ay);
        az = fmaf(f, dz, az);
        if (kPot) {
            const float d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
            ph -= d2 > 0.0f ? mi : 0.0f;  // self potential excluded (traversal.cpp:78)
        }
    }
}

template <bool kPot, bool kEps0, bool kCheck>
__global__ void __launch_bounds__(kThreads) walk_kernel(TreeView t, WalkParams p, WalkBuffers b, DevFlags* flags) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    WarpSmem& sm = reinterpret_cast<WarpSmem*>(smem_raw)[w];
    uint32_t* spill = b.spill + (size_t(blockIdx.x) * kWarps + w) * kSpillWords;
    uint32_t* q_head = b.qstate;
    uint32_t* q_tail = b.qstate + 1;
    uint32_t* q_pending = b.qstate + 2;
    const uint32_t ng = b.qstate[3];  // initial tasks (written by walk_init)
    const uint32_t glo = b.group_lo;
    const float eps2 = float(p.eps * p.eps);
    const float G = float(p.G);
    const int donate_below = int(gridDim.x) * kWarps / 4 + 1;

    while (true) {
        // ---------------- acquire a task
        uint32_t ti = 0;
        if (lane == 0) ti = atomicAdd(q_head, 1u);
        ti = __shfl_sync(kFull, ti, 0);
        uint32_t grp, root;
        if (ti < ng) {
            grp = glo + ti;
            root = 0;
        } else {
            uint64_t e = kEmpty;
            if (lane == 0) {
                const uint32_t qi = ti - ng;
                unsigned backoff = 32;
                while (true) {
                    if (qi < b.queue_cap) {
                        e = ld_vol64(&b.queue[qi]);
                        if (e != kEmpty) {
                            st_vol64(&b.queue[qi], kEmpty);  // self-cleaning for the next launch
                            break;
                        }
                    }
                    if (ld_vol(q_pending) == 0) break;
                    __nanosleep(backoff);
                    backoff = backoff < 1024 ? backoff * 2 : 1024;
                }
            }
            e = __shfl_sync(kFull, e, 0);
            if (e == kEmpty) return;
            grp = uint32_t(e >> 32);
            root = uint32_t(e);
        }

        // ---------------- group and sinks
        const GroupRec g = b.groups[grp];
        const bool geom = p.force_geometric || g.a_min <= 0.0;  // engine.cpp:66
        const double rhs = dmul(p.dacc, g.a_min);
        const bool has_sink = uint32_t(lane) < g.count;
        float sx = 0.f, sy = 0.f, sz = 0.f;
        if (has_sink) {
            const double4 q = t.xyzm[b.sinks[g.first + lane]];
            sx = float(dsub(q.x, g.cx)), sy = float(dsub(q.y, g.cy)), sz = float(dsub(q.z, g.cz));
        }
        float ax = 0.f, ay = 0.f, az = 0.f, ph = 0.f;
        uint32_t macs = 0, pushes = 0;
        // logical LIFO = spill[gbase, gtop) (bottom, global) ++ sm.stack[0, ssize) (top, shared)
        int ssize = 1, gbase = 0, gtop = 0, lsize = 0, iter = 0;
        if (lane == 0) sm.stack[0] = root;
        __syncwarp();

        while (ssize + gtop - gbase > 0) {
            // ---- pop up to 32 cells, one per lane
            int take;
            uint32_t c = 0;
            if (ssize > 0) {
                take = min(ssize, 32);
                if (lane < take) c = sm.stack[ssize - 1 - lane];
                ssize -= take;
            } else {
                take = min(gtop - gbase, 32);
                if (lane < take) c = spill[gtop - 1 - lane];
                gtop -= take;
                if (gtop == gbase) gtop = gbase = 0;
            }
            __syncwarp();
            macs += take;
            const bool valid = lane < take;

            // ---- acceleration / geometric MAC, FP64 exact (traversal.cpp:40-56)
            bool accept = false, leaf = false;
            uint32_t link = 0, info = 0;
            double ncx = 0, ncy = 0, ncz = 0, nm = 0;
            if (valid) {
                const WNode nd = t.nodes[c];
                link = nd.link, info = nd.info;
                leaf = (info & kLeafBit) != 0;
                ncx = nd.cx, ncy = nd.cy, ncz = nd.cz, nm = nd.mass;
                const double dx = dsub(g.cx, nd.cx), dy = dsub(g.cy, nd.cy), dz = dsub(g.cz, nd.cz);
                const double d = smax(0.0, dsub(dsqrt(norm2(dx, dy, dz)), g.radius));
                if (d > 0.0) {
                    if (geom) {
                        accept = nd.extent <= dmul(p.theta, d);
                    } else {
                        const double d2 = dmul(d, d);
                        const double lhs = ddiv(dmul(dmul(dmul(p.G, nd.mass), nd.extent), nd.extent), dmul(d2, d2));
                        accept = lhs <= rhs;
                    }
                }
            }
            const uint32_t npush = valid ? (accept ? 1u : (leaf ? (info & ~kLeafBit) : 0u)) : 0u;
            const uint32_t nchild = (valid && !accept && !leaf) ? (info & 0xffu) : 0u;

            // ---- rejected internal cells: children onto the stack
            uint32_t ctot;
            const uint32_t cofs = warp_excl_scan(nchild, ctot);
            if (ctot) {
                if (kCheck && nchild)
                    atomicAdd(&b.level_count[size_t(grp - glo) * (kMaxDepth + 1) + ((info >> 8) & 31u) + 1u], nchild);
                if (ssize + int(ctot) > kScap) {
                    // shared part full: move it onto the spill top, keeping one logical
                    // LIFO (spill = bottom, shared = top) so the depth-first bound holds
                    if (gtop + ssize > int(kSpillWords) && gbase > 0) {  // compact the deque
                        for (int i0 = 0; i0 < gtop - gbase; i0 += 32) {
                            const int i = i0 + lane;
                            const uint32_t v = i < gtop - gbase ? spill[gbase + i] : 0u;
                            __syncwarp();
                            if (i < gtop - gbase) spill[i] = v;
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
                if (ssize + int(ctot) <= kScap) {
                    for (uint32_t j = 0; j < nchild; ++j) sm.stack[ssize + cofs + j] = link + j;
                    ssize += int(ctot);
                }
            }

            // ---- accepted cells and opened leaves: interaction-list entries
            uint32_t ptot;
            const uint32_t pofs = warp_excl_scan(npush, ptot);
            pushes += ptot;
            if (ptot) {
                int pos = lsize + int(pofs), end_all = lsize + int(ptot);
                uint32_t j = 0;
                while (true) {
                    for (; j < npush && pos + int(j) < kLcap; ++j) {
                        float4 en;
                        if (accept) {
                            en = make_float4(float(dsub(ncx, g.cx)), float(dsub(ncy, g.cy)), float(dsub(ncz, g.cz)),
                                             float(nm));
                        } else {
                            const double4 q = t.xyzm[link + j];
                            en = make_float4(float(dsub(q.x, g.cx)), float(dsub(q.y, g.cy)), float(dsub(q.z, g.cz)),
                                             float(q.w));
                        }
                        sm.list[pos + j] = en;
                    }
                    if (end_all < kLcap) {
                        lsize = end_all;
                        break;
                    }
                    __syncwarp();
                    flush_list<kPot, kEps0>(sm.list, kLcap, sx, sy, sz, eps2, ax, ay, az, ph);
                    __syncwarp();
                    pos -= kLcap;
                    end_all -= kLcap;
                    if (end_all == 0) {
                        lsize = 0;
                        break;
                    }
                }
            }
            __syncwarp();

            // ---- donate from the logical bottom (shallowest cells = largest subtrees)
            // when the queue runs dry: splits heavy groups across warps
            const int live = ssize + gtop - gbase;
            if ((++iter & 3) == 0 && live >= 64) {
                int k = 0;
                uint32_t r = 0;
                if (lane == 0) {
                    const int avail = int(ld_vol(q_tail)) - int(ld_vol(q_head));
                    if (avail < donate_below) {
                        k = min(live / 2, 32);
                        if (gtop == gbase) k = min(k, ssize);
                        else k = min(k, gtop - gbase);
                        r = atomicAdd(q_tail, uint32_t(k));
                        const long long room = (long long)ng + b.queue_cap - r;
                        k = int(room < 0 ? 0 : (room < k ? room : k));
                        if (k) {
                            atomicAdd(q_pending, uint32_t(k));
                            __threadfence();
                        }
                    }
                }
                k = __shfl_sync(kFull, k, 0);
                r = __shfl_sync(kFull, r, 0);
                if (k && gtop > gbase) {
                    if (lane < k) st_vol64(&b.queue[r - ng + lane], (uint64_t(grp) << 32) | spill[gbase + lane]);
                    gbase += k;
                    if (gbase == gtop) gbase = gtop = 0;
                    __syncwarp();
                } else if (k) {
                    if (lane < k) st_vol64(&b.queue[r - ng + lane], (uint64_t(grp) << 32) | sm.stack[lane]);
                    __syncwarp();
                    for (int base = 0; base < ssize - k; base += 32) {
                        const int i = base + lane;
                        const uint32_t v = i < ssize - k ? sm.stack[i + k] : 0u;
                        __syncwarp();
                        if (i < ssize - k) sm.stack[i] = v;
                        __syncwarp();
                    }
                    ssize -= k;
                }
            }
        }
        if (lsize) flush_list<kPot, kEps0>(sm.list, lsize, sx, sy, sz, eps2, ax, ay, az, ph);
        __syncwarp();

        // ---------------- results and events
        if (has_sink) {
            float4* acc = &b.accum[g.first + lane];
            atomicAdd(&acc->x, G * ax);
            atomicAdd(&acc->y, G * ay);
            atomicAdd(&acc->z, G * az);
            if (kPot) atomicAdd(&acc->w, G * ph);
        }
        if (lane == 0) {
            const unsigned long long inter = (unsigned long long)pushes * g.count;
            if (p.count_ops) {
                atomicAdd(&b.events[0], inter);
                atomicAdd(&b.events[1], (unsigned long long)macs);
                atomicAdd(&b.events[2], (unsigned long long)pushes);
            }
            if (b.group_inter) atomicAdd(reinterpret_cast<unsigned long long*>(&b.group_inter[grp]), inter);
            __threadfence();
            atomicSub(q_pending, 1u);
        }
    }
}

// one warp per group: AABB centre, radius and a_min (make_group, traversal.cpp:16-38)
__global__ void __launch_bounds__(256) groups_kernel(TreeView t, const double* __restrict__ amag, WalkBuffers b,
                                                     uint32_t gs) {
    const uint32_t n_sinks = *b.n_sinks;
    const uint32_t n_groups = (n_sinks + gs - 1) / gs;
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (gw == 0 && lane == 0) *b.n_groups = n_groups;
    for (uint32_t g = gw; g < n_groups; g += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t first = g * gs;
        const uint32_t cnt = min(gs, n_sinks - first);
        const bool on = uint32_t(lane) < cnt;
        double4 q = make_double4(0, 0, 0, 0);
        double am = INFINITY;
        if (on) {
            const uint32_t k = b.sinks[first + lane];
            q = t.xyzm[k];
            am = amag[k];
        }
        // members[0] seeds lo/hi; min/max are exact in any order
        const double q0x = __shfl_sync(kFull, q.x, 0), q0y = __shfl_sync(kFull, q.y, 0),
                     q0z = __shfl_sync(kFull, q.z, 0);
        double lx = on ? q.x : q0x, ly = on ? q.y : q0y, lz = on ? q.z : q0z;
        double hx = lx, hy = ly, hz = lz;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lx = smin(lx, __shfl_xor_sync(kFull, lx, o));
            ly = smin(ly, __shfl_xor_sync(kFull, ly, o));
            lz = smin(lz, __shfl_xor_sync(kFull, lz, o));
            hx = smax(hx, __shfl_xor_sync(kFull, hx, o));
            hy = smax(hy, __shfl_xor_sync(kFull, hy, o));
            hz = smax(hz, __shfl_xor_sync(kFull, hz, o));
            am = smin(am, __shfl_xor_sync(kFull, am, o));
        }
        const double cx = dmul(dadd(lx, hx), 0.5), cy = dmul(dadd(ly, hy), 0.5), cz = dmul(dadd(lz, hz), 0.5);
        double r2 = on ? norm2(dsub(q.x, cx), dsub(q.y, cy), dsub(q.z, cz)) : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r2 = smax(r2, __shfl_xor_sync(kFull, r2, o));
        if (lane == 0) b.groups[g] = GroupRec{cx, cy, cz, dsqrt(r2), am, first, cnt};
    }
}

__global__ void walk_init_kernel(WalkBuffers b) {
    if (threadIdx.x == 0) {
        const uint32_t n_groups = *b.n_groups;
        const uint32_t hi = min(b.group_hi, n_groups);
        const uint32_t ng = hi > b.group_lo ? hi - b.group_lo : 0u;
        b.qstate[0] = 0;
        b.qstate[1] = ng;
        b.qstate[2] = ng;
        b.qstate[3] = ng;
    }
}

__global__ void zero_accum_kernel(float4* accum, const uint32_t* n_sinks, uint32_t cap) {
    const uint32_t n = min(*n_sinks, cap);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
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

template <bool kPot, bool kEps0, bool kCheck>
int walk_blocks_per_sm() {
    static int v = 0;
    if (!v) {
        const int smem = kWarps * int(sizeof(WarpSmem));
        G2_CUDA(cudaFuncSetAttribute(walk_kernel<kPot, kEps0, kCheck>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     smem));
        G2_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, walk_kernel<kPot, kEps0, kCheck>, kThreads, smem));
        if (v < 1) v = 1;
    }
    return v;
}

template <bool kPot, bool kEps0, bool kCheck>
void walk_launch_t(const TreeView& t, const WalkParams& p, const WalkBuffers& b, DevFlags* flags, cudaStream_t s) {
    const int per_sm = walk_blocks_per_sm<kPot, kEps0, kCheck>();
    const unsigned grid = unsigned(per_sm * kNumSMs);
    G2_COUNT(1), walk_kernel<kPot, kEps0, kCheck><<<grid, kThreads, kWarps * sizeof(WarpSmem), s>>>(t, p, b, flags);
}

}  // namespace

size_t walk_spill_words() { return kSpillWords; }
size_t walk_resident_warps() {
    // upper bound over the template variants (same smem, similar registers)
    return size_t(kNumSMs) * 16 * kWarps;
}

void launch_groups(const TreeView& t, const double* acc_old_mag, const WalkBuffers& b, uint32_t group_size,
                   uint32_t n_sinks_cap, cudaStream_t s) {
    const uint32_t ng = (n_sinks_cap + group_size - 1) / group_size;
    const unsigned blocks = std::max(1u, std::min<unsigned>(ceil_div(size_t(ng) * 32, 256), kNumSMs * 16));
    G2_COUNT(1), groups_kernel<<<blocks, 256, 0, s>>>(t, acc_old_mag, b, group_size);
    G2_CUDA(cudaGetLastError());
}

void launch_walk(const TreeView& t, const WalkParams& p, const WalkBuffers& b, bool with_pot, uint32_t n_sinks_cap,
                 DevFlags* flags, cudaStream_t s) {
    const unsigned zb = std::max(1u, std::min<unsigned>(ceil_div(n_sinks_cap, 256), kNumSMs * 8));
    G2_COUNT(1), zero_accum_kernel<<<zb, 256, 0, s>>>(b.accum, b.n_sinks, n_sinks_cap);
    G2_COUNT(1), walk_init_kernel<<<1, 32, 0, s>>>(b);
    const bool eps0 = p.eps == 0.0;
    const bool check = b.level_count != nullptr;
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
    G2_CUDA(cudaGetLastError());
}

void launch_walk_finalize(const WalkBuffers& b, uint32_t n_sinks_cap, double* ax, double* ay, double* az,
                          double* pot, cudaStream_t s) {
    const unsigned blocks = std::max(1u, std::min<unsigned>(ceil_div(n_sinks_cap, 256), kNumSMs * 8));
    G2_COUNT(1), finalize_kernel<<<blocks, 256, 0, s>>>(b, n_sinks_cap, ax, ay, az, pot);
    G2_CUDA(cudaGetLastError());
}

}  // namespace g2
