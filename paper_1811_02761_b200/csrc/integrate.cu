// Block-time-step integrator (integrator.cpp:21-164), bootstrap direct sum
// (gravity.cpp:18-43) and active-set compaction on sm_100a.  FP64 state,
// explicit round-to-nearest intrinsics: given identical accelerations the
// predictor/corrector/level updates are bit-identical to the reference.
#include <algorithm>
#include <vector>

#include "kernels.cuh"

namespace g2 {
namespace {

constexpr int kBlock = 256;
inline unsigned grid_for(size_t n) { return std::max(1u, std::min<unsigned>(ceil_div(n, kBlock), kNumSMs * 16)); }

// ---- direct_sum: one thread per sink, sources in index order (bit-exact) -----
__global__ void __launch_bounds__(kBlock) direct_kernel(const double4* __restrict__ xyzm, uint32_t n, double G,
                                                        double eps2, double* __restrict__ ax, double* __restrict__ ay,
                                                        double* __restrict__ az, DevFlags* flags) {
    __shared__ double4 tile[kBlock];
    const uint32_t i = blockIdx.x * kBlock + threadIdx.x;
    const double4 ri = i < n ? xyzm[i] : make_double4(0, 0, 0, 0);
    double sx = 0.0, sy = 0.0, sz = 0.0;
    bool singular = false;
    for (uint32_t base = 0; base < n; base += kBlock) {
        __syncthreads();
        if (base + threadIdx.x < n) tile[threadIdx.x] = xyzm[base + threadIdx.x];
        __syncthreads();
        const uint32_t m = min(uint32_t(kBlock), n - base);
        if (i < n) {
            for (uint32_t jj = 0; jj < m; ++jj) {
                const uint32_t j = base + jj;
                if (j == i) continue;
                const double4 q = tile[jj];
                const double dx = dsub(q.x, ri.x), dy = dsub(q.y, ri.y), dz = dsub(q.z, ri.z);
                const double d2 = norm2(dx, dy, dz);
                if (eps2 == 0.0 && d2 == 0.0) {
                    singular = true;
                    continue;
                }
                const double r2 = dadd(d2, eps2);  // softened_accel (gravity.hpp:15-20)
                if (r2 == 0.0) continue;
                const double inv = ddiv(1.0, dsqrt(r2));
                const double f = dmul(dmul(dmul(dmul(G, q.w), inv), inv), inv);
                sx = dadd(sx, dmul(dx, f));
                sy = dadd(sy, dmul(dy, f));
                sz = dadd(sz, dmul(dz, f));
            }
        }
    }
    if (singular) flags->singularity = 1;
    if (i < n) ax[i] = sx, ay[i] = sy, az[i] = sz;
}

__global__ void __launch_bounds__(kBlock) norm3_kernel(const double* ax, const double* ay, const double* az,
                                                       double* out, size_t n) {
    for (size_t i = blockIdx.x * size_t(kBlock) + threadIdx.x; i < n; i += size_t(gridDim.x) * kBlock)
        out[i] = dsqrt(norm2(ax[i], ay[i], az[i]));
}

__device__ __forceinline__ uint64_t level_ticks(int level) { return 1ull << (kMaxBlockLevel - level); }

// ---- t_next = min_i last_update + ticks(level) (integrator.cpp:103-105) -------
// 16 particles per thread and step (one 16-byte load of levels, eight of update times), one atomic
// per block (a same-address atomic per warp serialised at L2)
__global__ void __launch_bounds__(kBlock) tnext_kernel(const uint8_t* __restrict__ level,
                                                       const uint64_t* __restrict__ last, size_t n,
                                                       unsigned long long* t_next) {
    unsigned long long m = ~0ull;
    const size_t n16 = n / 16;
    for (size_t i = blockIdx.x * size_t(kBlock) + threadIdx.x; i < n16; i += size_t(gridDim.x) * kBlock) {
        const uint4 lv = reinterpret_cast<const uint4*>(level)[i];
        const uint32_t lw[4] = {lv.x, lv.y, lv.z, lv.w};
        const ulonglong2* lp = reinterpret_cast<const ulonglong2*>(last) + 8 * i;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const ulonglong2 t = lp[q];
            const uint32_t w = lw[q >> 1], sh = 16 * (q & 1);
            m = min(m, (unsigned long long)(t.x + level_ticks(uint8_t(w >> sh))));
            m = min(m, (unsigned long long)(t.y + level_ticks(uint8_t(w >> (sh + 8)))));
        }
    }
    for (size_t i = 16 * n16 + blockIdx.x * size_t(kBlock) + threadIdx.x; i < n; i += size_t(gridDim.x) * kBlock)
        m = min(m, (unsigned long long)(last[i] + level_ticks(level[i])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    __shared__ unsigned long long wm[kBlock / 32];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 1; q < kBlock / 32; ++q) m = min(m, wm[q]);
        if (m != ~0ull) atomicMin(t_next, m);
    }
}

// ---- predict (integrator.cpp:40-45) on ALL particles + active flags (:107-110), two particles per
// thread with 16-byte loads/stores of the SoA arrays (more bytes in flight per thread; cudaMalloc'd
// arrays are 256-byte aligned, so pairs are 16-byte aligned)
__device__ __forceinline__ void predict_one(double4& p, double& vx, double& vy, double& vz, double ax, double ay,
                                            double az, double dt, double h) {
    p.x = dadd(p.x, dadd(dmul(vx, dt), dmul(ax, h)));
    p.y = dadd(p.y, dadd(dmul(vy, dt), dmul(ay, h)));
    p.z = dadd(p.z, dadd(dmul(vz, dt), dmul(az, h)));
    vx = dadd(vx, dmul(ax, dt));
    vy = dadd(vy, dmul(ay, dt));
    vz = dadd(vz, dmul(az, dt));
}
// bbox (nullable): also the bounding-cube partials of the predicted positions (bounding_cube,
// octree.cpp:24-49: min / max are exact in any order), one record of 6 per block, so a rebuild
// that follows needs only bbox_final_kernel instead of another pass over the positions
__global__ void __launch_bounds__(kBlock) predict_kernel(StepState st, size_t n, const unsigned long long* t_next_p,
                                                          uint64_t now, double tick, uint8_t* __restrict__ active,
                                                          double* __restrict__ bbox, DevFlags* flags) {
    G2_PDL_WAIT();  // programmatic dependent launch (launch_pdl)
    const uint64_t t_next = *t_next_p;
    const double dt = dmul(double(t_next - now), tick);
    const double h = dmul(dmul(0.5, dt), dt);
    const size_t np = n / 2;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    bool bad = false;
    auto fold = [&](const double4& p) {
        bad |= !(isfinite(p.x) && isfinite(p.y) && isfinite(p.z));
        lo[0] = smin(lo[0], p.x), lo[1] = smin(lo[1], p.y), lo[2] = smin(lo[2], p.z);
        hi[0] = smax(hi[0], p.x), hi[1] = smax(hi[1], p.y), hi[2] = smax(hi[2], p.z);
    };
    for (size_t i = blockIdx.x * size_t(kBlock) + threadIdx.x; i < np; i += size_t(gridDim.x) * kBlock) {
        double4 p0 = st.xyzm[2 * i], p1 = st.xyzm[2 * i + 1];
        double2 vx = reinterpret_cast<const double2*>(st.vx)[i], vy = reinterpret_cast<const double2*>(st.vy)[i];
        double2 vz = reinterpret_cast<const double2*>(st.vz)[i];
        const double2 ax = reinterpret_cast<const double2*>(st.ax)[i], ay = reinterpret_cast<const double2*>(st.ay)[i];
        const double2 az = reinterpret_cast<const double2*>(st.az)[i];
        const ulonglong2 lu = reinterpret_cast<const ulonglong2*>(st.last_update)[i];
        const uchar2 lv = reinterpret_cast<const uchar2*>(st.level)[i];
        predict_one(p0, vx.x, vy.x, vz.x, ax.x, ay.x, az.x, dt, h);
        predict_one(p1, vx.y, vy.y, vz.y, ax.y, ay.y, az.y, dt, h);
        st.xyzm[2 * i] = p0, st.xyzm[2 * i + 1] = p1;
        if (bbox) fold(p0), fold(p1);
        reinterpret_cast<double2*>(st.vx)[i] = vx, reinterpret_cast<double2*>(st.vy)[i] = vy;
        reinterpret_cast<double2*>(st.vz)[i] = vz;
        if (active)
            reinterpret_cast<uchar2*>(active)[i] =
                make_uchar2(lu.x + level_ticks(lv.x) == t_next ? 1 : 0, lu.y + level_ticks(lv.y) == t_next ? 1 : 0);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {  // odd tail
        const size_t i = n - 1;
        double4 p = st.xyzm[i];
        double vx = st.vx[i], vy = st.vy[i], vz = st.vz[i];
        predict_one(p, vx, vy, vz, st.ax[i], st.ay[i], st.az[i], dt, h);
        st.xyzm[i] = p, st.vx[i] = vx, st.vy[i] = vy, st.vz[i] = vz;
        if (active) active[i] = (st.last_update[i] + level_ticks(st.level[i]) == t_next) ? 1 : 0;
        if (bbox) fold(p);
    }
    if (!bbox) return;
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
        bbox[blockIdx.x * 6 + threadIdx.x] = v;
    }
}

// ---- block_level (integrator.cpp:21-33) ------------------------------------------
__device__ int block_level_dev(double acc_mag, const SchemeDev& s) {
    if (!s.adaptive) return max(0, min(s.fixed_level, kMaxBlockLevel));
    if (acc_mag <= 0.0) return 0;
    const double dt = dmul(s.eta, dsqrt(ddiv(s.eps, acc_mag)));
    if (dt <= 0.0) return kMaxBlockLevel;
    if (dt >= s.dt_max) return 0;
    const double lg = ceil(log2(ddiv(s.dt_max, dt)));
    int level = lg >= double(kMaxBlockLevel) ? kMaxBlockLevel : (lg <= 0.0 ? 0 : int(lg));
    // the fix-up loops make the result independent of log2 rounding
    while (level < kMaxBlockLevel && ddiv(s.dt_max, double(1ull << level)) > dt) ++level;
    while (level > 0 && ddiv(s.dt_max, double(1ull << (level - 1))) <= dt) --level;
    return level;
}

// ---- correct loop over active sinks (integrator.cpp:148-156, apply_level :86-95)
// new accelerations straight from the walk's FP32 accumulators (slot s = sink s): the same
// double(float) values the finalize pass would store, without the FP64 round trip
__global__ void __launch_bounds__(kBlock) correct_kernel(StepState st, const uint32_t* __restrict__ sinks,
                                                         const uint32_t* n_sinks, uint32_t cap,
                                                         const float4* __restrict__ acc4,
                                                         const unsigned long long* t_next_p, uint64_t now, double tick,
                                                         SchemeDev sc) {
    G2_PDL_WAIT();  // programmatic dependent launch (launch_pdl)
    const uint32_t na = min(*n_sinks, cap);
    const uint64_t t_next = *t_next_p;
    for (uint32_t s = blockIdx.x * kBlock + threadIdx.x; s < na; s += gridDim.x * kBlock) {
        const uint32_t i = sinks[s];
        const double h = dmul(0.5, dmul(double(t_next - st.last_update[i]), tick));
        const float4 a4 = acc4[s];
        const double ax = double(a4.x), ay = double(a4.y), az = double(a4.z);
        st.vx[i] = dadd(st.vx[i], dmul(dsub(ax, st.ax[i]), h));
        st.vy[i] = dadd(st.vy[i], dmul(dsub(ay, st.ay[i]), h));
        st.vz[i] = dadd(st.vz[i], dmul(dsub(az, st.az[i]), h));
        st.ax[i] = ax, st.ay[i] = ay, st.az[i] = az;
        const double amag = dsqrt(norm2(ax, ay, az));
        st.amag[i] = amag;
        st.last_update[i] = t_next;
        if (sc.adaptive) {
            const int target = block_level_dev(amag, sc);
            const int current = st.level[i];
            int next = max(current - 1, min(target, current + 1));  // at most one level per step
            next = max(0, min(next, kMaxBlockLevel));
            if (next < current && now % level_ticks(next) != 0) next = current;  // uses the previous sync time
            st.level[i] = uint8_t(next);
        }
    }
}

__global__ void __launch_bounds__(kBlock) assign_levels_kernel(StepState st, size_t n, SchemeDev sc) {
    for (size_t i = blockIdx.x * size_t(kBlock) + threadIdx.x; i < n; i += size_t(gridDim.x) * kBlock)
        st.level[i] = uint8_t(block_level_dev(dsqrt(norm2(st.ax[i], st.ay[i], st.az[i])), sc));
}

// ---- order-preserving compaction of byte flags (decoupled look-back) ----------
constexpr int kCItems = 16;
constexpr int kCTile = kBlock * kCItems;

__global__ void __launch_bounds__(kBlock) compact_kernel(const uint8_t* __restrict__ flags, size_t n,
                                                         uint32_t* __restrict__ out, uint32_t* __restrict__ n_out,
                                                         uint64_t* __restrict__ status, uint32_t* counter) {
    __shared__ uint32_t s_tile, s_wsum[kBlock / 32];
    __shared__ uint64_t s_excl;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const size_t base = size_t(tile) * kCTile + size_t(tid) * kCItems;  // blocked: thread owns 16 consecutive
    uint32_t bits = 0;
    if (base + kCItems <= n) {  // one 16-byte load of the thread's flags
        static_assert(kCItems == 16, "flag vector load");
        const uint4 v = *reinterpret_cast<const uint4*>(flags + base);
        const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < kCItems; ++k)
            if ((w4[k >> 2] >> (8 * (k & 3))) & 0xffu) bits |= 1u << k;
    } else {
#pragma unroll
        for (int k = 0; k < kCItems; ++k)
            if (base + k < n && flags[base + k]) bits |= 1u << k;
    }
    const uint32_t x = __popc(bits);
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) s_wsum[w] = inc;
    __syncthreads();
    uint32_t wpre = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < kBlock / 32; ++k) {
        if (k < w) wpre += s_wsum[k];
        tot += s_wsum[k];
    }
    if (w == 0) {
        const uint64_t e = lookback_warp(status, tile, tot);
        if (lane == 0) s_excl = e;
    }
    __syncthreads();
    uint32_t o = uint32_t(s_excl) + wpre + inc - x;
#pragma unroll
    for (int k = 0; k < kCItems; ++k)
        if (bits & (1u << k)) out[o++] = uint32_t(base + k);
    const uint32_t ntiles = uint32_t((n + kCTile - 1) / kCTile);
    if (tile == ntiles - 1 && tid == 0) *n_out = uint32_t(s_excl) + tot;
}

// ---- compute_diagnostics (diagnostics.cpp:10-38) ---------------------------------
// kinetic energy and momentum: per-block FP64 partial sums (fixed launch => reruns bit-identical)
__global__ void __launch_bounds__(kBlock) kinetic_kernel(const double* __restrict__ mass, const double* __restrict__ vel3,
                                                         size_t n, double* __restrict__ partial) {
    double k = 0.0, px = 0.0, py = 0.0, pz = 0.0;
    for (size_t i = blockIdx.x * size_t(kBlock) + threadIdx.x; i < n; i += size_t(gridDim.x) * kBlock) {
        const double m = mass[i], vx = vel3[3 * i], vy = vel3[3 * i + 1], vz = vel3[3 * i + 2];
        k = dadd(k, dmul(dmul(0.5, m), norm2(vx, vy, vz)));
        px = dadd(px, dmul(m, vx)), py = dadd(py, dmul(m, vy)), pz = dadd(pz, dmul(m, vz));
    }
    __shared__ double sh[4][kBlock / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        k += __shfl_xor_sync(0xffffffffu, k, o), px += __shfl_xor_sync(0xffffffffu, px, o);
        py += __shfl_xor_sync(0xffffffffu, py, o), pz += __shfl_xor_sync(0xffffffffu, pz, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) sh[0][w] = k, sh[1][w] = px, sh[2][w] = py, sh[3][w] = pz;
    __syncthreads();
    if (threadIdx.x < 4) {
        double v = 0.0;
        for (int q = 0; q < kBlock / 32; ++q) v += sh[threadIdx.x][q];
        partial[4 * blockIdx.x + threadIdx.x] = v;
    }
}

// direct potential energy: phi_i = sum_{j != i} -G m_j / sqrt(r2 + eps2) (softened_potential,
// gravity.hpp:22-26) in FP64, sources tiled through shared memory; W = 1/2 sum_i m_i phi_i
__global__ void __launch_bounds__(kBlock) direct_potential_kernel(const double4* __restrict__ xyzm, uint32_t n,
                                                                  double G, double eps2, double* __restrict__ wpart,
                                                                  DevFlags* flags) {
    __shared__ double4 tile[kBlock];
    const uint32_t i = blockIdx.x * kBlock + threadIdx.x;
    const double4 ri = i < n ? xyzm[i] : make_double4(0, 0, 0, 0);
    double phi = 0.0;
    for (uint32_t base = 0; base < n; base += kBlock) {
        __syncthreads();
        if (base + threadIdx.x < n) tile[threadIdx.x] = xyzm[base + threadIdx.x];
        __syncthreads();
        const uint32_t m = min(uint32_t(kBlock), n - base);
        for (uint32_t q = 0; q < m; ++q) {
            const double4 rj = tile[q];
            if (base + q == i) continue;
            const double d2 = norm2(dsub(rj.x, ri.x), dsub(rj.y, ri.y), dsub(rj.z, ri.z));
            if (eps2 == 0.0 && d2 == 0.0) {
                flags->singularity = 1;  // direct_potential_energy throws (gravity.cpp:55-56)
                continue;
            }
            const double r2 = dadd(d2, eps2);
            phi = dsub(phi, ddiv(dmul(G, rj.w), dsqrt(r2)));
        }
    }
    double w = i < n ? dmul(dmul(0.5, ri.w), phi) : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    __shared__ double sw[kBlock / 32];
    if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = w;
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int q = 0; q < kBlock / 32; ++q) v += sw[q];
        wpart[blockIdx.x] = v;
    }
}

__global__ void __launch_bounds__(kBlock) block_levels_kernel(const double* amag, size_t n, SchemeDev sc, int* out) {
    for (size_t i = blockIdx.x * size_t(kBlock) + threadIdx.x; i < n; i += size_t(gridDim.x) * kBlock)
        out[i] = block_level_dev(amag[i], sc);
}

// predict with an explicit dt on AoS arrays (the free function integrator.cpp:40-45)
__global__ void __launch_bounds__(kBlock) predict_aos_kernel(double* pos, double* vel, const double* acc, size_t n,
                                                             double dt) {
    const double h = dmul(dmul(0.5, dt), dt);
    for (size_t i = blockIdx.x * size_t(kBlock) + threadIdx.x; i < 3 * n; i += size_t(gridDim.x) * kBlock) {
        pos[i] = dadd(pos[i], dadd(dmul(vel[i], dt), dmul(acc[i], h)));
        vel[i] = dadd(vel[i], dmul(acc[i], dt));
    }
}

// Direct summation onto a target subset (accuracy oracle for large N, SURVEY §8f
// rank 2): FP64 pair terms, sources split into chunks across blocks and combined
// with FP64 atomics (summation order differs from the reference's serial loop by
// ~1e-16 relative, far below the tree errors it measures).
constexpr int kDsTargets = 128, kDsChunk = 16384;
__global__ void __launch_bounds__(kDsTargets) direct_targets_kernel(const double4* __restrict__ xyzm, uint32_t n,
                                                                    const uint32_t* __restrict__ targets, uint32_t nt,
                                                                    double G, double eps2, double* __restrict__ acc3) {
    __shared__ double4 tile[kDsTargets];
    const uint32_t t = blockIdx.x * kDsTargets + threadIdx.x;
    const uint32_t me = t < nt ? targets[t] : 0xffffffffu;
    const double4 ri = t < nt ? xyzm[me] : make_double4(0, 0, 0, 0);
    const uint32_t j0 = blockIdx.y * kDsChunk, j1 = min(n, j0 + kDsChunk);
    double sx = 0.0, sy = 0.0, sz = 0.0;
    for (uint32_t base = j0; base < j1; base += kDsTargets) {
        __syncthreads();
        if (base + threadIdx.x < j1) tile[threadIdx.x] = xyzm[base + threadIdx.x];
        __syncthreads();
        const uint32_t m = min(uint32_t(kDsTargets), j1 - base);
        for (uint32_t k = 0; k < m; ++k) {
            if (base + k == me) continue;
            const double4 q = tile[k];
            const double dx = q.x - ri.x, dy = q.y - ri.y, dz = q.z - ri.z;
            const double r2 = dx * dx + dy * dy + dz * dz + eps2;
            if (r2 == 0.0) continue;
            const double inv = rsqrt(r2);
            const double f = G * q.w * inv * inv * inv;
            sx += f * dx, sy += f * dy, sz += f * dz;
        }
    }
    if (t < nt) {
        atomicAdd(&acc3[3 * t], sx);
        atomicAdd(&acc3[3 * t + 1], sy);
        atomicAdd(&acc3[3 * t + 2], sz);
    }
}

}  // namespace

void launch_direct_targets(const double4* xyzm, size_t n, const uint32_t* targets, size_t nt, double G, double eps,
                           double* acc3, cudaStream_t s) {
    G2_CUDA(cudaMemsetAsync(acc3, 0, 3 * nt * sizeof(double), s));
    const dim3 grid(ceil_div(nt, kDsTargets), ceil_div(n, kDsChunk));
    G2_COUNT(1), direct_targets_kernel<<<grid, kDsTargets, 0, s>>>(xyzm, uint32_t(n), targets, uint32_t(nt), G,
                                                                  eps * eps, acc3);
    G2_CUDA(cudaGetLastError());
}

void launch_block_levels(const double* acc_mag, size_t n, SchemeDev sc, int* levels, cudaStream_t s) {
    if (n) G2_COUNT(1), block_levels_kernel<<<grid_for(n), kBlock, 0, s>>>(acc_mag, n, sc, levels);
}
void launch_predict_aos(double* pos3, double* vel3, const double* acc3, size_t n, double dt, cudaStream_t s) {
    if (n) G2_COUNT(1), predict_aos_kernel<<<grid_for(3 * n), kBlock, 0, s>>>(pos3, vel3, acc3, n, dt);
}

void launch_direct_sum(const double4* xyzm, size_t n, double G, double eps, double* ax, double* ay, double* az,
                       DevFlags* flags, cudaStream_t s) {
    G2_COUNT(1), direct_kernel<<<ceil_div(n, kBlock), kBlock, 0, s>>>(xyzm, uint32_t(n), G, eps * eps, ax, ay, az, flags);
    G2_CUDA(cudaGetLastError());
}

void diagnostics_device(const double* mass, const double* vel3, const double4* xyzm, size_t n, double G, double eps,
                        bool direct_potential, double* kin_mom4, double* w_direct, DevFlags* flags, cudaStream_t s) {
    const unsigned kb = std::max(1u, std::min<unsigned>(ceil_div(n, kBlock), kNumSMs * 4));
    DBuf<double> part;
    part.reserve(size_t(4) * kb + 4);
    G2_COUNT(1), kinetic_kernel<<<kb, kBlock, 0, s>>>(mass, vel3, n, part.p);
    std::vector<double> h(4 * size_t(kb));
    G2_CUDA(cudaMemcpyAsync(h.data(), part.p, h.size() * 8, cudaMemcpyDeviceToHost, s));
    DBuf<double> wp;
    const unsigned pb = ceil_div(n, kBlock);
    std::vector<double> hw;
    if (direct_potential) {
        wp.reserve(pb + 1);
        G2_COUNT(1), direct_potential_kernel<<<pb, kBlock, 0, s>>>(xyzm, uint32_t(n), G, eps * eps, wp.p, flags);
        hw.resize(pb);
        G2_CUDA(cudaMemcpyAsync(hw.data(), wp.p, pb * 8, cudaMemcpyDeviceToHost, s));
    }
    G2_CUDA(cudaStreamSynchronize(s));
    for (int q = 0; q < 4; ++q) {
        double v = 0.0;
        for (unsigned b = 0; b < kb; ++b) v += h[4 * b + q];  // fixed merge order
        kin_mom4[q] = v;
    }
    if (direct_potential) {
        double v = 0.0;
        for (unsigned b = 0; b < pb; ++b) v += hw[b];
        *w_direct = v;
    }
}

void launch_norm3(const double* ax, const double* ay, const double* az, double* out, size_t n, cudaStream_t s) {
    G2_COUNT(1), norm3_kernel<<<grid_for(n), kBlock, 0, s>>>(ax, ay, az, out, n);
}

void launch_tnext(const StepState& st, size_t n, unsigned long long* t_next, cudaStream_t s) {
    G2_CUDA(cudaMemsetAsync(t_next, 0xff, sizeof(unsigned long long), s));
    G2_COUNT(1), tnext_kernel<<<std::max(1u, std::min<unsigned>(ceil_div(n, size_t(kBlock) * 16), kNumSMs * 8)), kBlock, 0,
                                 s>>>(st.level, st.last_update, n, t_next);
}

unsigned predict_blocks(size_t n) { return grid_for(n / 2 + 1); }
void launch_predict(const StepState& st, size_t n, const unsigned long long* t_next, uint64_t now, double tick,
                    uint8_t* active_flag, cudaStream_t s, double* bbox_partials, DevFlags* flags) {
    G2_COUNT(1), launch_pdl(predict_kernel, dim3(predict_blocks(n)), dim3(kBlock), size_t(0), s, st, n, t_next, now, tick, active_flag,
                                                                     bbox_partials, flags);
}

void launch_compact(const uint8_t* flags, size_t n, uint32_t* out, uint32_t* n_out, uint64_t* status,
                    uint32_t* counter, cudaStream_t s) {
    const size_t tiles = (n + kCTile - 1) / kCTile;
    G2_CUDA(cudaMemsetAsync(status, 0, tiles * sizeof(uint64_t), s));
    G2_CUDA(cudaMemsetAsync(counter, 0, sizeof(uint32_t), s));
    G2_COUNT(1), compact_kernel<<<unsigned(tiles), kBlock, 0, s>>>(flags, n, out, n_out, status, counter);
    G2_CUDA(cudaGetLastError());
}

void launch_correct(const StepState& st, const uint32_t* sinks, const uint32_t* n_sinks, uint32_t n_cap,
                    const float4* acc4, const unsigned long long* t_next, uint64_t now, double tick, SchemeDev sc,
                    cudaStream_t s) {
    G2_COUNT(1), launch_pdl(correct_kernel, dim3(grid_for(n_cap)), dim3(kBlock), size_t(0), s, st, sinks, n_sinks, n_cap, acc4, t_next, now, tick,
                                                                   sc);
}

void launch_assign_levels(const StepState& st, size_t n, SchemeDev sc, cudaStream_t s) {
    G2_COUNT(1), assign_levels_kernel<<<grid_for(n), kBlock, 0, s>>>(st, n, sc);
}

}  // namespace g2
