// Shared device/host definitions for the g2 octree-gravity engine (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <utility>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace g2 {

// ---- status codes (mirror gravitree/errors.hpp:8-23 + main.cpp:30-33) ---------
enum Status : int { kOk = 0, kInternal = 1, kDataError = 3, kResourceError = 4, kSingularity = 5 };

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define G2_CUDA(expr)                                                                                  \
    do {                                                                                               \
        cudaError_t _e = (expr);                                                                       \
        if (_e != cudaSuccess)                                                                         \
            throw ::g2::Error(::g2::kInternal, std::string("CUDA: ") + cudaGetErrorString(_e) + " at " \
                                                   + __FILE__ + ":" + std::to_string(__LINE__));       \
    } while (0)

// Device-side error flags, read back at API boundaries.
struct DevFlags {
    int data_error;       // non-finite position / position outside root cube (morton.hpp:39, octree.cpp:31)
    int resource_error;   // frontier cap exceeded (traversal.cpp:145-146)
    int singularity;      // eps == 0 coincident pair in direct_sum (gravity.cpp:32-33)
    int cell_overflow;    // cell buffer too small: host grows it and rebuilds
    int stack_overflow;   // walk stack spill area exhausted (internal, sized to never trigger)
    int queue_overflow;   // walk task queue exhausted (internal)
    int tie_run;          // a run of equal keys too long for the in-place tie repair (host re-sorts by id)
    int task_pool;        // walk task records exhausted: a donation was skipped (host grows the pool)
    int peer_timeout;     // a peer rank did not arrive at the device-side exchange barrier in time
};

constexpr int kMaxDepth = 21;        // octree.hpp:47
constexpr int kMortonBits = 21;      // morton.hpp:9
constexpr int kMaxBlockLevel = 24;   // integrator.hpp:14
constexpr int kNumSMs = 148;

// Walk-ready node record: FP64 monopole (calc_node output, octree.hpp:26-30)
// plus the topology link the traversal needs, padded to two whole 32-B sectors so that records
// written in any order (leaves in particle order) never leave partially written sectors.
//   internal: link = first_child, info = child_count
//   leaf:     link = first particle (sorted index), info = count | kLeafBit
struct alignas(32) WNode {
    double cx, cy, cz, mass, extent;
    uint32_t link, info;
    uint32_t pad[4];
};
static_assert(sizeof(WNode) == 64, "WNode is two 32-B sectors");
constexpr uint32_t kLeafBit = 0x80000000u;

// Compact walk record (32 B, one 256-bit load): the FP32-rounded centre of mass,
// mass, extent and q = m b^2 for the FP32 MAC screen, and the same link/info as
// WNode.  The exact FP64 WNode is read only for undecided MAC evaluations.
struct alignas(32) WNode32 {
    float cx, cy, cz, m;
    float b, q;
    uint32_t link, info;
};
// Leaf particles are read by the walk as float4 rel[k] = (x_k - c, m_k): the
// position relative to the leaf's FP32-rounded centre of mass c (one FP64
// difference, rounded).  An opened leaf then yields list entries
// (c - group centre) + rel in FP32 with no FP64 work per particle.

// ---- exact FP64 helpers: explicit _rn intrinsics are never contracted into FMA,
// so device results match the reference's x86-64 SSE2 arithmetic bit for bit.
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }
// std::min / std::max argument conventions (matter only for signed zeros).
__device__ __forceinline__ double smin(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return a < b ? b : a; }
__device__ __forceinline__ double norm2(double x, double y, double z) {
    return dadd(dadd(dmul(x, x), dmul(y, y)), dmul(z, z));
}

// Host-side count of kernel launches issued by the library (bench evidence).
inline std::atomic<unsigned long long>& launch_counter() {
    static std::atomic<unsigned long long> c{0};
    return c;
}
#define G2_COUNT(k) (::g2::launch_counter() += (k))

// Programmatic dependent launch: a kernel launched with launch_pdl may start while the previous
// kernel of its stream drains; it must begin with G2_PDL_WAIT() (griddepcontrol.wait: the previous
// grid complete, its writes visible) before touching memory.  Used only where the previous operation
// in the stream is a kernel (no event wait, memset or copy in between).  G2_NO_PDL: plain launches.
#define G2_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
inline bool pdl_enabled() {
    static const bool on = std::getenv("G2_NO_PDL") == nullptr;
    return on;
}
template <typename... K, typename... A>
inline void launch_pdl(void (*kernel)(K...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid, cfg.blockDim = block, cfg.dynamicSmemBytes = smem, cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr, cfg.numAttrs = pdl_enabled() ? 1 : 0;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...);
    if (e != cudaSuccess) throw std::runtime_error(std::string("launch_pdl: ") + cudaGetErrorString(e));
}

inline unsigned ceil_div(size_t a, size_t b) { return static_cast<unsigned>((a + b - 1) / b); }

// Grow-only device buffer.
template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t cap = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() {
        if (p) cudaFree(p);
    }
    void reserve(size_t n) {
        if (n <= cap) return;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        if (n == 0) return;
        G2_CUDA(cudaMalloc(&p, n * sizeof(T)));
        cap = n;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    operator T*() const { return p; }
};

// ---- single-pass decoupled look-back scan (shared by split, compaction, sort) ----
// Status word per tile: bits 62-63 flag (1 = aggregate, 2 = inclusive prefix),
// bits 0-61 value.  One 64-bit word carries flag and value together, so a
// relaxed store/load pair is enough for correctness.
constexpr uint64_t kLbAgg = 1ull << 62;
constexpr uint64_t kLbInc = 2ull << 62;
constexpr uint64_t kLbMask = (1ull << 62) - 1;

__device__ __forceinline__ void lb_store(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t lb_load(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Called by ONE full warp of the tile.  Publishes `aggregate` for tile `tile`
// and returns the exclusive prefix of all earlier tiles (same on all lanes).
__device__ __forceinline__ uint64_t lookback_warp(uint64_t* status, uint32_t tile, uint64_t aggregate) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) lb_store(&status[0], kLbInc | aggregate);
        return 0;
    }
    if (lane == 0) lb_store(&status[tile], kLbAgg | aggregate);
    uint64_t excl = 0;
    int64_t base = static_cast<int64_t>(tile) - 1;  // lane l inspects tile base - l
    while (true) {
        const int64_t t = base - lane;
        uint64_t s = t >= 0 ? lb_load(&status[t]) : kLbInc;  // virtual inclusive 0 before tile 0
        // wait until every inspected predecessor has published something
        while (__any_sync(0xffffffffu, (s >> 62) == 0)) {
            if ((s >> 62) == 0) s = lb_load(&status[t]);
        }
        const unsigned inc = __ballot_sync(0xffffffffu, (s >> 62) == 2);
        // lanes up to and including the first inclusive one contribute
        const int stop = inc ? __ffs(inc) - 1 : 31;
        uint64_t v = lane <= stop ? (s & kLbMask) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (inc) break;
        base -= 32;
    }
    if (lane == 0) lb_store(&status[tile], kLbInc | (excl + aggregate));
    return excl;
}

}  // namespace g2
