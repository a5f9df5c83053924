// Morton key of a position in the root cube (morton.hpp:14-44), shared by the key kernel and the
// rebuild's bucket sort.  FP64 with explicit round-to-nearest intrinsics: bit-identical to the reference.
#pragma once

#include "kernels.cuh"

namespace g2 {

__device__ __forceinline__ uint64_t expand_bits(uint64_t v) {
    v &= 0x1fffff;
    v = (v | v << 32) & 0x001f00000000ffffULL;
    v = (v | v << 16) & 0x001f0000ff0000ffULL;
    v = (v | v << 8) & 0x100f00f00f00f00fULL;
    v = (v | v << 4) & 0x10c30c30c30c30c3ULL;
    v = (v | v << 2) & 0x1249249249249249ULL;
    return v;
}

__device__ __forceinline__ uint64_t quantize(double v, double lo, double width) {
    const double t = dmul(ddiv(dsub(v, lo), width), 2097152.0);
    if (t <= 0.0) return 0;
    const unsigned long long q = __double2ull_rz(t);
    return q > 2097151ull ? 2097151ull : q;
}

// quantize() without the FP64 division: y = (v - lo) * (1 / width) differs from the reference's
// correctly rounded quotient q = fl((v - lo) / width) by at most 3.4e-16 |y| (two roundings of the
// product and reciprocal plus q's own half ulp), i.e. t = 2^21 y is within 7.4e-10 of 2^21 q while
// |t| <= 2.2e6 (positions inside the cube give 0 <= t <= 2^21).  Where t is farther than 1e-9 from an integer
// (every coordinate but ~2e-9 of them) floor(t) is the reference's floor, bit for bit; otherwise
// the exact division decides.
__device__ __forceinline__ uint64_t quantize_fast(double v, double lo, double width, double rwidth) {
    const double a = dsub(v, lo);
    const double t = dmul(dmul(a, rwidth), 2097152.0);
    const double f = floor(t);
    const double fr = t - f;  // exact for |t| < 2^52
    if (!(fr > 1e-9 && fr < 1.0 - 1e-9 && fabs(t) <= 2.2e6)) return quantize(v, lo, width);
    if (t <= 0.0) return 0;
    const unsigned long long q = static_cast<unsigned long long>(f);
    return q > 2097151ull ? 2097151ull : q;
}

// expand_bits from a shared-memory table (6 loads per key instead of ~90 integer operations): the
// spread of 11 bits fits 31 bits, so a 21-bit coordinate is T[v & 2047] | T[v >> 11] << 33.
// Every thread of the block calls spread_init, then __syncthreads, before the first key.
struct SpreadTable {
    uint32_t t[2048];
};
__device__ __forceinline__ uint32_t spread11(uint32_t v) {
    v &= 0x7ffu;
    v = (v | v << 16) & 0x070000ffu;
    v = (v | v << 8) & 0x0700f00fu;
    v = (v | v << 4) & 0x430c30c3u;
    v = (v | v << 2) & 0x49249249u;
    return v;
}
__device__ __forceinline__ void spread_init(SpreadTable& st) {
    for (uint32_t i = threadIdx.x; i < 2048; i += blockDim.x) st.t[i] = spread11(i);
}
__device__ __forceinline__ uint64_t spread21(const SpreadTable& st, uint64_t v) {
    return uint64_t(st.t[v & 2047u]) | (uint64_t(st.t[(v >> 11) & 1023u]) << 33);
}

// the cube's lower corner, upper corner and width, in the reference's operation order
struct KeyFrame {
    double lox, loy, loz, hix, hiy, hiz, width, rwidth;
    __device__ __forceinline__ explicit KeyFrame(const Cube& c)
        : lox(dsub(c.cx, c.half)), loy(dsub(c.cy, c.half)), loz(dsub(c.cz, c.half)), hix(dadd(c.cx, c.half)),
          hiy(dadd(c.cy, c.half)), hiz(dadd(c.cz, c.half)), width(dmul(2.0, c.half)), rwidth(ddiv(1.0, width)) {}
    __device__ __forceinline__ bool inside(const double4& p) const {
        return p.x >= lox && p.x <= hix && p.y >= loy && p.y <= hiy && p.z >= loz && p.z <= hiz;
    }
    __device__ __forceinline__ uint64_t key(const double4& p, const SpreadTable& st) const {
        return (spread21(st, quantize_fast(p.x, lox, width, rwidth)) << 2) |
               (spread21(st, quantize_fast(p.y, loy, width, rwidth)) << 1) |
               spread21(st, quantize_fast(p.z, loz, width, rwidth));
    }
    __device__ __forceinline__ uint64_t key(const double4& p) const {
        return (expand_bits(quantize_fast(p.x, lox, width, rwidth)) << 2) |
               (expand_bits(quantize_fast(p.y, loy, width, rwidth)) << 1) |
               expand_bits(quantize_fast(p.z, loz, width, rwidth));
    }
};

}  // namespace g2
