// Measured FP32 CUDA-core peak of this B200 (the walk's roofline denominator).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_peak tools/fp32_peak.cu && ./fp32_peak
// Two kernels at full occupancy (148 SMs x 2048 threads), 8 independent FMA chains per thread:
//   ffma   scalar fma.rn.f32        (one FMA per lane per instruction)
//   ffma2  packed fma.rn.f32x2      (two FMAs per lane per instruction, the walk flush's form)
// Flop = 2 per FMA.  Best of 5 launches, CUDA events; prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 4096;
constexpr int kChains = 8;

__global__ void __launch_bounds__(256) ffma_kernel(float* out, float a, float b) {
    float x[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = threadIdx.x * 1e-3f + c;
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = fmaf(x[c], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 12345.678f) out[0] = s;  // keep the chains alive
}

__global__ void __launch_bounds__(256) ffma2_kernel(float* out, float a, float b) {
    unsigned long long x[kChains], av, bv;
    asm("mov.b64 %0, {%1, %1};" : "=l"(av) : "f"(a));
    asm("mov.b64 %0, {%1, %1};" : "=l"(bv) : "f"(b));
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        const float lo = threadIdx.x * 1e-3f + c, hi = lo + 0.5f;
        asm("mov.b64 %0, {%1, %2};" : "=l"(x[c]) : "f"(lo), "f"(hi));
    }
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(av), "l"(bv));
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[c]));
        s += lo + hi;
    }
    if (s == 12345.678f) out[0] = s;
}

template <typename K>
static double best_tflops(K kern, double fma_per_thread, int blocks, float* out) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0), cudaEventCreate(&e1);
    kern<<<blocks, 256>>>(out, 0.999f, 1e-3f);  // warm-up
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        kern<<<blocks, 256>>>(out, 0.999f, 1e-3f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    return 2.0 * fma_per_thread * double(blocks) * 256.0 / (best * 1e-3) / 1e12;
}

int main() {
    cudaDeviceProp pr;
    cudaGetDeviceProperties(&pr, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* out;
    cudaMalloc(&out, 4);
    const int blocks = pr.multiProcessorCount * 8 * 16;  // 16 waves of full occupancy
    const double t1 = best_tflops(ffma_kernel, double(kIters) * kChains, blocks, out);
    const double t2 = best_tflops(ffma2_kernel, 2.0 * kIters * kChains, blocks, out);
    const double nominal = pr.multiProcessorCount * 128.0 * 2.0 * (clk * 1e3) / 1e12;
    std::printf("{\"ffma_tflops\": %.2f, \"ffma2_tflops\": %.2f, \"nominal_tflops_at_max_clock\": %.2f, "
                "\"sms\": %d, \"max_clock_mhz\": %.0f, \"how\": \"%d blocks x 256 threads, %d chains x %d iters, "
                "best of 5, CUDA events\"}\n",
                t1, t2, nominal, pr.multiProcessorCount, clk / 1e3, blocks, kChains, kIters);
    return 0;
}
