// Measured FP64 (DFMA) and FP32 (FFMA, packed FFMA2) throughput of this B200:
// the compute-roofline denominators of the complex128 (cfg4) and complex64
// (cfg5) passes ("measure the DFMA and FFMA2 peaks on the box").
// Each thread runs 8 independent FMA chains (no dependency stalls), all SMs,
// enough warps to saturate; reported as FMA/s and FLOP/s (2 per FMA).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp_peaks scripts/micro/fp_peaks.cu
#include <cuda_runtime.h>

#include <cstdio>

template <typename T> __global__ void fma_chains(T *out, int iters, T a, T b) {
    T x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = static_cast<T>(threadIdx.x + j);
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = x[j] * a + b;
    T s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j];
    if (s == static_cast<T>(-12345)) out[threadIdx.x] = s;  // keep the chains alive
}

__global__ void ffma2_chains(float *out, int iters, float a, float b) {
    unsigned long long x[8];
    unsigned long long av, bv;
    asm("mov.b64 %0, {%1,%1};" : "=l"(av) : "f"(a));
    asm("mov.b64 %0, {%1,%1};" : "=l"(bv) : "f"(b));
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const float f = threadIdx.x + j;
        asm("mov.b64 %0, {%1,%1};" : "=l"(x[j]) : "f"(f));
    }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[j]) : "l"(av), "l"(bv));
    float s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        float lo, hi;
        asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[j]));
        s += lo + hi;
    }
    if (s == -12345.f) out[threadIdx.x] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *o;
    cudaMalloc(&o, 4096);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256, iters = 1 << 14;
    const double fmas = double(blocks) * threads * iters * 8;
    auto run = [&](const char *name, auto launch, double per) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= 5;
        const double rate = per * fmas / (ms / 1e3);
        std::printf("%-6s %8.3f ms  %7.2f T FMA/s  %7.2f TFLOP/s\n", name, ms, rate / 1e12, 2 * rate / 1e12);
    };
    run("DFMA", [&] { fma_chains<double><<<blocks, threads>>>(reinterpret_cast<double *>(o), iters, 0.999, 1e-3); }, 1.0);
    run("FFMA", [&] { fma_chains<float><<<blocks, threads>>>(o, iters, 0.999f, 1e-3f); }, 1.0);
    run("FFMA2", [&] { ffma2_chains<<<blocks, threads>>>(o, iters, 0.999f, 1e-3f); }, 2.0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    std::printf("SMs %d, max SM clock %.0f MHz\n", sms, clk / 1e3);
    return 0;
}
