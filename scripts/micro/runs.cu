// DRAM access-pattern microbenchmark (diagnostics, not part of the engine):
// in-place read+write of 2^n complex128 amplitudes in "tiles" of 2^K
// amplitudes = 2^(K-L) runs of 2^L contiguous amplitudes at a stride of 2^P
// amplitudes (the shape of a fused tile pass whose tile holds the L lowest
// bits plus K-L bits starting at P). Reports GB/s (read + write).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
typedef unsigned long long u64;
template <int AMPS>
__global__ void __launch_bounds__(256) runs_kernel(double2 *st, int L, int K, int P, u64 ntiles) {
    for (u64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
        // tile index bits: below L -> bits [L, P) ; rest -> above P + (K - L)
        const int lowb = P - L;  // tile-index bits placed between L and P
        const u64 tlo = t & ((1ull << lowb) - 1), thi = t >> lowb;
        const u64 tb = (tlo << L) | (thi << (P + K - L));
        double2 v[AMPS];
#pragma unroll
        for (int i = 0; i < AMPS; ++i) {
            const int u = threadIdx.x + i * 256;
            const u64 g = tb | ((u64)(u >> L) << P) | (u & ((1 << L) - 1));
            v[i] = __ldcs(&st[g]);
        }
#pragma unroll
        for (int i = 0; i < AMPS; ++i) {
            const int u = threadIdx.x + i * 256;
            const u64 g = tb | ((u64)(u >> L) << P) | (u & ((1 << L) - 1));
            v[i].x += 1.0;
            __stcs(&st[g], v[i]);
        }
    }
}
int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 30;
    double2 *st;
    cudaMalloc(&st, sizeof(double2) << n);
    cudaMemset(st, 0, sizeof(double2) << n);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int K = 11;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int Ls[] = {2, 3, 4, 5, 6, 8};
    int Ps[] = {0, 10, 14, 19};  // P = 0 means P = L (fully contiguous tile)
    for (int L : Ls)
        for (int Pi : Ps) {
            const int P = Pi == 0 ? L : (Pi < L ? L : Pi);
            if (P + K - L > n) continue;
            const u64 ntiles = 1ull << (n - K);
            int bpsm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpsm, runs_kernel<8>, 256, 0);
            for (int gm : {1, 0}) {
                const unsigned grid = gm ? bpsm * nsm : (unsigned)ntiles;
                runs_kernel<8><<<grid, 256>>>(st, L, K, P, ntiles);
                cudaEventRecord(e0);
                const int reps = 5;
                for (int r = 0; r < reps; ++r) runs_kernel<8><<<grid, 256>>>(st, L, K, P, ntiles);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                ms /= reps;
                const double gbs = 2.0 * 16.0 * (double)(1ull << n) / (ms * 1e-3) / 1e9;
                printf("L=%d run=%4dB P=%2d stride=%9lluB grid=%s: %.3f ms  %.0f GB/s\n", L, 16 << L, P,
                       16ull << P, gm ? "persist" : "all", ms, gbs);
            }
        }
    cudaError_t err = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(err));
    return 0;
}
