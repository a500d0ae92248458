// DRAM pattern microbenchmark 2 (diagnostics): 128-byte runs at a 64 MiB
// stride (the first QFT pass at 30 qubits), varying the load/store cache
// hints and how many neighbouring tiles one CTA handles back to back.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
typedef unsigned long long u64;
template <int LD, int ST>
__global__ void __launch_bounds__(256) k2(double2 *st, int L, int K, int P, u64 ntiles, int tpc) {
    const int lowb = P - L;
    for (u64 t = (u64)blockIdx.x * tpc; t < ntiles && t < (u64)(blockIdx.x + 1) * tpc; ++t) {
        const u64 tlo = t & ((1ull << lowb) - 1), thi = t >> lowb;
        const u64 tb = (tlo << L) | (thi << (P + K - L));
        double2 v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int u = threadIdx.x + i * 256;
            const u64 g = tb | ((u64)(u >> L) << P) | (u & ((1 << L) - 1));
            v[i] = LD == 0 ? __ldcs(&st[g]) : (LD == 1 ? __ldcg(&st[g]) : st[g]);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int u = threadIdx.x + i * 256;
            const u64 g = tb | ((u64)(u >> L) << P) | (u & ((1 << L) - 1));
            v[i].x += 1.0;
            if (ST == 0) __stcs(&st[g], v[i]);
            else if (ST == 1) __stcg(&st[g], v[i]);
            else st[g] = v[i];
        }
    }
}
template <int LD, int ST>
void run(double2 *st, int n, int L, int P, int tpc, const char *name) {
    const int K = 11;
    const u64 ntiles = 1ull << (n - K);
    const unsigned grid = (unsigned)((ntiles + tpc - 1) / tpc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k2<LD, ST><<<grid, 256>>>(st, L, K, P, ntiles, tpc);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k2<LD, ST><<<grid, 256>>>(st, L, K, P, ntiles, tpc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    printf("%-8s L=%d P=%2d tpc=%2d: %.3f ms %.0f GB/s\n", name, L, P, tpc, ms, 32.0 * (1ull << n) / (ms * 1e-3) / 1e9);
}
int main() {
    const int n = 30;
    double2 *st;
    cudaMalloc(&st, sizeof(double2) << n);
    cudaMemset(st, 0, sizeof(double2) << n);
    for (int P : {3, 14, 22}) {
        for (int tpc : {1, 2, 4}) {
            run<0, 0>(st, n, 3, P, tpc, "cs/cs");
            run<1, 1>(st, n, 3, P, tpc, "cg/cg");
            run<2, 2>(st, n, 3, P, tpc, "def/def");
            run<1, 2>(st, n, 3, P, tpc, "cg/def");
        }
        run<0, 0>(st, n, 4, P < 4 ? 4 : P, 1, "cs/cs");
        run<2, 2>(st, n, 4, P < 4 ? 4 : P, 1, "def/def");
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
