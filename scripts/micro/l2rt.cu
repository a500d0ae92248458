// L2 round-trip microbenchmark (diagnostics): in-place HBM streaming of 2^30
// complex128 (32 KiB tiles, 128-byte runs at a 64 MiB stride, one CTA per
// tile) with and without an extra write + read-back of every tile through a
// per-CTA global scratch slot that should stay resident in L2 (optionally
// discarded from L2 after the read-back so it is never written to DRAM).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
template <int MODE>  // 0 plain, 1 scratch round trip, 2 round trip + discard
__global__ void __launch_bounds__(256) k(double2 *st, double2 *scratch, int *slots, int L, int P, u64 ntiles, int nslot) {
    __shared__ int slot;
    const int K = 11;
    if (MODE) {
        if (threadIdx.x == 0) {
            const unsigned sm = smid();
            int s = -1;
            while (s < 0)
                for (int i = 0; i < nslot && s < 0; ++i)
                    if (atomicCAS(&slots[sm * nslot + i], 0, 1) == 0) s = sm * nslot + i;
            slot = s;
        }
        __syncthreads();
    }
    const u64 t = blockIdx.x;
    const int lowb = P - L;
    const u64 tlo = t & ((1ull << lowb) - 1), thi = t >> lowb;
    const u64 tb = (tlo << L) | (thi << (P + K - L));
    double2 v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int u = threadIdx.x + i * 256;
        v[i] = __ldcs(&st[tb | ((u64)(u >> L) << P) | (u & ((1 << L) - 1))]);
    }
    if (MODE) {
        double2 *sc = scratch + (size_t)slot * 2048;
#pragma unroll
        for (int i = 0; i < 8; ++i) sc[threadIdx.x + i * 256] = v[i];
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = __ldcg(&sc[(threadIdx.x ^ 32) + i * 256]);
        __syncthreads();
        if (MODE == 2) {
            // 32 KiB = 256 lines of 128 B: one discard per thread
            asm volatile("discard.global.L2 [%0], 128;" ::"l"(sc + threadIdx.x * 8) : "memory");
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int u = threadIdx.x + i * 256;
        v[i].x += 1.0;
        __stcs(&st[tb | ((u64)(u >> L) << P) | (u & ((1 << L) - 1))], v[i]);
    }
    if (MODE) {
        __syncthreads();
        if (threadIdx.x == 0) atomicExch(&slots[slot], 0);
    }
}
template <int MODE>
void run(double2 *st, double2 *sc, int *slots, int n, int L, int P, int nslot) {
    const u64 ntiles = 1ull << (n - 11);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<MODE><<<(unsigned)ntiles, 256>>>(st, sc, slots, L, P, ntiles, nslot);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k<MODE><<<(unsigned)ntiles, 256>>>(st, sc, slots, L, P, ntiles, nslot);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("mode=%d L=%d P=%2d: %.3f ms  %.0f GB/s (HBM algorithmic)\n", MODE, L, P, ms, 32.0 * (1ull << n) / (ms * 1e-3) / 1e9);
}
int main() {
    const int n = 30, nslot = 8;
    double2 *st, *sc; int *slots;
    cudaMalloc(&st, sizeof(double2) << n);
    cudaMemset(st, 0, sizeof(double2) << n);
    cudaMalloc(&sc, (size_t)148 * nslot * 2048 * sizeof(double2));
    cudaMalloc(&slots, 148 * nslot * sizeof(int));
    cudaMemset(slots, 0, 148 * nslot * sizeof(int));
    for (int P : {3, 22}) {
        run<0>(st, sc, slots, n, 3, P, nslot);
        run<1>(st, sc, slots, n, 3, P, nslot);
        run<2>(st, sc, slots, n, 3, P, nslot);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
