// Super-pass feasibility microbenchmark (diagnostics): two tile passes of the
// 30-qubit QFT geometry (pass A: tile bits {0,1,2} + {22..29}; pass B: tile
// bits {0,1,2} + {14..21}) over 2^30 complex128, each tile loaded to
// registers and stored back. Mode 0 runs them as two kernels (each one HBM
// read + write of the state). Mode 1 runs ONE kernel whose CTAs claim items
// (4 tiles of one pass) from an atomic ticket: the 2^19-amplitude chunks
// (bits {0..2} + {14..29}) are processed as A(c) then, D chunks later, B(c),
// which waits on a per-chunk counter -- so B reads what A wrote while it is
// still in L2 and the state crosses HBM once for two passes.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
typedef unsigned long long u64;

constexpr int NQ = 30, K = 11, TPC = 4, THREADS = 256;
constexpr int TILE_PER_CHUNK = 256;              // 2^(19 - 11)
constexpr u64 NTILES = 1ull << (NQ - K);
constexpr u64 NCHUNK = NTILES / TILE_PER_CHUNK;  // 2048
constexpr int IPC = TILE_PER_CHUNK / TPC;        // items per chunk and pass

// tile t of pass P -> global offset of its amplitude 0; amplitude u -> offset
__device__ __forceinline__ u64 tile_base(int P, u64 t) {
    const u64 in = t & 255, out = t >> 8;  // chunk-internal ext bits, chunk id
    return (out << 3) | (in << (P == 0 ? 14 : 22));
}
__device__ __forceinline__ u64 amp_off(int P, int u) {
    return (u64)(u & 7) | ((u64)(u >> 3) << (P == 0 ? 22 : 14));
}

template <int WB>  // store policy: 0 default (write-back into L2), 1 .cs streaming
__device__ __forceinline__ void st(double2 *p, double2 v) {
    if (WB == 0) *p = v;
    else __stcs(p, v);
}

template <int WB>
__device__ void do_item(double2 *s, int P, u64 t0) {
    for (u64 t = t0; t < t0 + TPC; ++t) {
        const u64 tb = tile_base(P, t);
        double2 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldcg(&s[tb | amp_off(P, k * THREADS + threadIdx.x)]);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            v[k].x *= 1.0000001;
            st<WB>(&s[tb | amp_off(P, k * THREADS + threadIdx.x)], v[k]);
        }
    }
}

template <int WB>
__global__ void __launch_bounds__(THREADS) pass_kernel(double2 *s, int P) { do_item<1>(s, P, (u64)blockIdx.x * TPC); }

template <int WBA>
__global__ void __launch_bounds__(THREADS) fused(double2 *s, unsigned *ticket, unsigned *done, int D) {
    __shared__ unsigned item;
    if (threadIdx.x == 0) item = atomicAdd(ticket, 1u);
    __syncthreads();
    const unsigned it = item;
    const unsigned m = it / (2 * IPC), r = it % (2 * IPC);
    if (r < IPC) {  // A(m)
        if (m >= NCHUNK) return;
        do_item<WBA>(s, 0, (u64)m * TILE_PER_CHUNK + (u64)r * TPC);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(&done[m], 1u);
        }
    } else {        // B(m - D)
        if (m < (unsigned)D) return;
        const unsigned c = m - D;
        if (c >= NCHUNK) return;
        if (threadIdx.x == 0) {
            unsigned v;
            while (true) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&done[c]) : "memory");
                if (v >= (unsigned)IPC) break;
                __nanosleep(100);
            }
        }
        __syncthreads();
        do_item<1>(s, 1, (u64)c * TILE_PER_CHUNK + (u64)(r - IPC) * TPC);
    }
}

int main(int argc, char **argv) {
    double2 *s;
    unsigned *ctr;
    if (cudaMalloc(&s, sizeof(double2) << NQ) != cudaSuccess) return 1;
    cudaMalloc(&ctr, (NCHUNK + 1) * 4);
    cudaMemset(s, 0, sizeof(double2) << NQ);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double gb = 2.0 * (sizeof(double2) << NQ) / 1e9;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        pass_kernel<1><<<NTILES / TPC, THREADS>>>(s, 0);
        pass_kernel<1><<<NTILES / TPC, THREADS>>>(s, 1);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("two kernels          : %.3f ms (%.0f GB/s per pass)\n", ms, 2 * gb / ms * 1e3);
        for (int D : {1, 2, 4, 8}) {
            for (int wb = 0; wb < 2; ++wb) {
                const unsigned nitems = (unsigned)((NCHUNK + D) * 2 * IPC);
                cudaEventRecord(e0);
                cudaMemsetAsync(ctr, 0, (NCHUNK + 1) * 4);
                if (wb == 0) fused<0><<<nitems, THREADS>>>(s, ctr + NCHUNK, ctr, D);
                else fused<1><<<nitems, THREADS>>>(s, ctr + NCHUNK, ctr, D);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                printf("fused D=%d A-stores=%s: %.3f ms (HBM-equivalent %.0f GB/s)\n", D, wb ? "cs     " : "default",
                       ms, gb / ms * 1e3);
            }
        }
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
