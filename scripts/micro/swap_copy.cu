// Times the qubit-swap gather / scatter kernel of dist.cu (the exact code,
// csrc/swap_copy.cuh) on one GPU at 33 qubits, against a plain
// cudaMemcpyAsync of the same bytes. A swap step of m bit pairs gathers
// (1 - 2^-m) of the local slice into staging and scatters the same amount
// back: per kernel read + write of the moved bytes.
//   nvcc -O3 -std=c++20 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -I paper_2512_18995_b200/csrc scripts/micro/swap_copy.cu -o /tmp/swap_copy
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

namespace qsv {
namespace {
#include "swap_copy.cuh"
}
} // namespace qsv
using namespace qsv;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

int main(int argc, char **argv) {
    const int nl = argc > 1 ? std::atoi(argv[1]) : 32;  // local qubits (33 c64 / 32 c128 = 64 GiB)
    const int amp = argc > 2 ? std::atoi(argv[2]) : 16;
    const uint64_t n = 1ull << nl;
    void *state = nullptr, *stage = nullptr;
    CK(cudaMalloc(&state, n * amp));
    const uint64_t set_cap = 256ull << 20;  // bytes per staging set, as dist.cu
    CK(cudaMalloc(&stage, 2 * set_cap));
    CK(cudaMemset(state, 0, n * amp));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    struct Case { int m; int pos[6]; const char *what; };
    std::vector<Case> cases = {
        {1, {nl - 1}, "1 pair, top local bit (contiguous halves)"},
        {1, {nl - 9}, "1 pair, mid bit"},
        {1, {3}, "1 pair, bit 3 (64/128-byte runs)"},
        {3, {nl - 3, nl - 2, nl - 1}, "3 pairs, top bits (8 ranks)"},
        {3, {4, 12, 20}, "3 pairs, scattered bits"},
    };
    for (const Case &c : cases) {
        BlockBits bb{};
        bb.m = c.m;
        for (int i = 0; i < c.m; ++i) bb.pos[i] = c.pos[i];
        const int nv = (1 << c.m) - 1;
        std::vector<unsigned> vs;
        for (int v = 1; v <= nv; ++v) vs.push_back(v);
        unsigned *d_vs;
        CK(cudaMalloc(&d_vs, sizeof(unsigned) * nv));
        CK(cudaMemcpy(d_vs, vs.data(), sizeof(unsigned) * nv, cudaMemcpyHostToDevice));
        const uint64_t block = n >> c.m;
        // elements per block per round: a power of two, as dist.cu
        uint64_t chunk = 1;
        while (chunk * 2 <= std::min<uint64_t>(block, (set_cap / amp) / nv)) chunk *= 2;
        const bool pair64 = amp == 8 && bb.pos[0] >= 1 && chunk % 2 == 0;
        BlockBits bbv = bb;
        if (pair64)
            for (int i = 0; i < c.m; ++i) bbv.pos[i] -= 1;
        auto run = [&](int dir) {
            for (uint64_t e0 = 0; e0 < block; e0 += chunk) {
                const uint64_t c = std::min(chunk, block - e0);
                const uint64_t cnt = pair64 ? c / 2 : c, s0 = pair64 ? e0 / 2 : e0;
                dim3 grid((unsigned)std::max<uint64_t>(1, std::min<uint64_t>((cnt + 255) / 256, (148 * 8 + nv - 1) / nv)), nv);
                if (amp == 16 || pair64)
                    block_copy_kernel<double2><<<grid, 256>>>((double2 *)state, (double2 *)stage, pair64 ? bbv : bb, s0, cnt, d_vs, dir);
                else
                    block_copy_kernel<float2><<<grid, 256>>>((float2 *)state, (float2 *)stage, bb, e0, c, d_vs, dir);
            }
        };
        const double moved = double(block) * nv * amp;  // bytes per gather (read + write each)
        for (int dir = 0; dir < 2; ++dir) {
            run(dir);
            CK(cudaDeviceSynchronize());
            cudaEventRecord(a);
            for (int it = 0; it < 3; ++it) run(dir);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            ms /= 3;
            std::printf("nl=%d amp=%d %-40s %s: %.3f ms  %.0f GB/s (read+write)\n", nl, amp, c.what,
                        dir ? "scatter" : "gather ", ms, 2 * moved / (ms / 1e3) / 1e9);
        }
        cudaFree(d_vs);
    }
    // reference: device-to-device copy of 1 GiB chunks totalling half the state
    {
        const uint64_t bytes = n * amp / 2;
        cudaEventRecord(a);
        for (uint64_t off = 0; off < bytes; off += set_cap)
            cudaMemcpyAsync(stage, (char *)state + off, set_cap, cudaMemcpyDeviceToDevice);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        std::printf("cudaMemcpyAsync D2D %.1f GiB in 256 MiB chunks: %.3f ms  %.0f GB/s (read+write)\n",
                    bytes / double(1 << 30), ms, 2.0 * bytes / (ms / 1e3) / 1e9);
    }
    return 0;
}
