// Gather / scatter of a qubit-swap all-to-all (dist.cu): shared with the
// micro-benchmark scripts/micro/swap_copy.cu so ncu can time the exact kernel
// on one GPU. Included inside namespace qsv's anonymous namespace.
#pragma once

// The m local bits of a swap step (ascending positions) and one block's
// values: element e of block v <-> the local index with v's bits deposited
// at those positions.
struct BlockBits {
    int m;
    int pos[8];
};
__device__ __forceinline__ uint64_t deposit(uint64_t e, const BlockBits &bb, unsigned v) {
    uint64_t x = e;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
        if (i >= bb.m) break;
        const int p = bb.pos[i];
        const uint64_t lo = x & ((1ull << p) - 1);
        x = ((x ^ lo) << 1) | (static_cast<uint64_t>((v >> i) & 1u) << p) | lo;
    }
    return x;
}
// gather (dir 0: state -> staging) or scatter (dir 1) of `count` elements
// starting at e0 of every block listed in vs[0..nv): blockIdx.y is the block
// (no per-element division), each thread moves VEC consecutive elements
// (V = 16-byte vector: one c128 or two c64 amplitudes per element pair when
// the lowest swapped bit is >= 1), grid-strided over the chunk.
template <typename V>
__global__ void __launch_bounds__(256) block_copy_kernel(V *__restrict__ state, V *__restrict__ stage, BlockBits bb,
                                                          uint64_t e0, uint64_t count,
                                                          const unsigned *__restrict__ vs, int dir) {
    const unsigned v = vs[blockIdx.y];
    V *const sblk = stage + static_cast<uint64_t>(blockIdx.y) * count;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t idx = deposit(e0 + i, bb, v);
        if (dir == 0) sblk[i] = __ldcs(&state[idx]);
        else __stcs(&state[idx], sblk[i]);
    }
}

