// Microbenchmark: one dense 5-qubit block (a 32x32 complex matrix U) applied
// to a complex64 state, three ways, against a plain copy of the state:
//
//   copy  : read + write every amplitude (the HBM ceiling of any pass)
//   fma   : CUDA cores, one thread per 32-amplitude set, U from shared memory
//           (128 FP32 FMAs per amplitude)
//   tc    : tcgen05 tensor cores, kind::tf32 with a 3xTF32 split
//           (x = hi + lo, D = A_hi B_hi + A_hi B_lo + A_lo B_hi) so the result
//           keeps ~FP32 accuracy. The block is the real 64x64 matrix
//           B[2i+a][2j+b] of U acting on (re, im) pairs; per CTA iteration
//           128 sets are the M = 128 rows of A (K-major, K = 64 reals per
//           set), B = 64 x 64 (N = 64 outputs), the accumulator sits in 64
//           TMEM columns and thread m reads its set's 64 outputs back from
//           TMEM lane m.
//
// The sets are the 5 lowest qubits (32 consecutive amplitudes). This
// measures whether a dense 5-qubit block can run at the HBM roofline on
// tensor cores while the CUDA-core version is FMA-bound -- the question the
// cfg5 family (FMA-pipe bound, profiles/r01_ncu_cfg45_28q.txt) raises.
//
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tc_dense5 tc_dense5.cu
// Run:   ./tc_dense5 [log2 amplitudes = 30]
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                          \
    do {                                                                                               \
        cudaError_t e = (x);                                                                           \
        if (e != cudaSuccess) {                                                                        \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));             \
            std::exit(1);                                                                              \
        }                                                                                              \
    } while (0)

constexpr int kSets = 128;          // sets per CTA iteration (MMA M)
constexpr int kK = 64;              // reals per set (MMA K)
constexpr int kN = 64;              // outputs per set (MMA N)
constexpr int kAbytes = kSets * kK * 4;  // 32 KiB
constexpr int kBbytes = kN * kK * 4;     // 16 KiB

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major, 128-byte swizzle: an atom is 8 rows x 128 B (32 TF32 along K),
// 16-byte chunk c of row r stored at chunk c ^ (r & 7); K = 64 is two atom
// columns, the second ROWS / 8 atoms after the first. Lanes writing 8
// consecutive chunks of one row hit 8 distinct bank groups.
template <int ROWS>
__device__ __forceinline__ uint32_t kmaj_off(int row, int chunk) {
    return (chunk >> 3) * (ROWS / 8) * 1024 + (row >> 3) * 1024 + (row & 7) * 128 + (((chunk & 7) ^ (row & 7)) << 4);
}

// input chunk (set row, 16-byte chunk c) handled by thread t at step j:
// lanes 0..7 take the 8 rows of one core matrix (one 128-byte shared-memory
// line per 8-lane phase: conflict-free), the 4 lane octets and 4 warps cover
// the 16 row groups, the 16 steps the 16 chunks
__device__ __forceinline__ int in_row(int t, int j) { return (t + 128 * j) >> 4; }
__device__ __forceinline__ int in_chunk(int t, int j) { return (t + 128 * j) & 15; }
__device__ __forceinline__ float4 ld_in(const float4 *base, int t, int j) { return __ldcs(base + t + 128 * j); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((addr >> 4) & 0x3fff);
    d |= 1ull << 16;                                          // LBO (unused with swizzle)
    d |= static_cast<uint64_t>((1024 >> 4) & 0x3fff) << 32;  // SBO: 8-row atoms 1 KiB apart
    d |= 1ull << 46;                                          // version (sm_100)
    d |= 2ull << 61;                                          // SWIZZLE_128B
    return d;
}
// start of MMA k-step ks (K = 8 TF32 = 32 B) of an operand with ROWS rows
template <int ROWS>
__device__ __forceinline__ uint32_t kstep(int ks) { return (ks >> 2) * (ROWS / 8) * 1024 + (ks & 3) * 32; }

__device__ __forceinline__ float tf32_hi(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// G warpgroups per CTA share B; each has its own A hi / lo, TMEM columns and
// mbarrier and runs the load / split / MMA / drain loop on its own sets
template <int G>
__global__ void __launch_bounds__(128 * G, G == 1 ? 2 : 1) tc_kernel(const float4 *__restrict__ in,
                                                                    float4 *__restrict__ out,
                                                                    const float *__restrict__ Bg,
                                                                    uint64_t nsets_total) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char *sm = sm_raw + ((1024 - (smem_u32(sm_raw) & 1023)) & 1023);  // swizzle atoms need 1 KiB alignment
    const int g = threadIdx.x >> 7, t = threadIdx.x & 127, warp = t >> 5;
    unsigned char *Ahi = sm + g * 2 * kAbytes, *Alo = Ahi + kAbytes, *Bhi = sm + G * 2 * kAbytes,
                  *Blo = Bhi + kBbytes;
    constexpr uint32_t kCols = G == 1 ? 64 : G == 2 ? 128 : 256;
    __shared__ uint64_t mbars[G];
    uint64_t &mbar = mbars[g];
    __shared__ uint32_t tmem_base;
    // B hi / lo (row n = output, k contiguous)
    for (int q = threadIdx.x; q < kN * kK / 4; q += 128 * G) {
        const int n = q / (kK / 4), c = q % (kK / 4);
        float4 v = reinterpret_cast<const float4 *>(Bg)[q];
        float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
        float4 l = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
        *reinterpret_cast<float4 *>(Bhi + kmaj_off<kN>(n, c)) = h;
        *reinterpret_cast<float4 *>(Blo + kmaj_off<kN>(n, c)) = l;
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base + g * 64;
    // kind::tf32, D f32, A/B tf32 K-major, N = 64, M = 128
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((kN >> 3) << 17) | ((128 >> 4) << 24);
    uint32_t phase = 0;
    const uint64_t iters = nsets_total / kSets;
    // software pipeline: the next iteration's 32 KiB are loaded into
    // registers while this iteration's MMAs and output stores run
    float4 v[16];
    const uint64_t step = static_cast<uint64_t>(gridDim.x) * G;
    uint64_t it = static_cast<uint64_t>(blockIdx.x) * G + g;
    if (it < iters) {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = ld_in(in + it * (kSets * kK / 4), t, j);
    }
    for (; it < iters; it += step) {
        // chunk q = t + 128 j = (set m, 4-real chunk c), split into hi / lo
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int m = in_row(t, j), c = in_chunk(t, j);
            float4 h = make_float4(tf32_hi(v[j].x), tf32_hi(v[j].y), tf32_hi(v[j].z), tf32_hi(v[j].w));
            float4 l = make_float4(v[j].x - h.x, v[j].y - h.y, v[j].z - h.z, v[j].w - h.w);
            *reinterpret_cast<float4 *>(Ahi + kmaj_off<kSets>(m, c)) = h;
            *reinterpret_cast<float4 *>(Alo + kmaj_off<kSets>(m, c)) = l;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync %0, 128;" ::"r"(g + 1) : "memory");
        if (t == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;");
            const unsigned char *As[3] = {Ahi, Ahi, Alo};
            const unsigned char *Bs[3] = {Bhi, Blo, Bhi};
            int acc = 0;
            for (int p = 0; p < 3; ++p)
                for (int ks = 0; ks < kK / 8; ++ks) {
                    const uint64_t ad = sdesc(smem_u32(As[p]) + kstep<kSets>(ks));
                    const uint64_t bd = sdesc(smem_u32(Bs[p]) + kstep<kN>(ks));
                    asm volatile(
                        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                        "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                    acc = 1;
                }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&mbar)));
        }
        if (it + step < iters) {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = ld_in(in + (it + step) * (kSets * kK / 4), t, j);
        }
        // wait for the MMAs (bounded spin: a wrong descriptor must not hang the box)
        {
            uint32_t done = 0;
            for (long spin = 0; !done; ++spin) {
                asm volatile(
                    "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                    : "=r"(done)
                    : "r"(smem_u32(&mbar)), "r"(phase));
                if (spin > (1l << 26)) __trap();
            }
        }
        phase ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;");
        uint32_t r[64];
        const uint32_t taddr = tmem + ((static_cast<uint32_t>(warp) * 32) << 16);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%"
            "19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%"
            "46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
              "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
              "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
              "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
              "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
              "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        // stage through Alo (its MMAs completed): row t, chunk c at the
        // XOR-swizzled slot c ^ (t & 15) -- conflict-free both ways -- then
        // coalesced 16-byte stores
        float4 *stg = reinterpret_cast<float4 *>(Alo);
#pragma unroll
        for (int c = 0; c < 16; ++c)
            stg[t * 16 + (c ^ (t & 15))] = make_float4(__uint_as_float(r[4 * c]), __uint_as_float(r[4 * c + 1]),
                                                       __uint_as_float(r[4 * c + 2]), __uint_as_float(r[4 * c + 3]));
        asm volatile("bar.sync %0, 128;" ::"r"(g + 1) : "memory");
        float4 *dst = out + it * (kSets * kK / 4);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int q = t + 128 * j, m = q >> 4, c = q & 15;
            __stcs(dst + q, stg[m * 16 + (c ^ (m & 15))]);
        }
        // the next iteration overwrites A: every thread's TMEM read is done
        // and no MMA is in flight (waited above)
        asm volatile("tcgen05.fence::before_thread_sync;");
        asm volatile("bar.sync %0, 128;" ::"r"(g + 1) : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kCols));
}

// NB dense blocks per tile, back to back: the question a fused pass with
// several 5-qubit stages asks (cfg5: ~7 one-layer blocks per 13-qubit tile).
// After each block's MMAs the accumulator is drained to registers, split
// into hi / lo again and written as the next block's A (thread t = set row
// t, conflict-free in the 128-byte-swizzled K-major layout); only the last
// block's output goes back to HBM. Same B for every block (timing only).
template <int NB>
__global__ void __launch_bounds__(128, 2) tc_chain_kernel(const float4 *__restrict__ in, float4 *__restrict__ out,
                                                         const float *__restrict__ Bg, uint64_t nsets_total) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char *sm = sm_raw + ((1024 - (smem_u32(sm_raw) & 1023)) & 1023);
    const int t = threadIdx.x, warp = t >> 5;
    unsigned char *Ahi = sm, *Alo = Ahi + kAbytes, *Bhi = sm + 2 * kAbytes, *Blo = Bhi + kBbytes;
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base;
    for (int q = t; q < kN * kK / 4; q += 128) {
        const int n = q / (kK / 4), c = q % (kK / 4);
        float4 v = reinterpret_cast<const float4 *>(Bg)[q];
        float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
        float4 l = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
        *reinterpret_cast<float4 *>(Bhi + kmaj_off<kN>(n, c)) = h;
        *reinterpret_cast<float4 *>(Blo + kmaj_off<kN>(n, c)) = l;
    }
    if (t < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(64));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((kN >> 3) << 17) | ((128 >> 4) << 24);
    uint32_t phase = 0;
    const uint64_t iters = nsets_total / kSets;
    for (uint64_t it = blockIdx.x; it < iters; it += gridDim.x) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const float4 v = ld_in(in + it * (kSets * kK / 4), t, j);
            const int m = in_row(t, j), c = in_chunk(t, j);
            float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
            float4 l = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
            *reinterpret_cast<float4 *>(Ahi + kmaj_off<kSets>(m, c)) = h;
            *reinterpret_cast<float4 *>(Alo + kmaj_off<kSets>(m, c)) = l;
        }
        uint32_t r[64];
        for (int b = 0; b < NB; ++b) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (t == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;");
                const unsigned char *As[3] = {Ahi, Ahi, Alo};
                const unsigned char *Bs[3] = {Bhi, Blo, Bhi};
                int acc = 0;
                for (int p = 0; p < 3; ++p)
                    for (int ks = 0; ks < kK / 8; ++ks) {
                        const uint64_t ad = sdesc(smem_u32(As[p]) + kstep<kSets>(ks));
                        const uint64_t bd = sdesc(smem_u32(Bs[p]) + kstep<kN>(ks));
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                        acc = 1;
                    }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    smem_u32(&mbar)));
            }
            {
                uint32_t done = 0;
                for (long spin = 0; !done; ++spin) {
                    asm volatile(
                        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                        : "=r"(done)
                        : "r"(smem_u32(&mbar)), "r"(phase));
                    if (spin > (1l << 26)) __trap();
                }
            }
            phase ^= 1;
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t taddr = tmem + ((static_cast<uint32_t>(warp) * 32) << 16);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%"
                "19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%"
                "46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                  "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                  "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
                  "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
                  "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
                  "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
                  "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncthreads();  // every MMA read of A is done (waited) before A is rewritten
            if (b + 1 < NB) {
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    const float4 v = make_float4(__uint_as_float(r[4 * c]), __uint_as_float(r[4 * c + 1]),
                                                 __uint_as_float(r[4 * c + 2]), __uint_as_float(r[4 * c + 3]));
                    float4 h = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
                    float4 l = make_float4(v.x - h.x, v.y - h.y, v.z - h.z, v.w - h.w);
                    *reinterpret_cast<float4 *>(Ahi + kmaj_off<kSets>(t, c)) = h;
                    *reinterpret_cast<float4 *>(Alo + kmaj_off<kSets>(t, c)) = l;
                }
            }
        }
        float4 *stg = reinterpret_cast<float4 *>(Alo);
#pragma unroll
        for (int c = 0; c < 16; ++c)
            stg[t * 16 + (c ^ (t & 15))] = make_float4(__uint_as_float(r[4 * c]), __uint_as_float(r[4 * c + 1]),
                                                       __uint_as_float(r[4 * c + 2]), __uint_as_float(r[4 * c + 3]));
        __syncthreads();
        float4 *dst = out + it * (kSets * kK / 4);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int q = t + 128 * j, m = q >> 4, c = q & 15;
            __stcs(dst + q, stg[m * 16 + (c ^ (m & 15))]);
        }
        __syncthreads();
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    __syncthreads();
    if (t < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(64));
}

// CUDA cores: thread = one set, D[n] = sum_k B[n][k] x[k] (B from shared memory)
__global__ void __launch_bounds__(128) fma_kernel(const float4 *__restrict__ in, float4 *__restrict__ out,
                                                  const float *__restrict__ Bg, uint64_t nsets_total) {
    __shared__ float Bs[kN * kK];
    for (int q = threadIdx.x; q < kN * kK; q += 128) Bs[q] = Bg[q];
    __syncthreads();
    for (uint64_t s = blockIdx.x * 128ull + threadIdx.x; s < nsets_total; s += gridDim.x * 128ull) {
        float x[kK];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            float4 v = __ldcs(in + s * 16 + c);
            x[4 * c] = v.x, x[4 * c + 1] = v.y, x[4 * c + 2] = v.z, x[4 * c + 3] = v.w;
        }
#pragma unroll 1
        for (int n = 0; n < kN; n += 4) {
            float y[4] = {0, 0, 0, 0};
#pragma unroll
            for (int k = 0; k < kK; ++k)
#pragma unroll
                for (int j = 0; j < 4; ++j) y[j] = fmaf(Bs[(n + j) * kK + k], x[k], y[j]);
            __stcs(out + s * 16 + n / 4, make_float4(y[0], y[1], y[2], y[3]));
        }
    }
}

__global__ void copy_kernel(const float4 *__restrict__ in, float4 *__restrict__ out, uint64_t n4) {
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n4; i += gridDim.x * 256ull) __stcs(out + i, __ldcs(in + i));
}

int main(int argc, char **argv) {
    const int lg = argc > 1 ? std::atoi(argv[1]) : 30;
    const uint64_t namp = 1ull << lg, nsets = namp / 32, n4 = namp * 2 / 4;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    // U: a seeded dense complex 32x32 (not unitary -- accuracy is relative)
    std::vector<float> Ur(32 * 32), Ui(32 * 32), B(kN * kK);
    uint64_t x = 0x9e3779b97f4a7c15ull;
    auto rnd = [&] {
        x ^= x << 13, x ^= x >> 7, x ^= x << 17;
        return static_cast<float>((x >> 11) * (1.0 / 9007199254740992.0)) - 0.5f;
    };
    for (int i = 0; i < 32 * 32; ++i) Ur[i] = rnd() * 0.35f, Ui[i] = rnd() * 0.35f;
    for (int i = 0; i < 32; ++i)
        for (int j = 0; j < 32; ++j) {
            B[(2 * i) * kK + 2 * j] = Ur[i * 32 + j];
            B[(2 * i) * kK + 2 * j + 1] = -Ui[i * 32 + j];
            B[(2 * i + 1) * kK + 2 * j] = Ui[i * 32 + j];
            B[(2 * i + 1) * kK + 2 * j + 1] = Ur[i * 32 + j];
        }
    float *dB, *din, *dout;
    CK(cudaMalloc(&dB, B.size() * 4));
    CK(cudaMalloc(&din, namp * 8));
    CK(cudaMalloc(&dout, namp * 8));
    CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
    {
        std::vector<float> h(1 << 20);
        for (uint64_t off = 0; off < namp * 2; off += h.size()) {
            for (auto &v : h) v = rnd();
            CK(cudaMemcpy(din + off, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
        }
    }
    const int smem = 2 * kAbytes + 2 * kBbytes + 1024, smem3 = 3 * 2 * kAbytes + 2 * kBbytes + 1024;
    CK(cudaFuncSetAttribute(tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(tc_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto timeit = [&](const char *name, auto launch, double flop_per_amp) {
        launch();
        CK(cudaDeviceSynchronize());
        const int reps = 10;
        CK(cudaEventRecord(e0));
        for (int i = 0; i < reps; ++i) launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        ms /= reps;
        const double gbs = 2.0 * namp * 8 / (ms * 1e-3) / 1e9;
        std::printf("%-5s %2dq c64: %8.3f ms  %7.1f GB/s (read+write)  %7.1f TFLOP/s useful\n", name, lg, ms, gbs,
                    flop_per_amp * namp / (ms * 1e-3) / 1e12);
        return ms;
    };
    timeit("copy", [&] { copy_kernel<<<sms * 8, 256>>>((const float4 *)din, (float4 *)dout, n4); }, 0.0);
    timeit("fma", [&] { fma_kernel<<<sms * 8, 128>>>((const float4 *)din, (float4 *)dout, dB, nsets); }, 256.0);
    std::vector<float> got_fma(64 * 64 * 4);
    CK(cudaMemcpy(got_fma.data(), dout, got_fma.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemset(dout, 0, namp * 8));
    timeit("tc", [&] { tc_kernel<1><<<sms * 2, 128, smem>>>((const float4 *)din, (float4 *)dout, dB, nsets); }, 256.0);
    CK(cudaGetLastError());
    CK(cudaMemset(dout, 0, namp * 8));
    timeit("tc3", [&] { tc_kernel<3><<<sms, 384, smem3>>>((const float4 *)din, (float4 *)dout, dB, nsets); }, 256.0);
    CK(cudaGetLastError());
    // accuracy on the first 1024 sets against an FP64 host evaluation
    const int chk = 1024;
    std::vector<float> hin(chk * 64), hout(chk * 64);
    CK(cudaMemcpy(hin.data(), din, hin.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hout.data(), dout, hout.size() * 4, cudaMemcpyDeviceToHost));
    double err_tc = 0, err_fma = 0, mag = 0;
    for (int s = 0; s < chk; ++s)
        for (int n = 0; n < kN; ++n) {
            double y = 0;
            for (int k = 0; k < kK; ++k) y += static_cast<double>(B[n * kK + k]) * hin[s * 64 + k];
            err_tc = std::fmax(err_tc, std::fabs(y - hout[s * 64 + n]));
            if (s < 64) err_fma = std::fmax(err_fma, std::fabs(y - got_fma[s * 64 + n]));
            mag = std::fmax(mag, std::fabs(y));
        }
    std::printf("max |err| vs FP64: tc (3xTF32) %.3e, fma %.3e (max |y| %.3f)\n", err_tc, err_fma, mag);
    // several dense blocks per tile (one HBM sweep): does the TC side stay
    // under the memory time as a pass fuses more 5-qubit stages?
    const int smemc = 2 * kAbytes + 2 * kBbytes + 1024;
    CK(cudaFuncSetAttribute(tc_chain_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemc));
    CK(cudaFuncSetAttribute(tc_chain_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemc));
    CK(cudaFuncSetAttribute(tc_chain_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemc));
    CK(cudaFuncSetAttribute(tc_chain_kernel<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemc));
    timeit("chn1", [&] { tc_chain_kernel<1><<<sms * 2, 128, smemc>>>((const float4 *)din, (float4 *)dout, dB, nsets); }, 256.0);
    timeit("chn2", [&] { tc_chain_kernel<2><<<sms * 2, 128, smemc>>>((const float4 *)din, (float4 *)dout, dB, nsets); }, 512.0);
    timeit("chn4", [&] { tc_chain_kernel<4><<<sms * 2, 128, smemc>>>((const float4 *)din, (float4 *)dout, dB, nsets); }, 1024.0);
    timeit("chn7", [&] { tc_chain_kernel<7><<<sms * 2, 128, smemc>>>((const float4 *)din, (float4 *)dout, dB, nsets); }, 1792.0);
    CK(cudaGetLastError());
    return 0;
}
