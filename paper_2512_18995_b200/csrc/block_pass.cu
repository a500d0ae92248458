// Dense-block passes on the tcgen05 tensor cores (complex64, opt-in
// qsv_opts.dense_blocks; host half in dense_blocks.cpp).
//
// One persistent CTA of 256 threads per SM. A pass streams 12-bit tiles
// (4096 amplitudes = 32 KiB) through shared memory, double-buffered with
// 8-byte cp.async. Per tile, each of the pass's blocks (a 32 x 32 complex
// unitary on 5 of the tile's bits) is one tensor-core product: thread t owns
// set t (the tile's 7 other bits) and gathers its 32 amplitudes from the
// XOR-swizzled tile into row t of A -- the 64 (re, im) reals split into TF32
// hi / lo, K-major, 128-byte swizzled (the UMMA canonical layout) -- thread 0
// issues tcgen05.mma.kind::tf32 for A_hi B_hi + A_hi B_lo + A_lo B_hi (M =
// 128 sets, N = 64 output reals, K = 64) into 64 TMEM columns, and each
// thread drains its row with tcgen05.ld and scatters the 32 new amplitudes
// back into the tile. B (the real 64 x 64 form of U, hi / lo, prepared on the
// host) stays in shared memory for the whole pass. Measured against the
// fused FFMA passes in DESIGN.md section 4.1b.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "qsv_internal.hpp"

namespace qsv {

struct DenseDev {
    float *bimg = nullptr;            // all blocks' B images (hi, lo: 2 x 16 KiB each)
    std::vector<size_t> bofs;         // per pass: offset (floats) of its first block's image
};

namespace {

constexpr int kRows = 128, kK = 64, kN = 64;
constexpr int kAbytes = kRows * kK * 4;  // 32 KiB
constexpr int kBbytes = kN * kK * 4;     // 16 KiB
constexpr int kTileAmps = 1 << kDenseTile;

struct DenseArgs {
    float2 *state;
    uint64_t ntiles;      // tiles of all rows
    int tpr_log;          // log2 tiles per row
    uint64_t row_stride;  // amplitudes per row
    const float4 *bimg;   // this pass's blocks, 2048 float4 (32 KiB) each
    int nb;
    int next;
    int tile_pos[kDenseTile];
    int ext_pos[kMaxQubits];
    int bbit[kDenseMaxBlocks][kDenseQ];
    int swm[4];
};

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int ROWS> __device__ __forceinline__ uint32_t kmaj_off(int row, int chunk) {
    return (chunk >> 3) * (ROWS / 8) * 1024 + (row >> 3) * 1024 + (row & 7) * 128 + (((chunk & 7) ^ (row & 7)) << 4);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((addr >> 4) & 0x3fff);
    d |= 1ull << 16;                                          // LBO (unused with swizzle)
    d |= static_cast<uint64_t>((1024 >> 4) & 0x3fff) << 32;  // SBO: 8-row atoms 1 KiB apart
    d |= 1ull << 46;                                          // sm_100 descriptor version
    d |= 2ull << 61;                                          // SWIZZLE_128B
    return d;
}
template <int ROWS> __device__ __forceinline__ uint32_t kstep(int ks) { return (ks >> 2) * (ROWS / 8) * 1024 + (ks & 3) * 32; }
__device__ __forceinline__ float tf32_hi(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
__device__ __forceinline__ int swz(int u, const int *m) {
    return u ^ ((__popc(u & m[0]) & 1) | ((__popc(u & m[1]) & 1) << 1) | ((__popc(u & m[2]) & 1) << 2) |
                ((__popc(u & m[3]) & 1) << 3));
}
__device__ __forceinline__ uint64_t scatter_bits(uint64_t x, const int *pos, int n) {
    uint64_t r = 0;
    for (int i = 0; i < n; ++i) r |= ((x >> i) & 1ull) << pos[i];
    return r;
}

#define LD32(R, ADDR)                                                                                                 \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
                 "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                          \
                 : "=r"(R[0]), "=r"(R[1]), "=r"(R[2]), "=r"(R[3]), "=r"(R[4]), "=r"(R[5]), "=r"(R[6]), "=r"(R[7]),       \
                   "=r"(R[8]), "=r"(R[9]), "=r"(R[10]), "=r"(R[11]), "=r"(R[12]), "=r"(R[13]), "=r"(R[14]), "=r"(R[15]), \
                   "=r"(R[16]), "=r"(R[17]), "=r"(R[18]), "=r"(R[19]), "=r"(R[20]), "=r"(R[21]), "=r"(R[22]),           \
                   "=r"(R[23]), "=r"(R[24]), "=r"(R[25]), "=r"(R[26]), "=r"(R[27]), "=r"(R[28]), "=r"(R[29]),           \
                   "=r"(R[30]), "=r"(R[31])                                                                              \
                 : "r"(ADDR))

// 256 threads: thread (t, h) = set row t (its TMEM lane) and half h of the
// row's 64 reals (amplitudes 16h .. 16h + 15): both warpgroups gather,
// split, drain and scatter; thread 0 issues the MMAs.
__global__ void __launch_bounds__(256, 1) dense_pass_kernel(const DenseArgs a) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char *sm = sm_raw + ((1024 - (smem_u32(sm_raw) & 1023)) & 1023);
    unsigned char *Ahi = sm, *Alo = sm + kAbytes, *Bs = sm + 2 * kAbytes;
    float2 *const T0 = reinterpret_cast<float2 *>(Bs + a.nb * 2 * kBbytes);  // two tile buffers
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base;
    __shared__ int sj[kDenseMaxBlocks][32];  // swizzled offsets of the 32 block indices
    __shared__ uint64_t gk[16];              // tile offsets of u = 256 k (copies)
    __shared__ int sk[16];                   // and their swizzled slots
    const int tid = threadIdx.x, t = tid & 127, h = tid >> 7, warp = tid >> 5;
    {  // B images of the pass's blocks -> shared memory
        const int n4 = a.nb * 2 * kBbytes / 16;
        float4 *dst = reinterpret_cast<float4 *>(Bs);
        for (int i = tid; i < n4; i += 256) dst[i] = a.bimg[i];
    }
    if (tid < a.nb * 32) {
        const int b = tid >> 5, j = tid & 31;
        int u = 0;
        for (int i = 0; i < kDenseQ; ++i) u |= ((j >> i) & 1) << a.bbit[b][i];
        sj[b][j] = swz(u, a.swm);
    }
    if (tid < 16) {
        gk[tid] = scatter_bits(static_cast<uint64_t>(tid) << 8, a.tile_pos, kDenseTile);
        sk[tid] = swz(tid << 8, a.swm);
    }
    if (tid < 32) {  // 128 columns: the hi x hi products, and the three corrections apart
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(128));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base;
    // kind::tf32: D f32, A / B tf32 K-major, N = 64, M = 128
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((kN >> 3) << 17) | ((kRows >> 4) << 24);
    uint32_t phase = 0;
    // this thread's set offset per block (the tile's non-block bits in order)
    int stb[kDenseMaxBlocks];
    for (int b = 0; b < kDenseMaxBlocks; ++b) {
        int ut = 0;
        if (b < a.nb) {
            int k = 0;
            for (int i = 0; i < kDenseTile; ++i) {
                bool in = false;
                for (int q = 0; q < kDenseQ; ++q) in = in || a.bbit[b][q] == i;
                if (!in) ut |= ((t >> k++) & 1) << i;
            }
        }
        stb[b] = swz(ut, a.swm);
    }
    // the copies: element u = tid + 256 k; scatter and swizzle are linear
    const uint64_t gt = scatter_bits(static_cast<uint64_t>(tid), a.tile_pos, 8);
    const int swt = swz(tid, a.swm);
    auto tile_base = [&](uint64_t tile) {
        const uint64_t row = tile >> a.tpr_log, tl = tile & ((1ull << a.tpr_log) - 1);
        return row * a.row_stride + scatter_bits(tl, a.ext_pos, a.next);
    };
    auto issue = [&](uint64_t tile, float2 *buf) {
        const float2 *src = a.state + tile_base(tile) + gt;
#pragma unroll
        for (int k = 0; k < 16; ++k)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(&buf[swt ^ sk[k]])),
                         "l"(src + gk[k])
                         : "memory");
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    int buf = 0;
    if (blockIdx.x < a.ntiles) issue(blockIdx.x, T0);
    for (uint64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
        const uint64_t nxt = tile + gridDim.x;
        if (nxt < a.ntiles) {
            issue(nxt, T0 + (buf ^ 1) * kTileAmps);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        float2 *tl = T0 + buf * kTileAmps;
        for (int b = 0; b < a.nb; ++b) {
            const int st = stb[b];
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
                const int c = 8 * h + cc;  // 16-byte chunk of the row: amplitudes 2c, 2c + 1
                const float2 x0 = tl[st ^ sj[b][2 * c]], x1 = tl[st ^ sj[b][2 * c + 1]];
                const float4 v = make_float4(x0.x, x0.y, x1.x, x1.y);
                const float4 hi = make_float4(tf32_hi(v.x), tf32_hi(v.y), tf32_hi(v.z), tf32_hi(v.w));
                *reinterpret_cast<float4 *>(Ahi + kmaj_off<kRows>(t, c)) = hi;
                *reinterpret_cast<float4 *>(Alo + kmaj_off<kRows>(t, c)) =
                    make_float4(v.x - hi.x, v.y - hi.y, v.z - hi.z, v.w - hi.w);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;");
                const unsigned char *Bhi = Bs + b * 2 * kBbytes, *Blo = Bhi + kBbytes;
                // D0 = A_hi B_hi (exact products) in columns 0..63; the small
                // terms A_hi B_lo + A_lo B_hi + A_lo B_lo in columns 64..127, so
                // they do not round against the large accumulator
                const unsigned char *As[4] = {Ahi, Ahi, Alo, Alo};
                const unsigned char *Bp[4] = {Bhi, Blo, Bhi, Blo};
                for (int p = 0; p < 4; ++p) {
                    int acc = p >= 2 ? 1 : 0;
                    const uint32_t d = tmem + (p == 0 ? 0u : 64u);
                    for (int ks = 0; ks < kK / 8; ++ks) {
                        const uint64_t ad = sdesc(smem_u32(As[p]) + kstep<kRows>(ks));
                        const uint64_t bd = sdesc(smem_u32(Bp[p]) + kstep<kN>(ks));
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
                            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                        acc = 1;
                    }
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    smem_u32(&mbar)));
            }
            {  // bounded wait: a malformed descriptor must not hang the device
                uint32_t done = 0;
                for (long spin = 0; !done; ++spin) {
                    asm volatile(
                        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, "
                        "p;\n}\n"
                        : "=r"(done)
                        : "r"(smem_u32(&mbar)), "r"(phase));
                    if (spin > (1l << 28)) __trap();
                }
            }
            phase ^= 1;
            asm volatile("tcgen05.fence::after_thread_sync;");
            uint32_t r[32], q[32];
            const uint32_t taddr = tmem + ((static_cast<uint32_t>(warp & 3) * 32) << 16) + 32u * h;
            LD32(r, taddr);
            LD32(q, taddr + 64u);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 16; ++j)
                tl[st ^ sj[b][16 * h + j]] = make_float2(__uint_as_float(r[2 * j]) + __uint_as_float(q[2 * j]),
                                                         __uint_as_float(r[2 * j + 1]) + __uint_as_float(q[2 * j + 1]));
            // A is rewritten by the next block and the tile read by the next
            // block / the stores: every thread's drain and scatter done first
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncthreads();
        }
        {  // the tile back to HBM, coalesced (streaming stores)
            float2 *dst = a.state + tile_base(tile) + gt;
#pragma unroll
            for (int k = 0; k < 16; ++k) __stcs(dst + gk[k], tl[swt ^ sk[k]]);
        }
        __syncthreads();  // the buffer is refilled by the copy issued next iteration
        buf ^= 1;
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(128));
}

#define ST64(ADDR, R)                                                                                                 \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"    \
                 "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,"  \
                 "%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};" ::"r"(ADDR),     \
                 "r"(R[0]), "r"(R[1]), "r"(R[2]), "r"(R[3]), "r"(R[4]), "r"(R[5]), "r"(R[6]), "r"(R[7]), "r"(R[8]),          \
                 "r"(R[9]), "r"(R[10]), "r"(R[11]), "r"(R[12]), "r"(R[13]), "r"(R[14]), "r"(R[15]), "r"(R[16]), "r"(R[17]),   \
                 "r"(R[18]), "r"(R[19]), "r"(R[20]), "r"(R[21]), "r"(R[22]), "r"(R[23]), "r"(R[24]), "r"(R[25]), "r"(R[26]),  \
                 "r"(R[27]), "r"(R[28]), "r"(R[29]), "r"(R[30]), "r"(R[31]), "r"(R[32]), "r"(R[33]), "r"(R[34]), "r"(R[35]),  \
                 "r"(R[36]), "r"(R[37]), "r"(R[38]), "r"(R[39]), "r"(R[40]), "r"(R[41]), "r"(R[42]), "r"(R[43]), "r"(R[44]),  \
                 "r"(R[45]), "r"(R[46]), "r"(R[47]), "r"(R[48]), "r"(R[49]), "r"(R[50]), "r"(R[51]), "r"(R[52]), "r"(R[53]),  \
                 "r"(R[54]), "r"(R[55]), "r"(R[56]), "r"(R[57]), "r"(R[58]), "r"(R[59]), "r"(R[60]), "r"(R[61]), "r"(R[62]),  \
                 "r"(R[63]))
#define LD64(R, ADDR)                                                                                                 \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"   \
                 "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,"   \
                 "%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"                 \
                 : "=r"(R[0]), "=r"(R[1]), "=r"(R[2]), "=r"(R[3]), "=r"(R[4]), "=r"(R[5]), "=r"(R[6]), "=r"(R[7]),       \
                   "=r"(R[8]), "=r"(R[9]), "=r"(R[10]), "=r"(R[11]), "=r"(R[12]), "=r"(R[13]), "=r"(R[14]), "=r"(R[15]), \
                   "=r"(R[16]), "=r"(R[17]), "=r"(R[18]), "=r"(R[19]), "=r"(R[20]), "=r"(R[21]), "=r"(R[22]),           \
                   "=r"(R[23]), "=r"(R[24]), "=r"(R[25]), "=r"(R[26]), "=r"(R[27]), "=r"(R[28]), "=r"(R[29]),           \
                   "=r"(R[30]), "=r"(R[31]), "=r"(R[32]), "=r"(R[33]), "=r"(R[34]), "=r"(R[35]), "=r"(R[36]),           \
                   "=r"(R[37]), "=r"(R[38]), "=r"(R[39]), "=r"(R[40]), "=r"(R[41]), "=r"(R[42]), "=r"(R[43]),           \
                   "=r"(R[44]), "=r"(R[45]), "=r"(R[46]), "=r"(R[47]), "=r"(R[48]), "=r"(R[49]), "=r"(R[50]),           \
                   "=r"(R[51]), "=r"(R[52]), "=r"(R[53]), "=r"(R[54]), "=r"(R[55]), "=r"(R[56]), "=r"(R[57]),           \
                   "=r"(R[58]), "=r"(R[59]), "=r"(R[60]), "=r"(R[61]), "=r"(R[62]), "=r"(R[63])                         \
                 : "r"(ADDR))

// Two tiles in flight per SM: warpgroup g (0 / 1) owns tile slot g -- its
// own double-buffered shared tile, mbarrier and 256 TMEM columns (A_hi,
// A_lo, the hi x hi accumulator, the correction accumulator) -- so one
// slot's gather / scatter overlaps the other's tensor-core products. A goes
// to TMEM with tcgen05.st (thread t = TMEM lane t = set row t, one TF32 per
// column) and the MMAs read it from there (the kind::tf32 TS form), so the
// shared memory holds only the tiles and the B images.
__global__ void __launch_bounds__(256, 1) dense_pass_kernel_v3(const DenseArgs a) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char *sm = sm_raw + ((1024 - (smem_u32(sm_raw) & 1023)) & 1023);
    unsigned char *Bs = sm;
    float2 *const T0 = reinterpret_cast<float2 *>(Bs + a.nb * 2 * kBbytes);  // [slot][buffer] tiles
    __shared__ uint64_t mbar[2];
    __shared__ uint32_t tmem_base;
    __shared__ int sj[kDenseMaxBlocks][32];
    __shared__ uint64_t gk[32];  // tile offsets of u = 128 k (copies by 128 threads)
    __shared__ int sk[32];
    const int tid = threadIdx.x, g = tid >> 7, t = tid & 127, warp = tid >> 5;
    {
        const int n4 = a.nb * 2 * kBbytes / 16;
        float4 *dst = reinterpret_cast<float4 *>(Bs);
        for (int i = tid; i < n4; i += 256) dst[i] = a.bimg[i];
    }
    if (tid < a.nb * 32) {
        const int b = tid >> 5, j = tid & 31;
        int u = 0;
        for (int i = 0; i < kDenseQ; ++i) u |= ((j >> i) & 1) << a.bbit[b][i];
        sj[b][j] = swz(u, a.swm);
    }
    if (tid < 32) {
        gk[tid] = scatter_bits(static_cast<uint64_t>(tid) << 7, a.tile_pos, kDenseTile);
        sk[tid] = swz(tid << 7, a.swm);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar[1])));
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t col0 = tmem_base + 256u * g;                         // this slot's columns
    const uint32_t lane = (static_cast<uint32_t>(warp & 3) * 32) << 16;  // this warp's TMEM lanes
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((kN >> 3) << 17) | ((kRows >> 4) << 24);
    uint32_t phase = 0;
    int stb[kDenseMaxBlocks];
    for (int b = 0; b < kDenseMaxBlocks; ++b) {
        int ut = 0;
        if (b < a.nb) {
            int k = 0;
            for (int i = 0; i < kDenseTile; ++i) {
                bool in = false;
                for (int q = 0; q < kDenseQ; ++q) in = in || a.bbit[b][q] == i;
                if (!in) ut |= ((t >> k++) & 1) << i;
            }
        }
        stb[b] = swz(ut, a.swm);
    }
    const uint64_t gt = scatter_bits(static_cast<uint64_t>(t), a.tile_pos, 7);
    const int swt = swz(t, a.swm);
    auto tile_base = [&](uint64_t tile) {
        const uint64_t row = tile >> a.tpr_log, tl = tile & ((1ull << a.tpr_log) - 1);
        return row * a.row_stride + scatter_bits(tl, a.ext_pos, a.next);
    };
    auto issue = [&](uint64_t tile, float2 *buf) {
        const float2 *src = a.state + tile_base(tile) + gt;
#pragma unroll 8
        for (int k = 0; k < 32; ++k)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(&buf[swt ^ sk[k]])),
                         "l"(src + gk[k])
                         : "memory");
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    auto slot_sync = [&] { asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory"); };
    float2 *const Tg = T0 + static_cast<size_t>(g) * 2 * kTileAmps;
    const uint64_t step = 2ull * gridDim.x;
    uint64_t tile = 2ull * blockIdx.x + g;
    int buf = 0;
    if (tile < a.ntiles) issue(tile, Tg);
    for (; tile < a.ntiles; tile += step) {
        if (tile + step < a.ntiles) {
            issue(tile + step, Tg + (buf ^ 1) * kTileAmps);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        slot_sync();
        float2 *tl = Tg + buf * kTileAmps;
        for (int b = 0; b < a.nb; ++b) {
            const int st = stb[b];
            {
                uint32_t hi[64], lo[64];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const float2 x = tl[st ^ sj[b][j]];
                    const float hr = tf32_hi(x.x), hm = tf32_hi(x.y);
                    hi[2 * j] = __float_as_uint(hr);
                    hi[2 * j + 1] = __float_as_uint(hm);
                    lo[2 * j] = __float_as_uint(x.x - hr);
                    lo[2 * j + 1] = __float_as_uint(x.y - hm);
                }
                ST64(col0 + lane, hi);
                ST64(col0 + lane + 64u, lo);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            slot_sync();
            if (t == 0) {
                asm volatile("tcgen05.fence::after_thread_sync;");
                const unsigned char *Bhi = Bs + b * 2 * kBbytes, *Blo = Bhi + kBbytes;
                // D0 (cols +128) = A_hi B_hi; Dc (cols +192) = A_hi B_lo + A_lo B_hi + A_lo B_lo
                const uint32_t Acol[4] = {col0, col0, col0 + 64u, col0 + 64u};
                const unsigned char *Bp[4] = {Bhi, Blo, Bhi, Blo};
                for (int p = 0; p < 4; ++p) {
                    int acc = p >= 2 ? 1 : 0;
                    const uint32_t d = col0 + (p == 0 ? 128u : 192u);
                    for (int ks = 0; ks < kK / 8; ++ks) {
                        const uint64_t bd = sdesc(smem_u32(Bp[p]) + kstep<kN>(ks));
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                            "r"(Acol[p] + 8u * ks), "l"(bd), "r"(idesc), "r"(acc));
                        acc = 1;
                    }
                }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    smem_u32(&mbar[g])));
            }
            {
                uint32_t done = 0;
                for (long spin = 0; !done; ++spin) {
                    asm volatile(
                        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, "
                        "p;\n}\n"
                        : "=r"(done)
                        : "r"(smem_u32(&mbar[g])), "r"(phase));
                    if (spin > (1l << 28)) __trap();
                }
            }
            phase ^= 1;
            asm volatile("tcgen05.fence::after_thread_sync;");
            {
                uint32_t r[64], q[64];
                LD64(r, col0 + lane + 128u);
                LD64(q, col0 + lane + 192u);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    tl[st ^ sj[b][j]] = make_float2(__uint_as_float(r[2 * j]) + __uint_as_float(q[2 * j]),
                                                    __uint_as_float(r[2 * j + 1]) + __uint_as_float(q[2 * j + 1]));
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            slot_sync();
        }
        {
            float2 *dst = a.state + tile_base(tile) + gt;
#pragma unroll 8
            for (int k = 0; k < 32; ++k) __stcs(dst + gk[k], tl[swt ^ sk[k]]);
        }
        slot_sync();
        buf ^= 1;
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
}

size_t dense_smem(int nb) { return 2 * kAbytes + static_cast<size_t>(nb) * 2 * kBbytes + 2 * kTileAmps * 8 + 1024; }
size_t dense_smem_v3(int nb) { return static_cast<size_t>(nb) * 2 * kBbytes + 4 * kTileAmps * 8 + 1024; }
// QSV_DENSE_V2=1: the single-slot kernel with A in shared memory (A/B)
bool dense_v2() {
    static const bool v = [] {
        const char *e = std::getenv("QSV_DENSE_V2");
        return e && e[0] == '1';
    }();
    return v;
}

} // namespace

void dense_upload(Plan &p) {
    DenseDev *d = new DenseDev();
    p.ddev = d;
    std::vector<float> all, one;
    for (const DensePass &dp : p.dpasses) {
        d->bofs.push_back(all.size());
        for (int bi : dp.blocks) {
            dense_b_operand(p.dblocks[bi], one);
            all.insert(all.end(), one.begin(), one.end());
        }
    }
    QSV_CUDA(cudaMalloc(&d->bimg, std::max<size_t>(all.size(), 4) * sizeof(float)));
    if (!all.empty()) QSV_CUDA(cudaMemcpy(d->bimg, all.data(), all.size() * sizeof(float), cudaMemcpyHostToDevice));
    QSV_CUDA(cudaFuncSetAttribute(dense_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dense_smem(kDenseMaxBlocks))));
    QSV_CUDA(cudaFuncSetAttribute(dense_pass_kernel_v3, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(dense_smem_v3(kDenseMaxBlocks))));
}

void dense_free(Plan &p) {
    if (!p.ddev) return;
    cudaFree(p.ddev->bimg);
    delete p.ddev;
    p.ddev = nullptr;
}

void dense_execute(Plan &p, State &st, cudaStream_t s, double *launch_ms) {
    require(p.ddev != nullptr, "dense plan not uploaded");
    const int nl = p.nlocal;
    std::vector<cudaEvent_t> ev;
    if (launch_ms) {
        ev.resize(2 * p.dpasses.size());
        for (auto &e : ev) QSV_CUDA(cudaEventCreate(&e));
    }
    for (size_t pi = 0; pi < p.dpasses.size(); ++pi) {
        const DensePass &dp = p.dpasses[pi];
        DenseArgs a{};
        a.tpr_log = nl - kDenseTile;
        a.ntiles = (1ull << a.tpr_log) * static_cast<uint64_t>(st.batch);
        a.row_stride = st.local_amps;
        a.bimg = reinterpret_cast<const float4 *>(p.ddev->bimg + p.ddev->bofs[pi]);
        a.nb = static_cast<int>(dp.blocks.size());
        for (int i = 0; i < kDenseTile; ++i) a.tile_pos[i] = dp.tile_pos[i];
        a.next = static_cast<int>(dp.ext_pos.size());
        for (int i = 0; i < a.next; ++i) a.ext_pos[i] = dp.ext_pos[i];
        for (int b = 0; b < a.nb; ++b)
            for (int i = 0; i < kDenseQ; ++i) a.bbit[b][i] = dp.bbit[b][i];
        for (int i = 0; i < 4; ++i) a.swm[i] = dp.swm[i];
        a.state = static_cast<float2 *>(st.d);
        if (launch_ms) QSV_CUDA(cudaEventRecord(ev[2 * pi], s));
        if (dense_v2()) {
            const int grid = static_cast<int>(std::min<uint64_t>(a.ntiles, static_cast<uint64_t>(p.ctx->sm_count)));
            dense_pass_kernel<<<grid, 256, dense_smem(a.nb), s>>>(a);
        } else {  // two tiles in flight per CTA
            const int grid = static_cast<int>(std::min<uint64_t>((a.ntiles + 1) / 2, static_cast<uint64_t>(p.ctx->sm_count)));
            dense_pass_kernel_v3<<<grid, 256, dense_smem_v3(a.nb), s>>>(a);
        }
        QSV_CUDA(cudaGetLastError());
        if (launch_ms) QSV_CUDA(cudaEventRecord(ev[2 * pi + 1], s));
    }
    if (launch_ms) {
        QSV_CUDA(cudaStreamSynchronize(s));
        for (size_t pi = 0; pi < p.dpasses.size(); ++pi) {
            float ms = 0;
            QSV_CUDA(cudaEventElapsedTime(&ms, ev[2 * pi], ev[2 * pi + 1]));
            launch_ms[pi] = ms;
        }
        for (auto &e : ev) cudaEventDestroy(e);
    }
}

} // namespace qsv
