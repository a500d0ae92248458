// The fused gate pass: the hot loop of the engine (sm_100a).
//
// Replaces the reference's per-gate strided sweep (apply_matrix_strided,
// /root/reference/proj/include/quasar/qubit/state.hpp:111-143, one full pass
// over 2^n amplitudes per gate, plus a full state copy per gate in
// apply_gate, state.hpp:153) with one HBM read + write per PASS of many
// gates (see planner.cpp for how gates become passes):
//
//   * persistent CTAs (2 per SM) stage the pass program (groups, op stream,
//     phase records) into shared memory once, then loop over tiles;
//   * a tile = 2^K amplitudes whose index bits are the pass's tile qubits,
//     copied HBM -> XOR-swizzled shared memory with 16-byte cp.async
//     (contiguous runs of 2^L amplitudes, L >= 3 for complex128);
//   * each group sweeps the tile once: a thread loads the 2^R amplitudes of a
//     register set, runs the group's op records (dense 2x2 / 4x4 / real /
//     Pauli-X / deferred phase flushes) from shared memory, and stores them
//     back; ops without conditions take a branch-free path;
//   * the tile goes back to HBM with streaming 16-byte stores.
#include <cuda_runtime.h>

#include "device_util.cuh"
#include "qsv_internal.hpp"

namespace qsv {

namespace {
using dev::cfma;
using dev::cmul;
using dev::cp_async16;
using dev::cp_async_wait_all;
using dev::st_cs16;
using dev::swz;
using dev::Vec2;

// ---- register-group gate application ---------------------------------------
// COND: the op has register conditions or zero_off_control (general path);
// otherwise every pair is transformed (fixed-bit conditions are resolved
// per set before the call).
template <typename T, int R, int J, bool COND>
__device__ __forceinline__ void dense1(typename Vec2<T>::type (&v)[1 << R], const T *m, bool fok, int rmask,
                                       int rval, bool zoc) {
    using V = typename Vec2<T>::type;
    const V m00 = {m[0], m[1]}, m01 = {m[2], m[3]}, m10 = {m[4], m[5]}, m11 = {m[6], m[7]};
#pragma unroll
    for (int r = 0; r < (1 << R); ++r) {
        if (r & (1 << J)) continue;
        const int r1 = r | (1 << J);
        const bool on = !COND || (fok && ((r & rmask) == rval));
        if (on) {
            const V x0 = v[r], x1 = v[r1];
            v[r] = cfma(m01, x1, cmul(m00, x0));
            v[r1] = cfma(m11, x1, cmul(m10, x0));
        } else if (zoc) {
            v[r] = V{0, 0};
            v[r1] = V{0, 0};
        }
    }
}

template <typename T, int R, int J, bool COND>
__device__ __forceinline__ void dense1r(typename Vec2<T>::type (&v)[1 << R], const T *m, bool fok, int rmask,
                                        int rval, bool zoc) {
    using V = typename Vec2<T>::type;
    const T a = m[0], b = m[1], c = m[2], d = m[3];
#pragma unroll
    for (int r = 0; r < (1 << R); ++r) {
        if (r & (1 << J)) continue;
        const int r1 = r | (1 << J);
        const bool on = !COND || (fok && ((r & rmask) == rval));
        if (on) {
            const V x0 = v[r], x1 = v[r1];
            v[r] = V{a * x0.x + b * x1.x, a * x0.y + b * x1.y};
            v[r1] = V{c * x0.x + d * x1.x, c * x0.y + d * x1.y};
        } else if (zoc) {
            v[r] = V{0, 0};
            v[r1] = V{0, 0};
        }
    }
}

template <typename T, int R, int J, bool COND>
__device__ __forceinline__ void x1(typename Vec2<T>::type (&v)[1 << R], bool fok, int rmask, int rval) {
    using V = typename Vec2<T>::type;
#pragma unroll
    for (int r = 0; r < (1 << R); ++r) {
        if (r & (1 << J)) continue;
        const int r1 = r | (1 << J);
        if (!COND) {
            const V t = v[r];
            v[r] = v[r1];
            v[r1] = t;
        } else if (fok && ((r & rmask) == rval)) {
            const V t = v[r];
            v[r] = v[r1];
            v[r1] = t;
        }
    }
}

template <typename T, int R, int A, int B, bool COND>
__device__ __forceinline__ void dense2(typename Vec2<T>::type (&v)[1 << R], const T *m, bool fok, int rmask,
                                       int rval, bool zoc) {
    using V = typename Vec2<T>::type;
    const V *mv = reinterpret_cast<const V *>(m);
#pragma unroll
    for (int r = 0; r < (1 << R); ++r) {
        if (r & ((1 << A) | (1 << B))) continue;
        const int idx[4] = {r, r | (1 << B), r | (1 << A), r | (1 << A) | (1 << B)};
        const bool on = !COND || (fok && ((r & rmask) == rval));
        if (on) {
            V x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] = v[idx[q]];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                V acc = cmul(mv[q * 4], x[0]);
                acc = cfma(mv[q * 4 + 1], x[1], acc);
                acc = cfma(mv[q * 4 + 2], x[2], acc);
                acc = cfma(mv[q * 4 + 3], x[3], acc);
                v[idx[q]] = acc;
            }
        } else if (zoc) {
#pragma unroll
            for (int q = 0; q < 4; ++q) v[idx[q]] = V{0, 0};
        }
    }
}

// Diagonal applied where it stands (rare: see planner.cpp).
template <typename T, int R>
__device__ __forceinline__ void diag_op(typename Vec2<T>::type (&v)[1 << R], const OpHdr &h, const T *m,
                                        uint64_t pb, bool fok) {
    using V = typename Vec2<T>::type;
    const V d0 = {m[0], m[1]}, d1 = {m[2], m[3]};
    V d2 = d0, d3 = d1;
    const int nt = h.nt;
    if (nt == 2) {
        d2 = V{m[4], m[5]};
        d3 = V{m[6], m[7]};
    }
    const int t0 = h.t0, t1 = h.t1;
    const bool t0r = h.treg & 1, t1r = (h.treg >> 1) & 1;
    const int f0 = t0r ? 0 : int((pb >> t0) & 1ull);
    const int f1 = (nt == 2 && !t1r) ? int((pb >> t1) & 1ull) : 0;
    const bool zoc = h.flags & OPF_ZERO_OFF_CONTROL;
#pragma unroll
    for (int r = 0; r < (1 << R); ++r) {
        const int b0 = t0r ? ((r >> t0) & 1) : f0;
        int sel = b0;
        if (nt == 2) sel = (b0 << 1) | (t1r ? ((r >> t1) & 1) : f1);
        const V d = sel == 0 ? d0 : sel == 1 ? d1 : sel == 2 ? d2 : d3;
        if (fok && ((r & h.rmask) == h.rval)) v[r] = cmul(v[r], d);
        else if (zoc) v[r] = V{0, 0};
    }
}

template <typename T, int R, int J>
__device__ __forceinline__ void scale_slot(typename Vec2<T>::type (&v)[1 << R], typename Vec2<T>::type f) {
#pragma unroll
    for (int r = 0; r < (1 << R); ++r)
        if (r & (1 << J)) v[r] = cmul(v[r], f);
}

// value of a phase record on the bits of `pb` (1 when its condition fails)
template <typename V> __device__ __forceinline__ V eval_rec(const DiagRec &rc, uint64_t pb) {
    using T = decltype(V{}.x);
    if ((pb & rc.fmask) != rc.fval) return V{1, 0};
    int idx = 0;
    if (rc.nt >= 1) idx = static_cast<int>((pb >> rc.tpos0) & 1ull);
    if (rc.nt == 2) idx = (idx << 1) | static_cast<int>((pb >> rc.tpos1) & 1ull);
    return V{static_cast<T>(rc.val[2 * idx]), static_cast<T>(rc.val[2 * idx + 1])};
}

template <typename T> struct OpCtx {
    using V = typename Vec2<T>::type;
    const FlushTarget *targets; // shared
    const DiagRec *recs;        // shared
    const V *tables;            // global
    const V *E;                 // shared, per tile
    const T *enc_table;         // global
    int batch, row, s;
    uint64_t pb;
};

template <typename T, int R>
__device__ __forceinline__ void flush_op(typename Vec2<T>::type (&v)[1 << R], const unsigned char *q,
                                         const OpCtx<T> &c) {
    using V = typename Vec2<T>::type;
    const FlushPay fp = *reinterpret_cast<const FlushPay *>(q);
    for (int ti = fp.tgt_begin; ti < fp.tgt_end; ++ti) {
        const FlushTarget ft = c.targets[ti];
        V f = ft.eidx >= 0 ? c.E[ft.eidx] : V{1, 0};
        if (ft.table >= 0) f = cmul(f, __ldg(c.tables + ft.table + c.s));
        if (ft.table_lo >= 0) f = cmul(f, __ldg(c.tables + ft.table_lo + (c.s & ((1 << ft.lo_bits) - 1))));
        if (ft.table_hi >= 0) f = cmul(f, __ldg(c.tables + ft.table_hi + (c.s >> ft.lo_bits)));
        for (int k = ft.mix_begin; k < ft.mix_end; ++k) f = cmul(f, eval_rec<V>(c.recs[k], c.pb));
        switch (ft.slot) {
        case -1:
#pragma unroll
            for (int r = 0; r < (1 << R); ++r) v[r] = cmul(v[r], f);
            break;
        case 0: scale_slot<T, R, 0>(v, f); break;
        case 1: if constexpr (R > 1) scale_slot<T, R, 1>(v, f); break;
        case 2: if constexpr (R > 2) scale_slot<T, R, 2>(v, f); break;
        case 3: if constexpr (R > 3) scale_slot<T, R, 3>(v, f); break;
        }
    }
    if (fp.regmask) {
        const V *D = reinterpret_cast<const V *>(q + sizeof(FlushPay));
#pragma unroll
        for (int r = 0; r < (1 << R); ++r)
            if ((fp.regmask >> r) & 1u) v[r] = cmul(v[r], D[r]);
    }
}

#define QSV_SLOT1(FN, ...)                                                                                             \
    switch (h.a) {                                                                                                     \
    case 0: FN<T, R, 0, COND>(__VA_ARGS__); break;                                                                    \
    case 1: if constexpr (R > 1) FN<T, R, 1, COND>(__VA_ARGS__); break;                                               \
    case 2: if constexpr (R > 2) FN<T, R, 2, COND>(__VA_ARGS__); break;                                               \
    case 3: if constexpr (R > 3) FN<T, R, 3, COND>(__VA_ARGS__); break;                                               \
    }

template <typename T, int R, bool COND>
__device__ __forceinline__ void apply_dense(typename Vec2<T>::type (&v)[1 << R], const OpHdr &h, const T *m,
                                            bool fok) {
    const bool zoc = h.flags & OPF_ZERO_OFF_CONTROL;
    switch (h.code) {
    case OP_DENSE1: QSV_SLOT1(dense1, v, m, fok, h.rmask, h.rval, zoc) break;
    case OP_DENSE1R: QSV_SLOT1(dense1r, v, m, fok, h.rmask, h.rval, zoc) break;
    case OP_X1: QSV_SLOT1(x1, v, fok, h.rmask, h.rval) break;
    case OP_DENSE2:
        if constexpr (R > 1) {
            switch (h.a * 8 + h.b) {
            case 1 * 8 + 0: dense2<T, R, 1, 0, COND>(v, m, fok, h.rmask, h.rval, zoc); break;
            case 2 * 8 + 0: if constexpr (R > 2) dense2<T, R, 2, 0, COND>(v, m, fok, h.rmask, h.rval, zoc); break;
            case 2 * 8 + 1: if constexpr (R > 2) dense2<T, R, 2, 1, COND>(v, m, fok, h.rmask, h.rval, zoc); break;
            case 3 * 8 + 0: if constexpr (R > 3) dense2<T, R, 3, 0, COND>(v, m, fok, h.rmask, h.rval, zoc); break;
            case 3 * 8 + 1: if constexpr (R > 3) dense2<T, R, 3, 1, COND>(v, m, fok, h.rmask, h.rval, zoc); break;
            case 3 * 8 + 2: if constexpr (R > 3) dense2<T, R, 3, 2, COND>(v, m, fok, h.rmask, h.rval, zoc); break;
            }
        }
        break;
    }
}

template <typename T, int R>
__device__ __forceinline__ void run_ops(typename Vec2<T>::type (&v)[1 << R], const unsigned char *p,
                                        const unsigned char *end, const OpCtx<T> &c) {
    while (p < end) {
        const OpHdr h = *reinterpret_cast<const OpHdr *>(p);
        const unsigned char *q = p + sizeof(OpHdr);
        p += h.size;
        bool fok = true;
        if (h.flags & OPF_FCOND) {
            const ulonglong2 fm = *reinterpret_cast<const ulonglong2 *>(q);
            fok = (c.pb & fm.x) == fm.y;
            q += 16;
        }
        if (h.code == OP_FLUSH) {
            flush_op<T, R>(v, q, c);
            continue;
        }
        const T *m = (h.flags & OPF_ENC) ? c.enc_table + (static_cast<size_t>(h.enc) * c.batch + c.row) * 32
                                         : reinterpret_cast<const T *>(q);
        if (h.code == OP_DIAG) {
            diag_op<T, R>(v, h, m, c.pb, fok);
            continue;
        }
        if (h.flags & (OPF_RCOND | OPF_ZERO_OFF_CONTROL)) apply_dense<T, R, true>(v, h, m, fok);
        else if (fok) apply_dense<T, R, false>(v, h, m, fok);
    }
}

template <typename T, int R>
__global__ void __launch_bounds__(256, 2) tile_pass_kernel(const PassArgs a) {
    using V = typename Vec2<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ V E[kMaxExtTargets];
    __shared__ int s_uoff[1 << R]; // tile offsets of the 2^R register amplitudes of a set
    const int K = a.K, L = a.L, H = K - L;
    V *tile = reinterpret_cast<V *>(smem_raw);
    uint64_t *hi_off = reinterpret_cast<uint64_t *>(smem_raw + (sizeof(V) << K));
    unsigned char *prog = smem_raw + tile_prog_offset(K, L, sizeof(V));

    // stage the pass program and the high-bit offset table once per CTA
    {
        const int4 *src = reinterpret_cast<const int4 *>(a.blob);
        int4 *dst = reinterpret_cast<int4 *>(prog);
        for (int i = threadIdx.x; i < a.blob_bytes / 16; i += blockDim.x) dst[i] = src[i];
        for (int h = threadIdx.x; h < (1 << H); h += blockDim.x) {
            uint64_t o = 0;
            for (int i = 0; i < H; ++i) o |= static_cast<uint64_t>((h >> i) & 1) << a.tile_pos[L + i];
            hi_off[h] = o;
        }
    }
    __syncthreads();
    const GroupDesc *groups = reinterpret_cast<const GroupDesc *>(prog);
    OpCtx<T> c;
    c.targets = reinterpret_cast<const FlushTarget *>(prog + a.off_targets);
    c.recs = reinterpret_cast<const DiagRec *>(prog + a.off_recs);
    c.tables = reinterpret_cast<const V *>(a.tables);
    c.E = E;
    c.enc_table = reinterpret_cast<const T *>(a.enc_table);
    c.batch = a.batch;
    const unsigned char *ops = prog + a.off_ops;

    constexpr int APU = 16 / sizeof(V); // amplitudes per 16-byte chunk
    const int nchunks = (1 << K) / APU;
    const int lmask = (1 << L) - 1;
    const int nsets = 1 << (K - R);

    for (uint64_t t = blockIdx.x; t < a.total_tiles; t += gridDim.x) {
        const int row = static_cast<int>(t / a.tiles_per_row);
        const uint64_t tid_in_row = t - static_cast<uint64_t>(row) * a.tiles_per_row;
        V *st = reinterpret_cast<V *>(a.state) + static_cast<size_t>(row) * a.row_stride;
        uint64_t tb = 0;
        for (int i = 0; i < a.next; ++i) tb |= ((tid_in_row >> i) & 1ull) << a.ext_pos[i];
        for (int ch = threadIdx.x; ch < nchunks; ch += blockDim.x) {
            const int u = ch * APU;
            cp_async16(&tile[swz<V>(u)], &st[tb + hi_off[u >> L] + (u & lmask)]);
        }
        cp_async_wait_all();
        __syncthreads();

        const uint64_t pbase = a.rank_base | tb;
        c.row = row;
        for (int gi = 0; gi < a.ngroups; ++gi) {
            const GroupDesc &gd = groups[gi];
            if (threadIdx.x < (1 << R)) {
                int u = 0;
#pragma unroll
                for (int j = 0; j < R; ++j)
                    if ((threadIdx.x >> j) & 1) u |= 1 << gd.slot_bit[j];
                s_uoff[threadIdx.x] = u;
            }
            if (gd.tgt_end > gd.tgt_begin) {
                for (int ti = gd.tgt_begin + threadIdx.x; ti < gd.tgt_end; ti += blockDim.x) {
                    const FlushTarget &ft = c.targets[ti];
                    if (ft.eidx < 0) continue;
                    V f{1, 0};
                    for (int k = ft.ext_rest; k < ft.ext_end; ++k) f = cmul(f, eval_rec<V>(c.recs[k], pbase));
                    for (int ch = 0; ch < ft.ext_chunks; ++ch)
                        f = cmul(f, __ldg(c.tables + ft.ext_tab + ch * 256 + ((tid_in_row >> (8 * ch)) & 255)));
                    E[ft.eidx] = f;
                }
            }
            __syncthreads();
            const unsigned char *ob = ops + gd.op_begin, *oe = ops + gd.op_end;
            for (int s = threadIdx.x; s < nsets; s += blockDim.x) {
                int ub = 0;
                uint64_t pb = pbase;
                for (int i = 0; i < K - R; ++i) {
                    const int bit = (s >> i) & 1;
                    const int tbit = gd.ng_bit[i];
                    ub |= bit << tbit;
                    pb |= static_cast<uint64_t>(bit) << a.tile_pos[tbit];
                }
                V v[1 << R];
#pragma unroll
                for (int r = 0; r < (1 << R); ++r) v[r] = tile[swz<V>(ub | s_uoff[r])];
                c.s = s;
                c.pb = pb;
                run_ops<T, R>(v, ob, oe, c);
#pragma unroll
                for (int r = 0; r < (1 << R); ++r) tile[swz<V>(ub | s_uoff[r])] = v[r];
            }
            __syncthreads();
        }

        for (int ch = threadIdx.x; ch < nchunks; ch += blockDim.x) {
            const int u = ch * APU;
            const float4 val = *reinterpret_cast<const float4 *>(&tile[swz<V>(u)]);
            st_cs16(&st[tb + hi_off[u >> L] + (u & lmask)], val);
        }
        __syncthreads(); // the next tile's cp.async overwrites the buffer
    }
}

template <typename T, int R> const void *kernel_ptr() { return reinterpret_cast<const void *>(tile_pass_kernel<T, R>); }

const void *select_kernel(int dtype, int R) {
    if (dtype == QSV_C64) {
        switch (R) {
        case 1: return kernel_ptr<float, 1>();
        case 2: return kernel_ptr<float, 2>();
        case 3: return kernel_ptr<float, 3>();
        default: return kernel_ptr<float, 4>();
        }
    }
    switch (R) {
    case 1: return kernel_ptr<double, 1>();
    case 2: return kernel_ptr<double, 2>();
    case 3: return kernel_ptr<double, 3>();
    default: return kernel_ptr<double, 4>();
    }
}

} // namespace

int tile_kernel_blocks_per_sm(int dtype, int R, int threads, size_t smem) {
    const void *k = select_kernel(dtype, R);
    int dev = 0, optin = 0;
    QSV_CUDA(cudaGetDevice(&dev));
    QSV_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    // the limit is per kernel: always the device maximum, never a pass's own size
    cudaFuncAttributes fa{};
    QSV_CUDA(cudaFuncGetAttributes(&fa, k));
    QSV_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  optin - static_cast<int>(fa.sharedSizeBytes)));
    int blocks = 0;
    QSV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k, threads, smem));
    return blocks;
}

void launch_pass(const DevPass &dp, int dtype, void *state, int rows, cudaStream_t s, double *zout) {
    if (dp.jit) {
        launch_jit(dp, state, state, rows, s, zout);
        return;
    }
    require(zout == nullptr, "fused <Z> needs a specialised pass kernel");
    PassArgs a = dp.args;
    a.state = state;
    a.total_tiles = a.tiles_per_row * static_cast<uint64_t>(rows);
    const void *k = select_kernel(dtype, dp.R);
    const uint64_t grid = std::min<uint64_t>(a.total_tiles, static_cast<uint64_t>(std::max(dp.grid, 1)));
    void *args[] = {&a};
    QSV_CUDA(cudaLaunchKernel(k, dim3(static_cast<unsigned>(grid)), dim3(dp.threads), args, dp.smem, s));
}

} // namespace qsv
