// sm_100a kernels of the qsv engine.
//
//   tile_pass_kernel   the fused gate pass (the hot loop). Replaces the
//                      reference's per-gate strided sweep
//                      (apply_matrix_strided, /root/reference/proj/include/
//                      quasar/qubit/state.hpp:111-143) with one HBM read+write
//                      per PASS of many gates: cp.async 16-byte staging of a
//                      2^K-amplitude tile into XOR-swizzled shared memory,
//                      register-resident groups of R qubits, coalesced
//                      streaming stores.
//   bind_kernel        device-side gate_matrix for encoded (per-row) gates
//                      (gate.hpp:89-154, circuit.hpp:139-147).
//   zsum/pauli/norm    FP64 warp->block->grid reductions for expectation_one
//                      (circuit.hpp:248-282) and the norm.
//   marginal_kernel    marginal_probabilities histogram (circuit.hpp:182-205).
#include <cuda_runtime.h>

#include <cstdio>

#include "qsv_internal.hpp"

namespace qsv {

void cuda_check(cudaError_t e, const char *what) {
    if (e != cudaSuccess) fail(QSV_ERR_INTERNAL, std::string("CUDA error ") + cudaGetErrorString(e) + " at " + what);
}

namespace {

template <typename T> struct Vec2;
template <> struct Vec2<float> { using type = float2; };
template <> struct Vec2<double> { using type = double2; };

template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
    V r;
    r.x = a.x * b.x - a.y * b.y;
    r.y = a.x * b.y + a.y * b.x;
    return r;
}
template <typename V> __device__ __forceinline__ V cfma(V a, V b, V acc) { // acc + a*b
    acc.x += a.x * b.x - a.y * b.y;
    acc.y += a.x * b.y + a.y * b.x;
    return acc;
}

// XOR-swizzle of a tile-local amplitude index into its shared-memory slot so
// that lanes walking any tile bit spread over the 8 sixteen-byte columns of a
// 128-byte bank row. Bijective inside the tile (only the low bits change).
template <typename V> __device__ __forceinline__ int swz(int u);
template <> __device__ __forceinline__ int swz<double2>(int u) {
    const int f = (u >> 3) ^ (u >> 6) ^ (u >> 9) ^ (u >> 12);
    return u ^ (f & 7);
}
template <> __device__ __forceinline__ int swz<float2>(int u) {
    const int w = u >> 1; // 16-byte unit = 2 amplitudes, kept adjacent
    const int f = (w >> 3) ^ (w >> 6) ^ (w >> 9) ^ (w >> 12);
    return ((w ^ (f & 7)) << 1) | (u & 1);
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void st_cs16(void *gmem, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"l"(gmem), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}

// ---- register-group gate application ---------------------------------------
template <typename T, int R, int J>
__device__ __forceinline__ void dense1(typename Vec2<T>::type (&v)[1 << R], const T *__restrict__ m, bool fok,
                                       int rmask, int rval, bool zoc) {
    using V = typename Vec2<T>::type;
    const V m00 = {m[0], m[1]}, m01 = {m[2], m[3]}, m10 = {m[4], m[5]}, m11 = {m[6], m[7]};
#pragma unroll
    for (int r = 0; r < (1 << R); ++r) {
        if (r & (1 << J)) continue;
        const int r1 = r | (1 << J);
        const bool on = fok && ((r & rmask) == rval);
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

template <typename T, int R, int A, int B>
__device__ __forceinline__ void dense2(typename Vec2<T>::type (&v)[1 << R], const T *__restrict__ m, bool fok,
                                       int rmask, int rval, bool zoc) {
    using V = typename Vec2<T>::type;
    // matrix entries are re-read (L1-resident, warp-uniform) instead of held
    // in 32 registers: the 2^R amplitudes already occupy the register budget.
    const V *mv = reinterpret_cast<const V *>(m);
#pragma unroll
    for (int r = 0; r < (1 << R); ++r) {
        if (r & ((1 << A) | (1 << B))) continue;
        const int idx[4] = {r, r | (1 << B), r | (1 << A), r | (1 << A) | (1 << B)};
        const bool on = fok && ((r & rmask) == rval);
        if (on) {
            V x[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) x[q] = v[idx[q]];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                V acc = cmul(__ldg(mv + q * 4), x[0]);
                acc = cfma(__ldg(mv + q * 4 + 1), x[1], acc);
                acc = cfma(__ldg(mv + q * 4 + 2), x[2], acc);
                acc = cfma(__ldg(mv + q * 4 + 3), x[3], acc);
                v[idx[q]] = acc;
            }
        } else if (zoc) {
#pragma unroll
            for (int q = 0; q < 4; ++q) v[idx[q]] = V{0, 0};
        }
    }
}

template <typename T, int R>
__device__ __forceinline__ void diag_op(typename Vec2<T>::type (&v)[1 << R], const TileOp<T> &o,
                                        const T *__restrict__ m, uint64_t pb, bool fok, bool zoc) {
    using V = typename Vec2<T>::type;
    const V d0 = {m[0], m[1]}, d1 = {m[2], m[3]};
    V d2 = d0, d3 = d1;
    const int nt = o.nt;
    if (nt == 2) {
        d2 = V{m[4], m[5]};
        d3 = V{m[6], m[7]};
    }
    const int t0 = o.t0, t1 = o.t1;
    const bool t0r = o.t0reg, t1r = o.t1reg;
    const int f0 = t0r ? 0 : int((pb >> t0) & 1ull);
    const int f1 = (nt == 2 && !t1r) ? int((pb >> t1) & 1ull) : 0;
    const int rmask = o.rmask, rval = o.rval;
#pragma unroll
    for (int r = 0; r < (1 << R); ++r) {
        const int b0 = t0r ? ((r >> t0) & 1) : f0;
        int sel = b0;
        if (nt == 2) sel = (b0 << 1) | (t1r ? ((r >> t1) & 1) : f1);
        const V d = sel == 0 ? d0 : sel == 1 ? d1 : sel == 2 ? d2 : d3;
        if (fok && ((r & rmask) == rval)) v[r] = cmul(v[r], d);
        else if (zoc) v[r] = V{0, 0};
    }
}

template <typename T, int R, int J>
__device__ __forceinline__ void dense1r(typename Vec2<T>::type (&v)[1 << R], const T *__restrict__ m, bool fok,
                                        int rmask, int rval) {
    using V = typename Vec2<T>::type;
    const T a = m[0], b = m[2], c = m[4], d = m[6];
#pragma unroll
    for (int r = 0; r < (1 << R); ++r) {
        if (r & (1 << J)) continue;
        const int r1 = r | (1 << J);
        if (fok && ((r & rmask) == rval)) {
            const V x0 = v[r], x1 = v[r1];
            v[r] = V{a * x0.x + b * x1.x, a * x0.y + b * x1.y};
            v[r1] = V{c * x0.x + d * x1.x, c * x0.y + d * x1.y};
        }
    }
}

template <typename T, int R, int J>
__device__ __forceinline__ void x1(typename Vec2<T>::type (&v)[1 << R], bool fok, int rmask, int rval) {
    using V = typename Vec2<T>::type;
#pragma unroll
    for (int r = 0; r < (1 << R); ++r) {
        if (r & (1 << J)) continue;
        const int r1 = r | (1 << J);
        const bool on = fok && ((r & rmask) == rval);
        const V x0 = v[r], x1v = v[r1];
        v[r] = on ? x1v : x0;
        v[r1] = on ? x0 : x1v;
    }
}

template <typename T, int R, int J>
__device__ __forceinline__ void scale_slot(typename Vec2<T>::type (&v)[1 << R], typename Vec2<T>::type f) {
#pragma unroll
    for (int r = 0; r < (1 << R); ++r)
        if (r & (1 << J)) v[r] = cmul(v[r], f);
}

// value of a phase record on the bits of `pb` (1 when its condition fails)
template <typename V>
__device__ __forceinline__ V eval_rec(const DiagRec &rc, uint64_t pb) {
    using T = decltype(V{}.x);
    if ((pb & rc.fmask) != rc.fval) return V{1, 0};
    int idx = 0;
    if (rc.nt >= 1) idx = static_cast<int>((pb >> rc.tpos0) & 1ull);
    if (rc.nt == 2) idx = (idx << 1) | static_cast<int>((pb >> rc.tpos1) & 1ull);
    return V{static_cast<T>(rc.val[2 * idx]), static_cast<T>(rc.val[2 * idx + 1])};
}

// Context a FLUSH needs besides the registers.
template <typename V> struct FlushCtx {
    const FlushTarget *targets;
    const DiagRec *recs;
    const V *tables;
    const V *E;  // shared memory, per-CTA external factors
    int s;       // set index
};

template <typename T, int R>
__device__ __forceinline__ void flush_op(typename Vec2<T>::type (&v)[1 << R], const TileOp<T> &o,
                                         const FlushCtx<typename Vec2<T>::type> &fc, uint64_t pb) {
    using V = typename Vec2<T>::type;
    for (int ti = o.a; ti < o.b; ++ti) {
        const FlushTarget ft = fc.targets[ti];
        V f = ft.eidx >= 0 ? fc.E[ft.eidx] : V{1, 0};
        if (ft.table >= 0) f = cmul(f, fc.tables[ft.table + fc.s]);
        for (int k = ft.mix_begin; k < ft.mix_end; ++k) f = cmul(f, eval_rec<V>(fc.recs[k], pb));
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
}

template <typename T, int R>
__device__ __forceinline__ void run_op(typename Vec2<T>::type (&v)[1 << R], const TileOp<T> &o,
                                       const T *__restrict__ enc_table, int batch, int row, uint64_t pb,
                                       const FlushCtx<typename Vec2<T>::type> &fc) {
    const bool fok = (pb & o.fmask) == o.fval;
    const T *m = o.enc >= 0 ? enc_table + (static_cast<size_t>(o.enc) * batch + row) * 32 : o.m;
    const bool zoc = (o.flags & OPF_ZERO_OFF_CONTROL) != 0;
    switch (o.type) {
    case OP_DENSE1:
        switch (o.a) {
        case 0: dense1<T, R, 0>(v, m, fok, o.rmask, o.rval, zoc); break;
        case 1: if constexpr (R > 1) dense1<T, R, 1>(v, m, fok, o.rmask, o.rval, zoc); break;
        case 2: if constexpr (R > 2) dense1<T, R, 2>(v, m, fok, o.rmask, o.rval, zoc); break;
        case 3: if constexpr (R > 3) dense1<T, R, 3>(v, m, fok, o.rmask, o.rval, zoc); break;
        }
        break;
    case OP_DENSE2:
        if constexpr (R > 1) {
            const int ab = o.a * 8 + o.b;
            switch (ab) {
            case 1 * 8 + 0: dense2<T, R, 1, 0>(v, m, fok, o.rmask, o.rval, zoc); break;
            case 2 * 8 + 0: if constexpr (R > 2) dense2<T, R, 2, 0>(v, m, fok, o.rmask, o.rval, zoc); break;
            case 2 * 8 + 1: if constexpr (R > 2) dense2<T, R, 2, 1>(v, m, fok, o.rmask, o.rval, zoc); break;
            case 3 * 8 + 0: if constexpr (R > 3) dense2<T, R, 3, 0>(v, m, fok, o.rmask, o.rval, zoc); break;
            case 3 * 8 + 1: if constexpr (R > 3) dense2<T, R, 3, 1>(v, m, fok, o.rmask, o.rval, zoc); break;
            case 3 * 8 + 2: if constexpr (R > 3) dense2<T, R, 3, 2>(v, m, fok, o.rmask, o.rval, zoc); break;
            }
        }
        break;
    case OP_DIAG: diag_op<T, R>(v, o, m, pb, fok, zoc); break;
    case OP_DENSE1R:
        switch (o.a) {
        case 0: dense1r<T, R, 0>(v, m, fok, o.rmask, o.rval); break;
        case 1: if constexpr (R > 1) dense1r<T, R, 1>(v, m, fok, o.rmask, o.rval); break;
        case 2: if constexpr (R > 2) dense1r<T, R, 2>(v, m, fok, o.rmask, o.rval); break;
        case 3: if constexpr (R > 3) dense1r<T, R, 3>(v, m, fok, o.rmask, o.rval); break;
        }
        break;
    case OP_X1:
        switch (o.a) {
        case 0: x1<T, R, 0>(v, fok, o.rmask, o.rval); break;
        case 1: if constexpr (R > 1) x1<T, R, 1>(v, fok, o.rmask, o.rval); break;
        case 2: if constexpr (R > 2) x1<T, R, 2>(v, fok, o.rmask, o.rval); break;
        case 3: if constexpr (R > 3) x1<T, R, 3>(v, fok, o.rmask, o.rval); break;
        }
        break;
    case OP_FLUSH: flush_op<T, R>(v, o, fc, pb); break;
    }
}

// One fused pass. grid = (tiles per row, rows); block handles one tile.
template <typename T, int R>
__global__ void __launch_bounds__(256, 2) tile_pass_kernel(const PassArgs a) {
    using V = typename Vec2<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V *tile = reinterpret_cast<V *>(smem_raw);
    uint64_t *hi_off = reinterpret_cast<uint64_t *>(smem_raw + (sizeof(V) << a.K));
    const int row = a.row0 + blockIdx.y;
    V *st = reinterpret_cast<V *>(a.state) + static_cast<size_t>(row) * a.row_stride;
    const TileOp<T> *ops = reinterpret_cast<const TileOp<T> *>(a.ops);
    const T *enc_table = reinterpret_cast<const T *>(a.enc_table);

    // tile base: blockIdx.x scattered over the non-tile local bits
    uint64_t tb = 0;
    {
        const uint64_t bid = blockIdx.x;
        for (int i = 0; i < a.next; ++i) tb |= ((bid >> i) & 1ull) << a.ext_pos[i];
    }
    const int K = a.K, L = a.L, H = K - L;
    for (int h = threadIdx.x; h < (1 << H); h += blockDim.x) {
        uint64_t o = 0;
        for (int i = 0; i < H; ++i) o |= static_cast<uint64_t>((h >> i) & 1) << a.tile_pos[L + i];
        hi_off[h] = o;
    }
    __syncthreads();

    constexpr int APU = 16 / sizeof(V); // amplitudes per 16-byte chunk
    const int nchunks = (1 << K) / APU;
    const int lmask = (1 << L) - 1;
    for (int c = threadIdx.x; c < nchunks; c += blockDim.x) {
        const int u = c * APU;
        const uint64_t g = tb + hi_off[u >> L] + (u & lmask);
        cp_async16(&tile[swz<V>(u)], &st[g]);
    }
    cp_async_wait_all();
    __syncthreads();

    const uint64_t pbase = a.rank_base | tb;
    const int nsets = 1 << (K - R);
    __shared__ V E[kMaxExtTargets];
    FlushCtx<V> fc{a.targets, a.recs, reinterpret_cast<const V *>(a.tables), E, 0};
    for (int gi = 0; gi < a.ngroups; ++gi) {
        const GroupDesc &gd = a.groups[gi];
        if (gd.tgt_end > gd.tgt_begin) {
            // per-CTA factors of records over bits outside the tile
            for (int t = gd.tgt_begin + threadIdx.x; t < gd.tgt_end; t += blockDim.x) {
                const FlushTarget ft = a.targets[t];
                if (ft.eidx < 0) continue;
                V f{1, 0};
                for (int k = ft.ext_begin; k < ft.ext_end; ++k) f = cmul(f, eval_rec<V>(a.recs[k], pbase));
                E[ft.eidx] = f;
            }
            __syncthreads();
        }
        int uoff[1 << R];
        uoff[0] = 0;
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int bit = 1 << gd.slot_bit[j];
#pragma unroll
            for (int r = 0; r < (1 << j); ++r) uoff[r | (1 << j)] = uoff[r] | bit;
        }
        const int ob = gd.op_begin, oe = gd.op_end;
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
            for (int r = 0; r < (1 << R); ++r) v[r] = tile[swz<V>(ub | uoff[r])];
            fc.s = s;
            for (int oi = ob; oi < oe; ++oi) run_op<T, R>(v, ops[oi], enc_table, a.batch, row, pb, fc);
#pragma unroll
            for (int r = 0; r < (1 << R); ++r) tile[swz<V>(ub | uoff[r])] = v[r];
        }
        __syncthreads();
    }

    for (int c = threadIdx.x; c < nchunks; c += blockDim.x) {
        const int u = c * APU;
        const uint64_t g = tb + hi_off[u >> L] + (u & lmask);
        const float4 val = *reinterpret_cast<const float4 *>(&tile[swz<V>(u)]);
        st_cs16(&st[g], val);
    }
}

// ---- encoded gates: device-side gate_matrix (gate.hpp:89-154) -------------
template <typename T>
__global__ void bind_kernel(const double *__restrict__ data, int rows, int slots, const EncDesc *__restrict__ encs,
                            int nenc, T *__restrict__ table) {
    const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= static_cast<int64_t>(rows) * nenc) return;
    const int e = static_cast<int>(i / rows), row = static_cast<int>(i % rows);
    const EncDesc d = encs[e];
    const double *p = data + static_cast<size_t>(row) * slots + d.slot;
    double re[16], im[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) re[q] = im[q] = 0.0;
    int dim = 2;
    double c, s;
    sincos(p[0] / 2, &s, &c);
    switch (d.kind) {
    case GK_RX: re[0] = c, im[1] = -s, im[2] = -s, re[3] = c; break;
    case GK_RY: re[0] = c, re[1] = -s, re[2] = s, re[3] = c; break;
    case GK_RZ: re[0] = c, im[0] = -s, re[3] = c, im[3] = s; break;
    case GK_P: {
        double sp, cp;
        sincos(p[0], &sp, &cp);
        re[0] = 1, re[3] = cp, im[3] = sp;
        break;
    }
    case GK_U3: {
        double sl, cl, sf, cf, sfl, cfl;
        sincos(p[2], &sl, &cl);
        sincos(p[1], &sf, &cf);
        sincos(p[1] + p[2], &sfl, &cfl);
        re[0] = c;
        re[1] = -cl * s, im[1] = -sl * s;
        re[2] = cf * s, im[2] = sf * s;
        re[3] = cfl * c, im[3] = sfl * c;
        break;
    }
    case GK_RXX: // c I - i s X(x)X
        dim = 4;
        for (int q = 0; q < 4; ++q) re[q * 5] = c;
        im[3] = im[6] = im[9] = im[12] = -s;
        break;
    case GK_RYY: // Y(x)Y = [[0,0,0,-1],[0,0,1,0],[0,1,0,0],[-1,0,0,0]]
        dim = 4;
        for (int q = 0; q < 4; ++q) re[q * 5] = c;
        im[3] = s, im[6] = -s, im[9] = -s, im[12] = s;
        break;
    case GK_RZZ:
        dim = 4;
        re[0] = c, im[0] = -s;
        re[5] = c, im[5] = s;
        re[10] = c, im[10] = s;
        re[15] = c, im[15] = -s;
        break;
    }
    T *out = table + (static_cast<size_t>(e) * rows + row) * 32;
    if (d.diag) {
        for (int q = 0; q < dim; ++q) {
            out[2 * q] = static_cast<T>(re[q * dim + q]);
            out[2 * q + 1] = static_cast<T>(im[q * dim + q]);
        }
        return;
    }
    for (int r = 0; r < dim; ++r)
        for (int cc = 0; cc < dim; ++cc) {
            int rr = r, c2 = cc;
            if (d.swapq) {
                rr = ((r & 1) << 1) | (r >> 1);
                c2 = ((cc & 1) << 1) | (cc >> 1);
            }
            out[2 * (r * dim + cc)] = static_cast<T>(re[rr * dim + c2]);
            out[2 * (r * dim + cc) + 1] = static_cast<T>(im[rr * dim + c2]);
        }
}

// ---- basis state / conversions ----------------------------------------------
template <typename T>
__global__ void set_basis_kernel(typename Vec2<T>::type *st, uint64_t amps, int batch, uint64_t idx, int on) {
    using V = typename Vec2<T>::type;
    const uint64_t total = amps * batch;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        st[i] = (on && (i % amps) == idx) ? V{1, 0} : V{0, 0};
}

__global__ void f64_to_f32_kernel(float *dst, const double *src, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        dst[i] = static_cast<float>(src[i]);
}
__global__ void f32_to_f64_kernel(double *dst, const float *src, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        dst[i] = static_cast<double>(src[i]);
}

// ---- reductions -----------------------------------------------------------
__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    return x;
}

constexpr int kZ = 41; // total + one accumulator per physical local bit (<= 40)

// Per row: acc[0] = sum |a|^2, acc[1+b] = sum over indices with bit b set.
// Each thread walks aligned chunks of 16 amplitudes: the 4 low bits are
// resolved per element at compile time, the high bits once per chunk.
template <typename T, int CL>
__global__ void __launch_bounds__(256) zsum_kernel(const typename Vec2<T>::type *__restrict__ st, uint64_t row_stride,
                                                   int nlocal, double *__restrict__ partial) {
    using V = typename Vec2<T>::type;
    const int row = blockIdx.y;
    const V *p = st + static_cast<size_t>(row) * row_stride;
    double acc[kZ];
#pragma unroll
    for (int b = 0; b < kZ; ++b) acc[b] = 0.0;
    const uint64_t nchunk = (1ull << nlocal) >> CL;
    for (uint64_t ch = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; ch < nchunk;
         ch += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t base = ch << CL;
        double tot = 0.0;
#pragma unroll
        for (int j = 0; j < (1 << CL); ++j) {
            const V x = p[base + j];
            const double w = static_cast<double>(x.x) * x.x + static_cast<double>(x.y) * x.y;
            tot += w;
#pragma unroll
            for (int b = 0; b < CL; ++b)
                if ((j >> b) & 1) acc[1 + b] += w;
        }
        acc[0] += tot;
#pragma unroll
        for (int b = CL; b < kZ - 1; ++b)
            if (b < nlocal && ((base >> b) & 1ull)) acc[1 + b] += tot;
    }
    __shared__ double red[8][kZ];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int b = 0; b < kZ; ++b) {
        const double s = warp_sum(acc[b]);
        if (lane == 0) red[wid][b] = s;
    }
    __syncthreads();
    if (threadIdx.x < kZ) {
        double s = 0.0;
        for (int w = 0; w < (blockDim.x >> 5); ++w) s += red[w][threadIdx.x];
        partial[(static_cast<size_t>(row) * gridDim.x + blockIdx.x) * kZ + threadIdx.x] = s;
    }
}

// sum_i conj(a_i) * (-1)^popc(i & zy) * a_{i ^ flip}   (re, im)
template <typename T>
__global__ void __launch_bounds__(256) pauli_kernel(const typename Vec2<T>::type *__restrict__ st,
                                                    uint64_t row_stride, uint64_t amps, uint64_t flip, uint64_t zy,
                                                    uint64_t rank_base, double *__restrict__ partial) {
    using V = typename Vec2<T>::type;
    const int row = blockIdx.y;
    const V *p = st + static_cast<size_t>(row) * row_stride;
    double re = 0.0, im = 0.0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < amps;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const V a = p[i], b = p[i ^ flip];
        const double sgn = (__popcll((rank_base | i) & zy) & 1) ? -1.0 : 1.0;
        re += sgn * (static_cast<double>(a.x) * b.x + static_cast<double>(a.y) * b.y);
        im += sgn * (static_cast<double>(a.x) * b.y - static_cast<double>(a.y) * b.x);
    }
    __shared__ double red[2][8];
    re = warp_sum(re);
    im = warp_sum(im);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) red[0][wid] = re, red[1][wid] = im;
    __syncthreads();
    if (threadIdx.x < 2) {
        double s = 0.0;
        for (int w = 0; w < (blockDim.x >> 5); ++w) s += red[threadIdx.x][w];
        partial[(static_cast<size_t>(row) * gridDim.x + blockIdx.x) * 2 + threadIdx.x] = s;
    }
}

// Rank bits of a distributed state: every local amplitude has the same value
// of a rank bit, so its "bit set" weight is the local total or zero.
__global__ void rank_bits_kernel(double *out, int rows, int nlocal, int n, int rank) {
    const int row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= rows) return;
    double *o = out + static_cast<size_t>(row) * kZ;
    for (int b = nlocal; b < n && b < kZ - 1; ++b) o[1 + b] = ((rank >> (b - nlocal)) & 1) ? o[0] : 0.0;
}

// Second stage: out[row * width + j] = sum over blocks of partial.
__global__ void reduce_partials_kernel(const double *__restrict__ partial, int blocks, int width,
                                       double *__restrict__ out) {
    const int row = blockIdx.x;
    for (int j = threadIdx.x; j < width; j += blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < blocks; ++b) s += partial[(static_cast<size_t>(row) * blocks + b) * width + j];
        out[static_cast<size_t>(row) * width + j] = s;
    }
}

// marginal_probabilities: k bins <= 4096 in shared memory, else global atomics.
template <typename T>
__global__ void __launch_bounds__(256) marginal_kernel(const typename Vec2<T>::type *__restrict__ p, uint64_t amps,
                                                       const int *__restrict__ bits, int k, uint64_t rank_base,
                                                       double *__restrict__ out_partial, int use_smem) {
    extern __shared__ double hist[];
    const int nb = 1 << k;
    if (use_smem)
        for (int j = threadIdx.x; j < nb; j += blockDim.x) hist[j] = 0.0;
    __syncthreads();
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < amps;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const auto x = p[i];
        const double w = static_cast<double>(x.x) * x.x + static_cast<double>(x.y) * x.y;
        const uint64_t gi = rank_base | i;
        int o = 0;
        for (int j = 0; j < k; ++j) o = (o << 1) | static_cast<int>((gi >> bits[j]) & 1ull);
        if (use_smem) atomicAdd(&hist[o], w);
        else atomicAdd(&out_partial[o], w);
    }
    if (!use_smem) return;
    __syncthreads();
    for (int j = threadIdx.x; j < nb; j += blockDim.x)
        out_partial[static_cast<size_t>(blockIdx.x) * nb + j] = hist[j];
}

template <typename T, int R> void set_attrs(size_t smem) {
    static size_t done = 0;
    if (smem > done) {
        QSV_CUDA(cudaFuncSetAttribute(tile_pass_kernel<T, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        done = smem;
    }
}

template <typename T, int R> void launch_tile(const DevPass &dp, void *state, int rows, cudaStream_t s) {
    set_attrs<T, R>(dp.smem);
    PassArgs a = dp.args;
    a.state = state;
    for (int r0 = 0; r0 < rows; r0 += 65535) {
        a.row0 = r0;
        const dim3 grid(static_cast<unsigned>(dp.tiles), static_cast<unsigned>(std::min(rows - r0, 65535)));
        tile_pass_kernel<T, R><<<grid, dp.threads, dp.smem, s>>>(a);
    }
    QSV_CUDA(cudaGetLastError());
}

int grid_for(uint64_t work, int threads, int sm_count) {
    const uint64_t want = (work + threads - 1) / threads;
    const uint64_t cap = static_cast<uint64_t>(sm_count) * 8;
    return static_cast<int>(std::max<uint64_t>(1, std::min(want, cap)));
}

} // namespace

// ---------------------------------------------------------------- launchers --
void launch_pass(const DevPass &dp, int dtype, void *state, int rows, cudaStream_t s) {
    const int R = std::min(kRegSlots, dp.args.K);
    if (dtype == QSV_C64) {
        switch (R) {
        case 1: launch_tile<float, 1>(dp, state, rows, s); break;
        case 2: launch_tile<float, 2>(dp, state, rows, s); break;
        case 3: launch_tile<float, 3>(dp, state, rows, s); break;
        default: launch_tile<float, 4>(dp, state, rows, s); break;
        }
    } else {
        switch (R) {
        case 1: launch_tile<double, 1>(dp, state, rows, s); break;
        case 2: launch_tile<double, 2>(dp, state, rows, s); break;
        case 3: launch_tile<double, 3>(dp, state, rows, s); break;
        default: launch_tile<double, 4>(dp, state, rows, s); break;
        }
    }
}

void launch_bind(const Plan &p, const double *d_data, int rows, int slots, cudaStream_t s) {
    const int nenc = static_cast<int>(p.encs.size());
    if (nenc == 0) return;
    const int64_t work = static_cast<int64_t>(rows) * nenc;
    const int threads = 128;
    const int blocks = static_cast<int>((work + threads - 1) / threads);
    if (p.dtype == QSV_C64)
        bind_kernel<float><<<blocks, threads, 0, s>>>(d_data, rows, slots, static_cast<const EncDesc *>(p.d_encs), nenc,
                                                      static_cast<float *>(p.d_enc_table));
    else
        bind_kernel<double><<<blocks, threads, 0, s>>>(d_data, rows, slots, static_cast<const EncDesc *>(p.d_encs),
                                                       nenc, static_cast<double *>(p.d_enc_table));
    QSV_CUDA(cudaGetLastError());
}

void launch_set_basis(State &st, uint64_t local_index, bool on_this_rank) {
    const uint64_t total = st.local_amps * st.batch;
    const int g = grid_for(total, 256, st.ctx->sm_count);
    if (st.dtype == QSV_C64)
        set_basis_kernel<float><<<g, 256, 0, st.ctx->stream>>>(static_cast<float2 *>(st.d), st.local_amps, st.batch,
                                                                local_index, on_this_rank);
    else
        set_basis_kernel<double><<<g, 256, 0, st.ctx->stream>>>(static_cast<double2 *>(st.d), st.local_amps, st.batch,
                                                                 local_index, on_this_rank);
    QSV_CUDA(cudaGetLastError());
}

void launch_convert(void *dst, int dst_dtype, const void *src, int src_dtype, uint64_t count, cudaStream_t s) {
    const int g = static_cast<int>(std::min<uint64_t>((count + 255) / 256, 148 * 16));
    if (dst_dtype == QSV_C64 && src_dtype == QSV_C128)
        f64_to_f32_kernel<<<std::max(g, 1), 256, 0, s>>>(static_cast<float *>(dst), static_cast<const double *>(src),
                                                          count);
    else if (dst_dtype == QSV_C128 && src_dtype == QSV_C64)
        f32_to_f64_kernel<<<std::max(g, 1), 256, 0, s>>>(static_cast<double *>(dst), static_cast<const float *>(src),
                                                          count);
    else fail(QSV_ERR_INTERNAL, "launch_convert: bad dtypes");
    QSV_CUDA(cudaGetLastError());
}

namespace {
struct DevBuf {
    void *p = nullptr;
    explicit DevBuf(size_t bytes) { QSV_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16))); }
    ~DevBuf() { cudaFree(p); }
    template <typename X> X *as() { return static_cast<X *>(p); }
};
} // namespace

void reduce_z_all(State &st, double *host_out) {
    const int rows = st.batch;
    const int CL = st.nlocal >= 4 ? 4 : 0;
    const uint64_t nchunk = st.local_amps >> CL;
    const int per_row = std::max(1, std::min<int>(static_cast<int>((nchunk + 255) / 256), st.ctx->sm_count * 4));
    DevBuf partial(sizeof(double) * rows * per_row * kZ), out(sizeof(double) * rows * kZ);
    const dim3 grid(per_row, rows);
    cudaStream_t s = st.ctx->stream;
    if (st.dtype == QSV_C64) {
        if (CL == 4) zsum_kernel<float, 4><<<grid, 256, 0, s>>>(static_cast<const float2 *>(st.d), st.local_amps, st.nlocal, partial.as<double>());
        else zsum_kernel<float, 0><<<grid, 256, 0, s>>>(static_cast<const float2 *>(st.d), st.local_amps, st.nlocal, partial.as<double>());
    } else {
        if (CL == 4) zsum_kernel<double, 4><<<grid, 256, 0, s>>>(static_cast<const double2 *>(st.d), st.local_amps, st.nlocal, partial.as<double>());
        else zsum_kernel<double, 0><<<grid, 256, 0, s>>>(static_cast<const double2 *>(st.d), st.local_amps, st.nlocal, partial.as<double>());
    }
    QSV_CUDA(cudaGetLastError());
    reduce_partials_kernel<<<rows, 64, 0, s>>>(partial.as<double>(), per_row, kZ, out.as<double>());
    QSV_CUDA(cudaGetLastError());
    if (st.n > st.nlocal) {
        rank_bits_kernel<<<(rows + 127) / 128, 128, 0, s>>>(out.as<double>(), rows, st.nlocal, st.n, st.ctx->rank);
        QSV_CUDA(cudaGetLastError());
    }
    if (st.ctx->world > 1) dist_allreduce_sum(*st.ctx, out.as<double>(), static_cast<size_t>(rows) * kZ);
    QSV_CUDA(cudaMemcpyAsync(host_out, out.p, sizeof(double) * rows * kZ, cudaMemcpyDeviceToHost, s));
    QSV_CUDA(cudaStreamSynchronize(s));
}

void reduce_pauli(State &st, uint64_t flip, uint64_t zy, double *host_out) {
    const int rows = st.batch;
    const int per_row = std::max(1, std::min<int>(static_cast<int>((st.local_amps + 255) / 256), st.ctx->sm_count * 4));
    DevBuf partial(sizeof(double) * rows * per_row * 2), out(sizeof(double) * rows * 2);
    const dim3 grid(per_row, rows);
    cudaStream_t s = st.ctx->stream;
    const uint64_t rank_base = static_cast<uint64_t>(st.ctx->rank) << st.nlocal;
    if (st.dtype == QSV_C64)
        pauli_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float2 *>(st.d), st.local_amps, st.local_amps, flip, zy, rank_base, partial.as<double>());
    else
        pauli_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double2 *>(st.d), st.local_amps, st.local_amps, flip, zy, rank_base, partial.as<double>());
    QSV_CUDA(cudaGetLastError());
    reduce_partials_kernel<<<rows, 64, 0, s>>>(partial.as<double>(), per_row, 2, out.as<double>());
    QSV_CUDA(cudaGetLastError());
    if (st.ctx->world > 1) dist_allreduce_sum(*st.ctx, out.as<double>(), static_cast<size_t>(rows) * 2);
    QSV_CUDA(cudaMemcpyAsync(host_out, out.p, sizeof(double) * rows * 2, cudaMemcpyDeviceToHost, s));
    QSV_CUDA(cudaStreamSynchronize(s));
}

void reduce_norm2(State &st, double *host_out) {
    std::vector<double> z(static_cast<size_t>(st.batch) * kZ);
    reduce_z_all(st, z.data());
    for (int b = 0; b < st.batch; ++b) host_out[b] = z[static_cast<size_t>(b) * kZ];
}

void reduce_marginal(State &st, int row, const std::vector<int> &phys_bits, double *host_out) {
    const int k = static_cast<int>(phys_bits.size());
    require(k >= 1 && k <= 26, "marginal_probs: 1..26 wires supported");
    const int nb = 1 << k;
    const bool use_smem = nb <= 4096;
    const int blocks = use_smem ? std::max(1, std::min<int>(static_cast<int>((st.local_amps + 255) / 256), st.ctx->sm_count * 2)) : st.ctx->sm_count * 4;
    DevBuf bits(sizeof(int) * k), partial(sizeof(double) * (use_smem ? static_cast<size_t>(blocks) * nb : nb)),
        out(sizeof(double) * nb);
    cudaStream_t s = st.ctx->stream;
    QSV_CUDA(cudaMemcpyAsync(bits.p, phys_bits.data(), sizeof(int) * k, cudaMemcpyHostToDevice, s));
    if (!use_smem) QSV_CUDA(cudaMemsetAsync(partial.p, 0, sizeof(double) * nb, s));
    const uint64_t rank_base = static_cast<uint64_t>(st.ctx->rank) << st.nlocal;
    const size_t smem = use_smem ? sizeof(double) * nb : 0;
    if (st.dtype == QSV_C64)
        marginal_kernel<float><<<blocks, 256, smem, s>>>(static_cast<const float2 *>(st.d) + static_cast<size_t>(row) * st.local_amps, st.local_amps, bits.as<int>(), k, rank_base, partial.as<double>(), use_smem);
    else
        marginal_kernel<double><<<blocks, 256, smem, s>>>(static_cast<const double2 *>(st.d) + static_cast<size_t>(row) * st.local_amps, st.local_amps, bits.as<int>(), k, rank_base, partial.as<double>(), use_smem);
    QSV_CUDA(cudaGetLastError());
    double *res = partial.as<double>();
    if (use_smem) {
        // sum block partials: treat each bin as a "row" of width 1 over blocks
        std::vector<double> host(static_cast<size_t>(blocks) * nb);
        QSV_CUDA(cudaMemcpyAsync(host.data(), partial.p, sizeof(double) * host.size(), cudaMemcpyDeviceToHost, s));
        QSV_CUDA(cudaStreamSynchronize(s));
        for (int j = 0; j < nb; ++j) {
            double acc = 0.0;
            for (int b = 0; b < blocks; ++b) acc += host[static_cast<size_t>(b) * nb + j];
            host_out[j] = acc;
        }
        if (st.ctx->world > 1) {
            QSV_CUDA(cudaMemcpyAsync(out.p, host_out, sizeof(double) * nb, cudaMemcpyHostToDevice, s));
            dist_allreduce_sum(*st.ctx, out.as<double>(), nb);
            QSV_CUDA(cudaMemcpyAsync(host_out, out.p, sizeof(double) * nb, cudaMemcpyDeviceToHost, s));
            QSV_CUDA(cudaStreamSynchronize(s));
        }
        return;
    }
    if (st.ctx->world > 1) dist_allreduce_sum(*st.ctx, res, nb);
    QSV_CUDA(cudaMemcpyAsync(host_out, res, sizeof(double) * nb, cudaMemcpyDeviceToHost, s));
    QSV_CUDA(cudaStreamSynchronize(s));
}

} // namespace qsv
