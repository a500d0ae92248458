// sm_100a support kernels of the qsv engine (the fused gate pass lives in
// tile_pass.cu):
//   bind_kernel        device-side gate_matrix for encoded (per-row) gates
//                      (gate.hpp:89-154, circuit.hpp:139-147).
//   zsum/pauli/norm    FP64 warp->block->grid reductions for expectation_one
//                      (circuit.hpp:248-282) and the norm.
//   marginal_kernel    marginal_probabilities histogram (circuit.hpp:182-205).
#include <cuda_runtime.h>

#include <cstdio>
#include <map>
#include <mutex>

#include "qsv_internal.hpp"

#include "device_util.cuh"

namespace qsv {

void cuda_check(cudaError_t e, const char *what) {
    if (e != cudaSuccess) fail(QSV_ERR_INTERNAL, std::string("CUDA error ") + cudaGetErrorString(e) + " at " + what);
}

namespace {
using dev::Vec2;
using dev::warp_sum;

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

// Mixed states: the engine holds rho (2^m x 2^m, row-major) as the 2m-qubit
// vector vec(rho)[r * 2^m + c] (row wires = the high m bits). Tr[rho P] for a
// Pauli string P is sum_r rho[r, r ^ flip] * (-1)^popc(r & zy) times i^#Y
// (applied by the caller): only the 2^m entries of one "diagonal" are read.
template <typename T>
__global__ void __launch_bounds__(256) dm_pauli_kernel(const typename Vec2<T>::type *__restrict__ st,
                                                       uint64_t row_stride, int m, uint64_t flip, uint64_t zy,
                                                       double *__restrict__ partial) {
    using V = typename Vec2<T>::type;
    const int row = blockIdx.y;
    const V *p = st + static_cast<size_t>(row) * row_stride;
    const uint64_t dim = 1ull << m;
    double re = 0.0, im = 0.0;
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < dim;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const V a = p[(r << m) | (r ^ flip)];
        const double sgn = (__popcll(r & zy) & 1) ? -1.0 : 1.0;
        re += sgn * static_cast<double>(a.x);
        im += sgn * static_cast<double>(a.y);
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

// marginal_probabilities of a mixed state: bins of Re rho[r, r] (circuit.hpp:199-203).
template <typename T>
__global__ void __launch_bounds__(256) dm_marginal_kernel(const typename Vec2<T>::type *__restrict__ p, int m,
                                                          const int *__restrict__ bits, int k,
                                                          double *__restrict__ out_partial) {
    extern __shared__ double hist[];
    const int nb = 1 << k;
    for (int j = threadIdx.x; j < nb; j += blockDim.x) hist[j] = 0.0;
    __syncthreads();
    const uint64_t dim = 1ull << m;
    for (uint64_t r = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; r < dim;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double w = static_cast<double>(p[(r << m) | r].x);
        int o = 0;
        for (int j = 0; j < k; ++j) o = (o << 1) | static_cast<int>((r >> bits[j]) & 1ull);
        atomicAdd(&hist[o], w);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < nb; j += blockDim.x) out_partial[static_cast<size_t>(blockIdx.x) * nb + j] = hist[j];
}

int grid_for(uint64_t work, int threads, int sm_count) {
    const uint64_t want = (work + threads - 1) / threads;
    const uint64_t cap = static_cast<uint64_t>(sm_count) * 8;
    return static_cast<int>(std::max<uint64_t>(1, std::min(want, cap)));
}

} // namespace

// Product-state prefix of a from-|0> plan: u_w = M_k ... M_1 |0> per (row,
// wire), written as out[(row * n + p) * 2 + b] = u_w[b] with p = n - 1 - w
// (the canonical physical bit of wire w).
template <typename T>
__global__ void prefix_kernel(const int *__restrict__ prog, const double *__restrict__ mats,
                              const T *__restrict__ enc_table, int rows, int n, typename Vec2<T>::type *out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= rows * n) return;
    const int row = i / n, w = i % n;
    double a0 = 1.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;  // (a0 + i a1, b0 + i b1)
    for (int k = prog[w]; k < prog[w + 1]; ++k) {
        const int e = prog[k];
        double m[8];
        if (e >= 0) {
            const T *t = enc_table + (static_cast<size_t>(e) * rows + row) * 32;
            for (int q = 0; q < 8; ++q) m[q] = static_cast<double>(t[q]);
        } else {
            const double *t = mats + static_cast<size_t>(-1 - e) * 8;
            for (int q = 0; q < 8; ++q) m[q] = t[q];
        }
        const double na0 = m[0] * a0 - m[1] * a1 + m[2] * b0 - m[3] * b1;
        const double na1 = m[0] * a1 + m[1] * a0 + m[2] * b1 + m[3] * b0;
        const double nb0 = m[4] * a0 - m[5] * a1 + m[6] * b0 - m[7] * b1;
        const double nb1 = m[4] * a1 + m[5] * a0 + m[6] * b1 + m[7] * b0;
        a0 = na0, a1 = na1, b0 = nb0, b1 = nb1;
    }
    using V = typename Vec2<T>::type;
    V *o = out + (static_cast<size_t>(row) * n + (n - 1 - w)) * 2;
    o[0] = V{static_cast<T>(a0), static_cast<T>(a1)};
    o[1] = V{static_cast<T>(b0), static_cast<T>(b1)};
}

void launch_prefix(const Plan &p, int rows, cudaStream_t s) {
    const int work = rows * p.nlocal;
    const int threads = 128, blocks = (work + threads - 1) / threads;
    if (p.dtype == QSV_C64)
        prefix_kernel<float><<<blocks, threads, 0, s>>>(static_cast<const int *>(p.d_prefix_prog),
            static_cast<const double *>(p.d_prefix_mats), static_cast<const float *>(p.d_enc_table), rows, p.nlocal,
            static_cast<float2 *>(p.d_prefix));
    else
        prefix_kernel<double><<<blocks, threads, 0, s>>>(static_cast<const int *>(p.d_prefix_prog),
            static_cast<const double *>(p.d_prefix_mats), static_cast<const double *>(p.d_enc_table), rows, p.nlocal,
            static_cast<double2 *>(p.d_prefix));
    QSV_CUDA(cudaGetLastError());
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

namespace {
// One gate, one launch (qsv_apply_gate / qsv_apply_matrix on one GPU): the
// reference's apply_matrix_strided (state.hpp:111-143) as a single sweep --
// each thread owns groups of 2^k amplitudes whose target bits are 0, applies
// the 2^k x 2^k matrix where every control bit is 1, and with
// zero_off_control zeroes the groups where one is 0. No plan, no program
// upload, no host synchronisation: a loop of apply_gate calls (the
// reference's usage) runs at one sweep per gate.
struct DirectGate {
    int t0 = 0, t1 = 0, zoc = 0;
    uint64_t cmask = 0;
    double m[32];  // 2^k x 2^k row-major (re, im); wires[0] is the matrix MSB
};

__device__ __forceinline__ uint64_t ins0(uint64_t x, int b) {
    return ((x >> b) << (b + 1)) | (x & ((1ull << b) - 1));
}

template <typename T, int K>
__global__ void __launch_bounds__(256) direct_gate_kernel(typename Vec2<T>::type *__restrict__ st, uint64_t local_amps,
                                                          int log_groups, uint64_t total, const DirectGate g) {
    constexpr int D = 1 << K;
    const int lo = K == 2 ? min(g.t0, g.t1) : g.t0, hi = K == 2 ? max(g.t0, g.t1) : g.t0;
    for (uint64_t w = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; w < total;
         w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t row = w >> log_groups, gi = w & ((1ull << log_groups) - 1);
        uint64_t base = ins0(gi, lo);
        if (K == 2) base = ins0(base, hi);
        typename Vec2<T>::type *v = st + row * local_amps;
        uint64_t off[D];
        if (K == 1) off[0] = 0, off[1] = 1ull << g.t0;
        else
            for (int r = 0; r < D; ++r) off[r] = ((r >> 1) & 1 ? 1ull << g.t0 : 0ull) | (r & 1 ? 1ull << g.t1 : 0ull);
        if ((base & g.cmask) != g.cmask) {
            if (g.zoc) {
                typename Vec2<T>::type z;
                z.x = 0, z.y = 0;
#pragma unroll
                for (int r = 0; r < D; ++r) v[base | off[r]] = z;
            }
            continue;
        }
        double xr[D], xi[D];
#pragma unroll
        for (int r = 0; r < D; ++r) {
            const auto a = v[base | off[r]];
            xr[r] = a.x, xi[r] = a.y;
        }
#pragma unroll
        for (int r = 0; r < D; ++r) {
            double yr = 0.0, yi = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const double mr = g.m[2 * (r * D + c)], mi = g.m[2 * (r * D + c) + 1];
                yr += mr * xr[c] - mi * xi[c];
                yi += mr * xi[c] + mi * xr[c];
            }
            typename Vec2<T>::type o;
            o.x = static_cast<T>(yr), o.y = static_cast<T>(yi);
            v[base | off[r]] = o;
        }
    }
}
} // namespace

bool apply_direct(State &st, const GateRec &g) {
    static const bool off = [] {  // QSV_X_NODIRECT=1: one-gate plans instead
        const char *e = std::getenv("QSV_X_NODIRECT");
        return e && e[0] == '1';
    }();
    if (off || st.ctx->world != 1 || g.encoded || g.k < 1 || g.k > 2) return false;
    DirectGate a;
    a.t0 = st.perm[g.wires[0]];
    a.t1 = g.k == 2 ? st.perm[g.wires[1]] : 0;
    for (int c : g.ctls) a.cmask |= 1ull << st.perm[c];
    a.zoc = (g.flags & OPF_ZERO_OFF_CONTROL) ? 1 : 0;
    const int d = 1 << g.k;
    for (int i = 0; i < d * d; ++i) a.m[2 * i] = g.m[i].real(), a.m[2 * i + 1] = g.m[i].imag();
    const int log_groups = st.nlocal - g.k;
    const uint64_t total = static_cast<uint64_t>(st.batch) << log_groups;
    const int grid = grid_for(total, 256, st.ctx->sm_count);
    cudaStream_t s = st.ctx->stream;
    if (st.dtype == QSV_C64) {
        auto *v = static_cast<float2 *>(st.d);
        if (g.k == 1) direct_gate_kernel<float, 1><<<grid, 256, 0, s>>>(v, st.local_amps, log_groups, total, a);
        else direct_gate_kernel<float, 2><<<grid, 256, 0, s>>>(v, st.local_amps, log_groups, total, a);
    } else {
        auto *v = static_cast<double2 *>(st.d);
        if (g.k == 1) direct_gate_kernel<double, 1><<<grid, 256, 0, s>>>(v, st.local_amps, log_groups, total, a);
        else direct_gate_kernel<double, 2><<<grid, 256, 0, s>>>(v, st.local_amps, log_groups, total, a);
    }
    QSV_CUDA(cudaGetLastError());
    return true;
}

// <Z_w> of every row from the fused epilogue's sums: z[b][0] is the row's
// total |a|^2, z[b][1 + bit] the |a|^2 with that physical bit set.
struct ZPerm {
    int bit[kMaxQubits];
};
__global__ void z_finish_kernel(const double *__restrict__ z, int k1, int rows, int n, const ZPerm perm,
                                double *__restrict__ out) {
    const int total = rows * n;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int b = i / n, w = i - b * n;
        const double *zb = z + static_cast<size_t>(b) * k1;
        out[i] = zb[0] - 2.0 * zb[1 + perm.bit[w]];
    }
}

void launch_z_finish(const double *z, int k1, int rows, int n, const std::vector<int> &perm, double *out,
                     cudaStream_t s) {
    require(n <= kMaxQubits, "z_finish: too many qubits");
    ZPerm pm{};
    for (int w = 0; w < n; ++w) pm.bit[w] = perm[w];
    const int total = rows * n;
    const int blocks = std::max(1, std::min((total + 255) / 256, 1024));
    z_finish_kernel<<<blocks, 256, 0, s>>>(z, k1, rows, n, pm, out);
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
// Small reduction buffers come from a per-device cache (cudaMalloc/cudaFree
// synchronise the device and cost milliseconds; the reductions run every step
// of a batched workload). Blocks are returned after the host has synchronised
// with the stream that used them, so reuse is ordered.
struct BufCache {
    std::mutex mu;
    std::multimap<size_t, std::pair<int, void *>> free_blocks; // size -> (device, ptr)
};
BufCache &buf_cache() {
    static BufCache *c = new BufCache(); // intentionally leaked: outlives static destruction
    return *c;
}
struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    int dev = 0;
    int unwinding = std::uncaught_exceptions();
    explicit DevBuf(size_t bytes) {
        bytes = std::max<size_t>(bytes, 256);
        QSV_CUDA(cudaGetDevice(&dev));
        BufCache &c = buf_cache();
        {
            std::lock_guard<std::mutex> lk(c.mu);
            for (auto it = c.free_blocks.lower_bound(bytes); it != c.free_blocks.end() && it->first <= 4 * bytes; ++it)
                if (it->second.first == dev) {
                    p = it->second.second;
                    cap = it->first;
                    c.free_blocks.erase(it);
                    return;
                }
        }
        QSV_CUDA(cudaMalloc(&p, bytes));
        cap = bytes;
    }
    ~DevBuf() {
        if (std::uncaught_exceptions() > unwinding) {
            // a reduction threw part-way: kernels using the block may still run
            // and the host never synchronised, so the block must not be reused;
            // cudaFree waits for the device before releasing it
            cudaFree(p);
            return;
        }
        BufCache &c = buf_cache();
        std::lock_guard<std::mutex> lk(c.mu);
        c.free_blocks.emplace(cap, std::make_pair(dev, p));
    }
    template <typename X> X *as() { return static_cast<X *>(p); }
};
} // namespace

namespace {
// State buffers up to 256 MiB are recycled per device (512 MiB cached at
// most): the reference's value semantics make every apply_gate /
// apply_channel return a new state, and a cudaMalloc + cudaFree pair
// synchronises the device and costs far more than a small state's sweep.
// A buffer is cached once its stream has drained.
constexpr size_t kStateCacheBlock = size_t(256) << 20, kStateCacheTotal = size_t(512) << 20;
struct StateCache {
    std::mutex mu;
    std::multimap<size_t, std::pair<int, void *>> blocks;  // bytes -> (device, ptr)
    size_t total = 0;
};
StateCache &state_cache() {
    static StateCache *c = new StateCache();  // intentionally leaked: outlives static destruction
    return *c;
}
} // namespace

cudaError_t state_alloc(void **p, size_t bytes) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (bytes <= kStateCacheBlock) {
        StateCache &c = state_cache();
        std::lock_guard<std::mutex> lk(c.mu);
        auto range = c.blocks.equal_range(bytes);
        for (auto it = range.first; it != range.second; ++it)
            if (it->second.first == dev) {
                *p = it->second.second;
                c.total -= bytes;
                c.blocks.erase(it);
                return cudaSuccess;
            }
    }
    e = cudaMalloc(p, bytes);
    if (e == cudaErrorMemoryAllocation) {
        // give the cached buffers of this device back and retry once
        cudaGetLastError();
        StateCache &c = state_cache();
        std::lock_guard<std::mutex> lk(c.mu);
        for (auto it = c.blocks.begin(); it != c.blocks.end();) {
            if (it->second.first == dev) {
                cudaFree(it->second.second);
                c.total -= it->first;
                it = c.blocks.erase(it);
            } else ++it;
        }
        e = cudaMalloc(p, bytes);
    }
    return e;
}

void state_release(void *p, size_t bytes) {
    if (!p) return;
    if (bytes <= kStateCacheBlock) {
        // the buffer's own device (a state may be destroyed on any thread,
        // after its context); cached once that device has drained -- what
        // cudaFree would have waited for anyway
        cudaPointerAttributes at{};
        int cur = 0;
        if (cudaPointerGetAttributes(&at, p) == cudaSuccess && at.type == cudaMemoryTypeDevice &&
            cudaGetDevice(&cur) == cudaSuccess) {
            const bool other = at.device != cur;
            bool ok = !other || cudaSetDevice(at.device) == cudaSuccess;
            ok = ok && cudaDeviceSynchronize() == cudaSuccess;
            if (other) cudaSetDevice(cur);
            if (ok) {
                StateCache &c = state_cache();
                std::lock_guard<std::mutex> lk(c.mu);
                if (c.total + bytes <= kStateCacheTotal) {
                    c.blocks.emplace(bytes, std::make_pair(at.device, p));
                    c.total += bytes;
                    return;
                }
            }
        }
        cudaGetLastError();
    }
    cudaFree(p);
}

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

void reduce_dm_pauli(State &st, int m, uint64_t flip, uint64_t zy, double *host_out) {
    require(2 * m == st.n && st.nlocal == st.n, "density: state is not a single-GPU vectorised density matrix");
    const int rows = st.batch;
    const uint64_t dim = 1ull << m;
    const int per_row = std::max(1, std::min<int>(static_cast<int>((dim + 255) / 256), st.ctx->sm_count * 4));
    DevBuf partial(sizeof(double) * rows * per_row * 2), out(sizeof(double) * rows * 2);
    const dim3 grid(per_row, rows);
    cudaStream_t s = st.ctx->stream;
    if (st.dtype == QSV_C64)
        dm_pauli_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float2 *>(st.d), st.local_amps, m, flip, zy, partial.as<double>());
    else
        dm_pauli_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double2 *>(st.d), st.local_amps, m, flip, zy, partial.as<double>());
    QSV_CUDA(cudaGetLastError());
    reduce_partials_kernel<<<rows, 64, 0, s>>>(partial.as<double>(), per_row, 2, out.as<double>());
    QSV_CUDA(cudaGetLastError());
    QSV_CUDA(cudaMemcpyAsync(host_out, out.p, sizeof(double) * rows * 2, cudaMemcpyDeviceToHost, s));
    QSV_CUDA(cudaStreamSynchronize(s));
}

void reduce_dm_marginal(State &st, int m, int row, const std::vector<int> &bits_r, double *host_out) {
    require(2 * m == st.n && st.nlocal == st.n, "density: state is not a single-GPU vectorised density matrix");
    const int k = static_cast<int>(bits_r.size());
    require(k >= 1 && k <= 12, "marginal_probs: 1..12 wires supported for density matrices");
    const int nb = 1 << k;
    const uint64_t dim = 1ull << m;
    const int blocks = std::max(1, std::min<int>(static_cast<int>((dim + 255) / 256), st.ctx->sm_count * 2));
    DevBuf bits(sizeof(int) * k), partial(sizeof(double) * static_cast<size_t>(blocks) * nb);
    cudaStream_t s = st.ctx->stream;
    QSV_CUDA(cudaMemcpyAsync(bits.p, bits_r.data(), sizeof(int) * k, cudaMemcpyHostToDevice, s));
    const size_t smem = sizeof(double) * nb;
    if (st.dtype == QSV_C64)
        dm_marginal_kernel<float><<<blocks, 256, smem, s>>>(static_cast<const float2 *>(st.d) + static_cast<size_t>(row) * st.local_amps, m, bits.as<int>(), k, partial.as<double>());
    else
        dm_marginal_kernel<double><<<blocks, 256, smem, s>>>(static_cast<const double2 *>(st.d) + static_cast<size_t>(row) * st.local_amps, m, bits.as<int>(), k, partial.as<double>());
    QSV_CUDA(cudaGetLastError());
    std::vector<double> host(static_cast<size_t>(blocks) * nb);
    QSV_CUDA(cudaMemcpyAsync(host.data(), partial.p, sizeof(double) * host.size(), cudaMemcpyDeviceToHost, s));
    QSV_CUDA(cudaStreamSynchronize(s));
    for (int j = 0; j < nb; ++j) {
        double acc = 0.0;
        for (int b = 0; b < blocks; ++b) acc += host[static_cast<size_t>(b) * nb + j];
        host_out[j] = acc;
    }
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
