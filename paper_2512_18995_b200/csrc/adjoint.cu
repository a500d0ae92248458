// Adjoint-method gradients on the GPU.
//
// Restates quasar::qubit::adjoint_gradients
// (/root/reference/proj/include/quasar/qubit/adjoint.hpp:52-110) on
// device-resident states:
//   * bind encoded parameters from the data row (adjoint.hpp:70-82): encoded
//     gates feed data_grads, trainable (non-encoded) gates param_grads;
//   * forward sweep psi = C |init> -- one fused plan (adjoint.hpp:84-86);
//   * lambda = sum_obs O psi (adjoint.hpp:30-45, 87);
//   * reverse sweep (adjoint.hpp:93-108): psi <- U^dagger psi; for each
//     parameter mu = dU psi with zero_off_control, grad = 2 Re<lambda|mu>;
//     lambda <- U^dagger lambda. On one GPU each gate is ONE fused kernel
//     (fused_sweep below); across ranks the steps run as whole-state
//     operations through one-gate plans.
// The derivative matrices restate gate_dmatrix (gate.hpp:157-190).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "device_util.cuh"
#include "qsv_internal.hpp"

namespace qsv {

void build_plan(Plan &p, Ctx *ctx, int n, int dtype, std::vector<GateRec> gates, int nslots, const qsv_opts *opts);

namespace {

using dev::Vec2;

template <typename T>
__global__ void axpy_kernel(typename Vec2<T>::type *__restrict__ y, const typename Vec2<T>::type *__restrict__ x,
                            uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        y[i].x += x[i].x;
        y[i].y += x[i].y;
    }
}

// sum conj(a_i) b_i in FP64 (the conjugate-linear Eigen dot, adjoint.hpp:102)
template <typename T>
__global__ void __launch_bounds__(256) dot_kernel(const typename Vec2<T>::type *__restrict__ a,
                                                  const typename Vec2<T>::type *__restrict__ b, uint64_t n,
                                                  double *__restrict__ partial) {
    double re = 0.0, im = 0.0;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double ax = a[i].x, ay = a[i].y, bx = b[i].x, by = b[i].y;
        re += ax * bx + ay * by;
        im += ax * by - ay * bx;
    }
    __shared__ double red[2][8];
    re = dev::warp_sum(re);
    im = dev::warp_sum(im);
    if ((threadIdx.x & 31) == 0) red[0][threadIdx.x >> 5] = re, red[1][threadIdx.x >> 5] = im;
    __syncthreads();
    if (threadIdx.x < 2) {
        double s = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += red[threadIdx.x][w];
        partial[2 * blockIdx.x + threadIdx.x] = s;
    }
}

struct DState { // RAII device state on a context
    State st;
    DState(Ctx *ctx, int n, int dtype) {
        st.ctx = ctx;
        st.n = n;
        st.nlocal = n - ctx->gbits;
        st.batch = 1;
        st.dtype = dtype;
        st.local_amps = 1ull << st.nlocal;
        st.perm.resize(n);
        for (int w = 0; w < n; ++w) st.perm[w] = n - 1 - w;
        const size_t bytes = st.local_amps * st.amp_bytes();
        if (cudaMalloc(&st.d, bytes) != cudaSuccess) {
            cudaGetLastError();
            fail(QSV_ERR_INTERNAL, "adjoint_gradients: cannot allocate a work state");
        }
    }
    size_t bytes() const { return st.local_amps * st.amp_bytes(); }
};

void copy_state(DState &dst, const DState &src, cudaStream_t s) {
    QSV_CUDA(cudaMemcpyAsync(dst.st.d, src.st.d, src.bytes(), cudaMemcpyDeviceToDevice, s));
}

void apply_rec(State &st, const GateRec &g) {
    Plan p;
    qsv_opts o{};
    o.fuse = 1;
    o.jit = -1; // one-gate passes: the interpreter, no compilation
    build_plan(p, st.ctx, st.n, st.dtype, {g}, 0, &o);
    execute_plan(p, st, nullptr, 0, 0);
}

double re_dot(const DState &a, const DState &b) {
    Ctx &c = *a.st.ctx;
    const uint64_t n = a.st.local_amps;
    const int blocks = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, c.sm_count * 4)));
    double *part = nullptr;
    QSV_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&part), sizeof(double) * 2 * blocks, c.stream));
    if (a.st.dtype == QSV_C64)
        dot_kernel<float><<<blocks, 256, 0, c.stream>>>(static_cast<const float2 *>(a.st.d),
                                                        static_cast<const float2 *>(b.st.d), n, part);
    else
        dot_kernel<double><<<blocks, 256, 0, c.stream>>>(static_cast<const double2 *>(a.st.d),
                                                         static_cast<const double2 *>(b.st.d), n, part);
    QSV_CUDA(cudaGetLastError());
    std::vector<double> h(2 * blocks);
    QSV_CUDA(cudaMemcpyAsync(h.data(), part, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, c.stream));
    QSV_CUDA(cudaFreeAsync(part, c.stream));
    QSV_CUDA(cudaStreamSynchronize(c.stream));
    double re = 0.0;
    for (int i = 0; i < blocks; ++i) re += h[2 * i];
    if (c.world > 1) {
        double *d = nullptr;
        QSV_CUDA(cudaMalloc(&d, sizeof(double)));
        QSV_CUDA(cudaMemcpy(d, &re, sizeof(double), cudaMemcpyHostToDevice));
        dist_allreduce_sum(c, d, 1);
        QSV_CUDA(cudaMemcpyAsync(&re, d, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        QSV_CUDA(cudaStreamSynchronize(c.stream));
        cudaFree(d);
    }
    return re;
}

// ---- fused single-GPU path ---------------------------------------------
// One kernel per reverse-sweep gate instead of the reference's sequence of
// full-state operations (apply U^dagger to psi; per parameter a copy, a
// zero-off-control dU apply and a dot; apply U^dagger to lambda): each thread
// owns groups of 2^k amplitudes (k <= 2), loads psi and lambda once, forms
// psi' = U^dagger psi, accumulates Re sum conj(lambda) (dU_q psi') over the
// groups whose controls are on (off-control groups contribute 0, as
// zero_off_control makes them, and keep psi / lambda unchanged), writes
// psi' and lambda' = U^dagger lambda, and adds its FP64 partial sums to the
// gradient slots. Same arithmetic as adjoint.hpp:93-108 per group; the
// gradients are read back once at the end.
struct AdjGate {
    int k = 1, t0 = 0, t1 = 0, nq = 0;
    uint64_t cmask = 0;
    int slot = -1;    // first gradient slot (params, then data slots)
    double u[32];     // U^dagger, 2^k x 2^k row-major (re, im)
    double du[3][32]; // d U / d params[q]
};

__device__ __forceinline__ uint64_t insert_zero(uint64_t x, int b) {
    const uint64_t lo = x & ((1ull << b) - 1);
    return ((x >> b) << (b + 1)) | lo;
}

template <typename T, int K, bool G>  // G: the gate has gradient parameters
__global__ void __launch_bounds__(256) adj_gate_kernel(typename Vec2<T>::type *__restrict__ psi,
                                                       typename Vec2<T>::type *__restrict__ lam, uint64_t ngroups,
                                                       const AdjGate g, double *__restrict__ part, int pb) {
    constexpr int D = 1 << K;
    double acc[3] = {0.0, 0.0, 0.0};
    const int lo = K == 2 ? (g.t0 < g.t1 ? g.t0 : g.t1) : g.t0, hi = K == 2 ? (g.t0 < g.t1 ? g.t1 : g.t0) : g.t0;
    for (uint64_t gi = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; gi < ngroups;
         gi += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t base = insert_zero(gi, lo);
        if (K == 2) base = insert_zero(base, hi);
        if ((base & g.cmask) != g.cmask) continue;
        uint64_t off[D];
        if (K == 1) off[0] = 0, off[1] = 1ull << g.t0;
        else
            for (int r = 0; r < D; ++r) off[r] = ((r >> 1) & 1 ? 1ull << g.t0 : 0ull) | (r & 1 ? 1ull << g.t1 : 0ull);
        double pr[D], pi[D], lr[D], li[D];
#pragma unroll
        for (int r = 0; r < D; ++r) {
            const auto a = psi[base | off[r]];
            const auto b = lam[base | off[r]];
            pr[r] = a.x, pi[r] = a.y, lr[r] = b.x, li[r] = b.y;
        }
        double nr[D], ni[D];
#pragma unroll
        for (int r = 0; r < D; ++r) {
            double xr = 0.0, xi = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const double ur = g.u[2 * (r * D + c)], ui = g.u[2 * (r * D + c) + 1];
                xr += ur * pr[c] - ui * pi[c];
                xi += ur * pi[c] + ui * pr[c];
            }
            nr[r] = xr, ni[r] = xi;
        }
        for (int q = 0; G && q < g.nq; ++q) {
            double s = 0.0;
#pragma unroll
            for (int r = 0; r < D; ++r) {
                double mr = 0.0, mi = 0.0;
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    const double dr = g.du[q][2 * (r * D + c)], di = g.du[q][2 * (r * D + c) + 1];
                    mr += dr * nr[c] - di * ni[c];
                    mi += dr * ni[c] + di * nr[c];
                }
                s += lr[r] * mr + li[r] * mi;  // Re(conj(lambda) mu)
            }
            acc[q] += s;
        }
#pragma unroll
        for (int r = 0; r < D; ++r) {
            double xr = 0.0, xi = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const double ur = g.u[2 * (r * D + c)], ui = g.u[2 * (r * D + c) + 1];
                xr += ur * lr[c] - ui * li[c];
                xi += ur * li[c] + ui * lr[c];
            }
            typename Vec2<T>::type a, b;
            a.x = static_cast<T>(nr[r]), a.y = static_cast<T>(ni[r]);
            b.x = static_cast<T>(xr), b.y = static_cast<T>(xi);
            psi[base | off[r]] = a;
            lam[base | off[r]] = b;
        }
    }
    if (!G || g.nq == 0) return;
    __shared__ double red[3][8];
    for (int q = 0; q < g.nq; ++q) {
        const double v = dev::warp_sum(acc[q]);
        if ((threadIdx.x & 31) == 0) red[q][threadIdx.x >> 5] = v;
    }
    __syncthreads();
    if (threadIdx.x < g.nq) {
        double s = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += red[threadIdx.x][w];
        part[static_cast<size_t>(g.slot + threadIdx.x) * pb + blockIdx.x] = 2.0 * s;
    }
}

// A run of single-qubit gates on one wire under one control mask (cfg1's rx,
// ry, rz per wire and layer): the reverse-sweep steps of every gate of the
// run on the thread's amplitude pair in registers -- psi and lambda loaded
// and stored once per run instead of once per gate. Per gate in sweep order:
// psi <- U^dag psi, each parameter's Re conj(lambda) dU psi, lambda <- U^dag
// lambda (adjoint.hpp:93-108); the pair stays in FP64 between the gates.
constexpr int kRunMax = 8;  // gates per run, and parameters per run
constexpr int kRunMinBlocks = 3;  // 256-thread blocks per SM the register budget must allow
struct AdjRun {
    int t0 = 0, n = 0, nacc = 0;
    uint64_t cmask = 0;
    int first[kRunMax + 1];    // gate k's parameters are accumulators [first[k], first[k + 1])
    int accslot[kRunMax];      // gradient slot of accumulator j
    double u[kRunMax][8];      // U^dagger of gate k, 2 x 2 row-major (re, im)
    double du[kRunMax][8];     // d U / d param of accumulator j
    int ut[kRunMax];           // sparsity class of u[k] (mat_class), of du[j]
    int dt[kRunMax];
};

// Sparsity class of a 2 x 2 complex matrix (re, im row-major): 1 diagonal
// (rz, p), 2 real (ry), 3 real diagonal with imaginary off-diagonal (rx),
// 0 general -- the products with exact zeros are not issued (FP64-bound
// sweep; without fast-math a multiply by 0.0 is not folded).
inline int mat_class(const double *m) {
    if (m[2] == 0 && m[3] == 0 && m[4] == 0 && m[5] == 0) return 1;
    if (m[1] == 0 && m[3] == 0 && m[5] == 0 && m[7] == 0) return 2;
    if (m[1] == 0 && m[7] == 0 && m[2] == 0 && m[4] == 0) return 3;
    return 0;
}

// y = M x for a 2 x 2 complex M of class ty; x, y = (x0r, x0i, x1r, x1i)
__device__ __forceinline__ void cmv2(int ty, const double *m, const double *x, double *y) {
    switch (ty) {
    case 1:
        y[0] = m[0] * x[0] - m[1] * x[1];
        y[1] = m[0] * x[1] + m[1] * x[0];
        y[2] = m[6] * x[2] - m[7] * x[3];
        y[3] = m[6] * x[3] + m[7] * x[2];
        break;
    case 2:
        y[0] = m[0] * x[0] + m[2] * x[2];
        y[1] = m[0] * x[1] + m[2] * x[3];
        y[2] = m[4] * x[0] + m[6] * x[2];
        y[3] = m[4] * x[1] + m[6] * x[3];
        break;
    case 3:
        y[0] = m[0] * x[0] - m[3] * x[3];
        y[1] = m[0] * x[1] + m[3] * x[2];
        y[2] = m[6] * x[2] - m[5] * x[1];
        y[3] = m[6] * x[3] + m[5] * x[0];
        break;
    default:
        y[0] = m[0] * x[0] - m[1] * x[1] + m[2] * x[2] - m[3] * x[3];
        y[1] = m[0] * x[1] + m[1] * x[0] + m[2] * x[3] + m[3] * x[2];
        y[2] = m[4] * x[0] - m[5] * x[1] + m[6] * x[2] - m[7] * x[3];
        y[3] = m[4] * x[1] + m[5] * x[0] + m[6] * x[3] + m[7] * x[2];
    }
}

// One run's steps on one amplitude pair: p = (psi0, psi1), l = (lambda0,
// lambda1) as (re, im, re, im), in place; acc: the run's parameter sums.
__device__ __forceinline__ void adj_run_steps(const AdjRun &g, double *p, double *l, double *acc) {
#pragma unroll
    for (int k = 0; k < kRunMax; ++k) {
        if (k >= g.n) break;
        double nv[4], xv[4];
        cmv2(g.ut[k], g.u[k], p, nv);  // psi' = U^dag psi
        for (int j = g.first[k]; j < g.first[k + 1]; ++j) {
            double mv[4];
            cmv2(g.dt[j], g.du[j], nv, mv);
            acc[j] += l[0] * mv[0] + l[1] * mv[1] + l[2] * mv[2] + l[3] * mv[3];  // Re(conj(lambda) mu)
        }
        cmv2(g.ut[k], g.u[k], l, xv);  // lambda' = U^dag lambda
        p[0] = nv[0], p[1] = nv[1], p[2] = nv[2], p[3] = nv[3];
        l[0] = xv[0], l[1] = xv[1], l[2] = xv[2], l[3] = xv[3];
    }
}

template <typename T>
__global__ void __launch_bounds__(256, kRunMinBlocks) adj_run_kernel(typename Vec2<T>::type *__restrict__ psi,
                                                      typename Vec2<T>::type *__restrict__ lam, uint64_t ngroups,
                                                      const AdjRun g, double *__restrict__ part, int pb) {
    __shared__ double sacc[256 * kRunMax];  // per-thread gradient sums (indexed at run time)
    double *acc = sacc + threadIdx.x * kRunMax;
#pragma unroll
    for (int j = 0; j < kRunMax; ++j) acc[j] = 0.0;
    for (uint64_t gi = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; gi < ngroups;
         gi += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t b0 = insert_zero(gi, g.t0);
        if ((b0 & g.cmask) != g.cmask) continue;
        const uint64_t b1 = b0 | (1ull << g.t0);
        const auto a0 = psi[b0], a1 = psi[b1], c0 = lam[b0], c1 = lam[b1];
        double p[4] = {a0.x, a0.y, a1.x, a1.y}, l[4] = {c0.x, c0.y, c1.x, c1.y};
        adj_run_steps(g, p, l, acc);
        const double p0r = p[0], p0i = p[1], p1r = p[2], p1i = p[3];
        const double l0r = l[0], l0i = l[1], l1r = l[2], l1i = l[3];
        typename Vec2<T>::type v;
        v.x = static_cast<T>(p0r), v.y = static_cast<T>(p0i);
        psi[b0] = v;
        v.x = static_cast<T>(p1r), v.y = static_cast<T>(p1i);
        psi[b1] = v;
        v.x = static_cast<T>(l0r), v.y = static_cast<T>(l0i);
        lam[b0] = v;
        v.x = static_cast<T>(l1r), v.y = static_cast<T>(l1i);
        lam[b1] = v;
    }
    __syncthreads();
    if (threadIdx.x < g.nacc) {
        double t = 0.0;
        for (int i = 0; i < static_cast<int>(blockDim.x); ++i) t += sacc[i * kRunMax + threadIdx.x];
        part[static_cast<size_t>(g.accslot[threadIdx.x]) * pb + blockIdx.x] = 2.0 * t;
    }
}

// Runs on up to 3 different wires, consecutive in the sweep and without
// controls (cfg1: the rx, ry, rz runs of neighbouring wires in a layer): the
// thread holds the 2^W amplitudes spanned by the W wires for psi and lambda
// and applies run 0 on local bit 0 (its wire), then run 1 on local bit 1,
// ... -- the sweep order -- so W runs cost one state round trip. Gradient
// sums per thread in shared memory (registers go to the 4 W amplitudes).
constexpr int kRunsMax = 3;
struct AdjRuns {
    int w = 0;
    int sorted[kRunsMax];  // the wires' bits, ascending (index insertion order)
    AdjRun r[kRunsMax];    // sweep order; run k acts on local bit k
};

template <typename T, int W>
__global__ void __launch_bounds__(256, 2) adj_runs_kernel(typename Vec2<T>::type *__restrict__ psi,
                                                          typename Vec2<T>::type *__restrict__ lam, uint64_t ngroups,
                                                          const AdjRuns g, double *__restrict__ part, int pb) {
    constexpr int A = 1 << W, S = W * kRunMax;
    __shared__ double sacc[256 * S];
    double *acc = sacc + threadIdx.x * S;
#pragma unroll
    for (int j = 0; j < S; ++j) acc[j] = 0.0;
    uint64_t off[A];
#pragma unroll
    for (int j = 0; j < A; ++j) {
        off[j] = 0;
#pragma unroll
        for (int k = 0; k < W; ++k)
            if ((j >> k) & 1) off[j] |= 1ull << g.r[k].t0;
    }
    for (uint64_t gi = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; gi < ngroups;
         gi += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t base = gi;
#pragma unroll
        for (int k = 0; k < W; ++k) base = insert_zero(base, g.sorted[k]);
        double p[A][2], l[A][2];
#pragma unroll
        for (int j = 0; j < A; ++j) {
            const auto a = psi[base | off[j]];
            const auto b = lam[base | off[j]];
            p[j][0] = a.x, p[j][1] = a.y, l[j][0] = b.x, l[j][1] = b.y;
        }
#pragma unroll
        for (int r = 0; r < W; ++r) {
            const AdjRun &rr = g.r[r];
            for (int k = 0; k < rr.n; ++k) {  // the run's gates in sweep order, every pair along local bit r
                const double *u = rr.u[k];
                const int ut = rr.ut[k];
#pragma unroll
                for (int j0 = 0; j0 < A; ++j0) {
                    if ((j0 >> r) & 1) continue;
                    const int j1 = j0 | (1 << r);
                    const double pp[4] = {p[j0][0], p[j0][1], p[j1][0], p[j1][1]};
                    const double ll[4] = {l[j0][0], l[j0][1], l[j1][0], l[j1][1]};
                    double nv[4], xv[4];
                    cmv2(ut, u, pp, nv);
                    for (int j = rr.first[k]; j < rr.first[k + 1]; ++j) {
                        double mv[4];
                        cmv2(rr.dt[j], rr.du[j], nv, mv);
                        acc[r * kRunMax + j] += ll[0] * mv[0] + ll[1] * mv[1] + ll[2] * mv[2] + ll[3] * mv[3];
                    }
                    cmv2(ut, u, ll, xv);
                    p[j0][0] = nv[0], p[j0][1] = nv[1], p[j1][0] = nv[2], p[j1][1] = nv[3];
                    l[j0][0] = xv[0], l[j0][1] = xv[1], l[j1][0] = xv[2], l[j1][1] = xv[3];
                }
            }
        }
#pragma unroll
        for (int j = 0; j < A; ++j) {
            typename Vec2<T>::type a, b;
            a.x = static_cast<T>(p[j][0]), a.y = static_cast<T>(p[j][1]);
            b.x = static_cast<T>(l[j][0]), b.y = static_cast<T>(l[j][1]);
            psi[base | off[j]] = a;
            lam[base | off[j]] = b;
        }
    }
    __syncthreads();
    if (threadIdx.x < S) {
        const int r = threadIdx.x / kRunMax, j = threadIdx.x % kRunMax;
        if (j < g.r[r].nacc) {
            double t = 0.0;
            for (int i = 0; i < static_cast<int>(blockDim.x); ++i) t += sacc[i * S + threadIdx.x];
            part[static_cast<size_t>(g.r[r].accslot[j]) * pb + blockIdx.x] = 2.0 * t;
        }
    }
}

// Gradient slot q = sum of its launch's per-block partials part[q * pb + b]
// (the other entries stay zero): a fixed-order sum, no atomics contending on
// one slot while the sweep runs.
__global__ void __launch_bounds__(256) partial_sum_kernel(const double *__restrict__ part, int pb,
                                                          double *__restrict__ grads) {
    double s = 0.0;
    for (int b = threadIdx.x; b < pb; b += blockDim.x) s += part[static_cast<size_t>(blockIdx.x) * pb + b];
    __shared__ double red[8];
    s = dev::warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
        grads[blockIdx.x] = t;
    }
}

// lambda = sum_obs O psi (adjoint.hpp:30-45): each observable's Paulis are
// applied wire by wire in order, so lambda_i walks them back from i: the row
// of the last-applied Pauli first. Entries: (bit, letter) runs per
// observable, `first[o]` .. `first[o + 1]`.
template <typename T>
__global__ void pauli_sum_kernel(const typename Vec2<T>::type *__restrict__ psi, typename Vec2<T>::type *__restrict__ lam,
                                 uint64_t n, int nobs, const int *__restrict__ first, const int *__restrict__ bit,
                                 const char *__restrict__ letter) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        double sr = 0.0, si = 0.0;
        for (int o = 0; o < nobs; ++o) {
            uint64_t j = i;
            double cr = 1.0, ci = 0.0;  // coefficient: (P_m ... P_1 psi)_i = c psi_j
            for (int e = first[o + 1] - 1; e >= first[o]; --e) {
                const uint64_t m = 1ull << bit[e];
                const int r = (j & m) ? 1 : 0;
                double er, ei;  // P[r][c], c = the one nonzero column of row r
                if (letter[e] == 'z') {
                    er = r ? -1.0 : 1.0, ei = 0.0;
                } else {
                    j ^= m;
                    if (letter[e] == 'x') er = 1.0, ei = 0.0;
                    else er = 0.0, ei = r ? 1.0 : -1.0;  // Y = [[0, -i], [i, 0]]
                }
                const double tr = cr * er - ci * ei, ti = cr * ei + ci * er;
                cr = tr, ci = ti;
            }
            const auto a = psi[j];
            sr += cr * a.x - ci * a.y;
            si += cr * a.y + ci * a.x;
        }
        typename Vec2<T>::type out;
        out.x = static_cast<T>(sr), out.y = static_cast<T>(si);
        lam[i] = out;
    }
}

GateRec pauli_rec(char c, int wire) {
    GateRec g;
    g.k = 1;
    g.wires[0] = wire;
    for (auto &x : g.m) x = 0;
    if (c == 'x') g.m[1] = g.m[2] = 1, g.kind = GK_X;
    else if (c == 'y') g.m[1] = cplx(0, -1), g.m[2] = cplx(0, 1), g.kind = GK_Y;
    else g.m[0] = 1, g.m[3] = -1, g.kind = GK_Z, g.diag = true;
    g.name = std::string(1, c);
    return g;
}

// gate_dmatrix (gate.hpp:157-190): d(matrix)/d(params[which]); returns k.
int dmatrix(const qsv_gate &g, int which, cplx *m) {
    const std::string name(g.name, strnlen(g.name, sizeof(g.name)));
    const double *p = g.params;
    for (int i = 0; i < 16; ++i) m[i] = 0;
    auto drot = [&](const cplx *G, int d, double th) {
        for (int r = 0; r < d; ++r)
            for (int c = 0; c < d; ++c)
                m[r * d + c] = (r == c ? cplx(-0.5 * std::sin(th / 2), 0) : cplx(0, 0)) -
                               cplx(0, 0.5) * std::cos(th / 2) * G[r * d + c];
    };
    static const cplx X[4] = {0, 1, 1, 0}, Y[4] = {0, cplx(0, -1), cplx(0, 1), 0}, Z[4] = {1, 0, 0, -1};
    auto kron = [](const cplx *a, const cplx *b, cplx *o) {
        for (int i = 0; i < 2; ++i)
            for (int j = 0; j < 2; ++j)
                for (int k = 0; k < 2; ++k)
                    for (int l = 0; l < 2; ++l) o[(i * 2 + k) * 4 + (j * 2 + l)] = a[i * 2 + j] * b[k * 2 + l];
    };
    if (name == "rx") return drot(X, 2, p[0]), 1;
    if (name == "ry") return drot(Y, 2, p[0]), 1;
    if (name == "rz") return drot(Z, 2, p[0]), 1;
    if (name == "rxx" || name == "ryy" || name == "rzz") {
        cplx G[16];
        const cplx *P = name[1] == 'x' ? X : name[1] == 'y' ? Y : Z;
        kron(P, P, G);
        drot(G, 4, p[0]);
        return 2;
    }
    if (name == "p") {
        m[3] = cplx(0, 1) * std::exp(cplx(0, p[0]));
        return 1;
    }
    if (name == "u3") {
        const double c = std::cos(p[0] / 2), s = std::sin(p[0] / 2);
        const cplx el = std::exp(cplx(0, p[2])), ef = std::exp(cplx(0, p[1]));
        if (which == 0) m[0] = -0.5 * s, m[1] = -0.5 * el * c, m[2] = 0.5 * ef * c, m[3] = -0.5 * ef * el * s;
        else if (which == 1) m[2] = cplx(0, 1) * ef * s, m[3] = cplx(0, 1) * ef * el * c;
        else m[1] = -cplx(0, 1) * el * s, m[3] = cplx(0, 1) * ef * el * c;
        return 1;
    }
    fail(QSV_ERR_INVALID, "gate " + name + " has no parameter derivative");
}

GateRec with_matrix(const GateRec &base, const cplx *m, int flags) {
    GateRec g = base;
    const int d = 1 << g.k;
    bool diag = true;
    for (int i = 0; i < d * d; ++i) {
        g.m[i] = m[i];
        if (i / d != i % d && m[i] != cplx(0, 0)) diag = false;
    }
    g.diag = diag;
    g.encoded = false;
    g.flags = flags;
    return g;
}

void fused_sweep(Ctx *ctx, int n, int dtype, const std::vector<qsv_gate> &bound, const std::vector<GateRec> &recs,
                 const std::vector<int> &pbase, const std::vector<int> &dbase, int nparams, int nobs,
                 const qsv_obs *obs, DState &psi, DState &lam, std::vector<double> &pg, std::vector<double> &dg) {
    cudaStream_t s = ctx->stream;
    const uint64_t N = psi.st.local_amps;
    const std::vector<int> &perm = psi.st.perm;  // wire -> physical bit after the forward plan
    const int blocks_all = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((N + 255) / 256, ctx->sm_count * 8)));
    // lambda
    std::vector<int> first(1, 0), bit;
    std::vector<char> letter;
    for (int o = 0; o < nobs; ++o) {
        require(obs[o].nwires >= 0 && (obs[o].nwires == 0 || (obs[o].wires && obs[o].basis)), "observable: bad wires");
        for (int j = 0; j < obs[o].nwires; ++j) {
            const char c = obs[o].basis[j];
            require(c == 'x' || c == 'y' || c == 'z', "observable: basis letter outside {x,y,z}");
            const int w = obs[o].wires[j];
            require(w >= 0 && w < n, "observable: wire out of range");
            bit.push_back(perm[w]);
            letter.push_back(c);
        }
        first.push_back(static_cast<int>(bit.size()));
    }
    const size_t tb = sizeof(int) * (first.size() + bit.size()) + letter.size() + 16;
    char *dtab = nullptr;
    QSV_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&dtab), tb, s));
    int *d_first = reinterpret_cast<int *>(dtab), *d_bit = d_first + first.size();
    char *d_letter = reinterpret_cast<char *>(d_bit + bit.size());
    QSV_CUDA(cudaMemcpyAsync(d_first, first.data(), sizeof(int) * first.size(), cudaMemcpyHostToDevice, s));
    if (!bit.empty()) {
        QSV_CUDA(cudaMemcpyAsync(d_bit, bit.data(), sizeof(int) * bit.size(), cudaMemcpyHostToDevice, s));
        QSV_CUDA(cudaMemcpyAsync(d_letter, letter.data(), letter.size(), cudaMemcpyHostToDevice, s));
    }
    if (dtype == QSV_C64)
        pauli_sum_kernel<float><<<blocks_all, 256, 0, s>>>(static_cast<const float2 *>(psi.st.d),
                                                           static_cast<float2 *>(lam.st.d), N, nobs, d_first, d_bit,
                                                           d_letter);
    else
        pauli_sum_kernel<double><<<blocks_all, 256, 0, s>>>(static_cast<const double2 *>(psi.st.d),
                                                            static_cast<double2 *>(lam.st.d), N, nobs, d_first, d_bit,
                                                            d_letter);
    QSV_CUDA(cudaGetLastError());
    // gradient slots: params, then data slots
    const int nslots = static_cast<int>(dg.size());
    const int ngrad = std::max(1, nparams + nslots);
    double *d_grad = nullptr;
    QSV_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&d_grad), sizeof(double) * ngrad, s));
    QSV_CUDA(cudaMemsetAsync(d_grad, 0, sizeof(double) * ngrad, s));
    static const int bps = [] {  // gradient launches: blocks per SM (QSV_ADJ_BLOCKS_PER_SM)
        const char *e = std::getenv("QSV_ADJ_BLOCKS_PER_SM");
        return e ? std::max(1, std::min(8, std::atoi(e))) : kRunMinBlocks;
    }();
    // per-block gradient partials: [slot][block], zero where a launch had
    // fewer blocks; summed once after the sweep
    const int pb = ctx->sm_count * 8;
    double *d_part = nullptr;
    QSV_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&d_part), sizeof(double) * ngrad * pb, s));
    QSV_CUDA(cudaMemsetAsync(d_part, 0, sizeof(double) * ngrad * pb, s));
    static const bool no_runs = [] {  // QSV_ADJ_NO_RUNS=1: one kernel per gate (A/B)
        const char *e = std::getenv("QSV_ADJ_NO_RUNS");
        return e && e[0] == '1';
    }();
    static const int max_wires = [] {  // QSV_ADJ_RUN_WIRES=2|3: wires per multi-run kernel (A/B)
        const char *e = std::getenv("QSV_ADJ_RUN_WIRES");
        return e ? std::max(2, std::min(kRunsMax, std::atoi(e))) : kRunsMax;
    }();
    static const bool no_multi = [] {  // QSV_ADJ_NO_MULTI=1: one kernel per run (A/B)
        const char *e = std::getenv("QSV_ADJ_NO_MULTI");
        return e && e[0] == '1';
    }();
    auto nparams_of = [&](int x) { return pbase[x] >= 0 || dbase[x] >= 0 ? bound[x].nparams : 0; };
    auto cmask_of = [&](int x) {
        uint64_t m = 0;
        for (int c : recs[x].ctls) m |= 1ull << perm[c];
        return m;
    };
    for (int i = static_cast<int>(recs.size()) - 1; i >= 0; --i) {
        const GateRec &g = recs[i];
        require(g.k >= 1 && g.k <= 2, "adjoint_gradients: gates act on 1 or 2 targets");
        if (g.k == 1 && !no_runs && nparams_of(i) <= 3) {  // a run of single-qubit gates on this wire
            // the run of gates i, i-1, ..., j on gate i's wire and control mask
            auto extent = [&](int top) {
                const int t0 = perm[recs[top].wires[0]];
                const uint64_t cm = cmask_of(top);
                int j = top, np = nparams_of(top);
                while (j > 0 && top - j + 1 < kRunMax && recs[j - 1].k == 1 && perm[recs[j - 1].wires[0]] == t0 &&
                       cmask_of(j - 1) == cm && nparams_of(j - 1) <= 3 && np + nparams_of(j - 1) <= kRunMax) {
                    --j;
                    np += nparams_of(j);
                }
                return j;
            };
            auto make_run = [&](int top, int j) {
                AdjRun r;
                r.t0 = perm[recs[top].wires[0]];
                r.cmask = cmask_of(top);
                r.n = top - j + 1;
                int acc = 0;
                for (int k = 0; k < r.n; ++k) {
                    const int x = top - k;  // sweep order
                    const GateRec &h = recs[x];
                    for (int rr = 0; rr < 2; ++rr)
                        for (int c = 0; c < 2; ++c) {
                            const cplx v = std::conj(h.m[c * 2 + rr]);
                            r.u[k][2 * (rr * 2 + c)] = v.real();
                            r.u[k][2 * (rr * 2 + c) + 1] = v.imag();
                        }
                    r.first[k] = acc;
                    const int base = pbase[x] >= 0 ? pbase[x] : dbase[x] >= 0 ? nparams + dbase[x] : -1;
                    for (int q = 0; q < nparams_of(x); ++q) {
                        cplx dm[16];
                        dmatrix(bound[x], q, dm);
                        for (int e = 0; e < 4; ++e) r.du[acc][2 * e] = dm[e].real(), r.du[acc][2 * e + 1] = dm[e].imag();
                        r.accslot[acc++] = base + q;
                    }
                }
                r.first[r.n] = acc;
                r.nacc = acc;
                for (int k = 0; k < r.n; ++k) r.ut[k] = mat_class(r.u[k]);
                for (int q = 0; q < acc; ++q) r.dt[q] = mat_class(r.du[q]);
                return r;
            };
            // consecutive uncontrolled runs on different wires: one kernel for up to 3
            if (!no_multi && cmask_of(i) == 0) {
                AdjRuns rs;
                int top = i;
                while (rs.w < max_wires && top >= 0 && recs[top].k == 1 && cmask_of(top) == 0 && nparams_of(top) <= 3) {
                    const int t0 = perm[recs[top].wires[0]];
                    bool dup = false;
                    for (int k = 0; k < rs.w; ++k) dup = dup || rs.r[k].t0 == t0;
                    if (dup) break;
                    const int j = extent(top);
                    rs.r[rs.w++] = make_run(top, j);
                    top = j - 1;
                }
                if (rs.w >= 2) {
                    for (int k = 0; k < rs.w; ++k) rs.sorted[k] = rs.r[k].t0;
                    std::sort(rs.sorted, rs.sorted + rs.w);
                    const uint64_t groups = N >> rs.w;
                    const int blocks = static_cast<int>(
                        std::max<uint64_t>(1, std::min<uint64_t>((groups + 255) / 256, ctx->sm_count * 2)));
                    auto *P64 = static_cast<float2 *>(psi.st.d);
                    auto *L64 = static_cast<float2 *>(lam.st.d);
                    auto *P128 = static_cast<double2 *>(psi.st.d);
                    auto *L128 = static_cast<double2 *>(lam.st.d);
                    if (dtype == QSV_C64) {
                        if (rs.w == 2) adj_runs_kernel<float, 2><<<blocks, 256, 0, s>>>(P64, L64, groups, rs, d_part, pb);
                        else adj_runs_kernel<float, 3><<<blocks, 256, 0, s>>>(P64, L64, groups, rs, d_part, pb);
                    } else {
                        if (rs.w == 2) adj_runs_kernel<double, 2><<<blocks, 256, 0, s>>>(P128, L128, groups, rs, d_part, pb);
                        else adj_runs_kernel<double, 3><<<blocks, 256, 0, s>>>(P128, L128, groups, rs, d_part, pb);
                    }
                    QSV_CUDA(cudaGetLastError());
                    i = top + 1;  // the loop's --i continues below the runs
                    continue;
                }
            }
            const int j = extent(i);
            if (j < i) {
                AdjRun r = make_run(i, j);
                const int acc = r.nacc;
                const uint64_t groups = N >> 1;
                const int blocks = static_cast<int>(std::max<uint64_t>(
                    1, std::min<uint64_t>((groups + 255) / 256, ctx->sm_count * (acc ? bps : 8))));
                if (dtype == QSV_C64)
                    adj_run_kernel<float><<<blocks, 256, 0, s>>>(static_cast<float2 *>(psi.st.d),
                                                                 static_cast<float2 *>(lam.st.d), groups, r, d_part, pb);
                else
                    adj_run_kernel<double><<<blocks, 256, 0, s>>>(static_cast<double2 *>(psi.st.d),
                                                                  static_cast<double2 *>(lam.st.d), groups, r, d_part, pb);
                QSV_CUDA(cudaGetLastError());
                i = j;  // the loop's --i continues below the run
                continue;
            }
        }
        const int d = 1 << g.k;
        AdjGate a;
        a.k = g.k;
        a.t0 = perm[g.wires[0]];
        a.t1 = g.k == 2 ? perm[g.wires[1]] : 0;
        a.cmask = 0;
        for (int c : g.ctls) a.cmask |= 1ull << perm[c];
        for (int r = 0; r < d; ++r)
            for (int c = 0; c < d; ++c) {
                const cplx v = std::conj(g.m[c * d + r]);
                a.u[2 * (r * d + c)] = v.real();
                a.u[2 * (r * d + c) + 1] = v.imag();
            }
        a.nq = 0;
        if (pbase[i] >= 0 || dbase[i] >= 0) {
            a.nq = bound[i].nparams;
            require(a.nq <= 3, "adjoint_gradients: at most 3 parameters per gate");
            a.slot = pbase[i] >= 0 ? pbase[i] : nparams + dbase[i];
            for (int q = 0; q < a.nq; ++q) {
                cplx dm[16];
                dmatrix(bound[i], q, dm);
                for (int e = 0; e < d * d; ++e) a.du[q][2 * e] = dm[e].real(), a.du[q][2 * e + 1] = dm[e].imag();
            }
        }
        const uint64_t groups = N >> g.k;
        // gradient gates: fewer, fuller blocks (one atomic per block and
        // parameter lands on the same slot); QSV_ADJ_BLOCKS_PER_SM overrides
        const int blocks = static_cast<int>(
            std::max<uint64_t>(1, std::min<uint64_t>((groups + 255) / 256, ctx->sm_count * (a.nq ? bps : 8))));
        if (dtype == QSV_C64) {
            auto *P = static_cast<float2 *>(psi.st.d);
            auto *Lm = static_cast<float2 *>(lam.st.d);
            if (g.k == 1) (a.nq ? adj_gate_kernel<float, 1, true> : adj_gate_kernel<float, 1, false>)<<<blocks, 256, 0, s>>>(P, Lm, groups, a, d_part, pb);
            else (a.nq ? adj_gate_kernel<float, 2, true> : adj_gate_kernel<float, 2, false>)<<<blocks, 256, 0, s>>>(P, Lm, groups, a, d_part, pb);
        } else {
            auto *P = static_cast<double2 *>(psi.st.d);
            auto *Lm = static_cast<double2 *>(lam.st.d);
            if (g.k == 1) (a.nq ? adj_gate_kernel<double, 1, true> : adj_gate_kernel<double, 1, false>)<<<blocks, 256, 0, s>>>(P, Lm, groups, a, d_part, pb);
            else (a.nq ? adj_gate_kernel<double, 2, true> : adj_gate_kernel<double, 2, false>)<<<blocks, 256, 0, s>>>(P, Lm, groups, a, d_part, pb);
        }
        QSV_CUDA(cudaGetLastError());
    }
    if (nparams + nslots > 0) {
        partial_sum_kernel<<<nparams + nslots, 256, 0, s>>>(d_part, pb, d_grad);
        QSV_CUDA(cudaGetLastError());
    }
    std::vector<double> h(ngrad);
    QSV_CUDA(cudaMemcpyAsync(h.data(), d_grad, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s));
    QSV_CUDA(cudaFreeAsync(d_part, s));
    QSV_CUDA(cudaFreeAsync(d_grad, s));
    QSV_CUDA(cudaFreeAsync(dtab, s));
    QSV_CUDA(cudaStreamSynchronize(s));
    for (int q = 0; q < nparams; ++q) pg[q] = h[q];
    for (int q = 0; q < nslots; ++q) dg[q] = h[nparams + q];
}

} // namespace

void adjoint_gradients(Ctx *ctx, int n, int dtype, const qsv_gate *gates, int ngates, int nobs, const qsv_obs *obs,
                       const double *init, const double *data, int slots, std::vector<double> &pg,
                       std::vector<double> &dg) {
    require(ngates >= 0 && (ngates == 0 || gates), "adjoint_gradients: bad gate list");
    require(nobs >= 0 && (nobs == 0 || obs), "adjoint_gradients: bad observables");
    // bind (adjoint.hpp:70-82)
    int enc_slots = 0;
    for (int i = 0; i < ngates; ++i)
        if (gates[i].encode) enc_slots += gates[i].nparams;
    require(slots == enc_slots, "adjoint_gradients: data length != encode slots"); // adjoint.hpp:61-62
    std::vector<qsv_gate> bound(gates, gates + ngates);
    std::vector<int> pbase(ngates, -1), dbase(ngates, -1);
    int nparams = 0, nslots = 0, cursor = 0;
    for (int i = 0; i < ngates; ++i) {
        qsv_gate &g = bound[i];
        if (g.encode) {
            dbase[i] = nslots;
            for (int q = 0; q < g.nparams; ++q) g.params[q] = data[cursor++];
            nslots += g.nparams;
        } else if (g.trainable) {
            pbase[i] = nparams;
            nparams += g.nparams;
        }
        g.encode = 0;
    }
    std::vector<GateRec> recs;
    for (int i = 0; i < ngates; ++i) {
        int cur = 0;
        recs.push_back(resolve_gate(bound[i], n, &cur));
    }
    cudaStream_t s = ctx->stream;
    DState psi(ctx, n, dtype), lam(ctx, n, dtype);
    // init (QubitState::basis(n) by default, adjoint.hpp:84)
    if (init) {
        const uint64_t la = psi.st.local_amps;
        if (dtype == QSV_C128)
            QSV_CUDA(cudaMemcpyAsync(psi.st.d, init, la * 16, cudaMemcpyHostToDevice, s));
        else {
            std::vector<float> f(2 * la);
            for (uint64_t i = 0; i < 2 * la; ++i) f[i] = static_cast<float>(init[i]);
            QSV_CUDA(cudaMemcpyAsync(psi.st.d, f.data(), la * 8, cudaMemcpyHostToDevice, s));
            QSV_CUDA(cudaStreamSynchronize(s));
        }
    } else {
        launch_set_basis(psi.st, 0, ctx->rank == 0);
    }
    // forward sweep, fused. The trainable and data-bound values are
    // compile-time constants the first time this circuit structure is met;
    // once it comes back with other values (a training loop) they enter as
    // run-time parameters bound on the device (lift_policy), so new values
    // reuse the compiled passes instead of an NVRTC compile per call
    {
        auto variable = [&](int i) {
            return (pbase[i] >= 0 || dbase[i] >= 0) && bound[i].nparams > 0 &&
                   std::strncmp(bound[i].name, "custom", sizeof(bound[i].name)) != 0;
        };
        bool lift = false;
        std::string sk("adjoint"), vk;
        {
            auto put = [](std::string &k, const void *p, size_t b) { k.append(static_cast<const char *>(p), b); };
            put(sk, &n, sizeof(int));
            put(sk, &dtype, sizeof(int));
            bool any = false;
            for (int i = 0; i < ngates; ++i) {
                const qsv_gate &g = gates[i];
                put(sk, g.name, sizeof(g.name));
                put(sk, &g.nwires, sizeof(g.nwires) + sizeof(g.wires) + sizeof(g.ncontrols) + sizeof(g.controls) +
                                       sizeof(g.nparams));
                put(sk, &g.trainable, sizeof(g.trainable) + sizeof(g.encode));
                if (variable(i)) {
                    any = true;
                    put(vk, bound[i].params, sizeof(double) * bound[i].nparams);
                } else {
                    put(sk, g.params, sizeof(double) * std::min(3, std::max(0, static_cast<int>(g.nparams))));
                }
                if (g.custom) {
                    const int k = std::max(1, std::min(2, static_cast<int>(g.nwires)));
                    put(sk, g.custom, sizeof(double) * 2 * (1u << (2 * k)));
                }
            }
            static const bool nolift = [] {
                const char *e = std::getenv("QSV_NO_LIFT");
                return e && e[0] == '1';
            }();
            lift = any && !nolift && lift_policy(*ctx, sk, vk);
        }
        std::vector<GateRec> fwd;
        std::vector<double> vals;
        int cur = 0;
        for (int i = 0; i < ngates; ++i) {
            qsv_gate g = bound[i];
            if (lift && variable(i)) {
                g.encode = 1;
                for (int q = 0; q < g.nparams; ++q) vals.push_back(g.params[q]);
            }
            fwd.push_back(resolve_gate(g, n, &cur));
        }
        // forward plans kept per context: a device-bound plan by structure
        // (it does not depend on the values), a constant one by structure
        // and values (planning 600+ gates costs more than the 20q sweep)
        const std::string key = lift ? sk : sk + std::string(1, '\1') + vk;
        std::shared_ptr<Plan> fw;
        {
            std::lock_guard<std::mutex> lk(ctx->lift_seen->mu);
            for (auto &e : ctx->adj_plans)
                if (e.first == key) fw = e.second;
        }
        if (!fw) {
            fw = std::make_shared<Plan>();
            build_plan(*fw, ctx, n, dtype, std::move(fwd), cur, nullptr);
            std::lock_guard<std::mutex> lk(ctx->lift_seen->mu);
            if (ctx->adj_plans.size() >= 4) ctx->adj_plans.erase(ctx->adj_plans.begin());
            ctx->adj_plans.emplace_back(key, fw);
        }
        execute_plan(*fw, psi.st, cur ? vals.data() : nullptr, cur ? 1 : 0, cur);
    }
    pg.assign(nparams, 0.0);
    dg.assign(nslots, 0.0);
    if (ctx->world == 1) {
        fused_sweep(ctx, n, dtype, bound, recs, pbase, dbase, nparams, nobs, obs, psi, lam, pg, dg);
        return;
    }
    // multi-rank: the reference's sequence of whole-state operations, every
    // gate through a one-gate plan (global wires take the swap path)
    DState mu(ctx, n, dtype);
    // lambda = sum_obs O psi (adjoint.hpp:30-45)
    QSV_CUDA(cudaMemsetAsync(lam.st.d, 0, lam.bytes(), s));
    for (int o = 0; o < nobs; ++o) {
        copy_state(mu, psi, s);
        require(obs[o].nwires >= 0 && (obs[o].nwires == 0 || (obs[o].wires && obs[o].basis)),
                "observable: bad wires");
        for (int j = 0; j < obs[o].nwires; ++j) {
            const char c = obs[o].basis[j];
            require(c == 'x' || c == 'y' || c == 'z', "observable: basis letter outside {x,y,z}");
            apply_rec(mu.st, pauli_rec(c, obs[o].wires[j]));
        }
        const uint64_t nn = lam.st.local_amps;
        const int blocks = static_cast<int>(std::min<uint64_t>((nn + 255) / 256, ctx->sm_count * 8));
        if (dtype == QSV_C64)
            axpy_kernel<float><<<std::max(blocks, 1), 256, 0, s>>>(static_cast<float2 *>(lam.st.d),
                                                                   static_cast<const float2 *>(mu.st.d), nn);
        else
            axpy_kernel<double><<<std::max(blocks, 1), 256, 0, s>>>(static_cast<double2 *>(lam.st.d),
                                                                    static_cast<const double2 *>(mu.st.d), nn);
        QSV_CUDA(cudaGetLastError());
    }
    // reverse sweep (adjoint.hpp:93-108)
    for (int i = ngates - 1; i >= 0; --i) {
        const GateRec &g = recs[i];
        const int d = 1 << g.k;
        cplx adj[16];
        for (int r = 0; r < d; ++r)
            for (int c = 0; c < d; ++c) adj[r * d + c] = std::conj(g.m[c * d + r]);
        const GateRec gdag = with_matrix(g, adj, 0);
        apply_rec(psi.st, gdag);
        if (pbase[i] >= 0 || dbase[i] >= 0) {
            for (int q = 0; q < bound[i].nparams; ++q) {
                copy_state(mu, psi, s);
                cplx dm[16];
                dmatrix(bound[i], q, dm);
                apply_rec(mu.st, with_matrix(g, dm, OPF_ZERO_OFF_CONTROL));
                const double grad = 2.0 * re_dot(lam, mu);
                if (pbase[i] >= 0) pg[pbase[i] + q] = grad;
                if (dbase[i] >= 0) dg[dbase[i] + q] = grad;
            }
        }
        apply_rec(lam.st, gdag);
    }
    QSV_CUDA(cudaStreamSynchronize(s));
}

} // namespace qsv
