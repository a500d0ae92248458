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
//     lambda <- U^dagger lambda.
// The derivative matrices restate gate_dmatrix (gate.hpp:157-190).
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
    DState psi(ctx, n, dtype), lam(ctx, n, dtype), mu(ctx, n, dtype);
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
    // forward sweep, fused
    {
        Plan fw;
        build_plan(fw, ctx, n, dtype, recs, 0, nullptr);
        execute_plan(fw, psi.st, nullptr, 0, 0);
    }
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
    pg.assign(nparams, 0.0);
    dg.assign(nslots, 0.0);
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
