// extern "C" entry points of include/qsv.h. Every call catches C++
// exceptions and maps them to the reference's status codes
// (tools/main.cpp:686-697): invalid_input -> 2, guard_error -> 3,
// transport_error -> 4, CUDA/internal -> 1. There is no CPU fallback: without
// a usable CUDA device every state/plan call fails with QSV_ERR_INTERNAL.
#include <algorithm>
#include <bit>
#include <cmath>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <string>
#include <thread>

#include "qsv_internal.hpp"

// A handle is either one rank's object or, on a context made by
// qsv_ctx_create_multi, a GROUP: one object per rank (`parts`, rank order),
// every call on it run by one host thread per rank (the reference's
// dist::run_on_ranks, tests/test_dist.cpp:66-94) with NCCL hidden inside.
// Plans of recent qsv_run_circuit calls (Circuit::forward through the ABI):
// a training loop calls forward with the same gates and new data every
// step; planning and kernel specialisation are done once per distinct
// (gates, n, dtype, opts) and the plan is re-executed.
struct PlanCache {
    static constexpr size_t kCap = 8;
    std::mutex mu;
    std::list<std::pair<std::string, std::unique_ptr<qsv::Plan>>> lru;  // most recent first
};
struct qsv_ctx : qsv::Ctx {
    std::vector<qsv_ctx *> parts;
    // independent single-GPU contexts on the same devices (row sharding of
    // batched circuits: no communicator, made on first use)
    std::vector<qsv_ctx *> solo;
    std::unique_ptr<PlanCache> plans = std::make_unique<PlanCache>();
    ~qsv_ctx();
};
struct qsv_state : qsv::State {
    std::vector<qsv_state *> parts;
    ~qsv_state() {
        for (qsv_state *x : parts) delete x;
    }
};
struct qsv_plan : qsv::Plan {
    std::vector<qsv_plan *> parts;
    ~qsv_plan() {
        for (qsv_plan *x : parts) delete x;
    }
};

qsv_ctx::~qsv_ctx() {
    if (parts.empty() && plans && !plans->lru.empty()) {
        cudaSetDevice(device);
        plans.reset();  // cached plans free their device buffers while the context lives
    }
    for (qsv_ctx *x : solo) delete x;
    // NCCL teardown may synchronise with the peers: every rank in its own thread
    std::vector<std::thread> th;
    for (qsv_ctx *x : parts)
        th.emplace_back([x] {
            cudaSetDevice(x->device);
            delete x;
        });
    for (auto &t : th) t.join();
}

namespace qsv {
void build_plan(Plan &p, Ctx *ctx, int n, int dtype, std::vector<GateRec> gates, int nslots, const qsv_opts *opts);
void build_plan_from_abi(Plan &p, Ctx *ctx, int n, int dtype, const qsv_gate *gates, int ngates,
                         const qsv_opts *opts);
void profile_plan(Plan &p, State &st, double *launch_ms);
int rng_fill(uint64_t seed, const char *label, int kind, uint64_t count, void *out, int nthreads, uint64_t offset);
void sample_counts(const double *probs, int k, int shots, uint64_t seed, const char *label, uint64_t *counter,
                   uint64_t *counts);
void adjoint_gradients(Ctx *ctx, int n, int dtype, const qsv_gate *gates, int ngates, int nobs, const qsv_obs *obs,
                       const double *init, const double *data, int slots, std::vector<double> &pg,
                       std::vector<double> &dg);
} // namespace qsv

using namespace qsv;

namespace {
thread_local std::string g_err;

template <typename F> int guard(F &&f) {
    try {
        f();
        return QSV_OK;
    } catch (const Error &e) {
        g_err = e.what();
        return e.code;
    } catch (const std::bad_alloc &) {
        g_err = "out of host memory";
        return QSV_ERR_INTERNAL;
    } catch (const std::exception &e) {
        g_err = e.what();
        return QSV_ERR_INTERNAL;
    }
}

// Runs f(r) (an ABI call on rank r's object, returning its status) for every
// rank of a group, one host thread per rank (collectives inside need every
// rank to arrive); the first failing rank's status and message are raised.
template <typename F> void on_ranks(const std::vector<qsv_ctx *> &ranks, F &&f) {
    const int P = static_cast<int>(ranks.size());
    std::vector<int> rc(P, 0);
    std::vector<std::string> msg(P);
    std::vector<std::thread> th;
    for (int r = 0; r < P; ++r)
        th.emplace_back([&, r] {
            cudaSetDevice(ranks[r]->device);
            rc[r] = f(r);
            if (rc[r]) msg[r] = g_err;
        });
    for (auto &t : th) t.join();
    for (int r = 0; r < P; ++r)
        if (rc[r]) fail(rc[r], "rank " + std::to_string(r) + ": " + msg[r]);
}
bool is_group(const qsv_ctx *c) { return c && !c->parts.empty(); }
bool is_group(const qsv_state *s) { return s && !s->parts.empty(); }
bool is_group(const qsv_plan *p) { return p && !p->parts.empty(); }
qsv_ctx *group_ctx(const qsv_state *s) { return static_cast<qsv_ctx *>(s->ctx); }

void init_ctx(Ctx &c, int device) {
    int ndev = 0;
    const cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        fail(QSV_ERR_INTERNAL, "qsv: no CUDA device available (the engine has no CPU fallback)");
    require(device >= 0 && device < ndev, "qsv: device index out of range");
    c.device = device;
    QSV_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    QSV_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) fail(QSV_ERR_INTERNAL, "qsv: built for sm_100a (B200); device is sm_" +
                                                    std::to_string(prop.major * 10 + prop.minor));
    c.sm_count = prop.multiProcessorCount;
    c.smem_optin = prop.sharedMemPerBlockOptin;
    QSV_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    // stream-ordered scratch (reductions, adjoint gradient partials): keep up
    // to 256 MiB in the device's pool across synchronisations instead of
    // unmapping and remapping it on every call
    cudaMemPool_t pool = nullptr;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = 256ull << 20;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    cudaGetLastError();
}

// Device staging owned for the scope of one transfer (freed on every path,
// after the stream has drained).
struct StageBuf {
    void *p = nullptr;
    cudaStream_t s;
    StageBuf(size_t bytes, cudaStream_t st) : s(st) { QSV_CUDA(cudaMalloc(&p, bytes)); }
    ~StageBuf() {
        cudaStreamSynchronize(s);
        cudaFree(p);
    }
};

// Chunked host(f64) -> device(dtype) transfer through a bounded staging buffer.
void upload_f64(State &st, void *dst, const double *host, uint64_t count) {
    cudaStream_t s = st.ctx->stream;
    if (st.dtype == QSV_C128) {
        QSV_CUDA(cudaMemcpyAsync(dst, host, count * 16, cudaMemcpyHostToDevice, s));
        QSV_CUDA(cudaStreamSynchronize(s));
        return;
    }
    const uint64_t chunk = std::min<uint64_t>(count, 1ull << 24); // 16 Mi amplitudes (256 MiB f64)
    StageBuf stage(chunk * 16, s);
    for (uint64_t off = 0; off < count; off += chunk) {
        const uint64_t c = std::min(chunk, count - off);
        QSV_CUDA(cudaMemcpyAsync(stage.p, host + 2 * off, c * 16, cudaMemcpyHostToDevice, s));
        launch_convert(static_cast<float *>(dst) + 2 * off, QSV_C64, stage.p, QSV_C128, 2 * c, s);
    }
    QSV_CUDA(cudaStreamSynchronize(s));
}

void download_f64(State &st, const void *src, double *host, uint64_t count) {
    cudaStream_t s = st.ctx->stream;
    if (st.dtype == QSV_C128) {
        QSV_CUDA(cudaMemcpyAsync(host, src, count * 16, cudaMemcpyDeviceToHost, s));
        QSV_CUDA(cudaStreamSynchronize(s));
        return;
    }
    const uint64_t chunk = std::min<uint64_t>(count, 1ull << 24);
    StageBuf stage(chunk * 16, s);
    for (uint64_t off = 0; off < count; off += chunk) {
        const uint64_t c = std::min(chunk, count - off);
        launch_convert(stage.p, QSV_C128, static_cast<const float *>(src) + 2 * off, QSV_C64, 2 * c, s);
        QSV_CUDA(cudaMemcpyAsync(host + 2 * off, stage.p, c * 16, cudaMemcpyDeviceToHost, s));
        QSV_CUDA(cudaStreamSynchronize(s));
    }
}

// Lazy layouts: a whole-state overwrite makes any layout canonical; a
// one-row upload into a batch first restores the other rows' layout.
void reset_layout(State &st) {
    for (int w = 0; w < st.n; ++w) st.perm[w] = st.n - 1 - w;
}
void upload_layout(State &st) {
    if (st.ctx->world != 1 || layout_canonical(st)) return;
    if (st.batch == 1) reset_layout(st);
    else normalize_layout(st);
}

void *row_ptr(State &st, int row) {
    require(row >= 0 && row < st.batch, "batch index out of range");
    return static_cast<unsigned char *>(st.d) + static_cast<size_t>(row) * st.local_amps * st.amp_bytes();
}

// One-gate plan, executed immediately (apply_gate / apply_matrix_strided).
// A single-qubit matrix on a global wire is the reference's pairwise
// exchange instead (one message per rank, test_dist.cpp:112-126): cheaper for
// one gate than a swap in and a swap back.
void run_single(State &st, const GateRec &g) {
    if (st.ctx->world > 1 && g.k == 1 && !g.diag && !g.encoded && st.perm[g.wires[0]] >= st.nlocal) {
        uint64_t lc = 0;
        bool on = true;
        for (int c : g.ctls) {
            const int pb = st.perm[c];
            if (pb < st.nlocal) lc |= 1ull << pb;
            else on = on && ((st.ctx->rank >> (pb - st.nlocal)) & 1);
        }
        QSV_CUDA(cudaSetDevice(st.ctx->device));
        dist_exchange_apply(st, st.perm[g.wires[0]], g.m, lc, on, (g.flags & OPF_ZERO_OFF_CONTROL) != 0);
        return;
    }
    if (apply_direct(st, g)) return;
    Plan p;
    build_plan(p, st.ctx, st.n, st.dtype, {g}, 0, nullptr);
    execute_plan(p, st, nullptr, 0, 0);
    QSV_CUDA(cudaStreamSynchronize(st.ctx->stream));
}

// Trainable gates as run-time parameters (Circuit::forward in a training
// loop: new angles every call). A copy of the gate list with every trainable
// parametric gate marked encoded, and data rows rewritten in slot order --
// the caller's encode values and the trainable parameters interleaved as the
// gates come, one row per state row. The pass kernels then do not depend on
// the trainable values (the bind kernel forms their matrices on the device),
// so new angles reuse the compiled passes and the plan cache entry instead
// of a code-generation + NVRTC compile per call.
struct Lifted {
    std::vector<qsv_gate> gates;
    std::vector<double> data;
    int rows = 0, slots = 0;
};
// Bytes of the parameters a gate uses (cache and policy keys: entries past
// nparams may hold anything a C caller left there).
size_t used_params(const qsv_gate &g) {
    return sizeof(double) * static_cast<size_t>(std::min(3, std::max(0, static_cast<int>(g.nparams))));
}
bool liftable(const qsv_gate &g) {
    return g.trainable && !g.encode && g.nparams > 0 && std::strncmp(g.name, "custom", sizeof(g.name)) != 0;
}
bool lift_trainable(const qsv_gate *gates, int ngates, int n, const double *data, int rows, int slots, int batch,
                    Lifted &out) {
    bool any = false;
    for (int i = 0; i < ngates; ++i) any = any || liftable(gates[i]);
    if (!any) return false;
    out.gates.assign(gates, gates + ngates);
    int user = 0, total = 0;
    for (qsv_gate &g : out.gates) {
        if (liftable(g)) {
            int scratch = 0;
            (void)resolve_gate(g, n, &scratch);  // the constant gate's own checks and messages
            g.encode = 1;
        }
        if (g.encode && g.nparams > 0) total += g.nparams;
    }
    for (int i = 0; i < ngates; ++i)
        if (gates[i].encode && gates[i].nparams > 0) user += gates[i].nparams;
    require(rows == 0 || slots == user, "data length " + std::to_string(slots) + " != encode slots " +
                                            std::to_string(user));  // circuit.hpp:134-136
    require(rows > 0 || user == 0, "circuit has encode slots but no data given");  // circuit.hpp:125
    out.rows = rows > 0 ? rows : batch;
    out.slots = total;
    out.data.resize(static_cast<size_t>(out.rows) * total);
    for (int r = 0; r < out.rows; ++r) {
        double *dst = out.data.data() + static_cast<size_t>(r) * total;
        const double *src = rows > 0 ? data + static_cast<size_t>(r) * slots : nullptr;
        for (int i = 0; i < ngates; ++i) {
            const qsv_gate &g = gates[i];
            if (g.encode && g.nparams > 0) {
                for (int q = 0; q < g.nparams; ++q) *dst++ = *src++;
            } else if (liftable(g)) {
                for (int q = 0; q < g.nparams; ++q) *dst++ = g.params[q];
            }
        }
    }
    return true;
}

// lift_policy's keys for a gate list: the structure (everything but the
// trainable values) and those values.
bool want_lift(Ctx &c, int n, int dtype, const qsv_opts *opts, const qsv_gate *gates, int ngates) {
    if ((opts && opts->dense_blocks > 0) || ngates <= 0 || !gates) return false;  // dense blocks: no encoded gates
    std::string sk, vk;
    auto put = [](std::string &k, const void *p, size_t b) { k.append(static_cast<const char *>(p), b); };
    put(sk, &n, sizeof(int));
    put(sk, &dtype, sizeof(int));
    if (opts) put(sk, opts, sizeof(qsv_opts));
    bool any = false;
    for (int i = 0; i < ngates; ++i) {
        const qsv_gate &g = gates[i];
        const bool l = liftable(g);
        any = any || l;
        put(sk, g.name, sizeof(g.name));
        put(sk, &g.nwires, sizeof(g.nwires) + sizeof(g.wires) + sizeof(g.ncontrols) + sizeof(g.controls) +
                               sizeof(g.nparams));
        put(sk, &g.trainable, sizeof(g.trainable) + sizeof(g.encode));
        if (l) put(vk, g.params, used_params(g));
        else if (!g.encode) put(sk, g.params, used_params(g));
        if (g.custom) {
            const int k = std::max(1, std::min(2, static_cast<int>(g.nwires)));
            put(sk, g.custom, sizeof(double) * 2 * (1u << (2 * k)));
        }
    }
    return any && lift_policy(c, sk, vk);
}

// A group's host view is the whole state: rank r takes amplitudes
// [r * 2^(n-g), (r + 1) * 2^(n-g)).
template <typename Ptr, typename F> void group_slices(qsv_state *st, Ptr host, uint64_t count, size_t elem, F &&f) {
    require(count == st->local_amps, "QubitState: amplitude length mismatch");
    const uint64_t per = st->parts[0]->local_amps;
    on_ranks(group_ctx(st)->parts, [&](int r) {
        return f(st->parts[r], reinterpret_cast<Ptr>(reinterpret_cast<uintptr_t>(host) + r * per * elem), per);
    });
}

// The context's plan for (n, dtype, options, gates), planned and specialised
// on first use: the key is everything build_plan reads -- n, dtype, the
// options and every gate field except the encoded parameters' values (bound
// per row at execute) and `trainable`; custom matrices by value. `lk` holds
// the cache (and so the plan) while the caller executes it.
Plan &cached_plan(qsv_ctx *c, int n, int dtype, const qsv_opts *opts, const qsv_gate *gates, int ngates,
                  std::unique_lock<std::mutex> &lk) {
    std::string key;
    auto put = [&](const void *p, size_t b) { key.append(static_cast<const char *>(p), b); };
    put(&n, sizeof(int));
    put(&dtype, sizeof(int));
    const int has_opts = opts != nullptr;
    put(&has_opts, sizeof(int));
    if (opts) put(opts, sizeof(qsv_opts));
    require(ngates >= 0 && (ngates == 0 || gates != nullptr), "plan: bad gate list");
    for (int i = 0; i < ngates; ++i) {
        const qsv_gate &g = gates[i];
        put(g.name, sizeof(g.name));
        put(&g.nwires, sizeof(g.nwires) + sizeof(g.wires) + sizeof(g.ncontrols) + sizeof(g.controls) +
                           sizeof(g.nparams));
        put(&g.encode, sizeof(g.encode));
        if (!g.encode) put(g.params, used_params(g));
        if (g.custom) {
            const int k = std::max(1, std::min(2, static_cast<int>(g.nwires)));
            put(g.custom, sizeof(double) * 2 * (1u << (2 * k)));
        }
    }
    lk = std::unique_lock<std::mutex>(c->plans->mu);
    auto &lru = c->plans->lru;
    auto it = std::find_if(lru.begin(), lru.end(), [&](const auto &e) { return e.first == key; });
    if (it == lru.end()) {
        auto np = std::make_unique<Plan>();
        build_plan_from_abi(*np, c, n, dtype, gates, ngates, opts);
        lru.emplace_front(std::move(key), std::move(np));
        if (lru.size() > PlanCache::kCap) lru.pop_back();
        it = lru.begin();
    } else if (it != lru.begin()) {
        lru.splice(lru.begin(), lru, it);
        it = lru.begin();
    }
    return *it->second;
}

// Batched circuit on one context: forward from |0...0> with the rows' encode
// data, then every <Z_w> per row (the fused epilogue when the pass holds a
// whole row); the plan and state are freed on every path.
void detail_run_rows(qsv_ctx *c, int n, int dtype, const qsv_gate *gates, int ngates, const double *data, int rows,
                     int slots, const qsv_opts *opts, double *out, qsv_plan **pp, qsv_state **ps) {
    struct Free {
        qsv_plan **p;
        qsv_state **s;
        ~Free() {
            if (*s) qsv_state_destroy(*s);
            if (*p) qsv_plan_destroy(*p);
        }
    } fr{pp, ps};
    qsv_opts o{};
    if (opts) o = *opts;
    else o.fuse = 1;
    o.from_zero = 1;
    auto chk = [](int rc) {
        if (rc) fail(rc, g_err);
    };
    static const bool nolift = [] {  // QSV_NO_LIFT=1: trainable values stay compile-time constants
        const char *e = std::getenv("QSV_NO_LIFT");
        return e && e[0] == '1';
    }();
    Lifted lf;  // a training loop's new shared angles: bound on the device
    if (!nolift && want_lift(*c, n, dtype, &o, gates, ngates) &&
        lift_trainable(gates, ngates, n, data, slots ? rows : 0, slots, rows, lf)) {
        gates = lf.gates.data();
        data = lf.data.data();
        slots = lf.slots;
    }
    (void)pp;
    chk(qsv_state_create(c, n, rows, dtype, ps));
    std::unique_lock<std::mutex> lk;
    Plan &plan = cached_plan(c, n, dtype, &o, gates, ngates, lk);  // a training loop re-plans once
    execute_plan_z(plan, **ps, slots ? data : nullptr, slots ? rows : 0, slots, out);
}

} // namespace

extern "C" {

const char *qsv_last_error(void) { return g_err.c_str(); }
int qsv_version(void) { return QSV_VERSION; }

int qsv_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int qsv_ctx_create(int device, qsv_ctx **out) {
    return guard([&] {
        require(out != nullptr, "qsv_ctx_create: null out");
        auto c = std::make_unique<qsv_ctx>();
        init_ctx(*c, device);
        *out = c.release();
    });
}

int qsv_nccl_unique_id(void *out128) {
    return guard([&] { nccl_unique_id(out128); });
}

int qsv_ctx_create_dist(int device, int rank, int world, const void *uid, qsv_ctx **out) {
    return guard([&] {
        require(out != nullptr, "qsv_ctx_create_dist: null out");
        require(world >= 1 && (world & (world - 1)) == 0, "world size must be a power of two"); // test_dist.cpp:90-94
        require(rank >= 0 && rank < world, "rank out of range");
        auto c = std::make_unique<qsv_ctx>();
        init_ctx(*c, device);
        c->rank = rank;
        c->world = world;
        c->gbits = std::countr_zero(static_cast<unsigned>(world));
        if (world > 1) nccl_init(*c, uid);
        *out = c.release();
    });
}

int qsv_ctx_create_multi(int ndev, const int *devices, qsv_ctx **out) {
    return guard([&] {
        require(out != nullptr && (ndev == 0 || devices != nullptr), "qsv_ctx_create_multi: null argument");
        require(ndev >= 1 && (ndev & (ndev - 1)) == 0, "world size must be a power of two"); // test_dist.cpp:90-94
        auto g = std::make_unique<qsv_ctx>();
        for (int r = 0; r < ndev; ++r) {
            auto c = std::make_unique<qsv_ctx>();
            init_ctx(*c, devices[r]);
            c->rank = r;
            c->world = ndev;
            c->gbits = std::countr_zero(static_cast<unsigned>(ndev));
            c->in_process = true;
            g->parts.push_back(c.release());
        }
        if (ndev > 1) {
            std::vector<Ctx *> rk(g->parts.begin(), g->parts.end());
            nccl_init_all(rk);
        }
        Ctx &c0 = *g->parts[0];
        g->device = c0.device;
        g->stream = nullptr;  // a group has no stream of its own (rank 0's is reported)
        g->rank = 0;
        g->world = ndev;
        g->gbits = c0.gbits;
        g->sm_count = c0.sm_count;
        g->smem_optin = c0.smem_optin;
        g->in_process = true;
        *out = g.release();
    });
}

int qsv_ctx_rank_ctx(qsv_ctx *group, int rank, qsv_ctx **out) {
    return guard([&] {
        require(group && out, "null argument");
        require(is_group(group), "qsv_ctx_rank_ctx: not a multi-device context");
        require(rank >= 0 && rank < static_cast<int>(group->parts.size()), "rank out of range");
        *out = group->parts[rank];
    });
}

int qsv_run_on_ranks(qsv_ctx *group, qsv_rank_fn fn, void *user) {
    return guard([&] {
        require(group && fn, "null argument");
        if (!is_group(group)) { // a single rank: run inline
            const int rc = fn(group, group->rank, user);
            if (rc) fail(rc, g_err);
            return;
        }
        on_ranks(group->parts, [&](int r) { return fn(group->parts[r], r, user); });
    });
}

int qsv_ctx_comm_stats(const qsv_ctx *ctx, uint64_t *messages, uint64_t *bytes, uint64_t *allreduces) {
    return guard([&] {
        require(ctx != nullptr, "null ctx");
        uint64_t m = ctx->stat_messages, b = ctx->stat_bytes, a = ctx->stat_allreduces;
        for (const qsv_ctx *x : ctx->parts) {
            m += x->stat_messages;
            b += x->stat_bytes;
            a += x->stat_allreduces;
        }
        if (messages) *messages = m;
        if (bytes) *bytes = b;
        if (allreduces) *allreduces = a;
    });
}

int qsv_ctx_comm_reset(qsv_ctx *ctx) {
    return guard([&] {
        require(ctx != nullptr, "null ctx");
        ctx->stat_messages = ctx->stat_bytes = ctx->stat_allreduces = 0;
        for (qsv_ctx *x : ctx->parts) x->stat_messages = x->stat_bytes = x->stat_allreduces = 0;
    });
}

int qsv_run_rows_expect_z(qsv_ctx *ctx, int nqubit, int dtype, const qsv_gate *gates, int ngates, const double *data,
                          int rows, int slots, const qsv_opts *opts, double *out) {
    return guard([&] {
        require(ctx && out && rows >= 1 && (slots == 0 || data), "null argument");
        if (!is_group(ctx)) {  // one GPU: the whole batch
            qsv_plan *p = nullptr;
            qsv_state *st = nullptr;
            detail_run_rows(ctx, nqubit, dtype, gates, ngates, data, rows, slots, opts, out, &p, &st);
            return;
        }
        const int P = static_cast<int>(ctx->parts.size());
        if (ctx->solo.empty())
            for (int r = 0; r < P; ++r) {
                auto c = std::make_unique<qsv_ctx>();
                init_ctx(*c, ctx->parts[r]->device);
                ctx->solo.push_back(c.release());
            }
        const int per = (rows + P - 1) / P;
        on_ranks(ctx->solo, [&](int r) {
            const int r0 = std::min(rows, r * per), r1 = std::min(rows, r0 + per);
            if (r1 <= r0) return static_cast<int>(QSV_OK);
            return guard([&] {
                qsv_plan *p = nullptr;
                qsv_state *st = nullptr;
                detail_run_rows(ctx->solo[r], nqubit, dtype, gates, ngates, data + static_cast<size_t>(r0) * slots,
                                r1 - r0, slots, opts, out + static_cast<size_t>(r0) * nqubit, &p, &st);
            });
        });
    });
}

int qsv_ctx_destroy(qsv_ctx *ctx) {
    return guard([&] { delete ctx; });
}

int qsv_ctx_sync(qsv_ctx *ctx) {
    return guard([&] {
        require(ctx != nullptr, "null ctx");
        if (is_group(ctx)) {
            on_ranks(ctx->parts, [&](int r) { return qsv_ctx_sync(ctx->parts[r]); });
            return;
        }
        QSV_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int qsv_ctx_stream(qsv_ctx *ctx, void **stream) {
    return guard([&] {
        require(ctx && stream, "null argument");
        *stream = is_group(ctx) ? ctx->parts[0]->stream : ctx->stream;
    });
}

int qsv_ctx_rank(qsv_ctx *ctx, int *rank, int *world) {
    return guard([&] {
        require(ctx && rank && world, "null argument");
        *rank = ctx->rank;
        *world = ctx->world;
    });
}

int qsv_state_create(qsv_ctx *ctx, int nqubit, int batch, int dtype, qsv_state **out) {
    return guard([&] {
        require(ctx && out, "null argument");
        require(nqubit >= 1 && nqubit <= kMaxQubits, "QubitState: nqubit out of range");
        require(batch >= 1, "QubitState: batch must be >= 1");
        require(dtype == QSV_C64 || dtype == QSV_C128, "QubitState: dtype must be QSV_C64 or QSV_C128");
        require(nqubit >= ctx->gbits, "QubitState: fewer amplitudes than ranks");
        if (is_group(ctx)) { // one slice per rank; the host view is the whole state
            auto g = std::make_unique<qsv_state>();
            g->parts.assign(ctx->parts.size(), nullptr);
            on_ranks(ctx->parts, [&](int r) { return qsv_state_create(ctx->parts[r], nqubit, batch, dtype, &g->parts[r]); });
            g->ctx = ctx;
            g->n = nqubit;
            g->nlocal = nqubit;
            g->batch = batch;
            g->dtype = dtype;
            g->local_amps = 1ull << nqubit;
            g->perm.resize(nqubit);
            for (int w = 0; w < nqubit; ++w) g->perm[w] = nqubit - 1 - w;
            *out = g.release();
            return;
        }
        auto st = std::make_unique<qsv_state>();
        st->ctx = ctx;
        st->n = nqubit;
        st->nlocal = nqubit - ctx->gbits;
        require(st->nlocal >= 1, "QubitState: need at least one local qubit per rank");
        st->batch = batch;
        st->dtype = dtype;
        st->local_amps = 1ull << st->nlocal;
        st->perm.resize(nqubit);
        for (int w = 0; w < nqubit; ++w) st->perm[w] = nqubit - 1 - w;
        QSV_CUDA(cudaSetDevice(ctx->device));
        const size_t bytes = st->local_amps * st->amp_bytes() * static_cast<size_t>(batch);
        const cudaError_t e = state_alloc(&st->d, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            fail(QSV_ERR_INTERNAL, "QubitState: cannot allocate " + std::to_string(bytes) + " bytes of HBM");
        }
        launch_set_basis(*st, 0, ctx->rank == 0);
        QSV_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = st.release();
    });
}

int qsv_state_destroy(qsv_state *st) {
    return guard([&] { delete st; });
}

int qsv_state_info(const qsv_state *st, int *nqubit, int *batch, int *dtype, int *global_bits, uint64_t *local_amps) {
    return guard([&] {
        require(st != nullptr, "null state");
        if (nqubit) *nqubit = st->n;
        if (batch) *batch = st->batch;
        if (dtype) *dtype = st->dtype;
        if (global_bits) *global_bits = st->ctx->gbits;  // a group: log2 of its ranks
        if (local_amps) *local_amps = st->local_amps;
    });
}

int qsv_state_set_basis(qsv_state *st, uint64_t index) {
    return guard([&] {
        require(st != nullptr, "null state");
        require(st->n >= 64 || index < (1ull << st->n), "QubitState: basis index out of range"); // state.hpp:36
        if (is_group(st)) {
            on_ranks(group_ctx(st)->parts, [&](int r) { return qsv_state_set_basis(st->parts[r], index); });
            return;
        }
        const uint64_t owner = index >> st->nlocal;
        if (st->ctx->world == 1) reset_layout(*st);  // every row is overwritten
        launch_set_basis(*st, index & (st->local_amps - 1), owner == static_cast<uint64_t>(st->ctx->rank));
        QSV_CUDA(cudaStreamSynchronize(st->ctx->stream));
    });
}

int qsv_state_upload(qsv_state *st, int row, const double *host, uint64_t count) {
    return guard([&] {
        require(st && host, "null argument");
        if (is_group(st))
            return group_slices(st, host, count, 16, [&](qsv_state *x, const double *h, uint64_t c) {
                return qsv_state_upload(x, row, h, c);
            });
        require(count == st->local_amps, "QubitState: amplitude length mismatch");
        upload_layout(*st);
        upload_f64(*st, row_ptr(*st, row), host, count);
    });
}

int qsv_state_download(qsv_state *st, int row, double *host, uint64_t count) {
    return guard([&] {
        require(st && host, "null argument");
        if (is_group(st))
            return group_slices(st, host, count, 16, [&](qsv_state *x, double *h, uint64_t c) {
                return qsv_state_download(x, row, h, c);
            });
        require(count == st->local_amps, "QubitState: amplitude length mismatch");
        normalize_layout(*st);  // lazy layouts: amplitudes leave in logical order
        download_f64(*st, row_ptr(*st, row), host, count);
    });
}

int qsv_state_upload_raw(qsv_state *st, int row, const void *host, uint64_t count) {
    return guard([&] {
        require(st && host, "null argument");
        if (is_group(st))
            return group_slices(st, host, count, st->amp_bytes(), [&](qsv_state *x, const void *h, uint64_t c) {
                return qsv_state_upload_raw(x, row, h, c);
            });
        require(count == st->local_amps, "QubitState: amplitude length mismatch");
        upload_layout(*st);
        QSV_CUDA(cudaMemcpyAsync(row_ptr(*st, row), host, count * st->amp_bytes(), cudaMemcpyHostToDevice,
                                 st->ctx->stream));
        QSV_CUDA(cudaStreamSynchronize(st->ctx->stream));  // the caller may reuse `host` on return
    });
}

int qsv_state_upload_raw_async(qsv_state *st, int row, const void *host, uint64_t count) {
    return guard([&] {
        require(st && host, "null argument");
        if (is_group(st))
            return group_slices(st, host, count, st->amp_bytes(), [&](qsv_state *x, const void *h, uint64_t c) {
                return qsv_state_upload_raw_async(x, row, h, c);
            });
        require(count == st->local_amps, "QubitState: amplitude length mismatch");
        upload_layout(*st);
        QSV_CUDA(cudaMemcpyAsync(row_ptr(*st, row), host, count * st->amp_bytes(), cudaMemcpyHostToDevice,
                                 st->ctx->stream));
    });
}

int qsv_state_download_raw_async(qsv_state *st, int row, void *host, uint64_t count) {
    return guard([&] {
        require(st && host, "null argument");
        if (is_group(st))
            return group_slices(st, host, count, st->amp_bytes(), [&](qsv_state *x, void *h, uint64_t c) {
                return qsv_state_download_raw_async(x, row, h, c);
            });
        require(count == st->local_amps, "QubitState: amplitude length mismatch");
        normalize_layout(*st);  // lazy layouts: amplitudes leave in logical order
        QSV_CUDA(cudaMemcpyAsync(host, row_ptr(*st, row), count * st->amp_bytes(), cudaMemcpyDeviceToHost,
                                 st->ctx->stream));
    });
}

int qsv_state_download_raw(qsv_state *st, int row, void *host, uint64_t count) {
    return guard([&] {
        require(st && host, "null argument");
        if (is_group(st))
            return group_slices(st, host, count, st->amp_bytes(), [&](qsv_state *x, void *h, uint64_t c) {
                return qsv_state_download_raw(x, row, h, c);
            });
        require(count == st->local_amps, "QubitState: amplitude length mismatch");
        normalize_layout(*st);  // lazy layouts: amplitudes leave in logical order
        QSV_CUDA(cudaMemcpyAsync(host, row_ptr(*st, row), count * st->amp_bytes(), cudaMemcpyDeviceToHost,
                                 st->ctx->stream));
        QSV_CUDA(cudaStreamSynchronize(st->ctx->stream));
    });
}

int qsv_state_clone(const qsv_state *src, qsv_state **out) {
    return guard([&] {
        require(src && out, "null argument");
        if (is_group(src)) {
            auto g = std::make_unique<qsv_state>();
            static_cast<qsv::State &>(*g) = static_cast<const qsv::State &>(*src);
            g->parts.assign(src->parts.size(), nullptr);
            on_ranks(group_ctx(src)->parts, [&](int r) { return qsv_state_clone(src->parts[r], &g->parts[r]); });
            *out = g.release();
            return;
        }
        auto st = std::make_unique<qsv_state>();
        st->ctx = src->ctx;
        st->n = src->n;
        st->nlocal = src->nlocal;
        st->batch = src->batch;
        st->dtype = src->dtype;
        st->local_amps = src->local_amps;
        st->perm = src->perm;
        const size_t bytes = st->local_amps * st->amp_bytes() * static_cast<size_t>(st->batch);
        QSV_CUDA(state_alloc(&st->d, bytes));
        QSV_CUDA(cudaMemcpyAsync(st->d, src->d, bytes, cudaMemcpyDeviceToDevice, src->ctx->stream));
        QSV_CUDA(cudaStreamSynchronize(src->ctx->stream));
        *out = st.release();
    });
}

int qsv_state_device_ptr(qsv_state *st, int row, void **ptr) {
    return guard([&] {
        require(st && ptr, "null argument");
        require(!is_group(st), "device_ptr: a multi-device state has one pointer per rank (use the rank contexts)");
        normalize_layout(*st);  // the pointer's amplitudes are in logical order
        *ptr = row_ptr(*st, row);
    });
}

int qsv_state_peer_memory(const qsv_state *st, int *out) {
    return guard([&] {
        require(st && out, "null argument");
        *out = is_group(st) ? st->parts[0]->p2p : st->p2p;
    });
}

int qsv_gate_matrix(const qsv_gate *g, double *out, int *k) {
    return guard([&] {
        require(g && out, "null argument");
        cplx m[16];
        const int kk = gate_matrix(*g, m);
        const int d = 1 << kk;
        for (int i = 0; i < d * d; ++i) {
            out[2 * i] = m[i].real();
            out[2 * i + 1] = m[i].imag();
        }
        if (k) *k = kk;
    });
}

int qsv_apply_matrix(qsv_state *st, int k, const int32_t *wires, int nctl, const int32_t *ctls, const double *m,
                     int flags) {
    return guard([&] {
        require(st && wires && m, "null argument");
        if (is_group(st)) {
            on_ranks(group_ctx(st)->parts,
                     [&](int r) { return qsv_apply_matrix(st->parts[r], k, wires, nctl, ctls, m, flags); });
            return;
        }
        require(k >= 1 && k <= 2, "apply_matrix: 1 or 2 target wires supported");
        require(nctl >= 0 && nctl <= 6 && (nctl == 0 || ctls), "apply_matrix: bad controls");
        GateRec g;
        g.name = "matrix";
        g.kind = GK_CUSTOM;
        g.k = k;
        for (int i = 0; i < k; ++i) {
            require(wires[i] >= 0 && wires[i] < st->n, "target wire out of range"); // state.hpp:116
            g.wires[i] = wires[i];
        }
        require(k == 1 || wires[0] != wires[1], "apply_matrix: duplicate target wires");
        for (int i = 0; i < nctl; ++i) {
            require(ctls[i] >= 0 && ctls[i] < st->n, "control wire out of range"); // state.hpp:117
            for (int j = 0; j < k; ++j) require(ctls[i] != wires[j], "gate wires and controls must be disjoint");
            g.ctls.push_back(ctls[i]);
        }
        const int d = 1 << k;
        bool diag = true;
        for (int i = 0; i < d * d; ++i) {
            g.m[i] = cplx(m[2 * i], m[2 * i + 1]);
            if (i / d != i % d && g.m[i] != cplx(0, 0)) diag = false;
        }
        g.diag = diag;
        require((flags & ~(QSV_ZERO_OFF_CONTROL | QSV_HINT_DIAGONAL | QSV_HINT_PERMUTATION)) == 0,
                "apply_matrix: unknown flags");
        require(!(flags & QSV_HINT_DIAGONAL) || diag, "apply_matrix: DIAGONAL hint on a non-diagonal matrix");
        if (flags & QSV_HINT_PERMUTATION) {
            bool perm = true;
            for (int r = 0; r < d && perm; ++r) {
                int ones = 0;
                for (int c = 0; c < d; ++c) {
                    const cplx &e = g.m[r * d + c];
                    if (e == cplx(1, 0)) ++ones;
                    else if (e != cplx(0, 0)) perm = false;
                }
                perm = perm && ones == 1;
            }
            require(perm, "apply_matrix: PERMUTATION hint on a matrix that is not a 0/1 permutation");
        }
        g.flags = (flags & QSV_ZERO_OFF_CONTROL) ? OPF_ZERO_OFF_CONTROL : 0;
        run_single(*st, g);
    });
}

int qsv_apply_gate(qsv_state *st, const qsv_gate *gate) {
    return guard([&] {
        require(st && gate, "null argument");
        if (is_group(st)) {
            on_ranks(group_ctx(st)->parts, [&](int r) { return qsv_apply_gate(st->parts[r], gate); });
            return;
        }
        int cursor = 0;
        qsv_gate g = *gate;
        g.encode = 0; // apply_gate uses the gate's own params (state.hpp:149-151)
        GateRec r = resolve_gate(g, st->n, &cursor);
        run_single(*st, r);
    });
}

int qsv_run_circuit(qsv_state *st, const qsv_gate *gates, int ngates, const double *data, int rows, int slots,
                    const qsv_opts *opts) {
    return guard([&] {
        require(st != nullptr, "null state");
        if (is_group(st)) {
            on_ranks(group_ctx(st)->parts,
                     [&](int r) { return qsv_run_circuit(st->parts[r], gates, ngates, data, rows, slots, opts); });
            return;
        }
        qsv_ctx *c = static_cast<qsv_ctx *>(st->ctx);
        static const bool nocache = [] {  // QSV_NO_PLAN_CACHE=1: plan every call
            const char *e = std::getenv("QSV_NO_PLAN_CACHE");
            return e && e[0] == '1';
        }();
        static const bool nolift = [] {  // QSV_NO_LIFT=1: trainable angles stay compile-time constants
            const char *e = std::getenv("QSV_NO_LIFT");
            return e && e[0] == '1';
        }();
        Lifted lf;
        const bool lift = !nolift && want_lift(*c, st->n, st->dtype, opts, gates, ngates);
        if (lift && lift_trainable(gates, ngates, st->n, data, rows, slots, st->batch, lf)) {
            gates = lf.gates.data();
            data = lf.data.data();
            rows = lf.rows;
            slots = lf.slots;
        }
        if (nocache || c->world != 1 || ngates > 4096) {
            Plan p;
            build_plan_from_abi(p, st->ctx, st->n, st->dtype, gates, ngates, opts);
            execute_plan(p, *st, data, rows, slots);
            QSV_CUDA(cudaStreamSynchronize(st->ctx->stream));
            return;
        }
        std::unique_lock<std::mutex> lk;
        Plan &plan = cached_plan(c, st->n, st->dtype, opts, gates, ngates, lk);
        execute_plan(plan, *st, data, rows, slots);
        QSV_CUDA(cudaStreamSynchronize(st->ctx->stream));
    });
}

int qsv_plan_create(qsv_ctx *ctx, int nqubit, int dtype, const qsv_gate *gates, int ngates, const qsv_opts *opts,
                    qsv_plan **out) {
    return guard([&] {
        require(ctx && out, "null argument");
        auto q = std::make_unique<qsv_plan>();
        if (is_group(ctx)) {
            q->parts.assign(ctx->parts.size(), nullptr);
            on_ranks(ctx->parts, [&](int r) {
                return qsv_plan_create(ctx->parts[r], nqubit, dtype, gates, ngates, opts, &q->parts[r]);
            });
            q->ctx = ctx;
            q->n = nqubit;
            q->dtype = dtype;
            *out = q.release();
            return;
        }
        build_plan_from_abi(*q, ctx, nqubit, dtype, gates, ngates, opts);
        *out = q.release();
    });
}

int qsv_plan_destroy(qsv_plan *plan) {
    return guard([&] { delete plan; });
}

int qsv_plan_info_get(const qsv_plan *p, qsv_plan_info *info) {
    return guard([&] {
        require(p && info, "null argument");
        if (is_group(p)) p = p->parts[0];
        std::memset(info, 0, sizeof(*info));
        info->ngates = p->ngates;
        if (p->dense) {
            info->npasses = info->ntile_passes = static_cast<int>(p->dpasses.size());
            info->nblocks = static_cast<int>(p->dblocks.size());
            info->max_tile_bits = kDenseTile;
            info->bytes_per_exec = p->dpasses.size() * 2.0 * 8 * std::ldexp(1.0, p->nlocal);
            return;
        }
        for (const Step &s : p->steps) {
            if (s.kind == 0) {
                info->ntile_passes += 1;
                if (p->passes[s.pass].pair == 2) continue;  // inside its head's launch
                info->npasses += 1;
                info->bytes_per_exec += p->dev[s.pass].bytes;
                info->max_tile_bits = std::max(info->max_tile_bits, p->passes[s.pass].K);
            } else {
                info->nswaps += static_cast<int>(s.swap_bits.size());
                const double amp = p->dtype == QSV_C64 ? 8 : 16;
                info->comm_bytes_per_exec += s.swap_bits.size() * amp * std::ldexp(1.0, p->nlocal - 1);
            }
        }
    });
}

int qsv_plan_execute(qsv_plan *plan, qsv_state *st, const double *data, int rows, int slots) {
    return guard([&] {
        require(plan && st, "null argument");
        if (is_group(plan) || is_group(st)) {
            require(is_group(plan) && is_group(st) && plan->parts.size() == st->parts.size(),
                    "plan/state belong to different contexts");
            on_ranks(group_ctx(st)->parts,
                     [&](int r) { return qsv_plan_execute(plan->parts[r], st->parts[r], data, rows, slots); });
            return;
        }
        execute_plan(*plan, *st, data, rows, slots);
    });
}

int qsv_plan_execute_expect_z(qsv_plan *plan, qsv_state *st, const double *data, int rows, int slots, double *out) {
    return guard([&] {
        require(plan && st && out, "null argument");
        if (is_group(plan) || is_group(st)) {
            require(is_group(plan) && is_group(st) && plan->parts.size() == st->parts.size(),
                    "plan/state belong to different contexts");
            std::vector<double> other(static_cast<size_t>(st->batch) * st->n * st->parts.size());
            on_ranks(group_ctx(st)->parts, [&](int r) {
                double *o = r == 0 ? out : other.data() + static_cast<size_t>(r) * st->batch * st->n;
                return qsv_plan_execute_expect_z(plan->parts[r], st->parts[r], data, rows, slots, o);
            });
            return;
        }
        execute_plan_z(*plan, *st, data, rows, slots, out);
    });
}

int qsv_plan_profile(qsv_plan *plan, qsv_state *st, double *launch_ms) {
    return guard([&] {
        require(plan && st && launch_ms, "null argument");
        if (is_group(plan) || is_group(st)) {  // rank 0's launch times (every rank runs the same steps)
            require(is_group(plan) && is_group(st) && plan->parts.size() == st->parts.size(),
                    "plan/state belong to different contexts");
            std::vector<double> other(plan->parts[0]->steps.size() * st->parts.size());
            on_ranks(group_ctx(st)->parts, [&](int r) {
                double *o = r == 0 ? launch_ms : other.data() + r * plan->parts[0]->steps.size();
                return qsv_plan_profile(plan->parts[r], st->parts[r], o);
            });
            return;
        }
        profile_plan(*plan, *st, launch_ms);
    });
}

int qsv_norm2(qsv_state *st, double *out) {
    return guard([&] {
        require(st && out, "null argument");
        if (is_group(st)) {
            std::vector<double> other(static_cast<size_t>(st->batch) * st->parts.size());
            on_ranks(group_ctx(st)->parts,
                     [&](int r) { return qsv_norm2(st->parts[r], r == 0 ? out : other.data() + r * st->batch); });
            return;
        }
        reduce_norm2(*st, out);
    });
}

int qsv_expect_z_all(qsv_state *st, double *out) {
    return guard([&] {
        require(st && out, "null argument");
        if (is_group(st)) {
            const size_t per = static_cast<size_t>(st->batch) * st->n;
            std::vector<double> other(per * st->parts.size());
            on_ranks(group_ctx(st)->parts,
                     [&](int r) { return qsv_expect_z_all(st->parts[r], r == 0 ? out : other.data() + r * per); });
            return;
        }
        constexpr int kZ = 41;
        std::vector<double> z(static_cast<size_t>(st->batch) * kZ);
        reduce_z_all(*st, z.data());
        for (int b = 0; b < st->batch; ++b) {
            const double *zb = z.data() + static_cast<size_t>(b) * kZ;
            for (int w = 0; w < st->n; ++w)
                out[static_cast<size_t>(b) * st->n + w] = zb[0] - 2.0 * zb[1 + st->perm[w]];
        }
    });
}

namespace {
// X/Y of an observable on a global (rank) qubit: swap that qubit with a local
// bit the observable does not use -- the same exchange a gate on the wire
// triggers (dist.cu) -- so the Pauli kernel sees it locally; swapping the
// same pairs again restores the layout (tests/test_dist.cpp:189-204 measures
// X on a rank wire).
std::vector<std::pair<int, int>> localise_xy(qsv_state *st, const qsv_obs &o) {
    std::vector<std::pair<int, int>> pairs;
    if (st->nlocal == st->n) return pairs;
    std::vector<char> used(st->n, 0);
    for (int j = 0; j < o.nwires; ++j)
        if (o.wires[j] >= 0 && o.wires[j] < st->n) used[st->perm[o.wires[j]]] = 1;
    int next_lb = 0;
    for (int j = 0; j < o.nwires; ++j) {
        const char c = o.basis[j];
        if (c == 'z' || o.wires[j] < 0 || o.wires[j] >= st->n) continue;
        const int gb = st->perm[o.wires[j]];
        if (gb < st->nlocal) continue;
        bool done = false;  // a repeated wire is localised once
        for (const auto &pr : pairs) done = done || pr.first == gb;
        if (done) continue;
        while (next_lb < st->nlocal && used[next_lb]) ++next_lb;
        require(next_lb < st->nlocal, "observable: no free local qubit to localise a global x/y");
        used[next_lb] = 1;
        pairs.emplace_back(gb, next_lb);
    }
    return pairs;
}
void apply_swaps(qsv_state *st, const std::vector<std::pair<int, int>> &pairs) {
    if (pairs.empty()) return;
    dist_swap_bits(*st, pairs, nullptr, 0);
    for (const auto &[gb, lb] : pairs) {
        int wa = -1, wb = -1;
        for (int w = 0; w < st->n; ++w) {
            if (st->perm[w] == gb) wa = w;
            if (st->perm[w] == lb) wb = w;
        }
        std::swap(st->perm[wa], st->perm[wb]);
    }
}
} // namespace

int qsv_expect_pauli(qsv_state *st, int nobs, const qsv_obs *obs, double *out) {
    return guard([&] {
        require(st && (nobs == 0 || (obs && out)), "null argument");
        if (is_group(st)) {
            const size_t per = static_cast<size_t>(st->batch) * std::max(nobs, 1);
            std::vector<double> other(per * st->parts.size());
            on_ranks(group_ctx(st)->parts, [&](int r) {
                return qsv_expect_pauli(st->parts[r], nobs, obs, r == 0 ? out : other.data() + r * per);
            });
            return;
        }
        for (int i = 0; i < nobs; ++i) {
            const qsv_obs &o = obs[i];
            const auto moved = localise_xy(st, o);
            apply_swaps(st, moved);
            struct Restore {  // the layout comes back even when the observable fails
                qsv_state *st;
                std::vector<std::pair<int, int>> pairs;
                ~Restore() {
                    try {
                        apply_swaps(st, pairs);
                    } catch (...) {
                    }
                }
            } restore{st, std::vector<std::pair<int, int>>(moved.rbegin(), moved.rend())};
            require(o.nwires >= 0 && (o.nwires == 0 || (o.wires && o.basis)), "observable: bad wires");
            require(static_cast<int>(std::strlen(o.basis ? o.basis : "")) == o.nwires,
                    "observable: one basis letter per wire"); // circuit.hpp:97
            // the Paulis applied wire by wire like expectation_one
            // (circuit.hpp:255-259): per wire the product is i^k X^x Z^z
            // (X = X, Z = Z, Y = i X Z; Q * i^k X^x Z^z = i^(q+k) (-1)^(b x)
            // X^(a^x) Z^(b^z) for Q = i^q X^a Z^b), so a repeated wire composes
            uint64_t flip = 0, zy = 0;
            int kph = 0;
            for (int j = 0; j < o.nwires; ++j) {
                const char c = o.basis[j];
                require(c == 'x' || c == 'y' || c == 'z', "observable: basis letter outside {x,y,z}");
                const int w = o.wires[j];
                require(w >= 0 && w < st->n, "target wire out of range");
                const int pb = st->perm[w];
                require(pb < st->nlocal || c == 'z', "observable: internal: x/y on a global qubit after localisation");
                const uint64_t bit = 1ull << pb;
                const int q = c == 'y' ? 1 : 0, a = c != 'z', b = c != 'x';
                kph += q + ((b && (flip & bit)) ? 2 : 0);
                if (a) flip ^= bit;
                if (b) zy ^= bit;
            }
            // the kernel sums conj(a_i) (-1)^popc(i & zy) a_(i ^ flip); X^x Z^z
            // reads (-1)^popc((i ^ x) & z): a further (-1)^popc(x & z)
            const int ny = (kph + 2 * std::popcount(flip & zy)) & 3;  // result = i^ny * sum
            std::vector<double> v(static_cast<size_t>(st->batch) * 2);
            reduce_pauli(*st, flip, zy, v.data());
            for (int b = 0; b < st->batch; ++b) {
                double re = v[2 * b], im = v[2 * b + 1];
                for (int t = 0; t < ny; ++t) {
                    const double nre = -im, nim = re; // multiply by i
                    re = nre, im = nim;
                }
                if (std::abs(im) >= 1e-10) fail(QSV_ERR_INVALID, "expectation: imaginary residue"); // circuit.hpp:261
                out[static_cast<size_t>(b) * nobs + i] = re;
            }
        }
    });
}

int qsv_marginal_probs(qsv_state *st, int row, int k, const int32_t *wires, double *out) {
    return guard([&] {
        require(st && out, "null argument");
        require(k >= 1 && wires, "measure: empty wire list"); // circuit.hpp:185
        require(row >= 0 && row < st->batch, "batch index out of range");
        if (is_group(st)) {
            require(k <= 26, "marginal_probs: 1..26 wires supported");
            std::vector<double> other((size_t(1) << k) * st->parts.size());
            on_ranks(group_ctx(st)->parts, [&](int r) {
                return qsv_marginal_probs(st->parts[r], row, k, wires, r == 0 ? out : other.data() + (size_t(r) << k));
            });
            return;
        }
        std::vector<int> bits;
        for (int i = 0; i < k; ++i) {
            require(wires[i] >= 0 && wires[i] < st->n, "target wire out of range");
            bits.push_back(st->perm[wires[i]]);
        }
        reduce_marginal(*st, row, bits, out);
    });
}

int qsv_measure(qsv_state *st, int row, int k, const int32_t *wires, int shots, uint64_t seed, const char *label,
                uint64_t *rng_counter, uint64_t *counts, double *probs) {
    return guard([&] {
        require(st && counts, "null argument");
        require(shots >= 1, "measure: shots must be >= 1");  // circuit.hpp:221
        require(k >= 1 && k <= 26 && wires, "measure: 1..26 wires");
        std::vector<double> p(size_t(1) << k);
        const int rc = qsv_marginal_probs(st, row, k, wires, p.data());
        if (rc) fail(rc, g_err);
        sample_counts(p.data(), k, shots, seed, label, rng_counter, counts);
        if (probs) std::copy(p.begin(), p.end(), probs);
    });
}

namespace {
void require_canonical_density(qsv_state *st) {
    require(!is_group(st), "density: mixed states run on one GPU");
    normalize_layout(*st);
    require(st->n % 2 == 0 && st->n >= 2, "density: a mixed state of m qubits is held on 2m engine qubits");
    require(st->nlocal == st->n, "density: mixed states run on one GPU");
    for (int w = 0; w < st->n; ++w)
        require(st->perm[w] == st->n - 1 - w, "density: state layout is not canonical");
}
} // namespace

int qsv_density_expect_pauli(qsv_state *st, int nobs, const qsv_obs *obs, double *out) {
    return guard([&] {
        require(st && (nobs == 0 || (obs && out)), "null argument");
        require_canonical_density(st);
        const int m = st->n / 2;
        for (int i = 0; i < nobs; ++i) {
            const qsv_obs &o = obs[i];
            require(o.nwires >= 0 && (o.nwires == 0 || (o.wires && o.basis)), "observable: bad wires");
            require(static_cast<int>(std::strlen(o.basis ? o.basis : "")) == o.nwires,
                    "observable: one basis letter per wire"); // circuit.hpp:97
            // per wire the product i^k X^x Z^z, composed like expectation_one
            uint64_t flip = 0, zy = 0;
            int kph = 0;
            for (int j = 0; j < o.nwires; ++j) {
                const char c = o.basis[j];
                require(c == 'x' || c == 'y' || c == 'z', "observable: basis letter outside {x,y,z}");
                const int w = o.wires[j];
                require(w >= 0 && w < m, "target wire out of range");
                const uint64_t bit = 1ull << (m - 1 - w);
                const int q = c == 'y' ? 1 : 0, a = c != 'z', b = c != 'x';
                kph += q + ((b && (flip & bit)) ? 2 : 0);
                if (a) flip ^= bit;
                if (b) zy ^= bit;
            }
            const int ny = kph & 3;
            std::vector<double> v(static_cast<size_t>(st->batch) * 2);
            reduce_dm_pauli(*st, m, flip, zy, v.data());
            // Tr[rho X^x Z^z] = sum_r rho[r, r ^ x] (-1)^popc(r & z)
            for (int b = 0; b < st->batch; ++b) {
                double re = v[2 * b], im = v[2 * b + 1];
                for (int t = 0; t < ny; ++t) {
                    const double nre = -im, nim = re; // multiply by i
                    re = nre, im = nim;
                }
                // circuit.hpp:280 (1e-10 in double; a complex64 rho is Hermitian to ~1e-7)
                if (std::abs(im) >= (st->dtype == QSV_C64 ? 1e-5 : 1e-10))
                    fail(QSV_ERR_INVALID, "expectation: imaginary residue");
                out[static_cast<size_t>(b) * nobs + i] = re;
            }
        }
    });
}

int qsv_density_marginal_probs(qsv_state *st, int row, int k, const int32_t *wires, double *out) {
    return guard([&] {
        require(st && out, "null argument");
        require(k >= 1 && wires, "measure: empty wire list"); // circuit.hpp:185
        require(row >= 0 && row < st->batch, "batch index out of range");
        require_canonical_density(st);
        const int m = st->n / 2;
        std::vector<int> bits;
        for (int i = 0; i < k; ++i) {
            require(wires[i] >= 0 && wires[i] < m, "target wire out of range");
            bits.push_back(m - 1 - wires[i]);
        }
        reduce_dm_marginal(*st, m, row, bits, out);
    });
}

int qsv_adjoint_gradients(qsv_ctx *ctx, int nqubit, int dtype, const qsv_gate *gates, int ngates, int nobs,
                          const qsv_obs *obs, const double *init, const double *data, int slots,
                          double *param_grads, int param_cap, int *nparams, double *data_grads) {
    return guard([&] {
        require(ctx != nullptr, "null ctx");
        require(nqubit >= 1 && nqubit <= kMaxQubits, "adjoint_gradients: nqubit out of range");
        require(dtype == QSV_C64 || dtype == QSV_C128, "adjoint_gradients: bad dtype");
        require(slots == 0 || data, "adjoint_gradients: data missing");
        if (is_group(ctx)) {
            const int P = static_cast<int>(ctx->parts.size());
            std::vector<std::vector<double>> pgs(P, std::vector<double>(std::max(param_cap, 1))),
                dgs(P, std::vector<double>(std::max(slots, 1)));
            std::vector<int> nps(P, 0);
            on_ranks(ctx->parts, [&](int r) {
                return qsv_adjoint_gradients(ctx->parts[r], nqubit, dtype, gates, ngates, nobs, obs, init, data, slots,
                                             pgs[r].data(), param_cap, &nps[r], dgs[r].data());
            });
            if (nparams) *nparams = nps[0];
            if (param_grads)
                for (int i = 0; i < std::min(param_cap, nps[0]); ++i) param_grads[i] = pgs[0][i];
            if (data_grads)
                for (int i = 0; i < slots; ++i) data_grads[i] = dgs[0][i];
            return;
        }
        std::vector<double> pg, dg;
        adjoint_gradients(ctx, nqubit, dtype, gates, ngates, nobs, obs, init, data, slots, pg, dg);
        if (nparams) *nparams = static_cast<int>(pg.size());
        if (param_grads)
            for (int i = 0; i < std::min<int>(param_cap, static_cast<int>(pg.size())); ++i) param_grads[i] = pg[i];
        if (data_grads)
            for (size_t i = 0; i < dg.size(); ++i) data_grads[i] = dg[i];
    });
}

int qsv_plan_dry(int nqubit, int dtype, int world, const qsv_gate *gates, int ngates, const qsv_opts *opts,
                 qsv_plan_info *info, int pass_index, char *src, size_t cap) {
    return guard([&] {
        require(world >= 1 && (world & (world - 1)) == 0, "world size must be a power of two");
        Ctx ctx;
        ctx.device = -1;
        ctx.world = world;
        ctx.gbits = std::countr_zero(static_cast<unsigned>(world));
        Plan p;
        build_plan_from_abi(p, &ctx, nqubit, dtype, gates, ngates, opts);
        if (info) {
            std::memset(info, 0, sizeof(*info));
            info->ngates = p.ngates;
            const double amp = dtype == QSV_C64 ? 8 : 16;
            if (p.dense) {
                info->npasses = info->ntile_passes = static_cast<int>(p.dpasses.size());
                info->nblocks = static_cast<int>(p.dblocks.size());
                info->max_tile_bits = kDenseTile;
                info->bytes_per_exec = p.dpasses.size() * 2.0 * amp * std::ldexp(1.0, p.nlocal);
            }
            for (const Step &s : p.steps) {
                if (s.kind == 0) {
                    info->ntile_passes += 1;
                    if (p.passes[s.pass].pair == 2) continue;
                    info->npasses += 1;
                    info->bytes_per_exec += 2.0 * amp * std::ldexp(1.0, p.nlocal);
                    info->max_tile_bits = std::max(info->max_tile_bits, p.passes[s.pass].K);
                } else {
                    info->nswaps += static_cast<int>(s.swap_bits.size());
                    info->comm_bytes_per_exec += s.swap_bits.size() * amp * std::ldexp(1.0, p.nlocal - 1);
                }
            }
        }
        if (src && cap && pass_index == -2) { // the whole step schedule as JSON
            std::string js = "{\"n\":" + std::to_string(p.n) + ",\"nlocal\":" + std::to_string(p.nlocal) +
                             ",\"steps\":[";
            char num[64];
            auto dbl = [&](double v) {
                std::snprintf(num, sizeof num, "%.17g", v);
                return std::string(num);
            };
            for (size_t si = 0; si < p.steps.size(); ++si) {
                const Step &s = p.steps[si];
                if (si) js += ",";
                if (s.kind == 1) {
                    js += std::string("{\"kind\":\"swap\",\"fused\":") + (s.fused ? "true" : "false") + ",\"pairs\":[";
                    for (size_t k = 0; k < s.swap_bits.size(); ++k)
                        js += (k ? ",[" : "[") + std::to_string(s.swap_bits[k].first) + "," +
                              std::to_string(s.swap_bits[k].second) + "]";
                    js += "]}";
                    continue;
                }
                const PassHost &ph = p.passes[s.pass];
                js += "{\"kind\":\"pass\",\"pair\":" + std::to_string(ph.pair) + ",\"fused\":" +
                      (s.fused ? "true" : "false") + ",\"tile\":[";
                for (size_t k = 0; k < ph.tile_pos.size(); ++k) js += (k ? "," : "") + std::to_string(ph.tile_pos[k]);
                js += "],\"gperm\":[";
                for (size_t k = 0; k < ph.gperm.size(); ++k) js += (k ? "," : "") + std::to_string(ph.gperm[k]);
                js += "],\"out_perm\":[";
                for (size_t k = 0; k < ph.out_perm.size(); ++k) js += (k ? "," : "") + std::to_string(ph.out_perm[k]);
                js += "],\"gates\":[";
                for (size_t gi = 0; gi < ph.exec_gates.size(); ++gi) {
                    const GateRec &g = ph.exec_gates[gi];
                    js += gi ? ",{" : "{";
                    js += "\"t\":[" + std::to_string(g.wires[0]) + (g.k == 2 ? "," + std::to_string(g.wires[1]) : "") +
                          "],\"c\":[";
                    for (size_t c = 0; c < g.ctls.size(); ++c) js += (c ? "," : "") + std::to_string(g.ctls[c]);
                    js += "],\"enc\":" + std::to_string(g.encoded ? g.enc_slot : -1) + ",\"m\":[";
                    const int d = 1 << g.k;
                    for (int i = 0; i < d * d; ++i)
                        js += (i ? ",[" : "[") + dbl(g.m[i].real()) + "," + dbl(g.m[i].imag()) + "]";
                    js += "]}";
                }
                js += "]}";
            }
            js += "]}";
            require(js.size() + 1 <= cap, "plan_dry: schedule buffer too small");
            std::memcpy(src, js.c_str(), js.size() + 1);
        } else if (src && cap && pass_index <= -3) { // the peer-memory variant of pass -3 - index
            src[0] = 0;
            const int pi = -3 - pass_index;
            if (pi < static_cast<int>(p.passes.size()) && !p.passes[pi].gperm.empty())
                std::snprintf(src, cap, "%s", jit_gout_source(p.passes[pi], dtype).c_str());
        } else if (src && cap) {
            src[0] = 0;
            if (pass_index >= 0 && pass_index < static_cast<int>(p.passes.size())) {
                const PassHost &ph = p.passes[pass_index];
                const std::string s = ph.pair == 1 ? jit_pair_source(ph, p.passes[pass_index + 1], dtype)
                                                   : jit_source(ph, dtype);
                std::snprintf(src, cap, "%s", s.c_str());
            }
        }
        p.ctx = nullptr;
    });
}

int qsv_rng_fill(uint64_t seed, const char *label, int kind, uint64_t count, void *out, int nthreads) {
    return guard([&] {
        require(out != nullptr || count == 0, "null out");
        rng_fill(seed, label, kind, count, out, nthreads, 0);
    });
}

int qsv_rng_fill_at(uint64_t seed, const char *label, int kind, uint64_t offset, uint64_t count, void *out,
                    int nthreads) {
    return guard([&] {
        require(out != nullptr || count == 0, "null out");
        rng_fill(seed, label, kind, count, out, nthreads, offset);
    });
}

int qsv_plan_steps(const qsv_plan *plan, int *kinds, int cap) {
    if (!plan) return -QSV_ERR_INVALID;
    if (is_group(plan)) plan = plan->parts[0];
    if (plan->dense) {  // one launch per dense-block pass
        const int n = static_cast<int>(plan->dpasses.size());
        for (int i = 0; i < n && i < cap && kinds; ++i) kinds[i] = 0;
        return n;
    }
    const int n = static_cast<int>(plan->steps.size());
    for (int i = 0; i < n && i < cap && kinds; ++i) {
        const Step &s = plan->steps[i];
        kinds[i] = s.fused ? 3 : s.kind == 0 && plan->passes[s.pass].pair == 2 ? 2 : s.kind;
    }
    return n;
}

} // extern "C"
