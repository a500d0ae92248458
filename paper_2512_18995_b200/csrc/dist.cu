// Distributed transport over NCCL (NVLink 5 / NVSwitch), one process per GPU.
//
// Replaces the reference's Transport / PartitionedState exchange
// (quasar::dist, source absent from /root/reference; contract in
// proj/tests/test_dist.cpp:66-174 and SPEC.md:719-798). The reference sends
// the WHOLE slice pairwise for every non-diagonal gate on a global wire
// (test_dist.cpp:112-126); here a global qubit is instead SWAPPED with a local
// one: each rank keeps the half of its slice whose local bit already matches
// and exchanges the other half with the partner rank, so every later gate on
// that qubit is local. Several pairs swap at once as ONE all-to-all: with m
// pairs the local index space splits into 2^m blocks by the values v of the
// m local bits; block v of rank r belongs to the peer whose m rank bits are v
// and that peer's block holding r's rank bits comes back into the same
// positions, so each rank sends (1 - 2^-m) of its slice once (m sequential
// pairwise swaps would send m/2 of it). The exchange is chunked through
// persistent staging and is in place (no second copy of the state).
//
// NCCL is dlopen'ed (libnccl.so.2, the one torch bundles) so the library
// loads and single-GPU runs need no NCCL at all.
#include <dlfcn.h>

#include <algorithm>
#include <bit>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "qsv_internal.hpp"

namespace qsv {

namespace {
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef void *ncclComm_t;
typedef int ncclResult_t;
constexpr int ncclUint8 = 1, ncclFloat64 = 8, ncclSum = 0;
} // namespace

struct Nccl {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitAll)(ncclComm_t *, int, const int *) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
    ~Nccl() {
        if (h) dlclose(h);
    }
};

namespace {

std::unique_ptr<Nccl> load_nccl() {
    auto n = std::make_unique<Nccl>();
    const char *env = std::getenv("QSV_NCCL_LIB");
    const char *cands[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char *c : cands) {
        if (!c) continue;
        n->h = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
        if (n->h) break;
    }
    if (!n->h) fail(QSV_ERR_TRANSPORT, "NCCL not found (set QSV_NCCL_LIB to libnccl.so.2)");
#define LOAD(f)                                                                                                        \
    n->f = reinterpret_cast<decltype(n->f)>(dlsym(n->h, "nccl" #f));                                                   \
    if (!n->f) fail(QSV_ERR_TRANSPORT, "NCCL symbol missing: nccl" #f);
    LOAD(GetUniqueId) LOAD(CommInitRank) LOAD(CommDestroy) LOAD(Send) LOAD(Recv) LOAD(GroupStart) LOAD(GroupEnd)
    LOAD(AllReduce) LOAD(GetErrorString)
#undef LOAD
    n->CommInitAll = reinterpret_cast<decltype(n->CommInitAll)>(dlsym(n->h, "ncclCommInitAll"));
    return n;
}

void nccl_ok(const Nccl &n, ncclResult_t r, const char *what) {
    if (r != 0) fail(QSV_ERR_TRANSPORT, std::string("NCCL ") + what + ": " + n.GetErrorString(r));
}

#include "swap_copy.cuh"  // BlockBits, deposit, block_copy_kernel

// new = a * mine + b * theirs on control-satisfied elements (local control
// bits cmask all set); zero_off_control zeroes the others
template <typename T, typename V>
__global__ void exchange_combine_kernel(V *__restrict__ mine, const V *__restrict__ theirs, uint64_t count,
                                        uint64_t e0, uint64_t cmask, int zoc, double ar, double ai, double br,
                                        double bi) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (((e0 + i) & cmask) != cmask) {
            if (zoc) mine[i] = V{T(0), T(0)};
            continue;
        }
        const V x = mine[i], y = theirs[i];
        V o;
        o.x = static_cast<T>(ar * x.x - ai * x.y + br * y.x - bi * y.y);
        o.y = static_cast<T>(ar * x.y + ai * x.x + br * y.y + bi * y.x);
        mine[i] = o;
    }
}

template <typename V> __global__ void zero_kernel(V *p, uint64_t count) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        p[i] = V{};
}

} // namespace

void nccl_unique_id(void *out128) {
    auto n = load_nccl();
    ncclUniqueId id;
    nccl_ok(*n, n->GetUniqueId(&id), "GetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
}

void nccl_init(Ctx &ctx, const void *uid) {
    require(uid != nullptr, "distributed context needs an NCCL unique id");
    ctx.nccl = load_nccl().release();
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    QSV_CUDA(cudaSetDevice(ctx.device));
    ncclComm_t comm = nullptr;
    nccl_ok(*ctx.nccl, ctx.nccl->CommInitRank(&comm, ctx.world, id, ctx.rank), "CommInitRank");
    ctx.comm = comm;
}

void nccl_init_all(const std::vector<Ctx *> &ranks) {
    const int W = static_cast<int>(ranks.size());
    std::vector<int> devs(W);
    for (int r = 0; r < W; ++r) {
        ranks[r]->nccl = load_nccl().release();
        devs[r] = ranks[r]->device;
    }
    const Nccl &n = *ranks[0]->nccl;
    if (!n.CommInitAll) fail(QSV_ERR_TRANSPORT, "NCCL symbol missing: ncclCommInitAll");
    std::vector<ncclComm_t> comms(W, nullptr);
    nccl_ok(n, n.CommInitAll(comms.data(), W, devs.data()), "CommInitAll");
    for (int r = 0; r < W; ++r) ranks[r]->comm = comms[r];
}

void nccl_destroy(Ctx &ctx) {
    if (ctx.stage) {
        cudaStreamSynchronize(ctx.stream);
        cudaFree(ctx.stage);
        ctx.stage = nullptr;
        ctx.stage_bytes = 0;
    }
    if (ctx.comm_stream) {
        cudaStreamSynchronize(ctx.comm_stream);
        cudaStreamDestroy(ctx.comm_stream);
        ctx.comm_stream = nullptr;
    }
    if (ctx.comm && ctx.nccl) ctx.nccl->CommDestroy(static_cast<ncclComm_t>(ctx.comm));
    ctx.comm = nullptr;
    delete ctx.nccl;
    ctx.nccl = nullptr;
}

void dist_allreduce_sum(Ctx &ctx, double *d_buf, size_t count) {
    if (ctx.world == 1) return;
    const Nccl &n = *ctx.nccl;
    nccl_ok(n, n.AllReduce(d_buf, d_buf, count, ncclFloat64, ncclSum, static_cast<ncclComm_t>(ctx.comm), ctx.stream),
            "AllReduce");
    ctx.stat_allreduces += 1;
}

namespace {
void swap_disjoint(State &st, const std::vector<std::pair<int, int>> &pairs);

// every rank's flag summed (a float all-reduce on the state's stream, then
// read back): agreement on whether the peer-memory path is usable
int agree_failures(State &st, int mine) {
    Ctx &ctx = *st.ctx;
    const Nccl &n = *ctx.nccl;
    if (!st.d_barrier) QSV_CUDA(cudaMalloc(&st.d_barrier, sizeof(double)));
    const double f = static_cast<double>(mine);
    QSV_CUDA(cudaMemcpyAsync(st.d_barrier, &f, sizeof f, cudaMemcpyHostToDevice, ctx.stream));
    nccl_ok(n, n.AllReduce(st.d_barrier, st.d_barrier, 1, ncclFloat64, ncclSum, static_cast<ncclComm_t>(ctx.comm),
                           ctx.stream), "AllReduce");
    ctx.stat_allreduces += 1;
    double tot = 0;
    QSV_CUDA(cudaMemcpyAsync(&tot, st.d_barrier, sizeof tot, cudaMemcpyDeviceToHost, ctx.stream));
    QSV_CUDA(cudaStreamSynchronize(ctx.stream));
    return static_cast<int>(tot + 0.5);
}
} // namespace

// Peer memory for qubit swaps fused into passes (plan.cpp run_gout): both
// state buffers of every rank are mapped into every rank with CUDA IPC
// (handles exchanged over NCCL send / recv), so a pass can store each tile
// straight into its destination rank's scratch state over NVLink. Collective:
// all ranks reach it at the same step of the same plan, and they agree on
// the outcome (a failure anywhere -- no room for the scratch state, no peer
// access -- leaves every rank on the NCCL swaps). QSV_P2P_SWAP=0 disables it.
bool dist_p2p_ready(State &st) {
    if (st.p2p != 0) return st.p2p > 0;
    Ctx &ctx = *st.ctx;
    require(ctx.world > 1 && ctx.comm, "peer memory on a non-distributed state");
    const Nccl &n = *ctx.nccl;
    const char *env = std::getenv("QSV_P2P_SWAP");
    int bad = env && env[0] == '0' ? 1 : 0;
    const size_t bytes = st.local_amps * st.amp_bytes() * static_cast<size_t>(st.batch);
    if (!bad && !st.scratch && cudaMalloc(&st.scratch, bytes) != cudaSuccess) {
        cudaGetLastError();
        st.scratch = nullptr;
        bad = 1;
    }
    // what every rank publishes: IPC handles of its two buffers (one process
    // per GPU) or, when every rank lives in this process (qsv_ctx_create_multi),
    // the raw pointers and the device they live on
    struct Pub {
        cudaIpcMemHandle_t h[2];
        void *p[2];
        int dev, pad;
    };
    Pub mine;
    std::memset(&mine, 0, sizeof mine);
    mine.dev = ctx.device;
    if (!bad) {
        st.p2p_buf[0] = st.d;
        st.p2p_buf[1] = st.scratch;
        for (int i = 0; i < 2; ++i) mine.p[i] = st.p2p_buf[i];
        for (int i = 0; i < 2 && !bad && !ctx.in_process; ++i)
            if (cudaIpcGetMemHandle(&mine.h[i], st.p2p_buf[i]) != cudaSuccess) {
                cudaGetLastError();
                bad = 1;
            }
    }
    if (agree_failures(st, bad) > 0) {
        st.p2p = -1;
        return false;
    }
    // exchange: rank r's record lands in slot r on every rank
    const int W = ctx.world;
    const size_t hb = sizeof(Pub);
    unsigned char *d_h = nullptr;
    QSV_CUDA(cudaMalloc(&d_h, hb * W));
    QSV_CUDA(cudaMemcpyAsync(d_h + hb * ctx.rank, &mine, hb, cudaMemcpyHostToDevice, ctx.stream));
    nccl_ok(n, n.GroupStart(), "GroupStart");
    for (int r = 0; r < W; ++r) {
        if (r == ctx.rank) continue;
        nccl_ok(n, n.Send(d_h + hb * ctx.rank, hb, ncclUint8, r, static_cast<ncclComm_t>(ctx.comm), ctx.stream),
                "Send");
        ctx.stat_messages += 1;
        ctx.stat_bytes += hb;
        nccl_ok(n, n.Recv(d_h + hb * r, hb, ncclUint8, r, static_cast<ncclComm_t>(ctx.comm), ctx.stream), "Recv");
    }
    nccl_ok(n, n.GroupEnd(), "GroupEnd");
    std::vector<Pub> all(static_cast<size_t>(W));
    QSV_CUDA(cudaMemcpyAsync(all.data(), d_h, hb * W, cudaMemcpyDeviceToHost, ctx.stream));
    QSV_CUDA(cudaStreamSynchronize(ctx.stream));
    cudaFree(d_h);
    std::vector<void *> table(2 * static_cast<size_t>(W), nullptr);
    for (int r = 0; r < W && !bad; ++r) {
        if (ctx.in_process && r != ctx.rank && all[r].dev != ctx.device) {
            const cudaError_t e = cudaDeviceEnablePeerAccess(all[r].dev, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) bad = 1;
            cudaGetLastError();
        }
        for (int i = 0; i < 2 && !bad; ++i) {
            if (r == ctx.rank || ctx.in_process) {
                table[static_cast<size_t>(i) * W + r] = r == ctx.rank ? st.p2p_buf[i] : all[r].p[i];
                continue;
            }
            void *ptr = nullptr;
            if (cudaIpcOpenMemHandle(&ptr, all[r].h[i], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                cudaGetLastError();
                bad = 1;
                break;
            }
            st.p2p_opened.push_back(ptr);
            table[static_cast<size_t>(i) * W + r] = ptr;
        }
    }
    if (!bad) {
        if (cudaMalloc(reinterpret_cast<void **>(&st.d_peers), table.size() * sizeof(void *)) != cudaSuccess) {
            cudaGetLastError();
            st.d_peers = nullptr;
            bad = 1;
        } else {
            QSV_CUDA(cudaMemcpy(st.d_peers, table.data(), table.size() * sizeof(void *), cudaMemcpyHostToDevice));
        }
    }
    if (agree_failures(st, bad) > 0) {
        dist_p2p_release(st);
        st.p2p = -1;
        return false;
    }
    st.p2p_cur = 0;
    st.p2p = 1;
    return true;
}

// Orders a fused pass's peer stores before anything that reads them: every
// rank's pass kernel has completed once this all-reduce (on the same
// stream) completes anywhere.
void dist_p2p_barrier(State &st) {
    Ctx &ctx = *st.ctx;
    const Nccl &n = *ctx.nccl;
    nccl_ok(n, n.AllReduce(st.d_barrier, st.d_barrier, 1, ncclFloat64, ncclSum, static_cast<ncclComm_t>(ctx.comm),
                           ctx.stream), "AllReduce");
    ctx.stat_allreduces += 1;
}

void dist_p2p_release(State &st) {
    for (void *p : st.p2p_opened) cudaIpcCloseMemHandle(p);
    st.p2p_opened.clear();
    if (st.d_peers) cudaFree(st.d_peers);
    st.d_peers = nullptr;
    if (st.d_barrier) cudaFree(st.d_barrier);
    st.d_barrier = nullptr;
    st.p2p = 0;
}

// A step's pairs apply in order (a later pair may reuse a bit of an earlier
// one, e.g. when the layout is restored); maximal runs of pairwise-disjoint
// pairs commute and go as one all-to-all each.
void dist_swap_bits(State &st, const std::vector<std::pair<int, int>> &pairs, void *, size_t) {
    std::vector<std::pair<int, int>> run;
    for (const auto &p : pairs) {
        bool clash = false;
        for (const auto &q : run) clash = clash || q.first == p.first || q.second == p.second;
        if (clash) {
            swap_disjoint(st, run);
            run.clear();
        }
        run.push_back(p);
    }
    if (!run.empty()) swap_disjoint(st, run);
}

namespace {
void swap_disjoint(State &st, const std::vector<std::pair<int, int>> &pairs) {
    Ctx &ctx = *st.ctx;
    require(ctx.world > 1 && ctx.comm, "swap on a non-distributed state");
    const Nccl &n = *ctx.nccl;
    const int m = static_cast<int>(pairs.size());
    require(m >= 1 && m <= 6, "swap: 1..6 bit pairs per step");
    const int amp = static_cast<int>(st.amp_bytes());
    // local bits ascending, each with its rank bit
    std::vector<std::pair<int, int>> pr(pairs.begin(), pairs.end());
    for (const auto &[gb, lb] : pr)
        require(gb >= st.nlocal && gb < st.n && lb >= 0 && lb < st.nlocal, "swap: bad bit pair");
    std::sort(pr.begin(), pr.end(), [](auto &a, auto &b) { return a.second < b.second; });
    BlockBits bb{};
    bb.m = m;
    unsigned own = 0;
    for (int i = 0; i < m; ++i) {
        bb.pos[i] = pr[i].second;
        own |= static_cast<unsigned>((ctx.rank >> (pr[i].first - st.nlocal)) & 1) << i;
    }
    // peers: block v goes to the rank whose swapped rank bits equal v
    std::vector<unsigned> vs;
    std::vector<int> peers;
    for (unsigned v = 0; v < (1u << m); ++v) {
        if (v == own) continue;
        int peer = ctx.rank;
        for (int i = 0; i < m; ++i) {
            const int rb = pr[i].first - st.nlocal;
            peer = (peer & ~(1 << rb)) | static_cast<int>(((v >> i) & 1u) << rb);
        }
        vs.push_back(v);
        peers.push_back(peer);
    }
    const int nv = static_cast<int>(vs.size());
    const uint64_t block = st.local_amps >> m;
    // persistent staging: two sets (send + receive each), a set <= 2 x 256 MiB
    // QSV_SWAP_STAGE_BYTES (tests): a small per-set payload forces many
    // pipelined rounds on small states
    static const uint64_t set_cap = [] {
        const char *e = std::getenv("QSV_SWAP_STAGE_BYTES");
        return e ? std::max<uint64_t>(256, std::strtoull(e, nullptr, 10)) : (256ull << 20);
    }();
    const uint64_t want = std::min<uint64_t>(block * nv, set_cap / amp);
    // elements per block per round, a power of two (rounds stay aligned)
    const uint64_t chunk = std::bit_floor(std::max<uint64_t>(1, want / nv));
    const size_t set_bytes = 2 * chunk * nv * static_cast<size_t>(amp);
    if (ctx.stage_bytes < 2 * set_bytes) {
        QSV_CUDA(cudaStreamSynchronize(ctx.stream));
        if (ctx.comm_stream) QSV_CUDA(cudaStreamSynchronize(ctx.comm_stream));
        cudaFree(ctx.stage);
        ctx.stage = nullptr;
        ctx.stage_bytes = 0;
        QSV_CUDA(cudaMalloc(&ctx.stage, 2 * set_bytes));
        ctx.stage_bytes = 2 * set_bytes;
    }
    if (!ctx.comm_stream) QSV_CUDA(cudaStreamCreateWithFlags(&ctx.comm_stream, cudaStreamNonBlocking));
    unsigned *d_vs = nullptr;
    QSV_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&d_vs), sizeof(unsigned) * nv, ctx.stream));
    QSV_CUDA(cudaMemcpyAsync(d_vs, vs.data(), sizeof(unsigned) * nv, cudaMemcpyHostToDevice, ctx.stream));
    // rounds (row, chunk) in order; round k uses staging set k % 2. The copy
    // stream issues gather(k + 1) before scatter(k), so the next chunk is
    // gathered while chunk k is on the wire; scatter(k - 1) precedes
    // gather(k + 1) on the copy stream, which frees set (k + 1) % 2.
    struct Round {
        int row;
        uint64_t e0, c;
    };
    std::vector<Round> rounds;
    for (int row = 0; row < st.batch; ++row)
        for (uint64_t e0 = 0; e0 < block; e0 += chunk) rounds.push_back({row, e0, std::min(chunk, block - e0)});
    const size_t K = rounds.size();
    std::vector<cudaEvent_t> ev_g(K), ev_c(K);
    for (size_t k = 0; k < K; ++k) {
        QSV_CUDA(cudaEventCreateWithFlags(&ev_g[k], cudaEventDisableTiming));
        QSV_CUDA(cudaEventCreateWithFlags(&ev_c[k], cudaEventDisableTiming));
    }
    auto set_ptr = [&](size_t k, int recv) {
        return static_cast<unsigned char *>(ctx.stage) + (k % 2) * set_bytes + (recv ? set_bytes / 2 : 0);
    };
    // 16-byte vectors: a c64 pair of neighbouring amplitudes moves as one
    // float4 when bit 0 is not a swapped bit (element e = amplitude pair)
    const bool pair64 = amp == 8 && bb.pos[0] >= 1 && chunk % 2 == 0;
    BlockBits bbv = bb;
    if (pair64)
        for (int i = 0; i < m; ++i) bbv.pos[i] -= 1;
    auto copy = [&](size_t k, int dir) {
        const Round &r = rounds[k];
        unsigned char *base = static_cast<unsigned char *>(st.d) + static_cast<size_t>(r.row) * st.local_amps * amp;
        unsigned char *buf = set_ptr(k, dir);
        const uint64_t cnt = pair64 ? r.c / 2 : r.c, e0 = pair64 ? r.e0 / 2 : r.e0;
        const dim3 grid(static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((cnt + 255) / 256,
                                                                                       (148 * 8 + nv - 1) / nv))),
                        static_cast<unsigned>(nv));
        if (amp == 16 || pair64)
            block_copy_kernel<double2><<<grid, 256, 0, ctx.stream>>>(reinterpret_cast<double2 *>(base),
                reinterpret_cast<double2 *>(buf), pair64 ? bbv : bb, e0, cnt, d_vs, dir);
        else
            block_copy_kernel<float2><<<grid, 256, 0, ctx.stream>>>(reinterpret_cast<float2 *>(base),
                reinterpret_cast<float2 *>(buf), bb, r.e0, r.c, d_vs, dir);
        QSV_CUDA(cudaGetLastError());
    };
    auto transfer = [&](size_t k) {
        const Round &r = rounds[k];
        QSV_CUDA(cudaStreamWaitEvent(ctx.comm_stream, ev_g[k], 0));
        unsigned char *sb = set_ptr(k, 0), *rb = set_ptr(k, 1);
        nccl_ok(n, n.GroupStart(), "GroupStart");
        for (int j = 0; j < nv; ++j) {
            nccl_ok(n, n.Send(sb + static_cast<size_t>(j) * r.c * amp, r.c * amp, ncclUint8, peers[j],
                              static_cast<ncclComm_t>(ctx.comm), ctx.comm_stream), "Send");
            ctx.stat_messages += 1;
            ctx.stat_bytes += r.c * amp;
            nccl_ok(n, n.Recv(rb + static_cast<size_t>(j) * r.c * amp, r.c * amp, ncclUint8, peers[j],
                              static_cast<ncclComm_t>(ctx.comm), ctx.comm_stream), "Recv");
        }
        nccl_ok(n, n.GroupEnd(), "GroupEnd");
        QSV_CUDA(cudaEventRecord(ev_c[k], ctx.comm_stream));
    };
    copy(0, 0);
    QSV_CUDA(cudaEventRecord(ev_g[0], ctx.stream));
    for (size_t k = 0; k < K; ++k) {
        transfer(k);
        if (k + 1 < K) {
            copy(k + 1, 0);
            QSV_CUDA(cudaEventRecord(ev_g[k + 1], ctx.stream));
        }
        QSV_CUDA(cudaStreamWaitEvent(ctx.stream, ev_c[k], 0));
        copy(k, 1);
    }
    for (size_t k = 0; k < K; ++k) {
        cudaEventDestroy(ev_g[k]);
        cudaEventDestroy(ev_c[k]);
    }
    QSV_CUDA(cudaFreeAsync(d_vs, ctx.stream));
}
} // namespace

void dist_exchange_apply(State &st, int gbit, const cplx *m, uint64_t local_cmask, bool on, bool zero_off_control) {
    Ctx &ctx = *st.ctx;
    require(ctx.world > 1 && ctx.comm, "exchange on a non-distributed state");
    require(gbit >= st.nlocal && gbit < st.n, "exchange: target is not a rank bit");
    const int amp = static_cast<int>(st.amp_bytes());
    const uint64_t total = st.local_amps * static_cast<uint64_t>(st.batch);
    const int blocks = 148 * 8;
    if (!on) { // a global control is |0> on this rank and its partner alike
        if (zero_off_control) {
            if (amp == 16) zero_kernel<double2><<<blocks, 256, 0, ctx.stream>>>(static_cast<double2 *>(st.d), total);
            else zero_kernel<float2><<<blocks, 256, 0, ctx.stream>>>(static_cast<float2 *>(st.d), total);
            QSV_CUDA(cudaGetLastError());
        }
        return;
    }
    const Nccl &n = *ctx.nccl;
    const int rb = gbit - st.nlocal;
    const int peer = ctx.rank ^ (1 << rb);
    const int b = (ctx.rank >> rb) & 1;
    const cplx a = m[b * 2 + b], c = m[b * 2 + (1 - b)];
    static const uint64_t set_cap = [] {
        const char *e = std::getenv("QSV_SWAP_STAGE_BYTES");
        return e ? std::max<uint64_t>(256, std::strtoull(e, nullptr, 10)) : (256ull << 20);
    }();
    const uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(total, std::bit_floor(set_cap / amp)));
    const size_t need = 2 * chunk * static_cast<size_t>(amp);
    if (ctx.stage_bytes < need) {
        QSV_CUDA(cudaStreamSynchronize(ctx.stream));
        if (ctx.comm_stream) QSV_CUDA(cudaStreamSynchronize(ctx.comm_stream));
        cudaFree(ctx.stage);
        ctx.stage = nullptr;
        ctx.stage_bytes = 0;
        QSV_CUDA(cudaMalloc(&ctx.stage, need));
        ctx.stage_bytes = need;
    }
    if (!ctx.comm_stream) QSV_CUDA(cudaStreamCreateWithFlags(&ctx.comm_stream, cudaStreamNonBlocking));
    struct Ev {  // destroyed on every path (an NCCL failure throws mid-loop)
        cudaEvent_t e = nullptr;
        Ev() { QSV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); }
        ~Ev() {
            if (e) cudaEventDestroy(e);
        }
    } ev_ready, ev_done;
    cudaEvent_t ready = ev_ready.e, done = ev_done.e;
    // rounds alternate between the two halves of the staging buffer; each
    // round's send reads the state chunk BEFORE its combine rewrites it
    int k = 0;
    for (uint64_t e0 = 0; e0 < total; e0 += chunk, ++k) {
        const uint64_t cnt = std::min(chunk, total - e0);
        unsigned char *mine = static_cast<unsigned char *>(st.d) + e0 * amp;
        unsigned char *recv = static_cast<unsigned char *>(ctx.stage) + (k % 2) * chunk * amp;
        QSV_CUDA(cudaEventRecord(ready, ctx.stream));
        QSV_CUDA(cudaStreamWaitEvent(ctx.comm_stream, ready, 0));
        nccl_ok(n, n.GroupStart(), "GroupStart");
        nccl_ok(n, n.Send(mine, cnt * amp, ncclUint8, peer, static_cast<ncclComm_t>(ctx.comm), ctx.comm_stream),
                "Send");
        nccl_ok(n, n.Recv(recv, cnt * amp, ncclUint8, peer, static_cast<ncclComm_t>(ctx.comm), ctx.comm_stream),
                "Recv");
        nccl_ok(n, n.GroupEnd(), "GroupEnd");
        ctx.stat_messages += 1;
        ctx.stat_bytes += cnt * amp;
        QSV_CUDA(cudaEventRecord(done, ctx.comm_stream));
        QSV_CUDA(cudaStreamWaitEvent(ctx.stream, done, 0));
        // element e of the flat (row, index) range: only its bits below nlocal
        // (its local index) meet the control mask
        const int g = static_cast<int>(std::min<uint64_t>((cnt + 255) / 256, blocks));
        if (amp == 16)
            exchange_combine_kernel<double, double2><<<g, 256, 0, ctx.stream>>>(
                reinterpret_cast<double2 *>(mine), reinterpret_cast<const double2 *>(recv), cnt, e0, local_cmask,
                zero_off_control, a.real(), a.imag(), c.real(), c.imag());
        else
            exchange_combine_kernel<float, float2><<<g, 256, 0, ctx.stream>>>(
                reinterpret_cast<float2 *>(mine), reinterpret_cast<const float2 *>(recv), cnt, e0, local_cmask,
                zero_off_control, a.real(), a.imag(), c.real(), c.imag());
        QSV_CUDA(cudaGetLastError());
    }
    QSV_CUDA(cudaStreamSynchronize(ctx.stream));
}

} // namespace qsv
