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
#include <cstdlib>
#include <cstring>
#include <string>

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
    return n;
}

void nccl_ok(const Nccl &n, ncclResult_t r, const char *what) {
    if (r != 0) fail(QSV_ERR_TRANSPORT, std::string("NCCL ") + what + ": " + n.GetErrorString(r));
}

// The m local bits of a swap step (ascending positions) and one block's
// values: element e of block v <-> the local index with v's bits deposited
// at those positions.
struct BlockBits {
    int m;
    int pos[8];
};
__device__ __forceinline__ uint64_t deposit(uint64_t e, const BlockBits &bb, unsigned v) {
    uint64_t x = e;
    for (int i = 0; i < bb.m; ++i) {
        const int p = bb.pos[i];
        x = ((x >> p) << (p + 1)) | (static_cast<uint64_t>((v >> i) & 1u) << p) | (x & ((1ull << p) - 1));
    }
    return x;
}
// gather (dir 0: state -> staging) or scatter (dir 1) of `count` elements
// starting at e0 of every block listed in vs[0..nv) (slot j <-> vs[j])
template <typename V>
__global__ void block_copy_kernel(V *__restrict__ state, V *__restrict__ stage, BlockBits bb, uint64_t e0,
                                  uint64_t count, const unsigned *__restrict__ vs, int nv, int dir) {
    const uint64_t total = count * static_cast<uint64_t>(nv);
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(i / count);
        const uint64_t e = e0 + (i - static_cast<uint64_t>(j) * count);
        const uint64_t idx = deposit(e, bb, vs[j]);
        if (dir == 0) stage[i] = state[idx];
        else state[idx] = stage[i];
    }
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

void nccl_destroy(Ctx &ctx) {
    if (ctx.stage) {
        cudaStreamSynchronize(ctx.stream);
        cudaFree(ctx.stage);
        ctx.stage = nullptr;
        ctx.stage_bytes = 0;
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
}

namespace {
void swap_disjoint(State &st, const std::vector<std::pair<int, int>> &pairs);
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
    // persistent staging: send + receive halves, up to 512 MiB each
    const uint64_t want = std::min<uint64_t>(block * nv, (512ull << 20) / amp);
    const uint64_t chunk = std::max<uint64_t>(1, want / nv);  // elements per block per round
    const size_t need = 2 * chunk * nv * static_cast<size_t>(amp);
    if (ctx.stage_bytes < need) {
        QSV_CUDA(cudaStreamSynchronize(ctx.stream));
        cudaFree(ctx.stage);
        ctx.stage = nullptr;
        ctx.stage_bytes = 0;
        QSV_CUDA(cudaMalloc(&ctx.stage, need));
        ctx.stage_bytes = need;
    }
    unsigned char *sbuf = static_cast<unsigned char *>(ctx.stage);
    unsigned char *rbuf = sbuf + chunk * nv * amp;
    unsigned *d_vs = nullptr;
    QSV_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&d_vs), sizeof(unsigned) * nv, ctx.stream));
    QSV_CUDA(cudaMemcpyAsync(d_vs, vs.data(), sizeof(unsigned) * nv, cudaMemcpyHostToDevice, ctx.stream));
    for (int row = 0; row < st.batch; ++row) {
        unsigned char *base = static_cast<unsigned char *>(st.d) + static_cast<size_t>(row) * st.local_amps * amp;
        for (uint64_t e0 = 0; e0 < block; e0 += chunk) {
            const uint64_t c = std::min(chunk, block - e0);
            const int blocks = static_cast<int>(std::min<uint64_t>((c * nv + 255) / 256, 148 * 8));
            if (amp == 16)
                block_copy_kernel<double2><<<blocks, 256, 0, ctx.stream>>>(reinterpret_cast<double2 *>(base),
                    reinterpret_cast<double2 *>(sbuf), bb, e0, c, d_vs, nv, 0);
            else
                block_copy_kernel<float2><<<blocks, 256, 0, ctx.stream>>>(reinterpret_cast<float2 *>(base),
                    reinterpret_cast<float2 *>(sbuf), bb, e0, c, d_vs, nv, 0);
            QSV_CUDA(cudaGetLastError());
            nccl_ok(n, n.GroupStart(), "GroupStart");
            for (int j = 0; j < nv; ++j) {
                nccl_ok(n, n.Send(sbuf + static_cast<size_t>(j) * c * amp, c * amp, ncclUint8, peers[j],
                                  static_cast<ncclComm_t>(ctx.comm), ctx.stream), "Send");
                nccl_ok(n, n.Recv(rbuf + static_cast<size_t>(j) * c * amp, c * amp, ncclUint8, peers[j],
                                  static_cast<ncclComm_t>(ctx.comm), ctx.stream), "Recv");
            }
            nccl_ok(n, n.GroupEnd(), "GroupEnd");
            if (amp == 16)
                block_copy_kernel<double2><<<blocks, 256, 0, ctx.stream>>>(reinterpret_cast<double2 *>(base),
                    reinterpret_cast<double2 *>(rbuf), bb, e0, c, d_vs, nv, 1);
            else
                block_copy_kernel<float2><<<blocks, 256, 0, ctx.stream>>>(reinterpret_cast<float2 *>(base),
                    reinterpret_cast<float2 *>(rbuf), bb, e0, c, d_vs, nv, 1);
            QSV_CUDA(cudaGetLastError());
        }
    }
    QSV_CUDA(cudaFreeAsync(d_vs, ctx.stream));
}
} // namespace

} // namespace qsv
