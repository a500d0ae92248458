// TEST INFRASTRUCTURE ONLY -- a stand-in for libnccl.so.2 that lets the
// engine's multi-rank path (dist.cu: qubit swaps, all-reduced reductions,
// the distributed schedule) run as several processes sharing ONE GPU.
//
// NCCL itself refuses two ranks on one device, and kernels that wait on each
// other across processes on one GPU are unsafe; this shim therefore does all
// communication from the HOST: at ncclGroupEnd every rank synchronises its
// stream, publishes CUDA IPC handles of its send buffers in a POSIX
// shared-memory block, meets the other ranks at a shared-memory barrier, and
// copies what it receives with cudaMemcpy from the peers' IPC-mapped buffers.
// No kernel ever waits for another process. Only what dist.cu uses is
// implemented: GetUniqueId, CommInitRank, CommDestroy, Send/Recv inside
// GroupStart/GroupEnd, AllReduce (float64, sum), GetErrorString.
// Selected with QSV_NCCL_LIB=<this .so>; never used by the product.
//
// Only the CUDA DRIVER API is used (the calling thread's current context is
// the runtime's primary context): a second runtime instance would not share
// libqsv's view of its streams.
#include <cuda.h>
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

namespace {
constexpr int kMaxRanks = 16;
constexpr size_t kRedDoubles = 1 << 17;
constexpr size_t kArea = 8u << 20;

struct Slot {
    uint64_t off, bytes;
    int valid;
};
// Point-to-point is pairwise (only the two ranks of a send / receive meet:
// ranks whose global control is |0> skip an exchange, as with NCCL): src
// posts its bytes and bumps seq[src][dst]; dst waits for that sequence
// number, copies, and acknowledges in ack[src][dst]; src's staging area is
// reused only once every receiver has acknowledged.
struct Ctl {
    std::atomic<int> joined;
    std::atomic<int> count;
    std::atomic<int> gen;
    Slot send[kMaxRanks][kMaxRanks];  // [src][dst]
    std::atomic<uint64_t> seq[kMaxRanks][kMaxRanks];
    std::atomic<uint64_t> ack[kMaxRanks][kMaxRanks];
    double red[kMaxRanks][kRedDoubles];
    unsigned char area[kMaxRanks][kArea];
};
struct Comm {
    Ctl *ctl = nullptr;
    int rank = 0, nranks = 1;
    char name[128] = {};
    uint64_t sent[kMaxRanks] = {}, recvd[kMaxRanks] = {};  // this rank's sequence numbers per peer
};
struct Op {
    bool send;
    void *buf;
    size_t bytes;
    int peer;
    Comm *comm;
    CUstream stream;
};
thread_local int g_depth = 0;
thread_local std::vector<Op> g_ops;

int elem_bytes(int t) {
    switch (t) {
    case 0: case 1: return 1;
    case 2: case 3: case 7: return 4;
    case 4: case 5: case 8: return 8;
    case 6: case 9: return 2;
    default: return 1;
    }
}

void barrier(Comm *c) {
    Ctl *k = c->ctl;
    const int g = k->gen.load();
    if (k->count.fetch_add(1) == c->nranks - 1) {
        k->count.store(0);
        k->gen.fetch_add(1);
    } else {
        while (k->gen.load() == g) sched_yield();
    }
}

bool cu_ok(CUresult r, const char *what) {
    if (r == CUDA_SUCCESS) return true;
    const char *name = nullptr;
    cuGetErrorName(r, &name);
    std::fprintf(stderr, "fake nccl: %s failed: %s\n", what, name ? name : "?");
    return false;
}

int run_group(std::vector<Op> &ops) {
    if (ops.empty()) return 0;
    Comm *c = ops[0].comm;
    Ctl *k = c->ctl;
    for (const Op &o : ops)
        if (!cu_ok(cuCtxSynchronize(), "cuCtxSynchronize") || !cu_ok(cuStreamSynchronize(o.stream), "cuStreamSynchronize"))
            return 1;
    uint64_t used = 0;
    for (const Op &o : ops) {
        if (!o.send) continue;
        if (used + o.bytes > kArea) {
            std::fprintf(stderr, "fake nccl: more than %zu bytes sent per rank per group\n", kArea);
            return 4;
        }
        if (!cu_ok(cuMemcpyDtoH(k->area[c->rank] + used, reinterpret_cast<CUdeviceptr>(o.buf), o.bytes),
                   "cuMemcpyDtoH"))
            return 1;
        Slot &sl = k->send[c->rank][o.peer];
        sl.off = used;
        sl.bytes = o.bytes;
        sl.valid = 1;
        k->seq[c->rank][o.peer].store(++c->sent[o.peer], std::memory_order_release);
        used += (o.bytes + 255) & ~uint64_t(255);
    }
    int rc = 0;
    for (const Op &o : ops) {
        if (o.send) continue;
        const uint64_t want = ++c->recvd[o.peer];
        while (k->seq[o.peer][c->rank].load(std::memory_order_acquire) < want) sched_yield();
        Slot &sl = k->send[o.peer][c->rank];
        if (!sl.valid || sl.bytes != o.bytes) {
            std::fprintf(stderr, "fake nccl: unmatched receive from rank %d\n", o.peer);
            rc = 4;
        } else if (!cu_ok(cuMemcpyHtoD(reinterpret_cast<CUdeviceptr>(o.buf), k->area[o.peer] + sl.off, o.bytes),
                          "cuMemcpyHtoD"))
            rc = 1;
        k->ack[o.peer][c->rank].store(want, std::memory_order_release);
    }
    if (cuCtxSynchronize() != CUDA_SUCCESS) rc = 1;  // the copies land before the caller's stream goes on
    for (const Op &o : ops)  // the staging area is reused by the next group: wait for every receiver
        if (o.send)
            while (k->ack[c->rank][o.peer].load(std::memory_order_acquire) < c->sent[o.peer]) sched_yield();
    return rc;
}
} // namespace

extern "C" {
typedef struct {
    char internal[128];
} ncclUniqueId;

int ncclGetUniqueId(ncclUniqueId *id) {
    std::random_device rd;
    std::memset(id, 0, sizeof(*id));
    std::snprintf(id->internal, sizeof(id->internal), "/qsv_fake_nccl_%d_%08x%08x", static_cast<int>(getpid()), rd(), rd());
    return 0;
}

int ncclCommInitRank(void **comm, int nranks, ncclUniqueId id, int rank) {
    if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) return 4;
    auto *c = new Comm();
    c->rank = rank;
    c->nranks = nranks;
    std::memcpy(c->name, id.internal, sizeof(c->name));
    const int fd = shm_open(c->name, O_CREAT | O_RDWR, 0600);
    if (fd < 0 || ftruncate(fd, sizeof(Ctl)) != 0) return 2;
    void *m = mmap(nullptr, sizeof(Ctl), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED) return 2;
    c->ctl = static_cast<Ctl *>(m);
    c->ctl->joined.fetch_add(1);
    while (c->ctl->joined.load() < nranks) sched_yield();
    *comm = c;
    return 0;
}

// One process driving every rank (qsv_ctx_create_multi): the ranks share one
// control block; each rank's calls still come from its own host thread
// (qsv's per-rank workers), so the barriers above work unchanged.
int ncclCommInitAll(void **comms, int ndev, const int *) {
    if (ndev < 1 || ndev > kMaxRanks) return 4;
    ncclUniqueId id;
    ncclGetUniqueId(&id);
    for (int r = 0; r < ndev; ++r) {
        auto *c = new Comm();
        c->rank = r;
        c->nranks = ndev;
        std::memcpy(c->name, id.internal, sizeof(c->name));
        const int fd = shm_open(c->name, O_CREAT | O_RDWR, 0600);
        if (fd < 0 || ftruncate(fd, sizeof(Ctl)) != 0) return 2;
        void *m = mmap(nullptr, sizeof(Ctl), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
        close(fd);
        if (m == MAP_FAILED) return 2;
        c->ctl = static_cast<Ctl *>(m);
        c->ctl->joined.fetch_add(1);
        comms[r] = c;
    }
    return 0;
}

int ncclCommDestroy(void *comm) {
    auto *c = static_cast<Comm *>(comm);
    barrier(c);
    if (c->rank == 0) shm_unlink(c->name);
    munmap(c->ctl, sizeof(Ctl));
    delete c;
    return 0;
}

int ncclGroupStart() {
    ++g_depth;
    return 0;
}

int ncclGroupEnd() {
    if (--g_depth > 0) return 0;
    std::vector<Op> ops;
    ops.swap(g_ops);
    return run_group(ops);
}

static int enqueue(Op o) {
    g_ops.push_back(o);
    if (g_depth == 0) {
        std::vector<Op> ops;
        ops.swap(g_ops);
        return run_group(ops);
    }
    return 0;
}

int ncclSend(const void *buf, size_t count, int type, int peer, void *comm, CUstream stream) {
    return enqueue({true, const_cast<void *>(buf), count * elem_bytes(type), peer, static_cast<Comm *>(comm), stream});
}

int ncclRecv(void *buf, size_t count, int type, int peer, void *comm, CUstream stream) {
    return enqueue({false, buf, count * elem_bytes(type), peer, static_cast<Comm *>(comm), stream});
}

int ncclAllReduce(const void *send, void *recv, size_t count, int type, int op, void *comm, CUstream stream) {
    auto *c = static_cast<Comm *>(comm);
    if (type != 8 || op != 0 || count > kRedDoubles) return 5;  // float64 sum only
    if (cuCtxSynchronize() != CUDA_SUCCESS || cuStreamSynchronize(stream) != CUDA_SUCCESS) return 1;
    if (cuMemcpyDtoH(c->ctl->red[c->rank], reinterpret_cast<CUdeviceptr>(send), count * 8) != CUDA_SUCCESS) return 1;
    barrier(c);
    std::vector<double> acc(count, 0.0);
    for (int r = 0; r < c->nranks; ++r)
        for (size_t i = 0; i < count; ++i) acc[i] += c->ctl->red[r][i];

    barrier(c);
    // a pageable HtoD returns before its DMA lands: wait for it, or the
    // caller's stream can read the buffer first
    if (cuMemcpyHtoD(reinterpret_cast<CUdeviceptr>(recv), acc.data(), count * 8) != CUDA_SUCCESS) return 1;
    if (cuCtxSynchronize() != CUDA_SUCCESS) return 1;
    return 0;
}

const char *ncclGetErrorString(int r) {
    static const char *msg[] = {"ncclSuccess", "fake nccl: CUDA error", "fake nccl: shared memory error",
                                "fake nccl: internal error", "fake nccl: invalid argument", "fake nccl: unsupported"};
    return (r >= 0 && r <= 5) ? msg[r] : "fake nccl: unknown error";
}
}
