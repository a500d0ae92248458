// NVRTC compilation and loading of specialised pass kernels (codegen.cpp).
//
// libnvrtc is dlopen'ed (the CUDA 12.9 toolkit's, or the one torch ships) so
// libqsv.so itself still loads on GPU-less hosts; kernels are compiled for
// sm_100a only, loaded with cudaLibraryLoadData and launched like any other
// kernel. Compiled cubins are cached in-process and, when writable, on disk
// ($QSV_JIT_CACHE or ~/.cache/qsv_jit) keyed by a hash of the source; the
// cache is an optimisation only -- nothing depends on it persisting.
#include <dlfcn.h>
#include <sys/stat.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "qsv_internal.hpp"

namespace qsv {

std::string generate_pass_source(const PassHost &ph, int dtype, const std::string &name, int *threads, bool dbuf,
                                 bool zsum = false, size_t *smem = nullptr, bool gout = false);
int dbuf_stages(const PassHost &ph, int dtype);
std::string generate_pair_source(const PassHost &A, const PassHost &B, int dtype, const std::string &name,
                                 int *threads, bool dbuf, size_t *smem = nullptr);

namespace {

typedef int nvrtcResult;
typedef struct _nvrtcProgram *nvrtcProgram;

struct Nvrtc {
    void *h = nullptr;
    nvrtcResult (*CreateProgram)(nvrtcProgram *, const char *, const char *, int, const char *const *,
                                 const char *const *) = nullptr;
    nvrtcResult (*CompileProgram)(nvrtcProgram, int, const char *const *) = nullptr;
    nvrtcResult (*GetCUBINSize)(nvrtcProgram, size_t *) = nullptr;
    nvrtcResult (*GetCUBIN)(nvrtcProgram, char *) = nullptr;
    nvrtcResult (*GetProgramLogSize)(nvrtcProgram, size_t *) = nullptr;
    nvrtcResult (*GetProgramLog)(nvrtcProgram, char *) = nullptr;
    nvrtcResult (*DestroyProgram)(nvrtcProgram *) = nullptr;
    const char *(*GetErrorString)(nvrtcResult) = nullptr;
};

Nvrtc *nvrtc() {
    static Nvrtc *inst = nullptr;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (inst) return inst;
    auto *n = new Nvrtc();
    const char *env = std::getenv("QSV_NVRTC_LIB");
    const char *cands[] = {env, "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so.12", "libnvrtc.so"};
    for (const char *c : cands) {
        if (!c) continue;
        n->h = dlopen(c, RTLD_NOW | RTLD_LOCAL);
        if (n->h) break;
    }
    if (!n->h) {
        delete n;
        fail(QSV_ERR_INTERNAL, "NVRTC not found (set QSV_NVRTC_LIB to libnvrtc.so.12)");
    }
#define LOAD(f)                                                                                                        \
    n->f = reinterpret_cast<decltype(n->f)>(dlsym(n->h, "nvrtc" #f));                                                  \
    if (!n->f) fail(QSV_ERR_INTERNAL, "NVRTC symbol missing: nvrtc" #f);
    LOAD(CreateProgram) LOAD(CompileProgram) LOAD(GetCUBINSize) LOAD(GetCUBIN) LOAD(GetProgramLogSize)
    LOAD(GetProgramLog) LOAD(DestroyProgram) LOAD(GetErrorString)
#undef LOAD
    inst = n;
    return inst;
}

uint64_t fnv64(const std::string &s) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (unsigned char c : s) {
        h ^= c;
        h *= 0x100000001b3ull;
    }
    return h;
}

std::string cache_dir() {
    const char *env = std::getenv("QSV_JIT_CACHE");
    if (env) return env;
    const char *home = std::getenv("HOME");
    return std::string(home ? home : "/tmp") + "/.cache/qsv_jit";
}

std::vector<char> compile(const std::string &src, const std::string &key) {
    static std::map<std::string, std::vector<char>> mem;
    static std::mutex mu;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = mem.find(key);
        if (it != mem.end()) return it->second;
    }
    const std::string path = cache_dir() + "/" + key + ".cubin";
    {
        std::ifstream f(path, std::ios::binary);
        if (f) {
            std::vector<char> b((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
            if (!b.empty()) {
                std::lock_guard<std::mutex> lk(mu);
                mem[key] = b;
                return b;
            }
        }
    }
    Nvrtc *n = nvrtc();
    nvrtcProgram prog = nullptr;
    // the source goes next to the cubin and names the program, so -lineinfo
    // points ncu (--import-source) at the generated code
    const std::string dir0 = cache_dir();
    mkdir((dir0.substr(0, dir0.rfind('/'))).c_str(), 0755);
    mkdir(dir0.c_str(), 0755);
    const std::string src_path = dir0 + "/" + key + ".cu";
    {
        std::ofstream f(src_path);
        if (f) f << src;
    }
    if (n->CreateProgram(&prog, src.c_str(), src_path.c_str(), 0, nullptr, nullptr) != 0)
        fail(QSV_ERR_INTERNAL, "nvrtcCreateProgram failed");
    const char *opts[] = {"-arch=sm_100a", "-std=c++17", "-default-device", "-lineinfo", "--extra-device-vectorization"};
    const nvrtcResult rc = n->CompileProgram(prog, 5, opts);
    if (rc != 0) {
        size_t ls = 0;
        n->GetProgramLogSize(prog, &ls);
        std::string log(ls, '\0');
        n->GetProgramLog(prog, log.data());
        n->DestroyProgram(&prog);
        fail(QSV_ERR_INTERNAL, std::string("NVRTC compile failed: ") + n->GetErrorString(rc) + "\n" + log.substr(0, 4000));
    }
    size_t sz = 0;
    n->GetCUBINSize(prog, &sz);
    std::vector<char> cubin(sz);
    n->GetCUBIN(prog, cubin.data());
    n->DestroyProgram(&prog);
    {
        std::lock_guard<std::mutex> lk(mu);
        mem[key] = cubin;
    }
    // best-effort disk cache (atomic rename)
    const std::string dir = cache_dir();
    mkdir((dir.substr(0, dir.rfind('/'))).c_str(), 0755);
    mkdir(dir.c_str(), 0755);
    const std::string tmp = path + ".tmp" + std::to_string(reinterpret_cast<uintptr_t>(&cubin));
    {
        std::ofstream f(tmp, std::ios::binary);
        if (f) f.write(cubin.data(), static_cast<std::streamsize>(cubin.size()));
    }
    std::rename(tmp.c_str(), path.c_str());
    return cubin;
}

} // namespace

struct JitKernel {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kernel = nullptr;
};

namespace {
JitKernel load_kernel(const std::string &src, const std::string &name) {
    char key[32];
    std::snprintf(key, sizeof key, "p%016llx%08zx", static_cast<unsigned long long>(fnv64(src)), src.size());
    std::vector<char> cubin = compile(src, key);
    static std::map<std::string, JitKernel> loaded;
    static std::mutex mu;
    JitKernel jk;
    int dev = 0;
    QSV_CUDA(cudaGetDevice(&dev));
    const std::string lkey = std::string(key) + ":" + std::to_string(dev);
    std::lock_guard<std::mutex> lk(mu);
    auto it = loaded.find(lkey);
    if (it != loaded.end()) return it->second;
    QSV_CUDA(cudaLibraryLoadData(&jk.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    QSV_CUDA(cudaLibraryGetKernel(&jk.kernel, jk.lib, name.c_str()));
    loaded[lkey] = jk;
    return jk;
}

bool use_prefetch(const PassHost &ph, int dtype) { return pass_prefetches(ph, dtype); }
} // namespace

// Double-buffered (prefetching) tiles hide HBM latency; a pass whose gate
// math outweighs its memory time runs better single-buffered, with a CTA
// more per SM (more warps to hide the FP64 / FMA latencies). Heavy = more
// dense register-group matrices than 3x the tile bits (the QFT passes: ~8
// per 11-bit tile, prefetching; the brickwork passes of cfg4: 40-130).
// Interleaved A/B, cfg4 family: 32q 912 -> 887 ms, 28q 51.9 -> 49.6 ms; QFT
// with prefetching off 22.6 -> 26.2 ms. QSV_PREFETCH=0 / 1 forces it.
bool pass_prefetches(const PassHost &ph, int dtype) {
    const int amp0 = dtype == QSV_C64 ? 8 : 16;
    const char *pe = std::getenv("QSV_PREFETCH");
    if (pe && pe[0] == '0') return false;
    const bool fits = (2 * (static_cast<size_t>(amp0) << ph.K) <= (64u << 10)) && (1 << ph.K) * amp0 >= 16 * 32 &&
                      !ph.synth;
    if (!fits) return false;
    if (pe && pe[0] == '1') return true;
    int dense = 0;
    for (const HostOp &op : ph.ops)
        if (op.code == OP_DENSE1 || op.code == OP_DENSE1R || op.code == OP_DENSE2) ++dense;
    return dense <= 3 * ph.K;
}

void jit_prepare_pair(DevPass &head, const PassHost &a, const PassHost &b, int dtype, int sm_count) {
    (void)sm_count;
    const bool dbuf = use_prefetch(a, dtype);
    require(dbuf == use_prefetch(b, dtype), "jit: super-pass halves differ in staging");
    int threads = 0;
    size_t smem = 0;
    const std::string src = generate_pair_source(a, b, dtype, "qsv_pair", &threads, dbuf, &smem);
    const JitKernel jk = load_kernel(src, "qsv_pair");
    head.jit_pair = reinterpret_cast<const void *>(jk.kernel);
    head.threads = threads;
    head.smem = smem;
    head.pair = 1;
    head.chunk_tiles_log = a.chunk_bits - a.K;
    int dev = 0, optin = 0;
    QSV_CUDA(cudaGetDevice(&dev));
    QSV_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa{};
    QSV_CUDA(cudaFuncGetAttributes(&fa, head.jit_pair));
    QSV_CUDA(cudaFuncSetAttribute(head.jit_pair, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  optin - static_cast<int>(fa.sharedSizeBytes)));
    head.jit_regs = fa.numRegs;
    head.jit_spill = static_cast<int>(fa.localSizeBytes);
}

// Compiles (or fetches) the specialised kernel of one pass and fills dp
// (zsum: the variant with the fused <Z> epilogue, dp.jit_z / dp.grid_z).
static void jit_build(DevPass &dp, const PassHost &ph, int dtype, int sm_count, bool zsum) {
    const std::string name = "qsv_pass";
    int threads = 256;
    // prefetch (two shared tiles, cp.async of the next tile in flight) when
    // both buffers fit in 64 KiB: K <= 11 for complex128, K <= 12 for complex64
    const bool dbuf = use_prefetch(ph, dtype);
    size_t smem = 0;
    std::string src = generate_pass_source(ph, dtype, name, &threads, dbuf, zsum, &smem);
    const JitKernel jk = load_kernel(src, name);
    int dev = 0;
    QSV_CUDA(cudaGetDevice(&dev));
    const int amp = dtype == QSV_C64 ? 8 : 16;
    const void *kern = reinterpret_cast<const void *>(jk.kernel);
    if (zsum) {
        require(threads == dp.threads, "jit: <Z> variant changed the CTA shape");
        int optin = 0;
        QSV_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        cudaFuncAttributes fa{};
        QSV_CUDA(cudaFuncGetAttributes(&fa, kern));
        QSV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      optin - static_cast<int>(fa.sharedSizeBytes)));
        int blocks = 0;
        QSV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, dp.threads, dp.smem));
        dp.jit_z = kern;
        dp.grid_z = std::max(1, blocks) * sm_count;
        return;
    }
    dp.jit = kern;
    dp.threads = threads;
    // groups between the first (loads from HBM) and the last (stores to HBM)
    // exchange amplitudes through a shared tile; a one-group pass needs none
    dp.smem = smem;
    int optin = 0;
    QSV_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa{};
    QSV_CUDA(cudaFuncGetAttributes(&fa, dp.jit));
    QSV_CUDA(cudaFuncSetAttribute(dp.jit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  optin - static_cast<int>(fa.sharedSizeBytes)));
    int blocks = 0;
    QSV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, dp.jit, dp.threads, dp.smem));
    dp.grid = std::max(1, blocks) * sm_count;
    dp.jit_regs = fa.numRegs;
    dp.jit_spill = static_cast<int>(fa.localSizeBytes);
}

// Source of a pass's specialised kernel (diagnostics / tests).
std::string jit_source(const PassHost &ph, int dtype) {
    int threads = 0;
    return generate_pass_source(ph, dtype, "qsv_pass", &threads, use_prefetch(ph, dtype));
}

std::string jit_gout_source(const PassHost &ph, int dtype) {
    int threads = 0;
    return generate_pass_source(ph, dtype, "qsv_pass", &threads, use_prefetch(ph, dtype), false, nullptr, true);
}

std::string jit_pair_source(const PassHost &a, const PassHost &b, int dtype) {
    int threads = 0;
    return generate_pair_source(a, b, dtype, "qsv_pair", &threads, use_prefetch(a, dtype));
}

void jit_prepare(DevPass &dp, const PassHost &ph, int dtype, int sm_count) { jit_build(dp, ph, dtype, sm_count, false); }

void jit_prepare_gout(DevPass &dp, const PassHost &ph, int dtype, int sm_count) {
    (void)sm_count;
    int threads = 0;
    size_t smem = 0;
    const std::string src =
        generate_pass_source(ph, dtype, "qsv_pass", &threads, use_prefetch(ph, dtype), false, &smem, true);
    require(threads == dp.threads && smem == dp.smem, "jit: peer-memory variant changed the CTA shape");
    const JitKernel jk = load_kernel(src, "qsv_pass");
    const void *kern = reinterpret_cast<const void *>(jk.kernel);
    int dev = 0, optin = 0;
    QSV_CUDA(cudaGetDevice(&dev));
    QSV_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa{};
    QSV_CUDA(cudaFuncGetAttributes(&fa, kern));
    QSV_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  optin - static_cast<int>(fa.sharedSizeBytes)));
    dp.jit_gout = kern;
}
void jit_prepare_z(DevPass &dp, const PassHost &ph, int dtype, int sm_count) { jit_build(dp, ph, dtype, sm_count, true); }

namespace {
// Kernel parameters of a generated pass (codegen.cpp Args, same layout).
struct JArgs {
    void *state;
    uint64_t row_stride, rank_base, tiles_per_row, total_tiles;
    const void *tables;
    const void *enc_table;
    int batch;
    int tpc;             // > 0: each CTA runs a block of tpc consecutive tiles
    void *out;
    double *zout;        // fused <Z> epilogue: batch x (K + 1) sums
    const void *prefix;  // synthesising pass: product-state vectors
    void *const *peers;  // peer-memory stores: destination buffer per rank
    uint64_t out_lconst;
    int out_rconst;
};

JArgs make_args(const DevPass &dp, void *state, void *out, int rows) {
    JArgs a{};
    a.state = state;
    a.out = out;
    a.row_stride = dp.args.row_stride;
    a.rank_base = dp.args.rank_base;
    a.tiles_per_row = dp.args.tiles_per_row;
    a.total_tiles = dp.args.tiles_per_row * static_cast<uint64_t>(rows);
    a.tables = dp.args.tables;
    a.enc_table = dp.args.enc_table;
    a.batch = dp.args.batch;
    a.prefix = dp.args.prefix;
    return a;
}

// A few tiles per CTA rather than one persistent wave: CTAs that start and
// retire at different times keep HBM reads and writes interleaved, where a
// persistent grid moves in lock-step read / compute / write phases (measured
// on cfg3 30q: 29.7 -> 23.1 ms for 4 passes; 128-byte runs at large strides
// suffer most, scripts/micro/runs.cu).
void launch_tiles(const void *kern, const DevPass &dp, JArgs &a, int grid_cap, cudaStream_t s) {
    require(kern != nullptr, "jit: kernel variant not prepared");
    uint64_t grid = std::min<uint64_t>(a.total_tiles, static_cast<uint64_t>(std::max(grid_cap, 1)));
    // tiles per CTA: 4 on large states; small ones (a few tiles per
    // resident CTA slot) need every tile in flight at once -- measured:
    // cfg1 20q (512 tiles) 59 -> 51 us with 1, 22q (2048 tiles) best with 2,
    // cfg2 (4096 tiles) and >= 24q best with 4
    static const int tpc_env = [] {
        const char *e = std::getenv("QSV_TILES_PER_CTA");
        return e ? std::atoi(e) : -1;
    }();
    const uint64_t cap = static_cast<uint64_t>(std::max(grid_cap, 1));
    const int tpc = tpc_env >= 0 ? tpc_env : a.total_tiles <= 2 * cap ? 1 : a.total_tiles <= 8 * cap ? 2 : 4;
    static const bool blocked = [] {
        const char *e = std::getenv("QSV_TILE_ORDER");
        return !(e && e[0] == 's');
    }();
    if (tpc > 0) {
        grid = std::min<uint64_t>(a.total_tiles, std::max<uint64_t>(grid, (a.total_tiles + tpc - 1) / tpc));
        if (blocked) a.tpc = static_cast<int>((a.total_tiles + grid - 1) / grid);
    }
    void *args[] = {&a};
    QSV_CUDA(cudaLaunchKernel(kern, dim3(static_cast<unsigned>(grid)), dim3(dp.threads), args, dp.smem, s));
}
} // namespace

void launch_jit(const DevPass &dp, void *state, void *out, int rows, cudaStream_t s, double *zout) {
    JArgs a = make_args(dp, state, out, rows);
    a.zout = zout;
    launch_tiles(zout ? dp.jit_z : dp.jit, dp, a, zout ? dp.grid_z : dp.grid, s);
}

void launch_gout(const DevPass &dp, void *state, int rows, void *const *peers, uint64_t out_lconst, int out_rconst,
                 cudaStream_t s) {
    JArgs a = make_args(dp, state, state, rows);
    a.peers = peers;
    a.out_lconst = out_lconst;
    a.out_rconst = out_rconst;
    launch_tiles(dp.jit_gout, dp, a, dp.grid, s);
}

} // namespace qsv

namespace qsv {
void launch_pair(const DevPass &head, const DevPass &tail, void *state, void *out, int rows, unsigned *sync,
                 uint64_t nchunks, cudaStream_t s) {
    JArgs a{}, b{};
    struct Pair {
        unsigned *sync;
        uint64_t nchunks;
        int chunk_tiles_log;
        int tpi;
        int lookahead;
    } q{};
    const DevPass *dps[2] = {&head, &tail};
    JArgs *as[2] = {&a, &b};
    for (int i = 0; i < 2; ++i) {
        JArgs &x = *as[i];
        const DevPass &dp = *dps[i];
        x.state = state;
        x.out = i == 0 ? state : out;
        x.row_stride = dp.args.row_stride;
        x.rank_base = dp.args.rank_base;
        x.tiles_per_row = dp.args.tiles_per_row;
        x.total_tiles = dp.args.tiles_per_row * static_cast<uint64_t>(rows);
        x.tables = dp.args.tables;
        x.batch = rows;
    }
    static const int look = [] {
        const char *e = std::getenv("QSV_SUPER_LOOKAHEAD");
        return e ? std::max(1, std::atoi(e)) : 2;
    }();
    q.sync = sync;
    q.nchunks = nchunks;
    q.chunk_tiles_log = head.chunk_tiles_log;
    static const int tpi = [] {
        const char *e = std::getenv("QSV_SUPER_TPI");
        return e ? std::max(1, std::atoi(e)) : 4;
    }();
    q.tpi = std::min(tpi, 1 << head.chunk_tiles_log);
    q.lookahead = look;
    const uint64_t ipc = (1ull << head.chunk_tiles_log) / static_cast<uint64_t>(q.tpi);
    const uint64_t items = (nchunks + static_cast<uint64_t>(look)) * 2 * ipc;
    require(items < (1ull << 32), "super-pass: too many items");
    void *args[] = {&a, &b, &q};
    QSV_CUDA(cudaLaunchKernel(head.jit_pair, dim3(static_cast<unsigned>(items)), dim3(head.threads), args, head.smem,
                              s));
}
} // namespace qsv
