// Internal declarations shared by the host runtime (C++) and the CUDA
// kernels of the qsv engine. Not part of the ABI (include/qsv.h is).
#pragma once

#include <cuda_runtime.h>

#include <complex>
#include <map>
#include <mutex>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/qsv.h"

namespace qsv {

using cplx = std::complex<double>;

// ---- errors (mirror quasar core.hpp:34-47 + CUDA) --------------------------
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string &msg) { throw Error(code, msg); }
inline void require(bool cond, const std::string &msg) {
    if (!cond) fail(QSV_ERR_INVALID, msg);
}
void cuda_check(cudaError_t e, const char *what);
#define QSV_CUDA(x) ::qsv::cuda_check((x), #x)

// ---- limits -----------------------------------------------------------------
constexpr int kMaxQubits = 40;      // global qubits (36q configs + headroom)
constexpr int kMaxTileBits = 14;    // K: 2^K amplitudes per CTA tile
constexpr int kMaxSlots = 4;        // R: register-resident qubits per group
constexpr int kRegSlots = 4;        // R used by the fused kernel
constexpr int kMaxExtTargets = 64;  // per-CTA external phase factors per group
constexpr int kProgramBudget = 40 * 1024;  // bytes of pass program staged in shared memory

// ---- device program (tile passes) ---------------------------------------
// A pass program is one blob staged into shared memory by every CTA:
//   [GroupDesc x ngroups][FlushTarget x ntargets][DiagRec x nrecs][op stream]
// The op stream is a sequence of 16-byte-aligned variable-length records:
//   OpHdr (16 B) [, uint64 fmask, fval (16 B) if OPF_FCOND] [, payload]
// payload (T = float or double):
//   DENSE1  4 complex T        DENSE1R  4 real T (padded to 16 B)
//   DENSE2  16 complex T       DIAG     4 complex T        X1  none
//   FLUSH   FlushPay (16 B) [, 2^R complex T register table if regmask]
enum OpCode : uint8_t {
    OP_DENSE1 = 1,   // complex 2x2 on one register slot
    OP_DENSE2 = 2,   // complex 4x4 on two register slots (a = MSB slot > b)
    OP_DIAG = 3,     // diagonal applied where it stands (>= 2 register deps + fixed bits, or non-unitary)
    OP_DENSE1R = 4,  // real 2x2 (h, ry, ...)
    OP_X1 = 5,       // Pauli-X on one slot: register swap, no FLOPs
    OP_FLUSH = 6     // apply pending phase factors
};
enum OpFlag : uint8_t { OPF_ZERO_OFF_CONTROL = 1, OPF_FCOND = 2, OPF_ENC = 4, OPF_RCOND = 8 };

struct alignas(16) OpHdr {
    uint8_t code, a, b, flags;
    uint8_t rmask, rval;    // condition over register slots
    uint8_t nt, t0, t1;     // DIAG: target count, slot or physical position
    uint8_t treg;           // DIAG: bit0 t0 is a slot, bit1 t1 is a slot
    uint16_t enc;           // encoded gate index (OPF_ENC)
    uint16_t size;          // record size in bytes
    uint16_t aux;
};
static_assert(sizeof(OpHdr) == 16, "OpHdr layout");

struct alignas(16) FlushPay {
    int32_t tgt_begin, tgt_end;
    uint32_t regmask;       // registers multiplied by the register table
    int32_t pad;
};

// A phase factor that depends only on bits OUTSIDE the register group
// ("fixed" bits of a register set): value = cond ? val[index of the fixed
// target bits] : 1, cond = (index & fmask) == fval.
struct alignas(16) DiagRec {
    uint64_t fmask, fval;
    int32_t nt;             // fixed target bits (0..2)
    int32_t tpos0, tpos1;   // their physical positions (tpos0 is the MSB of the index)
    int32_t pad;
    double val[8];          // up to 4 complex values
};

// One factor applied at a FLUSH: to every register (slot < 0) or to the
// registers whose slot bit is 1. factor = E[eidx] (per tile: records over
// bits outside the tile) * table[s] (host-precomputed over the set index s:
// records over tile bits outside the group) * prod(mixed records, per set).
struct alignas(16) FlushTarget {
    int32_t slot;
    int32_t table;          // offset (complex entries) into the pass's table, or -1
    int32_t ext_begin, ext_end;
    int32_t mix_begin, mix_end;
    int32_t eidx;           // index into the CTA's shared E array, or -1
    // separable part of the tile records: table_lo[s & lo_mask] * table_hi[s >> lo_bits]
    int32_t table_lo, table_hi, lo_bits;
    // separable part of the per-tile (EXT) records: prod_c ext_tab[c * 256 + ((tile >> 8c) & 255)];
    // the records in [ext_rest, ext_end) span chunks or read rank bits and are evaluated per tile
    int32_t ext_tab, ext_chunks, ext_rest;
    int32_t pad[3];
};

struct alignas(16) GroupDesc {
    int32_t op_begin, op_end;          // byte offsets into the op stream
    int32_t slot_bit[kMaxSlots];       // tile-local bit of each register slot
    int32_t ng_bit[kMaxTileBits];      // tile-local bits NOT in the group, ascending
    int32_t tgt_begin, tgt_end;        // flush targets of this group (E precompute)
};

// Per-row matrix binding of an encoded gate (device-side gate_matrix).
struct EncDesc {
    int32_t kind;        // GateKind
    int32_t slot;        // first data column
    int32_t nparams;
    int32_t swapq;       // DENSE2 stored with swapped qubit order
    int32_t diag;        // store the diagonal (DIAG op layout)
};

enum GateKind : int32_t {
    GK_X, GK_Y, GK_Z, GK_H, GK_S, GK_T, GK_RX, GK_RY, GK_RZ, GK_P, GK_U3, GK_SWAP, GK_RXX, GK_RYY, GK_RZZ, GK_CUSTOM
};

struct PassArgs {
    void *state;
    uint64_t row_stride;      // amplitudes per batch row
    uint64_t rank_base;       // rank << nlocal (global physical index offset)
    uint64_t tiles_per_row;
    uint64_t total_tiles;     // tiles_per_row * rows
    const void *blob;         // pass program (device)
    const void *tables;       // complex T
    const void *enc_table;    // [nenc][batch][32] T
    int32_t blob_bytes;
    int32_t off_targets, off_recs, off_ops;
    int32_t batch;
    int32_t nlocal, K, L, ngroups, next;
    int32_t tile_pos[kMaxTileBits];  // physical position of tile-local bit i
    int32_t ext_pos[kMaxQubits];     // physical positions of non-tile local bits
    const void *prefix;              // synthesising first pass: [row][phys bit][0/1] complex T
};

// Shared-memory layout of a tile CTA: [tile 2^K amps][hi_off 2^(K-L) u64][program]
__host__ __device__ inline int tile_prog_offset(int K, int L, int amp_bytes) {
    const int b = (amp_bytes << K) + (8 << (K - L));
    return (b + 15) & ~15;
}

// ---- resolved gate ----------------------------------------------------------
struct GateRec {
    std::string name;
    int kind = 0;
    int k = 1;                 // targets
    int wires[2] = {0, 0};     // logical (or physical, for internal swap gates)
    std::vector<int> ctls;     // logical
    bool diag = false;
    bool encoded = false;
    int enc_slot = -1;         // first data column when encoded
    int nparams = 0;
    int flags = 0;             // OPF_ZERO_OFF_CONTROL for apply_matrix
    cplx m[16];                // 2^k x 2^k row-major (non-encoded)
};

int gate_kind(const std::string &name);
// gate_matrix with reference semantics (gate.hpp:89-154); returns k.
int gate_matrix(const qsv_gate &g, cplx *m);
bool approx_unitary(const cplx *m, int d, double tol);
bool kind_is_diagonal(int kind);
GateRec resolve_gate(const qsv_gate &g, int nqubit, int *enc_cursor);

// ---- host-side program ---------------------------------------------------
struct HostOp {
    uint8_t code = 0, a = 0, b = 0, flags = 0, rmask = 0, rval = 0, nt = 0, t0 = 0, t1 = 0, treg = 0;
    int enc = -1;
    uint64_t fmask = 0, fval = 0;
    std::vector<cplx> pay;     // DENSE1/DENSE1R: 4, DENSE2: 16, DIAG: 4
    FlushPay flush{};
    std::vector<cplx> regtab;  // FLUSH register table (2^R) when flush.regmask != 0
};

struct HostGroup {
    int op_begin = 0, op_end = 0;   // indices into PassHost::ops
    int slot_bit[kMaxSlots] = {};
    int ng_bit[kMaxTileBits] = {};
    int tgt_begin = 0, tgt_end = 0;
};

// A single state pass: the tile geometry plus the groups/ops to run on it.
struct PassHost {
    int K = 0, L = 0, R = kRegSlots;
    std::vector<int> tile_pos;        // size K
    std::vector<int> ext_pos;         // nlocal - K
    std::vector<HostGroup> groups;
    std::vector<HostOp> ops;
    std::vector<FlushTarget> targets;
    std::vector<DiagRec> recs;
    std::vector<cplx> tables;
    int ngates = 0;                   // gates in this pass (after 1q fusion)
    double scale = 1.0;               // deferred real scale (butterfly normalisation)
    // Output bit permutation (input physical bit -> output physical bit);
    // empty = identity. A permuting pass writes out of place (State::scratch).
    std::vector<int> out_perm;
    // First pass of a from-|0> plan: the register sets are synthesised from
    // the per-row, per-bit product-state vectors instead of loaded.
    bool synth = false;
    // L2 super-pass: 1 = first pass of a pair (its launch runs both), 2 =
    // second; chunk_bits = bits spanned by the pair's two tiles (the ext bits
    // inside the chunk come first in ext_pos, so a chunk is a tile range)
    int pair = 0;
    int chunk_bits = 0;
    // Multi-GPU: the qubit swaps that follow this pass, fused into it (when
    // peer memory is available): input global bit -> output global bit
    // (size n; rank bits >= nlocal). The pass then writes every tile straight
    // into its destination rank's scratch state over NVLink.
    std::vector<int> gperm;
    // One GPU: gperm (size nlocal) is the plan's final layout permutation,
    // applied by the last register group storing every amplitude straight to
    // its output position (out of place, write-back stores merged into whole
    // lines in L2) instead of a shared-memory copy-out in output order -- so
    // the pass needs no room in its tile for the output's coalescing run.
    bool local_gperm = false;
    // The pass's gates in execution order, wires mapped to physical bits
    // (schedule export for host-side verification, qsv_plan_dry).
    std::vector<GateRec> exec_gates;
};
// Serialised pass program for dtype.
std::vector<unsigned char> serialize_program(const PassHost &ph, int dtype, int *off_targets, int *off_recs,
                                             int *off_ops);
size_t op_record_bytes(const HostOp &op, int dtype, int R);

// ---- dense-block passes (tensor cores, complex64) -------------------------
// A fused block: up to 5 physical bits (q[i] <-> bit i of the block index)
// and its 2^5 x 2^5 unitary (row-major, padded to exactly 5 bits).
constexpr int kDenseQ = 5;
constexpr int kDenseTile = 12;   // tile bits of a dense-block pass: 128 sets x 32 amplitudes
constexpr int kDenseMaxBlocks = 3;
constexpr int kDenseAutoPerBlock = 12;  // auto mode: dense multi-qubit gates per block to prefer tensor cores
struct DenseBlock {
    int q[kDenseQ] = {0, 0, 0, 0, 0};
    std::vector<cplx> u;         // 32 x 32
    int ngates = 0;
    int ndense = 0;              // absorbed gates that are dense on two or more qubits
};
struct DensePass {
    int tile_pos[kDenseTile];    // physical bit of tile-local bit i (0..3 = the low bits)
    std::vector<int> ext_pos;    // the other local bits, ascending
    std::vector<int> blocks;     // indices into Plan::dblocks, in order
    int bbit[kDenseMaxBlocks][kDenseQ];  // tile-local bit of each block qubit
    int swm[4] = {0, 0, 0, 0};   // shared-tile swizzle masks (slot bit i ^= parity(u & swm[i]))
};
// Fuses gates (wires = physical bits, canonical layout) into dense blocks of
// at most 5 qubits (greedy, gate order kept: a gate joins the open block when
// its qubits fit and none is held by an earlier skipped gate), then packs the
// blocks into passes of a 12-bit tile with the 4 low bits always in it.
void plan_dense(const std::vector<GateRec> &gates, int nlocal, std::vector<DenseBlock> &blocks,
                std::vector<DensePass> &passes);
// B operand of a block: the real 64 x 64 matrix on (re, im) pairs split into
// TF32 hi / lo, in the K-major 128-byte-swizzled UMMA layout (2 x 16 KiB).
void dense_b_operand(const DenseBlock &b, std::vector<float> &out);
struct DenseDev;  // device state of a dense plan (block_pass.cu)
void dense_upload(struct Plan &p);
void dense_execute(struct Plan &p, struct State &st, cudaStream_t s, double *launch_ms = nullptr);
void dense_free(struct Plan &p);

// ---- runtime objects ----------------------------------------------------
struct Nccl;  // dlopen'd NCCL

// Circuit structures met on a context and whether their trainable values
// have varied (lift_policy).
struct LiftSeen {
    std::mutex mu;
    std::map<size_t, std::pair<size_t, bool>> m;  // hash(structure) -> (hash(last values), varied)
};

struct Ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int rank = 0, world = 1, gbits = 0;
    int sm_count = 148;
    size_t smem_optin = 0;
    void *comm = nullptr;       // ncclComm_t
    Nccl *nccl = nullptr;       // owned; freed by nccl_destroy
    void *stage = nullptr;      // qubit-swap staging (2 sets of send + receive), persistent
    size_t stage_bytes = 0;
    cudaStream_t comm_stream = nullptr;  // NCCL transfers of a swap, overlapped with its copies
    // Transport counters (the reference's Transport::messages_sent /
    // bytes_sent, tests/test_dist.cpp:96-126), counted as this rank issues
    // them: point-to-point sends (one per peer per chunk round) and peer-memory
    // stores of swaps fused into passes (one message per destination rank);
    // all-reduces (reductions and the peer-memory ordering barrier) apart.
    uint64_t stat_messages = 0, stat_bytes = 0, stat_allreduces = 0;
    // every rank is driven from this process (qsv_ctx_create_multi): peer
    // memory is shared by raw pointers instead of CUDA IPC handles
    bool in_process = false;
    // permutation-only plans restoring the canonical layout, by input layout
    std::vector<std::pair<std::vector<int>, std::shared_ptr<struct Plan>>> layout_plans;
    std::shared_ptr<LiftSeen> lift_seen = std::make_shared<LiftSeen>();
    // adjoint forward plans of device-bound (lifted) structures, by structure
    std::vector<std::pair<std::string, std::shared_ptr<struct Plan>>> adj_plans;
    ~Ctx();
};

struct State {
    Ctx *ctx = nullptr;
    int n = 0, nlocal = 0, batch = 1, dtype = QSV_C128;
    uint64_t local_amps = 0;
    void *d = nullptr;          // batch * local_amps amplitudes
    void *scratch = nullptr;    // same size; target of out-of-place (permuting) passes
    std::vector<int> perm;      // logical wire -> physical bit (>= nlocal: rank bit)
    // peer memory (multi-GPU swaps fused into passes, dist.cu): 0 = not set
    // up, 1 = ready, -1 = unavailable (NCCL swaps). p2p_buf[i] are this
    // rank's two state buffers (p2p_buf[p2p_cur] == d); d_peers holds
    // 2 x world device pointers: buffer i of rank r at [i * world + r].
    int p2p = 0;
    int p2p_cur = 0;
    void *p2p_buf[2] = {nullptr, nullptr};
    std::vector<void *> p2p_opened;  // peer mappings to close
    void **d_peers = nullptr;
    double *d_barrier = nullptr;
    size_t amp_bytes() const { return dtype == QSV_C64 ? 8 : 16; }
    ~State();
};

struct DevPass {
    PassArgs args{};
    int threads = 256;
    int R = kRegSlots;
    size_t smem = 0;
    int grid = 0;               // persistent CTAs (occupancy x SMs)
    const void *jit = nullptr;  // specialised kernel (cudaKernel_t), else the interpreter
    bool out_of_place = false;  // writes State::scratch (bit-permuting pass)
    int jit_regs = 0, jit_spill = 0;
    const void *jit_z = nullptr;  // variant with the fused <Z> epilogue (prepared on first use)
    int grid_z = 0;
    int pair = 0;                 // L2 super-pass: 1 = head (jit_pair runs it and the next pass), 2 = tail
    const void *jit_pair = nullptr;
    int chunk_tiles_log = 0;      // log2 tiles per chunk (head)
    const void *jit_gout = nullptr;  // variant writing through peer memory (PassHost::gperm), on first use
    double bytes = 0;
    int ngates = 0;
};

// One step of an executable program: a local pass or a global<->local swap.
struct Step {
    int kind = 0;              // 0 pass, 1 swap
    int pass = -1;             // index into passes
    std::vector<std::pair<int, int>> swap_bits;  // (global physical bit, local physical bit)
    bool fused = false;        // swap: done by the preceding pass when peer memory is ready
};

struct Plan {
    Ctx *ctx = nullptr;
    int n = 0, nlocal = 0, dtype = QSV_C128;
    int ngates = 0;
    int nslots = 0;            // encode slots
    std::vector<GateRec> gates;
    std::vector<PassHost> passes;
    std::vector<Step> steps;
    std::vector<int> perm_in, perm_out;  // layout before/after
    std::vector<EncDesc> encs;
    // device buffers
    void *d_blob = nullptr, *d_tables = nullptr, *d_encs = nullptr;
    void *d_enc_table = nullptr;
    size_t enc_table_rows = 0;
    void *d_data = nullptr;
    size_t d_data_cap = 0;
    void *d_z = nullptr;       // fused <Z> sums: batch x (nlocal + 1)
    // product-state prefix of a from-|0> plan: per wire, its leading
    // single-qubit gates (prog: n + 1 offsets, then entries enc index >= 0 or
    // -(1 + constant matrix index)); d_prefix: [row][phys bit][2] complex T
    bool synth = false;
    std::vector<int> prefix_prog;
    std::vector<cplx> prefix_mats;
    void *d_prefix_prog = nullptr, *d_prefix_mats = nullptr, *d_prefix = nullptr;
    size_t prefix_rows = 0;
    size_t d_z_cap = 0;
    double *d_zout = nullptr, *h_zout = nullptr;  // fused <Z>: device result, pinned staging
    size_t zout_cap = 0;
    void *d_sync = nullptr;    // L2 super-passes: per-chunk counters + the item ticket
    size_t d_sync_cap = 0;
    // opts.use_graph: the launch sequence captured per (state buffers, rows)
    struct Graph {
        void *d = nullptr, *scratch = nullptr;
        int batch = 0;
        bool flips = false;      // the sequence ends with d and scratch exchanged
        cudaGraphExec_t exec = nullptr;
    };
    std::vector<Graph> graphs;
    std::vector<DevPass> dev;
    qsv_opts opts{};
    // dense-block plan (opts.dense_blocks): blocks, passes, device buffers
    bool dense = false;
    std::vector<DenseBlock> dblocks;
    std::vector<DensePass> dpasses;
    DenseDev *ddev = nullptr;
    // opts.lazy_layout: the source gates, and one plan per input layout met
    // so far (a lazily laid-out state alternates between a few layouts)
    std::vector<GateRec> src_gates;
    std::vector<std::pair<std::vector<int>, std::unique_ptr<Plan>>> variants;
    ~Plan();
};

// ---- planner (planner.cpp) --------------------------------------------------
struct PlanConfig {
    int nlocal = 0, K = 12, L = 3, R = kRegSlots;
    bool fuse = true;         // tile passes with many gates (false: one gate per pass)
    bool fuse_1q = true;      // pre-multiply runs of single-qubit gates
    bool phase_flush = true;  // lazy phase factors for diagonal gates
    int dtype = QSV_C128;
    // L2 super-passes: consecutive passes whose tiles together span at most
    // this many bits run as one launch, chunk by chunk (0: off)
    int super_bits = 0;
    // one GPU, specialised kernels: a final layout permutation that does not
    // fit the last pass's tile is applied by scattered stores (local_gperm)
    // instead of an extra permutation-only pass
    bool scatter_out = false;
};
// Swap gates as qubit relabelings: rewrites `gates` onto physical bits (the
// returned gates' wires ARE physical bits), dropping uncontrolled swaps and
// tracking the layout; `final_phys` receives the layout after the last gate.
std::vector<GateRec> relabel_swaps(const std::vector<GateRec> &gates, const std::vector<int> &phys_in,
                                   std::vector<int> &final_phys);
// Host-side gate fusion: runs of uncontrolled, non-encoded single-qubit gates
// on the same wire (nothing else touching it in between) become one matrix.
std::vector<GateRec> fuse_single_qubit_runs(const std::vector<GateRec> &gates);
// Lowers gates (wires mapped to PHYSICAL bits by phys_of_wire; every
// non-diagonal target local) to tile passes.
std::vector<PassHost> plan_passes(const std::vector<GateRec> &gates, const std::vector<int> &phys_of_wire,
                                  const PlanConfig &cfg, std::vector<EncDesc> &encs,
                                  const std::vector<int> &out_perm = {}, uint64_t last_need = 0);
int default_tile_bits(int dtype, int nlocal);
int default_low_bits(int dtype, int nlocal);

// ---- device launchers (engine.cu) -----------------------------------------
void upload_plan(Plan &p);
void launch_pass(const DevPass &dp, int dtype, void *state, int rows, cudaStream_t s, double *zout = nullptr);
// Runs one pass on `st`; an out-of-place pass writes State::scratch and swaps it in.
void run_pass(const DevPass &dp, int dtype, State &st, cudaStream_t s, double *zout = nullptr);
// Circuit::forward + expectation() of every single-Z observable in one call:
// out[b * n + w] = <Z_w>. The <Z> sums are fused into the last pass when its
// tile is the whole row (batched small circuits, cfg2), else one extra
// reduction pass.
void execute_plan_z(Plan &p, State &st, const double *data, int rows, int slots, double *host_out);
void execute_plan(Plan &p, State &st, const double *data, int rows, int slots, double *zout = nullptr);
// Lazy layouts (opts.lazy_layout): whether the state's wire -> bit map is the
// canonical one (wire w at bit n-1-w), and the permutation pass restoring it
// (a no-op when it is; single GPU).
bool layout_canonical(const State &st);
// Trainable values as compile-time constants (specialised passes) the first
// time a circuit structure is met on a context, as run-time parameters bound
// on the device (encoded slots: no new code per value) once the same
// structure comes back with other values -- a training loop.
inline bool lift_policy(Ctx &c, const std::string &structure, const std::string &values) {
    // hashes only: a collision costs a compile or a device-bound run, never a
    // wrong result (both forms compute the same circuit)
    const size_t hs = std::hash<std::string>{}(structure), hv = std::hash<std::string>{}(values);
    std::lock_guard<std::mutex> lk(c.lift_seen->mu);
    auto &m = c.lift_seen->m;
    auto it = m.find(hs);
    if (it == m.end()) {
        if (m.size() >= 1024) m.clear();
        m.emplace(hs, std::make_pair(hv, false));
        return false;
    }
    const size_t &values_seen = it->second.first;
    if (!it->second.second && values_seen != hv) it->second.second = true;
    return it->second.second;
}
void normalize_layout(State &st);
void launch_bind(const Plan &p, const double *d_data, int rows, int slots, cudaStream_t s);
// per-row, per-bit product-state vectors of a from-|0> plan into p.d_prefix
void launch_prefix(const Plan &p, int rows, cudaStream_t s);
void launch_set_basis(State &st, uint64_t local_index, bool on_this_rank);
// out[b * n + w] = z[b * k1] - 2 z[b * k1 + 1 + perm[w]] (device arrays)
void launch_z_finish(const double *z, int k1, int rows, int n, const std::vector<int> &perm, double *out,
                     cudaStream_t s);
// state buffers: recycled per device up to 256 MiB each (engine.cu)
cudaError_t state_alloc(void **p, size_t bytes);
void state_release(void *p, size_t bytes);
// one gate as one sweep kernel (single GPU, k <= 2, not encoded); false = not eligible
bool apply_direct(State &st, const GateRec &g);
void launch_convert(void *dst, int dst_dtype, const void *src, int src_dtype, uint64_t count, cudaStream_t s);
int tile_kernel_blocks_per_sm(int dtype, int R, int threads, size_t smem);
// ---- pass specialisation (codegen.cpp, jit.cpp) ----------------------------
// whether a pass's kernel double-buffers its tiles (jit.cpp)
bool pass_prefetches(const PassHost &ph, int dtype);
// threads per CTA of a pass's generated kernel (codegen.cpp)
int kernel_threads(const PassHost &ph, int dtype);
void jit_prepare(DevPass &dp, const PassHost &ph, int dtype, int sm_count);
void launch_jit(const DevPass &dp, void *state, void *out, int rows, cudaStream_t s, double *zout = nullptr);
// L2 super-pass (PassHost::pair): compiles the pair kernel into head; the
// launch runs head's pass in place on state and the tail's into out.
void jit_prepare_pair(DevPass &head, const PassHost &a, const PassHost &b, int dtype, int sm_count);
void launch_pair(const DevPass &head, const DevPass &tail, void *state, void *out, int rows, unsigned *sync,
                 uint64_t nchunks, cudaStream_t s);
void jit_prepare_z(DevPass &dp, const PassHost &ph, int dtype, int sm_count);
// Pass variant whose last group stores straight into the destination rank's
// buffer (PassHost::gperm; peers = world device pointers of the destination
// buffers, out_lconst / out_rconst = this rank's own rank bits mapped to
// local / rank output bits).
void jit_prepare_gout(DevPass &dp, const PassHost &ph, int dtype, int sm_count);
void launch_gout(const DevPass &dp, void *state, int rows, void *const *peers, uint64_t out_lconst, int out_rconst,
                 cudaStream_t s);
std::string jit_source(const PassHost &ph, int dtype);
std::string jit_pair_source(const PassHost &a, const PassHost &b, int dtype);
std::string jit_gout_source(const PassHost &ph, int dtype);
// Reductions write FP64 results to device memory, then copy to host.
void reduce_norm2(State &st, double *host_out);
void reduce_z_all(State &st, double *host_out /* batch x kZ: [total, S_bit0..] */);
void reduce_pauli(State &st, uint64_t flip, uint64_t zy, double *host_out /* batch x 2 */);
void reduce_marginal(State &st, int row, const std::vector<int> &phys_bits, double *host_out);
// Mixed states held as vec(rho) on 2m qubits (row wires high): Tr-type sums
// along the flip-diagonal, and diagonal marginals (bits are positions in r).
void reduce_dm_pauli(State &st, int m, uint64_t flip, uint64_t zy, double *host_out /* batch x 2 */);
void reduce_dm_marginal(State &st, int m, int row, const std::vector<int> &bits_r, double *host_out);

// ---- distributed (dist.cu) -------------------------------------------------
void nccl_unique_id(void *out128);
void nccl_init(Ctx &ctx, const void *uid);
// One process driving every rank: ncclCommInitAll over the ranks' devices.
void nccl_init_all(const std::vector<Ctx *> &ranks);
void nccl_destroy(Ctx &ctx);
// Exchange: swap every physical rank bit `gbit` (>= nlocal) with its local
// bit `lbit` at once -- one in-place all-to-all over the 2^m - 1 peer ranks
// (m = pairs), for every batch row, chunked through persistent staging.
void dist_swap_bits(State &st, const std::vector<std::pair<int, int>> &pairs, void *staging, size_t staging_bytes);
void dist_allreduce_sum(Ctx &ctx, double *d_buf, size_t count);
// A single-qubit matrix on a GLOBAL target (physical rank bit gbit): the
// reference's pairwise exchange (tests/test_dist.cpp:112-126) --
// each rank sends its whole slice to the partner across that bit and
// combines the partner's slice with its own, new = m[b][b] * mine +
// m[b][1-b] * theirs (b = this rank's bit); local controls select elements,
// global controls whole slices (off-control: untouched, or zeroed with
// zero_off_control). One message per rank per chunk round.
void dist_exchange_apply(State &st, int gbit, const cplx *m, uint64_t local_cmask, bool on, bool zero_off_control);
// Peer memory for swaps fused into passes (collective; agreed by all ranks).
bool dist_p2p_ready(State &st);
void dist_p2p_barrier(State &st);
void dist_p2p_release(State &st);

} // namespace qsv
