/*
 * qsv — B200-native state-vector engine for the DeepQuantum / quasar qubit
 * hot path. This is the C ABI (the drop-in boundary): plain pointers and
 * sizes, no C++ or torch types. Everything above it (the quasar-compatible
 * C++ headers in include/quasar/, the Python mirror in
 * paper_2512_18995_b200/qsv.py) is a thin host layer over these calls.
 *
 * Reference interfaces replaced (paths under /root/reference/proj):
 *   qsv_apply_matrix     quasar::qubit::detail::apply_matrix_strided
 *                        include/quasar/qubit/state.hpp:111-143
 *   qsv_apply_gate       quasar::qubit::apply_gate (pure states)
 *                        include/quasar/qubit/state.hpp:149-157
 *   qsv_gate_matrix      quasar::qubit::gate_matrix  include/quasar/qubit/gate.hpp:89-154
 *   qsv_run_circuit      quasar::qubit::Circuit::forward  include/quasar/qubit/circuit.hpp:121-157
 *   qsv_plan_*           (same, with planning hoisted out of the timed loop)
 *   qsv_expect_pauli     quasar::qubit::expectation_one / expectation
 *                        include/quasar/qubit/circuit.hpp:248-282
 *   qsv_expect_z_all     expectation() over the n single-Z observables (cfg1/cfg2)
 *   qsv_marginal_probs   quasar::qubit::marginal_probabilities circuit.hpp:182-205
 *   qsv_state_*          quasar::qubit::QubitState (basis / from_amplitudes /
 *                        amplitudes(b)) state.hpp:29-91
 *   qsv_ctx_create_dist, qsv_ctx_create_multi, qsv_run_on_ranks,
 *   qsv_ctx_comm_stats, qsv_state_info (global bits), qsv_norm2 (global)
 *                        quasar::dist::PartitionedState / run_on_ranks /
 *                        global_norm2 (source absent from the reference;
 *                        contract from tests/test_dist.cpp:66-174 and
 *                        SPEC.md:719-798)
 *
 * Conventions (identical to the reference):
 *   - wire 0 is the MOST significant bit of a basis index (state.hpp:21-24);
 *   - a k-qubit matrix is 2^k x 2^k row-major with wires[0] as its MSB
 *     (gate.hpp:30); complex numbers are interleaved (re, im) doubles;
 *   - amplitudes cross the boundary in LOGICAL index order whatever
 *     internal qubit permutation the engine is using.
 *
 * Status codes mirror the reference CLI exit codes (tools/main.cpp:686-697)
 * and error classes (core.hpp:34-47). Every call returns one; the message of
 * the last failure on the calling thread is qsv_last_error().
 *
 * Threading: calls on distinct states are independent; calls on the same
 * state must be serialised by the caller (reference: SPEC.md:216).
 */
#ifndef QSV_H_
#define QSV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QSV_VERSION 1

enum qsv_status {
    QSV_OK = 0,
    QSV_ERR_INTERNAL = 1,  /* CUDA / internal failure */
    QSV_ERR_INVALID = 2,   /* quasar::invalid_input */
    QSV_ERR_GUARD = 3,     /* quasar::guard_error (numerical guard) */
    QSV_ERR_TRANSPORT = 4  /* quasar::transport_error (NCCL) */
};

enum qsv_dtype { QSV_C64 = 1, QSV_C128 = 2 };

/* apply flags */
enum {
    QSV_ZERO_OFF_CONTROL = 1, /* apply_matrix_strided(..., zero_off_control=true) */
    /* Structure hints. The engine classifies every matrix
     * itself (diagonal -> deferred phases, 0/1 permutation -> register
     * relabel), so a hint changes nothing on the GPU path; a hint the matrix
     * contradicts fails with QSV_ERR_INVALID. */
    QSV_HINT_DIAGONAL = 2,
    QSV_HINT_PERMUTATION = 4
};

typedef struct qsv_ctx qsv_ctx;
typedef struct qsv_state qsv_state;
typedef struct qsv_plan qsv_plan;

/* A gate record with the meaning of quasar::qubit::Gate (gate.hpp:28-38). */
typedef struct qsv_gate {
    char name[16];          /* x y z h s t rx ry rz p u3 swap rxx ryy rzz custom */
    int32_t nwires;         /* targets; wires[0] is the matrix MSB */
    int32_t wires[2];
    int32_t ncontrols;      /* all controls must be |1> */
    int32_t controls[6];
    int32_t nparams;
    double params[3];       /* radians */
    int32_t trainable;
    int32_t encode;         /* parameters bound from data rows at run time */
    const double *custom;   /* name=="custom": 2^k x 2^k row-major (re,im) */
} qsv_gate;

/* Tensor product of single-qubit Paulis (circuit.hpp:25-28). */
typedef struct qsv_obs {
    int32_t nwires;
    const int32_t *wires;
    const char *basis;      /* one of 'x','y','z' per wire */
} qsv_obs;

/* Planner / executor options (0 = engine default). */
typedef struct qsv_opts {
    int32_t fuse;           /* 1 = fused tile passes (default), 0 = one kernel per gate */
    int32_t tile_bits;      /* qubits per shared-memory tile (K) */
    int32_t low_bits;       /* lowest physical qubits always in a tile (coalescing) */
    int32_t use_graph;      /* 1 = replay the launch sequence as a CUDA graph (one
                               per state buffer pair and row count; single GPU,
                               no encoded data): for launch-bound small states */
    int32_t no_fuse_1q;     /* 1 = keep runs of single-qubit gates unfused */
    int32_t no_phase_flush; /* 1 = apply every diagonal gate eagerly */
    int32_t jit;            /* 1 = specialised (NVRTC) pass kernels, -1 = interpreter, 0 = auto */
    int32_t reg_slots;      /* qubits per register group R (1..4; 0 = 4) */
    int32_t no_relabel;     /* 1 = apply swap gates as data moves (no scratch state needed) */
    int32_t from_zero;      /* 1 = execute starts from |0...0> whatever the state holds
                               (Circuit::forward without init); the leading
                               single-qubit gates of every wire then become a
                               product state synthesised inside the first pass */
    int32_t super_bits;     /* L2 super-passes: pairs of passes whose tiles span at
                               most this many qubits run as one launch, chunk by
                               chunk through L2 (> 0 = on with this chunk size;
                               0 = $QSV_SUPER_BITS, default off; -1 = off) */
    int32_t dense_blocks;   /* complex64, one GPU: fuse the circuit into dense <= 5-qubit
                               blocks (32 x 32 unitaries) applied on the tcgen05 tensor
                               cores (3xTF32, TMEM accumulators), up to 3 blocks per HBM
                               pass. 1 = on; -1 = off (the fused FFMA tile passes);
                               0 = auto: on when the blocks average >= 12 dense
                               multi-qubit gates (deep local circuits, where it is
                               measured 2.7-5.4x faster); the BASELINE configs stay on
                               the FFMA passes */
    int32_t lazy_layout;    /* one GPU: swap gates stay qubit relabelings past the end of
                               the execute -- the state keeps its permuted physical
                               layout (its wire -> bit map travels with it) instead of
                               paying a layout-restoring pass; the next execute plans
                               from that layout, and anything that reads amplitudes in
                               logical order (downloads, device_ptr, density calls)
                               restores it first (one permutation pass). 0 = off */
} qsv_opts;

/* What a plan does, for measurement (bench.py roofline). */
typedef struct qsv_plan_info {
    int32_t ngates;          /* source gates */
    int32_t npasses;         /* pass launches per execute (an L2 super-pass is one) */
    int32_t nswaps;          /* global<->local qubit swaps (multi-GPU) */
    int32_t max_tile_bits;
    double bytes_per_exec;   /* algorithmic HBM bytes per execute (all passes) */
    double comm_bytes_per_exec; /* bytes sent per rank per execute */
    int32_t ntile_passes;    /* tile passes per execute (>= npasses: super-passes run two) */
    int32_t nblocks;         /* dense-block plans (opts.dense_blocks): fused 5-qubit blocks */
} qsv_plan_info;

/* ---- library --------------------------------------------------------- */
const char *qsv_last_error(void);
int qsv_version(void);
/* Number of CUDA devices (0 on a host without a GPU; never fails). */
int qsv_device_count(void);

/* ---- context (owns the CUDA stream, the NCCL communicator) ----------- */
int qsv_ctx_create(int device, qsv_ctx **out);
/* One process per GPU: rank/world with an NCCL unique id produced by
 * qsv_nccl_unique_id on rank 0 and broadcast by the caller (e.g. with
 * torch.distributed). world must be a power of two (test_dist.cpp:90-94). */
int qsv_nccl_unique_id(void *out128);
int qsv_ctx_create_dist(int device, int rank, int world, const void *unique_id128, qsv_ctx **out);
/* One process, P GPUs (the reference's in-process
 * dist::run_on_ranks, tests/test_dist.cpp:66-94, tools/main.cpp:95): rank r
 * on devices[r] with its own stream, one NCCL communicator per rank from
 * ncclCommInitAll, ndev a power of two. Every call on this context and on the
 * states / plans made from it runs on all ranks (one host thread per rank,
 * NCCL inside); a state's host view (upload / download) is the WHOLE state in
 * logical order, and reductions return the all-reduced values. */
int qsv_ctx_create_multi(int ndev, const int *devices, qsv_ctx **out);
/* Rank r's own context inside a multi-device one (owned by it): the ABI
 * calls on it act on that rank's slice, as with qsv_ctx_create_dist. */
int qsv_ctx_rank_ctx(qsv_ctx *multi, int rank, qsv_ctx **out);
/* dist::run_on_ranks: fn(rank context, rank, user) on one host thread per
 * rank, all joined; the first failing rank's status is returned (its message
 * in qsv_last_error). On a single-rank context fn runs inline. Collective
 * calls inside fn must be made by every rank, as in the reference. */
typedef int (*qsv_rank_fn)(qsv_ctx *rank_ctx, int rank, void *user);
int qsv_run_on_ranks(qsv_ctx *multi, qsv_rank_fn fn, void *user);
/* Transport counters (Transport::messages_sent / bytes_sent / reset_counters,
 * tests/test_dist.cpp:96-126), measured as the rank issues them: one message
 * per point-to-point send (per peer, per chunk round) and per destination
 * rank of a swap fused into a pass (peer-memory stores), bytes = payload;
 * all-reduces counted apart. On a multi-device context: summed over ranks. */
int qsv_ctx_comm_stats(const qsv_ctx *ctx, uint64_t *messages, uint64_t *bytes, uint64_t *allreduces);
int qsv_ctx_comm_reset(qsv_ctx *ctx);
/* Batched small circuits as independent units: the
 * `rows` data rows split into contiguous chunks over the devices of a
 * multi-device context (one independent single-GPU context per device, no
 * communication), each chunk a from-|0...0> forward with its rows' encode data
 * followed by every <Z_w>: out[row * nqubit + w] (circuit.hpp:121-157,
 * 248-282). On a single-GPU context the whole batch runs there. */
int qsv_run_rows_expect_z(qsv_ctx *ctx, int nqubit, int dtype, const qsv_gate *gates, int ngates, const double *data,
                          int rows, int slots, const qsv_opts *opts, double *out);
int qsv_ctx_destroy(qsv_ctx *ctx);
int qsv_ctx_sync(qsv_ctx *ctx);
/* The cudaStream_t the engine launches on (for events), as void*. */
int qsv_ctx_stream(qsv_ctx *ctx, void **stream);
int qsv_ctx_rank(qsv_ctx *ctx, int *rank, int *world);

/* ---- states (QubitState) --------------------------------------------- */
/* nqubit is the GLOBAL qubit count; each rank holds 2^(nqubit-g) amplitudes
 * per batch row, g = log2(world). Initialised to |0...0>. */
int qsv_state_create(qsv_ctx *ctx, int nqubit, int batch, int dtype, qsv_state **out);
int qsv_state_destroy(qsv_state *st);
int qsv_state_info(const qsv_state *st, int *nqubit, int *batch, int *dtype, int *global_bits,
                   uint64_t *local_amps);
/* |index> on every batch row (QubitState::basis, state.hpp:34-42). */
int qsv_state_set_basis(qsv_state *st, uint64_t index);
/* Host <-> device, interleaved (re,im) float64 for BOTH dtypes, logical
 * order. On a distributed context these move this rank's slice (the
 * 2^(n-g) indices whose top g bits equal the rank). */
int qsv_state_upload(qsv_state *st, int row, const double *host, uint64_t count);
int qsv_state_download(qsv_state *st, int row, double *host, uint64_t count);
/* Raw dtype-native host buffers (float32 pairs for C64): one DMA each way.
 * Both return after the copy has completed (the host buffer may be reused). */
int qsv_state_upload_raw(qsv_state *st, int row, const void *host, uint64_t count);
int qsv_state_download_raw(qsv_state *st, int row, void *host, uint64_t count);
/* Stream-ordered variants (the e2e benchmark's pipeline): the copy is queued
 * on the context's stream and the call returns at once; `host` (pinned for an
 * asynchronous DMA) must stay untouched until qsv_ctx_sync. */
int qsv_state_upload_raw_async(qsv_state *st, int row, const void *host, uint64_t count);
int qsv_state_download_raw_async(qsv_state *st, int row, void *host, uint64_t count);
int qsv_state_clone(const qsv_state *st, qsv_state **out);
/* Device pointer of row `row` in the engine's PHYSICAL order (tests). */
int qsv_state_device_ptr(qsv_state *st, int row, void **ptr);
/* Multi-GPU: whether this state's qubit swaps run fused into the passes
 * through peer memory (1), as NCCL all-to-alls (-1: peer memory unavailable
 * or QSV_P2P_SWAP=0), or not decided yet (0: set up on the first swap). */
int qsv_state_peer_memory(const qsv_state *st, int *out);

/* ---- gates ------------------------------------------------------------- */
/* gate_matrix() with reference semantics; out is 2^k x 2^k (re,im). */
int qsv_gate_matrix(const qsv_gate *g, double *out, int *k);
/* apply_matrix_strided on every batch row. */
int qsv_apply_matrix(qsv_state *st, int k, const int32_t *wires, int nctl, const int32_t *ctls, const double *m,
                     int flags);
/* apply_gate: gate_matrix + unitarity check (1e-10) + strided update. */
int qsv_apply_gate(qsv_state *st, const qsv_gate *g);

/* ---- circuits (Circuit::forward) --------------------------------------- */
/* rows == 0: apply the gates to every batch row (no encode slots allowed).
 * rows  > 0: rows must equal the state's batch; row b binds the encode slots
 * from data[b*slots ...] in circuit order; slots must equal the circuit's
 * encode-slot count exactly (circuit.hpp:133-136). */
int qsv_run_circuit(qsv_state *st, const qsv_gate *gates, int ngates, const double *data, int rows, int slots,
                    const qsv_opts *opts);
int qsv_plan_create(qsv_ctx *ctx, int nqubit, int dtype, const qsv_gate *gates, int ngates, const qsv_opts *opts,
                    qsv_plan **out);
int qsv_plan_destroy(qsv_plan *plan);
int qsv_plan_info_get(const qsv_plan *plan, qsv_plan_info *info);
int qsv_plan_execute(qsv_plan *plan, qsv_state *st, const double *data, int rows, int slots);
/* Circuit::forward(data) followed by expectation() of the n single-qubit Z
 * observables (circuit.hpp:121-157, 248-282): out[b * n + w] = <Z_w> for every
 * batch row. When the plan's last pass holds a whole row per tile (batched
 * small circuits) the |a|^2 sums are fused into that pass (no second read of
 * the state); otherwise one extra reduction pass runs. */
int qsv_plan_execute_expect_z(qsv_plan *plan, qsv_state *st, const double *data, int rows, int slots, double *out);
/* Execute once with a CUDA event pair around every launch; launch_ms gets
 * npasses durations (ms). */
int qsv_plan_profile(qsv_plan *plan, qsv_state *st, double *launch_ms);

/* ---- reductions (FP64 accumulation) ------------------------------------ */
int qsv_norm2(qsv_state *st, double *out /* batch */);
/* <Z_w> for every wire w: out[b * n + w]. */
int qsv_expect_z_all(qsv_state *st, double *out);
/* <P> for each observable: out[b * nobs + i]; fails (QSV_ERR_INVALID) on an
 * imaginary residue >= 1e-10 like circuit.hpp:261. */
int qsv_expect_pauli(qsv_state *st, int nobs, const qsv_obs *obs, double *out);
/* marginal_probabilities on row `row`: out has 2^k entries. */
int qsv_marginal_probs(qsv_state *st, int row, int k, const int32_t *wires, double *out);

/* measure (circuit.hpp:217-244) on row `row`: the marginals of `wires` on the
 * device, then `shots` draws u = Rng(seed, label).uniform() * total (the
 * stream continues after *rng_counter draws and the counter is advanced; NULL
 * = from the start), outcome = lower_bound over the running sums -- the
 * reference's seeded histogram exactly. counts[2^k] per outcome (wires[0] is
 * the outcome's MSB); probs[2^k] receives the exact marginals (may be NULL:
 * the with_prob = false form). A multi-device state all-reduces the marginals
 * first (measure_dist). */
int qsv_measure(qsv_state *st, int row, int k, const int32_t *wires, int shots, uint64_t seed, const char *label,
                uint64_t *rng_counter, uint64_t *counts, double *probs);

/* ---- mixed states (density matrices, channels) --------------------------
 * A batch of m-qubit density matrices is an engine state of 2m qubits holding
 * vec(rho)[r * 2^m + c] per row (row wires = engine wires 0..m-1, column
 * wires = m..2m-1). A gate U on wires W acts as U on W and conj(U) on m + W
 * (state.hpp:159-172: U rho U^dagger); a single-qubit channel is the 4x4
 * superoperator sum_i K_i (x) conj(K_i) on wires {w, m + w}
 * (channel.hpp:73-100); both go through qsv_apply_matrix. The reductions read
 * rho's diagonal (or one flip-diagonal) only. */
/* Tr[rho P] per observable: out[b * nobs + i]; imaginary residue >= 1e-10
 * fails like circuit.hpp:280. Replaces expectation_one's mixed branch
 * (circuit.hpp:264-281). */
int qsv_density_expect_pauli(qsv_state *st, int nobs, const qsv_obs *obs, double *out);
/* marginal_probabilities' mixed branch (circuit.hpp:199-203): Re rho[i, i]
 * binned by the outcome bits of `wires` (1..12 wires). */
int qsv_density_marginal_probs(qsv_state *st, int row, int k, const int32_t *wires, double *out);

/* ---- gradients (quasar::qubit::adjoint_gradients, adjoint.hpp:52-110) ---- */
/* Gradient of sum_i <O_i> by the adjoint method: param_grads gets one entry
 * per parameter of each trainable, non-encoded gate (circuit order; *nparams
 * receives the count, at most param_cap are written), data_grads one per
 * encode slot (data order; `slots` must equal the circuit's encode slots).
 * init: 2^n interleaved (re,im) amplitudes of the initial state, or NULL for
 * |0...0>. Pure states, one data row per call, like the reference. */
int qsv_adjoint_gradients(qsv_ctx *ctx, int nqubit, int dtype, const qsv_gate *gates, int ngates, int nobs,
                          const qsv_obs *obs, const double *init, const double *data, int slots,
                          double *param_grads, int param_cap, int *nparams, double *data_grads);

/* Plans on the host only (no device, no upload): fills info as
 * qsv_plan_info_get would for a context of `world` ranks, and, when src is
 * non-null, the generated CUDA source of pass `pass_index`. For tests and
 * diagnostics on GPU-less hosts. */
int qsv_plan_dry(int nqubit, int dtype, int world, const qsv_gate *gates, int ngates, const qsv_opts *opts,
                 qsv_plan_info *info, int pass_index, char *src, size_t cap);

/* ---- seeded inputs (quasar::Rng, rng.hpp:29-103) ----------------------- */
/* Fills `out` with count draws of stream Rng(seed, label) (label may be
 * NULL for Rng(seed)); kind 0 next_u64, 1 uniform, 2 normal. Counter-based,
 * so it runs on nthreads host threads and still reproduces the sequential
 * stream exactly. */
int qsv_rng_fill(uint64_t seed, const char *label, int kind, uint64_t count, void *out, int nthreads);
/* The same stream starting `offset` draws in (even for normals): a rank fills
 * only its slice of a seeded input. */
int qsv_rng_fill_at(uint64_t seed, const char *label, int kind, uint64_t offset, uint64_t count, void *out,
                    int nthreads);
/* Step kinds of a plan in execution order (0 = local pass launch, 1 = qubit
 * swap, 2 = local pass run inside the previous step's launch: the second half
 * of an L2 super-pass, whose profiled time is 0; 3 = a qubit swap, or the
 * final permutation-only pass, fused into the preceding pass, which stores
 * its tiles through peer memory when every rank has it -- profiled time 0 --
 * else run as a swap / pass);
 * returns the step count (fills at most cap entries). */
int qsv_plan_steps(const qsv_plan *plan, int *kinds, int cap);

#ifdef __cplusplus
}
#endif

#endif /* QSV_H_ */
