// Host runtime: contexts, device-resident states, plans (planning hoisted out
// of execution), and the distributed step schedule.
//
// Reference correspondence (/root/reference/proj/include/quasar):
//   State            qubit::QubitState (state.hpp:29-91), device-resident, one
//                    row per batch element, no 30-qubit cap (state.hpp:35).
//   plan + execute   qubit::Circuit::forward (circuit.hpp:121-157) with the
//                    per-gate value copies (state.hpp:153) removed.
//   dist schedule    dist::apply_gate_dist / run_circuit_dist (source absent;
//                    SPEC.md:743-751, tests/test_dist.cpp:96-126): local gates
//                    and every diagonal gate run without communication; a
//                    non-diagonal gate on a global (rank) qubit first swaps
//                    that qubit with a local one.
#include <algorithm>
#include <bit>
#include <cstring>

#include <cmath>

#include "qsv_internal.hpp"

namespace qsv {

Ctx::~Ctx() {
    if (comm || nccl) nccl_destroy(*this);
    if (stream) cudaStreamDestroy(stream);
}

State::~State() {
    if (p2p_opened.size() || d_peers || d_barrier) dist_p2p_release(*this);
    const size_t bytes = local_amps * amp_bytes() * static_cast<size_t>(batch);
    // buffers once exported to peers (IPC) are freed, never recycled
    if (d) state_release(d, p2p ? SIZE_MAX : bytes);
    if (scratch) state_release(scratch, p2p ? SIZE_MAX : bytes);
}

bool plan_uses_jit(const Plan &p);

Plan::~Plan() {
    cudaFree(d_blob);
    cudaFree(d_tables);
    cudaFree(d_encs);
    cudaFree(d_enc_table);
    cudaFree(d_data);
    cudaFree(d_z);
    cudaFree(d_prefix_prog);
    cudaFree(d_prefix_mats);
    cudaFree(d_prefix);
    cudaFree(d_sync);
    cudaFree(d_zout);
    cudaFreeHost(h_zout);
    for (auto &g : graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    dense_free(*this);
}

namespace {

std::vector<int> canonical_perm(int n) {
    std::vector<int> p(n);
    for (int w = 0; w < n; ++w) p[w] = n - 1 - w; // wire 0 = MSB (state.hpp:21-24)
    return p;
}

// Qubit swaps fused into the pass before them (used when every rank has peer
// memory, dist.cu dist_p2p_ready): a run of swap steps is one permutation of
// the global index bits, and the pass writes every tile straight to where the
// permutation puts it -- the destination rank's scratch state, over NVLink --
// instead of writing in place and exchanging halves through NCCL afterwards.
// Needs a specialised kernel and no output permutation of its own. The swap
// steps stay in the plan: without peer memory they run as NCCL all-to-alls.
void fuse_swaps_into_passes(Plan &p) {
    const int n = p.n, nl = p.nlocal;
    if (!plan_uses_jit(p)) return;
    auto perm_only = [&](const Step &st) {
        if (st.kind != 0) return false;
        const PassHost &q = p.passes[st.pass];
        return !q.out_perm.empty() && q.ngates == 0;
    };
    for (size_t i = 1; i < p.steps.size(); ++i) {
        if ((p.steps[i].kind != 1 && !perm_only(p.steps[i])) || p.steps[i - 1].kind != 0) continue;
        PassHost &ph = p.passes[p.steps[i - 1].pass];
        if (!ph.out_perm.empty() || ph.synth || ph.pair || !ph.gperm.empty()) continue;
        std::vector<int> where(n); // input bit -> its position after the swaps
        for (int b = 0; b < n; ++b) where[b] = b;
        size_t j = i;
        for (; j < p.steps.size() && p.steps[j].kind == 1; ++j)
            for (const auto &[a, b] : p.steps[j].swap_bits)
                for (int &w : where) w = w == a ? b : w == b ? a : w;
        // a permutation-only pass right after (the final local layout) joins
        // when its coalescing run stays in this pass's tile: the input bits
        // landing on the L lowest output bits are tile bits
        if (j < p.steps.size() && perm_only(p.steps[j])) {
            const std::vector<int> &op = p.passes[p.steps[j].pass].out_perm;
            std::vector<int> w2 = where;
            for (int &x : w2)
                if (x < nl) x = op[x];
            bool ok = true;
            for (int b = 0; b < n && ok; ++b)
                if (w2[b] < ph.L)
                    ok = std::find(ph.tile_pos.begin(), ph.tile_pos.end(), b) != ph.tile_pos.end();
            if (ok) {
                where = w2;
                ++j;
            }
        }
        if (j == i) continue;
        ph.gperm = where;
        for (size_t k = i; k < j; ++k) p.steps[k].fused = true;
        i = j - 1;
    }
}

// Distributed schedule: split the gate list into local segments separated by
// global<->local qubit swaps. A non-diagonal target on a rank bit is swapped
// with the local bit whose next non-diagonal use is furthest away (Belady),
// preferring the highest local bits (contiguous halves).
void schedule_dist(Plan &p, const PlanConfig &cfg) {
    const int n = p.n, nl = p.nlocal;
    std::vector<int> phys = p.perm_in;
    std::vector<int> wire_at(n);
    for (int w = 0; w < n; ++w) wire_at[phys[w]] = w;
    // Gates still to schedule, in order. Each round runs the maximal
    // commutation-closed front that needs no communication (a gate joins when
    // it commutes with every earlier blocked gate and has no non-diagonal
    // target on a rank bit), then swaps in the rank-bit qubits the blocked
    // frontier needs.
    std::vector<int> rem(p.gates.size());
    for (size_t i = 0; i < rem.size(); ++i) rem[i] = static_cast<int>(i);
    // Swap gates as relabelings (as on one GPU): a swap gate exchanges the
    // two wires' physical bits in the mapping and moves no data -- local or
    // global -- and the final layout restore absorbs them (a permuting,
    // out-of-place pass for the local bits, so it needs room for a second
    // local state; else swap gates stay gates).
    bool relabel = cfg.fuse && p.opts.no_relabel == 0 && plan_uses_jit(p) && p.nslots == 0;
    if (relabel && p.ctx->stream) {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
            const double state = std::ldexp(static_cast<double>(p.dtype == QSV_C64 ? 8 : 16), nl);
            if (2.0 * state > 0.92 * static_cast<double>(total_b)) relabel = false;
        } else {
            cudaGetLastError();
        }
    }
    auto plain_swap = [](const GateRec &g) {
        return g.kind == GK_SWAP && g.k == 2 && g.ctls.empty() && !g.encoded && g.flags == 0;
    };
    std::vector<int> ident(n);
    for (int b = 0; b < n; ++b) ident[b] = b;
    auto next_use = [&](int wire, size_t from) -> size_t { // position in rem
        for (size_t j = from; j < rem.size(); ++j) {
            const GateRec &g = p.gates[rem[j]];
            if (g.diag) continue;
            for (int t = 0; t < g.k; ++t)
                if (g.wires[t] == wire) return j;
        }
        return rem.size() + 1;
    };
    std::vector<GateRec> last_seg; // the final front: planned once the layout restore is known
    while (!rem.empty()) {
        std::vector<int> blocked;
        std::vector<GateRec> seg; // the front, on physical bits (as admitted)
        uint64_t bN = 0, bD = 0; // wires (logical) blocked non-diagonally / diagonally
        for (int gi : rem) {
            const GateRec &g = p.gates[gi];
            if (relabel && plain_swap(g)) {
                const uint64_t wm = (1ull << g.wires[0]) | (1ull << g.wires[1]);
                if (wm & (bN | bD)) { // an earlier gate on either wire waits: so does the swap
                    bN |= wm;
                    blocked.push_back(gi);
                    continue;
                }
                const int a = g.wires[0], b = g.wires[1];
                std::swap(phys[a], phys[b]);
                wire_at[phys[a]] = a;
                wire_at[phys[b]] = b;
                continue;
            }
            uint64_t nm = 0, dm = 0;
            bool global_n = false;
            for (int t = 0; t < g.k; ++t) {
                if (g.diag) dm |= 1ull << g.wires[t];
                else {
                    nm |= 1ull << g.wires[t];
                    if (phys[g.wires[t]] >= nl) global_n = true;
                }
            }
            for (int c : g.ctls) dm |= 1ull << c;
            const bool conflict = (nm & (bN | bD)) || (dm & bN);
            if (conflict || global_n) {
                bN |= nm;
                bD |= dm;
                blocked.push_back(gi);
            } else {
                GateRec e = g;
                for (int t = 0; t < g.k; ++t) e.wires[t] = phys[g.wires[t]];
                for (int &c : e.ctls) c = phys[c];
                seg.push_back(std::move(e));
            }
        }
        if (blocked.empty()) {
            last_seg = std::move(seg);
            break;
        }
        if (!seg.empty()) {
            auto passes = plan_passes(seg, ident, cfg, p.encs);
            for (auto &ph : passes) {
                Step s;
                s.kind = 0;
                s.pass = static_cast<int>(p.passes.size());
                p.passes.push_back(std::move(ph));
                p.steps.push_back(std::move(s));
            }
        }
        rem.swap(blocked);
        // swap in the rank-bit targets of the first blocked gate (it is blocked
        // only by them: everything before it has run), plus those of the next
        // blocked gates (look-ahead) while rank bits remain, in one step
        Step s;
        s.kind = 1;
        std::vector<int> keep, want; // local bits that must stay / rank-bit wires to bring in
        {
            // look-ahead wants are bounded by the local bits left for victims
            // (a state with few local qubits cannot take the whole frontier)
            const size_t look = std::min<size_t>(rem.size(), 64);
            for (size_t j = 0; j < look && static_cast<int>(want.size()) < p.ctx->gbits; ++j) {
                const GateRec &h = p.gates[rem[j]];
                if (h.diag) continue;
                for (int t = 0; t < h.k; ++t) {
                    const int b = phys[h.wires[t]];
                    if (b < nl) {
                        if (j == 0) keep.push_back(b);
                    } else if (std::find(want.begin(), want.end(), h.wires[t]) == want.end() &&
                               (j == 0 || (static_cast<int>(want.size()) < p.ctx->gbits &&
                                           static_cast<int>(want.size() + keep.size()) < nl)))
                        want.push_back(h.wires[t]);
                }
            }
            require(static_cast<int>(want.size() + keep.size()) <= nl,
                    "dist: a gate needs more local qubits than each rank holds (" + std::to_string(nl) +
                        "); use fewer ranks");
        }
        for (int w : want) {
            const int gb = phys[w];
            if (gb < nl) continue;
            // victim: the local wire needed furthest in the future; among
            // equally distant ones (or ones not needed before the next few
            // gates) the highest bit, whose halves are contiguous runs
            // ties -> a bit outside the tile of the pass just before the
            // swap (the swap can then be fused into that pass, see
            // fuse_swaps_into_passes), then the highest bit
            uint64_t prev_tile = 0;
            if (!p.steps.empty() && p.steps.back().kind == 0)
                for (int t : p.passes[p.steps.back().pass].tile_pos) prev_tile |= 1ull << t;
            const char *slack_env = std::getenv("QSV_SWAP_SLACK");
            const size_t slack = slack_env ? std::strtoull(slack_env, nullptr, 10) : 0;
            size_t far = 0; // Belady: the furthest next use among the candidates
            auto candidate = [&](int lb) {
                if (std::find(keep.begin(), keep.end(), lb) != keep.end()) return false;
                for (int w : want)
                    if (wire_at[lb] == w) return false;
                return true;
            };
            for (int lb = nl - 1; lb >= 0; --lb)
                if (candidate(lb)) far = std::max(far, next_use(wire_at[lb], 0));
            // within `slack` gates of it (QSV_SWAP_SLACK, default 0: ties
            // only -- a one-layer slack measured more passes and swaps on the
            // cfg4 family), a bit outside the previous pass's tile wins (its
            // fused stores keep whole tiles together), then the furthest,
            // then the highest bit
            int best = -1;
            size_t best_use = 0;
            bool best_free = false;
            for (int lb = nl - 1; lb >= 0; --lb) {
                if (!candidate(lb)) continue;
                const size_t score = next_use(wire_at[lb], 0);
                const bool free_bit = !((prev_tile >> lb) & 1) && score + slack >= far;
                if (best < 0 || (free_bit && !best_free) || (free_bit == best_free && score > best_use))
                    best = lb, best_use = score, best_free = free_bit;
            }
            require(best >= 0, "dist: no local qubit available for a swap");
            keep.push_back(best);
            s.swap_bits.emplace_back(gb, best);
            const int wg = wire_at[gb], wl = wire_at[best];
            std::swap(phys[wg], phys[wl]);
            wire_at[gb] = wl;
            wire_at[best] = wg;
        }
        p.steps.push_back(std::move(s));
    }
    // Restore the canonical layout so the API always sees logical order.
    // Phase A: put the right wire on every rank bit (global<->local swaps).
    const std::vector<int> canon = p.perm_in;
    std::vector<int> wire_of_canon(n);
    for (int w = 0; w < n; ++w) wire_of_canon[canon[w]] = w;
    std::vector<int> where(n); // physical bit after the last gate -> after the restore
    for (int b = 0; b < n; ++b) where[b] = b;
    auto do_swap = [&](Step &s, int a, int b) { // exchange physical bits a, b
        s.swap_bits.emplace_back(a, b);
        const int wa = wire_at[a], wb = wire_at[b];
        std::swap(phys[wa], phys[wb]);
        wire_at[a] = wb;
        wire_at[b] = wa;
        for (int &x : where) x = x == a ? b : x == b ? a : x;
    };
    Step back;
    back.kind = 1;
    for (int gb = nl; gb < n; ++gb) {
        const int want = wire_of_canon[gb];
        int x = phys[want];
        if (x == gb) continue;
        if (x >= nl) { // parked on another rank bit: bring it local first
            int lb = nl - 1;
            do_swap(back, x, lb);
            x = lb;
        }
        do_swap(back, gb, x);
    }
    // Phase B: local bits permuted among themselves. With relabeled swap
    // gates: one permutation-only pass (out of place, balanced read / write
    // runs); else local swap gates, expressed on PHYSICAL bits (identity
    // mapping) and fused into passes.
    std::vector<int> out_perm;
    if (relabel) {
        out_perm.assign(nl, 0);
        bool moved = false;
        for (int b = 0; b < nl; ++b) {
            out_perm[b] = canon[wire_at[b]];
            moved = moved || out_perm[b] != b;
        }
        if (!moved) out_perm.clear();
        for (int &x : where)
            if (x < nl && !out_perm.empty()) x = out_perm[x];
    }
    // the final front, with the restore's coalescing run in its last tile
    // when it fits: the input bits that land on the L lowest output bits
    // (so the restore can be fused into it, fuse_swaps_into_passes)
    if (!last_seg.empty()) {
        uint64_t need = 0;
        bool ok = relabel;
        for (int b = 0; b < n && ok; ++b)
            if (where[b] < cfg.L) {
                if (b >= nl) ok = false;
                else need |= 1ull << b;
            }
        auto passes = plan_passes(last_seg, ident, cfg, p.encs, {}, ok ? need : 0);
        for (auto &ph : passes) {
            Step s;
            s.kind = 0;
            s.pass = static_cast<int>(p.passes.size());
            p.passes.push_back(std::move(ph));
            p.steps.push_back(std::move(s));
        }
    }
    if (!back.swap_bits.empty()) p.steps.push_back(std::move(back));
    if (!out_perm.empty()) {
        PlanConfig c1 = cfg;
        c1.super_bits = 0;
        auto passes = plan_passes({}, ident, c1, p.encs, out_perm);
        for (auto &ph : passes) {
            Step st;
            st.pass = static_cast<int>(p.passes.size());
            p.passes.push_back(std::move(ph));
            p.steps.push_back(std::move(st));
        }
        for (int w = 0; w < n; ++w) phys[w] = canon[w], wire_at[canon[w]] = w;
    }
    std::vector<GateRec> fix;
    for (int w = 0; w < n; ++w) {
        if (phys[w] == canon[w]) continue;
        const int a = phys[w], b = canon[w];
        GateRec sw;
        sw.name = "swap";
        sw.kind = GK_SWAP;
        sw.k = 2;
        sw.wires[0] = a;
        sw.wires[1] = b;
        for (auto &x : sw.m) x = 0;
        sw.m[0] = sw.m[15] = sw.m[6] = sw.m[9] = 1;
        fix.push_back(sw);
        const int wa = wire_at[a], wb = wire_at[b];
        std::swap(phys[wa], phys[wb]);
        wire_at[a] = wb;
        wire_at[b] = wa;
    }
    if (!fix.empty()) {
        auto passes = plan_passes(fix, ident, cfg, p.encs);
        for (auto &ph : passes) {
            Step s;
            s.pass = static_cast<int>(p.passes.size());
            p.passes.push_back(std::move(ph));
            p.steps.push_back(std::move(s));
        }
    }
    p.perm_out = phys;
    fuse_swaps_into_passes(p);
}

} // namespace

namespace {
// From |0...0>, the gates a wire sees before any multi-qubit gate, control
// or swap touches it leave it in a product state: per wire a 2-vector
// M_k ... M_1 |0>, evaluated per row on the device (encoded gates included)
// and synthesised inside the first pass instead of loading the state
// (cfg2: the encoding layer and the first U3 layer never run as gates).
void extract_prefix(Plan &p) {
    const int n = p.n;
    std::vector<std::vector<const GateRec *>> pre(n);
    std::vector<char> open(n, 1);
    std::vector<GateRec> rest;
    for (const GateRec &g : p.gates) {
        const bool single = g.k == 1 && g.ctls.empty() && g.flags == 0 && g.kind != GK_SWAP;
        if (single && open[g.wires[0]]) {
            pre[g.wires[0]].push_back(&g);
            continue;
        }
        for (int t = 0; t < g.k; ++t) open[g.wires[t]] = 0;
        for (int c : g.ctls) open[c] = 0;
        rest.push_back(g);
    }
    bool any = false;
    for (const auto &v : pre) any = any || !v.empty();
    if (!any || rest.empty()) return;
    std::vector<int> prog(n + 1, 0), entries;
    for (int w = 0; w < n; ++w) {
        prog[w] = static_cast<int>(entries.size());
        for (const GateRec *g : pre[w]) {
            if (g->encoded) {
                EncDesc e{};
                e.kind = g->kind;
                e.slot = g->enc_slot;
                e.nparams = g->nparams;
                e.diag = 0;  // the full 2x2 matrix
                entries.push_back(static_cast<int>(p.encs.size()));
                p.encs.push_back(e);
            } else {
                entries.push_back(-1 - static_cast<int>(p.prefix_mats.size() / 4));
                p.prefix_mats.insert(p.prefix_mats.end(), g->m, g->m + 4);
            }
        }
    }
    prog[n] = static_cast<int>(entries.size());
    for (int &o : prog) o += n + 1;  // entries follow the offset table
    prog.insert(prog.end(), entries.begin(), entries.end());
    p.prefix_prog = std::move(prog);
    std::vector<GateRec> keep;
    keep.swap(rest);
    p.gates = std::move(keep);
    p.synth = true;
}
} // namespace

namespace {
void build_plan_at(Plan &pl, Ctx *ctx, int n, int dtype, std::vector<GateRec> gates, int nslots, const qsv_opts *opts,
                   const std::vector<int> *layout);
}

void build_plan(Plan &pl, Ctx *ctx, int n, int dtype, std::vector<GateRec> gates, int nslots, const qsv_opts *opts) {
    build_plan_at(pl, ctx, n, dtype, std::move(gates), nslots, opts, nullptr);
}

namespace {
// `layout` (lazy layouts, one GPU): the wire -> physical bit map of the
// states this plan runs on; nullptr = canonical.
void build_plan_at(Plan &pl, Ctx *ctx, int n, int dtype, std::vector<GateRec> gates, int nslots, const qsv_opts *opts,
                   const std::vector<int> *layout) {
    require(n >= 1 && n <= kMaxQubits, "plan: nqubit out of range");
    require(dtype == QSV_C64 || dtype == QSV_C128, "plan: bad dtype");
    Plan *p = &pl;
    p->ctx = ctx;
    p->n = n;
    p->dtype = dtype;
    p->nlocal = n - ctx->gbits;
    require(p->nlocal >= 1, "plan: more ranks than amplitudes");
    if (opts) p->opts = *opts;
    else p->opts.fuse = 1;
    p->gates = std::move(gates);
    p->nslots = nslots;
    p->ngates = static_cast<int>(p->gates.size());
    PlanConfig cfg;
    cfg.nlocal = p->nlocal;
    cfg.dtype = dtype;
    cfg.K = p->opts.tile_bits > 0 ? std::min(p->opts.tile_bits, kMaxTileBits) : default_tile_bits(dtype, p->nlocal);
    cfg.K = std::min(cfg.K, p->nlocal);
    cfg.L = p->opts.low_bits > 0 ? p->opts.low_bits : default_low_bits(dtype, p->nlocal);
    cfg.L = std::max(dtype == QSV_C64 ? 1 : 0, std::min(cfg.L, cfg.K));
    cfg.fuse = p->opts.fuse != 0;
    cfg.fuse_1q = p->opts.no_fuse_1q == 0;
    cfg.phase_flush = p->opts.no_phase_flush == 0;
    // complex128: 3-qubit register groups (8 amplitudes = 32 registers) keep a
    // 512-thread CTA under 64 registers, i.e. 32 warps per SM at 2 CTAs/SM
    cfg.R = p->opts.reg_slots > 0 ? std::min(p->opts.reg_slots, kMaxSlots) : 0; // 0: per pass (planner.cpp)
    require(cfg.K - cfg.L >= 2 || cfg.K == p->nlocal, "plan: tile too small (need tile_bits - low_bits >= 2)");
    p->perm_in = canonical_perm(n);
    const bool lazy = p->opts.lazy_layout != 0 && ctx->world == 1 && !p->opts.from_zero;
    if (layout) {
        require(ctx->world == 1 && static_cast<int>(layout->size()) == n, "plan: layouts are single-GPU");
        p->perm_in = *layout;
    }
    const bool canon_in = p->perm_in == canonical_perm(n);
    if (lazy && canon_in) p->src_gates = p->gates;  // the base plan: variants are re-planned from these
    if (canon_in && p->opts.dense_blocks == 0 && dtype == QSV_C64 && ctx->world == 1 && p->nslots == 0 && p->nlocal >= kDenseTile &&
        cfg.fuse && p->opts.jit >= 0 && !p->gates.empty()) {
        // auto: tensor-core blocks when the fused 5-qubit blocks are deep in
        // genuinely dense gates (measured: ~40 dense two-qubit
        // gates per block run 2.7-5.4x faster on tensor cores; ~4 per block,
        // or layers of single-qubit rotations, run faster on the FFMA passes)
        std::vector<GateRec> phys = p->gates;
        for (GateRec &g : phys) {
            for (int t = 0; t < g.k; ++t) g.wires[t] = p->perm_in[g.wires[t]];
            for (int &c : g.ctls) c = p->perm_in[c];
        }
        std::vector<DenseBlock> blocks;
        std::vector<DensePass> dps;
        bool ok = true;
        for (const GateRec &g : phys)
            ok = ok && !g.encoded && g.flags == 0 && static_cast<int>(g.ctls.size()) + g.k <= kDenseQ;
        if (ok) {
            plan_dense(phys, p->nlocal, blocks, dps);
            long nd = 0;
            for (const DenseBlock &b : blocks) nd += b.ndense;
            if (!blocks.empty() && nd >= kDenseAutoPerBlock * static_cast<long>(blocks.size())) {
                p->dblocks = std::move(blocks);
                p->dpasses = std::move(dps);
                p->dense = true;
                p->perm_out = p->perm_in;
                if (ctx->stream || ctx->device >= 0) dense_upload(*p);
                return;
            }
        }
    }
    if (p->opts.dense_blocks > 0 && canon_in) {
        // dense-block plan (tensor cores): every gate fused into <= 5-qubit
        // blocks on physical bits (canonical layout: wire w is bit n-1-w)
        require(dtype == QSV_C64, "dense blocks: complex64 plans only (tf32 tensor cores)");
        require(ctx->world == 1, "dense blocks: one GPU");
        require(p->nslots == 0, "dense blocks: encoded gates are not supported");
        std::vector<GateRec> phys = p->gates;
        for (GateRec &g : phys) {
            for (int t = 0; t < g.k; ++t) g.wires[t] = p->perm_in[g.wires[t]];
            for (int &c : g.ctls) c = p->perm_in[c];
        }
        plan_dense(phys, p->nlocal, p->dblocks, p->dpasses);
        p->dense = true;
        p->perm_out = p->perm_in;
        if (ctx->stream || ctx->device >= 0) dense_upload(*p);
        return;
    }
    if (p->opts.from_zero && ctx->world == 1 && cfg.fuse && plan_uses_jit(*p)) extract_prefix(*p);
    // L2 super-passes (planner.cpp), opt-in: opts.super_bits (or
    // QSV_SUPER_BITS) = the largest chunk, e.g. 19 (C128) / 20 (C64) = 8 MiB.
    // Off by default: measured slower on B200 (DESIGN.md 4.1 -- a pass is
    // already co-limited by its shared-memory exchanges and latency, so two
    // passes' SM work in one launch costs what the saved HBM sweep gains).
    {
        static const int env = [] {
            const char *e = std::getenv("QSV_SUPER_BITS");
            return e ? std::atoi(e) : 0;
        }();
        int sb = p->opts.super_bits != 0 ? p->opts.super_bits : env;
        if (sb < 0 || !cfg.fuse || !plan_uses_jit(*p) || p->synth) sb = 0;
        cfg.super_bits = sb;
    }
    if (ctx->world == 1) {
        // swaps as relabelings, the final layout folded into the last pass
        bool relabel = cfg.fuse && p->opts.no_relabel == 0 && plan_uses_jit(*p) && p->nslots == 0;
        // relabelled swaps end in an out-of-place pass (a second state-sized
        // buffer); when two states do not fit, swaps move data in place
        if (relabel && ctx->stream) {
            size_t free_b = 0, total_b = 0;
            if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
                const double state = std::ldexp(static_cast<double>(dtype == QSV_C64 ? 8 : 16), p->nlocal);
                if (2.0 * state > 0.92 * static_cast<double>(total_b)) relabel = false;
            } else {
                cudaGetLastError();
            }
        }
        std::vector<GateRec> gl = p->gates;
        std::vector<int> phys = p->perm_in, out_perm;
        {  // QSV_SCATTER_OUT=1 (opt-in, measured slower): a final
           // permutation that does not fit the last tile by scattered stores
           // instead of an extra copy-out pass
            const char *e = std::getenv("QSV_SCATTER_OUT");
            cfg.scatter_out = relabel && e && e[0] == '1';
        }
        p->perm_out = p->perm_in;
        if (relabel) {
            std::vector<int> fin;
            gl = relabel_swaps(p->gates, p->perm_in, fin);
            for (int b = 0; b < n; ++b) phys[b] = b; // gates now name physical bits
            if (lazy) {
                p->perm_out = fin;  // the state leaves in the relabelled layout
            } else {                // restore the canonical layout in the last pass
                const std::vector<int> canon = canonical_perm(n);
                p->perm_out = canon;
                out_perm.assign(n, 0);
                bool moved = false;
                for (int w = 0; w < n; ++w) {
                    out_perm[fin[w]] = canon[w];
                    moved = moved || fin[w] != canon[w];
                }
                if (!moved) out_perm.clear();
            }
        }
        if (!gl.empty() || !out_perm.empty()) {
            const size_t encs0 = p->encs.size();
            auto passes = plan_passes(gl, phys, cfg, p->encs, out_perm);
            // complex64, default geometry: a memory-bound circuit (at most
            // 1.5 K dense register-group matrices per pass on average: the
            // QFT ~7.5, SU(4) brickworks ~17; cfg5's rotation layers ~27
            // stay on 13-bit tiles) runs faster on
            // 12-bit double-buffered tiles with 4-qubit register groups than
            // on the 13-bit single-buffered tiles that suit the compute-bound
            // ones (cfg5). Interleaved A/B, c64 QFT: 28q 4.10 -> 2.97 ms, 30q
            // 15.4 -> 12.0 ms, 32q 60.1 -> 53.8 ms. QSV_X_NOLIGHT=1: off.
            const char *nl_env = std::getenv("QSV_X_NOLIGHT");
            if (dtype == QSV_C64 && p->opts.tile_bits <= 0 && p->opts.reg_slots <= 0 && cfg.K == 13 &&
                p->nlocal > 13 && !(nl_env && nl_env[0] == '1')) {
                long dense = 0;
                for (const PassHost &ph : passes)
                    for (const HostOp &op : ph.ops)
                        if (op.code == OP_DENSE1 || op.code == OP_DENSE1R || op.code == OP_DENSE2) ++dense;
                if (2 * dense <= 3L * cfg.K * static_cast<long>(passes.size())) {  // <= 1.5 K per pass
                    PlanConfig light = cfg;
                    light.K = 12;
                    light.R = 4;
                    p->encs.resize(encs0);
                    passes = plan_passes(gl, phys, light, p->encs, out_perm);
                }
            }
            if (p->synth) {
                require(!passes.empty(), "plan: product-state prefix without a pass");
                passes.front().synth = true;
            }
            for (auto &ph : passes) {
                Step s;
                s.pass = static_cast<int>(p->passes.size());
                p->passes.push_back(std::move(ph));
                p->steps.push_back(std::move(s));
            }
        }
    } else {
        schedule_dist(*p, cfg);
    }
    if (ctx->stream || ctx->device >= 0) upload_plan(*p); // dry runs (qsv_plan_dry) stay on the host
}
} // namespace

void build_plan_from_abi(Plan &p, Ctx *ctx, int n, int dtype, const qsv_gate *gates, int ngates,
                         const qsv_opts *opts) {
    require(ngates >= 0 && (ngates == 0 || gates != nullptr), "plan: bad gate list");
    require(n >= 1 && n <= kMaxQubits, "plan: nqubit out of range");
    std::vector<GateRec> recs;
    int cursor = 0;
    for (int i = 0; i < ngates; ++i) recs.push_back(resolve_gate(gates[i], n, &cursor));
    build_plan(p, ctx, n, dtype, std::move(recs), cursor, opts);
}

bool plan_uses_jit(const Plan &p) {
    return p.opts.jit > 0 || (p.opts.jit == 0 && p.ngates >= 8 && p.nlocal >= 10);
}

// Cached CUDA graphs bake the device pointers of p.d_sync / p.d_prefix: a
// reallocation of either must drop them.
void drop_graphs(Plan &p) {
    for (auto &g : p.graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    p.graphs.clear();
}

namespace {
void ensure_scratch(State &st) {
    if (!st.scratch) {
        const size_t bytes = st.local_amps * st.amp_bytes() * static_cast<size_t>(st.batch);
        if (state_alloc(&st.scratch, bytes) != cudaSuccess) {
            cudaGetLastError();
            st.scratch = nullptr;
            fail(QSV_ERR_INTERNAL, "out-of-place pass: cannot allocate the scratch state (" + std::to_string(bytes) +
                                       " bytes); plan with opts.no_relabel = 1");
        }
    }
}

// One L2 super-pass launch: pass pi in place, then pass pi + 1 (in place or
// into the scratch state), chunk by chunk.
void run_pair(Plan &p, int pi, State &st, cudaStream_t s) {
    const DevPass &head = p.dev[pi], &tail = p.dev[pi + 1];
    const PassHost &ph = p.passes[pi];
    const uint64_t nchunks = static_cast<uint64_t>(st.batch) << (p.nlocal - ph.chunk_bits);
    const size_t bytes = (nchunks + 1) * sizeof(unsigned);
    if (bytes > p.d_sync_cap) {
        QSV_CUDA(cudaStreamSynchronize(s));
        drop_graphs(p);
        cudaFree(p.d_sync);
        p.d_sync = nullptr;
        QSV_CUDA(cudaMalloc(&p.d_sync, bytes));
        p.d_sync_cap = bytes;
    }
    QSV_CUDA(cudaMemsetAsync(p.d_sync, 0, bytes, s));
    void *out = st.d;
    if (tail.out_of_place) {
        ensure_scratch(st);
        out = st.scratch;
    }
    launch_pair(head, tail, st.d, out, st.batch, static_cast<unsigned *>(p.d_sync), nchunks, s);
    if (tail.out_of_place) {
        std::swap(st.d, st.scratch);
        st.p2p_cur ^= 1;
    }
}
} // namespace

// One GPU: the device array of the state's two buffers (the "peers" of a
// local_gperm pass's scattered stores), in the p2p_cur convention of the
// multi-GPU path: buffer i at [i], the current state at [p2p_cur].
void local_out_ready(State &st) {
    ensure_scratch(st);
    void *want[2];
    want[st.p2p_cur] = st.d;
    want[1 - st.p2p_cur] = st.scratch;
    if (st.d_peers && st.p2p_buf[0] == want[0] && st.p2p_buf[1] == want[1]) return;
    if (!st.d_peers) QSV_CUDA(cudaMalloc(reinterpret_cast<void **>(&st.d_peers), 2 * sizeof(void *)));
    st.p2p_buf[0] = want[0];
    st.p2p_buf[1] = want[1];
    QSV_CUDA(cudaMemcpy(st.d_peers, want, sizeof want, cudaMemcpyHostToDevice));
}

void run_local_gout(const DevPass &dp, State &st, cudaStream_t s) {
    local_out_ready(st);
    launch_gout(dp, st.d, st.batch, st.d_peers + (1 - st.p2p_cur), 0, 0, s);
    std::swap(st.d, st.scratch);
    st.p2p_cur ^= 1;
}

namespace {
// A pass that can do the swaps after it (PassHost::gperm) does so when every
// rank has peer memory (set up on first use, collectively).
bool use_gout(Plan &p, int pi, State &st) {
    if (p.ctx->world == 1 || p.passes[pi].gperm.empty() || !p.dev[pi].jit || p.passes[pi].local_gperm) return false;
    return dist_p2p_ready(st);
}

// The pass, then the swaps fused into it: every tile is stored straight into
// its destination rank's scratch state (peer memory over NVLink); once every
// rank's kernel is done (an all-reduce on the stream orders them) the scratch
// states become the states on every rank.
void run_gout(Plan &p, int pi, DevPass &dp, State &st, cudaStream_t s) {
    const PassHost &ph = p.passes[pi];
    DevPass &keep = p.dev[pi];
    if (!keep.jit_gout) {
        QSV_CUDA(cudaSetDevice(p.ctx->device));
        jit_prepare_gout(keep, ph, p.dtype, p.ctx->sm_count);
    }
    dp.jit_gout = keep.jit_gout;
    const int nl = p.nlocal, W = p.ctx->world;
    uint64_t lconst = 0;
    int rconst = 0;
    for (int b = nl; b < p.n; ++b) {
        const uint64_t bit = (static_cast<uint64_t>(p.ctx->rank) >> (b - nl)) & 1;
        const int q = ph.gperm[b];
        if (q < nl) lconst |= bit << q;
        else rconst |= static_cast<int>(bit << (q - nl));
    }
    void *const *dst = st.d_peers + static_cast<size_t>(1 - st.p2p_cur) * W;
    // write-after-read: a peer may still be reading the buffer this pass is
    // about to store into (its own out-of-place step, or the previous plan
    // execution's last step), so every rank must be here before anyone stores
    dist_p2p_barrier(st);
    launch_gout(dp, st.d, st.batch, dst, lconst, rconst, s);
    {  // transport counters: the amplitudes whose destination is another rank
        int m = 0;
        for (int b = 0; b < nl; ++b) m += ph.gperm[b] >= nl;
        if (m > 0) {
            p.ctx->stat_messages += (1ull << m) - 1;
            p.ctx->stat_bytes += static_cast<uint64_t>(std::ldexp(
                static_cast<double>(st.amp_bytes()) * st.batch * (1.0 - std::ldexp(1.0, -m)), nl));
        }
    }
    dist_p2p_barrier(st);
    std::swap(st.d, st.scratch);
    st.p2p_cur ^= 1;
}
} // namespace

void run_pass(const DevPass &dp, int dtype, State &st, cudaStream_t s, double *zout) {
    if (!dp.out_of_place) {
        launch_pass(dp, dtype, st.d, st.batch, s, zout);
        return;
    }
    require(zout == nullptr, "fused <Z>: not on a permuting pass");
    ensure_scratch(st);
    launch_jit(dp, st.d, st.scratch, st.batch, s);
    std::swap(st.d, st.scratch);
    st.p2p_cur ^= 1;
}

void upload_plan(Plan &p) {
    // one device blob holding every pass program (each 16-byte aligned), one
    // table array
    std::vector<unsigned char> blob;
    std::vector<unsigned char> tables;
    const size_t tsz = p.dtype == QSV_C64 ? 8 : 16;
    struct Off {
        size_t blob, bytes, table;
        int ot, orc, oo;
    };
    std::vector<Off> offs;
    for (const PassHost &ph : p.passes) {
        Off o{};
        std::vector<unsigned char> b = serialize_program(ph, p.dtype, &o.ot, &o.orc, &o.oo);
        o.blob = blob.size();
        o.bytes = (b.size() + 15) / 16 * 16;
        b.resize(o.bytes, 0);
        blob.insert(blob.end(), b.begin(), b.end());
        o.table = tables.size() / tsz;
        for (const cplx &c : ph.tables) {
            unsigned char buf[16];
            if (p.dtype == QSV_C64) {
                const float f[2] = {static_cast<float>(c.real()), static_cast<float>(c.imag())};
                std::memcpy(buf, f, 8);
            } else {
                const double f[2] = {c.real(), c.imag()};
                std::memcpy(buf, f, 16);
            }
            tables.insert(tables.end(), buf, buf + tsz);
        }
        offs.push_back(o);
    }
    QSV_CUDA(cudaSetDevice(p.ctx->device));
    auto up = [](void **dst, const void *src, size_t bytes) {
        QSV_CUDA(cudaMalloc(dst, std::max<size_t>(bytes, 16)));
        if (bytes) QSV_CUDA(cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice));
    };
    up(&p.d_blob, blob.data(), blob.size());
    up(&p.d_tables, tables.data(), tables.size());
    if (!p.encs.empty()) up(&p.d_encs, p.encs.data(), p.encs.size() * sizeof(EncDesc));
    if (p.synth) {
        up(&p.d_prefix_prog, p.prefix_prog.data(), p.prefix_prog.size() * sizeof(int));
        up(&p.d_prefix_mats, p.prefix_mats.data(), p.prefix_mats.size() * sizeof(cplx));
    }
    const size_t amp = p.dtype == QSV_C64 ? 8 : 16;
    p.dev.clear();
    for (size_t i = 0; i < p.passes.size(); ++i) {
        const PassHost &ph = p.passes[i];
        const Off &o = offs[i];
        DevPass dp;
        PassArgs &a = dp.args;
        a.row_stride = 1ull << p.nlocal;
        a.rank_base = static_cast<uint64_t>(p.ctx->rank) << p.nlocal;
        a.tiles_per_row = 1ull << (p.nlocal - ph.K);
        a.blob = static_cast<const unsigned char *>(p.d_blob) + o.blob;
        a.blob_bytes = static_cast<int>(o.bytes);
        a.off_targets = o.ot;
        a.off_recs = o.orc;
        a.off_ops = o.oo;
        a.tables = static_cast<const unsigned char *>(p.d_tables) + o.table * tsz;
        a.nlocal = p.nlocal;
        a.K = ph.K;
        a.L = ph.L;
        a.ngroups = static_cast<int>(ph.groups.size());
        a.next = static_cast<int>(ph.ext_pos.size());
        for (int j = 0; j < ph.K; ++j) a.tile_pos[j] = ph.tile_pos[j];
        for (int j = 0; j < a.next; ++j) a.ext_pos[j] = ph.ext_pos[j];
        dp.R = ph.R;
        const int nsets = 1 << (ph.K - ph.R);
        const int chunks = static_cast<int>(((1ull << ph.K) * amp) / 16);
        dp.threads = std::max(32, std::min(256, std::max(nsets, std::min(chunks, 256))));
        dp.threads = (dp.threads + 31) / 32 * 32;
        dp.smem = tile_prog_offset(ph.K, ph.L, static_cast<int>(amp)) + o.bytes;
        require(dp.smem + 1024 <= p.ctx->smem_optin || p.ctx->smem_optin == 0,
                "plan: pass program does not fit in shared memory");
        dp.grid = std::max(1, tile_kernel_blocks_per_sm(p.dtype, dp.R, dp.threads, dp.smem)) * p.ctx->sm_count;
        const bool use_jit = plan_uses_jit(p);
        require(!ph.synth || use_jit, "plan: a synthesising pass needs the specialised kernels");
        dp.out_of_place = !ph.out_perm.empty();
        require(!dp.out_of_place || use_jit, "plan: permuting passes need the specialised kernels");
        if (use_jit && ph.pair == 1) jit_prepare_pair(dp, ph, p.passes[i + 1], p.dtype, p.ctx->sm_count);
        else if (use_jit && ph.pair == 2) dp.pair = 2;  // runs inside its head's launch
        else if (use_jit) jit_prepare(dp, ph, p.dtype, p.ctx->sm_count);
        if (use_jit && ph.local_gperm) jit_prepare_gout(dp, ph, p.dtype, p.ctx->sm_count);  // scattered stores
        dp.bytes = 2.0 * amp * static_cast<double>(1ull << p.nlocal);
        dp.ngates = ph.ngates;
        p.dev.push_back(dp);
    }
}

namespace {
void execute_steps(Plan &p, State &st, const void *enc_table, int rows, double *zout);
}

// opts.use_graph: one CUDA graph per (state, its two buffers, rows) replays
// the whole launch sequence (prefix, passes, super-pass memsets) -- one
// launch instead of one per pass, for launch-bound small states. Single GPU,
// no encoded data (its host upload is per call), no fused <Z> epilogue.
bool execute_graph(Plan &p, State &st) {
    if (!p.opts.use_graph || p.ctx->world != 1 || p.nslots != 0 || !p.ctx->stream) return false;
    cudaStream_t s = p.ctx->stream;
    bool oop = false, lg = false;
    for (const DevPass &dp : p.dev) oop = oop || dp.out_of_place;
    for (const PassHost &ph : p.passes) lg = lg || ph.local_gperm;
    if (oop || lg) ensure_scratch(st);
    if (lg) local_out_ready(st);  // no allocation or copy inside the capture
    for (size_t i = 0; i < p.passes.size(); ++i)
        if (p.dev[i].pair == 1) { // counters sized before capture (no allocation inside)
            const uint64_t nchunks = static_cast<uint64_t>(st.batch) << (p.nlocal - p.passes[i].chunk_bits);
            const size_t bytes = (nchunks + 1) * sizeof(unsigned);
            if (bytes > p.d_sync_cap) {
                QSV_CUDA(cudaStreamSynchronize(s));
                drop_graphs(p);
                cudaFree(p.d_sync);
                p.d_sync = nullptr;
                QSV_CUDA(cudaMalloc(&p.d_sync, bytes));
                p.d_sync_cap = bytes;
            }
        }
    if (p.synth && static_cast<size_t>(st.batch) > p.prefix_rows) {
        QSV_CUDA(cudaStreamSynchronize(s));
        drop_graphs(p);
        cudaFree(p.d_prefix);
        p.d_prefix = nullptr;
        QSV_CUDA(cudaMalloc(&p.d_prefix, static_cast<size_t>(st.batch) * p.nlocal * 2 * (p.dtype == QSV_C64 ? 8 : 16)));
        p.prefix_rows = st.batch;
    }
    // the graph bakes the device pointers and the row count, nothing else
    for (auto &g : p.graphs)
        if (g.d == st.d && g.scratch == st.scratch && g.batch == st.batch) {
            QSV_CUDA(cudaGraphLaunch(g.exec, s));
            if (g.flips) {
                std::swap(st.d, st.scratch);
                st.p2p_cur ^= 1;
            }
            return true;
        }
    if (p.graphs.size() >= 8) { // states come and go: keep the newest few
        cudaGraphExecDestroy(p.graphs.front().exec);
        p.graphs.erase(p.graphs.begin());
    }
    Plan::Graph g;
    g.d = st.d;
    g.scratch = st.scratch;
    g.batch = st.batch;
    cudaGraph_t graph = nullptr;
    QSV_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    try {
        if (p.synth) launch_prefix(p, st.batch, s);
        execute_steps(p, st, nullptr, 0, nullptr);
    } catch (...) {
        cudaStreamEndCapture(s, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
    }
    QSV_CUDA(cudaStreamEndCapture(s, &graph));
    g.flips = st.d != g.d;
    const cudaError_t rc = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    QSV_CUDA(rc);
    QSV_CUDA(cudaGraphLaunch(g.exec, s)); // capture recorded the work; now run it
    p.graphs.push_back(g);
    return true;
}

bool layout_canonical(const State &st) {
    for (int w = 0; w < st.n; ++w)
        if (st.perm[w] != st.n - 1 - w) return false;
    return true;
}

// One permutation-only pass (out of place, balanced read / write runs) from
// the state's layout to the canonical one; the plan is kept per context and
// input layout (a lazily laid-out state meets only a few).
void normalize_layout(State &st) {
    if (st.ctx->world != 1 || layout_canonical(st)) return;
    Ctx &c = *st.ctx;
    Plan *q = nullptr;
    for (auto &e : c.layout_plans)
        if (e.first == st.perm && e.second->dtype == st.dtype && e.second->n == st.n) q = e.second.get();
    if (!q) {
        auto np = std::make_shared<Plan>();
        qsv_opts o{};
        o.fuse = 1;
        o.jit = 1;  // the permuting pass is a specialised kernel
        build_plan_at(*np, st.ctx, st.n, st.dtype, {}, 0, &o, &st.perm);
        require(np->perm_out == canonical_perm(st.n) && !np->passes.empty(),
                "layout restore: needs a second state buffer (relabelled layouts)");
        if (c.layout_plans.size() >= 8) c.layout_plans.erase(c.layout_plans.begin());
        c.layout_plans.emplace_back(st.perm, np);
        q = np.get();
    }
    execute_plan(*q, st, nullptr, 0, 0);
}

namespace {
// The plan that runs on the state's current layout: p itself, or (lazy
// layouts) p re-planned from that layout, once per layout met.
Plan &plan_for_layout(Plan &p, State &st) {
    if (p.ctx->world != 1 || st.perm == p.perm_in) return p;
    if (p.opts.from_zero) {  // the state's contents are replaced: any layout will do
        st.perm = p.perm_in;
        return p;
    }
    if (p.src_gates.empty() && p.ngates > 0) {  // not a lazy-layout plan
        normalize_layout(st);
        require(st.perm == p.perm_in, "plan: state layout");
        return p;
    }
    for (auto &v : p.variants)
        if (v.first == st.perm) return *v.second;
    auto v = std::make_unique<Plan>();
    build_plan_at(*v, p.ctx, p.n, p.dtype, p.src_gates, p.nslots, &p.opts, &st.perm);
    p.variants.emplace_back(st.perm, std::move(v));
    return *p.variants.back().second;
}
void execute_plan_body(Plan &p, State &st, const double *data, int rows, int slots, double *zout);
} // namespace

void execute_plan(Plan &p, State &st, const double *data, int rows, int slots, double *zout) {
    require(st.n == p.n && st.dtype == p.dtype, "plan/state mismatch (nqubit or dtype)");
    require(st.ctx == p.ctx, "plan/state belong to different contexts");
    Plan &q = plan_for_layout(p, st);
    execute_plan_body(q, st, data, rows, slots, zout);
    if (p.ctx->world == 1) {
        require(q.perm_out.size() == static_cast<size_t>(st.n), "plan: output layout");
        st.perm = q.perm_out;
    }
}

namespace {
void execute_plan_body(Plan &p, State &st, const double *data, int rows, int slots, double *zout) {
    require(st.n == p.n && st.dtype == p.dtype, "plan/state mismatch (nqubit or dtype)");
    require(st.ctx == p.ctx, "plan/state belong to different contexts");
    if (rows == 0) {
        require(p.nslots == 0, "circuit has encode slots but no data given"); // circuit.hpp:125
    } else {
        require(rows == st.batch, "data rows must equal the state's batch");
        require(slots == p.nslots, "data length " + std::to_string(slots) + " != encode slots " +
                                       std::to_string(p.nslots)); // circuit.hpp:134-136
    }
    cudaStream_t s = p.ctx->stream;
    QSV_CUDA(cudaSetDevice(p.ctx->device));
    if (p.dense) {
        require(zout == nullptr, "dense blocks: no fused <Z> epilogue");
        dense_execute(p, st, s);
        return;
    }
    if (zout == nullptr && rows == 0 && execute_graph(p, st)) return;
    const void *enc_table = nullptr;
    if (!p.encs.empty()) {
        const size_t dbytes = sizeof(double) * static_cast<size_t>(rows) * slots;
        if (dbytes > p.d_data_cap) {
            cudaFree(p.d_data);
            QSV_CUDA(cudaMalloc(&p.d_data, dbytes));
            p.d_data_cap = dbytes;
        }
        QSV_CUDA(cudaMemcpyAsync(p.d_data, data, dbytes, cudaMemcpyHostToDevice, s));
        if (static_cast<size_t>(rows) > p.enc_table_rows) {
            cudaFree(p.d_enc_table);
            const size_t tsz = (p.dtype == QSV_C64 ? 4 : 8) * 32 * p.encs.size() * static_cast<size_t>(rows);
            QSV_CUDA(cudaMalloc(&p.d_enc_table, tsz));
            p.enc_table_rows = rows;
        }
        launch_bind(p, static_cast<const double *>(p.d_data), rows, slots, s);
        enc_table = p.d_enc_table;
    }
    const int brows = rows > 0 ? rows : st.batch;
    if (p.synth) {
        const size_t need = static_cast<size_t>(brows) * p.nlocal * 2 * (p.dtype == QSV_C64 ? 8 : 16);
        if (static_cast<size_t>(brows) > p.prefix_rows) {
            QSV_CUDA(cudaStreamSynchronize(s));
            drop_graphs(p);
            cudaFree(p.d_prefix);
            p.d_prefix = nullptr;
            QSV_CUDA(cudaMalloc(&p.d_prefix, need));
            p.prefix_rows = brows;
        }
        launch_prefix(p, brows, s);
    }
    execute_steps(p, st, enc_table, rows, zout);
}
} // namespace

namespace {
void execute_steps(Plan &p, State &st, const void *enc_table, int rows, double *zout) {
    cudaStream_t s = p.ctx->stream;
    bool fused_done = false; // the last pass also did the swap steps after it
    for (size_t i = 0; i < p.steps.size(); ++i) {
        const Step &stp = p.steps[i];
        if (stp.fused && fused_done) continue;
        fused_done = false;
        if (stp.kind == 0 && p.dev[stp.pass].pair) {
            require(!zout || i + 1 < p.steps.size(), "fused <Z>: not on a super-pass");
            if (p.dev[stp.pass].pair == 1) run_pair(p, stp.pass, st, s);
        } else if (stp.kind == 0) {
            DevPass dp = p.dev[stp.pass];
            dp.args.enc_table = enc_table;
            dp.args.batch = rows > 0 ? rows : st.batch;
            dp.args.prefix = p.passes[stp.pass].synth ? p.d_prefix : nullptr;
            if (p.passes[stp.pass].local_gperm) {
                require(!zout, "fused <Z>: not on a permuting pass");
                run_local_gout(dp, st, s);
            } else if (use_gout(p, stp.pass, st)) {
                run_gout(p, stp.pass, dp, st, s);
                fused_done = true;
            } else {
                run_pass(dp, p.dtype, st, s, i + 1 == p.steps.size() ? zout : nullptr);
            }
        } else {
            dist_swap_bits(st, stp.swap_bits, nullptr, 0);
        }
    }
}
} // namespace

namespace {
// The last step can carry the fused <Z> epilogue: a specialised, in-place
// pass whose tile is the whole (single-GPU) row.
bool z_fusable(Plan &p) {
    if (p.steps.empty() || p.steps.back().kind != 0 || p.ctx->world != 1) return false;
    const int pi = p.steps.back().pass;
    const PassHost &ph = p.passes[pi];
    const DevPass &dp = p.dev[pi];
    return dp.jit != nullptr && !dp.out_of_place && !ph.local_gperm && ph.ext_pos.empty() && ph.out_perm.empty() &&
           ph.K == p.nlocal;
}
} // namespace

void execute_plan_z(Plan &p0, State &st, const double *data, int rows, int slots, double *host_out) {
    require(st.n == p0.n && st.dtype == p0.dtype, "plan/state mismatch (nqubit or dtype)");
    require(st.ctx == p0.ctx, "plan/state belong to different contexts");
    Plan &p = plan_for_layout(p0, st);
    const int n = st.n, K1 = p.nlocal + 1;
    if (!z_fusable(p)) {
        execute_plan_body(p, st, data, rows, slots, nullptr);
        if (p.ctx->world == 1) st.perm = p.perm_out;
        std::vector<double> z(static_cast<size_t>(st.batch) * 41);
        reduce_z_all(st, z.data());
        for (int b = 0; b < st.batch; ++b)
            for (int w = 0; w < n; ++w)
                host_out[static_cast<size_t>(b) * n + w] = z[b * 41] - 2.0 * z[b * 41 + 1 + st.perm[w]];
        return;
    }
    DevPass &last = p.dev[p.steps.back().pass];
    if (!last.jit_z) {
        QSV_CUDA(cudaSetDevice(p.ctx->device));
        jit_prepare_z(last, p.passes[p.steps.back().pass], p.dtype, p.ctx->sm_count);
    }
    const size_t zbytes = sizeof(double) * static_cast<size_t>(st.batch) * K1;
    if (zbytes > p.d_z_cap) {
        cudaFree(p.d_z);
        p.d_z = nullptr;
        QSV_CUDA(cudaMalloc(&p.d_z, zbytes));
        p.d_z_cap = zbytes;
    }
    execute_plan_body(p, st, data, rows, slots, static_cast<double *>(p.d_z));
    if (p.ctx->world == 1) st.perm = p.perm_out;
    // <Z_w> formed on the device, read back through pinned staging
    cudaStream_t s = p.ctx->stream;
    const size_t obytes = sizeof(double) * static_cast<size_t>(st.batch) * n;
    if (obytes > p.zout_cap) {
        QSV_CUDA(cudaStreamSynchronize(s));
        cudaFree(p.d_zout);
        cudaFreeHost(p.h_zout);
        p.d_zout = nullptr;
        p.h_zout = nullptr;
        p.zout_cap = 0;
        QSV_CUDA(cudaMalloc(reinterpret_cast<void **>(&p.d_zout), obytes));
        QSV_CUDA(cudaMallocHost(reinterpret_cast<void **>(&p.h_zout), obytes));
        p.zout_cap = obytes;
    }
    launch_z_finish(static_cast<const double *>(p.d_z), K1, st.batch, n, st.perm, p.d_zout, s);
    QSV_CUDA(cudaMemcpyAsync(p.h_zout, p.d_zout, obytes, cudaMemcpyDeviceToHost, s));
    QSV_CUDA(cudaStreamSynchronize(s));
    std::memcpy(host_out, p.h_zout, obytes);
}

void profile_plan(Plan &p0, State &st, double *launch_ms) {
    require(st.n == p0.n && st.dtype == p0.dtype, "plan/state mismatch (nqubit or dtype)");
    require(p0.nslots == 0, "profile: encoded plans not supported");
    Plan &p = plan_for_layout(p0, st);
    // launch_ms holds one entry per step of p0 (qsv_plan_info / qsv_plan_steps)
    require(p.steps.size() == p0.steps.size(), "profile: this layout's plan has another step count");
    struct SetLayout {  // the state leaves in the plan's output layout
        Plan &p;
        State &st;
        ~SetLayout() {
            if (p.ctx->world == 1) st.perm = p.perm_out;
        }
    } set_layout{p, st};
    cudaStream_t s = p.ctx->stream;
    if (p.dense) {
        dense_execute(p, st, s, launch_ms);
        return;
    }
    std::vector<cudaEvent_t> ev(2 * p.steps.size());
    for (auto &e : ev) QSV_CUDA(cudaEventCreate(&e));
    size_t k = 0;
    bool fused_done = false;
    for (const Step &stp : p.steps) {
        QSV_CUDA(cudaEventRecord(ev[2 * k], s));
        const bool skip = stp.fused && fused_done;
        fused_done = false;
        if (skip) {
            fused_done = true;
        } else if (stp.kind == 0 && p.dev[stp.pass].pair == 1) run_pair(p, stp.pass, st, s);
        else if (stp.kind == 0 && p.dev[stp.pass].pair == 2) {
        } else if (stp.kind == 0 && p.passes[stp.pass].local_gperm) {
            DevPass dp = p.dev[stp.pass];
            dp.args.batch = st.batch;
            run_local_gout(dp, st, s);
        } else if (stp.kind == 0 && use_gout(p, stp.pass, st)) {
            DevPass dp = p.dev[stp.pass];
            dp.args.batch = st.batch;
            run_gout(p, stp.pass, dp, st, s);
            fused_done = true;
        } else if (stp.kind == 0) run_pass(p.dev[stp.pass], p.dtype, st, s);
        else dist_swap_bits(st, stp.swap_bits, nullptr, 0);
        QSV_CUDA(cudaEventRecord(ev[2 * k + 1], s));
        ++k;
    }
    QSV_CUDA(cudaStreamSynchronize(s));
    for (size_t i = 0; i < p.steps.size(); ++i) {
        float ms = 0;
        QSV_CUDA(cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]));
        launch_ms[i] = ms;
    }
    for (auto &e : ev) cudaEventDestroy(e);
}

} // namespace qsv
