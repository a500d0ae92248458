// Fusion planner: lowers an ordered gate list onto shared-memory tile passes.
//
// The reference applies every gate as one full strided sweep of the state
// (Circuit::forward -> apply_gate -> apply_matrix_strided,
// /root/reference/proj/include/quasar/qubit/circuit.hpp:121-157,
// state.hpp:111-174). Here a PASS is one read+write of the state through
// shared memory: each CTA stages a tile of 2^K amplitudes whose index bits are
// the pass's K "tile qubits" (always including the L lowest physical bits so
// every global access is a contiguous >= 128 B run), applies every gate of the
// pass to it, and writes it back. Inside the tile the gates are applied in
// GROUPS: each thread holds 2^R amplitudes spanning the R group qubits in
// registers, so a group is one shared-memory sweep whatever its gate count.
//
// Scheduling is commutation-aware and greedy:
//   * a gate acts "N" (non-diagonal) on its targets when its matrix is not
//     diagonal, and "D" on its controls and on the targets of diagonal gates;
//   * two gates commute when every shared qubit is D for both (both are then
//     block diagonal in it and act on disjoint remaining qubits);
//   * only N qubits must live in the tile/group; D qubits are read from the
//     amplitude's index bits wherever they are (tile, outside the tile, or a
//     rank bit of a distributed state);
//   * a pass walks the remaining gates in order, admitting a gate when it does
//     not conflict with an earlier skipped gate and its N qubits fit in the
//     tile; otherwise the gate is skipped and blocks the qubits it touches.
// The same greedy, with capacity R over tile qubits, forms the groups.
#include <algorithm>
#include <bit>
#include <cmath>
#include <cstring>

#include "qsv_internal.hpp"

namespace qsv {

int default_tile_bits(int dtype, int nlocal) {
    const int k = dtype == QSV_C64 ? 13 : 12; // 64 KiB tiles: 3 CTAs per SM
    return std::min(k, nlocal);
}
int default_low_bits(int dtype, int nlocal) {
    const int l = dtype == QSV_C64 ? 4 : 3; // 128-byte contiguous runs
    return std::min(l, nlocal);
}

namespace {

struct PG {
    int idx;            // gate index
    uint64_t nmask = 0; // physical bits acted on non-diagonally
    uint64_t dmask = 0; // physical bits acted on diagonally (controls, diag targets)
};

inline bool conflicts(const PG &g, uint64_t bN, uint64_t bD) {
    return (g.nmask & (bN | bD)) || (g.dmask & bN);
}

// Greedy admission: returns admitted gate indices (positions into `order`),
// the qubits they claimed, and leaves the rest in `order`.
std::vector<int> admit(std::vector<int> &order, const std::vector<PG> &pg, uint64_t &active, int cap,
                       uint64_t allowed) {
    int cnt = std::popcount(active);
    uint64_t bN = 0, bD = 0;
    std::vector<int> took, rest;
    for (int i : order) {
        const PG &g = pg[i];
        bool ok = !conflicts(g, bN, bD);
        if (ok) {
            const uint64_t need = g.nmask & ~active;
            if ((need & ~allowed) || cnt + std::popcount(need) > cap) ok = false;
            else {
                active |= need;
                cnt += std::popcount(need);
            }
        }
        if (ok) took.push_back(i);
        else {
            bN |= g.nmask;
            bD |= g.dmask;
            rest.push_back(i);
        }
    }
    order.swap(rest);
    return took;
}

void set_m(TileOp<double> &op, const cplx *m, int d) {
    for (int i = 0; i < d * d; ++i) {
        op.m[2 * i] = m[i].real();
        op.m[2 * i + 1] = m[i].imag();
    }
}

} // namespace

// ---- single-qubit run fusion ----------------------------------------------
std::vector<GateRec> fuse_single_qubit_runs(const std::vector<GateRec> &gates) {
    std::vector<GateRec> out;
    std::vector<int> open(kMaxQubits, -1); // wire -> index in `out` of an open run
    for (const GateRec &g : gates) {
        const bool fusable = g.k == 1 && g.ctls.empty() && !g.encoded && g.flags == 0;
        if (fusable) {
            const int w = g.wires[0];
            if (open[w] >= 0) {
                GateRec &f = out[open[w]];
                cplx m[4];
                for (int r = 0; r < 2; ++r)
                    for (int c = 0; c < 2; ++c) m[r * 2 + c] = g.m[r * 2] * f.m[c] + g.m[r * 2 + 1] * f.m[2 + c];
                for (int i = 0; i < 4; ++i) f.m[i] = m[i];
                f.diag = (m[1] == cplx(0, 0) && m[2] == cplx(0, 0));
                f.name = "fused1q";
                f.kind = GK_CUSTOM;
                continue;
            }
            out.push_back(g);
            open[w] = static_cast<int>(out.size()) - 1;
            continue;
        }
        for (int t = 0; t < g.k; ++t) open[g.wires[t]] = -1;
        for (int c : g.ctls) open[c] = -1;
        out.push_back(g);
    }
    return out;
}

namespace {

bool is_unitary_diag(const GateRec &g) {
    const int d = 1 << g.k;
    for (int i = 0; i < d; ++i)
        if (std::abs(std::abs(g.m[i * d + i]) - 1.0) > 1e-12) return false;
    return true;
}

cplx eval_rec(const DiagRec &r, uint64_t pb) {
    if ((pb & r.fmask) != r.fval) return cplx(1, 0);
    int idx = 0;
    if (r.nt >= 1) idx = static_cast<int>((pb >> r.tpos0) & 1);
    if (r.nt == 2) idx = (idx << 1) | static_cast<int>((pb >> r.tpos1) & 1);
    return cplx(r.val[2 * idx], r.val[2 * idx + 1]);
}

uint64_t rec_deps(const DiagRec &r) {
    uint64_t d = r.fmask;
    if (r.nt >= 1) d |= 1ull << r.tpos0;
    if (r.nt == 2) d |= 1ull << r.tpos1;
    return d;
}

// Lowers the admitted gates of one register group into device ops. Unitary
// diagonal gates that depend on at most one register slot are not applied
// where they stand: their phase becomes a per-slot (or per-set "uniform")
// factor that floats forward -- diagonal gates commute with each other and
// with every gate not acting non-diagonally on their slot -- and is applied
// by one FLUSH right before the next non-diagonal gate on that slot, or at
// the end of the group. Each factor is split by the bits it reads:
//   EXT    only bits outside the tile: one value per CTA (shared memory);
//   TILE   only tile bits outside the group: a host-precomputed table over
//          the set index, shared by every CTA;
//   MIXED  both: evaluated per register set.
struct GroupLowering {
    PassHost &ph;
    const std::vector<GateRec> &gates;
    const std::vector<int> &phys;
    const int *slot_of_phys;
    int R;
    std::vector<EncDesc> &encs;
    bool flush_enabled;
    std::vector<int> ng_phys;                 // physical bits of the set index, LSB first
    std::vector<std::vector<DiagRec>> pend;   // per slot
    std::vector<DiagRec> pend_u;
    int n_ext = 0;

    GroupLowering(PassHost &p, const std::vector<GateRec> &g, const std::vector<int> &ph_, const int *sop, int r,
                  std::vector<EncDesc> &e, bool fe)
        : ph(p), gates(g), phys(ph_), slot_of_phys(sop), R(r), encs(e), flush_enabled(fe), pend(r) {}

    int slot(int wire) const {
        const int b = phys[wire];
        return b < 64 ? slot_of_phys[b] : -1;
    }

    void emit_target(int slot_id, const std::vector<DiagRec> &recs) {
        if (recs.empty()) return;
        uint64_t ngmask = 0;
        for (int b : ng_phys) ngmask |= 1ull << b;
        const uint64_t tilemask = ngmask;
        FlushTarget t{};
        t.slot = slot_id;
        t.table = -1;
        t.eidx = -1;
        std::vector<DiagRec> ext, tile, mix;
        for (const DiagRec &r : recs) {
            const uint64_t d = rec_deps(r);
            if ((d & ngmask) == 0) ext.push_back(r); // no tile dependence (tile group bits never appear)
            else if ((d & ~tilemask) == 0) tile.push_back(r);
            else mix.push_back(r);
        }
        if (!ext.empty() && n_ext >= kMaxExtTargets) {
            mix.insert(mix.end(), ext.begin(), ext.end());
            ext.clear();
        }
        t.ext_begin = static_cast<int>(ph.recs.size());
        ph.recs.insert(ph.recs.end(), ext.begin(), ext.end());
        t.ext_end = static_cast<int>(ph.recs.size());
        if (!ext.empty()) t.eidx = n_ext++;
        t.mix_begin = static_cast<int>(ph.recs.size());
        ph.recs.insert(ph.recs.end(), mix.begin(), mix.end());
        t.mix_end = static_cast<int>(ph.recs.size());
        if (!tile.empty()) {
            const int nset = 1 << ng_phys.size();
            t.table = static_cast<int>(ph.tables.size());
            for (int s = 0; s < nset; ++s) {
                uint64_t pb = 0;
                for (size_t i = 0; i < ng_phys.size(); ++i)
                    if ((s >> i) & 1) pb |= 1ull << ng_phys[i];
                cplx f(1, 0);
                for (const DiagRec &r : tile) f *= eval_rec(r, pb);
                ph.tables.push_back(f);
            }
        }
        ph.targets.push_back(t);
    }

    void flush(const std::vector<int> &slots, bool with_u) {
        const int t0 = static_cast<int>(ph.targets.size());
        for (int j : slots) {
            emit_target(j, pend[j]);
            pend[j].clear();
        }
        if (with_u) {
            emit_target(-1, pend_u);
            pend_u.clear();
        }
        const int t1 = static_cast<int>(ph.targets.size());
        if (t1 > t0) {
            TileOp<double> op{};
            op.type = OP_FLUSH;
            op.enc = -1;
            op.a = t0;
            op.b = t1;
            ph.ops.push_back(op);
        }
    }

    // Returns true when the diagonal gate was absorbed into pending factors.
    bool try_defer(const GateRec &g) {
        if (!flush_enabled || !g.diag || g.encoded || g.flags || !is_unitary_diag(g)) return false;
        DiagRec base{};
        int rc = -1, nrc = 0;
        for (int c : g.ctls) {
            const int s = slot(c);
            if (s >= 0) rc = s, ++nrc;
            else {
                base.fmask |= 1ull << phys[c];
                base.fval |= 1ull << phys[c];
            }
        }
        int rt = -1, rtpos = -1, nrt = 0;
        for (int t = 0; t < g.k; ++t)
            if (slot(g.wires[t]) >= 0) rt = slot(g.wires[t]), rtpos = t, ++nrt;
        const int d = 1 << g.k;
        cplx dv[4];
        for (int i = 0; i < d; ++i) dv[i] = g.m[i * d + i];
        auto setv = [](DiagRec &r, int i, cplx v) {
            r.val[2 * i] = v.real();
            r.val[2 * i + 1] = v.imag();
        };
        if (nrc + nrt == 0) {
            DiagRec r = base;
            r.nt = g.k;
            r.tpos0 = phys[g.wires[0]];
            if (g.k == 2) r.tpos1 = phys[g.wires[1]];
            for (int i = 0; i < d; ++i) setv(r, i, dv[i]);
            pend_u.push_back(r);
            return true;
        }
        if (nrc == 1 && nrt == 0) {
            DiagRec r = base;
            r.nt = g.k;
            r.tpos0 = phys[g.wires[0]];
            if (g.k == 2) r.tpos1 = phys[g.wires[1]];
            for (int i = 0; i < d; ++i) setv(r, i, dv[i]);
            pend[rc].push_back(r);
            return true;
        }
        if (nrc == 0 && nrt == 1) {
            DiagRec u = base, f = base;
            if (g.k == 1) {
                u.nt = f.nt = 0;
                setv(u, 0, dv[0]);
                setv(f, 0, dv[1] / dv[0]);
            } else {
                const int other = 1 - rtpos;
                u.nt = f.nt = 1;
                u.tpos0 = f.tpos0 = phys[g.wires[other]];
                for (int ob = 0; ob < 2; ++ob) {
                    const int i0 = rtpos == 0 ? (0 << 1) | ob : (ob << 1) | 0;
                    const int i1 = rtpos == 0 ? (1 << 1) | ob : (ob << 1) | 1;
                    setv(u, ob, dv[i0]);
                    setv(f, ob, dv[i1] / dv[i0]);
                }
            }
            pend_u.push_back(u);
            pend[rt].push_back(f);
            return true;
        }
        return false;
    }

    void add(int gi) {
        const GateRec &g = gates[gi];
        if (try_defer(g)) return;
        if (!g.diag) { // flush the pending factors of the slots it acts on non-diagonally
            std::vector<int> need;
            for (int t = 0; t < g.k; ++t) {
                const int s = slot(g.wires[t]);
                if (s >= 0 && !pend[s].empty()) need.push_back(s);
            }
            if (!need.empty()) flush(need, false);
        }
        lower(g);
    }

    void finish() {
        std::vector<int> all;
        for (int j = 0; j < R; ++j)
            if (!pend[j].empty()) all.push_back(j);
        flush(all, true);
    }

    void lower(const GateRec &g) {
        TileOp<double> op{};
        op.enc = -1;
        op.flags = g.flags & OPF_ZERO_OFF_CONTROL;
        for (int c : g.ctls) {
            const int s = slot(c);
            if (s >= 0) {
                op.rmask |= 1 << s;
                op.rval |= 1 << s;
            } else {
                op.fmask |= 1ull << phys[c];
                op.fval |= 1ull << phys[c];
            }
        }
        const int d = 1 << g.k;
        if (g.diag) {
            op.type = OP_DIAG;
            op.nt = g.k;
            int *tt[2] = {&op.t0, &op.t1};
            int *tr[2] = {&op.t0reg, &op.t1reg};
            for (int t = 0; t < g.k; ++t) {
                const int s = slot(g.wires[t]);
                *tt[t] = s >= 0 ? s : phys[g.wires[t]];
                *tr[t] = s >= 0 ? 1 : 0;
            }
            if (!g.encoded)
                for (int i = 0; i < d; ++i) {
                    op.m[2 * i] = g.m[i * d + i].real();
                    op.m[2 * i + 1] = g.m[i * d + i].imag();
                }
        } else if (g.k == 1) {
            op.a = slot(g.wires[0]);
            op.type = OP_DENSE1;
            if (!g.encoded) {
                set_m(op, g.m, 2);
                const bool real = g.m[0].imag() == 0 && g.m[1].imag() == 0 && g.m[2].imag() == 0 &&
                                  g.m[3].imag() == 0;
                if (real) op.type = OP_DENSE1R;
                if (g.m[0] == cplx(0, 0) && g.m[3] == cplx(0, 0) && g.m[1] == cplx(1, 0) && g.m[2] == cplx(1, 0) &&
                    !(g.flags & OPF_ZERO_OFF_CONTROL))
                    op.type = OP_X1;
            }
        } else {
            op.type = OP_DENSE2;
            const int s0 = slot(g.wires[0]), s1 = slot(g.wires[1]);
            const bool swapq = s0 < s1;
            op.a = swapq ? s1 : s0;
            op.b = swapq ? s0 : s1;
            if (!g.encoded) {
                cplx mm[16];
                for (int r = 0; r < 4; ++r)
                    for (int c = 0; c < 4; ++c) {
                        const int rr = swapq ? ((r & 1) << 1) | (r >> 1) : r;
                        const int cc = swapq ? ((c & 1) << 1) | (c >> 1) : c;
                        mm[r * 4 + c] = g.m[rr * 4 + cc];
                    }
                set_m(op, mm, 4);
            }
            if (g.encoded) {
                EncDesc e{};
                e.kind = g.kind;
                e.slot = g.enc_slot;
                e.nparams = g.nparams;
                e.swapq = swapq ? 1 : 0;
                e.diag = 0;
                op.enc = static_cast<int>(encs.size());
                encs.push_back(e);
            }
            ph.ops.push_back(op);
            return;
        }
        if (g.encoded) {
            EncDesc e{};
            e.kind = g.kind;
            e.slot = g.enc_slot;
            e.nparams = g.nparams;
            e.swapq = 0;
            e.diag = g.diag ? 1 : 0;
            op.enc = static_cast<int>(encs.size());
            encs.push_back(e);
        }
        ph.ops.push_back(op);
    }
};

} // namespace

std::vector<PassHost> plan_passes(const std::vector<GateRec> &gates_in, const std::vector<int> &phys,
                                  const PlanConfig &cfg, std::vector<EncDesc> &encs) {
    const int nl = cfg.nlocal;
    const int K = std::min(cfg.K, nl);
    const int L = std::min(cfg.L, K);
    const int R = std::min(cfg.R, K);
    require(K >= 1, "planner: empty local state");
    const uint64_t localmask = nl >= 64 ? ~0ull : ((1ull << nl) - 1);
    const std::vector<GateRec> fused = cfg.fuse_1q ? fuse_single_qubit_runs(gates_in) : gates_in;
    const std::vector<GateRec> &gates = fused;

    std::vector<PG> pg(gates.size());
    for (size_t i = 0; i < gates.size(); ++i) {
        const GateRec &g = gates[i];
        pg[i].idx = static_cast<int>(i);
        for (int t = 0; t < g.k; ++t) {
            const uint64_t b = 1ull << phys[g.wires[t]];
            if (g.diag) pg[i].dmask |= b;
            else {
                require(phys[g.wires[t]] < nl, "planner: non-diagonal target on a global qubit");
                pg[i].nmask |= b;
            }
        }
        for (int c : g.ctls) pg[i].dmask |= 1ull << phys[c];
    }

    // ---- passes -----------------------------------------------------------
    std::vector<std::vector<int>> pass_gates;
    std::vector<uint64_t> pass_active;
    std::vector<int> order(gates.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
    const uint64_t lowmask = (1ull << L) - 1;
    while (!order.empty()) {
        uint64_t active = lowmask;
        std::vector<int> took;
        if (cfg.fuse) took = admit(order, pg, active, K, localmask);
        else {
            const int i = order.front();
            order.erase(order.begin());
            active |= pg[i].nmask;
            took.push_back(i);
        }
        require(!took.empty(), "planner: no progress");
        pass_gates.push_back(std::move(took));
        pass_active.push_back(active);
    }

    std::vector<PassHost> passes;
    for (size_t p = 0; p < pass_gates.size(); ++p) {
        PassHost ph;
        ph.K = K;
        ph.L = L;
        uint64_t active = pass_active[p];
        // pad with the lowest free bits: lengthens the contiguous runs
        for (int b = 0; b < nl && std::popcount(active) < K; ++b) active |= 1ull << b;
        for (int b = 0; b < nl; ++b)
            if (active & (1ull << b)) ph.tile_pos.push_back(b);
            else ph.ext_pos.push_back(b);
        require(static_cast<int>(ph.tile_pos.size()) == K, "planner: tile size");
        int tile_of_phys[64];
        for (int &x : tile_of_phys) x = -1;
        for (int i = 0; i < K; ++i) tile_of_phys[ph.tile_pos[i]] = i;

        // ---- groups (capacity R over tile qubits) ---------------------------
        std::vector<int> gorder = pass_gates[p];
        ph.ngates = static_cast<int>(gorder.size()); // (after 1q fusion)
        while (!gorder.empty()) {
            uint64_t gact = 0;
            std::vector<int> took = admit(gorder, pg, gact, R, active);
            require(!took.empty(), "planner: no group progress");
            // slots: claimed tile bits, padded with the HIGHEST free tile bits so
            // the lanes of a warp walk the low (contiguous) tile bits.
            std::vector<int> slot_tile;
            for (int b = 0; b < nl; ++b)
                if (gact & (1ull << b)) slot_tile.push_back(tile_of_phys[b]);
            for (int t = K - 1; t >= 0 && static_cast<int>(slot_tile.size()) < R; --t)
                if (std::find(slot_tile.begin(), slot_tile.end(), t) == slot_tile.end()) slot_tile.push_back(t);
            GroupDesc gd{};
            gd.op_begin = static_cast<int>(ph.ops.size());
            int slot_of_phys[64];
            for (int &x : slot_of_phys) x = -1;
            for (int j = 0; j < R; ++j) {
                gd.slot_bit[j] = slot_tile[j];
                slot_of_phys[ph.tile_pos[slot_tile[j]]] = j;
            }
            int q = 0;
            for (int t = 0; t < K; ++t)
                if (std::find(slot_tile.begin(), slot_tile.end(), t) == slot_tile.end()) gd.ng_bit[q++] = t;

            GroupLowering low(ph, gates, phys, slot_of_phys, R, encs, cfg.phase_flush);
            low.ng_phys.clear();
            for (int i = 0; i < K - R; ++i) low.ng_phys.push_back(ph.tile_pos[gd.ng_bit[i]]);
            gd.tgt_begin = static_cast<int>(ph.targets.size());
            for (int gi : took) low.add(gi);
            low.finish();
            gd.tgt_end = static_cast<int>(ph.targets.size());
            gd.op_end = static_cast<int>(ph.ops.size());
            ph.groups.push_back(gd);
        }
        passes.push_back(std::move(ph));
    }
    return passes;
}

} // namespace qsv
