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
    // complex128: 32 KiB tiles, double-buffered (prefetch) -> 64 KiB per CTA;
    // complex64: 64 KiB single-buffered tiles (r01 sweep, scripts/sweep2.py)
    const int k = dtype == QSV_C64 ? 13 : 11;
    return std::min(k, nlocal);
}
int default_low_bits(int dtype, int nlocal) {
    const int l = dtype == QSV_C64 ? 4 : 3; // 128-byte contiguous runs
    return std::min(l, nlocal);
}

// ---- single-qubit run fusion ----------------------------------------------
std::vector<GateRec> fuse_single_qubit_runs(const std::vector<GateRec> &gates) {
    std::vector<GateRec> out;
    std::vector<int> open(64, -1); // wire -> index in `out` of an open run
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

struct PG {
    uint64_t nmask = 0; // physical bits acted on non-diagonally
    uint64_t dmask = 0; // physical bits acted on diagonally (controls, diag targets)
};

inline bool conflicts(const PG &g, uint64_t bN, uint64_t bD) { return (g.nmask & (bN | bD)) || (g.dmask & bN); }

// Greedy admission over `order` (ascending gate indices). Admitted gates are
// returned; the rest stay in `order`.
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

bool is_unitary_diag(const GateRec &g) {
    const int d = 1 << g.k;
    for (int i = 0; i < d; ++i)
        if (std::abs(std::abs(g.m[i * d + i]) - 1.0) > 1e-12) return false;
    return true;
}

// QSV_X_NOHOIST=1 (A/B switch): deferred diagonals stay in program order
bool hoist_diagonals() {
    const char *e = std::getenv("QSV_X_NOHOIST");
    return !(e && e[0] == '1');
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

void setv(DiagRec &r, int i, cplx v) {
    r.val[2 * i] = v.real();
    r.val[2 * i + 1] = v.imag();
}

// Lowers the admitted gates of one register group into HostOps.
//
// Unitary diagonal gates are not applied where they stand. Diagonal gates
// commute with each other and with every gate that is not non-diagonal on
// one of their qubits, so their phases are deferred and applied by a FLUSH
// right before the next non-diagonal gate on a register slot they depend on,
// or at the end of the group:
//   * phases over register slots only (no other bit) multiply into one
//     2^R-entry register table, computed here;
//   * phases over exactly one register slot plus fixed bits become per-slot
//     factors, phases over fixed bits only a per-set uniform factor. Each is
//     split by the fixed bits it reads: EXT (only bits outside the tile: one
//     value per tile, computed by the CTA), TILE (only tile bits outside the
//     group: a host table over the set index, shared by every CTA), MIXED
//     (both: evaluated per register set);
//   * anything else (two register slots AND fixed bits, non-unitary, or
//     encoded) is applied where it stands (OP_DIAG).
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
    std::vector<cplx> pend_reg;               // register table
    unsigned pend_reg_slots = 0;
    int n_ext = 0;
    bool x_through = [] {  // QSV_X_NOXPERM=1 (A/B): flush before every X instead
        const char *e = std::getenv("QSV_X_NOXPERM");
        return !(e && e[0] == '1');
    }();

    GroupLowering(PassHost &p, const std::vector<GateRec> &g, const std::vector<int> &ph_, const int *sop, int r,
                  std::vector<EncDesc> &e, bool fe)
        : ph(p), gates(g), phys(ph_), slot_of_phys(sop), R(r), encs(e), flush_enabled(fe), pend(r),
          pend_reg(1u << r, cplx(1, 0)) {}

    int slot(int wire) const {
        const int b = phys[wire];
        return b < 64 ? slot_of_phys[b] : -1;
    }

    int emit_target(int slot_id, const std::vector<DiagRec> &recs) {
        if (recs.empty()) return 0;
        uint64_t ngmask = 0;
        for (int b : ng_phys) ngmask |= 1ull << b;
        FlushTarget t{};
        t.slot = slot_id;
        t.table = -1;
        t.eidx = -1;
        std::vector<DiagRec> ext, tile, mix;
        for (const DiagRec &r : recs) {
            const uint64_t d = rec_deps(r);
            if ((d & ngmask) == 0) ext.push_back(r);      // bits outside the tile only
            else if ((d & ~ngmask) == 0) tile.push_back(r); // tile bits outside the group only
            else mix.push_back(r);
        }
        if (!ext.empty() && n_ext >= kMaxExtTargets) {
            mix.insert(mix.end(), ext.begin(), ext.end());
            ext.clear();
        }
        // per-tile records over the tile index bits (ext_pos) that stay inside
        // one 8-bit chunk of the tile index become chunk tables
        t.ext_tab = -1;
        t.ext_chunks = 0;
        std::vector<DiagRec> rest;
        {
            const int ne = static_cast<int>(ph.ext_pos.size());
            const int nch = (ne + 7) / 8;
            std::vector<std::vector<DiagRec>> by_chunk(nch);
            for (const DiagRec &r : ext) {
                const uint64_t d = rec_deps(r);
                int chunk = -1;
                bool ok = d != 0;
                for (int b = 0; b < 64 && ok; ++b) {
                    if (!((d >> b) & 1)) continue;
                    const auto it = std::find(ph.ext_pos.begin(), ph.ext_pos.end(), b);
                    if (it == ph.ext_pos.end()) ok = false; // a rank bit
                    else {
                        const int c = static_cast<int>(it - ph.ext_pos.begin()) / 8;
                        if (chunk >= 0 && c != chunk) ok = false;
                        chunk = c;
                    }
                }
                if (ok) by_chunk[chunk].push_back(r);
                else rest.push_back(r);
            }
            bool any = false;
            for (auto &v : by_chunk) any = any || !v.empty();
            if (any) {
                t.ext_tab = static_cast<int>(ph.tables.size());
                t.ext_chunks = nch;
                for (int c = 0; c < nch; ++c)
                    for (int j = 0; j < 256; ++j) {
                        uint64_t pb = 0;
                        for (int i = 0; i < 8 && 8 * c + i < ne; ++i)
                            if ((j >> i) & 1) pb |= 1ull << ph.ext_pos[8 * c + i];
                        cplx f(1, 0);
                        for (const DiagRec &r : by_chunk[c]) f *= eval_rec(r, pb);
                        ph.tables.push_back(f);
                    }
            }
        }
        // records evaluated per tile: [ext_rest, ext_end) (all of them without tables)
        t.ext_begin = t.ext_rest = static_cast<int>(ph.recs.size());
        if (t.ext_tab >= 0) ph.recs.insert(ph.recs.end(), rest.begin(), rest.end());
        else ph.recs.insert(ph.recs.end(), ext.begin(), ext.end());
        t.ext_end = static_cast<int>(ph.recs.size());
        if (!ext.empty()) t.eidx = n_ext++;
        t.mix_begin = static_cast<int>(ph.recs.size());
        ph.recs.insert(ph.recs.end(), mix.begin(), mix.end());
        t.mix_end = static_cast<int>(ph.recs.size());
        // tile records split by the set-index bits they read: low bits only,
        // high bits only (two small separable tables), or both (full table)
        const int nbits = static_cast<int>(ng_phys.size());
        const int lo_bits = std::min(5, nbits);
        uint64_t lomask = 0;
        for (int i = 0; i < lo_bits; ++i) lomask |= 1ull << ng_phys[i];
        std::vector<DiagRec> lo, hi, full;
        for (const DiagRec &r : tile) {
            const uint64_t d = rec_deps(r);
            if ((d & ~lomask) == 0) lo.push_back(r);
            else if ((d & lomask) == 0) hi.push_back(r);
            else full.push_back(r);
        }
        auto make_table = [&](const std::vector<DiagRec> &rs, int first_bit, int bits) {
            const int off = static_cast<int>(ph.tables.size());
            for (int s = 0; s < (1 << bits); ++s) {
                uint64_t pb = 0;
                for (int i = 0; i < bits; ++i)
                    if ((s >> i) & 1) pb |= 1ull << ng_phys[first_bit + i];
                cplx f(1, 0);
                for (const DiagRec &r : rs) f *= eval_rec(r, pb);
                ph.tables.push_back(f);
            }
            return off;
        };
        t.table_lo = t.table_hi = -1;
        t.lo_bits = lo_bits;
        if (!full.empty()) t.table = make_table(full, 0, nbits);
        if (!lo.empty()) t.table_lo = make_table(lo, 0, lo_bits);
        if (!hi.empty()) t.table_hi = make_table(hi, lo_bits, nbits - lo_bits);
        ph.targets.push_back(t);
        return 1;
    }

    void flush(unsigned slots, bool with_u, bool with_reg) {
        HostOp op;
        op.code = OP_FLUSH;
        op.flush.tgt_begin = static_cast<int>(ph.targets.size());
        for (int j = 0; j < R; ++j)
            if ((slots >> j) & 1) {
                emit_target(j, pend[j]);
                pend[j].clear();
            }
        if (with_u) {
            emit_target(-1, pend_u);
            pend_u.clear();
        }
        op.flush.tgt_end = static_cast<int>(ph.targets.size());
        if (with_reg && pend_reg_slots) {
            for (int r = 0; r < (1 << R); ++r)
                if (pend_reg[r] != cplx(1, 0)) op.flush.regmask |= 1u << r;
            if (op.flush.regmask) op.regtab = pend_reg;
            std::fill(pend_reg.begin(), pend_reg.end(), cplx(1, 0));
            pend_reg_slots = 0;
        }
        if (op.flush.tgt_end > op.flush.tgt_begin || op.flush.regmask) ph.ops.push_back(std::move(op));
    }

    // Returns true when the diagonal gate was absorbed into pending phases.
    bool try_defer(const GateRec &g) {
        if (!flush_enabled || !g.diag || g.encoded || g.flags || !is_unitary_diag(g)) return false;
        DiagRec base{};
        unsigned rc_slots = 0;
        for (int c : g.ctls) {
            const int s = slot(c);
            if (s >= 0) rc_slots |= 1u << s;
            else {
                base.fmask |= 1ull << phys[c];
                base.fval |= 1ull << phys[c];
            }
        }
        int tslot[2] = {-1, -1};
        unsigned rt_slots = 0;
        int nfixed_t = 0;
        for (int t = 0; t < g.k; ++t) {
            tslot[t] = slot(g.wires[t]);
            if (tslot[t] >= 0) rt_slots |= 1u << tslot[t];
            else ++nfixed_t;
        }
        const int d = 1 << g.k;
        cplx dv[4];
        for (int i = 0; i < d; ++i) dv[i] = g.m[i * d + i];
        const unsigned reg = rc_slots | rt_slots;
        const int nreg = std::popcount(reg);
        // register-only phase -> register table
        if (nreg >= 1 && base.fmask == 0 && nfixed_t == 0) {
            for (int r = 0; r < (1 << R); ++r) {
                if ((r & rc_slots) != rc_slots) continue;
                int idx = 0;
                for (int t = 0; t < g.k; ++t) idx = (idx << 1) | ((r >> tslot[t]) & 1);
                pend_reg[r] *= dv[idx];
            }
            pend_reg_slots |= reg;
            return true;
        }
        if (nreg == 0) {
            DiagRec r = base;
            r.nt = g.k;
            r.tpos0 = phys[g.wires[0]];
            if (g.k == 2) r.tpos1 = phys[g.wires[1]];
            for (int i = 0; i < d; ++i) setv(r, i, dv[i]);
            pend_u.push_back(r);
            return true;
        }
        if (nreg == 1 && rt_slots == 0) { // one register control, targets fixed
            const int j = std::countr_zero(rc_slots);
            DiagRec r = base;
            r.nt = g.k;
            r.tpos0 = phys[g.wires[0]];
            if (g.k == 2) r.tpos1 = phys[g.wires[1]];
            for (int i = 0; i < d; ++i) setv(r, i, dv[i]);
            pend[j].push_back(r);
            return true;
        }
        if (nreg == 1 && rc_slots == 0) { // one register target
            const int j = std::countr_zero(rt_slots);
            const int rtpos = tslot[0] == j ? 0 : 1;
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
            pend[j].push_back(f);
            return true;
        }
        return false;
    }

    // An X on a register slot whose controls are register slots (or none) only
    // relabels registers: the pending register table is permuted through it
    // instead of flushed, so one layer's closing phases and the next layer's
    // opening phases meet in one flush (brickwork CNOT layers).
    bool try_permute(const GateRec &g) {
        if (!flush_enabled || !x_through || g.diag || g.encoded || g.flags || g.k != 1) return false;
        if (!(g.m[0] == cplx(0, 0) && g.m[3] == cplx(0, 0) && g.m[1] == cplx(1, 0) && g.m[2] == cplx(1, 0)))
            return false;
        const int t = slot(g.wires[0]);
        if (t < 0) return false;
        unsigned rc = 0;
        for (int c : g.ctls) {
            const int s = slot(c);
            if (s < 0) return false;
            rc |= 1u << s;
        }
        if (!pend[t].empty()) flush(1u << t, false, false);
        if (pend_reg_slots) {
            for (int r = 0; r < (1 << R); ++r)
                if (!((r >> t) & 1) && (r & rc) == rc) std::swap(pend_reg[r], pend_reg[r | (1 << t)]);
            pend_reg_slots |= (1u << t) | rc;
        }
        lower(g);
        return true;
    }

    void add(int gi) {
        const GateRec &g = gates[gi];
        if (try_defer(g)) return;
        if (try_permute(g)) return;
        if (!g.diag) { // flush pending phases on the slots it acts on non-diagonally
            unsigned need = 0;
            for (int t = 0; t < g.k; ++t) {
                const int s = slot(g.wires[t]);
                if (s >= 0) need |= 1u << s;
            }
            unsigned slots = 0;
            for (int j = 0; j < R; ++j)
                if (((need >> j) & 1) && !pend[j].empty()) slots |= 1u << j;
            const bool reg = (pend_reg_slots & need) != 0;
            if (slots || reg) flush(slots, false, reg);
        }
        lower(g);
    }

    void finish() { flush((1u << R) - 1, true, true); }

    void lower(const GateRec &g) {
        HostOp op;
        if (g.flags & OPF_ZERO_OFF_CONTROL) op.flags |= OPF_ZERO_OFF_CONTROL;
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
        if (op.rmask) op.flags |= OPF_RCOND;
        if (op.fmask) op.flags |= OPF_FCOND;
        if (g.encoded) {
            op.flags |= OPF_ENC;
            EncDesc e{};
            e.kind = g.kind;
            e.slot = g.enc_slot;
            e.nparams = g.nparams;
            e.diag = g.diag ? 1 : 0;
            op.enc = static_cast<int>(encs.size());
            encs.push_back(e);
        }
        const int d = 1 << g.k;
        if (g.diag) {
            op.code = OP_DIAG;
            op.nt = static_cast<uint8_t>(g.k);
            uint8_t *tt[2] = {&op.t0, &op.t1};
            for (int t = 0; t < g.k; ++t) {
                const int s = slot(g.wires[t]);
                *tt[t] = static_cast<uint8_t>(s >= 0 ? s : phys[g.wires[t]]);
                if (s >= 0) op.treg |= 1 << t;
            }
            if (!g.encoded)
                for (int i = 0; i < d; ++i) op.pay.push_back(g.m[i * d + i]);
        } else if (g.k == 1) {
            op.a = static_cast<uint8_t>(slot(g.wires[0]));
            op.code = OP_DENSE1;
            if (!g.encoded) {
                op.pay.assign(g.m, g.m + 4);
                const bool real = g.m[0].imag() == 0 && g.m[1].imag() == 0 && g.m[2].imag() == 0 &&
                                  g.m[3].imag() == 0;
                if (real) op.code = OP_DENSE1R;
                // Tangent form: a real uncontrolled matrix is divided by its
                // largest |entry| c, which is deferred to one scale per pass
                // (scalars commute with every gate). Each row then holds a +-1,
                // so an output costs one FMA per component instead of a
                // multiply and an FMA: an orthogonal R = [[a, b], [b, -a]]
                // becomes a * [[1, t], [t, -1]], t = b / a (or its mirror with
                // 1 / t when |b| > |a|), and h becomes the +-1 butterfly.
                // |t| <= 1, so a pass's deferred scale stays >= 2^-(gates / 2).
                // QSV_X_NOTAN=1 keeps the h-only rule (all |entries| equal).
                double c = 0.0;
                for (int i = 0; i < 4; ++i) c = std::max(c, std::abs(g.m[i].real()));
                const char *notan_env = std::getenv("QSV_X_NOTAN");
                const bool notan = notan_env && notan_env[0] == '1';
                bool all_eq = true;
                for (int i = 1; i < 4; ++i) all_eq = all_eq && std::abs(g.m[i].real()) == std::abs(g.m[0].real());
                if (real && c != 0.0 && c != 1.0 && !(op.flags & OPF_ZERO_OFF_CONTROL) && op.rmask == 0 &&
                    op.fmask == 0 && (all_eq || !notan)) {
                    for (auto &x : op.pay) x /= c;
                    ph.scale *= c;
                }
                if (g.m[0] == cplx(0, 0) && g.m[3] == cplx(0, 0) && g.m[1] == cplx(1, 0) && g.m[2] == cplx(1, 0) &&
                    !(op.flags & OPF_ZERO_OFF_CONTROL)) {
                    op.code = OP_X1;
                    op.pay.clear();
                }
            }
        } else {
            op.code = OP_DENSE2;
            const int s0 = slot(g.wires[0]), s1 = slot(g.wires[1]);
            const bool swapq = s0 < s1;
            op.a = static_cast<uint8_t>(swapq ? s1 : s0);
            op.b = static_cast<uint8_t>(swapq ? s0 : s1);
            if (g.encoded) encs.back().swapq = swapq ? 1 : 0;
            else {
                op.pay.resize(16);
                for (int r = 0; r < 4; ++r)
                    for (int c = 0; c < 4; ++c) {
                        const int rr = swapq ? ((r & 1) << 1) | (r >> 1) : r;
                        const int cc = swapq ? ((c & 1) << 1) | (c >> 1) : c;
                        op.pay[r * 4 + c] = g.m[rr * 4 + cc];
                    }
            }
        }
        ph.ops.push_back(std::move(op));
    }
};

PassHost lower_pass(const std::vector<GateRec> &gates, const std::vector<PG> &pg, const std::vector<int> &took,
                    uint64_t active, const std::vector<int> &phys, const PlanConfig &cfg, int K, int L, int R,
                    std::vector<EncDesc> &encs, const std::vector<int> *out_perm = nullptr,
                    uint64_t ext_first = 0) {
    const int nl = cfg.nlocal;
    K = std::max(K, std::popcount(active));  // passenger bits (QSV_PASSENGERS) widen the tile
    PassHost ph;
    ph.K = K;
    ph.L = L;
    ph.R = R;
    if (out_perm) {
        // permuted pass: the tile is read in runs of 2^(lowest contiguous input
        // bits) amplitudes and written in runs of 2^(lowest contiguous output
        // bits); pad by lengthening the shorter run
        std::vector<int> src(nl, -1);
        for (int b = 0; b < nl; ++b) src[(*out_perm)[b]] = b;
        while (std::popcount(active) < K) {
            int in_run = 0, out_run = 0;
            while (in_run < nl && (active >> in_run & 1)) ++in_run;
            while (out_run < nl && (active >> src[out_run] & 1)) ++out_run;
            int b = -1;
            if (out_run < in_run && out_run < nl) b = src[out_run];
            else if (in_run < nl) b = in_run;
            else if (out_run < nl) b = src[out_run];
            if (b < 0) break;
            active |= 1ull << b;
        }
    }
    for (int b = 0; b < nl && std::popcount(active) < K; ++b) active |= 1ull << b; // lengthen contiguous runs
    for (int b = 0; b < nl; ++b)
        if (active & (1ull << b)) ph.tile_pos.push_back(b);
    // tile index bits: the ext bits in ext_first (an L2 super-pass chunk)
    // are the low ones, so a chunk's tiles are one contiguous index range
    for (int pass = 0; pass < 2; ++pass)
        for (int b = 0; b < nl; ++b)
            if (!(active & (1ull << b)) && (((ext_first >> b) & 1) != 0) == (pass == 0)) ph.ext_pos.push_back(b);
    require(static_cast<int>(ph.tile_pos.size()) == K, "planner: tile size");
    int tile_of_phys[64];
    for (int &x : tile_of_phys) x = -1;
    for (int i = 0; i < K; ++i) tile_of_phys[ph.tile_pos[i]] = i;
    std::vector<int> gorder = took;
    ph.ngates = static_cast<int>(gorder.size());
    if (gorder.empty()) { // permutation-only pass: one empty group moves the data
        HostGroup hg;
        int j = 0;
        for (int t = K - 1; t >= K - R; --t) hg.slot_bit[j++] = t;
        for (int t = 0; t < K - R; ++t) hg.ng_bit[t] = t;
        ph.groups.push_back(hg);
    }
    // groups: admission first (all of them), then the lowering
    std::vector<std::vector<int>> gtooks;
    std::vector<std::vector<int>> gslots;  // slot tile bits per group
    while (!gorder.empty()) {
        uint64_t gact = 0;
        std::vector<int> gtook = admit(gorder, pg, gact, R, active);
        require(!gtook.empty(), "planner: no group progress");
        // slots: claimed tile bits, padded with the HIGHEST free tile bits so
        // the lanes of a warp walk the low (contiguous) tile bits.
        std::vector<int> slot_tile;
        for (int b = 0; b < nl; ++b)
            if (gact & (1ull << b)) slot_tile.push_back(tile_of_phys[b]);
        for (int t = K - 1; t >= 0 && static_cast<int>(slot_tile.size()) < R; --t)
            if (std::find(slot_tile.begin(), slot_tile.end(), t) == slot_tile.end()) slot_tile.push_back(t);
        gtooks.push_back(std::move(gtook));
        gslots.push_back(std::move(slot_tile));
    }
    for (size_t gix = 0; gix < gtooks.size(); ++gix) {
        std::vector<int> &gtook = gtooks[gix];
        const std::vector<int> &slot_tile = gslots[gix];
        HostGroup hg;
        int slot_of_phys[64];
        for (int &x : slot_of_phys) x = -1;
        for (int j = 0; j < R; ++j) {
            hg.slot_bit[j] = slot_tile[j];
            slot_of_phys[ph.tile_pos[slot_tile[j]]] = j;
        }
        int q = 0;
        for (int t = 0; t < K; ++t)
            if (std::find(slot_tile.begin(), slot_tile.end(), t) == slot_tile.end()) hg.ng_bit[q++] = t;
        GroupLowering low(ph, gates, phys, slot_of_phys, R, encs, cfg.phase_flush);
        for (int i = 0; i < K - R; ++i) low.ng_phys.push_back(ph.tile_pos[hg.ng_bit[i]]);
        hg.op_begin = static_cast<int>(ph.ops.size());
        hg.tgt_begin = static_cast<int>(ph.targets.size());
        if (cfg.phase_flush && hoist_diagonals()) {
            // deferred diagonals move to the front of the group as far as they
            // commute, so phases that are flushed anyway share one flush (an
            // Euler-split layer's opening phases diag(1, r) of all R slots
            // land before the layer's first rotation: one register-table
            // flush instead of one per slot)
            std::vector<int> ord;
            for (int gi : gtook) {
                size_t pos = ord.size();
                const GateRec &g = gates[gi];
                if (g.diag && !g.encoded && !g.flags && is_unitary_diag(g))
                    while (pos > 0 && !conflicts(pg[gi], pg[ord[pos - 1]].nmask, pg[ord[pos - 1]].dmask)) --pos;
                ord.insert(ord.begin() + static_cast<std::ptrdiff_t>(pos), gi);
            }
            gtook.swap(ord);
        }
        for (int gi : gtook) {
            GateRec e = gates[gi];
            for (int t = 0; t < e.k; ++t) e.wires[t] = phys[e.wires[t]];
            for (int &c : e.ctls) c = phys[c];
            ph.exec_gates.push_back(std::move(e));
            low.add(gi);
        }
        low.finish();
        hg.op_end = static_cast<int>(ph.ops.size());
        hg.tgt_end = static_cast<int>(ph.targets.size());
        ph.groups.push_back(hg);
    }
    if (ph.scale != 1.0) {
        // the deferred butterfly normalisation: one real scale on every
        // amplitude, folded into the last group's closing register table
        HostGroup &last = ph.groups.back();
        HostOp *fl = nullptr;
        if (last.op_end > last.op_begin && ph.ops[last.op_end - 1].code == OP_FLUSH) fl = &ph.ops[last.op_end - 1];
        if (!fl) {
            HostOp op;
            op.code = OP_FLUSH;
            op.flush.tgt_begin = op.flush.tgt_end = static_cast<int>(ph.targets.size());
            ph.ops.push_back(std::move(op));
            last.op_end = static_cast<int>(ph.ops.size());
            fl = &ph.ops.back();
        }
        if (fl->regtab.empty()) fl->regtab.assign(1u << R, cplx(1, 0));
        for (auto &x : fl->regtab) x *= ph.scale;
        fl->flush.regmask = (1u << (1u << R)) - 1;
        ph.scale = 1.0;
    }
    return ph;
}

size_t pass_program_bytes(const PassHost &ph, int dtype) {
    size_t b = ph.groups.size() * sizeof(GroupDesc) + ph.targets.size() * sizeof(FlushTarget) +
               ph.recs.size() * sizeof(DiagRec);
    for (const HostOp &op : ph.ops) b += op_record_bytes(op, dtype, ph.R);
    return b;
}

} // namespace

size_t op_record_bytes(const HostOp &op, int dtype, int R) {
    const size_t t = dtype == QSV_C64 ? 4 : 8;
    size_t b = sizeof(OpHdr) + ((op.flags & OPF_FCOND) ? 16 : 0);
    const bool enc = (op.flags & OPF_ENC) != 0;
    switch (op.code) {
    case OP_DENSE1: b += enc ? 0 : 8 * t; break;
    case OP_DENSE1R: b += (4 * t + 15) / 16 * 16; break;
    case OP_DENSE2: b += enc ? 0 : 32 * t; break;
    case OP_DIAG: b += enc ? 0 : 8 * t; break;
    case OP_X1: break;
    case OP_FLUSH: b += sizeof(FlushPay) + (op.flush.regmask ? (2 * t << R) : 0); break;
    }
    return (b + 15) / 16 * 16;
}

std::vector<unsigned char> serialize_program(const PassHost &ph, int dtype, int *off_targets, int *off_recs,
                                             int *off_ops) {
    const bool f32 = dtype == QSV_C64;
    std::vector<size_t> op_off(ph.ops.size() + 1, 0);
    for (size_t i = 0; i < ph.ops.size(); ++i) op_off[i + 1] = op_off[i] + op_record_bytes(ph.ops[i], dtype, ph.R);
    const size_t g_bytes = ph.groups.size() * sizeof(GroupDesc);
    const size_t t_bytes = ph.targets.size() * sizeof(FlushTarget);
    const size_t r_bytes = ph.recs.size() * sizeof(DiagRec);
    std::vector<unsigned char> blob(g_bytes + t_bytes + r_bytes + op_off.back(), 0);
    *off_targets = static_cast<int>(g_bytes);
    *off_recs = static_cast<int>(g_bytes + t_bytes);
    *off_ops = static_cast<int>(g_bytes + t_bytes + r_bytes);
    for (size_t i = 0; i < ph.groups.size(); ++i) {
        const HostGroup &hg = ph.groups[i];
        GroupDesc gd{};
        gd.op_begin = static_cast<int>(op_off[hg.op_begin]);
        gd.op_end = static_cast<int>(op_off[hg.op_end]);
        for (int j = 0; j < kMaxSlots; ++j) gd.slot_bit[j] = hg.slot_bit[j];
        for (int j = 0; j < kMaxTileBits; ++j) gd.ng_bit[j] = hg.ng_bit[j];
        gd.tgt_begin = hg.tgt_begin;
        gd.tgt_end = hg.tgt_end;
        std::memcpy(blob.data() + i * sizeof(GroupDesc), &gd, sizeof(gd));
    }
    if (t_bytes) std::memcpy(blob.data() + g_bytes, ph.targets.data(), t_bytes);
    if (r_bytes) std::memcpy(blob.data() + g_bytes + t_bytes, ph.recs.data(), r_bytes);
    auto put = [&](unsigned char *&p, double v) {
        if (f32) {
            const float f = static_cast<float>(v);
            std::memcpy(p, &f, 4);
            p += 4;
        } else {
            std::memcpy(p, &v, 8);
            p += 8;
        }
    };
    for (size_t i = 0; i < ph.ops.size(); ++i) {
        const HostOp &op = ph.ops[i];
        unsigned char *p = blob.data() + *off_ops + op_off[i];
        OpHdr h{};
        h.code = op.code, h.a = op.a, h.b = op.b, h.flags = op.flags, h.rmask = op.rmask, h.rval = op.rval;
        h.nt = op.nt, h.t0 = op.t0, h.t1 = op.t1, h.treg = op.treg;
        h.enc = static_cast<uint16_t>(op.enc < 0 ? 0 : op.enc);
        h.size = static_cast<uint16_t>(op_off[i + 1] - op_off[i]);
        std::memcpy(p, &h, sizeof h);
        p += sizeof h;
        if (op.flags & OPF_FCOND) {
            std::memcpy(p, &op.fmask, 8);
            std::memcpy(p + 8, &op.fval, 8);
            p += 16;
        }
        if (op.code == OP_FLUSH) {
            std::memcpy(p, &op.flush, sizeof(FlushPay));
            p += sizeof(FlushPay);
            if (op.flush.regmask)
                for (const cplx &c : op.regtab) put(p, c.real()), put(p, c.imag());
        } else if (op.code == OP_DENSE1R) {
            for (const cplx &c : op.pay) put(p, c.real());
        } else {
            for (const cplx &c : op.pay) put(p, c.real()), put(p, c.imag());
        }
    }
    return blob;
}

// Euler split of dense complex single-qubit gates: M = g * diag(1, l) * R *
// diag(1, r) with R real and g a global phase. R costs half the FP work of a
// complex 2x2 (4 instead of 8 real multiply-adds per amplitude); the two
// diagonals join the deferred phases (consecutive layers' diagonals merge,
// and commute through CZ / controls), and the plan's global phases become
// one constant folded into a register table. Measured with 3-qubit register
// groups (interleaved A/B at 28q): cfg5 family 11.22 -> 9.81 ms, cfg4 family
// 15.81 -> 15.12 ms. QSV_X_NOSPLIT=1 keeps the dense complex matrices.
std::vector<GateRec> split_dense_1q(const std::vector<GateRec> &gates, cplx &gphase) {
    const char *off = std::getenv("QSV_X_NOSPLIT");
    if (off && off[0] == '1') return gates;
    std::vector<GateRec> out;
    out.reserve(gates.size() * 2);
    for (const GateRec &g : gates) {
        bool cand = g.k == 1 && g.ctls.empty() && !g.encoded && g.flags == 0 && !g.diag;
        if (cand) {
            bool real = true;
            for (int i = 0; i < 4; ++i) real = real && g.m[i].imag() == 0.0;
            cand = !real;
        }
        const cplx a = g.m[0], b = g.m[1], c = g.m[2], d = g.m[3];
        if (cand) cand = std::abs(a) > 1e-12 && std::abs(b) > 1e-12 && std::abs(c) > 1e-12 && std::abs(d) > 1e-12;
        if (!cand) {
            out.push_back(g);
            continue;
        }
        const cplx p0 = a / std::abs(a), p1 = c / std::abs(c);
        const cplx q1 = (b / p0) / std::abs(b);
        const cplx r11 = d / (p1 * q1);
        if (std::abs(r11.imag()) > 1e-12 * std::max(1.0, std::abs(r11))) {
            out.push_back(g);
            continue;
        }
        GateRec dr = g, rr = g, dl = g;
        for (GateRec *x : {&dr, &rr, &dl}) {
            x->kind = GK_CUSTOM;
            x->nparams = 0;
            for (int i = 0; i < 16; ++i) x->m[i] = cplx(0, 0);
        }
        dr.name = "split-r";
        dr.diag = true;
        dr.m[0] = cplx(1, 0), dr.m[3] = q1;
        rr.name = "split-real";
        rr.diag = false;
        rr.m[0] = std::abs(a), rr.m[1] = std::abs(b), rr.m[2] = std::abs(c), rr.m[3] = r11.real();
        dl.name = "split-l";
        dl.diag = true;
        dl.m[0] = cplx(1, 0), dl.m[3] = p1 / p0;
        out.push_back(dr);
        out.push_back(rr);
        out.push_back(dl);
        gphase *= p0;
    }
    return out;
}

// A uniform complex factor on every amplitude of a pass, folded into its
// last group's closing register table (created if absent).
void fold_uniform(PassHost &ph, cplx f) {
    const int R = ph.R;
    HostGroup &last = ph.groups.back();
    HostOp *fl = nullptr;
    if (last.op_end > last.op_begin && ph.ops[last.op_end - 1].code == OP_FLUSH) fl = &ph.ops[last.op_end - 1];
    if (!fl) {
        HostOp op;
        op.code = OP_FLUSH;
        op.flush.tgt_begin = op.flush.tgt_end = static_cast<int>(ph.targets.size());
        require(last.op_end == static_cast<int>(ph.ops.size()), "planner: cannot append a flush");
        ph.ops.push_back(std::move(op));
        last.op_end = static_cast<int>(ph.ops.size());
        fl = &ph.ops.back();
    }
    if (fl->regtab.empty()) fl->regtab.assign(1u << R, cplx(1, 0));
    for (auto &x : fl->regtab) x *= f;
    fl->flush.regmask = (1u << (1u << R)) - 1;
    // the schedule export (qsv_plan_dry) lists it as a uniform diagonal gate
    GateRec e;
    e.name = "global-phase";
    e.kind = GK_CUSTOM;
    e.k = 1;
    e.wires[0] = 0;
    e.diag = true;
    e.m[0] = e.m[3] = f;
    ph.exec_gates.push_back(e);
}

std::vector<PassHost> plan_passes(const std::vector<GateRec> &gates_in, const std::vector<int> &phys,
                                  const PlanConfig &cfg, std::vector<EncDesc> &encs,
                                  const std::vector<int> &out_perm, uint64_t last_need) {
    std::vector<int> last_took;
    uint64_t last_active = 0;
    const int nl = cfg.nlocal;
    const int K = std::min(cfg.K, nl);
    const int L = std::min(cfg.L, K);
    int R = cfg.R > 0 ? std::min(cfg.R, K) : std::min(3, K); // cfg.R <= 0: chosen per pass below
    require(K >= 1, "planner: empty local state");
    const uint64_t localmask = nl >= 64 ? ~0ull : ((1ull << nl) - 1);
    std::vector<GateRec> fused = cfg.fuse_1q ? fuse_single_qubit_runs(gates_in) : gates_in;
    cplx gphase(1, 0);
    if (cfg.fuse_1q) fused = split_dense_1q(fused, gphase);
    const std::vector<GateRec> &gates = fused;

    std::vector<PG> pg(gates.size());
    for (size_t i = 0; i < gates.size(); ++i) {
        const GateRec &g = gates[i];
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

    std::vector<PassHost> passes;
    struct Lowering {
        std::vector<int> took;
        uint64_t active;
        bool permuted;
    };
    std::vector<Lowering> how; // per pass: what lower_pass was given (re-lowered for super-passes)
    std::vector<int> order(gates.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
    const uint64_t lowmask = (1ull << L) - 1;
    // Longer contiguous runs where they are free: the first pass starts from
    // the L + 1 lowest bits instead of L (256-byte instead of 128-byte
    // complex128 runs: +9 % DRAM throughput at 64 MiB strides,
    // scripts/micro/runs.cu) when that admits fewer gates to it but does not
    // add a pass overall (admission-only pass counts). The first pass of the
    // 30q QFT strides 64 MiB between runs: measured (interleaved A/B, 30
    // reps) 25.4 -> 23.9 ms median for the 4 passes. Extending later passes
    // too (QSV_RUN_EXTEND = number of leading passes tried) pushes gates into
    // the permuting last pass, whose write runs then shrink: 24.7 ms.
    std::vector<int> extra;
    auto lowmask_of = [&](size_t pi) {
        const int l = std::min(K, L + (pi < extra.size() ? extra[pi] : 0));
        return l >= 64 ? ~0ull : (1ull << l) - 1;
    };
    std::vector<int> out_need_bits;
    uint64_t out_need = 0;
    {
        bool ident = true;
        for (size_t b = 0; b < out_perm.size(); ++b) ident = ident && out_perm[b] == static_cast<int>(b);
        if (!ident)
            for (int b = 0; b < nl; ++b)
                if (out_perm[b] < L) out_need |= 1ull << b;
    }
    auto count_passes = [&]() {
        std::vector<int> ord = order;
        int np = 0;
        uint64_t act = 0;
        while (!ord.empty()) {
            act = lowmask_of(static_cast<size_t>(np));
            if (admit(ord, pg, act, K, localmask).empty()) return 1 << 30;
            ++np;
        }
        if (out_need && !cfg.scatter_out && (np == 0 || std::popcount(act | out_need) > K)) ++np;
        return np;
    };
    const char *ext_env = std::getenv("QSV_RUN_EXTEND");
    const int ext_passes = ext_env ? std::atoi(ext_env) : 1;
    if (cfg.fuse && L < K && ext_passes > 0) {
        const int base = count_passes();
        for (int pi = 0; pi < base && pi < ext_passes; ++pi) {
            extra.resize(static_cast<size_t>(pi) + 1, 0);
            extra[pi] = 1;
            if (count_passes() > base) extra[pi] = 0;
        }
    }
    // Tile search: besides the greedy admission (tile bits claimed by the
    // first admissible gates in order), every window of contiguous bits
    // above the coalescing run is tried as the tile and whichever admits the
    // most gates wins. Light-cone-shaped circuits (cfg4's brickwork) then get
    // a trapezoid of neighbouring wires per pass instead of ~one layer of
    // scattered ones (32q cfg4: 32 -> 17 passes). QSV_TILE_SEARCH=0: greedy.
    static const bool tile_search = [] {
        const char *e = std::getenv("QSV_TILE_SEARCH");
        return !(e && e[0] == '0');
    }();
    while (!order.empty()) {
        uint64_t active = lowmask_of(passes.size());
        if (cfg.fuse && tile_search) {
            std::vector<int> ord = order;
            uint64_t act = active;
            size_t best = admit(ord, pg, act, K, localmask).size();
            uint64_t best_pre = 0;
            const int free_bits = K - std::popcount(active);
            for (int s0 = 0; free_bits > 0 && s0 + free_bits <= nl; ++s0) {
                uint64_t win = 0;
                for (int b = s0; b < s0 + free_bits; ++b) win |= 1ull << b;
                if (win & active) continue;
                ord = order;
                act = active | win;
                const size_t got = admit(ord, pg, act, K, localmask).size();
                if (got > best) best = got, best_pre = win;
            }
            active |= best_pre;
        }
        std::vector<int> took;
        if (cfg.fuse) took = admit(order, pg, active, K, localmask);
        else {
            const int i = order.front();
            order.erase(order.begin());
            active |= pg[i].nmask;
            took.push_back(i);
        }
        require(!took.empty(), "planner: no progress");
        size_t first_encs = encs.size();
        if (cfg.R <= 0) {
            // auto: 4-qubit register groups. With the tangent form and
            // per-register scales the c128 passes are FP64-bound and fewer
            // groups (fewer shared-tile round trips, longer runs of deferred
            // phases) win (28q A/B against 3 when a pass held complex or
            // dense 2-qubit matrices: cfg4 family 12.17 -> 11.52 ms). For
            // complex64, 3-qubit groups won while the passes ran 512-thread
            // CTAs; with the 256-thread CTAs of compute-bound c64 passes
            // (codegen.cpp threads_for) 4 wins: cfg5 family 28q 22.8 -> 22.3
            // ms, 30q 95.3 -> 89.3 ms, 32q 413 -> 395 ms, cfg2 unchanged.
            R = std::min(4, K);
        }
        PassHost ph = lower_pass(gates, pg, took, active, phys, cfg, K, L, R, encs);
        // keep the program within the shared-memory budget: give the tail of
        // the admitted gates back (they commute with everything skipped before
        // them, so they stay valid for a later pass)
        while (pass_program_bytes(ph, cfg.dtype) > static_cast<size_t>(kProgramBudget) && took.size() > 1) {
            const size_t keep = std::max<size_t>(1, took.size() * 2 / 3);
            std::vector<int> back(took.begin() + keep, took.end());
            took.resize(keep);
            order.insert(order.end(), back.begin(), back.end());
            std::sort(order.begin(), order.end());
            active = lowmask_of(passes.size());
            for (int i : took) active |= pg[i].nmask;
            encs.resize(first_encs);
            ph = lower_pass(gates, pg, took, active, phys, cfg, K, L, R, encs);
        }
        {
            // Passenger bit: a compute-bound pass (more dense register-group
            // matrices than 3x its tile bits: single-buffered, jit.cpp) also
            // carries the lowest free bit in its tile, untouched by its gates,
            // so one CTA runs two of the planned tiles in lock-step through
            // the same group code. The deep straight-line passes are
            // instruction-cache bound (ncu: no_instruction the top stall);
            // half as many CTAs at different points of the code per SM.
            // Interleaved A/B, cfg4 family: 28q 49.4 -> 47.0 ms, 30q 201.7 ->
            // 188.5 ms; two passenger bits lose (215.5 ms). QSV_PASSENGERS=P
            // overrides (0 = off); the widened tile must stay <= 64 KiB.
            const char *e = std::getenv("QSV_PASSENGERS");
            const int P = e ? std::atoi(e) : 1;
            int dense = 0;
            for (const HostOp &op : ph.ops)
                if (op.code == OP_DENSE1 || op.code == OP_DENSE1R || op.code == OP_DENSE2) ++dense;
            const size_t amp = cfg.dtype == QSV_C64 ? 8 : 16;
            if (P > 0 && dense > 3 * K && std::popcount(active) + P <= nl &&
                (amp << (std::popcount(active) + P)) <= (64u << 10)) {
                uint64_t a2 = active;
                for (int b = 0, got = 0; b < nl && got < P; ++b)
                    if (!((a2 >> b) & 1)) a2 |= 1ull << b, ++got;
                encs.resize(first_encs);
                ph = lower_pass(gates, pg, took, a2, phys, cfg, K, L, R, encs);
                active = a2;
            }
        }
        passes.push_back(std::move(ph));
        how.push_back({took, active, false});
        last_took = took;
        last_active = active;
    }
    // Final layout permutation: folded into the last pass when its tile can
    // also hold the input bits that land on the L lowest output bits
    // (coalesced permuted writes), else one extra permutation-only pass.
    bool ident = true;
    for (size_t b = 0; b < out_perm.size(); ++b) ident = ident && out_perm[b] == static_cast<int>(b);
    if (!ident) {
        uint64_t need = 0;
        for (int b = 0; b < nl; ++b)
            if (out_perm[b] < L) need |= 1ull << b;
        bool done = false;
        if (!passes.empty() && std::popcount(last_active | need) <= K) {
            const size_t first_encs = encs.size();
            (void)first_encs;
            PassHost ph = lower_pass(gates, pg, last_took, last_active | need, phys, cfg, K, L, R, encs, &out_perm);
            // the re-lowered pass re-registered its encoded gates: drop the old ones
            if (pass_program_bytes(ph, cfg.dtype) <= static_cast<size_t>(kProgramBudget)) {
                ph.out_perm = out_perm;
                passes.back() = std::move(ph);
                how.back() = {last_took, last_active | need, true};
                done = true;
            }
        }
        if (!done && cfg.scatter_out && !passes.empty() && !last_took.empty()) {
            // scattered permuted stores: the last pass keeps its tile; the
            // input bits landing on the output's low bits become its lowest
            // tile-index bits, so neighbouring tiles complete the same output
            // lines while they sit in L2
            PassHost ph = lower_pass(gates, pg, last_took, last_active, phys, cfg, K, L, passes.back().R, encs,
                                     nullptr, need);
            if (pass_program_bytes(ph, cfg.dtype) <= static_cast<size_t>(kProgramBudget)) {
                ph.gperm = out_perm;
                ph.local_gperm = true;
                passes.back() = std::move(ph);
                done = true;
            }
        }
        if (!done) {
            PassHost ph = lower_pass(gates, pg, {}, lowmask | need, phys, cfg, K, L, R, encs, &out_perm);
            ph.out_perm = out_perm;
            passes.push_back(std::move(ph));
            how.push_back({{}, lowmask | need, true});
        }
    }
    // Bits the caller wants in the last pass's tile (the coalescing run of a
    // permutation fused into it later, plan.cpp fuse_swaps_into_passes):
    // added when they fit and the pass has no output permutation of its own.
    if (last_need && !passes.empty() && passes.back().out_perm.empty() && how.back().took.size() &&
        std::popcount(how.back().active | last_need) <= K) {
        const uint64_t act = how.back().active | last_need;
        PassHost ph = lower_pass(gates, pg, how.back().took, act, phys, cfg, K, L, passes.back().R, encs);
        if (pass_program_bytes(ph, cfg.dtype) <= static_cast<size_t>(kProgramBudget)) {
            passes.back() = std::move(ph);
            how.back().active = act;
        }
    }
    // L2 super-passes: pair consecutive passes whose two tiles span at most
    // cfg.super_bits bits. The pair runs as one launch over chunks (the
    // 2^chunk_bits amplitudes of fixed values of every other bit): the first
    // pass's tiles of a chunk, then -- a few chunks later, while they are
    // still in L2 -- the second pass's tiles of it, so the state crosses HBM
    // once for both passes (codegen.cpp generate_pair_source).
    bool any_enc = false;
    for (const GateRec &g : gates) any_enc = any_enc || g.encoded;
    if (cfg.super_bits > 0 && !any_enc) {
        for (size_t i = 0; i + 1 < passes.size();) {
            const PassHost &A = passes[i], &B = passes[i + 1];
            uint64_t cm = 0;
            for (int b : A.tile_pos) cm |= 1ull << b;
            for (int b : B.tile_pos) cm |= 1ull << b;
            const int cb = std::popcount(cm);
            const bool ok = A.K == B.K && A.R == B.R && !A.synth && !B.synth && A.out_perm.empty() &&
                            !A.local_gperm && !B.local_gperm &&
                            pass_prefetches(A, cfg.dtype) == pass_prefetches(B, cfg.dtype) &&
                            kernel_threads(A, cfg.dtype) == kernel_threads(B, cfg.dtype) &&
                            cb <= cfg.super_bits && cb >= A.K + 2 && cb < nl;
            if (!ok) {
                ++i;
                continue;
            }
            for (int j = 0; j < 2; ++j) {
                const Lowering &h = how[i + j];
                const int Rj = passes[i + j].R;
                PassHost ph = lower_pass(gates, pg, h.took, h.active, phys, cfg, K, L, Rj, encs,
                                         h.permuted ? &out_perm : nullptr, cm);
                if (h.permuted) ph.out_perm = out_perm;
                ph.pair = j + 1;
                ph.chunk_bits = cb;
                passes[i + j] = std::move(ph);
            }
            i += 2;
        }
    }
    if (gphase != cplx(1, 0)) {
        require(!passes.empty(), "planner: global phase without a pass");
        fold_uniform(passes.back(), gphase);
    }
    return passes;
}

std::vector<GateRec> relabel_swaps(const std::vector<GateRec> &gates, const std::vector<int> &phys_in,
                                   std::vector<int> &final_phys) {
    std::vector<int> phys = phys_in;
    std::vector<GateRec> out;
    out.reserve(gates.size());
    for (const GateRec &g : gates) {
        if (g.kind == GK_SWAP && g.k == 2 && g.ctls.empty() && !g.encoded && g.flags == 0) {
            std::swap(phys[g.wires[0]], phys[g.wires[1]]);
            continue;
        }
        GateRec p = g;
        for (int t = 0; t < g.k; ++t) p.wires[t] = phys[g.wires[t]];
        for (int &c : p.ctls) c = phys[c];
        out.push_back(std::move(p));
    }
    final_phys = phys;
    return out;
}

} // namespace qsv
