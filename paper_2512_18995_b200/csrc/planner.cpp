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

std::vector<PassHost> plan_passes(const std::vector<GateRec> &gates, const std::vector<int> &phys,
                                  const PlanConfig &cfg, std::vector<EncDesc> &encs) {
    const int nl = cfg.nlocal;
    const int K = std::min(cfg.K, nl);
    const int L = std::min(cfg.L, K);
    const int R = std::min(cfg.R, K);
    require(K >= 1, "planner: empty local state");
    const uint64_t localmask = nl >= 64 ? ~0ull : ((1ull << nl) - 1);

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
        ph.ngates = static_cast<int>(gorder.size());
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

            for (int gi : took) {
                const GateRec &g = gates[gi];
                TileOp<double> op{};
                op.enc = -1;
                op.flags = g.flags & OPF_ZERO_OFF_CONTROL;
                // controls
                for (int c : g.ctls) {
                    const int b = phys[c];
                    if (b < 64 && slot_of_phys[b] >= 0) {
                        op.rmask |= 1 << slot_of_phys[b];
                        op.rval |= 1 << slot_of_phys[b];
                    } else {
                        op.fmask |= 1ull << b;
                        op.fval |= 1ull << b;
                    }
                }
                const int d = 1 << g.k;
                if (g.diag) {
                    op.type = OP_DIAG;
                    op.nt = g.k;
                    int *tt[2] = {&op.t0, &op.t1};
                    int *tr[2] = {&op.t0reg, &op.t1reg};
                    for (int t = 0; t < g.k; ++t) {
                        const int b = phys[g.wires[t]];
                        if (slot_of_phys[b] >= 0) {
                            *tt[t] = slot_of_phys[b];
                            *tr[t] = 1;
                        } else {
                            *tt[t] = b;
                            *tr[t] = 0;
                        }
                    }
                    if (!g.encoded)
                        for (int i = 0; i < d; ++i) {
                            op.m[2 * i] = g.m[i * d + i].real();
                            op.m[2 * i + 1] = g.m[i * d + i].imag();
                        }
                } else if (g.k == 1) {
                    op.type = OP_DENSE1;
                    op.a = slot_of_phys[phys[g.wires[0]]];
                    if (!g.encoded) set_m(op, g.m, 2);
                } else {
                    op.type = OP_DENSE2;
                    const int s0 = slot_of_phys[phys[g.wires[0]]], s1 = slot_of_phys[phys[g.wires[1]]];
                    const bool swapq = s0 < s1;
                    op.a = swapq ? s1 : s0;
                    op.b = swapq ? s0 : s1;
                    if (!g.encoded) {
                        cplx mm[16];
                        for (int r = 0; r < 4; ++r)
                            for (int c = 0; c < 4; ++c) {
                                // swap the two qubits of the row/column index
                                const int rr = swapq ? ((r & 1) << 1) | (r >> 1) : r;
                                const int cc = swapq ? ((c & 1) << 1) | (c >> 1) : c;
                                mm[r * 4 + c] = g.m[rr * 4 + cc];
                            }
                        set_m(op, mm, 4);
                    }
                    if (g.encoded) op.flags |= swapq ? 2 : 0;
                }
                if (g.encoded) {
                    EncDesc e{};
                    e.kind = g.kind;
                    e.slot = g.enc_slot;
                    e.nparams = g.nparams;
                    e.swapq = (op.type == OP_DENSE2 && (op.flags & 2)) ? 1 : 0;
                    e.diag = g.diag ? 1 : 0;
                    op.enc = static_cast<int>(encs.size());
                    encs.push_back(e);
                }
                op.flags &= ~2; // (bit 1 was scratch for the qubit swap)
                ph.ops.push_back(op);
            }
            gd.op_end = static_cast<int>(ph.ops.size());
            ph.groups.push_back(gd);
        }
        passes.push_back(std::move(ph));
    }
    return passes;
}

} // namespace qsv
