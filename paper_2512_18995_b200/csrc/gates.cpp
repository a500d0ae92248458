// Gate matrices with the reference's semantics and the host-side resolution
// of a qsv_gate into the engine's GateRec.
//
// gate_matrix restates quasar::qubit::gate_matrix
// (/root/reference/proj/include/quasar/qubit/gate.hpp:89-154):
//   rot(G, t) = cos(t/2) I - i sin(t/2) G  (gate.hpp:63-68)
//   u3(t,f,l) = [[c, -e^{il} s], [e^{if} s, e^{i(f+l)} c]]  (gate.hpp:70-76)
//   two-qubit matrices index wires[0] as the MSB (kron, gate.hpp:78-84).
#include <cmath>
#include <cstring>

#include "qsv_internal.hpp"

namespace qsv {

namespace {
constexpr double kPi = 3.141592653589793238462643383279502884;

void rot(const cplx *G, int d, double theta, cplx *out) {
    const double c = std::cos(theta / 2), s = std::sin(theta / 2);
    for (int r = 0; r < d; ++r)
        for (int k = 0; k < d; ++k) out[r * d + k] = (r == k ? cplx(c, 0) : cplx(0, 0)) - cplx(0, s) * G[r * d + k];
}

void kron2(const cplx *a, const cplx *b, cplx *out) {
    for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
            for (int k = 0; k < 2; ++k)
                for (int l = 0; l < 2; ++l) out[(i * 2 + k) * 4 + (j * 2 + l)] = a[i * 2 + j] * b[k * 2 + l];
}

const cplx PX[4] = {0, 1, 1, 0};
const cplx PY[4] = {0, cplx(0, -1), cplx(0, 1), 0};
const cplx PZ[4] = {1, 0, 0, -1};

int arity(int kind) {
    switch (kind) {
    case GK_SWAP:
    case GK_RXX:
    case GK_RYY:
    case GK_RZZ: return 2;
    case GK_CUSTOM: return -1;
    default: return 1;
    }
}

int nparams_of(int kind) {
    switch (kind) {
    case GK_RX:
    case GK_RY:
    case GK_RZ:
    case GK_P:
    case GK_RXX:
    case GK_RYY:
    case GK_RZZ: return 1;
    case GK_U3: return 3;
    default: return 0;
    }
}
} // namespace

int gate_kind(const std::string &n) {
    static const char *names[] = {"x", "y", "z", "h", "s", "t", "rx", "ry", "rz", "p", "u3", "swap", "rxx", "ryy",
                                  "rzz", "custom"};
    for (int i = 0; i < 16; ++i)
        if (n == names[i]) return i;
    fail(QSV_ERR_INVALID, "unknown gate: " + n); // gate.hpp:153
}

bool kind_is_diagonal(int kind) {
    return kind == GK_Z || kind == GK_S || kind == GK_T || kind == GK_RZ || kind == GK_P || kind == GK_RZZ;
}

int gate_matrix(const qsv_gate &g, cplx *m) {
    const std::string name(g.name, strnlen(g.name, sizeof(g.name)));
    const int kind = gate_kind(name);
    const double *p = g.params;
    const int need = nparams_of(kind);
    if (kind != GK_CUSTOM && need > 0)
        require(g.nparams == need, "gate " + name + ": expected " + std::to_string(need) + " params");
    for (int i = 0; i < 16; ++i) m[i] = 0;
    switch (kind) {
    case GK_X: std::copy(PX, PX + 4, m); return 1;
    case GK_Y: std::copy(PY, PY + 4, m); return 1;
    case GK_Z: std::copy(PZ, PZ + 4, m); return 1;
    case GK_H: {
        const double r = 1.0 / std::sqrt(2.0);
        m[0] = r, m[1] = r, m[2] = r, m[3] = -r;
        return 1;
    }
    case GK_S: m[0] = 1, m[3] = cplx(0, 1); return 1;
    case GK_T: m[0] = 1, m[3] = std::exp(cplx(0, kPi / 4)); return 1;
    case GK_RX: rot(PX, 2, p[0], m); return 1;
    case GK_RY: rot(PY, 2, p[0], m); return 1;
    case GK_RZ: rot(PZ, 2, p[0], m); return 1;
    case GK_P: m[0] = 1, m[3] = std::exp(cplx(0, p[0])); return 1;
    case GK_U3: {
        const double c = std::cos(p[0] / 2), s = std::sin(p[0] / 2);
        m[0] = c;
        m[1] = -std::exp(cplx(0, p[2])) * s;
        m[2] = std::exp(cplx(0, p[1])) * s;
        m[3] = std::exp(cplx(0, p[1] + p[2])) * c;
        return 1;
    }
    case GK_SWAP: m[0] = m[15] = m[6] = m[9] = 1; return 2;
    case GK_RXX:
    case GK_RYY:
    case GK_RZZ: {
        const cplx *P = kind == GK_RXX ? PX : kind == GK_RYY ? PY : PZ;
        cplx G[16];
        kron2(P, P, G);
        rot(G, 4, p[0], m);
        return 2;
    }
    case GK_CUSTOM: {
        require(g.custom != nullptr, "custom gate without matrix");
        require(g.nwires >= 1 && g.nwires <= 2, "custom gate: 1 or 2 target wires supported");
        const int d = 1 << g.nwires;
        for (int i = 0; i < d * d; ++i) m[i] = cplx(g.custom[2 * i], g.custom[2 * i + 1]);
        require(approx_unitary(m, d, 1e-10), "custom gate matrix not unitary");
        return g.nwires;
    }
    }
    fail(QSV_ERR_INVALID, "unknown gate: " + name);
}

bool approx_unitary(const cplx *u, int d, double tol) { // core.hpp:53-57
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) {
            cplx acc = 0;
            for (int k = 0; k < d; ++k) acc += std::conj(u[k * d + i]) * u[k * d + j];
            if (std::abs(acc - cplx(i == j ? 1.0 : 0.0, 0.0)) >= tol) return false;
        }
    return true;
}

GateRec resolve_gate(const qsv_gate &g, int nqubit, int *enc_cursor) {
    GateRec r;
    r.name.assign(g.name, strnlen(g.name, sizeof(g.name)));
    r.kind = gate_kind(r.name);
    require(g.nwires >= 1 && g.nwires <= 2, "gate " + r.name + ": 1 or 2 target wires supported");
    require(g.ncontrols >= 0 && g.ncontrols <= 6, "gate " + r.name + ": at most 6 controls");
    r.k = g.nwires;
    for (int i = 0; i < g.nwires; ++i) {
        require(g.wires[i] >= 0 && g.wires[i] < nqubit, "gate wire out of range"); // circuit.hpp:51
        r.wires[i] = g.wires[i];
    }
    require(r.k == 1 || r.wires[0] != r.wires[1], "gate " + r.name + ": duplicate target wires");
    for (int i = 0; i < g.ncontrols; ++i) {
        const int c = g.controls[i];
        require(c >= 0 && c < nqubit, "control wire out of range"); // circuit.hpp:52
        for (int j = 0; j < r.k; ++j)
            require(c != r.wires[j], "gate wires and controls must be disjoint"); // gate.hpp:203-205
        r.ctls.push_back(c);
    }
    const int ar = arity(r.kind);
    // apply_matrix_strided: "gate matrix shape mismatch" (state.hpp:115)
    require(ar < 0 || ar == r.k, "gate matrix shape mismatch");
    r.nparams = g.nparams;
    r.encoded = g.encode != 0 && g.nparams > 0;
    if (r.encoded) {
        require(r.kind != GK_CUSTOM, "custom gates cannot be encoded");
        require(g.nparams == nparams_of(r.kind), "gate " + r.name + ": expected " +
                                                     std::to_string(nparams_of(r.kind)) + " params");
        r.enc_slot = *enc_cursor;
        *enc_cursor += g.nparams;
        r.diag = kind_is_diagonal(r.kind);
        return r;
    }
    const int k = gate_matrix(g, r.m);
    require(k == r.k, "gate matrix shape mismatch");
    require(approx_unitary(r.m, 1 << k, 1e-10), "gate " + r.name + ": matrix not unitary"); // state.hpp:152
    bool diag = true;
    const int d = 1 << k;
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j)
            if (i != j && r.m[i * d + j] != cplx(0, 0)) diag = false;
    r.diag = diag;
    return r;
}

} // namespace qsv
