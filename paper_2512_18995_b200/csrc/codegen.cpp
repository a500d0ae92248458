// Pass specialiser: emits the CUDA source of one fused tile pass with the
// pass program compiled in (see jit.cpp for NVRTC + loading).
//
// The generated kernel has the structure of the interpreter in tile_pass.cu
// (persistent CTAs, cp.async tile staging into swizzled shared memory,
// register groups, streaming stores) but every gate is straight-line code:
//   * matrix entries become exact hexfloat immediates; zero and +-1 terms are
//     folded away, so h / x / ry / cz / diag phases cost only what they must;
//   * register-slot conditions (controls inside the group) are resolved at
//     generation time -- only the control-satisfied pairs are emitted;
//   * bit scatters (tile index -> global offset, set index -> tile offset) are
//     runs of constant shift/mask operations;
//   * deferred phases (planner.cpp GroupLowering) keep their split: per-tile
//     EXT factors in shared memory, TILE tables in global memory, MIXED
//     records as inline predicated multiplies, register tables as constants.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <sstream>
#include <string>

#include "qsv_internal.hpp"

namespace qsv {

namespace {

// Matrix / phase entries within 1e-15 of 0 or +-1 become exact (sin/cos of
// multiples of pi/2 leave ~6e-17 residues): the folded term costs no FLOPs and
// the change is far below the 1e-12 (complex128) parity bound.
double snap(double v) {
    if (std::fabs(v) < 1e-15) return 0.0;
    if (std::fabs(v - 1.0) < 1e-15) return 1.0;
    if (std::fabs(v + 1.0) < 1e-15) return -1.0;
    return v;
}

// The shared-tile swizzle (same formula as the generated swz()); it is
// linear over GF(2), so swz(a | b) = swz(a) ^ swz(b) for disjoint a, b.
int swz_host(int u, bool f32) {
    if (f32) {
        const int w = u >> 1;
        const int f = (w >> 3) ^ (w >> 6) ^ (w >> 9) ^ (w >> 12);
        return ((w ^ (f & 7)) << 1) | (u & 1);
    }
    const int f = (u >> 3) ^ (u >> 6) ^ (u >> 9) ^ (u >> 12);
    return u ^ (f & 7);
}

std::string lit(double v, bool f32) {
    char buf[64];
    if (f32) {
        std::snprintf(buf, sizeof buf, "%af", static_cast<double>(static_cast<float>(v)));
    } else {
        std::snprintf(buf, sizeof buf, "%a", v);
    }
    return buf;
}

// Runs of a bit scatter: source bit i -> destination bit pos[i] (ascending).
struct Run {
    int src, len, dst;
};
std::vector<Run> runs_of(const std::vector<int> &pos) {
    std::vector<Run> rs;
    for (size_t i = 0; i < pos.size(); ++i) {
        if (!rs.empty() && rs.back().src + rs.back().len == static_cast<int>(i) &&
            rs.back().dst + rs.back().len == pos[i])
            rs.back().len++;
        else rs.push_back({static_cast<int>(i), 1, pos[i]});
    }
    return rs;
}
// Scatter of selected source bits: (source bit, destination bit) pairs.
std::string scatter_sel(const std::string &x, const std::vector<std::pair<int, int>> &sd) {
    if (sd.empty()) return "0ull";
    std::ostringstream o;
    size_t k = 0;
    bool first = true;
    while (k < sd.size()) {
        size_t e = k + 1;
        while (e < sd.size() && sd[e].first == sd[e - 1].first + 1 && sd[e].second == sd[e - 1].second + 1) ++e;
        const int len = static_cast<int>(e - k);
        if (!first) o << " | ";
        first = false;
        o << "(((((unsigned long long)(" << x << ")) >> " << sd[k].first << ") & " << ((1ull << len) - 1) << "ull) << "
          << sd[k].second << ")";
        k = e;
    }
    return o.str();
}
std::string scatter(const std::string &x, const std::vector<int> &pos, bool wide) {
    auto rs = runs_of(pos);
    if (rs.empty()) return wide ? "0ull" : "0";
    std::ostringstream o;
    for (size_t k = 0; k < rs.size(); ++k) {
        const Run &r = rs[k];
        if (k) o << " | ";
        const std::string mask = wide ? std::to_string((1ull << r.len) - 1) + "ull" : std::to_string((1u << r.len) - 1);
        std::string src = wide ? "((unsigned long long)(" + x + "))" : "(" + x + ")";
        o << "(((" << src << " >> " << r.src << ") & " << mask << ") << " << r.dst << ")";
    }
    return o.str();
}

// One register set per thread per group (up to 512 threads: 2 CTAs x 16 warps
// per SM), at least one 16-byte chunk per thread for the tile copies.
//
// A compute-bound complex64 pass (more dense register-group matrices than
// tile bits) runs 256-thread CTAs instead: several register sets per thread,
// three CTAs per SM (shared memory) instead of two, so one CTA's tile load
// overlaps two others' arithmetic. Interleaved A/B: cfg5 family 30q 99.2 ->
// 95.5 ms, 33q 855 -> 823 ms; cfg2 execute 0.358 -> 0.297 ms; the light
// (memory-bound) passes keep 512 (the cfg5 tail passes lose 5-17 % at 256).
// QSV_MAX_THREADS overrides the cap.
int threads_for(const PassHost &ph, int dtype) {
    const int nsets = 1 << (ph.K - ph.R); // one register set per thread per group, up to the cap
    int cap = 512;
    if (dtype == QSV_C64) {
        int dense = 0;
        for (const HostOp &op : ph.ops)
            if (op.code == OP_DENSE1 || op.code == OP_DENSE1R || op.code == OP_DENSE2) ++dense;
        if (dense > ph.K) cap = 256;
    }
    const char *mt = std::getenv("QSV_MAX_THREADS");
    if (mt && std::atoi(mt) > 0) cap = std::atoi(mt);
    const int th = std::max(32, std::min(cap, nsets));
    return (th + 31) / 32 * 32;
}

// CTAs per SM the register budget is sized for: 2^R amplitudes per thread
// (R = 4 -> up to 128 registers, R <= 3 -> 64).
int kernel_min_blocks(const PassHost &ph, int threads) {
    const int regcap = ph.R >= 4 ? 128 : 64;
    return std::max(1, std::min(8, 65536 / (threads * regcap)));
}

struct Gen {
    const PassHost &ph;
    bool f32;
    bool packed; // complex64 arithmetic on f32x2 pairs (QSV_X_NOPACK=1: scalar FP32)
    // Deferred per-register real scales (QSV_X_NOSCALE=1: off). Register r
    // holds sc[r]^-1 times its amplitude: a constant phase p = d (1 + i t)
    // costs one FMA per component (the real d joins sc[r]), a real matrix
    // absorbs the scales of its inputs and leaves each output row divided by
    // its largest entry (one +-1 term per row). Runtime complex factors
    // commute with the scales; they are multiplied in by the group's last
    // constant multiply or before its stores.
    bool track = true;
    bool untracked = false; // inside a runtime-conditional op
    bool final_op = false;  // emitting the group's last op
    std::vector<double> sc;
    int R;
    std::ostringstream o;
    std::string T, V;

    Gen(const PassHost &p, int dtype) : ph(p), f32(dtype == QSV_C64), R(p.R) {
        T = f32 ? "float" : "double";
        V = f32 ? "cf" : "cd";
        const char *np = std::getenv("QSV_X_NOPACK");
        packed = f32 && !(np && np[0] == '1');
        const char *ns = std::getenv("QSV_X_NOSCALE");
        track = !(ns && ns[0] == '1');
        sc.assign(static_cast<size_t>(1) << R, 1.0);
    }

    // multiplies the pending scales of the registers in `mask` into them
    void materialize(const std::string &ind, uint64_t mask = ~0ull) {
        for (size_t r = 0; r < sc.size(); ++r)
            if (((mask >> r) & 1) && sc[r] != 1.0) {
                o << ind << "v" << r << " = " << rscale("v" + std::to_string(r), sc[r]) << ";\n";
                sc[r] = 1.0;
            }
    }

    // complex128 constants: hexfloat immediates (a DFMA takes no 64-bit
    // immediate, so each distinct value costs two UMOVs in the instruction
    // stream), or with `pool` one __constant__ table per kernel read by
    // LDCU.128 (two values per instruction)
    bool pool = [] {
        const char *e = std::getenv("QSV_X_CPOOL");
        return e && e[0] == '1';
    }();
    mutable std::map<uint64_t, int> pool_idx;
    mutable std::vector<double> pool_vals;
    std::string c(double x) const {
        if (f32 || !pool) return lit(x, f32);
        const double a = std::fabs(x);
        uint64_t bits;
        std::memcpy(&bits, &a, 8);
        auto it = pool_idx.find(bits);
        int i;
        if (it == pool_idx.end()) {
            i = static_cast<int>(pool_vals.size());
            pool_idx.emplace(bits, i);
            pool_vals.push_back(a);
        } else i = it->second;
        return std::string(x < 0 ? "(-KC[" : "(KC[") + std::to_string(i) + "])";
    }
    std::string pool_decl() const {
        if (pool_vals.empty()) return "";
        std::ostringstream d;
        d << "__constant__ double KC[" << pool_vals.size() << "] = {";
        for (size_t i = 0; i < pool_vals.size(); ++i) d << (i ? ", " : "") << lit(pool_vals[i], false);
        d << "};\n";
        return d.str();
    }

    // complex128 tile swizzle: the 16-byte slot of amplitude u is u with its
    // low 3 bits XORed with parities of the high bits (swm[i] = the high bits
    // folded into bit i). Any such map is linear over GF(2). It is chosen per
    // pass so that every 8-thread phase of the pass's shared-memory accesses
    // (each group's set -> slot mapping, the permuted copy-out) hits 8
    // distinct 16-byte bank groups; the default folds bits 3+i, 6+i, 9+i, 12+i.
    //
    // complex64 (8-byte amplitudes): the same construction on 16-byte CHUNKS
    // (amplitude pairs u, u ^ 1 stay together, so the 16-byte cp.async copies
    // and the pair accesses below keep working): chunk w = u >> 1 becomes
    // w ^ f(w). A group whose slots hold tile bit 0 moves each register pair
    // as one 16-byte access (8 threads per shared-memory wavefront: the set's
    // first three bits must reach 8 distinct chunks); otherwise a thread moves
    // 8 bytes (16 threads per wavefront: tile bit 0 is the set's first bit,
    // and its next three bits must reach 8 distinct chunks).
    int swm[3] = {0, 0, 0};
    bool noswz() const { return swm[0] == 0 && swm[1] == 0 && swm[2] == 0; }
    int swz_of(int u) const {
        const int w = f32 ? u >> 1 : u;
        int f = 0;
        for (int i = 0; i < 3; ++i) f |= (__builtin_popcount(w & swm[i]) & 1) << i;
        return f32 ? (((w ^ f) << 1) | (u & 1)) : u ^ f;
    }
    void choose_swizzle(const std::vector<std::vector<int>> &patterns) {
        const int K = f32 ? ph.K - 1 : ph.K;  // bits of the swizzled unit (chunk for complex64)
        auto ok = [&](const int m[3], const std::vector<int> &b) {
            // the three phase-varying tile bits must map to independent low-bit vectors
            int v[3];
            for (int j = 0; j < 3; ++j) {
                if (b[j] < 3) v[j] = 1 << b[j];
                else {
                    v[j] = 0;
                    for (int i = 0; i < 3; ++i) v[j] |= ((m[i] >> b[j]) & 1) << i;
                }
            }
            return v[0] && v[1] && v[2] && v[0] != v[1] && v[0] != v[2] && v[1] != v[2] && (v[0] ^ v[1]) != v[2];
        };
        auto score = [&](const int m[3]) {
            int n = 0;
            for (const auto &b : patterns) n += ok(m, b);
            return n;
        };
        // no swizzle at all when every pattern's phase-varying bits are the 3
        // lowest tile bits (the usual case: they are the contiguous-run bits):
        // then a register slot's offset is a plain immediate on the set's base
        const int zero[3] = {0, 0, 0};
        if (score(zero) == static_cast<int>(patterns.size())) {
            swm[0] = swm[1] = swm[2] = 0;
            return;
        }
        int best[3];
        for (int i = 0; i < 3; ++i) {
            best[i] = 0;
            for (int k = 3 + i; k < K; k += 3) best[i] |= 1 << k;
        }
        int bs = score(best);
        uint64_t x = 0x9e3779b97f4a7c15ull;
        for (int it = 0; it < 4000 && bs < static_cast<int>(patterns.size()); ++it) {
            int m[3];
            for (int i = 0; i < 3; ++i) {
                x ^= x << 13, x ^= x >> 7, x ^= x << 17;
                m[i] = static_cast<int>(x) & (((1 << K) - 1) & ~7);
            }
            const int sc = score(m);
            if (sc > bs) bs = sc, std::copy(m, m + 3, best);
        }
        std::copy(best, best + 3, swm);
    }

    // dst = coefficient * x (complex), with constant folding; returns terms
    // for the real and imaginary parts (appended to re/im lists)
    void term(const cplx &m, const std::string &x, std::vector<std::string> &re, std::vector<std::string> &im) {
        const double a = snap(m.real()), b = snap(m.imag());
        auto mulstr = [&](double k, const std::string &v) -> std::string {
            if (k == 1.0) return "+" + v;
            if (k == -1.0) return "-" + v;
            return "+" + c(k) + "*" + v;
        };
        // (a + ib)(x + iy) = (a x - b y) + i(a y + b x)
        if (a != 0.0) {
            re.push_back(mulstr(a, x + ".x"));
            im.push_back(mulstr(a, x + ".y"));
        }
        if (b != 0.0) {
            re.push_back(mulstr(-b, x + ".y"));
            im.push_back(mulstr(b, x + ".x"));
        }
    }
    static std::string sum(const std::vector<std::string> &ts) {
        if (ts.empty()) return "0";
        std::string s;
        for (size_t i = 0; i < ts.size(); ++i) {
            std::string t = ts[i];
            if (i == 0 && t[0] == '+') t = t.substr(1);
            s += t;
        }
        return s;
    }

    // complex64: sum_k m_k x_k as a chain of packed f32x2 operations (the
    // helpers of common()): a real coefficient is one FMUL2/FFMA2, a complex
    // one two (the i*x half reads x with its halves swapped, which ptxas
    // folds into the operand), +-1 an FADD2.
    std::string packed_sum(const std::vector<std::pair<cplx, std::string>> &ts_in) const {
        // a +1 term starts the chain (acc = x, no instruction), so a real
        // row [c, 1] is one FFMA2 instead of FMUL2 + FADD2 (the scale
        // tracking leaves a +1 in every real row)
        std::vector<std::pair<cplx, std::string>> ts = ts_in;
        std::stable_partition(ts.begin(), ts.end(), [&](const std::pair<cplx, std::string> &t) {
            return snap(t.first.real()) == 1.0 && snap(t.first.imag()) == 0.0;
        });
        std::string acc;
        for (const auto &t : ts) {
            const double a = snap(t.first.real()), b = snap(t.first.imag());
            if (a == 0.0 && b == 0.0) continue;
            const std::string &x = t.second;
            if (acc.empty()) {
                if (b == 0.0) acc = a == 1.0 ? x : a == -1.0 ? "cneg(" + x + ")" : "rmul(" + x + ", " + c(a) + ")";
                else if (a == 0.0) acc = "imul(" + x + ", " + c(b) + ")";
                else acc = "cmc(" + x + ", " + c(a) + ", " + c(b) + ")";
            } else {
                if (b == 0.0)
                    acc = a == 1.0    ? "cadd(" + acc + ", " + x + ")"
                          : a == -1.0 ? "csub(" + acc + ", " + x + ")"
                                      : "rfma(" + acc + ", " + x + ", " + c(a) + ")";
                else if (a == 0.0) acc = "ifma(" + acc + ", " + x + ", " + c(b) + ")";
                else acc = "cfc(" + acc + ", " + x + ", " + c(a) + ", " + c(b) + ")";
            }
        }
        return acc.empty() ? "mk(0, 0)" : acc;
    }

    // v[r] = sum_k M[row][k] * x[k]
    void matvec(const std::vector<int> &regs, const std::vector<cplx> &m_in, int d, const std::string &ind) {
        std::vector<cplx> m = m_in;
        if (track && !untracked) {
            // absorb the input scales, then divide every all-real row by its
            // largest |entry| (the divisor becomes that output's scale)
            for (int r = 0; r < d; ++r)
                for (int k = 0; k < d; ++k) m[r * d + k] *= sc[regs[k]];
            std::vector<double> out(d, 1.0);
            for (int r = 0; r < d; ++r) {
                bool real = true;
                double big = 0.0, sgn = 1.0;
                for (int k = 0; k < d; ++k) {
                    const cplx &e = m[r * d + k];
                    real = real && e.imag() == 0.0;
                    if (std::abs(e.real()) > big) big = std::abs(e.real()), sgn = e.real() < 0 ? -1.0 : 1.0;
                }
                if (real && big != 0.0) {
                    out[r] = big * sgn;
                    for (int k = 0; k < d; ++k) m[r * d + k] /= out[r];
                }
            }
            for (int r = 0; r < d; ++r) sc[regs[r]] = out[r];
        }
        o << ind << "{ ";
        for (int k = 0; k < d; ++k) o << "const " << V << " x" << k << " = v" << regs[k] << "; ";
        o << "\n";
        for (int r = 0; r < d; ++r) {
            if (packed) {
                std::vector<std::pair<cplx, std::string>> ts;
                for (int k = 0; k < d; ++k) ts.emplace_back(m[r * d + k], "x" + std::to_string(k));
                o << ind << "  v" << regs[r] << " = " << packed_sum(ts) << ";\n";
                continue;
            }
            std::vector<std::string> re, im;
            for (int k = 0; k < d; ++k) term(m[r * d + k], "x" + std::to_string(k), re, im);
            o << ind << "  v" << regs[r] << " = mk(" << sum(re) << ", " << sum(im) << ");\n";
        }
        o << ind << "}\n";
    }

    void cmul_const(int r, const cplx &f_in, const std::string &ind) {
        cplx f = f_in;
        if (track && !untracked) {
            f *= sc[r];
            sc[r] = 1.0;
            const double a = f.real(), b = f.imag();
            if (!final_op && !untracked) {
                // f = d (1 + i t) or d (t + i), |t| <= 1; d joins the scale
                if (b == 0.0 || std::abs(a) >= std::abs(b)) {
                    sc[r] = a;
                    f = cplx(1.0, b / a);
                } else {
                    sc[r] = b;
                    f = cplx(a / b, 1.0);
                }
            }
        }
        if (snap(f.real()) == 1.0 && snap(f.imag()) == 0.0) return;
        if (packed && snap(f.real()) == 1.0) {
            o << ind << "v" << r << " = cti(v" << r << ", " << c(f.imag()) << ");\n";
            return;
        }
        if (packed && snap(f.imag()) == 1.0) {
            o << ind << "v" << r << " = cit(v" << r << ", " << c(f.real()) << ");\n";
            return;
        }
        if (packed) {
            o << ind << "v" << r << " = " << packed_sum({{f, "v" + std::to_string(r)}}) << ";\n";
            return;
        }
        std::vector<std::string> re, im;
        term(f, "v" + std::to_string(r), re, im);
        o << ind << "v" << r << " = mk(" << sum(re) << ", " << sum(im) << ");\n";
    }

    // x scaled by a real constant
    std::string rscale(const std::string &x, double k) const {
        if (packed) return "rmul(" + x + ", " + c(k) + ")";
        return "mk(" + c(k) + "*" + x + ".x, " + c(k) + "*" + x + ".y)";
    }

    std::string fcond(uint64_t fmask, uint64_t fval) {
        std::ostringstream s;
        s << "((pb & " << fmask << "ull) == " << fval << "ull)";
        return s.str();
    }

    void emit_rec_factor(const DiagRec &r, const std::string &base, const std::string &f, const std::string &ind) {
        // f = f * (cond(base) ? val[idx(base)] : 1)
        std::string cond = r.fmask ? "((" + base + " & " + std::to_string(r.fmask) + "ull) == " +
                                         std::to_string(r.fval) + "ull)"
                                   : "true";
        o << ind << "if (" << cond << ") {\n";
        const int nv = 1 << r.nt;
        if (nv == 1) {
            o << ind << "  " << f << " = cmulv(" << f << ", mk(" << c(r.val[0]) << ", " << c(r.val[1]) << "));\n";
        } else {
            o << ind << "  const int ix = ";
            if (r.nt == 1) o << "(int)((" << base << " >> " << r.tpos0 << ") & 1ull);\n";
            else
                o << "(int)(((" << base << " >> " << r.tpos0 << ") & 1ull) << 1 | ((" << base << " >> " << r.tpos1
                  << ") & 1ull));\n";
            o << ind << "  " << V << " q;\n";
            for (int i = 0; i < nv; ++i)
                o << ind << "  " << (i ? "else " : "") << "if (ix == " << i << ") q = mk(" << c(r.val[2 * i]) << ", "
                  << c(r.val[2 * i + 1]) << ");\n";
            o << ind << "  " << f << " = cmulv(" << f << ", q);\n";
        }
        o << ind << "}\n";
    }

    void emit_op(const HostOp &op, const std::string &ind) {
        const int NR = 1 << R;
        std::string ind2 = ind;
        const bool fc = (op.flags & OPF_FCOND) != 0;
        const bool zoc = (op.flags & OPF_ZERO_OFF_CONTROL) != 0;
        const bool enc = (op.flags & OPF_ENC) != 0;
        if (op.code == OP_FLUSH) {
            emit_flush(op, ind);
            return;
        }
        // a runtime condition (or a runtime matrix) makes the op's effect on
        // the scales unknown at generation time: it sees materialised registers
        struct Untrack {
            bool &u;
            bool prev;
            ~Untrack() { u = prev; }
        } untrack{untracked, untracked};
        if (track && (fc || enc)) {
            // equal scales commute with any linear map of the registers they
            // share, so only a pair / quad with unequal scales is materialised;
            // per-register (diagonal) factors commute with every scale
            std::vector<int> touched;
            if (op.code == OP_DENSE1 || op.code == OP_DENSE1R || op.code == OP_X1) touched = {0, 1 << op.a};
            else if (op.code == OP_DENSE2) touched = {0, 1 << op.b, 1 << op.a, (1 << op.a) | (1 << op.b)};
            const int span = touched.empty() ? 0 : touched.back();
            for (int r = 0; r < NR && !touched.empty(); ++r) {
                if (r & span) continue;
                uint64_t mask = 0;
                bool same = true;
                for (int t : touched) {
                    mask |= 1ull << (r | t);
                    same = same && sc[r | t] == sc[r];
                }
                if (!same) materialize(ind, mask);
            }
            untracked = true;
        }
        if (fc && !zoc) {
            o << ind << "if " << fcond(op.fmask, op.fval) << " {\n";
            ind2 = ind + "  ";
        }
        std::vector<cplx> m = op.pay;
        if (enc) {
            // matrix / diagonal from the per-row table
            o << ind2 << "{ const " << T << " *em = a.enc_table + ((size_t)" << op.enc
              << " * a.batch + row) * 32;\n";
            const int cnt = op.code == OP_DENSE2 ? 16 : 4;
            o << ind2 << "  " << V << " ";
            for (int i = 0; i < cnt; ++i) o << (i ? ", " : "") << "e" << i << " = mk(em[" << 2 * i << "], em[" << 2 * i + 1 << "])";
            o << ";\n";
        }
        auto pair_on = [&](int r) { return (r & op.rmask) == op.rval; };
        auto zero_regs = [&](const std::vector<int> &regs, const std::string &in) {
            for (int r : regs) o << in << "v" << r << " = mk(0, 0);\n";
        };
        switch (op.code) {
        case OP_DENSE1:
        case OP_DENSE1R:
        case OP_X1: {
            const int J = op.a;
            if (op.code == OP_X1) m = {0, 1, 1, 0};
            for (int r = 0; r < NR; ++r) {
                if (r & (1 << J)) continue;
                const int r1 = r | (1 << J);
                std::vector<int> regs = {r, r1};
                if (!pair_on(r)) {
                    if (zoc) zero_regs(regs, ind2);
                    continue;
                }
                if (zoc && fc) {
                    o << ind2 << "if " << fcond(op.fmask, op.fval) << " {\n";
                    emit_mv(regs, m, 2, enc, ind2 + "  ");
                    o << ind2 << "} else {\n";
                    zero_regs(regs, ind2 + "  ");
                    o << ind2 << "}\n";
                } else emit_mv(regs, m, 2, enc, ind2);
            }
            break;
        }
        case OP_DENSE2: {
            const int A = op.a, B = op.b;
            for (int r = 0; r < NR; ++r) {
                if (r & ((1 << A) | (1 << B))) continue;
                std::vector<int> regs = {r, r | (1 << B), r | (1 << A), r | (1 << A) | (1 << B)};
                if (!pair_on(r)) {
                    if (zoc) zero_regs(regs, ind2);
                    continue;
                }
                if (zoc && fc) {
                    o << ind2 << "if " << fcond(op.fmask, op.fval) << " {\n";
                    emit_mv(regs, m, 4, enc, ind2 + "  ");
                    o << ind2 << "} else {\n";
                    zero_regs(regs, ind2 + "  ");
                    o << ind2 << "}\n";
                } else emit_mv(regs, m, 4, enc, ind2);
            }
            break;
        }
        case OP_DIAG: {
            // value index from target bits: register bits are compile-time,
            // fixed bits are read from pb
            const bool t0r = op.treg & 1, t1r = (op.treg >> 1) & 1;
            for (int r = 0; r < NR; ++r) {
                const bool on = pair_on(r);
                if (!on) {
                    if (zoc) o << ind2 << "v" << r << " = mk(0, 0);\n";
                    continue;
                }
                std::string body;
                auto bitexpr = [&](bool reg, int t) -> std::string {
                    if (reg) return std::to_string((r >> t) & 1);
                    return "(int)((pb >> " + std::to_string(t) + ") & 1ull)";
                };
                const std::string b0 = bitexpr(t0r, op.t0);
                const std::string idx = op.nt == 2 ? "((" + b0 + ") << 1 | (" + bitexpr(t1r, op.t1) + "))" : b0;
                const bool static_idx = (t0r && (op.nt == 1 || t1r));
                std::string in3 = ind2;
                if (zoc && fc) {
                    o << ind2 << "if " << fcond(op.fmask, op.fval) << " {\n";
                    in3 = ind2 + "  ";
                }
                if (static_idx && !enc) {
                    int ix = (r >> op.t0) & 1;
                    if (op.nt == 2) ix = (ix << 1) | ((r >> op.t1) & 1);
                    cmul_const(r, m[ix], in3);
                } else {
                    o << in3 << "{ const int ix = " << idx << "; " << V << " q = ";
                    const int nv = 1 << op.nt;
                    for (int i = 0; i < nv; ++i) {
                        const std::string val = enc ? "e" + std::to_string(i)
                                                    : "mk(" + c(m[i].real()) + ", " + c(m[i].imag()) + ")";
                        if (i + 1 < nv) o << "ix == " << i << " ? " << val << " : ";
                        else o << val;
                    }
                    o << "; v" << r << " = cmulv(v" << r << ", q); }\n";
                }
                if (zoc && fc) {
                    o << ind2 << "} else {\n" << ind2 << "  v" << r << " = mk(0, 0);\n" << ind2 << "}\n";
                }
            }
            break;
        }
        }
        if (enc) o << ind2 << "}\n";
        if (fc && !zoc) o << ind << "}\n";
    }

    void emit_mv(const std::vector<int> &regs, const std::vector<cplx> &m, int d, bool enc, const std::string &ind) {
        if (!enc) {
            matvec(regs, m, d, ind);
            return;
        }
        o << ind << "{ ";
        for (int k = 0; k < d; ++k) o << "const " << V << " x" << k << " = v" << regs[k] << "; ";
        o << "\n";
        for (int r = 0; r < d; ++r) {
            o << ind << "  v" << regs[r] << " = ";
            for (int k = 0; k < d; ++k) {
                if (k == 0) o << "cmulv(e" << r * d << ", x0)";
                else o << ";\n" << ind << "  v" << regs[r] << " = cfmav(e" << r * d + k << ", x" << k << ", v" << regs[r]
                       << ")";
            }
            o << ";\n";
        }
        o << ind << "}\n";
    }

    // A FLUSH multiplies register slot r by the product of the factors of its
    // targets (slot -1: every slot; slot b: slots with bit b set). The
    // factors of one slot class are merged first (g_all, g_b), then the
    // per-slot products are built down a binary tree over the bits
    // (ph[r | 1<<b] = ph[r] * g_b, depth-first so at most R + 1 are live)
    // and applied once per slot: 2^R - 1 + 2^R complex multiplies at most,
    // against 2^(R-1) per single-bit target + 2^R per all-slot target when
    // every target is applied on its own. A uniform real register scale
    // (the deferred 1/sqrt(2)^h of the butterflies) rides on the root.
    // Every value a flush target's factor can take is exactly +-1 (CZ-type
    // phases against bits outside the register group, e.g. cfg5's random-pair
    // CZs): the factor is then a sign and the flush a sign-bit XOR on the
    // integer pipe instead of complex multiplies on the FMA pipe.
    static bool pm1(const cplx &v) { return v.imag() == 0.0 && (v.real() == 1.0 || v.real() == -1.0); }
    bool target_is_sign(const FlushTarget &t) const {
        auto tab_ok = [&](int off, int len) {
            for (int i = 0; i < len; ++i)
                if (!pm1(ph.tables[off + i])) return false;
            return true;
        };
        auto rec_ok = [&](int b, int e) {
            for (int k = b; k < e; ++k) {
                const DiagRec &r = ph.recs[k];
                for (int i = 0; i < (1 << r.nt); ++i)
                    if (!pm1(cplx(r.val[2 * i], r.val[2 * i + 1]))) return false;
            }
            return true;
        };
        const int nb = ph.K - ph.R;
        if (t.ext_tab >= 0 && !tab_ok(t.ext_tab, 256 * t.ext_chunks)) return false;
        if (!rec_ok(t.ext_rest, t.ext_end) || !rec_ok(t.mix_begin, t.mix_end)) return false;
        if (t.table >= 0 && !tab_ok(t.table, 1 << nb)) return false;
        if (t.table_lo >= 0 && !tab_ok(t.table_lo, 1 << t.lo_bits)) return false;
        if (t.table_hi >= 0 && !tab_ok(t.table_hi, 1 << (nb - t.lo_bits))) return false;
        return true;
    }
    std::string sgn(const std::string &x) const { return "(" + std::string(f32 ? "__float_as_uint" : "__double2hiint") + "(" + x + ".x) & 0x80000000u)"; }
    void emit_rec_sign(const DiagRec &r, const std::string &base, const std::string &f, const std::string &ind) {
        std::string cond = r.fmask ? "((" + base + " & " + std::to_string(r.fmask) + "ull) == " +
                                         std::to_string(r.fval) + "ull)"
                                   : "true";
        const int nv = 1 << r.nt;
        unsigned m[4];
        for (int i = 0; i < nv; ++i) m[i] = r.val[2 * i] < 0 ? 0x80000000u : 0u;
        if (nv == 1) {
            if (m[0]) o << ind << "if (" << cond << ") " << f << " ^= 0x80000000u;\n";
            return;
        }
        o << ind << "if (" << cond << ") {\n" << ind << "  const int ix = ";
        if (r.nt == 1) o << "(int)((" << base << " >> " << r.tpos0 << ") & 1ull);\n";
        else
            o << "(int)(((" << base << " >> " << r.tpos0 << ") & 1ull) << 1 | ((" << base << " >> " << r.tpos1
              << ") & 1ull));\n";
        o << ind << "  " << f << " ^= ";
        for (int i = 0; i < nv; ++i) o << (i + 1 < nv ? "ix == " + std::to_string(i) + " ? " : "") << m[i] << "u" << (i + 1 < nv ? " : " : "");
        o << ";\n" << ind << "}\n";
    }
    bool emit_flush_sign(const HostOp &op, const std::string &ind) {
        const bool off = [] {  // QSV_X_NOSIGN=1 (A/B): complex multiplies
            const char *e = std::getenv("QSV_X_NOSIGN");
            return e && e[0] == '1';
        }();
        if (off || op.flush.tgt_end <= op.flush.tgt_begin) return false;
        for (int ti = op.flush.tgt_begin; ti < op.flush.tgt_end; ++ti)
            if (!target_is_sign(ph.targets[ti])) return false;
        const int NR = 1 << R;
        bool uniform = op.flush.regmask == (NR >= 32 ? 0xffffffffu : ((1u << NR) - 1)) &&
                       static_cast<int>(op.regtab.size()) >= NR && op.regtab[0].imag() == 0.0;
        for (int r = 1; uniform && r < NR; ++r) uniform = op.regtab[r] == op.regtab[0];
        const double rc = uniform ? op.regtab[0].real() : 1.0;
        if (rc != 1.0 && !track) return false;  // a runtime scale would need a multiply anyway
        if (rc != 1.0) {
            for (double &x : sc) x *= rc;
            if (final_op) materialize(ind);
        }
        o << ind << "{\n";
        const std::string in = ind + "  ";
        std::vector<int> nfac(R + 1, 0);
        for (int ti = op.flush.tgt_begin; ti < op.flush.tgt_end; ++ti) {
            const FlushTarget &t = ph.targets[ti];
            const int cls = t.slot < 0 ? R : t.slot;
            const std::string g = "m" + std::to_string(cls);
            const std::string f = "n" + std::to_string(ti);
            std::vector<std::string> terms;
            if (t.eidx >= 0) terms.push_back(sgn("E[" + eoff() + std::to_string(ebase[cur_group] + t.eidx) + "]"));
            if (t.table >= 0) terms.push_back(sgn("tab" + std::to_string(ti)));
            if (t.table_lo >= 0)
                terms.push_back(sgn("stab[" + std::to_string(stab_off.at(t.table_lo)) + " + (s & " +
                                    std::to_string((1 << t.lo_bits) - 1) + ")]"));
            if (t.table_hi >= 0)
                terms.push_back(sgn("stab[" + std::to_string(stab_off.at(t.table_hi)) + " + (s >> " +
                                    std::to_string(t.lo_bits) + ")]"));
            o << in << "unsigned " << f << " = " << (terms.empty() ? std::string("0u") : terms[0]);
            for (size_t k = 1; k < terms.size(); ++k) o << " ^ " << terms[k];
            o << ";\n";
            for (int k = t.mix_begin; k < t.mix_end; ++k) emit_rec_sign(ph.recs[k], "pb", f, in);
            if (nfac[cls]++ == 0) o << in << "unsigned " << g << " = " << f << ";\n";
            else o << in << g << " ^= " << f << ";\n";
        }
        int nph = 0;
        std::function<void(int, const std::string &)> visit = [&](int r, const std::string &p) {
            if (!p.empty()) o << in << "v" << r << " = sxor(v" << r << ", " << p << ");\n";
            const int top = r ? 64 - __builtin_clzll(static_cast<unsigned long long>(r)) : 0;
            for (int b = top; b < R; ++b) {
                const int ch = r | (1 << b);
                if (!nfac[b]) {
                    visit(ch, p);
                    continue;
                }
                const std::string gb = "m" + std::to_string(b);
                std::string q = gb;
                if (!p.empty()) {
                    q = "q" + std::to_string(nph++);
                    o << in << "const unsigned " << q << " = " << p << " ^ " << gb << ";\n";
                }
                visit(ch, q);
            }
        };
        visit(0, nfac[R] ? "m" + std::to_string(R) : "");
        o << ind << "}\n";
        if (op.flush.regmask && !uniform)
            for (int r = 0; r < NR; ++r)
                if ((op.flush.regmask >> r) & 1) cmul_const(r, op.regtab[r], ind);
        return true;
    }

    void emit_flush(const HostOp &op, const std::string &ind) {
        if (emit_flush_sign(op, ind)) return;
        const int NR = 1 << R;
        o << ind << "{\n";
        const std::string in = ind + "  ";
        std::vector<int> nfac(R + 1, 0); // index R: the all-slot class
        for (int ti = op.flush.tgt_begin; ti < op.flush.tgt_end; ++ti) {
            const FlushTarget &t = ph.targets[ti];
            const int cls = t.slot < 0 ? R : t.slot;
            const std::string g = "g" + std::to_string(cls);
            const std::string f = "f" + std::to_string(ti);
            // the factor's terms (no multiplication by a constant 1: without
            // fast-math 0 * x does not fold, so it would cost FP64 work)
            std::vector<std::string> terms;
            if (t.eidx >= 0) terms.push_back("E[" + eoff() + std::to_string(ebase[cur_group] + t.eidx) + "]");
            if (t.table >= 0) terms.push_back("tab" + std::to_string(ti));
            if (t.table_lo >= 0)
                terms.push_back("stab[" + std::to_string(stab_off.at(t.table_lo)) + " + (s & " +
                                std::to_string((1 << t.lo_bits) - 1) + ")]");
            if (t.table_hi >= 0)
                terms.push_back("stab[" + std::to_string(stab_off.at(t.table_hi)) + " + (s >> " +
                                std::to_string(t.lo_bits) + ")]");
            if (terms.empty()) terms.push_back("mk(1, 0)");
            o << in << V << " " << f << " = " << terms[0] << ";\n";
            for (size_t k = 1; k < terms.size(); ++k) o << in << f << " = cmulv(" << f << ", " << terms[k] << ");\n";
            for (int k = t.mix_begin; k < t.mix_end; ++k) emit_rec_factor(ph.recs[k], "pb", f, in);
            if (nfac[cls]++ == 0) o << in << V << " " << g << " = " << f << ";\n";
            else o << in << g << " = cmulv(" << g << ", " << f << ");\n";
        }
        bool uniform = op.flush.regmask == (NR >= 32 ? 0xffffffffu : ((1u << NR) - 1)) &&
                       static_cast<int>(op.regtab.size()) >= NR && op.regtab[0].imag() == 0.0;
        for (int r = 1; uniform && r < NR; ++r) uniform = op.regtab[r] == op.regtab[0];
        // root: "" (identity), a real constant, or the all-slot factor
        std::string root;
        double rc = 1.0;
        if (uniform) rc = op.regtab[0].real();
        if (track && uniform && rc != 1.0) {
            for (double &x : sc) x *= rc;
            rc = 1.0;
            if (final_op) materialize(ind);
        }
        if (nfac[R]) {
            root = "g" + std::to_string(R);
            if (rc != 1.0) o << in << root << " = " << rscale(root, rc) << ";\n";
        }
        int nph = 0;
        // ph: variable holding the product for slot r ("" = identity), or the
        // real constant rc when the slot carries only the scale
        std::function<void(int, const std::string &, bool)> visit = [&](int r, const std::string &p, bool scaled) {
            if (!p.empty()) o << in << "v" << r << " = cmulv(v" << r << ", " << p << ");\n";
            else if (scaled && rc != 1.0)
                o << in << "v" << r << " = " << rscale("v" + std::to_string(r), rc) << ";\n";
            const int top = r ? 64 - __builtin_clzll(static_cast<unsigned long long>(r)) : 0;
            for (int b = top; b < R; ++b) {
                const int ch = r | (1 << b);
                if (!nfac[b]) {
                    visit(ch, p, scaled);
                    continue;
                }
                const std::string gb = "g" + std::to_string(b);
                std::string q;
                if (!p.empty()) {
                    q = "p" + std::to_string(nph++);
                    o << in << V << " " << q << " = cmulv(" << p << ", " << gb << ");\n";
                } else if (scaled && rc != 1.0) {
                    q = "p" + std::to_string(nph++);
                    o << in << V << " " << q << " = " << rscale(gb, rc) << ";\n";
                } else q = gb;
                visit(ch, q, false);
            }
        };
        visit(0, root, root.empty() && uniform);
        o << ind << "}\n";
        if (op.flush.regmask && !uniform)
            for (int r = 0; r < NR; ++r)
                if ((op.flush.regmask >> r) & 1) cmul_const(r, op.regtab[r], ind);
    }

    // Types and helpers shared by every pass body of one source.
    std::string common() const {
        std::ostringstream c;
        c << "typedef unsigned long long u64;\n";
        c << "struct __align__(" << (f32 ? 8 : 16) << ") " << V << " { " << T << " x, y; };\n";
        c << "static __device__ __forceinline__ " << V << " mk(" << T << " x, " << T << " y) { " << V
          << " r; r.x = x; r.y = y; return r; }\n";
        if (packed) {
            // complex64 arithmetic on packed f32x2 registers (FFMA2 / FMUL2 /
            // FADD2, sm_100a): (a + ib) x = a (x.x, x.y) + b (-x.y, x.x), the
            // swapped and sign-flipped halves fold into the operand modifiers
            c << "#define QD static __device__ __forceinline__\n"
                 "QD u64 pk(float a, float b) { u64 r; asm(\"mov.b64 %0, {%1,%2};\" : \"=l\"(r) : \"f\"(a), \"f\"(b)); return r; }\n"
                 "QD u64 pv(cf v) { return pk(v.x, v.y); }\n"
                 "QD u64 bc(float k) { return pk(k, k); }\n"
                 "QD cf up(u64 r) { cf v; asm(\"mov.b64 {%0,%1}, %2;\" : \"=f\"(v.x), \"=f\"(v.y) : \"l\"(r)); return v; }\n"
                 "QD u64 fma2(u64 a, u64 b, u64 c) { u64 r; asm(\"fma.rn.f32x2 %0, %1, %2, %3;\" : \"=l\"(r) : \"l\"(a), \"l\"(b), \"l\"(c)); return r; }\n"
                 "QD u64 mul2(u64 a, u64 b) { u64 r; asm(\"mul.rn.f32x2 %0, %1, %2;\" : \"=l\"(r) : \"l\"(a), \"l\"(b)); return r; }\n"
                 "QD u64 add2(u64 a, u64 b) { u64 r; asm(\"add.rn.f32x2 %0, %1, %2;\" : \"=l\"(r) : \"l\"(a), \"l\"(b)); return r; }\n"
                 "QD u64 sub2(u64 a, u64 b) { u64 r; asm(\"sub.rn.f32x2 %0, %1, %2;\" : \"=l\"(r) : \"l\"(a), \"l\"(b)); return r; }\n"
                 "QD cf cneg(cf x) { return mk(-x.x, -x.y); }\n"
                 "QD cf cadd(cf a, cf x) { return up(add2(pv(a), pv(x))); }\n"
                 "QD cf csub(cf a, cf x) { return up(sub2(pv(a), pv(x))); }\n"
                 "QD cf rmul(cf x, float k) { return up(mul2(bc(k), pv(x))); }\n"
                 "QD cf rfma(cf a, cf x, float k) { return up(fma2(bc(k), pv(x), pv(a))); }\n"
                 "QD u64 pn(cf v) { return pk(-v.y, v.x); }\n"
                 "QD cf imul(cf x, float k) { return up(mul2(bc(k), pn(x))); }\n"
                 "QD cf ifma(cf a, cf x, float k) { return up(fma2(bc(k), pn(x), pv(a))); }\n"
                 "QD cf cmc(cf x, float re, float im) { return up(fma2(bc(im), pn(x), mul2(bc(re), pv(x)))); }\n"
                 "QD cf cfc(cf a, cf x, float re, float im) { return up(fma2(bc(im), pn(x), fma2(bc(re), pv(x), pv(a)))); }\n"
                 "QD cf cti(cf x, float t) { return up(fma2(bc(t), pn(x), pv(x))); }\n"
                 "QD cf cit(cf x, float t) { return up(fma2(bc(t), pv(x), pn(x))); }\n"
                 "QD cf cmulv(cf a, cf b) { return cmc(b, a.x, a.y); }\n"
                 "QD cf cfmav(cf a, cf b, cf c) { return cfc(c, b, a.x, a.y); }\n";
        } else {
            c << "static __device__ __forceinline__ " << V << " cmulv(" << V << " a, " << V
              << " b) { return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }\n";
            c << "static __device__ __forceinline__ " << V << " cfmav(" << V << " a, " << V << " b, " << V
              << " c) { return mk(c.x + a.x * b.x - a.y * b.y, c.y + a.x * b.y + a.y * b.x); }\n";
        }
        // a +-1 factor as a sign mask (0 or 0x80000000 on the high word of each component)
        const char *nosign_dbg = std::getenv("QSV_DEBUG_NOSIGN");  // diagnostics only: wrong results
        if (nosign_dbg && nosign_dbg[0] == '1')
            c << "static __device__ __forceinline__ " << V << " sxor(" << V << " v, unsigned s) { (void)s; return v; }\n";
        else if (f32)
            c << "static __device__ __forceinline__ cf sxor(cf v, unsigned s) { return mk(__uint_as_float(__float_as_uint(v.x) ^ s), "
                 "__uint_as_float(__float_as_uint(v.y) ^ s)); }\n";
        else
            c << "static __device__ __forceinline__ cd sxor(cd v, unsigned s) { return mk(__hiloint2double(__double2hiint(v.x) ^ (int)s, "
                 "__double2loint(v.x)), __hiloint2double(__double2hiint(v.y) ^ (int)s, __double2loint(v.y))); }\n";
        // streaming (evict-first) 8/16-byte amplitude loads and stores; stwb:
        // a plain write-back store (the first pass of an L2 super-pass keeps
        // its output in L2 for the second)
        const char *sfx = f32 ? "v2.f32" : "v2.f64";
        const char *rc = f32 ? "f" : "d";
        c << "static __device__ __forceinline__ " << V << " ldcs(const " << V << " *p) { " << V
          << " r; asm volatile(\"ld.global.cs." << sfx << " {%0,%1}, [%2];\" : \"=" << rc << "\"(r.x), \"=" << rc
          << "\"(r.y) : \"l\"(p)); return r; }\n";
        c << "static __device__ __forceinline__ " << V << " ldcg(const " << V << " *p) { " << V
          << " r; asm volatile(\"ld.global.cg." << sfx << " {%0,%1}, [%2];\" : \"=" << rc << "\"(r.x), \"=" << rc
          << "\"(r.y) : \"l\"(p) : \"memory\"); return r; }\n";
        c << "static __device__ __forceinline__ void stcs(" << V << " *p, " << V << " v) { asm volatile(\"st.global.cs."
          << sfx << " [%0], {%1,%2};\" :: \"l\"(p), \"" << rc << "\"(v.x), \"" << rc << "\"(v.y) : \"memory\"); }\n";
        c << "static __device__ __forceinline__ void stwb(" << V << " *p, " << V << " v) { asm volatile(\"st.global."
          << sfx << " [%0], {%1,%2};\" :: \"l\"(p), \"" << rc << "\"(v.x), \"" << rc << "\"(v.y) : \"memory\"); }\n";
        c << "struct Args { void *state; u64 row_stride, rank_base, tiles_per_row, total_tiles; const " << V
          << " *tables; const " << T << " *enc_table; int batch; int tpc; void *out; double *zout; const " << V
          << " *prefix; void *const *peers; u64 out_lconst; int out_rconst; };\n";
        return c.str();
    }

    // complex64: the register slot whose tile bit is 0 (its register pairs
    // are adjacent amplitudes, one 16-byte shared-memory access), or -1
    int pair_slot(const HostGroup &g) const {
        for (int j = 0; j < R; ++j)
            if (g.slot_bit[j] == 0) return j;
        return -1;
    }
    // QSV_X_NOPAIR=1 (A/B switch): complex64 register pairs as two 8-byte accesses
    bool noswz_pairs = [] {
        const char *e = std::getenv("QSV_X_NOPAIR");
        return e && e[0] == '1';
    }();

    int threads_of() const { return (threads_for(ph, f32 ? QSV_C64 : QSV_C128) + 31) / 32 * 32; }

    // A whole single-pass kernel: the pass body over this CTA's tiles (a
    // block of a.tpc consecutive tiles, or with a.tpc == 0 a grid-strided
    // sequence).
    std::string source(const std::string &name) {
        const int threads = threads_of();
        const std::string body = body_fn("pass_body");
        std::ostringstream k;
        k << "// generated by qsv codegen.cpp: one fused tile pass\n" << common() << pool_decl() << body;
        k << "extern \"C\" __global__ void __launch_bounds__(" << threads << ", "
          << (double_buffer ? 1 : kernel_min_blocks(ph, threads)) << ") " << name << "(const Args a) {\n";
        k << "  extern __shared__ __align__(16) unsigned char smem_raw[];\n";
        k << "  const u64 t0 = a.tpc > 0 ? (u64)blockIdx.x * a.tpc : (u64)blockIdx.x;\n";
        k << "  const u64 tend = a.tpc > 0 ? (t0 + a.tpc < a.total_tiles ? t0 + a.tpc : a.total_tiles) : a.total_tiles;\n";
        k << "  const u64 tstep = a.tpc > 0 ? 1ull : (u64)gridDim.x;\n";
        k << "  pass_body(a, t0, tend, tstep, smem_raw);\n";
        // peer-memory stores: performed system-wide before the CTA retires
        if (gout) k << "  __threadfence_system();\n";
        k << "}\n";
        return k.str();
    }

    // The pass as a device function over tiles t0, t0 + tstep, ... < tend.
    std::string body_fn(const std::string &fname) {
        const int K = ph.K, L = ph.L, NR = 1 << R;
        const int amp = f32 ? 8 : 16;
        const int apu = 16 / amp;
        const int nchunks = (1 << K) / apu;
        const int nsets = 1 << (K - R);
        const int threads = threads_of();
        const bool dbuf = double_buffer;
        if (f32) {
            // patterns in chunk bits (tile bit b >= 1 is chunk bit b - 1): per
            // group the first three thread-varying chunk bits of one wavefront
            std::vector<std::vector<int>> pats;
            for (const HostGroup &g : ph.groups) {
                if (ph.K - ph.R < 4) continue;
                const bool pair = pair_slot(g) >= 0;
                const int first = pair ? 0 : 1;  // tile bit 0 is ng_bit[0] when it is not a slot
                if (!pair && g.ng_bit[0] != 0) continue;
                pats.push_back({g.ng_bit[first] - 1, g.ng_bit[first + 1] - 1, g.ng_bit[first + 2] - 1});
            }
            if (!ph.out_perm.empty()) {
                std::vector<std::pair<int, int>> q;
                for (int i = 0; i < ph.K; ++i) q.emplace_back(ph.out_perm[ph.tile_pos[i]], i);
                std::sort(q.begin(), q.end());
                // 8-byte reads in output order: 16 per wavefront
                std::vector<int> b;
                for (int i = 0; i < 4 && i < ph.K; ++i)
                    if (q[i].second != 0) b.push_back(q[i].second - 1);
                if (b.size() >= 3) pats.push_back({b[0], b[1], b[2]});
            }
            choose_swizzle(pats);
            const bool oldswz = [] {  // QSV_X_OLDSWZ=1 (A/B): the fixed fold of round 1
                const char *e = std::getenv("QSV_X_OLDSWZ");
                return e && e[0] == '1';
            }();
            if (oldswz)
                for (int i = 0; i < 3; ++i) swm[i] = (1 << (3 + i)) | (1 << (6 + i)) | (1 << (9 + i)) | (1 << (12 + i));
            o << "static __device__ __forceinline__ int swz(int u) { const int w = u >> 1; return ((w ^ ((__popc(w & "
              << swm[0] << ") & 1) | ((__popc(w & " << swm[1] << ") & 1) << 1) | ((__popc(w & " << swm[2]
              << ") & 1) << 2))) << 1) | (u & 1); }\n";
        } else {
            // patterns of this pass: each group's first three set bits, the
            // copy-out's first three input bits
            std::vector<std::vector<int>> pats;
            for (const HostGroup &g : ph.groups)
                if (ph.K - ph.R >= 3) pats.push_back({g.ng_bit[0], g.ng_bit[1], g.ng_bit[2]});
            if (!ph.out_perm.empty()) {
                std::vector<std::pair<int, int>> q;
                for (int i = 0; i < ph.K; ++i) q.emplace_back(ph.out_perm[ph.tile_pos[i]], i);
                std::sort(q.begin(), q.end());
                pats.push_back({q[0].second, q[1].second, q[2].second});
            }
            choose_swizzle(pats);
            o << "static __device__ __forceinline__ int swz(int u) { return u ^ ((__popc(u & " << swm[0]
              << ") & 1) | ((__popc(u & " << swm[1] << ") & 1) << 1) | ((__popc(u & " << swm[2] << ") & 1) << 2)); }\n";
        }
        o << "static __device__ __forceinline__ void " << fname
          << "(const Args &a, const u64 t0, const u64 tend, const u64 tstep, unsigned char *smem_raw) {\n";
        // per-tile external phase factors of ALL groups get distinct slots
        ebase.assign(ph.groups.size(), 0);
        int next_max = 0;
        for (size_t gi = 0; gi < ph.groups.size(); ++gi) {
            const HostGroup &g = ph.groups[gi];
            int ne = 0;
            for (int ti = g.tgt_begin; ti < g.tgt_end; ++ti)
                if (ph.targets[ti].eidx >= 0) ne = std::max(ne, ph.targets[ti].eidx + 1);
            ebase[gi] = next_max;
            next_max += ne;
        }
        const bool pf = prefetch;
        late = pf;  // prefetching passes issue tile t + 1 after tile t's first barrier
        // late-issue prefetch rewrites E while other warps may still read the
        // previous tile's factors: one E set per shared tile
        // dynamic shared memory: the tile ring first, then this pass's E /
        // stab / Eraw arrays (not static __shared__: the two passes of a
        // super-pass share one launch and must not add up)
        {
            const size_t tile = static_cast<size_t>(amp) << K;
            const bool shared_tile = ph.groups.size() >= 2 || !ph.out_perm.empty();
            dyn_base = pf ? static_cast<size_t>(stages) * tile : shared_tile ? tile : 0;
            dyn_extra = 0;
        }
        if (next_max) salloc("E", late ? 2 * next_max : next_max);
        e_stride = next_max;
        // separable phase tables (low / high set-index bits) live in shared memory
        {
            std::vector<std::pair<int, int>> ranges; // (global offset, length)
            for (const FlushTarget &t : ph.targets) {
                const int nb = ph.K - ph.R;
                if (t.table_lo >= 0) ranges.emplace_back(t.table_lo, 1 << t.lo_bits);
                if (t.table_hi >= 0) ranges.emplace_back(t.table_hi, 1 << (nb - t.lo_bits));
            }
            int total = 0;
            for (auto &r : ranges) {
                stab_off[r.first] = total;
                total += r.second;
            }
            if (total) {
                salloc("stab", total);
                for (auto &r : ranges)
                    o << "  for (int i = threadIdx.x; i < " << r.second << "; i += " << threads << ") stab["
                      << stab_off[r.first] << " + i] = a.tables[" << r.first << " + i];\n";
                o << "  __syncthreads();\n";
            }
        }
        std::vector<int> hi(ph.tile_pos.begin() + L, ph.tile_pos.end());
        int tpr_log = static_cast<int>(ph.ext_pos.size());
        // The first group reads its register sets straight from HBM and the
        // last group writes them straight back; only the groups in between
        // exchange amplitudes through the shared-memory tile. A one-group pass
        // is a pure streaming kernel.
        (void)dbuf;
        (void)hi;
        (void)apu;
        (void)nchunks;
        const int G = static_cast<int>(ph.groups.size());
        const bool permuted = !ph.out_perm.empty();
        const bool any_e = next_max > 0;
        // prefetch mode: two shared tiles; while tile t is transformed, the
        // cp.async copies of tile t + gridDim stream into the other buffer and
        // the first group reads shared memory instead of HBM
        // Per-tile external phase factors E (one per FlushTarget with eidx >= 0),
        // each owned by one thread spread over the warps. Pipelined (prefetch +
        // late issue): the owner cp.asyncs the table entries of tile t + gridDim
        // together with that tile's data and multiplies them out at the end of
        // tile t, so no L2 round trip sits in front of a tile's first barrier.
        struct ETask {
            int thr, slot, ti, raw;
        };
        std::vector<ETask> etasks;
        int nraw = 0;
        {
            int k = 0;
            const int nwarps = threads / 32;
            for (size_t gi = 0; gi < ph.groups.size(); ++gi) {
                const HostGroup &g = ph.groups[gi];
                for (int ti = g.tgt_begin; ti < g.tgt_end; ++ti) {
                    const FlushTarget &t = ph.targets[ti];
                    if (t.eidx < 0) continue;
                    const int thr = (k % nwarps) * 32 + (k / nwarps) % 32;
                    ++k;
                    etasks.push_back({thr, ebase[gi] + t.eidx, ti, nraw});
                    nraw += t.ext_chunks;
                }
            }
        }
        auto emit_e_store = [&](const ETask &e, const std::string &eofs, const std::string &ind) {
            o << ind << "E[" << eofs << e.slot << "] = f;\n";
        };
        const bool epipe = pf && late && any_e;
        const std::string tmask = std::to_string((1ull << tpr_log) - 1) + "ull";
        auto emit_e_direct = [&](const std::string &ind) {
            for (const ETask &e : etasks) {
                const FlushTarget &t = ph.targets[e.ti];
                o << ind << "if (threadIdx.x == " << e.thr << ") {\n" << ind << "  " << V << " f = mk(1, 0);\n";
                for (int c = 0; c < t.ext_chunks; ++c)
                    o << ind << "  f = cmulv(f, a.tables[" << t.ext_tab + c * 256 << " + ((tl >> " << 8 * c
                      << ") & 255)]);\n";
                for (int q = t.ext_rest; q < t.ext_end; ++q) emit_rec_factor(ph.recs[q], "pbase", "f", ind + "  ");
                emit_e_store(e, eoff(), ind + "  ");
                o << ind << "}\n";
            }
        };
        auto emit_e_issue = [&](const std::string &tv, const std::string &nb, const std::string &ind) {
            if (!nraw) return;
            o << ind << "{ const u64 tlx = (" << tv << ") & " << tmask << ";\n";
            for (const ETask &e : etasks) {
                const FlushTarget &t = ph.targets[e.ti];
                if (!t.ext_chunks) continue;
                o << ind << "  if (threadIdx.x == " << e.thr << ") {\n";
                for (int c = 0; c < t.ext_chunks; ++c) {
                    o << ind << "    asm volatile(\"cp.async." << (f32 ? "ca" : "cg") << ".shared.global [%0], [%1], "
                      << (f32 ? 8 : 16) << ";\\n\" :: \"r\"((unsigned)__cvta_generic_to_shared(&Eraw[(" << nb << ") * "
                      << nraw << " + " << e.raw + c << "])), \"l\"(&a.tables[" << t.ext_tab + c * 256
                      << " + ((tlx >> " << 8 * c << ") & 255)]) : \"memory\");\n";
                }
                o << ind << "  }\n";
            }
            o << ind << "}\n";
        };
        auto emit_e_compute = [&](const std::string &tv, const std::string &nb, const std::string &ind) {
            o << ind << "{ const u64 tlx = (" << tv << ") & " << tmask << ";\n";
            o << ind << "  const u64 pbx = a.rank_base | " << scatter("tlx", ph.ext_pos, true) << ";\n";
            o << ind << "  (void)pbx;\n";
            for (const ETask &e : etasks) {
                const FlushTarget &t = ph.targets[e.ti];
                o << ind << "  if (threadIdx.x == " << e.thr << ") {\n" << ind << "    " << V << " f = mk(1, 0);\n";
                for (int c = 0; c < t.ext_chunks; ++c)
                    o << ind << "    f = " << (c ? "cmulv(f, " : "(") << "Eraw[(" << nb << ") * " << nraw << " + "
                      << e.raw + c << "]);\n";
                for (int q = t.ext_rest; q < t.ext_end; ++q) emit_rec_factor(ph.recs[q], "pbx", "f", ind + "    ");
                emit_e_store(e, "(" + nb + ") * " + std::to_string(e_stride) + " + ", ind + "    ");
                o << ind << "  }\n";
            }
            o << ind << "}\n";
        };
        const std::string commit = "asm volatile(\"cp.async.commit_group;\\n\" ::: \"memory\");\n";
        if (epipe && nraw) salloc("Eraw", 2 * nraw);
        // tiles of this CTA: a block of a.tpc consecutive tiles (neighbouring
        // DRAM runs back to back) or, with a.tpc == 0, a grid-strided sequence
        if (pf) {
            o << "  auto issue = [&](u64 t, " << V << " *buf) {\n";
            o << "    const int row = (int)(t >> " << tpr_log << ");\n";
            o << "    const u64 tl = t & " << tmask << ";\n";
            o << "    const " << V << " *src = (const " << V << " *)a.state + (u64)row * a.row_stride;\n";
            o << "    const u64 tb = " << scatter("tl", ph.ext_pos, true) << ";\n";
            // chunk u = tid * apu + k * threads * apu: bit scatter and swizzle are
            // linear, so the per-thread parts are computed once
            const int step = threads * apu;
            o << "    const int u0 = threadIdx.x * " << apu << ";\n";
            o << "    const u64 g0 = tb | (" << scatter("(u0 >> " + std::to_string(L) + ")", hi, true) << ") | (u0 & "
              << ((1 << L) - 1) << ");\n";
            o << "    const int s0 = swz(u0);\n";
            if (nchunks % threads == 0) {
                // unrolled: per chunk one constant global offset (its tile bits
                // are disjoint from g0's, so OR = ADD) and one constant XOR
                o << "    const " << V << " *p0 = src + g0;\n";
                for (int k = 0; k < nchunks / threads; ++k) {
                    const int uk = k * step;
                    uint64_t gk = static_cast<uint64_t>(uk & ((1 << L) - 1));
                    for (size_t i = 0; i < hi.size(); ++i)
                        if (((uk >> L) >> i) & 1) gk |= 1ull << hi[i];
                    o << "    asm volatile(\"cp.async.cg.shared.global [%0], [%1], 16;\\n\" :: \"r\"((unsigned)"
                         "__cvta_generic_to_shared(&buf[s0 "
                      << (noswz() ? "+ " : "^ ") << swz_of(uk) << "])), \"l\"(p0 + " << gk << "ull) : \"memory\");\n";
                }
                o << "  };\n";
            } else {
                o << "    for (int k = 0; k * " << threads << " + threadIdx.x < " << nchunks << "; ++k) {\n";
            // k * step has bits only at or above log2(step) (a power of two)
            o << "      const int uk = k * " << step << ";\n";
            o << "      const u64 g = g0 | (" << scatter("(uk >> " + std::to_string(L) + ")", hi, true) << ") | (uk & "
              << ((1 << L) - 1) << ");\n";
            o << "      const unsigned sa = (unsigned)__cvta_generic_to_shared(&buf[s0 ^ swz(uk)]);\n";
            o << "      asm volatile(\"cp.async.cg.shared.global [%0], [%1], 16;\\n\" :: \"r\"(sa), \"l\"(&src[g]) : "
                 "\"memory\");\n";
            o << "    }\n  };\n";
            }
            // S-stage ring (late issue): tile t + (S-1) steps is issued at the
            // top of tile t; per iteration the commit groups are [Eraw of the
            // next tile] (epipe only) and [tile data], so tile t is complete
            // once at most (S-2) * gpi younger groups are pending
            const int S = late ? stages : 2;
            const int gpi = epipe ? 2 : 1;  // commit groups per iteration
            o << "  int cur = 0, ec = 0;\n";
            if (epipe) {
                o << "  if (t0 < tend) {\n";
                emit_e_issue("t0", "0", "    ");
                o << "  }\n  " << commit;
            }
            o << "  if (t0 < tend) issue(t0, (" << V << " *)smem_raw);\n";
            o << "  " << commit;
            for (int j = 1; j + 1 < S; ++j) {
                if (epipe) o << "  " << commit;  // (empty) Eraw slot keeps the group count uniform
                o << "  if (t0 + " << j << " * tstep < tend) issue(t0 + " << j << " * tstep, (" << V
                  << " *)smem_raw + (" << j << " << " << K << "));\n";
                o << "  " << commit;
            }
            if (epipe) {
                o << "  asm volatile(\"cp.async.wait_group " << 1 + (S - 2) * gpi << ";\\n\" ::: \"memory\");\n";
                o << "  if (t0 < tend) {\n";
                emit_e_compute("t0", "0", "    ");
                o << "  }\n";
            }
        } else {
            o << "  " << V << " *tile = (" << V << " *)smem_raw;\n";
            o << "  (void)tile;\n";
        }
        const int S = (pf && late) ? stages : 2;
        const int gpi = epipe ? 2 : 1;
        o << "  for (u64 t = t0; t < tend; t += tstep) {\n";
        const std::string nb = S == 2 ? "(cur ^ 1)" : "((cur + " + std::to_string(S - 1) + ") % " + std::to_string(S) + ")";
        const std::string issue_next = "    if (t + " + std::to_string(S - 1) + " * tstep < tend) issue(t + " +
                                       std::to_string(S - 1) + " * tstep, (" + std::string(V) + " *)smem_raw + (" + nb +
                                       " << " + std::to_string(K) + "));\n    " + commit;
        if (pf) {
            o << "    " << V << " *tile = (" << V << " *)smem_raw + (cur << " << K << ");\n";
            if (!late) o << issue_next;
        }
        o << "    const int row = (int)(t >> " << tpr_log << ");\n";
        o << "    (void)row;\n";
        o << "    const u64 tl = t & " << tmask << ";\n";
        o << "    " << V << " *st = (" << V << " *)a.state + (u64)row * a.row_stride;\n";
        o << "    const u64 tb = " << scatter("tl", ph.ext_pos, true) << ";\n";
        o << "    const u64 pbase = a.rank_base | tb;\n";
        if (gout) {
            // stores go to the destination rank's buffer: the ext bits map to
            // local output bits or to rank bits (tile bits map to themselves)
            const int nl = K + static_cast<int>(ph.ext_pos.size());
            std::vector<std::pair<int, int>> lp, rp;
            for (size_t i = 0; i < ph.ext_pos.size(); ++i) {
                const int q = ph.gperm[ph.ext_pos[i]];
                if (q < nl) lp.emplace_back(static_cast<int>(i), q);
                else rp.emplace_back(static_cast<int>(i), q - nl);
            }
            o << "    const u64 tbo = " << scatter_sel("tl", lp) << ";\n";
            o << "    const int drk = a.out_rconst | (int)(" << scatter_sel("tl", rp) << ");\n";
            o << "    const u64 rowoff = (u64)row * a.row_stride + a.out_lconst;\n";
        }
        if (!epipe) emit_e_direct("    ");
        if (pf) {
            // early issue: tile t + gridDim is already in flight, wait for the
            // older group only. Late issue: this barrier also retires every
            // read of the buffer about to be refilled (the previous tile), so
            // the next copy goes out now and no end-of-tile barrier is needed.
            o << "    asm volatile(\"cp.async.wait_group " << (late ? (S - 2) * gpi : 1) << ";\\n\" ::: \"memory\");\n";
            o << "    __syncthreads();\n";
            if (epipe) {
                o << "    if (t + tstep < tend) {\n";
                emit_e_issue("t + tstep", "ec ^ 1", "      ");
                o << "    }\n    " << commit;
            }
            if (late) o << issue_next;
        } else if (any_e) o << "    __syncthreads();\n";
        for (size_t gi = 0; gi < ph.groups.size(); ++gi) {
            const HostGroup &g = ph.groups[gi];
            cur_group = static_cast<int>(gi);
            const bool from_hbm = gi == 0 && !pf, to_hbm = static_cast<int>(gi) == G - 1 && !permuted;
            o << "    // ---- group " << gi << "\n";
            std::vector<int> ngt(g.ng_bit, g.ng_bit + (K - R)), ngp;
            for (int b : ngt) ngp.push_back(ph.tile_pos[b]);
            const bool zhere = zsum && to_hbm;
            if (zhere) {
                // fused <Z> epilogue (one tile = one whole row): per-thread sums of
                // |a|^2 in total and per physical bit, FP64
                o << "    double zacc[" << K + 1 << "];\n";
                o << "#pragma unroll\n    for (int j = 0; j < " << K + 1 << "; ++j) zacc[j] = 0.0;\n";
            }
            o << "    for (int s = threadIdx.x; s < " << nsets << "; s += " << threads << ") {\n";
            o << "      const int ub = " << scatter("s", ngt, false) << ";\n";
            o << "      const int sb = swz(ub);\n";
            o << "      const u64 ls = " << scatter("s", ngp, true) << ";\n";
            o << "      const u64 pb = pbase | ls;\n";
            o << "      const u64 gb = tb | ls;\n";
            // peer-memory stores (last group): the set's bits and each
            // register's slot bits map to output local bits or rank bits
            std::vector<uint64_t> poffo(NR, 0);
            std::vector<int> rkr(NR, 0);
            if (gout && to_hbm) {
                const int nl = K + static_cast<int>(ph.ext_pos.size());
                std::vector<std::pair<int, int>> lsp, rsp;
                for (size_t i = 0; i < ngt.size(); ++i) {
                    const int q = ph.gperm[ph.tile_pos[ngt[i]]];
                    if (q < nl) lsp.emplace_back(static_cast<int>(i), q);
                    else rsp.emplace_back(static_cast<int>(i), q - nl);
                }
                o << "      const u64 lso = " << scatter_sel("s", lsp) << ";\n";
                o << "      const int rks = drk | (int)(" << scatter_sel("s", rsp) << ");\n";
                std::map<int, int> ptrs;
                for (int r = 0; r < NR; ++r) {
                    for (int j = 0; j < R; ++j)
                        if ((r >> j) & 1) {
                            const int q = ph.gperm[ph.tile_pos[g.slot_bit[j]]];
                            if (q < nl) poffo[r] |= 1ull << q;
                            else rkr[r] |= 1 << (q - nl);
                        }
                    if (!ptrs.count(rkr[r])) {
                        const int id = static_cast<int>(ptrs.size());
                        ptrs[rkr[r]] = id;
                        o << "      " << V << " *const pd" << id << " = (" << V << " *)a.peers[rks | " << rkr[r]
                          << "] + rowoff + lso;\n";
                    }
                    rkr[r] = ptrs[rkr[r]];
                }
            }
            o << "      (void)ub; (void)sb; (void)gb;\n";
            // phase tables: issue the (L2-resident) loads before the gate math
            for (int oi = g.op_begin; oi < g.op_end; ++oi) {
                const HostOp &op = ph.ops[oi];
                if (op.code != OP_FLUSH) continue;
                for (int ti = op.flush.tgt_begin; ti < op.flush.tgt_end; ++ti)
                    if (ph.targets[ti].table >= 0)
                        o << "      const " << V << " tab" << ti << " = a.tables[" << ph.targets[ti].table
                          << " + s];\n";
            }
            std::vector<int> uoff(NR, 0);
            const int pj = f32 && !noswz_pairs ? pair_slot(g) : -1;  // complex64: register slot holding tile bit 0
            std::vector<uint64_t> poff(NR, 0); // physical offsets of the register amplitudes
            for (int r = 0; r < NR; ++r)
                for (int j = 0; j < R; ++j)
                    if ((r >> j) & 1) {
                        uoff[r] |= 1 << g.slot_bit[j];
                        poff[r] |= 1ull << ph.tile_pos[g.slot_bit[j]];
                    }
            if (from_hbm && ph.synth) {
                // product state M_k..M_1|0> per wire: the set's factor over its
                // non-slot bits, then a binary tree over the R slot bits
                const int nl = K + static_cast<int>(ph.ext_pos.size());
                o << "      const " << V << " *U = a.prefix + (u64)row * " << 2 * nl << ";\n";
                o << "      " << V << " f = mk(1, 0);\n";
                for (size_t i = 0; i < ngt.size(); ++i)
                    o << "      f = cmulv(f, U[" << 2 * ph.tile_pos[ngt[i]] << " + ((s >> " << i << ") & 1)]);\n";
                for (int e : ph.ext_pos)
                    o << "      f = cmulv(f, U[" << 2 * e << " + (int)((tb >> " << e << ") & 1ull)]);\n";
                std::vector<std::string> cur{"f"};
                for (int j = 0; j < R; ++j) {
                    const int pj = ph.tile_pos[g.slot_bit[j]];
                    std::vector<std::string> nxt(cur.size() * 2);
                    for (size_t r = 0; r < cur.size(); ++r)
                        for (int b = 0; b < 2; ++b) {
                            const size_t idx = r | (static_cast<size_t>(b) << j);
                            const std::string nm = j + 1 == R ? "v" + std::to_string(idx)
                                                              : "t" + std::to_string(j) + "_" + std::to_string(idx);
                            o << "      " << V << " " << nm << " = cmulv(" << cur[r] << ", U[" << 2 * pj + b << "]);\n";
                            nxt[idx] = nm;
                        }
                    cur.swap(nxt);
                }
                if (R == 0) o << "      " << V << " v0 = f;\n";
            } else
                for (int r = 0; r < NR; ++r) {
                    if (from_hbm)
                        o << "      " << V << " v" << r << " = " << ld_in << "(&st[gb + " << poff[r] << "ull]);\n";
                    else if (pj >= 0) {  // complex64 pair (tile bit 0 is slot pj): one 16-byte load
                        if ((r >> pj) & 1) continue;
                        const int r1 = r | (1 << pj);
                        o << "      " << V << " v" << r << ", v" << r1 << "; { const float4 q = *(const float4 *)&tile[sb "
                          << (noswz() ? "+ " : "^ ") << swz_of(uoff[r]) << "]; v" << r << " = mk(q.x, q.y); v" << r1
                          << " = mk(q.z, q.w); }\n";
                    } else o << "      " << V << " v" << r << " = tile[sb " << (noswz() ? "+ " : "^ ") << swz_of(uoff[r])
                           << "];\n";
                }
            // QSV_DEBUG_NOCOMPUTE=1 (diagnostics only): the pass moves data without
            // applying its gates -- the memory-structure ceiling of its geometry
            static const bool nocompute = [] {
                const char *e = std::getenv("QSV_DEBUG_NOCOMPUTE");
                return e && e[0] == '1';
            }();
            std::fill(sc.begin(), sc.end(), 1.0);
            if (!nocompute)
                for (int oi = g.op_begin; oi < g.op_end; ++oi) {
                    final_op = oi == g.op_end - 1;
                    emit_op(ph.ops[oi], "      ");
                }
            final_op = false;
            materialize("      ");
            if (zhere) {
                o << "      { double zt = 0.0";
                for (int j = 0; j < R; ++j) o << ", zs" << j << " = 0.0";
                o << ";\n";
                for (int r = 0; r < NR; ++r) {
                    o << "        { const double q = (double)v" << r << ".x * v" << r << ".x + (double)v" << r << ".y * v" << r
                      << ".y; zt += q;";
                    for (int j = 0; j < R; ++j)
                        if ((r >> j) & 1) o << " zs" << j << " += q;";
                    o << " }\n";
                }
                o << "        zacc[0] += zt;\n";
                for (int j = 0; j < R; ++j) o << "        zacc[" << 1 + ph.tile_pos[g.slot_bit[j]] << "] += zs" << j << ";\n";
                for (size_t i = 0; i < ngt.size(); ++i)
                    o << "        if ((s >> " << i << ") & 1) zacc[" << 1 + ph.tile_pos[ngt[i]] << "] += zt;\n";
                o << "      }\n";
            }
            for (int r = 0; r < NR; ++r) {
                if (to_hbm && gout) o << "      " << st_out << "(&pd" << rkr[r] << "[tbo + " << poffo[r] << "ull], v" << r << ");\n";
                else if (to_hbm) o << "      " << st_out << "(&st[gb + " << poff[r] << "ull], v" << r << ");\n";
                else if (pj >= 0) {
                    if ((r >> pj) & 1) continue;
                    const int r1 = r | (1 << pj);
                    o << "      *(float4 *)&tile[sb " << (noswz() ? "+ " : "^ ") << swz_of(uoff[r]) << "] = make_float4(v"
                      << r << ".x, v" << r << ".y, v" << r1 << ".x, v" << r1 << ".y);\n";
                } else o << "      tile[sb " << (noswz() ? "+ " : "^ ") << swz_of(uoff[r]) << "] = v" << r << ";\n";
            }
            o << "      (void)pb;\n    }\n";
            if (zhere) {
                // block reduction: warp shuffles, then one partial per warp
                const int nw = threads / 32;
                o << "    {\n      __shared__ double zred[" << nw << "][" << K + 1 << "];\n";
                o << "#pragma unroll\n      for (int j = 0; j < " << K + 1 << "; ++j) {\n";
                o << "        double x = zacc[j];\n";
                o << "        for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);\n";
                o << "        if ((threadIdx.x & 31) == 0) zred[threadIdx.x >> 5][j] = x;\n      }\n";
                o << "      __syncthreads();\n";
                o << "      if (threadIdx.x < " << K + 1 << ") {\n        double x = 0.0;\n";
                o << "        for (int w = 0; w < " << nw << "; ++w) x += zred[w][threadIdx.x];\n";
                o << "        a.zout[(u64)row * " << K + 1 << " + threadIdx.x] = x;\n      }\n";
                o << "      __syncthreads();\n    }\n";
            }
            if (!to_hbm) o << "    __syncthreads();\n";
        }
        if (permuted) {
            // out-of-place copy-out in OUTPUT order: w enumerates the tile's
            // output bit positions ascending (the L lowest output bits first,
            // so the writes are contiguous runs); u is the same amplitude's
            // input tile index.
            std::vector<std::pair<int, int>> q; // (output position, input tile bit)
            for (int i = 0; i < K; ++i) q.emplace_back(ph.out_perm[ph.tile_pos[i]], i);
            std::sort(q.begin(), q.end());
            std::vector<int> w2u, w2out, ext_out;
            for (auto &pr : q) w2out.push_back(pr.first), w2u.push_back(pr.second);
            for (int e : ph.ext_pos) ext_out.push_back(ph.out_perm[e]);
            o << "    {\n      " << V << " *dst = (" << V << " *)a.out + (u64)row * a.row_stride;\n";
            o << "      const u64 tbo = " << scatter("tl", ext_out, true) << ";\n";
            if ((1 << K) % threads == 0 && (threads & (threads - 1)) == 0) {
                // w = tid + k * threads: both bit scatters and the swizzle are
                // linear, so the per-thread parts are computed once and every
                // k adds constants (the unrolled loop needs no index math)
                o << "      const int su0 = swz(" << scatter("threadIdx.x", w2u, false) << ");\n";
                o << "      " << V << " *d0 = dst + (tbo | " << scatter("threadIdx.x", w2out, true) << ");\n";
                for (int k = 0; k < (1 << K) / threads; ++k) {
                    const int wk = k * threads;
                    int uk = 0;
                    uint64_t ok = 0;
                    for (size_t i = 0; i < w2u.size(); ++i)
                        if ((wk >> i) & 1) uk |= 1 << w2u[i], ok |= 1ull << w2out[i];
                    o << "      stcs(d0 + " << ok << "ull, tile[su0 ^ " << swz_of(uk) << "]);\n";
                }
                o << "    }\n";
            } else {
                o << "      for (int w = threadIdx.x; w < " << (1 << K) << "; w += " << threads << ") {\n";
                o << "        const int u = " << scatter("w", w2u, false) << ";\n";
                o << "        stcs(&dst[tbo | " << scatter("w", w2out, true) << "], tile[swz(u)]);\n";
                o << "      }\n    }\n";
            }
        }
        // the next tile's first group rewrites the shared tile / E
        if (!late && (G >= 2 || any_e || permuted || pf)) o << "    __syncthreads();\n";
        if (epipe) {
            o << "    asm volatile(\"cp.async.wait_group 1;\\n\" ::: \"memory\");\n";
            o << "    if (t + tstep < tend) {\n";
            emit_e_compute("t + tstep", "ec ^ 1", "      ");
            o << "    }\n";
        }
        if (pf) {
            if (S == 2) o << "    cur ^= 1;\n";
            else o << "    cur = cur + 1 == " << S << " ? 0 : cur + 1;\n";
            o << "    ec ^= 1;\n";
        }
        o << "  }\n";
        if (pf) o << "  asm volatile(\"cp.async.wait_group 0;\\n\" ::: \"memory\");\n";
        o << "}\n";
        return o.str();
    }
    bool double_buffer = true;
    bool prefetch = false;
    bool late = false;
    int e_stride = 0;
    std::string eoff() const { return late ? "(ec * " + std::to_string(e_stride) + ") + " : ""; }
    int stages = 2;  // shared tile buffers in prefetch mode (late issue)
    bool zsum = false; // fused <Z> epilogue in the last group (whole-row tiles)
    std::string st_out = "stcs"; // the last group's stores (stwb: keep the output in L2)
    std::string ld_in = "ldcs";  // the first group's direct loads (ldcg: L2 only, data written in this launch)
    bool gout = false;           // last group stores through peer memory (PassHost::gperm)
    size_t dyn_base = 0, dyn_extra = 0; // dynamic shared memory: tile ring, then salloc'ed arrays
    size_t dyn_bytes() const { return dyn_base + dyn_extra; }
    void salloc(const char *name, int count) {
        o << "  " << V << " *const " << name << " = (" << V << " *)(smem_raw + " << dyn_base + dyn_extra << ");\n";
        dyn_extra += (static_cast<size_t>(count) * (f32 ? 8 : 16) + 15) / 16 * 16;
    }
    std::vector<int> ebase; // first E slot of each group
    int cur_group = 0;
    std::map<int, int> stab_off; // global table offset -> shared-memory offset
};

} // namespace

int kernel_threads(const PassHost &ph, int dtype) { return threads_for(ph, dtype); }

// Shared tile buffers of a prefetching pass: QSV_STAGES (default 2), capped
// so the ring stays within 160 KiB.
int dbuf_stages(const PassHost &ph, int dtype) {
    static const int env = [] {
        const char *e = std::getenv("QSV_STAGES");
        return e ? std::atoi(e) : 2;
    }();
    const size_t tile = static_cast<size_t>(dtype == QSV_C64 ? 8 : 16) << ph.K;
    int s = std::max(2, std::min(4, env));
    while (s > 2 && s * tile > (160u << 10)) --s;
    return s;
}

// L2 super-pass: passes A (pair = 1) and B (pair = 2) as one kernel. Each
// CTA takes one item -- tpi consecutive tiles of one pass inside one chunk --
// from an atomic ticket; tickets run A(0 .. D-1), then per chunk m the items
// of A(m + D) followed by those of B(m). A's items store with plain
// write-back stores and signal a per-chunk counter; a B item waits for all of
// its chunk's A items and reads through L2 (cp.async.cg / ld.global.cg), so
// B finds A's output in L2 and the state crosses HBM once for both passes.
// Tickets are taken in order by running CTAs, so every A item a B item waits
// for is held by a running CTA that never waits: no deadlock, whatever else
// shares the GPU.
std::string generate_pair_source(const PassHost &A, const PassHost &B, int dtype, const std::string &name,
                                 int *threads, bool dbuf, size_t *smem) {
    Gen ga(A, dtype), gb(B, dtype);
    for (Gen *g : {&ga, &gb}) {
        g->pool = false;
        g->double_buffer = false;
        g->prefetch = dbuf;
        g->stages = dbuf_stages(g->ph, dtype);
    }
    ga.st_out = "stwb";
    gb.ld_in = "ldcg";
    const int th = ga.threads_of();
    require(th == gb.threads_of(), "codegen: super-pass halves differ in CTA shape");
    *threads = th;
    std::ostringstream k;
    k << "// generated by qsv codegen.cpp: an L2 super-pass (two tile passes, chunk by chunk)\n" << ga.common();
    k << "namespace pa {\n" << ga.body_fn("body") << "}\n";
    k << "namespace pb {\n" << gb.body_fn("body") << "}\n";
    if (smem) *smem = std::max(ga.dyn_bytes(), gb.dyn_bytes());
    k << "struct Pair { unsigned *sync; u64 nchunks; int chunk_tiles_log; int tpi; int lookahead; };\n";
    k << "extern \"C\" __global__ void __launch_bounds__(" << th << ", " << kernel_min_blocks(A, th) << ") " << name
      << "(const Args a, const Args b, const Pair q) {\n";
    k << "  extern __shared__ __align__(16) unsigned char smem_raw[];\n";
    k << "  __shared__ unsigned tk;\n";
    k << "  if (threadIdx.x == 0) tk = atomicAdd(q.sync + q.nchunks, 1u);\n";
    k << "  __syncthreads();\n";
    k << "  const u64 ipc = (1ull << q.chunk_tiles_log) / (u64)q.tpi;\n";
    k << "  const u64 m = tk / (2 * ipc), r = tk % (2 * ipc);\n";
    k << "  if (r < ipc) {\n";
    k << "    if (m >= q.nchunks) return;\n";
    k << "    const u64 t0 = (m << q.chunk_tiles_log) + r * q.tpi;\n";
    k << "    pa::body(a, t0, t0 + q.tpi, 1, smem_raw);\n";
    k << "    __syncthreads();\n";
    k << "    if (threadIdx.x == 0) { __threadfence(); atomicAdd(q.sync + m, 1u); }\n";
    k << "  } else {\n";
    k << "    if (m < (u64)q.lookahead) return;\n";
    k << "    const u64 c = m - q.lookahead;\n";
    k << "    if (c >= q.nchunks) return;\n";
    k << "    if (threadIdx.x == 0) {\n";
    k << "      unsigned v;\n";
    k << "      for (;;) {\n";
    k << "        asm volatile(\"ld.acquire.gpu.global.u32 %0, [%1];\" : \"=r\"(v) : \"l\"(q.sync + c) : \"memory\");\n";
    k << "        if ((u64)v >= ipc) break;\n";
    k << "        __nanosleep(64);\n";
    k << "      }\n";
    k << "    }\n";
    k << "    __syncthreads();\n";
    k << "    const u64 t0 = (c << q.chunk_tiles_log) + (r - ipc) * q.tpi;\n";
    k << "    pb::body(b, t0, t0 + q.tpi, 1, smem_raw);\n";
    k << "  }\n}\n";
    return k.str();
}

std::string generate_pass_source(const PassHost &ph, int dtype, const std::string &name, int *threads, bool dbuf,
                                 bool zsum, size_t *smem, bool gout) {
    Gen g(ph, dtype);
    g.zsum = zsum;
    g.gout = gout;
    // a one-GPU output permutation by scattered stores: plain write-back
    // stores, so the partial lines of neighbouring tiles merge in L2
    if (gout && ph.local_gperm) g.st_out = "stwb";
    require(!gout || !ph.gperm.empty(), "codegen: peer-memory pass without a global permutation");
    require(!gout || (!zsum && ph.out_perm.empty()), "codegen: peer-memory stores on a permuting / <Z> pass");
    g.double_buffer = false;
    g.prefetch = dbuf;
    g.stages = dbuf_stages(ph, dtype);
    *threads = g.threads_of();
    std::string src = g.source(name);
    if (smem) *smem = g.dyn_bytes();
    return src;
}

} // namespace qsv
