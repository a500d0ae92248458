// Dense-block fusion for the tensor-core path (complex64, opt-in
// qsv_opts.dense_blocks): the host half. North_star (2): "a gate-fusion pass
// that packs runs of gates on k <= 5 local qubits into one dense 2^k x 2^k
// block ... using tensor cores only if the fused block is a real dense
// contraction". The blocks replace the reference's per-gate strided loop
// (state.hpp:127-142) by one 32 x 32 product per set of 32 amplitudes; the
// kernels are in block_pass.cu.
#include <algorithm>
#include <bit>
#include <cstring>

#include "qsv_internal.hpp"

namespace qsv {

namespace {

// The gate as a 2^m x 2^m matrix on the block's qubits q (bit i of the block
// index <-> q[i]); targets index the gate matrix MSB first (gate.hpp:30).
std::vector<cplx> embed(const GateRec &g, const std::vector<int> &q) {
    const int m = static_cast<int>(q.size()), d = 1 << m;
    auto pos = [&](int bit) {
        for (int i = 0; i < m; ++i)
            if (q[i] == bit) return i;
        fail(QSV_ERR_INTERNAL, "dense: gate qubit outside its block");
    };
    std::vector<cplx> e(static_cast<size_t>(d) * d, cplx(0, 0));
    int tp[2] = {0, 0};
    for (int t = 0; t < g.k; ++t) tp[t] = pos(g.wires[t]);
    int cmask = 0;
    for (int c : g.ctls) cmask |= 1 << pos(c);
    const int gd = 1 << g.k;
    for (int x = 0; x < d; ++x) {
        if ((x & cmask) != cmask) {
            e[static_cast<size_t>(x) * d + x] = 1;
            continue;
        }
        int a = 0;
        for (int t = 0; t < g.k; ++t) a = (a << 1) | ((x >> tp[t]) & 1);
        for (int r = 0; r < gd; ++r) {
            int y = x;
            for (int t = 0; t < g.k; ++t) {
                const int bit = (r >> (g.k - 1 - t)) & 1;
                y = (y & ~(1 << tp[t])) | (bit << tp[t]);
            }
            e[static_cast<size_t>(y) * d + x] += g.m[r * gd + a];
        }
    }
    return e;
}

std::vector<cplx> matmul(const std::vector<cplx> &a, const std::vector<cplx> &b, int d) {
    std::vector<cplx> c(static_cast<size_t>(d) * d, cplx(0, 0));
    for (int i = 0; i < d; ++i)
        for (int k = 0; k < d; ++k) {
            const cplx x = a[static_cast<size_t>(i) * d + k];
            if (x == cplx(0, 0)) continue;
            for (int j = 0; j < d; ++j) c[static_cast<size_t>(i) * d + j] += x * b[static_cast<size_t>(k) * d + j];
        }
    return c;
}

// U (2^m) -> U (x) I on `extra` more qubits (appended as the high block bits)
std::vector<cplx> widen(const std::vector<cplx> &u, int m, int extra) {
    const int d = 1 << m, D = d << extra;
    std::vector<cplx> w(static_cast<size_t>(D) * D, cplx(0, 0));
    for (int y = 0; y < D; ++y)
        for (int x = 0; x < D; ++x)
            if ((y >> m) == (x >> m)) w[static_cast<size_t>(y) * D + x] = u[static_cast<size_t>(y & (d - 1)) * d + (x & (d - 1))];
    return w;
}

uint64_t gate_mask(const GateRec &g) {
    uint64_t m = 0;
    for (int t = 0; t < g.k; ++t) m |= 1ull << g.wires[t];
    for (int c : g.ctls) m |= 1ull << c;
    return m;
}

// tf32 as cvt.rna.tf32.f32 (round to nearest, ties away: on the magnitude)
float tf32_hi(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    u = (u + 0x1000u) & ~0x1fffu;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
}

} // namespace

void plan_dense(const std::vector<GateRec> &gates, int nlocal, std::vector<DenseBlock> &blocks,
                std::vector<DensePass> &passes) {
    require(nlocal >= kDenseTile, "dense blocks: need at least 12 qubits");
    for (const GateRec &g : gates) {
        require(!g.encoded, "dense blocks: encoded gates are not supported (use the default passes)");
        require(g.flags == 0, "dense blocks: zero_off_control is not supported");
        require(static_cast<int>(g.ctls.size()) + g.k <= kDenseQ, "dense blocks: a gate spans more than 5 qubits");
    }
    // ---- fusion: greedy, in gate order ----
    std::vector<int> rem(gates.size());
    for (size_t i = 0; i < rem.size(); ++i) rem[i] = static_cast<int>(i);
    while (!rem.empty()) {
        std::vector<int> q;
        std::vector<cplx> u(1, cplx(1, 0));
        uint64_t qm = 0, blocked = 0;
        std::vector<int> skipped;
        int ng = 0, nd = 0;
        for (int gi : rem) {
            const GateRec &g = gates[gi];
            const uint64_t gm = gate_mask(g);
            if ((gm & blocked) || std::popcount(qm | gm) > kDenseQ) {
                blocked |= gm;
                skipped.push_back(gi);
                continue;
            }
            const uint64_t add = gm & ~qm;
            if (add) {
                const int m = static_cast<int>(q.size());
                for (int b = 0; b < 64; ++b)
                    if ((add >> b) & 1) q.push_back(b);
                u = widen(u, m, static_cast<int>(q.size()) - m);
                qm |= add;
            }
            u = matmul(embed(g, q), u, 1 << q.size());
            ++ng;
            nd += !g.diag && std::popcount(gm) >= 2;
        }
        // pad to exactly 5 qubits with the lowest free bits
        const int m = static_cast<int>(q.size());
        for (int b = 0; static_cast<int>(q.size()) < kDenseQ && b < nlocal; ++b)
            if (!((qm >> b) & 1)) q.push_back(b), qm |= 1ull << b;
        u = widen(u, m, kDenseQ - m);
        DenseBlock blk;
        for (int i = 0; i < kDenseQ; ++i) blk.q[i] = q[i];
        blk.u = std::move(u);
        blk.ngates = ng;
        blk.ndense = nd;
        blocks.push_back(std::move(blk));
        rem.swap(skipped);
    }
    // ---- passes: a 12-bit tile (4 low bits always in it), blocks in order ----
    std::vector<int> pend(blocks.size());
    for (size_t i = 0; i < pend.size(); ++i) pend[i] = static_cast<int>(i);
    const uint64_t low = 0xFull;
    while (!pend.empty()) {
        uint64_t tile = low, blockedq = 0;
        std::vector<int> chosen, rest;
        for (int bi : pend) {
            uint64_t bm = 0;
            for (int i = 0; i < kDenseQ; ++i) bm |= 1ull << blocks[bi].q[i];
            if (static_cast<int>(chosen.size()) < kDenseMaxBlocks && !(bm & blockedq) &&
                std::popcount(tile | bm) <= kDenseTile) {
                chosen.push_back(bi);
                tile |= bm;
            } else {
                blockedq |= bm;
                rest.push_back(bi);
            }
        }
        for (int b = 0; std::popcount(tile) < kDenseTile && b < nlocal; ++b) tile |= 1ull << b;
        DensePass dp;
        int k = 0;
        for (int b = 0; b < nlocal; ++b) {
            if ((tile >> b) & 1) dp.tile_pos[k++] = b;
            else dp.ext_pos.push_back(b);
        }
        dp.blocks = chosen;
        for (size_t j = 0; j < chosen.size(); ++j)
            for (int i = 0; i < kDenseQ; ++i)
                for (int t = 0; t < kDenseTile; ++t)
                    if (dp.tile_pos[t] == blocks[chosen[j]].q[i]) dp.bbit[j][i] = t;
        // shared-tile swizzle: for every block, the four lowest set bits a
        // half-warp walks must reach 16 distinct 8-byte slots (conflict-free
        // LDS.64 / STS.64); masks over tile bits 4..11 only (invertible)
        std::vector<std::vector<int>> pats;
        for (size_t j = 0; j < chosen.size(); ++j) {
            std::vector<int> nbits;
            for (int t = 0; t < kDenseTile && nbits.size() < 4; ++t) {
                bool in = false;
                for (int i = 0; i < kDenseQ; ++i) in = in || dp.bbit[j][i] == t;
                if (!in) nbits.push_back(t);
            }
            pats.push_back(nbits);
        }
        auto vec = [&](const int m[4], int bit) {
            if (bit < 4) return 1 << bit;
            int v = 0;
            for (int i = 0; i < 4; ++i) v |= ((m[i] >> bit) & 1) << i;
            return v;
        };
        auto ok = [&](const int m[4], const std::vector<int> &b) {
            int basis[4] = {0, 0, 0, 0};  // GF(2) rank of the four vectors == 4
            int rank = 0;
            for (int bit : b) {
                int v = vec(m, bit);
                for (int i = 3; i >= 0; --i)
                    if ((v >> i) & 1) {
                        if (!basis[i]) {
                            basis[i] = v;
                            ++rank;
                            break;
                        }
                        v ^= basis[i];
                    }
            }
            return rank == 4;
        };
        int best[4] = {0, 0, 0, 0}, bs = -1;
        uint64_t x = 0x9e3779b97f4a7c15ull;
        for (int it = 0; it < 6000 && bs < static_cast<int>(pats.size()); ++it) {
            int m[4];
            for (int i = 0; i < 4; ++i) {
                x ^= x << 13, x ^= x >> 7, x ^= x << 17;
                m[i] = it == 0 ? 0 : static_cast<int>(x) & 0xFF0;
            }
            int sc = 0;
            for (const auto &p : pats) sc += ok(m, p);
            if (sc > bs) bs = sc, std::copy(m, m + 4, best);
        }
        std::copy(best, best + 4, dp.swm);
        passes.push_back(std::move(dp));
        pend.swap(rest);
    }
}

void dense_b_operand(const DenseBlock &b, std::vector<float> &out) {
    // B[n][k]: n = output real index 2i + a, k = input real index 2j + c
    constexpr int N = 64, K = 64;
    std::vector<float> B(N * K);
    for (int i = 0; i < 32; ++i)
        for (int j = 0; j < 32; ++j) {
            const cplx v = b.u[static_cast<size_t>(i) * 32 + j];
            const float re = static_cast<float>(v.real()), im = static_cast<float>(v.imag());
            B[(2 * i) * K + 2 * j] = re;
            B[(2 * i) * K + 2 * j + 1] = -im;
            B[(2 * i + 1) * K + 2 * j] = im;
            B[(2 * i + 1) * K + 2 * j + 1] = re;
        }
    // K-major, 128-byte swizzle: 16-byte chunk c of row r at chunk c ^ (r & 7)
    // within its 8-row x 128-byte atom; K = 64 floats = two atom columns
    out.assign(2 * N * K, 0.0f);  // hi image, then lo image (16 KiB each)
    for (int n = 0; n < N; ++n)
        for (int c = 0; c < K / 4; ++c) {
            const int off = ((c >> 3) * (N / 8) * 1024 + (n >> 3) * 1024 + (n & 7) * 128 + (((c & 7) ^ (n & 7)) << 4)) / 4;
            for (int e = 0; e < 4; ++e) {
                const float v = B[n * K + 4 * c + e];
                const float h = tf32_hi(v);
                out[off + e] = h;
                out[N * K + off + e] = v - h;
            }
        }
}

} // namespace qsv
