// Drop-in bridge: the reference's C++ qubit API (quasar::qubit, header-only,
// /root/reference/proj/include/quasar/qubit/*.hpp) routed to the qsv C ABI.
//
// A maintainer includes the quasar headers as usual, then this header, and
// calls quasar::qubit::gpu::forward / expectation / apply_gate where the
// reference calls Circuit::forward (circuit.hpp:121-157), expectation
// (circuit.hpp:277-282) and apply_gate (state.hpp:149-157). Semantics and
// errors are the reference's: encode slots must match exactly, value
// semantics for states, invalid_input / guard_error / transport_error for
// status 2 / 3 / 4 (core.hpp:34-47). Nothing here computes amplitudes: all of
// it marshals through include/qsv.h.
#pragma once

#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../qsv.h"

namespace quasar::qubit::gpu {

namespace detail {

inline void check(int rc) {
    if (rc == QSV_OK) return;
    const std::string msg = qsv_last_error();
    if (rc == QSV_ERR_INVALID) throw ::quasar::invalid_input(msg);
    if (rc == QSV_ERR_GUARD) throw ::quasar::guard_error(msg);
    if (rc == QSV_ERR_TRANSPORT) throw ::quasar::transport_error(msg);
    throw std::runtime_error("qsv: " + msg);
}

struct Ctx {
    qsv_ctx *h = nullptr;
    Ctx() { check(qsv_ctx_create(0, &h)); }
    ~Ctx() { qsv_ctx_destroy(h); }
};
inline qsv_ctx *context() {
    static Ctx c; // one stream on device 0 (one process per GPU)
    return c.h;
}

struct State {
    qsv_state *h = nullptr;
    explicit State(qsv_state *s) : h(s) {}
    ~State() { qsv_state_destroy(h); }
};

// quasar::qubit::Gate (gate.hpp:28-38) -> qsv_gate; `keep` owns custom matrices.
inline qsv_gate to_qsv(const Gate &g, std::vector<std::vector<double>> &keep) {
    if (g.wires.size() > 2 || g.controls.size() > 6 || g.params.size() > 3)
        throw ::quasar::invalid_input("gate " + g.name + ": outside the supported shape (<= 2 targets)");
    qsv_gate q{};
    std::strncpy(q.name, g.name.c_str(), sizeof(q.name) - 1);
    q.nwires = static_cast<int32_t>(g.wires.size());
    for (size_t i = 0; i < g.wires.size(); ++i) q.wires[i] = g.wires[i];
    q.ncontrols = static_cast<int32_t>(g.controls.size());
    for (size_t i = 0; i < g.controls.size(); ++i) q.controls[i] = g.controls[i];
    q.nparams = static_cast<int32_t>(g.params.size());
    for (size_t i = 0; i < g.params.size(); ++i) q.params[i] = g.params[i];
    q.trainable = g.trainable;
    q.encode = g.encode;
    if (g.custom) {
        const auto &m = *g.custom;
        std::vector<double> buf(2 * m.rows() * m.cols());
        for (long r = 0; r < m.rows(); ++r)
            for (long c = 0; c < m.cols(); ++c) {
                buf[2 * (r * m.cols() + c)] = m(r, c).real();
                buf[2 * (r * m.cols() + c) + 1] = m(r, c).imag();
            }
        keep.push_back(std::move(buf));
        q.custom = keep.back().data();
    }
    return q;
}

inline std::unique_ptr<State> upload(const QubitState &s, int batch_rows) {
    if (s.is_mixed()) throw ::quasar::invalid_input("qsv: pure states only");
    qsv_state *h = nullptr;
    check(qsv_state_create(context(), s.nqubit(), batch_rows, QSV_C128, &h));
    auto st = std::make_unique<State>(h);
    const uint64_t dim = uint64_t(1) << s.nqubit();
    std::vector<double> buf(2 * dim);
    for (int b = 0; b < batch_rows; ++b) {
        const cvec &v = s.amplitudes(s.batch() == 1 ? 0 : b);
        for (uint64_t i = 0; i < dim; ++i) {
            buf[2 * i] = v(static_cast<long>(i)).real();
            buf[2 * i + 1] = v(static_cast<long>(i)).imag();
        }
        check(qsv_state_upload(h, b, buf.data(), dim));
    }
    return st;
}

inline QubitState download(State &st, int n, int rows) {
    const uint64_t dim = uint64_t(1) << n;
    std::vector<double> buf(2 * dim);
    std::vector<cvec> out;
    for (int b = 0; b < rows; ++b) {
        check(qsv_state_download(st.h, b, buf.data(), dim));
        cvec v(static_cast<long>(dim));
        for (uint64_t i = 0; i < dim; ++i) v(static_cast<long>(i)) = cdouble(buf[2 * i], buf[2 * i + 1]);
        out.push_back(std::move(v));
    }
    QubitState s = QubitState::basis(n);
    s.set_batch_pure(std::move(out));
    return s;
}

} // namespace detail

/// Circuit::forward (circuit.hpp:121-157) on the GPU.
inline QubitState forward(const Circuit &cir, const QubitState &init,
                          const std::vector<std::vector<double>> &data = {}) {
    const int n = cir.nqubit();
    const int slots = cir.encode_slots();
    std::vector<std::vector<double>> keep;
    std::vector<qsv_gate> gs;
    for (const Gate &g : cir.gates()) gs.push_back(detail::to_qsv(g, keep));
    if (data.empty()) {
        if (slots != 0) throw ::quasar::invalid_input("circuit has encode slots but no data given");
        auto st = detail::upload(init, static_cast<int>(init.batch()));
        detail::check(qsv_run_circuit(st->h, gs.data(), static_cast<int>(gs.size()), nullptr, 0, 0, nullptr));
        return detail::download(*st, n, static_cast<int>(init.batch()));
    }
    if (init.batch() != 1) throw ::quasar::invalid_input("encoded runs broadcast a single initial state");
    std::vector<double> flat;
    for (const auto &row : data) {
        if (static_cast<int>(row.size()) != slots)
            throw ::quasar::invalid_input("data length " + std::to_string(row.size()) + " != encode slots " +
                                          std::to_string(slots));
        flat.insert(flat.end(), row.begin(), row.end());
    }
    const int rows = static_cast<int>(data.size());
    auto st = detail::upload(init, rows);
    detail::check(qsv_run_circuit(st->h, gs.data(), static_cast<int>(gs.size()), flat.data(), rows, slots, nullptr));
    return detail::download(*st, n, rows);
}

inline QubitState forward(const Circuit &cir, const std::vector<std::vector<double>> &data = {}) {
    return forward(cir, QubitState::basis(cir.nqubit()), data);
}

/// apply_gate (state.hpp:149-157): value semantics, every batch row.
inline QubitState apply_gate(const QubitState &s, const Gate &g) {
    std::vector<std::vector<double>> keep;
    qsv_gate q = detail::to_qsv(g, keep);
    auto st = detail::upload(s, static_cast<int>(s.batch()));
    detail::check(qsv_apply_gate(st->h, &q));
    return detail::download(*st, s.nqubit(), static_cast<int>(s.batch()));
}

/// expectation (circuit.hpp:277-282): one value per registered observable.
inline std::vector<double> expectation(const QubitState &s, const Circuit &cir, std::size_t batch_index = 0) {
    QubitState one = QubitState::from_amplitudes(s.nqubit(), s.amplitudes(batch_index));
    auto st = detail::upload(one, 1);
    const auto &obs = cir.observables();
    std::vector<qsv_obs> qo(obs.size());
    std::vector<std::vector<int32_t>> wires(obs.size());
    for (size_t i = 0; i < obs.size(); ++i) {
        wires[i].assign(obs[i].wires.begin(), obs[i].wires.end());
        qo[i].nwires = static_cast<int32_t>(wires[i].size());
        qo[i].wires = wires[i].data();
        qo[i].basis = obs[i].basis.c_str();
    }
    std::vector<double> out(obs.size());
    if (!obs.empty()) detail::check(qsv_expect_pauli(st->h, static_cast<int>(qo.size()), qo.data(), out.data()));
    return out;
}

} // namespace quasar::qubit::gpu
