// Drop-in bridge: the reference's C++ qubit API (quasar::qubit, header-only,
// /root/reference/proj/include/quasar/qubit/*.hpp) routed to the qsv C ABI.
//
// A maintainer includes the quasar headers as usual, then this header, and
// calls quasar::qubit::gpu::forward / expectation / apply_gate /
// marginal_probabilities / measure / adjoint_gradients where the reference
// calls Circuit::forward (circuit.hpp:121-157), expectation
// (circuit.hpp:277-282), apply_gate (state.hpp:149-157), marginal_probabilities
// / measure (circuit.hpp:182-244) and adjoint_gradients (adjoint.hpp:52-110);
// quasar::qubit::gpu::dist mirrors the reference's distributed API
// (dist::run_on_ranks, Transport, PartitionedState, apply_gate_dist,
// run_circuit_dist, expectation_dist, probabilities_dist, measure_dist,
// adjoint_gradients_dist, gather_amplitudes -- tests/test_dist.cpp,
// tools/main.cpp:86-131) over one process driving P GPUs. Semantics and
// errors are the reference's: encode slots must match exactly, value
// semantics for states, invalid_input / guard_error / transport_error for
// status 2 / 3 / 4 (core.hpp:34-47). Nothing here computes amplitudes: all of
// it marshals through include/qsv.h.
#pragma once

#include <algorithm>
#include <barrier>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../qsv.h"
#include "quasar/qubit/adjoint.hpp"
#include "quasar/qubit/circuit.hpp"

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

// Circuit observables -> qsv_obs (views into the circuit's storage + `wires`).
inline std::vector<qsv_obs> to_obs(const std::vector<Observable> &obs, std::vector<std::vector<int32_t>> &wires) {
    std::vector<qsv_obs> qo(obs.size());
    wires.assign(obs.size(), {});
    for (size_t i = 0; i < obs.size(); ++i) {
        wires[i].assign(obs[i].wires.begin(), obs[i].wires.end());
        qo[i].nwires = static_cast<int32_t>(wires[i].size());
        qo[i].wires = wires[i].data();
        qo[i].basis = obs[i].basis.c_str();
    }
    return qo;
}

// measure()'s sampling (circuit.hpp:217-244) over device-computed marginals.
inline std::map<std::string, MeasureEntry> sample(const std::vector<double> &probs, int k, int shots, Rng &rng,
                                                  bool with_prob) {
    if (shots < 1) throw ::quasar::invalid_input("measure: shots must be >= 1");
    std::vector<double> cdf(probs.size());
    double acc = 0.0;
    for (size_t i = 0; i < probs.size(); ++i) {
        acc += probs[i];
        cdf[i] = acc;
    }
    std::map<std::string, MeasureEntry> out;
    for (int s = 0; s < shots; ++s) {
        const double u = rng.uniform() * acc;
        const size_t idx = std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin();
        out[bits_to_string(std::min(idx, probs.size() - 1), k)].count += 1;
    }
    if (with_prob)
        for (size_t i = 0; i < probs.size(); ++i) {
            if (probs[i] <= 0 && out.find(bits_to_string(i, k)) == out.end()) continue;
            out[bits_to_string(i, k)].probability = probs[i];
        }
    return out;
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

/// marginal_probabilities (circuit.hpp:182-205), pure states.
inline std::vector<double> marginal_probabilities(const QubitState &s, const std::vector<int> &wires,
                                                  std::size_t batch_index = 0) {
    if (wires.empty()) throw ::quasar::invalid_input("measure: empty wire list");
    QubitState one = QubitState::from_amplitudes(s.nqubit(), s.amplitudes(batch_index));
    auto st = detail::upload(one, 1);
    std::vector<int32_t> w(wires.begin(), wires.end());
    std::vector<double> out(std::size_t(1) << wires.size());
    detail::check(qsv_marginal_probs(st->h, 0, static_cast<int>(w.size()), w.data(), out.data()));
    return out;
}

/// measure (circuit.hpp:217-244): the marginals on the GPU, the reference's
/// seeded CDF sampling on the host (identical histograms for the same Rng).
inline std::map<std::string, MeasureEntry> measure(const QubitState &s, int shots, const std::vector<int> &wires,
                                                   Rng &rng, bool with_prob = false, std::size_t batch_index = 0) {
    if (shots < 1) throw ::quasar::invalid_input("measure: shots must be >= 1");
    return detail::sample(gpu::marginal_probabilities(s, wires, batch_index), static_cast<int>(wires.size()), shots, rng,
                          with_prob);
}

/// adjoint_gradients (adjoint.hpp:52-110): gradient of the summed
/// expectation of the circuit's observables.
inline AdjointGradients adjoint_gradients(const Circuit &cir, const QubitState &init,
                                          const std::vector<double> &data = {}) {
    if (init.is_mixed()) throw ::quasar::invalid_input("adjoint_gradients: pure states only");
    if (init.batch() != 1) throw ::quasar::invalid_input("adjoint_gradients: one batch row at a time");
    std::vector<std::vector<double>> keep;
    std::vector<qsv_gate> gs;
    int cap = 0;
    for (const Gate &g : cir.gates()) {
        gs.push_back(detail::to_qsv(g, keep));
        cap += g.num_params();
    }
    std::vector<std::vector<int32_t>> wires;
    auto qo = detail::to_obs(cir.observables(), wires);
    const uint64_t dim = uint64_t(1) << cir.nqubit();
    std::vector<double> ini(2 * dim);
    for (uint64_t i = 0; i < dim; ++i) {
        ini[2 * i] = init.amplitudes(0)(static_cast<long>(i)).real();
        ini[2 * i + 1] = init.amplitudes(0)(static_cast<long>(i)).imag();
    }
    AdjointGradients out;
    std::vector<double> pg(std::max(cap, 1)), dg(std::max<size_t>(data.size(), 1));
    int np = 0;
    detail::check(qsv_adjoint_gradients(detail::context(), cir.nqubit(), QSV_C128, gs.data(), static_cast<int>(gs.size()),
                                        static_cast<int>(qo.size()), qo.data(), ini.data(),
                                        data.empty() ? nullptr : data.data(), static_cast<int>(data.size()), pg.data(),
                                        cap, &np, dg.data()));
    out.param_grads.assign(pg.begin(), pg.begin() + np);
    out.data_grads.assign(dg.begin(), dg.begin() + static_cast<long>(data.size()));
    return out;
}

// ---------------------------------------------------------------------------
// Distributed: the reference's quasar::dist API (source absent from the
// reference; contract from tests/test_dist.cpp and tools/main.cpp:86-131) on
// one process driving P GPUs (qsv_ctx_create_multi + qsv_run_on_ranks): the
// top log2 P wires are global, every rank a host thread with its own stream
// and NCCL communicator.
// ---------------------------------------------------------------------------
namespace dist {

/// One rank's endpoint inside run_on_ranks (the reference's Transport&).
class Transport {
  public:
    Transport(qsv_ctx *ctx, int rank, int world, std::barrier<> *bar, std::vector<double> *shared)
        : ctx_(ctx), rank_(rank), world_(world), bar_(bar), shared_(shared) {}
    int rank() const { return rank_; }
    int world() const { return world_; }
    qsv_ctx *ctx() const { return ctx_; }
    void barrier() { bar_->arrive_and_wait(); }
    /// Measured counters (tests/test_dist.cpp:96-126): point-to-point sends
    /// and bytes this rank issued since the last reset.
    std::uint64_t messages_sent() const {
        std::uint64_t m = 0;
        detail::check(qsv_ctx_comm_stats(ctx_, &m, nullptr, nullptr));
        return m;
    }
    std::uint64_t bytes_sent() const {
        std::uint64_t b = 0;
        detail::check(qsv_ctx_comm_stats(ctx_, nullptr, &b, nullptr));
        return b;
    }
    void reset_counters() { detail::check(qsv_ctx_comm_reset(ctx_)); }
    std::vector<double> &shared() { return *shared_; }

  private:
    qsv_ctx *ctx_;
    int rank_, world_;
    std::barrier<> *bar_;
    std::vector<double> *shared_;
};

/// A rank's slice: 2^(n-g) amplitudes, the indices whose top g bits equal
/// the rank.
class PartitionedState {
  public:
    PartitionedState(Transport &tr, int nqubit) : tr_(&tr), n_(nqubit) {
        if (tr.world() < 1 || (tr.world() & (tr.world() - 1)))
            throw ::quasar::invalid_input("world size must be a power of two");
        qsv_state *h = nullptr;
        detail::check(qsv_state_create(tr.ctx(), nqubit, 1, QSV_C128, &h));
        st_ = std::make_shared<detail::State>(h);
    }
    int nqubit() const { return n_; }
    int global_bits() const {
        int g = 0;
        detail::check(qsv_state_info(st_->h, nullptr, nullptr, nullptr, &g, nullptr));
        return g;
    }
    cvec slice() const {
        std::uint64_t la = 0;
        detail::check(qsv_state_info(st_->h, nullptr, nullptr, nullptr, nullptr, &la));
        std::vector<double> buf(2 * la);
        detail::check(qsv_state_download(st_->h, 0, buf.data(), la));
        cvec v(static_cast<long>(la));
        for (std::uint64_t i = 0; i < la; ++i) v(static_cast<long>(i)) = cdouble(buf[2 * i], buf[2 * i + 1]);
        return v;
    }
    double global_norm2() const {
        double x = 0;
        detail::check(qsv_norm2(st_->h, &x));
        return x;
    }
    qsv_state *handle() const { return st_->h; }
    Transport &transport() const { return *tr_; }

  private:
    Transport *tr_;
    int n_;
    std::shared_ptr<detail::State> st_;
};

/// dist::run_on_ranks: fn(Transport&) on `ranks` host threads, rank r on GPU
/// r mod (device count); the first rank's exception is rethrown.
template <typename Fn> void run_on_ranks(int ranks, Fn &&fn) {
    if (ranks < 1 || (ranks & (ranks - 1))) throw ::quasar::invalid_input("world size must be a power of two");
    const int nd = std::max(1, qsv_device_count());
    std::vector<int> devs(ranks);
    for (int r = 0; r < ranks; ++r) devs[r] = r % nd;
    qsv_ctx *multi = nullptr;
    detail::check(qsv_ctx_create_multi(ranks, devs.data(), &multi));
    struct Run {
        Fn *fn;
        std::barrier<> bar;
        std::vector<double> shared;
        std::vector<std::exception_ptr> err;
        int world;
    } run{&fn, std::barrier<>(ranks), {}, std::vector<std::exception_ptr>(ranks), ranks};
    auto tramp = [](qsv_ctx *rc, int rank, void *user) -> int {
        auto *r = static_cast<Run *>(user);
        try {
            Transport tr(rc, rank, r->world, &r->bar, &r->shared);
            (*r->fn)(tr);
            return QSV_OK;
        } catch (...) {
            r->err[rank] = std::current_exception();
            return QSV_ERR_INTERNAL;
        }
    };
    const int rc = qsv_run_on_ranks(multi, tramp, &run);
    qsv_ctx_destroy(multi);
    for (auto &e : run.err)
        if (e) std::rethrow_exception(e);
    detail::check(rc);
}

/// apply_gate_dist: local and diagonal gates send nothing; a single-qubit
/// gate on a global wire is one pairwise exchange of the slice.
inline void apply_gate_dist(PartitionedState &st, const Gate &g) {
    std::vector<std::vector<double>> keep;
    qsv_gate q = detail::to_qsv(g, keep);
    detail::check(qsv_apply_gate(st.handle(), &q));
}

/// run_circuit_dist: |0...0>, the circuit fused into passes with global
/// qubits swapped in as needed; `row` binds the encode slots.
inline PartitionedState run_circuit_dist(Transport &tr, const Circuit &cir, const std::vector<double> &row = {}) {
    PartitionedState st(tr, cir.nqubit());
    std::vector<std::vector<double>> keep;
    std::vector<qsv_gate> gs;
    for (const Gate &g : cir.gates()) gs.push_back(detail::to_qsv(g, keep));
    if (static_cast<int>(row.size()) != cir.encode_slots())
        throw ::quasar::invalid_input("data length " + std::to_string(row.size()) + " != encode slots " +
                                      std::to_string(cir.encode_slots()));
    detail::check(qsv_run_circuit(st.handle(), gs.data(), static_cast<int>(gs.size()), row.empty() ? nullptr : row.data(),
                                  row.empty() ? 0 : 1, static_cast<int>(row.size()), nullptr));
    return st;
}

inline std::vector<double> expectation_dist(PartitionedState &st, const std::vector<Observable> &obs) {
    std::vector<std::vector<int32_t>> wires;
    auto qo = detail::to_obs(obs, wires);
    std::vector<double> out(obs.size());
    if (!obs.empty()) detail::check(qsv_expect_pauli(st.handle(), static_cast<int>(qo.size()), qo.data(), out.data()));
    return out;
}

inline std::vector<double> probabilities_dist(PartitionedState &st, const std::vector<int> &wires) {
    if (wires.empty()) throw ::quasar::invalid_input("measure: empty wire list");
    std::vector<int32_t> w(wires.begin(), wires.end());
    std::vector<double> out(std::size_t(1) << wires.size());
    detail::check(qsv_marginal_probs(st.handle(), 0, static_cast<int>(w.size()), w.data(), out.data()));
    return out;
}

inline std::map<std::string, MeasureEntry> measure_dist(PartitionedState &st, int shots, const std::vector<int> &wires,
                                                        Rng &rng, bool with_prob = false) {
    if (shots < 1) throw ::quasar::invalid_input("measure: shots must be >= 1");
    return detail::sample(probabilities_dist(st, wires), static_cast<int>(wires.size()), shots, rng, with_prob);
}

inline AdjointGradients adjoint_gradients_dist(Transport &tr, const Circuit &cir, const std::vector<double> &row = {}) {
    std::vector<std::vector<double>> keep;
    std::vector<qsv_gate> gs;
    int cap = 0;
    for (const Gate &g : cir.gates()) {
        gs.push_back(detail::to_qsv(g, keep));
        cap += g.num_params();
    }
    std::vector<std::vector<int32_t>> wires;
    auto qo = detail::to_obs(cir.observables(), wires);
    std::vector<double> pg(std::max(cap, 1)), dg(std::max<size_t>(row.size(), 1));
    int np = 0;
    detail::check(qsv_adjoint_gradients(tr.ctx(), cir.nqubit(), QSV_C128, gs.data(), static_cast<int>(gs.size()),
                                        static_cast<int>(qo.size()), qo.data(), nullptr,
                                        row.empty() ? nullptr : row.data(), static_cast<int>(row.size()), pg.data(),
                                        cap, &np, dg.data()));
    AdjointGradients out;
    out.param_grads.assign(pg.begin(), pg.begin() + np);
    out.data_grads.assign(dg.begin(), dg.begin() + static_cast<long>(row.size()));
    return out;
}

/// gather_amplitudes: every rank receives the whole state (collective).
inline cvec gather_amplitudes(PartitionedState &st) {
    Transport &tr = st.transport();
    const cvec mine = st.slice();
    const long per = mine.size();
    tr.barrier();
    if (tr.rank() == 0) tr.shared().assign(2 * static_cast<size_t>(per) * tr.world(), 0.0);
    tr.barrier();
    for (long i = 0; i < per; ++i) {
        tr.shared()[2 * (tr.rank() * per + i)] = mine(i).real();
        tr.shared()[2 * (tr.rank() * per + i) + 1] = mine(i).imag();
    }
    tr.barrier();
    cvec full(per * tr.world());
    for (long i = 0; i < full.size(); ++i) full(i) = cdouble(tr.shared()[2 * i], tr.shared()[2 * i + 1]);
    tr.barrier();
    return full;
}

} // namespace dist

} // namespace quasar::qubit::gpu
