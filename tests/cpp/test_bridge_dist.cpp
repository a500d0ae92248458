// The reference's distributed KATs (proj/tests/test_dist.cpp) restated over
// quasar::qubit::gpu::dist (include/qsv/quasar_bridge.hpp): one process,
// P ranks as host threads (qsv_ctx_create_multi), the reference's own
// single-rank CPU path (quasar headers, unchanged) as the oracle, as
// test_dist.cpp:59-62 does. On a one-GPU host every rank shares device 0,
// which needs the host-driven NCCL stand-in (QSV_NCCL_LIB=tests/fake_nccl).
#include <cmath>
#include <cstdio>
#include <string>

#include "quasar/qubit/adjoint.hpp"
#include "quasar/qubit/circuit.hpp"
#include "qsv/quasar_bridge.hpp"

using namespace quasar;
using namespace quasar::qubit;
namespace D = quasar::qubit::gpu::dist;

static int failures = 0, checks = 0;
#define CHECK(cond, what)                                                                                              \
    do {                                                                                                               \
        ++checks;                                                                                                      \
        if (!(cond)) {                                                                                                 \
            ++failures;                                                                                                \
            std::printf("FAIL %s (%s:%d)\n", std::string(what).c_str(), __FILE__, __LINE__);                        \
        }                                                                                                              \
    } while (0)

// tests/test_dist.cpp:28-57 gate mix, draws sequenced explicitly
static Circuit random_circuit(Rng &rng, int nq, int ngates) {
    Circuit cir(nq);
    for (int i = 0; i < ngates; ++i) {
        const double u = rng.uniform();
        const int a = static_cast<int>(rng.next_below(nq));
        int b = a;
        while (nq > 1 && b == a) b = static_cast<int>(rng.next_below(nq));
        if (u < 0.2) cir.cnot(a, b);
        else if (u < 0.3) cir.cp(a, b, rng.uniform(-kPi, kPi));
        else if (u < 0.4) cir.swap(a, b);
        else if (u < 0.5) cir.rzz(a, b, rng.uniform(-kPi, kPi));
        else if (u < 0.56) cir.rxx(a, b, rng.uniform(-kPi, kPi));
        else if (u < 0.62) cir.ryy(a, b, rng.uniform(-kPi, kPi));
        else if (u < 0.72) cir.h(a);
        else if (u < 0.82) cir.ry(a, rng.uniform(-kPi, kPi), true);
        else if (u < 0.92) cir.rz(a, rng.uniform(-kPi, kPi), true);
        else cir.cry(a, b, rng.uniform(-kPi, kPi), true);
    }
    return cir;
}

static double maxdiff(const cvec &a, const cvec &b) { return (a - b).cwiseAbs().maxCoeff(); }

int main() {
    D::run_on_ranks(4, [](D::Transport &tr) {  // Setup.SliceSizesMatchArithmetic
        D::PartitionedState st(tr, 4);
        CHECK(st.slice().size() == 4 && st.global_bits() == 2, "slice sizes");
    });
    D::run_on_ranks(4, [](D::Transport &tr) {  // Communication.LocalGatesSendNothing
        D::PartitionedState st(tr, 6);
        tr.reset_counters();
        D::apply_gate_dist(st, make_gate("h", {3}));
        D::apply_gate_dist(st, make_gate("x", {2}));
        D::apply_gate_dist(st, make_gate("rzz", {4, 5}, {}, {0.7}));
        D::apply_gate_dist(st, make_gate("rz", {0}, {}, {0.3}));
        D::apply_gate_dist(st, make_gate("p", {1}, {0}, {0.9}));
        CHECK(tr.messages_sent() == 0u && tr.bytes_sent() == 0u, "local gates send nothing");
    });
    {   // Communication.GlobalTargetDoesOnePairwiseExchange
        Circuit cir(3);
        cir.h(0);
        const cvec want = cir.forward().amplitudes();
        D::run_on_ranks(2, [&](D::Transport &tr) {
            D::PartitionedState st(tr, 3);
            tr.reset_counters();
            D::apply_gate_dist(st, make_gate("h", {0}));
            CHECK(tr.messages_sent() == 1u, "one message");
            CHECK(tr.bytes_sent() == st.slice().size() * sizeof(cdouble), "one slice of bytes");
            const cvec got = D::gather_amplitudes(st);
            if (tr.rank() == 0) CHECK(maxdiff(got, want) < 1e-12, "global h state");
        });
    }
    {   // Equivalence.RandomCircuitsAcrossWorldSizes
        Rng rng(7, "dist-equiv");
        for (int world : {2, 4, 8})
            for (int trial = 0; trial < 6; ++trial) {
                const int n = 4 + static_cast<int>(rng.next_below(5));
                if ((1 << n) < 4 * world) continue;  // two local qubits per rank
                Circuit cir = random_circuit(rng, n, 18);
                const cvec want = cir.forward().amplitudes();
                D::run_on_ranks(world, [&](D::Transport &tr) {
                    D::PartitionedState st = D::run_circuit_dist(tr, cir);
                    const cvec got = D::gather_amplitudes(st);
                    if (tr.rank() == 0)
                        CHECK(maxdiff(got, want) < 1e-12, "world " + std::to_string(world) + " trial " + std::to_string(trial));
                });
            }
    }
    {   // Equivalence.NormPreservedAcrossExchanges
        Rng rng(11, "dist-norm");
        Circuit cir = random_circuit(rng, 6, 25);
        D::run_on_ranks(4, [&](D::Transport &tr) {
            D::PartitionedState st(tr, 6);
            bool ok = true;
            for (const auto &g : cir.gates()) {
                D::apply_gate_dist(st, g);
                ok = ok && std::abs(st.global_norm2() - 1.0) < 1e-10;
            }
            CHECK(ok, "norm preserved");
        });
    }
    {   // MeasureExpectation.BellPairHistogramAndCode31Circuit
        D::run_on_ranks(2, [](D::Transport &tr) {
            D::PartitionedState st(tr, 2);
            D::apply_gate_dist(st, make_gate("h", {0}));
            D::apply_gate_dist(st, make_gate("x", {1}, {0}));
            auto probs = D::probabilities_dist(st, {0, 1});
            CHECK(std::abs(probs[0] - 0.5) < 1e-12 && std::abs(probs[3] - 0.5) < 1e-12, "bell probabilities");
            Rng rng(0, "dist-bell");
            auto counts = D::measure_dist(st, 1000, {0, 1}, rng, true);
            CHECK(counts.at("00").count + counts.at("11").count == 1000u, "bell counts");
        });
        Circuit cir(4);
        cir.rylayer(true);
        cir.cnot_ring();
        cir.observable({0}, "z");
        cir.observable({1}, "x");
        const std::vector<double> data{0.0, 1.0, 2.0, 3.0};
        const auto want = expectation(cir.forward({data}), cir);
        D::run_on_ranks(4, [&](D::Transport &tr) {
            D::PartitionedState st = D::run_circuit_dist(tr, cir, data);
            const auto got = D::expectation_dist(st, cir.observables());
            bool ok = got.size() == want.size();
            for (size_t i = 0; ok && i < want.size(); ++i) ok = std::abs(got[i] - want[i]) < 1e-12;
            CHECK(ok, "encoded expectations");
        });
    }
    {   // MeasureExpectation.HistogramMatchesSeededSingleRank
        Circuit cir(3);
        cir.h(0);
        cir.cnot(0, 1);
        cir.ry(2, 0.7);
        Rng rs(9, "hist");
        const auto want = measure(cir.forward(), 500, {0, 1, 2}, rs);
        D::run_on_ranks(2, [&](D::Transport &tr) {
            D::PartitionedState st = D::run_circuit_dist(tr, cir);
            Rng rng(9, "hist");
            const auto got = D::measure_dist(st, 500, {0, 1, 2}, rng);
            bool ok = got.size() == want.size();
            for (const auto &[k, e] : want) ok = ok && got.count(k) && got.at(k).count == e.count;
            CHECK(ok, "seeded histogram");
        });
    }
    {   // Adjoint.AnalyticAndAgainstSingleRank (the 1-qubit-on-2-ranks case is
        // refused: a state needs one local qubit per rank)
        Rng rng(13, "dist-adj");
        for (int world : {2, 4})
            for (int trial = 0; trial < 5; ++trial) {
                Circuit c = random_circuit(rng, 5, 14);
                c.observable({0}, "z");
                c.observable({2}, "x");
                const auto want = adjoint_gradients(c, QubitState::basis(5));
                D::run_on_ranks(world, [&](D::Transport &tr) {
                    const auto got = D::adjoint_gradients_dist(tr, c);
                    bool ok = got.param_grads.size() == want.param_grads.size();
                    for (size_t i = 0; ok && i < want.param_grads.size(); ++i)
                        ok = std::abs(got.param_grads[i] - want.param_grads[i]) < 1e-10;
                    if (tr.rank() == 0) CHECK(ok, "adjoint " + std::to_string(world) + ":" + std::to_string(trial));
                });
            }
    }
    {   // run_on_ranks rethrows a rank's exception
        bool threw = false;
        try {
            D::run_on_ranks(2, [](D::Transport &tr) {
                if (tr.rank() == 1) throw invalid_input("rank one");
            });
        } catch (const invalid_input &) {
            threw = true;
        }
        CHECK(threw, "exception propagates");
    }
    std::printf("%d/%d checks passed\n", checks - failures, checks);
    return failures ? 1 : 0;
}
