// The reference's C++ API, unchanged, with Circuit::forward / apply_gate /
// expectation routed to the GPU through include/qsv/quasar_bridge.hpp.
// Each check mirrors a known-answer test of proj/tests/test_qubit.cpp and
// compares the GPU result with the reference's own CPU result.
#include <cmath>
#include <cstdio>
#include <string>

#include "quasar/qubit/adjoint.hpp"
#include "quasar/qubit/circuit.hpp"
#include "qsv/quasar_bridge.hpp"

using namespace quasar;
using namespace quasar::qubit;

static int failures = 0, checks = 0;
#define CHECK(cond, what)                                                                                              \
    do {                                                                                                               \
        ++checks;                                                                                                      \
        if (!(cond)) {                                                                                                 \
            ++failures;                                                                                                \
            std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__);                                              \
        }                                                                                                              \
    } while (0)

static double maxdiff(const cvec &a, const cvec &b) { return (a - b).cwiseAbs().maxCoeff(); }

// A seeded gate mix in the spirit of test_qubit.cpp's random gates (1- and
// 2-qubit, parameterised, 30% controlled), draws sequenced explicitly.
static Gate seeded_gate(Rng &rng, int n) {
    static const char *one[] = {"x", "y", "z", "h", "s", "t", "rx", "ry", "rz", "u3"};
    static const char *two[] = {"swap", "rxx", "ryy", "rzz"};
    if (n >= 2 && rng.uniform() < 0.4) {
        const std::string name = two[rng.next_below(4)];
        const int a = static_cast<int>(rng.next_below(n));
        int b = static_cast<int>(rng.next_below(n));
        while (b == a) b = static_cast<int>(rng.next_below(n));
        std::vector<double> p;
        if (name != "swap") p.push_back(rng.uniform(-kPi, kPi));
        return make_gate(name, {a, b}, {}, p);
    }
    const std::string name = one[rng.next_below(10)];
    const int w = static_cast<int>(rng.next_below(n));
    std::vector<double> p;
    if (name == "rx" || name == "ry" || name == "rz") p.push_back(rng.uniform(-kPi, kPi));
    if (name == "u3")
        for (int i = 0; i < 3; ++i) p.push_back(rng.uniform(-kPi, kPi));
    std::vector<int> ctl;
    if (n >= 2 && rng.uniform() < 0.3) {
        const int c = static_cast<int>(rng.next_below(n));
        if (c != w) ctl.push_back(c);
    }
    return make_gate(name, {w}, ctl, p);
}

int main() {
    {   // HadamardOnZero
        QubitState s = gpu::apply_gate(QubitState::basis(1), make_gate("h", {0}));
        CHECK(std::abs(s.amplitudes()(0) - cdouble(1 / std::sqrt(2.0), 0)) < 1e-12, "HadamardOnZero");
    }
    {   // ToffoliLike
        QubitState s = gpu::apply_gate(QubitState::basis(3, 0b110), make_gate("x", {2}, {0, 1}));
        CHECK(std::abs(std::abs(s.amplitudes()(0b111)) - 1.0) < 1e-12, "ToffoliLike");
    }
    {   // gate-by-gate against the reference apply_gate, n = 1..8
        Rng rng(31, "bridge");
        for (int n = 1; n <= 8; ++n) {
            QubitState ref = QubitState::basis(n), gpu_s = QubitState::basis(n);
            for (int rep = 0; rep < 25; ++rep) {
                Gate g = seeded_gate(rng, n);
                ref = apply_gate(ref, g);
                gpu_s = gpu::apply_gate(gpu_s, g);
            }
            CHECK(maxdiff(ref.amplitudes(), gpu_s.amplitudes()) < 1e-12, ("striding n=" + std::to_string(n)).c_str());
        }
    }
    {   // EncodingCircuit with data rows (test_qubit.cpp:145-193)
        Circuit cir(3);
        cir.h(0);
        cir.cnot(0, 1);
        cir.x(2, {0});
        cir.rylayer(true);
        cir.cnot_ring();
        cir.rylayer(false);
        cir.observable({0, 1, 2}, "xzx");
        const std::vector<std::vector<double>> data{{1.0, 2.0, 3.0}, {0.1, -0.4, 2.2}};
        QubitState want = cir.forward(data), got = gpu::forward(cir, data);
        CHECK(got.batch() == 2, "batch rows");
        for (size_t b = 0; b < 2; ++b) CHECK(maxdiff(want.amplitudes(b), got.amplitudes(b)) < 1e-12, "encoded rows");
        const auto ew = expectation(want, cir), eg = gpu::expectation(got, cir);
        CHECK(std::abs(ew[0] - eg[0]) < 1e-12, "xzx expectation");
        bool threw = false;
        try {
            gpu::forward(cir, {{0.1, 0.2}});
        } catch (const invalid_input &) {
            threw = true;
        }
        CHECK(threw, "DataLengthMismatchFailsFast");
    }
    {   // GHZ expectations (test_qubit.cpp:262-270)
        Circuit cir(3);
        cir.h(0);
        cir.cnot(0, 1);
        cir.cnot(1, 2);
        cir.observable({0, 1, 2}, "zzz");
        cir.observable({0, 1, 2}, "xxx");
        const auto e = gpu::expectation(gpu::forward(cir), cir);
        CHECK(std::abs(e[0]) < 1e-12 && std::abs(e[1] - 1.0) < 1e-12, "Ghz3");
    }
    {   // QFT (circuit.hpp:167-178) at 14 qubits against the reference
        Circuit q = qft_circuit(14);
        Rng rng(5, "bridge-qft");
        for (int i = 0; i < 7; ++i) q.swap(i, 13 - i);
        QubitState init = QubitState::basis(14, 12345);
        CHECK(maxdiff(q.forward(init).amplitudes(), gpu::forward(q, init).amplitudes()) < 1e-12, "qft14");
    }
    {   // measure: seeded histograms equal to the reference's (circuit.hpp:217-244)
        Circuit cir(3);
        cir.h(0);
        cir.cnot(0, 1);
        cir.ry(2, 0.7);
        QubitState s = cir.forward();
        Rng r1(9, "hist"), r2(9, "hist");
        const auto want = measure(s, 500, {0, 1, 2}, r1, true);
        const auto got = gpu::measure(gpu::forward(cir), 500, {0, 1, 2}, r2, true);
        bool same = want.size() == got.size();
        for (const auto &[k, e] : want)
            same = same && got.count(k) && got.at(k).count == e.count &&
                   std::abs(got.at(k).probability - e.probability) < 1e-12;
        CHECK(same, "measure histogram");
        const auto pw = marginal_probabilities(s, {2, 0}), pg = gpu::marginal_probabilities(s, {2, 0});
        double d = 0;
        for (size_t i = 0; i < pw.size(); ++i) d = std::max(d, std::abs(pw[i] - pg[i]));
        CHECK(d < 1e-12, "marginal_probabilities");
    }
    {   // adjoint_gradients (adjoint.hpp:52-110), trainable + encoded
        Circuit cir(4);
        cir.rylayer(true);
        cir.cnot_ring();
        cir.rx(1, 0.3, true);
        cir.cry(2, 3, 1.1, true);
        cir.add(make_gate("u3", {0}, {}, {0.2, 0.4, 0.6}, true));
        cir.observable({0}, "z");
        cir.observable({1, 3}, "xy");
        const std::vector<double> data{0.1, 0.5, -0.9, 2.0};
        const auto want = adjoint_gradients(cir, QubitState::basis(4), data);
        const auto got = gpu::adjoint_gradients(cir, QubitState::basis(4), data);
        double d = 0;
        bool shape = want.param_grads.size() == got.param_grads.size() && want.data_grads.size() == got.data_grads.size();
        for (size_t i = 0; shape && i < want.param_grads.size(); ++i)
            d = std::max(d, std::abs(want.param_grads[i] - got.param_grads[i]));
        for (size_t i = 0; shape && i < want.data_grads.size(); ++i)
            d = std::max(d, std::abs(want.data_grads[i] - got.data_grads[i]));
        CHECK(shape && d < 1e-10, "adjoint_gradients");
    }
    std::printf("%d/%d checks passed\n", checks - failures, checks);
    return failures ? 1 : 0;
}
