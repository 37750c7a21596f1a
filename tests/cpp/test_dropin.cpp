// Drop-in check of the reference's C++ surface on the device path: the same
// calls a reference user makes (proj/include/simdiag/{hamiltonian,
// diagonalize,statevector,evolve}.hpp), written like the reference's own
// tests (proj/tests/*.cpp) but with plain asserts (doctest is not vendored).
//   test_dropin <hamiltonian.txt> <neel|plus> <dt> <steps> <out.raw>
// evolves the state and writes it with StateVector::save_raw, plus side
// outputs (out.raw.<what>) of the rest of the reference surface:
//   .loop      evolve_grouped called n_steps times with n_steps = 1 (plan cache)
//   .baseline  evolve_baseline(Hamiltonian) from the same start
//   .gbase     evolve_baseline(span<CommutingGroup>) (group-major order)
//   .gates     apply_single_qubit / apply_two_qubit / apply_pauli_rotation
//              sequence on |0...0>
//   .exact     exact_evolve(h, start, dt*steps)
//   .expect    expectation(h, evolved state) and its imaginary residue (text)
// The Python test compares each with the reference compiled from its sources
// (exact_evolve: with a dense scipy expm, the reference's own needs Eigen).
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <stdexcept>
#include <string>

#include "simdiag/diagonalize.hpp"
#include "simdiag/evolve.hpp"
#include "simdiag/hamiltonian.hpp"
#include "simdiag/statevector.hpp"

#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::fprintf(stderr, "CHECK failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__); \
            std::exit(1);                                                        \
        }                                                                        \
    } while (0)

template <typename E, typename F>
bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main(int argc, char** argv) {
    if (argc != 6) {
        std::fprintf(stderr, "usage: test_dropin H.txt neel|plus dt steps out.raw\n");
        return 2;
    }
    std::ifstream hin(argv[1]);
    const simdiag::Hamiltonian h = simdiag::Hamiltonian::load(hin);
    const int n = h.n_qubits();
    std::vector<simdiag::DiagonalGroup> groups;
    for (const auto& g : simdiag::greedy_partition(h)) groups.push_back(simdiag::diagonalize_group(g));

    // exception contract of the reference (statevector.cpp:96-98, 180-185)
    {
        simdiag::StateVector t(4);
        CHECK(throws<std::out_of_range>([&] { t.apply_hadamard(4); }));
        CHECK(throws<std::invalid_argument>([&] { t.apply_batched_cnot(1, 0); }));
        CHECK(throws<std::invalid_argument>([&] {
            simdiag::EvolutionPlan p;
            p.n_steps = -1;
            p.validate();
        }));
        t.apply_hadamard(0);
        CHECK(std::abs(t[1].real() - 0.7071067811865476) < 1e-15);
        CHECK(t.stats().kernel_calls == 1);
    }

    simdiag::StateVector psi = std::string(argv[2]) == "plus" ? simdiag::StateVector::plus_state(n)
                                                               : simdiag::StateVector(n);
    if (std::string(argv[2]) == "neel") {
        std::uint64_t idx = 0;
        for (int q = 1; q < n; q += 2) idx |= std::uint64_t(1) << q;
        psi[0] = 0.0;
        psi[idx] = 1.0;
    }
    const std::string base = argv[5];
    auto save = [&](const simdiag::StateVector& v, const std::string& suffix) {
        std::ofstream out(base + suffix, std::ios::binary);
        v.save_raw(out);
    };
    auto start = [&]() {
        simdiag::StateVector v = std::string(argv[2]) == "plus" ? simdiag::StateVector::plus_state(n)
                                                                 : simdiag::StateVector(n);
        if (std::string(argv[2]) == "neel") {
            std::uint64_t idx = 0;
            for (int q = 1; q < n; q += 2) idx |= std::uint64_t(1) << q;
            v[0] = 0.0;
            v[idx] = 1.0;
        }
        return v;
    };
    simdiag::EvolutionPlan plan;
    CHECK(plan.method == simdiag::Method::baseline);  // the reference's default (evolve.hpp:18)
    plan.n_steps = std::atoi(argv[4]);
    const double dt = std::atof(argv[3]);
    plan.total_time = dt * plan.n_steps;
    simdiag::evolve_grouped(groups, psi, plan);
    CHECK(std::abs(simdiag::norm(psi) - 1.0) < 1e-12);
    save(psi, "");

    // step-and-measure loop: one evolve_grouped call per step
    {
        simdiag::StateVector v = start();
        simdiag::EvolutionPlan one;
        one.n_steps = 1;
        one.total_time = dt;
        double e_prev = 0.0;
        for (int k = 0; k < plan.n_steps; ++k) {
            simdiag::evolve_grouped(groups, v, one);
            e_prev = simdiag::expectation(h, v);
        }
        (void)e_prev;
        save(v, ".loop");
    }
    {
        simdiag::StateVector v = start();
        simdiag::evolve_baseline(h, v, plan);
        save(v, ".baseline");
    }
    {
        simdiag::StateVector v = start();
        const auto parts = simdiag::greedy_partition(h);
        simdiag::evolve_baseline(std::span<const simdiag::CommutingGroup>(parts), v, plan);
        save(v, ".gbase");
    }
    {
        simdiag::StateVector v(n);
        const double c = std::cos(0.3), s = std::sin(0.3);
        const simdiag::Mat2 ry{simdiag::Amplitude(c, 0), simdiag::Amplitude(-s, 0), simdiag::Amplitude(s, 0),
                               simdiag::Amplitude(c, 0)};
        const simdiag::Mat2 ph{simdiag::Amplitude(1, 0), 0.0, 0.0, std::polar(1.0, 0.7)};
        for (int q = 0; q < n; ++q) v.apply_single_qubit(q % 2 ? ry : ph, q);
        for (int q = 0; q < n; ++q) v.apply_single_qubit(ry, q);
        simdiag::Mat4 u{};  // CNOT(q1 -> q2) then a phase on |11>
        u[0] = 1.0;
        u[5] = 1.0;
        u[11] = std::polar(1.0, 0.4);
        u[14] = 1.0;
        for (int q = 0; q + 1 < n; q += 2) v.apply_two_qubit(u, q, q + 1);
        v.apply_two_qubit(u, n - 1, 0);
        for (const auto& t : h.terms()) v.apply_pauli_rotation(t, 0.37);
        CHECK(throws<std::invalid_argument>([&] {
            simdiag::Mat2 bad{simdiag::Amplitude(1, 0), simdiag::Amplitude(1, 0), 0.0, simdiag::Amplitude(1, 0)};
            v.apply_single_qubit(bad, 0);
        }));
        CHECK(throws<std::invalid_argument>([&] { v.apply_two_qubit(u, 1, 1); }));
        CHECK(throws<std::out_of_range>([&] { v.apply_single_qubit(ry, n); }));
        save(v, ".gates");
    }
    if (n <= simdiag::kExactEvolveMaxQubits) {
        const simdiag::StateVector v = start();
        save(simdiag::exact_evolve(h, v, dt * plan.n_steps), ".exact");
    }
    CHECK(throws<std::invalid_argument>([&] {
        simdiag::StateVector big(simdiag::kExactEvolveMaxQubits + 1);
        simdiag::Hamiltonian hb = simdiag::Hamiltonian::from_terms(
            simdiag::kExactEvolveMaxQubits + 1,
            {simdiag::WeightedTerm{1.0, simdiag::PauliString::parse(std::string(simdiag::kExactEvolveMaxQubits + 1, 'Z'))}});
        (void)simdiag::exact_evolve(hb, big, 0.1);
    }));
    {
        double im = -1.0;
        const double e = simdiag::expectation(h, psi, &im);
        std::ofstream out(base + ".expect");
        out.precision(17);
        out << e << " " << im << "\n";
    }
    std::printf("ok n=%d groups=%zu\n", n, groups.size());
    return 0;
}
