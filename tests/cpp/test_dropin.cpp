// Drop-in check of the reference's C++ surface on the device path: the same
// calls a reference user makes (proj/include/simdiag/{hamiltonian,
// diagonalize,statevector,evolve}.hpp), written like the reference's own
// tests (proj/tests/*.cpp) but with plain asserts (doctest is not vendored).
//   test_dropin <hamiltonian.txt> <neel|plus> <dt> <steps> <out.raw>
// evolves the state and writes it with StateVector::save_raw; the Python
// test compares it with the reference compiled from its sources.
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
    simdiag::EvolutionPlan plan;
    plan.n_steps = std::atoi(argv[4]);
    plan.total_time = std::atof(argv[3]) * plan.n_steps;
    simdiag::evolve_grouped(groups, psi, plan);
    CHECK(std::abs(simdiag::norm(psi) - 1.0) < 1e-12);
    std::ofstream out(argv[5], std::ios::binary);
    psi.save_raw(out);
    std::printf("ok n=%d groups=%zu\n", n, groups.size());
    return 0;
}
