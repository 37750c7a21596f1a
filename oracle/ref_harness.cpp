// ref_harness.cpp -- TEST INFRASTRUCTURE ONLY (oracle side).
//
// A C-ABI shim over the reference implementation compiled from its own
// sources (/root/reference/proj/src/{pauli,hamiltonian,tableau,diagonalize,
// statevector}.cpp) into oracle/_ref/libsimdiag_ref.so by oracle/Makefile.
// It lets tests/ and bench.py (--impl reference, cpu_baseline) drive the
// reference's public C++ API through ctypes. evolve.cpp needs Eigen (absent
// in this image), so evolve_grouped's 12-line loop (proj/src/evolve.cpp:47-58)
// is restated here with the same calls in the same order; S2 is the
// composition SURVEY §8a D1 defines (the reference has no S2).
#include <algorithm>
#include <bit>
#include <chrono>
#include <complex>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include <omp.h>

#include "simdiag/diagonalize.hpp"
#include "simdiag/serialize.hpp"
#include "simdiag/hamiltonian.hpp"
#include "simdiag/models.hpp"
#include "simdiag/statevector.hpp"

namespace {
thread_local std::string g_err;

struct RefGroups {
    int n = 0;
    std::vector<simdiag::CommutingGroup> parts;
    std::vector<simdiag::DiagonalGroup> diags;
    std::vector<std::vector<int>> cnots, czs;
};

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

void apply_group(simdiag::StateVector& psi, const simdiag::DiagonalGroup& g, double dt) {
    psi.apply_clifford(g.circuit);
    psi.apply_diagonal_exp(g, dt);
    psi.apply_clifford_inverse(g.circuit);
}

void load_state(simdiag::StateVector& psi, const double* re_im) {
    for (std::uint64_t i = 0; i < psi.dim(); ++i) psi[i] = {re_im[2 * i], re_im[2 * i + 1]};
}
void store_state(const simdiag::StateVector& psi, double* re_im) {
    for (std::uint64_t i = 0; i < psi.dim(); ++i) {
        re_im[2 * i] = psi[i].real();
        re_im[2 * i + 1] = psi[i].imag();
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Hamiltonian::load -> greedy_partition -> diagonalize_group for each group.
int ref_partition_text(const char* text, size_t len, int synthesize, void** out) {
    return guarded([&] {
        std::istringstream in(std::string(text, len));
        auto h = simdiag::Hamiltonian::load(in);
        auto r = std::make_unique<RefGroups>();
        r->n = h.n_qubits();
        r->parts = simdiag::greedy_partition(h);
        for (const auto& p : r->parts) {
            simdiag::DiagonalGroup d;
            if (synthesize) d = simdiag::diagonalize_group(p);
            std::vector<int> cx, cz;
            for (auto [a, b] : d.circuit.cnots) cx.insert(cx.end(), {a, b});
            for (auto [a, b] : d.circuit.czs) cz.insert(cz.end(), {a, b});
            r->cnots.push_back(std::move(cx));
            r->czs.push_back(std::move(cz));
            r->diags.push_back(std::move(d));
        }
        *out = r.release();
    });
}

// gen_tfim (model 0) / gen_syk (model 1) (models.cpp:17-92) -> save() text.
int ref_gen_save_text(int model, int n, uint64_t seed, char* buf, size_t cap, size_t* out_len, uint64_t* info) {
    return guarded([&] {
        simdiag::SykInfo si;
        const simdiag::Hamiltonian h = model == 0 ? simdiag::gen_tfim(n, seed) : simdiag::gen_syk(n, seed, &si);
        std::ostringstream os;
        h.save(os);
        const std::string s = os.str();
        *out_len = s.size();
        if (info) {
            info[0] = si.candidate_quadruples;
            info[1] = si.merge_collisions;
        }
        if (buf && cap) {
            const size_t k = s.size() < cap - 1 ? s.size() : cap - 1;
            std::memcpy(buf, s.data(), k);
            buf[k] = 0;
        }
    });
}

// greedy_partition alone (hamiltonian.cpp:135-158), timed: seconds and group count.
int ref_partition_timed(const char* text, size_t len, double* secs, size_t* n_groups) {
    return guarded([&] {
        std::istringstream in(std::string(text, len));
        const auto h = simdiag::Hamiltonian::load(in);
        const auto t0 = std::chrono::steady_clock::now();
        const auto parts = simdiag::greedy_partition(h);
        *secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *n_groups = parts.size();
    });
}

// Hamiltonian::load + save (round trip text).
int ref_load_save(const char* text, size_t len, char* buf, size_t cap, size_t* out_len) {
    return guarded([&] {
        std::istringstream in(std::string(text, len));
        auto h = simdiag::Hamiltonian::load(in);
        std::ostringstream os;
        h.save(os);
        const std::string s = os.str();
        *out_len = s.size();
        if (buf && cap) {
            const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
            std::memcpy(buf, s.data(), n);
            buf[n] = 0;
        }
    });
}

// diagonalize_group on an explicit term list.
int ref_diagonalize_terms(int n, const uint64_t* x, const uint64_t* z, const double* c, size_t m, void** out) {
    return guarded([&] {
        simdiag::CommutingGroup g;
        for (size_t k = 0; k < m; ++k) g.terms.push_back({c[k], simdiag::PauliString::from_masks(n, x[k], z[k])});
        auto r = std::make_unique<RefGroups>();
        r->n = n;
        r->parts.push_back(g);
        auto d = simdiag::diagonalize_group(g);
        std::vector<int> cx, cz;
        for (auto [a, b] : d.circuit.cnots) cx.insert(cx.end(), {a, b});
        for (auto [a, b] : d.circuit.czs) cz.insert(cz.end(), {a, b});
        r->cnots.push_back(std::move(cx));
        r->czs.push_back(std::move(cz));
        r->diags.push_back(std::move(d));
        *out = r.release();
    });
}

void ref_groups_free(void* h) { delete static_cast<RefGroups*>(h); }
int ref_groups_count(void* h) { return static_cast<int>(static_cast<RefGroups*>(h)->parts.size()); }
int ref_groups_nqubits(void* h) { return static_cast<RefGroups*>(h)->n; }

// sizes[0..5] = h_pre, cnots, czs, s, h_post, terms
void ref_group_sizes(void* h, int g, int64_t* sizes) {
    auto* r = static_cast<RefGroups*>(h);
    const auto& c = r->diags[g].circuit;
    sizes[0] = c.h_pre.size();
    sizes[1] = c.cnots.size();
    sizes[2] = c.czs.size();
    sizes[3] = c.s_layer.size();
    sizes[4] = c.h_post.size();
    sizes[5] = r->parts[g].terms.size();
}

void ref_group_data(void* h, int g, int32_t* h_pre, int32_t* cnots, int32_t* czs, int32_t* s, int32_t* h_post,
                    uint64_t* src_x, uint64_t* src_z, double* src_c, uint64_t* zm, double* cf) {
    auto* r = static_cast<RefGroups*>(h);
    const auto& d = r->diags[g];
    const auto& c = d.circuit;
    for (size_t i = 0; i < c.h_pre.size(); ++i) h_pre[i] = c.h_pre[i];
    for (size_t i = 0; i < r->cnots[g].size(); ++i) cnots[i] = r->cnots[g][i];
    for (size_t i = 0; i < r->czs[g].size(); ++i) czs[i] = r->czs[g][i];
    for (size_t i = 0; i < c.s_layer.size(); ++i) s[i] = c.s_layer[i];
    for (size_t i = 0; i < c.h_post.size(); ++i) h_post[i] = c.h_post[i];
    const auto& t = r->parts[g].terms;
    for (size_t i = 0; i < t.size(); ++i) {
        src_x[i] = t[i].pauli.x_mask();
        src_z[i] = t[i].pauli.z_mask();
        src_c[i] = t[i].coeff;
        if (i < d.z_masks.size()) {
            zm[i] = d.z_masks[i];
            cf[i] = d.signed_coeffs[i];
        }
    }
}

// evolve_grouped (evolve.cpp:47-58) over every group of `h`, in place on
// re_im (2^n interleaved doubles). order 2 = S2 composition. stats (may be
// NULL) receives KernelStats {reads, writes, calls}.
int ref_evolve_grouped(void* h, double* re_im, int n, double dt, int steps, int order, uint64_t* stats) {
    return guarded([&] {
        auto* r = static_cast<RefGroups*>(h);
        simdiag::StateVector psi(n);
        load_state(psi, re_im);
        const auto& gs = r->diags;
        const size_t G = gs.size();
        for (int s = 0; s < steps; ++s) {
            if (order == 1 || G <= 1) {
                for (const auto& g : gs) apply_group(psi, g, dt);
            } else {
                for (size_t g = 0; g + 1 < G; ++g) apply_group(psi, gs[g], 0.5 * dt);
                apply_group(psi, gs[G - 1], dt);
                for (size_t g = G - 1; g-- > 0;) apply_group(psi, gs[g], 0.5 * dt);
            }
        }
        store_state(psi, re_im);
        if (stats) {
            stats[0] = psi.stats().amp_reads;
            stats[1] = psi.stats().amp_writes;
            stats[2] = psi.stats().kernel_calls;
        }
    });
}

// A reference StateVector that persists across calls, so the CPU timings
// (bench.py cpu_baseline / --impl reference) cover evolve_grouped's loop
// only, not a 16 GiB copy in and out per call.
void* ref_sv_create(int n) {
    void* out = nullptr;
    const int rc = guarded([&] { out = new simdiag::StateVector(n); });
    return rc == 0 ? out : nullptr;
}
void ref_sv_free(void* sv) { delete static_cast<simdiag::StateVector*>(sv); }
int ref_sv_set_basis(void* sv, uint64_t index) {
    return guarded([&] {
        auto& psi = *static_cast<simdiag::StateVector*>(sv);
        for (uint64_t i = 0; i < psi.dim(); ++i) psi[i] = 0.0;
        psi[index] = 1.0;
    });
}
int ref_sv_write(void* sv, uint64_t first, uint64_t count, const double* re_im) {
    return guarded([&] {
        auto& psi = *static_cast<simdiag::StateVector*>(sv);
        for (uint64_t i = 0; i < count; ++i) psi[first + i] = {re_im[2 * i], re_im[2 * i + 1]};
    });
}
int ref_sv_read(void* sv, uint64_t first, uint64_t count, double* re_im) {
    return guarded([&] {
        const auto& psi = *static_cast<simdiag::StateVector*>(sv);
        for (uint64_t i = 0; i < count; ++i) {
            re_im[2 * i] = psi[first + i].real();
            re_im[2 * i + 1] = psi[first + i].imag();
        }
    });
}
// evolve_grouped's loop (evolve.cpp:47-58) on the persistent state.
int ref_sv_evolve(void* sv, void* h, double dt, int steps, int order) {
    return guarded([&] {
        auto& psi = *static_cast<simdiag::StateVector*>(sv);
        const auto& gs = static_cast<RefGroups*>(h)->diags;
        const size_t G = gs.size();
        for (int s = 0; s < steps; ++s) {
            if (order == 1 || G <= 1) {
                for (const auto& g : gs) apply_group(psi, g, dt);
            } else {
                for (size_t g = 0; g + 1 < G; ++g) apply_group(psi, gs[g], 0.5 * dt);
                apply_group(psi, gs[G - 1], dt);
                for (size_t g = G - 1; g-- > 0;) apply_group(psi, gs[g], 0.5 * dt);
            }
        }
    });
}
double ref_sv_norm(void* sv) { return simdiag::norm(*static_cast<simdiag::StateVector*>(sv)); }
void ref_set_threads(int t) { omp_set_num_threads(t); }
int ref_get_threads() { return omp_get_max_threads(); }

int ref_random_state(int n, uint64_t seed, double* re_im) {
    return guarded([&] { store_state(simdiag::StateVector::random_state(n, seed), re_im); });
}

int ref_plus_state(int n, double* re_im) {
    return guarded([&] { store_state(simdiag::StateVector::plus_state(n), re_im); });
}

// Single-kernel entry points (statevector.cpp:156-286) on a host buffer.
int ref_kernel(int which, double* re_im, int n, int a, uint64_t mask, const int32_t* pairs, size_t np,
               const uint64_t* zm, const double* cf, size_t m, double dt) {
    return guarded([&] {
        simdiag::StateVector psi(n);
        load_state(psi, re_im);
        std::vector<std::pair<int, int>> pv;
        for (size_t k = 0; k < np; ++k) pv.emplace_back(pairs[2 * k], pairs[2 * k + 1]);
        switch (which) {
            case 0: psi.apply_hadamard(a); break;
            case 1: psi.apply_batched_cnot(a, mask); break;
            case 2: psi.apply_phase_layer(mask, pv, a != 0); break;
            case 3: psi.apply_diagonal_exp(std::span<const uint64_t>(zm, m), std::span<const double>(cf, m), dt); break;
            default: throw std::invalid_argument("unknown kernel");
        }
        store_state(psi, re_im);
    });
}

// StateVector::apply_pauli_rotation (statevector.cpp:288-337) on one term.
int ref_pauli_rotation(double* re_im, int n, uint64_t x, uint64_t z, double coeff, double dt) {
    return guarded([&] {
        simdiag::StateVector psi(n);
        load_state(psi, re_im);
        psi.apply_pauli_rotation(simdiag::WeightedTerm{coeff, simdiag::PauliString::from_masks(n, x, z)}, dt);
        store_state(psi, re_im);
    });
}

// apply_single_qubit / apply_two_qubit (statevector.cpp:101-154); u =
// row-major complex entries as (re, im) pairs.
int ref_generic_gate(double* re_im, int n, const double* u, int q1, int q2) {
    return guarded([&] {
        simdiag::StateVector psi(n);
        load_state(psi, re_im);
        if (q2 < 0) {
            simdiag::Mat2 m;
            for (int k = 0; k < 4; ++k) m[k] = {u[2 * k], u[2 * k + 1]};
            psi.apply_single_qubit(m, q1);
        } else {
            simdiag::Mat4 m;
            for (int k = 0; k < 16; ++k) m[k] = {u[2 * k], u[2 * k + 1]};
            psi.apply_two_qubit(m, q1, q2);
        }
        store_state(psi, re_im);
    });
}

// evolve_baseline(span<const CommutingGroup>, ...) restated (evolve.cpp:34-45)
// over a partition_text handle's groups.
int ref_evolve_baseline_groups(void* h, double* re_im, int n, double dt, int steps) {
    return guarded([&] {
        auto* r = static_cast<RefGroups*>(h);
        simdiag::StateVector psi(n);
        load_state(psi, re_im);
        for (int s = 0; s < steps; ++s)
            for (const auto& g : r->parts)
                for (const auto& term : g.terms) psi.apply_pauli_rotation(term, dt);
        store_state(psi, re_im);
    });
}

// evolve_baseline(const Hamiltonian&, ...) restated (evolve.cpp:21-32: same
// calls, same order; evolve.cpp itself needs Eigen).
int ref_evolve_baseline_text(const char* text, size_t len, double* re_im, int n, double dt, int steps) {
    return guarded([&] {
        std::istringstream in(std::string(text, len));
        const auto h = simdiag::Hamiltonian::load(in);
        simdiag::StateVector psi(n);
        load_state(psi, re_im);
        for (int s = 0; s < steps; ++s)
            for (const auto& term : h.terms()) psi.apply_pauli_rotation(term, dt);
        store_state(psi, re_im);
    });
}

// expectation (evolve.cpp:99-135) restated: the same 256 fixed chunks per term.
int ref_expectation_text(const char* text, size_t len, const double* re_im, int n, double* re, double* imag) {
    return guarded([&] {
        std::istringstream in(std::string(text, len));
        const auto h = simdiag::Hamiltonian::load(in);
        simdiag::StateVector psi(n);
        load_state(psi, re_im);
        const std::uint64_t dim = psi.dim();
        const std::complex<double> i_pow[4] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};
        std::complex<double> total = 0.0;
        for (const auto& term : h.terms()) {
            const std::uint64_t x = term.pauli.x_mask();
            const std::uint64_t z = term.pauli.z_mask();
            const std::complex<double> base = i_pow[term.pauli.phase_exp()];
            constexpr int kChunks = 256;
            std::complex<double> partial[kChunks] = {};
            const std::uint64_t chunk_len = (dim + kChunks - 1) / kChunks;
            for (int c = 0; c < kChunks; ++c) {
                const std::uint64_t begin = c * chunk_len;
                const std::uint64_t end = std::min(dim, begin + chunk_len);
                std::complex<double> acc = 0.0;
                for (std::uint64_t b = begin; b < end; ++b) {
                    const bool parity = std::popcount((b ^ x) & z) & 1;
                    const std::complex<double> ph = parity ? -base : base;
                    acc += std::conj(psi[b]) * ph * psi[b ^ x];
                }
                partial[c] = acc;
            }
            std::complex<double> sum = 0.0;
            for (int c = 0; c < kChunks; ++c) sum += partial[c];
            total += term.coeff * sum;
        }
        *re = total.real();
        *imag = std::abs(total.imag());
    });
}

// diag_document (serialize.cpp:46-66) of a partition_text handle, dumped.
int ref_diag_json(void* h, char* buf, size_t cap, size_t* len) {
    return guarded([&] {
        auto* r = static_cast<RefGroups*>(h);
        const std::string s = simdiag::diag_document(r->n, r->diags).dump();
        *len = s.size();
        if (buf && cap) {
            const size_t k = std::min(cap - 1, s.size());
            std::memcpy(buf, s.data(), k);
            buf[k] = 0;
        }
    });
}

double ref_norm(const double* re_im, int n) {
    simdiag::StateVector psi(n);
    for (std::uint64_t i = 0; i < psi.dim(); ++i) psi[i] = {re_im[2 * i], re_im[2 * i + 1]};
    return simdiag::norm(psi);
}

}  // extern "C"
