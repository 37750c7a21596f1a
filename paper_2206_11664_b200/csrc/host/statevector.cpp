// simdiag::StateVector / evolve_grouped over the C ABI (include/simdiag/
// statevector.hpp, evolve.hpp): the reference's C++ surface for the device
// path. Every call maps an sd_status back onto the reference's exception
// types (proj/src/statevector.cpp, proj/src/evolve.cpp).
#include "simdiag/statevector.hpp"

#include <cmath>
#include <deque>
#include <cstring>
#include <istream>
#include <ostream>
#include <stdexcept>
#include <string>

#include "simdiag/evolve.hpp"
#include "simdiag_c.h"

namespace simdiag {

// evolve_grouped's compiled schedules (sd_plan) for one state, keyed by the
// exact bytes of the group list and the Trotter order: a caller that steps and
// measures in a loop plans once. Bounded, least recently used first out.
struct PlanCache {
    static constexpr size_t kMax = 4;
    std::vector<std::pair<std::string, sd_plan*>> entries;  // most recent last
    ~PlanCache() {
        for (auto& e : entries) sd_plan_destroy(e.second);
    }
};

namespace {

void check(sd_status st) {
    if (st == SD_OK) return;
    const std::string m = sd_last_error();
    if (st == SD_INVALID_ARGUMENT) throw std::invalid_argument(m);
    if (st == SD_OUT_OF_RANGE) throw std::out_of_range(m);
    throw std::runtime_error(m);
}

sd_group_desc desc_of(const DiagonalGroup& g, std::deque<std::vector<int32_t>>& keep) {
    const CliffordCircuit& c = g.circuit;
    auto& h0 = keep.emplace_back(c.h_pre.begin(), c.h_pre.end());
    auto& cx = keep.emplace_back();
    for (auto [a, b] : c.cnots) cx.insert(cx.end(), {a, b});
    auto& cz = keep.emplace_back();
    for (auto [a, b] : c.czs) cz.insert(cz.end(), {a, b});
    auto& s = keep.emplace_back(c.s_layer.begin(), c.s_layer.end());
    auto& h1 = keep.emplace_back(c.h_post.begin(), c.h_post.end());
    sd_group_desc d{};
    d.group_index = g.group_index;
    d.n_qubits = c.n_qubits;
    d.n_h_pre = h0.size();
    d.h_pre = h0.data();
    d.n_cnots = c.cnots.size();
    d.cnots = cx.data();
    d.n_czs = c.czs.size();
    d.czs = cz.data();
    d.n_s = s.size();
    d.s_layer = s.data();
    d.n_h_post = h1.size();
    d.h_post = h1.data();
    d.n_terms = g.z_masks.size();
    d.z_masks = g.z_masks.data();
    d.signed_coeffs = g.signed_coeffs.data();
    return d;
}

}  // namespace

StateVector::StateVector(int n_qubits, int device) : n_qubits_(n_qubits) {
    if (n_qubits < 0) throw std::invalid_argument("state vector qubit count out of range");
    check(sd_state_create(n_qubits, device, &s_));
}

StateVector::~StateVector() {
    delete plans_;  // plans reference the state: destroyed first
    sd_state_destroy(s_);
}

StateVector::StateVector(StateVector&& o) noexcept
    : n_qubits_(o.n_qubits_), s_(o.s_), host_(std::move(o.host_)), host_valid_(o.host_valid_), host_dirty_(o.host_dirty_),
      plans_(o.plans_) {
    o.s_ = nullptr;
    o.plans_ = nullptr;
}

StateVector& StateVector::operator=(StateVector&& o) noexcept {
    if (this != &o) {
        delete plans_;
        sd_state_destroy(s_);
        n_qubits_ = o.n_qubits_;
        s_ = o.s_;
        host_ = std::move(o.host_);
        host_valid_ = o.host_valid_;
        host_dirty_ = o.host_dirty_;
        plans_ = o.plans_;
        o.s_ = nullptr;
        o.plans_ = nullptr;
    }
    return *this;
}

StateVector StateVector::zero_state(int n) { return StateVector(n); }

StateVector StateVector::plus_state(int n) {
    StateVector v(n);
    check(sd_state_set_plus(v.s_));
    return v;
}

StateVector StateVector::random_state(int n, std::uint64_t seed) {
    StateVector v(n);
    check(sd_state_set_random(v.s_, seed));
    return v;
}

void StateVector::fetch() const {
    if (host_valid_) return;
    host_.resize(dim());
    check(sd_state_download(s_, reinterpret_cast<double*>(host_.data()), dim()));
    host_valid_ = true;
}

sd_state* StateVector::sync_to_device() {
    if (host_dirty_) {
        check(sd_state_upload(s_, reinterpret_cast<const double*>(host_.data()), dim()));
        host_dirty_ = false;
    }
    host_valid_ = false;  // the caller is about to mutate the device copy
    return s_;
}

std::span<const Amplitude> StateVector::amplitudes() const {
    fetch();
    return host_;
}

Amplitude& StateVector::operator[](std::uint64_t i) {
    fetch();
    host_dirty_ = true;
    return host_.at(i);
}

const Amplitude& StateVector::operator[](std::uint64_t i) const {
    fetch();
    return host_.at(i);
}

void StateVector::apply_single_qubit(const Mat2& u, int target) {
    check(sd_apply_single_qubit(sync_to_device(), reinterpret_cast<const double*>(u.data()), target));
}

void StateVector::apply_two_qubit(const Mat4& u, int q1, int q2) {
    check(sd_apply_two_qubit(sync_to_device(), reinterpret_cast<const double*>(u.data()), q1, q2));
}

void StateVector::apply_pauli_rotation(const WeightedTerm& term, double dt) {
    if (term.pauli.n_qubits() != n_qubits_) throw std::invalid_argument("pauli rotation: qubit count mismatch");
    check(sd_apply_pauli_rotation(sync_to_device(), term.pauli.x_mask(), term.pauli.z_mask(), term.coeff, dt));
}

void StateVector::apply_hadamard(int target) { check(sd_apply_hadamard(sync_to_device(), target)); }

void StateVector::apply_batched_cnot(int control, std::uint64_t targets) {
    check(sd_apply_batched_cnot(sync_to_device(), control, targets));
}

void StateVector::apply_phase_layer(std::uint64_t s_mask, std::span<const std::pair<int, int>> cz_pairs, bool dagger) {
    std::vector<int32_t> flat;
    for (auto [a, b] : cz_pairs) flat.insert(flat.end(), {a, b});
    check(sd_apply_phase_layer(sync_to_device(), s_mask, flat.data(), cz_pairs.size(), dagger ? 1 : 0));
}

void StateVector::apply_diagonal_exp(std::span<const std::uint64_t> z_masks, std::span<const double> coeffs, double dt) {
    if (z_masks.size() != coeffs.size()) throw std::invalid_argument("diagonal exp: mask/coefficient size mismatch");
    check(sd_apply_diagonal_exp(sync_to_device(), z_masks.data(), coeffs.data(), z_masks.size(), dt));
}

void StateVector::apply_diagonal_exp(const DiagonalGroup& group, double dt) {
    apply_diagonal_exp(group.z_masks, group.signed_coeffs, dt);
}

void StateVector::apply_clifford(const CliffordCircuit& c) {
    DiagonalGroup g;
    g.circuit = c;
    std::deque<std::vector<int32_t>> keep;  // stable element addresses
    const sd_group_desc d = desc_of(g, keep);
    check(sd_apply_clifford(sync_to_device(), &d));
}

void StateVector::apply_clifford_inverse(const CliffordCircuit& c) {
    DiagonalGroup g;
    g.circuit = c;
    std::deque<std::vector<int32_t>> keep;  // stable element addresses
    const sd_group_desc d = desc_of(g, keep);
    check(sd_apply_clifford_inverse(sync_to_device(), &d));
}

void StateVector::save_raw(std::ostream& out) const {
    fetch();
    out.write(reinterpret_cast<const char*>(host_.data()), static_cast<std::streamsize>(host_.size() * sizeof(Amplitude)));
}

StateVector StateVector::load_raw(std::istream& in) {
    std::vector<char> bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    const size_t amps = bytes.size() / sizeof(Amplitude);
    if (amps == 0 || (amps & (amps - 1)) || bytes.size() % sizeof(Amplitude)) {
        throw std::invalid_argument("load_raw: size is not a power of two of (re, im) pairs");
    }
    int n = 0;
    while ((size_t(1) << n) < amps) ++n;
    StateVector v(n);
    check(sd_state_upload(v.s_, reinterpret_cast<const double*>(bytes.data()), amps));
    return v;
}

KernelStats StateVector::stats() const {
    sd_kernel_stats k{};
    check(sd_kernel_stats_get(s_, &k));
    return KernelStats{k.amp_reads, k.amp_writes, k.kernel_calls};
}

void StateVector::reset_stats() { check(sd_kernel_stats_reset(s_)); }

double norm(const StateVector& a) {
    double v = 0.0;
    check(sd_state_norm_sq(const_cast<StateVector&>(a).handle(), &v));
    return std::sqrt(v);
}

double fidelity(const StateVector& a, const StateVector& b) {
    if (a.n_qubits() != b.n_qubits()) throw std::invalid_argument("fidelity: dimension mismatch");
    double re = 0.0, im = 0.0;
    check(sd_state_inner(const_cast<StateVector&>(a).handle(), const_cast<StateVector&>(b).handle(), &re, &im));
    return std::hypot(re, im);
}

void EvolutionPlan::validate() const {
    if (n_steps < 0) throw std::invalid_argument("plan needs n_steps >= 0");
    if (!std::isfinite(total_time)) throw std::invalid_argument("plan needs finite total_time");
    if (order != 1 && order != 2) throw std::invalid_argument("trotter order must be 1 or 2");
}

namespace {

void append_bytes(std::string& k, const void* p, size_t n) { k.append(static_cast<const char*>(p), n); }

std::string plan_key(std::span<const DiagonalGroup> groups, int order) {
    std::string k;
    append_bytes(k, &order, sizeof order);
    for (const DiagonalGroup& g : groups) {
        const CliffordCircuit& c = g.circuit;
        const size_t sizes[6] = {c.h_pre.size(), c.cnots.size(), c.czs.size(), c.s_layer.size(), c.h_post.size(),
                                 g.z_masks.size()};
        append_bytes(k, sizes, sizeof sizes);
        append_bytes(k, &c.n_qubits, sizeof c.n_qubits);
        append_bytes(k, c.h_pre.data(), c.h_pre.size() * sizeof(int));
        append_bytes(k, c.cnots.data(), c.cnots.size() * sizeof(c.cnots[0]));
        append_bytes(k, c.czs.data(), c.czs.size() * sizeof(c.czs[0]));
        append_bytes(k, c.s_layer.data(), c.s_layer.size() * sizeof(int));
        append_bytes(k, c.h_post.data(), c.h_post.size() * sizeof(int));
        append_bytes(k, g.z_masks.data(), g.z_masks.size() * sizeof(std::uint64_t));
        append_bytes(k, g.signed_coeffs.data(), g.signed_coeffs.size() * sizeof(double));
    }
    return k;
}

struct TermArrays {
    std::vector<std::uint64_t> x, z;
    std::vector<double> c;
    void add(const WeightedTerm& t) {
        x.push_back(t.pauli.x_mask());
        z.push_back(t.pauli.z_mask());
        c.push_back(t.coeff);
    }
};

TermArrays arrays_of(const Hamiltonian& h) {
    TermArrays a;
    for (const WeightedTerm& t : h.terms()) a.add(t);
    return a;
}

}  // namespace

void evolve_grouped(std::span<const DiagonalGroup> groups, StateVector& psi, const EvolutionPlan& plan) {
    plan.validate();
    if (plan.n_steps == 0) return;
    sd_state* h = psi.handle();
    if (!psi.plans_) psi.plans_ = new PlanCache();
    PlanCache& cache = *psi.plans_;
    const std::string key = plan_key(groups, plan.order);
    sd_plan* p = nullptr;
    for (size_t i = 0; i < cache.entries.size(); ++i) {
        if (cache.entries[i].first == key) {
            auto e = cache.entries[i];
            cache.entries.erase(cache.entries.begin() + static_cast<std::ptrdiff_t>(i));
            cache.entries.push_back(e);
            p = e.second;
            break;
        }
    }
    if (!p) {
        std::deque<std::vector<int32_t>> keep;  // stable element addresses
        std::vector<sd_group_desc> descs;
        for (const DiagonalGroup& g : groups) descs.push_back(desc_of(g, keep));
        sd_plan_options o;
        check(sd_plan_options_default(&o));
        o.order = plan.order;
        check(sd_plan_create(h, descs.data(), descs.size(), &o, &p));
        if (cache.entries.size() >= PlanCache::kMax) {
            sd_plan_destroy(cache.entries.front().second);
            cache.entries.erase(cache.entries.begin());
        }
        cache.entries.emplace_back(key, p);
    }
    check(sd_evolve(p, plan.dt(), plan.n_steps));
}

void evolve_baseline(const Hamiltonian& h, StateVector& psi, const EvolutionPlan& plan) {
    plan.validate();
    if (h.n_qubits() != psi.n_qubits()) throw std::invalid_argument("hamiltonian/state qubit counts differ");
    const TermArrays a = arrays_of(h);
    const double dt = plan.n_steps > 0 ? plan.dt() : 0.0;
    check(sd_evolve_baseline(psi.handle(), a.x.data(), a.z.data(), a.c.data(), a.c.size(), dt, plan.n_steps));
}

void evolve_baseline(std::span<const CommutingGroup> groups, StateVector& psi, const EvolutionPlan& plan) {
    plan.validate();
    TermArrays a;
    for (const CommutingGroup& g : groups)
        for (const WeightedTerm& t : g.terms) a.add(t);
    const double dt = plan.n_steps > 0 ? plan.dt() : 0.0;
    check(sd_evolve_baseline(psi.handle(), a.x.data(), a.z.data(), a.c.data(), a.c.size(), dt, plan.n_steps));
}

StateVector exact_evolve(const Hamiltonian& h, const StateVector& psi, double t) {
    const int n = h.n_qubits();
    if (n != psi.n_qubits()) throw std::invalid_argument("hamiltonian/state qubit counts differ");
    if (n > kExactEvolveMaxQubits) {
        throw std::invalid_argument("exact_evolve limited to n <= " + std::to_string(kExactEvolveMaxQubits) +
                                    " qubits");
    }
    StateVector out(n);
    check(sd_state_copy(out.handle(), const_cast<StateVector&>(psi).handle()));
    const TermArrays a = arrays_of(h);
    check(sd_exact_evolve(out.handle(), a.x.data(), a.z.data(), a.c.data(), a.c.size(), t));
    return out;
}

double expectation(const Hamiltonian& h, const StateVector& psi, double* imag_residue) {
    if (h.n_qubits() != psi.n_qubits()) throw std::invalid_argument("hamiltonian/state qubit counts differ");
    const TermArrays a = arrays_of(h);
    double re = 0.0, im = 0.0;
    check(sd_expectation(const_cast<StateVector&>(psi).handle(), a.x.data(), a.z.data(), a.c.data(), a.c.size(), &re,
                         &im));
    if (imag_residue) *imag_residue = im;
    return re;
}

}  // namespace simdiag
