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

StateVector::~StateVector() { sd_state_destroy(s_); }

StateVector::StateVector(StateVector&& o) noexcept
    : n_qubits_(o.n_qubits_), s_(o.s_), host_(std::move(o.host_)), host_valid_(o.host_valid_), host_dirty_(o.host_dirty_) {
    o.s_ = nullptr;
}

StateVector& StateVector::operator=(StateVector&& o) noexcept {
    if (this != &o) {
        sd_state_destroy(s_);
        n_qubits_ = o.n_qubits_;
        s_ = o.s_;
        host_ = std::move(o.host_);
        host_valid_ = o.host_valid_;
        host_dirty_ = o.host_dirty_;
        o.s_ = nullptr;
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

void evolve_grouped(std::span<const DiagonalGroup> groups, StateVector& psi, const EvolutionPlan& plan) {
    plan.validate();
    if (plan.n_steps == 0) return;
    std::deque<std::vector<int32_t>> keep;  // stable element addresses
    std::vector<sd_group_desc> descs;
    for (const DiagonalGroup& g : groups) descs.push_back(desc_of(g, keep));
    sd_plan_options o;
    check(sd_plan_options_default(&o));
    o.order = plan.order;
    sd_plan* p = nullptr;
    check(sd_plan_create(psi.handle(), descs.data(), descs.size(), &o, &p));
    const sd_status st = sd_evolve(p, plan.dt(), plan.n_steps);
    sd_plan_destroy(p);
    check(st);
}

}  // namespace simdiag
