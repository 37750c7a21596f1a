// extern "C" host entry points: Hamiltonian I/O, greedy grouping and
// Clifford synthesis (all computed by the from-scratch C++ in csrc/host).
#include <charconv>
#include <cstdio>
#include <cstring>
#include <memory>
#include <sstream>

#include "guard.hpp"
#include "simdiag/diagonalize.hpp"
#include "simdiag/hamiltonian.hpp"
#include "simdiag/models.hpp"

struct sd_hamiltonian {
    simdiag::Hamiltonian h;
};

struct sd_group_store {
    simdiag::DiagonalGroup diag;
    std::vector<int32_t> h_pre, cnots, czs, s_layer, h_post;
    std::vector<uint64_t> src_x, src_z;
    std::vector<double> src_c;
    bool synthesized = true;
};

struct sd_groups {
    std::vector<sd_group_store> g;
};

namespace sdb {

namespace {
thread_local std::string g_last_error;

void fill_store(sd_group_store& st, const simdiag::CommutingGroup& cg, bool synth) {
    st.synthesized = synth;
    if (synth) st.diag = simdiag::diagonalize_group(cg);
    st.diag.group_index = cg.group_index;
    const auto& c = st.diag.circuit;
    st.h_pre.assign(c.h_pre.begin(), c.h_pre.end());
    st.s_layer.assign(c.s_layer.begin(), c.s_layer.end());
    st.h_post.assign(c.h_post.begin(), c.h_post.end());
    for (auto [a, b] : c.cnots) st.cnots.insert(st.cnots.end(), {a, b});
    for (auto [a, b] : c.czs) st.czs.insert(st.czs.end(), {a, b});
    for (const auto& t : cg.terms) {
        st.src_x.push_back(t.pauli.x_mask());
        st.src_z.push_back(t.pauli.z_mask());
        st.src_c.push_back(t.coeff);
    }
}

void write_text(const std::string& s, char* buf, size_t cap, size_t* len) {
    if (len) *len = s.size();
    if (buf && cap) {
        const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
        std::memcpy(buf, s.data(), n);
        buf[n] = '\0';
    }
}
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }
void write_text_out(const std::string& s, char* buf, size_t cap, size_t* len) { write_text(s, buf, cap, len); }

}  // namespace sdb

using sdb::guard;
using sdb::require;

extern "C" {

const char* sd_last_error(void) { return sdb::last_error(); }
const char* sd_version(void) { return "simdiag-b200 0.1 (sm_100a)"; }

sd_status sd_gen_tfim(int n_qubits, uint64_t seed, sd_hamiltonian** out) {
    return guard([&] {
        require(out != nullptr, "out is null");
        auto h = std::make_unique<sd_hamiltonian>();
        h->h = simdiag::gen_tfim(n_qubits, seed);
        *out = h.release();
    });
}

sd_status sd_gen_syk(int n_qubits, uint64_t seed, size_t* candidate_quadruples, size_t* merge_collisions,
                     sd_hamiltonian** out) {
    return guard([&] {
        require(out != nullptr, "out is null");
        simdiag::SykInfo info;
        auto h = std::make_unique<sd_hamiltonian>();
        h->h = simdiag::gen_syk(n_qubits, seed, &info);
        if (candidate_quadruples) *candidate_quadruples = info.candidate_quadruples;
        if (merge_collisions) *merge_collisions = info.merge_collisions;
        *out = h.release();
    });
}

sd_status sd_hamiltonian_from_terms(int n_qubits, const uint64_t* x, const uint64_t* z, const double* c,
                                    size_t m, double tol, size_t* merged, sd_hamiltonian** out) {
    return guard([&] {
        require(out != nullptr, "out is null");
        require(m == 0 || (x && z && c), "null term arrays");
        std::vector<simdiag::WeightedTerm> terms;
        terms.reserve(m);
        for (size_t k = 0; k < m; ++k) {
            terms.push_back({c[k], simdiag::PauliString::from_masks(n_qubits, x[k], z[k])});
        }
        auto h = std::make_unique<sd_hamiltonian>();
        h->h = simdiag::Hamiltonian::from_terms(n_qubits, std::move(terms), tol, merged);
        *out = h.release();
    });
}

sd_status sd_hamiltonian_load_text(const char* text, size_t len, double tol, sd_hamiltonian** out) {
    return guard([&] {
        require(out != nullptr && (text != nullptr || len == 0), "null argument");
        std::istringstream in(std::string(text ? text : "", len));
        auto h = std::make_unique<sd_hamiltonian>();
        h->h = simdiag::Hamiltonian::load(in, tol);
        *out = h.release();
    });
}

sd_status sd_hamiltonian_load_file(const char* path, double tol, sd_hamiltonian** out) {
    return guard([&] {
        require(out != nullptr && path != nullptr, "null argument");
        auto h = std::make_unique<sd_hamiltonian>();
        h->h = simdiag::Hamiltonian::load_file(path, tol);
        *out = h.release();
    });
}

sd_status sd_hamiltonian_save_text(const sd_hamiltonian* h, char* buf, size_t cap, size_t* len) {
    return guard([&] {
        require(h != nullptr, "null hamiltonian");
        std::ostringstream os;
        h->h.save(os);
        sdb::write_text_out(os.str(), buf, cap, len);
    });
}

sd_status sd_hamiltonian_info(const sd_hamiltonian* h, int* n, size_t* m) {
    return guard([&] {
        require(h != nullptr, "null hamiltonian");
        if (n) *n = h->h.n_qubits();
        if (m) *m = h->h.term_count();
    });
}

sd_status sd_hamiltonian_terms(const sd_hamiltonian* h, uint64_t* x, uint64_t* z, double* c) {
    return guard([&] {
        require(h != nullptr, "null hamiltonian");
        size_t k = 0;
        for (const auto& t : h->h.terms()) {
            if (x) x[k] = t.pauli.x_mask();
            if (z) z[k] = t.pauli.z_mask();
            if (c) c[k] = t.coeff;
            ++k;
        }
    });
}

void sd_hamiltonian_destroy(sd_hamiltonian* h) { delete h; }

sd_status sd_partition(const sd_hamiltonian* h, sd_groups** out) {
    return guard([&] {
        require(h != nullptr && out != nullptr, "null argument");
        auto gs = std::make_unique<sd_groups>();
        const auto parts = simdiag::greedy_partition(h->h);
        gs->g.resize(parts.size());
        for (size_t i = 0; i < parts.size(); ++i) sdb::fill_store(gs->g[i], parts[i], true);
        *out = gs.release();
    });
}

sd_status sd_partition_only(const sd_hamiltonian* h, sd_groups** out) {
    return guard([&] {
        require(h != nullptr && out != nullptr, "null argument");
        auto gs = std::make_unique<sd_groups>();
        const auto parts = simdiag::greedy_partition(h->h);
        gs->g.resize(parts.size());
        for (size_t i = 0; i < parts.size(); ++i) sdb::fill_store(gs->g[i], parts[i], false);
        *out = gs.release();
    });
}

sd_status sd_diagonalize_terms(int n_qubits, const uint64_t* x, const uint64_t* z, const double* c,
                               size_t m, sd_groups** out) {
    return guard([&] {
        require(out != nullptr, "out is null");
        require(m == 0 || (x && z && c), "null term arrays");
        simdiag::CommutingGroup g;
        for (size_t k = 0; k < m; ++k) {
            g.terms.push_back({c[k], simdiag::PauliString::from_masks(n_qubits, x[k], z[k])});
        }
        auto gs = std::make_unique<sd_groups>();
        gs->g.resize(1);
        sdb::fill_store(gs->g[0], g, true);
        *out = gs.release();
    });
}

sd_status sd_groups_count(const sd_groups* g, size_t* n) {
    return guard([&] {
        require(g != nullptr && n != nullptr, "null argument");
        *n = g->g.size();
    });
}

void sd_groups_destroy(sd_groups* g) { delete g; }

sd_status sd_group_get(const sd_groups* g, size_t index, sd_group_desc* d) {
    return guard([&] {
        require(g != nullptr && d != nullptr, "null argument");
        if (index >= g->g.size()) throw std::out_of_range("group index out of range");
        const sd_group_store& s = g->g[index];
        d->group_index = s.diag.group_index;
        d->n_qubits = s.diag.circuit.n_qubits;
        d->n_h_pre = s.h_pre.size();
        d->h_pre = s.h_pre.data();
        d->n_cnots = s.cnots.size() / 2;
        d->cnots = s.cnots.data();
        d->n_czs = s.czs.size() / 2;
        d->czs = s.czs.data();
        d->n_s = s.s_layer.size();
        d->s_layer = s.s_layer.data();
        d->n_h_post = s.h_post.size();
        d->h_post = s.h_post.data();
        d->n_terms = s.src_c.size();
        d->z_masks = s.synthesized ? s.diag.z_masks.data() : nullptr;
        d->signed_coeffs = s.synthesized ? s.diag.signed_coeffs.data() : nullptr;
        d->src_x = s.src_x.data();
        d->src_z = s.src_z.data();
        d->src_coeffs = s.src_c.data();
    });
}

// `diag` document of a synthesised partition (the reference's
// diag_document, proj/src/serialize.cpp:46-66): the bit-exact grouping /
// circuit diff format. Keys in nlohmann::json's (sorted) order; z-masks as
// "0x.." hex strings; coefficients as shortest round-trip doubles.
sd_status sd_groups_diag_json(const sd_groups* g, int n_qubits, char* buf, size_t cap, size_t* len) {
    return sdb::guard([&] {
        sdb::require(g != nullptr, "null groups");
        auto ints = [](std::ostringstream& os, const std::vector<int32_t>& v) {
            os << "[";
            for (size_t i = 0; i < v.size(); ++i) os << (i ? "," : "") << v[i];
            os << "]";
        };
        auto pairs = [](std::ostringstream& os, const std::vector<int32_t>& v) {
            os << "[";
            for (size_t i = 0; i + 1 < v.size(); i += 2) os << (i ? "," : "") << "[" << v[i] << "," << v[i + 1] << "]";
            os << "]";
        };
        auto dbl = [](std::ostringstream& os, double d) {
            char b[64];
            auto r = std::to_chars(b, b + sizeof b, d);
            std::string t(b, r.ptr);
            if (t.find_first_of(".eEn") == std::string::npos) t += ".0";
            os << t;
        };
        std::ostringstream os;
        os << "{\"groups\":[";
        for (size_t i = 0; i < g->g.size(); ++i) {
            const sd_group_store& st = g->g[i];
            if (!st.synthesized) throw std::invalid_argument("groups are not synthesised (sd_partition_only)");
            os << (i ? "," : "") << "{\"circuit\":{\"cnot\":";
            pairs(os, st.cnots);
            os << ",\"cz\":";
            pairs(os, st.czs);
            os << ",\"h_post\":";
            ints(os, st.h_post);
            os << ",\"h_pre\":";
            ints(os, st.h_pre);
            os << ",\"n_qubits\":" << st.diag.circuit.n_qubits << ",\"s\":";
            ints(os, st.s_layer);
            os << "},\"coeffs\":[";
            for (size_t k = 0; k < st.diag.signed_coeffs.size(); ++k) {
                if (k) os << ",";
                dbl(os, st.diag.signed_coeffs[k]);
            }
            os << "],\"group\":" << st.diag.group_index << ",\"z_masks\":[";
            for (size_t k = 0; k < st.diag.z_masks.size(); ++k) {
                char b[24];
                std::snprintf(b, sizeof b, "0x%llx", static_cast<unsigned long long>(st.diag.z_masks[k]));
                os << (k ? "," : "") << "\"" << b << "\"";
            }
            os << "]}";
        }
        os << "],\"n_groups\":" << g->g.size() << ",\"n_qubits\":" << n_qubits << "}";
        sdb::write_text_out(os.str(), buf, cap, len);
    });
}

}  // extern "C"
