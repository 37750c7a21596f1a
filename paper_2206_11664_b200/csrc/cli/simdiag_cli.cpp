// simdiag -- command-line front end (SPEC.md module `cli`; the reference
// ships only a placeholder, proj/tools/main.cpp:1-6).
//
//   simdiag gen --model tfim|syk --qubits N [--seed S] [--out FILE]
//   simdiag partition FILE [--out ASSIGNMENT]
//   simdiag diag FILE [--out JSON]
//   simdiag run FILE --t T --steps K [--method grouped|baseline]
//               [--init zero|plus|neel|random[:SEED]] [--csv FILE] [--verify]
//   simdiag bench --model tfim|syk --qubits A[:B] [--repeats R] [--seed S] [--steps K]
//   simdiag verify FILE [--t T] [--steps K]
//
// Written purely against the drop-in C++ API (include/simdiag/*.hpp): every
// evolution runs on the GPU through libsimdiag_b200.so. Exit codes: 0 ok,
// 2 input error (std::invalid_argument / std::out_of_range / unreadable
// file), 3 internal invariant failure (std::runtime_error).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "simdiag/diagonalize.hpp"
#include "simdiag/evolve.hpp"
#include "simdiag/hamiltonian.hpp"
#include "simdiag/models.hpp"
#include "simdiag/statevector.hpp"
#include "simdiag_c.h"

namespace {

using namespace simdiag;

struct Args {
    std::vector<std::string> pos;
    std::map<std::string, std::string> opt;
    bool has(const std::string& k) const { return opt.count(k) != 0; }
    std::string get(const std::string& k, const std::string& dflt = "") const {
        auto it = opt.find(k);
        return it == opt.end() ? dflt : it->second;
    }
};

Args parse(int argc, char** argv, int first) {
    Args a;
    for (int i = first; i < argc; ++i) {
        std::string s = argv[i];
        if (s.rfind("--", 0) == 0) {
            const std::string k = s.substr(2);
            if (k == "verify") {
                a.opt[k] = "1";
            } else {
                if (i + 1 >= argc) throw std::invalid_argument("option --" + k + " needs a value");
                a.opt[k] = argv[++i];
            }
        } else {
            a.pos.push_back(s);
        }
    }
    return a;
}

Hamiltonian load_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::invalid_argument("cannot open " + path);
    return Hamiltonian::load(in);
}

Hamiltonian generate(const std::string& model, int n, std::uint64_t seed, SykInfo* info = nullptr) {
    if (model == "tfim") return gen_tfim(n, seed);
    if (model == "syk") return gen_syk(n, seed, info);
    throw std::invalid_argument("unknown model '" + model + "' (tfim|syk)");
}

std::vector<DiagonalGroup> synthesize(const std::vector<CommutingGroup>& parts) {
    std::vector<DiagonalGroup> out;
    out.reserve(parts.size());
    for (const CommutingGroup& g : parts) out.push_back(diagonalize_group(g));
    return out;
}

StateVector initial(const std::string& init, int n) {
    if (init == "zero") return StateVector::zero_state(n);
    if (init == "plus") return StateVector::plus_state(n);
    if (init == "neel") {
        StateVector v(n);
        std::uint64_t idx = 0;
        for (int q = 1; q < n; q += 2) idx |= std::uint64_t(1) << q;
        v[0] = 0.0;
        v[idx] = 1.0;
        return v;
    }
    if (init.rfind("random", 0) == 0) {
        const std::uint64_t seed = init.size() > 7 ? std::strtoull(init.c_str() + 7, nullptr, 10) : 0;
        return StateVector::random_state(n, seed);
    }
    throw std::invalid_argument("unknown --init '" + init + "' (zero|plus|neel|random[:seed])");
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int cmd_gen(const Args& a) {
    const int n = std::stoi(a.get("qubits", "0"));
    const std::uint64_t seed = std::stoull(a.get("seed", "0"));
    SykInfo info;
    const Hamiltonian h = generate(a.get("model"), n, seed, &info);
    if (a.has("out")) {
        std::ofstream out(a.get("out"));
        h.save(out);
    } else {
        h.save(std::cout);
    }
    std::fprintf(stderr, "model=%s n=%d seed=%llu m=%zu", a.get("model").c_str(), n,
                 static_cast<unsigned long long>(seed), h.term_count());
    if (a.get("model") == "syk")
        std::fprintf(stderr, " quadruples=%zu collisions=%zu", info.candidate_quadruples, info.merge_collisions);
    std::fprintf(stderr, "\n");
    return 0;
}

int cmd_partition(const Args& a) {
    if (a.pos.empty()) throw std::invalid_argument("partition needs a hamiltonian file");
    const Hamiltonian h = load_file(a.pos[0]);
    if (h.term_count() == 0) throw std::invalid_argument("hamiltonian has no terms");
    const auto t0 = std::chrono::steady_clock::now();
    const auto parts = greedy_partition(h);
    const double secs = seconds_since(t0);
    const PartitionStats st = partition_stats(h.n_qubits(), parts);
    std::printf("n=%d m=%zu n_g=%zu max_group=%zu predicted_speedup=%.4f partition_s=%.3f\n", h.n_qubits(),
                st.term_count, st.group_count, st.max_group_size, st.predicted_speedup, secs);
    std::printf("group_sizes");
    for (const CommutingGroup& g : parts) std::printf(" %zu", g.terms.size());
    std::printf("\n");
    if (a.has("out")) {
        // one line per input term (load order): "<term index> <group index>"
        std::map<std::pair<std::uint64_t, std::uint64_t>, int> where;
        for (const CommutingGroup& g : parts)
            for (const WeightedTerm& t : g.terms) where[{t.pauli.x_mask(), t.pauli.z_mask()}] = g.group_index;
        std::ofstream out(a.get("out"));
        for (size_t k = 0; k < h.terms().size(); ++k) {
            const auto& p = h.terms()[k].pauli;
            out << k << ' ' << where[{p.x_mask(), p.z_mask()}] << '\n';
        }
    }
    return 0;
}

int cmd_diag(const Args& a) {
    if (a.pos.empty()) throw std::invalid_argument("diag needs a hamiltonian file");
    const Hamiltonian h = load_file(a.pos[0]);
    // through the C ABI: greedy_partition + diagonalize_group (X blocks
    // verified zero) rendered as the reference's `diag` document
    std::ostringstream text;
    h.save(text);
    const std::string s = text.str();
    sd_hamiltonian* hh = nullptr;
    sd_groups* gs = nullptr;
    auto fail = [](sd_status st) {
        const std::string m = sd_last_error();
        if (st == SD_INVALID_ARGUMENT || st == SD_OUT_OF_RANGE) throw std::invalid_argument(m);
        throw std::runtime_error(m);
    };
    sd_status st = sd_hamiltonian_load_text(s.data(), s.size(), 0.0, &hh);
    if (st != SD_OK) fail(st);
    st = sd_partition(hh, &gs);
    if (st != SD_OK) {
        sd_hamiltonian_destroy(hh);
        fail(st);
    }
    size_t len = 0;
    sd_groups_diag_json(gs, h.n_qubits(), nullptr, 0, &len);
    std::string js(len + 1, '\0');
    st = sd_groups_diag_json(gs, h.n_qubits(), js.data(), js.size(), &len);
    js.resize(len);
    sd_groups_destroy(gs);
    sd_hamiltonian_destroy(hh);
    if (st != SD_OK) fail(st);
    if (a.has("out")) {
        std::ofstream out(a.get("out"));
        out << js << '\n';
    } else {
        std::cout << js << '\n';
    }
    return 0;
}

int cmd_run(const Args& a) {
    if (a.pos.empty()) throw std::invalid_argument("run needs a hamiltonian file");
    const Hamiltonian h = load_file(a.pos[0]);
    const int n = h.n_qubits();
    const double t = std::stod(a.get("t", "0"));
    const int steps = std::stoi(a.get("steps", "1"));
    const std::string method = a.get("method", "grouped");
    if (method != "grouped" && method != "baseline") throw std::invalid_argument("--method grouped|baseline");
    const auto parts = greedy_partition(h);
    const auto groups = synthesize(parts);
    StateVector psi = initial(a.get("init", "zero"), n);
    const StateVector start = initial(a.get("init", "zero"), n);
    EvolutionPlan one;
    one.n_steps = 1;
    one.total_time = steps > 0 ? t / steps : 0.0;
    std::ofstream csv_file;
    std::ostream* csv = &std::cout;
    if (a.has("csv")) {
        csv_file.open(a.get("csv"));
        csv = &csv_file;
    }
    *csv << "step,time,energy\n";
    csv->precision(17);
    *csv << 0 << ',' << 0.0 << ',' << expectation(h, psi) << '\n';
    const auto t0 = std::chrono::steady_clock::now();
    for (int k = 1; k <= steps; ++k) {
        if (method == "grouped") evolve_grouped(groups, psi, one);
        else evolve_baseline(h, psi, one);
        *csv << k << ',' << one.total_time * k << ',' << expectation(h, psi) << '\n';
    }
    const double secs = seconds_since(t0);
    std::fprintf(stderr, "n=%d m=%zu n_g=%zu method=%s dt=%.17g steps=%d wall_s=%.3f final_norm=%.17g\n", n,
                 h.term_count(), groups.size(), method.c_str(), one.total_time, steps, secs, norm(psi));
    if (a.has("verify")) {
        // the same Trotter product as a group-major per-term baseline
        // (SPEC driver equivalence): fidelity deficit must vanish
        StateVector ref = initial(a.get("init", "zero"), n);
        EvolutionPlan p;
        p.n_steps = steps;
        p.total_time = t;
        evolve_baseline(std::span<const CommutingGroup>(parts), ref, p);
        if (method == "baseline") {
            ref = initial(a.get("init", "zero"), n);
            evolve_baseline(h, ref, p);
        }
        const double deficit = 1.0 - fidelity(psi, ref);
        std::fprintf(stderr, "verify: fidelity deficit vs %s = %.3e\n",
                     method == "grouped" ? "group-major baseline" : "baseline", deficit);
        if (!(std::fabs(deficit) < 1e-10)) throw std::runtime_error("verify: fidelity deficit above 1e-10");
    }
    (void)start;
    return 0;
}

double median(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v.empty() ? 0.0 : v[v.size() / 2];
}

int cmd_bench(const Args& a) {
    const std::string model = a.get("model", "tfim");
    const std::string q = a.get("qubits", "10");
    const size_t colon = q.find(':');
    const int n0 = std::stoi(q.substr(0, colon)), n1 = colon == std::string::npos ? n0 : std::stoi(q.substr(colon + 1));
    const int repeats = std::max(1, std::stoi(a.get("repeats", "5")));
    const std::uint64_t seed = std::stoull(a.get("seed", "0"));
    std::printf("model,n_qubits,m,n_g,method,n_steps,wall_time_per_step,speedup_vs_baseline,"
                "predicted_speedup,worker_count\n");
    for (int n = n0; n <= n1; ++n) {
        const Hamiltonian h = generate(model, n, seed);
        const auto parts = greedy_partition(h);
        const auto groups = synthesize(parts);
        const PartitionStats st = partition_stats(n, parts);
        EvolutionPlan one;
        one.n_steps = 1;
        one.total_time = 0.01;
        StateVector psi = StateVector::plus_state(n);
        auto time_steps = [&](auto&& step) {
            for (int w = 0; w < 3; ++w) step();  // warm-up (plans, caches) discarded
            std::vector<double> ts;
            for (int r = 0; r < repeats; ++r) {
                const auto t0 = std::chrono::steady_clock::now();
                step();
                ts.push_back(seconds_since(t0));
            }
            return median(ts);
        };
        const double tg = time_steps([&] { evolve_grouped(groups, psi, one); });
        const double tb = time_steps([&] { evolve_baseline(h, psi, one); });
        std::printf("%s,%d,%zu,%zu,grouped,1,%.6e,%.4f,%.4f,1\n", model.c_str(), n, h.term_count(), groups.size(), tg,
                    tb / tg, st.predicted_speedup);
        std::printf("%s,%d,%zu,%zu,baseline,1,%.6e,1.0,%.4f,1\n", model.c_str(), n, h.term_count(), groups.size(), tb,
                    st.predicted_speedup);
        std::fflush(stdout);
    }
    return 0;
}

int cmd_verify(const Args& a) {
    if (a.pos.empty()) throw std::invalid_argument("verify needs a hamiltonian file");
    const Hamiltonian h = load_file(a.pos[0]);
    const int n = h.n_qubits();
    const double t = std::stod(a.get("t", "0.1"));
    const int steps = std::stoi(a.get("steps", "10"));
    const auto parts = greedy_partition(h);
    const auto groups = synthesize(parts);
    EvolutionPlan p;
    p.n_steps = steps;
    p.total_time = t;
    StateVector g = StateVector::random_state(n, 1), b = StateVector::random_state(n, 1);
    evolve_grouped(groups, g, p);
    evolve_baseline(std::span<const CommutingGroup>(parts), b, p);
    const double d = 1.0 - fidelity(g, b);
    std::printf("grouped vs group-major baseline: fidelity deficit %.3e (n=%d, m=%zu, n_g=%zu, steps=%d)\n", d, n,
                h.term_count(), groups.size(), steps);
    if (n <= kExactEvolveMaxQubits) {
        const StateVector e = exact_evolve(h, StateVector::random_state(n, 1), t);
        std::printf("grouped vs exact_evolve: fidelity deficit %.3e (Trotter error)\n", 1.0 - fidelity(g, e));
    }
    if (!(std::fabs(d) < 1e-10)) throw std::runtime_error("verify: grouped and baseline evolutions differ");
    return 0;
}

void usage() {
    std::fprintf(stderr,
                 "usage: simdiag gen|partition|diag|run|bench|verify ...\n"
                 "  gen --model tfim|syk --qubits N [--seed S] [--out FILE]\n"
                 "  partition FILE [--out ASSIGNMENT]\n"
                 "  diag FILE [--out JSON]\n"
                 "  run FILE --t T --steps K [--method grouped|baseline] [--init zero|plus|neel|random[:S]]"
                 " [--csv FILE] [--verify]\n"
                 "  bench --model tfim|syk --qubits A[:B] [--repeats R] [--seed S]\n"
                 "  verify FILE [--t T] [--steps K]\n");
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return 2;
    }
    const std::string cmd = argv[1];
    try {
        const Args a = parse(argc, argv, 2);
        if (cmd == "gen") return cmd_gen(a);
        if (cmd == "partition") return cmd_partition(a);
        if (cmd == "diag") return cmd_diag(a);
        if (cmd == "run") return cmd_run(a);
        if (cmd == "bench") return cmd_bench(a);
        if (cmd == "verify") return cmd_verify(a);
        usage();
        return 2;
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "simdiag %s: %s\n", cmd.c_str(), e.what());
        return 2;
    } catch (const std::out_of_range& e) {
        std::fprintf(stderr, "simdiag %s: %s\n", cmd.c_str(), e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "simdiag %s: %s\n", cmd.c_str(), e.what());
        return 3;
    }
}
