/*
 * simdiag_oracle.c -- CPU ORACLE for the simdiag-b200 parity tests.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product (paper_2206_11664_b200/)
 * links or calls this file; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs load it, as the checker.
 *
 * A plain-C restatement of the reference's hot path (arXiv 2206.11664
 * `simdiag`, reference root /root/reference), function by function:
 *   or_commutes            proj/src/pauli.cpp:92-98
 *   or_from_terms          proj/src/hamiltonian.cpp:36-69
 *   or_greedy_partition    proj/src/hamiltonian.cpp:135-158
 *   tab_* gate rules       proj/src/tableau.cpp:39-96
 *   rank_x                 proj/src/tableau.cpp:102-118
 *   or_independent_subset  proj/src/tableau.cpp:142-199
 *   or_diagonalize         proj/src/diagonalize.cpp:27-212 (all steps)
 *   or_random_state        proj/src/statevector.cpp:81-93, rng.hpp:15-49
 *   sv_hadamard            proj/src/statevector.cpp:156-174
 *   sv_batched_cnot        proj/src/statevector.cpp:176-203
 *   sv_phase_layer         proj/src/statevector.cpp:205-245
 *   sv_diagonal_exp        proj/src/statevector.cpp:247-286
 *   or_apply_clifford(_inv) proj/src/statevector.cpp:339-381
 *   or_evolve_grouped      proj/src/evolve.cpp:47-58 (+ S2 composition,
 *                          groups 1..G at dt/2 then G..1)
 * Parity of this restatement is pinned against (a) the reference's own
 * known-answer tests (tests/test_oracle_kat.py) and (b) the reference
 * compiled from its sources into oracle/_ref (tests/test_oracle_vs_ref.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_PAR_CUTOFF (1ull << 16) /* statevector.cpp:16 */

static inline int pc64(uint64_t v) { return __builtin_popcountll(v); }

/* ------------------------------------------------------------ Pauli / H */

int or_commutes(uint64_t ax, uint64_t az, uint64_t bx, uint64_t bz) {
    return ((pc64(ax & bz) ^ pc64(az & bx)) & 1) == 0;
}

/* Merge duplicates in first-seen order (sums in input order), then drop
 * |c| <= tol. Writes the kept terms to out_* and returns their count. */
int64_t or_from_terms(const uint64_t* x, const uint64_t* z, const double* c, int64_t m, double tol,
                      uint64_t* ox, uint64_t* oz, double* oc) {
    int64_t cap = 16;
    while (cap < 2 * m + 2) cap <<= 1;
    int64_t* slot = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
    uint64_t* ux = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(m + 1));
    uint64_t* uz = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(m + 1));
    double* uc = (double*)malloc(sizeof(double) * (size_t)(m + 1));
    int64_t nu = 0, k, kept = 0;
    for (k = 0; k < cap; ++k) slot[k] = -1;
    for (k = 0; k < m; ++k) {
        uint64_t h = (x[k] * 0x9e3779b97f4a7c15ull) ^ (z[k] + 0x632be59bd9b4e019ull);
        h ^= h >> 31;
        int64_t p = (int64_t)(h & (uint64_t)(cap - 1));
        for (;;) {
            if (slot[p] < 0) {
                slot[p] = nu;
                ux[nu] = x[k];
                uz[nu] = z[k];
                uc[nu] = c[k];
                ++nu;
                break;
            }
            if (ux[slot[p]] == x[k] && uz[slot[p]] == z[k]) {
                uc[slot[p]] += c[k];
                break;
            }
            p = (p + 1) & (cap - 1);
        }
    }
    for (k = 0; k < nu; ++k) {
        if (fabs(uc[k]) > tol) {
            ox[kept] = ux[k];
            oz[kept] = uz[k];
            oc[kept] = uc[k];
            ++kept;
        }
    }
    free(slot);
    free(ux);
    free(uz);
    free(uc);
    return kept;
}

/* First fit. group_of[k] receives term k's group; returns group count. */
int64_t or_greedy_partition(const uint64_t* x, const uint64_t* z, int64_t m, int64_t* group_of) {
    int64_t* first = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1)); /* member lists */
    int64_t* next = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
    int64_t* last = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
    int64_t ng = 0, k, g, e;
    for (k = 0; k < m; ++k) {
        int64_t home = -1;
        for (g = 0; g < ng && home < 0; ++g) {
            int ok = 1;
            for (e = first[g]; e >= 0; e = next[e]) {
                if (!or_commutes(x[k], z[k], x[e], z[e])) {
                    ok = 0;
                    break;
                }
            }
            if (ok) home = g;
        }
        next[k] = -1;
        if (home < 0) {
            home = ng++;
            first[home] = k;
            last[home] = k;
        } else {
            next[last[home]] = k;
            last[home] = k;
        }
        group_of[k] = home;
    }
    free(first);
    free(next);
    free(last);
    return ng;
}

/* ------------------------------------------------------------- tableau */

typedef struct {
    uint64_t x, z;
    int sign;
} row_t;

static inline int bit(uint64_t w, int q) { return (int)((w >> q) & 1u); }

static void tab_h(row_t* r, int64_t nr, int t) {
    for (int64_t k = 0; k < nr; ++k) {
        int xt = bit(r[k].x, t), zt = bit(r[k].z, t);
        r[k].sign ^= xt & zt;
        r[k].x = (r[k].x & ~(1ull << t)) | ((uint64_t)zt << t);
        r[k].z = (r[k].z & ~(1ull << t)) | ((uint64_t)xt << t);
    }
}
static void tab_s(row_t* r, int64_t nr, int t) {
    for (int64_t k = 0; k < nr; ++k) {
        int xt = bit(r[k].x, t), zt = bit(r[k].z, t);
        r[k].sign ^= xt & zt;
        r[k].z ^= (uint64_t)xt << t;
    }
}
static void tab_cnot(row_t* r, int64_t nr, int c, int t) {
    for (int64_t k = 0; k < nr; ++k) {
        int xc = bit(r[k].x, c), zc = bit(r[k].z, c), xt = bit(r[k].x, t), zt = bit(r[k].z, t);
        r[k].sign ^= xc & zt & (xt == zc);
        r[k].x ^= (uint64_t)xc << t;
        r[k].z ^= (uint64_t)zt << c;
    }
}
static void tab_cz(row_t* r, int64_t nr, int c, int t) {
    for (int64_t k = 0; k < nr; ++k) {
        int xc = bit(r[k].x, c), zc = bit(r[k].z, c), xt = bit(r[k].x, t), zt = bit(r[k].z, t);
        r[k].sign ^= xc & xt & (zt != zc);
        r[k].z ^= (uint64_t)xc << t;
        r[k].z ^= (uint64_t)xt << c;
    }
}

static int rank_x(const row_t* r, int64_t nr) {
    uint64_t piv[64];
    int rank = 0;
    memset(piv, 0, sizeof(piv));
    for (int64_t k = 0; k < nr; ++k) {
        uint64_t w = r[k].x;
        while (w) {
            int lead = __builtin_ctzll(w);
            if (!piv[lead]) {
                piv[lead] = w;
                ++rank;
                break;
            }
            w ^= piv[lead];
        }
    }
    return rank;
}

/* Returns the count of kept indices written to idx (final row order). */
int64_t or_independent_subset(const uint64_t* x, const uint64_t* z, int64_t m, int n, int64_t* idx) {
    typedef struct {
        uint64_t x, z;
        int64_t origin;
    } sr_t;
    sr_t* rows = (sr_t*)malloc(sizeof(sr_t) * (size_t)(m + 1));
    int64_t k, cur = 0, kept = 0;
    int col = 0;
    for (k = 0; k < m; ++k) {
        rows[k].x = x[k];
        rows[k].z = z[k];
        rows[k].origin = k;
    }
#define COLBIT(R, C) ((C) < n ? bit((R).x, (C)) : bit((R).z, (C) - n))
    while (cur < m && col < 2 * n) {
        if (!COLBIT(rows[cur], col)) {
            int64_t found = m;
            for (k = cur + 1; k < m; ++k) {
                if (COLBIT(rows[k], col)) {
                    found = k;
                    break;
                }
            }
            if (found == m) {
                ++col;
                continue;
            }
            sr_t tmp = rows[cur];
            rows[cur] = rows[found];
            rows[found] = tmp;
        }
        for (k = cur + 1; k < m; ++k) {
            if (COLBIT(rows[k], col)) {
                rows[k].x ^= rows[cur].x;
                rows[k].z ^= rows[cur].z;
            }
        }
        ++cur;
        ++col;
    }
#undef COLBIT
    for (k = 0; k < m; ++k) {
        if (rows[k].x || rows[k].z) idx[kept++] = rows[k].origin;
    }
    free(rows);
    return kept;
}

/* Circuit layout (int32 arrays sized by the caller to >= n*n*2):
 * counts[0..4] = |h_pre|, |cnots|, |czs|, |s|, |h_post|.
 * Returns 0 ok, 1 invalid_argument (empty/too many rows), 2 runtime_error
 * (X block not cleared / term keeps X). */
static int cmp_int(const void* a, const void* b) {
    int x = *(const int*)a, y = *(const int*)b;
    return (x > y) - (x < y);
}
static int cmp_pair(const void* a, const void* b) {
    const int* p = (const int*)a;
    const int* q = (const int*)b;
    if (p[0] != q[0]) return (p[0] > q[0]) - (p[0] < q[0]);
    return (p[1] > q[1]) - (p[1] < q[1]);
}

int or_diagonalize(int n, const uint64_t* x, const uint64_t* z, const double* c, int64_t m, int32_t* h_pre,
                   int32_t* cnots, int32_t* czs, int32_t* s_layer, int32_t* h_post, int64_t* counts,
                   uint64_t* z_out, double* c_out) {
    uint64_t xu = 0, zu = 0, active = 0;
    int64_t k, nh = 0, ncx = 0, ncz = 0, ns = 0, nhp = 0;
    int q, rc = 0;
    if (m <= 0) return 1;
    for (k = 0; k < m; ++k) {
        xu |= x[k];
        zu |= z[k];
    }
    for (q = 0; q < n; ++q) /* classify_columns: general = X and Z both present */
        if (bit(xu, q) && bit(zu, q)) active |= 1ull << q;

    int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
    int64_t ni = or_independent_subset(x, z, m, n, idx);
    if (ni > n) {
        free(idx);
        return 1; /* padded_to_square throws invalid_argument */
    }
    if (ni > 0) {
        row_t* tab = (row_t*)calloc((size_t)n, sizeof(row_t));
        row_t* trial = (row_t*)calloc((size_t)n, sizeof(row_t));
        for (k = 0; k < ni; ++k) {
            tab[k].x = x[idx[k]];
            tab[k].z = z[idx[k]];
        }
        /* (i) maximize_x_rank, high -> low over active columns */
        int rank = rank_x(tab, n);
        for (q = n - 1; q >= 0; --q) {
            if (!bit(active, q)) continue;
            memcpy(trial, tab, sizeof(row_t) * (size_t)n);
            tab_h(trial, n, q);
            int r2 = rank_x(trial, n);
            if (r2 > rank) {
                memcpy(tab, trial, sizeof(row_t) * (size_t)n);
                rank = r2;
                h_pre[nh++] = q;
            }
        }
        /* (ii) clear_upper_x with a row cursor advancing on pivots only */
        int64_t* prow = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
        int* pcol = (int*)malloc(sizeof(int) * (size_t)n);
        int64_t np = 0, cursor = 0;
        for (int col = 0; col < n && cursor < n; ++col) {
            if (!bit(active, col)) continue;
            if (!bit(tab[cursor].x, col)) {
                int64_t found = n;
                for (k = cursor + 1; k < n; ++k)
                    if (bit(tab[k].x, col)) {
                        found = k;
                        break;
                    }
                if (found == n) continue;
                row_t t = tab[cursor];
                tab[cursor] = tab[found];
                tab[found] = t;
            }
            for (int t = col + 1; t < n; ++t) {
                if (bit(active, t) && bit(tab[cursor].x, t)) {
                    tab_cnot(tab, n, col, t);
                    cnots[2 * ncx] = col;
                    cnots[2 * ncx + 1] = t;
                    ++ncx;
                }
            }
            prow[np] = cursor;
            pcol[np] = col;
            ++np;
            ++cursor;
        }
        /* (iii) clear_z_block */
        for (int64_t p = 0; p < np; ++p) {
            int64_t row = prow[p];
            int col = pcol[p];
            for (int j = 0; j < n; ++j) {
                if (j == col || !bit(active, j)) continue;
                if (bit(tab[row].z, j)) {
                    tab_cz(tab, n, col, j);
                    czs[2 * ncz] = col;
                    czs[2 * ncz + 1] = j;
                    ++ncz;
                }
            }
            if (bit(tab[row].z, col)) {
                tab_s(tab, n, col);
                s_layer[ns++] = col;
            }
        }
        /* (iv) x_to_z */
        for (q = 0; q < n; ++q) {
            int has = 0;
            for (k = 0; k < n && !has; ++k) has = bit(tab[k].x, q);
            if (has) {
                tab_h(tab, n, q);
                h_post[nhp++] = q;
            }
        }
        for (k = 0; k < n; ++k)
            if (tab[k].x) rc = 2;
        free(prow);
        free(pcol);
        free(tab);
        free(trial);
        /* canonical ordering: sort H/S layers, normalise + sort CZ pairs */
        qsort(h_pre, (size_t)nh, sizeof(int32_t), cmp_int);
        qsort(s_layer, (size_t)ns, sizeof(int32_t), cmp_int);
        qsort(h_post, (size_t)nhp, sizeof(int32_t), cmp_int);
        for (k = 0; k < ncz; ++k) {
            if (czs[2 * k] > czs[2 * k + 1]) {
                int32_t t = czs[2 * k];
                czs[2 * k] = czs[2 * k + 1];
                czs[2 * k + 1] = t;
            }
        }
        qsort(czs, (size_t)ncz, 2 * sizeof(int32_t), cmp_pair);
    }
    free(idx);
    counts[0] = nh;
    counts[1] = ncx;
    counts[2] = ncz;
    counts[3] = ns;
    counts[4] = nhp;
    if (rc) return rc;
    /* replay over all terms in for_each_gate order */
    row_t* all = (row_t*)calloc((size_t)m, sizeof(row_t));
    for (k = 0; k < m; ++k) {
        all[k].x = x[k];
        all[k].z = z[k];
    }
    for (k = 0; k < nh; ++k) tab_h(all, m, h_pre[k]);
    for (k = 0; k < ncx; ++k) tab_cnot(all, m, cnots[2 * k], cnots[2 * k + 1]);
    for (k = 0; k < ncz; ++k) tab_cz(all, m, czs[2 * k], czs[2 * k + 1]);
    for (k = 0; k < ns; ++k) tab_s(all, m, s_layer[k]);
    for (k = 0; k < nhp; ++k) tab_h(all, m, h_post[k]);
    for (k = 0; k < m; ++k) {
        if (all[k].x) rc = 2;
        z_out[k] = all[k].z;
        c_out[k] = all[k].sign ? -c[k] : c[k];
    }
    free(all);
    return rc;
}

/* --------------------------------------------------------- state kernels */
/* amp: 2^n complex doubles, interleaved (re, im). */

static inline uint64_t ins0(uint64_t b, int p) {
    uint64_t low = (1ull << p) - 1;
    return ((b & ~low) << 1) | (b & low);
}

void sv_hadamard(double* a, int n, int t) {
    const int64_t pairs = (int64_t)((1ull << n) >> 1);
    const uint64_t tb = 1ull << t;
    const double s = 0.7071067811865475244;
#pragma omp parallel for schedule(static) if ((1ull << n) >= OR_PAR_CUTOFF)
    for (int64_t b = 0; b < pairs; ++b) {
        uint64_t i0 = ins0((uint64_t)b, t), i1 = i0 | tb;
        double r0 = a[2 * i0], m0 = a[2 * i0 + 1], r1 = a[2 * i1], m1 = a[2 * i1 + 1];
        a[2 * i0] = (r0 + r1) * s;
        a[2 * i0 + 1] = (m0 + m1) * s;
        a[2 * i1] = (r0 - r1) * s;
        a[2 * i1 + 1] = (m0 - m1) * s;
    }
}

void sv_batched_cnot(double* a, int n, int control, uint64_t targets) {
    const int t0 = __builtin_ctzll(targets);
    const int lo = control < t0 ? control : t0, hi = control < t0 ? t0 : control;
    const int64_t quads = (int64_t)((1ull << n) >> 2);
    const uint64_t cb = 1ull << control;
#pragma omp parallel for schedule(static) if ((1ull << n) >= OR_PAR_CUTOFF)
    for (int64_t b = 0; b < quads; ++b) {
        uint64_t i = ins0(ins0((uint64_t)b, lo), hi) | cb, j = i ^ targets;
        double r = a[2 * i], m = a[2 * i + 1];
        a[2 * i] = a[2 * j];
        a[2 * i + 1] = a[2 * j + 1];
        a[2 * j] = r;
        a[2 * j + 1] = m;
    }
}

void sv_phase_layer(double* a, int n, uint64_t s_mask, const int32_t* pairs, int64_t np, int dagger) {
    const int64_t dim = (int64_t)(1ull << n);
    uint64_t* pm = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(np + 1));
    for (int64_t k = 0; k < np; ++k) pm[k] = (1ull << pairs[2 * k]) | (1ull << pairs[2 * k + 1]);
#pragma omp parallel for schedule(static) if ((uint64_t)dim >= OR_PAR_CUTOFF)
    for (int64_t b = 0; b < dim; ++b) {
        uint64_t bits = (uint64_t)b;
        unsigned p = (unsigned)pc64(bits & s_mask) & 3u, cz = 0;
        if (dagger) p = (4u - p) & 3u;
        for (int64_t k = 0; k < np; ++k) cz ^= ((bits & pm[k]) == pm[k]) ? 1u : 0u;
        unsigned quarter = (p + 2u * cz) & 3u;
        double r = a[2 * b], m = a[2 * b + 1];
        if (quarter == 1) {
            a[2 * b] = -m;
            a[2 * b + 1] = r;
        } else if (quarter == 2) {
            a[2 * b] = -r;
            a[2 * b + 1] = -m;
        } else if (quarter == 3) {
            a[2 * b] = m;
            a[2 * b + 1] = -r;
        }
    }
    free(pm);
}

void sv_diagonal_exp(double* a, int n, const uint64_t* zm, const double* cf, int64_t m, double dt) {
    const int64_t dim = (int64_t)(1ull << n);
#pragma omp parallel for schedule(static) if ((uint64_t)dim >= OR_PAR_CUTOFF)
    for (int64_t b = 0; b < dim; ++b) {
        double angle = 0.0;
        for (int64_t k = 0; k < m; ++k) {
            union {
                double d;
                uint64_t u;
            } v;
            v.d = cf[k];
            v.u ^= ((uint64_t)(pc64((uint64_t)b & zm[k]) & 1)) << 63;
            angle += v.d;
        }
        double phi = -dt * angle, cs = cos(phi), sn = sin(phi);
        double r = a[2 * b], im = a[2 * b + 1];
        a[2 * b] = r * cs - im * sn;
        a[2 * b + 1] = r * sn + im * cs;
    }
}

/* One group: layer arrays as produced by or_diagonalize. */
typedef struct {
    int64_t counts[5];
    const int32_t *h_pre, *cnots, *czs, *s_layer, *h_post;
    int64_t m;
    const uint64_t* zm;
    const double* cf;
} or_group;

static void clifford(double* a, int n, const or_group* g, int inverse) {
    int64_t k;
    uint64_t smask = 0;
    /* CNOT runs with one control */
    int64_t nr = 0;
    int* rc = (int*)malloc(sizeof(int) * (size_t)(g->counts[1] + 1));
    uint64_t* rt = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(g->counts[1] + 1));
    for (k = 0; k < g->counts[1];) {
        int c = g->cnots[2 * k];
        uint64_t t = 0;
        while (k < g->counts[1] && g->cnots[2 * k] == c) {
            t |= 1ull << g->cnots[2 * k + 1];
            ++k;
        }
        rc[nr] = c;
        rt[nr] = t;
        ++nr;
    }
    for (k = 0; k < g->counts[3]; ++k) smask |= 1ull << g->s_layer[k];
    int phase = g->counts[2] > 0 || g->counts[3] > 0;
    if (!inverse) {
        for (k = 0; k < g->counts[0]; ++k) sv_hadamard(a, n, g->h_pre[k]);
        for (k = 0; k < nr; ++k) sv_batched_cnot(a, n, rc[k], rt[k]);
        if (phase) sv_phase_layer(a, n, smask, g->czs, g->counts[2], 0);
        for (k = 0; k < g->counts[4]; ++k) sv_hadamard(a, n, g->h_post[k]);
    } else {
        for (k = 0; k < g->counts[4]; ++k) sv_hadamard(a, n, g->h_post[k]);
        if (phase) sv_phase_layer(a, n, smask, g->czs, g->counts[2], 1);
        for (k = nr - 1; k >= 0; --k) sv_batched_cnot(a, n, rc[k], rt[k]);
        for (k = 0; k < g->counts[0]; ++k) sv_hadamard(a, n, g->h_pre[k]);
    }
    free(rc);
    free(rt);
}

void or_apply_clifford(double* a, int n, const or_group* g) { clifford(a, n, g, 0); }
void or_apply_clifford_inverse(double* a, int n, const or_group* g) { clifford(a, n, g, 1); }

static void apply_group(double* a, int n, const or_group* g, double dt) {
    clifford(a, n, g, 0);
    sv_diagonal_exp(a, n, g->zm, g->cf, g->m, dt);
    clifford(a, n, g, 1);
}

void or_evolve_grouped(double* a, int n, const or_group* groups, int64_t ng, double dt, int64_t steps, int order) {
    for (int64_t s = 0; s < steps; ++s) {
        if (order == 1 || ng <= 1) {
            for (int64_t g = 0; g < ng; ++g) apply_group(a, n, &groups[g], dt);
        } else {
            for (int64_t g = 0; g < ng - 1; ++g) apply_group(a, n, &groups[g], 0.5 * dt);
            apply_group(a, n, &groups[ng - 1], dt);
            for (int64_t g = ng - 2; g >= 0; --g) apply_group(a, n, &groups[g], 0.5 * dt);
        }
    }
}

size_t or_group_size(void) { return sizeof(or_group); }

/* ------------------------------------------------------------- states */

static inline uint64_t sm64(uint64_t v) {
    v += 0x9e3779b97f4a7c15ull;
    v = (v ^ (v >> 30)) * 0xbf58476d1ce4e5b9ull;
    v = (v ^ (v >> 27)) * 0x94d049bb133111ebull;
    return v ^ (v >> 31);
}
uint64_t or_hash(uint64_t seed, uint64_t tag, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    uint64_t h = sm64(seed ^ 0x243f6a8885a308d3ull);
    h = sm64(h ^ tag);
    h = sm64(h ^ a);
    h = sm64(h ^ b);
    h = sm64(h ^ c);
    h = sm64(h ^ d);
    return h;
}
double or_gaussian(uint64_t w) {
    double u1 = (double)(sm64(w ^ 0x5bf0a8dcull) >> 11) * 0x1.0p-53;
    double u2 = (double)(sm64(w ^ 0x94d0ca12ull) >> 11) * 0x1.0p-53;
    return sqrt(-2.0 * log1p(-u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

void or_random_state(double* a, int n, uint64_t seed) {
    const uint64_t dim = 1ull << n;
    double ns = 0.0;
    for (uint64_t i = 0; i < dim; ++i) {
        double re = or_gaussian(or_hash(seed, 0x57a7eull, i, 0, 0, 0));
        double im = or_gaussian(or_hash(seed, 0x57a7eull, i, 1, 0, 0));
        a[2 * i] = re;
        a[2 * i + 1] = im;
        ns += re * re + im * im;
    }
    double inv = 1.0 / sqrt(ns);
    for (uint64_t i = 0; i < 2 * dim; ++i) a[i] *= inv;
}

double or_norm(const double* a, int n) {
    double s = 0.0;
    for (uint64_t i = 0; i < (1ull << n); ++i) s += a[2 * i] * a[2 * i] + a[2 * i + 1] * a[2 * i + 1];
    return sqrt(s);
}

int or_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
