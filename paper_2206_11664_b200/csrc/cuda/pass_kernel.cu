// Fused Clifford/diagonal tile pass for sm_100a (north star (a) + (b)).
//
// One launch = one HBM read + write of the state. CTA t owns the 2^K
// amplitudes whose physical index bits outside the pass's local set are the
// bits of t (the tile's "outer" bits); it stages them in shared memory and
// runs the pass's stage list on them:
//   WHT   - unnormalised radix-2^R butterflies over local coordinates, R <= 4
//           coordinates per shared-memory round trip, in registers;
//   CX    - a CNOT run (one control, several local targets) as an in-tile
//           swap permutation (the GF(2) index map of the run);
//   POINT - the S/CZ quarter-turn phase of apply_phase_layer and the
//           exp(-i dt Lambda) of apply_diagonal_exp, fused into one complex
//           multiply. Many-term diagonals build a per-tile angle table with a
//           Walsh-Hadamard transform in shared memory (no HBM traffic).
// The store applies the pass's exact power-of-two scale (Hadamards are
// normalised in pairs, which keeps |1-||psi||| at rounding level).
//
// Reference semantics per stage: proj/src/statevector.cpp:156-286.
#include <cuda_runtime.h>

#include "../internal.hpp"

namespace sdb {

namespace {

constexpr int kPassThreads = 256;

// 16-byte slots; XOR-swizzle the low 3 slot bits with bits 3..5 so that the
// quarter-warp phases of strided butterfly accesses hit distinct banks.
__device__ __forceinline__ int swz(int l) { return l ^ ((l >> 3) & 7); }

__device__ __forceinline__ uint32_t insert_zero32(uint32_t v, int p) {
    const uint32_t low = (1u << p) - 1u;
    return ((v & ~low) << 1) | (v & low);
}

template <int R>
__device__ __forceinline__ void wht_chunk_c(double2* __restrict__ tile, int n, const int* c) {
    const int groups = n >> R;
    for (int g = threadIdx.x; g < groups; g += kPassThreads) {
        uint32_t b = static_cast<uint32_t>(g);
#pragma unroll
        for (int j = 0; j < R; ++j) b = insert_zero32(b, c[j]);
        uint32_t idx[1 << R];
        double2 v[1 << R];
#pragma unroll
        for (int s = 0; s < (1 << R); ++s) {
            uint32_t x = b;
#pragma unroll
            for (int j = 0; j < R; ++j)
                if ((s >> j) & 1) x |= 1u << c[j];
            idx[s] = static_cast<uint32_t>(swz(static_cast<int>(x)));
            v[s] = tile[idx[s]];
        }
#pragma unroll
        for (int j = 0; j < R; ++j) {
#pragma unroll
            for (int s = 0; s < (1 << R); ++s) {
                if ((s >> j) & 1) continue;
                const double2 a = v[s], d = v[s | (1 << j)];
                v[s] = make_double2(a.x + d.x, a.y + d.y);
                v[s | (1 << j)] = make_double2(a.x - d.x, a.y - d.y);
            }
        }
#pragma unroll
        for (int s = 0; s < (1 << R); ++s) tile[idx[s]] = v[s];
    }
}

template <int R>
__device__ __forceinline__ void wht_chunk_r(double* __restrict__ tab, int n, const int* c) {
    const int groups = n >> R;
    for (int g = threadIdx.x; g < groups; g += kPassThreads) {
        uint32_t b = static_cast<uint32_t>(g);
#pragma unroll
        for (int j = 0; j < R; ++j) b = insert_zero32(b, c[j]);
        uint32_t idx[1 << R];
        double v[1 << R];
#pragma unroll
        for (int s = 0; s < (1 << R); ++s) {
            uint32_t x = b;
#pragma unroll
            for (int j = 0; j < R; ++j)
                if ((s >> j) & 1) x |= 1u << c[j];
            idx[s] = x;
            v[s] = tab[x];
        }
#pragma unroll
        for (int j = 0; j < R; ++j) {
#pragma unroll
            for (int s = 0; s < (1 << R); ++s) {
                if ((s >> j) & 1) continue;
                const double a = v[s], d = v[s | (1 << j)];
                v[s] = a + d;
                v[s | (1 << j)] = a - d;
            }
        }
#pragma unroll
        for (int s = 0; s < (1 << R); ++s) tab[idx[s]] = v[s];
    }
}

// Butterflies over every coordinate in `mask`, up to 4 per round trip.
template <bool kComplex>
__device__ void wht_stage(void* buf, int n, uint32_t mask) {
    while (mask) {
        int c[4];
        int r = 0;
        while (mask && r < 4) {
            c[r++] = __ffs(mask) - 1;
            mask &= mask - 1;
        }
        if (kComplex) {
            double2* t = static_cast<double2*>(buf);
            if (r == 4) wht_chunk_c<4>(t, n, c);
            else if (r == 3) wht_chunk_c<3>(t, n, c);
            else if (r == 2) wht_chunk_c<2>(t, n, c);
            else wht_chunk_c<1>(t, n, c);
        } else {
            double* t = static_cast<double*>(buf);
            if (r == 4) wht_chunk_r<4>(t, n, c);
            else if (r == 3) wht_chunk_r<3>(t, n, c);
            else if (r == 2) wht_chunk_r<2>(t, n, c);
            else wht_chunk_r<1>(t, n, c);
        }
        __syncthreads();
    }
}

template <int K>
__global__ void __launch_bounds__(kPassThreads)
k_tile_pass(double2* __restrict__ psi, PlanDev plan, int pass_index, double neg_dt,
            uint64_t rank_bits) {
    constexpr int N = 1 << K;
    constexpr int LO = K < 6 ? K : 6;
    constexpr int HI = K - LO;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* tile = reinterpret_cast<double2*>(smem_raw);
    double* tab = reinterpret_cast<double*>(smem_raw + sizeof(double2) * N);
    __shared__ uint64_t off_lo[1 << LO];
    __shared__ uint64_t off_hi[1 << HI];

    const PassDev& P = plan.passes[pass_index];
    const int tid = threadIdx.x;

    // outer bits of this tile
    uint64_t base = 0;
    {
        const uint64_t t = blockIdx.x;
        const int no = P.n_outer;
        for (int j = 0; j < no; ++j) base |= ((t >> j) & 1ull) << P.opos[j];
    }
    if (tid < (1 << LO)) {
        uint64_t o = 0;
#pragma unroll
        for (int j = 0; j < LO; ++j)
            if ((tid >> j) & 1) o |= 1ull << P.lpos[j];
        off_lo[tid] = o;
    }
    if (tid < (1 << HI)) {
        uint64_t o = 0;
#pragma unroll
        for (int j = 0; j < HI; ++j)
            if ((tid >> j) & 1) o |= 1ull << P.lpos[LO + j];
        off_hi[tid] = o;
    }
    __syncthreads();

    double2* __restrict__ g = psi + base;
#pragma unroll 8
    for (int l = tid; l < N; l += kPassThreads) {
        tile[swz(l)] = g[off_lo[l & ((1 << LO) - 1)] | off_hi[l >> LO]];
    }
    __syncthreads();

    const uint64_t full_base = rank_bits | base;
    const int ns = P.n_stages;
    for (int si = 0; si < ns; ++si) {
        const StageDev st = plan.stages[P.stage_off + si];
        if (st.kind == kStageWht) {
            wht_stage<true>(tile, N, st.mask);
        } else if (st.kind == kStageCx) {
            const uint32_t T = st.mask;
            const int t0 = __ffs(T) - 1;
            const bool outer_on = st.ctrl_phys >= 0 && ((full_base >> st.ctrl_phys) & 1ull);
            for (int l = tid; l < N; l += kPassThreads) {
                const bool on = st.ctrl_local >= 0 ? ((l >> st.ctrl_local) & 1) : outer_on;
                if (on && !((l >> t0) & 1)) {
                    const int a = swz(l), b = swz(l ^ static_cast<int>(T));
                    const double2 x = tile[a];
                    tile[a] = tile[b];
                    tile[b] = x;
                }
            }
            __syncthreads();
        } else {
            const PointDev pt = plan.points[st.point];
            const bool table = pt.n_seg > 0;
            if (table) {
                for (int l = tid; l < N; l += kPassThreads) tab[l] = 0.0;
                __syncthreads();
                const uint64_t* zm = plan.term_masks + pt.term_off;
                const double* cf = plan.term_coeffs + pt.term_off;
                for (int s = tid; s < pt.n_seg; s += kPassThreads) {
                    const SegDev sg = plan.segs[pt.seg_off + s];
                    double acc = 0.0;
                    for (int t = sg.begin; t < sg.end; ++t) {
                        const uint64_t par = __popcll(full_base & __ldg(zm + t)) & 1ull;
                        acc += __longlong_as_double(__double_as_longlong(__ldg(cf + t)) ^
                                                    static_cast<long long>(par << 63));
                    }
                    tab[sg.u] = acc;
                }
                __syncthreads();
                wht_stage<false>(tab, N, pt.table_mask);
            }
            const uint64_t* zm = plan.term_masks + pt.term_off;
            const double* cf = plan.term_coeffs + pt.term_off;
            const uint64_t* czm = plan.cz_masks + pt.cz_off;
            for (int l = tid; l < N; l += kPassThreads) {
                const uint64_t i = full_base | off_lo[l & ((1 << LO) - 1)] | off_hi[l >> LO];
                unsigned q = __popcll(i & pt.s1) + 2u * __popcll(i & pt.s2);
                unsigned cz = 0;
                for (int c = 0; c < pt.n_cz; ++c) {
                    const uint64_t m = __ldg(czm + c);
                    cz ^= ((i & m) == m) ? 1u : 0u;
                }
                q = (q + 2u * cz) & 3u;
                double ang;
                if (table) {
                    ang = tab[l & pt.table_mask];  // phi depends on l only through the table bits
                } else {
                    ang = 0.0;
                    for (int t = 0; t < pt.n_terms; ++t) {
                        const uint64_t par = __popcll(i & __ldg(zm + t)) & 1ull;
                        ang += __longlong_as_double(__double_as_longlong(__ldg(cf + t)) ^
                                                    static_cast<long long>(par << 63));
                    }
                }
                const int a = swz(l);
                double2 v = tile[a];
                if (q == 1) v = make_double2(-v.y, v.x);
                else if (q == 2) v = make_double2(-v.x, -v.y);
                else if (q == 3) v = make_double2(v.y, -v.x);
                if (pt.n_terms > 0) {
                    double sn, cs;
                    sincos(neg_dt * ang, &sn, &cs);
                    v = make_double2(v.x * cs - v.y * sn, v.x * sn + v.y * cs);
                }
                tile[a] = v;
            }
            __syncthreads();
        }
    }

    const double sc = P.scale;
#pragma unroll 8
    for (int l = tid; l < N; l += kPassThreads) {
        const double2 v = tile[swz(l)];
        g[off_lo[l & ((1 << LO) - 1)] | off_hi[l >> LO]] = make_double2(v.x * sc, v.y * sc);
    }
}

template <int K>
void launch_k(StateImpl& s, int pass_index, const PlanDev& plan, double dt, uint64_t rank_bits,
              bool need_table, int n_outer) {
    const size_t smem = sizeof(double2) * (size_t(1) << K) + (need_table ? sizeof(double) * (size_t(1) << K) : 0);
    static bool configured[2] = {false, false};
    if (!configured[need_table ? 1 : 0]) {
        SDB_CUDA(cudaFuncSetAttribute(k_tile_pass<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        configured[need_table ? 1 : 0] = true;
    }
    const unsigned grid = static_cast<unsigned>(1ull << n_outer);
    k_tile_pass<K><<<grid, kPassThreads, smem, s.stream>>>(reinterpret_cast<double2*>(s.amps), plan,
                                                          pass_index, -dt, rank_bits);
    SDB_CUDA(cudaGetLastError());
}

}  // namespace

int max_tile_qubits() { return 13; }

void launch_tile_pass(StateImpl& s, const PassDev& ph, int pass_index, const PlanDev& plan, double dt,
                      uint64_t rank_bits) {
    const bool tbl = (ph.flags & kPassNeedsTable) != 0;
    switch (ph.k) {
#define SDB_K(KK) \
    case KK: launch_k<KK>(s, pass_index, plan, dt, rank_bits, tbl, ph.n_outer); break;
        SDB_K(1) SDB_K(2) SDB_K(3) SDB_K(4) SDB_K(5) SDB_K(6) SDB_K(7) SDB_K(8) SDB_K(9) SDB_K(10)
        SDB_K(11) SDB_K(12) SDB_K(13)
#undef SDB_K
        default: throw std::invalid_argument("tile qubits out of range");
    }
}

}  // namespace sdb
