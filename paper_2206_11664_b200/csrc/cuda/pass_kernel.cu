// Fused Clifford/diagonal tile pass for sm_100a (north star (a) + (b)).
//
// Persistent CTAs (one per SM) walk the tiles of a pass. Tile t+stride is
// prefetched with cp.async into the second shared-memory buffer while tile t
// is processed, so HBM streaming overlaps the in-tile work. Each thread keeps
// 2^R amplitudes of the tile in registers and executes the pass's host-
// compiled micro-program (internal.hpp): register butterflies for Hadamard
// layers, shared-memory transposes between register configs (pending CNOT
// index maps applied on the write side), pointwise quarter-turn phases and
// exp(-i dt Lambda) with a per-tile Walsh-Hadamard angle table, and a store
// that goes straight from registers to HBM when a warp's lanes cover whole
// 128-byte lines. The program (ops + per-thread config bases) is staged in
// shared memory once per launch; the angle table is built at the start of
// each tile, before any amplitude occupies registers.
//
// Reference semantics per op: proj/src/statevector.cpp:156-286
// (apply_hadamard, apply_batched_cnot, apply_phase_layer, apply_diagonal_exp).
#include <cuda_runtime.h>

#include "../internal.hpp"

namespace sdb {

namespace {

// 16-byte amplitude slots: XOR the low 3 slot bits with bits 3-5, 6-8, 9-11
// so the 8 lanes of a quarter-warp hit distinct 16-byte bank groups for any
// three consecutive thread coordinates. GF(2)-linear (host_swz twin).
__host__ __device__ constexpr uint32_t swz(uint32_t l) {
    return l ^ ((l >> 3) & 7u) ^ ((l >> 6) & 7u) ^ ((l >> 9) & 7u);
}
// 8-byte angle-table slots: same idea over 16-element rows.
__device__ __forceinline__ uint32_t tsw(uint32_t u) { return u ^ ((u >> 4) & 15u) ^ ((u >> 8) & 15u); }

// scatter the low bits of v into the set bits of mask (ascending)
__device__ __forceinline__ uint32_t pdep32(uint32_t v, uint32_t mask) {
    uint32_t out = 0;
    for (uint32_t m = mask; m; m &= m - 1) {
        if (v & 1u) out |= m & (~m + 1u);
        v >>= 1;
    }
    return out;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// Butterflies on the register coordinates selected by the compile-time mask M.
template <int R, int M>
__device__ __forceinline__ void bfly(double2 (&v)[1 << R]) {
#pragma unroll
    for (int j = 0; j < R; ++j) {
        if (!((M >> j) & 1)) continue;
#pragma unroll
        for (int s = 0; s < (1 << R); ++s) {
            if ((s >> j) & 1) continue;
            const double2 a = v[s], d = v[s | (1 << j)];
            v[s] = cadd(a, d);
            v[s | (1 << j)] = csub(a, d);
        }
    }
}

template <int R>
__device__ __forceinline__ void bfly_dispatch(double2 (&v)[1 << R], uint32_t mask) {
    switch (mask & ((1u << R) - 1u)) {
#define SDB_B(M) \
    case M:      \
        if constexpr (M < (1 << R)) bfly<R, M>(v); \
        break;
        SDB_B(1) SDB_B(2) SDB_B(3) SDB_B(4) SDB_B(5) SDB_B(6) SDB_B(7) SDB_B(8) SDB_B(9) SDB_B(10) SDB_B(11)
        SDB_B(12) SDB_B(13) SDB_B(14) SDB_B(15)
#undef SDB_B
        default: break;
    }
}

// Angle table for one tile: A[u] from the term segments, then a real WHT
// over `tmask` (up to RT coordinates per shared-memory round trip).
template <int K, int NT>
__device__ void build_angle_table(double* __restrict__ tab, const PlanDev& plan, const PointDev& pt, uint64_t full) {
    constexpr int N = 1 << K;
    constexpr int RT = K < 4 ? K : 4;
    const int tid = threadIdx.x;
    for (int u = tid; u < N; u += NT) tab[tsw(static_cast<uint32_t>(u))] = 0.0;
    __syncthreads();
    const uint64_t* zm = plan.term_masks + pt.term_off;
    const double* cf = plan.term_coeffs + pt.term_off;
    for (int s = tid; s < pt.n_seg; s += NT) {
        const SegDev sg = plan.segs[pt.seg_off + s];
        double acc = 0.0;
        for (int q = sg.begin; q < sg.end; ++q) {
            const uint64_t par = __popcll(full & __ldg(zm + q)) & 1ull;
            acc += __longlong_as_double(__double_as_longlong(__ldg(cf + q)) ^ static_cast<long long>(par << 63));
        }
        tab[tsw(sg.u)] = acc;
    }
    __syncthreads();
    uint32_t rem = pt.table_mask;
    while (rem) {
        uint32_t cb4[RT];
        int r = 0;
#pragma unroll
        for (int j = 0; j < RT; ++j) {
            cb4[j] = rem & (~rem + 1u);
            rem &= rem - 1u;
            if (cb4[j]) ++r;
        }
        uint32_t cm = 0;
#pragma unroll
        for (int j = 0; j < RT; ++j) cm |= cb4[j];
        const uint32_t others = (static_cast<uint32_t>(N) - 1u) & ~cm;
        const int groups = N >> r;
        for (int gi = tid; gi < groups; gi += NT) {
            const uint32_t b = pdep32(static_cast<uint32_t>(gi), others);
            double w[1 << RT];
            uint32_t idx[1 << RT];
#pragma unroll
            for (int s = 0; s < (1 << RT); ++s) {
                uint32_t x = b;
                bool valid = true;
#pragma unroll
                for (int j = 0; j < RT; ++j) {
                    if ((s >> j) & 1) {
                        if (!cb4[j]) valid = false;
                        x |= cb4[j];
                    }
                }
                idx[s] = tsw(x);
                w[s] = valid ? tab[idx[s]] : 0.0;
            }
#pragma unroll
            for (int j = 0; j < RT; ++j) {
                if (!cb4[j]) continue;
#pragma unroll
                for (int s = 0; s < (1 << RT); ++s) {
                    if ((s >> j) & 1) continue;
                    const double a = w[s], d = w[s | (1 << j)];
                    w[s] = a + d;
                    w[s | (1 << j)] = a - d;
                }
            }
#pragma unroll
            for (int s = 0; s < (1 << RT); ++s) {
                bool valid = true;
#pragma unroll
                for (int j = 0; j < RT; ++j)
                    if (((s >> j) & 1) && !cb4[j]) valid = false;
                if (valid) tab[idx[s]] = w[s];
            }
        }
        __syncthreads();
    }
}

template <int K, int RB>
struct Cfg {
    static constexpr int R = K < RB ? K : RB;
    static constexpr int NR = 1 << R;        // amplitudes per thread
    static constexpr int NT = 1 << (K - R);  // threads per CTA
    static constexpr int N = 1 << K;
    static constexpr int LO = K < 6 ? K : 6;
    static constexpr int HI = K - LO;
};

template <int K, int RB>
__global__ void __launch_bounds__(Cfg<K, RB>::NT)
k_tile_pass(double2* __restrict__ psi, PlanDev plan, int pass_index, double neg_dt, uint64_t rank_bits,
            uint64_t n_tiles) {
    using C = Cfg<K, RB>;
    constexpr int R = C::R, NR = C::NR, NT = C::NT, N = C::N, LO = C::LO, HI = C::HI;
    constexpr int TB = K - R;  // thread bits
    const PassDev& P = plan.passes[pass_index];
    const int tid = threadIdx.x;
    const int n_outer = P.n_outer;
    const int n_ops = P.n_ops;
    const int n_cfg = P.n_cfg;
    const bool has_table = P.table_point >= 0;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* const ring = reinterpret_cast<double2*>(smem_raw);  // 2 tile buffers
    double* const tab = reinterpret_cast<double*>(ring + 2 * N);  // angle table (if any)
    MicroOpDev* const s_ops = reinterpret_cast<MicroOpDev*>(tab + (has_table ? N : 0));
    uint32_t* const s_cfg = reinterpret_cast<uint32_t*>(s_ops + n_ops);  // n_cfg x NT
    __shared__ uint64_t off_lo[1 << LO];
    __shared__ uint64_t off_hi[1 << HI];
    __shared__ uint64_t s_tbase[3][128];  // tile index (7 bits per chunk) -> outer offset
    __shared__ uint64_t s_offj[NR];       // offset of local index j << TB

    // ---- stage the program and the index tables (once per launch)
    {
        const int4* src = reinterpret_cast<const int4*>(plan.ops + P.op_off);
        int4* dst = reinterpret_cast<int4*>(s_ops);
        const int words = n_ops * static_cast<int>(sizeof(MicroOpDev) / sizeof(int4));
        for (int i = tid; i < words; i += NT) dst[i] = __ldg(src + i);
        for (int i = tid; i < n_cfg * NT; i += NT) s_cfg[i] = __ldg(plan.cfg_tb + P.cfg_off + i);
    }
    for (int i = tid; i < (1 << LO); i += NT) {
        uint64_t o = 0;
        for (int j = 0; j < LO; ++j)
            if ((i >> j) & 1) o |= 1ull << P.lpos[j];
        off_lo[i] = o;
    }
    for (int i = tid; i < (1 << HI); i += NT) {
        uint64_t o = 0;
        for (int j = 0; j < HI; ++j)
            if ((i >> j) & 1) o |= 1ull << P.lpos[LO + j];
        off_hi[i] = o;
    }
    for (int i = tid; i < 3 * 128; i += NT) {
        const int c = i >> 7, v = i & 127;
        uint64_t o = 0;
        for (int j = 0; j < 7; ++j) {
            const int q = 7 * c + j;
            if (q < n_outer && ((v >> j) & 1)) o |= 1ull << P.opos[q];
        }
        s_tbase[c][v] = o;
    }
    for (int j = tid; j < NR; j += NT) {
        uint64_t o = 0;
        for (int b = 0; b < R; ++b)
            if ((j >> b) & 1) o |= 1ull << P.lpos[TB + b];
        s_offj[j] = o;
    }
    const double scale = P.scale;  // exact power of two
    const PointDev* const tpt = has_table ? plan.points + P.table_point : nullptr;
    __syncthreads();

    auto tile_base = [&](uint64_t t) {
        return s_tbase[0][t & 127] | s_tbase[1][(t >> 7) & 127] | s_tbase[2][(t >> 14) & 127];
    };
    auto off_of = [&](uint32_t l) -> uint64_t { return off_lo[l & ((1u << LO) - 1u)] | off_hi[l >> LO]; };
    // prefetch: this thread copies local indices tid + j*NT (= tid | j << TB)
    const uint32_t pf_sw = swz(static_cast<uint32_t>(tid));
    const uint64_t pf_off = off_of(static_cast<uint32_t>(tid));
    auto prefetch = [&](uint64_t t, double2* dst) {
        const double2* g = psi + (tile_base(t) | pf_off);
#pragma unroll
        for (int j = 0; j < NR; ++j) {
            const uint32_t sj = swz(static_cast<uint32_t>(j) << TB);  // compile-time
            cp_async16(dst + (pf_sw ^ sj), g + s_offj[j]);
        }
        cp_async_commit();
    };

    const uint64_t stride = gridDim.x;
    uint64_t t = blockIdx.x;
    if (t < n_tiles) prefetch(t, ring);
    for (int it = 0; t < n_tiles; t += stride, ++it) {
        double2* const cb = ring + (it & 1) * N;
        cp_async_wait_all();
        __syncthreads();  // tile t resident in cb; everyone is done with the other buffer
        if (t + stride < n_tiles) prefetch(t + stride, ring + ((it + 1) & 1) * N);

        const uint64_t base = tile_base(t);
        const uint64_t full = rank_bits | base;
        double2* const g = psi + base;
        if (has_table) build_angle_table<K, NT>(tab, plan, *tpt, full);

        double2 v[NR];
        bool in_regs = false;
        uint32_t tb = 0, swt = 0;  // local index / slot of this thread's register 0
        uint32_t cidx = 0;         // local coordinate index of register coordinate j (byte j)
        uint32_t swc[R];           // slot offset of register coordinate j
#pragma unroll
        for (int j = 0; j < R; ++j) swc[j] = 0;

        for (int oi = 0; oi < n_ops; ++oi) {
            const int4 hdr = reinterpret_cast<const int4*>(s_ops + oi)[0];
            const int kind = hdr.x;
            const uint32_t mask = static_cast<uint32_t>(hdr.y);
            const int perm = hdr.z;
            const int arg = hdr.w;
            if (kind == kOpCfg) {
                if (in_regs || perm >= 0) {
                    uint32_t sb = 0;
                    const PermDev* pm = perm >= 0 ? plan.perms + perm : nullptr;
                    if (pm) {
                        for (int j = 0; j < pm->n_ctrl; ++j)
                            if ((full >> pm->ctrl_phys[j]) & 1ull) sb ^= pm->flip[j];
                    }
                    if (!in_regs) {
                        // permutation straight out of the load buffer: identity config
#pragma unroll
                        for (int j = 0; j < NR; ++j) v[j] = cb[pf_sw ^ swz(static_cast<uint32_t>(j) << TB)];
                        tb = static_cast<uint32_t>(tid);
                        cidx = 0;
#pragma unroll
                        for (int j = 0; j < R; ++j) cidx |= static_cast<uint32_t>(TB + j) << (8 * j);
                        __syncthreads();
                    }
                    if (pm) {
                        uint32_t l[NR];
                        l[0] = tb;
#pragma unroll
                        for (int j = 0; j < R; ++j)
#pragma unroll
                            for (int s = 0; s < (1 << j); ++s)
                                l[s + (1 << j)] = l[s] | (1u << ((cidx >> (8 * j)) & 255u));
#pragma unroll
                        for (int s = 0; s < NR; ++s) {
                            const uint32_t m = static_cast<uint32_t>(pm->lo[l[s] & 63u]) ^
                                               static_cast<uint32_t>(pm->hi[l[s] >> 6]) ^ sb;
                            cb[m] = v[s];
                        }
                    } else {
                        uint32_t a[NR];
                        a[0] = swt;
#pragma unroll
                        for (int j = 0; j < R; ++j)
#pragma unroll
                            for (int s = 0; s < (1 << j); ++s) a[s + (1 << j)] = a[s] ^ swc[j];
#pragma unroll
                        for (int s = 0; s < NR; ++s) cb[a[s]] = v[s];
                    }
                    __syncthreads();
                }
                const int4 ext = reinterpret_cast<const int4*>(s_ops + oi)[1];
                const uint32_t w = s_cfg[arg * NT + tid];
                tb = w & 0xffffu;
                swt = w >> 16;
                cidx = static_cast<uint32_t>(ext.z);
                swc[0] = static_cast<uint32_t>(ext.x) & 0xffffu;
                if (R > 1) swc[1 % R] = static_cast<uint32_t>(ext.x) >> 16;
                if (R > 2) swc[2 % R] = static_cast<uint32_t>(ext.y) & 0xffffu;
                if (R > 3) swc[3 % R] = static_cast<uint32_t>(ext.y) >> 16;
                {
                    uint32_t a[NR];
                    a[0] = swt;
#pragma unroll
                    for (int j = 0; j < R; ++j)
#pragma unroll
                        for (int s = 0; s < (1 << j); ++s) a[s + (1 << j)] = a[s] ^ swc[j];
#pragma unroll
                    for (int s = 0; s < NR; ++s) v[s] = cb[a[s]];
                }
                in_regs = true;
                __syncthreads();
            } else if (kind == kOpBfly) {
                bfly_dispatch<R>(v, mask);
            } else if (kind == kOpPoint) {
                const PointDev& pt = plan.points[arg];
                const bool table = arg == P.table_point;
                const bool scale_here = (mask & 1u) != 0;
                const int n_terms = pt.n_terms;
                const uint64_t s1 = pt.s1, s2 = pt.s2;
                // per-tile CZ pieces: local ends of local-outer pairs, outer-outer parity
                uint32_t mh = 0, cc = 0;
                for (int j = 0; j < pt.n_lo; ++j) {
                    const uint32_t wl = __ldg(plan.lo_pairs + pt.lo_off + j);
                    if ((full >> (wl & 0xffu)) & 1ull) mh ^= 1u << (wl >> 8);
                }
                for (int j = 0; j < pt.n_oo; ++j) {
                    const uint64_t m = __ldg(plan.oo_pairs + pt.oo_off + j);
                    cc ^= ((full & m) == m) ? 1u : 0u;
                }
                const uint32_t tmask = pt.table_mask;
                const uint64_t* zm = plan.term_masks + pt.term_off;
                const double* cf = plan.term_coeffs + pt.term_off;
                const uint64_t* qt = pt.qt_off >= 0 ? plan.qt_words + pt.qt_off : nullptr;
                uint32_t l[NR];
                uint64_t o[NR];
                l[0] = tb;
                o[0] = off_of(tb);
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const uint32_t cbit = 1u << ((cidx >> (8 * j)) & 255u);
                    const uint64_t coff = off_of(cbit);
#pragma unroll
                    for (int s = 0; s < (1 << j); ++s) {
                        l[s + (1 << j)] = l[s] | cbit;
                        o[s + (1 << j)] = o[s] | coff;
                    }
                }
#pragma unroll
                for (int s = 0; s < NR; ++s) {
                    const uint64_t i = full | o[s];
                    uint32_t czp = cc ^ (__popc(l[s] & mh) & 1u);
                    if (qt) czp ^= static_cast<uint32_t>((__ldg(qt + (l[s] >> 6)) >> (l[s] & 63u)) & 1ull);
                    const unsigned q = (__popcll(i & s1) + 2u * __popcll(i & s2) + 2u * czp) & 3u;
                    double2 a = v[s];
                    if (q & 2u) a = make_double2(-a.x, -a.y);
                    if (q & 1u) a = make_double2(-a.y, a.x);
                    if (n_terms > 0) {
                        double ang;
                        if (table) {
                            ang = tab[tsw(l[s] & tmask)];
                        } else {
                            ang = 0.0;
                            for (int q2 = 0; q2 < n_terms; ++q2) {
                                const uint64_t par = __popcll(i & __ldg(zm + q2)) & 1ull;
                                ang += __longlong_as_double(__double_as_longlong(__ldg(cf + q2)) ^
                                                            static_cast<long long>(par << 63));
                            }
                        }
                        double sn, cs;
                        sincos(neg_dt * ang, &sn, &cs);
                        if (scale_here) {
                            sn *= scale;
                            cs *= scale;
                        }
                        a = make_double2(a.x * cs - a.y * sn, a.x * sn + a.y * cs);
                    }
                    v[s] = a;
                }
            } else {  // kOpStore
                const double sc = (mask & 2u) ? scale : 1.0;
                if (mask & 1u) {
                    uint64_t o[NR];
                    o[0] = off_of(tb);
#pragma unroll
                    for (int j = 0; j < R; ++j) {
                        const uint64_t coff = off_of(1u << ((cidx >> (8 * j)) & 255u));
#pragma unroll
                        for (int s = 0; s < (1 << j); ++s) o[s + (1 << j)] = o[s] | coff;
                    }
                    if (mask & 2u) {
#pragma unroll
                        for (int s = 0; s < NR; ++s) __stcs(g + o[s], make_double2(v[s].x * sc, v[s].y * sc));
                    } else {
#pragma unroll
                        for (int s = 0; s < NR; ++s) __stcs(g + o[s], v[s]);
                    }
                } else {
                    uint32_t a[NR];
                    a[0] = swt;
#pragma unroll
                    for (int j = 0; j < R; ++j)
#pragma unroll
                        for (int s = 0; s < (1 << j); ++s) a[s + (1 << j)] = a[s] ^ swc[j];
#pragma unroll
                    for (int s = 0; s < NR; ++s) cb[a[s]] = v[s];
                    __syncthreads();
                    double2* gp = g + pf_off;
#pragma unroll
                    for (int j = 0; j < NR; ++j) {
                        const double2 x = cb[pf_sw ^ swz(static_cast<uint32_t>(j) << TB)];
                        __stcs(gp + s_offj[j], make_double2(x.x * sc, x.y * sc));
                    }
                }
            }
        }
    }
    cp_async_wait_all();
}

template <int K, int RB>
void launch_kr(StateImpl& s, const PassDev& ph, int pass_index, const PlanDev& plan, double dt, uint64_t rank_bits) {
    using C = Cfg<K, RB>;
    const bool need_table = ph.table_point >= 0;
    const size_t smem = sizeof(double2) * 2 * C::N + (need_table ? sizeof(double) * C::N : 0) +
                        sizeof(MicroOpDev) * ph.n_ops + sizeof(uint32_t) * ph.n_cfg * C::NT;
    static size_t configured = 0;
    if (smem > configured) {
        SDB_CUDA(cudaFuncSetAttribute(k_tile_pass<K, RB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        configured = smem;
    }
    int occ = 0;
    SDB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tile_pass<K, RB>, C::NT, smem));
    if (occ < 1) throw std::runtime_error("tile pass does not fit on an SM (shared memory / registers)");
    if (s.sm_count == 0) SDB_CUDA(cudaDeviceGetAttribute(&s.sm_count, cudaDevAttrMultiProcessorCount, s.device));
    const uint64_t n_tiles = 1ull << ph.n_outer;
    uint64_t grid = static_cast<uint64_t>(s.sm_count) * static_cast<uint64_t>(occ);
    if (grid > n_tiles) grid = n_tiles;
    k_tile_pass<K, RB><<<static_cast<unsigned>(grid), C::NT, smem, s.stream>>>(
        reinterpret_cast<double2*>(s.amps), plan, pass_index, -dt, rank_bits, n_tiles);
    SDB_CUDA(cudaGetLastError());
}

template <int K>
void launch_k(StateImpl& s, const PassDev& ph, int pass_index, const PlanDev& plan, double dt, uint64_t rank_bits) {
    if (ph.rbits == 3) launch_kr<K, 3>(s, ph, pass_index, plan, dt, rank_bits);
    else launch_kr<K, 4>(s, ph, pass_index, plan, dt, rank_bits);
}

}  // namespace

int max_tile_qubits() { return 12; }

void launch_tile_pass(StateImpl& s, const PassDev& ph, int pass_index, const PlanDev& plan, double dt,
                      uint64_t rank_bits) {
    switch (ph.k) {
#define SDB_K(KK) \
    case KK: launch_k<KK>(s, ph, pass_index, plan, dt, rank_bits); break;
        SDB_K(1) SDB_K(2) SDB_K(3) SDB_K(4) SDB_K(5) SDB_K(6) SDB_K(7) SDB_K(8) SDB_K(9) SDB_K(10)
        SDB_K(11) SDB_K(12)
#undef SDB_K
        default: throw std::invalid_argument("tile qubits out of range");
    }
}

}  // namespace sdb
