// Device code of the fused Clifford/diagonal tile pass (north star (a)+(b)),
// shared by the compiled interpreter kernel (pass_kernel.cu) and the run-time
// specialised kernels (jit.cpp compiles this header with NVRTC).
//
// Two persistent CTAs per SM walk the tiles of a pass. A tile of 2^k
// amplitudes is loaded from HBM straight into registers (16 amplitudes per
// thread, 128-byte coalesced lines), transformed by the pass's host-compiled
// micro-program (plan_dev.h) and stored straight back: register butterflies
// for Hadamard layers, shared-memory transposes between register configs
// (pending CNOT index maps applied on the write side), pointwise quarter-turn
// phases and exp(-i dt Lambda) with per-tile Walsh-Hadamard phase tables.
//
// Reference semantics per op: proj/src/statevector.cpp:156-286
// (apply_hadamard, apply_batched_cnot, apply_phase_layer, apply_diagonal_exp).
#pragma once

#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>
#endif

#include "../plan_dev.h"

namespace sdb {
namespace dev {

// 16-byte amplitude slots (host_swz twin, see internal.hpp / plan_dev.h).
__host__ __device__ constexpr uint32_t swz(uint32_t l) {
    return l ^ ((l >> 3) & 7u) ^ ((l >> 6) & 7u) ^ ((l >> 9) & 7u);
}
// 8-byte angle-table slots: XOR the low 4 bits with bits 4-7 and 8-11 so the
// radix-16 table butterflies (lanes 16 entries apart) spread over the banks.
__device__ __forceinline__ uint32_t tsw(uint32_t u) { return u ^ ((u >> 4) & 15u) ^ ((u >> 8) & 15u); }

// gather the bits of v selected by mask into the low bits (ascending)
__device__ __forceinline__ uint32_t pext32(uint32_t v, uint32_t mask) {
    uint32_t out = 0, bit = 1;
    for (uint32_t m = mask; m; m &= m - 1, bit <<= 1) {
        if (v & m & (~m + 1u)) out |= bit;
    }
    return out;
}

// Cache hints of the tile loads/stores (timing experiments may override).
#ifndef SDB_TILE_LOAD
#define SDB_TILE_LOAD __ldcs
#endif
#ifndef SDB_TILE_STORE
#define SDB_TILE_STORE __stcs
#endif

// Ring mode (SDB_RING, specialised TMA programs): one CTA per SM runs kGroups
// warp groups of NT threads on alternate tiles of the CTA's sequence; three
// shared-memory stages rotate between them, so a tile's TMA boxes are issued
// when the tile three places earlier has finished its last transpose (about a
// tile of lead time instead of the tail of one). Group barriers are named
// barriers 1..kGroups of NT threads; barrier 0 (__syncthreads) stays CTA-wide.
#ifdef SDB_RING
constexpr int kGroups = 2;
constexpr int kStages = 3;
#else
constexpr int kGroups = 1;
constexpr int kStages = 1;
#endif
template <int NT>
__device__ __forceinline__ void gsync() {
    if constexpr (kGroups > 1) {
        asm volatile("bar.sync %0, %1;\n" ::"r"(1u + threadIdx.x / NT), "n"(NT) : "memory");
    } else {
        __syncthreads();
    }
}
// thread index within its warp group
template <int NT>
__device__ __forceinline__ uint32_t ltid() {
    return kGroups > 1 ? (threadIdx.x & (NT - 1u)) : threadIdx.x;
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}

// ---- TMA staging of tile loads (specialised kernels, SDB_TMA): one thread
// issues cp.async.bulk.tensor boxes of the tile into the transpose buffer
// once the previous tile's last transpose has read it, completing on an
// mbarrier; the LOAD op then reads its register config from shared memory.
// The tensor map (a __grid_constant__ kernel parameter) views the shard as a
// rank-5 tensor whose dimensions start at the pass's runs of consecutive local
// physical bits (host side: jit.cpp tma_spec).
struct alignas(64) TmapParam {
    unsigned long long w[16];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t mbar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mbar));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(mbar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void tma_load_5d(uint32_t dst, const void* tmap, int c0, int c1, int c2, int c3, int c4,
                                            uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(mbar)
        : "memory");
}

// TMA store of one box from shared memory (bulk async-group of the issuing thread)
__device__ __forceinline__ void tma_store_5d(const void* tmap, int c0, int c1, int c2, int c3, int c4, uint32_t src) {
    asm volatile(
        "cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group"
        " [%0, {%1, %2, %3, %4, %5}], [%6];\n" ::"l"(tmap),
        "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(src)
        : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// the thread's committed bulk stores have finished reading shared memory
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
// ... and have completed
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ void tma_prefetch_5d(const void* tmap, int c0, int c1, int c2, int c3, int c4) {
    asm volatile("cp.async.bulk.prefetch.tensor.5d.L2.global.tile [%0, {%1, %2, %3, %4, %5}];\n" ::"l"(tmap),
                 "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
                 : "memory");
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// sin/cos of a phase. Cody-Waite reduction by pi/2 and the fdlibm kernels on
// [-pi/4, pi/4] (errors < 1 ulp); arguments beyond 2^20 take CUDA's sincos.
__device__ __forceinline__ void phase_sincos(double x, double* s, double* c) {
    if (fabs(x) > 1048576.0) {
        sincos(x, s, c);
        return;
    }
    const double q = rint(x * 0.63661977236758134308);
    double r = fma(-q, 1.57079632673412561417e+00, x);
    r = fma(-q, 6.07710050650619224932e-11, r);
    r = fma(-q, 2.02226624879595063154e-21, r);
    const double z = r * r;
    const double ps = fma(z, fma(z, fma(z, fma(z, fma(z, 1.58969099521155010221e-10, -2.50507602534068634195e-08),
                                                2.75573137070700676789e-06),
                                        -1.98412698298579493134e-04),
                                8.33333333332248946124e-03),
                          -1.66666666666666324348e-01);
    const double sn = fma(r * z, ps, r);
    const double pc = z * fma(z, fma(z, fma(z, fma(z, fma(z, -1.13596475577881948265e-11, 2.08757232129817482790e-09),
                                                   -2.75573143513906633035e-07),
                                           2.48015872894767294178e-05),
                                   -1.38888888888741095749e-03),
                             4.16666666666666019037e-02);
    const double hz = 0.5 * z;
    const double w = 1.0 - hz;
    const double cs = w + (((1.0 - w) - hz) + z * pc);
    const int quad = static_cast<int>(static_cast<long long>(q) & 3);
    double so = sn, co = cs;
    if (quad & 1) {
        so = cs;
        co = -sn;
    }
    if (quad & 2) {
        so = -so;
        co = -co;
    }
    *s = so;
    *c = co;
}

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

// Swaps register coordinate J with lane bit B through warp shuffles (no
// shared memory, no block barrier): afterwards register bit J holds the
// coordinate lane bit B held and vice versa. 2^(R-1) double2 move per thread.
template <int R, int J, int B>
__device__ __forceinline__ void lane_swap(double2 (&v)[1 << R]) {
#ifdef SDB_EXPERIMENT_FASTSWAP
    // timing experiment only (wrong results): the select-free data movement
#pragma unroll
    for (int s = 0; s < (1 << R); ++s) {
        if ((s >> J) & 1) continue;
        const int s1 = s | (1 << J);
        v[s1].x = __shfl_xor_sync(0xffffffffu, v[s1].x, 1 << B);
        v[s1].y = __shfl_xor_sync(0xffffffffu, v[s1].y, 1 << B);
    }
    return;
#endif
    const bool hi = (threadIdx.x >> B) & 1u;
#pragma unroll
    for (int s = 0; s < (1 << R); ++s) {
        if ((s >> J) & 1) continue;
        const int s1 = s | (1 << J);
        double2 x = hi ? v[s] : v[s1];
        x.x = __shfl_xor_sync(0xffffffffu, x.x, 1 << B);
        x.y = __shfl_xor_sync(0xffffffffu, x.y, 1 << B);
        if (hi) v[s] = x;
        else v[s1] = x;
    }
}

// Butterfly on the coordinate held by lane bit B: the low lane gets a + d, the
// high lane a - d (fma with +-1 rounds exactly like the register butterfly's
// add / subtract, so the result is bit-identical). 2 shuffles per double, no
// selects, config unchanged.
template <int R, int B>
__device__ __forceinline__ void lane_bfly(double2 (&v)[1 << R]) {
    const double sg = ((threadIdx.x >> B) & 1u) ? -1.0 : 1.0;
#pragma unroll
    for (int s = 0; s < (1 << R); ++s) {
        const double yx = __shfl_xor_sync(0xffffffffu, v[s].x, 1 << B);
        const double yy = __shfl_xor_sync(0xffffffffu, v[s].y, 1 << B);
        v[s] = make_double2(fma(sg, v[s].x, yx), fma(sg, v[s].y, yy));
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

// One radix-2^RB round of the in-place table WHT over compact coordinates
// LO..LO+RB-1 (the swizzle is linear: slot(base | s << LO) = tsw(base) ^ tsw(s << LO)).
template <int NT, int LO, int RB>
__device__ __forceinline__ void wht_round(double* __restrict__ tab, int size) {
    constexpr int M = 1 << RB;
    const int groups = size >> RB;
    constexpr uint32_t lowm = (1u << LO) - 1u;
    for (int gi = static_cast<int>(ltid<NT>()); gi < groups; gi += NT) {
        const uint32_t g = static_cast<uint32_t>(gi);
        const uint32_t b = tsw(((g >> LO) << (LO + RB)) | (g & lowm));
        double w[M];
#pragma unroll
        for (int s = 0; s < M; ++s) w[s] = tab[b ^ tsw(static_cast<uint32_t>(s) << LO)];
#pragma unroll
        for (int j = 0; j < RB; ++j)
#pragma unroll
            for (int s = 0; s < M; ++s) {
                if ((s >> j) & 1) continue;
                const double a = w[s], d = w[s | (1 << j)];
                w[s] = a + d;
                w[s | (1 << j)] = a - d;
            }
#pragma unroll
        for (int s = 0; s < M; ++s) tab[b ^ tsw(static_cast<uint32_t>(s) << LO)] = w[s];
    }
}

// Radix-4 rounds (the tables are built while the tile's loads are in flight,
// so the round keeps few registers live).
template <int NT, int LO, int BITS>
__device__ __forceinline__ void wht_rounds(double* __restrict__ tab) {
    if constexpr (LO < BITS) {
        constexpr int RB = BITS - LO >= 2 ? 2 : 1;
        wht_round<NT, LO, RB>(tab, 1 << BITS);
        gsync<NT>();
        wht_rounds<NT, LO + RB, BITS>(tab);
    }
}

template <int NT, int BITS>
__device__ __forceinline__ void wht_fixed(double* __restrict__ tab) {
    wht_rounds<NT, 0, BITS>(tab);
}

// In-place WHT of a 2^bits table (tsw-swizzled); ends with a barrier.
template <int NT>
__device__ void wht_table(double* __restrict__ tab, int bits) {
    switch (bits) {
#define SDB_W(BB) \
    case BB: wht_fixed<NT, BB>(tab); break;
        SDB_W(1) SDB_W(2) SDB_W(3) SDB_W(4) SDB_W(5) SDB_W(6) SDB_W(7) SDB_W(8) SDB_W(9) SDB_W(10) SDB_W(11)
        SDB_W(12)
#undef SDB_W
        default: break;
    }
}

// Factor tables of one tile, every thread computing entries directly: entry
// u of factor f (entries of all factors numbered consecutively) is
//   E_f[u] = exp(-i dt sum_{segments s of f} A_s (-1)^{popc(u & u_s)}) (* sc),
// A_s = sum_{terms q of s} c_q (-1)^{popc(h & zh_q)} -- a handful of terms per
// factor, so no transform pass and no cross-thread exchange is needed.
template <int NT>
__device__ __forceinline__ void build_factor_tables(double* __restrict__ tab, const PlanDev& plan, const PointDev& pt,
                                                    uint64_t full, double neg_dt, double tscale) {
    const uint64_t* zh = plan.term_hmask + pt.term_off;
    const double* cf = plan.term_coeffs + pt.term_off;
    const SegDev* segs = plan.segs + pt.seg_off;
    const int n0 = 1 << pt.fac_bits[0];
    const int n1 = pt.n_fac > 1 ? 1 << pt.fac_bits[1] : 0;
    const int n2 = pt.n_fac > 2 ? 1 << pt.fac_bits[2] : 0;
    for (int e = static_cast<int>(ltid<NT>()); e < n0 + n1 + n2; e += NT) {
        const int f = e < n0 ? 0 : (e < n0 + n1 ? 1 : 2);
        const uint32_t u = static_cast<uint32_t>(e - (f == 0 ? 0 : (f == 1 ? n0 : n0 + n1)));
        double th = 0.0;
        for (int sg = pt.fac_sbeg[f]; sg < pt.fac_send[f]; ++sg) {
            const SegDev d = segs[sg];
            double acc = 0.0;
            for (int q = d.begin; q < d.end; ++q) {
                const uint64_t par = __popcll(full & __ldg(zh + q)) & 1ull;
                acc += __longlong_as_double(__double_as_longlong(__ldg(cf + q)) ^ static_cast<long long>(par << 63));
            }
            th += (__popc(u & d.u) & 1) ? -acc : acc;
        }
        double sn, cs;
        phase_sincos(neg_dt * th, &sn, &cs);
        const double sc = f == 0 ? tscale : 1.0;
        reinterpret_cast<double2*>(tab + pt.fac_coff[f])[swz(u)] = make_double2(cs * sc, sn * sc);
    }
}

// exp(-i dt theta_0(t)) of a pass's tile-constant table terms for tile t
// (tile index in the pass's own tile order).
__device__ __forceinline__ double2 tile_constant_phase(const PlanDev& plan, const PassDev& P, uint64_t t,
                                                      uint64_t rank_bits, double neg_dt) {
    uint64_t base = 0;
    for (int j = 0; j < P.n_outer; ++j)
        if ((t >> j) & 1ull) base |= 1ull << P.opos[j];
    const uint64_t full = rank_bits | base;
    const PointDev& pt = plan.points[P.table_point];
    const SegDev d = plan.segs[pt.seg_off + pt.c0_seg];
    double th = 0.0;
    for (int q = d.begin; q < d.end; ++q) {
        const uint64_t par = __popcll(full & plan.term_hmask[pt.term_off + q]) & 1ull;
        th += __longlong_as_double(__double_as_longlong(plan.term_coeffs[pt.term_off + q]) ^
                                   static_cast<long long>(par << 63));
    }
    double sn, cs;
    phase_sincos(neg_dt * th, &sn, &cs);
    return make_double2(cs, sn);
}

// Per-tile tables of the pass's table point, built while the tile's loads
// are in flight. Factor mode: warp f builds factor f's complex table
// E_f = exp(-i dt theta_f) (E_0 carries table_scale) -- two block barriers
// per tile. Full mode: angle table A[u] from the term segments, WHT over the
// table_bits compact coordinates (phi/(-dt) per local index).
template <int NT>
__device__ void build_tables(double* __restrict__ tab, const PlanDev& plan, const PointDev& pt, uint64_t full,
                             double neg_dt, double tscale, bool nosync) {
    const int tid = static_cast<int>(ltid<NT>());
    if (pt.n_fac > 0 && nosync) {
        // double-buffered tables; the program's transposes order the writes
        // before the POINT reads and this tile's reads before the reuse
        build_factor_tables<NT>(tab, plan, pt, full, neg_dt, tscale);
        return;
    }
    gsync<NT>();  // previous tile's readers are done with tab
    if (pt.n_fac > 0) {
        build_factor_tables<NT>(tab, plan, pt, full, neg_dt, tscale);
        gsync<NT>();
        return;
    }
    for (int u = tid; u < (1 << pt.table_bits); u += NT) tab[u] = 0.0;
    gsync<NT>();
    const uint64_t* zh = plan.term_hmask + pt.term_off;
    const double* cf = plan.term_coeffs + pt.term_off;
    for (int s = tid; s < pt.n_seg; s += NT) {
        const SegDev sg = plan.segs[pt.seg_off + s];
        double acc = 0.0;
        for (int q = sg.begin; q < sg.end; ++q) {
            const uint64_t par = __popcll(full & __ldg(zh + q)) & 1ull;
            acc += __longlong_as_double(__double_as_longlong(__ldg(cf + q)) ^ static_cast<long long>(par << 63));
        }
        tab[tsw(sg.u)] = acc;
    }
    gsync<NT>();
    wht_table<NT>(tab, pt.table_bits);
}

template <int K, int RB>
struct Cfg {
    static constexpr int R = K < RB ? K : RB;
    static constexpr int NR = 1 << R;        // amplitudes per thread
    static constexpr int NT = 1 << (K - R);  // threads per CTA
    static constexpr int N = 1 << K;
    static constexpr int LO = K < 6 ? K : 6;
    static constexpr int HI = K - LO;
    static constexpr int MINB = K >= 12 ? 2 : 1;  // resident CTAs per SM the register budget is cut for
};

constexpr int kTbaseChunks = 4;  // outer bits covered by the tile-base tables: 4 x 7
constexpr int kPatTerms = 6;     // POINT mode 5: at most 2^6 sign patterns per tile


// Register config of the current micro-program point: the thread's register-0
// local index / swizzled slot, the local coordinate (byte j of cidx) and
// slot offset of register coordinate j, and its physical offset.
struct RegCfg {
    uint32_t tb, swt;
    uint64_t cidx;
    uint32_t swc[kMaxR];
    uint64_t coff[kMaxR];
};

// Per-CTA state of one tile pass plus the op implementations. The compiled
// interpreter (pass_kernel.cu) feeds the ops from the staged program; the
// run-time specialised kernels (jit.cpp) call the same ops in a straight line
// with the register configs as literals, so the compiler folds them.
template <int K, int RB>
struct PassCtx {
    using C = Cfg<K, RB>;
    static constexpr int R = C::R, NR = C::NR, NT = C::NT, N = C::N, LO = C::LO, HI = C::HI;

    const PassDev& P;
    const PlanDev& plan;
    const double2* psi;   // may alias out (in-place passes): no __restrict__
    double2* out;
    double2* const* xdst;  // fused exchange destinations per chunk (nullptr: local store)
    double neg_dt;
    uint64_t rank_bits, n_tiles, stride;
    uint64_t t_first, t_last;  // this CTA's tiles: strided (t_first += grid) or a contiguous block
    int tid;
    bool has_table, store_perm;
    double scale;
    double2* buf;
    double* tab;
    MicroOpDev* s_ops;
    const uint32_t* s_cfg;
    const uint32_t* s_qt;
    uint64_t *st_lo, *st_hi, *st_tbase;
    uint32_t* qt_smem;  // QT bit tables staged in shared memory
    uint64_t *off_lo, *off_hi, *s_tbase;  // s_tbase: [kTbaseChunks][128]
    uint32_t *s_pl, *s_ph;                // [3][64]
    // per tile
    uint64_t t, base, full;
    const double2* g;
    bool smem_busy;
    uint64_t last_pat;  // sign pattern the current phase tables were built for
    RegCfg rc;
    double2* pat_tab = nullptr;  // POINT mode 5: [1 << kPatTerms] phase per sign pattern of the terms
    uint32_t mbar = 0;       // TMA: mbarrier of the tile staged in buf
    uint32_t mbar2 = 0;      // TMA split stage: mbarrier of the early half (0: one stage)
    const void* tmap = nullptr;  // TMA: the tensor map (address of the __grid_constant__ parameter)
    const void* tmap_out = nullptr;  // TMA store: the same view of the output buffer
    uint32_t tma_phase = 0;  // TMA: parity of the next completion to wait for
    double2* ring = nullptr; // ring mode: the kStages tile stages
    uint32_t mbar0 = 0;      // ring mode: the 2 kStages mbarriers (see set_stage)
    uint64_t ring_i = 0;     // ring mode: index of the current tile in this CTA's sequence
    uint64_t ahead;          // tile distance of the TMA issue (ring: kStages tiles of this CTA)

    __device__ __forceinline__ PassCtx(const PassDev& P_, const PlanDev& plan_, const double2* psi_, double2* out_,
                                       double2* const* xdst_, double neg_dt_, uint64_t rank_bits_, uint64_t n_tiles_,
                                       unsigned char* smem_raw,
                                       uint64_t* off_lo_, uint64_t* off_hi_, uint64_t* s_tbase_, uint32_t* s_pl_,
                                       uint32_t* s_ph_, int stage_extra = 0)
        : P(P_), plan(plan_), psi(psi_), out(out_), xdst(xdst_), neg_dt(neg_dt_), rank_bits(rank_bits_), n_tiles(n_tiles_),
          off_lo(off_lo_), off_hi(off_hi_), s_tbase(s_tbase_), s_pl(s_pl_), s_ph(s_ph_) {
        tid = static_cast<int>(ltid<NT>());
        if (P.blocked) {
            // contiguous block of tiles per CTA: consecutive tiles share the
            // phase tables' sign pattern (PassDev::pat_shift)
            const uint64_t per = (n_tiles + gridDim.x - 1) / gridDim.x;
            t_first = blockIdx.x * per;
            t_last = t_first + per < n_tiles ? t_first + per : n_tiles;
            stride = 1;
        } else {
            t_first = blockIdx.x;
            t_last = n_tiles;
            stride = gridDim.x;
        }
        ahead = stride * kStages;
        has_table = P.table_point >= 0;
        last_pat = ~0ull;
        store_perm = P.store_perm != 0;
        scale = P.scale;  // exact power of two
        buf = reinterpret_cast<double2*>(smem_raw);  // transpose buffer
        ring = buf;
        // TMA split stage: stage_extra more amplitude slots after the transpose
        // buffer hold the early half of the next tile (SDB_PASS_KERNEL_BODY_TMA);
        // ring mode: kStages stages, then one table region per warp group
        double* const tab0 = reinterpret_cast<double*>(buf + kStages * N + stage_extra);
        tab = tab0 + (threadIdx.x / NT) * P.tab_words;  // per-tile tables (if any)
        // The micro-ops are staged in shared memory (the planner caps a pass's
        // length); per-thread config bases and QT tables are read through L1.
        s_ops = reinterpret_cast<MicroOpDev*>(tab0 + kGroups * P.tab_words);
        s_cfg = plan.cfg_tb + P.cfg_off;
        s_qt = reinterpret_cast<const uint32_t*>(plan.qt_words + P.qt_off);  // staged into smem in setup()
        // store-side index tables (only for passes that store through a local
        // bit permutation sigma, i.e. in front of a qubit-remap exchange)
        st_lo = reinterpret_cast<uint64_t*>(s_ops + P.n_ops);
        st_hi = st_lo + (1 << LO);
        st_tbase = st_hi + (1 << HI);
        qt_smem = reinterpret_cast<uint32_t*>(st_lo + (P.store_perm ? (1 << LO) + (1 << HI) + kTbaseChunks * 128 : 0));
    }

    // ---- stage the program and the index tables (once per launch)
    __device__ __forceinline__ void setup() {
        // every thread of the CTA (all warp groups) stages the shared tables
        const int tid = static_cast<int>(threadIdx.x);
        constexpr int NT = C::NT * kGroups;
        const int n_outer = P.n_outer;
        {
            const int4* src = reinterpret_cast<const int4*>(plan.ops + P.op_off);
            int4* dst = reinterpret_cast<int4*>(s_ops);
            const int words = P.n_ops * static_cast<int>(sizeof(MicroOpDev) / sizeof(int4));
            for (int i = tid; i < words; i += NT) dst[i] = __ldg(src + i);
        }
        for (int i = tid; i < 2 * P.n_qt_words; i += NT) qt_smem[i] = __ldg(s_qt + i);
        s_qt = qt_smem;
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
        for (int i = tid; i < kTbaseChunks * 128; i += NT) {
            const int c = i >> 7, v = i & 127;
            uint64_t o = 0, os = 0;
            for (int j = 0; j < 7; ++j) {
                const int q = 7 * c + j;
                if (q < n_outer && ((v >> j) & 1)) {
                    o |= 1ull << P.opos[q];
                    os |= 1ull << P.st_opos[q];
                }
            }
            s_tbase[i] = o;
            if (store_perm) st_tbase[i] = os;
        }
        if (store_perm) {
            for (int i = tid; i < (1 << LO); i += NT) {
                uint64_t o = 0;
                for (int j = 0; j < LO; ++j)
                    if ((i >> j) & 1) o |= 1ull << P.st_lpos[j];
                st_lo[i] = o;
            }
            for (int i = tid; i < (1 << HI); i += NT) {
                uint64_t o = 0;
                for (int j = 0; j < HI; ++j)
                    if ((i >> j) & 1) o |= 1ull << P.st_lpos[LO + j];
                st_hi[i] = o;
            }
        }
        if (has_table) {
            const PointDev& tp = plan.points[P.table_point];
            const int nf = tp.n_fac > 0 ? tp.n_fac : 1;
            for (int f = 0; f < nf; ++f) {
                const uint32_t tm = tp.n_fac > 0 ? tp.fac_mask[f] : tp.table_mask;
                const int nlo = __popc(tm & 63u);
                for (int i = tid; i < 64; i += NT) {
                    const uint32_t lo = pext32(static_cast<uint32_t>(i), tm & 63u);
                    const uint32_t hi = pext32(static_cast<uint32_t>(i), tm >> 6) << nlo;
                    // factor tables hold complex entries in amplitude-swizzled slots
                    s_pl[f * 64 + i] = tp.n_fac > 0 ? swz(lo) : tsw(lo);
                    s_ph[f * 64 + i] = tp.n_fac > 0 ? swz(hi) : tsw(hi);
                }
            }
        }
        __syncthreads();  // CTA-wide: every group reads the staged tables
    }

    __device__ __forceinline__ uint64_t tile_base(uint64_t tt) const {
        uint64_t b = 0;
#pragma unroll
        for (int c = 0; c < kTbaseChunks; ++c) b |= s_tbase[c * 128 + ((tt >> (7 * c)) & 127)];
        return b;
    }
    __device__ __forceinline__ uint64_t off_of(uint32_t l) const {
        return off_lo[l & ((1u << LO) - 1u)] | off_hi[l >> LO];
    }

    // Ring mode: tile i of this CTA's sequence is staged in stage i % kStages.
    // Each stage alternates between two mbarriers, so tile i completes barrier
    // (stage, (i / kStages) & 1) for the (i / 2 kStages)-th time. With a single
    // barrier per stage the group waiting for tile i could run ahead of the
    // other group's tile i - kStages and see that older phase's parity
    // (aliasing); with two, the previous completion of tile i's barrier is
    // tile i - 2 kStages, which the same group consumed before.
    __device__ __forceinline__ uint32_t mbar_of(uint64_t i) const {
        return mbar0 + 8u * static_cast<uint32_t>((i % kStages) * 2 + ((i / kStages) & 1u));
    }
    __device__ __forceinline__ void set_stage(uint64_t i) {
        ring_i = i;
        buf = ring + static_cast<uint32_t>(i % kStages) * N;
        mbar = mbar_of(i);
        tma_phase = static_cast<uint32_t>((i / (2 * kStages)) & 1u);
    }
    // mbarrier the boxes of tile t + ahead complete on (issued from this stage)
    __device__ __forceinline__ uint32_t mbar_next() const { return kStages > 1 ? mbar_of(ring_i + kStages) : mbar; }

    __device__ __forceinline__ void begin_tile(uint64_t tt) {
        t = tt;
        base = tile_base(tt);
        full = rank_bits | base;
        g = psi + base;
        smem_busy = true;  // smem may still be read by other threads (sync before writing)
    }
    __device__ __forceinline__ double* tabc() const { return tab; }

    // register config from the staged program (interpreter)
    __device__ __forceinline__ RegCfg cfg_of(const MicroOpDev& op) const {
        RegCfg r;
        const uint32_t w = __ldg(s_cfg + op.arg * NT + tid);
        r.tb = w & 0xffffu;
        r.swt = w >> 16;
        r.cidx = op.cidx;
#pragma unroll
        for (int j = 0; j < kMaxR; ++j) {
            r.swc[j] = op.swc[j];
            r.coff[j] = op.c_off[j];
        }
        return r;
    }

    // Register part of the physical offsets (the thread part is off_of(rc.tb)):
    // local coordinates are distinct bits, so base | thread | register ==
    // base + thread + register, and a tile address is one per-thread pointer
    // plus a per-register offset (an immediate when the JIT bakes the
    // config's offsets in).
    __device__ __forceinline__ void reg_offsets(uint64_t (&o)[NR], const uint64_t (&coff)[kMaxR]) const {
        o[0] = 0;
#pragma unroll
        for (int j = 0; j < R; ++j)
#pragma unroll
            for (int s = 0; s < (1 << j); ++s) o[s + (1 << j)] = o[s] | coff[j];
    }


    __device__ __forceinline__ void slots(uint32_t (&a)[NR]) const {
        a[0] = rc.swt;
#pragma unroll
        for (int j = 0; j < R; ++j)
#pragma unroll
            for (int s = 0; s < (1 << j); ++s) a[s + (1 << j)] = a[s] ^ rc.swc[j];
    }

    __device__ __forceinline__ void load(const RegCfg& r, double2 (&v)[NR]) {
        rc = r;
        uint64_t o[NR];
        reg_offsets(o, rc.coff);
        const uint64_t o0 = off_of(rc.tb);
        const double2* gt = g + o0;
#ifdef SDB_EXPERIMENT_NOLOAD
        // timing experiment only (wrong results): tile data from shared memory
#pragma unroll
        for (int s = 0; s < NR; ++s) v[s] = buf[(static_cast<uint32_t>(o0 + o[s]) ^ static_cast<uint32_t>(t)) & (N - 1)];
#else
#pragma unroll
        for (int s = 0; s < NR; ++s) v[s] = SDB_TILE_LOAD(gt + o[s]);
#endif
        // Pull this CTA's next tile into L2 while the current one is
        // transformed: HBM keeps streaming through the compute phase
        // without holding registers or shared memory.
#ifndef SDB_NO_PREFETCH
#ifndef SDB_PREFETCH_DIST
#define SDB_PREFETCH_DIST 1
#endif
        if (t + SDB_PREFETCH_DIST * stride < t_last) {
            const double2* gn = psi + (tile_base(t + SDB_PREFETCH_DIST * stride) + o0);
#pragma unroll
            for (int s = 0; s < NR; ++s) prefetch_l2(gn + o[s]);
        }
#endif
        // per-tile phase tables, built while the loads are in flight
        // (rebuilt only when the tile's table sign pattern changes, see PassDev::pat_shift)
        if (has_table) {
            const uint64_t pat = P.pat_shift >= 64 ? t : (t >> P.pat_shift);
            if (pat != last_pat) {
                // the previous tile's POINT may still be reading the tables when
                // no transpose (block barrier) follows it in the program
                if (last_pat != ~0ull) gsync<NT>();
                last_pat = pat;
                build_tables<NT>(tabc(), plan, plan.points[P.table_point], full, neg_dt, P.table_scale, false);
            }
        }
    }

    // LOAD from the TMA-staged tile: amplitude of local index l sits at slot
    // tsl(l) (the box layout, GF(2)-linear in l); tsl0 is this thread's
    // register-0 slot, tso[j] the slot offset of register coordinate j.
    __device__ __forceinline__ void load_tma(const RegCfg& r, double2 (&v)[NR], uint32_t tsl0,
                                             const uint32_t (&tso)[kMaxR]) {
        rc = r;
        // per-tile phase tables are built while the tile's boxes are in flight
        if (has_table) {
            const uint64_t pat = P.pat_shift >= 64 ? t : (t >> P.pat_shift);
            if (pat != last_pat) {
                if (last_pat != ~0ull) gsync<NT>();
                last_pat = pat;
                build_tables<NT>(tabc(), plan, plan.points[P.table_point], full, neg_dt, P.table_scale, false);
            }
        }
#ifndef SDB_NO_PREFETCH
        if (t + SDB_PREFETCH_DIST * stride < t_last) {
            // next tile into L2 (its TMA boxes are issued from there)
            uint64_t o[NR];
            reg_offsets(o, rc.coff);
            const double2* gn = psi + (tile_base(t + SDB_PREFETCH_DIST * stride) + off_of(rc.tb));
#pragma unroll
            for (int s = 0; s < NR; ++s) prefetch_l2(gn + o[s]);
        }
#endif
        // split stage: the early half (issued during the previous tile's
        // transposes) first, then the late half
#ifndef SDB_EXPERIMENT_NOTMA
        if (mbar2) mbar_wait(mbar2, tma_phase);
        mbar_wait(mbar, tma_phase);
#endif
        tma_phase ^= 1u;
        // slots -> buffer positions are GF(2)-affine (the split stage moves the
        // early half behind the transpose buffer): XOR-combine the offsets
        uint32_t a[NR];
        a[0] = tsl0;
#pragma unroll
        for (int j = 0; j < R; ++j)
#pragma unroll
            for (int s = 0; s < (1 << j); ++s) a[s + (1 << j)] = a[s] ^ tso[j];
#pragma unroll
        for (int s = 0; s < NR; ++s) v[s] = buf[a[s]];
    }

    // shared-memory transpose into config r; op.perm >= 0 applies a pending
    // CNOT index map on the write side
    __device__ __forceinline__ void cfg(const MicroOpDev& op, const RegCfg& r, double2 (&v)[NR]) {
        if (smem_busy) gsync<NT>();
        if (op.perm >= 0) {
            const PermDev* pm = plan.perms + op.perm;
            uint32_t sb = 0;
            for (int j = 0; j < pm->n_ctrl; ++j)
                if ((full >> pm->ctrl_phys[j]) & 1ull) sb ^= pm->flip[j];
            uint32_t l[NR];
            l[0] = rc.tb;
#pragma unroll
            for (int j = 0; j < R; ++j)
#pragma unroll
                for (int s = 0; s < (1 << j); ++s) l[s + (1 << j)] = l[s] | (1u << ((rc.cidx >> (8 * j)) & 255u));
#pragma unroll
            for (int s = 0; s < NR; ++s) {
                const uint32_t m = static_cast<uint32_t>(__ldg(&pm->lo[l[s] & 63u])) ^
                                   static_cast<uint32_t>(__ldg(&pm->hi[l[s] >> 6])) ^ sb;
                buf[m] = v[s];
            }
        } else {
            uint32_t a[NR];
            slots(a);
#pragma unroll
            for (int s = 0; s < NR; ++s) buf[a[s]] = v[s];
        }
        gsync<NT>();
        rc = r;
        {
            uint32_t a[NR];
            slots(a);
#pragma unroll
            for (int s = 0; s < NR; ++s) v[s] = buf[a[s]];
        }
        smem_busy = true;
    }

    // Transpose whose write side applies a pending CNOT map, with the map's
    // images of the register coordinates as literals: the map is GF(2)-linear
    // (PermDev lo/hi are XORs of its columns), so register s of the thread
    // lands at slot m(tb) ^ XOR_{j in s} lm[j] -- two table reads per thread
    // instead of two per amplitude.
    __device__ __forceinline__ void cfg_lin(const MicroOpDev& op, const RegCfg& r, double2 (&v)[NR],
                                            const uint32_t (&lm)[kMaxR]) {
        if (smem_busy) gsync<NT>();
        const PermDev* pm = plan.perms + op.perm;
        uint32_t sb = 0;
        for (int j = 0; j < pm->n_ctrl; ++j)
            if ((full >> pm->ctrl_phys[j]) & 1ull) sb ^= pm->flip[j];
        uint32_t m[NR];
        m[0] = static_cast<uint32_t>(__ldg(&pm->lo[rc.tb & 63u])) ^ static_cast<uint32_t>(__ldg(&pm->hi[rc.tb >> 6])) ^
               sb;
#pragma unroll
        for (int j = 0; j < R; ++j)
#pragma unroll
            for (int s = 0; s < (1 << j); ++s) m[s + (1 << j)] = m[s] ^ lm[j];
#pragma unroll
        for (int s = 0; s < NR; ++s) buf[m[s]] = v[s];
        gsync<NT>();
        rc = r;
        {
            uint32_t a[NR];
            slots(a);
#pragma unroll
            for (int s = 0; s < NR; ++s) v[s] = buf[a[s]];
        }
        smem_busy = true;
    }

    // register slot J <-> lane bit B by warp shuffles, then config r
    template <int J, int B>
    __device__ __forceinline__ void swap(const RegCfg& r, double2 (&v)[NR]) {
        if constexpr (J < R) lane_swap<R, J, B>(v);
        rc = r;
    }
    __device__ __forceinline__ void swap_any(const MicroOpDev& op, const RegCfg& r, double2 (&v)[NR]) {
        switch (op.mask) {
#define SDB_SW(J, B) \
    case (J) | ((B) << 4): swap<J, B>(r, v); break;
            SDB_SW(0, 3) SDB_SW(1, 3) SDB_SW(2, 3) SDB_SW(3, 3) SDB_SW(0, 4) SDB_SW(1, 4) SDB_SW(2, 4) SDB_SW(3, 4)
#undef SDB_SW
            default: __trap();
        }
    }

    // Phase mode of a POINT op (template parameter of point()):
    //   0 quarter turns only, 1 <= 8 terms summed directly, 2 more terms
    //   summed directly (no table left in the pass), 3 full angle table,
    //   4 factor tables (NFAC of them).
    //   5 <= kPatTerms terms: per-tile table of the 2^m sign patterns (the
    //     same angle sums as mode 1, one sincos per pattern instead of one per
    //     amplitude).
    static __device__ __forceinline__ int point_mode(const PassDev& P, const PointDev& pt, int arg) {
        if (pt.n_terms == 0) return 0;
        if (arg == P.table_point) return pt.n_fac > 0 ? 4 : 3;
        if (pt.n_terms <= kPatTerms) return 5;
        return pt.n_terms <= 8 ? 1 : 2;
    }

    // Per-op constants of a POINT in the current register config: the JIT
    // passes literals, the interpreter decodes the staged op (point_cfg).
    struct PointCfg {
        uint32_t qr;         // bit s: QT(r_s)
        uint32_t tc[kMaxR];      // full table: swizzled compact offsets of the register coordinates
        uint32_t fo[3][kMaxR];   // factor tables: swizzled compact offsets per factor
        int coffE[3];        // factor tables: double offsets in the table region
        // S/CZ quadratic form of the tile (literals in specialised kernels;
        // n_lo < 0: read PointDev's pair lists at run time)
        int quarter;         // 0: the point has no S/CZ quarter turns at all
        int tph;             // the pass multiplies by a per-tile constant phase here (MODE 4)
        int n_lo, n_oo;
        uint32_t lo[kMaxLitPairs];  // (local coordinate mask << 8) | outer physical bit
        uint64_t oo[kMaxLitPairs];  // (1 << a) | outer partners of a above a
        uint32_t s1L, s2L;
        uint64_t s1H, s2H;
    };
    __device__ __forceinline__ PointCfg point_cfg(const MicroOpDev& op, const PointDev& pt) const {
        PointCfg c;
        c.qr = static_cast<uint32_t>(op.pad);
#pragma unroll
        for (int j = 0; j < kMaxR; ++j) c.tc[j] = tsw(op.swc[j]);
#pragma unroll
        for (int f = 0; f < 3; ++f) {
            c.coffE[f] = pt.fac_coff[f];
#pragma unroll
            for (int j = 0; j < kMaxR; ++j) c.fo[f][j] = op.fo[f][j];
        }
        c.n_lo = -1;
        c.n_oo = 0;
        c.quarter = (pt.s1L | pt.s2L) != 0u || (pt.s1H | pt.s2H) != 0ull || pt.n_lo > 0 || pt.n_oo > 0 ||
                    pt.qt_word >= 0;
        c.tph = P.tphase_off >= 0;
        c.s1L = pt.s1L;
        c.s2L = pt.s2L;
        c.s1H = pt.s1H;
        c.s2H = pt.s2H;
        return c;
    }

    // pointwise S/CZ quarter turns and exp(-i dt Lambda) (PointDev)
    template <int MODE, int NFAC>
    __device__ __forceinline__ void point(const MicroOpDev& op, const PointCfg& pc, double2 (&v)[NR]) {
        const PointDev& pt = plan.points[op.arg];
        const bool scale_here = (op.mask & 1u) != 0;
        uint32_t cb[R];
#pragma unroll
        for (int j = 0; j < R; ++j) cb[j] = 1u << ((rc.cidx >> (8 * j)) & 255u);
        // ---- quarter turns: q(tb ^ r_s) = q0 + sum_{j in s} dq_j + 2 QT(r_s)  (mod 4)
        // (QT is a quadratic form: QT(a^b) = QT(a) + QT(b) + B(a,b), B bilinear)
        uint32_t m2 = pc.s2L;
        unsigned q0 = 0;
        unsigned dq[R];
#pragma unroll
        for (int j = 0; j < R; ++j) dq[j] = 0u;
        auto oo_term = [&](uint64_t m) -> unsigned {
            // 2 * bit_a * popc(full & partners(a)), a = lowest bit of m
            return ((full & m & (~m + 1ull)) != 0ull) ? 2u * __popcll(full & (m & (m - 1ull))) : 0u;
        };
        if (pc.quarter) {
        q0 = __popcll(full & pc.s1H) + 2u * __popcll(full & pc.s2H);
        if (pc.n_lo >= 0) {
#pragma unroll
            for (int j = 0; j < kMaxLitPairs; ++j)
                if (j < pc.n_lo && ((full >> (pc.lo[j] & 0xffu)) & 1ull)) m2 ^= pc.lo[j] >> 8;
#pragma unroll
            for (int j = 0; j < kMaxLitPairs; ++j)
                if (j < pc.n_oo) q0 += oo_term(pc.oo[j]);
        } else {
            for (int j = 0; j < pt.n_lo; ++j) {
                const uint32_t wl = __ldg(plan.lo_pairs + pt.lo_off + j);
                if ((full >> (wl & 0xffu)) & 1ull) m2 ^= wl >> 8;
            }
            for (int j = 0; j < pt.n_oo; ++j) q0 += oo_term(__ldg(plan.oo_pairs + pt.oo_off + j));
        }
        const uint32_t* qt = pt.qt_word >= 0 ? s_qt + 2 * pt.qt_word : nullptr;
        auto qtb = [&](uint32_t l) -> unsigned { return qt ? (qt[l >> 5] >> (l & 31u)) & 1u : 0u; };
        const unsigned qt_tb = qtb(rc.tb);
        q0 += __popc(rc.tb & pc.s1L) + 2u * (__popc(rc.tb & m2) + qt_tb);
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const unsigned bil = qt ? (qtb(rc.tb ^ cb[j]) ^ qt_tb ^ qtb(cb[j])) : 0u;
            dq[j] = __popc(cb[j] & pc.s1L) + 2u * (__popc(cb[j] & m2) + bil);
        }
        }  // pc.quarter
        // ---- table slots of this thread's registers (compact index, swizzle linear)
        uint32_t ts0 = 0, fb[3] = {0, 0, 0};
        const double2* E[3] = {nullptr, nullptr, nullptr};
        if constexpr (MODE == 3) ts0 = s_pl[rc.tb & 63u] ^ s_ph[rc.tb >> 6];
        double2 tph = make_double2(1.0, 0.0);
        if constexpr (MODE == 4) {
            if (pc.tph) tph = plan.tile_phase[P.tphase_off + t];
            const double* tb_ = tabc();
#pragma unroll
            for (int f = 0; f < NFAC; ++f) {
                fb[f] = s_pl[f * 64 + (rc.tb & 63u)] ^ s_ph[f * 64 + (rc.tb >> 6)];
                E[f] = reinterpret_cast<const double2*>(tb_ + pc.coffE[f]);
            }
        }
        // ---- direct-mode terms (few) with the tile's outer sign folded in
        double dc[(MODE == 1 || MODE == 5) ? 8 : 1];
        uint32_t dz[(MODE == 1 || MODE == 5) ? 8 : 1];
        if constexpr (MODE == 1 || MODE == 5) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                dc[q] = 0.0;
                dz[q] = 0u;
                if (q < pt.n_terms) {
                    const uint64_t par = __popcll(full & __ldg(plan.term_hmask + pt.term_off + q)) & 1ull;
                    dc[q] = __longlong_as_double(__double_as_longlong(__ldg(plan.term_coeffs + pt.term_off + q)) ^
                                                 static_cast<long long>(par << 63));
                    dz[q] = __ldg(plan.term_lmask + pt.term_off + q);
                }
            }
        }
        // mode 5: the tile's phase per sign pattern of its terms, summed in
        // term order exactly as mode 1 does per amplitude
        const double2* ptab = nullptr;
        uint32_t pidx0 = 0, pidx[R];
        if constexpr (MODE == 5) {
#pragma unroll
            for (int j = 0; j < R; ++j) pidx[j] = 0u;
#pragma unroll
            for (int q = 0; q < kPatTerms; ++q) {
                pidx0 |= static_cast<uint32_t>(__popc(rc.tb & dz[q]) & 1) << q;
#pragma unroll
                for (int j = 0; j < R; ++j) pidx[j] |= static_cast<uint32_t>(__popc(cb[j] & dz[q]) & 1) << q;
            }
        }
        if constexpr (MODE == 5) {
            // barriers on both sides: earlier readers (this tile's previous mode-5
            // POINT, the previous tile's) are done before the table is rewritten
            double2* tabp = pat_tab;
            const int m = pt.n_terms;
            gsync<NT>();
            for (int e = tid; e < (1 << m); e += NT) {
                double ang = 0.0;
#pragma unroll
                for (int q = 0; q < kPatTerms; ++q)
                    if (q < m) ang += __longlong_as_double(__double_as_longlong(dc[q]) ^
                                                           (static_cast<long long>((e >> q) & 1) << 63));
                double sn, cs;
                phase_sincos(neg_dt * ang, &sn, &cs);
                if (scale_here) {
                    sn *= scale;
                    cs *= scale;
                }
                tabp[e] = make_double2(cs, sn);
            }
            gsync<NT>();
            ptab = tabp;
        }
        // q of every register combination, one add each
        unsigned qs[NR];
        qs[0] = q0;
#pragma unroll
        for (int j = 0; j < R; ++j)
#pragma unroll
            for (int s = 0; s < (1 << j); ++s) qs[s + (1 << j)] = qs[s] + dq[j];
#pragma unroll
        for (int s2 = 0; s2 < NR; ++s2) {
            double2 a = v[s2];
            if (pc.quarter) {
                // a * i^q: swap the parts for odd q, then flip sign bits on the
                // integer pipe (re for q = 1, 2; im for q = 2, 3) -- no FP64 work
                const unsigned q = (qs[s2] + 2u * ((pc.qr >> s2) & 1u)) & 3u;
#ifdef SDB_EXPERIMENT_QT_FP64
                if (q & 2u) a = make_double2(-a.x, -a.y);  // timing comparison: negations as FP64 ops
                if (q & 1u) a = make_double2(-a.y, a.x);
#else
                if (q & 1u) a = make_double2(a.y, a.x);
                a.x = __longlong_as_double(__double_as_longlong(a.x) ^
                                           (static_cast<long long>((q ^ (q >> 1)) & 1u) << 63));
                a.y = __longlong_as_double(__double_as_longlong(a.y) ^ (static_cast<long long>((q >> 1) & 1u) << 63));
#endif
            }
            if constexpr (MODE == 4) {
                double2 e;
#pragma unroll
                for (int f = 0; f < NFAC; ++f) {
                    uint32_t x = fb[f];
#pragma unroll
                    for (int j = 0; j < R; ++j)
                        if ((s2 >> j) & 1) x ^= pc.fo[f][j];
                    const double2 t = E[f][x];
                    e = f == 0 ? t : make_double2(e.x * t.x - e.y * t.y, e.x * t.y + e.y * t.x);
                }
                // the tile's constant phase goes onto the table entry, not the
                // amplitude: e depends only on the register coordinates the
                // factors span, so registers that share them share the product
                // (common-subexpression), one complex multiply per amplitude
                if (pc.tph) e = make_double2(e.x * tph.x - e.y * tph.y, e.x * tph.y + e.y * tph.x);
                a = make_double2(a.x * e.x - a.y * e.y, a.x * e.y + a.y * e.x);
            } else if constexpr (MODE == 5) {
                // the sign pattern is GF(2)-linear in the local index: the
                // thread's base pattern XOR the patterns of its register bits
                uint32_t idx = pidx0;
#pragma unroll
                for (int j = 0; j < R; ++j)
                    if ((s2 >> j) & 1) idx ^= pidx[j];
                const double2 e = ptab[idx];
                a = make_double2(a.x * e.x - a.y * e.y, a.x * e.y + a.y * e.x);
            } else if constexpr (MODE != 0) {
                double ang = 0.0;
                uint32_t l = rc.tb;
#pragma unroll
                for (int j = 0; j < R; ++j)
                    if ((s2 >> j) & 1) l |= cb[j];
                if constexpr (MODE == 3) {
                    uint32_t ti = ts0;
#pragma unroll
                    for (int j = 0; j < R; ++j)
                        if ((s2 >> j) & 1) ti ^= pc.tc[j];
                    ang = tabc()[ti];
                } else if constexpr (MODE == 1) {
#pragma unroll
                    for (int q2 = 0; q2 < 8; ++q2) {
                        const long long sg = static_cast<long long>(__popc(l & dz[q2]) & 1u) << 63;
                        ang += __longlong_as_double(__double_as_longlong(dc[q2]) ^ sg);
                    }
                } else {
                    for (int q2 = 0; q2 < pt.n_terms; ++q2) {
                        const uint64_t zm = __ldg(plan.term_hmask + pt.term_off + q2);
                        const uint32_t zl = __ldg(plan.term_lmask + pt.term_off + q2);
                        const long long sg = static_cast<long long>((__popcll(full & zm) + __popc(l & zl)) & 1u) << 63;
                        ang += __longlong_as_double(__double_as_longlong(__ldg(plan.term_coeffs + pt.term_off + q2)) ^ sg);
                    }
                }
                double sn, cs;
                phase_sincos(neg_dt * ang, &sn, &cs);
                if (scale_here) {
                    sn *= scale;
                    cs *= scale;
                }
                a = make_double2(a.x * cs - a.y * sn, a.x * sn + a.y * cs);
            }
            v[s2] = a;
        }
    }

    // interpreter entry: decode the mode and the per-op constants at run time
    __device__ __forceinline__ void point_any(const MicroOpDev& op, double2 (&v)[NR]) {
        const PointDev& pt = plan.points[op.arg];
        const PointCfg pc = point_cfg(op, pt);
        switch (point_mode(P, pt, op.arg)) {
            case 0: point<0, 0>(op, pc, v); break;
            case 1: point<1, 0>(op, pc, v); break;
            case 5: point<5, 0>(op, pc, v); break;
            case 2: point<2, 0>(op, pc, v); break;
            case 3: point<3, 0>(op, pc, v); break;
            default:
                if (pt.n_fac == 1) point<4, 1>(op, pc, v);
                else if (pt.n_fac == 2) point<4, 2>(op, pc, v);
                else point<4, 3>(op, pc, v);
                break;
        }
    }

    // STORE through TMA (ring pipeline, plain stores): the registers go to the
    // tile's stage in box layout (slot of local index l = tsl(l), the LOAD's
    // map), then the group's warp 0 issues the boxes as bulk tensor stores
    // (Prog::tma_store_issue). The stage is reused for a later tile's load
    // only after those stores have read it (bulk wait_group.read).
    __device__ __forceinline__ void store_tma(bool sc, uint32_t tsl0, const uint32_t (&tso)[kMaxR], double2 (&v)[NR]) {
        if (smem_busy) gsync<NT>();  // every thread has read the last transpose
        uint32_t a[NR];
        a[0] = tsl0;
#pragma unroll
        for (int j = 0; j < R; ++j)
#pragma unroll
            for (int s = 0; s < (1 << j); ++s) a[s + (1 << j)] = a[s] ^ tso[j];
        if (sc) {
#pragma unroll
            for (int s = 0; s < NR; ++s) buf[a[s]] = make_double2(v[s].x * scale, v[s].y * scale);
        } else {
#pragma unroll
            for (int s = 0; s < NR; ++s) buf[a[s]] = v[s];
        }
        fence_proxy_async();  // generic-proxy writes visible to the bulk copy
        gsync<NT>();
    }

    // STORE flags: the specialised kernels pass them as a template constant
    // (F >= 0), so only the path the op takes is compiled; the interpreter
    // decodes them from the staged op (F < 0).
    static constexpr int kStPerm = 1, kStSigma = 2, kStScale = 4, kStSync = 8, kStXchg = 16;
    // with kStPerm: soff holds the physical offsets of the map's images of the
    // register coordinates (host-computed; the map and the offsets are linear)
    static constexpr int kStPermLin = 32;
    __device__ __forceinline__ int store_flags(const MicroOpDev& op) const {
        return (op.perm >= 0 ? kStPerm : 0) | (store_perm ? kStSigma : 0) | ((op.mask & 2u) ? kStScale : 0) |
               ((op.mask & 4u) ? kStSync : 0) | (P.x_bits > 0 ? kStXchg : 0);
    }

    __device__ __forceinline__ void store(const MicroOpDev& op, double2 (&v)[NR]) {
        uint64_t so[kMaxR];
#pragma unroll
        for (int j = 0; j < kMaxR; ++j) so[j] = op.c_off[j];
        store_f<-1>(op, so, v);
    }

    // soff: sigma-mapped physical offsets of the register coordinates (kStSigma)
    template <int F>
    __device__ __forceinline__ void store_f(const MicroOpDev& op, const uint64_t (&soff)[kMaxR], double2 (&v)[NR]) {
        const int f = F >= 0 ? F : store_flags(op);
        if (f & kStSync) gsync<NT>();  // cross-warp in-place store with no barrier since the load
        uint64_t o[NR];
        double2* go;
        if (f & kStSigma) {
            // sigma is a bit permutation: sigma(base | off) = sigma(base) | sigma(off)
            uint64_t sb = 0;
#pragma unroll
            for (int c = 0; c < kTbaseChunks; ++c) sb |= st_tbase[c * 128 + ((t >> (7 * c)) & 127)];
            go = out + sb;
            go += st_lo[rc.tb & ((1u << LO) - 1u)] | st_hi[rc.tb >> LO];
            reg_offsets(o, soff);
        } else if ((f & kStPerm) && (f & kStPermLin)) {
            // pending CNOT map by the addressing, linear form: physical offset
            // of register s = off(P(tb)) ^ XOR_{j in s} soff[j]
            go = out + base;
            const PermDev* pm = plan.perms + op.perm;
            uint32_t sb = 0;
            for (int j = 0; j < pm->n_ctrl; ++j)
                if ((full >> pm->ctrl_phys[j]) & 1ull) sb ^= pm->flip[j];
            const uint32_t m0 = swz(static_cast<uint32_t>(__ldg(&pm->lo[rc.tb & 63u])) ^
                                    static_cast<uint32_t>(__ldg(&pm->hi[rc.tb >> 6])) ^ sb);
            o[0] = off_of(m0);
#pragma unroll
            for (int j = 0; j < R; ++j)
#pragma unroll
                for (int s = 0; s < (1 << j); ++s) o[s + (1 << j)] = o[s] ^ soff[j];
        } else if (f & kStPerm) {
            // pending CNOT map applied by the addressing: register s (local
            // index l) goes to P(l) = swz(lo[l & 63] ^ hi[l >> 6] ^ b(h))
            go = out + base;
            const PermDev* pm = plan.perms + op.perm;
            uint32_t sb = 0;
            for (int j = 0; j < pm->n_ctrl; ++j)
                if ((full >> pm->ctrl_phys[j]) & 1ull) sb ^= pm->flip[j];
#pragma unroll
            for (int s = 0; s < NR; ++s) {
                uint32_t ls = rc.tb;
#pragma unroll
                for (int j = 0; j < R; ++j)
                    if ((s >> j) & 1) ls |= 1u << ((rc.cidx >> (8 * j)) & 255u);
                const uint32_t m = swz(static_cast<uint32_t>(__ldg(&pm->lo[ls & 63u])) ^
                                       static_cast<uint32_t>(__ldg(&pm->hi[ls >> 6])) ^ sb);
                o[s] = off_of(m);
            }
        } else {
            go = out + (base + off_of(rc.tb));
            reg_offsets(o, rc.coff);
        }
        const bool sc = (f & kStScale) != 0;
#ifdef SDB_EXPERIMENT_NOSTORE
        if (neg_dt != 1234.5) return;
#endif
        if ((f & kStXchg) && xdst) {
            // fused exchange: every amplitude goes straight to its receiving
            // rank's buffer (peer memory over NVLink), at its final position
            const uint64_t sb = static_cast<uint64_t>(go - out);
            uint64_t own = 0;
            for (int i = 0; i < P.x_bits; ++i) own |= ((rank_bits >> P.x_gpos[i]) & 1ull) << i;
            const uint64_t low = (1ull << P.x_t0) - 1ull;
            const uint64_t ownsh = own << P.x_t0;
#pragma unroll
            for (int s = 0; s < NR; ++s) {
                const uint64_t y = sb | o[s];
                double2* const d = xdst[y >> P.x_t0] + ((y & low) | ownsh);
                SDB_TILE_STORE(d, sc ? make_double2(v[s].x * scale, v[s].y * scale) : v[s]);
            }
            return;
        }
        if (sc) {
#pragma unroll
            for (int s = 0; s < NR; ++s) SDB_TILE_STORE(go + o[s], make_double2(v[s].x * scale, v[s].y * scale));
        } else {
#pragma unroll
            for (int s = 0; s < NR; ++s) SDB_TILE_STORE(go + o[s], v[s]);
        }
    }
};

// Shared memory the pass kernels declare statically, then the persistent
// loop over tiles; `prog(ctx, v)` runs one tile's micro-program.
#define SDB_PASS_KERNEL_BODY(K, RB, PROG)                                                                  \
    using Ctx = ::sdb::dev::PassCtx<K, RB>;                                                                \
    extern __shared__ __align__(16) unsigned char smem_raw[];                                              \
    __shared__ uint64_t sdb_off_lo[1 << Ctx::LO];                                                          \
    __shared__ uint64_t sdb_off_hi[1 << Ctx::HI];                                                          \
    __shared__ uint64_t sdb_tbase[::sdb::dev::kTbaseChunks * 128];                                         \
    __shared__ uint32_t sdb_pl[3 * 64], sdb_ph[3 * 64];                                                    \
    Ctx ctx(plan.passes[pass_index], plan, psi, out, xdst, neg_dt, rank_bits, n_tiles, smem_raw, sdb_off_lo, \
            sdb_off_hi, sdb_tbase, sdb_pl, sdb_ph);                                                        \
    __shared__ double2 sdb_pat[1 << ::sdb::dev::kPatTerms];                                                 \
    ctx.pat_tab = sdb_pat;                                                                                 \
    ctx.setup();                                                                                           \
    for (uint64_t t = ctx.t_first; t < ctx.t_last; t += ctx.stride) {                                      \
        ctx.begin_tile(t);                                                                                 \
        double2 v[Ctx::NR];                                                                                \
        PROG(ctx, v);                                                                                      \
    }

// TMA variant: the first tile's boxes are issued after setup; each program
// issues the next tile's boxes itself once its last transpose is done
// (Prog::tma_next), and its LOAD waits on the mbarrier. With SPLIT the next
// tile's early half goes to a half-tile stage behind the transpose buffer
// right after the program's first transpose (Prog::tma_early; mbarrier 1), the
// late half into the transpose buffer after the last one (mbarrier 0).
#define SDB_PASS_KERNEL_BODY_TMA(K, RB, PROG, SPLIT)                                                       \
    using Ctx = ::sdb::dev::PassCtx<K, RB>;                                                                \
    extern __shared__ __align__(128) unsigned char smem_raw[];                                             \
    __shared__ uint64_t sdb_off_lo[1 << Ctx::LO];                                                          \
    __shared__ uint64_t sdb_off_hi[1 << Ctx::HI];                                                          \
    __shared__ uint64_t sdb_tbase[::sdb::dev::kTbaseChunks * 128];                                         \
    __shared__ uint32_t sdb_pl[3 * 64], sdb_ph[3 * 64];                                                    \
    __shared__ __align__(8) uint64_t sdb_mbar[2];                                                          \
    Ctx ctx(plan.passes[pass_index], plan, psi, out, xdst, neg_dt, rank_bits, n_tiles, smem_raw, sdb_off_lo, \
            sdb_off_hi, sdb_tbase, sdb_pl, sdb_ph, (SPLIT) ? Ctx::N / 2 : 0);                              \
    ctx.mbar = ::sdb::dev::smem_u32(&sdb_mbar[0]);                                                         \
    ctx.mbar2 = (SPLIT) ? ::sdb::dev::smem_u32(&sdb_mbar[1]) : 0u;                                         \
    ctx.tmap = &tmap;                                                                                      \
    if (threadIdx.x == 0) {                                                                                \
        ::sdb::dev::mbar_init(ctx.mbar);                                                                   \
        if (SPLIT) ::sdb::dev::mbar_init(ctx.mbar2);                                                       \
    }                                                                                                      \
    __shared__ double2 sdb_pat[1 << ::sdb::dev::kPatTerms];                                                 \
    ctx.pat_tab = sdb_pat;                                                                                 \
    ctx.setup();                                                                                           \
    if (threadIdx.x < 32u && ctx.t_first < ctx.t_last)                                                    \
        PROG.tma_issue(ctx, ctx.tile_base(ctx.t_first), threadIdx.x, ctx.mbar);                            \
    for (uint64_t t = ctx.t_first; t < ctx.t_last; t += ctx.stride) {                                      \
        ctx.begin_tile(t);                                                                                 \
        double2 v[Ctx::NR];                                                                                \
        PROG(ctx, v);                                                                                      \
    }

// Ring variant (SDB_RING): kGroups warp groups of NT threads take alternate
// tiles of the CTA's sequence; stages 0..kStages-1 are issued after setup and
// each program re-issues its stage for the tile kStages places later once its
// last transpose is done (Prog::tma_next with ctx.ahead).
#define SDB_PASS_KERNEL_BODY_RING(K, RB, PROG)                                                             \
    using Ctx = ::sdb::dev::PassCtx<K, RB>;                                                                \
    extern __shared__ __align__(128) unsigned char smem_raw[];                                             \
    __shared__ uint64_t sdb_off_lo[1 << Ctx::LO];                                                          \
    __shared__ uint64_t sdb_off_hi[1 << Ctx::HI];                                                          \
    __shared__ uint64_t sdb_tbase[::sdb::dev::kTbaseChunks * 128];                                         \
    __shared__ uint32_t sdb_pl[3 * 64], sdb_ph[3 * 64];                                                    \
    __shared__ __align__(8) uint64_t sdb_mbar[2 * ::sdb::dev::kStages];                                    \
    Ctx ctx(plan.passes[pass_index], plan, psi, out, xdst, neg_dt, rank_bits, n_tiles, smem_raw, sdb_off_lo, \
            sdb_off_hi, sdb_tbase, sdb_pl, sdb_ph);                                                        \
    ctx.mbar0 = ::sdb::dev::smem_u32(&sdb_mbar[0]);                                                        \
    ctx.tmap = &tmap;                                                                                      \
    ctx.tmap_out = &tmap_out;                                                                              \
    if (threadIdx.x == 0) {                                                                                \
        for (int st = 0; st < 2 * ::sdb::dev::kStages; ++st) ::sdb::dev::mbar_init(ctx.mbar0 + 8u * st);   \
    }                                                                                                      \
    __shared__ double2 sdb_pat[::sdb::dev::kGroups][1 << ::sdb::dev::kPatTerms];                           \
    const uint32_t sdb_group = threadIdx.x / Ctx::NT;                                                      \
    ctx.pat_tab = sdb_pat[sdb_group];                                                                      \
    ctx.setup();                                                                                           \
    if (threadIdx.x < 32u) {                                                                               \
        for (uint64_t st = 0; st < ::sdb::dev::kStages; ++st) {                                            \
            const uint64_t tt = ctx.t_first + st * ctx.stride;                                             \
            if (tt >= ctx.t_last) break;                                                                   \
            ctx.set_stage(st);                                                                             \
            PROG.tma_issue(ctx, ctx.tile_base(tt), threadIdx.x, ctx.mbar);                                 \
        }                                                                                                  \
    }                                                                                                      \
    for (uint64_t i = sdb_group;; i += ::sdb::dev::kGroups) {                                              \
        const uint64_t t = ctx.t_first + i * ctx.stride;                                                   \
        if (t >= ctx.t_last) break;                                                                        \
        ctx.set_stage(i);                                                                                  \
        ctx.begin_tile(t);                                                                                 \
        double2 v[Ctx::NR];                                                                                \
        PROG(ctx, v);                                                                                      \
    }                                                                                                      \
    if (ctx.tid < 32) ::sdb::dev::bulk_wait0(); /* TMA stores complete before the CTA exits */

}  // namespace dev
}  // namespace sdb
