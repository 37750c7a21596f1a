// Single-sweep state kernels for sm_100a: initialisation, reductions and the
// reference's unfused gate sweeps (the StateVector methods of reference
// proj/src/statevector.cpp). These back the sd_apply_* entry points and the
// `fuse = 0` schedule; the Trotter hot path uses pass_kernel.cu.
//
// Memory layout: 2^n_local interleaved (re, im) doubles = double2 per
// amplitude; every kernel is a grid-stride stream over amplitudes or
// amplitude pairs with 16-byte vector loads.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "../internal.hpp"

namespace sdb {

namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(uint64_t work) {
    uint64_t blocks = (work + kThreads - 1) / kThreads;
    const uint64_t cap = 148ull * 16;  // 16 resident waves of 256-thread CTAs
    if (blocks > cap) blocks = cap;
    if (blocks == 0) blocks = 1;
    return static_cast<unsigned>(blocks);
}

__device__ __forceinline__ uint64_t insert_zero(uint64_t v, int p) {
    const uint64_t low = (1ull << p) - 1ull;
    return ((v & ~low) << 1) | (v & low);
}

// --- counter RNG, identical integer stream to reference rng.hpp:15-49
__device__ __forceinline__ uint64_t mix64(uint64_t v) {
    v += 0x9e3779b97f4a7c15ull;
    v = (v ^ (v >> 30)) * 0xbf58476d1ce4e5b9ull;
    v = (v ^ (v >> 27)) * 0x94d049bb133111ebull;
    return v ^ (v >> 31);
}
__device__ __forceinline__ uint64_t key_hash(uint64_t seed, uint64_t tag, uint64_t a, uint64_t b) {
    uint64_t h = mix64(seed ^ 0x243f6a8885a308d3ull);
    h = mix64(h ^ tag);
    h = mix64(h ^ a);
    h = mix64(h ^ b);
    h = mix64(h ^ 0ull);
    h = mix64(h ^ 0ull);
    return h;
}
__device__ __forceinline__ double unit53(uint64_t w) { return double(w >> 11) * 0x1.0p-53; }
__device__ __forceinline__ double normal_draw(uint64_t w) {
    const double u1 = unit53(mix64(w ^ 0x5bf0a8dcull));
    const double u2 = unit53(mix64(w ^ 0x94d0ca12ull));
    // Same argument rounding as the reference (2*pi*u2 in double).
    return sqrt(-2.0 * log1p(-u1)) * cos(2.0 * 3.141592653589793 * u2);
}

__global__ void k_fill(double2* __restrict__ a, uint64_t n, double re, double im) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x)
        a[i] = make_double2(re, im);
}

__global__ void k_set_one(double2* a, uint64_t idx) { a[idx] = make_double2(1.0, 0.0); }

__global__ void k_random(double2* __restrict__ a, uint64_t n, uint64_t seed, uint64_t first) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t g = first + i;
        a[i] = make_double2(normal_draw(key_hash(seed, 0x57a7eull, g, 0)),
                            normal_draw(key_hash(seed, 0x57a7eull, g, 1)));
    }
}

__global__ void k_scale(double2* __restrict__ a, uint64_t n, double f) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        double2 v = a[i];
        a[i] = make_double2(v.x * f, v.y * f);
    }
}

// Deterministic two-level reduction: block b sums a fixed strided subset in
// a fixed order, then a tree inside the block; the host-side second level
// adds the block partials in index order.
template <bool kInner>
__global__ void k_reduce(const double2* __restrict__ a, const double2* __restrict__ b, uint64_t n,
                         double2* __restrict__ partial) {
    __shared__ double2 red[kThreads];
    double sr = 0.0, si = 0.0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const double2 x = a[i];
        if (kInner) {
            const double2 y = b[i];
            sr += x.x * y.x + x.y * y.y;  // conj(x) * y
            si += x.x * y.y - x.y * y.x;
        } else {
            sr += x.x * x.x + x.y * x.y;
        }
    }
    red[threadIdx.x] = make_double2(sr, si);
    __syncthreads();
    for (int w = kThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            red[threadIdx.x].x += red[threadIdx.x + w].x;
            red[threadIdx.x].y += red[threadIdx.x + w].y;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

// <psi| P |psi> partial sums for one Pauli term P = i^{phase} X^x Z^z
// (expectation, reference evolve.cpp:99-135): sum_b conj(psi[b]) ph(b) psi[b^x],
// ph(b) = base * (-1)^{popc((b^x) & z)}; same fixed-order block partials as
// k_reduce. Sharded: b = rank_bits | i over this shard, psi[b^x] is element
// i ^ x_lo of `p` (this shard, or a copy of shard rank ^ x_hi when x has
// global bits); x and z are physical masks including the global bits.
__global__ void k_expect(const double2* __restrict__ a, const double2* __restrict__ p, uint64_t n, uint64_t x_lo,
                         uint64_t x, uint64_t z, uint64_t rank_bits, double2 base, double2* __restrict__ partial) {
    __shared__ double2 red[kThreads];
    double sr = 0.0, si = 0.0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const double2 u = a[i];
        const double2 w = p[i ^ x_lo];
        const bool odd = __popcll(((rank_bits | i) ^ x) & z) & 1;
        const double pr = odd ? -base.x : base.x, pi = odd ? -base.y : base.y;
        const double tr = pr * w.x - pi * w.y, ti = pr * w.y + pi * w.x;  // ph * psi[b^x]
        sr += u.x * tr + u.y * ti;                                        // conj(psi[b]) * (...)
        si += u.x * ti - u.y * tr;
    }
    red[threadIdx.x] = make_double2(sr, si);
    __syncthreads();
    for (int w = kThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            red[threadIdx.x].x += red[threadIdx.x + w].x;
            red[threadIdx.x].y += red[threadIdx.x + w].y;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

// exp(-i theta P) on a shard whose partner amplitudes b^x live on another
// rank (x has global bits): new[b] = cos(theta) a[b] + (-1)^{popc((b^x)&z)} w
// a[b^x], the per-amplitude form of the reference's pair update
// (statevector.cpp:313-333), with a[b^x] = element i ^ x_lo of p, a copy of
// shard rank ^ x_hi taken before the update.
__global__ void k_pauli_rotation_remote(double2* __restrict__ a, const double2* __restrict__ p, uint64_t n,
                                        uint64_t x_lo, uint64_t x, uint64_t z, uint64_t rank_bits, double c,
                                        double2 w) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const bool par = __popcll(((rank_bits | i) ^ x) & z) & 1;
        const double2 wi = par ? make_double2(-w.x, -w.y) : w;
        const double2 a0 = a[i], a1 = p[i ^ x_lo];
        a[i] = make_double2(c * a0.x + (wi.x * a1.x - wi.y * a1.y), c * a0.y + (wi.x * a1.y + wi.y * a1.x));
    }
}

// One Taylor term of exact_evolve: nxt = f * H cur, acc += nxt, with H the
// Pauli sum (H cur)[b'] = sum_k c_k i^{s_k} (-1)^{popc(z_k & (b' ^ x_k))}
// cur[b' ^ x_k] (P|b> = i^s (-1)^{<z,b>} |b^x>, reference evolve.cpp:70-79).
__global__ void k_taylor_term(const double2* __restrict__ cur, double2* __restrict__ nxt, double2* __restrict__ acc,
                              uint64_t n, const uint64_t* __restrict__ xm, const uint64_t* __restrict__ zm,
                              const double2* __restrict__ cb, int m, double2 f) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        double sr = 0.0, si = 0.0;
        for (int k = 0; k < m; ++k) {
            const uint64_t x = __ldg(xm + k);
            const double2 b = __ldg(cb + k);
            const double2 v = cur[i ^ x];
            const double sg = (__popcll(__ldg(zm + k) & (i ^ x)) & 1) ? -1.0 : 1.0;
            sr += sg * (b.x * v.x - b.y * v.y);
            si += sg * (b.x * v.y + b.y * v.x);
        }
        const double2 t = make_double2(f.x * sr - f.y * si, f.x * si + f.y * sr);
        nxt[i] = t;
        acc[i] = make_double2(acc[i].x + t.x, acc[i].y + t.y);
    }
}

// apply_single_qubit (reference statevector.cpp:101-122): one sweep over the
// pairs (i0, i0|t), u row-major 2x2 complex.
struct Mat2D {
    double2 u[4];
};
struct Mat4D {
    double2 u[16];
};
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

__global__ void k_single_qubit(double2* __restrict__ a, uint64_t pairs, int t, Mat2D m) {
    const uint64_t tb = 1ull << t;
    for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < pairs;
         q += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i0 = insert_zero(q, t), i1 = i0 | tb;
        const double2 a0 = a[i0], a1 = a[i1];
        a[i0] = cadd2(cmul(m.u[0], a0), cmul(m.u[1], a1));
        a[i1] = cadd2(cmul(m.u[2], a0), cmul(m.u[3], a1));
    }
}

// apply_two_qubit (reference statevector.cpp:124-154): local index
// 2*bit(q1) + bit(q2); row r accumulates u[r][0] v0 + u[r][1] v1 + ... in order.
__global__ void k_two_qubit(double2* __restrict__ a, uint64_t quads, int lo, int hi, uint64_t b1, uint64_t b2,
                            Mat4D m) {
    for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < quads;
         q += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i00 = insert_zero(insert_zero(q, lo), hi);
        const uint64_t idx[4] = {i00, i00 | b2, i00 | b1, i00 | b1 | b2};
        double2 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = a[idx[k]];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            double2 acc = cmul(m.u[r * 4], v[0]);
#pragma unroll
            for (int k = 1; k < 4; ++k) acc = cadd2(acc, cmul(m.u[r * 4 + k], v[k]));
            a[idx[r]] = acc;
        }
    }
}

// apply_pauli_rotation (reference statevector.cpp:288-337): exp(-i theta P).
// x == 0: a[b] *= (cos, -+sin) by the parity of b & z; otherwise over pairs
// (b, b^x): a0' = c a0 + w0 a1, a1' = c a1 + w1 a0 with w = -i sin(theta) i^{phase}
// and its sign from the parities of the pair's z bits.
__global__ void k_pauli_rotation(double2* __restrict__ a, uint64_t n, uint64_t x, uint64_t z, double c, double s,
                                 double2 w, int t0, int y_parity, uint64_t rank_bits) {
    if (x == 0) {
        for (uint64_t b = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; b < n;
             b += uint64_t(gridDim.x) * blockDim.x) {
            const bool odd = __popcll((rank_bits | b) & z) & 1;
            const double fr = c, fi = odd ? s : -s;
            const double2 v = a[b];
            a[b] = make_double2(v.x * fr - v.y * fi, v.x * fi + v.y * fr);
        }
        return;
    }
    const uint64_t pairs = n >> 1;
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < pairs;
         p += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i0 = insert_zero(p, t0);
        const uint64_t i1 = i0 ^ x;
        const bool par0 = __popcll((rank_bits | i0) & z) & 1;
        const bool par1 = par0 ^ (y_parity != 0);
        const double2 w0 = par1 ? make_double2(-w.x, -w.y) : w;
        const double2 w1 = par0 ? make_double2(-w.x, -w.y) : w;
        const double2 a0 = a[i0], a1 = a[i1];
        a[i0] = make_double2(c * a0.x + (w0.x * a1.x - w0.y * a1.y), c * a0.y + (w0.x * a1.y + w0.y * a1.x));
        a[i1] = make_double2(c * a1.x + (w1.x * a0.x - w1.y * a0.y), c * a1.y + (w1.x * a0.y + w1.y * a0.x));
    }
}

// apply_hadamard (reference statevector.cpp:156-174): one sweep over pairs,
// scaled by fl(1/sqrt2) per gate exactly as the reference does.
__global__ void k_hadamard(double2* __restrict__ a, uint64_t pairs, int t) {
    const double c = 0.7071067811865475244;
    const uint64_t tb = 1ull << t;
    for (uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; p < pairs;
         p += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i0 = insert_zero(p, t), i1 = i0 | tb;
        const double2 x = a[i0], y = a[i1];
        a[i0] = make_double2((x.x + y.x) * c, (x.y + y.y) * c);
        a[i1] = make_double2((x.x - y.x) * c, (x.y - y.y) * c);
    }
}

// apply_batched_cnot (statevector.cpp:176-203): swap amp[i] <-> amp[i^T] for
// the representative with control 1 and lowest target 0.
__global__ void k_batched_cnot(double2* __restrict__ a, uint64_t quads, int lo, int hi,
                               uint64_t cbit, uint64_t targets) {
    for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < quads;
         q += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = insert_zero(insert_zero(q, lo), hi) | cbit;
        const uint64_t j = i ^ targets;
        const double2 x = a[i];
        a[i] = a[j];
        a[j] = x;
    }
}

// apply_phase_layer (statevector.cpp:205-245): multiply by i^quarter, exact.
__global__ void k_phase_layer(double2* __restrict__ a, uint64_t n, uint64_t s_mask,
                              const uint64_t* __restrict__ pairs, int n_pairs, int dagger) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        unsigned q = __popcll(i & s_mask) & 3u;
        if (dagger) q = (4u - q) & 3u;
        unsigned cz = 0;
        for (int k = 0; k < n_pairs; ++k) {
            const uint64_t pm = __ldg(pairs + k);
            cz ^= ((i & pm) == pm) ? 1u : 0u;
        }
        q = (q + 2u * cz) & 3u;
        if (q == 0) continue;
        const double2 v = a[i];
        a[i] = q == 1 ? make_double2(-v.y, v.x) : q == 2 ? make_double2(-v.x, -v.y)
                                                         : make_double2(v.y, -v.x);
    }
}

// apply_diagonal_exp (statevector.cpp:247-286): angle summed in term order
// with the sign-bit flip, phi = -dt*angle, multiply by (cos phi, sin phi).
__global__ void k_diag_exp(double2* __restrict__ a, uint64_t n, const uint64_t* __restrict__ zm,
                           const double* __restrict__ cf, int m, double dt) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        double ang = 0.0;
        for (int k = 0; k < m; ++k) {
            const uint64_t par = __popcll(i & __ldg(zm + k)) & 1ull;
            ang += __longlong_as_double(__double_as_longlong(__ldg(cf + k)) ^ (long long)(par << 63));
        }
        double sn, cs;
        sincos(-dt * ang, &sn, &cs);
        const double2 v = a[i];
        a[i] = make_double2(v.x * cs - v.y * sn, v.x * sn + v.y * cs);
    }
}

// Physical bit permutation dst[pi(i)] = src[i] with bit j of i moved to
// bit new_pos[j] (used to restore logical order on download).
// Gather form (dst bit c comes from src bit src_of[c]): the writes stay
// coalesced and scattered reads only waste sector bandwidth, where scattered
// 16-byte writes would force partial-sector merges.
__global__ void k_permute_bits(const double2* __restrict__ src, double2* __restrict__ dst,
                               uint64_t n, const int* __restrict__ src_of, int n_bits) {
    for (uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; j < n;
         j += uint64_t(gridDim.x) * blockDim.x) {
        uint64_t i = 0;
        for (int c = 0; c < n_bits; ++c) i |= ((j >> c) & 1ull) << __ldg(src_of + c);
        dst[j] = __ldcs(src + i);
    }
}

double2* d2(StateImpl& s) { return reinterpret_cast<double2*>(s.amps); }

template <typename T>
T* upload_scratch(const std::vector<T>& v, cudaStream_t st) {
    T* d = nullptr;
    if (v.empty()) return nullptr;
    SDB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), v.size() * sizeof(T), st));
    SDB_CUDA(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    return d;
}

}  // namespace

void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        throw OomError(std::string("CUDA out of memory: ") + what);
    }
    throw CudaError(std::string(cudaGetErrorString(e)) + " at " + what);
}

void launch_fill(StateImpl& s, double re, double im) {
    const uint64_t n = s.amps_count();
    k_fill<<<grid_for(n), kThreads, 0, s.stream>>>(d2(s), n, re, im);
    SDB_CUDA(cudaGetLastError());
}

void launch_set_basis(StateImpl& s, uint64_t local_index) {
    launch_fill(s, 0.0, 0.0);
    if (local_index < s.amps_count()) {
        k_set_one<<<1, 1, 0, s.stream>>>(d2(s), local_index);
        SDB_CUDA(cudaGetLastError());
    }
}

void launch_random(StateImpl& s, uint64_t seed) {
    const uint64_t n = s.amps_count();
    k_random<<<grid_for(n), kThreads, 0, s.stream>>>(d2(s), n, seed, uint64_t(s.rank) << s.n_local);
    SDB_CUDA(cudaGetLastError());
}

void launch_scale(StateImpl& s, double f) {
    const uint64_t n = s.amps_count();
    k_scale<<<grid_for(n), kThreads, 0, s.stream>>>(d2(s), n, f);
    SDB_CUDA(cudaGetLastError());
}

static void reduce_impl(StateImpl& a, StateImpl* b, double* re, double* im) {
    const uint64_t n = a.amps_count();
    const unsigned blocks = grid_for(n);
    if (!a.reduce_buf) SDB_CUDA(cudaMalloc(reinterpret_cast<void**>(&a.reduce_buf), 148 * 16 * sizeof(double2)));
    double2* part = reinterpret_cast<double2*>(a.reduce_buf);
    if (b)
        k_reduce<true><<<blocks, kThreads, 0, a.stream>>>(d2(a), d2(*b), n, part);
    else
        k_reduce<false><<<blocks, kThreads, 0, a.stream>>>(d2(a), nullptr, n, part);
    SDB_CUDA(cudaGetLastError());
    std::vector<double2> h(blocks);
    SDB_CUDA(cudaMemcpyAsync(h.data(), part, blocks * sizeof(double2), cudaMemcpyDeviceToHost, a.stream));
    SDB_CUDA(cudaStreamSynchronize(a.stream));
    // Pairwise sum of the block partials (fixed order).
    while (h.size() > 1) {
        std::vector<double2> nx((h.size() + 1) / 2);
        for (size_t i = 0; i < nx.size(); ++i) {
            nx[i] = h[2 * i];
            if (2 * i + 1 < h.size()) {
                nx[i].x += h[2 * i + 1].x;
                nx[i].y += h[2 * i + 1].y;
            }
        }
        h.swap(nx);
    }
    *re = h[0].x;
    if (im) *im = h[0].y;
}

double device_norm_sq(StateImpl& s) {
    double r = 0.0;
    reduce_impl(s, nullptr, &r, nullptr);
    return r;
}

void device_inner(StateImpl& a, StateImpl& b, double* re, double* im) { reduce_impl(a, &b, re, im); }

void launch_hadamard(StateImpl& s, int t) {
    const uint64_t pairs = s.amps_count() >> 1;
    k_hadamard<<<grid_for(pairs), kThreads, 0, s.stream>>>(d2(s), pairs, t);
    SDB_CUDA(cudaGetLastError());
}

void launch_batched_cnot(StateImpl& s, int control, uint64_t targets) {
    const int t0 = __builtin_ctzll(targets);
    const int lo = control < t0 ? control : t0, hi = control < t0 ? t0 : control;
    const uint64_t quads = s.amps_count() >> 2;
    k_batched_cnot<<<grid_for(quads), kThreads, 0, s.stream>>>(d2(s), quads, lo, hi, 1ull << control,
                                                              targets);
    SDB_CUDA(cudaGetLastError());
}

void launch_phase_layer(StateImpl& s, uint64_t s_mask, const std::vector<uint64_t>& pair_masks,
                        bool dagger) {
    uint64_t* dp = upload_scratch(pair_masks, s.stream);
    const uint64_t n = s.amps_count();
    k_phase_layer<<<grid_for(n), kThreads, 0, s.stream>>>(d2(s), n, s_mask, dp,
                                                         static_cast<int>(pair_masks.size()), dagger ? 1 : 0);
    SDB_CUDA(cudaGetLastError());
    if (dp) SDB_CUDA(cudaFreeAsync(dp, s.stream));
}

void launch_diag_exp(StateImpl& s, const std::vector<uint64_t>& masks,
                     const std::vector<double>& coeffs, double dt) {
    uint64_t* dm = upload_scratch(masks, s.stream);
    double* dc = upload_scratch(coeffs, s.stream);
    const uint64_t n = s.amps_count();
    k_diag_exp<<<grid_for(n), kThreads, 0, s.stream>>>(d2(s), n, dm, dc, static_cast<int>(masks.size()), dt);
    SDB_CUDA(cudaGetLastError());
    if (dm) SDB_CUDA(cudaFreeAsync(dm, s.stream));
    if (dc) SDB_CUDA(cudaFreeAsync(dc, s.stream));
}

namespace {
double2 rotation_w(uint64_t x, uint64_t z, double sn) {
    // w = -i sin(theta) * i^{phase_exp}, phase_exp = popc(x & z) & 3 (pauli.cpp:64-66)
    double wr = 0.0, wi = -sn;
    const int ph = __builtin_popcountll(x & z) & 3;
    for (int k = 0; k < ph; ++k) {
        const double t = wr;
        wr = -wi;
        wi = t;
    }
    return make_double2(wr, wi);
}
}  // namespace

void launch_pauli_rotation(StateImpl& s, uint64_t x, uint64_t z, double coeff, double dt, const double* partner) {
    const double theta = coeff * dt;
    const double c = std::cos(theta), sn = std::sin(theta);
    const double2 w = rotation_w(x, z, sn);
    const uint64_t n = s.amps_count();
    const uint64_t rank_bits = uint64_t(s.rank) << s.n_local;
    const uint64_t x_lo = x & (n - 1);
    if (x >> s.n_local) {
        if (!partner) throw std::logic_error("pauli rotation across shards needs the partner shard");
        k_pauli_rotation_remote<<<grid_for(n), kThreads, 0, s.stream>>>(
            d2(s), reinterpret_cast<const double2*>(partner), n, x_lo, x, z, rank_bits, c, w);
    } else {
        const int t0 = x ? __builtin_ctzll(x) : 0;
        const int ypar = __builtin_popcountll(z & x) & 1;
        k_pauli_rotation<<<grid_for(x ? n >> 1 : n), kThreads, 0, s.stream>>>(d2(s), n, x, z, c, sn, w, t0, ypar,
                                                                             rank_bits);
    }
    SDB_CUDA(cudaGetLastError());
}

void device_expectation_term(StateImpl& s, uint64_t x, uint64_t z, const double* partner, double* re, double* im) {
    const uint64_t n = s.amps_count();
    const unsigned blocks = grid_for(n);
    if (!s.reduce_buf) SDB_CUDA(cudaMalloc(reinterpret_cast<void**>(&s.reduce_buf), 148 * 16 * sizeof(double2)));
    double2* part = reinterpret_cast<double2*>(s.reduce_buf);
    const int ph = __builtin_popcountll(x & z) & 3;
    const double2 base[4] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};
    const double2* p = (x >> s.n_local) ? reinterpret_cast<const double2*>(partner) : d2(s);
    if (!p) throw std::logic_error("expectation across shards needs the partner shard");
    k_expect<<<blocks, kThreads, 0, s.stream>>>(d2(s), p, n, x & (n - 1), x, z, uint64_t(s.rank) << s.n_local,
                                                base[ph], part);
    SDB_CUDA(cudaGetLastError());
    std::vector<double2> h(blocks);
    SDB_CUDA(cudaMemcpyAsync(h.data(), part, blocks * sizeof(double2), cudaMemcpyDeviceToHost, s.stream));
    SDB_CUDA(cudaStreamSynchronize(s.stream));
    while (h.size() > 1) {
        std::vector<double2> nx((h.size() + 1) / 2);
        for (size_t i = 0; i < nx.size(); ++i) {
            nx[i] = h[2 * i];
            if (2 * i + 1 < h.size()) {
                nx[i].x += h[2 * i + 1].x;
                nx[i].y += h[2 * i + 1].y;
            }
        }
        h.swap(nx);
    }
    *re = h[0].x;
    *im = h[0].y;
}

// exact_evolve (reference evolve.cpp:60-97) for n <= 12: psi <- exp(-i H t)
// psi by a Taylor series, time-sliced so each slice has ||H dt|| <= 1/2
// (||H|| <= sum |c_k|) and truncated at 24 terms (remainder < 2^-24/24! ~ 1e-31
// of the slice's norm); the reference diagonalises the dense matrix instead.
void launch_exact_evolve(StateImpl& s, const uint64_t* x, const uint64_t* z, const double* c, size_t m, double t) {
    const uint64_t n = s.amps_count();
    double hnorm = 0.0;
    std::vector<double2> cb(m);
    for (size_t k = 0; k < m; ++k) {
        hnorm += std::fabs(c[k]);
        const int ph = __builtin_popcountll(x[k] & z[k]) & 3;
        const double2 ip[4] = {{1, 0}, {0, 1}, {-1, 0}, {0, -1}};
        cb[k] = make_double2(c[k] * ip[ph].x, c[k] * ip[ph].y);
    }
    if (m == 0 || t == 0.0) return;
    const int slices = std::max(1, static_cast<int>(std::ceil(2.0 * hnorm * std::fabs(t))));
    const double dt = t / slices;
    uint64_t* dx = upload_scratch(std::vector<uint64_t>(x, x + m), s.stream);
    uint64_t* dz = upload_scratch(std::vector<uint64_t>(z, z + m), s.stream);
    double2* dc = upload_scratch(cb, s.stream);
    double2* buf = nullptr;
    SDB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), 2 * n * sizeof(double2), s.stream));
    for (int sl = 0; sl < slices; ++sl) {
        SDB_CUDA(cudaMemcpyAsync(buf, s.amps, n * sizeof(double2), cudaMemcpyDeviceToDevice, s.stream));
        for (int j = 1; j <= 24; ++j) {
            const double2 f = make_double2(0.0, -dt / j);  // (-i dt) / j
            const double2* cur = buf + ((j - 1) & 1) * n;
            double2* nxt = buf + (j & 1) * n;
            k_taylor_term<<<grid_for(n), kThreads, 0, s.stream>>>(cur, nxt, d2(s), n, dx, dz, dc, static_cast<int>(m), f);
            SDB_CUDA(cudaGetLastError());
        }
    }
    SDB_CUDA(cudaFreeAsync(buf, s.stream));
    SDB_CUDA(cudaFreeAsync(dx, s.stream));
    SDB_CUDA(cudaFreeAsync(dz, s.stream));
    SDB_CUDA(cudaFreeAsync(dc, s.stream));
}

void launch_single_qubit(StateImpl& s, const double* u, int t) {
    Mat2D m;
    for (int k = 0; k < 4; ++k) m.u[k] = make_double2(u[2 * k], u[2 * k + 1]);
    const uint64_t pairs = s.amps_count() >> 1;
    k_single_qubit<<<grid_for(pairs), kThreads, 0, s.stream>>>(d2(s), pairs, t, m);
    SDB_CUDA(cudaGetLastError());
}

void launch_two_qubit(StateImpl& s, const double* u, int q1, int q2) {
    Mat4D m;
    for (int k = 0; k < 16; ++k) m.u[k] = make_double2(u[2 * k], u[2 * k + 1]);
    const uint64_t quads = s.amps_count() >> 2;
    const int lo = q1 < q2 ? q1 : q2, hi = q1 < q2 ? q2 : q1;
    k_two_qubit<<<grid_for(quads), kThreads, 0, s.stream>>>(d2(s), quads, lo, hi, 1ull << q1, 1ull << q2, m);
    SDB_CUDA(cudaGetLastError());
}

void launch_permute_bits(StateImpl& s, const double* src, double* dst, const int* new_pos_host,
                         int n_bits) {
    std::vector<int> pos(n_bits);
    for (int b = 0; b < n_bits; ++b) pos[new_pos_host[b]] = b;  // inverse: source bit of each target bit
    int* dpos = upload_scratch(pos, s.stream);
    const uint64_t n = uint64_t(1) << n_bits;
    k_permute_bits<<<grid_for(n), kThreads, 0, s.stream>>>(reinterpret_cast<const double2*>(src),
                                                          reinterpret_cast<double2*>(dst), n, dpos, n_bits);
    SDB_CUDA(cudaGetLastError());
    SDB_CUDA(cudaFreeAsync(dpos, s.stream));
}

}  // namespace sdb
