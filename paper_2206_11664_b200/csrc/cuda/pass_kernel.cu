// Fused Clifford/diagonal tile pass: the compiled interpreter. The device
// code lives in pass_device.cuh; this kernel feeds its ops from the staged
// micro-program. Large states can instead run a kernel specialised for the
// pass's program at plan time (jit.cpp).
#include <cuda_runtime.h>

#include <cstdlib>

#include "../internal.hpp"
#include "jit.hpp"
#include "pass_device.cuh"

namespace sdb {

namespace {

using dev::Cfg;
using dev::kTbaseChunks;

struct Interpreter {
    template <class Ctx, int NR>
    __device__ __forceinline__ void operator()(Ctx& ctx, double2 (&v)[NR]) const {
        const int n_ops = ctx.P.n_ops;
        for (int oi = 0; oi < n_ops; ++oi) {
            const MicroOpDev& op = ctx.s_ops[oi];
            const int kind = op.kind;
            if (kind == kOpLoad) {
                ctx.load(ctx.cfg_of(op), v);
            } else if (kind == kOpCfg) {
                ctx.cfg(op, ctx.cfg_of(op), v);
            } else if (kind == kOpSwap) {
                ctx.swap_any(op, ctx.cfg_of(op), v);
            } else if (kind == kOpBfly) {
                dev::bfly_dispatch<Ctx::R>(v, op.mask);
            } else if (kind == kOpLaneBfly) {
                if (op.mask == 3) dev::lane_bfly<Ctx::R, 3>(v);
                else dev::lane_bfly<Ctx::R, 4>(v);
            } else if (kind == kOpPoint) {
                ctx.point_any(op, v);
            } else {
                ctx.store(op, v);
            }
        }
    }
};

__global__ void k_tile_phase(PlanDev plan, int pass_index, double neg_dt, uint64_t rank_bits, uint64_t n_tiles,
                             double2* __restrict__ out) {
    const PassDev& P = plan.passes[pass_index];
    for (uint64_t t = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; t < n_tiles; t += uint64_t(gridDim.x) * blockDim.x)
        out[t] = dev::tile_constant_phase(plan, P, t, rank_bits, neg_dt);
}

template <int K, int RB>
__global__ void __launch_bounds__(Cfg<K, RB>::NT, Cfg<K, RB>::MINB)
k_tile_pass(const double2* psi, double2* out, double2* const* xdst, PlanDev plan,
            int pass_index, double neg_dt, uint64_t rank_bits, uint64_t n_tiles) {
    const Interpreter prog;
    SDB_PASS_KERNEL_BODY(K, RB, prog)
}

template <int K, int RB>
size_t smem_bytes(const PassDev& ph) {
    using C = Cfg<K, RB>;
    return sizeof(double2) * C::N + sizeof(double) * ph.tab_words + sizeof(MicroOpDev) * ph.n_ops +
           sizeof(uint64_t) * ph.n_qt_words +
           (ph.store_perm ? sizeof(uint64_t) * ((1 << C::LO) + (1 << C::HI) + kTbaseChunks * 128) : 0);
}

template <int K, int RB>
void launch_kr(StateImpl& s, const PassDev& ph, int pass_index, const PlanDev& plan, double dt, uint64_t rank_bits,
               double* out, double2* const* xdst) {
    using C = Cfg<K, RB>;
    const size_t smem = smem_bytes<K, RB>(ph);
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
    if (const char* e = std::getenv("SDB_MAX_CTAS"); e && std::atoi(e) > 0 && grid > uint64_t(std::atoi(e)))
        grid = std::atoi(e);  // debugging: many tiles per CTA at small n
    k_tile_pass<K, RB><<<static_cast<unsigned>(grid), C::NT, smem, s.stream>>>(
        reinterpret_cast<const double2*>(s.amps), reinterpret_cast<double2*>(out ? out : s.amps), xdst, plan,
        pass_index, -dt, rank_bits, n_tiles);
    SDB_CUDA(cudaGetLastError());
}

template <int K>
void launch_k(StateImpl& s, const PassDev& ph, int pass_index, const PlanDev& plan, double dt, uint64_t rank_bits,
              double* out, double2* const* xdst) {
    // R = 4 register coordinates (16 amplitudes per thread). R = 3 with twice the
    // threads spills at the 2-CTA/SM register budget and measured 1.5x slower
    // per step (profiles/r1_notes.md).
    if (ph.rbits != 4 && K >= 4) throw std::invalid_argument("tile pass: unsupported register config");
    launch_kr<K, 4>(s, ph, pass_index, plan, dt, rank_bits, out, xdst);
}

}  // namespace

int max_tile_qubits() { return 12; }

void launch_tile_phase(StateImpl& s, const PassDev& ph, int pass_index, const PlanDev& plan, double dt,
                       uint64_t rank_bits, double2* out) {
    const uint64_t n_tiles = 1ull << ph.n_outer;
    uint64_t blocks = (n_tiles + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    k_tile_phase<<<static_cast<unsigned>(blocks), 256, 0, s.stream>>>(plan, pass_index, -dt, rank_bits, n_tiles, out);
    SDB_CUDA(cudaGetLastError());
}

size_t tile_pass_smem(const PassDev& ph) {
    if (ph.k == 12 && ph.rbits == 3) return smem_bytes<12, 3>(ph);
    switch (ph.k) {
#define SDB_K(KK) \
    case KK: return smem_bytes<KK, 4>(ph);
        SDB_K(1) SDB_K(2) SDB_K(3) SDB_K(4) SDB_K(5) SDB_K(6) SDB_K(7) SDB_K(8) SDB_K(9) SDB_K(10)
        SDB_K(11) SDB_K(12)
#undef SDB_K
        default: throw std::invalid_argument("tile qubits out of range");
    }
}

void launch_tile_pass(StateImpl& s, const PassDev& ph, int pass_index, const PlanDev& plan, double dt,
                      uint64_t rank_bits, double* out, double2* const* xdst) {
    if (ph.n_outer > 7 * kTbaseChunks) throw std::invalid_argument("tile pass: too many outer bits");
    switch (ph.k) {
#define SDB_K(KK) \
    case KK: launch_k<KK>(s, ph, pass_index, plan, dt, rank_bits, out, xdst); break;
        SDB_K(1) SDB_K(2) SDB_K(3) SDB_K(4) SDB_K(5) SDB_K(6) SDB_K(7) SDB_K(8) SDB_K(9) SDB_K(10)
        SDB_K(11) SDB_K(12)
#undef SDB_K
        default: throw std::invalid_argument("tile qubits out of range");
    }
}

}  // namespace sdb
