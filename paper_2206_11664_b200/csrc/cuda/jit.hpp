// Run-time specialised tile-pass kernels (jit.cpp).
#pragma once

#include <cstddef>
#include <vector>

#include "../internal.hpp"
#include "../plan/lower.hpp"

namespace sdb {

// Whether plans for a state of this shard size use specialised kernels
// (SDB_JIT=0/1 overrides; default: n_local >= 22, where compile time amortises).
bool jit_wanted(int n_local);
// CUfunction of every pass's specialised kernel (distinct programs compiled in
// parallel, cached in-process and on disk).
std::vector<void*> jit_pass_kernels(const HostPlanArrays& A, int device);
void launch_tile_pass_jit(void* fn, StateImpl& s, const PassDev& ph, int pass_index, const PlanDev& plan, double dt,
                          uint64_t rank_bits, double* out, size_t smem, double2* const* xdst = nullptr,
                          int threads = 0);
// Host-only: generate and NVRTC-compile every distinct pass program of A
// (no device needed); returns the number of distinct programs.
size_t jit_compile_only(const HostPlanArrays& A);
// dynamic shared memory of a tile pass (same for both kernel kinds)
size_t tile_pass_smem(const PassDev& ph);
// extra dynamic shared memory of pass `pass`'s specialised kernel (TMA split stage)
size_t jit_pass_smem_extra(const HostPlanArrays& A, size_t pass);
// block size of pass `pass`'s specialised kernel (two warp groups in ring mode)
int jit_pass_threads(const HostPlanArrays& A, size_t pass);

}  // namespace sdb
