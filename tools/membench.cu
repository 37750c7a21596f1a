// Memory-system microbenchmark for the tile-pass access pattern (B200).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/membench tools/membench.cu
// Runs in-place read+write passes over a 2^n complex128 state with:
//   A  grid-stride streaming (LDG.128 -> STG.128)
//   B  tile gather via cp.async ring (STAGES, 256 thr, 16 amps/thread), direct store
//   C  tile gather via plain LDG into registers (no smem), 2^k tile, 256 thr
// with the tile's local bit set either contiguous {0..k-1} or "split"
// {0,1,2} + {s..s+k-4} (the pass pattern with strided 128-byte runs).
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e = (x);                                                                    \
        if (e != cudaSuccess) {                                                                 \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);             \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

__global__ void k_stream(double2* a, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        double2 v = a[i];
        v.x = -v.x;
        a[i] = v;
    }
}

struct Layout {
    int lpos[16];
    int opos[48];
    int k, n_outer;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

__device__ __forceinline__ uint64_t tile_base(const Layout& L, uint64_t t) {
    uint64_t b = 0;
    for (int j = 0; j < L.n_outer; ++j) b |= ((t >> j) & 1ull) << L.opos[j];
    return b;
}
__device__ __forceinline__ uint64_t loc(const Layout& L, uint32_t l) {
    uint64_t o = 0;
    for (int j = 0; j < L.k; ++j) o |= uint64_t((l >> j) & 1u) << L.lpos[j];
    return o;
}

template <int STAGES>
__global__ void __launch_bounds__(256) k_ring(double2* psi, Layout L, uint64_t n_tiles) {
    extern __shared__ __align__(16) double2 ring[];
    constexpr int N = 4096;
    const int tid = threadIdx.x;
    uint64_t off[16];
    for (int j = 0; j < 16; ++j) off[j] = loc(L, tid + j * 256);
    const uint64_t stride = gridDim.x;
    uint64_t t = blockIdx.x;
    for (int j = 0; j < STAGES - 1; ++j) {
        if (t + j * stride < n_tiles) {
            const double2* g = psi + tile_base(L, t + j * stride);
            for (int q = 0; q < 16; ++q) cp_async16(ring + j * N + tid + q * 256, g + off[q]);
        }
        cp_commit();
    }
    for (int it = 0; t < n_tiles; t += stride, ++it) {
        double2* cb = ring + (it % STAGES) * N;
        cp_wait<STAGES - 2>();
        __syncthreads();
        const uint64_t tn = t + (STAGES - 1) * stride;
        if (tn < n_tiles) {
            const double2* g = psi + tile_base(L, tn);
            double2* nb = ring + ((it + STAGES - 1) % STAGES) * N;
            for (int q = 0; q < 16; ++q) cp_async16(nb + tid + q * 256, g + off[q]);
        }
        cp_commit();
        double2* g = psi + tile_base(L, t);
        for (int q = 0; q < 16; ++q) {
            double2 v = cb[tid + q * 256];
            v.x = -v.x;
            __stcs(g + off[q], v);
        }
    }
    cp_wait<0>();
}

__global__ void __launch_bounds__(256) k_regs(double2* psi, Layout L, uint64_t n_tiles) {
    const int tid = threadIdx.x;
    uint64_t off[16];
    for (int j = 0; j < 16; ++j) off[j] = loc(L, tid + j * 256);
    for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        double2* g = psi + tile_base(L, t);
        double2 v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = __ldcs(g + off[q]);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            v[q].x = -v[q].x;
            __stcs(g + off[q], v[q]);
        }
    }
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 30;
    const uint64_t amps = 1ull << n;
    double2* a;
    CK(cudaMalloc(&a, amps * 16));
    CK(cudaMemset(a, 0, amps * 16));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const double bytes = 2.0 * 16.0 * double(amps);
    auto report = [&](const char* name, auto&& launch) {
        launch();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        const int reps = 5;
        for (int r = 0; r < reps; ++r) launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        ms /= reps;
        printf("%-44s %8.3f ms  %8.1f GB/s\n", name, ms, bytes / (ms * 1e-3) / 1e9);
    };
    report("stream grid-stride 148x16x256", [&] { k_stream<<<sms * 16, 256>>>(a, amps); });
    report("stream grid-stride 148x4x1024", [&] { k_stream<<<sms * 4, 1024>>>(a, amps); });
    for (int split = 0; split < 3; ++split) {
        Layout L{};
        L.k = 12;
        int s0 = split == 0 ? 3 : (split == 1 ? 7 : 18);
        for (int j = 0; j < 12; ++j) L.lpos[j] = j < 3 ? j : (split == 0 ? j : s0 + j - 3);
        int no = 0;
        for (int b = 0; b < n; ++b) {
            bool local = false;
            for (int j = 0; j < 12; ++j) local |= L.lpos[j] == b;
            if (!local) L.opos[no++] = b;
        }
        L.n_outer = no;
        const uint64_t tiles = 1ull << no;
        char nm[128];
        const char* lname = split == 0 ? "contig{0..11}" : (split == 1 ? "split{0-2,7-15}" : "split{0-2,18-26}");
        snprintf(nm, sizeof nm, "ring2 %s", lname);
        CK(cudaFuncSetAttribute(k_ring<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 65536));
        report(nm, [&] { k_ring<2><<<sms, 256, 2 * 65536>>>(a, L, tiles); });
        snprintf(nm, sizeof nm, "ring3 %s", lname);
        CK(cudaFuncSetAttribute(k_ring<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 65536));
        report(nm, [&] { k_ring<3><<<sms, 256, 3 * 65536>>>(a, L, tiles); });
        snprintf(nm, sizeof nm, "regs 1/SM %s", lname);
        report(nm, [&] { k_regs<<<sms, 256>>>(a, L, tiles); });
        snprintf(nm, sizeof nm, "regs 4/SM %s", lname);
        report(nm, [&] { k_regs<<<sms * 4, 256>>>(a, L, tiles); });
    }
    return 0;
}
