// Memory-pattern microbenchmark, tile-order variants (B200). In-place
// read+negate+write of a 2^n complex128 state in tiles of 2^12 amplitudes whose
// local bits are listed (registers = the 4 highest local bits, threads = the
// other 8). Variants:
//   mode 0: 2 CTAs/SM x 256 threads, grid-stride over tiles (k_tile_pass shape)
//   mode 1: mode 0 + prefetch.global.L2 of the CTA's next tile (as k_tile_pass)
//   mode 2: 1 CTA/SM x 512 threads, each CTA takes the tile pair differing in
//           the lowest outer bit (256 contiguous bytes per DRAM page visit)
//   mode 3: mode 2 + L2 prefetch of the next pair
//   mode 4: 1 CTA/SM x 1024 threads, 8 amplitudes per thread, tile quadruple
// Usage: membench3 n "0,1,2,..." mode
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/membench3 tools/membench3.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e = (x);                                                         \
        if (e != cudaSuccess) {                                                      \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                                 \
        }                                                                            \
    } while (0)

struct Layout {
    uint64_t off[16];    // register j offset
    uint64_t toff[256];  // thread offsets
    uint64_t tb[4][128]; // tile index chunks
};

__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

template <int SUB, int NA, bool PF>
__global__ void __launch_bounds__(SUB * 256 * 16 / NA, SUB == 1 ? 2 : 1) k_tiles(double2* psi, const Layout* __restrict__ L, uint64_t n_groups) {
    // SUB tiles per CTA, NA amplitudes per thread, 256 * 16 / NA threads per tile
    constexpr int TPT = 256 * 16 / NA;
    __shared__ uint64_t s_tb[4][128];
    for (int i = threadIdx.x; i < 512; i += blockDim.x) s_tb[i >> 7][i & 127] = L->tb[i >> 7][i & 127];
    const int sub = threadIdx.x / TPT;
    const int lt = threadIdx.x % TPT;
    uint64_t off[NA];
    if constexpr (NA == 16) {
        const uint64_t to = L->toff[lt];
        for (int j = 0; j < 16; ++j) off[j] = L->off[j] | to;
    } else {
        // 8 amplitudes: registers = 3 highest local bits, thread bit 8 = the 4th
        const uint64_t to = L->toff[lt & 255] | ((lt >> 8) ? L->off[1] : 0);
        for (int j = 0; j < 8; ++j) off[j] = L->off[j << 1] | to;
    }
    __syncthreads();
    auto base = [&](uint64_t t) {
        return s_tb[0][t & 127] | s_tb[1][(t >> 7) & 127] | s_tb[2][(t >> 14) & 127] | s_tb[3][(t >> 21) & 127];
    };
    for (uint64_t gidx = blockIdx.x; gidx < n_groups; gidx += gridDim.x) {
        double2* g = psi + base(gidx * SUB + sub);
        double2 v[NA];
#pragma unroll
        for (int q = 0; q < NA; ++q) v[q] = __ldcs(g + off[q]);
        if constexpr (PF) {
            if (gidx + gridDim.x < n_groups) {
                const double2* gn = psi + base((gidx + gridDim.x) * SUB + sub);
#pragma unroll
                for (int q = 0; q < NA; ++q) prefetch_l2(gn + off[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < NA; ++q) {
            v[q].x = -v[q].x;
            __stcs(g + off[q], v[q]);
        }
    }
}

int main(int argc, char** argv) {
    const int n = atoi(argv[1]);
    std::vector<int> lpos;
    std::string spec = argv[2];
    for (char* p = strtok(argv[2], ","); p; p = strtok(nullptr, ",")) lpos.push_back(atoi(p));
    const int mode = argc > 3 ? atoi(argv[3]) : 0;
    Layout h{};
    for (int j = 0; j < 16; ++j) {
        uint64_t o = 0;
        for (int b = 0; b < 4; ++b)
            if ((j >> b) & 1) o |= 1ull << lpos[8 + b];
        h.off[j] = o;
    }
    for (int t = 0; t < 256; ++t) {
        uint64_t o = 0;
        for (int b = 0; b < 8; ++b)
            if ((t >> b) & 1) o |= 1ull << lpos[b];
        h.toff[t] = o;
    }
    std::vector<int> opos;
    for (int b = 0; b < n; ++b) {
        bool loc = false;
        for (int x : lpos) loc |= x == b;
        if (!loc) opos.push_back(b);
    }
    for (int c = 0; c < 4; ++c)
        for (int v = 0; v < 128; ++v) {
            uint64_t o = 0;
            for (int j = 0; j < 7; ++j)
                if (7 * c + j < (int)opos.size() && ((v >> j) & 1)) o |= 1ull << opos[7 * c + j];
            h.tb[c][v] = o;
        }
    double2* a;
    Layout* dL;
    CK(cudaMalloc(&a, (1ull << n) * 16));
    CK(cudaMemset(a, 0, (1ull << n) * 16));
    CK(cudaMalloc(&dL, sizeof(Layout)));
    CK(cudaMemcpy(dL, &h, sizeof(Layout), cudaMemcpyHostToDevice));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint64_t tiles = 1ull << opos.size();
    auto launch = [&]() {
        switch (mode) {
            case 0: k_tiles<1, 16, false><<<sms * 2, 256>>>(a, dL, tiles); break;
            case 1: k_tiles<1, 16, true><<<sms * 2, 256>>>(a, dL, tiles); break;
            case 2: k_tiles<2, 16, false><<<sms, 512>>>(a, dL, tiles / 2); break;
            case 3: k_tiles<2, 16, true><<<sms, 512>>>(a, dL, tiles / 2); break;
            default: k_tiles<2, 8, true><<<sms, 1024>>>(a, dL, tiles / 2); break;
        }
    };
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    launch();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= 5;
    printf("n=%d mode=%d lpos=%s : %.3f ms %.1f GB/s\n", n, mode, spec.c_str(), ms, 32.0 * (1ull << n) / (ms * 1e-3) / 1e9);
    return 0;
}
