// Memory-pattern microbenchmark for tile passes (B200). In-place read+write
// of a 2^n complex128 state, one tile = 2^12 amplitudes whose local bits are
// given as a list; 256 threads x 16 amplitudes, loads straight to registers
// (the k_tile_pass LOAD/STORE shape). Usage: membench2 n "0,1,2,3,5,7,..." [ctas_per_sm]
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/membench2 tools/membench2.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#define CK(x)                                                                               \
    do {                                                                                    \
        cudaError_t e = (x);                                                                \
        if (e != cudaSuccess) {                                                             \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);        \
            exit(1);                                                                        \
        }                                                                                   \
    } while (0)

struct Layout {
    uint64_t off[16];     // register j offset
    uint64_t toff[256];   // thread offsets
    uint64_t tb[4][128];  // tile index chunks
};

__global__ void __launch_bounds__(256, 2) k_regs(double2* psi, const Layout* __restrict__ L, uint64_t n_tiles) {
    __shared__ uint64_t s_tb[4][128];
    for (int i = threadIdx.x; i < 512; i += 256) s_tb[i >> 7][i & 127] = L->tb[i >> 7][i & 127];
    const uint64_t to = L->toff[threadIdx.x];
    uint64_t off[16];
    for (int j = 0; j < 16; ++j) off[j] = L->off[j] | to;
    __syncthreads();
    for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const uint64_t b = s_tb[0][t & 127] | s_tb[1][(t >> 7) & 127] | s_tb[2][(t >> 14) & 127] | s_tb[3][(t >> 21) & 127];
        double2* g = psi + b;
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
    const int n = atoi(argv[1]);
    std::vector<int> lpos;
    std::string spec = argv[2];
    for (char* p = strtok(argv[2], ","); p; p = strtok(nullptr, ",")) lpos.push_back(atoi(p));
    const int per_sm = argc > 3 ? atoi(argv[3]) : 2;
    // register coords = the 4 highest local bits, thread coords = the other 8 ascending
    Layout h{};
    for (int j = 0; j < 16; ++j) {
        uint64_t o = 0;
        for (int b = 0; b < 4; ++b) if ((j >> b) & 1) o |= 1ull << lpos[8 + b];
        h.off[j] = o;
    }
    for (int t = 0; t < 256; ++t) {
        uint64_t o = 0;
        for (int b = 0; b < 8; ++b) if ((t >> b) & 1) o |= 1ull << lpos[b];
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
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    k_regs<<<sms * per_sm, 256>>>(a, dL, tiles);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) k_regs<<<sms * per_sm, 256>>>(a, dL, tiles);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= 5;
    printf("n=%d ctas/sm=%d lpos=%s : %.3f ms %.1f GB/s\n", n, per_sm, spec.c_str(), ms, 32.0 * (1ull << n) / (ms * 1e-3) / 1e9);
    return 0;
}
