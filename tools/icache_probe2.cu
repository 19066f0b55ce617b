// icache_probe2.cu -- cost of cold, branchy code: NB blocks, each = a runtime-trip-count
// loop (8 iterations: smem load -> compare -> ballot -> popc), then a branch over COLD
// bytes of never-executed code (runtime-false condition), a CTA barrier and a stamp.
// pass 0 cold, pass 1 warm.  usage: ./icache_probe2 [ctas] [iters]
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#ifndef NB
#define NB 32
#endif
#ifndef COLD
#define COLD 64
#endif
__device__ __forceinline__ uint64_t clk() { uint64_t t; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory"); return t; }
template <int I>
__device__ __forceinline__ void blk(float& acc, const uint32_t* sm, int iters, int never) {
    uint32_t c = 0;
    for (int j = 0; j < iters; ++j) {
        const uint32_t k = sm[(threadIdx.x + 37 * j + I) & 1023];
        c += __popc(__ballot_sync(0xffffffffu, (k ^ (uint32_t)I) > 0x7fffffffu));
    }
    acc += (float)c;
    if (never) {
        float x = acc;
#pragma unroll
        for (int j = 0; j < COLD; ++j) x = fmaf(x, 1.0f + (float)(I * COLD + j) * 1e-7f, (float)(I ^ j));
        acc = x;
    }
}
template <int I>
__device__ __forceinline__ void chain(float& acc, const uint32_t* sm, int iters, int never, uint64_t* st) {
    if constexpr (I < NB) {
        blk<I>(acc, sm, iters, never);
        __syncthreads();
        if (threadIdx.x == 0) st[I] = clk();
        chain<I + 1>(acc, sm, iters, never, st);
    }
}
__global__ void __launch_bounds__(512, 1) probe(float* out, uint64_t* stamps, int iters, int never) {
    __shared__ uint64_t st[2][NB + 1];
    __shared__ uint32_t sm[1024];
    for (int i = threadIdx.x; i < 1024; i += 512) sm[i] = i * 2654435761u;
    __syncthreads();
    float acc = (float)threadIdx.x;
    for (int pass = 0; pass < 2; ++pass) {
        __syncthreads();
        if (threadIdx.x == 0) st[pass][NB] = clk();
        chain<0>(acc, sm, iters, never, st[pass]);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x < 2 * (NB + 1)) stamps[blockIdx.x * 2 * (NB + 1) + threadIdx.x] = (&st[0][0])[threadIdx.x];
}
int main(int argc, char** argv) {
    const int ctas = argc > 1 ? atoi(argv[1]) : 64, iters = argc > 2 ? atoi(argv[2]) : 8;
    float* out; uint64_t* stamps;
    cudaMalloc(&out, ctas * 512 * 4); cudaMalloc(&stamps, ctas * 2 * (NB + 1) * 8);
    for (int rep = 0; rep < 3; ++rep) probe<<<ctas, 512>>>(out, stamps, iters, 0);
    cudaDeviceSynchronize();
    uint64_t* h = new uint64_t[ctas * 2 * (NB + 1)];
    cudaMemcpy(h, stamps, ctas * 2 * (NB + 1) * 8, cudaMemcpyDeviceToHost);
    double tot[2] = {0, 0};
    for (int c = 0; c < ctas; ++c) for (int pass = 0; pass < 2; ++pass) {
        const uint64_t* s = h + c * 2 * (NB + 1) + pass * (NB + 1);
        tot[pass] += (double)(s[NB - 1] - s[NB]);
    }
    printf("NB=%d COLD=%d iters=%d ctas=%d: cycles per block pass0 %.0f  pass1 %.0f\n", NB, COLD, iters, ctas,
           tot[0] / ctas / NB, tot[1] / ctas / NB);
    return 0;
}
