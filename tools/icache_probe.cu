// icache_probe.cu -- is cold straight-line code the fused kernel's post-stream cost?
// NB blocks of distinct code (each: 48 dependent FMAs with block-specific constants, a
// CTA barrier, a timer stamp), executed twice in a row by 512-thread CTAs.  Pass 0 runs
// every block's code cold, pass 1 warm (if it fits the instruction caches).
// usage: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/icache_probe tools/icache_probe.cu
//        ./tools/icache_probe [ctas]
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#ifndef NB
#define NB 96
#endif

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    return t;
}

template <int I>
__device__ __forceinline__ void blk(float& acc) {
    float x = acc;
#pragma unroll
    for (int j = 0; j < 48; ++j) x = fmaf(x, 1.0f + (float)(I * 48 + j) * 1e-7f, (float)(I ^ j) * 1e-3f);
    acc = x;
}

template <int I>
__device__ __forceinline__ void chain(float& acc, uint64_t* st) {
    if constexpr (I < NB) {
        blk<I>(acc);
        __syncthreads();
        if (threadIdx.x == 0) st[I] = gtimer();
        chain<I + 1>(acc, st);
    }
}

__global__ void __launch_bounds__(512, 1) probe(float* out, uint64_t* stamps) {
    __shared__ uint64_t st[2][NB + 1];
    float acc = (float)threadIdx.x;
    for (int pass = 0; pass < 2; ++pass) {
        __syncthreads();
        if (threadIdx.x == 0) st[pass][NB] = gtimer();
        chain<0>(acc, st[pass]);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x < 2 * (NB + 1)) stamps[blockIdx.x * 2 * (NB + 1) + threadIdx.x] = (&st[0][0])[threadIdx.x];
}

int main(int argc, char** argv) {
    const int ctas = argc > 1 ? atoi(argv[1]) : 64;
    float* out;
    uint64_t* stamps;
    cudaMalloc(&out, ctas * 512 * 4);
    cudaMalloc(&stamps, ctas * 2 * (NB + 1) * 8);
    for (int rep = 0; rep < 3; ++rep) probe<<<ctas, 512>>>(out, stamps);
    cudaDeviceSynchronize();
    uint64_t* h = new uint64_t[ctas * 2 * (NB + 1)];
    cudaMemcpy(h, stamps, ctas * 2 * (NB + 1) * 8, cudaMemcpyDeviceToHost);
    double tot[2] = {0, 0};
    for (int c = 0; c < ctas; ++c)
        for (int pass = 0; pass < 2; ++pass) {
            const uint64_t* s = h + c * 2 * (NB + 1) + pass * (NB + 1);
            tot[pass] += (double)(s[NB - 1] - s[NB]);
        }
    printf("NB=%d blocks (~%d instrs each), %d CTAs: pass0 (cold) %.2f us, pass1 (warm) %.2f us, per block %.1f / %.1f ns\n",
           NB, 48 + 8, ctas, tot[0] / ctas / 1e3, tot[1] / ctas / 1e3, tot[0] / ctas / NB, tot[1] / ctas / NB);
    return 0;
}
