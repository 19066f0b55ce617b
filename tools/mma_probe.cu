// mma_probe.cu -- legacy mma.sync m16n8k16 bf16 throughput on sm_100a: cycles per MMA per
// SMSP with W warps per CTA (one CTA per SM), A independent accumulator chains per warp.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void mma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <int A>
__global__ void probe(float* out, long long* cyc, int iters) {
    uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
    float d[A][4] = {};
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int j = 0; j < A; ++j) mma(d[j], a, 0x3f803f80u + i, 0x3f803f80u);
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int j = 0; j < A; ++j) s += d[j][0] + d[j][1] + d[j][2] + d[j][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
    const int iters = 2000;
    for (int W : {4, 8, 16, 32}) {
        for (int A : {1, 4, 8}) {
            long long h = 0;
            for (int rep = 0; rep < 2; ++rep) {
                if (A == 1) probe<1><<<148, 32 * W>>>(out, cyc, iters);
                if (A == 4) probe<4><<<148, 32 * W>>>(out, cyc, iters);
                if (A == 8) probe<8><<<148, 32 * W>>>(out, cyc, iters);
                cudaDeviceSynchronize();
                cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
            }
            const double mmas_per_smsp = (double)W / 4 * A * iters;
            printf("warps %2d chains %d: %.2f cycles per MMA per SMSP (%.1f cycles per MMA per warp)\n", W, A,
                   h / mmas_per_smsp, (double)h / (A * iters));
        }
    }
    return 0;
}
