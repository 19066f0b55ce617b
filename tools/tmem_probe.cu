// tmem_probe.cu -- which (TMEM lane, column) does each thread get from
// tcgen05.ld.16x256b?  (layout check for mixing mma.sync fragments with TMEM)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void probe(uint32_t* out) {
    __shared__ uint32_t slot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = slot;
    // every warp w writes its lane quarter: value = lane_global * 1000 + col, cols 0..15
    uint32_t v[16];
    for (int c = 0; c < 16; ++c) v[c] = (uint32_t)((warp * 32 + lane) * 1000 + c);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 ::"r"(tb + ((uint32_t)(warp * 32) << 16)), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                 "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) {
        uint32_t r[8];
        // 16 lanes starting at lane 0 (of quarter 0), columns 0..15: .x2
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\ntcgen05.wait::ld.sync.aligned;"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(tb));
        for (int i = 0; i < 8; ++i) out[lane * 8 + i] = r[i];
        uint32_t r2[4];
        asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];\ntcgen05.wait::ld.sync.aligned;"
                     : "=r"(r2[0]), "=r"(r2[1]), "=r"(r2[2]), "=r"(r2[3]) : "r"(tb + (16u << 16)));
        for (int i = 0; i < 4; ++i) out[256 + lane * 4 + i] = r2[i];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tb));
}

int main() {
    uint32_t* d;
    cudaMalloc(&d, 4096 * 4);
    probe<<<1, 128>>>(d);
    uint32_t h[512];
    cudaError_t e = cudaMemcpy(h, d, 512 * 4, cudaMemcpyDeviceToHost);
    printf("err=%s\n", cudaGetErrorString(e));
    printf("16x256b.x2 at lane 0 (value = lane*1000 + col):\n");
    for (int t = 0; t < 32; ++t) {
        printf("T%2d:", t);
        for (int i = 0; i < 8; ++i) printf(" (%u,%u)", h[t * 8 + i] / 1000, h[t * 8 + i] % 1000);
        printf("\n");
    }
    printf("16x256b.x1 at lane 16:\n");
    for (int t = 0; t < 4; ++t) {
        printf("T%2d:", t);
        for (int i = 0; i < 4; ++i) printf(" (%u,%u)", h[256 + t * 4 + i] / 1000, h[256 + t * 4 + i] % 1000);
        printf("\n");
    }
    return 0;
}
