// gather_probe.cu -- how fast can one CTA gather R scattered 256-B rows (one
// V row of d=128 bf16) from HBM into shared memory?  Design probe for the
// decode-side V gather (not part of the library).
//   m0: cp.async.bulk per row, rows spread over all 512 threads
//   m1: cp.async.bulk per row, issued by one warp
//   m2: ld.global.nc.v4 -> registers -> st.shared (16 lanes per row, all loads in flight)
//   m3: cp.async.cg 16 B, all threads
//   m4: cp.async.bulk.tensor tile::gather4 (4 rows / request, 128B swizzle, 2 col halves), one warp
// Each launch: G CTAs x R rows, random rows of a 1 GiB buffer (L2 misses);
// per-launch time from CUDA events over 50 launches (graph-free, so includes
// ~2-4 us launch overhead: compare methods, not absolutes; also reports a
// "null" kernel).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(bar), "r"(ph) : "memory");
}
constexpr int ROWB = 256;
constexpr int NT = 512;

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
template <int M>
__global__ void __launch_bounds__(NT, 1) gather_kernel(const uint8_t* V, const int* idx, int R, const __grid_constant__ CUtensorMap tmap, unsigned* sink, uint64_t* tdur) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    const int* my = idx + (size_t)blockIdx.x * R;
    const uint32_t b = smem_u32(&bar);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    const uint64_t tstart = gtimer();
    if (M == 0 || M == 1 || M == 4 || M == 5 || M == 6) {
        if (tid == 0) asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(R * ROWB) : "memory");
        if (M == 0) {
            for (int r = tid; r < R; r += NT)
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sm + r * ROWB)),
                             "l"(V + (size_t)my[r] * ROWB), "r"(ROWB), "r"(b) : "memory");
        } else if (M == 1) {
            if (tid < 32)
                for (int r = tid; r < R; r += 32)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sm + r * ROWB)),
                                 "l"(V + (size_t)my[r] * ROWB), "r"(ROWB), "r"(b) : "memory");
        } else if (M == 5) {  // bulk per row, lane 0 of every warp
            if ((tid & 31) == 0)
                for (int r = tid >> 5; r < R; r += NT / 32)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sm + r * ROWB)),
                                 "l"(V + (size_t)my[r] * ROWB), "r"(ROWB), "r"(b) : "memory");
        } else {
            // 4 rows x 64 cols (128 B) per request; two requests per 4-row group (cols 0, 64)
            // M == 4: lanes of warp 0; M == 6: lane 0 of every warp
            const bool issuer = (M == 4) ? (tid < 32) : ((tid & 31) == 0);
            const int q0 = (M == 4) ? tid : (tid >> 5), qs = (M == 4) ? 32 : NT / 32;
            if (issuer)
                for (int q = q0; q < 2 * (R / 4); q += qs) {
                    const int grp = q >> 1, half = q & 1;
                    const uint32_t dst = smem_u32(sm + grp * 4 * ROWB + half * 512);
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
                        "l"(&tmap), "r"(half * 64), "r"(my[4 * grp]), "r"(my[4 * grp + 1]), "r"(my[4 * grp + 2]), "r"(my[4 * grp + 3]), "r"(b)
                        : "memory");
                }
        }
        mbar_wait(b, 0);
    } else if (M == 2) {
        // 16 lanes per row, every thread keeps up to 8 loads in flight
        const int per = (R * 16 + NT - 1) / NT;
        uint4 v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int e = tid + u * NT;
            if (u < per && e < R * 16) {
                const uint8_t* src = V + (size_t)my[e >> 4] * ROWB + (e & 15) * 16;
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src));
            }
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int e = tid + u * NT;
            if (u < per && e < R * 16) *reinterpret_cast<uint4*>(sm + (size_t)e * 16) = v[u];
        }
    } else if (M == 3) {
        for (int e = tid; e < R * 16; e += NT) {
            const uint8_t* src = V + (size_t)my[e >> 4] * ROWB + (e & 15) * 16;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm + (size_t)e * 16)), "l"(src) : "memory");
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) tdur[blockIdx.x] = gtimer() - tstart;
    if (sm[(tid * 97) % (R * ROWB)] == 0x5a && tid == 7) atomicAdd(sink, 1u);
}

__global__ void null_kernel(unsigned* sink) {
    if (threadIdx.x == 9999) *sink = 1;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const size_t NROWS = (size_t)1 << 22;  // 1 GiB of 256-B rows
    uint8_t* V;
    cudaMalloc(&V, NROWS * ROWB);
    cudaMemset(V, 1, NROWS * ROWB);
    unsigned* sink;
    cudaMalloc(&sink, 4);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap tmap;
    {
        cuuint64_t dims[2] = {128, NROWS};
        cuuint64_t strides[1] = {ROWB};
        cuuint32_t box[2] = {64, 1};
        cuuint32_t es[2] = {1, 1};
        CUresult r = ((EncodeFn)fn)(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, V, dims, strides, box, es,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("tensor map encode: %d\n", (int)r);
    }
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(gather_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gather_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gather_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gather_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gather_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gather_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(gather_kernel<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    uint64_t* tdur;
    cudaMalloc(&tdur, 148 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int NREP = 50;
    for (int G : {64, 148}) {
        for (int R : {64, 256, 512}) {
            std::vector<int> h((size_t)NREP * G * R);
            srand(1234);
            for (auto& x : h) x = (int)(((uint64_t)rand() * 2654435761ull) % NROWS);
            int* idx;
            cudaMalloc(&idx, h.size() * 4);
            cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
            float tnull = 0;
            for (int m = -1; m < 7; ++m) {
                for (int pass = 0; pass < 2; ++pass) {
                    cudaEventRecord(e0);
                    for (int rep = 0; rep < NREP; ++rep) {
                        const int* ix = idx + (size_t)rep * G * R;
                        switch (m) {
                            case -1: null_kernel<<<G, NT>>>(sink); break;
                            case 0: gather_kernel<0><<<G, NT, smem>>>(V, ix, R, tmap, sink, tdur); break;
                            case 1: gather_kernel<1><<<G, NT, smem>>>(V, ix, R, tmap, sink, tdur); break;
                            case 2: gather_kernel<2><<<G, NT, smem>>>(V, ix, R, tmap, sink, tdur); break;
                            case 3: gather_kernel<3><<<G, NT, smem>>>(V, ix, R, tmap, sink, tdur); break;
                            case 4: gather_kernel<4><<<G, NT, smem>>>(V, ix, R, tmap, sink, tdur); break;
                            case 5: gather_kernel<5><<<G, NT, smem>>>(V, ix, R, tmap, sink, tdur); break;
                            case 6: gather_kernel<6><<<G, NT, smem>>>(V, ix, R, tmap, sink, tdur); break;
                        }
                    }
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                }
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                const float us = ms * 1000.f / NREP;
                if (m == -1) tnull = us;
                const char* names[] = {"null", "bulk/row all-thr", "bulk/row 1 warp", "ldg->sts", "cp.async16", "gather4 1 warp", "bulk/row lane0/warp", "gather4 lane0/warp"};
                double med = 0, mx = 0;
                if (m >= 0) {
                    std::vector<uint64_t> hd(G);
                    cudaMemcpy(hd.data(), tdur, G * 8, cudaMemcpyDeviceToHost);
                    std::sort(hd.begin(), hd.end());
                    med = hd[G / 2] / 1e3; mx = hd[G - 1] / 1e3;
                }
                printf("G=%3d R=%3d %-20s %7.2f us/launch; in-kernel gather median %6.2f max %6.2f us\n", G, R, names[m + 1], us, med, mx);
            }
            cudaError_t err = cudaGetLastError();
            if (err != cudaSuccess) printf("error: %s\n", cudaGetErrorString(err));
            cudaFree(idx);
        }
    }
    return 0;
}
