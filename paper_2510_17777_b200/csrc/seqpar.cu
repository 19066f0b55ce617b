// seqpar.cu -- the small kernels of the sequence-split (context-parallel)
// fresh step: a (b, KV group) unit's visual span
// split over P_s ranks (B = 1 on 8 GPUs: 4 KV heads x 2 sequence halves), with
// three latency-bound exchanges between the shards (PAPER.md:351 long-context
// retention motivates keeping B = 1 requests fast at scale):
//   1. LSE partials -> svl_lse_combine: LSE = M + log sum_p exp(lse_p - M);
//   2. relevance scores of every shard -> one global top-k (svl_topk) ->
//      svl_shard_indices: the shard's kept rows, relative, padded with -1;
//   3. decode partials (out_p, lse_p) -> svl_merge_partials (north star a5):
//      out = sum_p e^{lse_p - M} out_p / sum_p e^{lse_p - M}, lse = M + log(...).
// lse_from_partials_kernel turns the score kernel's per-chunk base-2 (max,
// sum) partials of a shard view into that view's natural-log LSE (exchange 1).
#include "common.cuh"
#include "kernels.h"

namespace svl {

namespace {

// one warp per (unit, query column): the chunk partials merged in chunk order
__global__ void lse_from_partials_kernel(const float2* part, int units, int C, int NCP, int NC, int g, int n_q,
                                         int H, int Hkv, float* lse_out) {
    const int warps = (blockDim.x >> 5) * gridDim.x;
    const int lane = threadIdx.x & 31;
    for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < units * NC; w += warps) {
        const int u = w / NC, col = w % NC;
        float m = -INFINITY, l = 0.f;
        for (int i = lane; i < C; i += 32) {
            const float2 pr = part[((int64_t)u * C + i) * NCP + col];
            const float M = fmaxf(m, pr.x);
            if (M != -INFINITY) {
                l = l * exp2f(m - M) + pr.y * exp2f(pr.x - M);
                m = M;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, m, off);
            const float l2 = __shfl_xor_sync(0xffffffffu, l, off);
            const float M = fmaxf(m, m2);
            if (M != -INFINITY) {
                l = l * exp2f(m - M) + l2 * exp2f(m2 - M);
                m = M;
            }
        }
        if (lane == 0) {
            const int b = u / Hkv, G = u % Hkv, r = col / g, h = G * g + col % g;
            lse_out[((int64_t)b * n_q + r) * H + h] = (m == -INFINITY) ? -INFINITY : (m + log2f(l)) * kLn2;
        }
    }
}

// lse[i] = M + log sum_p exp(parts[p][i] - M), p in rank order
__global__ void lse_combine_kernel(const float* parts, int P, int n, float* out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        float M = -INFINITY;
        for (int p = 0; p < P; ++p) M = fmaxf(M, parts[(int64_t)p * n + i]);
        float s = 0.f;
        if (M != -INFINITY)
            for (int p = 0; p < P; ++p) s += expf(parts[(int64_t)p * n + i] - M);
        out[i] = (M == -INFINITY) ? -INFINITY : M + logf(s);
    }
}

// per unit (one warp): the ascending global kept list's entries inside [lo, hi),
// relative to lo, then -1 padding to k entries (a contiguous run: the list is ascending)
__global__ void shard_indices_kernel(const int32_t* idx, int units, int k, int lo, int hi, int32_t* out) {
    const int lane = threadIdx.x & 31;
    for (int u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < units; u += (blockDim.x >> 5) * gridDim.x) {
        const int32_t* src = idx + (int64_t)u * k;
        int32_t* dst = out + (int64_t)u * k;
        // first entry >= lo (binary search, lane 0) then a coalesced copy
        int a = 0;
        if (lane == 0) {
            int l0 = 0, h0 = k;
            while (l0 < h0) {
                const int m = (l0 + h0) >> 1;
                if (src[m] < lo) l0 = m + 1;
                else h0 = m;
            }
            a = l0;
        }
        a = __shfl_sync(0xffffffffu, a, 0);
        for (int i = lane; i < k; i += 32) {
            const int j = a + i;
            const int32_t v = (j < k) ? src[j] : hi;
            dst[i] = (v < hi) ? v - lo : -1;
        }
    }
}

// out[b][h][c] from P partials (natural-log lse), rank order
__global__ void merge_partials_kernel(const float* out_parts, const float* lse_parts, int P, int rows, int d,
                                      float* out, float* lse_out) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * d; e += gridDim.x * blockDim.x) {
        const int r = e / d, c = e % d;
        float M = -INFINITY;
        for (int p = 0; p < P; ++p) M = fmaxf(M, lse_parts[(int64_t)p * rows + r]);
        float num = 0.f, den = 0.f;
        if (M != -INFINITY)
            for (int p = 0; p < P; ++p) {
                const float w = expf(lse_parts[(int64_t)p * rows + r] - M);
                num += w * out_parts[((int64_t)p * rows + r) * d + c];
                den += w;
            }
        out[e] = (den > 0.f) ? num / den : 0.f;
        if (c == 0 && lse_out) lse_out[r] = (den > 0.f) ? M + logf(den) : -INFINITY;
    }
}

int grid_for(int64_t n, int per) {
    const int64_t g = (n + per - 1) / per;
    return (int)(g < 1 ? 1 : (g > 4L * device_sm_count() ? 4L * device_sm_count() : g));
}

}  // namespace

cudaError_t launch_lse_from_partials(const float2* part, int units, int C, int NCP, int NC, int g, int n_q, int H,
                                     int Hkv, float* lse_out, cudaStream_t s) {
    lse_from_partials_kernel<<<grid_for((int64_t)units * NC * 32, 256), 256, 0, s>>>(part, units, C, NCP, NC, g, n_q,
                                                                                    H, Hkv, lse_out);
    return cudaGetLastError();
}

cudaError_t launch_lse_combine(const float* parts, int P, int n, float* out, cudaStream_t s) {
    lse_combine_kernel<<<grid_for(n, 256), 256, 0, s>>>(parts, P, n, out);
    return cudaGetLastError();
}

cudaError_t launch_shard_indices(const int32_t* idx, int units, int k, int lo, int hi, int32_t* out, cudaStream_t s) {
    shard_indices_kernel<<<grid_for((int64_t)units * 32, 256), 256, 0, s>>>(idx, units, k, lo, hi, out);
    return cudaGetLastError();
}

cudaError_t launch_merge_partials(const float* out_parts, const float* lse_parts, int P, int rows, int d, float* out,
                                  float* lse_out, cudaStream_t s) {
    merge_partials_kernel<<<grid_for((int64_t)rows * d, 256), 256, 0, s>>>(out_parts, lse_parts, P, rows, d, out,
                                                                         lse_out);
    return cudaGetLastError();
}

}  // namespace svl
