// pages.cu -- retrieval on page summaries (Quest-style:
// PAPER.md:527 "Quest estimates upper-bound attention scores for each page";
// north star "optionally on a page/chunk summary"; reading A22 in DESIGN.md).
//
// svl_page_summary: per (b, KV group) and page of `page` consecutive visual
// rows, the elementwise max and min of the keys (bf16, exact).  Built once per
// retained cache (prefill / round start); HBM-bound: reads the visual K once.
//
// svl_retrieve_pages, per unit (b, G), n_q * g <= 32 query rows:
//   1. page_score_kernel: ub2[n][p] = log2(e) * scale * sum_c max(q_n,c kmax_p,c,
//      q_n,c kmin_p,c) -- Quest's upper bound of every row logit of page p (one
//      warp per page, lanes over d, fixed shuffle tree); reads 2 d bf16 per page
//      instead of page * d: the scored-K bytes drop by page / 2;
//   2. page_norm_kernel: LSE2 over the unit's pages per query row (warp per row),
//      then score[p] = sum_n exp2(ub2[n][p] - LSE2[n]) in row order;
//   3. the cluster top-k of select.cu on the page scores (ties -> lower page);
//   4. page_expand_kernel: the kept pages' rows, ascending (relative to vb), for
//      svl_sparse_decode_attn.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace svl {

namespace {

__global__ void page_summary_kernel(const PageSumParams p) {
    const int CH = p.d / 8;
    const int64_t total = (int64_t)p.units * p.np * CH;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(e % CH);
        const int64_t t = e / CH;
        const int pg = (int)(t % p.np);
        const int u = (int)(t / p.np);
        const int b = u / p.Hkv, G = u % p.Hkv;
        const uint16_t* base = p.K + (int64_t)b * p.ksb + (int64_t)G * p.ksh + (int64_t)(p.vb + pg * p.page) * p.kst + c * 8;
        uint4 v = __ldg(reinterpret_cast<const uint4*>(base));
        __nv_bfloat162 mx[4], mn[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) mx[i] = mn[i] = reinterpret_cast<const __nv_bfloat162*>(&v)[i];
        for (int r = 1; r < p.page; ++r) {
            v = __ldg(reinterpret_cast<const uint4*>(base + (int64_t)r * p.kst));
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const __nv_bfloat162 x = reinterpret_cast<const __nv_bfloat162*>(&v)[i];
                mx[i] = __hmax2(mx[i], x);
                mn[i] = __hmin2(mn[i], x);
            }
        }
        const int64_t o = ((int64_t)u * p.np + pg) * p.d + c * 8;
        *reinterpret_cast<uint4*>(p.kmax + o) = *reinterpret_cast<const uint4*>(mx);
        *reinterpret_cast<uint4*>(p.kmin + o) = *reinterpret_cast<const uint4*>(mn);
    }
}

constexpr int kPageThreads = 256;
constexpr int kPagesPerBlock = 64;

// one warp per page: lane l holds dims [l * D/32, (l + 1) * D/32) of kmax / kmin
template <int D>
__global__ void __launch_bounds__(kPageThreads) page_score_kernel(const PageRetrParams p) {
    constexpr int PER = D / 32;
    __shared__ float qs[32 * D];  // the unit's query rows n = r * g + hh, fp32
    const int u = blockIdx.y, b = u / p.Hkv, G = u % p.Hkv;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int e = tid; e < p.NC * D; e += kPageThreads) {
        const int n = e / D, c = e % D, r = n / p.g, hh = n % p.g;
        qs[e] = __bfloat162float(__ushort_as_bfloat16(p.q[(((int64_t)b * p.n_q + r) * p.H + G * p.g + hh) * D + c]));
    }
    __syncthreads();
    for (int pg = blockIdx.x * kPagesPerBlock + warp; pg < min(p.np, (int)(blockIdx.x + 1) * kPagesPerBlock);
         pg += kPageThreads / 32) {
        const uint16_t* mxr = p.kmax + ((int64_t)u * p.np + pg) * D + lane * PER;
        const uint16_t* mnr = p.kmin + ((int64_t)u * p.np + pg) * D + lane * PER;
        float mx[PER], mn[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            mx[i] = __bfloat162float(__ushort_as_bfloat16(mxr[i]));
            mn[i] = __bfloat162float(__ushort_as_bfloat16(mnr[i]));
        }
        for (int n = 0; n < p.NC; ++n) {
            float acc = 0.f;
#pragma unroll
            for (int i = 0; i < PER; ++i) {
                const float qc = qs[n * D + lane * PER + i];
                acc += fmaxf(qc * mx[i], qc * mn[i]);
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            if (lane == 0) p.ub2[((int64_t)u * p.NC + n) * p.np + pg] = acc * p.scale2;
        }
    }
}

// per unit: warp n -> LSE2 of query row n over the pages; then the page scores
__global__ void __launch_bounds__(1024) page_norm_kernel(const PageRetrParams p) {
    __shared__ float lse2[32];
    const int u = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp < p.NC) {
        const float* row = p.ub2 + ((int64_t)u * p.NC + warp) * p.np;
        float m = -INFINITY;
        for (int pg = lane; pg < p.np; pg += 32) m = fmaxf(m, row[pg]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
        float s = 0.f;
        if (m != -INFINITY)
            for (int pg = lane; pg < p.np; pg += 32) s += exp2f(row[pg] - m);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane == 0) lse2[warp] = m + log2f(s);
    }
    __syncthreads();
    for (int pg = tid; pg < p.np; pg += blockDim.x) {
        float sc = 0.f;
        for (int n = 0; n < p.NC; ++n) sc += exp2f(p.ub2[((int64_t)u * p.NC + n) * p.np + pg] - lse2[n]);
        p.scores[(int64_t)u * p.np + pg] = sc;
    }
}

__global__ void page_expand_kernel(const int32_t* pidx, int units, int kp, int page, int32_t* rows) {
    const int64_t total = (int64_t)units * kp * page;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t um = e / page;  // (unit, m)
        rows[e] = pidx[um] * page + (int)(e % page);
    }
}

}  // namespace

cudaError_t launch_page_summary(const PageSumParams& p, cudaStream_t s) {
    const int64_t total = (int64_t)p.units * p.np * (p.d / 8);
    const int grid = (int)std::min<int64_t>((total + 255) / 256, 16L * device_sm_count());
    page_summary_kernel<<<std::max(grid, 1), 256, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_page_scores(const PageRetrParams& p, cudaStream_t s) {
    const dim3 grid((p.np + kPagesPerBlock - 1) / kPagesPerBlock, p.units);
    if (p.d == 128) page_score_kernel<128><<<grid, kPageThreads, 0, s>>>(p);
    else page_score_kernel<64><<<grid, kPageThreads, 0, s>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    page_norm_kernel<<<p.units, 1024, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_page_expand(const int32_t* pidx, int units, int kp, int page, int32_t* rows, cudaStream_t s) {
    const int64_t total = (int64_t)units * kp * page;
    if (total == 0) return cudaSuccess;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, 4L * device_sm_count());
    page_expand_kernel<<<grid, 256, 0, s>>>(pidx, units, kp, page, rows);
    return cudaGetLastError();
}

}  // namespace svl
