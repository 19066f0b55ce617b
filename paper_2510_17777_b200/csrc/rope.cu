// rope.cu -- unified RoPE remap after prefill pruning:
// svl_rope_remap.
//
// for unified RoPE, SparseVILA "simply retain[s] a contiguous range
// of position indices corresponding to the preserved visual tokens"
// recomputes post-RoPE keys from the stored pre-RoPE keys.  Per batch row b the
// compacted cache row w (= its new position) takes
//   old row w (w < vb) | vb + kept[b][w - vb] (w < vb + k) | w - k + N_v (later text)
// and K_out[w] = RoPE(K_pre[old], w) in the rotate-half convention, pairs
// (c, c + d/2), theta_c = w * base^(-2c/d); V rows are copied unchanged.
// The angle, its sine / cosine and the rotation are evaluated in double (the
// position reaches 10^5: a float angle would be off by ~10^-2 rad; fp32 products
// lose the small results of x1 cos - x2 sin), the output rounded to bf16 (RNE).  One thread per (row, pair c); the Hkv heads of
// the row reuse its sine and cosine.  HBM-bound: 2 x (K + V) rows moved.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace svl {

namespace {

__global__ void __launch_bounds__(256) rope_remap_kernel(const RopeParams p) {
    const int b = blockIdx.y;
    const int half = p.d / 2;
    int L = p.seq_len[b];
    if (L < p.vb + p.nv || L > p.capacity) {
        if (threadIdx.x == 0 && blockIdx.x == 0) raise_flag(p.flags, 4u /*SPAN*/);
        L = min(max(L, p.vb + p.nv), p.capacity);
    }
    const int n_out = p.vb + p.k + (L - p.vb - p.nv);
    const int hp = half / 2;  // one thread per (row, two adjacent pairs c, c + 1): 4-byte accesses
    const int64_t total = (int64_t)n_out * hp;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int w = (int)(e / hp), c = 2 * (int)(e % hp);
        int old;
        if (w < p.vb) {
            old = w;
        } else if (w < p.vb + p.k) {
            const int i = w - p.vb;
            const int x = p.kept[(int64_t)b * p.k + i];
            if (c == 0 && (!(x >= 0 && x < p.nv) || (i > 0 && p.kept[(int64_t)b * p.k + i - 1] >= x)))
                raise_flag(p.flags, 1u /*SVL_DEVFLAG_INDEX*/);
            old = p.vb + min(max(x, 0), p.nv - 1);
        } else {
            old = w - p.k + p.nv;
        }
        double sn0, cs0, sn1, cs1;
        sincos((double)w * exp2(-2.0 * (double)c / (double)p.d * p.log2_base), &sn0, &cs0);
        sincos((double)w * exp2(-2.0 * (double)(c + 1) / (double)p.d * p.log2_base), &sn1, &cs1);
        for (int G = 0; G < p.Hkv; ++G) {
            const __nv_bfloat162* x = reinterpret_cast<const __nv_bfloat162*>(
                p.K + (int64_t)b * p.ksb + (int64_t)G * p.ksh + (int64_t)old * p.kst);
            __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(p.Ko + (int64_t)b * p.osb + (int64_t)G * p.osh +
                                                                  (int64_t)w * p.ost);
            // rotation in double too (fp32 loses the small results of x1 cos - x2 sin to
            // cancellation): the output is the bf16 rounding of the exact value
            const float2 a = __bfloat1622float2(x[c / 2]), z = __bfloat1622float2(x[(c + half) / 2]);
            const double a0 = a.x, a1 = a.y, z0 = z.x, z1 = z.y;
            o[c / 2] = __halves2bfloat162(__double2bfloat16(a0 * cs0 - z0 * sn0), __double2bfloat16(a1 * cs1 - z1 * sn1));
            o[(c + half) / 2] =
                __halves2bfloat162(__double2bfloat16(z0 * cs0 + a0 * sn0), __double2bfloat16(z1 * cs1 + a1 * sn1));
            if (p.V) {
                const uint2* v = reinterpret_cast<const uint2*>(p.V + (int64_t)b * p.vsb + (int64_t)G * p.vsh +
                                                                (int64_t)old * p.vst);
                uint2* vo = reinterpret_cast<uint2*>(p.Vo + (int64_t)b * p.vosb + (int64_t)G * p.vosh + (int64_t)w * p.vost);
                vo[c / 2] = v[c / 2];  // d/4 chunks of 8 bytes = the whole row
            }
        }
    }
}

}  // namespace

cudaError_t launch_rope_remap(const RopeParams& p, int max_rows, cudaStream_t s) {
    const int64_t per_b = (int64_t)max_rows * (p.d / 4);
    const int blocks = (int)std::min<int64_t>((per_b + 255) / 256, 4096);
    rope_remap_kernel<<<dim3(blocks, p.B), 256, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace svl
