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

// ---------------------------------------------------------------- mRoPE
// Plan ("reconstruct the minimal contiguous positional grid along
// temporal, height, and width dimensions"; reading A23): one CTA
// per (dimension x, batch row b).  The kept tokens' coordinates in x are marked in
// a 65536-bit shared-memory bitmap; a block scan of the word popcounts gives
// every value its rank among the distinct kept values (coordinate compression,
// order-preserving); the CTA's largest rank goes to the workspace for the text
// start.  Coordinates outside [0, 65536) or a kept list that is not strictly
// ascending in [0, N_v) raise SVL_DEVFLAG_INDEX (and are clamped).
constexpr int kMropeMaxCoord = 65536;
constexpr int kMropeThreads = 1024;

__global__ void __launch_bounds__(kMropeThreads) mrope_plan_kernel(const MropeParams p) {
    __shared__ uint32_t bits[kMropeMaxCoord / 32];
    __shared__ uint32_t base[kMropeMaxCoord / 32];
    __shared__ uint32_t wsum[kMropeThreads / 32];
    __shared__ int rmax;
    const int x = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
    constexpr int WORDS = kMropeMaxCoord / 32, PER = WORDS / kMropeThreads;  // 2 words per thread
    for (int i = tid; i < WORDS; i += kMropeThreads) bits[i] = 0u;
    if (tid == 0) rmax = -1;
    __syncthreads();
    const int32_t* kb = p.kept + (int64_t)b * p.k;
    auto coord = [&](int i) {
        int m = kb[i];
        if (!(m >= 0 && m < p.nv) || (i > 0 && kb[i - 1] >= m)) {
            if (x == 0) raise_flag(p.flags, 1u /*SVL_DEVFLAG_INDEX*/);
            m = min(max(m, 0), p.nv - 1);
        }
        int v = p.coords[((int64_t)b * p.nv + m) * 3 + x];
        if (v < 0 || v >= kMropeMaxCoord) {
            raise_flag(p.flags, 1u /*SVL_DEVFLAG_INDEX*/);
            v = min(max(v, 0), kMropeMaxCoord - 1);
        }
        return v;
    };
    for (int i = tid; i < p.k; i += kMropeThreads) {
        const int v = coord(i);
        atomicOr(&bits[v >> 5], 1u << (v & 31));
    }
    __syncthreads();
    // exclusive prefix of the word popcounts: PER words per thread, then a block scan
    uint32_t c[PER], tot = 0u;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        c[j] = (uint32_t)__popc(bits[tid * PER + j]);
        tot += c[j];
    }
    const int lane = tid & 31, warp = tid >> 5;
    uint32_t incl = tot;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = wsum[lane];
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, off);
            if (lane >= off) w += y;
        }
        wsum[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    uint32_t run = incl - tot + (warp > 0 ? wsum[warp - 1] : 0u);
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        base[tid * PER + j] = run;
        run += c[j];
    }
    __syncthreads();
    int my_max = -1;
    for (int i = tid; i < p.k; i += kMropeThreads) {
        const int v = coord(i);
        const int r = (int)(base[v >> 5] + (uint32_t)__popc(bits[v >> 5] & ((1u << (v & 31)) - 1u)));
        p.new_coords[((int64_t)b * p.k + i) * 3 + x] = r;
        my_max = max(my_max, r);
    }
    atomicMax(&rmax, my_max);
    __syncthreads();
    if (tid == 0) p.dim_max[b * 3 + x] = rmax;
}

// Apply (post-RoPE keys recomputed from the stored pre-RoPE keys):
// output row w as in the unified remap; pair c takes the position of its section
// (t for c < sec0, h for c < sec0 + sec1, else w); text rows take their scalar
// position on every section (system row w: w; later text row i: text_start + i,
// text_start = vb + 1 + max over dimensions of the kept ranks).  Angles, sine,
// cosine and rotation in double, bf16 RNE output; V compacted.
__global__ void __launch_bounds__(256) mrope_apply_kernel(const MropeParams p) {
    const int b = blockIdx.y;
    const int half = p.d / 2;
    int L = p.seq_len[b];
    if (L < p.vb + p.nv || L > p.capacity) {
        if (threadIdx.x == 0 && blockIdx.x == 0) raise_flag(p.flags, 4u /*SPAN*/);
        L = min(max(L, p.vb + p.nv), p.capacity);
    }
    const int n_out = p.vb + p.k + (L - p.vb - p.nv);
    const int mx = max(p.dim_max[b * 3], max(p.dim_max[b * 3 + 1], p.dim_max[b * 3 + 2]));
    const int text_start = (p.k > 0) ? p.vb + 1 + mx : p.vb;
    if (p.text_start_out && blockIdx.x == 0 && threadIdx.x == 0) p.text_start_out[b] = text_start;
    const int hp = half / 2;  // one thread per (row, two adjacent pairs)
    const int64_t total = (int64_t)n_out * hp;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int w = (int)(e / hp), c = 2 * (int)(e % hp);
        int old;
        double pos[3];
        if (w < p.vb) {
            old = w;
            pos[0] = pos[1] = pos[2] = (double)w;
        } else if (w < p.vb + p.k) {
            const int i = w - p.vb;
            old = p.vb + min(max(p.kept[(int64_t)b * p.k + i], 0), p.nv - 1);
#pragma unroll
            for (int x = 0; x < 3; ++x) pos[x] = (double)(p.vb + p.new_coords[((int64_t)b * p.k + i) * 3 + x]);
        } else {
            old = w - p.k + p.nv;
            pos[0] = pos[1] = pos[2] = (double)(text_start + (w - p.vb - p.k));
        }
        const int s0 = (c < p.sec0) ? 0 : (c < p.sec0 + p.sec1) ? 1 : 2;
        const int s1 = (c + 1 < p.sec0) ? 0 : (c + 1 < p.sec0 + p.sec1) ? 1 : 2;
        double sn0, cs0, sn1, cs1;
        sincos(pos[s0] * exp2(-2.0 * (double)c / (double)p.d * p.log2_base), &sn0, &cs0);
        sincos(pos[s1] * exp2(-2.0 * (double)(c + 1) / (double)p.d * p.log2_base), &sn1, &cs1);
        for (int G = 0; G < p.Hkv; ++G) {
            const __nv_bfloat162* xk = reinterpret_cast<const __nv_bfloat162*>(
                p.K + (int64_t)b * p.ksb + (int64_t)G * p.ksh + (int64_t)old * p.kst);
            __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(p.Ko + (int64_t)b * p.osb + (int64_t)G * p.osh +
                                                                  (int64_t)w * p.ost);
            const float2 a = __bfloat1622float2(xk[c / 2]), z = __bfloat1622float2(xk[(c + half) / 2]);
            const double a0 = a.x, a1 = a.y, z0 = z.x, z1 = z.y;
            o[c / 2] = __halves2bfloat162(__double2bfloat16(a0 * cs0 - z0 * sn0), __double2bfloat16(a1 * cs1 - z1 * sn1));
            o[(c + half) / 2] =
                __halves2bfloat162(__double2bfloat16(z0 * cs0 + a0 * sn0), __double2bfloat16(z1 * cs1 + a1 * sn1));
            if (p.V) {
                const uint2* v = reinterpret_cast<const uint2*>(p.V + (int64_t)b * p.vsb + (int64_t)G * p.vsh +
                                                                (int64_t)old * p.vst);
                uint2* vo = reinterpret_cast<uint2*>(p.Vo + (int64_t)b * p.vosb + (int64_t)G * p.vosh + (int64_t)w * p.vost);
                vo[c / 2] = v[c / 2];
            }
        }
    }
}

}  // namespace

cudaError_t launch_mrope_remap(const MropeParams& p, int max_rows, cudaStream_t s) {
    mrope_plan_kernel<<<dim3(3, p.B), kMropeThreads, 0, s>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int64_t per_b = (int64_t)max_rows * (p.d / 4);
    const int blocks = (int)std::min<int64_t>((per_b + 255) / 256, 4096);
    mrope_apply_kernel<<<dim3(std::max(blocks, 1), p.B), 256, 0, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_rope_remap(const RopeParams& p, int max_rows, cudaStream_t s) {
    const int64_t per_b = (int64_t)max_rows * (p.d / 4);
    const int blocks = (int)std::min<int64_t>((per_b + 255) / 256, 4096);
    rope_remap_kernel<<<dim3(blocks, p.B), 256, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace svl
