// pack.cu -- pack-once of the retained KV: svl_pack_kv.
//
// the selected visual KV "are compactly packed into a contiguous
// memory region" so that the decode steps of a round attend a dense cache
// (SPEC.md:315-323 pack_active).  Per unit (b, KV group G) the packed cache holds
//   [0, vb)                 the system rows
//   [vb, vb + k)            K/V[vb + vis_idx[b][G][m]], m ascending
//   [vb + k, vb + k + T_a)  the rows after the visual span, T_a = seq_len - vb - N_v
// so svl_sparse_decode_attn over it (visual_len = k, vis_idx = 0..k-1, seq_len - N_v + k)
// attends exactly the same rows, in the same order, as over the original cache.
// HBM-bound copy: one 16-byte chunk per thread, K and V interleaved.
#include "common.cuh"
#include "kernels.h"

namespace svl {

namespace {

template <int D>
__global__ void __launch_bounds__(256) pack_kernel(const PackParams p) {
    constexpr int CH = D / 8;
    const int u = blockIdx.y;
    const int b = u / p.Hkv, G = u % p.Hkv;
    int L = p.seq_len[b];
    if (L < p.vb + p.nv || L > p.capacity) {
        if (threadIdx.x == 0 && blockIdx.x == 0) raise_flag(p.flags, 4u /*SPAN*/);
        L = min(max(L, p.vb + p.nv), p.capacity);
    }
    const int n_out = p.vb + p.k + (L - p.vb - p.nv);
    const int32_t* idx = p.idx + ((int64_t)b * (p.shared ? 1 : p.Hkv) + (p.shared ? 0 : G)) * p.k;
    const uint16_t* Kb = p.K + (int64_t)b * p.ksb + (int64_t)G * p.ksh;
    const uint16_t* Vb = p.V + (int64_t)b * p.vsb + (int64_t)G * p.vsh;
    uint16_t* Pk = p.Kp + (int64_t)b * p.pksb + (int64_t)G * p.pksh;
    uint16_t* Pv = p.Vp + (int64_t)b * p.pvsb + (int64_t)G * p.pvsh;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n_out * CH * 2; e += gridDim.x * blockDim.x) {
        const int kv = e & 1, c = (e >> 1) % CH, w = (e >> 1) / CH;
        int row;
        if (w < p.vb) {
            row = w;
        } else if (w < p.vb + p.k) {
            const int m = w - p.vb;
            const int x = idx[m];
            if (!(x >= 0 && x < p.nv) || (m > 0 && idx[m - 1] >= x)) {
                if (c == 0 && kv == 0) raise_flag(p.flags, 1u /*SVL_DEVFLAG_INDEX*/);
            }
            row = p.vb + min(max(x, 0), p.nv - 1);
        } else {
            row = w - p.k + p.nv;
        }
        if (kv == 0)
            reinterpret_cast<uint4*>(Pk + (int64_t)w * p.pkst)[c] = reinterpret_cast<const uint4*>(Kb + (int64_t)row * p.kst)[c];
        else
            reinterpret_cast<uint4*>(Pv + (int64_t)w * p.pvst)[c] = reinterpret_cast<const uint4*>(Vb + (int64_t)row * p.vst)[c];
    }
}

}  // namespace

cudaError_t launch_pack(const PackParams& p, int d, int max_rows, cudaStream_t s) {
    const int per_unit = max_rows * (d / 8) * 2;
    const dim3 grid((unsigned)((per_unit + 255) / 256), (unsigned)(p.B * p.Hkv));
    if (d == 128) pack_kernel<128><<<grid, 256, 0, s>>>(p);
    else if (d == 64) pack_kernel<64><<<grid, 256, 0, s>>>(p);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

}  // namespace svl
