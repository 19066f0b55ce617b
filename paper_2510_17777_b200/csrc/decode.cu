// decode.cu -- split-K gathered flash-decoding + log-sum-exp merge
// (SURVEY.md 8(a) a4, a5).
//
// PAPER.md:121 / 433: decode attention over the active set only -- all text
// rows plus the k retrieved visual rows ("less relevant tokens
// remain cached but inactive"; SPEC.md:315-323 pack_active order).  For each
// unit (b, KV group G) the attended row list
//     [0, vb)  U  {vb + idx[m]}  U  [vb + N_v, seq_len)
// (ascending) is cut into S contiguous splits.  One CTA per (split, unit):
//   1. builds its row ids (validating idx: in range, strictly ascending),
//   2. gathers the K and V rows with cp.async (16-byte, L1-bypassing) into
//      XOR-swizzled shared memory -- all of the split's rows in flight at once,
//   3. per warp and 16-row tile: S = q K^T with mma.sync m16n8k16 (heads are
//      M, rows are N, the contraction d is permuted consistently so K chunks
//      are read with conflict-free 128-bit LDS), online softmax in base 2,
//      O += P V with P split into bf16 hi + lo parts (two MMAs; ~2^-17
//      relative error instead of bf16's 2^-9) and V B-fragments from
//      ldmatrix.trans,
//   4. merges its 4 warps and stores the unnormalised partial (o, m, l).
// merge_kernel then combines the S partials of each (unit, head) in split
// order: M = max m_i, out = sum e^{m_i-M} o_i / sum e^{m_i-M} l_i,
// lse = M + log sum e^{m_i-M} l_i (north star step 3).
#include "common.cuh"
#include "kernels.h"

namespace svl {

namespace {

constexpr int NTH = kDecodeThreads;
constexpr int RM = kDecodeRowsMax;

template <int D>
struct DecodeSmem {
    static constexpr int CH = D / 8;             // 16-byte chunks per row
    static constexpr int ROW_BYTES = D * 2;
    static constexpr int K_OFF = 0;
    static constexpr int V_OFF = RM * ROW_BYTES;
    static constexpr int ROWS_OFF = 2 * RM * ROW_BYTES;
    static constexpr int BYTES = ROWS_OFF + RM * 4;
};

// swizzles (physical 16-byte chunk within a row)
SVL_DEV int swz_k(int row, int c) { return c ^ ((row & 1) << 2); }  // LDS.128 pattern
SVL_DEV int swz_v(int row, int c) { return c ^ (row & 7); }         // ldmatrix.trans pattern

template <int D>
__global__ void __launch_bounds__(NTH) decode_kernel(const DecodeParams p) {
    using SM = DecodeSmem<D>;
    constexpr int CH = SM::CH;
    constexpr int NCH = D / 32;  // chunks per thread per row in the permuted-k layout
    constexpr int NVT = D / 8;   // n-tiles of the output
    extern __shared__ __align__(128) uint8_t smem[];
    const uint32_t sK = smem_u32(smem + SM::K_OFF);
    const uint32_t sV = smem_u32(smem + SM::V_OFF);
    int* rows = reinterpret_cast<int*>(smem + SM::ROWS_OFF);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int gid = lane >> 2, t = lane & 3;
    const int u = blockIdx.y, sp = blockIdx.x;
    const int b = u / p.Hkv, G = u % p.Hkv;
    const int U = p.shared ? 1 : p.Hkv;
    const int uG = p.shared ? 0 : G;

    int L = p.seq_len[b];
    if (L < p.vb + p.nv || L > p.capacity) {
        if (tid == 0 && sp == 0) raise_flag(p.flags, 4u /*SPAN*/);
        L = min(max(L, p.vb + p.nv), p.capacity);
    }
    const int n_att = p.vb + p.k + (L - p.vb - p.nv);
    const int w0 = (int)((int64_t)sp * n_att / p.S);
    const int w1 = (int)((int64_t)(sp + 1) * n_att / p.S);
    const int nrows = w1 - w0;  // <= RM (host guarantees)
    const int ntiles = (nrows + 15) >> 4;

    // ---- 1. row ids
    const int32_t* idx = p.idx + ((int64_t)b * U + uG) * p.k;
    bool bad = false;
    for (int i = tid; i < ntiles * 16; i += NTH) {
        int row = -1;
        const int w = w0 + i;
        if (i < nrows) {
            if (w < p.vb) {
                row = w;
            } else if (w < p.vb + p.k) {
                const int m = w - p.vb;
                const int x = idx[m];
                const bool ok = (x >= 0 && x < p.nv) && (m == 0 || idx[m - 1] < x);
                if (ok) row = p.vb + x;
                else bad = true;
            } else {
                row = w - p.k + p.nv;
            }
        }
        rows[i] = row;
    }
    if (bad) raise_flag(p.flags, 1u /*SVL_DEVFLAG_INDEX*/);
    __syncthreads();

    // ---- 2. gather K and V rows (two commit groups: tiles [0,4) and [4,8))
    const uint16_t* Kb = p.K + (int64_t)b * p.ksb + (int64_t)G * p.ksh;
    const uint16_t* Vb = p.V + (int64_t)b * p.vsb + (int64_t)G * p.vsh;
    for (int grp = 0; grp < 2; ++grp) {
        const int r0 = grp * 64, r1 = min(ntiles * 16, r0 + 64);
        for (int i = tid; i < (r1 - r0) * CH; i += NTH) {
            const int r = r0 + i / CH, c = i % CH;
            const int row = rows[r];
            const bool valid = row >= 0;
            const int rr = valid ? row : 0;
            cp_async16(sK + r * SM::ROW_BYTES + swz_k(r, c) * 16, Kb + (int64_t)rr * p.kst + c * 8, valid);
            cp_async16(sV + r * SM::ROW_BYTES + swz_v(r, c) * 16, Vb + (int64_t)rr * p.vst + c * 8, valid);
        }
        cp_async_commit();
    }

    // ---- q A-fragments (heads gid, gid+8 of the group; zero beyond g)
    uint4 qa[NCH], qb[NCH];
    {
        const int ha = gid, hb = gid + 8;
#pragma unroll
        for (int i = 0; i < NCH; ++i) qa[i] = qb[i] = make_uint4(0, 0, 0, 0);
        if (ha < p.g) {
            const uint4* qr = reinterpret_cast<const uint4*>(p.q + ((int64_t)b * p.H + G * p.g + ha) * D);
#pragma unroll
            for (int i = 0; i < NCH; ++i) qa[i] = qr[t + 4 * i];
        }
        if (hb < p.g) {
            const uint4* qr = reinterpret_cast<const uint4*>(p.q + ((int64_t)b * p.H + G * p.g + hb) * D);
#pragma unroll
            for (int i = 0; i < NCH; ++i) qb[i] = qr[t + 4 * i];
        }
    }

    float o[NVT][4];
#pragma unroll
    for (int n = 0; n < NVT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;

    for (int grp = 0; grp < 2; ++grp) {
        if (grp == 0) cp_async_wait<1>();
        else cp_async_wait<0>();
        __syncthreads();
        const int tile = grp * 4 + warp;
        if (tile >= ntiles) continue;
        const int tb = tile * 16;
        // S = q K^T : two n-tiles of 8 rows
        float s[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
            const int r = tb + nt * 8 + gid;
#pragma unroll
            for (int i = 0; i < NCH; ++i) {
                const uint4 kc = lds128(sK + r * SM::ROW_BYTES + swz_k(r, t + 4 * i) * 16);
                {
                    const uint32_t a[4] = {qa[i].x, qb[i].x, qa[i].y, qb[i].y};
                    mma_bf16_16816(s[nt], a, kc.x, kc.y);
                }
                {
                    const uint32_t a[4] = {qa[i].z, qb[i].z, qa[i].w, qb[i].w};
                    mma_bf16_16816(s[nt], a, kc.z, kc.w);
                }
            }
        }
        // scale + mask (C layout: c0,c1 -> head gid, rows 2t,2t+1; c2,c3 -> head gid+8)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int r = tb + nt * 8 + 2 * t + (e & 1);
                s[nt][e] = (rows[r] >= 0) ? s[nt][e] * p.scale2 : -INFINITY;
            }
        float mx_a = fmaxf(fmaxf(s[0][0], s[0][1]), fmaxf(s[1][0], s[1][1]));
        float mx_b = fmaxf(fmaxf(s[0][2], s[0][3]), fmaxf(s[1][2], s[1][3]));
        mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, 1));
        mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, 2));
        mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, 1));
        mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, 2));
        const float mn_a = fmaxf(m_a, mx_a), mn_b = fmaxf(m_b, mx_b);
        const float al_a = (mn_a == -INFINITY) ? 1.f : fast_exp2(m_a - mn_a);
        const float al_b = (mn_b == -INFINITY) ? 1.f : fast_exp2(m_b - mn_b);
        m_a = mn_a;
        m_b = mn_b;
        float pr[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            pr[nt][0] = (mn_a == -INFINITY) ? 0.f : fast_exp2(s[nt][0] - mn_a);
            pr[nt][1] = (mn_a == -INFINITY) ? 0.f : fast_exp2(s[nt][1] - mn_a);
            pr[nt][2] = (mn_b == -INFINITY) ? 0.f : fast_exp2(s[nt][2] - mn_b);
            pr[nt][3] = (mn_b == -INFINITY) ? 0.f : fast_exp2(s[nt][3] - mn_b);
        }
        l_a = l_a * al_a + (pr[0][0] + pr[0][1] + pr[1][0] + pr[1][1]);
        l_b = l_b * al_b + (pr[0][2] + pr[0][3] + pr[1][2] + pr[1][3]);
#pragma unroll
        for (int n = 0; n < NVT; ++n) {
            o[n][0] *= al_a; o[n][1] *= al_a;
            o[n][2] *= al_b; o[n][3] *= al_b;
        }
        // P as A operand (k = 16 tile rows), split hi + lo
        uint32_t ph[4], pl[4];
        {
            const float v[4][2] = {{pr[0][0], pr[0][1]}, {pr[0][2], pr[0][3]},
                                   {pr[1][0], pr[1][1]}, {pr[1][2], pr[1][3]}};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                ph[i] = pack_bf16(v[i][0], v[i][1]);
                pl[i] = pack_bf16(v[i][0] - bf16lo(ph[i]), v[i][1] - bf16hi(ph[i]));
            }
        }
        // O += P V : V B-fragments via ldmatrix.trans, two n-tiles per x4
        const int mi = lane >> 3, rin = lane & 7;
        const int vrow = tb + (mi & 1) * 8 + rin;
#pragma unroll
        for (int j = 0; j < NVT / 2; ++j) {
            const int c = 2 * j + (mi >> 1);
            uint32_t v0, v1, v2, v3;
            ldsm_x4_trans(sV + vrow * SM::ROW_BYTES + swz_v(vrow, c) * 16, v0, v1, v2, v3);
            mma_bf16_16816(o[2 * j], ph, v0, v1);
            mma_bf16_16816(o[2 * j], pl, v0, v1);
            mma_bf16_16816(o[2 * j + 1], ph, v2, v3);
            mma_bf16_16816(o[2 * j + 1], pl, v2, v3);
        }
    }

    // ---- 4. warp -> CTA merge (fixed warp order), partial store
    l_a += __shfl_xor_sync(0xffffffffu, l_a, 1);
    l_a += __shfl_xor_sync(0xffffffffu, l_a, 2);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, 1);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, 2);
    __syncthreads();  // staging buffers are free now
    float* wo = reinterpret_cast<float*>(smem);          // [4][16][D]
    float* wm = wo + 4 * 16 * D;                          // [4][16]
    float* wl = wm + 4 * 16;                              // [4][16]
#pragma unroll
    for (int n = 0; n < NVT; ++n) {
        const int col = n * 8 + 2 * t;
        wo[(warp * 16 + gid) * D + col] = o[n][0];
        wo[(warp * 16 + gid) * D + col + 1] = o[n][1];
        wo[(warp * 16 + gid + 8) * D + col] = o[n][2];
        wo[(warp * 16 + gid + 8) * D + col + 1] = o[n][3];
    }
    if (t == 0) {
        wm[warp * 16 + gid] = m_a;
        wm[warp * 16 + gid + 8] = m_b;
        wl[warp * 16 + gid] = l_a;
        wl[warp * 16 + gid + 8] = l_b;
    }
    __syncthreads();
    float* part = p.part + ((int64_t)u * p.S + sp) * p.g * (D + 2);
    for (int i = tid; i < p.g * D; i += NTH) {
        const int h = i / D, dd = i % D;
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < 4; ++w) M = fmaxf(M, wm[w * 16 + h]);
        float acc = 0.f;
        if (M != -INFINITY) {
#pragma unroll
            for (int w = 0; w < 4; ++w) acc += fast_exp2(wm[w * 16 + h] - M) * wo[(w * 16 + h) * D + dd];
        }
        part[h * D + dd] = acc;
    }
    for (int h = tid; h < p.g; h += NTH) {
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < 4; ++w) M = fmaxf(M, wm[w * 16 + h]);
        float l = 0.f;
        if (M != -INFINITY) {
#pragma unroll
            for (int w = 0; w < 4; ++w) l += fast_exp2(wm[w * 16 + h] - M) * wl[w * 16 + h];
        }
        part[p.g * D + h] = M;
        part[p.g * D + p.g + h] = l;
    }
}

// one CTA per (unit, head); threads over d
template <int D>
__global__ void __launch_bounds__(D / 2) merge_kernel(const DecodeParams p) {
    const int u = blockIdx.y, h = blockIdx.x;
    const int b = u / p.Hkv, G = u % p.Hkv;
    const int dd = threadIdx.x * 2;
    const float* base = p.part + (int64_t)u * p.S * p.g * (D + 2);
    const int stride = p.g * (D + 2);
    // split weights: all (m_s, l_s) loads issued in parallel, then reduced in
    // a fixed order (deterministic)
    __shared__ float sw[kMergeMaxSplits], sl[kMergeMaxSplits];
    __shared__ float sM;
    for (int s = threadIdx.x; s < p.S; s += blockDim.x) {
        sw[s] = base[s * stride + p.g * D + h];
        sl[s] = base[s * stride + p.g * D + p.g + h];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float M = -INFINITY;
        for (int s = 0; s < p.S; ++s) M = fmaxf(M, sw[s]);
        sM = M;
    }
    __syncthreads();
    const float M = sM;
    for (int s = threadIdx.x; s < p.S; s += blockDim.x)
        sw[s] = (M == -INFINITY) ? 0.f : exp2f(sw[s] - M);
    __syncthreads();
    float o0 = 0.f, o1 = 0.f, l = 0.f;
#pragma unroll 8
    for (int s = 0; s < p.S; ++s) {
        const float2 ov = *reinterpret_cast<const float2*>(base + s * stride + h * D + dd);
        o0 += sw[s] * ov.x;
        o1 += sw[s] * ov.y;
        l += sw[s] * sl[s];
    }
    const int hh = G * p.g + h;
    const float inv = (l > 0.f) ? 1.f / l : 0.f;
    *reinterpret_cast<float2*>(p.out + ((int64_t)b * p.H + hh) * D + dd) = make_float2(o0 * inv, o1 * inv);
    if (p.lse_out && threadIdx.x == 0)
        p.lse_out[(int64_t)b * p.H + hh] = (l > 0.f) ? (M + log2f(l)) * kLn2 : -INFINITY;
}

template <int D>
cudaError_t launch_decode_t(const DecodeParams& p, cudaStream_t s) {
    using SM = DecodeSmem<D>;
    static bool attr_done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_done[dev]) {
        cudaError_t e = cudaFuncSetAttribute(decode_kernel<D>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, SM::BYTES);
        if (e == cudaSuccess) e = set_max_carveout(decode_kernel<D>);
        if (e == cudaSuccess) e = set_max_carveout(merge_kernel<D>);
        if (e != cudaSuccess) return e;
        attr_done[dev] = true;
    }
    static_assert(4 * 16 * D * 4 + 4 * 16 * 8 <= SM::BYTES, "merge scratch must fit");
    dim3 grid(p.S, p.B * p.Hkv);
    decode_kernel<D><<<grid, NTH, SM::BYTES, s>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    merge_kernel<D><<<dim3(p.g, p.B * p.Hkv), D / 2, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_decode(const DecodeParams& p, int d, cudaStream_t s) {
    if (d == 128) return launch_decode_t<128>(p, s);
    if (d == 64) return launch_decode_t<64>(p, s);
    return cudaErrorInvalidValue;
}

}  // namespace svl
