// retrieve_tc.cu -- question-chunk retrieval on the 5th-generation tensor cores
// (SURVEY.md 8(f) f1): svl_retrieve when n_q * g > 32.
//
// PAPER.md:124 (section 3.2): the query-aware relevance of every visual token is
// computed from the *question* rows, "concurrently with the FlashAttention2
// path during prefill".  With n_q question rows the per-unit work is a real
// contraction (M = n_q * g query columns against N_v keys, arithmetic
// intensity ~ n_q * g flop/B), so it runs on tcgen05:
//
//   qpack     Q_u = the n_q * g query rows of unit (b, G), row n = r * g + hh,
//             packed contiguous and zero padded to NQP (multiple of 256) rows.
//   pass 0    (only without lse_in) row log-sum-exp: S = Q_blk K_chunk^T with
//             M = 128 query rows, N = 256 keys per stage (TMEM accumulator);
//             one thread per query row folds a running (max, sum) over its
//             columns, causal limit j <= seq_len - n_q + r (FULL_PREFIX) or the
//             visual span only (VISUAL_ONLY); partials per (row, key chunk,
//             column quarter) -> workspace.
//   combine   LSE2[u][n] (base 2) from the partials, or lse_in * log2(e).
//   pass 1    column mass, operands swapped: S^T = K_blk Q_chunk^T with
//             M = 128 visual keys, N = 256 query rows per stage; one thread per
//             key sums exp2(s * scale2 - LSE2[n]) over its columns, so the
//             "visual share of the attention mass" of a
//             key is a per-thread row sum -- no cross-thread reduction.
//   select    the cluster top-k of select.cu (mode 2: precomputed scores).
//
// Both tensor-core passes share one kernel: a resident X tile (128 rows) and
// a 2-stage ring of Y tiles (256 rows), both loaded by tiled TMA with the
// 128-B swizzle (K-major UMMA operands), one elected thread issuing
// tcgen05.mma (M128 N256 K16) into a double-buffered TMEM accumulator
// (2 x 256 columns), 16 epilogue warps (four per TMEM lane quarter, 64
// columns each) reading it back with tcgen05.ld.
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace svl {

namespace {

constexpr int RT_THREADS = 640;  // w0 TMA producer, w1 MMA issuer, w2 TMEM owner, w3 spare, w4-w19 epilogue
constexpr int RT_EPI_WARPS = 16;  // 4 per TMEM lane quarter, 64 accumulator columns each
constexpr int RT_XROWS = 128;    // UMMA M
constexpr int RT_YROWS = 256;    // UMMA N per stage
constexpr int RT_NST = 2;        // Y ring stages

template <int D>
struct RtSmem {
    static constexpr int NB = D / 64;                          // 64-column (128-B) TMA boxes
    static constexpr int X_BYTES = NB * RT_XROWS * 128;
    static constexpr int Y_BYTES = NB * RT_YROWS * 128;
    static constexpr int X_OFF = 0;
    static constexpr int Y_OFF = X_OFF + X_BYTES;
    static constexpr int LSE_OFF = Y_OFF + RT_NST * Y_BYTES;  // pass 1: LSE2 of the unit's query rows
    static constexpr int RED_OFF = LSE_OFF + kRtMaxNQ * 4;    // pass 1: [2 halves][128 rows] column-half sums
    static constexpr int BAR_OFF = RED_OFF + 4 * RT_XROWS * 4;
    static constexpr int BYTES = BAR_OFF + 128;
    static_assert(X_OFF % 1024 == 0 && Y_OFF % 1024 == 0 && Y_BYTES % 1024 == 0, "swizzle atoms");
    static_assert(BYTES <= 227 * 1024, "shared memory");
};

__global__ void qpack_kernel(const RetrTcParams p, int D) {
    // one 16-B chunk per thread: Qpack[u][n][c] = q[b][r][G g + hh][c], zero past NQ
    const int CH = D / 8;
    const int64_t total = (int64_t)p.B * p.Hkv * p.NQP * CH;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(e % CH);
        const int64_t row = e / CH;
        const int n = (int)(row % p.NQP);
        const int u = (int)(row / p.NQP);
        const int b = u / p.Hkv, G = u % p.Hkv;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (n < p.NQ) {
            const int r = n / p.g, hh = n % p.g;
            v = reinterpret_cast<const uint4*>(p.q + (((int64_t)b * p.n_q + r) * p.H + G * p.g + hh) * D)[c];
        }
        reinterpret_cast<uint4*>(p.qpack + row * D)[c] = v;
    }
}

// One warp per query row: lanes fold a lane-strided share of the row's chunk
// partials, then a fixed butterfly -- deterministic, and the row's partials are
// read coalesced.
__global__ void lse_combine_kernel(const RetrTcParams p) {
    const int lane = threadIdx.x & 31;
    const int64_t total = (int64_t)p.B * p.Hkv * p.NQP;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t e = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); e < total; e += nwarps) {
        const int n = (int)(e % p.NQP);
        const int u = (int)(e / p.NQP);
        const int b = u / p.Hkv, G = u % p.Hkv;
        float out = INFINITY;  // padding rows: exp2(x - inf) = 0
        if (n < p.NQ) {
            const int r = n / p.g, hh = n % p.g;
            if (p.lse_in) {
                out = p.lse_in[((int64_t)b * p.n_q + r) * p.H + G * p.g + hh] * kLog2e;
            } else {
                float m = -INFINITY, l = 0.f;
                const float2* pp = p.part + e * p.npart;
                for (int i = lane; i < p.npart; i += 32) {
                    const float2 x = pp[i];
                    const float M = fmaxf(m, x.x);
                    if (M != -INFINITY) {
                        l = l * exp2f(m - M) + x.y * exp2f(x.x - M);
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
                out = m + log2f(l);
            }
            if (lane == 0 && out != out) raise_flag(p.flags, 2u /*NONFINITE*/);
        }
        if (lane == 0) p.lse2[e] = out;
    }
}

// MODE 0: row LSE partials (X = Q block, Y = K chunk stages).
// MODE 1: column mass      (X = K block, Y = Q chunk stages).
template <int MODE, int D>
__global__ void __launch_bounds__(RT_THREADS, 1) retr_tc_kernel(const __grid_constant__ RetrTcParams p) {
    using SM = RtSmem<D>;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr uint32_t IDESC = umma_idesc_bf16(RT_XROWS, RT_YROWS);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
    const uint32_t xfull = smem_u32(bars), yfull0 = smem_u32(bars + 1), yempty0 = smem_u32(bars + 1 + RT_NST);
    const uint32_t afull0 = smem_u32(bars + 1 + 2 * RT_NST), aempty0 = smem_u32(bars + 3 + 2 * RT_NST);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 5 + 2 * RT_NST);
    const uint32_t sX = smem_u32(smem + SM::X_OFF), sY = smem_u32(smem + SM::Y_OFF);

    const int u = (MODE == 0) ? blockIdx.z : blockIdx.y;
    const int b = u / p.Hkv, G = u % p.Hkv;
    int L = p.seq_len[b];
    if (L < p.vb + p.nv + p.n_q || L > p.capacity) {
        if (tid == 0 && blockIdx.x == 0) raise_flag(p.flags, 4u /*SPAN*/);
        L = min(max(L, p.vb + p.nv + p.n_q), p.capacity);
    }
    // geometry: X rows, Y stages
    int xrow0, y0 = 0, y1 = 0, nst;
    if (MODE == 0) {
        const int lo = p.visual_only ? p.vb : 0;
        const int hi = p.visual_only ? p.vb + p.nv : L;
        y0 = lo + blockIdx.x * p.chunk;
        y1 = min(hi, y0 + p.chunk);
        xrow0 = blockIdx.y * RT_XROWS;
        nst = y1 > y0 ? (y1 - y0 + RT_YROWS - 1) / RT_YROWS : 0;
    } else {
        xrow0 = p.vb + blockIdx.x * RT_XROWS;
        nst = p.NQP / RT_YROWS;
    }
    const int q4 = warp & 3, ch = (warp - 4) >> 2;  // epilogue: TMEM lane quarter, column half
    float2* part_out = nullptr;
    if (MODE == 0) {
        const int n = xrow0 + 32 * q4 + lane;
        part_out = p.part + ((int64_t)u * p.NQP + n) * p.npart + blockIdx.x * 4 + ch;
        if (nst == 0) {  // empty key chunk (seq_len shorter than the planned range)
            if (warp >= 4) *part_out = make_float2(-INFINITY, 0.f);
            return;
        }
    }

    if (tid == 0) {
        mbar_init(xfull, 1);
        for (int s = 0; s < RT_NST; ++s) {
            mbar_init(yfull0 + 8 * s, 1);
            mbar_init(yempty0 + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(afull0 + 8 * a, 1);
            mbar_init(aempty0 + 8 * a, RT_EPI_WARPS);
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(smem_u32(tslot), 512);
    float* lse_s = reinterpret_cast<float*>(smem + SM::LSE_OFF);
    if (MODE == 1)
        for (int i = tid; i < p.NQP; i += RT_THREADS) lse_s[i] = p.lse2[(int64_t)u * p.NQP + i];
    tc_fence_before();
    cta_sync();
    tc_fence_after();
    const uint32_t tbase = *tslot;

    if (warp == 0) {
        if (lane == 0) {
            mbar_arrive_expect_tx(xfull, (uint32_t)SM::X_BYTES);
#pragma unroll
            for (int hf = 0; hf < SM::NB; ++hf) {
                if (MODE == 0)
                    tma_load_4d(sX + hf * (RT_XROWS * 128), &p.xmap, hf * 64, xrow0, 0, u, xfull);
                else
                    tma_load_4d(sX + hf * (RT_XROWS * 128), &p.xmap, hf * 64, xrow0, G, b, xfull);
            }
            for (int s = 0; s < nst; ++s) {
                const int slot = s % RT_NST;
                if (s >= RT_NST) mbar_wait(yempty0 + 8 * slot, ((s / RT_NST) - 1) & 1);
                const uint32_t bar = yfull0 + 8 * slot;
                mbar_arrive_expect_tx(bar, (uint32_t)SM::Y_BYTES);
#pragma unroll
                for (int hf = 0; hf < SM::NB; ++hf) {
                    const uint32_t dst = sY + slot * SM::Y_BYTES + hf * (RT_YROWS * 128);
                    if (MODE == 0)
                        tma_load_4d(dst, &p.ymap, hf * 64, y0 + s * RT_YROWS, G, b, bar);
                    else
                        tma_load_4d(dst, &p.ymap, hf * 64, s * RT_YROWS, 0, u, bar);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            mbar_wait(xfull, 0);
            for (int s = 0; s < nst; ++s) {
                const int slot = s % RT_NST, a = s & 1;
                mbar_wait(yfull0 + 8 * slot, (s / RT_NST) & 1);
                if (s >= 2) mbar_wait(aempty0 + 8 * a, ((s >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t yb = sY + slot * SM::Y_BYTES;
#pragma unroll
                for (int j = 0; j < D / 16; ++j) {
                    const int hf = j >> 2, kk = j & 3;
                    umma_bf16(tbase + a * RT_YROWS, sw128_desc(sX + hf * (RT_XROWS * 128) + kk * 32),
                              sw128_desc(yb + hf * (RT_YROWS * 128) + kk * 32), IDESC, j > 0 ? 1u : 0u);
                }
                umma_commit(yempty0 + 8 * slot);
                umma_commit(afull0 + 8 * a);
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        const uint32_t trow = tbase + ((uint32_t)(32 * q4) << 16);
        // one warp = 32 accumulator rows x 64 columns per stage: both 32-column loads
        // in flight together, one wait, then the accumulator buffer is released to
        // the MMA issuer before the exponentials are computed from registers
        auto load64 = [&](int a, uint32_t (&va)[32], uint32_t (&vb)[32]) {
            const uint32_t t0 = trow + a * RT_YROWS + ch * 64;
            tmem_ld32_nowait(t0, va);
            tmem_ld32_nowait(t0 + 32, vb);
            tmem_wait_ld_tie(va);
            tmem_wait_ld_tie(vb);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(aempty0 + 8 * a);
        };
        if (MODE == 0) {
            const int n = xrow0 + 32 * q4 + lane;
            const int r = n / p.g;
            // causal limit of query row r (FULL_PREFIX): keys j <= L - n_q + r
            const int jend = p.visual_only ? y1 : min(y1, L - p.n_q + r + 1);
            float m = -INFINITY, l = 0.f;
            for (int s = 0; s < nst; ++s) {
                const int a = s & 1;
                mbar_wait(afull0 + 8 * a, (s >> 1) & 1);
                __syncwarp();  // tcgen05.ld is .aligned
                tc_fence_after();
                uint32_t va[32], vb[32];
                load64(a, va, vb);
                const int j0 = y0 + s * RT_YROWS + ch * 64;
                if (j0 + 64 > jend) {  // a stage crossing the causal / range limit: mask
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        if (j0 + i >= jend) va[i] = __float_as_uint(-INFINITY);
                        if (j0 + 32 + i >= jend) vb[i] = __float_as_uint(-INFINITY);
                    }
                }
                // max on the raw dot products (scale2 > 0), then 2^(s*scale2 - M) by one FMA +
                // one exponential per element; 3 of 4 exponentials on the SFU, 1 on the FP32 pipe
                float cm = -INFINITY;
#pragma unroll
                for (int i = 0; i < 32; ++i) cm = fmaxf(cm, fmaxf(__uint_as_float(va[i]), __uint_as_float(vb[i])));
                const float M = fmaxf(m, cm * p.scale2);  // an all-masked stage leaves (m, l) unchanged
                const float Ms = (M == -INFINITY) ? 0.f : M;
                float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const float ya = fmaf(__uint_as_float(va[i]), p.scale2, -Ms);
                    const float yb = fmaf(__uint_as_float(vb[i]), p.scale2, -Ms);
                    acc0 += fast_exp2(ya);
                    acc1 += ((i & 1) == 0) ? fast_exp2(yb) : ((yb < -126.f) ? 0.f : poly_exp2(yb));
                }
                l = l * fast_exp2(m - Ms) + (acc0 + acc1);
                m = M;
            }
            if (n < p.NQP) *part_out = make_float2(m, l);
        } else {
            float acc0 = 0.f, acc1 = 0.f;
            for (int s = 0; s < nst; ++s) {
                const int a = s & 1;
                mbar_wait(afull0 + 8 * a, (s >> 1) & 1);
                __syncwarp();  // tcgen05.ld is .aligned
                tc_fence_after();
                uint32_t va[32], vb[32];
                load64(a, va, vb);
                const float4* ls4 = reinterpret_cast<const float4*>(lse_s + s * RT_YROWS + ch * 64);
#pragma unroll
                for (int i4 = 0; i4 < 8; ++i4) {  // 3 of 4 exponentials on the SFU, 1 on the FP32 pipe
                    const float4 la = ls4[i4], lb = ls4[8 + i4];
                    const float* lav = reinterpret_cast<const float*>(&la);
                    const float* lbv = reinterpret_cast<const float*>(&lb);
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int i = 4 * i4 + e;
                        const float ya = fmaf(__uint_as_float(va[i]), p.scale2, -lav[e]);
                        const float yb = fmaf(__uint_as_float(vb[i]), p.scale2, -lbv[e]);
                        acc0 += fast_exp2(ya);
                        acc1 += (e != 3) ? fast_exp2(yb) : ((yb < -126.f) ? 0.f : poly_exp2(yb));  // padded: 0
                    }
                }
            }
            reinterpret_cast<float*>(smem + SM::RED_OFF)[ch * RT_XROWS + 32 * q4 + lane] = acc0 + acc1;
        }
    }
    tc_fence_before();
    cta_sync();
    if (MODE == 1 && tid < RT_XROWS) {
        const float* red = reinterpret_cast<const float*>(smem + SM::RED_OFF);
        const int j = blockIdx.x * RT_XROWS + tid;
        const float sc = (red[tid] + red[RT_XROWS + tid]) + (red[2 * RT_XROWS + tid] + red[3 * RT_XROWS + tid]);
        if (j < p.nv) {
            if (!(sc == sc) || sc == INFINITY) raise_flag(p.flags, 2u /*NONFINITE*/);
            p.scores[(int64_t)u * p.nv + j] = sc;
        }
    }
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tbase, 512);
    }
}


// Column mass with the query tile RESIDENT (NQP == 256: n_q * g <= 256, e.g. a
// 32-row question at g = 7): one 256-row Q tile per unit stays in shared memory
// and the CTA walks key blocks kb = blockIdx.x, += gridDim.x through a 2-slot
// X ring, so the per-CTA setup (TMEM, barriers, Q and LSE loads) is paid once
// instead of once per 128 keys.  Same math and summation order as mode 1.
template <int D>
struct RqSmem {
    static constexpr int NB = D / 64;
    static constexpr int X_BYTES = NB * RT_XROWS * 128;
    static constexpr int Y_BYTES = NB * RT_YROWS * 128;
    static constexpr int X_OFF = 0;                               // [2 slots] K blocks
    static constexpr int Y_OFF = X_OFF + 2 * X_BYTES;             // the unit's Q tile
    static constexpr int LSE_OFF = Y_OFF + Y_BYTES;               // LSE2 [256]
    static constexpr int RED_OFF = LSE_OFF + RT_YROWS * 4;        // [2 items][4 quarters][128 rows]
    static constexpr int BAR_OFF = RED_OFF + 2 * 4 * RT_XROWS * 4;
    static constexpr int BYTES = BAR_OFF + 128;
    static_assert(Y_OFF % 1024 == 0 && X_BYTES % 1024 == 0, "swizzle atoms");
    static_assert(BYTES <= 227 * 1024, "shared memory");
};

template <int D>
__global__ void __launch_bounds__(RT_THREADS, 1) retr_mass_qres_kernel(const __grid_constant__ RetrTcParams p) {
    using SM = RqSmem<D>;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr uint32_t IDESC = umma_idesc_bf16(RT_XROWS, RT_YROWS);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
    const uint32_t yfull = smem_u32(bars), xfull0 = smem_u32(bars + 1), xempty0 = smem_u32(bars + 3);
    const uint32_t afull0 = smem_u32(bars + 5), aempty0 = smem_u32(bars + 7);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 9);
    const uint32_t sX = smem_u32(smem + SM::X_OFF), sY = smem_u32(smem + SM::Y_OFF);
    float* lse_s = reinterpret_cast<float*>(smem + SM::LSE_OFF);
    float* red = reinterpret_cast<float*>(smem + SM::RED_OFF);
    const int u = blockIdx.y, b = u / p.Hkv, G = u % p.Hkv;
    const int nkb = (p.nv + RT_XROWS - 1) / RT_XROWS;
    const int nit = blockIdx.x < nkb ? (nkb - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (nit == 0) return;
    const int q4 = warp & 3, ch = (warp - 4) >> 2;

    if (tid == 0) {
        mbar_init(yfull, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(xfull0 + 8 * i, 1);
            mbar_init(xempty0 + 8 * i, 1);
            mbar_init(afull0 + 8 * i, 1);
            mbar_init(aempty0 + 8 * i, RT_EPI_WARPS);
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(smem_u32(tslot), 512);
    for (int i = tid; i < RT_YROWS; i += RT_THREADS) lse_s[i] = p.lse2[(int64_t)u * p.NQP + i];
    tc_fence_before();
    cta_sync();
    tc_fence_after();
    const uint32_t tbase = *tslot;

    if (warp == 0) {
        if (lane == 0) {
            mbar_arrive_expect_tx(yfull, (uint32_t)SM::Y_BYTES);
#pragma unroll
            for (int hf = 0; hf < SM::NB; ++hf)
                tma_load_4d(sY + hf * (RT_YROWS * 128), &p.ymap, hf * 64, 0, 0, u, yfull);
            for (int j = 0; j < nit; ++j) {
                const int slot = j & 1, kb = blockIdx.x + j * gridDim.x;
                if (j >= 2) mbar_wait(xempty0 + 8 * slot, ((j >> 1) - 1) & 1);
                mbar_arrive_expect_tx(xfull0 + 8 * slot, (uint32_t)SM::X_BYTES);
#pragma unroll
                for (int hf = 0; hf < SM::NB; ++hf)
                    tma_load_4d(sX + slot * SM::X_BYTES + hf * (RT_XROWS * 128), &p.xmap, hf * 64,
                                p.vb + kb * RT_XROWS, G, b, xfull0 + 8 * slot);
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            mbar_wait(yfull, 0);
            for (int j = 0; j < nit; ++j) {
                const int slot = j & 1, a = j & 1;
                mbar_wait(xfull0 + 8 * slot, (j >> 1) & 1);
                if (j >= 2) mbar_wait(aempty0 + 8 * a, ((j >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t xb = sX + slot * SM::X_BYTES;
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                    const int hf = k >> 2, kk = k & 3;
                    umma_bf16(tbase + a * RT_YROWS, sw128_desc(xb + hf * (RT_XROWS * 128) + kk * 32),
                              sw128_desc(sY + hf * (RT_YROWS * 128) + kk * 32), IDESC, k > 0 ? 1u : 0u);
                }
                umma_commit(xempty0 + 8 * slot);
                umma_commit(afull0 + 8 * a);
            }
        }
        __syncwarp();
    } else if (warp >= 4) {
        const uint32_t trow = tbase + ((uint32_t)(32 * q4) << 16);
        const float4* ls4 = reinterpret_cast<const float4*>(lse_s + ch * 64);
        for (int j = 0; j < nit; ++j) {
            const int a = j & 1;
            mbar_wait(afull0 + 8 * a, (j >> 1) & 1);
            __syncwarp();  // tcgen05.ld is .aligned
            tc_fence_after();
            uint32_t va[32], vb[32];
            const uint32_t t0 = trow + a * RT_YROWS + ch * 64;
            tmem_ld32_nowait(t0, va);
            tmem_ld32_nowait(t0 + 32, vb);
            tmem_wait_ld_tie(va);
            tmem_wait_ld_tie(vb);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(aempty0 + 8 * a);
            float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
            for (int i4 = 0; i4 < 8; ++i4) {  // 3 of 4 exponentials on the SFU, 1 on the FP32 pipe
                const float4 la = ls4[i4], lb = ls4[8 + i4];
                const float* lav = reinterpret_cast<const float*>(&la);
                const float* lbv = reinterpret_cast<const float*>(&lb);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int i = 4 * i4 + e;
                    const float ya = fmaf(__uint_as_float(va[i]), p.scale2, -lav[e]);
                    const float yb = fmaf(__uint_as_float(vb[i]), p.scale2, -lbv[e]);
                    acc0 += fast_exp2(ya);
                    acc1 += (e != 3) ? fast_exp2(yb) : ((yb < -126.f) ? 0.f : poly_exp2(yb));
                }
            }
            float* rj = red + (j & 1) * (4 * RT_XROWS);
            rj[ch * RT_XROWS + 32 * q4 + lane] = acc0 + acc1;
            asm volatile("bar.sync 1, %0;" ::"n"(RT_EPI_WARPS * 32) : "memory");  // the 16 epilogue warps
            if (ch == 0) {
                const int row = 32 * q4 + lane;
                const int jj = (blockIdx.x + j * gridDim.x) * RT_XROWS + row;
                const float sc = (rj[row] + rj[RT_XROWS + row]) + (rj[2 * RT_XROWS + row] + rj[3 * RT_XROWS + row]);
                if (jj < p.nv) {
                    if (!(sc == sc) || sc == INFINITY) raise_flag(p.flags, 2u /*NONFINITE*/);
                    p.scores[(int64_t)u * p.nv + jj] = sc;
                }
            }
        }
    }
    tc_fence_before();
    cta_sync();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tbase, 512);
    }
}

// ---------------------------------------------------------------------------
// Question-chunk attention output (svl_question_attention):
// the attention output the prefill pass produces beside the row LSE
// (PAPER.md:124 runs the retrieval "concurrently with the FlashAttention2
// path"; this is that path on the same tensor-core machinery):
//   O[n] = sum_j 2^(s[n,j] * scale2 - LSE2[n]) V[j]
// over exactly the key range and causal limit pass 0 folds, with the FINAL
// LSE2 (pass 0 + combine, or lse_in), so a key chunk's partial output is
// already normalised and the chunks add without rescaling (no online-softmax
// correction in TMEM).  Per stage of 128 keys:
//   S_a = Q_blk K_s^T        tcgen05 M128 N128 K16 x D/16, TMEM columns a*128
//   P   = 2^(S*scale2 - LSE2) masked, rounded to bf16 (as FlashAttention-2 does
//         on bf16 inputs, reading A24), written by the epilogue warps into a
//         K-major 128-B-swizzled shared tile
//   O  += P V_s              tcgen05 M128 N=D K16 x 8, B = V stage MN-major
//                            (the TMA tile of V is [keys][d]: d contiguous),
//                            TMEM columns 256..256+D
// The MMA issuer runs one stage ahead (S of stage s before P.V of stage s-1),
// so the exponentials of one stage overlap the products of the next.
// PT (default): P goes to tensor memory and the P.V product takes its A operand
// from TMEM (tcgen05.mma [d], [a_tmem], b_desc) -- no shared-memory P tile, so
// the K/V ring gets three stages; !PT (A/B builds, SVL_QA_P_SMEM): P in a
// 128-B-swizzled shared tile, two K/V stages.
#ifdef SVL_QA_P_SMEM
constexpr bool kQaPTmem = false;
#else
constexpr bool kQaPTmem = true;
#endif

template <int D, bool PT>
struct RoSmem {
    static constexpr int NB = D / 64;
    static constexpr int KROWS = 128;                    // keys per stage
    static constexpr int NKV = PT ? 3 : 2;               // K/V ring stages
    static constexpr int Q_BYTES = NB * RT_XROWS * 128;  // resident Q block
    static constexpr int KV_BYTES = NB * KROWS * 128;    // one K (or V) stage
    static constexpr int P_BYTES = PT ? 0 : 2 * RT_XROWS * 128;  // 128 rows x 128 keys bf16, two 64-key blocks
    static constexpr int Q_OFF = 0;
    static constexpr int K_OFF = Q_OFF + Q_BYTES;         // [NKV] K stages
    static constexpr int V_OFF = K_OFF + NKV * KV_BYTES;  // [NKV] V stages
    static constexpr int P_OFF = V_OFF + NKV * KV_BYTES;  // [2] P tiles (!PT)
    static constexpr int LSE_OFF = P_OFF + 2 * P_BYTES;
    static constexpr int BAR_OFF = LSE_OFF + RT_XROWS * 4;
    static constexpr int BYTES = BAR_OFF + 256;
    static_assert(K_OFF % 1024 == 0 && V_OFF % 1024 == 0 && P_OFF % 1024 == 0, "swizzle atoms");
    static_assert(BYTES <= 227 * 1024, "shared memory");
};

// MN-major operand, 128-B swizzle: 8 K-rows of 128 B (64 MN elements) per
// 1024-B atom; SBO = 1024 (next 8 K rows), LBO = `lbo` bytes (next 64 MN
// elements).  Advancing K by 16 = +2048 B on the start address.
SVL_DEV uint64_t sw128_mn_desc(uint32_t saddr, uint32_t lbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)(1024u >> 4) << 32) | ((uint64_t)1u << 46) | ((uint64_t)2u << 61);
}
// D[tmem] (+)= A[tmem] . B[smem]^T: A (M x 16, bf16 pairs per 32-bit column, lane = row)
// read from tensor memory.
SVL_DEV void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// TMEM columns: S_0 [0,128), S_1 [128,256), O [256,256+D), P_0 [384,448), P_1 [448,512)
template <int D, bool PT>
__global__ void __launch_bounds__(RT_THREADS, 1) retr_out_kernel(const __grid_constant__ RetrTcParams p) {
    using SM = RoSmem<D, PT>;
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int KR = SM::KROWS, NKV = SM::NKV;
    constexpr int OCOL = 2 * KR, PCOL = 384;
    constexpr uint32_t IDESC_S = umma_idesc_bf16(RT_XROWS, KR);
    constexpr uint32_t IDESC_O = umma_idesc_bf16(RT_XROWS, D) | (1u << 16);  // B (= V) MN-major
    constexpr int OCOLS = D / 4;                                             // O columns per epilogue warp
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::BAR_OFF);
    const uint32_t qfull = smem_u32(bars), kvfull0 = smem_u32(bars + 1), kvempty0 = smem_u32(bars + 4);
    const uint32_t sfull0 = smem_u32(bars + 7), sempty0 = smem_u32(bars + 9);
    const uint32_t pfull0 = smem_u32(bars + 11), pempty0 = smem_u32(bars + 13), ofull = smem_u32(bars + 15);
    const uint32_t vfix = smem_u32(bars + 16);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 17);
    const uint32_t sQ = smem_u32(smem + SM::Q_OFF), sK = smem_u32(smem + SM::K_OFF);
    const uint32_t sV = smem_u32(smem + SM::V_OFF), sP = smem_u32(smem + SM::P_OFF);
    float* lse_s = reinterpret_cast<float*>(smem + SM::LSE_OFF);

    const int u = blockIdx.z, b = u / p.Hkv, G = u % p.Hkv;
    int L = p.seq_len[b];
    if (L < p.vb + p.nv + p.n_q || L > p.capacity) {
        if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0) raise_flag(p.flags, 4u /*SPAN*/);
        L = min(max(L, p.vb + p.nv + p.n_q), p.capacity);
    }
    const int lo = p.visual_only ? p.vb : 0;
    const int hi = p.visual_only ? p.vb + p.nv : L;
    const int y0 = lo + blockIdx.x * p.chunk;
    const int y1 = min(hi, y0 + p.chunk);
    const int xrow0 = blockIdx.y * RT_XROWS;
    const int nst = y1 > y0 ? (y1 - y0 + KR - 1) / KR : 0;
    const int q4 = warp & 3, cg = (warp - 4) >> 2;  // epilogue: TMEM lane quarter, 32-key column group
    const int row = 32 * q4 + lane;
    // valid rows of the last stage: V rows past the key range (past seq_len: possibly never
    // written) are zeroed in shared memory before the last P.V, since 0 * NaN = NaN
    const int tail = y1 - (y0 + (nst - 1) * KR);
    float* po = p.part_o + (((int64_t)u * p.NQP + xrow0 + row) * p.nkc + blockIdx.x) * D + cg * OCOLS;
    if (nst == 0) {  // empty key chunk: a zero partial
        if (warp >= 4)
            for (int c = 0; c < OCOLS; c += 4) *reinterpret_cast<float4*>(po + c) = make_float4(0.f, 0.f, 0.f, 0.f);
        return;
    }

    if (tid == 0) {
        mbar_init(qfull, 1);
        mbar_init(ofull, 1);
        mbar_init(vfix, 1);
        for (int i = 0; i < NKV; ++i) {
            mbar_init(kvfull0 + 8 * i, 1);
            mbar_init(kvempty0 + 8 * i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(sfull0 + 8 * i, 1);
            mbar_init(sempty0 + 8 * i, RT_EPI_WARPS);
            mbar_init(pfull0 + 8 * i, RT_EPI_WARPS);
            mbar_init(pempty0 + 8 * i, 1);
        }
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(smem_u32(tslot), 512);
    for (int i = tid; i < RT_XROWS; i += RT_THREADS) lse_s[i] = p.lse2[(int64_t)u * p.NQP + xrow0 + i];
    tc_fence_before();
    cta_sync();
    tc_fence_after();
    const uint32_t tbase = *tslot;

    if (warp == 0) {
        if (lane == 0) {
            mbar_arrive_expect_tx(qfull, (uint32_t)SM::Q_BYTES);
#pragma unroll
            for (int hf = 0; hf < SM::NB; ++hf)
                tma_load_4d(sQ + hf * (RT_XROWS * 128), &p.xmap, hf * 64, xrow0, 0, u, qfull);
            for (int s = 0; s < nst; ++s) {
                const int slot = s % NKV;
                if (s >= NKV) mbar_wait(kvempty0 + 8 * slot, ((s / NKV) - 1) & 1);
                const uint32_t bar = kvfull0 + 8 * slot;
                mbar_arrive_expect_tx(bar, (uint32_t)(2 * SM::KV_BYTES));
#pragma unroll
                for (int hf = 0; hf < SM::NB; ++hf) {
                    const int off = slot * SM::KV_BYTES + hf * (KR * 128);
                    tma_load_4d(sK + off, &p.ymap, hf * 64, y0 + s * KR, G, b, bar);
                    tma_load_4d(sV + off, &p.vmap, hf * 64, y0 + s * KR, G, b, bar);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            mbar_wait(qfull, 0);
            for (int s = 0; s <= nst; ++s) {
                if (s < nst) {  // S of stage s
                    const int a = s & 1, slot = s % NKV;
                    mbar_wait(kvfull0 + 8 * slot, (s / NKV) & 1);
                    if (s >= 2) mbar_wait(sempty0 + 8 * a, ((s >> 1) - 1) & 1);
                    tc_fence_after();
                    const uint32_t kb = sK + slot * SM::KV_BYTES;
#pragma unroll
                    for (int j = 0; j < D / 16; ++j) {
                        const int hf = j >> 2, kk = j & 3;
                        umma_bf16(tbase + a * KR, sw128_desc(sQ + hf * (RT_XROWS * 128) + kk * 32),
                                  sw128_desc(kb + hf * (KR * 128) + kk * 32), IDESC_S, j > 0 ? 1u : 0u);
                    }
                    umma_commit(sfull0 + 8 * a);
                }
                if (s >= 1) {  // P.V of stage s - 1
                    const int t = s - 1, a = t & 1, slot = t % NKV;
                    mbar_wait(pfull0 + 8 * a, (t >> 1) & 1);
                    if (t == nst - 1 && tail < KR) mbar_wait(vfix, 0);
                    tc_fence_after();
                    const uint32_t vb = sV + slot * SM::KV_BYTES;
#pragma unroll
                    for (int j = 0; j < KR / 16; ++j) {
                        const uint64_t bd = sw128_mn_desc(vb + j * 16 * 128, KR * 128);
                        const uint32_t acc = (t > 0 || j > 0) ? 1u : 0u;
                        if constexpr (PT) {
                            umma_bf16_ts(tbase + OCOL, tbase + PCOL + a * 64 + j * 8, bd, IDESC_O, acc);
                        } else {
                            const int hf = j >> 2, kk = j & 3;
                            umma_bf16(tbase + OCOL,
                                      sw128_desc(sP + a * SM::P_BYTES + hf * (RT_XROWS * 128) + kk * 32), bd,
                                      IDESC_O, acc);
                        }
                    }
                    umma_commit(kvempty0 + 8 * slot);  // K and V of stage t consumed
                    umma_commit(pempty0 + 8 * a);
                }
            }
            umma_commit(ofull);
        }
        __syncwarp();
    } else if (warp == 3) {
        if (tail < KR) {
            const int slot = (nst - 1) % NKV;
            mbar_wait(kvfull0 + 8 * slot, ((nst - 1) / NKV) & 1);
#pragma unroll
            for (int hf = 0; hf < SM::NB; ++hf)
                for (int i = tail * 8 + lane; i < KR * 8; i += 32)  // 16-B chunks, 8 per 128-B row
                    asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(sV + slot * SM::KV_BYTES +
                                                                                hf * (KR * 128) + i * 16),
                                 "r"(0u)
                                 : "memory");
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(vfix);
        }
    } else if (warp >= 4) {
        const uint32_t trow = tbase + ((uint32_t)(32 * q4) << 16);
        const int n = xrow0 + row;
        const int r = n / p.g;
        const int jend = p.visual_only ? y1 : min(y1, L - p.n_q + r + 1);
        const float lse = lse_s[row];  // +inf on padding rows: P = 0
        const uint32_t prow = (uint32_t)((cg >> 1) * (RT_XROWS * 128) + row * 128);
        for (int s = 0; s < nst; ++s) {
            const int a = s & 1;
            mbar_wait(sfull0 + 8 * a, (s >> 1) & 1);
            __syncwarp();  // tcgen05.ld is .aligned
            tc_fence_after();
            uint32_t v[32];
            tmem_ld32_nowait(trow + a * KR + cg * 32, v);
            tmem_wait_ld_tie(v);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(sempty0 + 8 * a);
            const int j0 = y0 + s * KR + cg * 32;
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                const float x0 = fmaf(__uint_as_float(v[i]), p.scale2, -lse);
                const float x1 = fmaf(__uint_as_float(v[i + 1]), p.scale2, -lse);
                float e0 = fast_exp2(x0);
                float e1 = ((i & 2) == 0) ? fast_exp2(x1) : ((x1 < -126.f) ? 0.f : poly_exp2(x1));
                if (j0 + i >= jend) e0 = 0.f;
                if (j0 + i + 1 >= jend) e1 = 0.f;
                pk[i >> 1] = pack_bf16(e0, e1);
            }
            if (s >= 2) mbar_wait(pempty0 + 8 * a, ((s >> 1) - 1) & 1);
            if constexpr (PT) {
                float pf[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) pf[i] = __uint_as_float(pk[i]);
                tmem_st16(trow + PCOL + a * 64 + cg * 16, pf);  // includes tcgen05.wait::st
                tc_fence_before();
            } else {
                const uint32_t pbase = sP + a * SM::P_BYTES + prow;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const uint32_t chunk = (uint32_t)((cg & 1) * 4 + c) ^ (uint32_t)(row & 7);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(pbase + chunk * 16), "r"(pk[4 * c]),
                                 "r"(pk[4 * c + 1]), "r"(pk[4 * c + 2]), "r"(pk[4 * c + 3])
                                 : "memory");
                }
                fence_proxy_async_smem();
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(pfull0 + 8 * a);
        }
        mbar_wait(ofull, 0);
        __syncwarp();
        tc_fence_after();
        const uint32_t to = trow + OCOL + cg * OCOLS;
        if constexpr (OCOLS == 32) {
            uint32_t o[32];
            tmem_ld32(to, o);
#pragma unroll
            for (int c = 0; c < 32; c += 4)
                *reinterpret_cast<float4*>(po + c) = make_float4(__uint_as_float(o[c]), __uint_as_float(o[c + 1]),
                                                                 __uint_as_float(o[c + 2]), __uint_as_float(o[c + 3]));
        } else {
            uint32_t o[16];
            tmem_ld16(to, o);
#pragma unroll
            for (int c = 0; c < 16; c += 4)
                *reinterpret_cast<float4*>(po + c) = make_float4(__uint_as_float(o[c]), __uint_as_float(o[c + 1]),
                                                                 __uint_as_float(o[c + 2]), __uint_as_float(o[c + 3]));
        }
    }
    tc_fence_before();
    cta_sync();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tbase, 512);
    }
}

// out[b][r][h][:] = sum over key chunks (chunk order) of the partial outputs;
// lse_out = LSE2 * ln 2.  One thread per (row, 4 columns).
__global__ void out_combine_kernel(const RetrTcParams p, int D) {
    const int C4 = D / 4;
    const int64_t total = (int64_t)p.B * p.Hkv * p.NQ * C4;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int c4 = (int)(e % C4);
        const int n = (int)((e / C4) % p.NQ);
        const int u = (int)(e / C4 / p.NQ);
        const float4* src = reinterpret_cast<const float4*>(p.part_o + ((int64_t)u * p.NQP + n) * p.nkc * D) + c4;
        float4 acc = src[0];
        for (int k = 1; k < p.nkc; ++k) {
            const float4 x = src[(int64_t)k * C4];
            acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
        }
        const int b = u / p.Hkv, G = u % p.Hkv, r = n / p.g, h = G * p.g + n % p.g;
        const int64_t orow = ((int64_t)b * p.n_q + r) * p.H + h;
        reinterpret_cast<float4*>(p.out + orow * D)[c4] = acc;
        if (c4 == 0 && p.lse_out) p.lse_out[orow] = p.lse2[(int64_t)u * p.NQP + n] * kLn2;
    }
}

template <int MODE, int D>
cudaError_t launch_tc(const RetrTcParams& p, dim3 grid, cudaStream_t s) {
    static bool attr_done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_done[dev]) {
        cudaError_t e = cudaFuncSetAttribute(retr_tc_kernel<MODE, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             RtSmem<D>::BYTES);
        if (e == cudaSuccess) e = set_max_carveout(retr_tc_kernel<MODE, D>);
        if (e != cudaSuccess) return e;
        attr_done[dev] = true;
    }
    retr_tc_kernel<MODE, D><<<grid, RT_THREADS, RtSmem<D>::BYTES, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_question_attn_tc(const RetrTcParams& p, int d, cudaStream_t s) {
    const int units = p.B * p.Hkv;
    const int sms = device_sm_count();
    const int64_t qchunks = (int64_t)units * p.NQP * (d / 8);
    qpack_kernel<<<(int)std::min<int64_t>((qchunks + 255) / 256, 8L * sms), 256, 0, s>>>(p, d);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    RetrTcParams p0 = p;
    p0.xmap = p.qmap_x;  // X = Q blocks
    p0.ymap = p.kmap_y;  // Y = K stages (256 rows)
    const int nqb = (p.NQ + RT_XROWS - 1) / RT_XROWS;
    if (!p.lse_in) {
        const dim3 g0(p.nkc, nqb, units);
        e = d == 128 ? launch_tc<0, 128>(p0, g0, s) : launch_tc<0, 64>(p0, g0, s);
        if (e != cudaSuccess) return e;
    }
    const int64_t rows = (int64_t)units * p.NQP;
    lse_combine_kernel<<<(int)std::min<int64_t>((rows + 7) / 8, 8L * sms), 256, 0, s>>>(p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    RetrTcParams p2 = p;
    p2.xmap = p.qmap_x;  // X = Q blocks
    p2.ymap = p.kmap_x;  // K stages of 128 rows (p.vmap: V stages of 128 rows)
    static bool attr_done[64][2] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_done[dev][d == 128]) {
        e = d == 128 ? cudaFuncSetAttribute(retr_out_kernel<128, kQaPTmem>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, RoSmem<128, kQaPTmem>::BYTES)
                     : cudaFuncSetAttribute(retr_out_kernel<64, kQaPTmem>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, RoSmem<64, kQaPTmem>::BYTES);
        if (e != cudaSuccess) return e;
        attr_done[dev][d == 128] = true;
    }
    const dim3 g2(p.nkc, nqb, units);
    if (d == 128) retr_out_kernel<128, kQaPTmem><<<g2, RT_THREADS, RoSmem<128, kQaPTmem>::BYTES, s>>>(p2);
    else retr_out_kernel<64, kQaPTmem><<<g2, RT_THREADS, RoSmem<64, kQaPTmem>::BYTES, s>>>(p2);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int64_t n4 = (int64_t)units * p.NQ * (d / 4);
    out_combine_kernel<<<(int)std::min<int64_t>((n4 + 255) / 256, 8L * sms), 256, 0, s>>>(p, d);
    return cudaGetLastError();
}

// host plan of pass 0: a fixed number of key chunks per (unit, query block) --
// about two waves of CTAs, independent of the key range (so the workspace size
// does not depend on the capacity) -- each chunk a multiple of 256 keys
void plan_retrieve_tc(int units, int n_q, int g, int nv, int capacity, bool visual_only, int sms, int* chunk,
                      int* nkc) {
    const int NQ = n_q * g;
    const int nqb = (NQ + RT_XROWS - 1) / RT_XROWS;
    const int range = visual_only ? nv : capacity;
    // CTA budget in waves (measured on the long-video cache, FULL_PREFIX, us: n_q = 32: 1 wave
    // 61.8 vs 2 waves 65.8; n_q = 128: 148.8 vs 154.3; n_q = 512 (112 query blocks): 4 waves
    // 414 vs 2 waves 450): few query blocks -> one wave of long key chunks, many -> 4 waves
    int waves = (units * nqb * 2 >= sms) ? 4 : 1;
#ifdef SVL_RT_WAVES
    waves = SVL_RT_WAVES;  // A/B builds only
#endif
    const int n = std::max(1, std::min(64, waves * sms / std::max(1, units * nqb)));
    *nkc = n;
    *chunk = ((range + n - 1) / n + RT_YROWS - 1) / RT_YROWS * RT_YROWS;
}

cudaError_t launch_retrieve_tc(const RetrTcParams& p, int d, cudaStream_t s) {
    const int units = p.B * p.Hkv;
    const int sms = device_sm_count();
    const int64_t qchunks = (int64_t)units * p.NQP * (d / 8);
    qpack_kernel<<<(int)std::min<int64_t>((qchunks + 255) / 256, 8L * sms), 256, 0, s>>>(p, d);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    RetrTcParams p0 = p;
    p0.xmap = p.qmap_x;  // X = Q blocks
    p0.ymap = p.kmap_y;  // Y = K stages
    if (!p.lse_in) {
        const dim3 g0(p.nkc, (p.NQ + RT_XROWS - 1) / RT_XROWS, units);
        e = d == 128 ? launch_tc<0, 128>(p0, g0, s) : launch_tc<0, 64>(p0, g0, s);
        if (e != cudaSuccess) return e;
    }
    const int64_t rows = (int64_t)units * p.NQP;
    lse_combine_kernel<<<(int)std::min<int64_t>((rows + 7) / 8, 8L * sms), 256, 0, s>>>(p);  // 8 rows / block
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    RetrTcParams p1 = p;
    p1.xmap = p.kmap_x;  // X = K blocks
    p1.ymap = p.qmap_y;  // Y = Q chunks
    const int nkb = (p.nv + RT_XROWS - 1) / RT_XROWS;
#ifndef SVL_RT_NO_QRES
    constexpr bool qres = true;
#else
    constexpr bool qres = false;  // A/B builds only
#endif
    if (p.NQP == RT_YROWS && qres) {  // Q tile resident, CTAs walk key blocks
        const int per_unit = std::max(1, std::min(nkb, (2 * sms + units - 1) / units));
        const dim3 g2(per_unit, units, 1);
        static bool attr_done[64][2] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 64 && !attr_done[dev][d == 128]) {
            e = d == 128 ? cudaFuncSetAttribute(retr_mass_qres_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                RqSmem<128>::BYTES)
                         : cudaFuncSetAttribute(retr_mass_qres_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                RqSmem<64>::BYTES);
            if (e != cudaSuccess) return e;
            attr_done[dev][d == 128] = true;
        }
        if (d == 128) retr_mass_qres_kernel<128><<<g2, RT_THREADS, RqSmem<128>::BYTES, s>>>(p1);
        else retr_mass_qres_kernel<64><<<g2, RT_THREADS, RqSmem<64>::BYTES, s>>>(p1);
        return cudaGetLastError();
    }
    const dim3 g1(nkb, units, 1);
    return d == 128 ? launch_tc<1, 128>(p1, g1, s) : launch_tc<1, 64>(p1, g1, s);
}

}  // namespace svl
