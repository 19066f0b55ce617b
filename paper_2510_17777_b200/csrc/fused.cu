// fused.cu -- the fresh-retrieval decode step in ONE kernel per layer
// (SURVEY.md 8(a) a1-a5 fused): svl_fresh_decode_step.
//
// at a decode step with a new query, score every cached
// visual token by its attention mass (query-aware relevance), keep the top-k
// per KV group, and run decode attention over [text rows] U [kept visual
// rows].  When the retrieval query IS the decode query (n_q = 1, the
// per-step fresh retrieval this library benchmarks), both need the same
// logits s = scale * q.K_j, so K is streamed from HBM exactly once.
//
// One thread-block cluster (CS <= 16 CTAs, distributed shared memory) per
// unit (b, KV group G); CTA r owns visual rows [r*slice, (r+1)*slice) and a
// 1/CS share of the text rows.  Per CTA (8 consumer warps + 1 TMA warp):
//   1. the TMA warp streams the CTA's K rows (visual slice, then text share)
//      with cp.async.bulk into a 4-stage x 32 KB mbarrier ring; consumer warps
//      compute the base-2 logits of all g heads per 16-row tile with
//      mma.sync (swap-AB, permuted contraction, as in score.cu) and keep them
//      in shared memory (never written to HBM), plus a running (max, sum);
//   2. cluster reduction of the (max, sum) partials over DSMEM -> the
//      full-prefix LSE of every head (same value in every CTA);
//   3. score_j = sum_h exp2(s2[j,h] - LSE2[h]) -> order-preserving keys;
//   4. cluster_topk_push (select_push.cuh) -> threshold; kept indices written to
//      idx_out (ascending, ties to the lower index);
//   5. decode attention over this CTA's kept rows + text share, reusing the
//      logits: fixed max M_h, l_h = sum exp2(s2 - M_h), O_h = sum p V with V
//      rows gathered by cp.async (swizzled) and P split bf16 hi+lo for
//      mma.sync (ldmatrix.trans V fragments);
//   6. cluster merge of (M, l, O) over DSMEM -> out fp32 [B][H][d], lse.
// HBM traffic per unit: visual K + text K once + kept V + text V.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"
#include "select_push.cuh"

namespace svl {

namespace {

constexpr int FT = kFusedThreads;  // 8 consumer warps + 1 producer warp
constexpr int FCW = 8;
constexpr int STAGE_ROWS = 128;
constexpr int RING = 128 * 1024;
constexpr int TMAX = kFusedTextMax;
constexpr int VB_ROWS = 256;  // V rows per staging batch (two batches in the ring)

template <int D, int NT>
struct FGeom {
    static constexpr int NCP = 8 * NT;
    static constexpr int SMAX = kFusedSliceMax / NT;
    static constexpr int NST = 512 / D;  // ring stages
    static constexpr int ROWB = 2 * D;
    static constexpr int STAGE_BYTES = STAGE_ROWS * ROWB;
    static constexpr int LOG_OFF = RING;
    static constexpr int LOG_BYTES = (SMAX + TMAX) * NCP * 4;
    static constexpr int ATT_OFF = LOG_OFF + LOG_BYTES;
    static constexpr int ATT_BYTES = (SMAX + TMAX) * 4;
    static constexpr int MISC_OFF = ATT_OFF + ATT_BYTES;
    static constexpr int MISC_BYTES = 2 * NST * 8 + FCW * NCP * 8 + 16 * NCP * 8 + NCP * 4 + 64 * 4;
    static constexpr int BYTES = MISC_OFF + MISC_BYTES;
    static constexpr int KEYS_OFF = 96 * 1024;  // inside the ring once streaming is over
    static constexpr int STATE_OFF = KEYS_OFF + SMAX * 4;
    static constexpr int VBUF_BYTES = VB_ROWS * ROWB;
    static constexpr int OCTA_OFF = 64 * 1024;  // CTA O [16][D] fp32 inside the ring at the end
};

SVL_DEV int swz_v(int row, int c) { return c ^ (row & 7); }

template <int D, int NT>
__global__ void __launch_bounds__(FT, 1) fresh_kernel(const FreshParams p) {
    using GM = FGeom<D, NT>;
    constexpr int NCP = GM::NCP, NST = GM::NST, ROWB = GM::ROWB;
    constexpr int NCH = D / 32;  // 16-byte chunks per thread per row (permuted contraction)
    constexpr int CH = D / 8;    // 16-byte chunks per row
    constexpr int NVT = D / 8;   // output n-tiles
    static_assert(GM::STATE_OFF + GM::SMAX <= RING, "keys + state must fit in the ring");
    static_assert(sizeof(PushTopkSmem) <= GM::KEYS_OFF, "top-k scratch must fit in the ring");
    static_assert(GM::BYTES <= 227 * 1024, "shared memory budget");

    extern __shared__ __align__(1024) uint8_t smem[];
    cg::cluster_group cl = cg::this_cluster();
    const int CS = (int)cl.num_blocks();
    const int rank = (int)cl.block_rank();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gid = lane >> 2, t = lane & 3;
    const int u = blockIdx.y;
    const int b = u / p.Hkv, G = u % p.Hkv;
    const int g = p.g;

    float* logits = reinterpret_cast<float*>(smem + GM::LOG_OFF);
    int* att = reinterpret_cast<int*>(smem + GM::ATT_OFF);
    uint8_t* misc = smem + GM::MISC_OFF;
    uint64_t* full = reinterpret_cast<uint64_t*>(misc);
    uint64_t* empty = full + NST;
    float2* wpart = reinterpret_cast<float2*>(empty + NST);  // [FCW][NCP]
    float2* allpart = wpart + FCW * NCP;                       // [16][NCP] pushed by the peers
    float* lse2 = reinterpret_cast<float*>(allpart + 16 * NCP);  // [NCP]
    float* Mh = lse2 + NCP;                                  // [16]
    float* lh = Mh + 16;                                     // [16]
    int* cnt = reinterpret_cast<int*>(lh + 16);              // [4]
    const uint32_t ring = smem_u32(smem);
#define SVL_TRACE(ph)                                                                     \
    if (p.trace && tid == 0) {                                                            \
        uint64_t tnow;                                                                    \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));                          \
        p.trace[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 32 + (ph)] = tnow;        \
    }
    SVL_TRACE(0);

    // ------------------------------------------------------------ geometry
    int L = p.seq_len[b];
    if (L < p.vb + p.nv + 1 || L > p.capacity) {
        if (tid == 0 && rank == 0) raise_flag(p.flags, 4u /*SPAN*/);
        L = min(max(L, p.vb + p.nv + 1), p.capacity);
    }
    const int slice = p.slice;
    const int v0 = min(p.nv, rank * slice);
    const int nvis = min(p.nv, v0 + slice) - v0;
    const int T = p.vb + (L - p.vb - p.nv);
    const int t0 = (int)((int64_t)rank * T / CS);
    int ntext = (int)((int64_t)(rank + 1) * T / CS) - t0;
    if (ntext > TMAX) {
        if (tid == 0) raise_flag(p.flags, 4u /*SPAN*/);
        ntext = TMAX;
    }
    const int nwork = nvis + ntext;
    const int nstages = (nwork + STAGE_ROWS - 1) / STAGE_ROWS;
    const uint16_t* Kb = p.K + (int64_t)b * p.ksb + (int64_t)G * p.ksh;
    const uint16_t* Vb = p.V + (int64_t)b * p.vsb + (int64_t)G * p.vsh;
    auto text_row = [&](int ti) {  // text share index -> cache row
        const int tt = t0 + ti;
        return tt < p.vb ? tt : tt + p.nv;
    };
    auto work_row = [&](int w) { return w < nvis ? p.vb + v0 + w : text_row(w - nvis); };

    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), FCW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    // ------------------------------------------------ 1. stream K, logits
    if (warp == FCW) {
        if (lane == 0) {
            // the work list is <= 3 contiguous row segments: visual slice, system
            // text, after-visual text; each stage is their intersection with it
            const int nsys = max(0, min(ntext, p.vb - t0));
            const int seg_w0[3] = {0, nvis, nvis + nsys};
            const int seg_w1[3] = {nvis, nvis + nsys, nwork};
            const int seg_row0[3] = {p.vb + v0, t0, t0 + nsys + p.nv};  // cache row of the segment start
            const bool dense = (p.kst == D);
            const int64_t kst = p.kst;
            for (int i = 0; i < nstages; ++i) {
                const int slot = i % NST;
                if (i >= NST) mbar_wait(smem_u32(&empty[slot]), ((i / NST) - 1) & 1);
                const int w0 = i * STAGE_ROWS, w1 = min(nwork, w0 + STAGE_ROWS);
                const uint32_t bar = smem_u32(&full[slot]);
                mbar_arrive_expect_tx(bar, (uint32_t)((w1 - w0) * ROWB));
                const uint32_t dst0 = ring + slot * GM::STAGE_BYTES;
#pragma unroll
                for (int sg = 0; sg < 3; ++sg) {
                    const int a = max(w0, seg_w0[sg]), z = min(w1, seg_w1[sg]);
                    if (a >= z) continue;
                    const int row = seg_row0[sg] + (a - seg_w0[sg]);
                    if (dense) {
                        bulk_g2s(dst0 + (a - w0) * ROWB, Kb + (int64_t)row * kst, (uint32_t)((z - a) * ROWB), bar);
                    } else {
                        for (int w = a; w < z; ++w)
                            bulk_g2s(dst0 + (w - w0) * ROWB, Kb + (int64_t)(row + w - a) * kst, ROWB, bar);
                    }
                }
            }
        }
    } else if (warp < FCW) {
        // query B fragments: column c = head G*g + c (c < g), same chunk layout as K
        uint4 bq[NT][NCH];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            const int col = nt * 8 + gid;
#pragma unroll
            for (int i = 0; i < NCH; ++i) bq[nt][i] = make_uint4(0, 0, 0, 0);
            if (col < g) {
                const uint4* qr = reinterpret_cast<const uint4*>(p.q + ((int64_t)b * p.H + G * g + col) * D);
#pragma unroll
                for (int i = 0; i < NCH; ++i) bq[nt][i] = qr[t + 4 * i];
            }
        }
        float rm[NT][2], rl[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) rm[nt][0] = rm[nt][1] = -INFINITY, rl[nt][0] = rl[nt][1] = 0.f;
        const bool text_in_lse = !(p.flags_in & 1u /*VISUAL_ONLY*/);
        for (int i = 0; i < nstages; ++i) {
            const int slot = i % NST;
            mbar_wait(smem_u32(&full[slot]), (i / NST) & 1);
            const int tb = i * STAGE_ROWS + warp * 16;
            if (tb < nwork) {
                const uint32_t base = ring + slot * GM::STAGE_BYTES + (warp * 16 + gid) * ROWB;
                float acc[NT][4];
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
                for (int c4 = 0; c4 < NCH; ++c4) {
                    const uint4 ra = lds128(base + (t + 4 * c4) * 16);
                    const uint4 rb = lds128(base + 8 * ROWB + (t + 4 * c4) * 16);
                    const uint32_t a0[4] = {ra.x, rb.x, ra.y, rb.y};
                    const uint32_t a1[4] = {ra.z, rb.z, ra.w, rb.w};
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) {
                        mma_bf16_16816(acc[nt], a0, bq[nt][c4].x, bq[nt][c4].y);
                        mma_bf16_16816(acc[nt], a1, bq[nt][c4].z, bq[nt][c4].w);
                    }
                }
                const int wa = tb + gid, wb = wa + 8;
                const bool va = wa < nwork, vbv = wb < nwork;
                const bool la = va && (wa < nvis || text_in_lse);
                const bool lb = vbv && (wb < nvis || text_in_lse);
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const float x0 = acc[nt][0] * p.scale2, x1 = acc[nt][1] * p.scale2;
                    const float x2 = acc[nt][2] * p.scale2, x3 = acc[nt][3] * p.scale2;
                    if (va) *reinterpret_cast<float2*>(logits + wa * NCP + nt * 8 + 2 * t) = make_float2(x0, x1);
                    if (vbv) *reinterpret_cast<float2*>(logits + wb * NCP + nt * 8 + 2 * t) = make_float2(x2, x3);
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) {
                        const float ya = la ? (e2 ? x1 : x0) : -INFINITY;
                        const float yb = lb ? (e2 ? x3 : x2) : -INFINITY;
                        const float mx = fmaxf(ya, yb);
                        if (mx != -INFINITY) {
                            const float M = fmaxf(rm[nt][e2], mx);
                            rl[nt][e2] = rl[nt][e2] * fast_exp2(rm[nt][e2] - M) + fast_exp2(ya - M) +
                                         fast_exp2(yb - M);
                            rm[nt][e2] = M;
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&empty[slot]));
        }
        // (max, sum) of each column over this warp
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e2 = 0; e2 < 2; ++e2) {
#pragma unroll
                for (int off = 4; off < 32; off <<= 1) {
                    const float m2 = __shfl_xor_sync(0xffffffffu, rm[nt][e2], off);
                    const float l2 = __shfl_xor_sync(0xffffffffu, rl[nt][e2], off);
                    const float M = fmaxf(rm[nt][e2], m2);
                    if (M != -INFINITY) {
                        rl[nt][e2] = rl[nt][e2] * fast_exp2(rm[nt][e2] - M) + l2 * fast_exp2(m2 - M);
                        rm[nt][e2] = M;
                    }
                }
                if (gid == 0) wpart[warp * NCP + nt * 8 + 2 * t + e2] = make_float2(rm[nt][e2], rl[nt][e2]);
            }
    }
    __syncthreads();

    SVL_TRACE(1);
    // ------------------------------------------------ 2. cluster LSE
    if (tid < NCP) {
        float m = -INFINITY, l = 0.f;
        for (int w = 0; w < FCW; ++w) {
            const float2 x = wpart[w * NCP + tid];
            const float M = fmaxf(m, x.x);
            if (M != -INFINITY) {
                l = l * exp2f(m - M) + x.y * exp2f(x.x - M);
                m = M;
            }
        }
        // push this CTA's partial into every peer's allpart[rank] (no remote reads)
        for (int q = 0; q < CS; ++q) cl.map_shared_rank(allpart, q)[rank * NCP + tid] = make_float2(m, l);
    }
    cl.sync();
    if (tid < NCP) {
        float2 x[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) x[q] = (q < CS) ? allpart[q * NCP + tid] : make_float2(-INFINITY, 0.f);
        float m = -INFINITY, l = 0.f;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const float M = fmaxf(m, x[q].x);
            if (M != -INFINITY) {
                l = l * exp2f(m - M) + x[q].y * exp2f(x[q].x - M);
                m = M;
            }
        }
        lse2[tid] = m + log2f(l);
    }
    __syncthreads();

    SVL_TRACE(2);
    if (p.trace && tid == 0) p.trace[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 32 + 12] = clock64();
    // ------------------------------------------------ 3. keys
    uint32_t* keys_s = reinterpret_cast<uint32_t*>(smem + GM::KEYS_OFF);
    for (int rep = 0; rep < (p.trace ? 2 : 1); ++rep) {  // (trace builds: run twice, i-cache probe)
        if (rep == 1) {
            __syncthreads();
            SVL_TRACE(11);
        }
        bool nan_seen = false;
        // normalisers in registers; padded columns get +inf so they add exp2(-inf) = 0
        // (no per-column branch: all NCP exponentials of a row issue back to back)
        float nl[NCP];
#pragma unroll
        for (int c = 0; c < NCP; ++c) nl[c] = (c < g) ? lse2[c] : INFINITY;
#pragma unroll 2
        for (int i = tid; i < nvis; i += FT) {
            const float4* lr = reinterpret_cast<const float4*>(logits + i * NCP);
            float sc = 0.f;
#pragma unroll
            for (int c4 = 0; c4 < NCP / 4; ++c4) {
                const float4 x = lr[c4];
                sc += fast_exp2(x.x - nl[4 * c4]) + fast_exp2(x.y - nl[4 * c4 + 1]) +
                      fast_exp2(x.z - nl[4 * c4 + 2]) + fast_exp2(x.w - nl[4 * c4 + 3]);
            }
            keys_s[i] = float_key(sc, nan_seen);
        }
        if (nan_seen) raise_flag(p.flags, 2u /*NONFINITE*/);
    }
    __syncthreads();

    // ------------------------------------------------ 4. top-k
    PushTopkSmem& ts = *reinterpret_cast<PushTopkSmem*>(smem);
    uint8_t* state_s = smem + GM::STATE_OFF;
    SVL_TRACE(3);
    if (p.trace && tid == 0) p.trace[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 32 + 13] = clock64();
    uint32_t sel_off;
    const int nsel = (int)cluster_topk_push<FT>(
        cl, ts, keys_s, state_s, nvis, v0, slice, p.nv, p.k, /*relevance=*/true, &sel_off,
        p.trace ? p.trace + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 32 + 16 : nullptr);
    SVL_TRACE(4);
    {
        int32_t* idx_out = p.idx_out + (int64_t)u * p.k;
        push_emit<FT>(ts, state_s, nvis, sel_off, [&](int i, uint32_t slot) {
            idx_out[slot] = v0 + i;
            att[slot - sel_off] = i;
        });
    }
    for (int i = tid; i < ntext; i += FT) att[nsel + i] = nvis + i;
    __syncthreads();
    const int natt = nsel + ntext;

    // ------------------------------------------------ 5. decode over the kept rows
    auto issue_batch = [&](int bi) {
        const int r0 = bi * VB_ROWS, n = min(VB_ROWS, natt - r0);
        const uint32_t vbuf = ring + (bi & 1) * GM::VBUF_BYTES;
        const int nr = (n + 15) & ~15;
        for (int i = tid; i < nr * CH; i += FT) {
            const int rr = i / CH, c = i % CH;
            const bool valid = rr < n;
            const int row = valid ? work_row(att[r0 + rr]) : 0;
            cp_async16(vbuf + rr * ROWB + swz_v(rr, c) * 16, Vb + (int64_t)row * p.vst + c * 8, valid);
        }
        cp_async_commit();
    };
    const int nbatch = (natt + VB_ROWS - 1) / VB_ROWS;
    // the V gather of the first batch overlaps the max / sum pass below (the
    // ring is free: the top-k exchange finished with a cluster barrier)
    if (nbatch > 0) issue_batch(0);
    // fixed per-head max / sum over this CTA's attended rows (logits are all known)
    {
        for (int h = warp; h < 16; h += FT / 32) {
            float m = -INFINITY;
            if (h < g)
                for (int i = lane; i < natt; i += 32) m = fmaxf(m, logits[att[i] * NCP + h]);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
            float l = 0.f;
            if (h < g && m != -INFINITY)
                for (int i = lane; i < natt; i += 32) l += fast_exp2(logits[att[i] * NCP + h] - m);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
            if (lane == 0) {
                Mh[h] = m;
                lh[h] = l;
            }
        }
    }
    __syncthreads();  // Mh/lh visible
    SVL_TRACE(5);
    float o[NVT][4];
#pragma unroll
    for (int n = 0; n < NVT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    for (int bi = 0; bi < nbatch; ++bi) {
        if (bi + 1 < nbatch) {
            issue_batch(bi + 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const int r0 = bi * VB_ROWS, n = min(VB_ROWS, natt - r0);
        const uint32_t vbuf = ring + (bi & 1) * GM::VBUF_BYTES;
        if (warp < FCW) {
            const float Ma = (gid < g) ? Mh[gid] : 0.f, Mb = (gid + 8 < g) ? Mh[gid + 8] : 0.f;
            for (int tile = warp; tile * 16 < n; tile += FCW) {
                const int tb = tile * 16;
                float pv[2][4];  // [k-half][a-rows]: (gid,2t),(gid,2t+1),(gid+8,2t),(gid+8,2t+1)
#pragma unroll
                for (int kh = 0; kh < 2; ++kh)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int rr = tb + kh * 8 + 2 * t + e;
                        const bool ok = rr < n;
                        const float* lr = logits + (ok ? att[r0 + rr] : 0) * NCP;
                        pv[kh][e] = (ok && gid < g && Ma != -INFINITY) ? fast_exp2(lr[gid] - Ma) : 0.f;
                        pv[kh][2 + e] = (ok && gid + 8 < g && Mb != -INFINITY) ? fast_exp2(lr[gid + 8] - Mb) : 0.f;
                    }
                uint32_t ph[4], pl[4];
                {
                    const float v[4][2] = {{pv[0][0], pv[0][1]}, {pv[0][2], pv[0][3]},
                                           {pv[1][0], pv[1][1]}, {pv[1][2], pv[1][3]}};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        ph[i] = pack_bf16(v[i][0], v[i][1]);
                        pl[i] = pack_bf16(v[i][0] - bf16lo(ph[i]), v[i][1] - bf16hi(ph[i]));
                    }
                }
                const int mi = lane >> 3, rin = lane & 7;
                const int vrow = tb + (mi & 1) * 8 + rin;
#pragma unroll
                for (int j = 0; j < NVT / 2; ++j) {
                    const int c = 2 * j + (mi >> 1);
                    uint32_t v0r, v1r, v2r, v3r;
                    ldsm_x4_trans(vbuf + vrow * ROWB + swz_v(vrow, c) * 16, v0r, v1r, v2r, v3r);
                    mma_bf16_16816(o[2 * j], ph, v0r, v1r);
                    mma_bf16_16816(o[2 * j], pl, v0r, v1r);
                    mma_bf16_16816(o[2 * j + 1], ph, v2r, v3r);
                    mma_bf16_16816(o[2 * j + 1], pl, v2r, v3r);
                }
            }
        }
        __syncthreads();  // batch buffer free for batch bi + 2
    }
    SVL_TRACE(6);
    // warp partials -> CTA O (fixed warp order); ring [0, 64K) as [FCW][16][D]
    float* wo = reinterpret_cast<float*>(smem);
    if (warp < FCW) {
#pragma unroll
        for (int n = 0; n < NVT; ++n) {
            const int col = n * 8 + 2 * t;
            *reinterpret_cast<float2*>(wo + (warp * 16 + gid) * D + col) = make_float2(o[n][0], o[n][1]);
            *reinterpret_cast<float2*>(wo + (warp * 16 + gid + 8) * D + col) = make_float2(o[n][2], o[n][3]);
        }
    }
    __syncthreads();
    float* octa = reinterpret_cast<float*>(smem + GM::OCTA_OFF);  // [16][D]
    for (int i = tid; i < g * D; i += FT) {
        const int h = i / D, dd = i % D;
        float acc = 0.f;
#pragma unroll
        for (int w = 0; w < FCW; ++w) acc += wo[(w * 16 + h) * D + dd];
        octa[h * D + dd] = acc;
    }
    // ------------------------------------------------ 6. cluster merge
    SVL_TRACE(7);
    cl.sync();
    SVL_TRACE(8);
    const int items = g * D;
    const int per = (items + CS - 1) / CS;
    for (int i = rank * per + tid; i < min(items, (rank + 1) * per); i += FT) {
        const int h = i / D, dd = i % D;
        // all 3 x CS remote loads issued before any use (one DSMEM round trip)
        float mq[16], oq[16], lq[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            mq[q] = (q < CS) ? cl.map_shared_rank(Mh, q)[h] : -INFINITY;
            oq[q] = (q < CS) ? cl.map_shared_rank(octa, q)[h * D + dd] : 0.f;
            lq[q] = (q < CS) ? cl.map_shared_rank(lh, q)[h] : 0.f;
        }
        float M = -INFINITY;
#pragma unroll
        for (int q = 0; q < 16; ++q) M = fmaxf(M, mq[q]);
        float num = 0.f, den = 0.f;
        if (M != -INFINITY) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                if (mq[q] != -INFINITY) {
                    const float w = exp2f(mq[q] - M);
                    num += w * oq[q];
                    den += w * lq[q];
                }
            }
        }
        const int hh = G * g + h;
        p.out[((int64_t)b * p.H + hh) * D + dd] = (den > 0.f) ? num / den : 0.f;
        if (dd == 0 && p.lse_out) p.lse_out[(int64_t)b * p.H + hh] = (den > 0.f) ? (M + log2f(den)) * kLn2 : -INFINITY;
    }
    (void)cnt;
    SVL_TRACE(9);
    cl.sync();  // peers may still read this CTA's shared memory until here
    SVL_TRACE(10);
#undef SVL_TRACE
}

template <int D, int NT>
cudaError_t launch_fresh_t(const FreshParams& p, int CS, cudaStream_t s) {
    using GM = FGeom<D, NT>;
    static bool attr_done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_done[dev]) {
        cudaError_t e = cudaFuncSetAttribute(fresh_kernel<D, NT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(fresh_kernel<D, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, GM::BYTES);
        if (e == cudaSuccess) e = set_max_carveout(fresh_kernel<D, NT>);
        if (e != cudaSuccess) return e;
        attr_done[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS, p.B * p.Hkv, 1);
    cfg.blockDim = dim3(FT, 1, 1);
    cfg.dynamicSmemBytes = GM::BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fresh_kernel<D, NT>, p);
}

}  // namespace

cudaError_t launch_fresh(const FreshParams& p, int d, int CS, cudaStream_t s) {
    const int NT = (p.g + 7) / 8;
    if (d == 128 && NT == 1) return launch_fresh_t<128, 1>(p, CS, s);
    if (d == 128 && NT == 2) return launch_fresh_t<128, 2>(p, CS, s);
    if (d == 64 && NT == 1) return launch_fresh_t<64, 1>(p, CS, s);
    if (d == 64 && NT == 2) return launch_fresh_t<64, 2>(p, CS, s);
    return cudaErrorInvalidValue;
}

}  // namespace svl
