// decode.cu -- gathered flash-decoding over the active set on every SM, with
// a log-sum-exp merge of the splits through L2.
//
// PAPER.md:121 / 433: decode attention over the active set only -- all text
// rows plus the k retrieved visual rows ("less relevant tokens
// remain cached but inactive"; SPEC.md:315-323 pack_active order).  For each
// unit (b, KV group G) the attended rows
//     [0, vb)  U  {vb + idx[m] : m < k}  U  [vb + N_v, seq_len)
// are cut into S splits, one CTA each, the grid (S x units) sized to the
// co-resident CTA count (B = 1: 4 units x 37 splits = all 148 SMs).  Split s
// takes the s-th S-th of each of the three segments (system rows, kept visual
// rows, later text rows), so its visual share -- the idx loads and the K/V
// gathers -- does not wait for seq_len.  Per CTA (256 threads, one per SM):
//   1. software pipeline over 128-row batches: row ids of batch j + NBUF are
//      loaded (idx validated: in range, strictly ascending) while batch j is
//      computed; K and V rows of batch j + NBUF - 1 are gathered with cp.async
//      (16-byte, L1-bypassing) into XOR-swizzled shared memory;
//   2. per warp and 16-row tile: S = q K^T with mma.sync m16n8k16 (heads are M,
//      rows are N, the contraction permuted so K chunks are read with
//      conflict-free 128-bit LDS), online softmax in base 2, O += P V with P
//      split into bf16 hi + lo (two MMAs: ~2^-17 relative error instead of
//      bf16's 2^-9) and V B-fragments from ldmatrix.trans;
//   3. S > 1: the CTA's partial (o, m, l) is stored (coalesced) to the
//      workspace; a barrier over the unit's CTAs (release add / acquire spin
//      on a counter in the workspace header; every CTA is co-resident: the
//      grid is sized for it and launched cooperatively); then CTA s merges a
//      1/S slice of its unit's (head, column) items over the S partials,
//      staged in shared memory with one round of coalesced loads:
//      M = max m_i, out = sum e^{m_i-M} o_i / sum e^{m_i-M} l_i,
//      lse = M + log sum e^{m_i-M} l_i (north star step 3), in a fixed order.
//      The counters reset themselves (the unit's last CTA out zeroes them).
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace svl {

namespace {

constexpr int NTH = kDecodeThreads;  // 256: 8 warps
constexpr int NW = NTH / 32;
constexpr int RB = kDecodeRowsMax;   // 128 rows per batch = 8 warps x one 16-row tile
static_assert(RB == 16 * NW, "one 16-row tile per warp and batch");
#ifndef SVL_DECODE_NBUF
#define SVL_DECODE_NBUF 3
#endif
constexpr int NBUF = SVL_DECODE_NBUF;  // gather buffers: NBUF - 1 batches in flight while one is computed
static_assert(NBUF >= 2 && (NBUF - 1) * RB <= NTH, "prologue: one row id per thread");

template <int D>
struct DecodeSmem {
    static constexpr int ROW_BYTES = D * 2;
    static constexpr int BUF_BYTES = 2 * RB * ROW_BYTES;        // K + V of one batch
    static constexpr int ROWS_OFF = NBUF * BUF_BYTES;            // row ids [NBUF][RB]
    static constexpr int TRED_OFF = ROWS_OFF + NBUF * RB * 4;    // tile max / sum [2][NW][16] fp32
    static constexpr int PT_OFF = TRED_OFF + 2 * NW * 16 * 4;    // P hi + lo [RB][16] bf16
    static constexpr int RUN_OFF = PT_OFF + 2 * RB * 16 * 2;     // running M[16], l[16]
    static constexpr int BYTES = RUN_OFF + 32 * 4;
    // merge staging (the gather buffers are free by then)
    static constexpr int MRG_FLOATS = BUF_BYTES / 4;
};

// swizzles (physical 16-byte chunk within a row)
SVL_DEV int swz_k(int row, int c) { return c ^ ((row & 1) << 2); }  // LDS.128 pattern
SVL_DEV int swz_v(int row, int c) { return c ^ (row & 7); }         // ldmatrix.trans pattern

// tagged partials: (float bits, tag) in one 64-bit relaxed (single-copy atomic) access
SVL_DEV void st_tagged(uint64_t* p, float a, uint32_t tag) {
    const uint64_t v = (uint64_t)__float_as_uint(a) | ((uint64_t)tag << 32);
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
SVL_DEV void st_tagged2(uint64_t* p, float a, float b, uint32_t tag) {
    const uint64_t va = (uint64_t)__float_as_uint(a) | ((uint64_t)tag << 32);
    const uint64_t vb = (uint64_t)__float_as_uint(b) | ((uint64_t)tag << 32);
    asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(va), "l"(vb) : "memory");
}
SVL_DEV uint32_t partial_tag(uint32_t epoch, uint32_t u, uint32_t S) {
    uint32_t h = epoch * 0x9E3779B9u ^ (u * 0x85EBCA6Bu + S * 0xC2B2AE35u);
    h ^= h >> 16;
    h *= 0x7FEB352Du;
    h ^= h >> 15;
    h *= 0x846CA68Bu;
    h ^= h >> 16;
    return h ? h : 1u;
}
SVL_DEV uint64_t ld_relaxed_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
SVL_DEV uint32_t ld_relaxed_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int D>
__global__ void __launch_bounds__(NTH, 1) decode_kernel(const __grid_constant__ DecodeParams p) {
    using SM = DecodeSmem<D>;
    constexpr int CH = D / 8;    // 16-byte chunks per row
    constexpr int NCH = D / 32;  // chunks per thread per row in the permuted-k layout
    extern __shared__ __align__(128) uint8_t smem[];
    const int S = (int)gridDim.x, split = (int)blockIdx.x, u = (int)blockIdx.y;
    int* rows_s = reinterpret_cast<int*>(smem + SM::ROWS_OFF);  // [NBUF][RB]
    float* tred = reinterpret_cast<float*>(smem + SM::TRED_OFF);
    uint16_t* pth = reinterpret_cast<uint16_t*>(smem + SM::PT_OFF);  // [RB][16] P hi
    uint16_t* ptl = pth + RB * 16;                                    // [RB][16] P lo
    float* run = reinterpret_cast<float*>(smem + SM::RUN_OFF);       // M[16], l[16]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int gid = lane >> 2, t = lane & 3;
#if SVL_TRACE_BUILD
    uint64_t* trace = p.trace ? p.trace + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16 : nullptr;
    auto stamp = [&](int i) {
        if (trace && tid == 0) {
            uint64_t tnow;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
            trace[i] = tnow;
        }
    };
#else
    auto stamp = [](int) {};
#endif
    stamp(0);
#if SVL_TRACE_BUILD
    if (trace && tid == 0) trace[14] = clock64();
#endif
    // programmatic dependent launch: nothing an upstream kernel may write (seq_len,
    // idx, q, the appended K/V row) is read before the wait
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int b = u / p.Hkv, G = u % p.Hkv;
    const int U = p.shared ? 1 : p.Hkv;
    const int uG = p.shared ? 0 : G;
    // this call's epoch of the unit (advanced by split 0 at the end of the previous call)
    const uint32_t tag_epoch = (S > 1) ? ld_relaxed_u32(p.epochs + u) : 0u;
    // tag = hash(epoch, unit, S): a slot left by another call -- another epoch, or another
    // split layout of the same workspace -- does not match (zero-filled slots never do)
    const uint32_t tag = partial_tag(tag_epoch, (uint32_t)u, (uint32_t)S);
    const int32_t* idx = p.idx + ((int64_t)b * U + uG) * p.k;
    const uint16_t* Kb = p.K + (int64_t)b * p.ksb + (int64_t)G * p.ksh;
    const uint16_t* Vb = p.V + (int64_t)b * p.vsb + (int64_t)G * p.vsh;

    // this split's share of the segments: system rows [s0, s0 + ns), kept visual m in
    // [m0, m0 + nm), later text rows t in [t0, t0 + na) (the last needs seq_len)
    const int s0 = (int)((int64_t)split * p.vb / S), ns = (int)((int64_t)(split + 1) * p.vb / S) - s0;
    const int m0 = (int)((int64_t)split * p.k / S), nm = (int)((int64_t)(split + 1) * p.k / S) - m0;
    struct Pending {
        int x, xp;
    };
    auto fetch = [&](int i) -> Pending {  // list item i: issue its idx loads (visual items only)
        Pending r{0, -1};
        const int m = m0 + (i - ns);
        if (i >= ns && i < ns + nm) {
            r.x = __ldg(idx + m);
            r.xp = m > 0 ? __ldg(idx + m - 1) : -1;
        }
        return r;
    };
    // the first NBUF - 1 batches' idx loads go out together with seq_len's
    Pending pre = fetch(tid);
    int L = __ldg(p.seq_len + b);
    if (L < p.vb + p.nv || L > p.capacity) {
        if (tid == 0 && split == 0) raise_flag(p.flags, 4u /*SPAN*/);
        L = min(max(L, p.vb + p.nv), p.capacity);
    }
    const int T = L - p.vb - p.nv;
    const int t0 = (int)((int64_t)split * T / S), na = (int)((int64_t)(split + 1) * T / S) - t0;
    const int n = ns + nm + na;  // this CTA's attended rows
    const int nb = (n + RB - 1) / RB;
    stamp(1);
    // row id of list item i (-1: past the list, or a bad index -> device flag)
    auto resolve = [&](int i, const Pending& r) -> int {
        if (i < 0 || i >= n) return -1;
        if (i < ns) return s0 + i;
        if (i < ns + nm) {
            if (r.x >= 0 && r.x < p.nv && r.xp < r.x) return p.vb + r.x;
            raise_flag(p.flags, 1u /*SVL_DEVFLAG_INDEX*/);
            return -1;
        }
        return p.vb + p.nv + t0 + (i - ns - nm);
    };
    auto issue = [&](int j) {  // gather batch j (row ids in rows_s[j % NBUF]) -- one commit group
        if (j < nb) {
            const int* rows = rows_s + (j % NBUF) * RB;
            const uint32_t sK = smem_u32(smem + (j % NBUF) * SM::BUF_BYTES);
            const uint32_t sV = sK + RB * SM::ROW_BYTES;
            const int nj = min(RB, n - j * RB);
            const int nr = (nj + 15) & ~15;
            // thread -> chunk c of rows r0, r0 + NTH/CH, ...: every row id read first, then
            // all the copies back to back (no shared-memory load between two copies)
            constexpr int RPP = NTH / CH, PASSES = RB / RPP;
            const int c = tid % CH, r0 = tid / CH;
            int rw[PASSES];
#pragma unroll
            for (int k = 0; k < PASSES; ++k) rw[k] = (r0 + k * RPP < nr) ? rows[r0 + k * RPP] : -2;
#pragma unroll
            for (int k = 0; k < PASSES; ++k) {
                const int r = r0 + k * RPP;
                if (rw[k] == -2) continue;
                const bool valid = rw[k] >= 0;
                const int rr = valid ? rw[k] : 0;
                cp_async16(sK + r * SM::ROW_BYTES + swz_k(r, c) * 16, Kb + (int64_t)rr * p.kst + c * 8, valid);
                cp_async16(sV + r * SM::ROW_BYTES + swz_v(r, c) * 16, Vb + (int64_t)rr * p.vst + c * 8, valid);
            }
        }
        cp_async_commit();  // (empty groups keep the wait_group arithmetic uniform)
    };

    // ---- prologue: row ids of batches [0, NBUF - 1) (one per thread), their gathers, and
    // the idx loads of batch NBUF - 1 (consumed at the top of iteration 0)
    if (tid < (NBUF - 1) * RB) rows_s[tid] = resolve(tid, pre);
    Pending pend = tid < RB ? fetch((NBUF - 1) * RB + tid) : Pending{0, -1};
    if (tid < 16) {
        run[tid] = -INFINITY;
        run[16 + tid] = 0.f;
    }
    cta_sync();
    stamp(2);
    for (int j = 0; j < NBUF - 1; ++j) issue(j);

    // q A-fragments (heads gid, gid + 8 of the group; zero beyond g)
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

    float o[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    static_assert(D / 16 <= NW, "one warp per 16 output columns");

    for (int j = 0; j < nb; ++j) {
        // row ids of batch j + NBUF - 1 (loads issued one iteration ago), then the loads of
        // batch j + NBUF's; the barrier publishes the ids and frees buffer (j - 1) % NBUF
        if (tid < RB) rows_s[((j + NBUF - 1) % NBUF) * RB + tid] = resolve((j + NBUF - 1) * RB + tid, pend);
        if (tid < RB) pend = fetch((j + NBUF) * RB + tid);
        cta_sync();
        issue(j + NBUF - 1);
        cp_async_wait<NBUF - 1>();  // batch j landed (this thread's copies)
        cta_sync();                 // ... and everyone's
        if (j == 0) stamp(3);
#if SVL_EXP_NOCOMPUTE  // timing experiment: gather only
        continue;
#endif
        const int* rows = rows_s + (j % NBUF) * RB;
        const uint32_t sK = smem_u32(smem + (j % NBUF) * SM::BUF_BYTES);
        const uint32_t sV = sK + RB * SM::ROW_BYTES;
        const int nj = min(RB, n - j * RB);
        const int nr = (nj + 15) & ~15;  // rows padded to whole 16-row tiles
        const int tb = warp * 16;
        const int ntl = nr >> 4;
        float s[2][4];  // n-tile nt: c0, c1 -> head gid, rows tb + 8nt + 2t, +1; c2, c3 -> head gid + 8
        if (tb < nr) {
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
            float mx_a = -INFINITY, mx_b = -INFINITY;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int rr = tb + nt * 8 + 2 * t + (e & 1);
                    const int h = gid + 8 * (e >> 1);
                    s[nt][e] = (rr < nj && rows[rr] >= 0 && h < p.g) ? s[nt][e] * p.scale2 : -INFINITY;
                    if (e < 2) mx_a = fmaxf(mx_a, s[nt][e]);
                    else mx_b = fmaxf(mx_b, s[nt][e]);
                }
            mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, 1));
            mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, 2));
            mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, 1));
            mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, 2));
            if (t == 0) {
                tred[warp * 16 + gid] = mx_a;
                tred[warp * 16 + gid + 8] = mx_b;
            }
        }
        cta_sync();
        if (j == 0) stamp(10);
        // batch max of heads gid, gid + 8 (every thread, same fixed order) -> new running max
        float bm_a = -INFINITY, bm_b = -INFINITY;
        for (int w = 0; w < ntl; ++w) {
            bm_a = fmaxf(bm_a, tred[w * 16 + gid]);
            bm_b = fmaxf(bm_b, tred[w * 16 + gid + 8]);
        }
        const float mo_a = run[gid], mo_b = run[gid + 8];
        const float mn_a = fmaxf(mo_a, bm_a), mn_b = fmaxf(mo_b, bm_b);
        if (tb < nr) {
            // P = exp2(s - M) into the split bf16 table; tile sums of the weights the PV uses
            float ls_a = 0.f, ls_b = 0.f;
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float mn = (e < 2) ? mn_a : mn_b;
                    const float pv = (s[nt][e] == -INFINITY) ? 0.f : fast_exp2(s[nt][e] - mn);
                    const __nv_bfloat16 hi = __float2bfloat16_rn(pv);
                    const __nv_bfloat16 lo = __float2bfloat16_rn(pv - __bfloat162float(hi));
                    const int rr = tb + nt * 8 + 2 * t + (e & 1), h = gid + 8 * (e >> 1);
                    pth[rr * 16 + h] = *reinterpret_cast<const uint16_t*>(&hi);
                    ptl[rr * 16 + h] = *reinterpret_cast<const uint16_t*>(&lo);
                    const float w = __bfloat162float(hi) + __bfloat162float(lo);
                    if (e < 2) ls_a += w;
                    else ls_b += w;
                }
            ls_a += __shfl_xor_sync(0xffffffffu, ls_a, 1);
            ls_a += __shfl_xor_sync(0xffffffffu, ls_a, 2);
            ls_b += __shfl_xor_sync(0xffffffffu, ls_b, 1);
            ls_b += __shfl_xor_sync(0xffffffffu, ls_b, 2);
            if (t == 0) {
                tred[NW * 16 + warp * 16 + gid] = ls_a;
                tred[NW * 16 + warp * 16 + gid + 8] = ls_b;
            }
        }
        cta_sync();
        if (j == 0) stamp(11);
        if (tid < 16) {  // running (M, l) of head tid; fixed tile order
            const float mo = run[tid];
            float mn = mo, ls = 0.f;
            for (int w = 0; w < ntl; ++w) {
                mn = fmaxf(mn, tred[w * 16 + tid]);
                ls += tred[NW * 16 + w * 16 + tid];
            }
            const float al = (mn == -INFINITY) ? 1.f : fast_exp2(mo - mn);
            run[16 + tid] = run[16 + tid] * al + ls;
            run[tid] = mn;
        }
        const float al_a = (mn_a == -INFINITY) ? 1.f : fast_exp2(mo_a - mn_a);
        const float al_b = (mn_b == -INFINITY) ? 1.f : fast_exp2(mo_b - mn_b);
        if (warp < D / 16) {
            // rescale this warp's accumulator rows (heads gid, gid + 8), then O += P V
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                o[nt][0] *= al_a; o[nt][1] *= al_a;
                o[nt][2] *= al_b; o[nt][3] *= al_b;
            }
            const int mi = lane >> 3, rin = lane & 7;
            const uint32_t aph = smem_u32(pth), apl = smem_u32(ptl);
            // k-steps of 16 rows; the hi and lo products go to separate accumulators (two
            // independent MMA chains per n-tile), summed once after the batch
            float ol[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
            for (int tt = 0; tt < RB; tt += 16) {
                if (tt < nr) {
                    // P fragment (m = heads, k = rows): matrices (h0-7,k0-7) (h8-15,k0-7) (h0-7,k8-15) (h8-15,k8-15)
                    const int prow = tt + (mi >> 1) * 8 + rin;
                    uint32_t ph[4], pl4[4];
                    ldsm_x4_trans(aph + prow * 32 + (mi & 1) * 16, ph[0], ph[1], ph[2], ph[3]);
                    ldsm_x4_trans(apl + prow * 32 + (mi & 1) * 16, pl4[0], pl4[1], pl4[2], pl4[3]);
                    const int vrow = tt + (mi & 1) * 8 + rin;
                    const int c = 2 * warp + (mi >> 1);
                    uint32_t v0, v1, v2, v3;
                    ldsm_x4_trans(sV + vrow * SM::ROW_BYTES + swz_v(vrow, c) * 16, v0, v1, v2, v3);
                    mma_bf16_16816(o[0], ph, v0, v1);
                    mma_bf16_16816(ol[0], pl4, v0, v1);
                    mma_bf16_16816(o[1], ph, v2, v3);
                    mma_bf16_16816(ol[1], pl4, v2, v3);
                }
            }
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) o[nt][e] += ol[nt][e];
        }
    }
    cp_async_wait<0>();
    cta_sync();  // run[] final (also when this CTA had no rows); the gather buffers are free
    stamp(4);

    constexpr int PSTRIDE = kDecodePartStride<D>;
    auto finalize = [&](int h, int dd, float ov, float M, float den) {
        const int hh = G * p.g + h;
        if (p.out) p.out[((int64_t)b * p.H + hh) * D + dd] = ov;
        if (dd == 0 && p.lse_out)
            p.lse_out[(int64_t)b * p.H + hh] = (den > 0.f) ? (M + log2f(den)) * kLn2 : -INFINITY;
        if (p.P > 0) {  // push variant: the same value into every peer's gathered output (NVLink stores)
            const int64_t go = ((int64_t)(p.b0 + b) * p.H_total + p.h0 + hh) * D + dd;
            for (int r = 0; r < p.P; ++r) p.peer_out[r][go] = ov;
        }
    };
    if (S == 1) {
        if (warp < D / 16) {
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int h = gid + 8 * (e >> 1), dd = warp * 16 + nt * 8 + 2 * t + (e & 1);
                    if (h < p.g) {
                        const float den = run[16 + h];
                        finalize(h, dd, den > 0.f ? o[nt][e] / den : 0.f, run[h], den);
                    }
                }
        }
    } else {
        // Partial (o, M, l) of this split -> workspace slot (u, split), every value stored as a
        // 64-bit (bits, tag) pair with one single-copy-atomic store; tag = the unit's call
        // epoch.  A reader that sees the tag sees the value: no barrier, no flag round trip.
        uint64_t* mine = p.part + (int64_t)(u * S + split) * PSTRIDE;
        if (warp < D / 16) {
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                const int col = warp * 16 + nt * 8 + 2 * t;
                if (gid < p.g) st_tagged2(mine + gid * D + col, o[nt][0], o[nt][1], tag);
                if (gid + 8 < p.g) st_tagged2(mine + (gid + 8) * D + col, o[nt][2], o[nt][3], tag);
            }
        }
        if (tid < 32) st_tagged(mine + 16 * D + tid, run[tid], tag);  // M[16], l[16]
        stamp(5);
        // merge this CTA's slice [i0, i0 + ni) of the unit's g x D items over the S partials:
        // every value loaded at once (relaxed 64-bit loads), the ones whose tag is not this
        // call's re-polled until they are (bounded), then staged in shared memory
        const int items = p.g * D, per = (items + S - 1) / S;
        const int i0 = split * per, ni = max(0, min(per, items - i0));
        if (ni > 0) {
            const int h0 = i0 / D, nh = (i0 + ni - 1) / D - h0 + 1;
            float* ob = reinterpret_cast<float*>(smem);  // [S][ni]
            float* mb = ob + S * ni;                     // [S][nh] m, then the weights
            float* lb = mb + S * nh;                     // [S][nh]
            float* hM = lb + S * nh;                     // [nh] M, den
            const uint64_t* up = p.part + (int64_t)u * S * PSTRIDE;
            constexpr int MAXL = (16 * D + kDecodeMaxSplits + NTH - 1) / NTH;  // S * ni <= g D + S
            uint64_t v[MAXL], vm[2], vl[2];  // S * nh <= max(2 S, S + 16) <= 2 NTH
            auto addr_o = [&](int e) { const int q = e / ni; return up + (int64_t)q * PSTRIDE + i0 + (e - q * ni); };
            auto addr_m = [&](int e) { const int q = e / nh; return up + (int64_t)q * PSTRIDE + 16 * D + h0 + (e - q * nh); };
#pragma unroll
            for (int r = 0; r < MAXL; ++r) {
                const int e = tid + r * NTH;
                v[r] = (e < S * ni) ? ld_relaxed_u64(addr_o(e)) : ((uint64_t)tag << 32);
            }
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int e = tid + r * NTH;
                vm[r] = (e < S * nh) ? ld_relaxed_u64(addr_m(e)) : ((uint64_t)tag << 32);
                vl[r] = (e < S * nh) ? ld_relaxed_u64(addr_m(e) + 16) : ((uint64_t)tag << 32);
            }
            for (uint32_t it = 0;; ++it) {
                bool ready = true;
#pragma unroll
                for (int r = 0; r < MAXL; ++r) ready &= (uint32_t)(v[r] >> 32) == tag;
#pragma unroll
                for (int r = 0; r < 2; ++r) ready &= (uint32_t)(vm[r] >> 32) == tag && (uint32_t)(vl[r] >> 32) == tag;
                if (ready) break;
                if (it > (1u << 22)) {  // ~seconds: a broken co-residency assumption, not a hang
                    raise_flag(p.flags, 8u /*SVL_DEVFLAG_WAIT_TIMEOUT*/);
                    break;
                }
                __nanosleep(64);
#pragma unroll
                for (int r = 0; r < MAXL; ++r)
                    if ((uint32_t)(v[r] >> 32) != tag) v[r] = ld_relaxed_u64(addr_o(tid + r * NTH));
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    if ((uint32_t)(vm[r] >> 32) != tag) vm[r] = ld_relaxed_u64(addr_m(tid + r * NTH));
                    if ((uint32_t)(vl[r] >> 32) != tag) vl[r] = ld_relaxed_u64(addr_m(tid + r * NTH) + 16);
                }
            }
#pragma unroll
            for (int r = 0; r < MAXL; ++r) {
                const int e = tid + r * NTH;
                if (e < S * ni) ob[e] = __uint_as_float((uint32_t)v[r]);
            }
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const int e = tid + r * NTH;
                if (e < S * nh) {
                    mb[e] = __uint_as_float((uint32_t)vm[r]);
                    lb[e] = __uint_as_float((uint32_t)vl[r]);
                }
            }
            cta_sync();
            stamp(8);
            for (int hh = warp; hh < nh; hh += NW) {  // per head: M, weights, den (lanes over splits)
                float M = -INFINITY;
                for (int q = lane; q < S; q += 32) M = fmaxf(M, mb[q * nh + hh]);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
                float den = 0.f;
                for (int q = lane; q < S; q += 32) {
                    const float w = (M == -INFINITY) ? 0.f : fast_exp2(mb[q * nh + hh] - M);
                    mb[q * nh + hh] = w;
                    den += w * lb[q * nh + hh];
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) den += __shfl_xor_sync(0xffffffffu, den, off);
                if (lane == 0) {
                    hM[2 * hh] = M;
                    hM[2 * hh + 1] = den;
                }
            }
            cta_sync();
            stamp(9);
            // per item: T threads (a power of two <= 32) stride over the splits, then a
            // fixed xor tree inside the T-lane group; every lane takes part in the shuffles
            int T = 32;
            while (T > 1 && T * ni > 2 * NTH) T >>= 1;
            for (int jb = 0; jb < ni; jb += NTH / T) {
                const int j = jb + tid / T, sub = tid & (T - 1);
                const int hh = (j < ni) ? (i0 + j) / D - h0 : 0;
                float num = 0.f;
                if (j < ni) {
#pragma unroll 4
                    for (int q = sub; q < S; q += T) num += mb[q * nh + hh] * ob[q * ni + j];
                }
                for (int off = T >> 1; off > 0; off >>= 1) num += __shfl_xor_sync(0xffffffffu, num, off);
                if (sub == 0 && j < ni) {
                    const float den = hM[2 * hh + 1];
                    finalize(h0 + hh, (i0 + j) % D, (den > 0.f) ? num / den : 0.f, hM[2 * hh], den);
                }
            }
        }
        // split 0 advances the unit's epoch once its own merge has seen every split's
        // partial -- so every CTA of the unit has read the current epoch already
        if (split == 0 && tid == 0) p.epochs[u] = tag_epoch + 1u;
    }
    stamp(7);
#if SVL_TRACE_BUILD
    if (trace && tid == 0) trace[15] = clock64();
#endif
    // push variant: the grid's last CTA publishes the epoch flags once every CTA's peer
    // stores are fenced at system scope (self-resetting counter, header word 3)
    if (p.P > 0) {
        cta_sync();
        if (tid == 0) {
            __threadfence_system();
            const uint32_t total = gridDim.x * gridDim.y;
            if (atomicAdd(p.sync + 3, 1u) == total - 1u) {
                p.sync[3] = 0u;
                __threadfence_system();
                for (int r = 0; r < p.P; ++r)
                    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p.peer_flags[r] + p.rank), "r"(p.epoch)
                                 : "memory");
            }
        }
    }
}

// consumer side of the push variant: one thread spins (acquire, system scope)
// until flags[s] has reached epoch for every producer s; bounded (~2 s), a
// timeout sets SVL_DEVFLAG_WAIT_TIMEOUT instead of hanging the stream.
__global__ void wait_flags_kernel(const uint32_t* flags, int P, uint32_t epoch, uint32_t* ws_flags) {
    if (threadIdx.x != 0) return;
    for (int s = 0; s < P; ++s) {
        for (uint32_t it = 0;; ++it) {
            uint32_t v;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + s) : "memory");
            if ((int32_t)(v - epoch) >= 0) break;
            if (it > (1u << 21)) {
                atomicOr(ws_flags, 8u /*SVL_DEVFLAG_WAIT_TIMEOUT*/);
                return;
            }
            __nanosleep(1000);
        }
    }
}

template <int D>
cudaError_t prepare_decode_t() {
    using SM = DecodeSmem<D>;
    static bool attr_done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && attr_done[dev]) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::BYTES);
    if (e == cudaSuccess) e = set_max_carveout(decode_kernel<D>);
    if (e == cudaSuccess && dev < 64) attr_done[dev] = true;
    return e;
}

template <int D>
cudaError_t launch_decode_t(const DecodeParams& p, cudaStream_t s) {
    using SM = DecodeSmem<D>;
    cudaError_t e = prepare_decode_t<D>();
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.S, p.B * p.Hkv);
    cfg.blockDim = dim3(NTH);
    cfg.dynamicSmemBytes = SM::BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see griddepcontrol in the kernel
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    // the grid barrier needs every CTA resident: the grid is sized to the co-resident count,
    // and a cooperative launch makes the runtime guarantee it
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
#if SVL_DECODE_NO_COOP  // A/B builds: co-residency by grid sizing alone
    cfg.numAttrs = 1;
#else
    cfg.numAttrs = p.S > 1 ? 2 : 1;
#endif
#if SVL_DECODE_NO_PDL  // A/B builds
    attr[0] = attr[1];
    cfg.numAttrs -= 1;
#endif
    return cudaLaunchKernelEx(&cfg, decode_kernel<D>, p);
}

template <int D>
int decode_ctas_per_sm_t() {
    if (prepare_decode_t<D>() != cudaSuccess) return 0;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, decode_kernel<D>, NTH, DecodeSmem<D>::BYTES) !=
        cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

}  // namespace

cudaError_t launch_wait_flags(const uint32_t* flags, int P, uint32_t epoch, uint32_t* ws_flags, cudaStream_t s) {
    wait_flags_kernel<<<1, 32, 0, s>>>(flags, P, epoch, ws_flags);
    return cudaGetLastError();
}

cudaError_t launch_decode(const DecodeParams& p, int d, cudaStream_t s) {
    if (d == 128) return launch_decode_t<128>(p, s);
    if (d == 64) return launch_decode_t<64>(p, s);
    return cudaErrorInvalidValue;
}

int decode_ctas_per_sm(int d) {
    static int cache[64][2] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 1;
    int& c = cache[dev][d == 128];
    if (c == 0) {
        c = (d == 128) ? decode_ctas_per_sm_t<128>() : decode_ctas_per_sm_t<64>();
        if (c <= 0) c = 1;
    }
    return c;
}

}  // namespace svl
