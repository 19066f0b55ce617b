// decode.cu -- gathered flash-decoding over the active set, split across a
// thread-block cluster with an on-chip log-sum-exp merge.
//
// PAPER.md:121 / 433: decode attention over the active set only -- all text
// rows plus the k retrieved visual rows ("less relevant tokens
// remain cached but inactive"; SPEC.md:315-323 pack_active order).  For each
// unit (b, KV group G) the attended row list
//     [0, vb)  U  {vb + idx[m]}  U  [vb + N_v, seq_len)
// (ascending) is cut into CS contiguous splits, one per CTA of a cluster:
//   1. per batch of <= 128 rows: row ids (validating idx: in range, strictly
//      ascending), K and V rows gathered with cp.async (16-byte, L1-bypassing)
//      into XOR-swizzled shared memory, double buffered (batch j+1 in flight
//      while batch j is computed);
//   2. per warp and 16-row tile: S = q K^T with mma.sync m16n8k16 (heads are M,
//      rows are N, the contraction d permuted so K chunks are read with
//      conflict-free 128-bit LDS), online softmax in base 2, O += P V with P
//      split into bf16 hi + lo (two MMAs; ~2^-17 relative error instead of
//      bf16's 2^-9) and V B-fragments from ldmatrix.trans;
//   3. warps -> CTA partial (o, m, l) in shared memory; cluster barrier; CTA r
//      merges a 1/CS share of the (head, column) items from the CS partials
//      over DSMEM in rank order: M = max m_i, out = sum e^{m_i-M} o_i /
//      sum e^{m_i-M} l_i, lse = M + log sum e^{m_i-M} l_i (north star step 3).
// No second kernel and no global partials.
#include <cooperative_groups.h>

#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace svl {

namespace {

constexpr int NTH = kDecodeThreads;  // 256: 8 warps, one 16-row tile each per batch
constexpr int RB = kDecodeRowsMax;   // 128 rows per batch
#ifndef SVL_DECODE_NBUF
#define SVL_DECODE_NBUF 2  // measured: 3 buffers (220 KB) gave no gain (9.5 vs 9.4 us long-video, 92.4 vs 92.9 sweep)
#endif
constexpr int NBUF = SVL_DECODE_NBUF;  // gather buffers (NBUF - 1 batches in flight)
constexpr int NW = NTH / 32;

template <int D>
struct DecodeSmem {
    static constexpr int CH = D / 8;  // 16-byte chunks per row
    static constexpr int ROW_BYTES = D * 2;
    static constexpr int BUF_BYTES = 2 * RB * ROW_BYTES;  // K + V of one batch
    static constexpr int ROWS_OFF = NBUF * BUF_BYTES;     // NBUF gather buffers
    static constexpr int SL_OFF = ROWS_OFF + NBUF * RB * 4;  // tile max / sum [2][128] fp32
    static constexpr int PT_OFF = SL_OFF + RB * 16 * 4;   // P hi + lo [RB][16] bf16
    static constexpr int RUN_OFF = PT_OFF + 2 * RB * 16 * 2;  // running M, l, al [3][16]
    static constexpr int RCV_OFF = RUN_OFF + 64 * 4;      // [CS][per] pushed o (CS * per <= 16 D + 16)
    static constexpr int RML_OFF = RCV_OFF + (16 * D + 16) * 4;  // [16][32] pushed M, l
    static constexpr int MB_OFF = RML_OFF + 16 * 32 * 4;     // merge mbarrier (st.async byte count)
    static constexpr int BYTES = MB_OFF + 16;
};

// swizzles (physical 16-byte chunk within a row)
SVL_DEV int swz_k(int row, int c) { return c ^ ((row & 1) << 2); }  // LDS.128 pattern
SVL_DEV int swz_v(int row, int c) { return c ^ (row & 7); }         // ldmatrix.trans pattern

template <int D>
__global__ void __launch_bounds__(NTH, 1) decode_kernel(const DecodeParams p) {
    using SM = DecodeSmem<D>;
    constexpr int CH = SM::CH;
    constexpr int NCH = D / 32;  // chunks per thread per row in the permuted-k layout
    constexpr int NVT = D / 8;   // n-tiles of the output
    extern __shared__ __align__(128) uint8_t smem[];
    cg::cluster_group cl = cg::this_cluster();
    const int CS = (int)cl.num_blocks(), rank = (int)cl.block_rank();
    int* rows_s = reinterpret_cast<int*>(smem + SM::ROWS_OFF);  // [NBUF][RB]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int gid = lane >> 2, t = lane & 3;
    const int u = blockIdx.y;
    const uint32_t mb = smem_u32(smem + SM::MB_OFF);
    if (tid == 0) {  // merge barrier: one local arrival + the bytes every peer will store
        const int items = p.g * D, per = (items + CS - 1) / CS;
        const int mine = max(0, min(per, items - rank * per));
        mbar_init(mb, 1);
        mbar_arrive_expect_tx(mb, (uint32_t)(CS * (mine + 32) * 4));
        fence_mbar_init();
    }
    cluster_arrive_relaxed();  // this CTA is resident (peers push into it after their cluster_wait)
    // programmatic dependent launch: everything above overlaps the upstream kernel's tail;
    // nothing it may write (seq_len, idx, q, the appended K/V row) is read before this
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    uint64_t* trace = p.trace ? p.trace + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16 : nullptr;
    auto stamp = [&](int i) {
        if (trace && tid == 0) {
            uint64_t tnow;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
            trace[i] = tnow;
        }
    };
    stamp(0);
    const int b = u / p.Hkv, G = u % p.Hkv;
    const int U = p.shared ? 1 : p.Hkv;
    const int uG = p.shared ? 0 : G;

    int L = p.seq_len[b];
    if (L < p.vb + p.nv || L > p.capacity) {
        if (tid == 0 && rank == 0) raise_flag(p.flags, 4u /*SPAN*/);
        L = min(max(L, p.vb + p.nv), p.capacity);
    }
    const int n_att = p.vb + p.k + (L - p.vb - p.nv);
    const int w0 = (int)((int64_t)rank * n_att / CS);
    const int w1 = (int)((int64_t)(rank + 1) * n_att / CS);
    const int nb = (w1 - w0 + RB - 1) / RB;

    const int32_t* idx = p.idx + ((int64_t)b * U + uG) * p.k;
    const uint16_t* Kb = p.K + (int64_t)b * p.ksb + (int64_t)G * p.ksh;
    const uint16_t* Vb = p.V + (int64_t)b * p.vsb + (int64_t)G * p.vsh;

    // batch j: row ids into rows_s[j % NBUF], then the K/V gather (one commit group)
    auto load_batch = [&](int j) {
        int* rows = rows_s + (j % NBUF) * RB;
        const int a = w0 + j * RB, n = min(RB, w1 - a);
        bool bad = false;
        for (int i = tid; i < RB; i += NTH) {
            int row = -1;
            const int w = a + i;
            if (i < n) {
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
        cta_sync();
        const uint32_t sK = smem_u32(smem + (j % NBUF) * SM::BUF_BYTES);
        const uint32_t sV = sK + RB * SM::ROW_BYTES;
        const int nr = (n + 15) & ~15;
        for (int i = tid; i < nr * CH; i += NTH) {
            const int r = i / CH, c = i % CH;
            const int row = rows[r];
            const bool valid = row >= 0;
            const int rr = valid ? row : 0;
            cp_async16(sK + r * SM::ROW_BYTES + swz_k(r, c) * 16, Kb + (int64_t)rr * p.kst + c * 8, valid);
            cp_async16(sV + r * SM::ROW_BYTES + swz_v(r, c) * 16, Vb + (int64_t)rr * p.vst + c * 8, valid);
        }
        cp_async_commit();
    };

    for (int j = 0; j < min(nb, NBUF - 1); ++j) load_batch(j);  // NBUF - 1 batches in flight

    // q A-fragments (heads gid, gid+8 of the group; zero beyond g)
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

    // Per batch: every warp scores one 16-row tile (tile max per head to smem); the
    // CTA folds the batch into a running per-head max M (rescale factor al), writes
    // P = exp2(s - M) as a split bf16 hi + lo table, and warp w accumulates the
    // output columns [16w, 16w + 16) of all 16 heads over the batch's rows (no
    // cross-warp reduction at the end).
    float* tred = reinterpret_cast<float*>(smem + SM::SL_OFF);        // [2][NW][16] tile max, tile sum
    uint16_t* pth = reinterpret_cast<uint16_t*>(smem + SM::PT_OFF);    // [RB][16] P hi
    uint16_t* ptl = pth + RB * 16;                                      // [RB][16] P lo
    float* run = reinterpret_cast<float*>(smem + SM::RUN_OFF);         // M[16], l[16], al[16]
    if (tid < 16) {
        run[tid] = -INFINITY;
        run[16 + tid] = 0.f;
    }
    float o[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    static_assert(D / 16 <= NW, "one warp per 16 output columns");

    for (int j = 0; j < nb; ++j) {
        if (j + NBUF - 1 < nb) {
            cta_sync();  // buffer (j + NBUF - 1) % NBUF = (j - 1) % NBUF is no longer read
            load_batch(j + NBUF - 1);
            cp_async_wait<NBUF - 1>();
        } else if (NBUF > 2 && j + 1 < nb) {
            cp_async_wait<1>();  // batches j and j + 1 outstanding (no more issued)
        } else {
            cp_async_wait<0>();
        }
        cta_sync();
        stamp(1 + j);
        const int* rows = rows_s + (j % NBUF) * RB;
        const uint32_t sK = smem_u32(smem + (j % NBUF) * SM::BUF_BYTES);
        const uint32_t sV = sK + RB * SM::ROW_BYTES;
        const int n = min(RB, w1 - (w0 + j * RB));
        const int nr = (n + 15) & ~15;
        const int tb = warp * 16;
        const int ntl = nr >> 4;  // tiles in this batch
        float s[2][4];            // this warp's tile: C layout c0,c1 -> head gid, rows 2t,2t+1; c2,c3 -> head gid+8
        if (tb < nr) {
            // S = q K^T : two n-tiles of 8 rows
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
                    const int r = tb + nt * 8 + 2 * t + (e & 1);
                    const int h = gid + 8 * (e >> 1);
                    s[nt][e] = (r < n && rows[r] >= 0 && h < p.g) ? s[nt][e] * p.scale2 : -INFINITY;
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
                    const int r = tb + nt * 8 + 2 * t + (e & 1), h = gid + 8 * (e >> 1);
                    pth[r * 16 + h] = *reinterpret_cast<const uint16_t*>(&hi);
                    ptl[r * 16 + h] = *reinterpret_cast<const uint16_t*>(&lo);
                    const float w = __bfloat162float(hi) + __bfloat162float(lo);
                    if (e < 2) ls_a += w;
                    else ls_b += w;
                }
            ls_a += __shfl_xor_sync(0xffffffffu, ls_a, 1);
            ls_a += __shfl_xor_sync(0xffffffffu, ls_a, 2);
            ls_b += __shfl_xor_sync(0xffffffffu, ls_b, 1);
            ls_b += __shfl_xor_sync(0xffffffffu, ls_b, 2);
            if (t == 0) {
                tred[128 + warp * 16 + gid] = ls_a;
                tred[128 + warp * 16 + gid + 8] = ls_b;
            }
        }
        cta_sync();
        if (tid < 16) {  // running (M, l) of head tid; fixed tile order
            const float mo = run[tid];
            float mn = mo, ls = 0.f;
            for (int w = 0; w < ntl; ++w) {
                mn = fmaxf(mn, tred[w * 16 + tid]);
                ls += tred[128 + w * 16 + tid];
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
            for (int tt = 0; tt < nr; tt += 16) {
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
                mma_bf16_16816(o[0], pl4, v0, v1);
                mma_bf16_16816(o[1], ph, v2, v3);
                mma_bf16_16816(o[1], pl4, v2, v3);
            }
        }
    }
    cta_sync();  // run[] final (also when this CTA had no rows)
    stamp(10);
    cluster_wait();   // every peer has started (first DSMEM access below)

    // ---- 3. CTA partial pushed straight to the owning peers, then the owners merge
    // item i = h * D + dd is owned by CTA i / per; a CTA sends owner q its
    // (o, M, l) for q's items into slot [rank] of q's receive buffer.
    const int items = p.g * D;
    const int per = (items + CS - 1) / CS;
    float* rcv = reinterpret_cast<float*>(smem + SM::RCV_OFF);   // [CS][per] o
    float* rml = reinterpret_cast<float*>(smem + SM::RML_OFF);   // [16][2][16] M, l
    if (warp < D / 16) {
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int h = gid + 8 * (e >> 1), dd = warp * 16 + nt * 8 + 2 * t + (e & 1);
                if (h < p.g) {
                    const int i = h * D + dd, q = i / per;
                    st_async_f32(mapa_shared(smem_u32(&rcv[rank * per + (i - q * per)]), q), o[nt][e], mapa_shared(mb, q));
                }
            }
    }
    for (int i = tid; i < 32 * CS; i += NTH) {  // M[0, 16) and l[16, 32) of every head to every peer
        const int q = i >> 5, h = i & 31;
        st_async_f32(mapa_shared(smem_u32(&rml[rank * 32 + h]), q), run[h], mapa_shared(mb, q));
    }
    stamp(11);
    mbar_wait(mb, 0);  // the bytes of every peer landed (st.async counts them on this barrier)
    stamp(12);
    for (int i = rank * per + tid; i < min(items, (rank + 1) * per); i += NTH) {
        const int h = i / D, dd = i % D, li = i - rank * per;
        float M = -INFINITY;
        for (int q = 0; q < CS; ++q) M = fmaxf(M, rml[q * 32 + h]);
        float num = 0.f, den = 0.f;
        if (M != -INFINITY) {
            for (int q = 0; q < CS; ++q) {
                const float w = fast_exp2(rml[q * 32 + h] - M);
                num += w * rcv[q * per + li];
                den += w * rml[q * 32 + 16 + h];
            }
        }
        const int hh = G * p.g + h;
        const float ov = (den > 0.f) ? num / den : 0.f;
        if (p.out) p.out[((int64_t)b * p.H + hh) * D + dd] = ov;
        if (dd == 0 && p.lse_out)
            p.lse_out[(int64_t)b * p.H + hh] = (den > 0.f) ? (M + log2f(den)) * kLn2 : -INFINITY;
        // push variant: the same value into every peer's gathered output (NVLink stores)
        const int64_t go = ((int64_t)(p.b0 + b) * p.H_total + p.h0 + hh) * D + dd;
        for (int r = 0; r < p.P; ++r) p.peer_out[r][go] = ov;
    }
    stamp(13);
    if (p.P > 0) {
        // the last CTA of the grid publishes: every CTA's stores are fenced at system
        // scope before its arrival, so the last arrival sees them all
        cta_sync();
        if (tid == 0) {
            __threadfence_system();
            const uint32_t total = gridDim.x * gridDim.y;
            if (atomicAdd(p.done, 1u) == total - 1u) {
                atomicExch(p.done, 0u);  // the workspace counter is zero again for the next call
                __threadfence_system();
                for (int r = 0; r < p.P; ++r)
                    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p.peer_flags[r] + p.rank), "r"(p.epoch)
                                 : "memory");
            }
        }
    }
    // no closing cluster barrier: nobody reads a peer's shared memory, and every CTA waited
    // for all the bytes pushed into it before getting here
    stamp(14);
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
cudaError_t launch_decode_t(const DecodeParams& p, cudaStream_t s) {
    using SM = DecodeSmem<D>;
    static bool attr_done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_done[dev]) {
        cudaError_t e = cudaFuncSetAttribute(decode_kernel<D>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(decode_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::BYTES);
        if (e == cudaSuccess) e = set_max_carveout(decode_kernel<D>);
        if (e != cudaSuccess) return e;
        attr_done[dev] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.S, p.B * p.Hkv);
    cfg.blockDim = dim3(NTH);
    cfg.dynamicSmemBytes = SM::BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see griddepcontrol in the kernel
    attr[1].val.programmaticStreamSerializationAllowed = getenv("SVL_NO_PDL") ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, decode_kernel<D>, p);
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

}  // namespace svl
