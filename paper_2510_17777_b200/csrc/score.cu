// score.cu -- retrieval scoring, phase 1 of svl_retrieve.
//
// relevance = "aggregate attention strength between the query
// embeddings and visual entries in the KV cache", streamed "directly between
// the query and cached visual tokens".  This kernel streams bf16 K rows of
// one unit (b, KV group G) from HBM once, computes the base-2 logits
//   s2[j, c] = scale*log2(e) * q[b, r, h] . K[b, G, j],   c = r*g + (h - G*g)
// for the unit's NC = n_q*g query columns, writes them (visual rows only) to
// an L2-resident fp32 scratch, and reduces each chunk's (max, sum) partial for
// the full-causal-prefix log-sum-exp (text rows included, never stored).
//
// B200 mapping: memory-bound GEMV (g*n_q flop/B).  Swap-AB mma.sync
// m16n8k16: K rows are M (16 per warp tile), query columns are N (8 per
// n-tile), d is the contraction.  Because the contraction index may be
// permuted consistently in A and B, each thread loads whole 16-byte chunks of
// its K rows straight from global (ld.global.nc, L1 no-allocate, L2
// evict-first) into A-fragment registers, and the query B fragments use the
// same chunk layout -- no shared memory, no ldmatrix, full 128-bit coalesced
// loads.  Tensor cores only free the FP32 pipe; HBM is the roofline.
#include "common.cuh"
#include "kernels.h"

namespace svl {

namespace {

template <int D>
struct RowLoad {
    static constexpr int NCH = D / 32;  // 16-byte chunks per thread per row
};

// merge (m, l) pairs in base 2; -inf-safe
SVL_DEV void lse_merge(float& m, float& l, float m2, float l2) {
    float M = fmaxf(m, m2);
    if (M == -INFINITY) return;
    l = l * fast_exp2(m - M) + l2 * fast_exp2(m2 - M);
    m = M;
}

template <int D, int NT>
__global__ void __launch_bounds__(kScoreThreads, 1) score_kernel(const ScoreParams p) {
    constexpr int NCH = RowLoad<D>::NCH;
    constexpr int NWARPS = kScoreThreads / 32;
    __shared__ float2 wpart[NWARPS][NT * 8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, t = lane & 3;
    const int n_items = p.B * p.Hkv * p.C;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int u = item / p.C, c = item % p.C;
    const int b = u / p.Hkv, G = u % p.Hkv;

    int L = p.seq_len[b];
    if (L < p.vb + p.nv + p.q_rows_in_view || L > p.capacity) {
        if (threadIdx.x == 0 && c == 0) raise_flag(p.flags, 4u /*SVL_DEVFLAG_SPAN*/);
        L = min(max(L, p.vb + p.nv + p.q_rows_in_view), p.capacity);
    }

    // ---- work list: visual rows of this chunk, then this chunk's share of text rows
    const int v0 = c * p.rows_per_chunk;
    const int v1 = min(p.nv, v0 + p.rows_per_chunk);
    const int nvis = max(0, v1 - v0);
    int t0 = 0, t1 = 0;
    if (p.use_text) {
        const int T = p.vb + (L - p.vb - p.nv);
        t0 = (int)((int64_t)c * T / p.C);
        t1 = (int)((int64_t)(c + 1) * T / p.C);
    }
    const int nwork = nvis + (t1 - t0);
    const int ntiles = (nwork + 15) >> 4;

    const uint16_t* Kb = p.K + (int64_t)b * p.sb + (int64_t)G * p.sh;
    const uint64_t pol = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();

    // ---- query B fragments (chunk layout identical to the K rows)
    uint4 bq[NT][NCH];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
        const int col = nt * 8 + gid;
#pragma unroll
        for (int i = 0; i < NCH; ++i) bq[nt][i] = make_uint4(0, 0, 0, 0);
        if (col < p.NC) {
            const int r = col / p.g, h = G * p.g + col % p.g;
            const uint4* qr = reinterpret_cast<const uint4*>(
                p.q + (((int64_t)b * p.n_q + r) * p.H + h) * D);
#pragma unroll
            for (int i = 0; i < NCH; ++i) bq[nt][i] = qr[t + 4 * i];
        }
    }

    // running (max, sum) for the 2*NT columns this thread owns
    float rm[NT][2], rl[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) rm[nt][0] = rm[nt][1] = -INFINITY, rl[nt][0] = rl[nt][1] = 0.f;

    auto row_of = [&](int w, bool& vis, int& j) -> int {
        if (w < nvis) {
            vis = true;
            j = v0 + w;
            return p.vb + j;
        }
        vis = false;
        j = -1;
        const int tt = t0 + (w - nvis);
        return tt < p.vb ? tt : tt + p.nv;
    };

    auto load_tile = [&](int tile, uint4 (&ra)[NCH], uint4 (&rb)[NCH]) {
        const int wa = tile * 16 + gid, wb = wa + 8;
        bool va, vb_;
        int ja, jb;
        if (wa < nwork) {
            const int row = row_of(wa, va, ja);
            const uint4* src = reinterpret_cast<const uint4*>(Kb + (int64_t)row * p.st);
#pragma unroll
            for (int i = 0; i < NCH; ++i) ra[i] = ldg_stream(src + t + 4 * i, pol);
        } else {
#pragma unroll
            for (int i = 0; i < NCH; ++i) ra[i] = make_uint4(0, 0, 0, 0);
        }
        if (wb < nwork) {
            const int row = row_of(wb, vb_, jb);
            const uint4* src = reinterpret_cast<const uint4*>(Kb + (int64_t)row * p.st);
#pragma unroll
            for (int i = 0; i < NCH; ++i) rb[i] = ldg_stream(src + t + 4 * i, pol);
        } else {
#pragma unroll
            for (int i = 0; i < NCH; ++i) rb[i] = make_uint4(0, 0, 0, 0);
        }
    };

    float* logits_u = p.logits + (int64_t)u * p.nv * p.NCP;

    auto compute_tile = [&](int tile, const uint4 (&ra)[NCH], const uint4 (&rb)[NCH]) {
        float acc[NT][4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
        for (int s = 0; s < D / 16; ++s) {
            const int i = s >> 1;
            uint32_t a[4];
            if ((s & 1) == 0) {
                a[0] = ra[i].x; a[1] = rb[i].x; a[2] = ra[i].y; a[3] = rb[i].y;
            } else {
                a[0] = ra[i].z; a[1] = rb[i].z; a[2] = ra[i].w; a[3] = rb[i].w;
            }
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const uint32_t b0 = (s & 1) ? bq[nt][i].z : bq[nt][i].x;
                const uint32_t b1 = (s & 1) ? bq[nt][i].w : bq[nt][i].y;
                mma_bf16_16816(acc[nt], a, b0, b1);
            }
        }
        // epilogue: scale, mask, store visual logits, fold into running LSE
        const int wa = tile * 16 + gid, wb = wa + 8;
        bool visa = false, visb = false;
        int ja = -1, jb = -1, rowa = -1, rowb = -1;
        if (wa < nwork) rowa = row_of(wa, visa, ja);
        if (wb < nwork) rowb = row_of(wb, visb, jb);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
            float v[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) v[e] = acc[nt][e] * p.scale2;
            if (visa) stg_hint_f2(logits_u + (int64_t)ja * p.NCP + nt * 8 + 2 * t, v[0], v[1], pol_keep);
            if (visb) stg_hint_f2(logits_u + (int64_t)jb * p.NCP + nt * 8 + 2 * t, v[2], v[3], pol_keep);
            if (p.need_partials) {
#pragma unroll
                for (int e2 = 0; e2 < 2; ++e2) {
                    const int col = nt * 8 + 2 * t + e2;
                    const int r = col / p.g;
                    const int lim = L - p.n_q + r;  // causal limit for query row r
                    float x0 = (rowa >= 0 && rowa <= lim) ? v[e2] : -INFINITY;
                    float x1 = (rowb >= 0 && rowb <= lim) ? v[2 + e2] : -INFINITY;
                    const float mx = fmaxf(x0, x1);
                    if (mx != -INFINITY) {
                        const float M = fmaxf(rm[nt][e2], mx);
                        rl[nt][e2] = rl[nt][e2] * fast_exp2(rm[nt][e2] - M) + fast_exp2(x0 - M) +
                                     fast_exp2(x1 - M);
                        rm[nt][e2] = M;
                    }
                }
            }
        }
    };

    // ---- main loop: register double buffering, one tile in flight per warp
    int tile = warp;
    uint4 ca[NCH], cb[NCH], na[NCH], nb[NCH];
    if (tile < ntiles) load_tile(tile, ca, cb);
    for (; tile < ntiles; tile += NWARPS) {
        const int nxt = tile + NWARPS;
        if (nxt < ntiles) load_tile(nxt, na, nb);
        compute_tile(tile, ca, cb);
#pragma unroll
        for (int i = 0; i < NCH; ++i) ca[i] = na[i], cb[i] = nb[i];
    }

    if (!p.need_partials) continue;

    // ---- chunk partials: reduce over the 8 row-groups (lanes with equal t)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e2 = 0; e2 < 2; ++e2) {
#pragma unroll
            for (int off = 4; off < 32; off <<= 1) {
                const float m2 = __shfl_xor_sync(0xffffffffu, rm[nt][e2], off);
                const float l2 = __shfl_xor_sync(0xffffffffu, rl[nt][e2], off);
                lse_merge(rm[nt][e2], rl[nt][e2], m2, l2);
            }
        }
    if (gid == 0) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e2 = 0; e2 < 2; ++e2)
                wpart[warp][nt * 8 + 2 * t + e2] = make_float2(rm[nt][e2], rl[nt][e2]);
    }
    cta_sync();
    if (threadIdx.x < NT * 8) {
        float m = -INFINITY, l = 0.f;
        for (int w = 0; w < NWARPS; ++w) lse_merge(m, l, wpart[w][threadIdx.x].x, wpart[w][threadIdx.x].y);
        p.part[((int64_t)u * p.C + c) * p.NCP + threadIdx.x] = make_float2(m, l);
    }
    cta_sync();  // wpart is reused by the next item
    }  // item loop
}

template <int D, int NT>
cudaError_t launch_score_t(const ScoreParams& p, cudaStream_t s) {
    static bool attr_done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_done[dev]) {
        attr_done[dev] = true;  // default carveout: this kernel keeps L1 for its register spills
    }
    const int n_items = p.B * p.Hkv * p.C;
    const int grid = n_items < device_sm_count() ? n_items : device_sm_count();
    score_kernel<D, NT><<<grid, kScoreThreads, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_score(const ScoreParams& p, int d, int NT, cudaStream_t s) {
    if (d == 128) {
        switch (NT) {
            case 1: return launch_score_t<128, 1>(p, s);
            case 2: return launch_score_t<128, 2>(p, s);
            case 3: return launch_score_t<128, 3>(p, s);
            case 4: return launch_score_t<128, 4>(p, s);
        }
    } else if (d == 64) {
        switch (NT) {
            case 1: return launch_score_t<64, 1>(p, s);
            case 2: return launch_score_t<64, 2>(p, s);
            case 3: return launch_score_t<64, 3>(p, s);
            case 4: return launch_score_t<64, 4>(p, s);
        }
    }
    return cudaErrorInvalidValue;
}

}  // namespace svl
