// select_core.cuh -- cluster-wide deterministic top-k over uint32 keys.
//
// Shared by the stand-alone selection kernel (select.cu: svl_retrieve phase 2,
// svl_prefill_prune) and the fused fresh-step kernel (fused.cu).
//
// Semantics (reading A8): select the k largest keys of a
// unit's n keys, ties to the lower index.  The keys of one unit are spread
// over the CS CTAs of a thread-block cluster, CTA r owning the index slice
// [r*slice, (r+1)*slice), thread tid the contiguous run [tid*E, tid*E + E).
//
// Algorithm (4 cluster barriers in the common case):
//   1. 12-bit digit histogram (key bits 31..20) per CTA; cluster barrier;
//      CTA r reduces bins [r*4096/CS, ...) over the cluster through DSMEM;
//      cluster barrier; every CTA locates the bin b* that holds the k-th
//      largest key (fixed-order scans -> identical on all CTAs).
//   2. The keys inside b* (typically a few hundred) go to rank 0's candidate
//      buffer over DSMEM; cluster barrier.
//   3. Rank 0 finds the exact threshold key T among the candidates (local
//      4 x 8-bit radix select), the tie cut (lowest indices win) by a second
//      local select on the indices, and each CTA's tie quota and output
//      offset; it writes them into every CTA's shared memory; cluster barrier.
//   Fallback (b* holds more than kCandMax keys, e.g. massive exact ties): two
//   more cluster-wide radix passes over bits 19..0 and a cluster prefix of the
//   per-CTA tie counts -- slower, identical result.
// Result per CTA: (T, quota, offset): the element at local position e is
// selected iff key > T, or key == T and it is among this CTA's first `quota`
// ties in index order; its output slot is offset + #selected before it.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace svl {

namespace cg = cooperative_groups;

constexpr int kTopkBins = 4096;
constexpr int kCandMax = 2048;

struct TopkSmem {
    uint32_t hist[2][kTopkBins];  // local digit histograms (double-buffered by pass)
    uint32_t own[2][kTopkBins];   // owner sums (bins of this CTA's range)
    uint32_t own_total[2];
    uint32_t warp_sums[32];
    uint32_t bcast[4];
    uint32_t cta_cnt[2];          // fallback: this CTA's (#gt, #eq)
    uint32_t ot_local[16];        // owner totals copied from the cluster
    uint32_t cand_count;          // rank 0: number of candidates appended
    uint32_t cta_above[16];       // rank 0: per-CTA #keys above the candidate bin
    uint32_t cta_sel[16];         // rank 0: per-CTA #selected candidates
    uint32_t cta_quota[16];       // rank 0: per-CTA #taken ties
    uint32_t lsel_hist[256];      // rank 0: local radix
    uint32_t lsel_res[3];
    uint32_t pub[4];              // published result: T, quota, offset
    uint2 cand[kCandMax];         // rank 0: (key, unit index)
    uint32_t aux[kCandMax];       // rank 0: tie values ~index (0 for non-ties)
};

// Exclusive block scan (sum) over all NTH threads of the CTA.
template <int NTH>
SVL_DEV uint32_t block_scan_excl(uint32_t v, uint32_t* warp_sums, uint32_t& total) {
    constexpr int NW = NTH / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    cta_sync();
    if (warp == 0) {
        uint32_t w = (lane < NW) ? warp_sums[lane] : 0u;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, off);
            if (lane >= off) w += y;
        }
        if (lane < NW) warp_sums[lane] = w;
    }
    cta_sync();
    const uint32_t before = (warp > 0 ? warp_sums[warp - 1] : 0u) + (x - v);
    total = warp_sums[NW - 1];
    cta_sync();
    return before;
}

// One warp: among `nbins` bin counts (cnt(i), bins ascending), find the bin
// holding the `need`-th largest element scanning from the top bin down.
// Returns the bin and the count strictly above it (warp-uniform).
template <typename F>
SVL_DEV void warp_find_from_top(int nbins, uint32_t need, F cnt, int& bin_out, uint32_t& above_out) {
    const int lane = threadIdx.x & 31;
    const int per = (nbins + 31) / 32;
    uint32_t grp = 0u;
    for (int i = 0; i < per; ++i) {
        const int b = lane * per + i;
        if (b < nbins) grp += cnt(b);
    }
    uint32_t suf = grp;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_down_sync(0xffffffffu, suf, off);
        if (lane + off < 32) suf += y;
    }
    const unsigned ball = __ballot_sync(0xffffffffu, suf >= need);
    const int lstar = ball ? 31 - __clz(ball) : 0;
    int bstar = 0;
    uint32_t above = 0u;
    if (lane == lstar) {
        above = suf - grp;
        bstar = lane * per;
        for (int i = per - 1; i >= 0; --i) {
            const int b = lane * per + i;
            if (b >= nbins) continue;
            const uint32_t c = cnt(b);
            if (above + c >= need) {
                bstar = b;
                break;
            }
            above += c;
        }
    }
    bin_out = __shfl_sync(0xffffffffu, bstar, lstar);
    above_out = __shfl_sync(0xffffffffu, above, lstar);
}

// Whole CTA: the `need`-th largest of vals[0..m) (1 <= need <= m), 4 passes
// of 8-bit digits over shared memory.  Returns T and #{values > T}.
template <int NTH>
SVL_DEV void local_kth_largest(TopkSmem& s, const uint32_t* vals, int vstride, int m, uint32_t need,
                               uint32_t& T, uint32_t& n_above) {
    const int tid = threadIdx.x;
    uint32_t P = 0u, M = 0u, krem = need, above_acc = 0u;
    for (int pass = 0; pass < 4; ++pass) {
        const int sh = 24 - 8 * pass;
        for (int i = tid; i < 256; i += NTH) s.lsel_hist[i] = 0u;
        cta_sync();
        for (int i = tid; i < m; i += NTH) {
            const uint32_t v = vals[i * vstride];
            if ((v & M) == P) atomicAdd(&s.lsel_hist[(v >> sh) & 255u], 1u);
        }
        cta_sync();
        if (tid < 32) {
            int b;
            uint32_t ab;
            warp_find_from_top(256, krem, [&](int i) { return s.lsel_hist[i]; }, b, ab);
            if (tid == 0) {
                s.lsel_res[0] = P | ((uint32_t)b << sh);
                s.lsel_res[1] = krem - ab;
                s.lsel_res[2] = above_acc + ab;
            }
        }
        cta_sync();
        P = s.lsel_res[0];
        M |= 255u << sh;
        krem = s.lsel_res[1];
        above_acc = s.lsel_res[2];
        cta_sync();
    }
    T = P;
    n_above = above_acc;
}

// One cluster-wide radix pass over digit (key >> sh) & (nbins-1) of the keys
// matching prefix (P, M).  Updates P, M, krem; returns the count in the bin.
template <int NTH, int EMAX>
SVL_DEV uint32_t cluster_radix_pass(cg::cluster_group& cl, TopkSmem& s, int buf,
                                    const uint32_t (&key)[EMAX], int nmine, int sh, int nbins,
                                    uint32_t& P, uint32_t& M, uint32_t& krem) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int CS = (int)cl.num_blocks();
    const int rank = (int)cl.block_rank();
    const uint32_t dmask = (uint32_t)(nbins - 1);
    for (int i = tid; i < nbins; i += NTH) s.hist[buf][i] = 0u;
    cta_sync();
#pragma unroll
    for (int e = 0; e < EMAX; ++e)
        if (e < nmine && (key[e] & M) == P) atomicAdd(&s.hist[buf][(key[e] >> sh) & dmask], 1u);
    cluster_sync(cl);
    const int bpo = nbins / CS;
    {
        // owner reduction: all CS remote loads of a bin are issued before use
        uint32_t part = 0u;
        for (int i = tid; i < bpo; i += NTH) {
            uint32_t v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q)
                v[q] = (q < CS) ? cl.map_shared_rank(&s.hist[buf][0], q)[rank * bpo + i] : 0u;
            uint32_t acc = 0u;
#pragma unroll
            for (int q = 0; q < 16; ++q) acc += v[q];
            s.own[buf][i] = acc;
            part += acc;
        }
        uint32_t tot;
        (void)block_scan_excl<NTH>(part, s.warp_sums, tot);
        if (tid == 0) s.own_total[buf] = tot;
    }
    cluster_sync(cl);
    // owner totals -> local, find the owner o*, then copy o*'s bins locally
    if (tid < CS) s.ot_local[tid] = *cl.map_shared_rank(&s.own_total[buf], tid);
    cta_sync();
    if (warp == 0) {
        int ostar;
        uint32_t above_o;
        warp_find_from_top(CS, krem, [&](int q) { return s.ot_local[q]; }, ostar, above_o);
        if (lane == 0) {
            s.bcast[0] = (uint32_t)ostar;
            s.bcast[1] = above_o;
        }
    }
    cta_sync();
    const int ostar = (int)s.bcast[0];
    const uint32_t above_o = s.bcast[1];
    uint32_t* lown = &s.hist[buf ^ 1][0];  // scratch copy of o*'s bins (other buffer is idle)
    {
        const uint32_t* rown = cl.map_shared_rank(&s.own[buf][0], ostar);
        for (int i = tid; i < bpo; i += NTH) lown[i] = rown[i];
    }
    cta_sync();
    if (warp == 0) {
        int bl;
        uint32_t above_b;
        warp_find_from_top(bpo, krem - above_o, [&](int i) { return lown[i]; }, bl, above_b);
        if (lane == 0) {
            s.bcast[0] = (uint32_t)(ostar * bpo + bl);
            s.bcast[1] = krem - above_o - above_b;
            s.bcast[2] = lown[bl];
        }
    }
    cta_sync();
    P |= s.bcast[0] << sh;
    M |= dmask << sh;
    krem = s.bcast[1];
    const uint32_t cnt = s.bcast[2];
    cta_sync();
    return cnt;
}

struct TopkResult {
    uint32_t T;       // threshold key
    uint32_t quota;   // ties (key == T) this CTA takes, lowest local index first
    uint32_t offset;  // output slot of this CTA's first selected element
};

// All NTH threads of every CTA of the cluster must call this with identical
// (n, k, slice).  key[e], e < nmine, are this thread's keys at unit index
// j0 + tid*E + e, where j0 = rank*slice is the CTA's first unit index.
template <int NTH, int EMAX>
SVL_DEV TopkResult cluster_topk(cg::cluster_group& cl, TopkSmem& s, const uint32_t (&key)[EMAX],
                                int nmine, int E, int j0, int slice, int n, int k) {
    const int tid = threadIdx.x;
    const int CS = (int)cl.num_blocks();
    const int rank = (int)cl.block_rank();
    TopkResult res;
    if (k <= 0) {
        res.T = 0xffffffffu; res.quota = 0u; res.offset = 0u;
        return res;
    }
    if (k >= n) {  // everything: all keys are >= T = 0 and every tie is taken
        res.T = 0u; res.quota = 0xffffffffu; res.offset = (uint32_t)j0;
        return res;
    }
    if (tid == 0) s.cand_count = 0u;  // ordered before any remote append by the first cl.sync

    uint32_t P = 0u, M = 0u, krem = (uint32_t)k;
    const uint32_t cnt_bin = cluster_radix_pass<NTH>(cl, s, 0, key, nmine, 20, kTopkBins, P, M, krem);
    const uint32_t bstar = P >> 20;

    if (cnt_bin <= (uint32_t)kCandMax) {
        // ---------------- common path: candidates of bin b* -> rank 0
        uint32_t n_above = 0u, n_cand = 0u;
#pragma unroll
        for (int e = 0; e < EMAX; ++e)
            if (e < nmine) {
                const uint32_t dg = key[e] >> 20;
                n_above += dg > bstar;
                n_cand += dg == bstar;
            }
        uint32_t cta_above;
        (void)block_scan_excl<NTH>(n_above, s.warp_sums, cta_above);
        TopkSmem* r0 = cl.map_shared_rank(&s, 0);
        if (tid == 0) r0->cta_above[rank] = cta_above;
        if (n_cand) {
            uint32_t pos = atomicAdd(&r0->cand_count, n_cand);
#pragma unroll
            for (int e = 0; e < EMAX; ++e)
                if (e < nmine && (key[e] >> 20) == bstar)
                    r0->cand[pos++] = make_uint2(key[e], (uint32_t)(j0 + tid * E + e));
        }
        cluster_sync(cl);
        if (rank == 0) {
            const int m = (int)s.cand_count;
            uint32_t T, n_gt;
            local_kth_largest<NTH>(s, &s.cand[0].x, 2, m, krem, T, n_gt);
            const uint32_t need_eq = krem - n_gt;  // >= 1 ties to take, lowest index first
            for (int i = tid; i < m; i += NTH) s.aux[i] = (s.cand[i].x == T) ? ~s.cand[i].y : 0u;
            if (tid < 16) s.cta_sel[tid] = s.cta_quota[tid] = 0u;
            cta_sync();
            uint32_t NI, unused;
            local_kth_largest<NTH>(s, s.aux, 1, m, need_eq, NI, unused);
            const uint32_t tie_max = ~NI;  // largest index among the taken ties
            for (int i = tid; i < m; i += NTH) {
                const uint2 c = s.cand[i];
                const uint32_t r = c.y / (uint32_t)slice;
                const bool tie_taken = (c.x == T) && (c.y <= tie_max);
                if (c.x > T || tie_taken) atomicAdd(&s.cta_sel[r], 1u);
                if (tie_taken) atomicAdd(&s.cta_quota[r], 1u);
            }
            cta_sync();
            if (tid < CS) {
                uint32_t off = 0u;
                for (int q = 0; q < tid; ++q) off += s.cta_above[q] + s.cta_sel[q];
                TopkSmem* rq = cl.map_shared_rank(&s, tid);
                rq->pub[0] = T;
                rq->pub[1] = s.cta_quota[tid];
                rq->pub[2] = off;
            }
        }
        cluster_sync(cl);
        res.T = s.pub[0];
        res.quota = s.pub[1];
        res.offset = s.pub[2];
        return res;
    }

    // ---------------- fallback: full radix on bits 19..0, then a tie prefix
    (void)cluster_radix_pass<NTH>(cl, s, 1, key, nmine, 10, 1024, P, M, krem);
    (void)cluster_radix_pass<NTH>(cl, s, 0, key, nmine, 0, 1024, P, M, krem);
    const uint32_t T = P;  // the exact k-th largest key; krem ties with key == T are taken
    uint32_t gt = 0u, eq = 0u;
#pragma unroll
    for (int e = 0; e < EMAX; ++e)
        if (e < nmine) {
            gt += key[e] > T;
            eq += key[e] == T;
        }
    uint32_t tot;
    (void)block_scan_excl<NTH>(gt | (eq << 16), s.warp_sums, tot);
    if (tid == 0) {
        s.cta_cnt[0] = tot & 0xffffu;
        s.cta_cnt[1] = tot >> 16;
    }
    cluster_sync(cl);
    uint32_t eq_acc = 0u, sel_before = 0u;
    for (int q = 0; q < rank; ++q) {
        const uint32_t* c = cl.map_shared_rank(&s.cta_cnt[0], q);
        const uint32_t qg = c[0], qe = c[1];
        sel_before += qg + ((krem > eq_acc) ? min(krem - eq_acc, qe) : 0u);
        eq_acc += qe;
    }
    res.T = T;
    res.quota = (krem > eq_acc) ? krem - eq_acc : 0u;
    res.offset = sel_before;
    cluster_sync(cl);  // peers finished reading cta_cnt
    return res;
}

// Compaction helper: calls emit(e, slot) for each selected key of this
// thread (index order), given the TopkResult.  All NTH threads must call it.
template <int NTH, int EMAX, typename Emit>
SVL_DEV uint32_t topk_emit(TopkSmem& s, const TopkResult& r, const uint32_t (&key)[EMAX], int nmine,
                           Emit emit) {
    uint32_t gt = 0u, eq = 0u;
#pragma unroll
    for (int e = 0; e < EMAX; ++e)
        if (e < nmine) {
            gt += key[e] > r.T;
            eq += key[e] == r.T;
        }
    uint32_t tot;
    const uint32_t excl = block_scan_excl<NTH>(gt | (eq << 16), s.warp_sums, tot);
    uint32_t gt_run = excl & 0xffffu, eq_run = excl >> 16;
#pragma unroll
    for (int e = 0; e < EMAX; ++e)
        if (e < nmine) {
            const bool isgt = key[e] > r.T, iseq = key[e] == r.T;
            if (isgt || (iseq && eq_run < r.quota)) emit(e, r.offset + gt_run + min(eq_run, r.quota));
            gt_run += isgt;
            eq_run += iseq;
        }
    return (tot & 0xffffu) + min(tot >> 16, r.quota);  // selected in this CTA
}

}  // namespace svl
