// select_push.cuh -- cluster top-k with push-style all-gathers.
//
// Semantics (reading A8): the k largest keys of a unit whose
// n keys are spread over the CS CTAs of a cluster (CTA r owns unit indices
// [r*slice, (r+1)*slice); its keys sit in shared memory, thread tid handles
// the run [tid*E, tid*E+E)), ties to the lower index.
//
// Built for latency: every exchange is a DSMEM *push* (st.shared::cluster into
// every peer) followed by ONE cluster barrier, after which every CTA decides
// locally and identically -- no owner CTA, no remote reads on the critical
// path.  Cold code is kept small (keys and per-key state live in shared
// memory, loops are not unrolled, helpers are not inlined): this code runs
// once per launch, so instruction-cache misses -- not arithmetic -- bound it.
//
//   relevance mode (scores in [0, 32]):
//     round 1  256-bin histogram of a value-adaptive digit (float exponent
//              101..132 x 3 mantissa bits: 1/8-binade bins; scores < 2^-26
//              share bin 0), all-gathered; every CTA finds the bin b* of the
//              k-th key;
//     round 2  the keys of b* (~1% of the unit) are all-gathered in index
//              order; each CTA finds the exact threshold among them (local
//              4 x 8-bit radix) and the lowest-index ties to keep.
//   generic mode (any fp32 key), or b* = catch-all / > kPushCand keys:
//     four exact 8-bit radix rounds on the full key; what stays active are
//     exact ties of the threshold, kept lowest index first from the gathered
//     per-CTA tie counts.
// Output: state[i] == 2 for selected keys, and the CTA's first output slot.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace svl {

namespace cg = cooperative_groups;

constexpr int kPushCand = 1024;

enum : uint8_t { kKeyOut = 0, kKeyActive = 1, kKeySel = 2 };

struct PushTopkSmem {
    uint32_t allhist[2][16][256];  // gathered histograms (double-buffered by round)
    uint2 cand[kPushCand];         // gathered candidates (key, unit index), index order
    uint32_t hist[256];            // local histogram / local-radix scratch
    uint32_t tot[256];             // summed histogram
    uint32_t warp_sums[32];
    uint32_t cand_sel[16];         // per-CTA selected candidates
    uint32_t above_q[16];          // per-CTA keys above the threshold bins
    uint32_t bcast[8];
    uint8_t cand_flag[kPushCand];  // candidate selected
};

// Exclusive block scan (sum) over all NTH threads of the CTA.
template <int NTH>
__device__ __noinline__ uint32_t block_scan_excl(uint32_t v, uint32_t* warp_sums, uint32_t* total) {
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
    *total = warp_sums[NW - 1];
    cta_sync();
    return before;
}

// One warp, 256 bins ascending in shared memory: the bin holding the
// `need`-th largest element (scanning from the top) and the count above it.
static __device__ __noinline__ void warp_find256(const uint32_t* bins, uint32_t need, uint32_t* out) {
    const int lane = threadIdx.x & 31;
    uint32_t c[8];
    uint32_t grp = 0u;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        c[i] = bins[lane * 8 + i];
        grp += c[i];
    }
    uint32_t suf = grp;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_down_sync(0xffffffffu, suf, off);
        if (lane + off < 32) suf += y;
    }
    const unsigned ball = __ballot_sync(0xffffffffu, suf >= need);
    const int lstar = ball ? 31 - __clz(ball) : 0;
    if (lane == lstar) {
        uint32_t above = suf - grp;
        int b = lane * 8;
        for (int i = 7; i >= 0; --i) {
            if (above + c[i] >= need) {
                b = lane * 8 + i;
                break;
            }
            above += c[i];
        }
        out[0] = (uint32_t)b;
        out[1] = above;
    }
}

SVL_DEV int push_digit(uint32_t key, int mode, int sh) {
    if (mode == 0) {  // value-adaptive relevance digit (keys of non-negative floats have bit 31 set)
        const int e = (int)((key >> 23) & 0xffu);
        const int b = (e - 101) * 8 + (int)((key >> 20) & 7u);
        return (key & 0x80000000u) ? min(max(b, 0), 255) : 0;
    }
    return (int)((key >> sh) & 255u);
}

// One histogram round over the active keys; returns the threshold bin and
// updates krem, the per-CTA "above" counts and the key states.
template <int NTH>
__device__ __noinline__ int push_round(cg::cluster_group& cl, PushTopkSmem& s, int buf, const uint32_t* keys,
                                       uint8_t* state, int E, int nmine, int mode, int sh, uint32_t* krem,
                                       uint64_t* tr = nullptr) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int CS = (int)cl.num_blocks(), rank = (int)cl.block_rank();
    for (int i = tid; i < 256; i += NTH) s.hist[i] = 0u;
    cta_sync();
#pragma unroll 1
    for (int e = 0; e < E; ++e) {  // E is CTA-uniform: every lane reaches the match
        const int i = tid * E + e;
        const bool on = e < nmine && state[i] == kKeyActive;
        const int bin = on ? push_digit(keys[i], mode, sh) : -1;
        const unsigned peers = __match_any_sync(0xffffffffu, bin);  // warp-aggregated atomics
        if (on && lane == __ffs(peers) - 1) atomicAdd(&s.hist[bin], (uint32_t)__popc(peers));
    }
    cta_sync();
    for (int i = tid; i < CS * 64; i += NTH) {
        const int q = i >> 6, c = i & 63;
        uint4* dst = reinterpret_cast<uint4*>(cl.map_shared_rank(&s.allhist[buf][rank][0], q));
        dst[c] = reinterpret_cast<const uint4*>(s.hist)[c];
    }
    if (tr && tid == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        tr[0] = t;
    }
    cluster_sync(cl);
    if (tr && tid == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        tr[1] = t;
    }
    for (int i = tid; i < 256; i += NTH) {
        uint32_t acc = 0u;
        for (int q = 0; q < CS; ++q) acc += s.allhist[buf][q][i];
        s.tot[i] = acc;
    }
    cta_sync();
    if (warp == 0) warp_find256(s.tot, *krem, s.bcast);
    cta_sync();
    if (tr && tid == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        tr[2] = t;
    }
    const int b = (int)s.bcast[0];
    *krem -= s.bcast[1];
    for (int q = warp; q < CS; q += NTH / 32) {  // per-CTA counts above the bin
        uint32_t a = 0u;
        for (int i = b + 1 + lane; i < 256; i += 32) a += s.allhist[buf][q][i];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
        if (lane == 0) s.above_q[q] += a;
    }
#pragma unroll 1
    for (int e = 0; e < nmine; ++e) {
        const int i = tid * E + e;
        if (state[i] != kKeyActive) continue;
        const int d = push_digit(keys[i], mode, sh);
        state[i] = (d > b) ? kKeySel : (d == b ? kKeyActive : kKeyOut);
    }
    cta_sync();
    return b;
}

// Whole CTA: the `need`-th largest key among s.cand[0..m).x (1 <= need <= m).
template <int NTH>
__device__ __noinline__ void block_kth_largest(PushTopkSmem& s, int m, uint32_t need, uint32_t* T,
                                               uint32_t* n_above) {
    const int tid = threadIdx.x;
    uint32_t P = 0u, M = 0u, krem = need, above_acc = 0u;
#pragma unroll 1
    for (int pass = 0; pass < 4; ++pass) {
        const int sh = 24 - 8 * pass;
        for (int i = tid; i < 256; i += NTH) s.hist[i] = 0u;
        cta_sync();
        for (int i = tid; i < m; i += NTH) {
            const uint32_t v = s.cand[i].x;
            if ((v & M) == P) atomicAdd(&s.hist[(v >> sh) & 255u], 1u);
        }
        cta_sync();
        if (tid < 32) warp_find256(s.hist, krem, s.bcast + 4);
        cta_sync();
        P |= s.bcast[4] << sh;
        M |= 255u << sh;
        krem -= s.bcast[5];
        above_acc += s.bcast[5];
        cta_sync();
    }
    *T = P;
    *n_above = above_acc;
}

// keys[0..nloc): this CTA's keys (unit indices j0 + i, j0 = rank*slice);
// state[0..nloc) is written (kKeySel = selected).  relevance: use the
// value-adaptive first round (keys of scores in [0, 32]).  Returns the CTA's
// selected count and its first output slot.
SVL_DEV void stamp(uint64_t* tr, int i) {
    if (tr && threadIdx.x == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        tr[i] = t;
    }
}

template <int NTH>
__device__ __noinline__ uint32_t cluster_topk_push(cg::cluster_group& cl, PushTopkSmem& s, const uint32_t* keys,
                                                   uint8_t* state, int nloc, int j0, int slice, int n, int k,
                                                   bool relevance, uint32_t* cta_offset,
                                                   uint64_t* tr = nullptr) {
    const int tid = threadIdx.x;
    const int CS = (int)cl.num_blocks(), rank = (int)cl.block_rank();
    const int E = (nloc + NTH - 1) / NTH;
    const int nmine = max(0, min(E, nloc - tid * E));
    const uint8_t init = (k >= n) ? kKeySel : (k <= 0 ? kKeyOut : kKeyActive);
    for (int i = tid; i < nloc; i += NTH) state[i] = init;
    uint32_t tot;
    if (k <= 0 || k >= n) {
        cta_sync();
        *cta_offset = (k <= 0) ? 0u : (uint32_t)j0;
        return (k <= 0) ? 0u : (uint32_t)nloc;
    }
    if (tid < 16) s.above_q[tid] = 0u;
    if (tid < 16) s.cand_sel[tid] = 0u;
    cta_sync();
    uint32_t krem = (uint32_t)k;
    int buf = 0;
    int blast = push_round<NTH>(cl, s, buf, keys, state, E, nmine, relevance ? 0 : 1, 24, &krem, tr);
    stamp(tr, 3);
    bool exact_ties = !relevance;
    if (relevance && (blast == 0 || s.tot[blast] > (uint32_t)kPushCand)) exact_ties = true;
    if (exact_ties) {
        // continue (or start) an exact radix over the full key; in generic mode
        // round 1 already handled bits 31..24
#pragma unroll 1
        for (int pass = relevance ? 0 : 1; pass < 4; ++pass) {
            buf ^= 1;
            blast = push_round<NTH>(cl, s, buf, keys, state, E, nmine, 1, 24 - 8 * pass, &krem);
        }
    }
    const uint32_t cnt = s.tot[blast];
    // candidates = the still-active keys, in index order across the cluster
    uint32_t my_cand = 0u;
    for (int e = 0; e < nmine; ++e) my_cand += state[tid * E + e] == kKeyActive;
    uint32_t pos = block_scan_excl<NTH>(my_cand, s.warp_sums, &tot);
    for (int q = 0; q < rank; ++q) pos += s.allhist[buf][q][blast];
    if (exact_ties) {
        // exact ties only: the first krem in index order are taken
        for (int e = 0; e < nmine; ++e) {
            const int i = tid * E + e;
            if (state[i] != kKeyActive) continue;
            state[i] = (pos < krem) ? kKeySel : kKeyOut;
            ++pos;
        }
        if (tid < CS) {
            uint32_t b0 = 0u;
            for (int q = 0; q < tid; ++q) b0 += s.allhist[buf][q][blast];
            const uint32_t cq = s.allhist[buf][tid][blast];
            s.cand_sel[tid] = (krem > b0) ? min(krem - b0, cq) : 0u;
        }
    } else {
        const uint32_t pos0 = pos;
        for (int e = 0; e < nmine; ++e) {
            const int i = tid * E + e;
            if (state[i] != kKeyActive) continue;
            const uint2 c = make_uint2(keys[i], (uint32_t)(j0 + i));
            for (int q = 0; q < CS; ++q) cl.map_shared_rank(&s.cand[0], q)[pos] = c;
            ++pos;
        }
        cluster_sync(cl);
        stamp(tr, 4);
        const int m = (int)cnt;
        uint32_t T, n_gt;
        block_kth_largest<NTH>(s, m, krem, &T, &n_gt);
        stamp(tr, 5);
        const uint32_t need_eq = krem - n_gt;  // ties of T to keep: the first need_eq in index order
        const int per = (m + NTH - 1) / NTH;
        const int i0 = min(m, tid * per), i1 = min(m, i0 + per);
        uint32_t nt = 0u;
        for (int i = i0; i < i1; ++i) nt += s.cand[i].x == T;
        uint32_t tie_rank = block_scan_excl<NTH>(nt, s.warp_sums, &tot);
        for (int i = i0; i < i1; ++i) {
            const uint2 ci = s.cand[i];
            bool take = ci.x > T;
            if (ci.x == T) take = (tie_rank++ < need_eq);
            s.cand_flag[i] = take;
            if (take) atomicAdd(&s.cand_sel[ci.y / (uint32_t)slice], 1u);
        }
        cta_sync();
        pos = pos0;
        for (int e = 0; e < nmine; ++e) {
            const int i = tid * E + e;
            if (state[i] != kKeyActive) continue;
            state[i] = s.cand_flag[pos] ? kKeySel : kKeyOut;
            ++pos;
        }
    }
    cta_sync();
    stamp(tr, 6);
    if (tid == 0) {
        uint32_t off = 0u, mine = 0u;
        for (int q = 0; q < CS; ++q) {
            const uint32_t c = s.above_q[q] + s.cand_sel[q];
            if (q < rank) off += c;
            if (q == rank) mine = c;
        }
        s.bcast[2] = off;
        s.bcast[3] = mine;
    }
    cta_sync();
    *cta_offset = s.bcast[2];
    stamp(tr, 7);
    return s.bcast[3];
}

// Writes emit(local index, output slot) for the selected keys, in index order.
template <int NTH, typename Emit>
SVL_DEV void push_emit(PushTopkSmem& s, const uint8_t* state, int nloc, uint32_t cta_offset, Emit emit) {
    const int tid = threadIdx.x;
    const int E = (nloc + NTH - 1) / NTH;
    const int nmine = max(0, min(E, nloc - tid * E));
    uint32_t mine = 0u, tot;
    for (int e = 0; e < nmine; ++e) mine += state[tid * E + e] == kKeySel;
    uint32_t slot = cta_offset + block_scan_excl<NTH>(mine, s.warp_sums, &tot);
    for (int e = 0; e < nmine; ++e) {
        const int i = tid * E + e;
        if (state[i] == kKeySel) emit(i, slot++);
    }
}

}  // namespace svl
