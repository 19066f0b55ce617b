// select_fast.cuh -- the fused kernel's relevance top-k, latency-trimmed.
//
// Same result as cluster_topk_push (select_push.cuh): the k largest relevance
// scores of a unit spread over the cluster, ties to the lower index, the kept
// indices written ascending.  Two cluster barriers in the common case:
//   histogram_and_threshold: keys (score -> order-preserving uint32) and a
//     256-bin value-adaptive histogram (float exponent 101..132 x 3 mantissa
//     bits; relevance scores are <= n_q*g <= 32) in one pass over the CTA's
//     logits; histogram pushed to every peer; cluster barrier; every CTA sums
//     the 16 histograms and finds the bin b* holding the k-th key;
//   assign_slots_and_push_candidates: rows at or above b* get decode V slots
//     (the caller starts their gather right away), the keys of b* (they share
//     key bits 31..20) are pushed to every peer in index order; cluster
//     barrier;
//   resolve_and_emit: every CTA resolves the exact cut inside b* with one
//     local 8-bit radix pass (bits 19..12) and an exact ranking within the
//     final sub-bin (key desc, index asc), derives every CTA's output offset
//     from the gathered counts, and writes its kept indices.
// If a CTA holds more than CANDS keys of b* (smooth score distributions over
// long slices) and the caller gave h2bar, one more all-gathered histogram of
// key bits 19..12 inside b* narrows the cut bin first (the resolve then uses
// bits 11..4).  If b* is the catch-all bin 0, or the refined bin still
// overflows, the generic exact radix of select_push.cuh takes over.
// Per-row state after the selection: 2 (kKeySel) = kept, 0 = not kept.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"
#include "select_push.cuh"

namespace svl {

constexpr int kFastCandPerCta = 64;
constexpr int kFastSub = 256;  // sub-bin members ranked by a short list

template <int CANDS>
struct FastSelSmemT {
    uint32_t allhist[16][256];
    uint2 cand[16][CANDS];
    uint32_t hist[256];
    uint32_t tot[256];
    uint32_t cnt_q[16], above_q[16], sel_q[16];
    uint32_t sel2[16][CANDS / 32];  // ballot masks of the kept candidates
    uint2 sub[kFastSub];
    uint32_t warp_sums[32];
    uint32_t bcast[16];
    uint8_t cflag[16][CANDS];
};
using FastSelSmem = FastSelSmemT<kFastCandPerCta>;

SVL_DEV int rel_digit(uint32_t key) {  // == push_digit(key, 0, .)
    const int e = (int)((key >> 23) & 0xffu);
    const int b = (e - 101) * 8 + (int)((key >> 20) & 7u);
    return (key & 0x80000000u) ? min(max(b, 0), 255) : 0;
}

// one warp: bin of the need-th largest over NB ascending bins
template <int NB>
__device__ __noinline__ void warp_find_nb(const uint32_t* bins, uint32_t need, uint32_t* out) {
    constexpr int PER = NB / 32;
    const int lane = threadIdx.x & 31;
    uint32_t c[PER];
    uint32_t grp = 0u;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        c[i] = bins[lane * PER + i];
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
        int b = lane * PER;
#pragma unroll
        for (int i = PER - 1; i >= 0; --i) {
            if (above + c[i] >= need) {
                b = lane * PER + i;
                break;
            }
            above += c[i];
        }
        out[0] = (uint32_t)b;
        out[1] = above;
    }
}

// CANDS: candidates of the threshold bin a CTA may hold (more -> the refinement round if
// REFINE, else / then the generic radix).  REFINE is a template switch: the refinement's
// code in threshold() measurably slows the instantiations that never need it (the fused
// kernel: 28.6 -> 29.25 us/layer at long-video).
template <int NTH, int CANDS = kFastCandPerCta, bool REFINE = false>
struct FastSelect {
    cg::cluster_group& cl;
    FastSelSmemT<CANDS>& s;
    int nvis, v0, slice, nv, k;
    uint32_t* keys;
    uint8_t* state;
    uint32_t* flags;
    uint32_t* whist;  // [NTH/32][256] private histograms (scratch, dead after the push)
    int bstar = 0;
    int sub = -1;   // >= 0: the cut was refined inside b* to sub-bin `sub` of key bits 19..12
    int rsh = 12;   // resolve radix: key bits rsh + 7 .. rsh (4 after the refinement)
    uint32_t krem = 0;
    uint32_t pre_gt = 0, pre_eq = 0;  // rows above the cut / candidates before this warp's rows (CTA-local)
    bool nan_seen = false;
    uint64_t* tr = nullptr;  // debug stamps (SVL_TRACE)
    // st.async exchange barriers (caller-initialised, count 1): hbar armed for CS x 1 KB of
    // histograms at init; cbar armed here once the candidate counts are known
    uint64_t* hbar = nullptr;
    uint64_t* cbar = nullptr;
    // optional (count 1, unarmed): the refinement round's histograms, CS x 1 KB into whist
    uint64_t* h2bar = nullptr;

    SVL_DEV FastSelect(cg::cluster_group& cl_, FastSelSmemT<CANDS>& s_, int nvis_, int v0_, int slice_, int nv_, int k_,
                       uint32_t* keys_, uint8_t* state_, uint32_t* flags_, uint32_t* whist_)
        : cl(cl_), s(s_), nvis(nvis_), v0(v0_), slice(slice_), nv(nv_), k(k_), keys(keys_), state(state_),
          flags(flags_), whist(whist_) {}

    // ownership for slots / emit: warp w takes the contiguous rows [32 E w, 32 E (w + 1)),
    // row base + 32 j + lane in step j (conflict-free key reads; positions in index order
    // from ballots and the warp's prefix)
    SVL_DEV void warp_rows(int& base, int& E) const {
        E = (nvis + NTH - 1) / NTH;
        base = (int)(threadIdx.x >> 5) * 32 * E;
    }
    // (REFINE = false, the fused kernel's short slices) contiguous ownership: thread tid
    // handles rows [i0, i1) -- measured faster there than the warp-interleaved loops
    SVL_DEV void my_rows(int& i0, int& i1) const {
        const int E = (nvis + NTH - 1) / NTH;
        i0 = min(nvis, (int)threadIdx.x * E);
        i1 = min(nvis, i0 + E);
    }

    SVL_DEV bool trivial() const { return k <= 0 || k >= nv; }

    // 2: above the cut bin (kept), 1: in it (a candidate), 0: below
    SVL_DEV int cls(uint32_t key) const {
        const int d = rel_digit(key);
        if (d != bstar) return d > bstar ? 2 : 0;
        if (!REFINE || sub < 0) return 1;
        const int sd = (int)((key >> 12) & 255u);
        return sd > sub ? 2 : (sd == sub ? 1 : 0);
    }

    // 1. (caller) zero_hist(); barrier; add_key(i, score) for every local row; then threshold()
    SVL_DEV void zero_hist() {
        for (int i = threadIdx.x; i < (NTH / 32) * 256; i += NTH) whist[i] = 0u;
    }
    SVL_DEV void add_key(int i, float score) {
        const uint32_t key = float_key(score, nan_seen);
        keys[i] = key;
#if SVL_HIST_MATCH
        // lanes with the same bin aggregate first (one atomic per distinct bin per warp)
        const int dg = rel_digit(key);
        const unsigned peers = __match_any_sync(__activemask(), dg);
        if ((int)(threadIdx.x & 31) == __ffs(peers) - 1)
            atomicAdd(&whist[(threadIdx.x >> 5) * 256 + dg], (uint32_t)__popc(peers));
#else
        atomicAdd(&whist[(threadIdx.x >> 5) * 256 + rel_digit(key)], 1u);
#endif
    }

    // returns 1 (fast path) or 2 (generic path); all threads, after the add_key pass
    SVL_DEV int threshold() {
        const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
        const int CS = (int)cl.num_blocks(), rank = (int)cl.block_rank();
        if (nan_seen) raise_flag(flags, 2u /*NONFINITE*/);
        stamp(tr, 8);
        cta_sync();
        stamp(tr, 9);
        // fold the private histograms and push bin b straight to every peer
        for (int b = tid; b < 256; b += NTH) {
            uint32_t acc = 0u;
#pragma unroll
            for (int w = 0; w < NTH / 32; ++w) acc += whist[w * 256 + b];
            s.hist[b] = acc;
        }
        cta_sync();
        for (int i = tid; i < CS * 64; i += NTH) {
            const int q = i >> 6, c = i & 63;
            st_async_u4(mapa_shared(smem_u32(&s.allhist[rank][4 * c]), q), reinterpret_cast<const uint4*>(s.hist)[c],
                        mapa_shared(smem_u32(hbar), q));
        }
        stamp(tr, 10);
        mbar_wait(smem_u32(hbar), 0);  // all CS histograms landed
        __syncwarp();
        stamp(tr, 11);
        for (int b = tid; b < 256; b += NTH) {
            uint32_t v[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) v[q] = (q < CS) ? s.allhist[q][b] : 0u;
            uint32_t acc = 0u;
#pragma unroll
            for (int q = 0; q < 16; ++q) acc += v[q];
            s.tot[b] = acc;
        }
        cta_sync();
        if (warp == 0) warp_find_nb<256>(s.tot, (uint32_t)k, s.bcast);
        cta_sync();
        stamp(tr, 12);
        bstar = (int)s.bcast[0];
        krem = (uint32_t)k - s.bcast[1];
        for (int q = warp; q < CS; q += NTH / 32) {
            uint32_t a = 0u;
            for (int b = bstar + 1 + lane; b < 256; b += 32) a += s.allhist[q][b];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
            if (lane == 0) {
                s.above_q[q] = a;
                s.cnt_q[q] = s.allhist[q][bstar];
                s.sel_q[q] = 0u;
            }
        }
        cta_sync();
        uint32_t maxc = 0u, totc = 0u;
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            maxc = max(maxc, (q < CS) ? s.cnt_q[q] : 0u);
            totc += (q < CS) ? s.cnt_q[q] : 0u;
        }
        int st = (bstar == 0 || maxc > (uint32_t)CANDS) ? 2 : 1;
        if (REFINE && st == 2 && bstar != 0 && bstar != 255 && h2bar != nullptr) {
            // Too many keys share b* (a smooth score distribution around the cut, e.g. 64k rows
            // per unit): one more all-gathered histogram, of key bits 19..12 inside b* (its
            // keys share bits 30..20), instead of the generic radix.
            if (tid == 0) mbar_arrive_expect_tx(smem_u32(h2bar), (uint32_t)(CS * 1024));
            for (int b = tid; b < 256; b += NTH) s.hist[b] = 0u;  // (round 1's values left by value)
            cta_sync();
            for (int i = tid; i < nvis; i += NTH) {
                const uint32_t key = keys[i];
                if (rel_digit(key) == bstar) atomicAdd(&s.hist[(key >> 12) & 255u], 1u);
            }
            cta_sync();
            uint32_t(*allh2)[256] = reinterpret_cast<uint32_t(*)[256]>(whist);  // dead since round 1's fold
            for (int i = tid; i < CS * 64; i += NTH) {
                const int q = i >> 6, c = i & 63;
                st_async_u4(mapa_shared(smem_u32(&allh2[rank][4 * c]), q), reinterpret_cast<const uint4*>(s.hist)[c],
                            mapa_shared(smem_u32(h2bar), q));
            }
            mbar_wait(smem_u32(h2bar), 0);
            __syncwarp();
            for (int b = tid; b < 256; b += NTH) {
                uint32_t acc = 0u;
                for (int q = 0; q < CS; ++q) acc += allh2[q][b];
                s.tot[b] = acc;
            }
            cta_sync();
            if (warp == 0) warp_find_nb<256>(s.tot, krem, s.bcast + 8);
            cta_sync();
            sub = (int)s.bcast[8];
            krem -= s.bcast[9];
            rsh = 4;
            for (int q = warp; q < CS; q += NTH / 32) {
                uint32_t a = 0u;
                for (int b = sub + 1 + lane; b < 256; b += 32) a += allh2[q][b];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
                if (lane == 0) {
                    s.above_q[q] += a;
                    s.cnt_q[q] = allh2[q][sub];
                }
            }
            cta_sync();
            maxc = 0u;
            totc = 0u;
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                maxc = max(maxc, (q < CS) ? s.cnt_q[q] : 0u);
                totc += (q < CS) ? s.cnt_q[q] : 0u;
            }
            st = (maxc > (uint32_t)CANDS) ? 2 : 1;
#if SVL_EXP_FLAG_STAGE2
            if (tid == 0 && rank == 0) raise_flag(flags, 0x200u);  // A/B builds: the refinement ran
#endif
        }
        if (st == 1 && tid == 0) mbar_arrive_expect_tx(smem_u32(cbar), totc * 8u);  // the candidates to come
        return st;
    }

    // V slots for every row with digit >= b* (att_sel[slot] = local row, in
    // index order); keys of b* pushed to the peers; returns the slot count.
    SVL_DEV int assign_slots_and_push_candidates(int* att_sel) {
        if constexpr (REFINE) return assign_warp_rows(att_sel);
        else return assign_contiguous(att_sel);
    }

    // (!REFINE) contiguous rows per thread, one block scan
    SVL_DEV int assign_contiguous(int* att_sel) {
        const int CS = (int)cl.num_blocks(), rank = (int)cl.block_rank();
        int i0, i1;
        my_rows(i0, i1);
        uint32_t ge = 0u, eq = 0u;
        for (int i = i0; i < i1; ++i) {
            const int c = cls(keys[i]);
            ge += c >= 1;
            eq += c == 1;
        }
        uint32_t tot;
        const uint32_t pre = block_scan_excl<NTH>(ge | (eq << 16), s.warp_sums, &tot);
        uint32_t pge = pre & 0xffffu, peq = pre >> 16;
        pre_gt = pge - peq;
        pre_eq = peq;
        for (int i = i0; i < i1; ++i) {
            const uint32_t key = keys[i];
            const int cl_ = cls(key);
            uint8_t st = 0;
            if (cl_ >= 1 && att_sel) att_sel[pge++] = i;  // (null: the caller needs no V slots)
            if (cl_ == 1) {
                st = (uint8_t)(CANDS > 254 ? min(peq + 1u, 255u) : peq + 1u);  // candidate marker
                const uint2 c = make_uint2(key, (uint32_t)(v0 + i));
                const uint32_t dst = smem_u32(&s.cand[rank][peq]), bar = smem_u32(cbar);
                if (peq < (uint32_t)CANDS)  // always true on this path (threshold() checked); defensive
                    for (int q = 0; q < CS; ++q) st_async_u2(mapa_shared(dst, q), c, mapa_shared(bar, q));
                ++peq;
            }
            state[i] = st;
        }
        mbar_wait(smem_u32(cbar), 0);  // every peer's candidates landed
        __syncwarp();
        return (int)(tot & 0xffffu);
    }

    // (REFINE: slices of up to 8192 rows) warp-interleaved rows, ballot prefixes
    SVL_DEV int assign_warp_rows(int* att_sel) {
        const int CS = (int)cl.num_blocks(), rank = (int)cl.block_rank();
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const unsigned lt = (1u << lane) - 1u;
        int base, E;
        warp_rows(base, E);
        uint32_t ge = 0u, eq = 0u;
        for (int j = 0; j < E; ++j) {
            const int i = base + 32 * j + lane;
            const int c = (i < nvis) ? cls(keys[i]) : 0;
            ge += (uint32_t)__popc(__ballot_sync(0xffffffffu, c >= 1));
            eq += (uint32_t)__popc(__ballot_sync(0xffffffffu, c == 1));
        }
        if (lane == 0) s.warp_sums[warp] = ge | (eq << 16);
        cta_sync();
        uint32_t pre = 0u, tot = 0u;
#pragma unroll
        for (int w = 0; w < NTH / 32; ++w) {
            const uint32_t x = s.warp_sums[w];
            pre += (w < warp) ? x : 0u;
            tot += x;
        }
        uint32_t pge = pre & 0xffffu, peq = pre >> 16;
        pre_gt = pge - peq;
        pre_eq = peq;
        for (int j = 0; j < E; ++j) {
            const int i = base + 32 * j + lane;
            const uint32_t key = (i < nvis) ? keys[i] : 0u;
            const int cl_ = (i < nvis) ? cls(key) : 0;
            const unsigned bg = __ballot_sync(0xffffffffu, cl_ >= 1), be = __ballot_sync(0xffffffffu, cl_ == 1);
            const uint32_t mg = pge + (uint32_t)__popc(bg & lt), me = peq + (uint32_t)__popc(be & lt);
            uint8_t st = 0;
            if (cl_ >= 1 && att_sel) att_sel[mg] = i;  // (null: the caller needs no V slots)
            if (cl_ == 1) {
                st = (uint8_t)(CANDS > 254 ? min(me + 1u, 255u) : me + 1u);  // candidate marker
                const uint2 c = make_uint2(key, (uint32_t)(v0 + i));
                const uint32_t dst = smem_u32(&s.cand[rank][me]), bar = smem_u32(cbar);
                if (me < (uint32_t)CANDS)  // always true on this path (threshold() checked); defensive
                    for (int q = 0; q < CS; ++q) st_async_u2(mapa_shared(dst, q), c, mapa_shared(bar, q));
            }
            if (i < nvis) state[i] = st;
            pge += (uint32_t)__popc(bg);
            peq += (uint32_t)__popc(be);
        }
        mbar_wait(smem_u32(cbar), 0);  // every peer's candidates landed
        __syncwarp();
        return (int)(tot & 0xffffu);
    }

    SVL_DEV void resolve_and_emit(int32_t* idx_out) {
        const int tid = threadIdx.x, warp = tid >> 5;
        const int rsh = REFINE ? this->rsh : 12;
        const int CS = (int)cl.num_blocks(), rank = (int)cl.block_rank();
        // one radix pass on key bits 19..12 over all candidates
        for (int i = tid; i < 256; i += NTH) s.hist[i] = 0u;
        if (tid == 0) s.bcast[6] = 0u;
        cta_sync();
        for (int sl = tid; sl < 16 * CANDS; sl += NTH) {
            const int q = sl / CANDS, j = sl % CANDS;
            if (q < CS && (uint32_t)j < s.cnt_q[q]) atomicAdd(&s.hist[(s.cand[q][j].x >> rsh) & 255u], 1u);
        }
        cta_sync();
        stamp(tr, 0);
        if (warp == 0) warp_find_nb<256>(s.hist, krem, s.bcast + 4);
        cta_sync();
        stamp(tr, 1);
        const uint32_t bA = s.bcast[4];
        const uint32_t need = krem - s.bcast[5];  // keys to keep inside sub-bin bA (>= 1)
        // (no shared atomics here: fire-and-forget ATOMS on a few hot counters
        // serialise and stall every later shared access of the CTA by microseconds)
        static_assert(CANDS % 32 == 0 && NTH % CANDS == 0, "one q per warp");
        // the members of sub-bin bA (usually a handful) compacted into sub[]
        const uint32_t nsub = s.hist[bA];
        if (nsub <= (uint32_t)kFastSub) {
            for (int sl = tid; sl < 16 * CANDS; sl += NTH) {
                const int q = sl / CANDS, j = sl % CANDS;
                if (q < CS && (uint32_t)j < s.cnt_q[q]) {
                    const uint2 c = s.cand[q][j];
                    if (((c.x >> rsh) & 255u) == bA) s.sub[atomicAdd(&s.bcast[6], 1u)] = c;
                }
            }
            cta_sync();
        }
        for (int sl = tid; sl < 16 * CANDS; sl += NTH) {
            const int q = sl / CANDS, j = sl % CANDS;
            bool take = false;
            if (q < CS && (uint32_t)j < s.cnt_q[q]) {
                const uint2 c = s.cand[q][j];
                const uint32_t dA = (c.x >> rsh) & 255u;
                take = dA > bA;
                if (dA == bA) {  // exact rank inside the sub-bin: (key desc, index asc)
                    uint32_t r = 0u;
                    if (nsub <= (uint32_t)kFastSub) {
                        for (uint32_t i = 0; i < nsub; ++i) {
                            const uint2 d = s.sub[i];
                            r += d.x > c.x || (d.x == c.x && d.y < c.y);
                        }
                    } else {
                        for (int q2 = 0; q2 < CS; ++q2)
                            for (uint32_t j2 = 0; j2 < s.cnt_q[q2]; ++j2) {
                                const uint2 d = s.cand[q2][j2];
                                r += (((d.x >> rsh) & 255u) == bA) && (d.x > c.x || (d.x == c.x && d.y < c.y));
                            }
                    }
                    take = r < need;
                }
                s.cflag[q][j] = take;
            }
            const unsigned bal = __ballot_sync(0xffffffffu, take);
            if ((tid & 31) == 0) s.sel2[q][j >> 5] = bal;
        }
        cta_sync();
        if constexpr (CANDS == 64) {  // (the fused kernel's instance: kept verbatim, it is latency-critical)
            if (tid < 16) s.sel_q[tid] = (uint32_t)(__popc(s.sel2[tid][0]) + __popc(s.sel2[tid][1]));
        } else if (tid < 16) {
            uint32_t c = 0u;
#pragma unroll
            for (int w = 0; w < CANDS / 32; ++w) c += (uint32_t)__popc(s.sel2[tid][w]);
            s.sel_q[tid] = c;
        }
        cta_sync();
        stamp(tr, 2);
        uint32_t off = 0u;
        for (int q = 0; q < rank; ++q) off += s.above_q[q] + s.sel_q[q];
        stamp(tr, 5);
        // output slot of a kept row = off + (rows above the cut before it) + (kept candidates
        // before it); both prefixes come from the slot-assignment prefixes and the candidate
        // ballot masks, so no second block scan
        const uint32_t* msk = s.sel2[rank];
        const uint32_t m0 = msk[0], m1 = msk[1];
        auto kept_cands_before = [&](uint32_t e) -> uint32_t {
            if constexpr (CANDS == 64) {
                return e >= 32u ? (uint32_t)__popc(m0) + (uint32_t)__popc(m1 & ((1u << (e - 32u)) - 1u))
                                : (uint32_t)__popc(m0 & ((1u << e) - 1u));
            } else {
                uint32_t c = 0u;
                for (uint32_t w = 0; w < (e >> 5); ++w) c += (uint32_t)__popc(msk[w]);
                if (e & 31u) c += (uint32_t)__popc(msk[e >> 5] & ((1u << (e & 31u)) - 1u));
                return c;
            }
        };
        if constexpr (!REFINE) {
            int i0, i1;
            my_rows(i0, i1);
            uint32_t gtc = pre_gt, eqc = pre_eq;
            for (int i = i0; i < i1; ++i) {
                const int c = cls(keys[i]);
                bool kept = c == 2;
                if (c == 1) kept = s.cflag[rank][eqc] != 0;
                if (kept) idx_out[off + gtc + kept_cands_before(eqc)] = v0 + i;
                gtc += c == 2;
                eqc += c == 1;
                state[i] = kept ? kKeySel : kKeyOut;
            }
        } else {
            const int lane = tid & 31;
            const unsigned lt = (1u << lane) - 1u;
            int base, E;
            warp_rows(base, E);
            uint32_t gtc = pre_gt, eqc = pre_eq;
            for (int j = 0; j < E; ++j) {
                const int i = base + 32 * j + lane;
                const int c = (i < nvis) ? cls(keys[i]) : 0;
                const unsigned ba = __ballot_sync(0xffffffffu, c == 2), be = __ballot_sync(0xffffffffu, c == 1);
                const uint32_t ma = gtc + (uint32_t)__popc(ba & lt), me = eqc + (uint32_t)__popc(be & lt);
                bool kept = c == 2;
                if (c == 1) kept = s.cflag[rank][me] != 0;
                if (kept) idx_out[off + ma + kept_cands_before(me)] = v0 + i;
                if (i < nvis) state[i] = kept ? kKeySel : kKeyOut;
                gtc += (uint32_t)__popc(ba);
                eqc += (uint32_t)__popc(be);
            }
        }
        stamp(tr, 3);
        stamp(tr, 4);
    }

    // stage 0: k <= 0 or k >= nv; stage 2: generic exact radix.  Writes
    // idx_out, att_sel (kept local rows in index order) and state; returns
    // the CTA's kept count.
    SVL_DEV int generic_or_trivial(int stage, PushTopkSmem& ps, int32_t* idx_out, int* att_sel) {
        const int tid = threadIdx.x;
        if (stage == 0) {
            const bool all = k >= nv;
            for (int i = tid; i < nvis; i += NTH) {
                state[i] = all ? kKeySel : kKeyOut;
                if (all) {
                    idx_out[v0 + i] = v0 + i;
                    att_sel[i] = i;
                }
            }
            cta_sync();
            return all ? nvis : 0;
        }
        uint32_t off;
        const int nsel = (int)cluster_topk_push<NTH>(cl, ps, keys, state, nvis, v0, slice, nv, k,
                                                     /*relevance=*/true, &off);
        push_emit<NTH>(ps, state, nvis, off, [&](int i, uint32_t slot) {
            idx_out[slot] = v0 + i;
            att_sel[slot - off] = i;
        });
        cta_sync();
        return nsel;
    }
};

}  // namespace svl
