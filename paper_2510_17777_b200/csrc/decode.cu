// decode.cu -- gathered flash-decoding over the active set on every SM, with
// a log-sum-exp merge of the splits through L2.
//
// PAPER.md:121 / 433: decode attention over the active set only -- all text
// rows plus the k retrieved visual rows ("less relevant tokens
// remain cached but inactive"; SPEC.md:315-323 pack_active order).  For each
// unit (b, KV group G) the attended rows
//     [0, vb)  U  {vb + idx[m] : m < k}  U  [vb + N_v, seq_len)
// are cut into S splits, one CTA each (api.cu plan_decode: S from the co-resident
// CTA count; B = 1: 4 units x 16 splits).  Split s takes the s-th S-th of each of
// the three segments (system rows, kept visual rows, later text rows), so its
// visual share -- the idx loads and the K/V gathers -- does not wait for seq_len.
// Per CTA (256 threads, one per SM):
//   1. software pipeline over 128-row batches: row ids of batch j + NBUF are
//      loaded (idx validated: in range, strictly ascending) while batch j is
//      computed; K and V rows of batch j + NBUF - 1 are gathered with cp.async
//      (16-byte, L1-bypassing) into XOR-swizzled shared memory.  With
//      SVL_DECODE_STATIC_PREFIX the first batches' rows (all but the current
//      token's) are gathered before the PDL wait, laid out by a speculative
//      seq_len read that is checked after the batch loop (a miss reruns it);
//   2. per warp and 16-row tile: S = q K^T with mma.sync m16n8k16 (heads are M,
//      rows are N, the contraction permuted so K chunks are read with
//      conflict-free 128-bit LDS), online softmax in base 2, O += P V with P
//      split into bf16 hi + lo (two MMAs: ~2^-17 relative error instead of
//      bf16's 2^-9) and V B-fragments from ldmatrix.trans; one cross-warp merge
//      per CTA gives its partial (o, M, l);
//   3. S > 1, the S CTAs of a unit one thread-block cluster (every cluster
//      co-resident): each CTA owns a 1/S share of the unit's (head, column)
//      items (a multiple of 4); every CTA pushes its partial's items to their
//      owners and its (M, l) to every peer with st.async (16-byte pushes,
//      mbarrier byte counts), each owner merges over the S partials in rank
//      order.  Otherwise a co-resident grid (cooperative launch): partials are
//      stored as 64-bit (value, tag) pairs tagged with the unit's call epoch
//      and each CTA merges its share once the tags it needs are this call's.
//      M = max m_i, out = sum e^{m_i-M} o_i / sum e^{m_i-M} l_i,
//      lse = M + log sum e^{m_i-M} l_i (north star step 3), in a fixed order.
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"

#ifndef SVL_OWNER_T
#define SVL_OWNER_T 1  // cluster merge: threads per owned item (measured: 1 -> 9.49 to 8.53 us at long-video)
#endif
#ifndef SVL_L2OWNER_T
#define SVL_L2OWNER_T 4  // L2 merge (S > 16): threads per owned item (at most; measured S = 37: 32 -> 10.35, 4 -> 9.59 us)
#endif
#ifndef SVL_EXP_NOOWNER
#define SVL_EXP_NOOWNER 0  // timing experiment: the cluster merge's owner loop skipped (no output)
#endif

namespace svl {

namespace {

constexpr int NTH = kDecodeThreads;  // 256: 8 warps
constexpr int NW = NTH / 32;
constexpr int RB = kDecodeRowsMax;   // 128 rows per batch = 8 warps x one 16-row tile
static_assert(RB == 16 * NW, "one 16-row tile per warp and batch");
// NB = gather buffers: NB - 1 batches in flight while one is computed.  NB = 1 when every
// CTA has a single batch (B = 1 shapes): 66 KB of shared memory, so the next launch's CTAs
// (programmatic dependent launch) are resident while this grid runs; NB = 3 otherwise.
template <int D, int NB>
struct DecodeSmem {
    static_assert(NB >= 1 && (NB - 1) * RB <= NTH, "prologue: one row id per thread");
    static constexpr int ROW_BYTES = D * 2;
    static constexpr int BUF_BYTES = 2 * RB * ROW_BYTES;           // K + V of one batch
    static_assert(NB * BUF_BYTES >= NW * 16 * D * 4, "cross-warp merge staging fits the gather buffers");
    static constexpr int ROWS_OFF = NB * BUF_BYTES;                 // row ids [NB][RB]
    static constexpr int WML_OFF = ROWS_OFF + NB * RB * 4;          // per-warp m, l [2][NW][16] fp32
    static constexpr int RUN_OFF = WML_OFF + 2 * NW * 16 * 4;       // CTA M[16], l[16]
    static constexpr int SC_OFF = RUN_OFF + 32 * 4;                 // warp scales [NW][16]
    // cluster merge (DSMEM): every peer's share of this CTA's items [S][per] and its M, l
    // [S][32]; per = ceil(g D / S) rounded up to 4 (16-byte pushes) -> S * per <= 16 D + 4 S
    // <= 16 D + 64; mbarrier counting the bytes
    static constexpr int RCV_OFF = SC_OFF + NW * 16 * 4;
    static constexpr int RML_OFF = RCV_OFF + (16 * D + 64) * 4;
    static constexpr int MB_OFF = RML_OFF + 16 * 33 * 4;  // rml rows padded to 33 (bank-conflict free)
    static constexpr int BYTES = MB_OFF + 16;
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

template <int D, int NBUF>
__global__ void __launch_bounds__(NTH, 1) decode_kernel(const __grid_constant__ DecodeParams p) {
    using SM = DecodeSmem<D, NBUF>;
    constexpr int CH = D / 8;    // 16-byte chunks per row
    constexpr int NCH = D / 32;  // chunks per thread per row in the permuted-k layout
    extern __shared__ __align__(128) uint8_t smem[];
    const int S = (int)gridDim.x, split = (int)blockIdx.x, u = (int)blockIdx.y;
    int* rows_s = reinterpret_cast<int*>(smem + SM::ROWS_OFF);  // [NBUF][RB]
    float* run = reinterpret_cast<float*>(smem + SM::RUN_OFF);       // M[16], l[16]

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int gid = lane >> 2, t = lane & 3;
#if SVL_TRACE_BUILD
    uint64_t* trace = p.trace ? p.trace + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 16 : nullptr;
    auto stamp = [&](int i) {  // SM cycles (clock64: exact within a CTA)
        if (trace && tid == 0) trace[i] = clock64();
    };
#else
    auto stamp = [](int) {};
#endif
    stamp(0);
#if SVL_TRACE_BUILD
    if (trace && tid == 0) {
        uint64_t tnow;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
        trace[14] = tnow;
    }
#endif
    // programmatic dependent launch: nothing an upstream kernel may write (seq_len,
    // idx, q, the appended K/V row) is read before the wait -- but see SVL_DECODE_STATIC_PREFIX
    // cluster merge: one local arrival + the bytes every peer will push (its share of this
    // CTA's items and its 32 M, l values); peers push only after their cluster_wait
    const uint32_t mbar = smem_u32(smem + SM::MB_OFF);
    if (p.cluster) {
        if (tid == 0) {
            const int items = p.g * D, per = (((items + S - 1) / S) + 3) & ~3;  // (16-B pushes)
            const int mine = max(0, min(per, items - split * per));
            mbar_init(mbar, 1);
            mbar_arrive_expect_tx(mbar, (uint32_t)(S * (mine + 32) * 4));
            fence_mbar_init();
        }
        cluster_arrive_relaxed();
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // SVL_DECODE_STATIC_PREFIX: vis_idx and every K, V row below seq_len - 1 (all but the
    // current token's) are not written by the upstream kernel, so the idx loads and the first
    // batches' gathers of those rows go out before the wait (overlapping the upstream kernel's
    // tail), their text share laid out by a speculative seq_len read that is checked after it;
    // q, seq_len, the current token's row and the workspace counters are read only after it
    const bool early = p.static_vis != 0;
    const int b = u / p.Hkv, G = u % p.Hkv;
    // q A-fragments (heads gid, gid + 8 of the group; zero beyond g); an early call loads
    // them right after the wait
    uint4 qa[NCH], qb[NCH];
    auto load_q = [&]() {
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
    };
    if (!early) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        stamp(6);
    }
    const int U = p.shared ? 1 : p.Hkv;
    const int uG = p.shared ? 0 : G;
    const int32_t* idx = p.idx + ((int64_t)b * U + uG) * p.k;
    const uint16_t* Kb = p.K + (int64_t)b * p.ksb + (int64_t)G * p.ksh;
    const uint16_t* Vb = p.V + (int64_t)b * p.vsb + (int64_t)G * p.vsh;

    // this split's share of the segments: system rows [s0, s0 + ns), kept visual m in
    // [m0, m0 + nm), later text rows t in [t0, t0 + na) (the last needs seq_len)
    const int s0 = (int)((int64_t)split * p.vb / S), ns = (int)((int64_t)(split + 1) * p.vb / S) - s0;
    const int m0 = (int)((int64_t)split * p.k / S), nm = (int)((int64_t)(split + 1) * p.k / S) - m0;
    const int nst = ns + nm;  // list items [0, nst) need no seq_len (system + visual rows)
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
    // row id of a system or visual list item i < nst (-1: a bad index -> device flag)
    auto resolve_st = [&](int i, const Pending& r) -> int {
        if (i < ns) return s0 + i;
        if (r.x >= 0 && r.x < p.nv && r.xp < r.x) return p.vb + r.x;
        if (p.padded && r.x == -1) return -1;  // trailing padding (SVL_IDX_PADDED)
        raise_flag(p.flags, 1u /*SVL_DEVFLAG_INDEX*/);
        return -1;
    };
    // batches [0, JE) of an early call had their system / visual rows gathered before the wait
    constexpr int JE = NBUF > 1 ? NBUF - 1 : 1;
    // gather list items [lo, hi) of batch j (row ids in rows_s[j % NBUF]; n_lim bounds the
    // batch's rows, padded to the 16-row tile with zero-filled copies) -- no commit
    auto issue_rows = [&](int j, auto take, int n_lim) {  // take(i): gather list item i
        const int* rows = rows_s + (j % NBUF) * RB;
        const uint32_t sK = smem_u32(smem + (j % NBUF) * SM::BUF_BYTES);
        const uint32_t sV = sK + RB * SM::ROW_BYTES;
        const int nj = min(RB, n_lim - j * RB);
        const int nr = (nj + 15) & ~15;
        // thread -> chunk c of rows r0, r0 + NTH/CH, ...: every row id read first, then
        // all the copies back to back (no shared-memory load between two copies)
        constexpr int RPP = NTH / CH, PASSES = RB / RPP;
        const int c = tid % CH, r0 = tid / CH;
        int rw[PASSES];
#pragma unroll
        for (int k = 0; k < PASSES; ++k) {
            const int r = r0 + k * RPP;
            rw[k] = (r < nr && take(j * RB + r)) ? rows[r] : -2;
        }
#pragma unroll
        for (int k = 0; k < PASSES; ++k) {
            const int r = r0 + k * RPP;
            if (rw[k] == -2) continue;
            const bool valid = rw[k] >= 0;
            const int rr = valid ? rw[k] : 0;
#if SVL_DEBUG_TRAP  // debug builds: every gathered row lies inside the cache
            if (rr >= p.capacity) __trap();
#endif
            cp_async16(sK + r * SM::ROW_BYTES + swz_k(r, c) * 16, Kb + (int64_t)rr * p.kst + c * 8, valid);
            cp_async16(sV + r * SM::ROW_BYTES + swz_v(r, c) * 16, Vb + (int64_t)rr * p.vst + c * 8, valid);
        }
    };
    // text share of this split for a seq_len value (clamped to the span; the device flag is
    // raised for the checked read only)
    auto clamp_len = [&](int Lv) { return min(max(Lv, p.vb + p.nv), p.capacity); };
    auto text_share = [&](int Lv, int& t0o, int& nao) {
        const int Tv = Lv - p.vb - p.nv;
        t0o = (int)((int64_t)split * Tv / S);
        nao = (int)((int64_t)(split + 1) * Tv / S) - t0o;
    };
    // the first NBUF - 1 batches' idx loads (one item per thread) go out first
    Pending pre = fetch(tid);
    int Ls = 0, t0s = 0, nas = 0;  // early: the speculative seq_len (clamped) and text share
    Pending pend{0, -1};            // idx loads of batch NBUF - 1 (consumed at the top of iteration 0)
    if (early) {
        if (tid < RB) pend = NBUF == 1 ? pre : fetch((NBUF - 1) * RB + tid);
        Ls = clamp_len((int)ld_relaxed_u32(reinterpret_cast<const uint32_t*>(p.seq_len + b)));
#if SVL_EXP_SPEC_MISS  // test build: the speculation always misses (the re-gather path)
        Ls = clamp_len(Ls - 1 - (int)(split & 3));
#endif
        text_share(Ls, t0s, nas);
        const int n_s = nst + nas;
        // every item of batches [0, JE) under the speculation; all gathered now but the
        // current token's row (Ls - 1), which goes out right after the wait
        if (tid < JE * RB)
            rows_s[tid] = tid < nst ? resolve_st(tid, pre) : (tid < n_s ? p.vb + p.nv + t0s + (tid - nst) : -1);
        cta_sync();
        const int i_cur = (nas > 0 && t0s + nas == Ls - p.vb - p.nv) ? n_s - 1 : -1;  // the current row's item
        for (int j = 0; j < JE; ++j) issue_rows(j, [&](int i) { return i != i_cur; }, n_s);
        cp_async_commit();  // (one group, older than every group below)
        asm volatile("griddepcontrol.wait;" ::: "memory");
        stamp(6);
        load_q();
        // one group per early batch, the current row's copies in its batch's group (batch 0's
        // compute does not wait for a later batch's row); these stand in for the prologue's
        // groups in the wait_group arithmetic (JE = NBUF - 1 when NBUF > 1)
        for (int j = 0; j < JE; ++j) {
            if (i_cur >= 0 && i_cur / RB == j) issue_rows(j, [&](int i) { return i == i_cur; }, n_s);
            cp_async_commit();
        }
    }
    // this call's epoch of the unit (advanced by split 0 at the end of the previous call)
    const uint32_t tag_epoch = (S > 1 && !p.cluster) ? ld_relaxed_u32(p.epochs + u) : 0u;
    // tag = hash(epoch, unit, S): a slot left by another call -- another epoch, or another
    // split layout of the same workspace -- does not match (zero-filled slots never do)
    const uint32_t tag = partial_tag(tag_epoch, (uint32_t)u, (uint32_t)S);
    // seq_len: an early call runs on its speculative value and checks this read after the
    // batch loop (its latency overlaps the compute); a miss reruns the pipeline on it
    const int L_raw = __ldg(p.seq_len + b);
    auto checked_len = [&]() {
        if (L_raw < p.vb + p.nv || L_raw > p.capacity) {
            if (tid == 0 && split == 0) raise_flag(p.flags, 4u /*SPAN*/);
            return clamp_len(L_raw);
        }
        return L_raw;
    };
    int L = early ? Ls : checked_len();
    int t0, na;
    text_share(L, t0, na);
    int n = nst + na;  // this CTA's attended rows
    int nb = (n + RB - 1) / RB;
    stamp(1);
    // row id of list item i (-1: past the list, or a bad index -> device flag)
    auto resolve = [&](int i, const Pending& r) -> int {
        if (i < 0 || i >= n) return -1;
        if (i < nst) return resolve_st(i, r);
        return p.vb + p.nv + t0 + (i - nst);
    };
    // an early call published (and gathered) every item of batches [0, JE) -- until a rerun
    bool pub_early = early;
    auto published = [&](int i) { return pub_early && i < JE * RB; };
    auto issue = [&](int j) {  // gather batch j -- one commit group (+ the tile's zero-filled padding)
        if (j < nb) issue_rows(j, [&](int i) { return !published(i); }, n);
        cp_async_commit();  // (empty groups keep the wait_group arithmetic uniform)
    };

    constexpr int NTO = D / 8;  // output n-tiles
    float o[NTO][4];
    float m_a, m_b;  // running max of heads gid, gid + 8 (quad-uniform)
    float l_a, l_b;  // this thread's share of the running sums
    for (;;) {  // one pass; an early call whose seq_len speculation missed takes a second
    // ---- prologue: row ids of batches [0, NBUF - 1) (one per thread), their gathers, and
    // the idx loads of batch NBUF - 1 (consumed at the top of iteration 0)
    if (tid < (NBUF - 1) * RB && !published(tid)) rows_s[tid] = resolve(tid, pre);
    if (!pub_early && tid < RB) pend = NBUF == 1 ? pre : fetch((NBUF - 1) * RB + tid);
    if (!pub_early) cta_sync();  // (an early pass wrote its prologue row ids before the wait)
    stamp(2);
    if (!pub_early)
        for (int j = 0; j < NBUF - 1; ++j) issue(j);
    if (!early) load_q();

    // FlashAttention-2 style per warp: warp w owns rows [16 w, 16 w + 16) of every batch,
    // scores them, keeps a running max per head, and multiplies P (still in registers: the
    // two n-tiles of the score accumulator ARE the A fragment of a k16 MMA) into its own
    // O[16 heads][D] -- no per-batch CTA barrier beyond the buffer hand-over.
#pragma unroll
    for (int i = 0; i < NTO; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    m_a = m_b = -INFINITY;
    l_a = l_b = 0.f;

    for (int j = 0; j < nb; ++j) {
        // row ids of batch j + NBUF - 1 (loads issued one iteration ago), then the loads of
        // batch j + NBUF's; the barrier publishes the ids and frees buffer (j - 1) % NBUF
        if (j + NBUF - 1 < nb) {  // (past the last batch: nothing to publish, no buffer to free)
            if (tid < RB && !published((j + NBUF - 1) * RB + tid))
                rows_s[((j + NBUF - 1) % NBUF) * RB + tid] = resolve((j + NBUF - 1) * RB + tid, pend);
            if (tid < RB) pend = fetch((j + NBUF) * RB + tid);
            cta_sync();
        }
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
        const int tb = warp * 16;
        if (tb >= nj) continue;  // (warp-uniform) no rows of this warp in the batch
        float s[2][4];  // n-tile nt: c0, c1 -> head gid, rows tb + 8nt + 2t, +1; c2, c3 -> head gid + 8
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
        const float mn_a = fmaxf(m_a, mx_a), mn_b = fmaxf(m_b, mx_b);
        const float al_a = (mn_a == -INFINITY) ? 1.f : fast_exp2(m_a - mn_a);
        const float al_b = (mn_b == -INFINITY) ? 1.f : fast_exp2(m_b - mn_b);
        m_a = mn_a;
        m_b = mn_b;
        // P = exp2(s - M) split into bf16 hi + lo, packed straight into A fragments:
        // a0 = (head gid, rows 2t, 2t+1), a1 = (gid + 8, ...), a2 / a3 = the same for rows + 8
        uint32_t ph[4], plo[4];
        float ls_a = 0.f, ls_b = 0.f;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int hb = 0; hb < 2; ++hb) {
                const float mn = hb ? mn_b : mn_a;
                const float p0 = (s[nt][2 * hb] == -INFINITY) ? 0.f : fast_exp2(s[nt][2 * hb] - mn);
                const float p1 = (s[nt][2 * hb + 1] == -INFINITY) ? 0.f : fast_exp2(s[nt][2 * hb + 1] - mn);
                const uint32_t hw = pack_bf16(p0, p1);
                const uint32_t lw = pack_bf16(p0 - bf16lo(hw), p1 - bf16hi(hw));
                ph[2 * nt + hb] = hw;
                plo[2 * nt + hb] = lw;
                const float w = bf16lo(hw) + bf16lo(lw) + bf16hi(hw) + bf16hi(lw);
                if (hb) ls_b += w;
                else ls_a += w;
            }
        l_a = l_a * al_a + ls_a;
        l_b = l_b * al_b + ls_b;
        // O = O * al + P V over the warp's 16 rows: V B-fragments by ldmatrix.trans, two
        // output n-tiles per load; all 2 x NTO MMAs independent
        const int mi = lane >> 3, rin = lane & 7;
        const int vrow = tb + (mi & 1) * 8 + rin;
#pragma unroll
        for (int cp = 0; cp < NTO / 2; ++cp) {
            uint32_t v0, v1, v2, v3;
            ldsm_x4_trans(sV + vrow * SM::ROW_BYTES + swz_v(vrow, 2 * cp + (mi >> 1)) * 16, v0, v1, v2, v3);
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                float* oo = o[2 * cp + h2];
                oo[0] *= al_a; oo[1] *= al_a;
                oo[2] *= al_b; oo[3] *= al_b;
                const uint32_t b0 = h2 ? v2 : v0, b1 = h2 ? v3 : v1;
                mma_bf16_16816(o[2 * cp + h2], ph, b0, b1);
                mma_bf16_16816(o[2 * cp + h2], plo, b0, b1);
            }
        }
    }
    cp_async_wait<0>();
    cta_sync();  // every warp's batches done; the gather buffers are free
    if (!early || !pub_early) break;
    const int L_chk = checked_len();
    if (L_chk == Ls) break;
#if SVL_EXP_MISS_FLAG  // test build: report a speculation miss in the device flags (bit 16)
    if (tid == 0) raise_flag(p.flags, 16u);
#endif
    // the speculation missed (seq_len changed upstream): rerun on the checked value with every
    // row gathered after the wait (the pipeline's buffers are idle: the barrier above)
    pub_early = false;
    L = L_chk;
    text_share(L, t0, na);
    n = nst + na;
    nb = (n + RB - 1) / RB;
    }
    stamp(4);

    // ---- cross-warp merge inside the CTA (shared memory, the gather buffers): each warp's
    // (m, l, O) rescaled to the CTA max; the result is the CTA's partial (o, M, l)
    float* wml = reinterpret_cast<float*>(smem + SM::WML_OFF);   // [2][NW][16] m, l
    float* wsc = reinterpret_cast<float*>(smem + SM::SC_OFF);    // [NW][16] exp2(m_w - M)
    float* wo = reinterpret_cast<float*>(smem);                   // [NW][16][D]
    {
        l_a += __shfl_xor_sync(0xffffffffu, l_a, 1);
        l_a += __shfl_xor_sync(0xffffffffu, l_a, 2);
        l_b += __shfl_xor_sync(0xffffffffu, l_b, 1);
        l_b += __shfl_xor_sync(0xffffffffu, l_b, 2);
        if (t == 0) {
            wml[warp * 16 + gid] = m_a;
            wml[warp * 16 + gid + 8] = m_b;
            wml[NW * 16 + warp * 16 + gid] = l_a;
            wml[NW * 16 + warp * 16 + gid + 8] = l_b;
        }
        // column swizzle c ^ 8 (h & 3): the 8 heads a warp's quarter-groups store land in
        // distinct banks (row stride D is a multiple of 32 words: 8-way conflicts otherwise)
#pragma unroll
        for (int i = 0; i < NTO; ++i) {
            const int col = (i * 8 + 2 * t) ^ ((gid & 3) << 3);
            if (gid < p.g) *reinterpret_cast<float2*>(wo + (warp * 16 + gid) * D + col) = make_float2(o[i][0], o[i][1]);
            if (gid + 8 < p.g)
                *reinterpret_cast<float2*>(wo + (warp * 16 + gid + 8) * D + col) = make_float2(o[i][2], o[i][3]);
        }
    }
    cta_sync();
    stamp(10);
    if (tid < 16) {  // CTA max, warp scales and sum of head tid (fixed warp order)
        float M = -INFINITY;
#pragma unroll
        for (int w = 0; w < NW; ++w) M = fmaxf(M, wml[w * 16 + tid]);
        float l = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const float mw = wml[w * 16 + tid];
            const float sc = (mw == -INFINITY) ? 0.f : fast_exp2(mw - M);
            wsc[w * 16 + tid] = sc;
            l += sc * wml[NW * 16 + w * 16 + tid];
        }
        run[tid] = M;
        run[16 + tid] = l;
    }
    cta_sync();
    // item (h, c) of the CTA partial: the warps' O rescaled to the CTA max, summed in warp order
    auto cta_o = [&](int h, int c) -> float {
        float acc = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) acc += wsc[w * 16 + h] * wo[(w * 16 + h) * D + (c ^ ((h & 3) << 3))];
        return acc;
    };

    constexpr int PSTRIDE = kDecodePartStride<D>;
    auto finalize = [&](int h, int dd, float ov, float M, float den) {
#if SVL_EXP_NOFINAL  // timing experiment: no output stores
        if (ov != 12345.f) return;
#endif
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
        for (int i = tid; i < p.g * D; i += NTH) {
            const int h = i / D, c = i % D;
            const float den = run[16 + h];
            finalize(h, c, den > 0.f ? cta_o(h, c) / den : 0.f, run[h], den);
        }
    } else if (p.cluster) {
        // the S CTAs of the unit form one cluster: every CTA pushes each item of the unit's
        // g x D block to its owner q = i / per (st.async into q's receive buffer, counted on
        // q's mbarrier) and its 32 (M, l) to every peer; owners merge in rank order
        const int items = p.g * D, per = (((items + S - 1) / S) + 3) & ~3;  // (16-B pushes)
        float* rcv = reinterpret_cast<float*>(smem + SM::RCV_OFF);  // [S][per]
        float* rml = reinterpret_cast<float*>(smem + SM::RML_OFF);  // [S][33]: M[16], l[16], pad
        stamp(11);
        cluster_wait();  // every peer has armed its barrier
        stamp(12);
        const uint32_t rcv_a = smem_u32(rcv), rml_a = smem_u32(rml);
        // four consecutive items per thread (one head: D % 4 == 0; one owner: per % 4 == 0):
        // 128-bit loads of the warps' staged O, one 16-byte push
        for (int i = 4 * tid; i < items; i += 4 * NTH) {
            const int q = i / per, h = i / D, c = (i % D) ^ ((h & 3) << 3);
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const float sc = wsc[w * 16 + h];
                const float4 v = *reinterpret_cast<const float4*>(wo + (w * 16 + h) * D + c);
                acc.x += sc * v.x; acc.y += sc * v.y; acc.z += sc * v.z; acc.w += sc * v.w;
            }
            st_async_u4(mapa_shared(rcv_a + (uint32_t)(split * per + (i - q * per)) * 4u, q),
                        make_uint4(__float_as_uint(acc.x), __float_as_uint(acc.y), __float_as_uint(acc.z),
                                   __float_as_uint(acc.w)),
                        mapa_shared(mbar, q));
        }
        for (int i = tid; i < 32 * S; i += NTH) {
            const int q = i >> 5, h = i & 31;
            st_async_f32(mapa_shared(rml_a + (uint32_t)(split * 33 + h) * 4u, q), run[h], mapa_shared(mbar, q));
        }
        stamp(5);
        mbar_wait(mbar, 0);  // every peer's bytes landed
        __syncwarp();
        stamp(8);
        const int i0 = split * per, ni = max(0, min(per, items - i0));
        int T = SVL_OWNER_T;  // threads per owned item (measured: 1 pass over the items with few
        while (T > 1 && T * ni > NTH) T >>= 1;  // threads each beats wide xor trees)
        for (int jb = 0; jb < (SVL_EXP_NOOWNER ? 0 : ni); jb += NTH / T) {
            const int j = jb + tid / T, sub = tid & (T - 1);
            const int h = (j < ni) ? (i0 + j) / D : 0;
            float M = -INFINITY;
            if (j < ni)
                for (int q = sub; q < S; q += T) M = fmaxf(M, rml[q * 33 + h]);
            for (int off = T >> 1; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
            float num = 0.f, den = 0.f;
            if (j < ni && M != -INFINITY)
                for (int q = sub; q < S; q += T) {
                    const float w = fast_exp2(rml[q * 33 + h] - M);
                    num += w * rcv[q * per + j];
                    den += w * rml[q * 33 + 16 + h];
                }
            for (int off = T >> 1; off > 0; off >>= 1) {
                num += __shfl_xor_sync(0xffffffffu, num, off);
                den += __shfl_xor_sync(0xffffffffu, den, off);
            }
            if (sub == 0 && j < ni) finalize(h, (i0 + j) % D, (den > 0.f) ? num / den : 0.f, M, den);
        }
        stamp(9);
        // no closing cluster barrier: nobody reads a peer's shared memory, and every CTA
        // waited for all the bytes pushed into it before getting here
    } else {
        // Partial (o, M, l) of this split -> workspace slot (u, split), every value stored as a
        // 64-bit (bits, tag) pair with one single-copy-atomic store; tag = the unit's call
        // epoch.  A reader that sees the tag sees the value: no barrier, no flag round trip.
        uint64_t* mine = p.part + (int64_t)(u * S + split) * PSTRIDE;
        for (int i = 2 * tid; i < p.g * D; i += 2 * NTH) {
            const int h = i / D, c = i % D;
            st_tagged2(mine + i, cta_o(h, c), cta_o(h, c + 1), tag);
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
            cta_sync();  // every thread's cta_o reads of the staging region are done
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
            // per item: T threads (a power of two <= 32) stride over the splits -- max, then the
            // weighted sums of o and l -- with fixed xor trees inside the T-lane group
            int T = SVL_L2OWNER_T;
            while (T > 1 && T * ni > 2 * NTH) T >>= 1;
            for (int jb = 0; jb < ni; jb += NTH / T) {
                const int j = jb + tid / T, sub = tid & (T - 1);
                const int hh = (j < ni) ? (i0 + j) / D - h0 : 0;
                float M = -INFINITY;
                if (j < ni) {
#pragma unroll 4
                    for (int q = sub; q < S; q += T) M = fmaxf(M, mb[q * nh + hh]);
                }
                for (int off = T >> 1; off > 0; off >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
                float num = 0.f, den = 0.f;
                if (j < ni && M != -INFINITY) {
#pragma unroll 4
                    for (int q = sub; q < S; q += T) {
                        const float w = fast_exp2(mb[q * nh + hh] - M);
                        num += w * ob[q * ni + j];
                        den += w * lb[q * nh + hh];
                    }
                }
                for (int off = T >> 1; off > 0; off >>= 1) {
                    num += __shfl_xor_sync(0xffffffffu, num, off);
                    den += __shfl_xor_sync(0xffffffffu, den, off);
                }
                if (sub == 0 && j < ni) finalize(h0 + hh, (i0 + j) % D, (den > 0.f) ? num / den : 0.f, M, den);
            }
            stamp(9);
        }
        // split 0 advances the unit's epoch once its own merge has seen every split's
        // partial -- so every CTA of the unit has read the current epoch already
        if (split == 0 && tid == 0) p.epochs[u] = tag_epoch + 1u;
    }
    stamp(7);
#if SVL_TRACE_BUILD
    if (trace && tid == 0) {
        uint64_t tnow;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
        trace[15] = tnow;
    }
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

template <int D, int NB>
cudaError_t prepare_decode_t() {
    using SM = DecodeSmem<D, NB>;
    static bool attr_done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && attr_done[dev]) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<D, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM::BYTES);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(decode_kernel<D, NB>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess) e = set_max_carveout(decode_kernel<D, NB>);
    if (e == cudaSuccess && dev < 64) attr_done[dev] = true;
    return e;
}

template <int D, int NB>
cudaError_t launch_decode_t(const DecodeParams& p, cudaStream_t s) {
    using SM = DecodeSmem<D, NB>;
    cudaError_t e = prepare_decode_t<D, NB>();
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.S, p.B * p.Hkv);
    cfg.blockDim = dim3(NTH);
    cfg.dynamicSmemBytes = SM::BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // see griddepcontrol in the kernel
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    if (p.cluster) {  // the unit's S CTAs merge over DSMEM
        attr[1].id = cudaLaunchAttributeClusterDimension;
        attr[1].val.clusterDim.x = p.S;
        attr[1].val.clusterDim.y = 1;
        attr[1].val.clusterDim.z = 1;
    } else {
        // the grid merge polls other CTAs' partials: every CTA must be resident -- the grid is
        // sized to the co-resident count, and a cooperative launch makes the runtime guarantee it
        attr[1].id = cudaLaunchAttributeCooperative;
        attr[1].val.cooperative = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = p.S > 1 ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, decode_kernel<D, NB>, p);
}

template <int D>
int decode_ctas_per_sm_t() {
    using SM = DecodeSmem<D, 3>;
    if (prepare_decode_t<D, 3>() != cudaSuccess) return 0;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, decode_kernel<D, 3>, NTH, SM::BYTES) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

template <int D>
int decode_max_active_clusters_t(int S) {
    using SM = DecodeSmem<D, 3>;
    if (prepare_decode_t<D, 3>() != cudaSuccess) return 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(S, 1, 1);
    cfg.blockDim = dim3(NTH, 1, 1);
    cfg.dynamicSmemBytes = SM::BYTES;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, decode_kernel<D, 3>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

}  // namespace

int decode_max_active_clusters(int d, int S) {
    static int cache[64][2][17] = {};
    int dev = 0;
    if (S < 1 || S > 16 || cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
    int& c = cache[dev][d == 128][S];
    if (c == 0) {
        c = (d == 128) ? decode_max_active_clusters_t<128>(S) : decode_max_active_clusters_t<64>(S);
        if (c <= 0) c = -1;
    }
    return c;
}

cudaError_t launch_wait_flags(const uint32_t* flags, int P, uint32_t epoch, uint32_t* ws_flags, cudaStream_t s) {
    wait_flags_kernel<<<1, 32, 0, s>>>(flags, P, epoch, ws_flags);
    return cudaGetLastError();
}

cudaError_t launch_decode(const DecodeParams& p, int d, cudaStream_t s) {
    if (p.single_batch) return d == 128 ? launch_decode_t<128, 1>(p, s) : launch_decode_t<64, 1>(p, s);
    return d == 128 ? launch_decode_t<128, 3>(p, s) : launch_decode_t<64, 3>(p, s);
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
