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
// 1/CS share of the text rows.  512 threads, 226 KB of shared memory, 512 TMEM
// columns per CTA.
//   1. stream: one thread issues 128-row TMA stages (128-B swizzle) into a ring;
//      d is split between tcgen05.mma (logits in TMEM) and mma.sync on warps
//      8-15; warps 4-7 fold a running (max, sum) per head.
//   2. LSE: (max, sum) partials pushed to every peer over DSMEM (st.async);
//      every CTA folds the same partials -> identical LSE2[h].
//   3. key pass: relevance = sum over the g heads of exp2(s2 - LSE2[h]) (the
//      exponentials are written back over the logits: they are the decode
//      weights), per-warp 256-bin value-adaptive histograms folded into 16-bit
//      counts and all-gathered; warp 0 finds the threshold bin b*.
//   4. split pipeline (stage 1: no CTA holds more than 64 keys of b*):
//      U, all warps: slots in index order for the rows above b* and the keys of
//        b* (candidates), P rows (bf16 hi + lo), one bulk V copy per row,
//        candidates pushed to every peer;
//      D, warps 0-7: swap-AB mma.sync P.V over the text + above rows as their V
//        lands (overflow batches if a CTA keeps more rows than its staging),
//        then over the candidates the cut keeps; O and l pushed from registers
//        to the owning peers;
//      S, warps 8-15: exact cut among the gathered candidates (one radix pass on
//        key bits 19..12, exact rank inside the cut sub-bin, ties to the lower
//        index) handed to D, then this CTA's kept indices, ascending.
//      Stage 2 (massive ties) / stage 0 (k <= 0 or k >= N_v): the generic exact
//      cluster radix (select_push.cuh) and the batched decode.
//   5. merge: every owner sums its items over the cluster -> out fp32, lse.
// The weights are relative to the GLOBAL normaliser (identical in every CTA),
// so the merge is a plain sum.  HBM traffic per unit: visual K + text K once +
// kept V + text V (+ the V of the cut-bin keys the cut drops).
#include <cooperative_groups.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"
#include "select_fast.cuh"

#ifndef SVL_TRACE_BUILD
#define SVL_TRACE_BUILD 0
#endif
#ifndef SVL_UGATHER_BULK
#define SVL_UGATHER_BULK 1  // U's V rows as one bulk copy each (A/B: 0 = 16-B cp.async per chunk)
#endif
#ifndef SVL_EXP_NOVG
#define SVL_EXP_NOVG 0  // timing experiment: U issues no V copies (wrong results)
#endif
#ifndef SVL_EXP_NOPROW
#define SVL_EXP_NOPROW 0  // timing experiment: U writes no P rows (wrong results)
#endif
#ifndef SVL_EXP_HOTONLY
#define SVL_EXP_HOTONLY 0  // timing experiment: the stage-0/2 and overflow paths compiled out
#endif

namespace svl {

namespace {

constexpr int FT = kFusedThreads;  // 512
constexpr int STAGE_ROWS = 128;    // = UMMA M: one K stage is one tcgen05.mma row block
#ifndef SVL_RING_KB
#define SVL_RING_KB 192
#endif
constexpr int RING = SVL_RING_KB * 1024;
constexpr int TMAX = kFusedTextMax;
constexpr int UMMA_N = 16;        // q columns per KV group (g <= 16, zero padded)
constexpr int TMEM_COLS = 512;    // [0, 256): tcgen05 half of d, [256, 512): mma.sync half; 16 cols per stage
constexpr int LDS_COL = 256;

// Stage-1 selection state of the split pipeline (fresh_kernel, after the threshold bin).
struct LeanSmem {
    uint2 cand[16][kFastCandPerCta];  // every CTA's keys of the threshold bin: (key, unit index)
    uint2 hdr[16];                    // every CTA's (rows above the threshold bin, candidates)
    uint32_t rhist[256];              // resolve radix: candidate key bits 19..12
    uint32_t ccnt[64];                // per 32-row chunk: rows above | candidates << 16
    int32_t attc[kFastCandPerCta];    // own candidate -> local row
    uint32_t wsum[8];
    uint32_t bc[16];                  // b*, keys left in b*, stage, own rows above, own candidates; sub-bin, above
    uint2 cut;                        // the last kept candidate (key, unit index)
    uint32_t nsub, offc;
    uint32_t sbc[8][2];               // per S warp: sub-bin, keys above it
    uint32_t kmask[2];                // own kept candidates (bit j = candidate j)
    uint16_t nab[kFastCandPerCta];    // candidate j: rows above b* before it
    uint16_t ncb[2048];               // above row i: candidates before it
};

template <int D, int NT>
struct FGeom {
    static constexpr int NCP = 8 * NT;
    static constexpr int SMAX = kFusedSliceMax / NT;
    static constexpr int ROWB = 2 * D;
    static constexpr int STAGE_BYTES = STAGE_ROWS * ROWB;
    static constexpr int TXT_BYTES = kFusedTextMax * ROWB;            // the CTA's text rows (own buffer)
    static constexpr int NST = (RING - TXT_BYTES) / STAGE_BYTES;      // visual K ring stages
    static constexpr int TXT_OFF = NST * STAGE_BYTES;
    static_assert(TXT_OFF + TXT_BYTES <= RING, "text buffer after the ring");
    static_assert(SMAX / STAGE_ROWS * UMMA_N <= LDS_COL, "visual stages fit the TMEM allocation");
    // persistent regions
    static constexpr int QT_OFF = RING;                        // q tile [16][D], K-major SW128 (UMMA B)
    static constexpr int QT_BYTES = UMMA_N * ROWB;
    static constexpr int TXL_OFF = QT_OFF + QT_BYTES;          // text-row logits [TMAX][NCP] fp32
    static constexpr int ATT_OFF = TXL_OFF + TMAX * NCP * 4;   // V slot -> local row
    static constexpr int ATT_BYTES = (SMAX + TMAX) * 4;
    static constexpr int MISC_OFF = ATT_OFF + ATT_BYTES;
    static constexpr int NVS_MAX = SMAX / STAGE_ROWS;
    static constexpr int MISC_BYTES = 2 * NST * 8 + 2 * NVS_MAX * 8 + 8 + 8 + 56 + (FT / 32) * NCP * 8 + 16 * NCP * 8 + NCP * 4 +
                                      16 * 4 + 64 * 4 + 64 * 8;
    static constexpr int RCV_OFF = MISC_OFF + MISC_BYTES;       // merge receive [CS][per] + l [16][16] fp32
    static constexpr int RCV_FLOATS = 16 * D + 32;              // CS * per <= g D + 2 CS (per even)
    static constexpr int BYTES = RCV_OFF + (RCV_FLOATS + 256) * 4;
    // ring re-use once streaming is over
    static constexpr int SEL_OFF = 0;                      // FastSelSmem
    static constexpr int KEYS_OFF = 44 * 1024;             // keys [SMAX]; then slot_of [SMAX] uint16
    static constexpr int STATE_OFF = KEYS_OFF + SMAX * 4;  // per-row state [SMAX]
    static constexpr int VST_OFF = 56 * 1024;              // V staging [VCAP][D], rows padded by 16 B
    static constexpr int VROWB = ROWB + 16;                // (conflict-free ldmatrix without a swizzle)
    static constexpr int VCAP = ((RING - VST_OFF) / VROWB) / 16 * 16 > 512 ? 512 : ((RING - VST_OFF) / VROWB) / 16 * 16;
    static constexpr int PUSH_OFF = VST_OFF;               // generic top-k scratch (fallback only)
    static constexpr int WHIST_OFF = RING - 16 * 1024;     // private histograms (before any selected-row V)
    static_assert(VST_OFF + TMAX * VROWB <= WHIST_OFF, "text-row V below the private histograms");
    static constexpr int PT_OFF = 0;                       // P table hi + lo [VCAP][16] (after top-k)
    static constexpr int OCTA_OFF = PT_OFF + 2 * VCAP * 16 * 2;  // CTA O [16][D] fp32
    static constexpr int LRED_OFF = OCTA_OFF + 16 * D * 4;       // [FT] fp32
    static_assert(STATE_OFF + SMAX <= VST_OFF, "keys + state below the V staging");
    static_assert(VST_OFF + VCAP * VROWB <= RING, "V staging inside the ring");
    static_assert(LRED_OFF + FT * 4 <= KEYS_OFF, "P table / O / l scratch below keys, state, slot_of");
    static_assert(RING % 1024 == 0 && QT_OFF % 1024 == 0, "128-B swizzle atoms are 1024-B aligned");
    // split pipeline (stage 1): P table [VCL][16] hi + lo, then LeanSmem, below the keys;
    // the gathered histograms and the resolve's sub-bin list in parts of the V staging /
    // private histograms that are dead by then
    static constexpr int LS_BYTES = (int)sizeof(LeanSmem);
    static constexpr int VCL0 = (KEYS_OFF - LS_BYTES) / 64 / 16 * 16;
    static constexpr int VCL1 = (WHIST_OFF - VST_OFF) / VROWB / 16 * 16;
    static constexpr int VCL = VCL0 < VCL1 ? (VCL0 < 512 ? VCL0 : 512) : (VCL1 < 512 ? VCL1 : 512);
    static constexpr int LPT_OFF = 0;
    static constexpr int LS_OFF = VCL * 64;
    static constexpr int LHIST_OFF = (VST_OFF + TMAX * VROWB + 1023) / 1024 * 1024;
    static constexpr int LSUB_OFF = WHIST_OFF;
    static_assert(LS_OFF + LS_BYTES <= KEYS_OFF, "P table + LeanSmem below the keys");
    static_assert(STATE_OFF + 2 * SMAX <= VST_OFF, "slot_of below the V staging");
    static_assert(LHIST_OFF + 16 * 1024 <= WHIST_OFF, "gathered histograms above the text rows' V");
    static_assert(VST_OFF + VCL * VROWB <= WHIST_OFF, "split-pipeline V staging below the sub-bin list");
    static_assert(LSUB_OFF + 2 * 16 * kFastCandPerCta * 8 <= RING, "the two cut-select member lists inside the ring");
    static_assert(16 * D * 4 + FT * 4 <= VCL * 64, "O + l scratch over the dead P table");
    static_assert(SMAX <= 2048 && VCL >= kFusedTextMax + kFastCandPerCta + 16, "chunk counts / batch sizes");
};


template <int D, int NT>
__global__ void __launch_bounds__(FT, 1) fresh_kernel(const __grid_constant__ FreshParams p) {
    using GM = FGeom<D, NT>;
    constexpr int NCP = GM::NCP, NST = GM::NST, ROWB = GM::ROWB, VCAP = GM::VCAP;
    constexpr int NCH = D / 32;  // 16-byte chunks per thread per row (permuted contraction)
    constexpr int CH = D / 8;    // 16-byte chunks per row
    constexpr uint32_t IDESC = umma_idesc_bf16(STAGE_ROWS, UMMA_N);
    static_assert(sizeof(FastSelSmem) <= GM::KEYS_OFF, "fast top-k scratch");
    static_assert(GM::PUSH_OFF + sizeof(PushTopkSmem) <= RING, "generic top-k scratch");
    static_assert(GM::BYTES <= 227 * 1024, "shared memory budget");

    extern __shared__ __align__(1024) uint8_t smem[];
    // phase stamps exist only in SVL_TRACE_BUILD builds: elsewhere the pointer is a
    // compile-time null and every stamp (and its code) disappears
    uint64_t* const trace_out = SVL_TRACE_BUILD ? p.trace : nullptr;
    cg::cluster_group cl = cg::this_cluster();
    const int CS = (int)cl.num_blocks();
    const int rank = (int)cl.block_rank();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gid = lane >> 2, t = lane & 3;
    const int q4 = warp & 3;  // this warp's TMEM lane quarter (rows 32*q4 .. 32*q4+31 of a stage)
    const int u = blockIdx.y;
    const int b = u / p.Hkv, G = u % p.Hkv;
    const int g = p.g;

    float* txl = reinterpret_cast<float*>(smem + GM::TXL_OFF);
    int* att = reinterpret_cast<int*>(smem + GM::ATT_OFF);
    uint8_t* misc = smem + GM::MISC_OFF;
    uint64_t* full = reinterpret_cast<uint64_t*>(misc);  // K stage landed
    uint64_t* empty = full + NST;                         // K stage consumed by the tensor core
    uint64_t* accf = empty + NST;                         // [NVS_MAX] stage i's tcgen05 half in TMEM (single use)
    uint64_t* ldsf = accf + GM::NVS_MAX;                  // [NVS_MAX] stage i's mma.sync half in TMEM (8 warps)
    uint64_t* mrg = ldsf + GM::NVS_MAX;                    // merge: CS remote arrivals
    uint64_t* vbar = ldsf + GM::NVS_MAX + 1;              // V gathers (TMA variant)
    uint32_t* tslot = reinterpret_cast<uint32_t*>(vbar + 1);                   // TMEM base address
    uint64_t* tfull = vbar + 2;                                                 // text rows landed
    uint64_t* xbar = vbar + 3;  // [5] LSE, histograms, candidates (st.async byte counts); split pipeline: slots, V
    float2* wpart = reinterpret_cast<float2*>(vbar + 8);                        // [16][NCP]
    float2* allpart = wpart + (FT / 32) * NCP;                   // [16][NCP] pushed by the peers
    float* lse2 = reinterpret_cast<float*>(allpart + 16 * NCP);  // [NCP]
    float* lh = lse2 + NCP;                                      // [16]
    int* ibc = reinterpret_cast<int*>(lh + 16);                  // broadcasts
    uint64_t* trs = reinterpret_cast<uint64_t*>(ibc + 64);       // debug stamps (SVL_TRACE), flushed at exit
    const uint32_t ring = smem_u32(smem);
    const uint32_t vst = ring + GM::VST_OFF;
    const uint32_t qt = ring + GM::QT_OFF;
    uint32_t* keys_s = reinterpret_cast<uint32_t*>(smem + GM::KEYS_OFF);
    uint16_t* slot_of = reinterpret_cast<uint16_t*>(smem + GM::KEYS_OFF);  // after the top-k
    uint8_t* state_s = smem + GM::STATE_OFF;
    FastSelSmem& fs = *reinterpret_cast<FastSelSmem*>(smem + GM::SEL_OFF);
    // stamps: SM cycles (clock64, one counter for every warp of the SM); slots 0 and 10 also
    // the global timer (CTA alignment), slots 30 / 31 the cycle counter at those two points
#define SVL_TRACE(ph)                                                                     \
    if (trace_out && tid == 0) {                                                          \
        uint64_t tnow;                                                                    \
        if ((ph) == 0 || (ph) == 10)                                                      \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow)::"memory");            \
        else                                                                              \
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(tnow)::"memory");               \
        trs[(ph)] = tnow;                                                                 \
    }
    auto tstamp = [&](int slot) {  // stamp from the calling thread (debug builds)
        if (trace_out) {
            uint64_t tnow;
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(tnow)::"memory");
            trs[slot] = tnow;
        }
    };
    if (trace_out && tid < 64) trs[tid] = 0;
    SVL_TRACE(0);
    if (trace_out && tid == 0) {
        uint64_t c0;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(c0)::"memory");
        trs[30] = c0;
    }

    // ------------------------------------------------------------ geometry
    // Programmatic dependent launch: the prologue (barrier init, TMEM allocation, L2
    // prefetch of the first visual stages) overlaps the previous kernel's tail; every
    // read of data an upstream kernel may write (seq_len, q, K, V) follows the wait.
    const int slice = p.slice;
    const int v0 = min(p.nv, rank * slice);
    const int nvis = min(p.nv, v0 + slice) - v0;
    // visual stages through the ring (tiled TMA, 128-B swizzle, tcgen05); the text rows
    // go to their own buffer (own barrier): sharing a ring slot with them made the
    // consumers that skip the text rows wait on a parity that a still-pending fill
    // satisfied (a barrier fault / stale logits when the text copy landed late)
    static_assert(TMAX <= STAGE_ROWS, "text rows fit one stage");
    const int nvs = (nvis + STAGE_ROWS - 1) / STAGE_ROWS;
    const int nstages = nvs;
    int L = 0, T = 0, t0 = 0, ntext = 0;  // set after griddepcontrol.wait
    const uint16_t* Kb = p.K + (int64_t)b * p.ksb + (int64_t)G * p.ksh;
    const uint16_t* Vb = p.V + (int64_t)b * p.vsb + (int64_t)G * p.vsh;
    auto work_row = [&](int w) {  // local work row -> cache row
        if (w < nvis) return p.vb + v0 + w;
        const int tt = t0 + (w - nvis);
        return tt < p.vb ? tt : tt + p.nv;
    };
    const uint32_t vbar_a = smem_u32(vbar);
#ifndef SVL_VGATHER_CPASYNC
#define SVL_VGATHER_CPASYNC 1  // measured: 30.9 vs 32.3 us/layer for TMA row copies (long-video)
#endif
#if SVL_VGATHER_CPASYNC
    // V gather of slots [s0, s1) (slot -> local row in att[]): cp.async 16-B chunks
    // over all 512 threads (LSU path); completion per thread (wait_group) + a CTA barrier
    auto gather_rows = [&](int s0, int s1, int base) {
        for (int e = tid; e < (s1 - s0) * CH; e += FT) {
            const int sl = s0 + e / CH, c = e % CH;
#if SVL_DEBUG_TRAP  // debug builds: a V slot must name a row of this CTA's work list
            if (att[sl] < 0 || att[sl] >= nvis + ntext || work_row(att[sl]) < 0 || work_row(att[sl]) >= L) __trap();
#endif
            cp_async16(vst + (sl - base) * GM::VROWB + c * 16, Vb + (int64_t)work_row(att[sl]) * p.vst + c * 8, true);
        }
        cp_async_commit();
    };
    auto v_expect = [&](uint32_t) {};
    auto v_wait = [&](uint32_t) {
        cp_async_wait<0>();
        cta_sync();
    };
#else
    // one TMA bulk copy per row, one issuing lane per warp (a bulk copy is a
    // uniform-datapath instruction: 32 active lanes would issue serially)
    auto gather_rows = [&](int s0, int s1, int base) {
        if (lane == 0)
            for (int sl = s0 + warp; sl < s1; sl += FT / 32)
                bulk_g2s(vst + (sl - base) * GM::VROWB, Vb + (int64_t)work_row(att[sl]) * p.vst, ROWB, vbar_a);
    };
    auto v_expect = [&](uint32_t bytes) {
        if (tid == 0) mbar_arrive_expect_tx(vbar_a, bytes);
    };
    auto v_wait = [&](uint32_t ph) { mbar_wait(vbar_a, ph); };
#endif

    // ------------------------------------------------ 1. stream K, logits -> TMEM
    // Visual stage i = cache rows vb + v0 + [128 i, 128 i + 128), loaded by the
    // tiled TMA (tensor map, 128-B swizzle) into ring slot i % NST; one
    // tcgen05.mma chain (M = 128 rows, N = 16 q columns, K = d) writes its dot
    // products to TMEM columns [16 i, 16 i + 16) -- the logits stay there for
    // the whole kernel (no shared-memory copy, so the ring can be deep).
    // Warp roles: w0 lane 0 = TMA producer, w1 lane 0 = MMA issuer (first half of
    // d -> TMEM columns [16 i, 16 i + 16)), w2 = TMEM owner, w8-15 = the text stage
    // (plain rows, mma.sync, logits to smem) and then the second half of d of every
    // visual stage by mma.sync from the swizzled stage -> TMEM columns LDS_COL + 16 i
    // (splitting d between the two datapaths: the tensor core's smem read of A is
    // the stream's bottleneck), w4-7 = running LSE of the visual rows from TMEM.
    int nsys = 0;
    auto issue = [&](int i) {  // visual stage i -> ring slot i % NST
        const int slot = i % NST;
        const uint32_t dst0 = ring + slot * GM::STAGE_BYTES;
        const uint32_t bar = smem_u32(&full[slot]);
        // 128 visual rows x D: D/64 boxes of 128 rows x 128 B (rows past the slice
        // are loaded and ignored; past the capacity the TMA zero-fills)
        mbar_arrive_expect_tx(bar, (uint32_t)GM::STAGE_BYTES);
#pragma unroll
        for (int hf = 0; hf < D / 64; ++hf)
            tma_load_4d(dst0 + hf * (STAGE_ROWS * 128), &p.ktmap, hf * 64, p.vb + v0 + i * STAGE_ROWS, G, b, bar);
    };
    auto issue_text = [&]() {  // text rows [t0, t0 + ntext): system rows, then after-visual rows
        const uint32_t dst0 = ring + GM::TXT_OFF;
        const uint32_t bar = smem_u32(tfull);
        mbar_arrive_expect_tx(bar, (uint32_t)(ntext * ROWB));
        const int seg_n[2] = {nsys, ntext - nsys};
        const int seg_row0[2] = {t0, t0 + nsys + p.nv};
        int w = 0;
#pragma unroll
        for (int sg = 0; sg < 2; ++sg) {
            if (seg_n[sg] <= 0) continue;
            if (p.kst == D) {
                bulk_g2s(dst0 + w * ROWB, Kb + (int64_t)seg_row0[sg] * p.kst, (uint32_t)(seg_n[sg] * ROWB), bar);
            } else {
                for (int r = 0; r < seg_n[sg]; ++r)
                    bulk_g2s(dst0 + (w + r) * ROWB, Kb + (int64_t)(seg_row0[sg] + r) * p.kst, ROWB, bar);
            }
            w += seg_n[sg];
        }
    };
    if (warp == 0) {
        if (lane == 0) {
            for (int s = 0; s < NST; ++s) {
                mbar_init(smem_u32(&full[s]), 1);
                mbar_init(smem_u32(&empty[s]), 1 + 8);  // tcgen05 commit + the 8 LDS warps
            }
            for (int s = 0; s < GM::NVS_MAX; ++s) {
                mbar_init(smem_u32(&accf[s]), 1);
                mbar_init(smem_u32(&ldsf[s]), 8);
            }
            mbar_init(vbar_a, 1);
            mbar_init(smem_u32(tfull), 1);
            // every exchange barrier: one local arrival + the bytes the peers will store
            mbar_init(smem_u32(&xbar[0]), 1);
            mbar_arrive_expect_tx(smem_u32(&xbar[0]), (uint32_t)(CS * NCP * 8));
            mbar_init(smem_u32(&xbar[1]), 1);  // top-k histograms: CS x 512 B
            mbar_arrive_expect_tx(smem_u32(&xbar[1]), (uint32_t)(CS * 512));
            mbar_init(smem_u32(&xbar[2]), 1);  // top-k candidates (armed once their count is known)
            mbar_init(smem_u32(&xbar[3]), FT);  // split pipeline: every thread's slots / P rows
            mbar_init(smem_u32(&xbar[4]), SVL_UGATHER_BULK ? 2 * FT : FT);  // ... and its V copies
            {
                const int items = g * D, per = (((items + CS - 1) / CS) + 1) & ~1;  // (as the merge)
                const int mine = max(0, min(per, items - rank * per));
                mbar_init(smem_u32(mrg), 1);
                mbar_arrive_expect_tx(smem_u32(mrg), (uint32_t)(CS * (mine + 16) * 4));
            }
            fence_mbar_init();
            // before the PDL wait only L2 prefetches of the first stages (a hint: the data
            // is read into shared memory after the wait, so an upstream kernel that writes
            // visual K rows -- svl_rope_remap, svl_pack_kv -- is always seen)
#ifndef SVL_L2PF_STAGES
#define SVL_L2PF_STAGES 0  // measured (28-layer graph, long-video): 0 stages 29.17, NST 29.50, all 16 30.50 us/layer
#endif
            for (int i = 0; i < min(SVL_L2PF_STAGES, nstages); ++i)
#pragma unroll
                for (int hf = 0; hf < D / 64; ++hf)
                    tma_prefetch_4d(&p.ktmap, hf * 64, p.vb + v0 + i * STAGE_ROWS, G, b);
        }
        __syncwarp();
    }
    if (warp == 2) tmem_alloc(smem_u32(tslot), TMEM_COLS);
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the upstream grid has completed
    L = p.seq_len[b];
    if (L < p.vb + p.nv + 1 || L > p.capacity) {
        if (tid == 0 && rank == 0) raise_flag(p.flags, 4u /*SPAN*/);
        L = min(max(L, p.vb + p.nv + 1), p.capacity);
    }
    T = p.vb + (L - p.vb - p.nv);
    t0 = (int)((int64_t)rank * T / CS);
    ntext = (int)((int64_t)(rank + 1) * T / CS) - t0;
    if (ntext > TMAX) {
        if (tid == 0) raise_flag(p.flags, 4u /*SPAN*/);
        ntext = TMAX;
    }
    nsys = max(0, min(ntext, p.vb - t0));
    // the private top-k histograms lie past the text rows' K buffer: zeroed during the stream
    const bool zero_early = GM::TXT_OFF + ntext * ROWB <= GM::WHIST_OFF;
    if (warp == 0) {
        if (lane == 0) {
            for (int i = 0; i < min(NST, nstages); ++i) issue(i);  // the first visual stages
            issue_text();  // the text rows (none: completes at once)
        }
        __syncwarp();
    }
    // q tile (UMMA B operand): row c = head G*g + c (zero for c >= g), K-major,
    // 128-B swizzle: chunk j of row r in half h at h*16*128 + r*128 + ((j ^ (r & 7)) << 4)
    for (int e = tid; e < UMMA_N * CH; e += FT) {
        const int r = e / CH, cf = e % CH, hf = cf >> 3, c = cf & 7;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (r < g) v = reinterpret_cast<const uint4*>(p.q + ((int64_t)b * p.H + G * g + r) * D)[cf];
        *reinterpret_cast<uint4*>(smem + GM::QT_OFF + hf * (UMMA_N * 128) + r * 128 + ((c ^ (r & 7)) << 4)) = v;
    }
    fence_proxy_async_smem();
    tc_fence_before();
    cta_sync();
    tc_fence_after();
    const uint32_t tbase = *tslot;
    cluster_arrive_relaxed();  // this CTA is resident: peers may push into it after their cluster_wait
    const bool text_in_lse = !(p.flags_in & 1u /*VISUAL_ONLY*/);
    // Full raw q.K of visual row i*128 + 32*q4 + lane (warp-collective): the tcgen05
    // half (lane = row) plus the mma.sync half, which the LDS warps stored in their
    // fragment order -- row q of a 16-row tile sits at lane perm^-1(q & 7) + (q & 8).
    const int lsrc = (lane & 16) | (lane & 8) | (((lane & 3) << 1) | ((lane >> 2) & 1));
    auto load_logits = [&](int i, float (&x)[16]) {
        uint32_t a[16], c[16];
        tmem_ld16(tbase + ((uint32_t)(q4 * 32) << 16) + i * UMMA_N, a);
        tmem_ld16(tbase + ((uint32_t)(q4 * 32) << 16) + LDS_COL + i * UMMA_N, c);
#pragma unroll
        for (int k = 0; k < 16; ++k)
            x[k] = __uint_as_float(a[k]) + __uint_as_float(__shfl_sync(0xffffffffu, c[k], lsrc));
    };
    // after the stream the LSE warps have written the sums back to columns [16 i, 16 i + 16)
    auto load_full = [&](int i, float (&x)[16]) {
        uint32_t a[16];
        tmem_ld16(tbase + ((uint32_t)(q4 * 32) << 16) + i * UMMA_N, a);
#pragma unroll
        for (int k = 0; k < 16; ++k) x[k] = __uint_as_float(a[k]);
    };

    if (warp == 0) {
        if (lane == 0)  // producer: refill a slot once the tensor core has consumed it
            for (int i = NST; i < nstages; ++i) {
                mbar_wait(smem_u32(&empty[i % NST]), ((i / NST) - 1) & 1);
                issue(i);
            }
        __syncwarp();
    } else if (warp == 1) {
        if (lane == 0) {
            for (int i = 0; i < nvs; ++i) {
                const int slot = i % NST;
                mbar_wait(smem_u32(&full[slot]), (i / NST) & 1);
                tc_fence_after();
                if (trace_out && i < 32) {
                    uint64_t tnow;
                    asm volatile("mov.u64 %0, %%clock64;" : "=l"(tnow)::"memory");
                    trs[32 + i] = tnow;
                }
                const uint32_t sb = ring + slot * GM::STAGE_BYTES;
#if !SVL_EXP_NOMATH  // timing experiment: stream only
#pragma unroll
                for (int j = 0; j < D / 32; ++j) {  // K = 16 per instruction, d in [0, D/2)
                    const int hf = j >> 2, kk = j & 3;
                    umma_bf16(tbase + i * UMMA_N, sw128_desc(sb + hf * (STAGE_ROWS * 128) + kk * 32),
                              sw128_desc(qt + hf * (UMMA_N * 128) + kk * 32), IDESC, j > 0 ? 1u : 0u);
                }
#endif
                umma_commit(smem_u32(&empty[slot]));
                umma_commit(smem_u32(&accf[i]));
            }
#if SVL_EXP_DRAIN
            // no asynchronous arrival may target this CTA's barriers after it exits:
            // wait for the final phase of every ring slot (commit + LDS warps)
            for (int st = max(0, nstages - NST); st < nstages; ++st)
                mbar_wait(smem_u32(&empty[st % NST]), (st / NST) & 1);
#endif
        }
        __syncwarp();
    } else if (warp == 3) {
        if (zero_early)
            for (int i = lane; i < (FT / 32) * 64; i += 32)
                reinterpret_cast<uint4*>(smem + GM::WHIST_OFF)[i] = make_uint4(0u, 0u, 0u, 0u);
    } else if (warp >= 4 && warp < 8) {
        // running (max, sum) of the visual logits, one TMEM lane (= stage row) per thread
        float rm[NCP], rl[NCP];
#pragma unroll
        for (int c = 0; c < NCP; ++c) rm[c] = -INFINITY, rl[c] = 0.f;
        for (int i = 0; i < nvs; ++i) {
            mbar_wait(smem_u32(&accf[i]), 0);
            mbar_wait(smem_u32(&ldsf[i]), 0);
            __syncwarp();  // lanes leave the spin at different times; tcgen05.ld is .aligned
            tc_fence_after();
            float x[16];
            load_logits(i, x);
            tmem_st16(tbase + ((uint32_t)(q4 * 32) << 16) + i * UMMA_N, x);  // full q.K for the later passes
            if (i * STAGE_ROWS + q4 * 32 + lane < nvis) {
#pragma unroll
                for (int c = 0; c < NCP; ++c) {
#ifndef SVL_LSE_ONE_EXP
#define SVL_LSE_ONE_EXP 1  // measured: 29.29 -> 28.81 us/layer (long-video 28-layer graph)
#endif
#if SVL_LSE_ONE_EXP
                    // one exponential per element: e = exp2(-|y - m|) rescales whichever side
                    // is smaller (y finite; m starts at -inf: d = +inf, e = 0 -> l = 1)
                    const float y = x[c] * p.scale2;
                    const float dd = y - rm[c];
                    const float e = fast_exp2(-fabsf(dd));
                    rl[c] = (dd > 0.f) ? fmaf(rl[c], e, 1.f) : rl[c] + e;
                    rm[c] = fmaxf(rm[c], y);
#else
                    const float y = x[c] * p.scale2;
                    const float M = fmaxf(rm[c], y);
                    rl[c] = rl[c] * fast_exp2(rm[c] - M) + fast_exp2(y - M);
                    rm[c] = M;
#endif
                }
            }
        }
        if (warp == 4 && lane == 0) tstamp(13);
        // warp fold: the max first (shuffles only), then each lane's sum rescaled to it
        // once and summed (one exponential per column instead of one per level)
#pragma unroll
        for (int c = 0; c < NCP; ++c) {
            float M = rm[c];
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, off));
            float l = (M == -INFINITY) ? 0.f : rl[c] * fast_exp2(rm[c] - M);
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) l += __shfl_xor_sync(0xffffffffu, l, off);
            rm[c] = M;
            rl[c] = l;
            if (lane == 0) wpart[warp * NCP + c] = make_float2(rm[c], rl[c]);
        }
        if (warp == 4 && lane == 0) tstamp(14);
    } else if (warp >= 8) {
        // visual stages, second half of d: warp w takes tile j = 2 (w % 4) + (w - 8) / 4
        // (rows 16 j .. 16 j + 15 lie in its TMEM lane quarter w % 4), mma.sync from the
        // swizzled stage, then adds the tcgen05 half from TMEM and writes the sum back;
        // the tensor core's shared-memory read of A is the stream's bottleneck, so
        // splitting d between the two datapaths shortens every stage.  Then the text
        // stage (plain rows, all of d) on the same warps.
        const int wig = warp - 8, r16v = 16 * (2 * (warp & 3) + (wig >> 2)), r16 = wig * 16;
        float rm[NT][2], rl[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) rm[nt][0] = rm[nt][1] = -INFINITY, rl[nt][0] = rl[nt][1] = 0.f;
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
        auto lse_fold = [&](int nt, float ya, float yb, int e2) {
            const float mx = fmaxf(ya, yb);
            if (mx != -INFINITY) {
                const float M = fmaxf(rm[nt][e2], mx);
                rl[nt][e2] = rl[nt][e2] * fast_exp2(rm[nt][e2] - M) + fast_exp2(ya - M) + fast_exp2(yb - M);
                rm[nt][e2] = M;
            }
        };
        // A rows ra = tile row pa, rb = pa + 8, pa = perm(gid): the two rows of a
        // quarter-warp are 4 apart, so their XOR-swizzled chunks fall in disjoint bank
        // halves.  TMEM (16x256b) holds rows gid / gid + 8 per thread: exchange by shuffle.
        const int pa = ((gid & 1) << 2) | (gid >> 1);
        const int src_ld = ((pa << 2) | t);                                   // holder of TMEM row pa
        const int src_st = (((((gid & 3) << 1) | (gid >> 2))) << 2) | t;      // holder of row gid (perm^-1)
        // text stage (stage 0, slot 0): 8 warps x 16 rows, mma.sync over all of d (swap-AB,
        // permuted contraction); every warp releases the slot, rows or not
        if (r16 < ntext) {
            mbar_wait(smem_u32(tfull), 0);
            __syncwarp();  // mma.sync is .aligned
            const uint32_t base = ring + GM::TXT_OFF + (r16 + gid) * ROWB;
            float acc[NT][2][4];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int h = 0; h < 2; ++h) acc[nt][h][0] = acc[nt][h][1] = acc[nt][h][2] = acc[nt][h][3] = 0.f;
#pragma unroll
            for (int c4 = 0; c4 < NCH; ++c4) {
                const uint4 ra = lds128(base + (t + 4 * c4) * 16);
                const uint4 rb = lds128(base + 8 * ROWB + (t + 4 * c4) * 16);
                const uint32_t a0[4] = {ra.x, rb.x, ra.y, rb.y};
                const uint32_t a1[4] = {ra.z, rb.z, ra.w, rb.w};
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    mma_bf16_16816(acc[nt][c4 & 1], a0, bq[nt][c4].x, bq[nt][c4].y);
                    mma_bf16_16816(acc[nt][c4 & 1], a1, bq[nt][c4].z, bq[nt][c4].w);
                }
            }
            const int ra_ = r16 + gid, rb_ = ra_ + 8;
            const bool va = ra_ < ntext, vbv = rb_ < ntext;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const float x0 = (acc[nt][0][0] + acc[nt][1][0]) * p.scale2;
                const float x1 = (acc[nt][0][1] + acc[nt][1][1]) * p.scale2;
                const float x2 = (acc[nt][0][2] + acc[nt][1][2]) * p.scale2;
                const float x3 = (acc[nt][0][3] + acc[nt][1][3]) * p.scale2;
                if (va) *reinterpret_cast<float2*>(txl + ra_ * NCP + nt * 8 + 2 * t) = make_float2(x0, x1);
                if (vbv) *reinterpret_cast<float2*>(txl + rb_ * NCP + nt * 8 + 2 * t) = make_float2(x2, x3);
                if (text_in_lse) {
                    lse_fold(nt, va ? x0 : -INFINITY, vbv ? x2 : -INFINITY, 0);
                    lse_fold(nt, va ? x1 : -INFINITY, vbv ? x3 : -INFINITY, 1);
                }
            }
        }
        for (int i = 0; i < nvs; ++i) {
            const int slot = i % NST;
            mbar_wait(smem_u32(&full[slot]), (i / NST) & 1);
            __syncwarp();  // mma.sync is .aligned
            const uint32_t sbase = ring + slot * GM::STAGE_BYTES;
            float acc[NT][4];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
            {
                const int rA = r16v + pa;  // rA & 7 == pa
                uint4 ra[NCH / 2], rb[NCH / 2];
#pragma unroll
                for (int c4 = NCH / 2; c4 < NCH; ++c4) {
                    const int hf = c4 >> 1, cc = t + 4 * (c4 & 1);
                    const uint32_t hb = sbase + hf * (STAGE_ROWS * 128) + ((cc ^ pa) << 4);
                    ra[c4 - NCH / 2] = lds128(hb + rA * 128);
                    rb[c4 - NCH / 2] = lds128(hb + (rA + 8) * 128);
                }
#pragma unroll
                for (int c4 = NCH / 2; c4 < NCH; ++c4) {
                    const uint4 x = ra[c4 - NCH / 2], y = rb[c4 - NCH / 2];
                    const uint32_t a0[4] = {x.x, y.x, x.y, y.y};
                    const uint32_t a1[4] = {x.z, y.z, x.w, y.w};
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) {
                        mma_bf16_16816(acc[nt], a0, bq[nt][c4].x, bq[nt][c4].y);
                        mma_bf16_16816(acc[nt], a1, bq[nt][c4].z, bq[nt][c4].w);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&empty[slot]));  // this warp's reads of the slot are done
            // raw partial to TMEM in fragment order (rows gid / gid + 8 hold tile rows pa / pa + 8)
            {
                float fr[8];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    fr[e] = acc[0][e];
                    fr[4 + e] = (NT > 1) ? acc[NT - 1][e] : 0.f;
                }
                tmem_st16x256_x2(tbase + ((uint32_t)r16v << 16) + LDS_COL + i * UMMA_N, fr);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&ldsf[i]));
            if (trace_out && tid == 256 && i < 8) {
                uint64_t tnow;
                asm volatile("mov.u64 %0, %%clock64;" : "=l"(tnow)::"memory");
                trs[48 + i] = tnow;
            }
        }
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
        if (warp == 8 && lane == 0) tstamp(15);
    }
    if (warp < 4)
        for (int c = lane; c < NCP; c += 32) wpart[warp * NCP + c] = make_float2(-INFINITY, 0.f);
    if (warp == 1 && lane == 0) tstamp(29);
    tc_fence_before();
    cta_sync();  // ring drained: every MMA completed (accf waited), text stage consumed
    tc_fence_after();

    for (int i = tid; i < ntext; i += FT) att[i] = nvis + i;
    SVL_TRACE(1);

    // ------------------------------------------------ 2. cluster LSE
    auto lse_merge = [](float& m, float& l, float m2, float l2) {
        const float M = fmaxf(m, m2);
        if (M != -INFINITY) {
            l = l * fast_exp2(m - M) + l2 * fast_exp2(m2 - M);
            m = M;
        }
    };
    cluster_wait();    // every peer has started (first DSMEM access below)
    if (warp < NCP) {  // warp c folds column c (fixed shuffle tree), lanes push to the peers
        float2 x = (lane < FT / 32) ? wpart[lane * NCP + warp] : make_float2(-INFINITY, 0.f);
#pragma unroll
        for (int off = 1; off < 16; off <<= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, x.x, off);
            const float l2 = __shfl_xor_sync(0xffffffffu, x.y, off);
            lse_merge(x.x, x.y, m2, l2);
        }
        if (lane < CS)
            st_async_f2(mapa_shared(smem_u32(&allpart[rank * NCP + warp]), lane), x.x, x.y,
                        mapa_shared(smem_u32(&xbar[0]), lane));
    }
    // all CS partials landed (this also means every peer has finished its K stream, so
    // the ring region that later exchanges write into is free everywhere)
    mbar_wait(smem_u32(&xbar[0]), 0);
    __syncwarp();
    if (warp < NCP) {
        float2 x = (lane < CS) ? allpart[lane * NCP + warp] : make_float2(-INFINITY, 0.f);
#pragma unroll
        for (int off = 1; off < 16; off <<= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, x.x, off);
            const float l2 = __shfl_xor_sync(0xffffffffu, x.y, off);
            lse_merge(x.x, x.y, m2, l2);
        }
        if (lane == 0) lse2[warp] = x.x + log2f(x.y);
    }
    // text rows' V: V slots [0, ntext); the gather overlaps everything up to the decode
    // (issued after the LSE barrier: a cluster arrive.release waits for in-flight copies;
    // the CTA barrier publishes att[0, ntext) to every gathering thread -- compute-sanitizer
    // racecheck)
    cta_sync();
    gather_rows(0, ntext, 0);
    SVL_TRACE(2);
    // per-thread copies of the normalisers (+inf pads: exp2(x - inf) = 0)
    float nl[NCP];
#pragma unroll
    for (int c = 0; c < NCP; ++c) nl[c] = (c < g) ? lse2[c] : INFINITY;

    // ------------------------------------------------ 3. top-k
    // Relevance keys + per-warp histograms (all warps), one all-gathered 256-bin
    // histogram -> the threshold bin b* (identical in every CTA).  Then, when no CTA
    // holds more than kFastCandPerCta keys of b* (stage 1, the common case), the
    // split pipeline below; otherwise (stage 2: massive ties, b* = the catch-all bin)
    // the generic exact radix and the batched decode; k <= 0 or k >= N_v: stage 0.
    int32_t* idx_out = p.idx_out + (int64_t)u * p.k;
    uint32_t* whist = reinterpret_cast<uint32_t*>(smem + GM::WHIST_OFF);
    FastSelect<FT> sel(cl, fs, nvis, v0, slice, p.nv, p.k, keys_s, state_s, p.flags, whist);
    if (trace_out) sel.tr = trs + 16;
    LeanSmem& ls = *reinterpret_cast<LeanSmem*>(smem + GM::LS_OFF);
    uint32_t* lhist = reinterpret_cast<uint32_t*>(smem + GM::LHIST_OFF);  // [CS][128] gathered histograms (16-bit bin pairs)
    int stage = 0;
    // the key pass's exponentials of this warp's stages (= U3's chunks 16 m + warp), kept in
    // registers for the split pipeline's P rows
    uint32_t lv[32];
    if (!sel.trivial()) {
        if (!zero_early) {  // (the text rows' K buffer reached the private histograms)
            sel.zero_hist();
            cta_sync();
        }
        // relevance of each visual row = its share of the softmax mass, summed over the g heads.
        // A warp's stages (lane quarter warp % 4) are loaded from TMEM at once, one wait: the
        // loop is a latency chain otherwise (load -> exponentials -> key -> histogram)
        {
            constexpr int NI = kFusedSliceMax / NT / STAGE_ROWS / (FT / 128);  // stages per warp
            static_assert(NI * NCP == 32, "32 logit registers per thread");
#pragma unroll
            for (int m = 0; m < NI; ++m) {
                const int i = (warp >> 2) + 4 * m;
                if (i < nvs) {
                    const uint32_t ta = tbase + ((uint32_t)(q4 * 32) << 16) + i * UMMA_N;
                    if constexpr (NCP == 8) tmem_ld8_nowait(ta, lv + m * NCP);
                    else tmem_ld16_nowait_p(ta, lv + m * NCP);
                }
            }
            tmem_wait_ld_tie(lv);
            // the exponentials p = exp2(s2 - LSE2[h]) replace the logits in TMEM: they are the
            // decode weights of the rows that get kept (U and the stage-0/2 path read them back)
#pragma unroll
            for (int m = 0; m < NI; ++m) {
                const int i = (warp >> 2) + 4 * m;
                const int row = i * STAGE_ROWS + q4 * 32 + lane;
                float sc = 0.f;
#pragma unroll
                for (int c = 0; c < NCP; ++c) {
                    const float pc = fast_exp2(__uint_as_float(lv[m * NCP + c]) * p.scale2 - nl[c]);
                    lv[m * NCP + c] = __float_as_uint(pc);
                    sc += pc;
                }
                if (i < nvs) {
                    const uint32_t ta = tbase + ((uint32_t)(q4 * 32) << 16) + i * UMMA_N;
                    if constexpr (NCP == 8) tmem_st8_nowait(ta, lv + m * NCP);
                    else tmem_st16_nowait(ta, lv + m * NCP);
                    if (row < nvis) sel.add_key(row, sc);
                }
            }
            tmem_wait_st();
        }
        if (sel.nan_seen) raise_flag(p.flags, 2u /*NONFINITE*/);
        if (tid == 0) tstamp(26);
        tc_fence_before();
        cta_sync();  // private histograms complete
        tc_fence_after();
        if (tid == 0) tstamp(27);
        // threads 0..31 fold 8 bins of the 16 private histograms into 16-bit counts (a slice
        // has <= 2048 rows, a unit <= 32768) and push them to every peer: 512 B per histogram
        // (the all-gather's shared-memory port traffic, 2 x CS x 512 B, is on the chain)
        if (tid < 32) {
            uint32_t acc[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
            for (int w = 0; w < FT / 32; ++w) {
                const uint4 h0 = *reinterpret_cast<const uint4*>(whist + w * 256 + 8 * tid);
                const uint4 h1 = *reinterpret_cast<const uint4*>(whist + w * 256 + 8 * tid + 4);
                acc[0] += h0.x, acc[1] += h0.y, acc[2] += h0.z, acc[3] += h0.w;
                acc[4] += h1.x, acc[5] += h1.y, acc[6] += h1.z, acc[7] += h1.w;
            }
            const uint4 pk = make_uint4(acc[0] | (acc[1] << 16), acc[2] | (acc[3] << 16), acc[4] | (acc[5] << 16),
                                        acc[6] | (acc[7] << 16));
            const uint32_t dst = smem_u32(lhist + rank * 128 + 4 * tid), hb = smem_u32(&xbar[1]);
            for (int q = 0; q < CS; ++q) st_async_u4(mapa_shared(dst, q), pk, mapa_shared(hb, q));
        }
        if (warp == 0) {
            // the threshold: bins 8 lane .. 8 lane + 7 summed over the CS histograms (16-bit
            // halves summed in place: a unit's count fits)
            mbar_wait(smem_u32(&xbar[1]), 0);
            __syncwarp();
            if (lane == 0) tstamp(28);
            uint4 sm = make_uint4(0u, 0u, 0u, 0u), mine = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
            for (int q = 0; q < 16; ++q) {  // one 16-B load per histogram, all independent
                if (q < CS) {
                    const uint4 a = *reinterpret_cast<const uint4*>(lhist + q * 128 + 4 * lane);
                    sm.x += a.x, sm.y += a.y, sm.z += a.z, sm.w += a.w;
                    if (q == rank) mine = a;
                }
            }
            uint32_t c[8] = {sm.x & 0xffffu, sm.x >> 16, sm.y & 0xffffu, sm.y >> 16,
                             sm.z & 0xffffu, sm.z >> 16, sm.w & 0xffffu, sm.w >> 16};
            const uint32_t cm[8] = {mine.x & 0xffffu, mine.x >> 16, mine.y & 0xffffu, mine.y >> 16,
                                    mine.z & 0xffffu, mine.z >> 16, mine.w & 0xffffu, mine.w >> 16};
            uint32_t grp = 0u, own = 0u;
#pragma unroll
            for (int i = 0; i < 8; ++i) grp += c[i];
            uint32_t suf = grp;  // keys in bins >= 8 lane
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t y = __shfl_down_sync(0xffffffffu, suf, off);
                if (lane + off < 32) suf += y;
            }
            const unsigned ball = __ballot_sync(0xffffffffu, suf >= (uint32_t)p.k);
            const int lstar = ball ? 31 - __clz(ball) : 0;
            uint32_t above = suf - grp;
            int bl = 8 * lane;
#pragma unroll
            for (int i = 7; i >= 0; --i) {
                if (above + c[i] >= (uint32_t)p.k) {
                    bl = 8 * lane + i;
                    break;
                }
                above += c[i];
            }
            const int bstar = __shfl_sync(0xffffffffu, bl, lstar);
            above = __shfl_sync(0xffffffffu, above, lstar);
            // per-CTA counts of b*, and this CTA's rows above it
            const uint32_t cq = (lane < CS) ? ((lhist[lane * 128 + (bstar >> 1)] >> (16 * (bstar & 1))) & 0xffffu) : 0u;
            uint32_t maxc = cq, totc = cq;
#pragma unroll
            for (int i = 0; i < 8; ++i) own += (8 * lane + i > bstar) ? cm[i] : 0u;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                maxc = max(maxc, __shfl_xor_sync(0xffffffffu, maxc, off));
                totc += __shfl_xor_sync(0xffffffffu, totc, off);
                own += __shfl_xor_sync(0xffffffffu, own, off);
            }
            const int st = (bstar == 0 || maxc > (uint32_t)kFastCandPerCta) ? 2 : 1;
            if (lane == 0) {
                ls.bc[0] = (uint32_t)bstar;
                ls.bc[1] = (uint32_t)p.k - above;  // keys still to keep inside b*
                ls.bc[2] = (uint32_t)st;
                ls.bc[3] = own;
                ls.bc[4] = (lhist[rank * 128 + (bstar >> 1)] >> (16 * (bstar & 1))) & 0xffffu;
                // every CTA's (above, count) header + its candidates
                if (st == 1) mbar_arrive_expect_tx(smem_u32(&xbar[2]), totc * 8u + (uint32_t)CS * 8u);
            }
        }
        else {
            // meanwhile (split pipeline) the text rows' P rows, exp2(s2 - LSE2[h]) as bf16 hi + lo
            // -- they do not depend on the threshold (the stage-2 path rebuilds its own table)
            uint16_t* pth = reinterpret_cast<uint16_t*>(smem + GM::LPT_OFF);
            uint16_t* ptl = pth + GM::VCL * 16;
            for (int i = tid - 32; i < ntext * 16; i += FT - 32) {
                const int rr = i >> 4, h = i & 15;
                float pv = 0.f;
                if (h < g) pv = fast_exp2(txl[rr * NCP + h] - lse2[h]);
                const __nv_bfloat16 hi = __float2bfloat16_rn(pv);
                const __nv_bfloat16 lo = __float2bfloat16_rn(pv - __bfloat162float(hi));
                pth[rr * 16 + h] = *reinterpret_cast<const uint16_t*>(&hi);
                ptl[rr * 16 + h] = *reinterpret_cast<const uint16_t*>(&lo);
            }
        }
        cta_sync();  // threshold published
        stage = (int)ls.bc[2];
    }
    SVL_TRACE(3);

    // ------------------------------------------------ 5. cluster merge layout (plain sums)
    // CTA q owns output items [q*per, (q+1)*per) of the unit's g x D block (per even, so an
    // element pair never straddles two owners); every CTA stores its partial of those items
    // and its 16 l sums straight into the owner's receive buffer with st.async, counted on
    // the owner's mbarrier; the owner waits for the bytes it expects and sums in sender order.
    const int items = g * D;
    const int per = (((items + CS - 1) / CS) + 1) & ~1;
    float* rcv = reinterpret_cast<float*>(smem + GM::RCV_OFF);  // [CS][per]
    float* lrcv = rcv + GM::RCV_FLOATS;                          // [16][16]
    const uint32_t rcv_a = smem_u32(rcv), lrcv_a = smem_u32(lrcv), mrg_a = smem_u32(mrg);
    int fin_threads = FT;  // threads that finish the owned items

    float o[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    if (stage == 1) {
        // ============================================ split pipeline (stage 1)
        // The post-stream chain is latency bound (a CTA barrier ~300 cycles, a cold branch
        // target ~500: tools/icache_probe2.cu), so it is arranged for few barriers:
        // U (all warps, one barrier): slots in index order for the rows above b* (kept for
        //   sure) and the keys of b* (candidates); each warp writes its rows' P, issues their
        //   V gathers and pushes its candidates to every peer.
        // D (warps 0-7): P.V over the text + above rows as soon as their V lands, then over
        //   the candidates once the cut is known; the output partials and the denominators
        //   (an MMA against ones) go from registers straight to the owning peers.
        // S (warps 8-15): the exact cut among the gathered candidates, handed to D, then this
        //   CTA's kept indices (ascending) from prefix counts recorded by U.
        const int bstar = (int)ls.bc[0];
        const uint32_t krem = ls.bc[1];
        const int na_loc = (int)ls.bc[3], nc_loc = (int)ls.bc[4];
        const int candR = (nc_loc + 15) & ~15;
        constexpr int VCL = GM::VCL;
        const int capA = VCL - candR;   // P / V rows of the text + above batches; candidates at [capA, VCL)
        const int nA = ntext + na_loc;  // virtual slots: text rows, then the above rows in index order
        const int n0 = min(nA, capA);
        uint16_t* pth = reinterpret_cast<uint16_t*>(smem + GM::LPT_OFF);
        uint16_t* ptl = pth + VCL * 16;
        uint2* lsub = reinterpret_cast<uint2*>(smem + GM::LSUB_OFF);
        const uint32_t ubar_s = smem_u32(&xbar[3]), ubar_v = smem_u32(&xbar[4]);
        const unsigned lt = (1u << lane) - 1u;
        const int nch = (nvis + 31) >> 5;
        auto cls_of = [&](uint32_t key) -> int {
            const int dg = rel_digit(key);
            return dg > bstar ? 2 : (dg == bstar ? 1 : 0);
        };
        // P row = exp2(s2 - LSE2[h]) of heads h < g (from TMEM) as split bf16 hi + lo, zero padded to 16 heads
        auto vaddr = [&](int r, int cc) -> uint32_t { return vst + (uint32_t)(r * GM::VROWB + cc * 16); };  // staging chunk
        auto zero16 = [](uint32_t a) { asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(a), "r"(0u) : "memory"); };
        auto write_p_row = [&](int prow, const float (&v)[16]) {
            uint32_t hw[8], lw[8];
#pragma unroll
            for (int c2 = 0; c2 < 8; ++c2) {
                hw[c2] = lw[c2] = 0u;
                if (2 * c2 < NCP) {  // (v = the exponentials the key pass left in TMEM)
                    const float pa = v[2 * c2], pb = v[2 * c2 + 1];
                    hw[c2] = pack_bf16(pa, pb);
                    lw[c2] = pack_bf16(pa - bf16lo(hw[c2]), pb - bf16hi(hw[c2]));
                }
            }
            uint4* dh = reinterpret_cast<uint4*>(pth + prow * 16);
            uint4* dl = reinterpret_cast<uint4*>(ptl + prow * 16);
            dh[0] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            dh[1] = make_uint4(hw[4], hw[5], hw[6], hw[7]);
            dl[0] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
            dl[1] = make_uint4(lw[4], lw[5], lw[6], lw[7]);
        };
        // U1: per-chunk counts (chunk c = 32 rows; warp w owns chunks 16 j + w, which lie in
        // its TMEM lane quarter: stage c / 4, quarter c % 4 = w % 4)
        unsigned cba[4], cbc[4];  // this warp's chunks: rows above b*, candidates (reused by U3)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = 16 * j + warp, r = 32 * c + lane;
            const int cl_ = (c < nch && r < nvis) ? cls_of(keys_s[r]) : 0;
            cba[j] = __ballot_sync(0xffffffffu, cl_ == 2);
            cbc[j] = __ballot_sync(0xffffffffu, cl_ == 1);
            if (c < nch && lane == 0) ls.ccnt[c] = (uint32_t)__popc(cba[j]) | ((uint32_t)__popc(cbc[j]) << 16);
        }
        if (warp >= 8) {  // S: zero the resolve scratch (published by the barrier below)
            const int ts = tid - 256;
            ls.rhist[ts] = 0u;
            if (ts == 0) ls.nsub = 0u, ls.offc = 0u;
        }
        cta_sync();  // chunk counts
        SVL_TRACE(56);
        // U2: exclusive prefixes of the chunk counts (every warp scans all 64)
        const uint32_t e0 = (2 * lane < nch) ? ls.ccnt[2 * lane] : 0u;
        const uint32_t e1 = (2 * lane + 1 < nch) ? ls.ccnt[2 * lane + 1] : 0u;
        uint32_t inc = e0 + e1;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, off);
            if (lane >= off) inc += y;
        }
        const uint32_t ex0 = inc - e0 - e1, ex1 = inc - e1;  // prefixes of chunks 2 lane, 2 lane + 1
        if (tid < CS)  // this CTA's header: (rows above b*, candidates)
            st_async_u2(mapa_shared(smem_u32(&ls.hdr[rank]), tid), make_uint2((uint32_t)na_loc, (uint32_t)nc_loc),
                        mapa_shared(smem_u32(&xbar[2]), tid));
        // U3: slots, prefix counts for the emission, P rows, candidate pushes, then the V
        // gathers.  A warp's chunks are its TMEM stages (lane quarter warp % 4): their logits
        // are loaded at once, one wait.
        constexpr int CPW = 32 / NCP;  // chunks per warp (4 for g <= 8, 2 for g <= 16)
        uint32_t vbytes = 0u;          // (bulk-copy variant) this thread's V bytes in flight
        if (tid == 0) tstamp(57);
#pragma unroll
        for (int m = 0; m < CPW; ++m) {
            const int c = 16 * m + warp;
            if (c >= nch) continue;
            const int r = 32 * c + lane;
            const unsigned ba = cba[m], bc = cbc[m];
            if ((ba | bc) == 0u) continue;  // (most chunks: nothing kept; U is issue-bound, 4 warps per SMSP)
            const uint32_t pre = __shfl_sync(0xffffffffu, (c & 1) ? ex1 : ex0, c >> 1);
            const int cl_ = ((ba >> lane) & 1u) ? 2 : (((bc >> lane) & 1u) ? 1 : 0);
            const uint32_t ck = (cl_ == 1) ? keys_s[r] : 0u;
            const int preA = (int)(pre & 0xffffu), preC = (int)(pre >> 16);
            const int ia = preA + __popc(ba & lt), jc = preC + __popc(bc & lt);  // rows above / candidates before r
            int prow = -1;
            if (cl_ == 2) {
                att[ntext + ia] = r;
                ls.ncb[ia] = (uint16_t)jc;
                if (ntext + ia < capA) prow = ntext + ia;
            } else if (cl_ == 1) {
                ls.attc[jc] = r;
                ls.nab[jc] = (uint16_t)ia;
                prow = capA + jc;
                const uint2 cv = make_uint2(ck, (uint32_t)(v0 + r));
                const uint32_t dst = smem_u32(&ls.cand[rank][jc]), cb = smem_u32(&xbar[2]);
                for (int q = 0; q < CS; ++q) st_async_u2(mapa_shared(dst, q), cv, mapa_shared(cb, q));
            }
            if (!SVL_EXP_NOVG && prow >= 0) {
#if SVL_UGATHER_BULK
                // the row's V as one bulk copy (one L2 request stream per row instead of 16
                // single-row 16-B requests per warp instruction), counted on ubar_v
                bulk_g2s(vaddr(prow, 0), Vb + (int64_t)(p.vb + v0 + r) * p.vst, (uint32_t)ROWB, ubar_v);
                vbytes += (uint32_t)ROWB;
#else
                // the row's V: its own lane issues the 16-B copies (no slot lookups)
#pragma unroll
                for (int cc = 0; cc < CH; ++cc)
                    cp_async16(vaddr(prow, cc), Vb + (int64_t)(p.vb + v0 + r) * p.vst + cc * 8, true);
#endif
            }
            if (!SVL_EXP_NOPROW && prow >= 0) {  // P row from the exponentials in TMEM
                float v[16];
#pragma unroll
                for (int k2 = 0; k2 < 16; ++k2) v[k2] = (k2 < NCP) ? __uint_as_float(lv[m * NCP + (k2 < NCP ? k2 : 0)]) : 0.f;
                write_p_row(prow, v);
            }
        }
        __syncwarp();  // this warp's att / attc entries
        if (tid == 0) tstamp(58);
        if (tid == 0) tstamp(59);
        // (the text rows' P rows were written while warp 0 found the threshold)
        // padding rows of the two regions: P = 0 and V = 0 (0 * stale NaN would poison P.V)
        {
            const int npa = ((n0 + 15) & ~15) - n0, npc = candR - nc_loc;
            for (int i = tid; i < (npa + npc) * 2; i += FT) {
                const int rr = (i >> 1) < npa ? n0 + (i >> 1) : capA + nc_loc + ((i >> 1) - npa);
                reinterpret_cast<uint4*>(pth + rr * 16)[i & 1] = make_uint4(0u, 0u, 0u, 0u);
                reinterpret_cast<uint4*>(ptl + rr * 16)[i & 1] = make_uint4(0u, 0u, 0u, 0u);
            }
            for (int i = tid; i < (npa + npc) * CH; i += FT) {
                const int k2 = i / CH, rr = k2 < npa ? n0 + k2 : capA + nc_loc + (k2 - npa);
                zero16(vaddr(rr, i % CH));
            }
        }
        if (tid == 0) tstamp(60);
        mbar_arrive(ubar_s);               // this thread's slots / P rows / prefix counts
        cp_async_mbar_arrive_noinc(ubar_v);  // ... and, once landed, its V copies
#if SVL_UGATHER_BULK
        mbar_arrive_expect_tx(ubar_v, vbytes);  // (its bulk row copies: bytes counted on ubar_v)
#endif
        SVL_TRACE(11);

        if (warp < 8) {
            // ---------------------------------------- D: decode
            // segments: batch 0 (prepared by U), overflow batches (a CTA keeping more rows than
            // the staging holds), the candidates once the cut is known -- one P.V call site
            const int nover = nA > capA ? (nA - capA + capA - 1) / capA : 0;
            float ot[NT][4], lt_[NT][4];  // O^T fragments (d x heads) and, warp 0, l (every row)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) ot[nt][0] = ot[nt][1] = ot[nt][2] = ot[nt][3] = lt_[nt][0] = lt_[nt][1] = lt_[nt][2] = lt_[nt][3] = 0.f;
#pragma unroll 1
            for (int sg = 0; sg <= nover + 1; ++sg) {
                int row0 = 0, nr;
                if (sg == 0) {
                    mbar_wait(ubar_s, 0);
                    mbar_wait(ubar_v, 0);
                    SVL_TRACE(16);
                    nr = (n0 + 15) & ~15;
                } else if (!SVL_EXP_HOTONLY && sg <= nover) {
                    const int s0 = capA * sg, n = min(capA, nA - s0);
                    nr = (n + 15) & ~15;
                    named_bar_sync(1, 256);  // the previous batch's P.V is done with the staging
                    for (int e = tid; e < n * CH; e += 256) {
                        const int sl = s0 + e / CH, cc = e % CH;
#if SVL_DEBUG_TRAP
                        if (att[sl] < 0 || att[sl] >= nvis) __trap();
#endif
                        cp_async16(vaddr(sl - s0, cc), Vb + (int64_t)work_row(att[sl]) * p.vst + cc * 8, true);
                    }
                    cp_async_commit();
                    for (int i = warp >> 2; i < nvs; i += 2) {  // P rows from TMEM (warp quarter = warp % 4)
                        // the row's virtual slot, recomputed as U assigned it (chunk prefix + ballot)
                        const int row = i * STAGE_ROWS + q4 * 32 + lane, c = row >> 5;
                        const uint32_t pre = __shfl_sync(0xffffffffu, (c & 1) ? ex1 : ex0, c >> 1);
                        const bool above = row < nvis && cls_of(keys_s[row]) == 2;
                        const unsigned ba = __ballot_sync(0xffffffffu, above);
                        const int sl = ntext + (int)(pre & 0xffffu) + __popc(ba & lt);
                        const int pr = (above && sl >= s0 && sl < s0 + n) ? sl - s0 : -1;
                        if (!__any_sync(0xffffffffu, pr >= 0)) continue;
                        float v[16];
                        load_full(i, v);
                        if (pr >= 0) write_p_row(pr, v);
                    }
                    for (int i = tid; i < (nr - n) * 2; i += 256) {
                        reinterpret_cast<uint4*>(pth + (n + (i >> 1)) * 16)[i & 1] = make_uint4(0u, 0u, 0u, 0u);
                        reinterpret_cast<uint4*>(ptl + (n + (i >> 1)) * 16)[i & 1] = make_uint4(0u, 0u, 0u, 0u);
                    }
                    for (int i = tid; i < (nr - n) * CH; i += 256) zero16(vaddr(n + i / CH, i % CH));
                    cp_async_wait<0>();
                    named_bar_sync(1, 256);
                } else {
                    named_bar_sync(3, 512);  // the cut (from S)
                    SVL_TRACE(18);
                    const uint2 cut = ls.cut;
                    for (int jc = tid; jc < nc_loc; jc += 256) {  // the candidates the cut drops: P = 0
                        const int r = ls.attc[jc];
                        const uint32_t key = keys_s[r], gi = (uint32_t)(v0 + r);
                        if (!(key > cut.x || (key == cut.x && gi <= cut.y))) {
                            uint4* dh = reinterpret_cast<uint4*>(pth + (capA + jc) * 16);
                            uint4* dl = reinterpret_cast<uint4*>(ptl + (capA + jc) * 16);
                            dh[0] = dh[1] = dl[0] = dl[1] = make_uint4(0u, 0u, 0u, 0u);
                        }
                    }
                    named_bar_sync(1, 256);
                    row0 = capA;
                    nr = candR;
                }
                if (warp < D / 16 && nr > 0) {
                    // O^T[d][h] += V^T . P, swap-AB: warp w owns d rows [16w, 16w + 16) as the MMA's M,
                    // heads are N (8 per tile), so every MMA does useful work (heads as M would be half
                    // zero rows for g <= 8).  Per 16-row k-tile: one ldmatrix.x4.trans of V (A = V^T)
                    // and one of P (hi and lo B fragments), hi / lo x even / odd tiles in separate
                    // accumulator chains, the next tile's fragments loaded before this tile's MMAs
                    // (legacy mma.sync: 8 cycles per m16n8k16 per SMSP); warp 0 also l += ones . P.
                    const int mi = lane >> 3, rin = lane & 7;
                    const uint32_t avv = vst + ((mi >> 1) * 8 + rin) * GM::VROWB + (2 * warp + (mi & 1)) * 16;
                    const uint32_t apb = smem_u32((mi >> 1) ? ptl : pth) + ((mi & 1) * 8 + rin) * 32;
                    constexpr uint32_t ONES = 0x3f803f80u;  // bf16 (1, 1)
                    const uint32_t ones4[4] = {ONES, ONES, ONES, ONES};
                    uint32_t va[4], pb[NT][4];
                    auto ld = [&](int tb) {
                        ldsm_x4_trans(avv + tb * GM::VROWB, va[0], va[1], va[2], va[3]);
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt)
                            ldsm_x4_trans(apb + tb * 32 + nt * 16, pb[nt][0], pb[nt][1], pb[nt][2], pb[nt][3]);
                    };
                    float acc[2][NT][4][4];  // [tile parity][nt][hi, lo, l hi, l lo]
#pragma unroll
                    for (int a2 = 0; a2 < 2; ++a2)
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                            for (int c = 0; c < 4; ++c) acc[a2][nt][c][0] = acc[a2][nt][c][1] = acc[a2][nt][c][2] = acc[a2][nt][c][3] = 0.f;
                    auto step = [&](float (&A)[NT][4][4], int tb) {
                        const uint32_t aa[4] = {va[0], va[1], va[2], va[3]};
                        uint32_t bb[NT][4];
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                            for (int c = 0; c < 4; ++c) bb[nt][c] = pb[nt][c];
                        if (tb + 16 < row0 + nr) ld(tb + 16);
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) {
                            mma_bf16_16816(A[nt][0], aa, bb[nt][0], bb[nt][1]);
                            mma_bf16_16816(A[nt][1], aa, bb[nt][2], bb[nt][3]);
                            if (warp == 0) {
                                mma_bf16_16816(A[nt][2], ones4, bb[nt][0], bb[nt][1]);
                                mma_bf16_16816(A[nt][3], ones4, bb[nt][2], bb[nt][3]);
                            }
                        }
                    };
                    ld(row0);
                    for (int tb = row0; tb < row0 + nr; tb += 32) {
                        step(acc[0], tb);
                        if (tb + 16 < row0 + nr) step(acc[1], tb + 16);
                    }
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            ot[nt][e] += (acc[0][nt][0][e] + acc[0][nt][1][e]) + (acc[1][nt][0][e] + acc[1][nt][1][e]);
                            lt_[nt][e] += (acc[0][nt][2][e] + acc[0][nt][3][e]) + (acc[1][nt][2][e] + acc[1][nt][3][e]);
                        }
                }
            }
            SVL_TRACE(19);
            // push O^T fragments: thread (gid, t) of warp w holds d = 16w + gid (+ 8), heads
            // 8 nt + 2t (+ 1); the d-neighbour (gid + 1) is 4 lanes up -> float2 pairs along d.
            // l: warp 0, lanes with gid == 0 hold l[8 nt + 2t], l[8 nt + 2t + 1].
            if (warp < D / 16) {
#pragma unroll
                for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float a0 = ot[nt][e], a1 = __shfl_down_sync(0xffffffffu, a0, 4);
                        const int h = 8 * nt + 2 * t + (e & 1), d = 16 * warp + gid + 8 * (e >> 1);
                        if ((gid & 1) == 0 && h < g) {
                            const int i = h * D + d, q = i / per, jj = i - q * per;
                            st_async_f2(mapa_shared(rcv_a + (uint32_t)(rank * per + jj) * 4u, q), a0, a1, mapa_shared(mrg_a, q));
                        }
                    }
                if (warp == 0 && gid == 0)
                    for (int q = 0; q < CS; ++q)
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                            for (int e = 0; e < 2; ++e) {  // heads 8 hh + 2t + e (zero past the NT tiles)
                                const float lv = (hh < NT) ? lt_[hh < NT ? hh : 0][e] : 0.f;
                                st_async_f32(mapa_shared(lrcv_a + (uint32_t)(rank * 16 + 8 * hh + 2 * t + e) * 4u, q), lv,
                                             mapa_shared(mrg_a, q));
                            }
            }
            fin_threads = 256;
        } else {
            // ---------------------------------------- S: exact cut + emit
            const int ts = tid - 256, ws = warp - 8;
            mbar_wait(smem_u32(&xbar[2]), 0);  // every CTA's header + candidates
            __syncwarp();
            if (ts == 0) tstamp(20);
            const int cq_ = ts >> 4;  // 16 threads per peer's candidate list
            const uint32_t ncq = (cq_ < CS) ? ls.hdr[cq_].y : 0u;
            for (uint32_t jc = ts & 15; jc < ncq; jc += 16)  // one radix pass, key bits 19..12
                atomicAdd(&ls.rhist[(ls.cand[cq_][jc].x >> 12) & 255u], 1u);
            named_bar_sync(2, 256);
            // every S warp finds the sub-bin holding the krem-th key (registers only, no barrier):
            // lane l holds bins 8l .. 8l + 7
            uint32_t bA, need;
            {
                const uint4 h0 = *reinterpret_cast<const uint4*>(ls.rhist + 8 * lane);
                const uint4 h1 = *reinterpret_cast<const uint4*>(ls.rhist + 8 * lane + 4);
                const uint32_t cb[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
                uint32_t grp = 0u;
#pragma unroll
                for (int i = 0; i < 8; ++i) grp += cb[i];
                uint32_t suf = grp;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint32_t y = __shfl_down_sync(0xffffffffu, suf, off);
                    if (lane + off < 32) suf += y;
                }
                const unsigned ball = __ballot_sync(0xffffffffu, suf >= krem);
                const int lstar = ball ? 31 - __clz(ball) : 0;
                uint32_t above = suf - grp, bl = 8u * lane;
#pragma unroll
                for (int i = 7; i >= 0; --i) {
                    const bool hit = above + cb[i] >= krem;
                    bl = hit ? 8u * lane + i : bl;
                    above = hit ? above : above + cb[i];
                    if (hit) break;
                }
                bA = __shfl_sync(0xffffffffu, bl, lstar);
                need = krem - __shfl_sync(0xffffffffu, above, lstar);  // keep `need` keys of sub-bin bA
            }
            for (uint32_t jc = ts & 15; jc < ncq; jc += 16) {
                const uint2 cv = ls.cand[cq_][jc];
                if (((cv.x >> 12) & 255u) == bA) lsub[atomicAdd(&ls.nsub, 1u)] = cv;
            }
            named_bar_sync(2, 256);
            const uint32_t nsub = ls.nsub;
            for (uint32_t m = ts; m < nsub; m += 256) {  // exact rank: (key desc, index asc)
                const uint2 cv = lsub[m];
                uint32_t rk = 0u;
#pragma unroll 8
                for (uint32_t i = 0; i < nsub; ++i) {
                    const uint2 d2 = lsub[i];
                    rk += d2.x > cv.x || (d2.x == cv.x && d2.y < cv.y);
                }
                if (rk == need - 1u) ls.cut = cv;
            }
            // hand the cut to D at once (the writer arrives after its store), then S's own barrier
            named_bar_arrive(3, 512);
            named_bar_sync(2, 256);
            if (ts == 0) tstamp(21);
            const uint2 cut = ls.cut;
            auto kept_c = [&](uint2 cv) { return cv.x > cut.x || (cv.x == cut.x && cv.y <= cut.y); };
            // own kept candidates (index order = candidate order) as a 64-bit mask; the
            // output offset = lower-ranked CTAs' rows above b* + their kept candidates
            if (ws == 0) {
                const unsigned k0 = __ballot_sync(0xffffffffu, (uint32_t)lane < (uint32_t)nc_loc && kept_c(ls.cand[rank][lane]));
                const unsigned k1 = __ballot_sync(0xffffffffu, (uint32_t)(lane + 32) < (uint32_t)nc_loc && kept_c(ls.cand[rank][lane + 32]));
                if (lane == 0) ls.kmask[0] = k0, ls.kmask[1] = k1;
            }
            uint32_t pc = 0u;
            if (cq_ < rank)
                for (uint32_t jc = ts & 15; jc < ncq; jc += 16) pc += kept_c(ls.cand[cq_][jc]);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) pc += __shfl_xor_sync(0xffffffffu, pc, off);
            if (lane == 0 && pc) atomicAdd(&ls.offc, pc);
            named_bar_sync(2, 256);
            mbar_wait(ubar_s, 0);  // U's slots and prefix counts
            uint32_t off = ls.offc;
#pragma unroll 4
            for (int q = 0; q < rank; ++q) off += ls.hdr[q].x;
            const uint64_t km = (uint64_t)ls.kmask[0] | ((uint64_t)ls.kmask[1] << 32);
            auto kept_before = [&](int n) { return (uint32_t)__popcll(n >= 64 ? km : (km & ((1ull << n) - 1ull))); };
            for (int ia = ts; ia < na_loc; ia += 256)  // rows above b*: all kept
                idx_out[off + ia + kept_before(ls.ncb[ia])] = v0 + att[ntext + ia];
            for (int jc = ts; jc < nc_loc; jc += 256)  // kept candidates
                if ((km >> jc) & 1ull) idx_out[off + ls.nab[jc] + kept_before(jc)] = v0 + ls.attc[jc];
            if (ts == 0) tstamp(22);
            fin_threads = 0;
        }
    } else {
        float lacc = 0.f;  // thread tid sums head tid % 16
#if !SVL_EXP_HOTONLY
        // ============================================ stage 0 (all / none) or 2 (generic)
        int nslots = ntext;
        uint32_t vphase = 0;
        if (stage == 2) {
            // the generic scratch aliases the V staging: every CTA's text-row gather
            // must land before any peer pushes into it (text rows are re-gathered)
            v_expect((uint32_t)(ntext * ROWB));
            v_wait(0);
            vphase = 1;
            cluster_sync(cl);
        }
        const int nsel = sel.generic_or_trivial(stage, *reinterpret_cast<PushTopkSmem*>(smem + GM::PUSH_OFF),
                                                idx_out, att + ntext);
        nslots = ntext + nsel;
        gather_rows(stage == 2 ? 0 : ntext, min(nslots, VCAP), 0);
        v_expect((uint32_t)(min(nslots, VCAP) * ROWB));
        SVL_TRACE(4);

        // p = exp2(s2 - LSE2[h]): the same reference in every CTA -> plain-sum merge.
        uint16_t* pth = reinterpret_cast<uint16_t*>(smem + GM::PT_OFF);
        uint16_t* ptl = pth + VCAP * 16;
        cta_sync();  // top-k scratch (aliased by the P table and slot_of) is dead
        for (int sl = ntext + tid; sl < nslots; sl += FT) slot_of[att[sl]] = (uint16_t)sl;
        for (int s0 = 0; s0 < nslots; s0 += VCAP) {
            const int n = min(VCAP, nslots - s0);
            const int nr = (n + 15) & ~15;
            if (s0 > 0) {  // overflow batches (rare): after the previous PV
                gather_rows(s0, s0 + n, s0);
                v_expect((uint32_t)(n * ROWB));
            }
            // P table rows [0, nr): zero, then the text rows and the kept visual rows
            for (int i = tid; i < nr * 2; i += FT) {  // 16 heads x 2 B = 32 B = 2 uint4 per row and table
                reinterpret_cast<uint4*>(pth)[i] = make_uint4(0, 0, 0, 0);
                reinterpret_cast<uint4*>(ptl)[i] = make_uint4(0, 0, 0, 0);
            }
            cta_sync();
            for (int i = tid; i < (min(ntext, s0 + n) - s0) * 16; i += FT) {
                const int rr = i >> 4, h = i & 15;
                if (h < g) {
                    const float pv = fast_exp2(txl[(att[s0 + rr] - nvis) * NCP + h] - lse2[h]);
                    const __nv_bfloat16 hi = __float2bfloat16_rn(pv);
                    const __nv_bfloat16 lo = __float2bfloat16_rn(pv - __bfloat162float(hi));
                    pth[rr * 16 + h] = *reinterpret_cast<const uint16_t*>(&hi);
                    ptl[rr * 16 + h] = *reinterpret_cast<const uint16_t*>(&lo);
                }
            }
            for (int i = warp >> 2; i < nvs; i += FT / 128) {
                const int row = i * STAGE_ROWS + q4 * 32 + lane;
                const bool kept = row < nvis && state_s[row] == kKeySel;
                if (!__any_sync(0xffffffffu, kept)) continue;
                float v[16];
                load_full(i, v);
                const int rr = kept ? (int)slot_of[row] - s0 : -1;
                if (rr >= 0 && rr < n) {
                    uint32_t hw[8], lw[8];
#pragma unroll
                    for (int c2 = 0; c2 < 8; ++c2) {
                        float pv2[2];
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int c = 2 * c2 + e;
                            // (stage 2: the key pass left the exponentials in TMEM; stage 0: logits)
                            pv2[e] = (c < NCP) ? (stage == 2 ? v[c] : fast_exp2(v[c] * p.scale2 - nl[c < NCP ? c : 0])) : 0.f;
                        }
                        hw[c2] = pack_bf16(pv2[0], pv2[1]);
                        lw[c2] = pack_bf16(pv2[0] - bf16lo(hw[c2]), pv2[1] - bf16hi(hw[c2]));
                    }
                    uint4* dh = reinterpret_cast<uint4*>(pth + rr * 16);
                    uint4* dl = reinterpret_cast<uint4*>(ptl + rr * 16);
                    dh[0] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                    dh[1] = make_uint4(hw[4], hw[5], hw[6], hw[7]);
                    dl[0] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
                    dl[1] = make_uint4(lw[4], lw[5], lw[6], lw[7]);
                }
            }
            // rows [n, nr) of the staging buffer: zero V (the P rows are zero, avoid NaN * 0)
            for (int i = n * CH + tid; i < nr * CH; i += FT) {
                const int rr = i / CH, c = i % CH;
                *reinterpret_cast<uint4*>(smem + GM::VST_OFF + rr * GM::VROWB + c * 16) = make_uint4(0, 0, 0, 0);
            }
            v_wait(vphase);
            vphase ^= 1u;
            cta_sync();
            // denominators from the table itself (hi + lo: the weights the PV uses)
            for (int i = tid; i < nr * 16; i += FT) {
                const uint32_t hv = pth[i], lv = ptl[i];
                lacc += __uint_as_float(hv << 16) + __uint_as_float(lv << 16);
            }
            SVL_TRACE(5);
            if (warp < D / 16) {
                const int mi = lane >> 3, rin = lane & 7;
                const uint32_t aph = smem_u32(pth), apl = smem_u32(ptl);
                for (int tb = 0; tb < nr; tb += 16) {
                    // P fragment (m = heads, k = rows): matrices (h0-7,k0-7) (h8-15,k0-7) (h0-7,k8-15) (h8-15,k8-15)
                    const int prow = tb + (mi >> 1) * 8 + rin;
                    uint32_t ph[4], pl[4];
                    ldsm_x4_trans(aph + prow * 32 + (mi & 1) * 16, ph[0], ph[1], ph[2], ph[3]);
                    ldsm_x4_trans(apl + prow * 32 + (mi & 1) * 16, pl[0], pl[1], pl[2], pl[3]);
                    const int vrow = tb + (mi & 1) * 8 + rin;
                    const int c = 2 * warp + (mi >> 1);
                    uint32_t v0r, v1r, v2r, v3r;
                    ldsm_x4_trans(vst + vrow * GM::VROWB + c * 16, v0r, v1r, v2r, v3r);
                    mma_bf16_16816(o[0], ph, v0r, v1r);
                    mma_bf16_16816(o[0], pl, v0r, v1r);
                    mma_bf16_16816(o[1], ph, v2r, v3r);
                    mma_bf16_16816(o[1], pl, v2r, v3r);
                }
            }
            cta_sync();  // staging + P table free for the next batch
        }
#endif
        float* octa = reinterpret_cast<float*>(smem + GM::OCTA_OFF);  // [16][D]
        float* lred = reinterpret_cast<float*>(smem + GM::LRED_OFF);
        cta_sync();  // P.V done everywhere
        SVL_TRACE(6);
        lred[tid] = lacc;
        if (warp < D / 16) {
#pragma unroll
            for (int nt = 0; nt < 2; ++nt) {
                const int col = warp * 16 + nt * 8 + 2 * t;
                if (gid < g) *reinterpret_cast<float2*>(octa + gid * D + col) = make_float2(o[nt][0], o[nt][1]);
                if (gid + 8 < g) *reinterpret_cast<float2*>(octa + (gid + 8) * D + col) = make_float2(o[nt][2], o[nt][3]);
            }
        }
        cta_sync();
        if (tid < 16) {
            float acc = 0.f;
#pragma unroll
            for (int j = 0; j < FT / 16; ++j) acc += lred[j * 16 + tid];
            lh[tid] = acc;
        }
        cta_sync();  // lh complete before it is pushed
        SVL_TRACE(7);
        for (int i = tid; i < items; i += FT) {
            const int q = i / per, j = i - q * per;
            st_async_f32(mapa_shared(rcv_a + (uint32_t)(rank * per + j) * 4u, q), octa[i], mapa_shared(mrg_a, q));
        }
        if (tid < 16 * CS)
            st_async_f32(mapa_shared(lrcv_a + (uint32_t)(rank * 16 + (tid & 15)) * 4u, tid >> 4), lh[tid & 15],
                         mapa_shared(mrg_a, tid >> 4));
    }
    tc_fence_before();  // every TMEM read of this CTA precedes the dealloc below
    SVL_TRACE(8);
    if (tid < fin_threads) mbar_wait(mrg_a, 0);
    for (int j = tid; j < per && tid < fin_threads; j += fin_threads) {
        const int i = rank * per + j;
        if (i >= items) break;
        const int h = i / D, dd = i % D;
        float num = 0.f, den = 0.f;
#pragma unroll
        for (int q = 0; q < 16; ++q) {  // (sender order; the loads are independent)
            if (q < CS) {
                num += rcv[q * per + j];
                den += lrcv[q * 16 + h];
            }
        }
        const int hh = G * g + h;
        p.out[((int64_t)b * p.H + hh) * D + dd] = (den > 0.f) ? num / den : 0.f;
        if (dd == 0 && p.lse_out)
            p.lse_out[(int64_t)b * p.H + hh] = (den > 0.f) ? (lse2[h] + log2f(den)) * kLn2 : -INFINITY;
    }
    (void)ibc;
    SVL_TRACE(9);
    tc_fence_before();
    SVL_TRACE(10);
    if (trace_out && tid == 0) {
        uint64_t c1;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(c1)::"memory");
        trs[31] = c1;
    }
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tbase, TMEM_COLS);
    }
    if (trace_out) {
        cta_sync();  // (trace builds) every warp's stamps
        if (tid < 64) trace_out[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 64 + tid] = trs[tid];
    }
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
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    // programmatic dependent launch: the prologue (barriers, TMEM, the first visual
    // K stages) may start while the previous kernel on the stream drains; the kernel
    // executes griddepcontrol.wait before reading anything that kernel may write
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, fresh_kernel<D, NT>, p);
}

template <int D, int NT>
int max_active_clusters_t(int CS) {
    using GM = FGeom<D, NT>;
    if (cudaFuncSetAttribute(fresh_kernel<D, NT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
        cudaFuncSetAttribute(fresh_kernel<D, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, GM::BYTES) != cudaSuccess)
        return 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS, 1, 1);
    cfg.blockDim = dim3(FT, 1, 1);
    cfg.dynamicSmemBytes = GM::BYTES;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fresh_kernel<D, NT>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

}  // namespace

// Co-resident clusters of the fused kernel at cluster size CS (cached per device; <= 0: unknown).
int fresh_max_active_clusters(int d, int g, int CS) {
    static int cache[8][2][2][17] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    const int NT = (g + 7) / 8;
    if (CS < 1 || CS > 16 || NT < 1 || NT > 2) return 0;
    int& c = cache[dev & 7][d == 128][NT - 1][CS];
    if (c == 0) {
        if (d == 128) c = NT == 1 ? max_active_clusters_t<128, 1>(CS) : max_active_clusters_t<128, 2>(CS);
        else c = NT == 1 ? max_active_clusters_t<64, 1>(CS) : max_active_clusters_t<64, 2>(CS);
        if (c == 0) c = -1;
    }
    return c;
}

cudaError_t launch_fresh(const FreshParams& p, int d, int CS, cudaStream_t s) {
    const int NT = (p.g + 7) / 8;
    if (d == 128 && NT == 1) return launch_fresh_t<128, 1>(p, CS, s);
    if (d == 128 && NT == 2) return launch_fresh_t<128, 2>(p, CS, s);
    if (d == 64 && NT == 1) return launch_fresh_t<64, 1>(p, CS, s);
    if (d == 64 && NT == 2) return launch_fresh_t<64, 2>(p, CS, s);
    return cudaErrorInvalidValue;
}

}  // namespace svl
