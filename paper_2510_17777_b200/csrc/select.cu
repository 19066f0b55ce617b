// select.cu -- stand-alone selection kernel (SURVEY.md 8(a) a2 + a3, a7).
//
// One thread-block cluster (CS <= 16 CTAs, distributed shared memory) per
// selection unit.  Used by
//   * svl_retrieve phase 2 (mode 0): score[j] = sum_c exp2(s2[j,c] - LSE2[c])
//     -- the visual share of the attention mass (SPEC.md:371,
//     394-396) -- from the phase-1 logits (L2-resident scratch) and the
//     cluster-reduced chunk partials, then the top-k of each unit;
//   * svl_prefill_prune (mode 1): the top-k_f of the given fp32 saliency of
//     each (batch row, frame).
// The top-k itself is cluster_topk (select_core.cuh): ties to the lower
// index, ascending output, bitwise reproducible.
#include <cooperative_groups.h>

#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "select_core.cuh"
#include "select_fast.cuh"

namespace svl {

namespace {

constexpr int NTH = kSelectThreads;
constexpr int EMAX = kSelectMaxPerThread;

struct SelectSmem {
    TopkSmem topk;
    float lse2[128];
};

template <int MODE, int NT>
SVL_DEV void select_body(const SelectParams& p, const PruneTable* tabp) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    SelectSmem& sm = *reinterpret_cast<SelectSmem*>(smem_raw);
    cg::cluster_group cluster = cg::this_cluster();
    cluster_arrive_relaxed();  // this CTA is resident (peers push into it after their cluster_wait)
    const int CS = p.CS;
    const int rank = (int)cluster.block_rank();
    const int u = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // ---------------------------------------------------------- unit geometry
    int n, k, b = 0, G0 = 0, nG = 1;
    int64_t src_off = 0, out_off;
    int idx_base = 0;  // added to written indices (prune: frame offset -> global index)
    if (MODE == 0 || MODE == 2) {
        n = p.nv;
        k = p.k;
        out_off = (int64_t)u * k;
        if (p.shared) {
            b = u; G0 = 0; nG = p.Hkv;
        } else {
            b = u / p.Hkv; G0 = u % p.Hkv; nG = 1;
        }
    } else {
        const int bb = u / p.nf, f = u % p.nf;
        const int2 a = tabp->fr[f], z = tabp->fr[f + 1];
        src_off = (int64_t)bb * p.N + a.x;
        n = z.x - a.x;
        k = z.y - a.y;
        out_off = (int64_t)bb * p.kept_cap + a.y;
        idx_base = a.x;
    }
    const int slice = (n + CS - 1) / CS;
    const int j0 = min(n, rank * slice);
    const int j1 = min(n, j0 + slice);
    const int E = (j1 - j0 + NTH - 1) / NTH;  // elements per thread (contiguous)
    const int my0 = j0 + tid * E;
    const int nmine = max(0, min(E, j1 - my0));

    // ------------------------------------------------------- normalisers (mode 0)
    if (MODE == 0) {
        const int ncols = p.NC * nG;
        for (int cc = warp; cc < ncols; cc += NTH / 32) {
            const int G = G0 + cc / p.NC, col = cc % p.NC;
            float lse2;
            if (p.lse_in) {
                const int r = col / p.g, h = G * p.g + col % p.g;
                lse2 = p.lse_in[((int64_t)b * p.n_q + r) * p.H + h] * kLog2e;
            } else {
                const int uu = b * p.Hkv + G;
                float m = -INFINITY, l = 0.f;
                for (int i = lane; i < p.C; i += 32) {
                    const float2 pr = p.part[((int64_t)uu * p.C + i) * p.NCP + col];
                    const float M = fmaxf(m, pr.x);
                    if (M != -INFINITY) {
                        l = l * exp2f(m - M) + pr.y * exp2f(pr.x - M);
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
                lse2 = m + log2f(l);
            }
            if (lane == 0) sm.lse2[cc] = lse2;
        }
        cta_sync();
    }

    // ------------------------------------------------------------------ keys
    uint32_t key[EMAX];
    bool nan_seen = false;
#pragma unroll
    for (int e = 0; e < EMAX; ++e) {
        key[e] = 0u;
        if (e < nmine) {
            const int j = my0 + e;
            float sc;
            if (MODE == 0) {
                sc = 0.f;
                for (int G = 0; G < nG; ++G) {
                    const float4* lr = reinterpret_cast<const float4*>(
                        p.logits + (((int64_t)(b * p.Hkv + G0 + G)) * p.nv + j) * (NT * 8));
                    float4 v[2 * NT];
#pragma unroll
                    for (int i = 0; i < 2 * NT; ++i) v[i] = lr[i];
                    const float* lv = reinterpret_cast<const float*>(v);
#pragma unroll
                    for (int col = 0; col < NT * 8; ++col)
                        if (col < p.NC) sc += exp2f(lv[col] - sm.lse2[G * p.NC + col]);
                }
                if (p.scores_out) p.scores_out[(int64_t)u * n + j] = sc;
            } else if (MODE == 2) {  // precomputed per-unit relevance (tensor-core retrieve), summed over G if SHARED
                sc = 0.f;
                for (int G = 0; G < nG; ++G) sc += p.scores_in[((int64_t)(b * p.Hkv + G0 + G)) * p.nv + j];
                if (p.scores_out) p.scores_out[(int64_t)u * n + j] = sc;
            } else {
                sc = p.scores_in[src_off + j];
            }
            key[e] = float_key(sc, nan_seen);
        }
    }
    if (nan_seen) raise_flag(p.flags, 2u /*SVL_DEVFLAG_NONFINITE*/);

    cluster_wait();  // every peer has started (cluster_topk pushes over DSMEM)
    const TopkResult r = cluster_topk<NTH>(cluster, sm.topk, key, nmine, E, j0, slice, n, k);
    topk_emit<NTH>(sm.topk, r, key, nmine, [&](int e, uint32_t slot) {
        p.idx_out[out_off + slot] = idx_base + my0 + e;
    });
    cluster_sync(cluster);  // no CTA leaves while a peer may still address its shared memory
}

// ----------------------------------------------------------------------------
// Retrieve selection with the fused kernel's two-exchange top-k (select_fast.cuh):
// relevance keys in shared memory, a 256-bin value-adaptive histogram and the
// threshold bin's candidates all-gathered with st.async, the exact cut resolved
// locally; massive ties fall back to the generic push radix.  Same result as
// select_body (ties to the lower index, ascending output).  Rows are read
// thread-strided (coalesced), keys kept per CTA slice (<= kFsSliceMax).
// threshold-bin candidates per CTA: 64 as in the fused kernel for relevance keys (mode 0),
// 256 for question-chunk scores (mode 2: sums over n_q * g rows concentrate near the cut
// and overflow 64 -> the generic radix); the slice bound keeps two CTAs per SM
template <int CANDS>
struct FsLayout {
    static constexpr int kFsSliceMax = CANDS > 64 ? 4096 : 8192;
    using FsSelSmem = FastSelSmemT<CANDS>;
    // [FastSelSmem | private histograms] is dead once threshold() has run, so the generic
    // fallback's scratch aliases it; the fallback's V-slot output (unused here) aliases the
    // keys, which are dead once its radix passes are done.  two CTAs per SM.
    static constexpr int FS_OFF = 0;
    static constexpr int WHIST_OFF = (int)((sizeof(FsSelSmem) + 15) / 16 * 16);
    static constexpr int PUSH_OFF = 0;
    static constexpr int KEYS_OFF = WHIST_OFF + 16 * 256 * 4 > (int)((sizeof(PushTopkSmem) + 15) / 16 * 16)
                                        ? WHIST_OFF + 16 * 256 * 4
                                        : (int)((sizeof(PushTopkSmem) + 15) / 16 * 16);
    static constexpr int STATE_OFF = KEYS_OFF + kFsSliceMax * 4;
    static constexpr int LSE_OFF = STATE_OFF + kFsSliceMax;
    static constexpr int BAR_OFF = LSE_OFF + 128 * 4;
    static constexpr int BYTES = BAR_OFF + 32;
    static_assert(BYTES <= 113 * 1024, "two CTAs per SM");
};

template <int MODE, int NT, int CANDS, bool REFINE = false>
__global__ void __launch_bounds__(NTH, 2) select_fast_kernel(const SelectParams p) {
    using FsLayout = svl::FsLayout<CANDS>;
    extern __shared__ __align__(16) uint8_t smem[];
    cg::cluster_group cl = cg::this_cluster();
    const int CS = (int)cl.num_blocks(), rank = (int)cl.block_rank();
    const int u = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + FsLayout::BAR_OFF);
    if (tid == 0) {
        mbar_init(smem_u32(&bars[0]), 1);  // histograms: CS x 1 KB
        mbar_arrive_expect_tx(smem_u32(&bars[0]), (uint32_t)(CS * 1024));
        mbar_init(smem_u32(&bars[1]), 1);  // candidates (armed in threshold())
        mbar_init(smem_u32(&bars[2]), 1);  // refinement histograms (armed in threshold(), if needed)
        fence_mbar_init();
    }
    cluster_arrive_relaxed();
    const int n = p.nv, k = p.k;
    const int64_t out_off = (int64_t)u * k;
    int b, G0, nG;
    if (p.shared) {
        b = u; G0 = 0; nG = p.Hkv;
    } else {
        b = u / p.Hkv; G0 = u % p.Hkv; nG = 1;
    }
    const int slice = (n + CS - 1) / CS;
    const int j0 = min(n, rank * slice);
    const int nloc = min(n, j0 + slice) - j0;
    float* lse2s = reinterpret_cast<float*>(smem + FsLayout::LSE_OFF);
    if (MODE == 0) {  // normalisers: lse_in, or the cluster of chunk partials (fixed fold order)
        const int ncols = p.NC * nG;
        for (int cc = warp; cc < ncols; cc += NTH / 32) {
            const int G = G0 + cc / p.NC, col = cc % p.NC;
            float lse2;
            if (p.lse_in) {
                const int r = col / p.g, h = G * p.g + col % p.g;
                lse2 = p.lse_in[((int64_t)b * p.n_q + r) * p.H + h] * kLog2e;
            } else {
                const int uu = b * p.Hkv + G;
                float m = -INFINITY, l = 0.f;
                for (int i = lane; i < p.C; i += 32) {
                    const float2 pr = p.part[((int64_t)uu * p.C + i) * p.NCP + col];
                    const float M = fmaxf(m, pr.x);
                    if (M != -INFINITY) {
                        l = l * exp2f(m - M) + pr.y * exp2f(pr.x - M);
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
                lse2 = m + log2f(l);
            }
            if (lane == 0) lse2s[cc] = lse2;
        }
    }
    FastSelect<NTH, CANDS, REFINE> sel(cl, *reinterpret_cast<typename FsLayout::FsSelSmem*>(smem + FsLayout::FS_OFF), nloc, j0,
                               slice, n, k,
                        reinterpret_cast<uint32_t*>(smem + FsLayout::KEYS_OFF), smem + FsLayout::STATE_OFF, p.flags,
                        reinterpret_cast<uint32_t*>(smem + FsLayout::WHIST_OFF));
    sel.hbar = &bars[0];
    sel.cbar = &bars[1];
    sel.h2bar = &bars[2];
    int stage = 0;
    if (!sel.trivial()) {
        sel.zero_hist();
        cta_sync();
        if (MODE == 2 && nG == 1) {
            // precomputed relevance: all of the thread's loads in flight before the first key
            constexpr int R = FsLayout::kFsSliceMax / NTH;
            const float* src = p.scores_in + ((int64_t)(b * p.Hkv + G0)) * p.nv + j0;
            float v[R];
#pragma unroll
            for (int q = 0; q < R; ++q) v[q] = (tid + q * NTH < nloc) ? src[tid + q * NTH] : 0.f;
#pragma unroll
            for (int q = 0; q < R; ++q)
                if (tid + q * NTH < nloc) sel.add_key(tid + q * NTH, v[q]);
        }
        for (int i = (MODE == 2 && nG == 1) ? nloc : tid; i < nloc; i += NTH) {
            const int j = j0 + i;
            float sc = 0.f;
            if (MODE == 0) {
                for (int G = 0; G < nG; ++G) {
                    const float4* lr = reinterpret_cast<const float4*>(
                        p.logits + (((int64_t)(b * p.Hkv + G0 + G)) * p.nv + j) * (NT * 8));
                    float4 v[2 * NT];
#pragma unroll
                    for (int q = 0; q < 2 * NT; ++q) v[q] = lr[q];
                    const float* lv = reinterpret_cast<const float*>(v);
#pragma unroll
                    for (int col = 0; col < NT * 8; ++col)
                        if (col < p.NC) sc += exp2f(lv[col] - lse2s[G * p.NC + col]);
                }
            } else {
                for (int G = 0; G < nG; ++G) sc += p.scores_in[((int64_t)(b * p.Hkv + G0 + G)) * p.nv + j];
            }
            if (p.scores_out) p.scores_out[(int64_t)u * n + j] = sc;
            sel.add_key(i, sc);
        }
        cluster_wait();  // every peer has started and armed its barriers
        stage = sel.threshold();
    } else {
        cluster_wait();
    }
    int32_t* idx_out = p.idx_out + out_off;
    if (stage == 1) {
        sel.assign_slots_and_push_candidates(nullptr);
        sel.resolve_and_emit(idx_out);
    } else {
        // (every CTA takes the same stage) the generic scratch aliases FastSelSmem, which a
        // slower peer may still be reading in threshold(): meet before anyone pushes into it
        if (stage == 2) cluster_sync(cl);
#if SVL_EXP_FLAG_STAGE2
        if (stage == 2 && tid == 0 && rank == 0) raise_flag(p.flags, 0x100u);
#endif
        sel.generic_or_trivial(stage, *reinterpret_cast<PushTopkSmem*>(smem + FsLayout::PUSH_OFF), idx_out,
                               reinterpret_cast<int*>(smem + FsLayout::KEYS_OFF));
    }
    cluster_sync(cl);  // no CTA leaves while a peer may still address its shared memory
}

// Relevance of every visual row, score[u][j] = sum_c exp2(s2[j,c] - LSE2[c]) (the
// select kernels' mode-0 arithmetic, same fold and summation order, so the scores
// are bitwise those mode 0 computes), as a plain streaming pass: every thread
// keeps RR rows' logits in flight, full occupancy; the cluster top-k then reads
// 4 B per row (mode 2) instead of the 8 NT logits.
constexpr int kRelThreads = 256;
constexpr int kRelRows = 4;       // rows per thread per pass (all loads issued first)
constexpr int kRelPasses = 4;     // passes per CTA
template <int NT>
__global__ void __launch_bounds__(kRelThreads) relevance_kernel(const SelectParams p, float* scores) {
    __shared__ float lse2s[NT * 8];
    const int u = blockIdx.y, b = u / p.Hkv, G = u % p.Hkv;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int col = warp; col < p.NC; col += kRelThreads / 32) {
        float lse2;
        if (p.lse_in) {
            const int r = col / p.g, h = G * p.g + col % p.g;
            lse2 = p.lse_in[((int64_t)b * p.n_q + r) * p.H + h] * kLog2e;
        } else {
            float m = -INFINITY, l = 0.f;
            for (int i = lane; i < p.C; i += 32) {
                const float2 pr = p.part[((int64_t)u * p.C + i) * p.NCP + col];
                const float M = fmaxf(m, pr.x);
                if (M != -INFINITY) {
                    l = l * exp2f(m - M) + pr.y * exp2f(pr.x - M);
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
            lse2 = m + log2f(l);
        }
        if (lane == 0) lse2s[col] = lse2;
    }
    __syncthreads();
    const float4* lg = reinterpret_cast<const float4*>(p.logits + (int64_t)u * p.nv * (NT * 8));
    float* out = scores + (int64_t)u * p.nv;
    constexpr int SPAN = kRelThreads * kRelRows;
    for (int j0 = blockIdx.x * SPAN; j0 < p.nv; j0 += gridDim.x * SPAN) {
        float4 v[kRelRows][2 * NT];
#pragma unroll
        for (int q = 0; q < kRelRows; ++q) {
            const int j = j0 + q * kRelThreads + tid;
#pragma unroll
            for (int i = 0; i < 2 * NT; ++i)
                v[q][i] = (j < p.nv) ? lg[(int64_t)j * (2 * NT) + i] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < kRelRows; ++q) {
            const int j = j0 + q * kRelThreads + tid;
            if (j >= p.nv) continue;
            const float* lv = reinterpret_cast<const float*>(v[q]);
            float sc = 0.f;
#pragma unroll
            for (int col = 0; col < NT * 8; ++col)
                if (col < p.NC) sc += exp2f(lv[col] - lse2s[col]);
            out[j] = sc;
        }
    }
}

template <int NT>
__global__ void __launch_bounds__(NTH, 1) select_retrieve_kernel(const SelectParams p) {
    select_body<0, NT>(p, nullptr);
}

__global__ void __launch_bounds__(NTH, 1) select_scores_kernel(const SelectParams p) {
    select_body<2, 1>(p, nullptr);
}

__global__ void __launch_bounds__(NTH, 1)
    select_prune_kernel(const SelectParams p, const __grid_constant__ PruneTable tab) {
    select_body<1, 1>(p, &tab);
}

// Per-frame prune for frames of <= 512 tokens (the encoder's frames): one CTA
// per (b, frame), one key per thread, a bitonic sort of the 64-bit composite
// (order-preserving key << 32 | ~index) descending -- i.e. saliency desc, index
// asc, exactly the oracle's stable order -- then the top k_f indices are
// re-emitted in ascending index order through a block prefix sum.  Stages with
// partner distance < 32 run inside a warp (shuffles, no barrier).
constexpr int kSmallFrame = 512;

__global__ void __launch_bounds__(kSmallFrame) prune_small_kernel(const SelectParams p,
                                                                 const __grid_constant__ PruneTable tab) {
    __shared__ uint64_t sv[kSmallFrame];
    __shared__ uint32_t wsum[kSmallFrame / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int u = blockIdx.x;
    const int bb = u / p.nf, f = u % p.nf;
    const int2 a = tab.fr[f], z = tab.fr[f + 1];
    const int n = z.x - a.x, k = z.y - a.y;
    const float* src = p.scores_in + (int64_t)bb * p.N + a.x;
    bool nan_seen = false;
    uint64_t v = 0ull;  // padding sorts last
    if (tid < n) v = ((uint64_t)float_key(src[tid], nan_seen) << 32) | (uint32_t)(~tid);
    if (nan_seen) raise_flag(p.flags, 2u /*SVL_DEVFLAG_NONFINITE*/);
    // bitonic sort, descending
    for (int size = 2; size <= kSmallFrame; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            uint64_t o;
            if (stride >= 32) {
                sv[tid] = v;
                cta_sync();
                o = sv[tid ^ stride];
                cta_sync();
            } else {
                o = __shfl_xor_sync(0xffffffffu, v, stride);
            }
            const bool desc = ((tid & size) == 0);      // direction of this bitonic block
            const bool lower = ((tid & stride) == 0);   // this thread holds the lower position
            const uint64_t hi = v > o ? v : o, lo = v > o ? o : v;
            v = (lower == desc) ? hi : lo;
        }
    }
    // position tid now holds the tid-th largest; the first k are kept
    sv[tid] = v;
    cta_sync();
    // kept flag per ORIGINAL index, then ascending emission by prefix sum
    const int idx_of_rank = (int)(~(uint32_t)(sv[tid] & 0xffffffffu));
    cta_sync();
    uint32_t* kept = reinterpret_cast<uint32_t*>(sv);  // reuse: kept[original index]
    kept[tid] = 0u;
    cta_sync();
    if (tid < k) kept[idx_of_rank] = 1u;
    cta_sync();
    const uint32_t mine = (tid < n) ? kept[tid] : 0u;
    uint32_t x = mine;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    cta_sync();
    uint32_t before = 0u;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    if (mine) p.idx_out[(int64_t)bb * p.kept_cap + a.y + before + x - 1u] = a.x + tid;
}

}  // namespace

int select_cluster_size(int n) {
    int cs = (n + 2047) / 2048;
    if (cs < 2) cs = 2;  // >= 2: st.async / DSMEM exchanges need a real cluster (compute-sanitizer)
    if (cs > 16) cs = 16;
    int c = 1;  // power of two: the 4096 / 1024 digit bins split evenly between owners
    while (c < cs) c <<= 1;
    return c;
}

template <typename Kern, typename... Args>
static cudaError_t launch_cluster(Kern kern, int CS, int n_units, cudaStream_t s, bool& attr_done,
                                  Args... args) {
    const int smem = (int)sizeof(SelectSmem);
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e == cudaSuccess) e = set_max_carveout(kern);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS, n_units, 1);
    cfg.blockDim = dim3(NTH, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

static bool* attr_flag(int which) {
    static bool done[16][64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    return &done[which][dev & 63];
}

template <int CANDS, typename Kern>
static cudaError_t launch_fast(Kern kern, const SelectParams& p, int n_units, cudaStream_t s, bool& attr_done) {
    using FsLayout = svl::FsLayout<CANDS>;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, FsLayout::BYTES);
        if (e == cudaSuccess) e = set_max_carveout(kern);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.CS, n_units, 1);
    cfg.blockDim = dim3(NTH, 1, 1);
    cfg.dynamicSmemBytes = FsLayout::BYTES;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

cudaError_t launch_select(const SelectParams& p, int n_units, cudaStream_t s) {
    const int slice = (p.nv + p.CS - 1) / p.CS;
#ifndef SVL_OLD_SELECT
    const bool fast = true;  // the generic cluster kernels below stay for slices past the fast-path capacity
#else
    const bool fast = false;  // A/B builds only
#endif
    if (p.mode == 3) {  // relevance scores of one decode query (svl_retrieve's split path): 64 candidates
        if (slice > FsLayout<64>::kFsSliceMax) return cudaErrorInvalidValue;
        SelectParams q = p;
        q.mode = 2;
        return launch_fast<64>(select_fast_kernel<2, 1, 64, true>, q, n_units, s, *attr_flag(11));
    }
    if (fast && p.mode == 2 && slice <= FsLayout<256>::kFsSliceMax)
        return launch_fast<256>(select_fast_kernel<2, 1, 256>, p, n_units, s, *attr_flag(6));
    if (fast && p.mode == 0 && slice <= FsLayout<64>::kFsSliceMax) {
        switch (p.NCP / 8) {
            case 1: return launch_fast<64>(select_fast_kernel<0, 1, 64>, p, n_units, s, *attr_flag(7));
            case 2: return launch_fast<64>(select_fast_kernel<0, 2, 64>, p, n_units, s, *attr_flag(8));
            case 3: return launch_fast<64>(select_fast_kernel<0, 3, 64>, p, n_units, s, *attr_flag(9));
            case 4: return launch_fast<64>(select_fast_kernel<0, 4, 64>, p, n_units, s, *attr_flag(10));
        }
        return cudaErrorInvalidValue;
    }
    if (p.mode == 2) return launch_cluster(select_scores_kernel, p.CS, n_units, s, *attr_flag(5), p);
    switch (p.NCP / 8) {
        case 1: return launch_cluster(select_retrieve_kernel<1>, p.CS, n_units, s, *attr_flag(1), p);
        case 2: return launch_cluster(select_retrieve_kernel<2>, p.CS, n_units, s, *attr_flag(2), p);
        case 3: return launch_cluster(select_retrieve_kernel<3>, p.CS, n_units, s, *attr_flag(3), p);
        case 4: return launch_cluster(select_retrieve_kernel<4>, p.CS, n_units, s, *attr_flag(4), p);
    }
    return cudaErrorInvalidValue;
}

// cluster size of the split path's select: slices of up to kFsSliceMax (8192) rows, so few
// small clusters -- the selection is a chain of cluster exchanges, paid once per wave
#ifndef SVL_REL_SLICE
#define SVL_REL_SLICE 8192  // rows per CTA of the mode-3 select (<= FsLayout<64>::kFsSliceMax)
#endif
int relevance_select_cs(int nv) {
    int cs = (nv + SVL_REL_SLICE - 1) / SVL_REL_SLICE;
    if (cs < 2) cs = 2;
    int c = 1;
    while (c < cs) c <<= 1;
    return c;
}

template <int NT>
static cudaError_t launch_relevance_t(const SelectParams& p, float* scores, int units, cudaStream_t s) {
    // one wave: CTAs per unit = resident CTAs / units (each grid-strides over its unit's rows)
    static int occ[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && occ[dev] == 0) {
        int o = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, relevance_kernel<NT>, kRelThreads, 0) != cudaSuccess)
            o = 1;
        occ[dev] = std::max(1, o);
    }
    const int slots = device_sm_count() * (dev < 64 ? occ[dev] : 1);
    constexpr int per = kRelThreads * kRelRows;
    int x = (p.nv + per - 1) / per;
#if !defined(SVL_REL_ONEWAVE) || SVL_REL_ONEWAVE
    x = std::max(1, std::min(x, slots / std::max(1, units)));
#else
    x = (p.nv + per * kRelPasses - 1) / (per * kRelPasses);
#endif
    relevance_kernel<NT><<<dim3((unsigned)x, (unsigned)units), kRelThreads, 0, s>>>(p, scores);
    return cudaGetLastError();
}

cudaError_t launch_relevance(const SelectParams& p, float* scores, int units, cudaStream_t s) {
    switch (p.NCP / 8) {
        case 1: return launch_relevance_t<1>(p, scores, units, s);
        case 2: return launch_relevance_t<2>(p, scores, units, s);
        case 3: return launch_relevance_t<3>(p, scores, units, s);
        case 4: return launch_relevance_t<4>(p, scores, units, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_prune_select(const SelectParams& p, const PruneTable& tab, int n_units,
                                cudaStream_t s) {
    int max_n = 0;
    for (int f = 0; f < p.nf; ++f) max_n = std::max(max_n, tab.fr[f + 1].x - tab.fr[f].x);
    if (max_n <= kSmallFrame) {
        prune_small_kernel<<<n_units, kSmallFrame, 0, s>>>(p, tab);
        return cudaGetLastError();
    }
    return launch_cluster(select_prune_kernel, p.CS, n_units, s, *attr_flag(0), p, tab);
}

}  // namespace svl
