// select.cu -- deterministic top-k selection (SURVEY.md 8(a) a2 + a3, a7).
//
// One thread-block cluster (CS <= 16 CTAs, distributed shared memory) per
// selection unit.  Used by
//   * svl_retrieve (mode 0): score[j] = sum_c exp2(s2[j,c] - LSE2[c]) -- the
//     visual share of the attention mass
//     -- from the phase-1 logits and the reduced chunk partials; then top-k.
//   * svl_prefill_prune (mode 1): top-k_f of the given fp32 saliency per
//     frame.
//
// Selection: the k largest keys, ties to the lower index, indices written
// ascending.  Keys are order-preserving uint32 images of
// the fp32 values (-0.0 == +0.0, NaN lowest, reading A8).  The k-th largest
// key T is found by an MSB-first radix select (digits of 11/11/10 bits) whose
// per-CTA shared-memory histograms are reduced across the cluster over
// DSMEM; selected = {key > T} + the first (k - #{key > T}) keys equal to T in
// index order, found with block scans plus a cluster prefix over CTA ranks.
// Every reduction has a fixed order: results are bitwise reproducible.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace svl {

namespace {

constexpr int NB = 2048;  // max bins per radix pass
constexpr int NTH = kSelectThreads;
constexpr int EMAX = kSelectMaxPerThread;

// exclusive block scan of a uint32 (sum), returns exclusive prefix and total
SVL_DEV uint32_t block_exclusive_scan(uint32_t v, uint32_t* warp_sums, uint32_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
        if (lane >= off) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = (lane < NTH / 32) ? warp_sums[lane] : 0u;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, off);
            if (lane >= off) w += y;
        }
        if (lane < NTH / 32) warp_sums[lane] = w;  // inclusive
    }
    __syncthreads();
    const uint32_t before = (warp > 0 ? warp_sums[warp - 1] : 0u) + (x - v);
    total = warp_sums[NTH / 32 - 1];
    __syncthreads();
    return before;
}

struct SelectShared {
    uint32_t hist[2][NB];
    uint32_t own[2][NB];  // owner sums (NB/CS bins used; CS may be 1)
    uint32_t own_total[2];
    uint32_t warp_sums[NTH / 32];
    uint32_t cta_gt, cta_eq;
    float lse2[128];
    // broadcast of the pass result
    uint32_t res_prefix, res_mask, res_krem;
};

template <int MODE>
SVL_DEV void select_body(const SelectParams& p, const PruneTable* tabp) {
    cg::cluster_group cluster = cg::this_cluster();
    const int CS = p.CS;
    const int rank = (int)cluster.block_rank();
    const int u = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ SelectShared sm;

    // ---------------------------------------------------------- unit geometry
    int n, k, b = 0, G0 = 0, nG = 1;
    int64_t src_off = 0, out_off;
    if (MODE == 0) {
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
    }
    const int slice = (n + CS - 1) / CS;
    const int j0 = min(n, rank * slice);
    const int j1 = min(n, j0 + slice);
    const int nloc = j1 - j0;
    const int E = (nloc + NTH - 1) / NTH;  // elements per thread (contiguous)
    const int my0 = j0 + tid * E;

    // ------------------------------------------------------- normalisers (mode 0)
    const int ncols = p.NC * nG;
    if (MODE == 0) {
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
        __syncthreads();
    }

    // ------------------------------------------------------------------ keys
    uint32_t key[EMAX];
    bool nan_seen = false;
#pragma unroll
    for (int e = 0; e < EMAX; ++e) {
        key[e] = 0u;
        if (e < E) {
            const int j = my0 + e;
            if (j < j1) {
                float sc;
                if (MODE == 0) {
                    sc = 0.f;
                    for (int G = 0; G < nG; ++G) {
                        const float* lr =
                            p.logits + (((int64_t)(b * p.Hkv + G0 + G)) * p.nv + j) * p.NCP;
                        for (int col = 0; col < p.NC; ++col)
                            sc += exp2f(lr[col] - sm.lse2[G * p.NC + col]);
                    }
                    if (p.scores_out) p.scores_out[(int64_t)u * n + j] = sc;
                } else {
                    sc = p.scores_in[src_off + j];
                }
                key[e] = float_key(sc, nan_seen);
            }
        }
    }
    if (nan_seen) raise_flag(p.flags, 2u /*SVL_DEVFLAG_NONFINITE*/);

    // ----------------------------------------------------------- radix select
    // Find prefix P / mask M / k_rem such that selected = {key&M > P} plus the
    // first k_rem (in index order) of {key&M == P}.
    uint32_t P = 0u, M = 0u, krem = (uint32_t)k;
    if (k > 0 && k < n) {
        const int shifts[3] = {21, 10, 0};
        const int widths[3] = {11, 11, 10};
        for (int pass = 0; pass < 3; ++pass) {
            const int buf = pass & 1;
            const int sh = shifts[pass];
            const int nb = 1 << widths[pass];
            const uint32_t dmask = (uint32_t)(nb - 1);
            for (int i = tid; i < nb; i += NTH) sm.hist[buf][i] = 0u;
            __syncthreads();
#pragma unroll
            for (int e = 0; e < EMAX; ++e)
                if (e < E && my0 + e < j1 && (key[e] & M) == P)
                    atomicAdd(&sm.hist[buf][(key[e] >> sh) & dmask], 1u);
            cluster.sync();
            // owner reduction: CTA `rank` owns bins [rank*bpo, (rank+1)*bpo)
            const int bpo = nb / CS;
            uint32_t own_part = 0u;
            for (int i = tid; i < bpo; i += NTH) {
                uint32_t s = 0u;
                for (int q = 0; q < CS; ++q) {
                    const uint32_t* rh = cluster.map_shared_rank(&sm.hist[buf][0], q);
                    s += rh[rank * bpo + i];
                }
                sm.own[buf][i] = s;
                own_part += s;
            }
            uint32_t tot;
            (void)block_exclusive_scan(own_part, sm.warp_sums, tot);
            if (tid == 0) sm.own_total[buf] = tot;
            cluster.sync();
            // locate the bin holding the krem-th largest (scan from the top)
            if (warp == 0) {
                uint32_t ot = 0u;
                if (lane < CS) ot = *cluster.map_shared_rank(&sm.own_total[buf], lane);
                // suffix sums over owners (descending owner = descending bins)
                uint32_t suf = ot;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint32_t y = __shfl_down_sync(0xffffffffu, suf, off);
                    if (lane + off < 32) suf += y;
                }
                // owner o*: largest lane with suf >= krem
                const unsigned ball = __ballot_sync(0xffffffffu, lane < CS && suf >= krem);
                const int ostar = 31 - __clz(ball);
                const uint32_t above_owner =
                    __shfl_sync(0xffffffffu, suf, ostar) - __shfl_sync(0xffffffffu, ot, ostar);
                // bins of o*: each lane takes a contiguous group, scan from top
                const uint32_t* rown = cluster.map_shared_rank(&sm.own[buf][0], ostar);
                const int per = (bpo + 31) / 32;
                uint32_t grp = 0u;
                for (int i = 0; i < per; ++i) {
                    const int bin = lane * per + i;
                    if (bin < bpo) grp += rown[bin];
                }
                uint32_t gsuf = grp;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint32_t y = __shfl_down_sync(0xffffffffu, gsuf, off);
                    if (lane + off < 32) gsuf += y;
                }
                const uint32_t need = krem - above_owner;
                const unsigned ball2 = __ballot_sync(0xffffffffu, gsuf >= need);
                const int lstar = 31 - __clz(ball2);
                if (lane == lstar) {
                    uint32_t above = gsuf - grp;  // bins of o* above this lane's group
                    int bstar = lane * per;
                    for (int i = per - 1; i >= 0; --i) {
                        const int bin = lane * per + i;
                        if (bin >= bpo) continue;
                        const uint32_t cnt = rown[bin];
                        if (above + cnt >= need) {
                            bstar = bin;
                            break;
                        }
                        above += cnt;
                    }
                    const uint32_t digit = (uint32_t)(ostar * bpo + bstar);
                    sm.res_prefix = P | (digit << sh);
                    sm.res_mask = M | (dmask << sh);
                    sm.res_krem = need - above;
                }
            }
            __syncthreads();
            P = sm.res_prefix;
            M = sm.res_mask;
            krem = sm.res_krem;
            __syncthreads();
        }
    } else if (k == n) {
        P = 0u; M = 0u; krem = (uint32_t)n;  // everything ties with the empty prefix
    }

    // ------------------------------------------------------------ compaction
    uint32_t gt = 0u, eq = 0u;
#pragma unroll
    for (int e = 0; e < EMAX; ++e)
        if (e < E && my0 + e < j1 && k > 0) {
            const uint32_t km = key[e] & M;
            gt += (km > P);
            eq += (km == P);
        }
    uint32_t tot;
    const uint32_t excl = block_exclusive_scan(gt | (eq << 16), sm.warp_sums, tot);
    if (tid == 0) {
        sm.cta_gt = tot & 0xffffu;
        sm.cta_eq = tot >> 16;
    }
    cluster.sync();
    uint32_t eq_before = 0u, sel_before = 0u;
    {
        // cluster prefix over lower ranks (fixed order)
        uint32_t eq_acc = 0u;
        for (int q = 0; q < rank; ++q) {
            const uint32_t qg = *cluster.map_shared_rank(&sm.cta_gt, q);
            const uint32_t qe = *cluster.map_shared_rank(&sm.cta_eq, q);
            const uint32_t quota = (krem > eq_acc) ? min(krem - eq_acc, qe) : 0u;
            sel_before += qg + quota;
            eq_acc += qe;
        }
        eq_before = eq_acc;
    }
    const uint32_t quota = (krem > eq_before) ? (krem - eq_before) : 0u;
    uint32_t gt_run = excl & 0xffffu, eq_run = excl >> 16;
    if (k > 0) {
#pragma unroll
        for (int e = 0; e < EMAX; ++e)
            if (e < E && my0 + e < j1) {
                const uint32_t km = key[e] & M;
                const bool isgt = km > P, iseq = km == P;
                if (isgt || (iseq && eq_run < quota)) {
                    const uint32_t pos = sel_before + gt_run + min(eq_run, quota);
                    p.idx_out[out_off + pos] = my0 + e;
                }
                gt_run += isgt;
                eq_run += iseq;
            }
    }
    cluster.sync();  // keep shared memory alive until every peer finished reading it
}

__global__ void __launch_bounds__(NTH, 1) select_retrieve_kernel(const SelectParams p) {
    select_body<0>(p, nullptr);
}

__global__ void __launch_bounds__(NTH, 1)
    select_prune_kernel(const SelectParams p, const __grid_constant__ PruneTable tab) {
    select_body<1>(p, &tab);
}

}  // namespace

int select_cluster_size(int n) {
    int cs = (n + 2047) / 2048;
    if (cs < 1) cs = 1;
    if (cs > 16) cs = 16;
    // power of two so that NB / CS bins split evenly between owners
    int c = 1;
    while (c < cs) c <<= 1;
    return c;
}

template <typename Kern, typename... Args>
static cudaError_t launch_cluster(Kern kern, int CS, int n_units, cudaStream_t s, bool& attr_done,
                                  Args... args) {
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS, n_units, 1);
    cfg.blockDim = dim3(NTH, 1, 1);
    cfg.dynamicSmemBytes = 0;
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
    static bool done[2][64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    return &done[which][dev & 63];
}

cudaError_t launch_select(const SelectParams& p, int n_units, cudaStream_t s) {
    return launch_cluster(select_retrieve_kernel, p.CS, n_units, s, *attr_flag(0), p);
}

cudaError_t launch_prune_select(const SelectParams& p, const PruneTable& tab, int n_units,
                                cudaStream_t s) {
    return launch_cluster(select_prune_kernel, p.CS, n_units, s, *attr_flag(1), p, tab);
}

}  // namespace svl
