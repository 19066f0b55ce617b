/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the SparseVILA
 * decode-stage hot path (arXiv 2510.17777).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (include/sparsevila.h, paper_2510_17777_b200/csrc) shares
 * no code, header, table or constant with this file and never calls it.
 *
 * Precision: every quantity is IEEE double; bf16 inputs are decoded exactly
 * ((uint32)bits << 16 reinterpreted as float, widened to double).  Plain
 * nested loops in the order the definitions are written; no blocking,
 * fusion or reordering.  OpenMP (optional) only distributes independent
 * units (b, KV group) -- each unit's summation order is fixed, so results are
 * bitwise identical for any thread count.
 *
 * Citations: PAPER.md = /root/reference/PAPER.md (line numbers), SPEC.md
 * likewise; "reading Ax" = DESIGN.md section "Readings of the paper".
 *
 * Error behaviour: functions return 0 on success and a negative code on an
 * invalid argument (the oracle is strict; it never clamps).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define O_VISUAL_ONLY 1u  /* normalise over visual rows only (reading A2)   */
#define O_SHARED 2u       /* one selection per batch row over all groups (A4) */

#define O_ERR_ARG (-1)
#define O_ERR_SHAPE (-2)
#define O_ERR_ORDER (-3)
#define O_ERR_NONFINITE (-4)
#define O_ERR_NOMEM (-5)

static double bf(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
}

/* keep_budget(n, s) = max(1, floor(n*(1-s) + 0.5)) for n > 0, 0 for n = 0;
 * s must lie in [0, 1).  SPEC.md:236-244 (half-up, >=1 clamp); evaluated
 * literally in IEEE double (reading A7). */
int64_t o_keep_budget(int64_t n, double s) {
    if (n < 0 || !(s >= 0.0 && s < 1.0)) return -1;
    if (n == 0) return 0;
    int64_t k = (int64_t)floor((double)n * (1.0 - s) + 0.5);
    if (k < 1) k = 1;
    if (k > n) k = n;
    return k;
}

typedef struct {
    double v;
    int32_t j;
} o_sv;

/* order: value descending, index ascending (ties -> lower index) */
static int cmp_desc_then_idx(const void* a, const void* b) {
    const o_sv* x = (const o_sv*)a;
    const o_sv* y = (const o_sv*)b;
    if (x->v > y->v) return -1;
    if (x->v < y->v) return 1;
    return (x->j < y->j) ? -1 : (x->j > y->j);
}

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x < y) ? -1 : (x > y);
}

/* top-k of v[0..n) by (value desc, index asc); writes ascending indices and
 * rel_gap = (S_(k) - S_(k+1)) / |S_(k)| (+inf when k == 0 or k == n).
 * SPEC.md:245-253 (top_k_indices), SPEC.md:377-385 (select_active). */
static int topk_select(const double* v, int32_t n, int32_t k, int32_t* idx, double* rel_gap) {
    o_sv* a = (o_sv*)malloc(sizeof(o_sv) * (size_t)(n > 0 ? n : 1));
    if (!a) return O_ERR_NOMEM;
    for (int32_t j = 0; j < n; ++j) {
        a[j].v = v[j];
        a[j].j = j;
    }
    qsort(a, (size_t)n, sizeof(o_sv), cmp_desc_then_idx);
    for (int32_t m = 0; m < k; ++m) idx[m] = a[m].j;
    qsort(idx, (size_t)k, sizeof(int32_t), cmp_i32);
    if (rel_gap) {
        if (k == 0 || k == n)
            *rel_gap = INFINITY;
        else
            *rel_gap = (a[k - 1].v - a[k].v) / fabs(a[k - 1].v);
    }
    free(a);
    return 0;
}

/*
 * o_retrieve -- query-aware relevance + per-unit top-k.
 *
 * PAPER.md:124 (section 3.2 "Query-Aware Token Selection"): relevance is "the
 * aggregate attention strength between the query embeddings and visual
 * entries in the KV cache"; "Tokens with the highest relevance scores are
 * retained".  SPEC.md:368-385 (accumulate_relevance, select_active) and
 * SPEC.md:394-396 (full-causal-prefix softmax, SUM over rows and heads).
 *
 * For each unit (b, G) (or b with O_SHARED), in this order:
 *  1. s[r,h,j] = scale * sum_c q[b,r,h,c] * K[b,G,j,c], h in [G*g, G*g+g)
 *     (GQA mapping kv = h / g, reading A5).
 *  2. LSE[r,h] = lse_in[b,r,h] if given, else log sum_j exp(s[r,h,j]) over
 *     the normalisation domain: visual rows, plus (unless O_VISUAL_ONLY) the
 *     text rows [0,vb) and [vb+nv, L) with j <= L - n_q + r (causal).
 *  3. score[j] = sum_r sum_h exp(s[r,h,j] - LSE[r,h]) for visual j, summed
 *     in (G asc,) r asc, h asc order.
 *  4. top-k by (score desc, j asc); indices output ascending, relative to vb.
 *
 * q: bf16 [B][n_q][H][d] contiguous.  K: bf16 with element strides
 * (ksb, ksh, kst), last dim contiguous.  seq_len: [B].  lse_in: nullable
 * [B][n_q][H].  idx_out: [B][U][k] where U = Hkv (or 1 with O_SHARED).
 * scores_out (nullable): [B][U][nv].  rel_gap_out (nullable): [B][U].
 */
int o_retrieve(const uint16_t* q, int B, int n_q, int H, int Hkv, int d,
               const uint16_t* K, int64_t ksb, int64_t ksh, int64_t kst,
               int vb, int nv, const int32_t* seq_len, const double* lse_in,
               int k, double scale, unsigned flags,
               int32_t* idx_out, double* scores_out, double* rel_gap_out,
               int nthreads) {
    if (B < 0 || n_q < 1 || H < 1 || Hkv < 1 || d < 1 || H % Hkv != 0) return O_ERR_SHAPE;
    if (nv < 1 || vb < 0) return O_ERR_SHAPE;
    if (k < 0 || k > nv) return O_ERR_ARG;
    const int g = H / Hkv;
    const int shared = (flags & O_SHARED) != 0;
    const int U = shared ? 1 : Hkv;
    for (int b = 0; b < B; ++b)
        if (seq_len[b] < vb + nv + n_q) return O_ERR_SHAPE;
    int err = 0;
    (void)nthreads;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1) reduction(min : err)
    for (int unit = 0; unit < B * U; ++unit) {
        const int b = unit / U;
        const int L = seq_len[b];
        double* score = (double*)calloc((size_t)nv, sizeof(double));
        double* s = (double*)malloc(sizeof(double) * (size_t)L);
        if (!score || !s) {
            err = O_ERR_NOMEM;
            free(score);
            free(s);
            continue;
        }
        const int G0 = shared ? 0 : unit % U;
        const int G1 = shared ? Hkv : G0 + 1;
        for (int G = G0; G < G1; ++G) {
            const uint16_t* Kb = K + (int64_t)b * ksb + (int64_t)G * ksh;
            for (int r = 0; r < n_q; ++r) {
                for (int h = G * g; h < G * g + g; ++h) {
                    const uint16_t* qv = q + (((int64_t)b * n_q + r) * H + h) * d;
                    const int lim = L - n_q + r; /* causal: j <= lim */
                    /* step 1: logits for every row of the domain */
                    for (int j = 0; j <= lim; ++j) {
                        const int is_vis = (j >= vb && j < vb + nv);
                        if (!is_vis && (flags & O_VISUAL_ONLY)) continue;
                        double acc = 0.0;
                        const uint16_t* kr = Kb + (int64_t)j * kst;
                        for (int c = 0; c < d; ++c) acc += bf(qv[c]) * bf(kr[c]);
                        s[j] = scale * acc;
                    }
                    /* step 2: log-sum-exp over the domain */
                    double lse;
                    if (lse_in) {
                        lse = lse_in[((int64_t)b * n_q + r) * H + h];
                    } else {
                        double m = -INFINITY;
                        for (int j = 0; j <= lim; ++j) {
                            const int is_vis = (j >= vb && j < vb + nv);
                            if (!is_vis && (flags & O_VISUAL_ONLY)) continue;
                            if (s[j] > m) m = s[j];
                        }
                        double sum = 0.0;
                        for (int j = 0; j <= lim; ++j) {
                            const int is_vis = (j >= vb && j < vb + nv);
                            if (!is_vis && (flags & O_VISUAL_ONLY)) continue;
                            sum += exp(s[j] - m);
                        }
                        lse = m + log(sum);
                    }
                    /* step 3: visual share of the attention mass */
                    for (int j = 0; j < nv; ++j) score[j] += exp(s[vb + j] - lse);
                }
            }
        }
        for (int j = 0; j < nv; ++j)
            if (!isfinite(score[j])) err = O_ERR_NONFINITE;
        if (scores_out) memcpy(scores_out + (int64_t)unit * nv, score, sizeof(double) * (size_t)nv);
        int e = topk_select(score, nv, k, idx_out + (int64_t)unit * k,
                            rel_gap_out ? rel_gap_out + unit : NULL);
        if (e) err = e;
        free(score);
        free(s);
    }
    return err;
}

/* Attention of one query row over an ascending row list:
 * s_j = scale * q . K_j ; m = max ; w_j = exp(s_j - m) ;
 * out = sum w_j V_j / sum w_j ; lse = m + log sum w_j.   SPEC.md:52 (attention),
 * SPEC.md:143-151 (decode step), north star step (3). */
static void attend_rows(const uint16_t* qv, int d, const uint16_t* Kb, int64_t kst,
                        const uint16_t* Vb, int64_t vst, const int32_t* rows, int n,
                        double scale, double* s, double* out, double* lse) {
    double m = -INFINITY;
    for (int i = 0; i < n; ++i) {
        double acc = 0.0;
        const uint16_t* kr = Kb + (int64_t)rows[i] * kst;
        for (int c = 0; c < d; ++c) acc += bf(qv[c]) * bf(kr[c]);
        s[i] = scale * acc;
        if (s[i] > m) m = s[i];
    }
    double l = 0.0;
    for (int c = 0; c < d; ++c) out[c] = 0.0;
    for (int i = 0; i < n; ++i) {
        const double w = exp(s[i] - m);
        l += w;
        const uint16_t* vr = Vb + (int64_t)rows[i] * vst;
        for (int c = 0; c < d; ++c) out[c] += w * bf(vr[c]);
    }
    for (int c = 0; c < d; ++c) out[c] /= l;
    *lse = m + log(l);
}

/*
 * o_sparse_decode -- decode attention over the active set.
 *
 * PAPER.md:121 ("selectively activates only the most query-relevant visual
 * tokens during decoding attention, while preserving the rest ... in the KV
 * cache"), PAPER.md:124 (selected entries packed, non-selected inactive),
 * SPEC.md:315-323 (pack_active: all non-visual entries PLUS the selected
 * visual entries, in original order).  For (b, h) the attended rows are,
 * ascending: [0, vb) U { vb + idx[b][G][m] : m < k } U [vb+nv, seq_len[b]),
 * G = h / g (or 0 with O_SHARED).  idx must be strictly ascending and in
 * [0, nv) (else O_ERR_ORDER).  q: bf16 [B][H][d]; out: [B][H][d]; lse: [B][H].
 * idx == NULL means every visual row (k must equal nv): dense attention.
 */
int o_sparse_decode(const uint16_t* q, int B, int H, int Hkv, int d,
                    const uint16_t* K, int64_t ksb, int64_t ksh, int64_t kst,
                    const uint16_t* V, int64_t vsb, int64_t vsh, int64_t vst,
                    int vb, int nv, const int32_t* seq_len,
                    const int32_t* idx, int k, unsigned flags, double scale,
                    double* out, double* lse, int nthreads) {
    if (B < 0 || H < 1 || Hkv < 1 || d < 1 || H % Hkv != 0) return O_ERR_SHAPE;
    if (vb < 0 || nv < 0 || k < 0 || k > nv) return O_ERR_ARG;
    if (!idx && k != nv) return O_ERR_ARG;
    const int g = H / Hkv;
    const int U = (flags & O_SHARED) ? 1 : Hkv;
    for (int b = 0; b < B; ++b)
        if (seq_len[b] < vb + nv) return O_ERR_SHAPE;
    if (idx) {
        for (int64_t u = 0; u < (int64_t)B * U; ++u)
            for (int m = 0; m < k; ++m) {
                const int32_t x = idx[u * k + m];
                if (x < 0 || x >= nv) return O_ERR_ORDER;
                if (m > 0 && x <= idx[u * k + m - 1]) return O_ERR_ORDER;
            }
    }
    int err = 0;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1) reduction(min : err)
    for (int bh = 0; bh < B * H; ++bh) {
        const int b = bh / H, h = bh % H, G = h / g;
        const int L = seq_len[b];
        int32_t* rows = (int32_t*)malloc(sizeof(int32_t) * (size_t)(L > 0 ? L : 1));
        double* s = (double*)malloc(sizeof(double) * (size_t)(L > 0 ? L : 1));
        if (!rows || !s) {
            err = O_ERR_NOMEM;
            free(rows);
            free(s);
            continue;
        }
        int n = 0;
        for (int j = 0; j < vb; ++j) rows[n++] = j;
        const int uG = (flags & O_SHARED) ? 0 : G;
        for (int m = 0; m < k; ++m)
            rows[n++] = vb + (idx ? idx[((int64_t)b * U + uG) * k + m] : m);
        for (int j = vb + nv; j < L; ++j) rows[n++] = j;
        double lse_dummy;
        attend_rows(q + (int64_t)bh * d, d, K + (int64_t)b * ksb + (int64_t)G * ksh, kst,
                    V + (int64_t)b * vsb + (int64_t)G * vsh, vst, rows, n, scale, s,
                    out + (int64_t)bh * d, lse ? lse + bh : &lse_dummy);
        free(rows);
        free(s);
    }
    return err;
}

/* Dense decode attention over rows [0, seq_len[b]) -- o_sparse_decode with
 * every visual row active ("decode with full view == dense"). */
int o_dense_attn(const uint16_t* q, int B, int H, int Hkv, int d,
                 const uint16_t* K, int64_t ksb, int64_t ksh, int64_t kst,
                 const uint16_t* V, int64_t vsb, int64_t vsh, int64_t vst,
                 const int32_t* seq_len, double scale, double* out, double* lse,
                 int nthreads) {
    return o_sparse_decode(q, B, H, Hkv, d, K, ksb, ksh, kst, V, vsb, vsh, vst,
                           0, 0, seq_len, NULL, 0, 0u, scale, out, lse, nthreads);
}

/*
 * o_salience -- query-agnostic visual-token salience from encoder attention.
 *
 * PAPER.md:113 (section 3.1 "Token Salience Estimation"): single summary
 * token (CLIP) -> attention of the summary token to each token; multiple
 * summary tokens (RADIO) -> mean attention toward the summary tokens... read
 * per SPEC.md:190 as the mean over summary rows of their attention to token
 * j; no summary token (SigLIP, QwenVL) -> average intra-visual attention.
 * P = softmax_rows(Q K^T / sqrt(d)) per head (all S+N_f
 * columns in the denominator), mean over heads (reading A12).
 *   mode 0 SUMMARY        (S == 1): sal_j = mean_h P_h[0, S+j]
 *   mode 1 MULTI_SUMMARY  (S >= 2): sal_j = mean_h (1/S) sum_{s<S} P_h[s, S+j]
 *   mode 2 INTRA_VISUAL   (S == 0): sal_j = mean_h (1/N_f) sum_{i<N_f} P_h[i, j]
 * Qe, Ke: bf16 [F][S+N_f][H_e][d_e] contiguous.  sal: [F][N_f].
 */
int o_salience(const uint16_t* Qe, const uint16_t* Ke, int F, int S, int Nf, int He, int de,
               int mode, double scale, double* sal, int nthreads) {
    if (F < 0 || S < 0 || Nf < 1 || He < 1 || de < 1) return O_ERR_SHAPE;
    if ((mode == 0 && S != 1) || (mode == 1 && S < 2) || (mode == 2 && S != 0) || mode < 0 ||
        mode > 2)
        return O_ERR_ARG;
    const int T = S + Nf;
    int err = 0;
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1) reduction(min : err)
    for (int f = 0; f < F; ++f) {
        double* p = (double*)malloc(sizeof(double) * (size_t)T);
        double* acc = (double*)calloc((size_t)Nf, sizeof(double));
        if (!p || !acc) {
            err = O_ERR_NOMEM;
            free(p);
            free(acc);
            continue;
        }
        const int n_rows = (mode == 2) ? Nf : S; /* the rows whose attention is read */
        for (int h = 0; h < He; ++h) {
            double* hacc = (double*)calloc((size_t)Nf, sizeof(double));
            for (int i = 0; i < n_rows; ++i) {
                const uint16_t* qi = Qe + (((int64_t)f * T + i) * He + h) * de;
                double m = -INFINITY;
                for (int j = 0; j < T; ++j) {
                    const uint16_t* kj = Ke + (((int64_t)f * T + j) * He + h) * de;
                    double a = 0.0;
                    for (int c = 0; c < de; ++c) a += bf(qi[c]) * bf(kj[c]);
                    p[j] = scale * a;
                    if (p[j] > m) m = p[j];
                }
                double z = 0.0;
                for (int j = 0; j < T; ++j) {
                    p[j] = exp(p[j] - m);
                    z += p[j];
                }
                for (int j = 0; j < Nf; ++j) hacc[j] += p[S + j] / z;
            }
            for (int j = 0; j < Nf; ++j) acc[j] += hacc[j] / (double)n_rows;
            free(hacc);
        }
        for (int j = 0; j < Nf; ++j) sal[(int64_t)f * Nf + j] = acc[j] / (double)He;
        free(p);
        free(acc);
    }
    return err;
}

/*
 * o_prune -- per-frame query-agnostic prefill pruning.
 *
 * PAPER.md:113 ("pruning those with the lowest aggregate salience"),
 * PAPER.md:199-200 ("a constant prefill sparsity before the LLM"),
 * SPEC.md:474-482 (salience -> keep_budget -> top_k -> pack_order), per frame
 * (north star; reading A13).  For each b and frame f = [o_f, o_{f+1}):
 * k_f = keep_budget(N_f, s); top-k_f by (saliency desc, index asc); frames
 * concatenated in order; output ascending global indices in [0, N).
 * frame_offsets == NULL means a single frame [0, N) (global pruning).
 * kept: [B][cap]; kept_total (out) = sum_f k_f; cap must be >= kept_total.
 * Saliency values are compared exactly as given (fp32 widened to double).
 */
int o_prune(const float* sal, int B, int N, const int32_t* frame_offsets, int n_frames,
            double s, int32_t* kept, int cap, int32_t* kept_total) {
    if (B < 0 || N < 0) return O_ERR_SHAPE;
    if (!(s >= 0.0 && s < 1.0)) return O_ERR_ARG;
    int32_t one[2] = {0, N};
    const int32_t* off = frame_offsets ? frame_offsets : one;
    const int nf = frame_offsets ? n_frames : 1;
    if (off[0] != 0 || off[nf] != N) return O_ERR_SHAPE;
    int64_t total = 0;
    for (int f = 0; f < nf; ++f) {
        if (off[f + 1] < off[f]) return O_ERR_SHAPE;
        total += o_keep_budget(off[f + 1] - off[f], s);
    }
    if (total > cap) return O_ERR_ARG;
    *kept_total = (int32_t)total;
    double* v = (double*)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
    int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(N > 0 ? N : 1));
    if (!v || !tmp) {
        free(v);
        free(tmp);
        return O_ERR_NOMEM;
    }
    int err = 0;
    for (int b = 0; b < B && !err; ++b) {
        int pos = 0;
        for (int f = 0; f < nf; ++f) {
            const int n = off[f + 1] - off[f];
            const int kf = (int)o_keep_budget(n, s);
            for (int j = 0; j < n; ++j) {
                v[j] = (double)sal[(int64_t)b * N + off[f] + j];
                if (!isfinite(v[j])) err = O_ERR_NONFINITE;
            }
            topk_select(v, n, kf, tmp, NULL);
            for (int m = 0; m < kf; ++m) kept[(int64_t)b * cap + pos++] = off[f] + tmp[m];
        }
    }
    free(v);
    free(tmp);
    return err;
}

/* ---------------------------------------------------------------------------
 * Unified RoPE remap after prefill pruning (PAPER.md:127
 * "we simply retain a contiguous range of position indices corresponding to
 * the preserved visual tokens"; SPEC.md:421-427 remap_unified
 * "remap recomputes post-RoPE keys from stored pre-RoPE keys").
 *
 * Plan (per batch row b, seq_len L = seq_len[b]):
 *   new row / position w in [0, vb)             <- old row w          (system text)
 *   w = vb + i, i < k                           <- old row vb + kept[b][i]
 *   w in [vb + k, vb + k + (L - vb - nv))       <- old row w - k + nv (later text)
 * so kept visual token i gets position vb + i, the text start moves from vb + nv
 * to vb + k (delta = k - nv <= 0).
 * Rotation (rotate-half convention of the cited model family, pairs (c, c + d/2)):
 *   theta_c = p * base^(-2c/d),  c < d/2
 *   out[c]       = x[c] cos theta_c - x[c + d/2] sin theta_c
 *   out[c + d/2] = x[c + d/2] cos theta_c + x[c] sin theta_c
 * in double, NOT rounded (the test compares the kernel's bf16 within one ulp).
 * rows_out[b][w] = the old row copied into w (or -1 past the packed length).
 * --------------------------------------------------------------------------- */
int o_rope_remap(const uint16_t* Kpre, int B, int Hkv, int d, int cap, const int32_t* seq_len, int vb, int nv,
                 const int32_t* kept, int k, double base, double* Kout, int cap_out, int32_t* rows_out) {
    if (B < 1 || Hkv < 1 || d < 2 || (d & 1) || vb < 0 || nv < 0 || k < 0 || k > nv || !(base > 1.0))
        return O_ERR_ARG;
    for (int b = 0; b < B; ++b) {
        const int L = seq_len[b];
        if (L < vb + nv || L > cap) return O_ERR_SHAPE;
        const int n_out = vb + k + (L - vb - nv);
        if (n_out > cap_out) return O_ERR_SHAPE;
        for (int i = 0; i < k; ++i) {
            const int x = kept[(int64_t)b * k + i];
            if (x < 0 || x >= nv || (i > 0 && kept[(int64_t)b * k + i - 1] >= x)) return O_ERR_ORDER;
        }
        for (int w = 0; w < cap_out; ++w) {
            int old = -1;
            if (w < vb) old = w;
            else if (w < vb + k) old = vb + kept[(int64_t)b * k + (w - vb)];
            else if (w < n_out) old = w - k + nv;
            rows_out[(int64_t)b * cap_out + w] = old;
            for (int G = 0; G < Hkv; ++G) {
                double* o = Kout + (((int64_t)b * Hkv + G) * cap_out + w) * d;
                if (old < 0) {
                    for (int c = 0; c < d; ++c) o[c] = 0.0;
                    continue;
                }
                const uint16_t* xk = Kpre + (((int64_t)b * Hkv + G) * cap + old) * d;
                const double p = (double)w;  /* unified: the new position is the new row */
                for (int c = 0; c < d / 2; ++c) {
                    const double theta = p * pow(base, -2.0 * (double)c / (double)d);
                    const double x1 = bf(xk[c]), x2 = bf(xk[c + d / 2]);
                    o[c] = x1 * cos(theta) - x2 * sin(theta);
                    o[c + d / 2] = x2 * cos(theta) + x1 * sin(theta);
                }
            }
        }
    }
    return 0;
}

/*
 * o_page_summary -- per-page elementwise key bounds (
 * PAPER.md:527 "Quest estimates upper-bound attention scores for each page").
 * For each unit (b, G) and page p of `page` consecutive visual rows
 * [vb + p*page, vb + (p+1)*page):
 *   kmax[b][G][p][c] = max_j K[b,G,j,c],  kmin[b][G][p][c] = min_j K[b,G,j,c]
 * (exact: the max / min of bf16 values is a bf16 value; returned as double).
 * nv % page == 0 (reading A22).
 */
int o_page_summary(const uint16_t* K, int B, int Hkv, int d, int64_t ksb, int64_t ksh, int64_t kst,
                   int vb, int nv, int page, double* kmax, double* kmin) {
    if (B < 0 || Hkv < 1 || d < 1 || vb < 0 || nv < 1 || page < 1 || nv % page) return O_ERR_SHAPE;
    const int np = nv / page;
    for (int b = 0; b < B; ++b)
        for (int G = 0; G < Hkv; ++G) {
            const uint16_t* Kb = K + (int64_t)b * ksb + (int64_t)G * ksh;
            for (int p = 0; p < np; ++p)
                for (int c = 0; c < d; ++c) {
                    double mx = -INFINITY, mn = INFINITY;
                    for (int j = vb + p * page; j < vb + (p + 1) * page; ++j) {
                        const double v = bf(Kb[(int64_t)j * kst + c]);
                        if (v > mx) mx = v;
                        if (v < mn) mn = v;
                    }
                    const int64_t o = (((int64_t)b * Hkv + G) * np + p) * d + c;
                    kmax[o] = mx;
                    kmin[o] = mn;
                }
        }
    return 0;
}

/*
 * o_retrieve_pages -- query-aware retrieval on page summaries (SURVEY.md 8(f)
 * f2(ii); PAPER.md:527 Quest; reading A22).  For each unit (b, G):
 *  1. ub[r,h,p] = scale * sum_c max(q[b,r,h,c] * kmax[p][c], q[b,r,h,c] * kmin[p][c])
 *     -- an upper bound of scale * q . K_j over every row j of page p (Quest);
 *  2. LSEp[r,h] = log sum_p exp(ub[r,h,p])   (softmax over the unit's pages);
 *  3. score[p] = sum_r sum_h exp(ub[r,h,p] - LSEp[r,h]), r asc, h asc  (the
 *     page analogue of the visual-only relevance, readings A2, A3);
 *  4. top-k_p pages by (score desc, p asc); page indices ascending.
 * With page = 1 this is o_retrieve with O_VISUAL_ONLY.
 * kmax, kmin: double [B][Hkv][np][d] (o_page_summary); q bf16 [B][n_q][H][d].
 */
int o_retrieve_pages(const uint16_t* q, int B, int n_q, int H, int Hkv, int d, const double* kmax,
                     const double* kmin, int np, int kp, double scale, int32_t* pidx_out,
                     double* scores_out, double* rel_gap_out) {
    if (B < 0 || n_q < 1 || H < 1 || Hkv < 1 || H % Hkv || d < 1 || np < 1) return O_ERR_SHAPE;
    if (kp < 0 || kp > np) return O_ERR_ARG;
    const int g = H / Hkv;
    double* ub = (double*)malloc(sizeof(double) * (size_t)np);
    double* score = (double*)malloc(sizeof(double) * (size_t)np);
    if (!ub || !score) {
        free(ub);
        free(score);
        return O_ERR_NOMEM;
    }
    int err = 0;
    for (int b = 0; b < B; ++b)
        for (int G = 0; G < Hkv; ++G) {
            for (int p = 0; p < np; ++p) score[p] = 0.0;
            const double* mx = kmax + ((int64_t)b * Hkv + G) * np * d;
            const double* mn = kmin + ((int64_t)b * Hkv + G) * np * d;
            for (int r = 0; r < n_q; ++r)
                for (int h = G * g; h < G * g + g; ++h) {
                    const uint16_t* qv = q + (((int64_t)b * n_q + r) * H + h) * d;
                    for (int p = 0; p < np; ++p) {
                        double acc = 0.0;
                        for (int c = 0; c < d; ++c) {
                            const double a = bf(qv[c]) * mx[(int64_t)p * d + c];
                            const double e = bf(qv[c]) * mn[(int64_t)p * d + c];
                            acc += (a > e) ? a : e;
                        }
                        ub[p] = scale * acc;
                    }
                    double m = -INFINITY;
                    for (int p = 0; p < np; ++p)
                        if (ub[p] > m) m = ub[p];
                    double sum = 0.0;
                    for (int p = 0; p < np; ++p) sum += exp(ub[p] - m);
                    const double lse = m + log(sum);
                    for (int p = 0; p < np; ++p) score[p] += exp(ub[p] - lse);
                }
            const int unit = b * Hkv + G;
            for (int p = 0; p < np; ++p)
                if (!isfinite(score[p])) err = O_ERR_NONFINITE;
            if (scores_out) memcpy(scores_out + (int64_t)unit * np, score, sizeof(double) * (size_t)np);
            const int e = topk_select(score, np, kp, pidx_out + (int64_t)unit * kp,
                                      rel_gap_out ? rel_gap_out + unit : NULL);
            if (e) err = e;
        }
    free(ub);
    free(score);
    return err;
}

/*
 * o_mrope_plan -- multimodal-RoPE remap plan after pruning (SURVEY.md 8(f)
 * f4(i); "reconstruct the minimal contiguous positional grid along
 * temporal, height, and width dimensions and then shift subsequent text
 * positions to maintain global continuity"; SPEC.md:428-433 remap_mrope;
 * reading A23).  Per batch row b, for each dimension x in (t, h, w)
 * independently: the distinct values of the kept tokens' coordinates, ranked
 * in increasing order (coordinate compression): x' = #{distinct kept values < x}.
 * Positions are offset by the text before the visual span: the kept token's
 * position in dimension x is vb + x'; the first later text token takes the
 * scalar position text_start = vb + 1 + max over kept tokens of max(t', h', w')
 * (Qwen-style continuation; 0-kept: vb).
 * coords: [B][nv][3] (t, h, w) of the original visual rows, each >= 0.
 * kept: [B][k] ascending in [0, nv).  Outputs new_coords [B][k][3] (t', h', w')
 * and text_start [B].  Duplicate kept triples -> O_ERR_ARG.
 */
int o_mrope_plan(const int32_t* coords, int B, int nv, int vb, const int32_t* kept, int k, int32_t* new_coords,
                 int32_t* text_start) {
    if (B < 1 || nv < 0 || vb < 0 || k < 0 || k > nv) return O_ERR_ARG;
    for (int b = 0; b < B; ++b) {
        const int32_t* kb = kept + (int64_t)b * k;
        for (int i = 0; i < k; ++i)
            if (kb[i] < 0 || kb[i] >= nv || (i > 0 && kb[i - 1] >= kb[i])) return O_ERR_ORDER;
        /* duplicate triples (brute force) */
        for (int i = 0; i < k; ++i)
            for (int j = i + 1; j < k; ++j) {
                const int32_t* a = coords + ((int64_t)b * nv + kb[i]) * 3;
                const int32_t* c = coords + ((int64_t)b * nv + kb[j]) * 3;
                if (a[0] == c[0] && a[1] == c[1] && a[2] == c[2]) return O_ERR_ARG;
            }
        int32_t mx = -1;
        int32_t* vals = (int32_t*)malloc(sizeof(int32_t) * (size_t)(k > 0 ? k : 1));
        if (!vals) return O_ERR_NOMEM;
        for (int x = 0; x < 3; ++x) {
            /* the distinct kept values of this dimension, ascending (sort + unique) */
            for (int i = 0; i < k; ++i) {
                vals[i] = coords[((int64_t)b * nv + kb[i]) * 3 + x];
                if (vals[i] < 0) {
                    free(vals);
                    return O_ERR_ARG;
                }
            }
            qsort(vals, (size_t)k, sizeof(int32_t), cmp_i32);
            int nd = 0;
            for (int i = 0; i < k; ++i)
                if (i == 0 || vals[i] != vals[i - 1]) vals[nd++] = vals[i];
            /* rank = number of distinct kept values below v = its position in vals */
            for (int i = 0; i < k; ++i) {
                const int32_t v = coords[((int64_t)b * nv + kb[i]) * 3 + x];
                int32_t r = 0;
                while (r < nd && vals[r] < v) ++r;
                new_coords[((int64_t)b * k + i) * 3 + x] = r;
                if (r > mx) mx = r;
            }
        }
        free(vals);
        text_start[b] = (k > 0) ? vb + 1 + mx : vb;
    }
    return 0;
}

/*
 * o_mrope_remap -- apply the plan to the cache (post-RoPE keys are
 * recomputed from the stored pre-RoPE keys; reading A23).  Output rows as in
 * o_rope_remap: [0, vb) system text, [vb, vb + k) kept visual, then the later
 * text rows.  Rotate-half pairs (c, c + d/2); pair c takes the position of its
 * section: c < sec[0] -> t, c < sec[0] + sec[1] -> h, else w; text rows use
 * their scalar position on every section (system row w: w; later text row i:
 * text_start + i).  theta_c = pos * base^(-2c/d), all in double.
 */
int o_mrope_remap(const uint16_t* Kpre, int B, int Hkv, int d, int cap, const int32_t* seq_len, int vb, int nv,
                  const int32_t* kept, int k, const int32_t* new_coords, const int32_t* text_start,
                  const int32_t* sec, double base, double* Kout, int cap_out, int32_t* rows_out) {
    if (B < 1 || Hkv < 1 || d < 2 || (d & 1) || vb < 0 || nv < 0 || k < 0 || k > nv || !(base > 1.0))
        return O_ERR_ARG;
    if (sec[0] < 0 || sec[1] < 0 || sec[2] < 0 || sec[0] + sec[1] + sec[2] != d / 2) return O_ERR_ARG;
    for (int b = 0; b < B; ++b) {
        const int L = seq_len[b];
        if (L < vb + nv || L > cap) return O_ERR_SHAPE;
        const int n_out = vb + k + (L - vb - nv);
        if (n_out > cap_out) return O_ERR_SHAPE;
        for (int w = 0; w < cap_out; ++w) {
            int old = -1;
            double pos[3] = {0.0, 0.0, 0.0};
            if (w < vb) {
                old = w;
                pos[0] = pos[1] = pos[2] = (double)w;
            } else if (w < vb + k) {
                const int i = w - vb;
                old = vb + kept[(int64_t)b * k + i];
                for (int x = 0; x < 3; ++x) pos[x] = (double)(vb + new_coords[((int64_t)b * k + i) * 3 + x]);
            } else if (w < n_out) {
                old = w - k + nv;
                pos[0] = pos[1] = pos[2] = (double)(text_start[b] + (w - vb - k));
            }
            rows_out[(int64_t)b * cap_out + w] = old;
            for (int G = 0; G < Hkv; ++G) {
                double* o = Kout + (((int64_t)b * Hkv + G) * cap_out + w) * d;
                if (old < 0) {
                    for (int c = 0; c < d; ++c) o[c] = 0.0;
                    continue;
                }
                const uint16_t* xk = Kpre + (((int64_t)b * Hkv + G) * cap + old) * d;
                for (int c = 0; c < d / 2; ++c) {
                    const int x = (c < sec[0]) ? 0 : (c < sec[0] + sec[1]) ? 1 : 2;
                    const double theta = pos[x] * pow(base, -2.0 * (double)c / (double)d);
                    const double x1 = bf(xk[c]), x2 = bf(xk[c + d / 2]);
                    o[c] = x1 * cos(theta) - x2 * sin(theta);
                    o[c + d / 2] = x2 * cos(theta) + x1 * sin(theta);
                }
            }
        }
    }
    return 0;
}
