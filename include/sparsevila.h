/*
 * sparsevila.h -- C ABI of libsparsevila.so, the B200 (sm_100a) decode-stage
 * hot path of SparseVILA (arXiv 2510.17777, "Decoupling Visual Sparsity for
 * Efficient VLM Inference").
 *
 * Calling rules:
 *  - Plain C types only; every pointer is caller-owned.  "device" pointers
 *    are CUDA global-memory addresses on the current device, "host" pointers
 *    are ordinary CPU memory.  The library never allocates or frees memory.
 *  - Every compute call is stream-ordered and asynchronous on `stream`
 *    (a cudaStream_t passed as void*; NULL = legacy default stream).  Host
 *    argument validation is synchronous: on any non-SVL_OK status nothing was
 *    launched.  No call synchronises the device except
 *    svl_read_device_flags (debug/test only).
 *  - Stateless and re-entrant.  The only globals are a thread-local
 *    last-error string and an immutable per-device attribute cache.
 *  - Scratch comes from a caller-supplied device `workspace` of at least
 *    svl_*_workspace_size(...) bytes (SVL_WORKSPACE_HEADER_BYTES for the calls
 *    without a size function), 256-byte aligned, which must be zero filled
 *    once before its first use (svl_workspace_init).  Its header
 *    (SVL_WORKSPACE_HEADER_BYTES) holds the device flag word and small
 *    self-maintained counters; calls never write another call's header words,
 *    so one workspace may serve any sequence of calls on one stream.  Two calls
 *    that may run concurrently need distinct workspaces.
 *  - bf16 tensors are IEEE bfloat16 bit patterns (uint16).  Row pointers and
 *    row strides must be 16-byte aligned.  Head dims d in {64, 128}.
 *
 * Citations: PAPER.md / SPEC.md line numbers refer to the paper text and the
 * spec written from it (DESIGN.md lists every reading taken where the paper
 * is silent; "reading Ax" below).
 */
#ifndef SPARSEVILA_H_
#define SPARSEVILA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- status */
typedef enum {
    SVL_OK = 0,
    SVL_ERR_INVALID_ARGUMENT = 1, /* k > N_v, sparsity outside [0,1), NULL pointer, bad flags */
    SVL_ERR_SHAPE = 2,            /* H % Hkv != 0, empty visual span, span outside capacity   */
    SVL_ERR_ALIGNMENT = 3,        /* pointer / stride not 16-byte aligned                     */
    SVL_ERR_WORKSPACE = 4,        /* workspace NULL, misaligned or smaller than required      */
    SVL_ERR_UNSUPPORTED = 5,      /* d not in {64,128}, g or n_q*g too large, N_v too large, no sm_100 device */
    SVL_ERR_CUDA = 6              /* a CUDA runtime call or kernel launch failed               */
} svl_status;

#define SVL_WORKSPACE_HEADER_BYTES 1024u

/* Device-side precondition bits, OR-ed into the workspace flag word
 * (svl_read_device_flags).  Offending elements are skipped / treated as the
 * lowest key so kernels never fault. */
#define SVL_DEVFLAG_INDEX 1u      /* vis_idx out of [0,N_v) or not strictly ascending */
#define SVL_DEVFLAG_NONFINITE 2u  /* NaN relevance / saliency; NaN ranks lowest          */
#define SVL_DEVFLAG_SPAN 4u       /* seq_len[b] < visual_begin + visual_len + n_q, or > capacity       */
#define SVL_DEVFLAG_WAIT_TIMEOUT 8u /* svl_wait_flags gave up (~2 s) before every producer flag arrived  */

/* ------------------------------------------------------------------ flags */
#define SVL_NORM_VISUAL_ONLY 1u /* softmax over visual rows only (default: full causal prefix, reading A2) */
#define SVL_SELECT_SHARED 2u    /* one selection per batch row, relevance summed over KV groups (reading A4) */
/* svl_retrieve phase split (profiling / overlap): SCORE_ONLY runs phase 1
 * (logits + chunk log-sum-exp partials into the workspace); SELECT_ONLY runs
 * phase 2 (normalise, aggregate, top-k) from a workspace filled by a
 * SCORE_ONLY call with identical arguments.  Neither bit = both phases. */
#define SVL_RETRIEVE_SCORE_ONLY 0x100u
#define SVL_RETRIEVE_SELECT_ONLY 0x200u
/* svl_fresh_decode_step: always run the two separate calls (svl_retrieve then
 * svl_sparse_decode_attn) instead of the fused kernel (A/B measurements, tests). */
#define SVL_FRESH_UNFUSED 0x400u
/* svl_sparse_decode_attn: vis_idx entries equal to -1 after the valid
 * (ascending) entries of a unit are padding, skipped without a device flag
 * (a shard's share of a sequence-split selection, svl_shard_indices). */
#define SVL_IDX_PADDED 0x800u
/* svl_retrieve / svl_retrieve_partial_lse: the K view is one shard of a
 * sequence-split cache: seq_len >= vb + visual_len suffices
 * (the query rows live in another shard's view). */
#define SVL_SHARD_VIEW 0x1000u
/* svl_sparse_decode_attn(_push): merge the splits through L2 (epoch-tagged
 * partials, co-resident grid) even when the split count would allow a
 * thread-block cluster per unit merged over DSMEM (A/B measurements, tests). */
#define SVL_DECODE_GRID_MERGE 0x2000u
/* svl_sparse_decode_attn(_push): the caller guarantees that vis_idx and every
 * K/V row below seq_len[b] - 1 (all rows but the current token's) are not
 * written by the work enqueued immediately before this call on the stream
 * (steady decode: vis_idx is the last fresh step's selection; the prompt and
 * the earlier tokens' rows were written by earlier steps).  The kernel then
 * loads vis_idx and starts gathering those rows before its programmatic-
 * dependent-launch wait, overlapping the upstream kernel's tail; their text
 * share is laid out from a speculative read of seq_len[b] that is checked after
 * the wait (a changed seq_len re-gathers the text rows).  q, seq_len and the
 * current token's row are read only after the wait.  Results are bitwise
 * identical with and without the flag. */
#define SVL_DECODE_STATIC_PREFIX 0x4000u
/* Split-count pin, flags bits 24..31 (0 = the planner's choice).
 * svl_sparse_decode_attn(_push): exactly n CTAs per (b, KV group) unit
 * (B*Hkv*n must not exceed the co-resident CTA count when n > 1, else
 * SVL_ERR_UNSUPPORTED); svl_fresh_decode_step: a cluster of n CTAs per unit
 * (n = 8 or 16; the fused kernel then runs even past one wave).  Results are a
 * deterministic function of the inputs and the split count, so a sharded run
 * reproduces the unsharded one bitwise when both pin the same n
 * (SURVEY.md 8(e) e5).  The workspace-size calls take the same flags. */
#define SVL_PIN_SPLITS(n) (((uint32_t)(n) & 0xffu) << 24)
#define SVL_PIN_SPLITS_MASK 0xff000000u

/* Salience modes */
#define SVL_SAL_SUMMARY 0       /* S == 1 summary token (CLIP)               */
#define SVL_SAL_MULTI_SUMMARY 1 /* S >= 2 summary tokens (RADIO)             */
#define SVL_SAL_INTRA_VISUAL 2  /* S == 0, mean intra-visual attention (SigLIP, QwenVL) */

/* ------------------------------------------------------------------ types */
/* A bf16 KV-cache view for one decoder layer: element (b, kv_head, row, c)
 * lives at data + b*stride_b + kv_head*stride_h + row*stride_t + c
 * (strides in elements, last dim contiguous).  `capacity` = rows allocated
 * per (b, kv_head).  Device memory. */
typedef struct {
    const void* data;
    int64_t stride_b, stride_h, stride_t;
    int32_t capacity;
} svl_kv;

/* Sequence layout per batch row b:
 * rows [0, visual_begin) are system text, [visual_begin, visual_begin +
 * visual_len) the retained visual tokens, [visual_begin + visual_len,
 * seq_len[b]) question / answer / generated text, the current token last.
 * seq_len is a DEVICE int32 [B] array (it changes every decode step). */
typedef struct {
    int32_t visual_begin;
    int32_t visual_len;
    const int32_t* seq_len;
} svl_span;

/* -------------------------------------------------------------- retrieve */
/*
 * svl_retrieve -- query-aware visual-token retrieval (section
 * 3.2 "Query-Aware Token Selection").
 *
 * For each unit (b, G) -- G a KV group, h in [G*g, G*g+g), g = H/Hkv
 * (kv = h / g, reading A5) -- or each b with SVL_SELECT_SHARED:
 *   s[r,h,j]  = scale * q[b,r,h,:] . K[b,G,j,:]
 *   LSE[r,h]  = lse_in[b,r,h] if lse_in != NULL, else the natural-log
 *               log-sum-exp of s over the causal prefix j <= seq_len-n_q+r
 *               (visual rows only with SVL_NORM_VISUAL_ONLY)
 *   score[j]  = sum_r sum_h exp(s[r,h,j] - LSE[r,h])     (visual j)
 *   idx       = the k visual rows with the largest score, ties to the lower
 *               index, written ascending, relative to visual_begin.
 *
 * q        device bf16 [B][n_q][H][d] contiguous (post-RoPE; reading A10).
 *          n_q*g <= 4096.  n_q*g <= 32 runs the CUDA-core GEMV path; larger
 *          n_q*g (a question chunk) runs the tensor-core path
 *          (tcgen05 row-LSE pass + column-mass pass), which
 *          needs K encodable as a TMA tensor map (SVL_ERR_UNSUPPORTED if not).
 * K        device KV view (see svl_kv).
 * span     visual span + device seq_len[B]; visual_len <= 131072.
 * lse_in   device fp32 [B][n_q][H] or NULL.
 * k        0 <= k <= visual_len (SVL_ERR_INVALID_ARGUMENT otherwise).
 * scale    softmax scale, normally 1/sqrt(d) (reading A6).
 * idx_out  device int32 [B][U][k], U = Hkv (or 1 with SVL_SELECT_SHARED).
 * scores_out  device fp32 [B][U][visual_len] or NULL.
 * Errors: host-checkable shape/argument errors return before launching;
 * NaN scores set SVL_DEVFLAG_NONFINITE; a bad seq_len sets SVL_DEVFLAG_SPAN.
 */
svl_status svl_retrieve(const void* q, int32_t B, int32_t n_q, int32_t H, int32_t Hkv,
                        int32_t d, svl_kv K, svl_span span, const float* lse_in, int32_t k,
                        float scale, uint32_t flags, int32_t* idx_out, float* scores_out,
                        void* workspace, size_t workspace_bytes, void* stream);

size_t svl_retrieve_workspace_size(int32_t B, int32_t n_q, int32_t H, int32_t Hkv, int32_t d,
                                   int32_t visual_len, uint32_t flags);

/*
 * svl_question_attention -- the attention output of the question chunk, the
 * prefill-attention product the retrieval pass accompanies (PAPER.md:124,
 * section 3.2: the relevance kernel "executes concurrently with the
 * FlashAttention2 path during prefill").  For each
 * (b, r, h), r < n_q the question rows (the last n_q rows of seq_len[b]),
 * G = h / g, over the key range j of svl_retrieve's normalisation (the causal
 * prefix j <= seq_len[b] - n_q + r, or the visual rows only with
 * SVL_NORM_VISUAL_ONLY):
 *   LSE[r,h]   = lse_in[b,r,h] if lse_in != NULL, else log sum_j exp(s[r,h,j])
 *   out[r,h,:] = sum_j exp(s[r,h,j] - LSE[r,h]) V[b,G,j,:]
 * with s = scale * q . K_j.  All steps run on the tensor cores (tcgen05): the
 * row-LSE pass of svl_retrieve (skipped with lse_in), then one pass per key
 * chunk computing S, P = exp(S - LSE) rounded to bf16 (reading A24) and P.V;
 * the chunks' partial outputs are summed in chunk order (deterministic).
 * Passing this call's lse_out as svl_retrieve's lse_in runs the retrieval's
 * column-mass pass on the same normalisation without recomputing the LSE.
 *
 * q        device bf16 [B][n_q][H][d] contiguous; n_q * g <= 4096.
 * K, V     device KV views (svl_kv), both encodable as TMA tensor maps
 *          (16-B aligned base, strides multiples of 8 elements), else
 *          SVL_ERR_UNSUPPORTED.
 * span     as svl_retrieve; visual_begin + visual_len + n_q <= capacity.
 * lse_in   device fp32 [B][n_q][H] (natural log) or NULL.
 * flags    0 or SVL_NORM_VISUAL_ONLY.
 * out      device fp32 [B][n_q][H][d] (written).
 * lse_out  device fp32 [B][n_q][H] natural-log LSE used, or NULL.
 * workspace  svl_question_attention_workspace_size bytes, 16-B aligned.
 * Device flags: SVL_DEVFLAG_SPAN when seq_len[b] is outside
 * [visual_begin + visual_len + n_q, capacity] (clamped).
 */
svl_status svl_question_attention(const void* q, int32_t B, int32_t n_q, int32_t H, int32_t Hkv, int32_t d,
                                  svl_kv K, svl_kv V, svl_span span, const float* lse_in, float scale,
                                  uint32_t flags, float* out, float* lse_out, void* workspace,
                                  size_t workspace_bytes, void* stream);
size_t svl_question_attention_workspace_size(int32_t B, int32_t n_q, int32_t H, int32_t Hkv, int32_t d,
                                             int32_t visual_len, uint32_t flags);

/* ---------------------------------------------------- sparse decode attn */
/*
 * svl_sparse_decode_attn -- decode attention over the active set
 * (SPEC.md:143-151, 315-323).
 *
 * For (b, h), G = h / g: attended rows, ascending,
 *   [0, vb)  U  { vb + vis_idx[b][G][m] : m < k }  U  [vb + N_v, seq_len[b])
 * (G replaced by 0 with SVL_SELECT_SHARED).  The caller appends the current
 * token's K/V before the call (reading A9).
 *   out[b,h,:] = sum_j softmax(scale * q.K_j)_j V_j   (fp32, reading A18)
 *   lse[b,h]   = natural-log log-sum-exp of the attended logits
 * Split-K flash-decoding with a log-sum-exp merge across splits, S splits
 * (CTAs) per unit, S from the co-resident CTA count.  While every unit's S
 * CTAs fit as co-resident thread-block clusters (S <= 16), each unit is one
 * cluster and the splits push their partials (o, m, l) to the owning CTAs
 * over distributed shared memory; otherwise the grid is launched
 * cooperatively, each split stores its partial to the workspace tagged with
 * the unit's call epoch (a counter in the workspace header that the unit's
 * first CTA advances once per call), and every split merges a 1/S slice of
 * the unit's outputs as soon as the tagged partials it needs are visible.
 * The merge order is fixed: results are bitwise reproducible for a given
 * split count and merge path.
 * flags    SVL_SELECT_SHARED, SVL_PIN_SPLITS(n), SVL_IDX_PADDED,
 *          SVL_DECODE_GRID_MERGE, SVL_DECODE_STATIC_PREFIX (see above).
 *
 * q        device bf16 [B][H][d] contiguous; g = H/Hkv <= 16.
 * K, V     device KV views with identical capacity.
 * vis_idx  device int32 [B][U][k], strictly ascending, in [0, N_v)
 *          (violations set SVL_DEVFLAG_INDEX; offending rows are skipped).
 *          k = 0 is allowed (text only).
 * out      device fp32 [B][H][d]; lse_out device fp32 [B][H] or NULL.
 */
svl_status svl_sparse_decode_attn(const void* q, int32_t B, int32_t H, int32_t Hkv, int32_t d,
                                  svl_kv K, svl_kv V, svl_span span, const int32_t* vis_idx,
                                  int32_t k, uint32_t flags, float scale, float* out,
                                  float* lse_out, void* workspace, size_t workspace_bytes,
                                  void* stream);

size_t svl_sparse_decode_workspace_size(int32_t B, int32_t H, int32_t Hkv, int32_t d, int32_t k,
                                        int32_t visual_len, int32_t capacity, uint32_t flags);

/*
 * svl_rope_remap -- unified RoPE remap after prefill pruning (SURVEY.md 8(f)
 * f4(i); "retain a contiguous range of position indices
 * corresponding to the preserved visual tokens").
 * For each batch row b (L = seq_len[b]) the compacted cache row w, which is
 * also its new position, takes
 *   old row w                      for w < vb                 (system text)
 *   old row vb + kept[b][w - vb]   for vb <= w < vb + k       (kept visual)
 *   old row w - k + N_v            for vb + k <= w < L - N_v + k  (later text)
 * K_out[b][G][w] = RoPE(K_pre[b][G][old], position w), rotate-half pairs
 * (c, c + d/2), theta_c = w * rope_base^(-2c/d) (angles in double, rotation
 * fp32, bf16 RNE output); V_out[b][G][w] = V[b][G][old] (skipped if V.data is
 * NULL).  The new seq_len is L - N_v + k (the caller's).  Applied once at
 * prefill-prune time; decode-stage retrieval does not remap.
 *
 * K_pre    PRE-RoPE keys at their original rows; V the values (or data NULL).
 * span     the original visual span and device seq_len [B].
 * kept     device int32 [B][k] ascending in [0, N_v) (svl_prefill_prune's output
 *          relative to vb); violations set SVL_DEVFLAG_INDEX and are clamped.
 * K_out, V_out  destination views, capacity >= vb + k + (K_pre.capacity - vb - N_v),
 *          not overlapping the sources.
 */
svl_status svl_rope_remap(svl_kv K_pre, svl_kv V, int32_t B, int32_t Hkv, int32_t d, svl_span span,
                          const int32_t* kept, int32_t k, double rope_base, svl_kv K_out, svl_kv V_out,
                          void* workspace, size_t workspace_bytes, void* stream);

/*
 * svl_mrope_remap -- multimodal-RoPE remap after prefill pruning (SURVEY.md 8(f)
 * f4(i); "reconstruct the minimal contiguous positional grid along
 * temporal, height, and width dimensions and then shift subsequent text
 * positions to maintain global continuity"; reading A23).
 * Plan, per batch row b and dimension x in (t, h, w) independently: the kept
 * tokens' coordinate x is replaced by its rank among the distinct kept values
 * (coordinate compression, order-preserving).  Positions: kept visual token
 * (t', h', w') -> (vb + t', vb + h', vb + w'); system rows keep w; the later
 * text rows continue at text_start = vb + 1 + max over kept of max(t', h', w').
 * Output rows as svl_rope_remap: [0, vb) system, [vb, vb + k) kept visual, then
 * the later text rows.  Rotate-half pairs (c, c + d/2); pair c uses the t
 * position for c < sections[0], h for c < sections[0] + sections[1], else w;
 * theta = pos * rope_base^(-2c/d) in double; bf16 RNE output; V compacted.
 *
 * coords   device int32 [B][visual_len][3] (t, h, w) of the original visual rows,
 *          each in [0, 65536); out-of-range values / a kept list that is not
 *          strictly ascending raise SVL_DEVFLAG_INDEX (clamped).  Duplicate kept
 *          triples are a precondition violation (not detected on the device).
 * kept     device int32 [B][k] ascending in [0, visual_len).
 * sections HOST int32 [3]: rotary pairs per section, sum d/2, first two even
 *          (Qwen2-VL at d = 128: {16, 24, 24}).
 * new_coords_out nullable device int32 [B][k][3]; text_start_out nullable device int32 [B].
 * Workspace: svl_mrope_remap_workspace_size(B, k).
 */
svl_status svl_mrope_remap(svl_kv K_pre, svl_kv V, int32_t B, int32_t Hkv, int32_t d, svl_span span,
                           const int32_t* coords, const int32_t* kept, int32_t k, double rope_base,
                           const int32_t* sections, svl_kv K_out, svl_kv V_out, int32_t* new_coords_out,
                           int32_t* text_start_out, void* workspace, size_t workspace_bytes, void* stream);

size_t svl_mrope_remap_workspace_size(int32_t B, int32_t k);

/*
 * svl_pack_kv -- pack-once of the retained KV cache (
 * PAPER.md:124 "compactly packed into a contiguous memory region";
 * SPEC.md:315-323).  For every unit (b, G) writes into the packed views Kp, Vp:
 *   rows [0, vb)            = K/V rows [0, vb)                     (system text)
 *   rows [vb, vb + k)       = K/V rows vb + vis_idx[b][G][m], m ascending
 *   rows [vb + k, vb + k + seq_len[b] - vb - N_v) = K/V rows [vb + N_v, seq_len[b])
 * so svl_sparse_decode_attn over (Kp, Vp) with visual_len = k, vis_idx = 0..k-1
 * and seq_len - N_v + k attends the same rows in the same order as over (K, V)
 * with vis_idx (bitwise-identical results).  The caller computes the packed
 * seq_len and appends later tokens to the packed views.
 *
 * K, V     source views (identical capacity); span = the source visual span.
 * vis_idx  device int32 [B][U][k] ascending in [0, N_v) (U = 1 with
 *          SVL_SELECT_SHARED); violations set SVL_DEVFLAG_INDEX and are clamped.
 * Kp, Vp   destination views, capacity >= vb + k + (K.capacity - vb - N_v);
 *          must not overlap the sources.
 * Workspace: SVL_WORKSPACE_HEADER_BYTES (device flags); asynchronous on `stream`.
 */
svl_status svl_pack_kv(svl_kv K, svl_kv V, int32_t B, int32_t Hkv, int32_t d, svl_span span,
                       const int32_t* vis_idx, int32_t k, uint32_t flags, svl_kv Kp, svl_kv Vp,
                       void* workspace, size_t workspace_bytes, void* stream);

/*
 * svl_sparse_decode_attn_push -- svl_sparse_decode_attn for one rank's shard of a
 * head-sharded multi-GPU decode (SURVEY.md 8(b) b7, 8(e) e3 "fused variant"),
 * with the all-gather of the head outputs folded into the kernel: the merged
 * output of every (b, h) of the shard is stored straight into EVERY rank's
 * gathered output buffer (NVLink peer stores through the unified address
 * space), and once all of this call's stores are visible system-wide the last
 * CTA sets peer_flags[r][rank] = epoch on every rank r (st.release.sys).  The
 * consumer side is svl_wait_flags.  Replaces the NCCL all-gather of the fp32
 * head outputs per layer (north star: "NCCL all-gather of head outputs").
 *
 * q, K, V, span, vis_idx, k, flags, scale, lse_out: the shard, exactly as for
 *   svl_sparse_decode_attn (B = this rank's batch rows, H / Hkv its heads).
 * out        device fp32 [B][H][d] local copy, or NULL.
 * peer_out   HOST array [P] of device pointers: rank r's gathered output fp32
 *            [B_total][H_total][d] (symmetric; peer access enabled, or all on
 *            one device); the shard lands at rows b0.., heads h0..
 * peer_flags HOST array [P] of device pointers: rank r's flag row uint32 [P].
 * rank, P    this rank, 1 <= P <= 8 (one NVLink/NVSwitch node).
 * epoch      > 0, increasing per call (flags compare modulo 2^32).
 * The workspace header's word 3 is the kernel's self-resetting CTA counter.
 */
svl_status svl_sparse_decode_attn_push(const void* q, int32_t B, int32_t H, int32_t Hkv, int32_t d,
                                       svl_kv K, svl_kv V, svl_span span, const int32_t* vis_idx,
                                       int32_t k, uint32_t flags, float scale, float* out,
                                       float* lse_out, float* const* peer_out,
                                       uint32_t* const* peer_flags, int32_t rank, int32_t P,
                                       uint32_t epoch, int32_t b0, int32_t h0, int32_t B_total,
                                       int32_t H_total, void* workspace, size_t workspace_bytes,
                                       void* stream);

/*
 * svl_wait_flags -- stream-ordered consumer of svl_sparse_decode_attn_push:
 * work enqueued on `stream` after this call starts once flags[s] >= epoch
 * (mod 2^32) for every producer s < P (acquire loads, system scope).  flags
 * is this rank's device flag row uint32 [P].  Bounded: after ~2 s it gives up
 * and sets SVL_DEVFLAG_WAIT_TIMEOUT in the workspace flag word.
 */
svl_status svl_wait_flags(const uint32_t* flags, int32_t P, uint32_t epoch, void* workspace, void* stream);

/* ------------------------------------------------ fused fresh decode step */
/*
 * svl_fresh_decode_step -- svl_retrieve (n_q = 1) followed by
 * svl_sparse_decode_attn with the SAME query, fused: the decode step that
 * re-retrieves its visual tokens.  Because the retrieval
 * logits s = scale*q.K_j are exactly the decode logits, K is read from HBM
 * once: one thread-block cluster per (b, KV group) streams K with tiled TMA into
 * tcgen05 (logits in TMEM), selects the top-k over DSMEM and attends
 * over [text rows] U [kept visual rows] (see fused.cu).  Results equal
 * svl_retrieve + svl_sparse_decode_attn up to fp32 rounding of the LSE.
 *
 * q        device bf16 [B][H][d] contiguous (the current token, post-RoPE).
 * flags    SVL_NORM_VISUAL_ONLY, SVL_FRESH_UNFUSED, SVL_PIN_SPLITS(8 or 16)
 *          (SVL_SELECT_SHARED -> UNSUPPORTED).
 * idx_out  device int32 [B][Hkv][k]: the kept visual indices (reusable by
 *          later svl_sparse_decode_attn steady steps).
 * out      device fp32 [B][H][d]; lse_out device fp32 [B][H] or NULL.
 * Shapes outside the fused kernel's on-chip budget (visual_len > 32768 with
 * g <= 8, > 16384 with 8 < g <= 16, or more than 4096 text rows), and batches
 * with more (b, KV group) units than co-resident clusters (the fused kernel
 * uses one 8- or 16-CTA cluster per unit; past one wave the two calls, which
 * spread over every SM, are faster), run the two separate calls instead (same
 * kernels as svl_retrieve / svl_sparse_decode_attn).  The workspace must be
 * sized by svl_fresh_decode_workspace_size, which covers either path.
 */
svl_status svl_fresh_decode_step(const void* q, int32_t B, int32_t H, int32_t Hkv, int32_t d,
                                 svl_kv K, svl_kv V, svl_span span, int32_t k, float scale,
                                 uint32_t flags, int32_t* idx_out, float* out, float* lse_out,
                                 void* workspace, size_t workspace_bytes, void* stream);

/* 1 if svl_fresh_decode_step runs the fused kernel for this shape and flags on the
 * current device (one launch per call), 0 if it runs the two separate calls
 * (host-only query; a K view that cannot be encoded as a TMA tensor map also
 * takes the two calls at run time). */
int32_t svl_fresh_decode_plan(int32_t B, int32_t H, int32_t Hkv, int32_t d, int32_t visual_len,
                              int32_t capacity, uint32_t flags);

size_t svl_fresh_decode_workspace_size(int32_t B, int32_t H, int32_t Hkv, int32_t d, int32_t k,
                                       int32_t visual_len, int32_t capacity, uint32_t flags);

/* -------------------- sequence split of one request */
/*
 * A (b, KV group) unit's visual span is split over P_s ranks (B = 1 on 8 GPUs:
 * 4 KV heads x 2 halves); each rank passes a K/V view of its shard (system text
 * on the first shard, later text on the last; SVL_SHARD_VIEW).  The fresh step
 * then needs three exchanges between the shards (the harness's collectives):
 *   1. svl_retrieve_partial_lse on the view -> local LSE [B][n_q][H];
 *      exchange; svl_lse_combine -> the full-prefix LSE;
 *   2. svl_retrieve(..., SVL_RETRIEVE_SELECT_ONLY | SVL_SHARD_VIEW, lse_in =
 *      that LSE, scores_out) -> the shard's relevance scores; exchange (the
 *      shards' scores side by side = the unit's scores); svl_topk -> the unit's
 *      kept rows (identical on every shard); svl_shard_indices -> this shard's;
 *   3. svl_sparse_decode_attn(view, SVL_IDX_PADDED) -> (out, lse) partial;
 *      exchange; svl_merge_partials -> out, lse.
 * paper_2510_17777_b200/seqpar.py drives the sequence (tests, bench).
 */
/* Natural-log LSE of scale * q . K_j over the view's normalisation domain (visual
 * rows, plus the view's text rows unless SVL_NORM_VISUAL_ONLY); leaves the
 * logits in the workspace for a following SVL_RETRIEVE_SELECT_ONLY call with
 * identical arguments.  n_q * g <= 32.  Workspace: svl_retrieve_workspace_size. */
svl_status svl_retrieve_partial_lse(const void* q, int32_t B, int32_t n_q, int32_t H, int32_t Hkv, int32_t d,
                                    svl_kv K, svl_span span, float scale, uint32_t flags, float* lse_out,
                                    void* workspace, size_t workspace_bytes, void* stream);
/* out[i] = M + log sum_p exp(parts[p][i] - M), p in rank order; device fp32. */
svl_status svl_lse_combine(const float* parts, int32_t P, int32_t n, float* out, void* stream);
/* Top-k of scores [units][n] per unit (ties -> lower index), ascending indices
 * [units][k]; the selection kernels of svl_retrieve.  Workspace: header. */
svl_status svl_topk(const float* scores, int32_t units, int32_t n, int32_t k, int32_t* idx_out, void* workspace,
                    size_t workspace_bytes, void* stream);
size_t svl_topk_workspace_size(int32_t units, int32_t n);
/* The entries of each unit's ascending idx [units][k] inside [lo, hi), minus
 * lo, then -1 padding: out [units][k] (SVL_IDX_PADDED vis_idx of the shard). */
svl_status svl_shard_indices(const int32_t* idx, int32_t units, int32_t k, int32_t lo, int32_t hi, int32_t* out,
                             void* stream);
/* out [rows][d], lse [rows] (nullable) from P partials out_parts [P][rows][d],
 * lse_parts [P][rows] (natural log), rank order: the a5 log-sum-exp merge. */
svl_status svl_merge_partials(const float* out_parts, const float* lse_parts, int32_t P, int32_t rows, int32_t d,
                              float* out, float* lse_out, void* stream);

/* ------------------------------------ page-summary retrieval (Quest-style) */
/*
 * svl_page_summary -- per-page key bounds for retrieval on page summaries
 * (north star "optionally on a page/chunk summary";
 * PAPER.md:527 Quest "estimates upper-bound attention scores for each page").
 * For each (b, G) and page p of `page` consecutive visual rows
 * [vb + p*page, vb + (p+1)*page):
 *   kmax[b][G][p][c] = max_j K[b,G,j,c],   kmin[b][G][p][c] = min_j K[b,G,j,c]
 * (bf16, exact).  visual_len % page == 0.  Built once per retained cache.
 * kmax, kmin  device bf16 [B][Hkv][visual_len/page][d] contiguous, caller-owned.
 * Workspace: SVL_WORKSPACE_HEADER_BYTES.
 */
svl_status svl_page_summary(svl_kv K, int32_t B, int32_t Hkv, int32_t d, svl_span span, int32_t page,
                            void* kmax, void* kmin, void* workspace, size_t workspace_bytes, void* stream);

/*
 * svl_retrieve_pages -- query-aware retrieval of whole pages from the page
 * summaries (reading A22).  For each unit (b, G):
 *   ub[r,h,p]  = scale * sum_c max(q[b,r,h,c] kmax[p][c], q[b,r,h,c] kmin[p][c])
 *                (an upper bound of every row logit of page p),
 *   score[p]   = sum_r sum_h softmax_p(ub[r,h,.])[p]   (softmax over the pages),
 *   the k_pages pages of largest score (ties -> lower page), ascending.
 * page = 1 reproduces svl_retrieve with SVL_NORM_VISUAL_ONLY.
 * q            device bf16 [B][n_q][H][d], n_q * H/Hkv <= 32.
 * kmax, kmin   svl_page_summary's output, n_pages = visual_len / page.
 * page_idx_out device int32 [B][Hkv][k_pages] ascending.
 * row_idx_out  nullable device int32 [B][Hkv][k_pages * page]: the kept pages' visual
 *              rows ascending, relative to vb -- svl_sparse_decode_attn's vis_idx
 *              with k = k_pages * page.
 * scores_out   nullable device fp32 [B][Hkv][n_pages].
 * flags        0.  Workspace: svl_retrieve_pages_workspace_size.
 */
svl_status svl_retrieve_pages(const void* q, int32_t B, int32_t n_q, int32_t H, int32_t Hkv, int32_t d,
                              const void* kmax, const void* kmin, int32_t n_pages, int32_t page, int32_t k_pages,
                              float scale, uint32_t flags, int32_t* page_idx_out, int32_t* row_idx_out,
                              float* scores_out, void* workspace, size_t workspace_bytes, void* stream);

size_t svl_retrieve_pages_workspace_size(int32_t B, int32_t n_q, int32_t H, int32_t Hkv, int32_t n_pages);

/* ----------------------------------------------------- prefill companion */
/*
 * svl_prefill_prune -- query-agnostic per-frame pruning (PAPER.md:113,
 * 199-200).  For each b and frame f = [o_f, o_{f+1}):
 * k_f = svl_keep_budget(N_f, prefill_sparsity); keep the k_f highest
 * saliency tokens (ties to the lower index); frames concatenated in order;
 * ascending global indices.  Bit-exact with the fp32 comparisons.
 *
 * saliency       device fp32 [B][N] (NaN ranks lowest, sets SVL_DEVFLAG_NONFINITE;
 *                -0.0 == +0.0).
 * frame_offsets  HOST int32 [n_frames+1], 0 = o_0 <= ... <= o_n = N, each
 *                frame <= 131072 tokens; NULL = one global frame (N <= 131072).
 * kept_idx       device int32 [B][kept_capacity].
 * kept_total     HOST out: sum_f k_f (computed synchronously on the host
 *                before launching; SVL_ERR_INVALID_ARGUMENT if > kept_capacity).
 */
svl_status svl_prefill_prune(const float* saliency, int32_t B, int32_t N,
                             const int32_t* frame_offsets, int32_t n_frames,
                             double prefill_sparsity, int32_t* kept_idx, int32_t kept_capacity,
                             int32_t* kept_total, void* workspace, size_t workspace_bytes,
                             void* stream);

size_t svl_prune_workspace_size(int32_t B, int32_t N, int32_t n_frames);

/*
 * svl_salience -- encoder-attention salience per visual token (PAPER.md:113,
 * 116 "streams softmax normalization and salience accumulation without
 * explicitly forming the full attention matrix").
 * Per frame f and encoder head h, P = softmax(scale * Q K^T) over all S+N_f
 * columns (never materialised; two streaming passes):
 *   SUMMARY        (S == 1): sal_j = mean_h P[0, S+j]
 *   MULTI_SUMMARY  (S >= 2): sal_j = mean_h (1/S) sum_{s<S} P[s, S+j]
 *   INTRA_VISUAL   (S == 0): sal_j = mean_h (1/N_f) sum_{i<N_f} P[i, j]
 * Qe, Ke   device bf16 [F][S+N_f][H_e][d_e] contiguous, d_e <= 128, d_e % 8 == 0.
 * saliency device fp32 [F][N_f].
 * Mode/summary-count mismatch -> SVL_ERR_INVALID_ARGUMENT.
 */
svl_status svl_salience(const void* Qe, const void* Ke, int32_t F, int32_t S, int32_t N_f,
                        int32_t H_e, int32_t d_e, int32_t mode, float scale, float* saliency,
                        void* workspace, size_t workspace_bytes, void* stream);

size_t svl_salience_workspace_size(int32_t F, int32_t S, int32_t N_f, int32_t H_e, int32_t d_e,
                                   int32_t mode);

/* --------------------------------------------------------------- helpers */
/* keep_budget(n, s) = max(1, floor(n*(1-s) + 0.5)) for n > 0, 0 for n == 0,
 * evaluated in IEEE double (reading A7); -1 if n < 0 or
 * s outside [0, 1). */
int64_t svl_keep_budget(int64_t n, double s);

/* Zero-fill a workspace (stream-ordered). */
svl_status svl_workspace_init(void* workspace, size_t workspace_bytes, void* stream);

const char* svl_status_string(svl_status s);

/* Thread-local description of the last non-OK status returned on this
 * thread (includes the cudaError_t name for SVL_ERR_CUDA). */
const char* svl_last_error_message(void);

/* Synchronises `stream` and reads the device flag word (debug/test only). */
svl_status svl_read_device_flags(void* workspace, void* stream, uint32_t* flags);
svl_status svl_reset_device_flags(void* workspace, void* stream);

/* Library build identifier ("sm_100a ..."). */
const char* svl_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SPARSEVILA_H_ */
