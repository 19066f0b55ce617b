// kernels.h -- internal launcher interface between the C-ABI host layer
// (api.cu) and the kernels.  Not part of the public ABI.
#pragma once

#include <cuda.h>  // CUtensorMap (encoded through the runtime's driver entry point)
#include <cuda_runtime.h>
#include <stdint.h>

namespace svl {

// ---------------------------------------------------------------- retrieve
struct ScoreParams {
    const uint16_t* q;  // [B][n_q][H][d]
    const uint16_t* K;  // KV view
    int64_t sb, sh, st;
    const int32_t* seq_len;
    int B, n_q, H, Hkv, g, NC, NCP;  // NC = n_q*g columns, NCP = padded (8*NT)
    int vb, nv, capacity;
    int C;               // chunks per unit
    int rows_per_chunk;  // visual rows per chunk (multiple of 16)
    int use_text;        // normalise over text rows too (FULL_PREFIX and no lse_in)
    int q_rows_in_view;  // n_q, or 0 for a shard view (SVL_SHARD_VIEW): seq_len >= vb + nv only
    int need_partials;   // 0 when lse_in supplies the normaliser
    float scale2;        // scale * log2(e)
    float* logits;       // [units][nv][NCP] base-2 logits
    float2* part;        // [units][C][NCP] chunk (max, sum) in base 2
    uint32_t* flags;
};

struct SelectParams {
    int mode;  // 0 = retrieve (logits + LSE), 1 = prune (float scores), 2 = retrieve from relevance scores,
               // 3 = as 2, one decode query's relevance (64 threshold candidates, 8192-row slices)
    // retrieve source
    const float* logits;
    const float2* part;
    const float* lse_in;  // natural log [B][n_q][H] or null
    int C, NC, NCP, g, n_q, H, Hkv, shared;
    // prune source
    const float* scores_in;
    int N, nf, kept_cap;  // prune: per b, frames f in [0, nf) of the row [b*N, b*N+N)
    // retrieve: uniform n = nv, k, out = u*k
    int nv, k;
    int32_t* idx_out;
    float* scores_out;  // retrieve only, nullable
    uint32_t* flags;
    int CS;  // cluster size (CTAs per selection unit)
};

// Prune frame table, passed by value as a kernel parameter (no host->device
// copy, no stream sync): fr[f] = (offset o_f, prefix sum of k over frames < f),
// f in [0, nf]; k_f = fr[f+1].y - fr[f].y.
constexpr int kMaxFrames = 2047;
struct PruneTable {
    int2 fr[kMaxFrames + 1];
};

constexpr int kMaxPeers = 8;  // GPUs of one NVLink/NVSwitch node

struct DecodeParams {
    const uint16_t* q;  // [B][H][d]
    const uint16_t* K;
    int64_t ksb, ksh, kst;
    const uint16_t* V;
    int64_t vsb, vsh, vst;
    const int32_t* seq_len;
    const int32_t* idx;  // [B][U][k]
    int B, H, Hkv, g, vb, nv, k, shared, capacity;
    int S;             // splits (CTAs) per unit; the grid (S x units) is co-resident
    int single_batch;  // every split has <= kDecodeRowsMax rows (host bound): one gather buffer
    int padded;        // SVL_IDX_PADDED: trailing -1 entries of vis_idx are skipped silently
    int cluster;       // 1: the S CTAs of a unit are one thread-block cluster, merged over DSMEM
    int static_vis;    // SVL_DECODE_STATIC_PREFIX: idx and rows < seq_len - 1 gathered before the PDL wait
    float scale2;  // scale * log2(e)
    float* out;    // [B][H][d]
    float* lse_out;
    uint32_t* flags;
    uint64_t* part;    // workspace: split partials [units * S][kDecodePartStride] (bits, tag) pairs (S > 1)
    uint32_t* sync;    // workspace header: word 3 = the push variant's departure counter (self-resetting)
    uint32_t* epochs;  // workspace header: per-unit call epochs [units] (tags of the partials)
    uint64_t* trace; // SVL_TRACE_BUILD only: per-CTA phase stamps [grid][16] (else null)
    // push variant (svl_sparse_decode_attn_push): P > 0 => the merged out tile is also
    // stored into every peer's gathered [B_total][H_total][d] buffer at (b0, h0), and
    // the last CTA raises peer_flags[r][rank] = epoch (release, system scope)
    int P, rank, b0, h0, B_total, H_total;
    uint32_t epoch;
    float* peer_out[kMaxPeers];
    uint32_t* peer_flags[kMaxPeers];
};
template <int D>
constexpr int kDecodePartStride = 16 * D + 32;  // o [16][D], M [16], l [16] (64-bit tagged fp32)
constexpr int kDecodeMaxSplits = 256;           // splits per unit (merge staging: S * slice <= g D + S)
int decode_ctas_per_sm(int d);                  // co-resident decode CTAs per SM
int decode_max_active_clusters(int d, int S);   // co-resident S-CTA decode clusters (<= 0: none)
cudaError_t launch_wait_flags(const uint32_t* flags, int P, uint32_t epoch, uint32_t* ws_flags, cudaStream_t s);

struct FreshParams {
    CUtensorMap ktmap;  // K as 4-D {d, capacity, Hkv, B}, box {64, 128, 1, 1}, 128-B swizzle
    const uint16_t* q;  // [B][H][d] -- retrieval query == decode query
    const uint16_t* K;
    int64_t ksb, ksh, kst;
    const uint16_t* V;
    int64_t vsb, vsh, vst;
    const int32_t* seq_len;
    int B, H, Hkv, g, vb, nv, k, capacity;
    int slice;          // visual rows per CTA of a unit's cluster
    uint32_t flags_in;  // SVL_NORM_VISUAL_ONLY
    float scale2;
    int32_t* idx_out;  // [B][Hkv][k]
    float* out;        // [B][H][d]
    float* lse_out;    // [B][H] or null
    uint32_t* flags;
    uint64_t* trace;   // debug: per-CTA phase timestamps (SVL_TRACE=1), else null
};
constexpr int kFusedThreads = 512;    // 8 stream-consumer warps + 1 TMA producer warp + 7 helper warps
constexpr int kFusedTextMax = 128;    // text rows per CTA
#ifndef SVL_SLICE_MAX
#define SVL_SLICE_MAX 2048
#endif
constexpr int kFusedSliceMax = SVL_SLICE_MAX;  // visual rows per CTA (halved for g > 8)
cudaError_t launch_fresh(const FreshParams& p, int d, int CS, cudaStream_t s);
int fresh_max_active_clusters(int d, int g, int CS);  // <= 0: unknown

struct SalienceParams {
    CUtensorMap qmap, kmap;  // tcgen05 path: Qe / Ke as 4-D {d_e, S+N_f, H_e, F}, box {64, 128}
    int use_tc;              // maps encoded (INTRA_VISUAL, S = 0, N_f <= 512)
    const uint16_t* Qe;
    const uint16_t* Ke;
    int F, S, Nf, He, de, mode;
    float scale2;
    float* lse;  // [F][He][rows] base-2 row LSE (pass 1)
    float* sal;  // [F][Nf]
    float* acc;  // [F][He][Nf] per-head column sums (pass 2) -- fp32
    uint32_t* flags;
};

// ------------------------------------------- retrieve, tensor-core path (n_q*g > 32)
constexpr int kRtMaxNQ = 4096;  // n_q * g query rows per unit (LSE2 table in shared memory)
struct RetrTcParams {
    CUtensorMap xmap, ymap;      // set by the launcher per pass (resident X tile, streamed Y stages)
    CUtensorMap qmap_x, qmap_y;  // Qpack as 4-D {d, NQP, 1, units}, boxes of 128 / 256 rows
    CUtensorMap kmap_x, kmap_y;  // K cache view {d, capacity, Hkv, B}, boxes of 128 / 256 rows
    CUtensorMap vmap;            // V cache view, boxes of 128 rows (svl_question_attention)
    const uint16_t* q;           // [B][n_q][H][d]
    uint16_t* qpack;             // [units][NQP][d] (workspace)
    const int32_t* seq_len;
    const float* lse_in;         // natural log [B][n_q][H] or null
    int B, n_q, H, Hkv, g, NQ, NQP, vb, nv, capacity;
    int visual_only;
    int chunk, nkc, npart;       // pass 0: keys per CTA, chunks per unit, partials per row (2 nkc)
    float scale2;
    float2* part;                // [units][NQP][npart] base-2 (max, sum)
    float* lse2;                 // [units][NQP] base-2 LSE (+inf on padding rows)
    float* scores;               // [units][nv] relevance
    uint32_t* flags;
    float* part_o;               // [units][NQP][nkc][d] partial outputs (svl_question_attention)
    float* out;                  // [B][n_q][H][d]
    float* lse_out;              // [B][n_q][H] natural log, or null
};
void plan_retrieve_tc(int units, int n_q, int g, int nv, int capacity, bool visual_only, int sms, int* chunk,
                      int* nkc);
cudaError_t launch_retrieve_tc(const RetrTcParams& p, int d, cudaStream_t s);
cudaError_t launch_question_attn_tc(const RetrTcParams& p, int d, cudaStream_t s);
// ------------------------------------------------------ pack-once
struct PackParams {
    const uint16_t* K;
    const uint16_t* V;
    int64_t ksb, ksh, kst, vsb, vsh, vst;
    uint16_t* Kp;
    uint16_t* Vp;
    int64_t pksb, pksh, pkst, pvsb, pvsh, pvst;
    const int32_t* seq_len;
    const int32_t* idx;  // [B][U][k]
    int B, Hkv, vb, nv, k, capacity, shared;
    uint32_t* flags;
};
cudaError_t launch_pack(const PackParams& p, int d, int max_rows, cudaStream_t s);
// ------------------------------------- page summaries
struct PageSumParams {
    const uint16_t* K;
    int64_t ksb, ksh, kst;
    int units, Hkv, d, vb, page, np;
    uint16_t* kmax;  // [units][np][d]
    uint16_t* kmin;
};
struct PageRetrParams {
    const uint16_t* q;  // [B][n_q][H][d]
    const uint16_t* kmax;
    const uint16_t* kmin;
    int units, n_q, H, Hkv, g, NC, d, np;
    float scale2;
    float* ub2;     // [units][NC][np] base-2 page bounds (workspace)
    float* scores;  // [units][np]
};
cudaError_t launch_page_summary(const PageSumParams& p, cudaStream_t s);
// --------------------------------- sequence-split exchanges
cudaError_t launch_lse_from_partials(const float2* part, int units, int C, int NCP, int NC, int g, int n_q, int H,
                                     int Hkv, float* lse_out, cudaStream_t s);
cudaError_t launch_lse_combine(const float* parts, int P, int n, float* out, cudaStream_t s);
cudaError_t launch_shard_indices(const int32_t* idx, int units, int k, int lo, int hi, int32_t* out, cudaStream_t s);
cudaError_t launch_merge_partials(const float* out_parts, const float* lse_parts, int P, int rows, int d, float* out,
                                  float* lse_out, cudaStream_t s);
cudaError_t launch_page_scores(const PageRetrParams& p, cudaStream_t s);
cudaError_t launch_page_expand(const int32_t* pidx, int units, int kp, int page, int32_t* rows, cudaStream_t s);
// -------------------------------------------- RoPE remap
struct RopeParams {
    const uint16_t* K;  // pre-RoPE keys
    int64_t ksb, ksh, kst;
    const uint16_t* V;  // nullable
    int64_t vsb, vsh, vst;
    uint16_t* Ko;
    int64_t osb, osh, ost;
    uint16_t* Vo;
    int64_t vosb, vosh, vost;
    const int32_t* seq_len;
    const int32_t* kept;  // [B][k]
    int B, Hkv, d, vb, nv, k, capacity;
    double log2_base;
    uint32_t* flags;
};
cudaError_t launch_rope_remap(const RopeParams& p, int max_rows, cudaStream_t s);
struct MropeParams {
    const uint16_t* K;  // pre-RoPE keys
    int64_t ksb, ksh, kst;
    const uint16_t* V;  // nullable
    int64_t vsb, vsh, vst;
    uint16_t* Ko;
    int64_t osb, osh, ost;
    uint16_t* Vo;
    int64_t vosb, vosh, vost;
    const int32_t* seq_len;
    const int32_t* kept;    // [B][k]
    const int32_t* coords;  // [B][nv][3] (t, h, w) of the original visual rows
    int B, Hkv, d, vb, nv, k, capacity;
    int sec0, sec1;         // rotary pairs of the t and h sections (w: the rest of d/2)
    double log2_base;
    int32_t* new_coords;    // [B][k][3]
    int32_t* dim_max;       // [B][3] workspace
    int32_t* text_start_out;  // nullable [B]
    uint32_t* flags;
};
cudaError_t launch_mrope_remap(const MropeParams& p, int max_rows, cudaStream_t s);
constexpr int kScoreThreads = 512;
constexpr int kSelectThreads = 512;
constexpr int kSelectMaxPerThread = 16;  // => <= 8192 keys per CTA
constexpr int kDecodeThreads = 256;  // 8 warps x one 16-row tile per batch
constexpr int kDecodeRowsMax = 128;  // rows per gather batch

cudaError_t launch_score(const ScoreParams& p, int d, int NT, cudaStream_t s);
cudaError_t launch_select(const SelectParams& p, int n_units, cudaStream_t s);
// relevance scores [units][nv] from the retrieve logits (mode-0 arithmetic), for a mode-2 select
cudaError_t launch_relevance(const SelectParams& p, float* scores, int units, cudaStream_t s);
int relevance_select_cs(int nv);  // cluster size of the mode-3 select (slices <= 8192 rows)
cudaError_t launch_prune_select(const SelectParams& p, const PruneTable& tab, int n_units, cudaStream_t s);
cudaError_t launch_decode(const DecodeParams& p, int d, cudaStream_t s);
cudaError_t launch_salience(const SalienceParams& p, cudaStream_t s);
bool salience_tc_eligible(const SalienceParams& p);
cudaError_t launch_salience_tc(const SalienceParams& p, cudaStream_t s);

int device_sm_count();

// All kernels request the maximum shared-memory carveout so that consecutive
// launches in a graph never force an L1/shared reconfiguration of the SMs.
template <typename K>
inline cudaError_t set_max_carveout(K kern) {
    return cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}
int select_cluster_size(int n);  // CTAs per selection unit for n keys

// K (or V) cache view as a 4-D TMA tensor map {d, capacity, Hkv, B} (strides in
// elements), box {64, box_rows, 1, 1}, 128-byte swizzle.  False if the driver
// entry point is missing or the view is not encodable (the caller falls back).
bool encode_kv_tensor_map(CUtensorMap* map, const void* data, int d, int capacity, int Hkv, int B,
                          int64_t stride_b, int64_t stride_h, int64_t stride_t, int box_rows);

}  // namespace svl
