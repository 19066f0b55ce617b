// api.cu -- C-ABI host layer of libsparsevila.so (include/sparsevila.h).
//
// Host-side validation (synchronous; nothing launches on error), workspace
// sizing and carving, launch heuristics (chunks / splits / cluster size from
// the device's SM count), error strings.  No allocation, no synchronisation.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "../../include/sparsevila.h"
#include "common.cuh"
#include "kernels.h"

namespace svl {

static thread_local char g_err[512] = "";

static svl_status fail(svl_status s, const char* fmt, const char* a = nullptr) {
    snprintf(g_err, sizeof g_err, fmt, a ? a : "");
    return s;
}

static svl_status cuda_fail(cudaError_t e, const char* where) {
    snprintf(g_err, sizeof g_err, "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
    return SVL_ERR_CUDA;
}

struct DevAttr {
    int sms = 0, major = 0, minor = 0;
};

static DevAttr dev_attr() {
    static DevAttr cache[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return DevAttr{};
    if (cache[dev].sms == 0) {
        DevAttr a;
        cudaDeviceGetAttribute(&a.sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&a.major, cudaDevAttrComputeCapabilityMajor, dev);
        cudaDeviceGetAttribute(&a.minor, cudaDevAttrComputeCapabilityMinor, dev);
        cache[dev] = a;
    }
    return cache[dev];
}

int device_sm_count() {
    const int s = dev_attr().sms;
    return s > 0 ? s : 148;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
static size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ------------------------------------------------------------------ retrieve
struct ScorePlan {
    int NT, NCP, C, rows_per_chunk;
};

// Chunks per unit: minimise the critical path ceil(units*C/SMs) * ceil(nv/C)
// (persistent grid of SM-count CTAs), chunks of >= 64 rows.
static ScorePlan plan_score(int units, int n_q, int g, int nv, int sms) {
    ScorePlan pl;
    pl.NT = (n_q * g + 7) / 8;
    pl.NCP = pl.NT * 8;
    long best = -1;
    int bestC = 1;
    const int cmax = std::max(1, std::min(4096, (nv + 63) / 64));
    for (int C = 1; C <= cmax; ++C) {
        const long rpc = ((nv + C - 1) / C + 15) / 16 * 16;
        const int Ceff = (int)((nv + rpc - 1) / rpc);
        if (Ceff != C) continue;
        const long waves = ((long)units * C + sms - 1) / sms;
        const long cost = waves * (rpc + 48);  // + per-item overhead in row units
        if (best < 0 || cost < best) {
            best = cost;
            bestC = C;
        }
    }
    pl.C = bestC;
    pl.rows_per_chunk = ((nv + bestC - 1) / bestC + 15) / 16 * 16;
    return pl;
}

struct RetrieveLayout {
    size_t logits, part, scores, total;
};

static RetrieveLayout retrieve_layout(int B, int Hkv, int nv, const ScorePlan& pl) {
    RetrieveLayout l;
    const size_t units = (size_t)B * Hkv;
    l.logits = kWsHeader;
    l.part = round_up(l.logits + units * nv * pl.NCP * sizeof(float), 256);
    l.scores = round_up(l.part + units * pl.C * pl.NCP * sizeof(float2), 256);  // relevance [units][nv]
    l.total = round_up(l.scores + units * nv * sizeof(float), 256);
    return l;
}

// tensor-core path (n_q * g > 32): Qpack, LSE partials, LSE2, scores
struct RetrieveTcLayout {
    size_t qpack, part, lse2, scores, total;
    int NQ, NQP, chunk, nkc;
};

static RetrieveTcLayout retrieve_tc_layout(int B, int n_q, int H, int Hkv, int d, int nv, int capacity,
                                           bool visual_only) {
    RetrieveTcLayout l;
    const size_t units = (size_t)B * Hkv;
    const int g = H / Hkv;
    l.NQ = n_q * g;
    l.NQP = (l.NQ + 255) / 256 * 256;
    plan_retrieve_tc((int)units, n_q, g, nv, capacity, visual_only, device_sm_count(), &l.chunk, &l.nkc);
    l.qpack = kWsHeader;
    l.part = round_up(l.qpack + units * l.NQP * d * 2, 256);
    l.lse2 = round_up(l.part + units * l.NQP * 4 * l.nkc * sizeof(float2), 256);
    l.scores = round_up(l.lse2 + units * l.NQP * sizeof(float), 256);
    l.total = round_up(l.scores + units * nv * sizeof(float), 256);
    return l;
}

// --------------------------------------------------------------- decode plan
// Splits per unit.  The grid (units x S CTAs) never exceeds the co-resident CTA
// count (the split merge is a grid-wide barrier), so S = floor(SMs * occ / units)
// for occ in {1, 2} CTAs per SM, at least kDecodeMinRows attended rows per CTA;
// of the two the one with the smaller per-SM row load (ties: more CTAs); see plan_decode for
// the merge path (cluster over DSMEM or co-resident grid over L2).
constexpr int kDecodeMinRows = 32;
#ifndef SVL_DECODE_OCC
#define SVL_DECODE_OCC 2  // (the kernel's shared memory allows one CTA per SM today)
#endif
static int decode_slots(int d) { return device_sm_count() * std::max(1, decode_ctas_per_sm(d)); }

// Split count S and merge path of the steady decode.  S <= 16 splits may run as one
// S-CTA cluster per unit merging over DSMEM, but only while every unit's cluster is
// co-resident: clusters that do not fit run as a second wave (measured long-video, us/layer:
// B = 3 as 12-CTA clusters 19.5 vs grid merge 13.5; B = 4 as 8-CTA clusters 22.5 vs grid
// merge at S = 9 15.0).  Past the co-resident cluster count the same S merges through L2.
struct DecodePlan {
    int S;
    int cluster;
};

static DecodePlan plan_decode(int units, int n_att_max, int d, uint32_t flags) {
    const bool grid_only = (flags & SVL_DECODE_GRID_MERGE) != 0;
    if (const int pin = (int)(flags >> 24)) return {pin, (pin > 1 && pin <= 16 && !grid_only) ? 1 : 0};
    const int sms = device_sm_count();
    const int occ_max = std::min(SVL_DECODE_OCC, std::max(1, decode_ctas_per_sm(d)));
    const int smax = std::max(1, n_att_max / kDecodeMinRows);
    int bestS = 1;
    long best = -1;
    for (int occ = 1; occ <= occ_max; ++occ) {
        const int S = std::max(1, std::min(smax, sms * occ / std::max(units, 1)));
        if (S > 1 && (long)units * S > (long)sms * occ) continue;
        const long ctas = (long)units * S;
        const long rows = (n_att_max + S - 1) / S;
        const long cost = ((ctas + sms - 1) / sms) * rows;
        if (best < 0 || cost < best || (cost == best && S > bestS)) {
            best = cost;
            bestS = S;
        }
    }
    if (bestS <= 1) return {1, 0};
    if (grid_only) return {bestS, 0};
    // few units: one 16-CTA cluster per unit merging over DSMEM beats spreading the unit over
    // more SMs with the L2 merge while the clusters are co-resident (measured, us/layer:
    // long-video 9.65 vs 10.37 at S = 37, nvila-4k 7.32 vs 8.69)
    if (bestS > 16) return units <= decode_max_active_clusters(d, 16) ? DecodePlan{16, 1} : DecodePlan{bestS, 0};
    if (units <= decode_max_active_clusters(d, bestS)) return {bestS, 1};
    // a slightly narrower cluster that fits in one wave still beats the L2 merge (B = 3:
    // 8-CTA clusters 12.0 vs grid merge at S = 12 13.5)
    for (int S2 = bestS - 1; 3 * S2 >= 2 * bestS && S2 > 1; --S2)
        if (units <= decode_max_active_clusters(d, S2)) return {S2, 1};
    return {bestS, 0};
}

static size_t decode_ws_bytes(int units, int S, int d) {
    if (S <= 1) return kWsHeader;
    const size_t stride = (d == 128) ? kDecodePartStride<128> : kDecodePartStride<64>;
    return kWsHeader + (size_t)units * S * stride * sizeof(uint64_t);
}

}  // namespace svl

using namespace svl;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static const EncodeTiledFn fn = []() -> EncodeTiledFn {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        return reinterpret_cast<EncodeTiledFn>(f);
    }();
    return fn;
}

namespace svl {
bool encode_kv_tensor_map(CUtensorMap* map, const void* data, int d, int capacity, int Hkv, int B,
                          int64_t stride_b, int64_t stride_h, int64_t stride_t, int box_rows) {
    const EncodeTiledFn fn = encode_fn();
    if (!fn || d % 8 || stride_t <= 0 || stride_h <= 0 || stride_b <= 0) return false;  // box cols past d zero-fill
    const cuuint64_t dims[4] = {(cuuint64_t)d, (cuuint64_t)capacity, (cuuint64_t)Hkv, (cuuint64_t)B};
    const cuuint64_t strides[3] = {(cuuint64_t)stride_t * 2, (cuuint64_t)stride_h * 2, (cuuint64_t)stride_b * 2};
    const cuuint32_t box[4] = {64, (cuuint32_t)box_rows, 1, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(data), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace svl

extern "C" {

const char* svl_version(void) {
    return "libsparsevila 0.5 sm_100a (fused fresh step: TMA + tcgen05 K stream, cluster top-k over DSMEM, split "
           "decode / selection warp groups after the threshold bin; "
           "steady decode: split-K gather (optionally started before the PDL wait), co-resident cluster DSMEM "
           "merge or epoch-tagged L2 merge; "
           "question chunk: tcgen05 row LSE, column mass and attention output (P from TMEM))";
}

const char* svl_status_string(svl_status s) {
    switch (s) {
        case SVL_OK: return "SVL_OK";
        case SVL_ERR_INVALID_ARGUMENT: return "SVL_ERR_INVALID_ARGUMENT";
        case SVL_ERR_SHAPE: return "SVL_ERR_SHAPE";
        case SVL_ERR_ALIGNMENT: return "SVL_ERR_ALIGNMENT";
        case SVL_ERR_WORKSPACE: return "SVL_ERR_WORKSPACE";
        case SVL_ERR_UNSUPPORTED: return "SVL_ERR_UNSUPPORTED";
        case SVL_ERR_CUDA: return "SVL_ERR_CUDA";
    }
    return "SVL_ERR_UNKNOWN";
}

const char* svl_last_error_message(void) { return g_err; }

int64_t svl_keep_budget(int64_t n, double s) {
    if (n < 0 || !(s >= 0.0 && s < 1.0)) return -1;
    if (n == 0) return 0;
    int64_t k = (int64_t)floor((double)n * (1.0 - s) + 0.5);
    if (k < 1) k = 1;
    if (k > n) k = n;
    return k;
}

svl_status svl_workspace_init(void* ws, size_t bytes, void* stream) {
    if (!ws) return fail(SVL_ERR_WORKSPACE, "workspace is NULL");
    cudaError_t e = cudaMemsetAsync(ws, 0, bytes, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "svl_workspace_init");
    return SVL_OK;
}

svl_status svl_read_device_flags(void* ws, void* stream, uint32_t* flags) {
    if (!ws || !flags) return fail(SVL_ERR_INVALID_ARGUMENT, "NULL argument");
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e == cudaSuccess) e = cudaMemcpy(flags, ws, sizeof(uint32_t), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "svl_read_device_flags");
    return SVL_OK;
}

svl_status svl_reset_device_flags(void* ws, void* stream) {
    if (!ws) return fail(SVL_ERR_INVALID_ARGUMENT, "NULL workspace");
    cudaError_t e = cudaMemsetAsync(ws, 0, sizeof(uint32_t), (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "svl_reset_device_flags");
    return SVL_OK;
}

static svl_status check_device() {
    DevAttr a = dev_attr();
    if (a.major != 10 || a.minor != 0)
        return fail(SVL_ERR_UNSUPPORTED, "libsparsevila needs an sm_100 (B200) device%s");
    return SVL_OK;
}

static svl_status check_kv(const svl_kv& kv, int B, int Hkv, int d, const char* name) {
    if (!kv.data) return fail(SVL_ERR_INVALID_ARGUMENT, "%s.data is NULL", name);
    if (!aligned16(kv.data)) return fail(SVL_ERR_ALIGNMENT, "%s.data not 16-byte aligned", name);
    if ((kv.stride_t * 2) % 16 || (kv.stride_h * 2) % 16 || (kv.stride_b * 2) % 16)
        return fail(SVL_ERR_ALIGNMENT, "%s strides must be multiples of 8 elements", name);
    if (kv.stride_t < d || kv.capacity < 1)
        return fail(SVL_ERR_SHAPE, "%s stride_t < d or capacity < 1", name);
    if (kv.stride_h < 0 || kv.stride_b < 0) return fail(SVL_ERR_SHAPE, "%s has a negative stride", name);
    (void)B;
    (void)Hkv;
    return SVL_OK;
}

// svl_retrieve, n_q * g > 32: qpack -> [row LSE pass] -> LSE2 -> column-mass pass -> cluster top-k
static svl_status retrieve_tc(const void* q, int B, int n_q, int H, int Hkv, int d, const svl_kv& K,
                              const svl_span& span, const float* lse_in, int k, float scale, uint32_t flags,
                              int32_t* idx_out, float* scores_out, void* ws, size_t ws_bytes, cudaStream_t s) {
    const int units = B * Hkv, g = H / Hkv;
    const bool vis_only = (flags & SVL_NORM_VISUAL_ONLY) != 0;
    const int shared = (flags & SVL_SELECT_SHARED) ? 1 : 0;
    RetrieveTcLayout lay = retrieve_tc_layout(B, n_q, H, Hkv, d, span.visual_len, K.capacity, vis_only);
    if (ws_bytes < lay.total) return fail(SVL_ERR_WORKSPACE, "workspace too small%s");
    uint8_t* w = static_cast<uint8_t*>(ws);
    RetrTcParams p;
    memset(&p, 0, sizeof(p));
    const int64_t qstride = (int64_t)lay.NQP * d;
    if (!encode_kv_tensor_map(&p.qmap_x, w + lay.qpack, d, lay.NQP, 1, units, qstride, qstride, d, 128) ||
        !encode_kv_tensor_map(&p.qmap_y, w + lay.qpack, d, lay.NQP, 1, units, qstride, qstride, d, 256) ||
        !encode_kv_tensor_map(&p.kmap_x, K.data, d, K.capacity, Hkv, B, K.stride_b, K.stride_h, K.stride_t, 128) ||
        !encode_kv_tensor_map(&p.kmap_y, K.data, d, K.capacity, Hkv, B, K.stride_b, K.stride_h, K.stride_t, 256))
        return fail(SVL_ERR_UNSUPPORTED, "tensor-core retrieve: K view not encodable as a TMA tensor map%s");
    p.q = static_cast<const uint16_t*>(q);
    p.qpack = reinterpret_cast<uint16_t*>(w + lay.qpack);
    p.seq_len = span.seq_len;
    p.lse_in = lse_in;
    p.B = B; p.n_q = n_q; p.H = H; p.Hkv = Hkv; p.g = g; p.NQ = lay.NQ; p.NQP = lay.NQP;
    p.vb = span.visual_begin; p.nv = span.visual_len; p.capacity = K.capacity;
    p.visual_only = vis_only ? 1 : 0;
    p.chunk = lay.chunk; p.nkc = lay.nkc; p.npart = 4 * lay.nkc;
    p.scale2 = scale * kLog2e;
    p.part = reinterpret_cast<float2*>(w + lay.part);
    p.lse2 = reinterpret_cast<float*>(w + lay.lse2);
    p.scores = (scores_out && !shared) ? scores_out : reinterpret_cast<float*>(w + lay.scores);
    p.flags = reinterpret_cast<uint32_t*>(w);
    cudaError_t e = cudaSuccess;
    if (!(flags & SVL_RETRIEVE_SELECT_ONLY)) {
        e = launch_retrieve_tc(p, d, s);
        if (e != cudaSuccess) return cuda_fail(e, "svl_retrieve/tensor-core scores");
    }
    if (flags & SVL_RETRIEVE_SCORE_ONLY) return SVL_OK;
    SelectParams se = {};
    se.mode = 2;
    se.scores_in = p.scores;
    se.Hkv = Hkv;
    se.shared = shared;
    se.nv = span.visual_len; se.k = k;
    se.idx_out = idx_out;
    se.scores_out = shared ? scores_out : nullptr;
    se.flags = p.flags;
    se.CS = select_cluster_size(span.visual_len);
    e = launch_select(se, shared ? B : units, s);
    if (e != cudaSuccess) return cuda_fail(e, "svl_retrieve/select");
    return SVL_OK;
}

size_t svl_retrieve_workspace_size(int32_t B, int32_t n_q, int32_t H, int32_t Hkv, int32_t d,
                                   int32_t visual_len, uint32_t flags) {
    if (B < 1 || n_q < 1 || Hkv < 1 || H % Hkv || visual_len < 1) return 0;
    const int g = H / Hkv;
    if (n_q * g > 32)  // tensor-core path (the layout does not depend on the capacity)
        return retrieve_tc_layout(B, n_q, H, Hkv, d, visual_len, visual_len, (flags & SVL_NORM_VISUAL_ONLY) != 0)
            .total;
    ScorePlan pl = plan_score(B * Hkv, n_q, g, visual_len, device_sm_count());
    return retrieve_layout(B, Hkv, visual_len, pl).total;
}

// ------------------------------------- question-chunk attention
static size_t question_attn_part_off(const RetrieveTcLayout& l) { return l.total; }
static size_t question_attn_total(const RetrieveTcLayout& l, int units, int d) {
    return round_up(l.total + (size_t)units * l.NQP * l.nkc * d * sizeof(float), 256);
}

size_t svl_question_attention_workspace_size(int32_t B, int32_t n_q, int32_t H, int32_t Hkv, int32_t d,
                                             int32_t visual_len, uint32_t flags) {
    if (B < 1 || n_q < 1 || Hkv < 1 || H % Hkv || visual_len < 1 || (d != 64 && d != 128)) return 0;
    const RetrieveTcLayout l =
        retrieve_tc_layout(B, n_q, H, Hkv, d, visual_len, visual_len, (flags & SVL_NORM_VISUAL_ONLY) != 0);
    return question_attn_total(l, B * Hkv, d);
}

svl_status svl_question_attention(const void* q, int32_t B, int32_t n_q, int32_t H, int32_t Hkv, int32_t d,
                                  svl_kv K, svl_kv V, svl_span span, const float* lse_in, float scale,
                                  uint32_t flags, float* out, float* lse_out, void* ws, size_t ws_bytes,
                                  void* stream) {
    if (!q || !out || !span.seq_len) return fail(SVL_ERR_INVALID_ARGUMENT, "NULL pointer argument%s");
    if (flags & ~SVL_NORM_VISUAL_ONLY) return fail(SVL_ERR_INVALID_ARGUMENT, "unknown flag bits%s");
    if (B < 1 || n_q < 1 || H < 1 || Hkv < 1) return fail(SVL_ERR_SHAPE, "B, n_q, H, Hkv must be >= 1%s");
    if (H % Hkv) return fail(SVL_ERR_SHAPE, "H %% Hkv != 0%s");
    if (span.visual_len < 1) return fail(SVL_ERR_SHAPE, "no visual rows%s");
    if (span.visual_begin < 0 || (int64_t)span.visual_begin + span.visual_len + n_q > (int64_t)K.capacity ||
        K.capacity != V.capacity)
        return fail(SVL_ERR_SHAPE, "visual span + query rows outside the KV capacity (or K/V capacities differ)%s");
    if (!(scale > 0.f) || !isfinite(scale)) return fail(SVL_ERR_INVALID_ARGUMENT, "scale must be finite > 0%s");
    if (d != 64 && d != 128) return fail(SVL_ERR_UNSUPPORTED, "head dim must be 64 or 128%s");
    const int g = H / Hkv;
    if (n_q * g > kRtMaxNQ) return fail(SVL_ERR_UNSUPPORTED, "n_q * g must be <= 4096%s");
    if (!aligned16(q) || !aligned16(out)) return fail(SVL_ERR_ALIGNMENT, "q / out not 16-byte aligned%s");
    svl_status st = check_kv(K, B, Hkv, d, "K");
    if (st != SVL_OK) return st;
    st = check_kv(V, B, Hkv, d, "V");
    if (st != SVL_OK) return st;
    if (!ws || !aligned16(ws)) return fail(SVL_ERR_WORKSPACE, "workspace NULL or misaligned%s");
    st = check_device();
    if (st != SVL_OK) return st;
    const int units = B * Hkv;
    const bool vis_only = (flags & SVL_NORM_VISUAL_ONLY) != 0;
    RetrieveTcLayout lay = retrieve_tc_layout(B, n_q, H, Hkv, d, span.visual_len, K.capacity, vis_only);
    if (ws_bytes < question_attn_total(lay, units, d)) return fail(SVL_ERR_WORKSPACE, "workspace too small%s");
    uint8_t* w = static_cast<uint8_t*>(ws);
    RetrTcParams p;
    memset(&p, 0, sizeof(p));
    const int64_t qstride = (int64_t)lay.NQP * d;
    if (!encode_kv_tensor_map(&p.qmap_x, w + lay.qpack, d, lay.NQP, 1, units, qstride, qstride, d, 128) ||
        !encode_kv_tensor_map(&p.kmap_x, K.data, d, K.capacity, Hkv, B, K.stride_b, K.stride_h, K.stride_t, 128) ||
        !encode_kv_tensor_map(&p.kmap_y, K.data, d, K.capacity, Hkv, B, K.stride_b, K.stride_h, K.stride_t, 256) ||
        !encode_kv_tensor_map(&p.vmap, V.data, d, V.capacity, Hkv, B, V.stride_b, V.stride_h, V.stride_t, 128))
        return fail(SVL_ERR_UNSUPPORTED, "question attention: K / V view not encodable as a TMA tensor map%s");
    p.q = static_cast<const uint16_t*>(q);
    p.qpack = reinterpret_cast<uint16_t*>(w + lay.qpack);
    p.seq_len = span.seq_len;
    p.lse_in = lse_in;
    p.B = B; p.n_q = n_q; p.H = H; p.Hkv = Hkv; p.g = g; p.NQ = lay.NQ; p.NQP = lay.NQP;
    p.vb = span.visual_begin; p.nv = span.visual_len; p.capacity = K.capacity;
    p.visual_only = vis_only ? 1 : 0;
    p.chunk = lay.chunk; p.nkc = lay.nkc; p.npart = 4 * lay.nkc;
    p.scale2 = scale * kLog2e;
    p.part = reinterpret_cast<float2*>(w + lay.part);
    p.lse2 = reinterpret_cast<float*>(w + lay.lse2);
    p.flags = reinterpret_cast<uint32_t*>(w);
    p.part_o = reinterpret_cast<float*>(w + question_attn_part_off(lay));
    p.out = out;
    p.lse_out = lse_out;
    const cudaError_t e = launch_question_attn_tc(p, d, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "svl_question_attention");
    return SVL_OK;
}

svl_status svl_retrieve(const void* q, int32_t B, int32_t n_q, int32_t H, int32_t Hkv, int32_t d,
                        svl_kv K, svl_span span, const float* lse_in, int32_t k, float scale,
                        uint32_t flags, int32_t* idx_out, float* scores_out, void* ws,
                        size_t ws_bytes, void* stream) {
    if (!q || (!idx_out && k > 0) || !span.seq_len)
        return fail(SVL_ERR_INVALID_ARGUMENT, "NULL pointer argument%s");
    if (flags & ~(SVL_NORM_VISUAL_ONLY | SVL_SELECT_SHARED | SVL_RETRIEVE_SCORE_ONLY |
                  SVL_RETRIEVE_SELECT_ONLY | SVL_SHARD_VIEW))
        return fail(SVL_ERR_INVALID_ARGUMENT, "unknown flag bits%s");
    if ((flags & SVL_RETRIEVE_SCORE_ONLY) && (flags & SVL_RETRIEVE_SELECT_ONLY))
        return fail(SVL_ERR_INVALID_ARGUMENT, "SCORE_ONLY and SELECT_ONLY are exclusive%s");
    if (B < 1 || n_q < 1 || H < 1 || Hkv < 1) return fail(SVL_ERR_SHAPE, "B, n_q, H, Hkv must be >= 1%s");
    if (H % Hkv) return fail(SVL_ERR_SHAPE, "H %% Hkv != 0%s");
    if (span.visual_len < 1) return fail(SVL_ERR_SHAPE, "no visual rows to retrieve from%s");
    const int q_rows = (flags & SVL_SHARD_VIEW) ? 0 : n_q;  // a shard view need not hold the query rows
    if (span.visual_begin < 0 ||
        (int64_t)span.visual_begin + span.visual_len + q_rows > (int64_t)K.capacity)
        return fail(SVL_ERR_SHAPE, "visual span + query rows outside the KV capacity%s");
    if (k < 0 || k > span.visual_len) return fail(SVL_ERR_INVALID_ARGUMENT, "k outside [0, visual_len]%s");
    if (!(scale > 0.f) || !isfinite(scale)) return fail(SVL_ERR_INVALID_ARGUMENT, "scale must be finite > 0%s");
    if (d != 64 && d != 128) return fail(SVL_ERR_UNSUPPORTED, "head dim must be 64 or 128%s");
    const int g = H / Hkv;
    const bool tc = n_q * g > 32;  // question chunk: tensor-core path (retrieve_tc.cu)
    if (tc && n_q * g > kRtMaxNQ) return fail(SVL_ERR_UNSUPPORTED, "n_q * g must be <= 4096%s");
    const int shared = (flags & SVL_SELECT_SHARED) ? 1 : 0;
    if (!tc && shared && n_q * g * Hkv > 128) return fail(SVL_ERR_UNSUPPORTED, "SHARED needs n_q*H <= 128%s");
    if (span.visual_len > 16 * kSelectThreads * kSelectMaxPerThread)
        return fail(SVL_ERR_UNSUPPORTED, "visual_len > 131072%s");
    if (!aligned16(q)) return fail(SVL_ERR_ALIGNMENT, "q not 16-byte aligned%s");
    svl_status st = check_kv(K, B, Hkv, d, "K");
    if (st != SVL_OK) return st;
    if (!ws || !aligned16(ws)) return fail(SVL_ERR_WORKSPACE, "workspace NULL or misaligned%s");
    st = check_device();
    if (st != SVL_OK) return st;

    const int units = B * Hkv;
    if (tc && (flags & SVL_SHARD_VIEW)) return fail(SVL_ERR_UNSUPPORTED, "SVL_SHARD_VIEW needs n_q * g <= 32%s");
    if (tc) return retrieve_tc(q, B, n_q, H, Hkv, d, K, span, lse_in, k, scale, flags, idx_out, scores_out,
                               ws, ws_bytes, (cudaStream_t)stream);
    ScorePlan pl = plan_score(units, n_q, g, span.visual_len, device_sm_count());
    RetrieveLayout lay = retrieve_layout(B, Hkv, span.visual_len, pl);
    if (ws_bytes < lay.total) return fail(SVL_ERR_WORKSPACE, "workspace too small%s");
    uint8_t* w = static_cast<uint8_t*>(ws);
    cudaStream_t s = (cudaStream_t)stream;

    ScoreParams sp;
    sp.q = static_cast<const uint16_t*>(q);
    sp.K = static_cast<const uint16_t*>(K.data);
    sp.sb = K.stride_b; sp.sh = K.stride_h; sp.st = K.stride_t;
    sp.seq_len = span.seq_len;
    sp.B = B; sp.n_q = n_q; sp.H = H; sp.Hkv = Hkv; sp.g = g;
    sp.NC = n_q * g; sp.NCP = pl.NCP;
    sp.vb = span.visual_begin; sp.nv = span.visual_len; sp.capacity = K.capacity;
    sp.C = pl.C; sp.rows_per_chunk = pl.rows_per_chunk;
    sp.need_partials = lse_in ? 0 : 1;
    sp.use_text = (!lse_in && !(flags & SVL_NORM_VISUAL_ONLY)) ? 1 : 0;
    sp.q_rows_in_view = (flags & SVL_SHARD_VIEW) ? 0 : n_q;
    sp.scale2 = scale * kLog2e;
    sp.logits = reinterpret_cast<float*>(w + lay.logits);
    sp.part = reinterpret_cast<float2*>(w + lay.part);
    sp.flags = reinterpret_cast<uint32_t*>(w);
    cudaError_t e = cudaSuccess;
    if (!(flags & SVL_RETRIEVE_SELECT_ONLY)) {
        e = launch_score(sp, d, pl.NT, s);
        if (e != cudaSuccess) return cuda_fail(e, "svl_retrieve/score");
    }
    if (flags & SVL_RETRIEVE_SCORE_ONLY) return SVL_OK;

    SelectParams se = {};
    se.mode = 0;
    se.logits = sp.logits;
    se.part = sp.part;
    se.lse_in = lse_in;
    se.C = pl.C; se.NC = sp.NC; se.NCP = pl.NCP; se.g = g; se.n_q = n_q; se.H = H; se.Hkv = Hkv;
    se.shared = shared;
    se.nv = span.visual_len; se.k = k;
    se.idx_out = idx_out;
    se.scores_out = scores_out;
    se.flags = sp.flags;
    se.CS = select_cluster_size(span.visual_len);
    // Past one wave of selection clusters (units x CS > 2 CTAs per SM), the relevance runs as
    // its own streaming pass (full occupancy) and the top-k over 4 B per row in few, larger
    // clusters (8192-row slices), since each wave of clusters pays the whole exchange chain.
#ifndef SVL_SELECT_MODE0
    const int cs3 = relevance_select_cs(span.visual_len);
    if (!shared && (long)units * se.CS > 2L * device_sm_count() &&
        (span.visual_len + cs3 - 1) / cs3 <= 8192) {
        float* rel = scores_out ? scores_out : reinterpret_cast<float*>(w + lay.scores);
        e = launch_relevance(se, rel, units, s);
        if (e != cudaSuccess) return cuda_fail(e, "svl_retrieve/relevance");
        se.mode = 3;
        se.scores_in = rel;
        se.scores_out = nullptr;
        se.CS = cs3;
    }
#endif
    e = launch_select(se, shared ? B : units, s);
    if (e != cudaSuccess) return cuda_fail(e, "svl_retrieve/select");
    return SVL_OK;
}

// ------------------------------------------- sequence split
svl_status svl_retrieve_partial_lse(const void* q, int32_t B, int32_t n_q, int32_t H, int32_t Hkv, int32_t d,
                                    svl_kv K, svl_span span, float scale, uint32_t flags, float* lse_out, void* ws,
                                    size_t ws_bytes, void* stream) {
    if (!q || !lse_out || !span.seq_len) return fail(SVL_ERR_INVALID_ARGUMENT, "NULL pointer argument%s");
    if (flags & ~(SVL_NORM_VISUAL_ONLY | SVL_SHARD_VIEW)) return fail(SVL_ERR_INVALID_ARGUMENT, "unknown flag bits%s");
    if (B < 1 || n_q < 1 || H < 1 || Hkv < 1) return fail(SVL_ERR_SHAPE, "B, n_q, H, Hkv must be >= 1%s");
    if (H % Hkv) return fail(SVL_ERR_SHAPE, "H %% Hkv != 0%s");
    if (span.visual_len < 1) return fail(SVL_ERR_SHAPE, "no visual rows%s");
    const int q_rows = (flags & SVL_SHARD_VIEW) ? 0 : n_q;
    if (span.visual_begin < 0 || (int64_t)span.visual_begin + span.visual_len + q_rows > (int64_t)K.capacity)
        return fail(SVL_ERR_SHAPE, "visual span + query rows outside the KV capacity%s");
    if (!(scale > 0.f) || !isfinite(scale)) return fail(SVL_ERR_INVALID_ARGUMENT, "scale must be finite > 0%s");
    if (d != 64 && d != 128) return fail(SVL_ERR_UNSUPPORTED, "head dim must be 64 or 128%s");
    const int g = H / Hkv;
    if (n_q * g > 32) return fail(SVL_ERR_UNSUPPORTED, "partial LSE needs n_q * g <= 32%s");
    if (!aligned16(q)) return fail(SVL_ERR_ALIGNMENT, "q not 16-byte aligned%s");
    svl_status st = check_kv(K, B, Hkv, d, "K");
    if (st != SVL_OK) return st;
    if (!ws || !aligned16(ws)) return fail(SVL_ERR_WORKSPACE, "workspace NULL or misaligned%s");
    st = check_device();
    if (st != SVL_OK) return st;
    const int units = B * Hkv;
    ScorePlan pl = plan_score(units, n_q, g, span.visual_len, device_sm_count());
    RetrieveLayout lay = retrieve_layout(B, Hkv, span.visual_len, pl);
    if (ws_bytes < lay.total) return fail(SVL_ERR_WORKSPACE, "workspace too small%s");
    uint8_t* w = static_cast<uint8_t*>(ws);
    ScoreParams sp;
    sp.q = static_cast<const uint16_t*>(q);
    sp.K = static_cast<const uint16_t*>(K.data);
    sp.sb = K.stride_b; sp.sh = K.stride_h; sp.st = K.stride_t;
    sp.seq_len = span.seq_len;
    sp.B = B; sp.n_q = n_q; sp.H = H; sp.Hkv = Hkv; sp.g = g;
    sp.NC = n_q * g; sp.NCP = pl.NCP;
    sp.vb = span.visual_begin; sp.nv = span.visual_len; sp.capacity = K.capacity;
    sp.C = pl.C; sp.rows_per_chunk = pl.rows_per_chunk;
    sp.need_partials = 1;
    sp.use_text = (flags & SVL_NORM_VISUAL_ONLY) ? 0 : 1;
    sp.q_rows_in_view = q_rows;
    sp.scale2 = scale * kLog2e;
    sp.logits = reinterpret_cast<float*>(w + lay.logits);
    sp.part = reinterpret_cast<float2*>(w + lay.part);
    sp.flags = reinterpret_cast<uint32_t*>(w);
    cudaError_t e = launch_score(sp, d, pl.NT, (cudaStream_t)stream);
    if (e == cudaSuccess)
        e = launch_lse_from_partials(sp.part, units, pl.C, pl.NCP, sp.NC, g, n_q, H, Hkv, lse_out, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "svl_retrieve_partial_lse");
    return SVL_OK;
}

svl_status svl_lse_combine(const float* parts, int32_t P, int32_t n, float* out, void* stream) {
    if (!parts || !out) return fail(SVL_ERR_INVALID_ARGUMENT, "NULL pointer argument%s");
    if (P < 1 || n < 0) return fail(SVL_ERR_SHAPE, "P >= 1, n >= 0%s");
    svl_status st = check_device();
    if (st != SVL_OK) return st;
    if (n == 0) return SVL_OK;
    cudaError_t e = launch_lse_combine(parts, P, n, out, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "svl_lse_combine");
    return SVL_OK;
}

size_t svl_topk_workspace_size(int32_t units, int32_t n) {
    (void)units;
    (void)n;
    return kWsHeader;
}

svl_status svl_topk(const float* scores, int32_t units, int32_t n, int32_t k, int32_t* idx_out, void* ws,
                    size_t ws_bytes, void* stream) {
    if (!scores || (!idx_out && k > 0)) return fail(SVL_ERR_INVALID_ARGUMENT, "NULL pointer argument%s");
    if (units < 1 || n < 1) return fail(SVL_ERR_SHAPE, "units, n must be >= 1%s");
    if (k < 0 || k > n) return fail(SVL_ERR_INVALID_ARGUMENT, "k outside [0, n]%s");
    if (n > 16 * kSelectThreads * kSelectMaxPerThread) return fail(SVL_ERR_UNSUPPORTED, "n > 131072%s");
    if (!ws || !aligned16(ws) || ws_bytes < kWsHeader) return fail(SVL_ERR_WORKSPACE, "workspace NULL, misaligned or too small%s");
    svl_status st = check_device();
    if (st != SVL_OK) return st;
    if (k == 0) return SVL_OK;
    SelectParams se = {};
    se.mode = 2;
    se.scores_in = scores;
    se.Hkv = 1;
    se.shared = 0;
    se.nv = n; se.k = k;
    se.idx_out = idx_out;
    se.flags = static_cast<uint32_t*>(ws);
    se.CS = select_cluster_size(n);
    cudaError_t e = launch_select(se, units, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "svl_topk");
    return SVL_OK;
}

svl_status svl_shard_indices(const int32_t* idx, int32_t units, int32_t k, int32_t lo, int32_t hi, int32_t* out,
                             void* stream) {
    if ((!idx || !out) && k > 0) return fail(SVL_ERR_INVALID_ARGUMENT, "NULL pointer argument%s");
    if (units < 1 || k < 0 || lo < 0 || hi < lo) return fail(SVL_ERR_SHAPE, "units >= 1, k >= 0, 0 <= lo <= hi%s");
    svl_status st = check_device();
    if (st != SVL_OK) return st;
    if (k == 0) return SVL_OK;
    cudaError_t e = launch_shard_indices(idx, units, k, lo, hi, out, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "svl_shard_indices");
    return SVL_OK;
}

svl_status svl_merge_partials(const float* out_parts, const float* lse_parts, int32_t P, int32_t rows, int32_t d,
                              float* out, float* lse_out, void* stream) {
    if (!out_parts || !lse_parts || !out) return fail(SVL_ERR_INVALID_ARGUMENT, "NULL pointer argument%s");
    if (P < 1 || rows < 1 || d < 1) return fail(SVL_ERR_SHAPE, "P, rows, d must be >= 1%s");
    svl_status st = check_device();
    if (st != SVL_OK) return st;
    cudaError_t e = launch_merge_partials(out_parts, lse_parts, P, rows, d, out, lse_out, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "svl_merge_partials");
    return SVL_OK;
}

// ------------------------------------------------------------ sparse decode
size_t svl_sparse_decode_workspace_size(int32_t B, int32_t H, int32_t Hkv, int32_t d, int32_t k,
                                        int32_t visual_len, int32_t capacity, uint32_t flags) {
    (void)flags;
    if (B < 1 || Hkv < 1 || H % Hkv || capacity < 1 || k < 0 || visual_len < 0) return 0;
    const int n_att_max = std::max(1, k + std::max(0, capacity - visual_len));
    const int units = B * Hkv;
    return decode_ws_bytes(units, plan_decode(units, n_att_max, d, flags).S, d);
}

struct PushArgs {
    int P = 0, rank = 0, b0 = 0, h0 = 0, B_total = 0, H_total = 0;
    uint32_t epoch = 0;
    float* const* peer_out = nullptr;
    uint32_t* const* peer_flags = nullptr;
};

static svl_status sparse_decode_impl(const void* q, int32_t B, int32_t H, int32_t Hkv, int32_t d,
                                     svl_kv K, svl_kv V, svl_span span, const int32_t* vis_idx,
                                     int32_t k, uint32_t flags, float scale, float* out,
                                     float* lse_out, void* ws, size_t ws_bytes, void* stream,
                                     const PushArgs& push, const char* name) {
    if (!q || (!out && push.P == 0) || !span.seq_len || (k > 0 && !vis_idx))
        return fail(SVL_ERR_INVALID_ARGUMENT, "NULL pointer argument%s");
    if (flags & ~(SVL_SELECT_SHARED | SVL_PIN_SPLITS_MASK | SVL_IDX_PADDED | SVL_DECODE_GRID_MERGE | SVL_DECODE_STATIC_PREFIX))
        return fail(SVL_ERR_INVALID_ARGUMENT, "unknown flag bits%s");
    if (B < 1 || H < 1 || Hkv < 1) return fail(SVL_ERR_SHAPE, "B, H, Hkv must be >= 1%s");
    if (H % Hkv) return fail(SVL_ERR_SHAPE, "H %% Hkv != 0%s");
    if (span.visual_begin < 0 || span.visual_len < 0 ||
        (int64_t)span.visual_begin + span.visual_len > (int64_t)K.capacity)
        return fail(SVL_ERR_SHAPE, "visual span outside the KV capacity%s");
    if (K.capacity != V.capacity) return fail(SVL_ERR_SHAPE, "K and V capacities differ%s");
    if (k < 0 || k > span.visual_len) return fail(SVL_ERR_INVALID_ARGUMENT, "k outside [0, visual_len]%s");
    if (!(scale > 0.f) || !isfinite(scale)) return fail(SVL_ERR_INVALID_ARGUMENT, "scale must be finite > 0%s");
    if (d != 64 && d != 128) return fail(SVL_ERR_UNSUPPORTED, "head dim must be 64 or 128%s");
    const int g = H / Hkv;
    if (g > 16) return fail(SVL_ERR_UNSUPPORTED, "g = H/Hkv must be <= 16 in this version%s");
    if (!aligned16(q)) return fail(SVL_ERR_ALIGNMENT, "q not 16-byte aligned%s");
    if (out && !aligned16(out)) return fail(SVL_ERR_ALIGNMENT, "out not 16-byte aligned%s");
    svl_status st = check_kv(K, B, Hkv, d, "K");
    if (st != SVL_OK) return st;
    st = check_kv(V, B, Hkv, d, "V");
    if (st != SVL_OK) return st;
    if (!ws || !aligned16(ws)) return fail(SVL_ERR_WORKSPACE, "workspace NULL or misaligned%s");
    st = check_device();
    if (st != SVL_OK) return st;

    const int units = B * Hkv;
    const int n_att_max = std::max(1, k + std::max(0, K.capacity - span.visual_len));
    const DecodePlan plan = plan_decode(units, n_att_max, d, flags);
    const int S = plan.S;
    // cluster: the unit's S CTAs merge over DSMEM; else the grid merge through L2 (co-resident grid)
    const int cluster = plan.cluster;
    if (S > 1 && !cluster && ((long)units * S > decode_slots(d) || units > kWsEpochs))
        return fail(SVL_ERR_UNSUPPORTED, "pinned split count: B*Hkv*n exceeds the co-resident CTA count%s");
    if (ws_bytes < decode_ws_bytes(units, S, d)) return fail(SVL_ERR_WORKSPACE, "workspace too small%s");

    DecodeParams p;
    p.q = static_cast<const uint16_t*>(q);
    p.K = static_cast<const uint16_t*>(K.data);
    p.ksb = K.stride_b; p.ksh = K.stride_h; p.kst = K.stride_t;
    p.V = static_cast<const uint16_t*>(V.data);
    p.vsb = V.stride_b; p.vsh = V.stride_h; p.vst = V.stride_t;
    p.seq_len = span.seq_len;
    p.idx = vis_idx;
    p.B = B; p.H = H; p.Hkv = Hkv; p.g = g;
    p.vb = span.visual_begin; p.nv = span.visual_len; p.k = k;
    p.shared = (flags & SVL_SELECT_SHARED) ? 1 : 0;
    p.padded = (flags & SVL_IDX_PADDED) ? 1 : 0;
    p.cluster = cluster;
    p.static_vis = (flags & SVL_DECODE_STATIC_PREFIX) ? 1 : 0;
    p.capacity = K.capacity;
    p.S = S;
    // rows of one split <= ceil(vb / S) + ceil(k / S) + ceil(T_max / S) (three segments)
    p.single_batch = ((span.visual_begin + S - 1) / S + (k + S - 1) / S +
                      (std::max(0, K.capacity - span.visual_begin - span.visual_len) + S - 1) / S) <= kDecodeRowsMax;
    p.scale2 = scale * kLog2e;
    p.out = out;
    p.lse_out = lse_out;
    p.flags = static_cast<uint32_t*>(ws);
    p.part = reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(ws) + kWsHeader);
    p.sync = static_cast<uint32_t*>(ws);  // header: word 0 is the flag word
    p.epochs = static_cast<uint32_t*>(ws) + kWsEpochWord;
    p.trace = nullptr;
#if SVL_TRACE_BUILD  // phase-stamp builds (tools/trace_decode.py): the last 1 MB of a larger workspace
    if (ws_bytes >= decode_ws_bytes(units, S, d) + ((size_t)1 << 20))
        p.trace = reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(ws) + ws_bytes - ((size_t)1 << 20));
#endif
    p.P = push.P;
    p.rank = push.rank;
    p.b0 = push.b0;
    p.h0 = push.h0;
    p.B_total = push.B_total;
    p.H_total = push.H_total;
    p.epoch = push.epoch;
    for (int r = 0; r < kMaxPeers; ++r) {
        p.peer_out[r] = (r < push.P) ? push.peer_out[r] : nullptr;
        p.peer_flags[r] = (r < push.P) ? push.peer_flags[r] : nullptr;
    }
    cudaError_t e = launch_decode(p, d, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, name);
    return SVL_OK;
}

svl_status svl_rope_remap(svl_kv K, svl_kv V, int32_t B, int32_t Hkv, int32_t d, svl_span span,
                          const int32_t* kept, int32_t k, double rope_base, svl_kv Ko, svl_kv Vo, void* ws,
                          size_t ws_bytes, void* stream) {
    if (!span.seq_len || (k > 0 && !kept) || !K.data || !Ko.data || (V.data && !Vo.data))
        return fail(SVL_ERR_INVALID_ARGUMENT, "NULL pointer argument%s");
    if (B < 1 || Hkv < 1) return fail(SVL_ERR_SHAPE, "B, Hkv must be >= 1%s");
    if (!(rope_base > 1.0) || !isfinite(rope_base)) return fail(SVL_ERR_INVALID_ARGUMENT, "rope_base must be finite > 1%s");
    if (span.visual_begin < 0 || span.visual_len < 0 ||
        (int64_t)span.visual_begin + span.visual_len > (int64_t)K.capacity)
        return fail(SVL_ERR_SHAPE, "visual span outside the KV capacity%s");
    if (k < 0 || k > span.visual_len) return fail(SVL_ERR_INVALID_ARGUMENT, "k outside [0, visual_len]%s");
    if (d != 64 && d != 128) return fail(SVL_ERR_UNSUPPORTED, "head dim must be 64 or 128%s");
    const int64_t need = (int64_t)span.visual_begin + k + (K.capacity - span.visual_begin - span.visual_len);
    if (Ko.capacity < need || (V.data && Vo.capacity < need))
        return fail(SVL_ERR_SHAPE, "output capacity < vb + k + (capacity - vb - N_v)%s");
    if (V.data && V.capacity != K.capacity) return fail(SVL_ERR_SHAPE, "K and V capacities differ%s");
    svl_status st = check_kv(K, B, Hkv, d, "K_pre");
    if (st == SVL_OK) st = check_kv(Ko, B, Hkv, d, "K_out");
    if (st == SVL_OK && V.data) st = check_kv(V, B, Hkv, d, "V");
    if (st == SVL_OK && V.data) st = check_kv(Vo, B, Hkv, d, "V_out");
    if (st != SVL_OK) return st;
    if (!ws || !aligned16(ws) || ws_bytes < kWsHeader) return fail(SVL_ERR_WORKSPACE, "workspace NULL, misaligned or too small%s");
    st = check_device();
    if (st != SVL_OK) return st;
    RopeParams p;
    p.K = static_cast<const uint16_t*>(K.data);
    p.ksb = K.stride_b; p.ksh = K.stride_h; p.kst = K.stride_t;
    p.V = static_cast<const uint16_t*>(V.data);
    p.vsb = V.stride_b; p.vsh = V.stride_h; p.vst = V.stride_t;
    p.Ko = static_cast<uint16_t*>(const_cast<void*>(Ko.data));
    p.osb = Ko.stride_b; p.osh = Ko.stride_h; p.ost = Ko.stride_t;
    p.Vo = static_cast<uint16_t*>(const_cast<void*>(Vo.data));
    p.vosb = Vo.stride_b; p.vosh = Vo.stride_h; p.vost = Vo.stride_t;
    p.seq_len = span.seq_len;
    p.kept = kept;
    p.B = B; p.Hkv = Hkv; p.d = d; p.vb = span.visual_begin; p.nv = span.visual_len; p.k = k;
    p.capacity = K.capacity;
    p.log2_base = log2(rope_base);
    p.flags = static_cast<uint32_t*>(ws);
    cudaError_t e = launch_rope_remap(p, (int)need, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "svl_rope_remap");
    return SVL_OK;
}

size_t svl_mrope_remap_workspace_size(int32_t B, int32_t k) {
    if (B < 1 || k < 0) return 0;
    return round_up(kWsHeader + (size_t)B * 3 * sizeof(int32_t), 256) + round_up((size_t)B * k * 3 * sizeof(int32_t), 256);
}

svl_status svl_mrope_remap(svl_kv K, svl_kv V, int32_t B, int32_t Hkv, int32_t d, svl_span span,
                           const int32_t* coords, const int32_t* kept, int32_t k, double rope_base,
                           const int32_t* sections, svl_kv Ko, svl_kv Vo, int32_t* new_coords_out,
                           int32_t* text_start_out, void* ws, size_t ws_bytes, void* stream) {
    if (!span.seq_len || (k > 0 && (!kept || !coords)) || !K.data || !Ko.data || (V.data && !Vo.data) || !sections)
        return fail(SVL_ERR_INVALID_ARGUMENT, "NULL pointer argument%s");
    if (B < 1 || Hkv < 1) return fail(SVL_ERR_SHAPE, "B, Hkv must be >= 1%s");
    if (!(rope_base > 1.0) || !isfinite(rope_base)) return fail(SVL_ERR_INVALID_ARGUMENT, "rope_base must be finite > 1%s");
    if (span.visual_begin < 0 || span.visual_len < 0 ||
        (int64_t)span.visual_begin + span.visual_len > (int64_t)K.capacity)
        return fail(SVL_ERR_SHAPE, "visual span outside the KV capacity%s");
    if (k < 0 || k > span.visual_len) return fail(SVL_ERR_INVALID_ARGUMENT, "k outside [0, visual_len]%s");
    if (d != 64 && d != 128) return fail(SVL_ERR_UNSUPPORTED, "head dim must be 64 or 128%s");
    if (sections[0] < 0 || sections[1] < 0 || sections[2] < 0 || sections[0] + sections[1] + sections[2] != d / 2 ||
        (sections[0] & 1) || (sections[1] & 1))
        return fail(SVL_ERR_INVALID_ARGUMENT, "sections must be >= 0, sum to d/2, the first two even%s");
    const int64_t need = (int64_t)span.visual_begin + k + (K.capacity - span.visual_begin - span.visual_len);
    if (Ko.capacity < need || (V.data && Vo.capacity < need))
        return fail(SVL_ERR_SHAPE, "output capacity < vb + k + (capacity - vb - N_v)%s");
    if (V.data && V.capacity != K.capacity) return fail(SVL_ERR_SHAPE, "K and V capacities differ%s");
    svl_status st = check_kv(K, B, Hkv, d, "K_pre");
    if (st == SVL_OK) st = check_kv(Ko, B, Hkv, d, "K_out");
    if (st == SVL_OK && V.data) st = check_kv(V, B, Hkv, d, "V");
    if (st == SVL_OK && V.data) st = check_kv(Vo, B, Hkv, d, "V_out");
    if (st != SVL_OK) return st;
    if (!ws || !aligned16(ws) || ws_bytes < svl_mrope_remap_workspace_size(B, k))
        return fail(SVL_ERR_WORKSPACE, "workspace NULL, misaligned or too small%s");
    st = check_device();
    if (st != SVL_OK) return st;
    uint8_t* w = static_cast<uint8_t*>(ws);
    MropeParams p;
    p.K = static_cast<const uint16_t*>(K.data);
    p.ksb = K.stride_b; p.ksh = K.stride_h; p.kst = K.stride_t;
    p.V = static_cast<const uint16_t*>(V.data);
    p.vsb = V.stride_b; p.vsh = V.stride_h; p.vst = V.stride_t;
    p.Ko = static_cast<uint16_t*>(const_cast<void*>(Ko.data));
    p.osb = Ko.stride_b; p.osh = Ko.stride_h; p.ost = Ko.stride_t;
    p.Vo = static_cast<uint16_t*>(const_cast<void*>(Vo.data));
    p.vosb = Vo.stride_b; p.vosh = Vo.stride_h; p.vost = Vo.stride_t;
    p.seq_len = span.seq_len;
    p.kept = kept;
    p.coords = coords;
    p.B = B; p.Hkv = Hkv; p.d = d; p.vb = span.visual_begin; p.nv = span.visual_len; p.k = k;
    p.capacity = K.capacity;
    p.sec0 = sections[0]; p.sec1 = sections[1];
    p.log2_base = log2(rope_base);
    p.dim_max = reinterpret_cast<int32_t*>(w + kWsHeader);
    p.new_coords = new_coords_out ? new_coords_out
                                  : reinterpret_cast<int32_t*>(w + round_up(kWsHeader + (size_t)B * 3 * sizeof(int32_t), 256));
    p.text_start_out = text_start_out;
    p.flags = static_cast<uint32_t*>(ws);
    cudaError_t e = launch_mrope_remap(p, (int)need, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "svl_mrope_remap");
    return SVL_OK;
}

svl_status svl_pack_kv(svl_kv K, svl_kv V, int32_t B, int32_t Hkv, int32_t d, svl_span span,
                       const int32_t* vis_idx, int32_t k, uint32_t flags, svl_kv Kp, svl_kv Vp, void* ws,
                       size_t ws_bytes, void* stream) {
    if (!span.seq_len || (k > 0 && !vis_idx)) return fail(SVL_ERR_INVALID_ARGUMENT, "NULL pointer argument%s");
    if (flags & ~(SVL_SELECT_SHARED)) return fail(SVL_ERR_INVALID_ARGUMENT, "unknown flag bits%s");
    if (B < 1 || Hkv < 1) return fail(SVL_ERR_SHAPE, "B, Hkv must be >= 1%s");
    if (span.visual_begin < 0 || span.visual_len < 0 ||
        (int64_t)span.visual_begin + span.visual_len > (int64_t)K.capacity)
        return fail(SVL_ERR_SHAPE, "visual span outside the KV capacity%s");
    if (K.capacity != V.capacity || Kp.capacity != Vp.capacity) return fail(SVL_ERR_SHAPE, "K/V capacities differ%s");
    if (k < 0 || k > span.visual_len) return fail(SVL_ERR_INVALID_ARGUMENT, "k outside [0, visual_len]%s");
    const int64_t need = (int64_t)span.visual_begin + k + (K.capacity - span.visual_begin - span.visual_len);
    if (Kp.capacity < need) return fail(SVL_ERR_SHAPE, "packed capacity < vb + k + (capacity - vb - N_v)%s");
    if (d != 64 && d != 128) return fail(SVL_ERR_UNSUPPORTED, "head dim must be 64 or 128%s");
    svl_status st = check_kv(K, B, Hkv, d, "K");
    if (st == SVL_OK) st = check_kv(V, B, Hkv, d, "V");
    if (st == SVL_OK) st = check_kv(Kp, B, Hkv, d, "Kp");
    if (st == SVL_OK) st = check_kv(Vp, B, Hkv, d, "Vp");
    if (st != SVL_OK) return st;
    if (!ws || !aligned16(ws) || ws_bytes < kWsHeader) return fail(SVL_ERR_WORKSPACE, "workspace NULL, misaligned or too small%s");
    st = check_device();
    if (st != SVL_OK) return st;
    PackParams p;
    p.K = static_cast<const uint16_t*>(K.data); p.V = static_cast<const uint16_t*>(V.data);
    p.ksb = K.stride_b; p.ksh = K.stride_h; p.kst = K.stride_t;
    p.vsb = V.stride_b; p.vsh = V.stride_h; p.vst = V.stride_t;
    p.Kp = static_cast<uint16_t*>(const_cast<void*>(Kp.data)); p.Vp = static_cast<uint16_t*>(const_cast<void*>(Vp.data));
    p.pksb = Kp.stride_b; p.pksh = Kp.stride_h; p.pkst = Kp.stride_t;
    p.pvsb = Vp.stride_b; p.pvsh = Vp.stride_h; p.pvst = Vp.stride_t;
    p.seq_len = span.seq_len;
    p.idx = vis_idx;
    p.B = B; p.Hkv = Hkv; p.vb = span.visual_begin; p.nv = span.visual_len; p.k = k; p.capacity = K.capacity;
    p.shared = (flags & SVL_SELECT_SHARED) ? 1 : 0;
    p.flags = static_cast<uint32_t*>(ws);
    cudaError_t e = launch_pack(p, d, (int)need, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "svl_pack_kv");
    return SVL_OK;
}

svl_status svl_sparse_decode_attn(const void* q, int32_t B, int32_t H, int32_t Hkv, int32_t d,
                                  svl_kv K, svl_kv V, svl_span span, const int32_t* vis_idx,
                                  int32_t k, uint32_t flags, float scale, float* out,
                                  float* lse_out, void* ws, size_t ws_bytes, void* stream) {
    return sparse_decode_impl(q, B, H, Hkv, d, K, V, span, vis_idx, k, flags, scale, out, lse_out, ws,
                              ws_bytes, stream, PushArgs(), "svl_sparse_decode_attn");
}

svl_status svl_sparse_decode_attn_push(const void* q, int32_t B, int32_t H, int32_t Hkv, int32_t d,
                                       svl_kv K, svl_kv V, svl_span span, const int32_t* vis_idx,
                                       int32_t k, uint32_t flags, float scale, float* out,
                                       float* lse_out, float* const* peer_out,
                                       uint32_t* const* peer_flags, int32_t rank, int32_t P,
                                       uint32_t epoch, int32_t b0, int32_t h0, int32_t B_total,
                                       int32_t H_total, void* ws, size_t ws_bytes, void* stream) {
    if (P < 1 || P > kMaxPeers) return fail(SVL_ERR_INVALID_ARGUMENT, "P outside [1, 8]%s");
    if (rank < 0 || rank >= P) return fail(SVL_ERR_INVALID_ARGUMENT, "rank outside [0, P)%s");
    if (epoch == 0) return fail(SVL_ERR_INVALID_ARGUMENT, "epoch must be > 0%s");
    if (!peer_out || !peer_flags) return fail(SVL_ERR_INVALID_ARGUMENT, "NULL peer arrays%s");
    for (int r = 0; r < P; ++r)
        if (!peer_out[r] || !peer_flags[r] || !aligned16(peer_out[r]))
            return fail(SVL_ERR_INVALID_ARGUMENT, "NULL or misaligned peer buffer%s");
    if (B < 1 || H < 1 || Hkv < 1 || H % Hkv) return fail(SVL_ERR_SHAPE, "B, H, Hkv must be >= 1 and H %% Hkv == 0%s");
    if (b0 < 0 || h0 < 0 || b0 + B > B_total || h0 + H > H_total || H_total % (H / Hkv))
        return fail(SVL_ERR_SHAPE, "shard (b0, h0, B, H) outside (B_total, H_total)%s");
    PushArgs push;
    push.P = P;
    push.rank = rank;
    push.b0 = b0;
    push.h0 = h0;
    push.B_total = B_total;
    push.H_total = H_total;
    push.epoch = epoch;
    push.peer_out = peer_out;
    push.peer_flags = peer_flags;
    return sparse_decode_impl(q, B, H, Hkv, d, K, V, span, vis_idx, k, flags, scale, out, lse_out, ws,
                              ws_bytes, stream, push, "svl_sparse_decode_attn_push");
}

svl_status svl_wait_flags(const uint32_t* flags, int32_t P, uint32_t epoch, void* ws, void* stream) {
    if (!flags || !ws) return fail(SVL_ERR_INVALID_ARGUMENT, "NULL pointer argument%s");
    if (P < 1 || P > kMaxPeers) return fail(SVL_ERR_INVALID_ARGUMENT, "P outside [1, 8]%s");
    if (epoch == 0) return fail(SVL_ERR_INVALID_ARGUMENT, "epoch must be > 0%s");
    svl_status st = check_device();
    if (st != SVL_OK) return st;
    cudaError_t e = launch_wait_flags(flags, P, epoch, static_cast<uint32_t*>(ws), (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "svl_wait_flags");
    return SVL_OK;
}

// ----------------------------------------------------- fused fresh step
// Cluster size and eligibility of the fused kernel for a shape.

static bool fresh_plan(int B, int Hkv, int g, int nv, int capacity, int& CS, int& slice, int d, uint32_t flags) {
    if (g > 16 || (flags & SVL_FRESH_UNFUSED)) return false;
    const int smax = kFusedSliceMax / ((g + 7) / 8);
    int cmin = (nv + smax - 1) / smax;
    if (cmin > 16) return false;
    const int units = B * Hkv;
    int c = 1;
    while (c < cmin) c <<= 1;
    // many SMs per unit while the units are few (HBM streaming is per-SM bound)
    const int want = (units * 16 <= 2 * device_sm_count()) ? 16 : 8;
    CS = std::max(c, want);
    bool pinned = false;
    if (const int v = (int)(flags >> 24)) {  // SVL_PIN_SPLITS(8 or 16)
        if ((v == 8 || v == 16) && v >= c) CS = v, pinned = true;
    }
    // The fused kernel while every unit's cluster is co-resident (one wave), or -- 16-CTA
    // clusters over long slices -- up to three waves; beyond that the two-call kernels, which
    // spread over every SM, are faster (round 1, us/layer fused vs two-call: 16k B=4 67.2 vs
    // 52.4, 4k B=8 55.9 vs 38.9; B=1: 32k 28.1 vs 34.2, 4k 17.3 vs 23.6; round 3 below)
    if (!pinned) {
        const int mac = fresh_max_active_clusters(d, g, CS);
        if (mac <= 0) return false;
        if (units > mac) {
            // several waves of clusters: still ahead of the two calls while a unit's slice is long
            // (round 3, us/layer fused vs two-call: 32k visual B = 3 / 4 / 5: 49.4 / 71.8 / 74.7 vs
            // 56.2 / 76.8 / 91.0; 24k B = 4: 63.8 vs 66.0; 16k B = 4 / 6: 55.6 / 74.5 vs 49.0 / 58.1)
            const int waves = (units + mac - 1) / mac;
            if (!(CS == 16 && (nv + CS - 1) / CS >= 1536 && waves <= 3)) return false;
        }
    }
    slice = (nv + CS - 1) / CS;
    if (slice > smax) return false;
    const int tmax = std::max(0, capacity - nv);  // every non-visual row could be text
    if ((tmax + CS - 1) / CS > kFusedTextMax) return false;
    return true;
}

int32_t svl_fresh_decode_plan(int32_t B, int32_t H, int32_t Hkv, int32_t d, int32_t visual_len, int32_t capacity,
                              uint32_t flags) {
    if (B < 1 || Hkv < 1 || H < 1 || H % Hkv || visual_len < 1 || (d != 64 && d != 128)) return 0;
    int CS, slice;
    return fresh_plan(B, Hkv, H / Hkv, visual_len, capacity, CS, slice, d, flags) ? 1 : 0;
}

size_t svl_fresh_decode_workspace_size(int32_t B, int32_t H, int32_t Hkv, int32_t d, int32_t k,
                                       int32_t visual_len, int32_t capacity, uint32_t flags) {
    if (B < 1 || Hkv < 1 || H % Hkv || visual_len < 1) return 0;
    int CS, slice;
    // (the fused plan needs the header only; the size covers the two-call path too, which
    // the step also takes when the K view cannot be encoded as a TMA tensor map)
    (void)CS; (void)slice;
    return std::max(svl_retrieve_workspace_size(B, 1, H, Hkv, d, visual_len, flags & SVL_NORM_VISUAL_ONLY),
                    svl_sparse_decode_workspace_size(B, H, Hkv, d, k, visual_len, capacity, 0u));
}

svl_status svl_fresh_decode_step(const void* q, int32_t B, int32_t H, int32_t Hkv, int32_t d,
                                 svl_kv K, svl_kv V, svl_span span, int32_t k, float scale,
                                 uint32_t flags, int32_t* idx_out, float* out, float* lse_out,
                                 void* ws, size_t ws_bytes, void* stream) {
    if (!q || !out || !span.seq_len || (k > 0 && !idx_out))
        return fail(SVL_ERR_INVALID_ARGUMENT, "NULL pointer argument%s");
    if (flags & ~(SVL_NORM_VISUAL_ONLY | SVL_FRESH_UNFUSED | SVL_PIN_SPLITS_MASK))
        return fail((flags & SVL_SELECT_SHARED) ? SVL_ERR_UNSUPPORTED : SVL_ERR_INVALID_ARGUMENT,
                    "svl_fresh_decode_step accepts SVL_NORM_VISUAL_ONLY, SVL_FRESH_UNFUSED, SVL_PIN_SPLITS%s");
    if (B < 1 || H < 1 || Hkv < 1) return fail(SVL_ERR_SHAPE, "B, H, Hkv must be >= 1%s");
    if (H % Hkv) return fail(SVL_ERR_SHAPE, "H %% Hkv != 0%s");
    if (span.visual_len < 1) return fail(SVL_ERR_SHAPE, "no visual rows to retrieve from%s");
    if (span.visual_begin < 0 || (int64_t)span.visual_begin + span.visual_len + 1 > (int64_t)K.capacity)
        return fail(SVL_ERR_SHAPE, "visual span + current token outside the KV capacity%s");
    if (K.capacity != V.capacity) return fail(SVL_ERR_SHAPE, "K and V capacities differ%s");
    if (k < 0 || k > span.visual_len) return fail(SVL_ERR_INVALID_ARGUMENT, "k outside [0, visual_len]%s");
    if (!(scale > 0.f) || !isfinite(scale)) return fail(SVL_ERR_INVALID_ARGUMENT, "scale must be finite > 0%s");
    if (d != 64 && d != 128) return fail(SVL_ERR_UNSUPPORTED, "head dim must be 64 or 128%s");
    const int g = H / Hkv;
    if (g > 16) return fail(SVL_ERR_UNSUPPORTED, "g = H/Hkv must be <= 16 in this version%s");
    if (!aligned16(q) || !aligned16(out)) return fail(SVL_ERR_ALIGNMENT, "q / out not 16-byte aligned%s");
    svl_status st = check_kv(K, B, Hkv, d, "K");
    if (st != SVL_OK) return st;
    st = check_kv(V, B, Hkv, d, "V");
    if (st != SVL_OK) return st;
    if (!ws || !aligned16(ws)) return fail(SVL_ERR_WORKSPACE, "workspace NULL or misaligned%s");
    if (ws_bytes < svl_fresh_decode_workspace_size(B, H, Hkv, d, k, span.visual_len, K.capacity, flags))
        return fail(SVL_ERR_WORKSPACE, "workspace too small%s");
    st = check_device();
    if (st != SVL_OK) return st;

    int CS, slice;
    FreshParams p;
    if (!fresh_plan(B, Hkv, g, span.visual_len, K.capacity, CS, slice, d, flags) ||
        !encode_kv_tensor_map(&p.ktmap, K.data, d, K.capacity, Hkv, B, K.stride_b, K.stride_h, K.stride_t, 128)) {
        // outside the on-chip budget: the two separate calls (same q as [B][1][H][d])
        st = svl_retrieve(q, B, 1, H, Hkv, d, K, span, nullptr, k, scale, flags & SVL_NORM_VISUAL_ONLY, idx_out,
                          nullptr, ws, ws_bytes, stream);
        if (st != SVL_OK) return st;
        return svl_sparse_decode_attn(q, B, H, Hkv, d, K, V, span, idx_out, k, 0u, scale, out,
                                      lse_out, ws, ws_bytes, stream);
    }
    p.q = static_cast<const uint16_t*>(q);
    p.K = static_cast<const uint16_t*>(K.data);
    p.ksb = K.stride_b; p.ksh = K.stride_h; p.kst = K.stride_t;
    p.V = static_cast<const uint16_t*>(V.data);
    p.vsb = V.stride_b; p.vsh = V.stride_h; p.vst = V.stride_t;
    p.seq_len = span.seq_len;
    p.B = B; p.H = H; p.Hkv = Hkv; p.g = g;
    p.vb = span.visual_begin; p.nv = span.visual_len; p.k = k; p.capacity = K.capacity;
    p.slice = slice;
    p.flags_in = flags & SVL_NORM_VISUAL_ONLY;
    p.scale2 = scale * kLog2e;
    p.idx_out = idx_out;
    p.out = out;
    p.lse_out = lse_out;
    p.flags = static_cast<uint32_t*>(ws);
    p.trace = nullptr;
#if SVL_TRACE_BUILD  // phase-stamp builds (tools/trace_fresh.py): 1 MB after the header
    if (ws_bytes >= kWsHeader + ((size_t)1 << 20))
        p.trace = reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(ws) + kWsHeader);
#endif
    cudaError_t e = launch_fresh(p, d, CS, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "svl_fresh_decode_step");
    return SVL_OK;
}

// ------------------------------------------------- page summaries (f2(ii))
svl_status svl_page_summary(svl_kv K, int32_t B, int32_t Hkv, int32_t d, svl_span span, int32_t page,
                            void* kmax, void* kmin, void* ws, size_t ws_bytes, void* stream) {
    if (!kmax || !kmin) return fail(SVL_ERR_INVALID_ARGUMENT, "NULL pointer argument%s");
    if (B < 1 || Hkv < 1) return fail(SVL_ERR_SHAPE, "B, Hkv must be >= 1%s");
    if (page < 1) return fail(SVL_ERR_INVALID_ARGUMENT, "page must be >= 1%s");
    if (span.visual_len < 1 || span.visual_len % page)
        return fail(SVL_ERR_SHAPE, "visual_len must be a positive multiple of page%s");
    if (span.visual_begin < 0 || (int64_t)span.visual_begin + span.visual_len > (int64_t)K.capacity)
        return fail(SVL_ERR_SHAPE, "visual span outside the KV capacity%s");
    if (d != 64 && d != 128) return fail(SVL_ERR_UNSUPPORTED, "head dim must be 64 or 128%s");
    if (!aligned16(kmax) || !aligned16(kmin)) return fail(SVL_ERR_ALIGNMENT, "kmax / kmin not 16-byte aligned%s");
    svl_status st = check_kv(K, B, Hkv, d, "K");
    if (st != SVL_OK) return st;
    if (!ws || !aligned16(ws) || ws_bytes < kWsHeader) return fail(SVL_ERR_WORKSPACE, "workspace NULL, misaligned or too small%s");
    st = check_device();
    if (st != SVL_OK) return st;
    PageSumParams p;
    p.K = static_cast<const uint16_t*>(K.data);
    p.ksb = K.stride_b; p.ksh = K.stride_h; p.kst = K.stride_t;
    p.units = B * Hkv; p.Hkv = Hkv; p.d = d; p.vb = span.visual_begin; p.page = page;
    p.np = span.visual_len / page;
    p.kmax = static_cast<uint16_t*>(kmax);
    p.kmin = static_cast<uint16_t*>(kmin);
    cudaError_t e = launch_page_summary(p, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "svl_page_summary");
    return SVL_OK;
}

struct PagesLayout {
    size_t ub2, scores, total;
};
static PagesLayout pages_layout(int units, int NC, int n_pages) {
    PagesLayout l;
    l.ub2 = kWsHeader;
    l.scores = round_up(l.ub2 + (size_t)units * NC * n_pages * sizeof(float), 256);
    l.total = round_up(l.scores + (size_t)units * n_pages * sizeof(float), 256);
    return l;
}

size_t svl_retrieve_pages_workspace_size(int32_t B, int32_t n_q, int32_t H, int32_t Hkv, int32_t n_pages) {
    if (B < 1 || n_q < 1 || Hkv < 1 || H % Hkv || n_pages < 1) return 0;
    return pages_layout(B * Hkv, n_q * (H / Hkv), n_pages).total;
}

svl_status svl_retrieve_pages(const void* q, int32_t B, int32_t n_q, int32_t H, int32_t Hkv, int32_t d,
                              const void* kmax, const void* kmin, int32_t n_pages, int32_t page, int32_t k_pages,
                              float scale, uint32_t flags, int32_t* page_idx_out, int32_t* row_idx_out,
                              float* scores_out, void* ws, size_t ws_bytes, void* stream) {
    if (!q || !kmax || !kmin || (!page_idx_out && k_pages > 0))
        return fail(SVL_ERR_INVALID_ARGUMENT, "NULL pointer argument%s");
    if (flags) return fail(SVL_ERR_INVALID_ARGUMENT, "unknown flag bits%s");
    if (B < 1 || n_q < 1 || H < 1 || Hkv < 1) return fail(SVL_ERR_SHAPE, "B, n_q, H, Hkv must be >= 1%s");
    if (H % Hkv) return fail(SVL_ERR_SHAPE, "H %% Hkv != 0%s");
    if (n_pages < 1 || page < 1) return fail(SVL_ERR_SHAPE, "n_pages and page must be >= 1%s");
    if (k_pages < 0 || k_pages > n_pages) return fail(SVL_ERR_INVALID_ARGUMENT, "k_pages outside [0, n_pages]%s");
    if (!(scale > 0.f) || !isfinite(scale)) return fail(SVL_ERR_INVALID_ARGUMENT, "scale must be finite > 0%s");
    if (d != 64 && d != 128) return fail(SVL_ERR_UNSUPPORTED, "head dim must be 64 or 128%s");
    const int g = H / Hkv;
    if (n_q * g > 32) return fail(SVL_ERR_UNSUPPORTED, "page retrieval needs n_q * g <= 32%s");
    if (n_pages > 16 * kSelectThreads * kSelectMaxPerThread) return fail(SVL_ERR_UNSUPPORTED, "n_pages > 131072%s");
    if (!aligned16(q) || !aligned16(kmax) || !aligned16(kmin)) return fail(SVL_ERR_ALIGNMENT, "q / kmax / kmin not 16-byte aligned%s");
    const int units = B * Hkv;
    PagesLayout lay = pages_layout(units, n_q * g, n_pages);
    if (!ws || !aligned16(ws) || ws_bytes < lay.total) return fail(SVL_ERR_WORKSPACE, "workspace NULL, misaligned or too small%s");
    svl_status st = check_device();
    if (st != SVL_OK) return st;
    uint8_t* w = static_cast<uint8_t*>(ws);
    cudaStream_t s = (cudaStream_t)stream;
    PageRetrParams p;
    p.q = static_cast<const uint16_t*>(q);
    p.kmax = static_cast<const uint16_t*>(kmax);
    p.kmin = static_cast<const uint16_t*>(kmin);
    p.units = units; p.n_q = n_q; p.H = H; p.Hkv = Hkv; p.g = g; p.NC = n_q * g; p.d = d; p.np = n_pages;
    p.scale2 = scale * kLog2e;
    p.ub2 = reinterpret_cast<float*>(w + lay.ub2);
    p.scores = scores_out ? scores_out : reinterpret_cast<float*>(w + lay.scores);
    cudaError_t e = launch_page_scores(p, s);
    if (e != cudaSuccess) return cuda_fail(e, "svl_retrieve_pages/scores");
    if (k_pages == 0) return SVL_OK;
    SelectParams se = {};
    se.mode = 2;
    se.scores_in = p.scores;
    se.Hkv = Hkv;
    se.shared = 0;
    se.nv = n_pages; se.k = k_pages;
    se.idx_out = page_idx_out;
    se.flags = reinterpret_cast<uint32_t*>(w);
    se.CS = select_cluster_size(n_pages);
    e = launch_select(se, units, s);
    if (e != cudaSuccess) return cuda_fail(e, "svl_retrieve_pages/select");
    if (row_idx_out) {
        e = launch_page_expand(page_idx_out, units, k_pages, page, row_idx_out, s);
        if (e != cudaSuccess) return cuda_fail(e, "svl_retrieve_pages/expand");
    }
    return SVL_OK;
}

// ---------------------------------------------------------------- prune
size_t svl_prune_workspace_size(int32_t B, int32_t N, int32_t n_frames) {
    (void)B;
    (void)N;
    (void)n_frames;
    return kWsHeader;
}

svl_status svl_prefill_prune(const float* saliency, int32_t B, int32_t N,
                             const int32_t* frame_offsets, int32_t n_frames,
                             double prefill_sparsity, int32_t* kept_idx, int32_t kept_capacity,
                             int32_t* kept_total, void* ws, size_t ws_bytes, void* stream) {
    if (!saliency || !kept_idx || !kept_total) return fail(SVL_ERR_INVALID_ARGUMENT, "NULL pointer argument%s");
    if (B < 1 || N < 1) return fail(SVL_ERR_SHAPE, "B and N must be >= 1%s");
    if (!(prefill_sparsity >= 0.0 && prefill_sparsity < 1.0))
        return fail(SVL_ERR_INVALID_ARGUMENT, "prefill_sparsity outside [0, 1)%s");
    const int nf = frame_offsets ? n_frames : 1;
    if (nf < 1) return fail(SVL_ERR_SHAPE, "n_frames must be >= 1%s");
    if (nf > kMaxFrames) return fail(SVL_ERR_UNSUPPORTED, "more than 2047 frames per call%s");
    PruneTable tab;
    int64_t total = 0;
    int max_n = 0;
    for (int f = 0; f < nf; ++f) {
        const int o0 = frame_offsets ? frame_offsets[f] : 0;
        const int o1 = frame_offsets ? frame_offsets[f + 1] : N;
        if (o1 < o0 || o0 < 0 || o1 > N) return fail(SVL_ERR_SHAPE, "frame_offsets not ascending within [0, N]%s");
        if (f == 0 && o0 != 0) return fail(SVL_ERR_SHAPE, "frame_offsets[0] must be 0%s");
        if (f == nf - 1 && o1 != N) return fail(SVL_ERR_SHAPE, "frame_offsets[n_frames] must be N%s");
        const int n = o1 - o0;
        if (n > 16 * kSelectThreads * kSelectMaxPerThread)
            return fail(SVL_ERR_UNSUPPORTED, "frame larger than 131072 tokens%s");
        max_n = std::max(max_n, n);
        tab.fr[f] = make_int2(o0, (int)total);
        total += svl_keep_budget(n, prefill_sparsity);
    }
    tab.fr[nf] = make_int2(N, (int)total);
    if (total > kept_capacity) return fail(SVL_ERR_INVALID_ARGUMENT, "kept_capacity < sum of frame budgets%s");
    *kept_total = (int32_t)total;
    if (!ws || !aligned16(ws)) return fail(SVL_ERR_WORKSPACE, "workspace NULL or misaligned%s");
    if (ws_bytes < kWsHeader) return fail(SVL_ERR_WORKSPACE, "workspace too small%s");
    if (!aligned16(saliency)) return fail(SVL_ERR_ALIGNMENT, "saliency not 16-byte aligned%s");
    svl_status st = check_device();
    if (st != SVL_OK) return st;
    SelectParams se = {};
    se.mode = 1;
    se.scores_in = saliency;
    se.N = N;
    se.nf = nf;
    se.kept_cap = kept_capacity;
    se.idx_out = kept_idx;
    se.flags = static_cast<uint32_t*>(ws);
    se.CS = select_cluster_size(max_n);
    cudaError_t e = launch_prune_select(se, tab, B * nf, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "svl_prefill_prune");
    return SVL_OK;
}

// --------------------------------------------------------------- salience
size_t svl_salience_workspace_size(int32_t F, int32_t S, int32_t N_f, int32_t H_e, int32_t d_e,
                                   int32_t mode) {
    (void)d_e;
    if (F < 1 || N_f < 1 || H_e < 1) return 0;
    const int rows = (mode == SVL_SAL_INTRA_VISUAL) ? N_f : S;
    return round_up(kWsHeader + (size_t)F * H_e * std::max(rows, 1) * sizeof(float), 256) +
           round_up((size_t)F * H_e * N_f * sizeof(float), 256);
}

svl_status svl_salience(const void* Qe, const void* Ke, int32_t F, int32_t S, int32_t N_f,
                        int32_t H_e, int32_t d_e, int32_t mode, float scale, float* saliency,
                        void* ws, size_t ws_bytes, void* stream) {
    if (!Qe || !Ke || !saliency) return fail(SVL_ERR_INVALID_ARGUMENT, "NULL pointer argument%s");
    if (F < 1 || N_f < 1 || H_e < 1 || S < 0) return fail(SVL_ERR_SHAPE, "bad F / N_f / H_e / S%s");
    if ((mode == SVL_SAL_SUMMARY && S != 1) || (mode == SVL_SAL_MULTI_SUMMARY && S < 2) ||
        (mode == SVL_SAL_INTRA_VISUAL && S != 0) || mode < 0 || mode > 2)
        return fail(SVL_ERR_INVALID_ARGUMENT, "salience mode does not match the summary-token count%s");
    if (d_e < 8 || d_e > 128 || d_e % 8) return fail(SVL_ERR_UNSUPPORTED, "d_e must be a multiple of 8 in [8, 128]%s");
    if (!(scale > 0.f) || !isfinite(scale)) return fail(SVL_ERR_INVALID_ARGUMENT, "scale must be finite > 0%s");
    if (!aligned16(Qe) || !aligned16(Ke)) return fail(SVL_ERR_ALIGNMENT, "Qe/Ke not 16-byte aligned%s");
    if (!ws || !aligned16(ws)) return fail(SVL_ERR_WORKSPACE, "workspace NULL or misaligned%s");
    if (ws_bytes < svl_salience_workspace_size(F, S, N_f, H_e, d_e, mode))
        return fail(SVL_ERR_WORKSPACE, "workspace too small%s");
    svl_status st = check_device();
    if (st != SVL_OK) return st;
    const int rows = (mode == SVL_SAL_INTRA_VISUAL) ? N_f : S;
    uint8_t* w = static_cast<uint8_t*>(ws);
    SalienceParams p;
    p.Qe = static_cast<const uint16_t*>(Qe);
    p.Ke = static_cast<const uint16_t*>(Ke);
    p.F = F; p.S = S; p.Nf = N_f; p.He = H_e; p.de = d_e; p.mode = mode;
    p.scale2 = scale * kLog2e;
    p.lse = reinterpret_cast<float*>(w + kWsHeader);
    p.acc = reinterpret_cast<float*>(w + round_up(kWsHeader + (size_t)F * H_e * std::max(rows, 1) * sizeof(float), 256));
    p.sal = saliency;
    p.flags = reinterpret_cast<uint32_t*>(w);
    // INTRA_VISUAL with no summary rows and frames of <= 512 tokens: the tcgen05 kernel
    // ([F][T][H_e][d_e] as 4-D {d_e, T, H_e, F} tensor maps); otherwise the mma.sync passes
    const int64_t T = (int64_t)S + N_f;
    p.use_tc = (mode == SVL_SAL_INTRA_VISUAL && S == 0 && N_f <= 512 && d_e % 8 == 0 &&
                encode_kv_tensor_map(&p.qmap, Qe, d_e, (int)T, H_e, F, T * H_e * d_e, d_e, (int64_t)H_e * d_e, 128) &&
                encode_kv_tensor_map(&p.kmap, Ke, d_e, (int)T, H_e, F, T * H_e * d_e, d_e, (int64_t)H_e * d_e, 128))
                   ? 1 : 0;
    cudaError_t e = launch_salience(p, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "svl_salience");
    return SVL_OK;
}

}  // extern "C"
