// salience.cu -- query-agnostic encoder-attention salience.
//
// PAPER.md:113 (three salience definitions) and PAPER.md:116: "streams
// softmax normalization and salience accumulation without explicitly forming
// the full attention matrix".  Two streaming passes per (frame f, head h),
// reading A15 (one column accumulator cannot be rescaled by many rows' running
// maxima, so the row normaliser is computed first):
//   pass 1  row_lse_kernel : LSE2[i] = log2 sum_j exp2(s2[i,j]) over all S+N_f
//                            columns, for the rows whose attention is read
//                            (the S summary rows, or all N_f rows);
//   pass 2  col_sum_kernel : acc[j] = sum_i exp2(s2[i,j] - LSE2[i]) for visual
//                            columns j, each CTA owning a column block (no
//                            atomics, fixed order);
//   final   finalize_kernel: sal[j] = (1/H_e) sum_h acc_h[j] / n_rows.
// s2 = scale*log2(e) * q.k from mma.sync m16n8k16 with the same permuted-
// contraction register layout as the retrieval kernel; K / Q tiles are staged
// in shared memory with a 64-byte row skew (conflict-free 128-bit reads).
// Memory is O(rows + N) per (f, h) -- never O(N^2).
#include "common.cuh"
#include "kernels.h"

namespace svl {

namespace {

constexpr int NTHS = 128;  // 4 warps x 16 rows
constexpr int TILE = 64;   // streamed tile (rows of the N operand)
constexpr int NCHMAX = 4;  // d_e <= 128 -> 4 chunks per thread

struct SalGeom {
    int T, rows, dep, nch, row_bytes;  // dep = d_e padded to a multiple of 32
};

SVL_DEV SalGeom geom(const SalienceParams& p) {
    SalGeom g;
    g.T = p.S + p.Nf;
    g.rows = (p.mode == 2) ? p.Nf : p.S;
    g.dep = (p.de + 31) / 32 * 32;
    g.nch = g.dep / 32;
    int rb = g.dep * 2;
    if (rb % 128 != 64) rb += 64;  // skew so that consecutive rows differ by 4 bank groups
    g.row_bytes = rb;
    return g;
}

// load 16-row A fragments (rows r0+gid, r0+gid+8) from global, permuted layout
SVL_DEV void load_rows_frag(const uint16_t* base, int64_t row_stride, int r0, int nrows, int de,
                            int nch, int gid, int t, uint4 (&ra)[NCHMAX], uint4 (&rb)[NCHMAX]) {
#pragma unroll
    for (int i = 0; i < NCHMAX; ++i) {
        ra[i] = rb[i] = make_uint4(0, 0, 0, 0);
        const int c = t + 4 * i;
        if (i < nch && c * 8 < de) {
            if (r0 + gid < nrows) ra[i] = *reinterpret_cast<const uint4*>(base + (int64_t)(r0 + gid) * row_stride + c * 8);
            if (r0 + gid + 8 < nrows) rb[i] = *reinterpret_cast<const uint4*>(base + (int64_t)(r0 + gid + 8) * row_stride + c * 8);
        }
    }
}

// stage `n` rows (starting at global row r0) of a [rows][He*de] operand into smem
SVL_DEV void stage_tile(uint32_t sdst, const uint16_t* base, int64_t row_stride, int r0, int n,
                        const SalGeom& g, int de) {
    const int CH = g.dep / 8;
    for (int i = threadIdx.x; i < TILE * CH; i += NTHS) {
        const int r = i / CH, c = i % CH;
        const bool valid = (r < n) && (c * 8 < de);
        const uint16_t* src = base + (int64_t)(valid ? r0 + r : 0) * row_stride + (valid ? c * 8 : 0);
        cp_async16(sdst + r * g.row_bytes + c * 16, src, valid);
    }
    cp_async_commit();
}

// 16 x 64 tile of s = A B^T (A rows in registers, B rows in smem)
SVL_DEV void tile_mma(float (&acc)[8][4], const uint4 (&ra)[NCHMAX], const uint4 (&rb)[NCHMAX],
                      uint32_t sB, const SalGeom& g, int gid, int t) {
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
        acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
        const int r = nt * 8 + gid;
#pragma unroll
        for (int i = 0; i < NCHMAX; ++i) {
            if (i < g.nch) {
                const uint4 kc = lds128(sB + r * g.row_bytes + (t + 4 * i) * 16);
                const uint32_t a0[4] = {ra[i].x, rb[i].x, ra[i].y, rb[i].y};
                mma_bf16_16816(acc[nt], a0, kc.x, kc.y);
                const uint32_t a1[4] = {ra[i].z, rb[i].z, ra[i].w, rb[i].w};
                mma_bf16_16816(acc[nt], a1, kc.z, kc.w);
            }
        }
    }
}

// pass 1: grid (ceil(rows/64), He, F)
__global__ void __launch_bounds__(NTHS) row_lse_kernel(const SalienceParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    const SalGeom g = geom(p);
    const int f = blockIdx.z, h = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gid = lane >> 2, t = lane & 3;
    const int64_t rs = (int64_t)p.He * p.de;
    const uint16_t* Qf = p.Qe + (int64_t)f * g.T * rs + (int64_t)h * p.de;
    const uint16_t* Kf = p.Ke + (int64_t)f * g.T * rs + (int64_t)h * p.de;
    const int r0 = blockIdx.x * 64 + warp * 16;  // query rows are rows 0..rows-1 of the frame
    uint4 ra[NCHMAX], rb[NCHMAX];
    load_rows_frag(Qf, rs, r0, g.rows, p.de, g.nch, gid, t, ra, rb);
    float ma = -INFINITY, mb = -INFINITY, la = 0.f, lb = 0.f;
    const uint32_t s0 = smem_u32(smem), s1 = s0 + TILE * g.row_bytes;
    const int ntile = (g.T + TILE - 1) / TILE;
    stage_tile(s0, Kf, rs, 0, min(TILE, g.T), g, p.de);
    for (int it = 0; it < ntile; ++it) {
        const uint32_t cur = (it & 1) ? s1 : s0, nxt = (it & 1) ? s0 : s1;
        if (it + 1 < ntile) stage_tile(nxt, Kf, rs, (it + 1) * TILE, min(TILE, g.T - (it + 1) * TILE), g, p.de);
        else cp_async_commit();
        cp_async_wait<1>();
        cta_sync();
        float acc[8][4];
        tile_mma(acc, ra, rb, cur, g, gid, t);
        float xa = -INFINITY, xb = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int col = it * TILE + nt * 8 + 2 * t + (e & 1);
                acc[nt][e] = (col < g.T) ? acc[nt][e] * p.scale2 : -INFINITY;
                if (e < 2) xa = fmaxf(xa, acc[nt][e]);
                else xb = fmaxf(xb, acc[nt][e]);
            }
        xa = fmaxf(xa, __shfl_xor_sync(0xffffffffu, xa, 1));
        xa = fmaxf(xa, __shfl_xor_sync(0xffffffffu, xa, 2));
        xb = fmaxf(xb, __shfl_xor_sync(0xffffffffu, xb, 1));
        xb = fmaxf(xb, __shfl_xor_sync(0xffffffffu, xb, 2));
        const float na = fmaxf(ma, xa), nb = fmaxf(mb, xb);
        float sa = 0.f, sb = 0.f;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
            sa += exp2f(acc[nt][0] - na) + exp2f(acc[nt][1] - na);
            sb += exp2f(acc[nt][2] - nb) + exp2f(acc[nt][3] - nb);
        }
        la = la * exp2f(ma - na) + sa;
        lb = lb * exp2f(mb - nb) + sb;
        ma = na;
        mb = nb;
        cta_sync();
    }
    la += __shfl_xor_sync(0xffffffffu, la, 1);
    la += __shfl_xor_sync(0xffffffffu, la, 2);
    lb += __shfl_xor_sync(0xffffffffu, lb, 1);
    lb += __shfl_xor_sync(0xffffffffu, lb, 2);
    if (t == 0) {
        float* lse = p.lse + ((int64_t)f * p.He + h) * g.rows;
        if (r0 + gid < g.rows) lse[r0 + gid] = ma + log2f(la);
        if (r0 + gid + 8 < g.rows) lse[r0 + gid + 8] = mb + log2f(lb);
    }
}

// pass 2: grid (ceil(Nf/64), He, F); warp owns 16 visual columns (A = K rows)
__global__ void __launch_bounds__(NTHS) col_sum_kernel(const SalienceParams p) {
    extern __shared__ __align__(128) uint8_t smem[];
    const SalGeom g = geom(p);
    const int f = blockIdx.z, h = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gid = lane >> 2, t = lane & 3;
    const int64_t rs = (int64_t)p.He * p.de;
    const uint16_t* Qf = p.Qe + (int64_t)f * g.T * rs + (int64_t)h * p.de;
    const uint16_t* Kv = p.Ke + ((int64_t)f * g.T + p.S) * rs + (int64_t)h * p.de;  // visual columns
    const float* lse = p.lse + ((int64_t)f * p.He + h) * g.rows;
    const int c0 = blockIdx.x * 64 + warp * 16;
    uint4 ra[NCHMAX], rb[NCHMAX];
    load_rows_frag(Kv, rs, c0, p.Nf, p.de, g.nch, gid, t, ra, rb);
    float* slse = reinterpret_cast<float*>(smem + 2 * TILE * g.row_bytes);  // [2][TILE]
    float suma = 0.f, sumb = 0.f;
    const uint32_t s0 = smem_u32(smem), s1 = s0 + TILE * g.row_bytes;
    const int ntile = (g.rows + TILE - 1) / TILE;
    stage_tile(s0, Qf, rs, 0, min(TILE, g.rows), g, p.de);
    if (threadIdx.x < TILE) slse[threadIdx.x] = (threadIdx.x < g.rows) ? lse[threadIdx.x] : INFINITY;
    for (int it = 0; it < ntile; ++it) {
        const uint32_t cur = (it & 1) ? s1 : s0, nxt = (it & 1) ? s0 : s1;
        const int nrow = (it + 1) * TILE;
        if (it + 1 < ntile) {
            stage_tile(nxt, Qf, rs, nrow, min(TILE, g.rows - nrow), g, p.de);
            if (threadIdx.x < TILE)
                slse[((it + 1) & 1) * TILE + threadIdx.x] = (nrow + threadIdx.x < g.rows) ? lse[nrow + threadIdx.x] : INFINITY;
        } else {
            cp_async_commit();
        }
        cp_async_wait<1>();
        cta_sync();
        float acc[8][4];
        tile_mma(acc, ra, rb, cur, g, gid, t);  // acc[nt]: (col gid/gid+8, rows nt*8+2t..)
        const float* L2 = slse + (it & 1) * TILE;
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) {
            const float l0 = L2[nt * 8 + 2 * t], l1 = L2[nt * 8 + 2 * t + 1];
            suma += exp2f(acc[nt][0] * p.scale2 - l0) + exp2f(acc[nt][1] * p.scale2 - l1);
            sumb += exp2f(acc[nt][2] * p.scale2 - l0) + exp2f(acc[nt][3] * p.scale2 - l1);
        }
        cta_sync();
    }
    suma += __shfl_xor_sync(0xffffffffu, suma, 1);
    suma += __shfl_xor_sync(0xffffffffu, suma, 2);
    sumb += __shfl_xor_sync(0xffffffffu, sumb, 1);
    sumb += __shfl_xor_sync(0xffffffffu, sumb, 2);
    if (t == 0) {
        float* acc = p.acc + ((int64_t)f * p.He + h) * p.Nf;
        if (c0 + gid < p.Nf) acc[c0 + gid] = suma;
        if (c0 + gid + 8 < p.Nf) acc[c0 + gid + 8] = sumb;
    }
}

__global__ void finalize_kernel(const SalienceParams p) {
    const int f = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= p.Nf) return;
    const int rows = (p.mode == 2) ? p.Nf : p.S;
    float s = 0.f;
    for (int h = 0; h < p.He; ++h) s += p.acc[((int64_t)f * p.He + h) * p.Nf + j] / (float)rows;
    const float v = s / (float)p.He;
    if (!(v == v)) raise_flag(p.flags, 2u /*NONFINITE*/);
    p.sal[(int64_t)f * p.Nf + j] = v;
}

}  // namespace

cudaError_t launch_salience(const SalienceParams& p, cudaStream_t s) {
    if (salience_tc_eligible(p)) {  // INTRA_VISUAL on tcgen05 (salience_tc.cu)
        cudaError_t e = launch_salience_tc(p, s);
        if (e != cudaSuccess) return e;
        finalize_kernel<<<dim3((p.Nf + 127) / 128, p.F), 128, 0, s>>>(p);
        return cudaGetLastError();
    }
    const int dep = (p.de + 31) / 32 * 32;
    int rb = dep * 2;
    if (rb % 128 != 64) rb += 64;
    const size_t sm1 = 2 * TILE * rb;
    const size_t sm2 = sm1 + 2 * TILE * sizeof(float);
    static bool attr_done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_done[dev]) {
        cudaError_t e = cudaFuncSetAttribute(row_lse_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * TILE * 320);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(col_sum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * TILE * 320 + 2 * TILE * 4);
        if (e != cudaSuccess) return e;
        attr_done[dev] = true;
    }
    const int rows = (p.mode == 2) ? p.Nf : p.S;
    row_lse_kernel<<<dim3((rows + 63) / 64, p.He, p.F), NTHS, sm1, s>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    col_sum_kernel<<<dim3((p.Nf + 63) / 64, p.He, p.F), NTHS, sm2, s>>>(p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    finalize_kernel<<<dim3((p.Nf + 127) / 128, p.F), 128, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace svl
