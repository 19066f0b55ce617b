// salience_tc.cu -- INTRA_VISUAL encoder salience on the 5th-generation tensor
// cores.
//
// For a frame f and encoder head h (S = 0 summary rows, N_f <= 512 tokens):
//   P = softmax_rows(scale * Q K^T)    (N_f x N_f, never written to memory)
//   acc[f][h][j] = sum_i P[i, j]        (the column mass; finalize_kernel then
//                                        takes mean_h acc / N_f -> saliency)
// One persistent CTA per SM walks the (f, h) items.  Per item, K (N_f x d_e,
// bf16) is loaded once by tiled TMA (4-D tensor map, 128-B swizzle, two 64-column
// boxes; columns past d_e are zero-filled) and every 128-row block of Q (double
// buffered, prefetched while the previous block is post-processed) is
// multiplied by it with tcgen05.mma (M = 128 query rows, N = 256 key columns,
// K = 16): S = Q_blk K^T lands in TMEM, all 512 columns.  The 4 warps then own
// one TMEM lane quarter each (thread = query row i):
//   pass 1  m_i = max_j S[i, j]                          (tcgen05.ld, x32 chunks)
//   pass 2  e = exp2((S - m_i) * scale * log2 e), l_i = sum_j e; e written back
//           to TMEM (one exponential per element)
//   pass 3  P = e / l_i; column sums over the warp's 32 rows by a 31-shuffle
//           butterfly per 32-column chunk; the 4 warps' partials are summed in
//           a fixed order (deterministic).
// S is computed once (not twice as the two-pass streaming kernels do), and the
// exponentials, not the tensor core, bound the kernel at d_e = 72: 2 d_e = 144
// flop per element vs ~16 exp2 per clock per SM.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace svl {

namespace {

constexpr int TC_NT = 512;    // 16 warps; warp w reads TMEM lanes [32 (w % 4), +32), column chunks c = w / 4 (mod 4)
constexpr int TC_NMAX = 512;  // key columns held in TMEM
constexpr int TC_ROWS = 128;  // query rows per MMA block (UMMA M)

struct TcSmem {
    static constexpr int K_OFF = 0;                            // [2 col boxes][512 rows][128 B]
    static constexpr int K_BYTES = 2 * TC_NMAX * 128;          // 128 KB
    static constexpr int Q_OFF = K_OFF + K_BYTES;              // [2 bufs][2 col boxes][128 rows][128 B]
    static constexpr int Q_BUF = 2 * TC_ROWS * 128;            // 32 KB
    static constexpr int CP_OFF = Q_OFF + 2 * Q_BUF;           // column partials [4 warps][512] fp32
    static constexpr int RED_OFF = CP_OFF + 4 * TC_NMAX * 4;   // row (max, sum) exchange [2][4 col groups][128 rows]
    static constexpr int BAR_OFF = RED_OFF + 8 * TC_ROWS * 4;   // kfull, qfull[2], mdone, tslot
    static constexpr int BYTES = BAR_OFF + 64;
};

__global__ void __launch_bounds__(TC_NT, 1) salience_tc_kernel(const __grid_constant__ SalienceParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int q4 = warp & 3, cg = warp >> 2;  // TMEM lane quarter, column group
    float* cpart = reinterpret_cast<float*>(smem + TcSmem::CP_OFF);
    float* red = reinterpret_cast<float*>(smem + TcSmem::RED_OFF);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + TcSmem::BAR_OFF);
    const uint32_t kfull = smem_u32(bars), qfull0 = smem_u32(bars + 1), mdone = smem_u32(bars + 3);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);
    const uint32_t sK = smem_u32(smem + TcSmem::K_OFF), sQ = smem_u32(smem + TcSmem::Q_OFF);
    const int Nf = p.Nf, ncb = (p.de + 63) / 64, ks = (p.de + 15) / 16;
    const int nrb = (Nf + TC_ROWS - 1) / TC_ROWS, nkb = (Nf + 127) / 128, nnh = (Nf + 255) / 256;
    const int nch = (Nf + 31) / 32;
    constexpr uint32_t IDESC = umma_idesc_bf16(TC_ROWS, 256);

    if (tid == 0) {
        mbar_init(kfull, 1);
        mbar_init(qfull0, 1);
        mbar_init(qfull0 + 8, 1);
        mbar_init(mdone, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(smem_u32(tslot), TC_NMAX);
    for (int i = tid; i < 4 * TC_NMAX; i += TC_NT) cpart[i] = 0.f;
    tc_fence_before();
    cta_sync();
    tc_fence_after();
    const uint32_t tbase = *tslot;

    auto load_q = [&](int f, int h, int rb, int buf) {  // thread 0
        const uint32_t bar = qfull0 + 8 * buf;
        mbar_arrive_expect_tx(bar, (uint32_t)(ncb * TC_ROWS * 128));
        for (int cb = 0; cb < ncb; ++cb)
            tma_load_4d(sQ + buf * TcSmem::Q_BUF + cb * (TC_ROWS * 128), &p.qmap, cb * 64, rb * TC_ROWS, h, f, bar);
    };
    uint32_t kph = 0, mph = 0, qph[2] = {0, 0};
    const float s2 = p.scale2;
    for (int item = blockIdx.x; item < p.F * p.He; item += gridDim.x) {
        const int f = item / p.He, h = item % p.He;
        if (tid == 0) {
            // the previous item's last MMA completed (mdone waited below) -> K and Q buffers free
            mbar_arrive_expect_tx(kfull, (uint32_t)(ncb * nkb * 128 * 128));
            for (int cb = 0; cb < ncb; ++cb)
                for (int kb = 0; kb < nkb; ++kb)
                    tma_load_4d(sK + cb * (TC_NMAX * 128) + kb * (128 * 128), &p.kmap, cb * 64, kb * 128, h, f, kfull);
            load_q(f, h, 0, 0);
        }
        for (int rb = 0; rb < nrb; ++rb) {
            const int buf = rb & 1;
            if (tid == 0) {
                if (rb == 0) {
                    mbar_wait(kfull, kph);
                    kph ^= 1u;
                }
                mbar_wait(qfull0 + 8 * buf, qph[buf]);
                qph[buf] ^= 1u;
                tc_fence_after();
                for (int nh = 0; nh < nnh; ++nh)
                    for (int j = 0; j < ks; ++j) {
                        const int cb = j >> 2, kk = j & 3;
                        umma_bf16(tbase + nh * 256,
                                  sw128_desc(sQ + buf * TcSmem::Q_BUF + cb * (TC_ROWS * 128) + kk * 32),
                                  sw128_desc(sK + cb * (TC_NMAX * 128) + nh * 256 * 128 + kk * 32), IDESC,
                                  j > 0 ? 1u : 0u);
                    }
                umma_commit(mdone);
            }
            mbar_wait(mdone, mph);
            __syncwarp();  // tcgen05.ld is .aligned
            mph ^= 1u;
            tc_fence_after();
            // the MMA has consumed buffer `buf`; prefetch the next row block into the other one
            if (tid == 0 && rb + 1 < nrb) load_q(f, h, rb + 1, buf ^ 1);

            const uint32_t trow = tbase + ((uint32_t)(q4 * 32) << 16);
            const int row = q4 * 32 + lane;  // within the block
            const bool valid = rb * TC_ROWS + row < Nf;
            // pass A: e = exp2((S - m) * s2) with a running max over this warp's chunks (chunk
            // maxima kept to rescale later), written back to TMEM; running row sum.  Even
            // columns on the SFU (ex2.approx), odd ones on the FP32 pipe (poly_exp2).
            constexpr int MAXC = TC_NMAX / 32 / 4;  // chunks per warp
            float mch[MAXC];
            float m = -INFINITY, l = 0.f;
#pragma unroll
            for (int ci = 0; ci < MAXC; ++ci) {
                const int c = cg + 4 * ci;
                mch[ci] = -INFINITY;
                if (c >= nch) continue;
                uint32_t v[32];
                tmem_ld32(trow + c * 32, v);
                const bool full = c * 32 + 32 <= Nf;  // mask-free fast path
                float cm = -INFINITY;
#pragma unroll
                for (int k = 0; k < 32; ++k)
                    if (full || c * 32 + k < Nf) cm = fmaxf(cm, __uint_as_float(v[k]));
                const float mn = fmaxf(m, cm);
                if (mn != -INFINITY) l *= fast_exp2((m - mn) * s2);
                m = mn;
                mch[ci] = mn;
                const float ms = mn * s2;
                float e[32];
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    const float x = fmaf(__uint_as_float(v[k]), s2, -ms);
#ifndef SVL_SAL_POLY
#define SVL_SAL_POLY 0  // measured: alternating with the FP32-pipe polynomial is slower (issue-bound)
#endif
                    e[k] = (full || c * 32 + k < Nf) ? ((SVL_SAL_POLY && (k & 1)) ? poly_exp2(x) : fast_exp2(x)) : 0.f;
                    l += e[k];
                }
                tmem_st32(trow + c * 32, e);
            }
            tmem_wait_st();
            // combine the 4 column groups of the row: M, L
            red[cg * TC_ROWS + row] = m;
            red[(4 + cg) * TC_ROWS + row] = l;
            cta_sync();
            float M = -INFINITY;
#pragma unroll
            for (int gq = 0; gq < 4; ++gq) M = fmaxf(M, red[gq * TC_ROWS + row]);
            float L = 0.f;
#pragma unroll
            for (int gq = 0; gq < 4; ++gq) {
                const float mg = red[gq * TC_ROWS + row];
                L += (mg == -INFINITY) ? 0.f : red[(4 + gq) * TC_ROWS + row] * fast_exp2((mg - M) * s2);
            }
            cta_sync();
            const float r = (valid && L > 0.f) ? 1.f / L : 0.f;
            // pass 3: column sums of e * r over the warp's 32 rows (butterfly transpose-reduce)
#pragma unroll
            for (int ci = 0; ci < MAXC; ++ci) {
                const int c = cg + 4 * ci;
                if (c >= nch) continue;
                uint32_t v[32];
                tmem_ld32(trow + c * 32, v);
                const float rc = (mch[ci] == -INFINITY) ? 0.f : r * fast_exp2((mch[ci] - M) * s2);
                float x[32];
#pragma unroll
                for (int k = 0; k < 32; ++k) x[k] = __uint_as_float(v[k]) * rc;
#pragma unroll
                for (int sft = 16; sft >= 1; sft >>= 1) {
                    const bool up = (lane & sft) != 0;
#pragma unroll
                    for (int k = 0; k < sft; ++k) {
                        const float send = up ? x[k] : x[k + sft];
                        const float keep = up ? x[k + sft] : x[k];
                        x[k] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
                    }
                }
                cpart[q4 * TC_NMAX + c * 32 + lane] += x[0];  // column c*32 + lane, rows of quarter q4
            }
            tc_fence_before();
            cta_sync();  // TMEM reads of this block done before the next block's MMA
            tc_fence_after();
        }
        // acc[f][h][j] = sum over the 4 warps (fixed order); reset the partials
        for (int j = tid; j < Nf; j += TC_NT) {
            const float a = cpart[j] + cpart[TC_NMAX + j] + cpart[2 * TC_NMAX + j] + cpart[3 * TC_NMAX + j];
            p.acc[((int64_t)f * p.He + h) * Nf + j] = a;
        }
        cta_sync();
        for (int i = tid; i < 4 * TC_NMAX; i += TC_NT) cpart[i] = 0.f;
        cta_sync();
    }
    tc_fence_before();
    cta_sync();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tbase, TC_NMAX);
    }
}

}  // namespace

bool salience_tc_eligible(const SalienceParams& p) {
    return p.use_tc && p.mode == 2 && p.S == 0 && p.Nf >= 1 && p.Nf <= TC_NMAX && p.de <= 128;
}

cudaError_t launch_salience_tc(const SalienceParams& p, cudaStream_t s) {
    static bool attr_done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_done[dev]) {
        cudaError_t e = cudaFuncSetAttribute(salience_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             TcSmem::BYTES);
        if (e != cudaSuccess) return e;
        attr_done[dev] = true;
    }
    const int items = p.F * p.He;
    const int grid = std::min(items, device_sm_count());
    salience_tc_kernel<<<grid, TC_NT, TcSmem::BYTES, s>>>(p);
    return cudaGetLastError();
}

}  // namespace svl
