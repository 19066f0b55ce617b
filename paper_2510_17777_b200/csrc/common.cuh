// common.cuh -- sm_100a PTX helpers shared by the libsparsevila kernels.
// (Product code: nothing here is shared with oracle/.)
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define SVL_DEV __device__ __forceinline__

namespace svl {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// ------------------------------------------------------------------ loads
// Streaming 128-bit load: read-only path, no L1 allocation, L2 evict-first
// (the K stream is touched once; keep L2 for the logit scratch).
SVL_DEV uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
SVL_DEV uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

SVL_DEV uint4 ldg_stream(const void* ptr, uint64_t pol) {
    uint4 r;
    asm volatile(
        "ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(ptr), "l"(pol));
    return r;
}

SVL_DEV void stg_hint_f2(float* ptr, float a, float b, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1,%2}, %3;" ::"l"(ptr), "f"(a), "f"(b),
                 "l"(pol)
                 : "memory");
}

// ---------------------------------------------------------------- cp.async
SVL_DEV uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
SVL_DEV void cp_async16(uint32_t dst, const void* src, bool valid) {
    // src-size 0 => the 16 destination bytes are zero-filled (masked rows)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
SVL_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
SVL_DEV void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ------------------------------------------------------- mbarrier + TMA bulk
SVL_DEV void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
SVL_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
SVL_DEV void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
SVL_DEV void mbar_expect_tx(uint32_t bar, uint32_t bytes) {  // no arrival
    asm volatile("mbarrier.expect_tx.shared.b64 [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
SVL_DEV void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"(bar) : "memory");
}
SVL_DEV void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`.
SVL_DEV void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

// ------------------------------------------------------------ tensor core
// D = A(16x16 bf16, row) * B(16x8 bf16, col) + C, fp32 accumulate.
SVL_DEV void mma_bf16_16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 "
        "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

SVL_DEV void ldsm_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                           uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}

SVL_DEV uint4 lds128(uint32_t addr) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"(addr));
    return r;
}

SVL_DEV uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
SVL_DEV float bf16lo(uint32_t v) { return __uint_as_float(v << 16); }
SVL_DEV float bf16hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

SVL_DEV float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Order-preserving float -> uint32 key (larger float => larger key).
// -0.0 is canonicalised to +0.0; NaN maps to 0 (ranks lowest, reading A8).
SVL_DEV uint32_t float_key(float f, bool& nonfinite_nan) {
    if (f != f) {
        nonfinite_nan = true;
        return 0u;
    }
    if (f == 0.0f) f = 0.0f;
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// ------------------------------------------------------------------ flags
// Workspace header: word 0 = device flag word (SVL_DEVFLAG_*).
constexpr size_t kWsHeader = 256;
SVL_DEV void raise_flag(uint32_t* ws_flags, uint32_t bit) { atomicOr(ws_flags, bit); }

}  // namespace svl
