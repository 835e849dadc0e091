// device_common.cuh — device helpers for the kvq kernels (sm_100a).
//
// Quantizer arithmetic (Eq. 7; readings Q1 half-even, Q2 fp32 IEEE
// quotient, Q4 clamp +-127, Q5 zero scale -> 0):
//
//   exact:  q = clamp(rint(fl32(x / s)), -127, 127)
//
// Fast path per element, with y = RN(1/s) computed ONCE per owned column:
//   fq = RN(x * y);  c = clamp(fq, +-127);  v = RN(c + 1.5*2^23)   (half-even rint)
//   q  = low byte of bits(v);  r = v - 1.5*2^23  (= (float)q exactly)
// Error bound (s normal, |x/s| <= 128): y = (1/s)(1+d1), fq = x*y*(1+d2),
// |d1|,|d2| <= 2^-24  =>  |fq - x/s| <= 128 * 2^-23 = 2^-16 and
// |RN(x/s) - x/s| <= 2^-18, so |fq - RN(x/s)| < 2^-15.  Whenever c is farther
// than 2^-14 (a 2x margin) from every half integer, fq and the exact quotient
// RN(x/s) lie strictly inside the same rounding interval and give the same
// code.  Otherwise ("danger", probability 2^-13 per element for uniform
// quotients) the element is recomputed with the IEEE division
// __fdiv_rn, which decides ties exactly as the oracle.  Quotients beyond
// +-127.5 clamp identically on both sides.  Subnormal scales (s < 2^-126,
// where RN(1/s) may overflow) take the exact path for the whole column.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace kvq {

constexpr float kMagic = 12582912.0f;          // 1.5 * 2^23: RN(c + kMagic) - kMagic == rint(c), |c| < 2^22
constexpr float kDangerThr = 0.5f - 0x1p-14f;  // distance to nearest integer above which we re-check
constexpr float kMinNormal = 1.17549435e-38f;  // 2^-126

struct ColQ {
    float s;     // scale
    float y;     // RN(1/s), 0 when s == 0
    bool exact;  // subnormal (or non-finite) scale: exact path for every element
};

__device__ __forceinline__ ColQ make_colq(float s) {
    ColQ c;
    c.s = s;
    if (s == 0.0f) {  // reading Q5: q = 0, K_hat = +0
        c.y = 0.0f;
        c.exact = false;
    } else if (s >= kMinNormal && s <= 3.0e38f) {
        c.y = __frcp_rn(s);  // IEEE round-to-nearest reciprocal
        c.exact = false;
    } else {
        c.y = 0.0f;
        c.exact = true;
    }
    return c;
}

// Exact reference arithmetic of the oracle (IEEE division, half-even, clamp).
static __device__ __noinline__ int quant_exact(float x, float s) {
    if (s == 0.0f) return 0;
    float v = __fdiv_rn(x, s);
    float r = rintf(v);
    r = fminf(fmaxf(r, -127.0f), 127.0f);
    return (int)r;
}

// Fast path for one element; returns v = RN(clamp(fq) + kMagic) whose low byte
// is the two's-complement code, and sets `danger` if the element must be
// recomputed exactly.
__device__ __forceinline__ float quant_fast(float x, const ColQ &c, bool &danger) {
    float fq = __fmul_rn(x, c.y);
    float cl = fminf(fmaxf(fq, -127.0f), 127.0f);
    float v = __fadd_rn(cl, kMagic);
    float r = __fsub_rn(v, kMagic);
    danger |= fabsf(__fsub_rn(cl, r)) > kDangerThr;
    return v;
}

__device__ __forceinline__ uint32_t code_byte(float v) { return __float_as_uint(v) & 0xffu; }

// Pack four codes (low bytes of four magic floats) into one uint32, byte j = element j.
__device__ __forceinline__ uint32_t pack4(float v0, float v1, float v2, float v3) {
    uint32_t a = __byte_perm(__float_as_uint(v0), __float_as_uint(v1), 0x0040);  // [v0.b0, v1.b0, 0, 0]
    uint32_t b = __byte_perm(__float_as_uint(v2), __float_as_uint(v3), 0x0040);
    return __byte_perm(a, b, 0x5410);  // a.b0 a.b1 b.b0 b.b1
}

// Streaming 128-bit load that does not allocate in L1 (read-once data).
__device__ __forceinline__ float4 ld_stream_f4(const float4 *p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}
// Same, with an L2 eviction-priority policy (createpolicy): evict-first keeps a read-once stream from pushing
// other lines (e.g. the previous pass's dirty output lines) out of the L2.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ float4 ld_stream_f4_hint(const float4 *p, uint64_t pol) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}
// The column-max streams (a1): experiments select the L2 policy (-DKVQ_COLMAX_EF: evict-first hint).
#ifdef KVQ_COLMAX_EF
#define KVQ_COLMAX_LD(ptr) ld_stream_f4_hint((ptr), l2_policy_evict_first())
#else
#define KVQ_COLMAX_LD(ptr) ld_stream_f4(ptr)
#endif
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t *p) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ uint4 ld_stream_u4(const uint4 *p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// Streaming (evict-first) stores for write-once outputs.
__device__ __forceinline__ void st_cs_f4(float4 *p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ void st_cs_u32(uint32_t *p, uint32_t v) {
    asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <int SP>
__device__ __forceinline__ void store_f4(float4 *p, float4 v) {
    if (SP) st_cs_f4(p, v); else *p = v;
}
template <int SP>
__device__ __forceinline__ void store_u32(uint32_t *p, uint32_t v) {
    if (SP) st_cs_u32(p, v); else *p = v;
}

__device__ __forceinline__ uint32_t absbits(float x) { return __float_as_uint(x) & 0x7fffffffu; }

// int8 code (as byte j of w) -> float, exact.
__device__ __forceinline__ float code_to_float(uint32_t w, int j) {
    return (float)(int)(int8_t)((w >> (8 * j)) & 0xffu);
}

// Programmatic dependent launch (kvq_internal.h launch_pdl): no-ops when launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

}  // namespace kvq
