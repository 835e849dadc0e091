// fp8_kernels.cu — NEXT-1: per-channel FP8 E4M3 variant of a3/a4
// (the paper's future-work FP8 format; reading Q17 in DESIGN.md §3):
//   s_d  = max_t |K[t,d]| / 448                        (kvq_compute_scales_fmt)
//   code = E4M3_RN_satfinite(fl32(K[t,d] / s_d)),  0 where s_d == 0
//   K_hat = fl32(decode(code) * s_d)
// Same column-owning streaming geometry as quant_kernels.cu; the quotient is the
// IEEE division (__fdiv_rn) and the conversion is the sm_100 hardware
// cvt.rn.satfinite.e4m3x2.f32 (round-to-nearest-even, saturating to +-448), the
// decode cvt.rn.f16x2.e4m3x2 (exact: E4M3 is a subset of fp16).
#include <cuda_fp16.h>

#include <algorithm>

#include "device_common.cuh"
#include "kvq_internal.h"

namespace kvq {

// two fp32 -> two E4M3 codes; lo -> byte 0, hi -> byte 1
__device__ __forceinline__ uint32_t e4m3x2(float lo, float hi) {
    uint16_t r;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
    return r;
}
// two E4M3 codes (bytes 0, 1 of v) -> two exact fp32
__device__ __forceinline__ float2 e4m3x2_decode(uint16_t v) {
    uint32_t h2;
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(v));
    const __half2 hh = *reinterpret_cast<const __half2 *>(&h2);
    return make_float2(__low2float(hh), __high2float(hh));
}

__device__ __forceinline__ float fp8_quot(float x, float s) { return s == 0.0f ? 0.0f : __fdiv_rn(x, s); }

template <int U, bool FUSED>
__global__ void __launch_bounds__(kThreads) e4m3_quant_v4_kernel(const float4 *__restrict__ K,
                                                                 const float *__restrict__ scales,
                                                                 uint32_t *__restrict__ Kq4, float4 *__restrict__ Kh4,
                                                                 int64_t n4, int64_t cols4, int64_t G) {
    const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (g >= G) return;
    const int64_t c4 = g % cols4;
    const float s0 = __ldg(scales + 4 * c4 + 0), s1 = __ldg(scales + 4 * c4 + 1);
    const float s2 = __ldg(scales + 4 * c4 + 2), s3 = __ldg(scales + 4 * c4 + 3);
    for (int64_t i = g; i < n4; i += U * G) {
        float4 v[U];
#pragma unroll
        for (int k = 0; k < U; k++)
            if (i + k * G < n4) v[k] = ld_stream_f4(K + i + k * G);
#pragma unroll
        for (int k = 0; k < U; k++) {
            const int64_t idx = i + k * G;
            if (idx < n4) {
                const uint32_t c01 = e4m3x2(fp8_quot(v[k].x, s0), fp8_quot(v[k].y, s1));
                const uint32_t c23 = e4m3x2(fp8_quot(v[k].z, s2), fp8_quot(v[k].w, s3));
                st_cs_u32(Kq4 + idx, c01 | (c23 << 16));
                if (FUSED) {
                    const float2 a = e4m3x2_decode((uint16_t)c01), b = e4m3x2_decode((uint16_t)c23);
                    st_cs_f4(Kh4 + idx, make_float4(__fmul_rn(a.x, s0), __fmul_rn(a.y, s1), __fmul_rn(b.x, s2),
                                                    __fmul_rn(b.y, s3)));
                }
            }
        }
    }
}

template <bool FUSED>
__global__ void __launch_bounds__(kThreads) e4m3_quant_scalar_kernel(const float *__restrict__ K,
                                                                     const float *__restrict__ scales,
                                                                     uint8_t *__restrict__ Kq, float *__restrict__ Kh,
                                                                     int64_t n, int64_t D, int64_t G) {
    const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (g >= G) return;
    const float s = __ldg(scales + g % D);
    for (int64_t i = g; i < n; i += G) {
        const uint32_t c = e4m3x2(fp8_quot(__ldg(K + i), s), 0.0f) & 0xffu;
        Kq[i] = (uint8_t)c;
        if (FUSED) Kh[i] = __fmul_rn(e4m3x2_decode((uint16_t)c).x, s);
    }
}

template <int U>
__global__ void __launch_bounds__(kThreads) e4m3_dequant_v4_kernel(const uint32_t *__restrict__ Kq4,
                                                                   const float *__restrict__ scales,
                                                                   float4 *__restrict__ Kh4, int64_t n4,
                                                                   int64_t cols4, int64_t G) {
    const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (g >= G) return;
    const int64_t c4 = g % cols4;
    const float s0 = __ldg(scales + 4 * c4 + 0), s1 = __ldg(scales + 4 * c4 + 1);
    const float s2 = __ldg(scales + 4 * c4 + 2), s3 = __ldg(scales + 4 * c4 + 3);
    for (int64_t i = g; i < n4; i += U * G) {
        uint32_t w[U];
#pragma unroll
        for (int k = 0; k < U; k++)
            if (i + k * G < n4) w[k] = ld_stream_u32(Kq4 + i + k * G);
#pragma unroll
        for (int k = 0; k < U; k++) {
            const int64_t idx = i + k * G;
            if (idx < n4) {
                const float2 a = e4m3x2_decode((uint16_t)(w[k] & 0xffffu));
                const float2 b = e4m3x2_decode((uint16_t)(w[k] >> 16));
                st_cs_f4(Kh4 + idx, make_float4(__fmul_rn(a.x, s0), __fmul_rn(a.y, s1), __fmul_rn(b.x, s2),
                                                __fmul_rn(b.y, s3)));
            }
        }
    }
}

__global__ void __launch_bounds__(kThreads) e4m3_dequant_scalar_kernel(const uint8_t *__restrict__ Kq,
                                                                       const float *__restrict__ scales,
                                                                       float *__restrict__ Kh, int64_t n, int64_t D,
                                                                       int64_t G) {
    const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (g >= G) return;
    const float s = __ldg(scales + g % D);
    for (int64_t i = g; i < n; i += G) Kh[i] = __fmul_rn(e4m3x2_decode((uint16_t)Kq[i]).x, s);
}

static inline bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

template <typename Kern>
static int resident(Kern kernel) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, kThreads, 0) != cudaSuccess || nb < 1) {
        cudaGetLastError();
        nb = 1;
    }
    return nb * kThreads;
}

kvq_status launch_quantize_e4m3(const float *K, const float *scales, int64_t T, int64_t D, uint8_t *Kq,
                                float *K_hat, cudaStream_t s) {
    const int64_t n = T * D;
    if (D % 4 == 0 && aligned(K, 16) && aligned(Kq, 4) && (!K_hat || aligned(K_hat, 16))) {
        const int64_t cols4 = D / 4;
        auto K4 = reinterpret_cast<const float4 *>(K);
        auto Q4 = reinterpret_cast<uint32_t *>(Kq);
        if (K_hat) {
            static const int r = resident(e4m3_quant_v4_kernel<4, true>);
            StreamPlan p = plan_stream(T, cols4, r);
            e4m3_quant_v4_kernel<4, true><<<p.blocks, kThreads, 0, s>>>(K4, scales, Q4,
                                                                        reinterpret_cast<float4 *>(K_hat), n / 4,
                                                                        cols4, p.G);
        } else {
            static const int r = resident(e4m3_quant_v4_kernel<4, false>);
            StreamPlan p = plan_stream(T, cols4, r);
            e4m3_quant_v4_kernel<4, false><<<p.blocks, kThreads, 0, s>>>(K4, scales, Q4, nullptr, n / 4, cols4, p.G);
        }
    } else {
        static const int r = resident(e4m3_quant_scalar_kernel<true>);
        StreamPlan p = plan_stream(T, D, r);
        if (K_hat)
            e4m3_quant_scalar_kernel<true><<<p.blocks, kThreads, 0, s>>>(K, scales, Kq, K_hat, n, D, p.G);
        else
            e4m3_quant_scalar_kernel<false><<<p.blocks, kThreads, 0, s>>>(K, scales, Kq, nullptr, n, D, p.G);
    }
    return check_launch("quantize_e4m3");
}

kvq_status launch_dequantize_e4m3(const uint8_t *Kq, const float *scales, int64_t T, int64_t D, float *K_hat,
                                  cudaStream_t s) {
    const int64_t n = T * D;
    if (D % 4 == 0 && aligned(Kq, 4) && aligned(K_hat, 16)) {
        const int64_t cols4 = D / 4;
        static const int r = resident(e4m3_dequant_v4_kernel<8>);
        StreamPlan p = plan_stream(T, cols4, r);
        e4m3_dequant_v4_kernel<8><<<p.blocks, kThreads, 0, s>>>(reinterpret_cast<const uint32_t *>(Kq), scales,
                                                                reinterpret_cast<float4 *>(K_hat), n / 4, cols4, p.G);
    } else {
        static const int r = resident(e4m3_dequant_scalar_kernel);
        StreamPlan p = plan_stream(T, D, r);
        e4m3_dequant_scalar_kernel<<<p.blocks, kThreads, 0, s>>>(Kq, scales, K_hat, n, D, p.G);
    }
    return check_launch("dequantize_e4m3");
}

}  // namespace kvq
