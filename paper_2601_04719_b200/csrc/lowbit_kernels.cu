// lowbit_kernels.cu — NEXT-3: per-channel INT4 / INT2 variant of
// a3 (+a4) with packed storage (future work P:562; reading Q19 in DESIGN.md §3):
//   s_d   = max_t |K[t,d]| / qmax                 (kvq_compute_scales_fmt, qmax 7 / 1)
//   q     = clamp(rint(fl32(K[t,d] / s_d)), -qmax, qmax),  0 where s_d == 0
//   K_hat = fl32(q * s_d)
// Storage: each row on its own, ceil(D * bits / 8) bytes; column d's code, in
// bits-bit two's complement, at bits [bits*(d % per), +bits) of byte d / per
// (per = 8 / bits, low bits first); unused bits are 0.
//
// Same column-owning streaming geometry and the same provably-exact division
// as the INT8 kernels (device_common.cuh: RN(1/s) hoisted per column, a 2^-14
// danger band around half-integers recomputed with the IEEE quotient; the bound
// needs |x/s| <= 128, far above qmax).  The magic-constant rint leaves the code's
// two's complement in the low bits of the float, so a word of packed codes is
// built with shifts and ORs.  One 32-bit word = 32/bits columns per thread step:
// INT4 reads 32 B (two float4) and writes 4 B; INT2 reads 64 B and writes 4 B.
#include <algorithm>

#include "device_common.cuh"
#include "kvq_internal.h"

namespace kvq {

__device__ __forceinline__ int quant_exact_q(float x, float s, float qmax) {
    if (s == 0.0f) return 0;
    const float r = rintf(__fdiv_rn(x, s));
    return (int)fminf(fmaxf(r, -qmax), qmax);
}

template <int BITS>
struct LowBits {
    static constexpr int C = 32 / BITS;          // columns per 32-bit word
    static constexpr int PER = 8 / BITS;         // columns per byte
    static constexpr float QMAX = BITS == 4 ? 7.0f : 1.0f;
    static constexpr uint32_t MASK = (1u << BITS) - 1u;
};

// fast path: v = RN(clamp(RN(x*y), +-qmax) + 1.5*2^23) (its low bits are the code)
__device__ __forceinline__ float quant_fast_q(float x, const ColQ &c, float qmax, bool &danger) {
    const float fq = __fmul_rn(x, c.y);
    const float cl = fminf(fmaxf(fq, -qmax), qmax);
    const float v = __fadd_rn(cl, kMagic);
    const float r = __fsub_rn(v, kMagic);
    danger |= fabsf(__fsub_rn(cl, r)) > kDangerThr;
    return v;
}

template <int BITS>
__device__ __forceinline__ int code_of(uint32_t w, int k) {  // sign-extended field k of a word
    return ((int32_t)(w << (32 - BITS * (k + 1)))) >> (32 - BITS);
}

// Vector path: D % C == 0, K and K_hat 16-B aligned, Kp 4-B aligned.  Thread g
// owns word-column wc = g % W (columns C*wc .. C*wc + C-1) for the whole loop.
template <int BITS, bool FUSED>
__global__ void __launch_bounds__(kThreads) lowbit_quant_kernel(const float4 *__restrict__ K,
                                                                const float *__restrict__ scales,
                                                                uint32_t *__restrict__ Kp, float4 *__restrict__ Kh,
                                                                int64_t nwords, int64_t W, int64_t G) {
    using LB = LowBits<BITS>;
    constexpr int C = LB::C, V = C / 4;
    const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (g >= G) return;
    const int64_t wc = g % W;
    ColQ cq[C];
    bool col_exact = false;
#pragma unroll
    for (int k = 0; k < C; k++) {
        cq[k] = make_colq(__ldg(scales + C * wc + k));
        col_exact |= cq[k].exact;
    }
    for (int64_t i = g; i < nwords; i += G) {
        float4 x[V];
#pragma unroll
        for (int v = 0; v < V; v++) x[v] = __ldg(K + i * V + v);  // L1-allocating: the V loads of a lane share sectors
        const float *xs = reinterpret_cast<const float *>(x);
        float vv[C];
        bool danger = col_exact;
#pragma unroll
        for (int k = 0; k < C; k++) vv[k] = cq[k].s == 0.0f ? kMagic : quant_fast_q(xs[k], cq[k], LB::QMAX, danger);
        uint32_t w = 0;
        float code[C];
        if (!danger) {
#pragma unroll
            for (int k = 0; k < C; k++) {
                w |= (__float_as_uint(vv[k]) & LB::MASK) << (BITS * k);
                code[k] = __fsub_rn(vv[k], kMagic);
            }
        } else {
#pragma unroll
            for (int k = 0; k < C; k++) {
                const int q = quant_exact_q(xs[k], cq[k].s, LB::QMAX);
                w |= ((uint32_t)q & LB::MASK) << (BITS * k);
                code[k] = (float)q;
            }
        }
        st_cs_u32(Kp + i, w);
        if (FUSED) {
#pragma unroll
            for (int v = 0; v < V; v++)
                st_cs_f4(Kh + i * V + v, make_float4(__fmul_rn(code[4 * v], cq[4 * v].s),
                                                     __fmul_rn(code[4 * v + 1], cq[4 * v + 1].s),
                                                     __fmul_rn(code[4 * v + 2], cq[4 * v + 2].s),
                                                     __fmul_rn(code[4 * v + 3], cq[4 * v + 3].s)));
        }
    }
}

template <int BITS>
__global__ void __launch_bounds__(kThreads) lowbit_dequant_kernel(const uint32_t *__restrict__ Kp,
                                                                  const float *__restrict__ scales,
                                                                  float4 *__restrict__ Kh, int64_t nwords, int64_t W,
                                                                  int64_t G) {
    constexpr int C = LowBits<BITS>::C, V = C / 4;
    const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (g >= G) return;
    const int64_t wc = g % W;
    float s[C];
#pragma unroll
    for (int k = 0; k < C; k++) s[k] = __ldg(scales + C * wc + k);
    for (int64_t i = g; i < nwords; i += G) {
        const uint32_t w = ld_stream_u32(Kp + i);
#pragma unroll
        for (int v = 0; v < V; v++)
            st_cs_f4(Kh + i * V + v, make_float4(__fmul_rn((float)code_of<BITS>(w, 4 * v), s[4 * v]),
                                                 __fmul_rn((float)code_of<BITS>(w, 4 * v + 1), s[4 * v + 1]),
                                                 __fmul_rn((float)code_of<BITS>(w, 4 * v + 2), s[4 * v + 2]),
                                                 __fmul_rn((float)code_of<BITS>(w, 4 * v + 3), s[4 * v + 3])));
    }
}

// Scalar path (any D, any alignment): one thread per packed byte, IEEE division.
template <int BITS>
__global__ void lowbit_quant_scalar_kernel(const float *__restrict__ K, const float *__restrict__ scales,
                                           uint8_t *__restrict__ Kp, float *__restrict__ Kh, int64_t T, int64_t D,
                                           int64_t rb) {
    using LB = LowBits<BITS>;
    const int64_t n = T * rb;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = o / rb, j = o % rb;
        uint32_t byte = 0;
#pragma unroll
        for (int k = 0; k < LB::PER; k++) {
            const int64_t d = j * LB::PER + k;
            if (d < D) {
                const float s = scales[d];
                const int q = quant_exact_q(K[t * D + d], s, LB::QMAX);
                byte |= ((uint32_t)q & LB::MASK) << (BITS * k);
                if (Kh) Kh[t * D + d] = __fmul_rn((float)q, s);
            }
        }
        Kp[o] = (uint8_t)byte;
    }
}

template <int BITS>
__global__ void lowbit_dequant_scalar_kernel(const uint8_t *__restrict__ Kp, const float *__restrict__ scales,
                                             float *__restrict__ Kh, int64_t T, int64_t D, int64_t rb) {
    using LB = LowBits<BITS>;
    const int64_t n = T * D;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < n; o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = o / D, d = o % D;
        const uint32_t byte = Kp[t * rb + d / LB::PER];
        const int q = code_of<BITS>(byte << (32 - 8), (int)(d % LB::PER) + (32 - 8) / BITS);
        Kh[o] = __fmul_rn((float)q, scales[d]);
    }
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

int64_t packed_row_bytes(int64_t D, int bits) {
    if (bits != 4 && bits != 2) return -1;
    const int64_t per = 8 / bits;
    return (D + per - 1) / per;
}

template <int BITS>
static kvq_status quant_bits(const float *K, const float *scales, int64_t T, int64_t D, uint8_t *Kp, float *K_hat,
                             cudaStream_t s) {
    constexpr int C = LowBits<BITS>::C;
    const int64_t rb = packed_row_bytes(D, BITS);
    if (D % C == 0 && aligned(K, 16) && aligned(Kp, 4) && (!K_hat || aligned(K_hat, 16))) {
        const int64_t W = D / C, nwords = T * W;
        auto K4 = reinterpret_cast<const float4 *>(K);
        auto P4 = reinterpret_cast<uint32_t *>(Kp);
        if (K_hat) {
            static const int r = resident(lowbit_quant_kernel<BITS, true>);
            const StreamPlan p = plan_stream(T, W, r);
            lowbit_quant_kernel<BITS, true><<<p.blocks, kThreads, 0, s>>>(K4, scales, P4,
                                                                          reinterpret_cast<float4 *>(K_hat), nwords,
                                                                          W, p.G);
        } else {
            static const int r = resident(lowbit_quant_kernel<BITS, false>);
            const StreamPlan p = plan_stream(T, W, r);
            lowbit_quant_kernel<BITS, false><<<p.blocks, kThreads, 0, s>>>(K4, scales, P4, nullptr, nwords, W, p.G);
        }
    } else {
        const int64_t n = T * rb;
        lowbit_quant_scalar_kernel<BITS><<<(unsigned)std::min<int64_t>((n + 255) / 256, 16384), 256, 0, s>>>(
            K, scales, Kp, K_hat, T, D, rb);
    }
    return check_launch("quantize_packed");
}

template <int BITS>
static kvq_status dequant_bits(const uint8_t *Kp, const float *scales, int64_t T, int64_t D, float *K_hat,
                               cudaStream_t s) {
    constexpr int C = LowBits<BITS>::C;
    const int64_t rb = packed_row_bytes(D, BITS);
    if (D % C == 0 && aligned(Kp, 4) && aligned(K_hat, 16)) {
        const int64_t W = D / C, nwords = T * W;
        static const int r = resident(lowbit_dequant_kernel<BITS>);
        const StreamPlan p = plan_stream(T, W, r);
        lowbit_dequant_kernel<BITS><<<p.blocks, kThreads, 0, s>>>(reinterpret_cast<const uint32_t *>(Kp), scales,
                                                                  reinterpret_cast<float4 *>(K_hat), nwords, W, p.G);
    } else {
        const int64_t n = T * D;
        lowbit_dequant_scalar_kernel<BITS><<<(unsigned)std::min<int64_t>((n + 255) / 256, 16384), 256, 0, s>>>(
            Kp, scales, K_hat, T, D, rb);
    }
    return check_launch("dequantize_packed");
}

kvq_status launch_quantize_packed(const float *K, const float *scales, int64_t T, int64_t D, int bits, uint8_t *Kp,
                                  float *K_hat, cudaStream_t s) {
    return bits == 4 ? quant_bits<4>(K, scales, T, D, Kp, K_hat, s) : quant_bits<2>(K, scales, T, D, Kp, K_hat, s);
}

kvq_status launch_dequantize_packed(const uint8_t *Kp, const float *scales, int64_t T, int64_t D, int bits,
                                    float *K_hat, cudaStream_t s) {
    return bits == 4 ? dequant_bits<4>(Kp, scales, T, D, K_hat, s) : dequant_bits<2>(Kp, scales, T, D, K_hat, s);
}

}  // namespace kvq
