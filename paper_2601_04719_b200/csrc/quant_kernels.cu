// quant_kernels.cu — a1 column abs-max, a2 scale finalize, a3 quantize,
// a4 dequantize (and a3+a4 fused) for sm_100a.
//
// All four are HBM-streaming kernels (arithmetic intensity ~1 op/byte), so the
// design is about bytes in flight and instruction count, not tensor cores:
//  * Column-owning grid-stride loops.  The flat float4 index space of K[T][D]
//    is walked with a stride G that is a multiple of D/4, so each thread owns
//    the same 4 columns for its whole life: scales, RN(1/s) and the running
//    column max stay in registers (the paper's "coarsened" idea, P:320-347,
//    with the vectorized kernel's 128-bit accesses).
//  * U independent 128-bit loads in flight per thread (LDG.128, L1 no-allocate)
//    and ~2048 resident threads per SM: >=128 KB of loads in flight per SM,
//    well above the ~40 KB Little's-law requirement at 8 TB/s.
//  * Codes are packed four per 32-bit store (P:365-370 char4), coalesced per warp.
//  * Any D and any alignment: a scalar variant of every kernel (same geometry
//    idea with stride a multiple of D) handles D % 4 != 0 or misaligned bases,
//    which the paper's vectorized kernel leaves unwritten.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "device_common.cuh"
#include "kvq_internal.h"

namespace kvq {

// ============================================================================ a1: column abs-max
// m_d = max_t |K[t,d]| as the uint32 max of (bits & 0x7fffffff): for finite
// non-negative floats IEEE order equals integer order, and Inf/NaN propagate
// (reading Q7).  Exact under any reduction order.
template <int U>
__global__ void __launch_bounds__(kThreads) colmax_v4_kernel(const float4 *__restrict__ K, int64_t n4,
                                                             int64_t cols4, int64_t G,
                                                             uint32_t *__restrict__ mbits) {
    extern __shared__ uint32_t smax[];  // [4*cols4] when cols4 <= kThreads
    const bool share = cols4 <= kThreads;
    const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (share) {
        for (int i = threadIdx.x; i < 4 * cols4; i += kThreads) smax[i] = 0u;
        __syncthreads();
    }
    uint32_t m0 = 0, m1 = 0, m2 = 0, m3 = 0;
    int64_t c4 = 0;
    if (g < G) {
        c4 = g % cols4;
        int64_t i = g;
        for (; i + (U - 1) * G < n4; i += U * G) {
            float4 v[U];
#pragma unroll
            for (int k = 0; k < U; k++) v[k] = KVQ_COLMAX_LD(K + i + k * G);
#pragma unroll
            for (int k = 0; k < U; k++) {
                m0 = max(m0, absbits(v[k].x));
                m1 = max(m1, absbits(v[k].y));
                m2 = max(m2, absbits(v[k].z));
                m3 = max(m3, absbits(v[k].w));
            }
        }
        for (; i < n4; i += G) {
            float4 v = KVQ_COLMAX_LD(K + i);
            m0 = max(m0, absbits(v.x));
            m1 = max(m1, absbits(v.y));
            m2 = max(m2, absbits(v.z));
            m3 = max(m3, absbits(v.w));
        }
    }
    if (share) {
        if (g < G) {
            atomicMax(&smax[4 * c4 + 0], m0);
            atomicMax(&smax[4 * c4 + 1], m1);
            atomicMax(&smax[4 * c4 + 2], m2);
            atomicMax(&smax[4 * c4 + 3], m3);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < 4 * cols4; i += kThreads)
            if (smax[i]) atomicMax(&mbits[i], smax[i]);
    } else if (g < G) {
        atomicMax(&mbits[4 * c4 + 0], m0);
        atomicMax(&mbits[4 * c4 + 1], m1);
        atomicMax(&mbits[4 * c4 + 2], m2);
        atomicMax(&mbits[4 * c4 + 3], m3);
    }
}

template <int U>
__global__ void __launch_bounds__(kThreads) colmax_scalar_kernel(const float *__restrict__ K, int64_t n,
                                                                 int64_t D, int64_t G,
                                                                 uint32_t *__restrict__ mbits) {
    const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (g >= G) return;
    uint32_t m = 0;
    int64_t i = g;
    for (; i + (U - 1) * G < n; i += U * G) {
        float v[U];
#pragma unroll
        for (int k = 0; k < U; k++) v[k] = __ldg(K + i + k * G);
#pragma unroll
        for (int k = 0; k < U; k++) m = max(m, absbits(v[k]));
    }
    for (; i < n; i += G) m = max(m, absbits(__ldg(K + i)));
    if (m) atomicMax(&mbits[g % D], m);
}

// ============================================================================ a2: finalize
// s_d = fl32(m_d / 127.0f), IEEE division (reading Q3); in place.
// (divisor 448 for the E4M3 variant, reading Q17)
__global__ void finalize_kernel(uint32_t *buf, int64_t D, float divisor) {
    pdl_wait();  // the column maxima of the preceding grid
    pdl_trigger();
    for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < D; d += (int64_t)gridDim.x * blockDim.x) {
        float m = __uint_as_float(buf[d]);
        reinterpret_cast<float *>(buf)[d] = __fdiv_rn(m, divisor);
    }
}

// ============================================================================ a3 (+a4): quantize
template <bool FUSED>
__device__ __forceinline__ void quant4(const float4 &x, const ColQ &q0, const ColQ &q1, const ColQ &q2,
                                       const ColQ &q3, bool col_exact, uint32_t &w, float4 &xh) {
    bool danger = col_exact;
    float a0 = quant_fast(x.x, q0, danger);
    float a1 = quant_fast(x.y, q1, danger);
    float a2 = quant_fast(x.z, q2, danger);
    float a3 = quant_fast(x.w, q3, danger);
    if (__builtin_expect(!danger, 1)) {
        w = pack4(a0, a1, a2, a3);
        if (FUSED) {
            xh.x = __fmul_rn(__fsub_rn(a0, kMagic), q0.s);
            xh.y = __fmul_rn(__fsub_rn(a1, kMagic), q1.s);
            xh.z = __fmul_rn(__fsub_rn(a2, kMagic), q2.s);
            xh.w = __fmul_rn(__fsub_rn(a3, kMagic), q3.s);
        }
    } else {
        int c0 = quant_exact(x.x, q0.s), c1 = quant_exact(x.y, q1.s);
        int c2 = quant_exact(x.z, q2.s), c3 = quant_exact(x.w, q3.s);
        w = (uint32_t)(c0 & 0xff) | ((uint32_t)(c1 & 0xff) << 8) | ((uint32_t)(c2 & 0xff) << 16) |
            ((uint32_t)(c3 & 0xff) << 24);
        if (FUSED) {
            xh.x = __fmul_rn((float)c0, q0.s);
            xh.y = __fmul_rn((float)c1, q1.s);
            xh.z = __fmul_rn((float)c2, q2.s);
            xh.w = __fmul_rn((float)c3, q3.s);
        }
    }
}

template <int U, bool FUSED, int SP = 0>
__global__ void __launch_bounds__(kThreads) quant_v4_kernel(const float4 *__restrict__ K,
                                                            const float *__restrict__ scales,
                                                            uint32_t *__restrict__ Kq4, float4 *__restrict__ Kh4,
                                                            int64_t n4, int64_t cols4, int64_t G) {
    const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (g >= G) return;
    const int64_t c4 = g % cols4;
    const ColQ q0 = make_colq(__ldg(scales + 4 * c4 + 0));
    const ColQ q1 = make_colq(__ldg(scales + 4 * c4 + 1));
    const ColQ q2 = make_colq(__ldg(scales + 4 * c4 + 2));
    const ColQ q3 = make_colq(__ldg(scales + 4 * c4 + 3));
    const bool col_exact = q0.exact | q1.exact | q2.exact | q3.exact;
    for (int64_t i = g; i < n4; i += U * G) {
        float4 v[U];
#pragma unroll
        for (int k = 0; k < U; k++)
            if (i + k * G < n4) v[k] = ld_stream_f4(K + i + k * G);
#pragma unroll
        for (int k = 0; k < U; k++) {
            const int64_t idx = i + k * G;
            if (idx < n4) {
                uint32_t w;
                float4 xh;
                quant4<FUSED>(v[k], q0, q1, q2, q3, col_exact, w, xh);
                store_u32<SP>(Kq4 + idx, w);
                if (FUSED) store_f4<SP>(Kh4 + idx, xh);
            }
        }
    }
}

template <int U, bool FUSED>
__global__ void __launch_bounds__(kThreads) quant_scalar_kernel(const float *__restrict__ K,
                                                                const float *__restrict__ scales,
                                                                int8_t *__restrict__ Kq, float *__restrict__ Kh,
                                                                int64_t n, int64_t D, int64_t G) {
    const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (g >= G) return;
    const ColQ q = make_colq(__ldg(scales + g % D));
    for (int64_t i = g; i < n; i += U * G) {
        float v[U];
#pragma unroll
        for (int k = 0; k < U; k++)
            if (i + k * G < n) v[k] = __ldg(K + i + k * G);
#pragma unroll
        for (int k = 0; k < U; k++) {
            const int64_t idx = i + k * G;
            if (idx < n) {
                bool danger = q.exact;
                float a = quant_fast(v[k], q, danger);
                int c = danger ? quant_exact(v[k], q.s) : (int)(int8_t)code_byte(a);
                Kq[idx] = (int8_t)c;
                if (FUSED) Kh[idx] = __fmul_rn((float)c, q.s);
            }
        }
    }
}

// ============================================================================ a4: dequantize
// x_hat = fl32((float)q * s_d): one IEEE multiply; (float)0 * s = +0.
template <int U, int SP = 0>
__global__ void __launch_bounds__(kThreads) dequant_v4_kernel(const uint32_t *__restrict__ Kq4,
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
                float4 o;
                o.x = __fmul_rn(code_to_float(w[k], 0), s0);
                o.y = __fmul_rn(code_to_float(w[k], 1), s1);
                o.z = __fmul_rn(code_to_float(w[k], 2), s2);
                o.w = __fmul_rn(code_to_float(w[k], 3), s3);
                store_f4<SP>(Kh4 + idx, o);
            }
        }
    }
}

// ============================================================================ row-slab grid variants
// The same element arithmetic as quant_v4_kernel / dequant_v4_kernel on a
// non-persistent grid: block b covers a slab of kSlabU x RS rows by CW float4
// columns (CW = min(D/4, 256), RS = 256 / CW) and retires.  Consecutive blocks
// take the adjacent column chunks of the same rows, so the hardware block
// scheduler walks K in address order and the DRAM pages written at any moment
// form one narrow moving window.  Measured on B200 at C4
// (scripts/probes/bw_mix2.cu, profiles/r01/hbm_patterns.md): such grids reach
// 6.9 TB/s on the quantize+dequantize traffic mix where persistent grid-stride
// loops (whose blocks drift apart and widen the window) reach 5.6 TB/s -- for
// write-heavy traffic the width of the window sets the bandwidth.  Each thread
// keeps the column-owning idea inside its slab: one float4 of columns, its
// scales and RN(1/s) formed once and reused for kSlabU rows.
constexpr int kSlabU = 4;

struct SlabGeom {
    uint32_t cols4, CW, RS, NCC;  // float4 columns, chunk width, rows per slice, chunks per row
    int64_t T;
};

static SlabGeom slab_geom(int64_t T, int64_t cols4) {
    SlabGeom g;
    g.cols4 = (uint32_t)cols4;
    g.CW = (uint32_t)std::min<int64_t>(cols4, kThreads);
    g.RS = kThreads / g.CW;
    g.NCC = (uint32_t)((cols4 + g.CW - 1) / g.CW);
    g.T = T;
    return g;
}
static int64_t slab_blocks(const SlabGeom &g) {
    return (int64_t)g.NCC * ((g.T + (int64_t)g.RS * kSlabU - 1) / ((int64_t)g.RS * kSlabU));
}

// thread -> (first row, float4 column); false if the thread has no column
__device__ __forceinline__ bool slab_coords(const SlabGeom &g, int64_t &row0, uint32_t &c) {
    const uint32_t rs = threadIdx.x / g.CW, cl = threadIdx.x - rs * g.CW;
    const uint32_t cc = blockIdx.x % g.NCC;
    c = cc * g.CW + cl;
    row0 = (int64_t)(blockIdx.x / g.NCC) * (g.RS * kSlabU) + rs;
    return rs < g.RS && c < g.cols4;
}

template <int SP = 1>
__global__ void __launch_bounds__(kThreads) dequant_slab_kernel(const uint32_t *__restrict__ Kq4,
                                                                const float4 *__restrict__ scales4,
                                                                float4 *__restrict__ Kh4, const SlabGeom g) {
    int64_t row0;
    uint32_t c;
    if (!slab_coords(g, row0, c)) return;
    uint32_t w[kSlabU];
#pragma unroll
    for (int k = 0; k < kSlabU; k++) {
        const int64_t row = row0 + (int64_t)k * g.RS;
        if (row < g.T) w[k] = ld_stream_u32(Kq4 + row * g.cols4 + c);
    }
    const float4 s = __ldg(scales4 + c);
#pragma unroll
    for (int k = 0; k < kSlabU; k++) {
        const int64_t row = row0 + (int64_t)k * g.RS;
        if (row < g.T) {
            float4 o;
            o.x = __fmul_rn(code_to_float(w[k], 0), s.x);
            o.y = __fmul_rn(code_to_float(w[k], 1), s.y);
            o.z = __fmul_rn(code_to_float(w[k], 2), s.z);
            o.w = __fmul_rn(code_to_float(w[k], 3), s.w);
            store_f4<SP>(Kh4 + row * g.cols4 + c, o);
        }
    }
}

template <bool FUSED, int SP = 1>
__global__ void __launch_bounds__(kThreads) quant_slab_kernel(const float4 *__restrict__ K,
                                                              const float4 *__restrict__ scales4,
                                                              uint32_t *__restrict__ Kq4, float4 *__restrict__ Kh4,
                                                              const SlabGeom g) {
    int64_t row0;
    uint32_t c;
    if (!slab_coords(g, row0, c)) return;
    float4 v[kSlabU];
#pragma unroll
    for (int k = 0; k < kSlabU; k++) {
        const int64_t row = row0 + (int64_t)k * g.RS;
        if (row < g.T) v[k] = ld_stream_f4(K + row * g.cols4 + c);
    }
    const float4 s = __ldg(scales4 + c);
    const ColQ q0 = make_colq(s.x), q1 = make_colq(s.y), q2 = make_colq(s.z), q3 = make_colq(s.w);
    const bool col_exact = q0.exact | q1.exact | q2.exact | q3.exact;
#pragma unroll
    for (int k = 0; k < kSlabU; k++) {
        const int64_t row = row0 + (int64_t)k * g.RS;
        if (row < g.T) {
            uint32_t w;
            float4 xh;
            quant4<FUSED>(v[k], q0, q1, q2, q3, col_exact, w, xh);
            store_u32<SP>(Kq4 + row * g.cols4 + c, w);
            if (FUSED) store_f4<SP>(Kh4 + row * g.cols4 + c, xh);
        }
    }
}

template <int U>
__global__ void __launch_bounds__(kThreads) dequant_scalar_kernel(const int8_t *__restrict__ Kq,
                                                                  const float *__restrict__ scales,
                                                                  float *__restrict__ Kh, int64_t n, int64_t D,
                                                                  int64_t G) {
    const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (g >= G) return;
    const float s = __ldg(scales + g % D);
    for (int64_t i = g; i < n; i += U * G) {
        int8_t c[U];
#pragma unroll
        for (int k = 0; k < U; k++)
            if (i + k * G < n) c[k] = Kq[i + k * G];
#pragma unroll
        for (int k = 0; k < U; k++)
            if (i + k * G < n) Kh[i + k * G] = __fmul_rn((float)(int)c[k], s);
    }
}

// ============================================================================ a1+a2+a3+a4 single pass
// One cooperative launch for L2-resident sizes: phase 1 is the column abs-max of
// colmax_v4_kernel, then a grid-wide barrier, then each thread forms the scales of
// its own 4 columns (Eq. 6, IEEE division) and runs the fused quantize+dequantize
// loop of quant_v4_kernel over the same elements, which the first phase has just
// pulled into the 126 MB L2.  Same geometry in both phases (column-owning threads).
__device__ __forceinline__ void grid_barrier_once(unsigned *ctr, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        while (*reinterpret_cast<volatile unsigned *>(ctr) < nblocks) __nanosleep(64);
        __threadfence();
    }
    __syncthreads();
}

template <int U>
__global__ void __launch_bounds__(kThreads) single_pass_v4_kernel(const float4 *__restrict__ K, int64_t n4,
                                                                  int64_t cols4, int64_t G, uint32_t *mbits,
                                                                  unsigned *barrier, float *__restrict__ scales,
                                                                  uint32_t *__restrict__ Kq4,
                                                                  float4 *__restrict__ Kh4) {
    extern __shared__ uint32_t smax[];  // [4*cols4] when cols4 <= kThreads
    const bool share = cols4 <= kThreads;
    const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    const int64_t c4 = g < G ? g % cols4 : 0;
    // ---- phase 1: a1 (colmax_v4_kernel)
    if (share) {
        for (int i = threadIdx.x; i < 4 * cols4; i += kThreads) smax[i] = 0u;
        __syncthreads();
    }
    uint32_t m0 = 0, m1 = 0, m2 = 0, m3 = 0;
    if (g < G) {
        int64_t i = g;
        for (; i + (U - 1) * G < n4; i += U * G) {
            float4 v[U];
#pragma unroll
            for (int k = 0; k < U; k++) v[k] = __ldcg(K + i + k * G);  // keep K in L2 for phase 2
#pragma unroll
            for (int k = 0; k < U; k++) {
                m0 = max(m0, absbits(v[k].x));
                m1 = max(m1, absbits(v[k].y));
                m2 = max(m2, absbits(v[k].z));
                m3 = max(m3, absbits(v[k].w));
            }
        }
        for (; i < n4; i += G) {
            float4 v = __ldcg(K + i);
            m0 = max(m0, absbits(v.x));
            m1 = max(m1, absbits(v.y));
            m2 = max(m2, absbits(v.z));
            m3 = max(m3, absbits(v.w));
        }
    }
    if (share) {
        if (g < G) {
            atomicMax(&smax[4 * c4 + 0], m0);
            atomicMax(&smax[4 * c4 + 1], m1);
            atomicMax(&smax[4 * c4 + 2], m2);
            atomicMax(&smax[4 * c4 + 3], m3);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < 4 * cols4; i += kThreads)
            if (smax[i]) atomicMax(&mbits[i], smax[i]);
    } else if (g < G) {
        atomicMax(&mbits[4 * c4 + 0], m0);
        atomicMax(&mbits[4 * c4 + 1], m1);
        atomicMax(&mbits[4 * c4 + 2], m2);
        atomicMax(&mbits[4 * c4 + 3], m3);
    }
    grid_barrier_once(barrier, gridDim.x);
    if (g >= G) return;
    // ---- a2 for the thread's own columns (Eq. 6), published by the threads of row-lane 0
    float sc[4];
#pragma unroll
    for (int j = 0; j < 4; j++) sc[j] = __fdiv_rn(__uint_as_float(__ldcg(mbits + 4 * c4 + j)), 127.0f);
    if (g < cols4) {
#pragma unroll
        for (int j = 0; j < 4; j++) scales[4 * c4 + j] = sc[j];
    }
    // ---- phase 2: a3 + a4 (quant_v4_kernel<.., true>)
    const ColQ q0 = make_colq(sc[0]), q1 = make_colq(sc[1]), q2 = make_colq(sc[2]), q3 = make_colq(sc[3]);
    const bool col_exact = q0.exact | q1.exact | q2.exact | q3.exact;
    for (int64_t i = g; i < n4; i += 4 * G) {
        float4 v[4];
#pragma unroll
        for (int k = 0; k < 4; k++)
            if (i + k * G < n4) v[k] = __ldcs(K + i + k * G);  // last use: evict
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int64_t idx = i + k * G;
            if (idx < n4) {
                uint32_t w;
                float4 xh;
                quant4<true>(v[k], q0, q1, q2, q3, col_exact, w, xh);
                Kq4[idx] = w;
                Kh4[idx] = xh;
            }
        }
    }
}

// ============================================================================ host launchers
static inline bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

StreamPlan plan_stream(int64_t rows, int64_t cols, int threads_per_sm) {
    const DeviceInfo &di = device_info();
    const int64_t target = (int64_t)di.num_sms * threads_per_sm;
    int64_t R = std::max<int64_t>(1, target / cols);
    R = std::min<int64_t>(R, rows);
    StreamPlan p;
    p.G = cols * R;
    p.blocks = (unsigned)((p.G + kThreads - 1) / kThreads);
    return p;
}

#ifndef KVQ_UQUANT
#define KVQ_UQUANT 8  // loads in flight per thread of the quantize-alone kernel (C4: 8 -> 0.848 ms, 4 -> 0.863-0.868, 2 -> 0.864-0.877)
#endif
constexpr int kUColmax = 8, kUQuant = KVQ_UQUANT, kUDequant = 8;

// Row-slab kernels: scales read as float4 (16-byte aligned), grid.x < 2^31, cols4 < 2^31.
static bool slab_ok(int64_t cols4, const float *scales) {
    return aligned(scales, 16) && cols4 < (1LL << 31);
}

// Resident threads per SM for `kernel` at kThreads per CTA: the grid is sized
// to exactly one full wave of resident threads (no tail wave).
template <typename Kern>
static int resident_threads(Kern kernel, size_t smem) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, kThreads, smem) != cudaSuccess || nb < 1) {
        cudaGetLastError();
        nb = 1;
    }
    return nb * kThreads;
}
#define KVQ_RESIDENT(kernel, smem)                                     \
    ([&]() {                                                           \
        static const int r_ = resident_threads(kernel, (smem));        \
        return r_;                                                     \
    }())

kvq_status launch_colmax(const float *K, int64_t T, int64_t D, uint32_t *mbits, cudaStream_t s) {
    const int64_t n = T * D;
    if (D % 4 == 0 && aligned(K, 16)) {
        const int64_t cols4 = D / 4;
        size_t smem = cols4 <= kThreads ? (size_t)4 * cols4 * sizeof(uint32_t) : 0;
        StreamPlan p = plan_stream(T, cols4, KVQ_RESIDENT(colmax_v4_kernel<kUColmax>, 4 * kThreads * sizeof(uint32_t)));
        colmax_v4_kernel<kUColmax><<<p.blocks, kThreads, smem, s>>>(reinterpret_cast<const float4 *>(K), n / 4,
                                                                   cols4, p.G, mbits);
    } else {
        StreamPlan p = plan_stream(T, D, KVQ_RESIDENT(colmax_scalar_kernel<kUColmax>, 0));
        colmax_scalar_kernel<kUColmax><<<p.blocks, kThreads, 0, s>>>(K, n, D, p.G, mbits);
    }
    return check_launch("colmax");
}

kvq_status launch_finalize(uint32_t *buf, int64_t D, cudaStream_t s, float divisor) {
    unsigned blocks = (unsigned)std::min<int64_t>((D + 255) / 256, 1024);
    if (cudaError_t e = launch_pdl(finalize_kernel, dim3(blocks), dim3(256), 0, s, buf, D, divisor); e != cudaSuccess)
        return check_launch("finalize");
    return check_launch("finalize");
}

// Outputs are written once and not re-read by this call: streaming (evict-first) stores
// keep them from displacing useful L2 lines (measured: the following column-max pass
// runs ~4% faster than after write-back-allocate stores).
kvq_status launch_quantize(const float *K, const float *scales, int64_t T, int64_t D, int8_t *Kq, float *K_hat,
                           cudaStream_t s) {
    const int64_t n = T * D;
    const bool vec = D % 4 == 0 && aligned(K, 16) && aligned(Kq, 4) && (!K_hat || aligned(K_hat, 16));
    if (vec) {
        const int64_t cols4 = D / 4;
        auto K4 = reinterpret_cast<const float4 *>(K);
        auto Q4 = reinterpret_cast<uint32_t *>(Kq);
        auto H4 = reinterpret_cast<float4 *>(K_hat);
        const SlabGeom sg = slab_geom(T, cols4);
        // quantize + dequantize (R4 W5, write-heavy): row-slab grid, 1.40 vs 1.75 ms at C4.
        // quantize alone (R4 W1, read-heavy): the persistent column-owning kernel stays ahead
        // (0.86 vs 0.92 ms at C4, same box), so it keeps the grid-stride geometry.
        if (K_hat && slab_ok(cols4, scales) && slab_blocks(sg) < (1LL << 31)) {
            quant_slab_kernel<true><<<(unsigned)slab_blocks(sg), kThreads, 0, s>>>(
                K4, reinterpret_cast<const float4 *>(scales), Q4, H4, sg);
#ifdef KVQ_QSLAB  // experiments: quantize alone on the row-slab grid
        } else if (!K_hat && slab_ok(cols4, scales) && slab_blocks(sg) < (1LL << 31)) {
            quant_slab_kernel<false><<<(unsigned)slab_blocks(sg), kThreads, 0, s>>>(
                K4, reinterpret_cast<const float4 *>(scales), Q4, nullptr, sg);
#endif
        } else if (K_hat) {
            StreamPlan p = plan_stream(T, cols4, KVQ_RESIDENT((quant_v4_kernel<kUQuant, true, 1>), 0));
            quant_v4_kernel<kUQuant, true, 1><<<p.blocks, kThreads, 0, s>>>(K4, scales, Q4, H4, n / 4, cols4, p.G);
        } else {
            StreamPlan p = plan_stream(T, cols4, KVQ_RESIDENT((quant_v4_kernel<kUQuant, false, 1>), 0));
            quant_v4_kernel<kUQuant, false, 1><<<p.blocks, kThreads, 0, s>>>(K4, scales, Q4, nullptr, n / 4, cols4,
                                                                             p.G);
        }
    } else {
        StreamPlan p = plan_stream(T, D, KVQ_RESIDENT((quant_scalar_kernel<kUQuant, true>), 0));
        if (K_hat)
            quant_scalar_kernel<kUQuant, true><<<p.blocks, kThreads, 0, s>>>(K, scales, Kq, K_hat, n, D, p.G);
        else
            quant_scalar_kernel<kUQuant, false><<<p.blocks, kThreads, 0, s>>>(K, scales, Kq, nullptr, n, D, p.G);
    }
    return check_launch(K_hat ? "quantize_dequantize" : "quantize");
}

kvq_status launch_dequantize(const int8_t *Kq, const float *scales, int64_t T, int64_t D, float *K_hat,
                             cudaStream_t s) {
    const int64_t n = T * D;
    if (D % 4 == 0 && aligned(Kq, 4) && aligned(K_hat, 16) && slab_ok(D / 4, scales) &&
        slab_blocks(slab_geom(T, D / 4)) < (1LL << 31)) {
        const SlabGeom sg = slab_geom(T, D / 4);
        dequant_slab_kernel<<<(unsigned)slab_blocks(sg), kThreads, 0, s>>>(reinterpret_cast<const uint32_t *>(Kq),
                                                                          reinterpret_cast<const float4 *>(scales),
                                                                          reinterpret_cast<float4 *>(K_hat), sg);
    } else if (D % 4 == 0 && aligned(Kq, 4) && aligned(K_hat, 16)) {
        const int64_t cols4 = D / 4;
        StreamPlan p = plan_stream(T, cols4, KVQ_RESIDENT((dequant_v4_kernel<kUDequant, 1>), 0));
        dequant_v4_kernel<kUDequant, 1><<<p.blocks, kThreads, 0, s>>>(
            reinterpret_cast<const uint32_t *>(Kq), scales, reinterpret_cast<float4 *>(K_hat), n / 4, cols4, p.G);
    } else {
        StreamPlan p = plan_stream(T, D, KVQ_RESIDENT(dequant_scalar_kernel<kUDequant>, 0));
        dequant_scalar_kernel<kUDequant><<<p.blocks, kThreads, 0, s>>>(Kq, scales, K_hat, n, D, p.G);
    }
    return check_launch("dequantize");
}

}  // namespace kvq

namespace kvq {

// D column maxima + the grid barrier word (64 B) at a 256-byte aligned offset of any caller pointer: up to
// 255 bytes of alignment slack
size_t single_pass_workspace_size(int64_t D) { return (size_t)D * 4 + 64 + 255; }

// Returns KVQ_ERR_UNSUPPORTED (nothing launched) when the shape or alignment does
// not allow the single cooperative pass; the caller then runs the two passes.
kvq_status launch_single_pass(const float *K, int64_t T, int64_t D, float *scales, int8_t *Kq, float *K_hat,
                              void *ws, cudaStream_t s) {
    if (D % 4 || !aligned(K, 16) || !aligned(Kq, 4) || !aligned(K_hat, 16))
        return KVQ_ERR_UNSUPPORTED;
    const int64_t cols4 = D / 4;
    if (cols4 > (int64_t)device_info().num_sms * kThreads) return KVQ_ERR_UNSUPPORTED;
    const size_t smem = cols4 <= kThreads ? (size_t)4 * cols4 * sizeof(uint32_t) : 0;
    static int nb_per_sm = [] {
        int nb = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, single_pass_v4_kernel<kUColmax>, kThreads,
                                                      4 * kThreads * sizeof(uint32_t));
        cudaGetLastError();
        return nb;
    }();
    if (nb_per_sm < 1) return KVQ_ERR_UNSUPPORTED;
    StreamPlan p = plan_stream(T, cols4, nb_per_sm * kThreads);
    if ((int64_t)p.blocks > (int64_t)nb_per_sm * device_info().num_sms) return KVQ_ERR_UNSUPPORTED;
    uint32_t *mbits = reinterpret_cast<uint32_t *>((reinterpret_cast<uintptr_t>(ws) + 255) & ~(uintptr_t)255);
    unsigned *bar = reinterpret_cast<unsigned *>(mbits + D);
    if (cudaMemsetAsync(mbits, 0, (size_t)D * 4 + 64, s) != cudaSuccess) return check_launch("single_pass memset");
    const float4 *K4 = reinterpret_cast<const float4 *>(K);
    int64_t n4 = T * D / 4, G = p.G;
    uint32_t *Q4 = reinterpret_cast<uint32_t *>(Kq);
    float4 *H4 = reinterpret_cast<float4 *>(K_hat);
    void *args[] = {(void *)&K4, (void *)&n4, (void *)&cols4, (void *)&G, (void *)&mbits, (void *)&bar,
                    (void *)&scales, (void *)&Q4, (void *)&H4};
    cudaError_t e = cudaLaunchCooperativeKernel((const void *)single_pass_v4_kernel<kUColmax>, dim3(p.blocks),
                                                dim3(kThreads), args, smem, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(KVQ_ERR_CUDA, std::string("single_pass cooperative launch: ") + cudaGetErrorString(e));
    }
    return KVQ_OK;
}

}  // namespace kvq
