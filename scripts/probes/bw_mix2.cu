// HBM access-pattern probe for the roundtrip's traffic mix (no arithmetic):
// read K (4 B/elem), write K_hat (4 B/elem) and codes (1 B/elem), C4 size.
// Compares SIMT linear streams (persistent one-wave and non-persistent grids,
// .cs vs default stores), 1-D bulk copies through smem (TMA cp.async.bulk), and
// the roundtrip kernel's own pattern: 2-D TMA boxes of 128 rows x 32 fp32 walked
// along the row (one 128-row tile per CTA, all D columns), at several box widths.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2601_04719_b200/csrc bw_mix2.cu
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>

#include "tc_common.cuh"

using namespace kvq::tc;

static const int64_t T = 131072, D = 8192, N = T * D;
static int g_hints = getenv("HINTS") ? atoi(getenv("HINTS")) : 3;

// ------------------------------------------------------------------ SIMT linear
template <int UNR, int CS, int WC>
__global__ void __launch_bounds__(256) lin_persist(const float4 *__restrict__ in, float4 *__restrict__ outk,
                                                   uint32_t *__restrict__ outc, int64_t n4) {
    const int64_t G = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += UNR * G) {
        float4 v[UNR];
#pragma unroll
        for (int k = 0; k < UNR; k++)
            if (i + k * G < n4)
                asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                             : "=f"(v[k].x), "=f"(v[k].y), "=f"(v[k].z), "=f"(v[k].w) : "l"(in + i + k * G));
#pragma unroll
        for (int k = 0; k < UNR; k++)
            if (i + k * G < n4) {
                if (CS)
                    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(outk + i + k * G), "f"(v[k].x),
                                 "f"(v[k].y), "f"(v[k].z), "f"(v[k].w) : "memory");
                else
                    outk[i + k * G] = v[k];
                if (WC) {
                    const uint32_t c = __float_as_uint(v[k].x) ^ __float_as_uint(v[k].w);
                    if (CS)
                        asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(outc + i + k * G), "r"(c) : "memory");
                    else
                        outc[i + k * G] = c;
                }
            }
    }
}

// non-persistent: each block handles a contiguous 256*UNR float4 chunk
template <int UNR, int CS, int WC>
__global__ void __launch_bounds__(256) lin_grid(const float4 *__restrict__ in, float4 *__restrict__ outk,
                                                uint32_t *__restrict__ outc, int64_t n4) {
    const int64_t base = (int64_t)blockIdx.x * 256 * UNR + threadIdx.x;
    float4 v[UNR];
#pragma unroll
    for (int k = 0; k < UNR; k++) v[k] = __ldcs(in + base + k * 256);
#pragma unroll
    for (int k = 0; k < UNR; k++) {
        if (CS)
            __stcs(outk + base + k * 256, v[k]);
        else
            outk[base + k * 256] = v[k];
        if (WC) {
            const uint32_t c = __float_as_uint(v[k].x) ^ __float_as_uint(v[k].w);
            if (CS)
                __stcs(outc + base + k * 256, c);
            else
                outc[base + k * 256] = c;
        }
    }
}

template <int UNR, int RW>
__global__ void __launch_bounds__(256) lin_grid_rw(const float4 *__restrict__ in, float4 *__restrict__ outk, int64_t n4) {
    const int64_t base = (int64_t)blockIdx.x * 256 * UNR + threadIdx.x;
    float4 v[UNR];
    if (RW & 1) {
#pragma unroll
        for (int k = 0; k < UNR; k++) v[k] = __ldcs(in + base + k * 256);
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < UNR; k++) acc += v[k].x + v[k].w;
        if (acc == 1.2345f) outk[0] = v[0];
    } else {
#pragma unroll
        for (int k = 0; k < UNR; k++) __stcs(outk + base + k * 256, make_float4(base, k, 0.f, 1.f));
    }
}

// ------------------------------------------------------------------ 1-D bulk (TMA) through smem
__device__ __forceinline__ void bulk_store(void *dst, const void *src, uint32_t bytes, uint64_t pol) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes), "l"(pol)
                 : "memory");
}

template <int ST, int CHUNK, int WC>
__global__ void __launch_bounds__(64, 1) bulk1d(const float *in, float *outk, uint8_t *outc, int64_t nchunks,
                                                int hints) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + ST * CHUNK + CHUNK / 4);
    uint64_t *empty = full + ST;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < ST; i++) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const uint64_t pin = (hints & 1) ? policy_evict_first() : policy_evict_normal();
    const uint64_t pout = (hints & 2) ? policy_evict_first() : policy_evict_normal();
    if (warp == 0 && lane == 0) {
        uint32_t g = 0;
        for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, g++) {
            const int sk = g % ST;
            mbar_wait(&empty[sk], ((g / ST) & 1) ^ 1);
            mbar_arrive_tx(&full[sk], CHUNK);
            bulk_load(sm + sk * CHUNK, reinterpret_cast<const uint8_t *>(in) + c * CHUNK, CHUNK, &full[sk], pin);
        }
    } else if (warp == 1 && lane == 0) {
        uint32_t g = 0;
        for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, g++) {
            const int sk = g % ST;
            mbar_wait(&full[sk], (g / ST) & 1);
            bulk_store(reinterpret_cast<uint8_t *>(outk) + c * CHUNK, sm + sk * CHUNK, CHUNK, pout);
            if (WC) bulk_store(outc + c * (CHUNK / 4), sm + ST * CHUNK, CHUNK / 4, pout);
            bulk_commit();
            if (g > 0) {
                bulk_wait_read<1>();
                mbar_arrive(&empty[(g - 1) % ST]);
            }
        }
        bulk_wait<0>();
    }
}

// ------------------------------------------------------------------ 2-D tile pattern (the roundtrip's)
// CTA walks 128-row tiles; per tile the K-blocks of BC columns left to right.
// codes: every (128/BC) K-blocks one [128 x 128 B] box.
template <int ST, int BC, int WC, int RW = 3, int BR = 128, int WD = 1>
__global__ void __launch_bounds__(64, 1) tile2d(const __grid_constant__ CUtensorMap mi,
                                                const __grid_constant__ CUtensorMap mo,
                                                const __grid_constant__ CUtensorMap mc, int ntiles, int nkb,
                                                int hints, int rot = 0) {
    extern __shared__ __align__(1024) uint8_t sm[];
    constexpr uint32_t BOX = (uint32_t)BR * BC * 4;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + ST * BOX + 16384);
    uint64_t *empty = full + ST;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < ST; i++) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const uint64_t pin = (hints & 1) ? policy_evict_first() : policy_evict_normal();
    const uint64_t pout = (hints & 2) ? policy_evict_first() : policy_evict_normal();
    constexpr int CKB = BC >= 128 ? 1 : 128 / BC;  // K-blocks per code box
    if (warp == 0 && lane == 0) {
        uint32_t g = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
            for (int k = 0; k < nkb; k++, g++) {
                const int kb = (k + tile * rot) % nkb;
                const int sk = g % ST;
                mbar_wait(&empty[sk], ((g / ST) & 1) ^ 1);
                if (RW & 1) {
                    mbar_arrive_tx(&full[sk], BOX);
                    tma_load_2d(sm + sk * BOX, &mi, &full[sk], kb * BC, tile * BR, pin);
                } else {
                    mbar_arrive(&full[sk]);
                }
            }
    } else if (warp == 1 && lane == 0) {
        uint32_t g = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
            for (int k = 0; k < nkb; k++, g++) {
                const int kb = (k + tile * rot) % nkb;
                const int sk = g % ST;
                mbar_wait(&full[sk], (g / ST) & 1);
                if (RW & 6) {
                    if (RW & 2) tma_store_2d(&mo, sm + sk * BOX, kb * BC, tile * BR, pout);
                    if (WC && (kb % CKB) == CKB - 1) {
                        if (BC >= 128) {
                            for (int j = 0; j < BC / 128; j++)
                                tma_store_2d(&mc, sm + ST * BOX, kb * BC + 128 * j, tile * BR, pout);
                        } else {
                            tma_store_2d(&mc, sm + ST * BOX, (kb / CKB) * 128, tile * BR, pout);
                        }
                    }
                }
                bulk_commit();
                if (g >= WD) {
                    bulk_wait_read<WD>();
                    mbar_arrive(&empty[(g - WD) % ST]);
                }
            }
        bulk_wait<0>();
    }
}

// Non-persistent SIMT version of the tile pattern: block b writes (and reads) one [128 x 32] fp32 box;
// resident blocks cover the same kb of 148 consecutive tiles at a time (the roundtrip's concurrency).
template <int RW>
__global__ void __launch_bounds__(256) simt_tile(const float *__restrict__ in, float *__restrict__ out,
                                                 uint8_t *__restrict__ oc, int ntiles, int nkb) {
    const int grpsz = 148;
    const int64_t b = blockIdx.x;
    const int64_t per_grp = (int64_t)grpsz * nkb;
    const int grp = (int)(b / per_grp);
    const int rem = (int)(b % per_grp);
    const int kb = rem / grpsz, tile = grp * grpsz + rem % grpsz;
    if (tile >= ntiles) return;
    // 256 threads: thread -> row (t/8) + 32 * k, 16-byte chunk t%8
    const int c = threadIdx.x % 8;
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int r = threadIdx.x / 8 + 32 * k;
        const int64_t off = ((int64_t)tile * 128 + r) * D + kb * 32 + c * 4;
        float4 v = make_float4(1.f, 2.f, 3.f, (float)r);
        if (RW & 1) v = __ldcs(reinterpret_cast<const float4 *>(in + off));
        if (RW & 2) __stcs(reinterpret_cast<float4 *>(out + off), v);
        if ((RW & 4) && c < 2) __stcs(reinterpret_cast<uint32_t *>(oc + off) + 0, __float_as_uint(v.x));
    }
}

// Persistent TMA-load + SIMT-store tile pattern: 4 store warps copy each staged box to global.
template <int ST>
__global__ void __launch_bounds__(160, 1) tile_tma_simt(const __grid_constant__ CUtensorMap mi, float *__restrict__ out,
                                                        int ntiles, int nkb) {
    extern __shared__ __align__(1024) uint8_t sm[];
    constexpr uint32_t BOX = 128u * 32 * 4;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + ST * BOX);
    uint64_t *empty = full + ST;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < ST; i++) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 128);
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (warp == 4) {
        if (lane == 0) {
            const uint64_t pin = policy_evict_first();
            uint32_t g = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
                for (int kb = 0; kb < nkb; kb++, g++) {
                    const int sk = g % ST;
                    mbar_wait(&empty[sk], ((g / ST) & 1) ^ 1);
                    mbar_arrive_tx(&full[sk], BOX);
                    tma_load_2d(sm + sk * BOX, &mi, &full[sk], kb * 32, tile * 128, pin);
                }
        }
    } else {
        uint32_t g = 0;
        const int t = threadIdx.x;  // 0..127
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
            for (int kb = 0; kb < nkb; kb++, g++) {
                const int sk = g % ST;
                mbar_wait(&full[sk], (g / ST) & 1);
                const uint32_t base = smem_u32(sm + sk * BOX);
#pragma unroll
                for (int k = 0; k < 8; k++) {
                    const int r = t / 8 + 16 * k, c = t % 8;
                    const float4 v = lds128(base + r * 128 + ((c ^ (r & 7)) << 4));
                    __stcs(reinterpret_cast<float4 *>(out + ((int64_t)tile * 128 + r) * D + kb * 32 + c * 4), v);
                }
                mbar_arrive(&empty[sk]);
            }
    }
}

// persistent, block-chunked: iteration i of block b handles the contiguous chunk b + i*gridDim.x
template <int UNR, int WC>
__global__ void __launch_bounds__(256) lin_chunk(const float4 *__restrict__ in, float4 *__restrict__ outk,
                                                 uint32_t *__restrict__ outc, int64_t n4) {
    const int64_t nch = n4 / (256 * UNR);
    for (int64_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {
        const int64_t base = ch * 256 * UNR + threadIdx.x;
        float4 v[UNR];
#pragma unroll
        for (int k = 0; k < UNR; k++) v[k] = __ldcs(in + base + k * 256);
#pragma unroll
        for (int k = 0; k < UNR; k++) {
            __stcs(outk + base + k * 256, v[k]);
            if (WC) __stcs(outc + base + k * 256, __float_as_uint(v[k].x) ^ __float_as_uint(v[k].w));
        }
    }
}
// dequant-shaped (R1W4) and quant-shaped (R4W1) linear grid kernels
template <int UNR>
__global__ void __launch_bounds__(256) g_r1w4(const uint32_t *__restrict__ c, float4 *__restrict__ out) {
    const int64_t base = (int64_t)blockIdx.x * 256 * UNR + threadIdx.x;
    uint32_t v[UNR];
#pragma unroll
    for (int k = 0; k < UNR; k++) v[k] = __ldcs(c + base + k * 256);
#pragma unroll
    for (int k = 0; k < UNR; k++) __stcs(out + base + k * 256, make_float4((float)(v[k] & 255), 0.f, 1.f, 2.f));
}
template <int UNR>
__global__ void __launch_bounds__(256) g_r4w1(const float4 *__restrict__ in, uint32_t *__restrict__ c) {
    const int64_t base = (int64_t)blockIdx.x * 256 * UNR + threadIdx.x;
    float4 v[UNR];
#pragma unroll
    for (int k = 0; k < UNR; k++) v[k] = __ldcs(in + base + k * 256);
#pragma unroll
    for (int k = 0; k < UNR; k++) __stcs(c + base + k * 256, __float_as_uint(v[k].x) ^ __float_as_uint(v[k].w));
}

// Group-interleaved tile pattern: G consecutive CTAs share one 128-row tile; CTA j of the group takes the
// K-blocks whose index / IL is congruent to j mod G.  Box [128 x 32] fp32, codes [128 x 32 B] per K-block
// (IL == 1) or [128 x 128 B] per 4 K-blocks (IL == 4).
template <int ST, int G, int IL>
__global__ void __launch_bounds__(64, 1) tile_grp(const __grid_constant__ CUtensorMap mi,
                                                  const __grid_constant__ CUtensorMap mo,
                                                  const __grid_constant__ CUtensorMap mc, int ntiles, int nkb) {
    extern __shared__ __align__(1024) uint8_t sm[];
    constexpr uint32_t BOX = 128u * 32 * 4;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + ST * BOX + 16384);
    uint64_t *empty = full + ST;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < ST; i++) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const int grp = blockIdx.x / G, j = blockIdx.x % G, ngrp = gridDim.x / G;
    const int my_kb = nkb / G;
    const uint64_t pin = policy_evict_first(), pout = policy_evict_first();
    if (warp == 0 && lane == 0) {
        uint32_t g = 0;
        for (int tile = grp; tile < ntiles; tile += ngrp)
            for (int k = 0; k < my_kb; k++, g++) {
                const int kb = (k / IL) * G * IL + j * IL + k % IL;
                const int sk = g % ST;
                mbar_wait(&empty[sk], ((g / ST) & 1) ^ 1);
                mbar_arrive_tx(&full[sk], BOX);
                tma_load_2d(sm + sk * BOX, &mi, &full[sk], kb * 32, tile * 128, pin);
            }
    } else if (warp == 1 && lane == 0) {
        uint32_t g = 0;
        for (int tile = grp; tile < ntiles; tile += ngrp)
            for (int k = 0; k < my_kb; k++, g++) {
                const int kb = (k / IL) * G * IL + j * IL + k % IL;
                const int sk = g % ST;
                mbar_wait(&full[sk], (g / ST) & 1);
                tma_store_2d(&mo, sm + sk * BOX, kb * 32, tile * 128, pout);
                if (IL == 1) tma_store_2d(&mc, sm + ST * BOX, kb * 32, tile * 128, pout);
                else if (k % IL == IL - 1) tma_store_2d(&mc, sm + ST * BOX, (kb / 4) * 128, tile * 128, pout);
                bulk_commit();
                if (g > 0) {
                    bulk_wait_read<1>();
                    mbar_arrive(&empty[(g - 1) % ST]);
                }
            }
        bulk_wait<0>();
    }
}

// ------------------------------------------------------------------ host
static PFN_cuTensorMapEncodeTiled_v12000 enc() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *ptr = nullptr;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}
static CUtensorMap map2d(void *base, CUtensorMapDataType ty, int elem, int box_cols, bool swz, int box_rows = 128) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)T};
    cuuint64_t strides[1] = {(cuuint64_t)D * elem};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc()(&m, ty, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d (box %d)\n", (int)r, box_cols);
    return m;
}

template <typename F>
static void timeit(const char *name, double bpe, F launch) {
    for (int w = 0; w < 3; w++) launch();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    std::vector<float> ts;
    for (int r = 0; r < 12; r++) {
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    const cudaError_t e = cudaGetLastError();
    printf("%-40s best %.3f ms  med %.3f ms  %6.0f GB/s (best)  %6.0f GB/s (med)  %.1f B/elem %s\n", name, ts[0],
           ts[ts.size() / 2], bpe * N / (ts[0] * 1e-3) / 1e9, bpe * N / (ts[ts.size() / 2] * 1e-3) / 1e9, bpe,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main(int argc, char **argv) {
    setvbuf(stdout, nullptr, _IONBF, 0);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *in, *ok;
    uint8_t *oc;
    cudaMalloc(&in, N * 4);
    cudaMalloc(&ok, N * 4);
    cudaMalloc(&oc, N);
    cudaMemset(in, 0, N * 4);
    const int64_t n4 = N / 4;
    const float4 *in4 = reinterpret_cast<const float4 *>(in);
    float4 *ok4 = reinterpret_cast<float4 *>(ok);
    uint32_t *oc4 = reinterpret_cast<uint32_t *>(oc);  // 4 codes per float4 -> one u32 per float4

#define PERSIST(U, CS, WC, name, bpe)                                                                     \
    {                                                                                                     \
        int nb = 0;                                                                                       \
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, lin_persist<U, CS, WC>, 256, 0);               \
        timeit(name, bpe, [&] { lin_persist<U, CS, WC><<<sms * nb, 256>>>(in4, ok4, oc4, n4); });        \
    }
#define TILE(ST, BC, BR, WC, RW, name, bpe) TILEW(ST, BC, BR, WC, RW, 1, name, bpe)
#define TILEW(ST, BC, BR, WC, RW, WD, name, bpe)                                                                      \
    {                                                                                                            \
        CUtensorMap mi = map2d(in, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, BC, BC == 32, BR);                        \
        CUtensorMap mo = map2d(ok, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, BC, BC == 32, BR);                        \
        CUtensorMap mc = map2d(oc, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, 128, true, BR);                             \
        const size_t smem = ST * BR * BC * 4 + 16384 + 1024;                                                     \
        cudaFuncSetAttribute(tile2d<ST, BC, WC, RW, BR, WD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        timeit(name, bpe, [&] {                                                                                  \
            tile2d<ST, BC, WC, RW, BR, WD><<<sms, 64, smem>>>(mi, mo, mc, (int)(T / BR), (int)(D / BC), g_hints, 0);     \
        });                                                                                                      \
    }
    const int ntl = (int)(T / 128), nkb = (int)(D / 32);
    CUtensorMap mi = map2d(in, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 32, true, 128);
    CUtensorMap mo = map2d(ok, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 32, true, 128);
    CUtensorMap mc128 = map2d(oc, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, 128, true, 128);
    CUtensorMap mc32 = map2d(oc, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, 32, false, 128);
    const size_t smem = 8 * 16384 + 16384 + 1024;
#define GRP(G, IL, name)                                                                                       \
    {                                                                                                          \
        cudaFuncSetAttribute(tile_grp<8, G, IL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
        const int grid = (sms / G) * G;                                                                        \
        timeit(name, 9, [&] {                                                                                  \
            tile_grp<8, G, IL><<<grid, 64, smem>>>(mi, mo, IL == 1 ? mc32 : mc128, ntl, nkb);                 \
        });                                                                                                    \
    }
    if (getenv("WIDE3")) {  // round 2: the 64-row geometries at the real kernel's 128 KB in flight
    TILE(8, 32, 128, 1, 3, "tile BR128 BC32  ST8  R4W5", 9);
    TILE(8, 64, 64, 1, 3, "tile BR64  BC64  ST8  R4W5", 9);
    TILE(6, 64, 64, 1, 3, "tile BR64  BC64  ST6  R4W5", 9);
    TILE(16, 32, 64, 1, 3, "tile BR64  BC32  ST16 R4W5", 9);
    TILE(4, 128, 64, 1, 3, "tile BR64  BC128 ST4  R4W5", 9);
    TILEW(8, 64, 64, 1, 3, 2, "tile BR64  BC64  ST8 WD2 R4W5", 9);
    TILE(8, 32, 128, 1, 3, "tile BR128 BC32  ST8  R4W5", 9);
    TILE(8, 64, 64, 1, 3, "tile BR64  BC64  ST8  R4W5", 9);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
    }
    if (getenv("WIDE2")) {  // round 2: shorter tiles with longer row segments (candidate M = 64 geometries)
    TILE(4, 32, 128, 1, 3, "tile BR128 BC32  ST4  R4W5", 9);
    TILE(8, 32, 128, 1, 3, "tile BR128 BC32  ST8  R4W5", 9);
    TILE(4, 32, 64, 1, 3, "tile BR64  BC32  ST4  R4W5", 9);
    TILE(8, 32, 64, 1, 3, "tile BR64  BC32  ST8  R4W5", 9);
    TILE(4, 64, 64, 1, 3, "tile BR64  BC64  ST4  R4W5", 9);
    TILE(2, 128, 64, 1, 3, "tile BR64  BC128 ST2  R4W5", 9);
    TILE(3, 128, 64, 1, 3, "tile BR64  BC128 ST3  R4W5", 9);
    TILE(4, 128, 64, 1, 3, "tile BR64  BC128 ST4  R4W5", 9);
    TILE(2, 256, 64, 1, 3, "tile BR64  BC256 ST2  R4W5", 9);
    TILE(4, 128, 32, 1, 3, "tile BR32  BC128 ST4  R4W5", 9);
    TILE(4, 256, 32, 1, 3, "tile BR32  BC256 ST4  R4W5", 9);
    TILE(8, 256, 16, 1, 3, "tile BR16  BC256 ST8  R4W5", 9);
    TILE(4, 256, 16, 1, 3, "tile BR16  BC256 ST4  R4W5", 9);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
    }
    if (getenv("WIDE")) {
    TILE(8, 32, 128, 1, 3, "tile BR128 BC32  ST8  R4W5", 9);
    TILE(4, 32, 128, 1, 3, "tile BR128 BC32  ST4  R4W5", 9);
    TILE(2, 64, 128, 1, 3, "tile BR128 BC64  ST2  R4W5", 9);
    TILE(3, 64, 128, 1, 3, "tile BR128 BC64  ST3  R4W5", 9);
    TILE(4, 64, 128, 1, 3, "tile BR128 BC64  ST4  R4W5", 9);
    TILE(6, 64, 128, 1, 3, "tile BR128 BC64  ST6  R4W5", 9);
    TILE(2, 128, 128, 1, 3, "tile BR128 BC128 ST2  R4W5", 9);
    TILE(3, 128, 128, 1, 3, "tile BR128 BC128 ST3  R4W5", 9);
    TILE(1, 256, 128, 1, 3, "tile BR128 BC256 ST1  R4W5", 9);
    TILE(4, 128, 64, 1, 3, "tile BR64  BC128 ST4  R4W5", 9);
    TILE(2, 256, 64, 1, 3, "tile BR64  BC256 ST2  R4W5", 9);
    TILE(4, 256, 32, 1, 3, "tile BR32  BC256 ST4  R4W5", 9);
    TILE(8, 256, 16, 1, 3, "tile BR16  BC256 ST8  R4W5", 9);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
    }
    if (getenv("DEPTH2")) {
    TILE(2, 32, 128, 1, 3, "tile BR128 BC32 ST2   R4W5", 9);
    TILE(3, 32, 128, 1, 3, "tile BR128 BC32 ST3   R4W5", 9);
    TILE(4, 32, 128, 1, 3, "tile BR128 BC32 ST4   R4W5", 9);
    TILE(5, 32, 128, 1, 3, "tile BR128 BC32 ST5   R4W5", 9);
    TILE(6, 32, 128, 1, 3, "tile BR128 BC32 ST6   R4W5", 9);
    TILE(8, 32, 128, 1, 3, "tile BR128 BC32 ST8   R4W5", 9);
    TILE(3, 32, 128, 0, 2, "tile BR128 BC32 ST3   W4 only", 4);
    TILE(4, 32, 128, 0, 2, "tile BR128 BC32 ST4   W4 only", 4);
    TILE(8, 32, 128, 0, 2, "tile BR128 BC32 ST8   W4 only", 4);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
    }
    if (getenv("DEPTH")) {
    TILE(4, 32, 128, 1, 3, "tile BR128 BC32 ST4   R4W5", 9);
    TILE(6, 32, 128, 1, 3, "tile BR128 BC32 ST6   R4W5", 9);
    TILE(8, 32, 128, 1, 3, "tile BR128 BC32 ST8   R4W5", 9);
    TILE(10, 32, 128, 1, 3, "tile BR128 BC32 ST10  R4W5", 9);
    TILE(12, 32, 128, 1, 3, "tile BR128 BC32 ST12  R4W5", 9);
    TILEW(8, 32, 128, 1, 3, 2, "tile BR128 BC32 ST8 WD2  R4W5", 9);
    TILEW(10, 32, 128, 1, 3, 2, "tile BR128 BC32 ST10 WD2 R4W5", 9);
    TILEW(12, 32, 128, 1, 3, 3, "tile BR128 BC32 ST12 WD3 R4W5", 9);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
    }
    if (getenv("GRP")) {
    GRP(1, 4, "tile grp G1 IL4 (current)  R4W5");
    GRP(2, 4, "tile grp G2 IL4            R4W5");
    GRP(4, 4, "tile grp G4 IL4            R4W5");
    GRP(8, 4, "tile grp G8 IL4            R4W5");
    GRP(2, 1, "tile grp G2 IL1            R4W5");
    GRP(4, 1, "tile grp G4 IL1            R4W5");
    GRP(8, 1, "tile grp G8 IL1            R4W5");
    GRP(16, 1, "tile grp G16 IL1           R4W5");
    GRP(37, 1, "tile grp G37 IL1           R4W5");
    GRP(74, 1, "tile grp G74 IL1           R4W5");
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
    }
    // round-1 session 3: tile height (rows written concurrently per CTA) and store L2 policy
    TILE(8, 32, 128, 1, 3, "tile BR128 BC32 (current)   R4W5", 9);
    TILE(16, 32, 64, 1, 3, "tile BR64  BC32             R4W5", 9);
    TILE(32, 32, 32, 1, 3, "tile BR32  BC32             R4W5", 9);
    TILE(64, 32, 16, 1, 3, "tile BR16  BC32             R4W5", 9);
    TILE(8, 32, 128, 0, 3, "tile BR128 BC32 no codes    R4W4", 8);
    TILE(16, 32, 64, 0, 3, "tile BR64  BC32 no codes    R4W4", 8);
    TILE(32, 32, 32, 0, 3, "tile BR32  BC32 no codes    R4W4", 8);
    TILE(8, 32, 128, 0, 2, "tile BR128 BC32 write only  W4", 4);
    TILE(16, 32, 64, 0, 2, "tile BR64  BC32 write only  W4", 4);
    TILE(32, 32, 32, 0, 2, "tile BR32  BC32 write only  W4", 4);
    TILE(64, 32, 16, 0, 2, "tile BR16  BC32 write only  W4", 4);
    {
        const int64_t nb = N / (256 * 2 * 4);
        timeit("linear grid R4W5 (reference)", 9, [&] { lin_grid<2, 1, 1><<<nb, 256>>>(in4, ok4, oc4, n4); });
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
