// scores_codes.cu — NEXT-2: raw attention scores straight from the
// compressed cache, on the tcgen05 tensor cores.
//
//   S'[i][t] = sum_d Q[i][d] * K_hat[t][d],  K_hat[t][d] = q[t][d] * s_d   (Eq. 8)
//            = sum_d W[i][d] * q[t][d],       W[i][d] = Q[i][d] * s_d
//
// The int8 codes are exact in bf16 (|q| <= 127 needs 7 bits), so the contraction
// runs as kind::f16 with bf16 operands: A = codes (converted on chip, from TMEM),
// B = W split into bf16 hi + lo (|W - hi - lo| <= 2^-18 |W|), fp32 accumulation
// in TMEM restarted every CHUNK_KB K-blocks and carried in fp64 (the tensor
// core's fp32 accumulation truncates).  HBM traffic is the 1 byte/element of
// the codes (vs 4 for K_hat): the cache is scored without being dequantized.
//
// Persistent CTA per SM, 128 token rows per tile, 128 code columns per K-block:
//   warp 0   TMA of [128 x 128] int8 code boxes (128B swizzle) into a 4-stage ring
//   warp 3   1-D bulk copies of the pre-split W tile (hi+lo, 2 x 16 KB) into a 3-stage ring
//   warp 1   16 x tcgen05.mma.kind::f16 (M=128, N=64, K=16) per K-block
//   warps 4-11  converters: int8 -> bf16 pairs, tcgen05.st into a 4-stage A ring in TMEM
//   warps 12-15 epilogue: fp64 carry of each chunk, store S' [nq][T] fp32
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <mutex>

#include "kvq_internal.h"
#include "tc_common.cuh"

namespace kvq {
namespace sc {

using namespace tc;

constexpr int BM = 128, BN = 64, BKC = 128;  // rows, queries, code columns per K-block
constexpr int KST = 4, WST = 3, AST = 4;
constexpr int NTHREADS = 512, NCONV = 256, CONV_W0 = 4, EPI_W0 = 12;
constexpr int CHUNK_KB = 2;                       // K-blocks per TMEM accumulation chunk (256 columns)
constexpr uint32_t CTILE = BM * BKC;              // 16 KB of codes
constexpr uint32_t WTILE = BN * BKC * 2;          // 16 KB of bf16 (one of hi/lo)
constexpr uint32_t TMEM_COLS = 512;               // acc 2 x 64 | A ring AST x 64 (packed bf16 pairs)
constexpr uint32_t A_COL0 = 128;
// kind::f16 instruction descriptor: D f32, A bf16, B bf16, K-major, M x N
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

struct __align__(1024) Smem {
    uint8_t c[KST][CTILE];
    uint8_t w[WST][2 * WTILE];
    uint64_t full_c[KST], empty_c[KST], full_w[WST], empty_w[WST];
    uint64_t full_a[AST], empty_a[AST], full_acc[2], empty_acc[2];
    uint32_t tmem_base;
};
static_assert(sizeof(Smem) <= 227 * 1024, "shared memory budget");

// W = Q * s split into bf16 hi + lo, per K-block kb: [hi | lo] tiles of BN x BKC
// in the canonical K-major SWIZZLE_NONE layout (core matrix = 8 rows x 16 B =
// 8 bf16 along K): core (kg = k/8, rg = n/8) at byte (kg*8 + rg)*128, row n%8 at
// +16*(n%8), element k%8 at +2*(k%8).  Rows >= nq and columns >= D are zero.
__global__ void wsplit_kernel(const float *__restrict__ Q, const float *__restrict__ scales, int64_t nq, int64_t D,
                              int64_t nkb, __nv_bfloat16 *__restrict__ out) {
    const int64_t total = nkb * BN * BKC;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t kb = i / (BN * BKC);
        const int rem = (int)(i % (BN * BKC));
        const int n = rem / BKC, k = rem % BKC;
        const int64_t col = kb * BKC + k;
        const float w = (n < nq && col < D) ? __fmul_rn(Q[n * D + col], scales[col]) : 0.0f;
        const __nv_bfloat16 hi = __float2bfloat16_rn(w);
        const __nv_bfloat16 lo = __float2bfloat16_rn(__fsub_rn(w, __bfloat162float(hi)));
        const int off = ((k / 8) * 8 + n / 8) * 64 + (n % 8) * 8 + (k % 8);  // in bf16 elements
        __nv_bfloat16 *tile = out + kb * (2 * BN * BKC);
        tile[off] = hi;
        tile[BN * BKC + off] = lo;
    }
}

__device__ __forceinline__ uint32_t swz(uint32_t base, int r, int c) { return base + r * 128 + ((c ^ (r & 7)) << 4); }

// 4 int8 codes (bytes of w) -> 2 packed bf16 pairs (exact)
__device__ __forceinline__ void codes4_to_bf16(uint32_t w, uint32_t &p0, uint32_t &p1) {
    const float f0 = (float)(int)(int8_t)(w & 0xffu), f1 = (float)(int)(int8_t)((w >> 8) & 0xffu);
    const float f2 = (float)(int)(int8_t)((w >> 16) & 0xffu), f3 = (float)(int)(int8_t)(w >> 24);
    const __nv_bfloat162 a = __floats2bfloat162_rn(f0, f1), b = __floats2bfloat162_rn(f2, f3);  // .x = low half
    p0 = *reinterpret_cast<const uint32_t *>(&a);
    p1 = *reinterpret_cast<const uint32_t *>(&b);
}

struct ScParams {
    const __nv_bfloat16 *wsplit;
    float *S;
    int64_t T;
    int nq, ntiles, nkb;
};

__global__ void __launch_bounds__(NTHREADS, 1)
    scores_codes_kernel(const __grid_constant__ CUtensorMap tmC, const __grid_constant__ ScParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem &s = *reinterpret_cast<Smem *>(smem_raw);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int ntiles = p.ntiles, nkb = p.nkb;
    if (threadIdx.x == 0) {
        if (smem_u32(smem_raw) & 1023u) __trap();
        for (int i = 0; i < KST; i++) {
            mbar_init(&s.full_c[i], 1);
            mbar_init(&s.empty_c[i], NCONV);
        }
        for (int i = 0; i < WST; i++) {
            mbar_init(&s.full_w[i], 1);
            mbar_init(&s.empty_w[i], 1);
        }
        for (int i = 0; i < AST; i++) {
            mbar_init(&s.full_a[i], NCONV);
            mbar_init(&s.empty_a[i], 1);
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(&s.full_acc[i], 1);
            mbar_init(&s.empty_acc[i], 128);
        }
        mbar_fence_init();
    }
    if (warp == 0 && lane == 0) prefetch_tmap(&tmC);
    if (warp == 1) tmem_alloc<TMEM_COLS>(&s.tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = s.tmem_base;

    if (warp < CONV_W0) {
        setmaxnreg_dec<56>();
        if (warp == 0 && lane == 0) {
            // ---- code producer (HBM stream)
            const uint64_t pol = policy_evict_first();
            uint32_t g = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
                for (int kb = 0; kb < nkb; kb++, g++) {
                    const int sk = g % KST;
                    mbar_wait_lazy(&s.empty_c[sk], ((g / KST) & 1) ^ 1);
                    mbar_arrive_tx(&s.full_c[sk], CTILE);
                    tma_load_2d(s.c[sk], &tmC, &s.full_c[sk], kb * BKC, tile * BM, pol);
                }
        } else if (warp == 3 && lane == 0) {
            // ---- W producer (L2-resident tiles)
            const uint64_t pol = policy_evict_last();
            uint32_t g = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
                for (int kb = 0; kb < nkb; kb++, g++) {
                    const int sw = g % WST;
                    mbar_wait_lazy(&s.empty_w[sw], ((g / WST) & 1) ^ 1);
                    mbar_arrive_tx(&s.full_w[sw], 2 * WTILE);
                    bulk_load(s.w[sw], p.wsplit + (size_t)kb * (2 * BN * BKC), 2 * WTILE, &s.full_w[sw], pol);
                }
        } else if (warp == 1 && lane == 0) {
            // ---- MMA issuer
            uint32_t g = 0, gc = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
                for (int kb = 0; kb < nkb; kb++, g++) {
                    const int ab = gc & 1;
                    const uint32_t d = tbase + ab * BN;
                    const bool first = (kb % CHUNK_KB) == 0;
                    const bool last = (kb % CHUNK_KB) == CHUNK_KB - 1 || kb == nkb - 1;
                    if (first) {
                        mbar_wait(&s.empty_acc[ab], ((gc >> 1) & 1) ^ 1);
                        tc_fence_after();
                    }
                    const int sa = g % AST, sw = g % WST;
                    mbar_wait(&s.full_a[sa], (g / AST) & 1);
                    mbar_wait(&s.full_w[sw], (g / WST) & 1);
                    tc_fence_after();
                    const uint32_t a0 = tbase + A_COL0 + sa * 64;
                    const uint32_t whi = smem_u32(s.w[sw]), wlo = whi + WTILE;
#pragma unroll
                    for (int j = 0; j < BKC / 16; j++) {
                        // K-step j: 16 bf16 = k-groups 2j, 2j+1 (LBO 1024 B apart), 8-row groups 128 B apart;
                        // A: 8 packed TMEM columns per K-step
                        const uint64_t bh = smem_desc(whi + j * 2048, 1024, 128);
                        const uint64_t bl = smem_desc(wlo + j * 2048, 1024, 128);
                        mma_f16_ts(d, a0 + 8 * j, bh, IDESC, (!first || j != 0) ? 1u : 0u);
                        mma_f16_ts(d, a0 + 8 * j, bl, IDESC, 1);
                    }
                    mma_commit(&s.empty_a[sa]);
                    mma_commit(&s.empty_w[sw]);
                    if (last) {
                        mma_commit(&s.full_acc[ab]);
                        gc++;
                    }
                }
        }
    } else if (warp < EPI_W0) {
        // ---- converters: thread = (row r, half h): codes 64h..64h+63 of the K-block
        const int quarter = warp & 3, h = (warp - CONV_W0) >> 2;
        const int r = quarter * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        uint32_t g = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
            for (int kb = 0; kb < nkb; kb++, g++) {
                const int sk = g % KST;
                mbar_wait(&s.full_c[sk], (g / KST) & 1);
                const uint32_t cb = smem_u32(s.c[sk]);
                uint32_t a[32];
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    const float4 v = lds128(swz(cb, r, 4 * h + c));
                    const uint32_t w4[4] = {__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z),
                                            __float_as_uint(v.w)};
#pragma unroll
                    for (int u = 0; u < 4; u++) codes4_to_bf16(w4[u], a[8 * c + 2 * u], a[8 * c + 2 * u + 1]);
                }
                mbar_arrive(&s.empty_c[sk]);
                const int sa = g % AST;
                mbar_wait(&s.empty_a[sa], ((g / AST) & 1) ^ 1);
                tc_fence_after();
                tmem_st32(tbase + lane_off + A_COL0 + sa * 64 + 32 * h, a);
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(&s.full_a[sa]);
            }
    } else {
        // ---- epilogue
        setmaxnreg_inc<200>();
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        const int nchunks = (nkb + CHUNK_KB - 1) / CHUNK_KB;
        uint32_t gc = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            double acc[BN];
#pragma unroll
            for (int j = 0; j < BN; j++) acc[j] = 0.0;
            for (int c = 0; c < nchunks; c++, gc++) {
                const int ab = gc & 1;
                mbar_wait_lazy(&s.full_acc[ab], (gc >> 1) & 1);
                tc_fence_after();
                uint32_t v[32];
#pragma unroll
                for (int hh = 0; hh < BN / 32; hh++) {
                    tmem_ld32(tbase + lane_off + ab * BN + 32 * hh, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; j++) acc[32 * hh + j] += (double)__uint_as_float(v[j]);
                }
                tc_fence_before();
                mbar_arrive(&s.empty_acc[ab]);
            }
            const int64_t row = (int64_t)tile * BM + r;
            if (row < p.T) {
#pragma unroll
                for (int j = 0; j < BN; j++)
                    if (j < p.nq) p.S[(int64_t)j * p.T + row] = (float)acc[j];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<TMEM_COLS>(tbase);
    }
}

// Reference-shaped CUDA-core path for shapes the tensor-core kernel does not take
// (nq > 64, D % 16 != 0, unaligned codes): one thread per score, fp64 sum.
__global__ void scores_codes_simt_kernel(const float *__restrict__ Q, const int8_t *__restrict__ Kq,
                                         const float *__restrict__ scales, int64_t nq, int64_t T, int64_t D,
                                         float *__restrict__ S) {
    const int64_t total = nq * T;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = o / T, t = o % T;
        double acc = 0.0;
        for (int64_t d = 0; d < D; d++)
            acc += (double)__fmul_rn(Q[i * D + d], scales[d]) * (double)Kq[t * D + d];
        S[i * T + t] = (float)acc;
    }
}

}  // namespace sc

size_t scores_codes_workspace_size(int64_t D) {
    return (size_t)((D + sc::BKC - 1) / sc::BKC) * 2 * sc::WTILE + 256;
}

kvq_status launch_scores_codes(const float *Q, int64_t nq, const int8_t *Kq, const float *scales, int64_t T,
                               int64_t D, float *S, void *ws, size_t ws_bytes, cudaStream_t s) {
    using namespace sc;
    const bool tc = ws && ws_bytes >= scores_codes_workspace_size(D) && nq >= 1 && nq <= BN && D % 16 == 0 &&
                    (reinterpret_cast<uintptr_t>(Kq) % 16) == 0 && !force_simt();
    if (!tc) {
        const int64_t total = nq * T;
        scores_codes_simt_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 65535), 256, 0, s>>>(
            Q, Kq, scales, nq, T, D, S);
        return check_launch("scores_codes_simt");
    }
    static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
        cudaDriverEntryPointQueryResult q;
        void *ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
        }
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }();
    if (!enc) return fail(KVQ_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap mC;
    cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)T};
    cuuint64_t strides[1] = {(cuuint64_t)D};
    cuuint32_t box[2] = {BKC, BM};
    cuuint32_t estr[2] = {1, 1};
    if (enc(&mC, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t *>(Kq), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return fail(KVQ_ERR_CUDA, "cuTensorMapEncodeTiled(Kq) failed");
    const int64_t nkb = (D + BKC - 1) / BKC;
    __nv_bfloat16 *wsplit =
        reinterpret_cast<__nv_bfloat16 *>((reinterpret_cast<uintptr_t>(ws) + 255) & ~(uintptr_t)255);
    {
        const int64_t total = nkb * BN * BKC;
        wsplit_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 4096), 256, 0, s>>>(Q, scales, nq, D, nkb,
                                                                                         wsplit);
        if (kvq_status st = check_launch("wsplit"); st != KVQ_OK) return st;
    }
    ScParams p{wsplit, S, T, (int)nq, (int)((T + BM - 1) / BM), (int)nkb};
    const int grid = std::min(p.ntiles, device_info().num_sms);
    static std::once_flag once;
    std::call_once(once, [] {
        cudaFuncSetAttribute(scores_codes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
    });
    scores_codes_kernel<<<grid, NTHREADS, sizeof(Smem), s>>>(mC, p);
    return check_launch("scores_codes");
}

}  // namespace kvq
