// attn_tc.cu — a5 + a6 on the 5th-generation tensor cores (tcgen05, TMEM, TMA).
//
// The attention-score error is a real dense contraction:
//     Delta[t][i] = sum_d E[t][d] * Q[i][d],   E = K - K_hat   (exact in fp32)
// with M = tokens, N = nq = 64 queries, K = D.  It runs on tcgen05 with fp32
// accuracy via the 3xTF32 split: E = E_hi + E_lo, Q = Q_hi + Q_lo (each part
// rounded to tf32), Delta = E_hi Q_hi + E_hi Q_lo + E_lo Q_hi (the dropped
// E_lo Q_lo term is ~2^-22 relative), accumulated in fp32 in TMEM.
//
// One persistent CTA per SM walks 128-row tiles; per 32-column K-block:
//   warp 0 (1 lane)  TMA: K and K_hat boxes [128 x 32] fp32 (128B swizzle) into a
//                    4-stage ring; 1-D bulk copy of the pre-split Q tile (hi+lo,
//                    16 KB, already in the canonical UMMA layout) into a 4-stage ring.
//   warps 2..5       converters, one token row per thread: read K/K_hat row
//                    segments from smem, E = K - K_hat, accumulate sum E^2 (fp64)
//                    and max |E| (a5), split E into tf32 hi/lo and tcgen05.st them
//                    into a 2-stage A ring in TMEM (A operand read from TMEM: no
//                    smem bandwidth for the 3 reads of E).
//   warp 1 (1 lane)  issues 3 x 4 tcgen05.mma (M=128, N=64, K=8) per K-block into a
//                    double-buffered TMEM accumulator, restarted every CHUNK_KB
//                    K-blocks, and commits to the barriers.
//   warps 6..9       epilogue, one row per thread: tcgen05.ld each finished
//                    [128 x 64] fp32 chunk accumulator and add it into fp64
//                    registers; at the end of a tile sum |Delta| (fp64) or store S.
// The tensor core's fp32 accumulation is not round-to-nearest: accumulating all
// D/8 * 3 MMA steps of D = 8192 in TMEM biased |Delta| by ~5e-5 (measured on
// B200).  Restarting the accumulator every 128 columns (48 MMA steps) and
// carrying the chunk sums in fp64 keeps the error ~1e-6.
// HBM traffic is the 8 bytes/element of K and K_hat read once (Q stays in L2).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "device_common.cuh"
#include "kvq_internal.h"
#include "tc_common.cuh"

namespace kvq {
namespace tc {

constexpr int BM = 128, BN = 64, BK = 32;
constexpr int KST = 4, QST = 4, AST = 2;
constexpr int NTHREADS = 320;
constexpr int CHUNK_KB = 4;  // K-blocks (of 32 columns) per TMEM accumulation chunk
constexpr uint32_t KTILE = BM * BK * 4;  // 16 KB
constexpr uint32_t QTILE = BN * BK * 4;  // 8 KB (one of hi/lo)
constexpr uint32_t TMEM_COLS = 256;      // acc 2 x 64 | A ring 2 x (hi 32 + lo 32)
constexpr uint32_t A_COL0 = 128;
constexpr uint32_t IDESC = idesc_tf32(BM, BN);

struct __align__(1024) Smem {
    uint8_t k[KST][KTILE];
    uint8_t kh[KST][KTILE];
    uint8_t q[QST][2 * QTILE];
    uint64_t full_k[KST], empty_k[KST], full_q[QST], empty_q[QST];
    uint64_t full_a[AST], empty_a[AST], full_acc[2], empty_acc[2];
    uint32_t tmem_base;
    double red[3][4];
};

// Q [nq][D] -> per K-block kb: [hi | lo] tiles of BN x BK tf32 in the canonical
// K-major SWIZZLE_NONE layout: core matrix (kg = k/4, rg = n/8) at byte
// (kg*8 + rg)*128, row n%8 at +16*(n%8), element k%4 at +4*(k%4).  Rows >= nq
// and columns >= D are zero.
__global__ void qsplit_kernel(const float *__restrict__ Q, int64_t nq, int64_t D, int64_t nkb,
                              uint32_t *__restrict__ out) {
    const int64_t total = nkb * BN * BK;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t kb = i / (BN * BK);
        const int rem = (int)(i % (BN * BK));
        const int n = rem / BK, k = rem % BK;
        const int64_t col = kb * BK + k;
        const float q = (n < nq && col < D) ? Q[n * D + col] : 0.0f;
        const uint32_t hi = to_tf32(q);
        const uint32_t lo = to_tf32(q - __uint_as_float(hi));
        const uint32_t off = ((k / 4) * 8 + n / 8) * 32 + (n % 8) * 4 + (k % 4);  // in 4-byte words
        uint32_t *tile = out + kb * (2 * BN * BK);
        tile[off] = hi;
        tile[BN * BK + off] = lo;
    }
}

template <int MODE>  // 0: metrics partials (E = K - K_hat), 1: scores S[i][t] (E = K or K - K_hat)
__global__ void __launch_bounds__(NTHREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmKh,
                   const uint32_t *__restrict__ qsplit, int64_t T, int nq, int ntiles, int nkb, int has_khat,
                   Partial *__restrict__ partials, float *__restrict__ S) {
    extern __shared__ uint8_t smem_raw[];
    Smem &s = *reinterpret_cast<Smem *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

    if (threadIdx.x == 0) {
        for (int i = 0; i < KST; i++) {
            mbar_init(&s.full_k[i], 1);
            mbar_init(&s.empty_k[i], 128);
        }
        for (int i = 0; i < QST; i++) {
            mbar_init(&s.full_q[i], 1);
            mbar_init(&s.empty_q[i], 1);
        }
        for (int i = 0; i < AST; i++) {
            mbar_init(&s.full_a[i], 128);
            mbar_init(&s.empty_a[i], 1);
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(&s.full_acc[i], 1);
            mbar_init(&s.empty_acc[i], 128);
        }
        mbar_fence_init();
    }
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmK);
        if (has_khat) prefetch_tmap(&tmKh);
    }
    if (warp == 1) tmem_alloc<TMEM_COLS>(&s.tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = s.tmem_base;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            const uint64_t pol_stream = policy_evict_first();
            const uint64_t pol_q = policy_evict_last();
            (void)pol_q;
            const uint32_t kbytes = has_khat ? 2 * KTILE : KTILE;
            uint32_t g = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (int kb = 0; kb < nkb; kb++, g++) {
                    const int sk = g % KST;
                    const uint32_t pk = (g / KST) & 1;
                    mbar_wait(&s.empty_k[sk], pk ^ 1);
                    mbar_arrive_tx(&s.full_k[sk], kbytes);
                    tma_load_2d(s.k[sk], &tmK, &s.full_k[sk], kb * BK, tile * BM, pol_stream);
                    if (has_khat) tma_load_2d(s.kh[sk], &tmKh, &s.full_k[sk], kb * BK, tile * BM, pol_stream);
                    const int sq = g % QST;
                    const uint32_t pq = (g / QST) & 1;
                    mbar_wait(&s.empty_q[sq], pq ^ 1);
                    mbar_arrive_tx(&s.full_q[sq], 2 * QTILE);
                    bulk_load(s.q[sq], qsplit + (size_t)kb * (2 * BN * BK), 2 * QTILE, &s.full_q[sq]);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            uint32_t g = 0, gc = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                for (int kb = 0; kb < nkb; kb++, g++) {
                    const int ab = gc & 1;
                    const uint32_t d = tbase + ab * BN;
                    const bool chunk_first = (kb % CHUNK_KB) == 0;
                    const bool chunk_last = (kb % CHUNK_KB) == CHUNK_KB - 1 || kb == nkb - 1;
                    if (chunk_first) {
                        mbar_wait(&s.empty_acc[ab], ((gc >> 1) & 1) ^ 1);
                        tc_fence_after();
                    }
                    const int sa = g % AST, sq = g % QST;
                    mbar_wait(&s.full_a[sa], (g / AST) & 1);
                    mbar_wait(&s.full_q[sq], (g / QST) & 1);
                    tc_fence_after();
                    const uint32_t ahi = tbase + A_COL0 + sa * 64, alo = ahi + 32;
                    const uint32_t qhi = smem_u32(s.q[sq]), qlo = qhi + QTILE;
#pragma unroll
                    for (int j = 0; j < BK / 8; j++) {
                        // K-step j covers k-groups 2j, 2j+1 (LBO apart = 1024 B), 8-row groups 128 B apart
                        const uint64_t bh = smem_desc(qhi + j * 2048, 1024, 128);
                        const uint64_t bl = smem_desc(qlo + j * 2048, 1024, 128);
                        mma_tf32_ts(d, ahi + 8 * j, bh, IDESC, (!chunk_first || j != 0) ? 1u : 0u);
                        mma_tf32_ts(d, ahi + 8 * j, bl, IDESC, 1);
                        mma_tf32_ts(d, alo + 8 * j, bh, IDESC, 1);
                    }
                    mma_commit(&s.empty_a[sa]);
                    mma_commit(&s.empty_q[sq]);
                    if (chunk_last) {
                        mma_commit(&s.full_acc[ab]);
                        gc++;
                    }
                }
            }
        }
    } else if (warp < 6) {
        // ------------------------------------------------------------ converters (warps 2..5)
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;  // row of the tile == TMEM lane
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        double ss = 0.0;
        float mx = 0.0f;
        uint32_t g = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            for (int kb = 0; kb < nkb; kb++, g++) {
                const int sk = g % KST;
                mbar_wait(&s.full_k[sk], (g / KST) & 1);
                const uint8_t *kr = s.k[sk] + r * 128;
                const uint8_t *hr = s.kh[sk] + r * 128;
                float e[32];
#pragma unroll
                for (int c = 0; c < 8; c++) {
                    const int pos = (c ^ (r & 7)) << 4;  // 128B swizzle: chunk c of row r
                    const float4 a = *reinterpret_cast<const float4 *>(kr + pos);
                    float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (has_khat) b = *reinterpret_cast<const float4 *>(hr + pos);
                    e[4 * c + 0] = __fsub_rn(a.x, b.x);
                    e[4 * c + 1] = __fsub_rn(a.y, b.y);
                    e[4 * c + 2] = __fsub_rn(a.z, b.z);
                    e[4 * c + 3] = __fsub_rn(a.w, b.w);
                }
                mbar_arrive(&s.empty_k[sk]);
                if (MODE == 0) {
                    // each e^2 is exact in fp64; 32 of them summed in fp64 per block
                    double blk = 0.0;
#pragma unroll
                    for (int i = 0; i < 32; i++) {
                        const double ed = (double)e[i];
                        blk = fma(ed, ed, blk);
                        mx = fmaxf(mx, fabsf(e[i]));
                    }
                    ss += blk;
                }
                uint32_t hi[32], lo[32];
#pragma unroll
                for (int i = 0; i < 32; i++) {
                    hi[i] = to_tf32(e[i]);
                    lo[i] = to_tf32(__fsub_rn(e[i], __uint_as_float(hi[i])));
                }
                const int sa = g % AST;
                mbar_wait(&s.empty_a[sa], ((g / AST) & 1) ^ 1);
                tc_fence_after();
                tmem_st32(tbase + lane_off + A_COL0 + sa * 64, hi);
                tmem_st32(tbase + lane_off + A_COL0 + sa * 64 + 32, lo);
                tmem_wait_st();
                tc_fence_before();
                mbar_arrive(&s.full_a[sa]);
            }
        }
        if (MODE == 0) {
            double mxd = (double)mx;
            for (int o = 16; o > 0; o >>= 1) {
                ss += __shfl_xor_sync(0xffffffffu, ss, o);
                mxd = fmax(mxd, __shfl_xor_sync(0xffffffffu, mxd, o));
            }
            if (lane == 0) {
                s.red[0][quarter] = ss;
                s.red[2][quarter] = mxd;
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue (warps 6..9)
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        double attn = 0.0;
        uint32_t gc = 0;
        const int nchunks = (nkb + CHUNK_KB - 1) / CHUNK_KB;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            double acc[BN];
#pragma unroll
            for (int j = 0; j < BN; j++) acc[j] = 0.0;
            for (int c = 0; c < nchunks; c++, gc++) {
                const int ab = gc & 1;
                mbar_wait(&s.full_acc[ab], (gc >> 1) & 1);
                tc_fence_after();
                uint32_t v[32];
#pragma unroll
                for (int h = 0; h < BN / 32; h++) {
                    tmem_ld32(tbase + lane_off + ab * BN + 32 * h, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; j++) acc[32 * h + j] += (double)__uint_as_float(v[j]);
                }
                tc_fence_before();
                mbar_arrive(&s.empty_acc[ab]);
            }
            const int64_t row = (int64_t)tile * BM + r;
            if (row < T) {
#pragma unroll
                for (int j = 0; j < BN; j++) {
                    if (j < nq) {
                        if (MODE == 0)
                            attn += fabs(acc[j]);
                        else
                            S[(int64_t)j * T + row] = (float)acc[j];
                    }
                }
            }
        }
        if (MODE == 0) {
            for (int o = 16; o > 0; o >>= 1) attn += __shfl_xor_sync(0xffffffffu, attn, o);
            if (lane == 0) s.red[1][quarter] = attn;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (MODE == 0 && threadIdx.x == 0) {
        Partial p{0.0, 0.0, 0.0, 0.0};
        for (int i = 0; i < 4; i++) {  // fixed order: deterministic
            p.sum_sq += s.red[0][i];
            p.attn_abs += s.red[1][i];
            p.max_abs = fmax(p.max_abs, s.red[2][i]);
        }
        partials[blockIdx.x] = p;
    }
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<TMEM_COLS>(tbase);
    }
}

// ---------------------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
        cudaGetLastError();
    });
    return fn;
}

static bool make_map(CUtensorMap *m, const float *base, int64_t T, int64_t D) {
    auto enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)T};
    cuuint64_t strides[1] = {(cuuint64_t)D * 4};
    cuuint32_t box[2] = {BK, BM};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace tc

bool tc_eligible(const float *K, const float *K_hat, int64_t T, int64_t D, int64_t nq) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(K) | reinterpret_cast<uintptr_t>(K_hat);
    return nq >= 1 && nq <= tc::BN && D % 4 == 0 && (a % 16) == 0 && (T + tc::BM - 1) / tc::BM < (1LL << 31) &&
           tc::encode_fn() != nullptr;
}

size_t tc_qsplit_bytes(int64_t D) { return (size_t)((D + tc::BK - 1) / tc::BK) * 2 * tc::QTILE; }

// Launch: qsplit (into ws_q) + the persistent tensor-core kernel.
kvq_status launch_attn_tc(int mode, const float *K, const float *K_hat, int64_t T, int64_t D, const float *Q,
                          int64_t nq, void *ws_q, void *partials, int *grid_out, float *S, cudaStream_t s) {
    using namespace tc;
    const int64_t nkb = (D + BK - 1) / BK;
    const int ntiles = (int)((T + BM - 1) / BM);
    CUtensorMap mK, mKh;
    if (!make_map(&mK, K, T, D)) return fail(KVQ_ERR_CUDA, "cuTensorMapEncodeTiled(K) failed");
    if (K_hat) {
        if (!make_map(&mKh, K_hat, T, D)) return fail(KVQ_ERR_CUDA, "cuTensorMapEncodeTiled(K_hat) failed");
    } else {
        mKh = mK;
    }
    uint32_t *qs = reinterpret_cast<uint32_t *>(ws_q);
    {
        const int64_t total = nkb * BN * BK;
        const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 4096);
        qsplit_kernel<<<blocks, 256, 0, s>>>(Q, nq, D, nkb, qs);
        if (kvq_status st = check_launch("qsplit"); st != KVQ_OK) return st;
    }
    const int grid = std::min(ntiles, device_info().num_sms);
    const size_t smem = sizeof(Smem) + 1024;
    if (grid_out) *grid_out = grid;
    if (mode == 0) {
        static std::once_flag once;
        std::call_once(once, [&] {
            cudaFuncSetAttribute(attn_tc_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        });
        attn_tc_kernel<0><<<grid, NTHREADS, smem, s>>>(mK, mKh, qs, T, (int)nq, ntiles, (int)nkb, K_hat != nullptr,
                                                        reinterpret_cast<Partial *>(partials), nullptr);
    } else {
        static std::once_flag once;
        std::call_once(once, [&] {
            cudaFuncSetAttribute(attn_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        });
        attn_tc_kernel<1><<<grid, NTHREADS, smem, s>>>(mK, mKh, qs, T, (int)nq, ntiles, (int)nkb, K_hat != nullptr,
                                                        nullptr, S);
    }
    return check_launch(mode == 0 ? "attn_tc(metrics)" : "attn_tc(scores)");
}

}  // namespace kvq
