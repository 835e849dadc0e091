// scores_codes.cu — NEXT-2: raw attention scores straight from the
// compressed cache, on the tcgen05 integer tensor cores.
//
//   S'[i][t] = sum_d Q[i][d] * K_hat[t][d],  K_hat[t][d] = q[t][d] * s_d   (Eq. 8)
//            ~ sum_d W[i][d] * q[t][d],       W[i][d] = fl32(Q[i][d] * s_d)
//
// The codes are int8 already, so the contraction runs as tcgen05.mma.kind::i8
// (s8 x s8 -> s32, EXACT accumulation) with both operands straight from shared
// memory: A = the 128B-swizzled TMA box of codes, B = W written as NDIG = 4
// signed base-2^7 digits per query row i, with a per-row exponent E_i
// (max_d |W[i][d]| < 2^(E_i - 1)):
//   W[i][d] = 2^E_i * (w1 2^-7 + w2 2^-14 + w3 2^-21 + w4 2^-28) + e,
//   |w_k| <= 64,  |e| <= 2^(E_i - 29) < 2^-27 max_d |W[i][d]|,
// each digit the round-to-nearest of the (exact, fp64) remainder.  The digits
// stack along N (n = 64 k + i), one M=128 x N=256 x K=32 MMA per 32 code
// columns; the int32 accumulators cannot overflow for D <= 2^31 / (64 * 127)
// and are drained once per tile: S' = sum_k acc_k 2^(E_i - 7k) in fp64.  So the
// only approximation is e (bound in DESIGN.md §5); no fp32 tensor-core
// accumulation is involved.  HBM traffic is the 1 byte/element of the codes.
//
// Persistent CTA pairs (clusters of 2), 256 token rows per tile, 128 code columns per K-block:
//   warp 0      (both CTAs) TMA of the CTA's [128 x 128] code box (128B swizzle), KST ring
//   warp 2      (both CTAs) TMA of its [128 x 128] half of the digit tile, WST ring
//   warp 1      (leader) 4 x tcgen05.mma.cta_group::2.kind::i8 (M=256, N=256, K=32)
//               per K-block, one elected lane
//   warps 4-7   (both CTAs) epilogue: tcgen05.ld of the s32 accumulators, fp64
//               recombination, S' [nq][T] fp32 (coalesced along t)
// Rows of Q whose W is not finite take an exact fp64 per-element path in the epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <climits>
#include <mutex>

#include "kvq_internal.h"
#include "tc_common.cuh"

namespace kvq {
namespace sc {

using namespace tc;

constexpr int BM = 256, HM = 128;   // token rows per CTA-pair tile / per CTA
constexpr int NQ = 64, NDIG = 4, NB = NQ * NDIG, BKC = 128;  // queries, digits, MMA N, K-block
constexpr int KST = 8, WST = 5, NACC = 2;  // code ring (HBM latency) / digit ring (L2)
constexpr int NTHREADS = 256, EPI_W0 = 4;
constexpr uint32_t CTILE = HM * BKC;        // 16 KB of codes per CTA per K-block
constexpr uint32_t WHALF = (NB / 2) * BKC;  // 16 KB: this CTA's half (128 digit rows) of the B tile
constexpr uint32_t TMEM_COLS = 512;         // NACC x 256 s32 accumulator columns
static_assert(NACC * NB <= (int)TMEM_COLS, "TMEM budget");
constexpr int64_t MAX_D = (int64_t(1) << 31) / (64 * 127);  // s32 accumulators cannot overflow below this
// kind::i8 instruction descriptor: D s32, A s8, B s8, both K-major, M=256 (pair) x N=256
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NB >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

struct __align__(1024) Smem {
    uint8_t c[KST][CTILE];
    uint8_t w[WST][WHALF];
    double f[NDIG][NQ];  // 2^(E_i - 7(k+1))
    int bad[NQ];         // row i of W not finite -> exact per-element path
    uint64_t full_c[KST], empty_c[KST], full_w[WST], empty_w[WST], full_acc[NACC], empty_acc[NACC];
    uint32_t tmem_base;
};
static_assert(sizeof(Smem) <= 227 * 1024, "shared memory budget");

// Workspace: [nkb digit tiles of NB x BKC][f: NDIG x NQ double][bad: NQ int][E: NQ int]
struct WsLayout {
    size_t tiles, f, bad, e, total;
    explicit WsLayout(int64_t D) {
        const int64_t nkb = (D + BKC - 1) / BKC;
        tiles = 0;
        f = (size_t)nkb * NB * BKC;
        bad = f + sizeof(double) * NDIG * NQ;
        e = bad + sizeof(int) * NQ;
        total = e + sizeof(int) * NQ;
    }
};

__device__ __forceinline__ float w_elem(const float *Q, const float *scales, int64_t D, int i, int64_t d) {
    return __fmul_rn(Q[(int64_t)i * D + d], scales[d]);
}

// wmax: one block per query row i < NQ (rows >= nq: zero factors): m_i =
// max_d |W[i][d]|, whether the row is finite, E_i (m_i < 2^(E_i - 1)) and the
// recombination factors 2^(E_i - 7(k+1)).
constexpr int WMAX_THREADS = 512;
__global__ void __launch_bounds__(WMAX_THREADS) wmax_kernel(const float *__restrict__ Q,
                                                            const float *__restrict__ scales, int nq, int64_t D,
                                                            double *__restrict__ f, int *__restrict__ bad,
                                                            int *__restrict__ E) {
    const int i = blockIdx.x;
    float m = 0.0f;
    int nonfinite = 0;
    if (i < nq) {
#pragma unroll 4
        for (int64_t d = threadIdx.x; d < D; d += WMAX_THREADS) {
            const float w = w_elem(Q, scales, D, i, d);
            nonfinite |= !isfinite(w);
            m = isfinite(w) ? fmaxf(m, fabsf(w)) : m;
        }
    }
    __shared__ float sm[32];
    __shared__ int sb[32];
    for (int o = 16; o; o >>= 1) {
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        nonfinite |= __shfl_xor_sync(0xffffffffu, nonfinite, o);
    }
    if ((threadIdx.x & 31) == 0) {
        sm[threadIdx.x / 32] = m;
        sb[threadIdx.x / 32] = nonfinite;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < WMAX_THREADS / 32; k++) {
            m = fmaxf(m, sm[k]);
            nonfinite |= sb[k];
        }
        const int e = (m > 0.0f) ? ilogbf(m) + 2 : 0;  // m < 2^(e-1)
        for (int k = 0; k < NDIG; k++) f[k * NQ + i] = (m > 0.0f && !nonfinite) ? ldexp(1.0, e - 7 * (k + 1)) : 0.0;
        bad[i] = nonfinite;
        E[i] = (i < nq && !nonfinite) ? e : INT_MIN;  // INT_MIN: all-zero digits
    }
}

// wdigits: the digits, row-major: tile kb, row n = 64 k + i, byte k' (code
// column kb*128 + k') at (kb*256 + n)*128 + k' (consecutive threads write
// consecutive bytes).  The TMA applies the 128B swizzle on the way into shared
// memory.  Lets the scores kernel (launched as its programmatic dependent) start
// streaming codes while this runs.
__global__ void wdigits_kernel(const float *__restrict__ Q, const float *__restrict__ scales, int nq, int64_t D,
                               int64_t nkb, const int *__restrict__ E, int8_t *__restrict__ tiles) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int64_t Dp = nkb * BKC;
    const int64_t total = (int64_t)NQ * Dp;
    for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(o / Dp);
        const int64_t d = o % Dp;
        const int e = E[i];
        double x = (e != INT_MIN && d < D) ? ldexp((double)w_elem(Q, scales, D, i, d), -e) : 0.0;  // |x| < 1/2, exact
        const int64_t kb = d / BKC;
        const int kk = (int)(d % BKC);
#pragma unroll
        for (int k = 0; k < NDIG; k++) {
            const double y = x * 128.0;  // exact
            const double w = rint(y);    // |w| <= 64
            x = y - w;                   // exact, |x| <= 1/2
            tiles[(kb * NB + k * NQ + i) * BKC + kk] = (int8_t)(int)w;
        }
    }
}

struct ScParams {
    const double *f;
    const int *bad;
    const float *Q, *scales;
    const int8_t *Kq;
    float *S;
    int64_t T, D;
    int nq, ntiles, nkb;
};

// Cluster of 2 CTAs (an SM pair) per 256-row tile: each CTA TMA-loads its 128
// code rows and its half (digits 0-1 or 2-3) of the B tile; the leader issues
// cta_group::2 MMAs (M=256: A rows split over the pair, N=256: B rows split),
// which halves each SM's digit traffic (L2 reads, TMA writes into shared memory)
// against one CTA per 128-row tile.  Each CTA's TMEM holds its own 128 rows x 256
// columns of s32 accumulators, drained by its own epilogue.  The kernel is
// launched as the programmatic dependent of wdigits: only the digit producer and
// the epilogue wait (griddepcontrol.wait) for the prep kernels; codes stream at once.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NTHREADS, 1)
    scores_codes_kernel(const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmW,
                        const __grid_constant__ ScParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem &s = *reinterpret_cast<Smem *>(smem_raw);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = cluster_rank();
    const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
    const int ntiles = p.ntiles, nkb = p.nkb;
    if (threadIdx.x == 0) {
        if (smem_u32(smem_raw) & 1023u) __trap();
        for (int i = 0; i < KST; i++) {
            mbar_init(&s.full_c[i], 1);
            mbar_init(&s.empty_c[i], 1);
        }
        for (int i = 0; i < WST; i++) {
            mbar_init(&s.full_w[i], 1);
            mbar_init(&s.empty_w[i], 1);
        }
        for (int i = 0; i < NACC; i++) {
            mbar_init(&s.full_acc[i], 1);
            mbar_init(&s.empty_acc[i], 2 * 128);
        }
        mbar_fence_init();
    }
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmC);
        prefetch_tmap(&tmW);
    }
    if (warp == 1) tmem_alloc_pair<TMEM_COLS>(&s.tmem_base);
    tc_fence_before();
    __syncthreads();  // CTA-local order of the alloc's smem write (racecheck models bar.sync, not barrier.cluster)
    cluster_sync();   // peer barriers initialised before any remote arrive / TMA complete_tx
    tc_fence_after();
    const uint32_t tbase = s.tmem_base;

    if (warp < EPI_W0) {
        if (warp == 0 && lane == 0) {
            // ---- code producer (both CTAs, HBM stream); completion on the leader's barrier
            const uint64_t pol = policy_evict_first();
            uint32_t g = 0;
            for (int tile = pair; tile < ntiles; tile += npairs)
                for (int kb = 0; kb < nkb; kb++, g++) {
                    const int st = g % KST;
                    mbar_wait(&s.empty_c[st], ((g / KST) & 1) ^ 1);
                    if (rank == 0) mbar_arrive_tx(&s.full_c[st], 2 * CTILE);
                    tma_load_2d_pair(s.c[st], &tmC, mapa(smem_u32(&s.full_c[st]), 0), kb * BKC,
                                     tile * BM + (int)rank * HM, pol);
                }
        } else if (warp == 2 && lane == 0) {
            // ---- digit producer (both CTAs, L2-resident half tiles)
            asm volatile("griddepcontrol.wait;" ::: "memory");  // digit tiles written by wdigits
            const uint64_t pol = policy_evict_last();
            uint32_t g = 0;
            for (int tile = pair; tile < ntiles; tile += npairs)
                for (int kb = 0; kb < nkb; kb++, g++) {
                    const int st = g % WST;
                    mbar_wait(&s.empty_w[st], ((g / WST) & 1) ^ 1);
                    if (rank == 0) mbar_arrive_tx(&s.full_w[st], 2 * WHALF);
                    tma_load_2d_pair(s.w[st], &tmW, mapa(smem_u32(&s.full_w[st]), 0), 0,
                                     kb * NB + (int)rank * (NB / 2), pol);
                }
        } else if (warp == 1 && rank == 0) {
            // ---- MMA issuer (leader CTA): the whole warp waits, one elected lane issues
            uint32_t g = 0, lt = 0;
            for (int tile = pair; tile < ntiles; tile += npairs, lt++) {
                const int ab = lt % NACC;
                const uint32_t d = tbase + ab * NB;
                mbar_wait(&s.empty_acc[ab], ((lt / NACC) & 1) ^ 1);
                tc_fence_after();
                for (int kb = 0; kb < nkb; kb++, g++) {
                    const int sk = g % KST, sw = g % WST;
                    mbar_wait(&s.full_c[sk], (g / KST) & 1);
                    mbar_wait(&s.full_w[sw], (g / WST) & 1);
                    tc_fence_after();
                    const uint64_t a0 = smem_desc_sw128(smem_u32(s.c[sk]));
                    const uint64_t b0 = smem_desc_sw128(smem_u32(s.w[sw]));
                    if (elect_one()) {
#pragma unroll
                        for (int j = 0; j < BKC / 32; j++)  // K step j: 32 codes = 32 B inside the swizzle atom
                            mma_i8_ss_pair(d, a0 + (uint64_t)(2 * j), b0 + (uint64_t)(2 * j), IDESC,
                                           (kb != 0 || j != 0) ? 1u : 0u);
                        mma_commit_pair(&s.empty_c[sk], 0x3);
                        mma_commit_pair(&s.empty_w[sw], 0x3);
                        if (kb == nkb - 1) mma_commit_pair(&s.full_acc[ab], 0x3);
                    }
                    __syncwarp();
                }
            }
        }
    } else {
        // ---- epilogue (both CTAs): thread = token row r of this CTA's half tile
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        asm volatile("griddepcontrol.wait;" ::: "memory");  // factors written by wmax
        for (int k = threadIdx.x - EPI_W0 * 32; k < NDIG * NQ; k += 128) (&s.f[0][0])[k] = p.f[k];
        for (int k = threadIdx.x - EPI_W0 * 32; k < NQ; k += 128) s.bad[k] = p.bad[k];
        named_bar_sync(1, 128);
        uint32_t lt = 0;
        for (int tile = pair; tile < ntiles; tile += npairs, lt++) {
            const int ab = lt % NACC;
            mbar_wait_lazy(&s.full_acc[ab], (lt / NACC) & 1);
            tc_fence_after();
            double acc[NQ];
#pragma unroll
            for (int j = 0; j < NQ; j++) acc[j] = 0.0;
            uint32_t v[32];
#pragma unroll
            for (int k = 0; k < NDIG; k++)
#pragma unroll
                for (int hh = 0; hh < NQ / 32; hh++) {
                    tmem_ld32(tbase + lane_off + ab * NB + k * NQ + 32 * hh, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; j++)
                        acc[32 * hh + j] = fma((double)(int)v[j], s.f[k][32 * hh + j], acc[32 * hh + j]);
                }
            tc_fence_before();
            mbar_arrive_cluster(mapa(smem_u32(&s.empty_acc[ab]), 0));
            const int64_t row = (int64_t)tile * BM + (int64_t)rank * HM + r;
            if (row < p.T) {
#pragma unroll
                for (int j = 0; j < NQ; j++) {
                    if (j >= p.nq) break;
                    float out = (float)acc[j];
                    if (s.bad[j]) {  // non-finite W row: plain fp64 sum (inf/nan propagate as in the definition)
                        double e = 0.0;
                        for (int64_t dd = 0; dd < p.D; dd++)
                            e += (double)w_elem(p.Q, p.scales, p.D, j, dd) * (double)p.Kq[row * p.D + dd];
                        out = (float)e;
                    }
                    p.S[(int64_t)j * p.T + row] = out;
                }
            }
        }
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair<TMEM_COLS>(tbase);
    }
}

// Reference-shaped CUDA-core path for shapes the tensor-core kernel does not take
// (nq > 64, D % 16 != 0, D > MAX_D, unaligned codes): one thread per score, fp64 sum.
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

size_t scores_codes_workspace_size(int64_t D) { return sc::WsLayout(D).total + 1024; }

kvq_status launch_scores_codes(const float *Q, int64_t nq, const int8_t *Kq, const float *scales, int64_t T,
                               int64_t D, float *S, void *ws, size_t ws_bytes, cudaStream_t s) {
    using namespace sc;
    const bool tc = ws && ws_bytes >= scores_codes_workspace_size(D) && nq >= 1 && nq <= NQ && D % 16 == 0 &&
                    D <= MAX_D && (reinterpret_cast<uintptr_t>(Kq) % 16) == 0 && !force_simt();
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
    const int64_t nkb = (D + BKC - 1) / BKC;
    const WsLayout L(D);
    uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(ws) + 1023) & ~(uintptr_t)1023);
    int8_t *tiles = reinterpret_cast<int8_t *>(base + L.tiles);
    double *f = reinterpret_cast<double *>(base + L.f);
    int *bad = reinterpret_cast<int *>(base + L.bad);
    int *E = reinterpret_cast<int *>(base + L.e);
    auto map2d = [&](CUtensorMap *m, const void *ptr, uint64_t cols, uint64_t rows) {
        cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
        cuuint64_t strides[1] = {(cuuint64_t)cols};
        cuuint32_t box[2] = {BKC, HM};
        cuuint32_t estr[2] = {1, 1};
        return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    CUtensorMap mC, mW;
    if (!map2d(&mC, Kq, (uint64_t)D, (uint64_t)T)) return fail(KVQ_ERR_CUDA, "cuTensorMapEncodeTiled(Kq) failed");
    if (!map2d(&mW, tiles, BKC, (uint64_t)nkb * NB)) return fail(KVQ_ERR_CUDA, "cuTensorMapEncodeTiled(W) failed");
    wmax_kernel<<<NQ, WMAX_THREADS, 0, s>>>(Q, scales, (int)nq, D, f, bad, E);
    if (kvq_status st = check_launch("scores_codes_wmax"); st != KVQ_OK) return st;
    {
        const int64_t total = (int64_t)NQ * nkb * BKC;
        wdigits_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, 8192), 256, 0, s>>>(Q, scales, (int)nq, D,
                                                                                           nkb, E, tiles);
        if (kvq_status st = check_launch("scores_codes_wdigits"); st != KVQ_OK) return st;
    }
    ScParams p{f, bad, Q, scales, Kq, S, T, D, (int)nq, (int)((T + BM - 1) / BM), (int)nkb};
    const int grid = 2 * std::min(p.ntiles, device_info().num_sms / 2);
    ensure_max_smem<scores_codes_kernel>((int)sizeof(Smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(NTHREADS);
    cfg.dynamicSmemBytes = sizeof(Smem);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, scores_codes_kernel, mC, mW, p) != cudaSuccess) return check_launch("scores_codes");
    return check_launch("scores_codes");
}

}  // namespace kvq
