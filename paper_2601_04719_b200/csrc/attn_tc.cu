// attn_tc.cu — a5 + a6 (and the single-pass a3+a4+a5+a6) on the 5th-generation
// tensor cores (tcgen05, TMEM, TMA).
//
// The attention-score error is a real dense contraction:
//     Delta[t][i] = sum_d E[t][d] * Q[i][d],   E = K - K_hat   (exact in fp32)
// with M = tokens, N = nq <= 64 queries, K = D.  It runs on tcgen05 with fp32
// accuracy via the 3xTF32 split: E = E_hi + E_lo, Q = Q_hi + Q_lo (each part
// rounded to tf32), Delta = E_hi Q_hi + E_hi Q_lo + E_lo Q_hi (the dropped
// E_lo Q_lo term is ~2^-22 relative), accumulated in fp32 in TMEM.
//
// One persistent CTA per SM walks 128-row tiles; per 32-column K-block:
//   warp 0 (1 lane)  TMA: K (and K_hat) boxes [128 x 32] fp32 (128B swizzle) and,
//                    in the fused mode, the 32 per-column quantizer constants into
//                    a 4-stage ring; 1-D bulk copy of the pre-split Q tile (hi+lo,
//                    16 KB, already in the canonical UMMA layout) into a 4-stage ring.
//   warps 4..11      converters, one token row and 16 columns per thread (ld.shared):
//                    [fused mode: quantize (Eq. 7) + dequantize (Eq. 8) the row
//                    segment, stage codes and K_hat in swizzled smem and write them
//                    with TMA bulk tensor stores (full 128-byte lines: no DRAM
//                    read-modify-write for the 32-byte code segments)]
//                    E = K - K_hat, sum E^2 and max |E| (a5), split E into tf32
//                    hi/lo and tcgen05.st them into a 2-stage A ring in TMEM (the A
//                    operand is read from TMEM: no smem bandwidth for E's 3 reads).
//   warp 1 (1 lane)  issues 3 x 4 tcgen05.mma (M=128, N=64, K=8) per K-block into a
//                    double-buffered TMEM accumulator, restarted every CHUNK_KB
//                    K-blocks, and commits to the barriers.
//   warps 12..15     epilogue (registers raised with setmaxnreg), one row per thread: tcgen05.ld each finished
//                    [128 x 64] fp32 chunk accumulator and add it into fp64
//                    registers; at the end of a tile sum |Delta| (fp64) or store S.
// The tensor core's fp32 accumulation is not round-to-nearest: accumulating all
// D/8 * 3 MMA steps of D = 8192 in TMEM biased |Delta| by ~5e-5 (measured on
// B200).  Restarting the accumulator every 128 columns (48 MMA steps) and
// carrying the chunk sums in fp64 keeps the error ~1e-6.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "device_common.cuh"
#include "kvq_internal.h"
#include "tc_common.cuh"

namespace kvq {
namespace tc {

constexpr int BM = 128, BN = 64, BK = 32;
constexpr int QST = 4, AST = 4;
// Input ring: modes 0/1 stage K and K_hat (32 KB) x 4; the fused mode stages K only
// (16 KB) x 8, i.e. 128 KB in flight per SM either way (Little's law at ~44 GB/s/SM).
constexpr int KST_MAX = 8;
#ifndef KVQ_TC_KST2
#define KVQ_TC_KST2 8  // fused-mode ring depth (16 KB stages; experiments: -DKVQ_TC_KST2=4..8)
#endif
#ifndef KVQ_TC_KST01
#define KVQ_TC_KST01 4  // modes 0/1 ring depth (experiments: -DKVQ_TC_KST01=5 fills the 160 KB buffer)
#endif
template <int MODE>
struct Ring {
    static constexpr int kst = MODE == 2 ? KVQ_TC_KST2 : KVQ_TC_KST01;
    static constexpr uint32_t stage = MODE == 2 ? 16384u : 32768u;
};
// warps: 0 K producer, 1 MMA (+TMEM alloc), 2 output stores (fused mode), 3 Q producer, 4-11 converters (2 per TMEM lane
// quarter, 16 columns each), 12-15 epilogue.  Warpgroup 0 gives registers to the
// epilogue warpgroup (setmaxnreg), which keeps 64 fp64 accumulators per row.
#ifndef KVQ_TC_TEAMS
#define KVQ_TC_TEAMS 2
#endif
constexpr int NTEAMS = KVQ_TC_TEAMS;  // converter teams; team t converts the K-blocks g with g % NTEAMS == t
constexpr int NCONV = 256;            // converter threads per team
constexpr int NCONV_W = NCONV / 32;   // converter warps per team (one elected arrival per warp after __syncwarp)
constexpr int CONV_W0 = 4, EPI_W0 = CONV_W0 + NTEAMS * NCONV_W;
constexpr int NTHREADS = (EPI_W0 + 4) * 32;
// setmaxnreg budgets (64K registers per SM): warpgroup 0 (single-lane roles) and the epilogue warpgroup
// (setmaxnreg only moves registers within the CTA's launch allocation: NTHREADS x the launch count)
constexpr uint32_t REG_LAUNCH = 65536 / NTHREADS / 8 * 8;
constexpr uint32_t REG_WG0 = NTEAMS == 1 ? 56 : 48, REG_EPI = NTEAMS == 1 ? 200 : 80;
constexpr uint32_t REG_CONV = NTEAMS == 1 ? 128 : (REG_LAUNCH * (NTHREADS / 128) - REG_WG0 - REG_EPI) / (NTEAMS * 2) / 8 * 8;
static_assert(REG_WG0 + REG_EPI + REG_CONV * NTEAMS * 2 <= REG_LAUNCH * (NTHREADS / 128), "register budget");
constexpr int CHUNK_KB = 4;              // K-blocks (of 32 columns) per TMEM accumulation chunk
constexpr int CODE_KB = 4;               // K-blocks per code store (128 codes = one 128 B line per row)
constexpr uint32_t KTILE = BM * BK * 4;  // 16 KB
constexpr uint32_t QTILE = BN * BK * 4;  // 8 KB (one of hi/lo)
constexpr uint32_t TMEM_COLS = 512;      // acc 2 x 64 | A ring AST x (hi 32 + lo 32) (| 128 spare)
constexpr uint32_t A_COL0 = 128;
constexpr uint32_t ACC_COL0 = 384;       // two converter teams: the tile's Delta as fp32 (hi, lo) pairs (2 x 64 columns)
constexpr uint32_t IDESC = idesc_tf32(BM, BN);

// Per K-block quantizer record (fused mode): RN(1/s) and s of the 32 columns (as two arrays, so that
// adjacent columns form the fp32 pairs of the packed arithmetic) and a
// flag set when one of them needs the exact path for every element.
struct __align__(16) ColRec {
    float y[BK];  // RN(1/s) per column (0: zero scale or exact path)
    float s[BK];  // s per column
    uint32_t any_exact;
    uint32_t pad[3];
};

// Timeline trace of CTA 0 (experiments only, -DKVQ_TRACE): clock64 of event e at K-block g in [TR_G0, TR_G0 + TR_N).
#ifdef KVQ_TRACE
constexpr int TR_G0 = 64, TR_N = 64, TR_E = 48;  // events 16..31: each team warp's staged arrival; 32..47: its loads done
__device__ unsigned long long g_kvq_trace[TR_N][TR_E];
#define KVQ_TR(e, cond)                                                                            \
    do {                                                                                           \
        if ((cond) && blockIdx.x == 0 && (int)g >= TR_G0 && (int)g < TR_G0 + TR_N)                 \
            g_kvq_trace[g - TR_G0][e] = clock64();                                                 \
    } while (0)
#else
#define KVQ_TR(e, cond) \
    do {                \
    } while (0)
#endif

// Waits on the critical path (MMA issuer, converters): a tight try_wait loop, or
// the hardware-suspending variant when built with -DKVQ_SLEEP_ALL.
#ifdef KVQ_SLEEP_ALL
#define KVQ_WAIT_HOT mbar_wait_sleep
#else
#define KVQ_WAIT_HOT mbar_wait
#endif

struct __align__(1024) Smem {
    // modes 0/1: stage i = [K box | K_hat box] at 32 KB * i (4 stages)
    // fused:     stage i = K box at 16 KB * i (8 stages; the converters overwrite it in place with
    //            the K_hat box, which the store warp writes out before the stage is refilled),
    //            codes staging at 128 KB + 16 KB * b (b = 0, 1)
    uint8_t buf[160 * 1024];
    uint8_t q[QST][2 * QTILE];
    ColRec cq[KST_MAX];      // fused mode: per-column quantizer constants of the K-block
    uint64_t full_k[KST_MAX], empty_k[KST_MAX], full_q[QST], empty_q[QST];
    uint64_t full_a[AST], empty_a[AST], full_acc[2], empty_acc[2];
    uint64_t staged[KST_MAX], cstored[2];  // fused mode: handoff converters -> store warp -> converters
    uint32_t tmem_base;
    double red[3][NTEAMS * 8];
};

static_assert(sizeof(Smem) <= 227 * 1024, "shared memory budget (227 KB per CTA on sm_100)");

struct TcParams {
    const uint32_t *qsplit;  // pre-split Q tiles (qsplit_kernel)
    int64_t T, D;
    int nq, ntiles, nkb, has_khat;
    Partial *partials;   // MODE 0, 2: one per CTA
    float *S;            // MODE 1: [nq][T]
    const ColRec *colq;  // MODE 2: per K-block quantizer records (colq_body, in prep_kernel)
    int hints;           // L2 policies: bit0 K loads evict-first, bit1 output stores evict-first (default both;
                         // evict-first loads with normal stores cost ~0.6 GB of extra DRAM reads at C4)
    float *Kh;           // MODE 2: K_hat output [T][D]
    int ngrp;            // work units (groups of CODE_KB K-blocks) per tile row
    double *split;       // MODE 0, 2: [Rt * pieces][BN][BM] fp64 Delta of the tail pieces (nullptr: whole tiles)
    int pieces;          // pieces per tail tile (divides ngrp) when split != nullptr
    int whole;           // with split: whole-tile waves every CTA takes before the tail (W)
    int rt;              // with split: tail tiles (ntiles - W * grid), each cut into `pieces` K-ranges
    // MODE 2 with a1 + a2 fused in front (cooperative launch, kvq_step on L2-resident K): the kernel first
    // computes the column maxima and the scales itself (pmax != nullptr), then runs the roundtrip
    uint32_t *pmax;      // [grid][D] per-CTA column maxima (abs bits)
    const float *Kin;    // K for the column-max phase (generic loads)
    float *scales_out;   // [D] s_d = fl32(m_d / 127)
    ColRec *colq_out;    // the per-K-block quantizer records the roundtrip then reads (== colq)
    // MODE 2 with whole tiles: the CTA that retires last reduces every CTA's partial in a fixed order and writes the
    // totals (and the metrics when no exchange follows) itself: no reduce_partials launch
    unsigned *ticket;        // zeroed by prep_kernel; nullptr: reduce_partials_kernel does it
    const float *scales_in;  // theoretical max = max_d s_d / 2
    double *sums;            // [4]: sum_sq, attn_abs, n_elems, n_scores (as reduce_partials_kernel)
    uint64_t *maxes;         // [2]: max_abs, theoretical max (fp64 bit patterns)
    kvq_metrics *final_out;  // nullable
    // MODE 2 with a1 + a2 fused in front: the Q split is done by the column-max phase too (no qsplit launch)
    const float *Qin;        // Q [nq][D] (nullptr when nq == 0)
    uint32_t *qsplit_out;    // == qsplit
};

// Work distribution.  A work unit is one group of CODE_KB K-blocks (one accumulator chunk, one code
// box) of one 128-row tile.  Every CTA first takes whole tiles in waves (tile b, b + G, ...: the G CTAs
// stream G adjacent tiles in lockstep, the write pattern the HBM measured best).  With a split tail (chosen
// on the host by a unit-count cost model, see launch_attn_tc) every CTA takes exactly W whole tiles, and the
// Rt = ntiles - W G tiles left are cut into P equal K-ranges ("pieces" of L = ngrp / P units), numbered
// piece-major: piece i is K-range i / Rt of tail tile W G + i mod Rt.  CTA b takes pieces b, b + G, b + 2G,
// ..., so in every round the CTAs work on the same K-range of adjacent tiles (still lockstep).  A piece's
// Delta goes, in fp64, to its own workspace slot; split_combine_kernel adds the P slots of a tile in piece
// order and takes |Delta|.  Mode 1 (scores) keeps whole tiles only.
struct Units {
    int n, nfull;   // units of this CTA; whole-tile units among them
    int G, ngrp;
    int wbase, rt, L;  // first tail tile (W * G), tail tiles, units per piece
};
// Computed once by every thread and broadcast from lane 0 (__shfl_sync), so that the compiler knows
// the loop state is warp-uniform: the MMA issuer's descriptors then stay in uniform registers.
__device__ __forceinline__ Units make_units(const TcParams &p) {
    const int b = blockIdx.x, G = gridDim.x;
    int n, nfull, wbase = 0, rt = 0, L = p.ngrp;
    if (!p.split) {
        nfull = n = (p.ntiles - b + G - 1) / G * p.ngrp;
    } else {
        nfull = p.whole * p.ngrp;
        wbase = p.whole * G;
        rt = p.rt;
        L = p.ngrp / p.pieces;
        const int np = p.rt * p.pieces;  // tail pieces in all
        n = nfull + (b < np ? (np - b + G - 1) / G : 0) * L;
    }
    Units us;
    us.n = __shfl_sync(0xffffffffu, n, 0);
    us.nfull = __shfl_sync(0xffffffffu, nfull, 0);
    us.wbase = __shfl_sync(0xffffffffu, wbase, 0);
    us.rt = __shfl_sync(0xffffffffu, rt, 0);
    us.L = __shfl_sync(0xffffffffu, L, 0);
    us.G = G;
    us.ngrp = p.ngrp;
    return us;
}
// Walks a CTA's units in order (whole-tile waves, then its tail pieces); integer division only at piece
// starts.
struct UnitWalk {
    int i, n, nfull, tile, grp, ngrp, G;
    int pi, pend, wbase, rt, L;  // current tail piece, its end group; tail geometry
    __device__ __forceinline__ explicit UnitWalk(const Units &u)
        : i(0), n(u.n), nfull(u.nfull), tile((int)blockIdx.x), grp(0), ngrp(u.ngrp), G(u.G), pi((int)blockIdx.x),
          pend(u.ngrp), wbase(u.wbase), rt(u.rt), L(u.L) {
        if (nfull == 0 && n > 0) start_piece();
    }
    __device__ __forceinline__ void start_piece() {
        tile = wbase + pi % rt;
        grp = (pi / rt) * L;
        pend = grp + L;
    }
    __device__ __forceinline__ bool ok() const { return i < n; }
    __device__ __forceinline__ bool in_piece() const { return i >= nfull; }
    __device__ __forceinline__ bool piece_first() const { return grp == pend - L; }
    __device__ __forceinline__ void next() {
        ++i;
        if (i < nfull) {
            if (++grp == ngrp) {
                grp = 0;
                tile += G;
            }
        } else if (i == nfull) {
            start_piece();  // pi == blockIdx.x: the CTA's first tail piece
        } else if (++grp == pend) {
            pi += G;
            start_piece();
        }
    }
};
static_assert(CHUNK_KB == CODE_KB, "one accumulator chunk per work unit");

// Q [nq][D] -> per K-block kb: [hi | lo] tiles of BN x BK tf32 in the canonical
// K-major SWIZZLE_NONE layout: core matrix (kg = k/4, rg = n/8) at byte
// (kg*8 + rg)*128, row n%8 at +16*(n%8), element k%4 at +4*(k%4).  Rows >= nq
// and columns >= D are zero.
__device__ __forceinline__ void qsplit_body(const float *__restrict__ Q, int64_t nq, int64_t D, int64_t nkb,
                                            uint32_t *__restrict__ out, int64_t blk, int64_t nblk) {
    // one thread per (K-block, query row, group of 4 columns): the 4 columns of a group are adjacent words of
    // one core-matrix row, so hi and lo each leave as one 16-byte store
    const int64_t total = nkb * BN * (BK / 4);
    for (int64_t i = blk * blockDim.x + threadIdx.x; i < total; i += nblk * blockDim.x) {
        const int64_t kb = i / (BN * (BK / 4));
        const int rem = (int)(i % (BN * (BK / 4)));
        const int n = rem / (BK / 4), kg = rem % (BK / 4);
        const int64_t col = kb * BK + kg * 4;
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const float q = (n < nq && col + e < D) ? Q[n * D + col + e] : 0.0f;
            hi[e] = to_tf32(q);
            lo[e] = to_tf32(q - __uint_as_float(hi[e]));
        }
        const uint32_t off = (kg * 8 + n / 8) * 32 + (n % 8) * 4;  // in 4-byte words (16-byte aligned)
        uint32_t *tile = out + kb * (2 * BN * BK);
        *reinterpret_cast<uint4 *>(tile + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4 *>(tile + BN * BK + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    }
}
__global__ void qsplit_kernel(const float *__restrict__ Q, int64_t nq, int64_t D, int64_t nkb,
                              uint32_t *__restrict__ out) {
    pdl_wait();
    pdl_trigger();
    qsplit_body(Q, nq, D, nkb, out, blockIdx.x, gridDim.x);
}

// Per-K-block quantizer records for the fused kernel: {s, RN(1/s)} per column,
// with y = 0 for s == 0 (code 0) and for subnormal/huge s, which need the exact
// path (flagged per block).
// (256-thread blocks: lane = column of the K-block, warp = K-block slot)
__device__ __forceinline__ void colq_body(const float *__restrict__ scales, int64_t D, int64_t nkb,
                                          ColRec *__restrict__ out, int64_t blk, int64_t nblk) {
    const int lx = threadIdx.x % 32, ly = threadIdx.x / 32;
    for (int64_t kb = blk * 8 + ly; kb < nkb; kb += nblk * 8) {
        const int64_t d = kb * BK + lx;
        const float sd = d < D ? scales[d] : 0.0f;
        const ColQ c = make_colq(sd);
        out[kb].y[lx] = c.y;
        out[kb].s[lx] = sd;
        const unsigned any = __ballot_sync(0xffffffffu, c.exact);
        if (lx == 0) {
            out[kb].any_exact = any ? 1u : 0u;
            out[kb].pad[0] = out[kb].pad[1] = out[kb].pad[2] = 0u;
        }
    }
}

// The fused mode's two small preparation passes in one launch: blocks [0, nbq) split Q, the rest build
// the column records.
__global__ void __launch_bounds__(256) prep_kernel(const float *__restrict__ Q, int64_t nq, int64_t D, int64_t nkb,
                                                   uint32_t *__restrict__ qs, const float *__restrict__ scales,
                                                   ColRec *__restrict__ cq, int nbq, unsigned *ticket) {
    pdl_wait();  // Q and the scales of the preceding calls
    pdl_trigger();
    if (ticket && blockIdx.x == 0 && threadIdx.x == 0) *ticket = 0u;  // the pass's last-CTA ticket
    if ((int)blockIdx.x < nbq)
        qsplit_body(Q, nq, D, nkb, qs, blockIdx.x, nbq);
    else
        colq_body(scales, D, nkb, cq, blockIdx.x - nbq, gridDim.x - nbq);
}

// Split tail (see make_units): block (r, y) adds the P pieces of tail tile r (slot pc * Rt + r holds K-range
// pc) in piece order for queries [16y, 16y + 16), takes |Delta| over the tile's rows < T and queries < nq,
// and writes the sum as partial G + r * COMBINE_JQ + y.  Fixed order throughout: deterministic.
constexpr int COMBINE_JQ = 4;  // query quarters per tile (blockIdx.y): 4x the loads in flight
__global__ void __launch_bounds__(BM) split_combine_kernel(const double *__restrict__ split, int64_t T, int nq,
                                                           int wbase, int rt, int G, int P, Partial *partials) {
    constexpr int JN = BN / COMBINE_JQ;
    const int r_t = blockIdx.x, r = threadIdx.x, j0 = blockIdx.y * JN;
    pdl_wait();  // the pieces written by the tensor-core pass
    pdl_trigger();
    const int64_t row = ((int64_t)wbase + r_t) * BM + r;
    double d[JN];
#pragma unroll
    for (int j = 0; j < JN; j++) d[j] = 0.0;
    for (int pc = 0; pc < P; pc++) {
        const double *sp = split + ((int64_t)pc * rt + r_t) * (BN * BM) + (int64_t)j0 * BM;
#pragma unroll
        for (int j = 0; j < JN; j++)
            if (j0 + j < nq) d[j] += sp[j * BM + r];
    }
    double attn = 0.0;
    if (row < T)
#pragma unroll
        for (int j = 0; j < JN; j++)
            if (j0 + j < nq) attn += fabs(d[j]);
    __shared__ double red[BM];
    red[r] = attn;
    __syncthreads();
    for (int o = BM / 2; o > 0; o >>= 1) {
        if (r < o) red[r] += red[r + o];
        __syncthreads();
    }
    if (r == 0) partials[G + r_t * COMBINE_JQ + blockIdx.y] = Partial{0.0, red[0], 0.0, 0.0};
}

// a1 + a2 in front of the fused roundtrip (kvq_step on an L2-resident K; cooperative launch, all threads of the
// CTA, before the warp roles start).  Alg. 1 / Eq. 6 over the CTA's row slab -> its row of partial maxima;
// grid barrier; Eq. 5/6 for the K-blocks this CTA owns (kb = b, b + G, ...): m_d = max over the partial rows
// (order-free), s_d = fl32(m_d / 127) (IEEE division), the K-block's quantizer record; grid barrier.  The
// roundtrip's producer then bulk-loads the records as usual.  `sm` is the (still unused) input ring.
template <bool QSPLIT = true>  // QSPLIT: also split Q (p.qsplit_out) before the second grid barrier
__device__ __forceinline__ void fused_scales_phase(const TcParams &p, uint8_t *sm) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const int b = blockIdx.x, G = gridDim.x, tid = threadIdx.x;
    const int64_t T = p.T, D = p.D, D4 = D / 4;  // D % 16 == 0 on this path
    const int64_t r0 = T * b / G, r1 = T * (b + 1) / G;
    uint32_t *smax = reinterpret_cast<uint32_t *>(sm);  // [D]
    for (int64_t d = tid; d < D; d += NTHREADS) smax[d] = 0u;
    __syncthreads();
    const float4 *K4 = reinterpret_cast<const float4 *>(p.Kin);
    if (NTHREADS % D4 == 0) {  // column-owning threads: D4 divides the block (D <= 3072)
        const int rpp = NTHREADS / (int)D4, c4 = tid % (int)D4;
        uint32_t m0 = 0, m1 = 0, m2 = 0, m3 = 0;
        constexpr int U = 8;  // loads in flight per thread
        for (int64_t r = r0 + tid / (int)D4; r < r1; r += (int64_t)U * rpp) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; u++)
                v[u] = r + (int64_t)u * rpp < r1 ? __ldcg(K4 + (r + (int64_t)u * rpp) * D4 + c4)  // stays in L2
                                                 : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < U; u++) {
                m0 = max(m0, absbits(v[u].x));
                m1 = max(m1, absbits(v[u].y));
                m2 = max(m2, absbits(v[u].z));
                m3 = max(m3, absbits(v[u].w));
            }
        }
        atomicMax(&smax[4 * c4 + 0], m0);
        atomicMax(&smax[4 * c4 + 1], m1);
        atomicMax(&smax[4 * c4 + 2], m2);
        atomicMax(&smax[4 * c4 + 3], m3);
    } else {
        for (int64_t r = r0; r < r1; r++)
            for (int64_t c4 = tid; c4 < D4; c4 += NTHREADS) {
                const float4 v = __ldcg(K4 + r * D4 + c4);
                atomicMax(&smax[4 * c4 + 0], absbits(v.x));
                atomicMax(&smax[4 * c4 + 1], absbits(v.y));
                atomicMax(&smax[4 * c4 + 2], absbits(v.z));
                atomicMax(&smax[4 * c4 + 3], absbits(v.w));
            }
    }
    __syncthreads();
    for (int64_t d = tid; d < D; d += NTHREADS) p.pmax[(int64_t)b * D + d] = smax[d];
    if (p.ticket && b == 0 && tid == 0) *p.ticket = 0u;  // the pass's last-CTA reduction (no prep launch here)
    grid.sync();
    // the K-blocks this CTA owns: warp w of the 24 folds row groups w, w + 24, ... of column `lane`
    const int lane = tid % 32, wv = tid / 32, nw = NTHREADS / 32;
    for (int kb = b; kb < p.nkb; kb += G) {
        __syncthreads();
        if (tid < 32) smax[tid] = 0u;
        __syncthreads();
        const int64_t d = (int64_t)kb * BK + lane;
        if (d < D) {
            uint32_t m = 0u;
            for (int c = wv; c < G; c += nw) m = max(m, __ldcg(p.pmax + (int64_t)c * D + d));
            atomicMax(&smax[lane], m);
        }
        __syncthreads();
        if (tid < 32) {
            const float sd = d < D ? __fdiv_rn(__uint_as_float(smax[lane]), 127.0f) : 0.0f;  // Eq. 5/6, Q3
            const ColQ c = make_colq(sd);
            p.colq_out[kb].y[lane] = c.y;
            p.colq_out[kb].s[lane] = sd;
            const unsigned any = __ballot_sync(0xffffffffu, c.exact);
            if (lane == 0) {
                p.colq_out[kb].any_exact = any ? 1u : 0u;
                p.colq_out[kb].pad[0] = p.colq_out[kb].pad[1] = p.colq_out[kb].pad[2] = 0u;
            }
            if (d < D) p.scales_out[d] = sd;
        }
    }
    if constexpr (QSPLIT) {
        if (p.qsplit_out) qsplit_body(p.Qin, p.nq, D, p.nkb, p.qsplit_out, b, G);  // (the Q split of the step)
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");  // records and Q tiles are read by bulk copies
    grid.sync();
}

// The end of the roundtrip pass with whole tiles (p.ticket set): after its partial is written (thread 0, then a block
// barrier), every CTA takes a ticket; the last one reduces all G partials in a fixed order with one warp (strided
// per-lane sums, xor butterfly: deterministic) and writes the totals as reduce_partials_kernel does.  Runs after the
// warp roles, within the smallest register budget (warpgroup 0's).
__device__ __forceinline__ void last_cta_reduce(const TcParams &p, int *flag) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, G = gridDim.x;
    constexpr int NW = NTHREADS / 32;
    double *sh = reinterpret_cast<double *>(flag + 4);  // [4][NW] (the free input ring)
    if (tid == 0) {
        __threadfence();  // this CTA's partial, before its ticket
        *flag = atomicAdd(p.ticket, 1u) == (unsigned)G - 1;
    }
    __syncthreads();
    if (!*flag) return;  // uniform: the whole CTA reduces (as reduce_partials_kernel, 768 instead of 1024 threads)
    __threadfence();     // the other CTAs' partials (their tickets came first)
    double ss = 0.0, at = 0.0, mx = 0.0, th = 0.0;
    for (int i = tid; i < G; i += NTHREADS) {
        ss += __ldcg(&p.partials[i].sum_sq);
        at += __ldcg(&p.partials[i].attn_abs);
        mx = fmax(mx, __ldcg(&p.partials[i].max_abs));
    }
    for (int64_t d = tid; d < p.D; d += NTHREADS) th = fmax(th, (double)__ldcg(p.scales_in + d) / 2.0);
    for (int o = 16; o > 0; o >>= 1) {
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
        at += __shfl_xor_sync(0xffffffffu, at, o);
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        th = fmax(th, __shfl_xor_sync(0xffffffffu, th, o));
    }
    if (lane == 0) {
        sh[wid] = ss;
        sh[NW + wid] = at;
        sh[2 * NW + wid] = mx;
        sh[3 * NW + wid] = th;
    }
    __syncthreads();
    if (wid != 0) return;
    ss = lane < NW ? sh[lane] : 0.0;
    at = lane < NW ? sh[NW + lane] : 0.0;
    mx = lane < NW ? sh[2 * NW + lane] : 0.0;
    th = lane < NW ? sh[3 * NW + lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
        at += __shfl_xor_sync(0xffffffffu, at, o);
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        th = fmax(th, __shfl_xor_sync(0xffffffffu, th, o));
    }
    if (lane == 0) {
        const double n_elems = (double)p.T * (double)p.D, n_scores = (double)p.nq * (double)p.T;
        const double maxabs = fmax(mx, 0.0);
        p.sums[0] = ss;
        p.sums[1] = at;
        p.sums[2] = n_elems;
        p.sums[3] = n_scores;
        p.maxes[0] = (uint64_t)__double_as_longlong(maxabs);
        p.maxes[1] = (uint64_t)__double_as_longlong(th);
        if (p.final_out) {
            kvq_metrics m;
            m.sum_sq = ss;
            m.attn_abs_sum = at;
            m.n_elems = (int64_t)n_elems;
            m.n_scores = (int64_t)n_scores;
            m.l2 = sqrt(ss);
            m.max_abs = maxabs;
            m.theoretical_max = th;
            m.attn_mean_abs = n_scores > 0.0 ? at / n_scores : 0.0;
            *p.final_out = m;
        }
    }
}

// byte address of 16-byte chunk c of row r in a [rows][128 B] tile with the TMA 128B swizzle
__device__ __forceinline__ uint32_t swz(uint32_t base, int r, int c) { return base + r * 128 + ((c ^ (r & 7)) << 4); }

// The fused converter's rare path for one thread's 16-column row segment (a near-tie quotient, a quotient past
// the clamp, or an exact-path column) in the FASTCONV variant: re-reads x from the stage, computes every element
// with the clamp and, where the fast quotient is within 2^-14 of a half-integer (or the column needs it), the IEEE
// division (quant_exact, the oracle's arithmetic), and writes K_hat in place and the 16 codes to `caddr` itself.
// The fast path's registers are not touched, so the common path carries no register merges for this branch.
__device__ __forceinline__ void rare_segment(uint32_t kbase, int r, int h, uint32_t caddr, const ColRec &rec) {
    uint32_t w[4];
#pragma unroll
    for (int c = 0; c < 4; c++) {
        const float4 a = lds128(swz(kbase, r, 4 * h + c));
        const float xs[4] = {a.x, a.y, a.z, a.w};
        float xh[4], vq[4];
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const int i = 16 * h + 4 * c + e;
            const float sc = rec.s[i], yy = rec.y[i], xi = xs[e];
            const float cl = fminf(fmaxf(__fmul_rn(xi, yy), -127.0f), 127.0f);
            float vv = __fadd_rn(cl, kMagic);
            const float rr = __fsub_rn(vv, kMagic);
            float x1 = __fmul_rn(rr, sc);
            if (fabsf(__fsub_rn(cl, rr)) > kDangerThr || (yy == 0.0f && sc != 0.0f)) {
                const int cd = quant_exact(xi, sc);
                vv = __fadd_rn((float)cd, kMagic);
                x1 = __fmul_rn((float)cd, sc);
            }
            xh[e] = x1;
            vq[e] = vv;
        }
        sts128(swz(kbase, r, 4 * h + c), make_float4(xh[0], xh[1], xh[2], xh[3]));
        w[c] = pack4(vq[0], vq[1], vq[2], vq[3]);
    }
    sts128u(caddr, make_uint4(w[0], w[1], w[2], w[3]));
}

// MODE 0: metrics partials (E = K - K_hat).
// MODE 1: scores S[i][t] (E = K, or K - K_hat).
// MODE 2: fused a3+a4+a5+a6: quantize and dequantize the K tile in the
//         converters (same arithmetic as quant_v4_kernel), write Kq and K_hat,
//         and contract E = K - K_hat with Q: one HBM pass, 9 bytes/element.
// FASTCONV (MODE 2 only): the converter variant without register merges on the rare path (253 instead of 325
// instructions per thread and K-block): faster per CTA, but 2.5% slower where the pass is HBM-bound (C4), so the
// host uses it only when the pass is bound per CTA (one round of work units: the 8-rank shard, C2).
template <int MODE, bool FASTCONV = false>
__global__ void __launch_bounds__(NTHREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmKh,
                   const __grid_constant__ CUtensorMap tmKq, const __grid_constant__ TcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem &s = *reinterpret_cast<Smem *>(smem_raw);
    const int64_t T = p.T;
    const int nq = p.nq, nkb = p.nkb, has_khat = p.has_khat;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    constexpr int KST = Ring<MODE>::kst;

    if (threadIdx.x == 0) {
        if (smem_u32(smem_raw) & 1023u) __trap();  // swizzle atoms need 1024-byte alignment
        for (int i = 0; i < Ring<MODE>::kst; i++) {
            mbar_init(&s.full_k[i], 1);
            // every converter thread of the team arrives on the barriers that release shared memory it read
            // (empty_k in modes 0/1, staged in the fused mode: the K stage and its column records are
            // overwritten by the next TMA / bulk load after them), so each generic-proxy read is ordered
            // before the async-proxy overwrite by its own release; full_a (TMEM hand-off) takes one
            // elected arrival per warp
            mbar_init(&s.empty_k[i], MODE == 2 ? 1 : NCONV);  // fused: the store warp frees the stage
            mbar_init(&s.staged[i], NCONV);
        }
        for (int i = 0; i < QST; i++) {
            mbar_init(&s.full_q[i], 1);
            mbar_init(&s.empty_q[i], 1);
        }
        for (int i = 0; i < AST; i++) {
            mbar_init(&s.full_a[i], NCONV_W);
            mbar_init(&s.empty_a[i], 1);
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(&s.full_acc[i], 1);
            mbar_init(&s.empty_acc[i], 128);
        }
        for (int i = 0; i < 2; i++) mbar_init(&s.cstored[i], 1);
        mbar_fence_init();
    }
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmK);
        if (has_khat || MODE == 2) prefetch_tmap(&tmKh);
        if (MODE == 2) prefetch_tmap(&tmKq);
    }
    if (warp == 1) tmem_alloc<TMEM_COLS>(&s.tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = s.tmem_base;
    // everything above (barrier init, TMEM allocation, tensor-map prefetch) overlaps the preceding grid;
    // from here on the pass reads Q tiles / column records of the preparation kernel and writes outputs
    pdl_wait();
    pdl_trigger();
    if constexpr (MODE == 2) {
        if (p.pmax) fused_scales_phase(p, s.buf);
    }
    const int ngrp = p.ngrp;
    const Units us = make_units(p);

    if (warp < CONV_W0) {
        setmaxnreg_dec<REG_WG0>();  // warpgroup 0: producer + MMA issuer need few registers
        if (warp == 0 && lane == 0) {
            // ------------------------------------------------------------ producer
            const uint64_t pol_stream = (p.hints & 1) ? policy_evict_first() : policy_evict_normal();
            const uint64_t pol_keep = policy_evict_last();  // column records: re-read by every tile
            const uint32_t kbytes = (has_khat ? 2 * KTILE : KTILE) + (MODE == 2 ? (uint32_t)sizeof(ColRec) : 0u);
            uint32_t g = 0;
            for (UnitWalk w(us); w.ok(); w.next()) {
                const int tile = w.tile, kb0 = w.grp * CODE_KB, kb1 = min(kb0 + CODE_KB, nkb);
                #pragma unroll 1
                for (int kb = kb0; kb < kb1; kb++, g++) {
                    const int sk = g % KST;
                    mbar_wait_sleep(&s.empty_k[sk], ((g / KST) & 1) ^ 1);
                    KVQ_TR(0, true);
                    mbar_arrive_tx(&s.full_k[sk], kbytes);
                    uint8_t *stg = s.buf + sk * Ring<MODE>::stage;
                    tma_load_2d(stg, &tmK, &s.full_k[sk], kb * BK, tile * BM, pol_stream);
                    if (has_khat) tma_load_2d(stg + KTILE, &tmKh, &s.full_k[sk], kb * BK, tile * BM, pol_stream);
                    if (MODE == 2) bulk_load(&s.cq[sk], p.colq + kb, sizeof(ColRec), &s.full_k[sk], pol_keep);
                }
            }
        } else if (warp == 3 && lane == 0) {
            // ------------------------------------------------------------ Q producer (L2-resident tiles)
            // Separate from the K producer so a late MMA never holds back the HBM stream.
            const uint64_t pol_keep = policy_evict_last();
            uint32_t g = 0;
            for (UnitWalk w(us); w.ok(); w.next()) {
                const int kb0 = w.grp * CODE_KB, kb1 = min(kb0 + CODE_KB, nkb);
                #pragma unroll 1
                for (int kb = kb0; kb < kb1; kb++, g++) {
                    const int sq = g % QST;
                    mbar_wait_sleep(&s.empty_q[sq], ((g / QST) & 1) ^ 1);
                    mbar_arrive_tx(&s.full_q[sq], 2 * QTILE);
                    bulk_load(s.q[sq], p.qsplit + (size_t)kb * (2 * BN * BK), 2 * QTILE, &s.full_q[sq], pol_keep);
                }
            }
        } else if (MODE == 2 && warp == 2 && lane == 0) {
            // ------------------------------------------------------------ output store warp (fused mode)
            // K-block g's K_hat box has been written by the converters into its own input stage
            // (g % KST); every CODE_KB blocks the group's codes ([128 rows x 128 B], full lines: no
            // DRAM read-modify-write) sit in code buffer grp & 1.  Store them with TMA; one block
            // later, when the bulk engine has read them out of smem, free the input stage for the
            // producer and (at group ends) the code buffer for the converters.
            const uint64_t pol_out = (p.hints & 2) ? policy_evict_first() : policy_evict_normal();
            uint32_t g = 0, grp = 0;
            bool prev_group_end = false;
            for (UnitWalk w(us); w.ok(); w.next()) {
                const int tile = w.tile, kb0 = w.grp * CODE_KB, kb1 = min(kb0 + CODE_KB, nkb);
                #pragma unroll 1
                for (int kb = kb0; kb < kb1; kb++, g++) {
                    const int sk = g % KST;
                    mbar_wait_sleep(&s.staged[sk], (g / KST) & 1);
                    KVQ_TR(7, true);
#ifndef KVQ_EXP_NOSTORE  // timing experiments only (outputs not written)
                    tma_store_2d(&tmKh, s.buf + sk * Ring<MODE>::stage, kb * BK, tile * BM, pol_out);
#endif
                    const bool group_end = kb == kb1 - 1;
#ifndef KVQ_EXP_NOSTORE
                    if (group_end)
#else
                    if (false)
#endif
                        tma_store_2d(&tmKq, s.buf + 128 * 1024 + (grp & 1) * KTILE, (kb / CODE_KB) * (BK * CODE_KB),
                                     tile * BM, pol_out);
                    bulk_commit();
                    if (g > 0) {
                        bulk_wait_read<1>();  // block g-1's boxes have left smem
                        KVQ_TR(8, true);
                        mbar_arrive(&s.empty_k[(g - 1) % KST]);
                        if (prev_group_end) mbar_arrive(&s.cstored[(grp - 1) & 1]);
                    }
                    prev_group_end = group_end;
                    if (group_end) grp++;
                }
            }
            bulk_wait<0>();  // all K_hat / code writes complete before the CTA retires
        } else if (warp == 1) {
            // ------------------------------------------------------------ MMA issuer
            // The whole warp walks the loop and waits (loop state and descriptors are warp-uniform, so they
            // live in uniform registers); one elected lane issues the MMAs and commits.  (A single-lane role
            // issues each tcgen05.mma through a per-instruction uniformization loop: ~1000 cycles per K-block.)
            uint32_t g = 0, gc = 0;
            for (UnitWalk w(us); w.ok(); w.next()) {
                const int kb0 = w.grp * CODE_KB, kb1 = min(kb0 + CODE_KB, nkb);
                #pragma unroll 1
                for (int kb = kb0; kb < kb1; kb++, g++) {
                    const int ab = gc & 1;
                    const uint32_t d = tbase + ab * BN;
                    const bool chunk_first = kb == kb0;
                    const bool chunk_last = kb == kb1 - 1;
                    if (chunk_first) {
                        KVQ_WAIT_HOT(&s.empty_acc[ab], ((gc >> 1) & 1) ^ 1);
                        tc_fence_after();
                    }
                    const int sa = g % AST, sq = g % QST;
                    KVQ_WAIT_HOT(&s.full_a[sa], (g / AST) & 1);
                    KVQ_TR(9, lane == 0);
                    KVQ_WAIT_HOT(&s.full_q[sq], (g / QST) & 1);
                    tc_fence_after();
                    const uint32_t ahi = tbase + A_COL0 + sa * 64, alo = ahi + 32;
                    const uint32_t qhi = smem_u32(s.q[sq]);
                    // K-step j covers k-groups 2j, 2j+1 (LBO apart = 1024 B), 8-row groups 128 B apart;
                    // step j starts 2048 B further (+128 in the descriptor's 16-byte address field)
                    const uint64_t bh0 = smem_desc(qhi, 1024, 128), bl0 = smem_desc(qhi + QTILE, 1024, 128);
                    if (elect_one()) {
#pragma unroll
                        for (int j = 0; j < BK / 8; j++) {
#ifndef KVQ_EXP_NOMMA  // timing experiments only (Delta not computed)
                            mma_tf32_ts(d, ahi + 8 * j, bh0 + 128u * j, IDESC, (!chunk_first || j != 0) ? 1u : 0u);
                            mma_tf32_ts(d, ahi + 8 * j, bl0 + 128u * j, IDESC, 1);
                            mma_tf32_ts(d, alo + 8 * j, bh0 + 128u * j, IDESC, 1);
#endif
                        }
                        mma_commit(&s.empty_a[sa]);
                        mma_commit(&s.empty_q[sq]);
                        if (chunk_last) mma_commit(&s.full_acc[ab]);
                    }
                    __syncwarp();
                    KVQ_TR(10, lane == 0);
                    if (chunk_last) gc++;
                }
            }
        }
    } else if (warp < EPI_W0) {
        // ------------------------------------------------------------ converters (warps 4..11)
        // thread = (row r, half h): columns 16h..16h+15 of every 32-column K-block
        if constexpr (REG_CONV > REG_LAUNCH) setmaxnreg_inc<REG_CONV>();
        const int team = (warp - CONV_W0) / NCONV_W;
        const int quarter = warp & 3;
        const int h = ((warp - CONV_W0) % NCONV_W) >> 2;
        const int r = quarter * 32 + lane;  // row of the tile == TMEM lane
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        double ss = 0.0;
        float mx = 0.0f;
        uint32_t g = 0, cgrp = 0;  // K-block and code-group counters (same order as the store warp)
        for (UnitWalk w(us); w.ok(); w.next()) {
            const int kb0 = w.grp * CODE_KB, kb1 = min(kb0 + CODE_KB, nkb);
            bool code_buf_ready = false;  // this team has waited for the group's code buffer
            #pragma unroll 1
            for (int kb = kb0; kb < kb1; kb++, g++) {
                if (NTEAMS > 1 && (int)(g % NTEAMS) != team) {  // the other team's K-block
                    if (kb == kb1 - 1) cgrp++;
                    continue;
                }
                const int sk = g % KST;
                KVQ_TR(14, lane == 0 && (warp - CONV_W0) % NCONV_W == 0);
                KVQ_WAIT_HOT(&s.full_k[sk], (g / KST) & 1);
                KVQ_TR(1, lane == 0 && (warp - CONV_W0) % NCONV_W == 0); KVQ_TR(5, lane == 0 && (warp - CONV_W0) % NCONV_W == NCONV_W - 1);
                const uint32_t kbase = smem_u32(s.buf + sk * Ring<MODE>::stage);
                uint64_t E[8];  // E = K - K_hat as fp32 pairs (columns 2j, 2j+1 of this thread's 16)
                if (MODE != 2) {
                    const uint32_t hbase = kbase + KTILE;
#pragma unroll
                    for (int c = 0; c < 4; c++) {
                        const float4 a = lds128(swz(kbase, r, 4 * h + c));
                        float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (has_khat) b = lds128(swz(hbase, r, 4 * h + c));
                        E[2 * c] = f2sub(f2pk(a.x, a.y), f2pk(b.x, b.y));
                        E[2 * c + 1] = f2sub(f2pk(a.z, a.w), f2pk(b.z, b.w));
                    }
                    mbar_arrive(&s.empty_k[sk]);
                } else {
                    // ---- a3 + a4 on the resident K row segment (Eq. 7, Eq. 8); same arithmetic and
                    // exactness argument as quant_v4_kernel (device_common.cuh), two columns per
                    // instruction (FMUL2/FADD2: each lane the IEEE RN operation of the scalar code).
                    // The clamp to +-127 is folded into the repair test: for a scale formed from the
                    // column's own maximum (Eq. 6) |fq| <= 127 (1 + 2^-22), so |fq| > 127.25 only happens
                    // for caller scales below max/127 and sends the segment to the exact path below.
                    uint64_t X[8], V[8], XH[8];
#pragma unroll
                    for (int c = 0; c < 4; c++) {
                        const float4 a = lds128(swz(kbase, r, 4 * h + c));
                        X[2 * c] = f2pk(a.x, a.y);
                        X[2 * c + 1] = f2pk(a.z, a.w);
                    }
                    const uint32_t cyb = smem_u32(&s.cq[sk]) + 64 * h;  // y[16h .. 16h+15], then s[...] at +128
                    const uint64_t M2 = f2pk(kMagic, kMagic);
                    float amax = 0.0f, dmax = 0.0f;
#pragma unroll
                    for (int c = 0; c < 4; c++) {
                        const float4 y4 = lds128(cyb + 16 * c);        // broadcast reads
                        const float4 s4 = lds128(cyb + 128 + 16 * c);
#pragma unroll
                        for (int u = 0; u < 2; u++) {
                            const int j = 2 * c + u;
                            const uint64_t fq = f2mul(X[j], u ? f2pk(y4.z, y4.w) : f2pk(y4.x, y4.y));
                            const uint64_t vv = f2add(fq, M2);
                            const uint64_t rr = f2sub(vv, M2);
                            const uint64_t dd = f2sub(fq, rr);
                            amax = fmaxf(amax, fmaxf(fabsf(f2lo(fq)), fabsf(f2hi(fq))));
                            dmax = fmaxf(dmax, fmaxf(fabsf(f2lo(dd)), fabsf(f2hi(dd))));
                            V[j] = vv;
                            XH[j] = f2mul(rr, u ? f2pk(s4.z, s4.w) : f2pk(s4.x, s4.y));
                        }
                    }
                  if constexpr (FASTCONV) {
                    const bool rare = dmax > kDangerThr || amax > 127.25f || s.cq[sk].any_exact;
                    if (!code_buf_ready) {
                        KVQ_WAIT_HOT(&s.cstored[cgrp & 1], ((cgrp >> 1) & 1) ^ 1);
                        code_buf_ready = true;
                    }
                    const uint32_t caddr =
                        swz(smem_u32(s.buf + 128 * 1024 + (cgrp & 1) * KTILE), r, (kb % CODE_KB) * 2 + h);
                    if (!rare) {
#pragma unroll
                        for (int c = 0; c < 4; c++)
                            sts128(swz(kbase, r, 4 * h + c), make_float4(f2lo(XH[2 * c]), f2hi(XH[2 * c]),
                                                                         f2lo(XH[2 * c + 1]), f2hi(XH[2 * c + 1])));
                        uint4 w;
                        w.x = pack4(f2lo(V[0]), f2hi(V[0]), f2lo(V[1]), f2hi(V[1]));
                        w.y = pack4(f2lo(V[2]), f2hi(V[2]), f2lo(V[3]), f2hi(V[3]));
                        w.z = pack4(f2lo(V[4]), f2hi(V[4]), f2lo(V[5]), f2hi(V[5]));
                        w.w = pack4(f2lo(V[6]), f2hi(V[6]), f2lo(V[7]), f2hi(V[7]));
                        sts128u(caddr, w);
                    } else {
                        rare_segment(kbase, r, h, caddr, s.cq[sk]);
                    }
                    fence_proxy_async();  // generic smem writes -> visible to the TMA (async proxy)
                    mbar_arrive(&s.staged[sk]);
                    if (kb == kb1 - 1) cgrp++;
                    // E from the K_hat the stage now holds (the fast path's or rare_segment's; this thread's own
                    // stores): no register merge between the two paths
#pragma unroll
                    for (int c = 0; c < 4; c++) {
                        const float4 b = lds128(swz(kbase, r, 4 * h + c));
                        E[2 * c] = f2sub(X[2 * c], f2pk(b.x, b.y));  // exact (fact 4)
                        E[2 * c + 1] = f2sub(X[2 * c + 1], f2pk(b.z, b.w));
                    }
                  } else {
#ifdef KVQ_EXP_NODANGER  // timing experiments only (near-tie quotients not repaired: codes may differ)
                    if (s.cq[sk].any_exact) {
#else
                    if (dmax > kDangerThr || amax > 127.25f || s.cq[sk].any_exact) {
#endif
                        // rare: a near-tie quotient, a quotient past the clamp or an exact-path column ->
                        // the whole segment again with the clamp and, where needed, the IEEE division
#pragma unroll
                        for (int i = 0; i < 16; i++) {
                            const float sc = s.cq[sk].s[16 * h + i], yy = s.cq[sk].y[16 * h + i];
                            const float xi = (i & 1) ? f2hi(X[i / 2]) : f2lo(X[i / 2]);
                            const float cl = fminf(fmaxf(__fmul_rn(xi, yy), -127.0f), 127.0f);
                            float vv = __fadd_rn(cl, kMagic);
                            const float rr = __fsub_rn(vv, kMagic);
                            float xh = __fmul_rn(rr, sc);
                            if (fabsf(__fsub_rn(cl, rr)) > kDangerThr || (yy == 0.0f && sc != 0.0f)) {
                                const int cd = quant_exact(xi, sc);
                                vv = __fadd_rn((float)cd, kMagic);
                                xh = __fmul_rn((float)cd, sc);
                            }
                            const int j = i / 2;
                            if (i & 1) {
                                V[j] = f2pk(f2lo(V[j]), vv);
                                XH[j] = f2pk(f2lo(XH[j]), xh);
                            } else {
                                V[j] = f2pk(vv, f2hi(V[j]));
                                XH[j] = f2pk(xh, f2hi(XH[j]));
                            }
                        }
                    }
                    // K_hat overwrites x in the input stage (same swizzled positions, read by this
                    // thread only); the codes go to the group's code buffer.  The store warp writes
                    // both out with TMA and then frees the stage (and the code buffer).
                    KVQ_TR(11, lane == 0 && (warp - CONV_W0) % NCONV_W == 0);
                    KVQ_TR(32 + (warp - CONV_W0) % NCONV_W, lane == 0);
                    if (!code_buf_ready) {
                        KVQ_WAIT_HOT(&s.cstored[cgrp & 1], ((cgrp >> 1) & 1) ^ 1);
                        code_buf_ready = true;
                    }
                    const uint32_t cds = smem_u32(s.buf + 128 * 1024 + (cgrp & 1) * KTILE);
#pragma unroll
                    for (int c = 0; c < 4; c++)
                        sts128(swz(kbase, r, 4 * h + c), make_float4(f2lo(XH[2 * c]), f2hi(XH[2 * c]),
                                                                     f2lo(XH[2 * c + 1]), f2hi(XH[2 * c + 1])));
                    uint4 w;
                    w.x = pack4(f2lo(V[0]), f2hi(V[0]), f2lo(V[1]), f2hi(V[1]));
                    w.y = pack4(f2lo(V[2]), f2hi(V[2]), f2lo(V[3]), f2hi(V[3]));
                    w.z = pack4(f2lo(V[4]), f2hi(V[4]), f2lo(V[5]), f2hi(V[5]));
                    w.w = pack4(f2lo(V[6]), f2hi(V[6]), f2lo(V[7]), f2hi(V[7]));
                    sts128u(swz(cds, r, (kb % CODE_KB) * 2 + h), w);
                    KVQ_TR(12, lane == 0 && (warp - CONV_W0) % NCONV_W == 0);
                    fence_proxy_async();  // generic smem writes -> visible to the TMA (async proxy)
                    KVQ_TR(13, lane == 0 && (warp - CONV_W0) % NCONV_W == 0);
                    mbar_arrive(&s.staged[sk]);
                    KVQ_TR(2, lane == 0 && (warp - CONV_W0) % NCONV_W == 0);
                    KVQ_TR(16 + (warp - CONV_W0) % NCONV_W, lane == 0);
                    if (kb == kb1 - 1) cgrp++;
#pragma unroll
                    for (int j = 0; j < 8; j++) E[j] = f2sub(X[j], XH[j]);  // exact (fact 4)
                  }
                }
                if (MODE != 1) {
                    // e^2 summed over the 16 columns in fp32 (two interleaved partial sums), blocks carried in fp64
                    uint64_t sq = f2mul(E[0], E[0]);
#pragma unroll
                    for (int j = 1; j < 8; j++) sq = f2fma(E[j], E[j], sq);
#pragma unroll
                    for (int j = 0; j < 8; j++) mx = fmaxf(mx, fmaxf(fabsf(f2lo(E[j])), fabsf(f2hi(E[j]))));
                    ss += (double)__fadd_rn(f2lo(sq), f2hi(sq));
                }
                // 3xTF32 split: hi = e with the 13 low mantissa bits cleared (a tf32 value),
                // lo = e - hi exactly (the tensor core reads lo's top 11 bits: error <= 2^-21 |e|)
                uint32_t hi[16], lo[16];
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    hi[2 * j] = __float_as_uint(f2lo(E[j])) & 0xFFFFE000u;
                    hi[2 * j + 1] = __float_as_uint(f2hi(E[j])) & 0xFFFFE000u;
                    const uint64_t l = f2sub(E[j], f2pk(__uint_as_float(hi[2 * j]), __uint_as_float(hi[2 * j + 1])));
                    lo[2 * j] = __float_as_uint(f2lo(l));
                    lo[2 * j + 1] = __float_as_uint(f2hi(l));
                }
                const int sa = g % AST;
                KVQ_WAIT_HOT(&s.empty_a[sa], ((g / AST) & 1) ^ 1);
                KVQ_TR(3, lane == 0 && (warp - CONV_W0) % NCONV_W == 0);
                tc_fence_after();
                tmem_st16(tbase + lane_off + A_COL0 + sa * 64 + 16 * h, hi);
                tmem_st16(tbase + lane_off + A_COL0 + sa * 64 + 32 + 16 * h, lo);
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.full_a[sa]);
                KVQ_TR(4, lane == 0 && (warp - CONV_W0) % NCONV_W == 0); KVQ_TR(6, lane == 0 && (warp - CONV_W0) % NCONV_W == NCONV_W - 1);
            }
        }
        if (MODE != 1) {
            double mxd = (double)mx;
            for (int o = 16; o > 0; o >>= 1) {
                ss += __shfl_xor_sync(0xffffffffu, ss, o);
                mxd = fmax(mxd, __shfl_xor_sync(0xffffffffu, mxd, o));
            }
            if (lane == 0) {
                s.red[0][warp - CONV_W0] = ss;
                s.red[2][warp - CONV_W0] = mxd;
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue (the last warpgroup)
        // Chunk sums (fp32 from the tensor core, 128 columns each) are carried across the tile: in fp64
        // registers with one converter team; with two teams (whose registers leave the epilogue 64) as
        // error-free (hi, lo) fp32 pairs in the 128 spare TMEM columns ACC_COL0.. .  (Restarting the
        // accumulator every 128 columns bounds the bias of the tensor core's truncating accumulation.)
        if constexpr (REG_EPI > REG_LAUNCH)
            setmaxnreg_inc<REG_EPI>();
        else if constexpr (REG_EPI < REG_LAUNCH)
            setmaxnreg_dec<REG_EPI>();
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        double attn = 0.0;
        uint32_t gc = 0;
        [[maybe_unused]] double acc[NTEAMS == 1 ? BN : 1];
        for (UnitWalk w(us); w.ok(); w.next(), gc++) {
            const int tile = w.tile, grp = w.grp;
            const bool piece = w.in_piece();  // a K-range of a split tail tile (else part of a whole tile)
            const bool first = piece ? w.piece_first() : grp == 0;
            const bool last = piece ? grp == w.pend - 1 : grp == ngrp - 1;
            const int ab = gc & 1;
            mbar_wait_sleep(&s.full_acc[ab], (gc >> 1) & 1);
            tc_fence_after();
            if constexpr (NTEAMS == 1) {
                if (first) {
#pragma unroll
                    for (int j = 0; j < BN; j++) acc[j] = 0.0;
                }
                uint32_t v[32];
#pragma unroll
                for (int hh = 0; hh < BN / 32; hh++) {
                    tmem_ld32(tbase + lane_off + ab * BN + 32 * hh, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; j++) acc[32 * hh + j] += (double)__uint_as_float(v[j]);
                }
            } else {
                // running sum (hi, lo) as an unevaluated fp32 pair (Knuth TwoSum per chunk: error-free
                // addition, so the carry is as accurate as the fp64 one it replaces)
#pragma unroll 1
                for (int hh = 0; hh < BN / 8; hh++) {
                    uint32_t v[8], a[8], b[8];
                    const uint32_t thi = tbase + lane_off + ACC_COL0 + 8 * hh, tlo = thi + BN;
                    tmem_ld8(tbase + lane_off + ab * BN + 8 * hh, v);
                    if (!first) {
                        tmem_ld8(thi, a);
                        tmem_ld8(tlo, b);
                    }
                    tmem_wait_ld();
                    if (first) {
#pragma unroll
                        for (int j = 0; j < 8; j++) b[j] = 0u;
                    } else {
#pragma unroll
                        for (int j = 0; j < 8; j += 2) {
                            const uint64_t x = f2pk(__uint_as_float(a[j]), __uint_as_float(a[j + 1]));
                            const uint64_t y = f2pk(__uint_as_float(v[j]), __uint_as_float(v[j + 1]));
                            const uint64_t sm = f2add(x, y);
                            const uint64_t yy = f2sub(sm, x);
                            const uint64_t er = f2add(f2sub(x, f2sub(sm, yy)), f2sub(y, yy));
                            const uint64_t lo = f2add(f2pk(__uint_as_float(b[j]), __uint_as_float(b[j + 1])), er);
                            v[j] = __float_as_uint(f2lo(sm));
                            v[j + 1] = __float_as_uint(f2hi(sm));
                            b[j] = __float_as_uint(f2lo(lo));
                            b[j + 1] = __float_as_uint(f2hi(lo));
                        }
                    }
                    tmem_st8(thi, v);
                    tmem_st8(tlo, b);
                }
                tmem_wait_st();
            }
            tc_fence_before();
            mbar_arrive(&s.empty_acc[ab]);
            if (!last) continue;  // tile / piece not finished
            const bool whole = !piece;  // the whole tile row-block is this CTA's: Delta is complete
            const int64_t row = (int64_t)tile * BM + r;
            // a piece of a split tail tile: its own fp64 slot (piece index w.pi), summed by split_combine_kernel
            double *slot = piece ? p.split + (int64_t)w.pi * (BN * BM) : nullptr;
#pragma unroll 1
            for (int hh = 0; hh < (NTEAMS == 1 ? 1 : BN / 8); hh++) {
                constexpr int NJ = NTEAMS == 1 ? BN : 8;
                uint32_t a[8], b[8];
                if constexpr (NTEAMS > 1) {
                    tmem_ld8(tbase + lane_off + ACC_COL0 + 8 * hh, a);
                    tmem_ld8(tbase + lane_off + ACC_COL0 + BN + 8 * hh, b);
                    tmem_wait_ld();
                }
#pragma unroll
                for (int jj = 0; jj < NJ; jj++) {
                    const int j = (NTEAMS == 1 ? 0 : 8 * hh) + jj;
                    double dv;
                    if constexpr (NTEAMS == 1)
                        dv = acc[jj];
                    else
                        dv = (double)__uint_as_float(a[jj]) + (double)__uint_as_float(b[jj]);
                    if (whole) {
                        if (row < T && j < nq) {
                            if (MODE != 1)
                                attn += fabs(dv);
                            else
                                p.S[(int64_t)j * T + row] = (float)dv;
                        }
                    } else if (MODE != 1) {
                        slot[j * BM + r] = dv;
                    }
                }
            }
        }
        if (MODE != 1) {
            for (int o = 16; o > 0; o >>= 1) attn += __shfl_xor_sync(0xffffffffu, attn, o);
            if (lane == 0) s.red[1][quarter] = attn;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (MODE != 1 && threadIdx.x == 0) {
        Partial pt{0.0, 0.0, 0.0, 0.0};
        for (int i = 0; i < NTEAMS * 8; i++) {  // fixed order: deterministic
            pt.sum_sq += s.red[0][i];
            pt.max_abs = fmax(pt.max_abs, s.red[2][i]);
        }
        for (int i = 0; i < 4; i++) pt.attn_abs += s.red[1][i];
        p.partials[blockIdx.x] = pt;
    }
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<TMEM_COLS>(tbase);
    }
    if constexpr (MODE == 2) {
        if (p.ticket) last_cta_reduce(p, reinterpret_cast<int *>(s.buf));
    }
}

}  // namespace tc
}  // namespace kvq
#include "rt64.cuh"
namespace kvq {
namespace tc {

// ---------------------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void *ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
        cudaGetLastError();
    });
    return fn;
}

// 2-D row-major [T][D] map, box {box_cols, box_rows}, 128B swizzle (box_cols * elem = 128 B).
static bool make_map(CUtensorMap *m, const void *base, CUtensorMapDataType ty, int elem, int64_t T, int64_t D,
                     int box_cols, int box_rows = BM) {
    auto enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)T};
    cuuint64_t strides[1] = {(cuuint64_t)D * elem};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, ty, 2, const_cast<void *>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}
static bool make_map_f32(CUtensorMap *m, const float *base, int64_t T, int64_t D, int box_rows = BM) {
    return make_map(m, base, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, T, D, BK, box_rows);
}
// KVQ_TC_RT64=1: the fused roundtrip on 64-row tiles (rt64.cuh; parity-green, measured slower: see there).
static bool use_rt64() {
    const char *e = std::getenv("KVQ_TC_RT64");
    return e && e[0] == '1';
}
// K-blocks of 32 columns, rounded up to whole 64-column stages (the padded Q tiles and column records are zero)
static int64_t nkb_padded(int64_t D) { return ((D + BK - 1) / BK + 1) & ~(int64_t)1; }

}  // namespace tc

bool tc_eligible(const float *K, const float *K_hat, int64_t T, int64_t D, int64_t nq) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(K) | reinterpret_cast<uintptr_t>(K_hat);
    return nq >= 1 && nq <= tc::BN && D % 4 == 0 && (a % 16) == 0 && (T + tc::BM - 1) / tc::BM < (1LL << 31) &&
           tc::encode_fn() != nullptr;
}

size_t tc_qsplit_bytes(int64_t D) { return (size_t)tc::nkb_padded(D) * 2 * tc::QTILE; }

bool tc_roundtrip_eligible(const float *K, const int8_t *Kq, const float *K_hat, int64_t T, int64_t D, int64_t nq) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(K) | reinterpret_cast<uintptr_t>(Kq) |
                        reinterpret_cast<uintptr_t>(K_hat);
    return tc_eligible(K, K_hat, T, D, nq) && D % 16 == 0 && (a % 16) == 0;
}

size_t tc_colq_bytes(int64_t D) { return (size_t)tc::nkb_padded(D) * sizeof(tc::ColRec); }

size_t tc_split_bytes(int64_t T, int64_t D) {
    // work units of either geometry: 128-row tiles x 4 K-blocks, 64-row tiles x 4 stages of 64 columns
    const int64_t n128 = (T + tc::BM - 1) / tc::BM * (((D + tc::BK - 1) / tc::BK + tc::CODE_KB - 1) / tc::CODE_KB);
    const int64_t n64 = (T + tc::r64::BR - 1) / tc::r64::BR * ((tc::nkb_padded(D) / 2 + tc::r64::UNIT_ST - 1) / tc::r64::UNIT_ST);
    const int64_t nunits = std::max(n128, n64);
    return (size_t)std::min<int64_t>(nunits, kSplitMaxPieces) * tc::BN * tc::BM * sizeof(double);
}

// Tail plan of the tensor-core pass (see make_units).  Cost model in work units on the critical path: W whole
// tiles + ceil(Rt P / G) pieces of L units, + 0.9 unit-equivalents per G pieces for the fp64 slots (64 KB
// written, then read by split_combine: ~0.9 of a unit's 144 KB of K/K_hat/code traffic) + 1.5 units for the
// combine launch.  Split only when the model gains >= 3% over whole tiles (C2, 64 tiles of 8 units: 2 pieces
// each, 55.7 -> 49.8 us per step back to back; the 8-rank C4 shard, 128 tiles of 64 units, stays whole: its
// split options save no unit on the critical path).  force: -1 auto, 0 whole tiles, 1 the best split.
TailPlan tc_plan_tail(int ntiles, int ngrp, int nsm, int force) {
    TailPlan whole{std::min(ntiles, nsm), 0, 0, 1, false};
    const int G = nsm, W0 = ntiles / G;
    if (force == 0) return whole;
    const double whole_cost = (double)((ntiles + G - 1) / G) * ngrp;
    double best = 1e300;
    TailPlan bp = whole;
    for (int W = W0; W >= std::max(0, W0 - 1); W--) {
        const int rt = ntiles - W * G;
        if (rt <= 0) continue;
        for (int P = 2; P <= ngrp; P++) {
            if (ngrp % P) continue;
            const int np = rt * P;
            if (np > kSplitMaxPieces) continue;
            const double cost = (double)W * ngrp + (double)((np + G - 1) / G) * (ngrp / P) + 0.9 * np / G + 1.5;
            if (cost < best) {
                best = cost;
                bp = TailPlan{G, W, rt, P, true};
            }
        }
    }
    if (bp.split && (force == 1 || best < 0.97 * whole_cost)) return bp;
    return whole;
}

template <int MODE, bool FASTCONV = false>
static void launch_mode(const CUtensorMap &mK, const CUtensorMap &mKh, const CUtensorMap &mKq, const tc::TcParams &p,
                        int grid, size_t smem, cudaStream_t s, bool cooperative = false) {
    ensure_max_smem<tc::attn_tc_kernel<MODE, FASTCONV>>((int)smem);
    if (!cooperative) {
        (void)launch_pdl(tc::attn_tc_kernel<MODE, FASTCONV>, dim3(grid), dim3(tc::NTHREADS), smem, s, mK, mKh, mKq, p);
        return;
    }
    // grid barriers inside (fused a1 + a2): a cooperative launch guarantees co-residency (1 CTA per SM)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(tc::NTHREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    (void)cudaLaunchKernelEx(&cfg, tc::attn_tc_kernel<MODE, FASTCONV>, mK, mKh, mKq, p);
}

static void launch_rt64(const CUtensorMap &mK, const CUtensorMap &mKh, const CUtensorMap &mKq, const tc::TcParams &p,
                        int grid, cudaStream_t s, bool cooperative) {
    const size_t smem = sizeof(tc::r64::Smem);
    ensure_max_smem<tc::r64::rt64_kernel>((int)smem);
    if (!cooperative) {
        (void)launch_pdl(tc::r64::rt64_kernel, dim3(grid), dim3(tc::NTHREADS), smem, s, mK, mKh, mKq, p);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(tc::NTHREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    (void)cudaLaunchKernelEx(&cfg, tc::r64::rt64_kernel, mK, mKh, mKq, p);
}

// Launch: qsplit (into ws_q) [+ colq] + the persistent tensor-core kernel.
kvq_status launch_attn_tc(int mode, const float *K, const float *K_hat, int64_t T, int64_t D, const float *Q,
                          int64_t nq, void *ws_q, void *partials, int *grid_out, float *S, cudaStream_t s,
                          const float *scales, void *ws_colq, int8_t *Kq_out, float *Kh_out, void *ws_split,
                          float *scales_out, void *ws_pmax, const MetricTotals *fin, unsigned *ticket,
                          bool *reduced) {
    using namespace tc;
    if (reduced) *reduced = false;
    const bool fused_a1 = mode == 2 && scales_out != nullptr && ws_pmax != nullptr;
    const bool r64 = mode == 2 && use_rt64();  // the fused roundtrip on 64-row tiles (rt64.cuh), opt-in
    const int trows = r64 ? r64::BR : BM;
    // r64: K-blocks padded to whole 64-column stages (zero Q tiles and column records past D)
    const int64_t nkb = r64 ? nkb_padded(D) : (D + BK - 1) / BK;
    const int ntiles = (int)((T + trows - 1) / trows);
    CUtensorMap mK, mKh, mKq;
    if (!make_map_f32(&mK, K, T, D, trows)) return fail(KVQ_ERR_CUDA, "cuTensorMapEncodeTiled(K) failed");
    mKh = mK;
    mKq = mK;
    if (mode == 2) {
        if (!make_map_f32(&mKh, Kh_out, T, D, trows)) return fail(KVQ_ERR_CUDA, "cuTensorMapEncodeTiled(K_hat) failed");
        if (!make_map(&mKq, Kq_out, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, T, D, BK * CODE_KB, trows))
            return fail(KVQ_ERR_CUDA, "cuTensorMapEncodeTiled(Kq) failed");
    } else if (K_hat) {
        if (!make_map_f32(&mKh, K_hat, T, D)) return fail(KVQ_ERR_CUDA, "cuTensorMapEncodeTiled(K_hat) failed");
    }
    uint32_t *qs = reinterpret_cast<uint32_t *>(ws_q);
    const unsigned qblocks = (unsigned)std::min<int64_t>((nkb * BN * (BK / 4) + 255) / 256, 4096);
    if (mode != 2 || (fused_a1 && r64)) {  // (fused a1: the tensor-core kernel writes the records and Q tiles itself)
        (void)launch_pdl(qsplit_kernel, dim3(qblocks), dim3(256), 0, s, Q, nq, D, nkb, qs);
        if (kvq_status st = check_launch("qsplit"); st != KVQ_OK) return st;
    }
    TcParams p{};
    p.qsplit = qs;
    p.T = T;
    p.D = D;
    p.nq = (int)nq;
    p.ntiles = ntiles;
    p.nkb = (int)nkb;
    p.has_khat = (K_hat != nullptr && mode != 2);
    p.partials = reinterpret_cast<Partial *>(partials);
    p.S = S;
    {
        const char *e = std::getenv("KVQ_TC_HINTS");  // experiments only
        p.hints = e ? std::atoi(e) : 3;
    }
    if (mode == 2) {
        ColRec *cq = reinterpret_cast<ColRec *>(ws_colq);
        if (fused_a1) {
            p.pmax = reinterpret_cast<uint32_t *>(ws_pmax);
            p.Kin = K;
            p.scales_out = scales_out;
            p.colq_out = cq;
            if (!r64) {
                p.Qin = Q;
                p.qsplit_out = qs;
            }
        } else {
            const unsigned cblocks = (unsigned)std::min<int64_t>((nkb + 7) / 8, 1024);
            (void)launch_pdl(prep_kernel, dim3(qblocks + cblocks), dim3(256), 0, s, Q, nq, D, nkb, qs, scales, cq,
                             (int)qblocks, ticket);
            if (kvq_status st = check_launch("qsplit+colq"); st != KVQ_OK) return st;
        }
        p.colq = cq;
        p.Kh = Kh_out;
    }
    p.ngrp = r64 ? (int)((nkb / 2 + r64::UNIT_ST - 1) / r64::UNIT_ST) : (int)((nkb + CODE_KB - 1) / CODE_KB);
    // modes 0/2: whole-tile waves + a split tail when the cost model says so (see make_units, tc_plan_tail);
    // mode 1 (scores): whole tiles
    const int nsm = std::min(device_info().num_sms, kSplitMaxCtas);
    const char *force = std::getenv("KVQ_TC_BALANCE");  // experiments / tests: 0 = whole tiles, 1 = best split
    const TailPlan plan = tc_plan_tail(ntiles, p.ngrp, nsm, force ? (force[0] == '1' ? 1 : 0) : -1);
    const bool balanced = mode != 1 && ws_split != nullptr && plan.split;
    const int grid = balanced ? plan.grid : std::min(ntiles, device_info().num_sms);
    p.split = balanced ? reinterpret_cast<double *>(ws_split) : nullptr;
    p.pieces = balanced ? plan.pieces : 1;
    p.whole = balanced ? plan.whole : 0;
    p.rt = balanced ? plan.rt : 0;
    const int R = balanced ? plan.rt : 0;
    // whole tiles (the ticket zeroed by prep, or by the fused column-max phase): the pass reduces its partials itself
    if (mode == 2 && !r64 && !balanced && fin && ticket) {
        p.ticket = ticket;
        p.scales_in = scales;
        p.sums = fin->sums;
        p.maxes = fin->maxes;
        p.final_out = fin->fused_out;
        if (reduced) *reduced = true;
    }
    const size_t smem = sizeof(Smem);
    // the pass is bound per CTA when every CTA gets at most one round of work (whole tiles in one wave, or a split
    // plan with no whole-tile wave): take the faster converter there (KVQ_TC_FASTCONV=0|1 forces it off / on)
    bool fastconv = balanced ? plan.whole == 0 : ntiles <= grid;
    if (const char *e = std::getenv("KVQ_TC_FASTCONV")) fastconv = e[0] == '1';
    if (grid_out) *grid_out = balanced ? grid + COMBINE_JQ * R : grid;  // + one partial per tail tile and quarter
    if (mode == 0)
        launch_mode<0>(mK, mKh, mKq, p, grid, smem, s);
    else if (mode == 1)
        launch_mode<1>(mK, mKh, mKq, p, grid, smem, s);
    else if (r64)
        launch_rt64(mK, mKh, mKq, p, grid, s, fused_a1);
    else if (fastconv)
        launch_mode<2, true>(mK, mKh, mKq, p, grid, smem, s, fused_a1);
    else
        launch_mode<2>(mK, mKh, mKq, p, grid, smem, s, fused_a1);
    if (kvq_status st = check_launch(mode == 0 ? "attn_tc(metrics)" : mode == 1 ? "attn_tc(scores)" : "attn_tc(roundtrip)");
        st != KVQ_OK || !balanced || R == 0)
        return st;
    if (r64)
        (void)launch_pdl(r64::split_combine64_kernel, dim3(R, COMBINE_JQ), dim3(r64::BR), 0, s, (const double *)p.split,
                         T, (int)nq, plan.whole * grid, plan.rt, grid, plan.pieces, reinterpret_cast<Partial *>(partials));
    else
        (void)launch_pdl(split_combine_kernel, dim3(R, COMBINE_JQ), dim3(BM), 0, s, (const double *)p.split, T, (int)nq,
                         plan.whole * grid, plan.rt, grid, plan.pieces, reinterpret_cast<Partial *>(partials));
    return check_launch("attn_tc(split_combine)");
}

}  // namespace kvq

#ifdef KVQ_TRACE
extern "C" int kvq_debug_trace_read(void *host, size_t bytes) {
    return (int)cudaMemcpyFromSymbol(host, kvq::tc::g_kvq_trace, bytes < sizeof(kvq::tc::g_kvq_trace) ? bytes : sizeof(kvq::tc::g_kvq_trace));
}
#endif
