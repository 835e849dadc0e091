// rt64.cuh — the fused roundtrip (a3 + a4 + a5 + a6, `kvq_roundtrip`) on 64-row tiles.
// Included by attn_tc.cu after attn_tc_kernel (it reuses ColRec, TcParams, Units/UnitWalk, the converter
// arithmetic and fused_scales_phase from there).
//
// Why 64 rows.  The pass is bound by how fast the HBM absorbs its K_hat / code writes, and that depends on how
// many DRAM rows the whole GPU writes at once: with one 128-row tile per CTA (148 x 128 rows written 128 bytes
// at a time) the same 9 B/elem of traffic with no arithmetic at all runs 1.736-1.741 ms at C4, with 64-row
// tiles and 64-column stages 1.649-1.669 ms (scripts/probes/bw_mix2.cu, WIDE3; profiles/r02/probes/).
//
// The contraction (Delta = E Q^T, E = K - K_hat) still runs as M = 128 tcgen05 MMAs, with the tile's two
// 32-column halves of a 64-column stage stacked along M ("block-diagonal" use of the MMA):
//   TMEM lane l < 64:  row l of the tile, columns [c0, c0 + 32)        (box A)
//   TMEM lane l >= 64: row l - 64 of the tile, columns [c0 + 32, c0 + 64) (box B)
// Per 8-column K-step j, the A operand (all 128 lanes of E, from TMEM) is multiplied once with the Q tile of
// box A's columns into accumulator columns [0, 64) and once with the Q tile of box B's columns into columns
// [64, 128).  Lanes < 64 of the first and lanes >= 64 of the second are the wanted partial sums; the other
// two quadrants multiply E with the other half's queries columns and are ignored (the price: twice the MMA
// work per element, still < 50% of the tensor pipe).  Delta[t] = D[t][0:64] + D[t + 64][64:128], added by
// the epilogue at the end of the tile (through shared memory: lanes t and t + 64 belong to different warps).
//
// Everything else is the 128-row kernel's design: one persistent CTA per SM, warp-specialised, mbarrier
// hand-offs; two converter teams alternating stages (thread = TMEM lane x 16 columns: the same 16 elements
// per thread per stage); K_hat written in place into the input stage and stored with TMA; codes staged as
// [64 rows x 128 B] boxes (full 128-byte lines); 3xTF32 with the accumulator restarted every work unit (4
// stages = 48 accumulation steps per lane, as before) and the tile's Delta carried as error-free fp32 (hi, lo)
// pairs in TMEM.
#pragma once

namespace kvq {
namespace tc {
namespace r64 {

constexpr int BR = 64;                      // tile rows
constexpr int SC = 64;                      // stage columns (two 32-column K-blocks, boxes A and B)
constexpr uint32_t BOX = BR * BK * 4;       // one [64 x 32] fp32 box: 8 KB
constexpr uint32_t STAGE = 2 * BOX;         // 16 KB
#ifndef KVQ_R64_KST
#define KVQ_R64_KST 8
#endif
#ifndef KVQ_R64_QST
#define KVQ_R64_QST 2
#endif
constexpr int KST = KVQ_R64_KST;            // input ring (16 KB stages)
constexpr int QST = KVQ_R64_QST;            // Q ring: the two K-blocks' [hi | lo] tiles of a stage (32 KB)
constexpr uint32_t QSTAGE = 4 * QTILE;      // 32 KB
#ifdef KVQ_R64_EXP_AST4  // timing experiment only: 4 A slots, no Delta carry (attention metric wrong)
constexpr int AST = 4;
#else
constexpr int AST = 2;                      // A ring in TMEM (one slot per converter team)
#endif
constexpr int UNIT_ST = 4;                  // stages per work unit (= accumulator chunk: 48 MMA steps per lane)
constexpr int CODE_ST = 2;                  // stages per code box ([64 x 128 B])
constexpr uint32_t CODEBOX = BR * 128;      // 8 KB
constexpr uint32_t ACC_COLS = 2 * BN;       // accumulator: two 64-column halves
constexpr uint32_t A_COL0 = 2 * ACC_COLS;   // 256: after the double-buffered accumulator
#ifdef KVQ_R64_EXP_AST4
constexpr uint32_t CARRY_COL0 = A_COL0 + 2 * 64;  // overlaps A slots 2, 3: carry not written in this experiment
#else
constexpr uint32_t CARRY_COL0 = A_COL0 + AST * 64;  // 384: the tile's Delta (hi 64 | lo 64)
static_assert(CARRY_COL0 + 2 * BN == TMEM_COLS, "TMEM budget");
#endif

struct __align__(1024) Smem {
    uint8_t buf[KST * STAGE];           // input ring; K_hat is written back in place
    uint8_t codes[2][CODEBOX];          // code staging, double-buffered
    uint8_t q[QST][QSTAGE];
    ColRec cq[KST][2];                  // the stage's two column records (boxes A, B)
    double xch[8][BR];                  // epilogue: box B lanes' Delta, 8 queries at a time
    uint64_t full_k[KST], empty_k[KST], staged[KST], full_q[QST], empty_q[QST];
    uint64_t full_a[AST], empty_a[AST], full_acc[2], empty_acc[2], cstored[2];
    uint32_t tmem_base;
    double red[3][NTEAMS * 8];
};
static_assert(sizeof(Smem) <= 227 * 1024, "shared memory budget (227 KB per CTA on sm_100)");

__global__ void __launch_bounds__(NTHREADS, 1)
    rt64_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmKh,
                const __grid_constant__ CUtensorMap tmKq, const __grid_constant__ TcParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem &s = *reinterpret_cast<Smem *>(smem_raw);
    const int64_t T = p.T;
    const int nq = p.nq, nst = p.nkb / 2;  // p.nkb is even here (records and Q tiles padded)
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

    if (threadIdx.x == 0) {
        if (smem_u32(smem_raw) & 1023u) __trap();
        for (int i = 0; i < KST; i++) {
            mbar_init(&s.full_k[i], 1);
            mbar_init(&s.empty_k[i], 1);   // the store warp frees the stage
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
            mbar_init(&s.cstored[i], 1);
        }
        mbar_fence_init();
    }
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmK);
        prefetch_tmap(&tmKh);
        prefetch_tmap(&tmKq);
    }
    if (warp == 1) tmem_alloc<TMEM_COLS>(&s.tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = s.tmem_base;
    pdl_wait();
    pdl_trigger();
    if (p.pmax) fused_scales_phase<false>(p, s.buf);  // (the Q split stays a launch on this path)
    const Units us = make_units(p);

    if (warp < CONV_W0) {
        setmaxnreg_dec<REG_WG0>();
        if (warp == 0 && lane == 0) {
            // ------------------------------------------------------------ K producer
            const uint64_t pol_stream = (p.hints & 1) ? policy_evict_first() : policy_evict_normal();
            const uint64_t pol_keep = policy_evict_last();
            uint32_t g = 0;
            for (UnitWalk w(us); w.ok(); w.next()) {
                const int tile = w.tile, st0 = w.grp * UNIT_ST, st1 = min(st0 + UNIT_ST, nst);
#pragma unroll 1
                for (int st = st0; st < st1; st++, g++) {
                    const int sk = g % KST;
                    mbar_wait_sleep(&s.empty_k[sk], ((g / KST) & 1) ^ 1);
                    KVQ_TR(0, true);
                    mbar_arrive_tx(&s.full_k[sk], STAGE + 2 * (uint32_t)sizeof(ColRec));
                    uint8_t *stg = s.buf + sk * STAGE;
                    tma_load_2d(stg, &tmK, &s.full_k[sk], st * SC, tile * BR, pol_stream);
                    tma_load_2d(stg + BOX, &tmK, &s.full_k[sk], st * SC + BK, tile * BR, pol_stream);
                    bulk_load(&s.cq[sk][0], p.colq + 2 * st, 2 * sizeof(ColRec), &s.full_k[sk], pol_keep);
                }
            }
        } else if (warp == 3 && lane == 0) {
            // ------------------------------------------------------------ Q producer (L2-resident tiles)
            const uint64_t pol_keep = policy_evict_last();
            uint32_t g = 0;
            for (UnitWalk w(us); w.ok(); w.next()) {
                const int st0 = w.grp * UNIT_ST, st1 = min(st0 + UNIT_ST, nst);
#pragma unroll 1
                for (int st = st0; st < st1; st++, g++) {
                    const int sq = g % QST;
                    mbar_wait_sleep(&s.empty_q[sq], ((g / QST) & 1) ^ 1);
                    mbar_arrive_tx(&s.full_q[sq], QSTAGE);
                    bulk_load(s.q[sq], p.qsplit + (size_t)(2 * st) * (2 * BN * BK), QSTAGE, &s.full_q[sq], pol_keep);
                }
            }
        } else if (warp == 2 && lane == 0) {
            // ------------------------------------------------------------ output stores
            const uint64_t pol_out = (p.hints & 2) ? policy_evict_first() : policy_evict_normal();
            uint32_t g = 0, cg = 0;
            bool prev_code_end = false;
            for (UnitWalk w(us); w.ok(); w.next()) {
                const int tile = w.tile, st0 = w.grp * UNIT_ST, st1 = min(st0 + UNIT_ST, nst);
#pragma unroll 1
                for (int st = st0; st < st1; st++, g++) {
                    const int sk = g % KST;
                    mbar_wait_sleep(&s.staged[sk], (g / KST) & 1);
                    KVQ_TR(7, true);
                    const uint8_t *stg = s.buf + sk * STAGE;
                    tma_store_2d(&tmKh, stg, st * SC, tile * BR, pol_out);
                    tma_store_2d(&tmKh, stg + BOX, st * SC + BK, tile * BR, pol_out);
                    const bool code_end = ((st - st0) % CODE_ST) == CODE_ST - 1 || st == st1 - 1;
                    if (code_end)
                        tma_store_2d(&tmKq, s.codes[cg & 1], (st - (st - st0) % CODE_ST) * SC, tile * BR, pol_out);
                    bulk_commit();
                    if (g > 0) {
                        bulk_wait_read<1>();  // stage g-1's boxes have left shared memory
                        KVQ_TR(8, true);
                        mbar_arrive(&s.empty_k[(g - 1) % KST]);
                        if (prev_code_end) mbar_arrive(&s.cstored[(cg - 1) & 1]);
                    }
                    prev_code_end = code_end;
                    if (code_end) cg++;
                }
            }
            bulk_wait<0>();
        } else if (warp == 1) {
            // ------------------------------------------------------------ MMA issuer (whole warp walks, one lane issues)
            uint32_t g = 0, gc = 0;
            for (UnitWalk w(us); w.ok(); w.next(), gc++) {
                const int st0 = w.grp * UNIT_ST, st1 = min(st0 + UNIT_ST, nst);
                const int ab = gc & 1;
                const uint32_t d0 = tbase + ab * ACC_COLS;
                KVQ_WAIT_HOT(&s.empty_acc[ab], ((gc >> 1) & 1) ^ 1);
                tc_fence_after();
#pragma unroll 1
                for (int st = st0; st < st1; st++, g++) {
                    const int sa = g % AST, sq = g % QST;
                    KVQ_WAIT_HOT(&s.full_a[sa], (g / AST) & 1);
                    KVQ_TR(9, lane == 0);
                    KVQ_WAIT_HOT(&s.full_q[sq], (g / QST) & 1);
                    KVQ_TR(15, lane == 0);
                    tc_fence_after();
                    const uint32_t ahi = tbase + A_COL0 + sa * 64, alo = ahi + 32;
                    const uint32_t qb = smem_u32(s.q[sq]);
                    const bool first = st == st0;
                    if (elect_one()) {
#pragma unroll
                        for (int x = 0; x < 2; x++) {  // x = 0: box A's queries columns -> D[:, 0:64]; x = 1 -> D[:, 64:128]
                            const uint64_t bh = smem_desc(qb + x * 2 * QTILE, 1024, 128);
                            const uint64_t bl = smem_desc(qb + x * 2 * QTILE + QTILE, 1024, 128);
                            const uint32_t d = d0 + x * BN;
#pragma unroll
                            for (int j = 0; j < BK / 8; j++) {
#ifndef KVQ_EXP_NOMMA  // timing experiments only (Delta not computed)
                                mma_tf32_ts(d, ahi + 8 * j, bh + 128u * j, IDESC, (!first || j != 0) ? 1u : 0u);
                                mma_tf32_ts(d, ahi + 8 * j, bl + 128u * j, IDESC, 1);
                                mma_tf32_ts(d, alo + 8 * j, bh + 128u * j, IDESC, 1);
#endif
                            }
                        }
                        mma_commit(&s.empty_a[sa]);
                        mma_commit(&s.empty_q[sq]);
                        if (st == st1 - 1) mma_commit(&s.full_acc[ab]);
                    }
                    __syncwarp();
                    KVQ_TR(10, lane == 0);
                }
            }
        }
    } else if (warp < EPI_W0) {
        // ------------------------------------------------------------ converters
        if constexpr (REG_CONV > REG_LAUNCH) setmaxnreg_inc<REG_CONV>();
        const int team = (warp - CONV_W0) / NCONV_W;
        const int quarter = warp & 3;
        const int h = ((warp - CONV_W0) % NCONV_W) >> 2;  // 16-column half of the box row
        const int l = quarter * 32 + lane;                // TMEM lane
        const int r = l & (BR - 1), bx = l >> 6;          // tile row, box (A: columns c0.., B: c0 + 32..)
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        double ss = 0.0;
        float mx = 0.0f;
        uint32_t g = 0, cg = 0;
        for (UnitWalk w(us); w.ok(); w.next()) {
            const int st0 = w.grp * UNIT_ST, st1 = min(st0 + UNIT_ST, nst);
            bool code_buf_ready = false;
#pragma unroll 1
            for (int st = st0; st < st1; st++, g++) {
                const bool code_end = ((st - st0) % CODE_ST) == CODE_ST - 1 || st == st1 - 1;
                if (NTEAMS > 1 && (int)(g % NTEAMS) != team) {
                    if (code_end) {
                        cg++;
                        code_buf_ready = false;
                    }
                    continue;
                }
                const int sk = g % KST;
                [[maybe_unused]] const bool tw0 = lane == 0 && (warp - CONV_W0) % NCONV_W == 0;
                KVQ_TR(14, tw0);
                KVQ_WAIT_HOT(&s.full_k[sk], (g / KST) & 1);
                KVQ_TR(1, tw0);
                KVQ_TR(5, lane == 0 && (warp - CONV_W0) % NCONV_W == NCONV_W - 1);
                const uint32_t kbase = smem_u32(s.buf + sk * STAGE) + bx * BOX;
                uint64_t X[8], V[8], XH[8], E[8];
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    const float4 a = lds128(swz(kbase, r, 4 * h + c));
                    X[2 * c] = f2pk(a.x, a.y);
                    X[2 * c + 1] = f2pk(a.z, a.w);
                }
                const ColRec &rec = s.cq[sk][bx];
                const uint32_t cyb = smem_u32(&rec) + 64 * h;
                const uint64_t M2 = f2pk(kMagic, kMagic);
                float amax = 0.0f, dmax = 0.0f;
#pragma unroll
                for (int c = 0; c < 4; c++) {
                    const float4 y4 = lds128(cyb + 16 * c);
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
                if (dmax > kDangerThr || amax > 127.25f || rec.any_exact) {
                    // rare: near-tie quotient, quotient past the clamp, or an exact-path column (see attn_tc_kernel)
#pragma unroll
                    for (int i = 0; i < 16; i++) {
                        const float sc = rec.s[16 * h + i], yy = rec.y[16 * h + i];
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
                KVQ_TR(11, tw0);
                KVQ_TR(32 + (warp - CONV_W0) % NCONV_W, lane == 0);
                if (!code_buf_ready) {
                    KVQ_WAIT_HOT(&s.cstored[cg & 1], ((cg >> 1) & 1) ^ 1);
                    code_buf_ready = true;
                }
                const uint32_t cds = smem_u32(s.codes[cg & 1]);
#pragma unroll
                for (int c = 0; c < 4; c++)
                    sts128(swz(kbase, r, 4 * h + c), make_float4(f2lo(XH[2 * c]), f2hi(XH[2 * c]),
                                                                 f2lo(XH[2 * c + 1]), f2hi(XH[2 * c + 1])));
                uint4 wv;
                wv.x = pack4(f2lo(V[0]), f2hi(V[0]), f2lo(V[1]), f2hi(V[1]));
                wv.y = pack4(f2lo(V[2]), f2hi(V[2]), f2lo(V[3]), f2hi(V[3]));
                wv.z = pack4(f2lo(V[4]), f2hi(V[4]), f2lo(V[5]), f2hi(V[5]));
                wv.w = pack4(f2lo(V[6]), f2hi(V[6]), f2lo(V[7]), f2hi(V[7]));
                // 16-byte chunk of the row's 128 B code line: stage (st - st0) % 2, box, half
                sts128u(swz(cds, r, 4 * ((st - st0) % CODE_ST) + 2 * bx + h), wv);
                KVQ_TR(12, tw0);
                fence_proxy_async();
                KVQ_TR(13, tw0);
                mbar_arrive(&s.staged[sk]);
                KVQ_TR(2, tw0);
                KVQ_TR(16 + (warp - CONV_W0) % NCONV_W, lane == 0);
                if (code_end) {
                    cg++;
                    code_buf_ready = false;
                }
#pragma unroll
                for (int j = 0; j < 8; j++) E[j] = f2sub(X[j], XH[j]);  // exact (fact 4)
                uint64_t sq = f2mul(E[0], E[0]);
#pragma unroll
                for (int j = 1; j < 8; j++) sq = f2fma(E[j], E[j], sq);
#pragma unroll
                for (int j = 0; j < 8; j++) mx = fmaxf(mx, fmaxf(fabsf(f2lo(E[j])), fabsf(f2hi(E[j]))));
                ss += (double)__fadd_rn(f2lo(sq), f2hi(sq));
                uint32_t hi[16], lo[16];
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    hi[2 * j] = __float_as_uint(f2lo(E[j])) & 0xFFFFE000u;
                    hi[2 * j + 1] = __float_as_uint(f2hi(E[j])) & 0xFFFFE000u;
                    const uint64_t lv = f2sub(E[j], f2pk(__uint_as_float(hi[2 * j]), __uint_as_float(hi[2 * j + 1])));
                    lo[2 * j] = __float_as_uint(f2lo(lv));
                    lo[2 * j + 1] = __float_as_uint(f2hi(lv));
                }
                const int sa = g % AST;
                KVQ_WAIT_HOT(&s.empty_a[sa], ((g / AST) & 1) ^ 1);
                KVQ_TR(3, tw0);
                tc_fence_after();
                tmem_st16(tbase + lane_off + A_COL0 + sa * 64 + 16 * h, hi);
                tmem_st16(tbase + lane_off + A_COL0 + sa * 64 + 32 + 16 * h, lo);
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.full_a[sa]);
                KVQ_TR(4, tw0);
                KVQ_TR(6, lane == 0 && (warp - CONV_W0) % NCONV_W == NCONV_W - 1);
            }
        }
        double mxd = (double)mx;
        for (int o = 16; o > 0; o >>= 1) {
            ss += __shfl_xor_sync(0xffffffffu, ss, o);
            mxd = fmax(mxd, __shfl_xor_sync(0xffffffffu, mxd, o));
        }
        if (lane == 0) {
            s.red[0][warp - CONV_W0] = ss;
            s.red[2][warp - CONV_W0] = mxd;
        }
    } else {
        // ------------------------------------------------------------ epilogue
        if constexpr (REG_EPI > REG_LAUNCH)
            setmaxnreg_inc<REG_EPI>();
        else if constexpr (REG_EPI < REG_LAUNCH)
            setmaxnreg_dec<REG_EPI>();
        const int quarter = warp & 3;
        const int l = quarter * 32 + lane, r = l & (BR - 1), bx = l >> 6;
        const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
        const uint32_t thi = tbase + lane_off + CARRY_COL0, tlo = thi + BN;
        double attn = 0.0;
        uint32_t gc = 0;
        for (UnitWalk w(us); w.ok(); w.next(), gc++) {
            const int tile = w.tile, grp = w.grp;
            const bool piece = w.in_piece();
            const bool first = piece ? w.piece_first() : grp == 0;
            const bool last = piece ? grp == w.pend - 1 : grp == p.ngrp - 1;
            const int ab = gc & 1;
            mbar_wait_sleep(&s.full_acc[ab], (gc >> 1) & 1);
            tc_fence_after();
            // this lane's wanted quadrant: box A lanes read accumulator columns [0, 64), box B lanes [64, 128)
            const uint32_t tacc = tbase + lane_off + ab * ACC_COLS + bx * BN;
#ifdef KVQ_R64_EXP_AST4
            if (true) {
                uint32_t v[8];
                tmem_ld8(tacc, v);
                tmem_wait_ld();
            } else
#endif
#pragma unroll 1
            for (int hh = 0; hh < BN / 8; hh++) {
                uint32_t v[8], a[8], b[8];
                tmem_ld8(tacc + 8 * hh, v);
                if (!first) {
                    tmem_ld8(thi + 8 * hh, a);
                    tmem_ld8(tlo + 8 * hh, b);
                }
                tmem_wait_ld();
                if (first) {
#pragma unroll
                    for (int j = 0; j < 8; j++) b[j] = 0u;
                } else {
#pragma unroll
                    for (int j = 0; j < 8; j += 2) {  // Knuth TwoSum on pairs: error-free carry
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
                tmem_st8(thi + 8 * hh, v);
                tmem_st8(tlo + 8 * hh, b);
            }
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&s.empty_acc[ab]);
            if (!last) continue;
            const int64_t row = (int64_t)tile * BR + r;
            if (piece) {
                // a K-range of a split tail tile: both boxes' lanes write their own fp64 slot rows; the combine
                // kernel adds lanes t and t + 64 of every piece in piece order
                double *slot = p.split + (int64_t)w.pi * (BN * BM);
#pragma unroll 1
                for (int hh = 0; hh < BN / 8; hh++) {
                    uint32_t a[8], b[8];
                    tmem_ld8(thi + 8 * hh, a);
                    tmem_ld8(tlo + 8 * hh, b);
                    tmem_wait_ld();
#pragma unroll
                    for (int jj = 0; jj < 8; jj++)
                        slot[(8 * hh + jj) * BM + l] = (double)__uint_as_float(a[jj]) + (double)__uint_as_float(b[jj]);
                }
                continue;
            }
            // whole tile: Delta[t][j] = carry(lane t) + carry(lane t + 64), 8 queries at a time through smem
#pragma unroll 1
            for (int hh = 0; hh < BN / 8; hh++) {
                uint32_t a[8], b[8];
                tmem_ld8(thi + 8 * hh, a);
                tmem_ld8(tlo + 8 * hh, b);
                tmem_wait_ld();
                if (bx == 1) {
#pragma unroll
                    for (int jj = 0; jj < 8; jj++)
                        s.xch[jj][r] = (double)__uint_as_float(a[jj]) + (double)__uint_as_float(b[jj]);
                }
                named_bar_sync(1, 128);
                if (bx == 0) {
#pragma unroll
                    for (int jj = 0; jj < 8; jj++) {
                        const int j = 8 * hh + jj;
                        const double dv = (double)__uint_as_float(a[jj]) + (double)__uint_as_float(b[jj]) + s.xch[jj][r];
                        if (row < T && j < nq) attn += fabs(dv);
                    }
                }
                named_bar_sync(1, 128);
            }
        }
        for (int o = 16; o > 0; o >>= 1) attn += __shfl_xor_sync(0xffffffffu, attn, o);
        if (lane == 0) s.red[1][quarter] = attn;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
        Partial pt{0.0, 0.0, 0.0, 0.0};
        for (int i = 0; i < NTEAMS * 8; i++) {
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
}

// Split tail on 64-row tiles: block (r, y) adds, for the 64 rows of tail tile r and queries [16y, 16y + 16),
// lanes t and t + 64 of the P piece slots in piece order, takes |Delta| and writes partial G + r * COMBINE_JQ + y.
__global__ void __launch_bounds__(BR) split_combine64_kernel(const double *__restrict__ split, int64_t T, int nq,
                                                             int wbase, int rt, int G, int P, Partial *partials) {
    constexpr int JN = BN / COMBINE_JQ;
    const int r_t = blockIdx.x, r = threadIdx.x, j0 = blockIdx.y * JN;
    pdl_wait();
    pdl_trigger();
    const int64_t row = ((int64_t)wbase + r_t) * BR + r;
    double d[JN];
#pragma unroll
    for (int j = 0; j < JN; j++) d[j] = 0.0;
    for (int pc = 0; pc < P; pc++) {
        const double *sp = split + ((int64_t)pc * rt + r_t) * (BN * BM) + (int64_t)j0 * BM;
#pragma unroll
        for (int j = 0; j < JN; j++)
            if (j0 + j < nq) d[j] += sp[j * BM + r] + sp[j * BM + BR + r];
    }
    double attn = 0.0;
    if (row < T)
#pragma unroll
        for (int j = 0; j < JN; j++) attn += fabs(d[j]);
    __shared__ double red[BR];
    red[r] = attn;
    __syncthreads();
    for (int o = BR / 2; o > 0; o >>= 1) {
        if (r < o) red[r] += red[r + o];
        __syncthreads();
    }
    if (r == 0) partials[G + r_t * COMBINE_JQ + blockIdx.y] = Partial{0.0, red[0], 0.0, 0.0};
}

}  // namespace r64
}  // namespace tc
}  // namespace kvq
