// metrics_kernels.cu — a5 reconstruction errors and a6 attention-score error
// (P:20-24), plus raw scores for parity.
//
// One CTA owns a tile of 64 key rows and all queries.  It streams K and K_hat
// across D in 32-column chunks, forms E = K - K_hat (exact in fp32, SURVEY
// §8(c) fact 4), accumulates sum E^2 (fp64; each square is exact in fp64) and
// max |E| (exact), and contracts E with the queries:
//     Delta[i][t] = sum_d Q[i][d] * E[t][d]  ( = S - S' exactly in real arithmetic)
// Computing the difference directly avoids the cancellation of S - S'
// (|S| ~ 30, |S - S'| ~ 0.1 at D = 8192).  Each 32-term chunk is summed in
// fp32 registers, chunks are carried in fp64, so the error is bounded by
// ~32 u sum|Q E| instead of D u sum|Q E|.  Per-CTA partials are reduced by a
// single CTA in a fixed order: metrics are deterministic run to run.
#include <algorithm>
#include <cstdlib>

#include "device_common.cuh"
#include "kvq_internal.h"

namespace kvq {

constexpr int kTileRows = 64, kTileQ = 64, kChunk = 32, kPad = 68;

// MODE 0: metrics partials (E = K - K_hat).  MODE 1: write S (E = K or K - K_hat) to `S`.
template <int MODE>
__global__ void __launch_bounds__(256) attn_tile_kernel(const float *__restrict__ K, const float *__restrict__ Kh,
                                                        const float *__restrict__ Q, int64_t T, int64_t D,
                                                        int64_t nq, Partial *__restrict__ partials,
                                                        float *__restrict__ S) {
    __shared__ __align__(16) float Es[kChunk][kPad];
    __shared__ __align__(16) float Qs[kChunk][kPad];
    __shared__ double red[3][8];
    const int tid = threadIdx.x;
    const int ty = tid / 16, tx = tid % 16;  // compute mapping: rows ty*4.., queries tx*4..
    const int lr = tid / 4, lk = (tid % 4) * 8;  // load mapping: row lr, columns lk..lk+7 of the chunk
    const int64_t row0 = (int64_t)blockIdx.x * kTileRows;
    const int64_t grow = row0 + lr;
    const bool vec = (D % 4 == 0) && ((reinterpret_cast<uintptr_t>(K) | reinterpret_cast<uintptr_t>(Kh) |
                                       reinterpret_cast<uintptr_t>(Q)) % 16 == 0);
    double ss = 0.0, attn = 0.0;
    float mx = 0.0f;
    const int64_t nqt = nq > 0 ? (nq + kTileQ - 1) / kTileQ : 1;
    for (int64_t qt = 0; qt < nqt; qt++) {
        double dacc[4][4];
#pragma unroll
        for (int i = 0; i < 4; i++)
#pragma unroll
            for (int j = 0; j < 4; j++) dacc[i][j] = 0.0;
        const int64_t gq = qt * kTileQ + lr;  // query row loaded by this thread
        for (int64_t k0 = 0; k0 < D; k0 += kChunk) {
            // ---- load E chunk (64 rows x 32 cols) and Q chunk (64 queries x 32 cols)
            float e[8], qv[8];
            if (vec && k0 + lk + 8 <= D) {
                float4 a0 = make_float4(0, 0, 0, 0), a1 = a0, b0 = a0, b1 = a0, c0 = a0, c1 = a0;
                if (grow < T) {
                    const float4 *kp = reinterpret_cast<const float4 *>(K + grow * D + k0 + lk);
                    a0 = ld_stream_f4(kp);
                    a1 = ld_stream_f4(kp + 1);
                    if (Kh) {
                        const float4 *hp = reinterpret_cast<const float4 *>(Kh + grow * D + k0 + lk);
                        b0 = ld_stream_f4(hp);
                        b1 = ld_stream_f4(hp + 1);
                    }
                }
                if (nq > 0 && gq < nq) {
                    const float4 *qp = reinterpret_cast<const float4 *>(Q + gq * D + k0 + lk);
                    c0 = __ldg(qp);
                    c1 = __ldg(qp + 1);
                }
                e[0] = a0.x - b0.x; e[1] = a0.y - b0.y; e[2] = a0.z - b0.z; e[3] = a0.w - b0.w;
                e[4] = a1.x - b1.x; e[5] = a1.y - b1.y; e[6] = a1.z - b1.z; e[7] = a1.w - b1.w;
                qv[0] = c0.x; qv[1] = c0.y; qv[2] = c0.z; qv[3] = c0.w;
                qv[4] = c1.x; qv[5] = c1.y; qv[6] = c1.z; qv[7] = c1.w;
            } else {
#pragma unroll
                for (int j = 0; j < 8; j++) {
                    const int64_t col = k0 + lk + j;
                    float a = 0.0f, b = 0.0f, c = 0.0f;
                    if (grow < T && col < D) {
                        a = K[grow * D + col];
                        if (Kh) b = Kh[grow * D + col];
                    }
                    if (nq > 0 && gq < nq && col < D) c = Q[gq * D + col];
                    e[j] = a - b;
                    qv[j] = c;
                }
            }
#pragma unroll
            for (int j = 0; j < 8; j++) {
                if (MODE == 0 && qt == 0) {
                    ss += (double)e[j] * (double)e[j];
                    mx = fmaxf(mx, fabsf(e[j]));
                }
                Es[lk + j][lr] = e[j];
                Qs[lk + j][lr] = qv[j];
            }
            __syncthreads();
            if (nq > 0) {
                float acc[4][4];
#pragma unroll
                for (int i = 0; i < 4; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++) acc[i][j] = 0.0f;
#pragma unroll 8
                for (int k = 0; k < kChunk; k++) {
                    const float4 a = *reinterpret_cast<const float4 *>(&Es[k][ty * 4]);
                    const float4 b = *reinterpret_cast<const float4 *>(&Qs[k][tx * 4]);
                    const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                    for (int i = 0; i < 4; i++)
#pragma unroll
                        for (int j = 0; j < 4; j++) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
                }
#pragma unroll
                for (int i = 0; i < 4; i++)
#pragma unroll
                    for (int j = 0; j < 4; j++) dacc[i][j] += (double)acc[i][j];
            }
            __syncthreads();
        }
        if (nq > 0) {
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const int64_t r = row0 + ty * 4 + i;
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const int64_t qi = qt * kTileQ + tx * 4 + j;
                    if (r < T && qi < nq) {
                        if (MODE == 0)
                            attn += fabs(dacc[i][j]);
                        else
                            S[qi * T + r] = (float)dacc[i][j];
                    }
                }
            }
        }
    }
    if (MODE == 0) {
        // fixed-order block reduction: warp shuffle tree, then warp 0 over the 8 warp results
        double mxd = (double)mx;
        for (int o = 16; o > 0; o >>= 1) {
            ss += __shfl_xor_sync(0xffffffffu, ss, o);
            attn += __shfl_xor_sync(0xffffffffu, attn, o);
            mxd = fmax(mxd, __shfl_xor_sync(0xffffffffu, mxd, o));
        }
        const int w = tid / 32, l = tid % 32;
        if (l == 0) {
            red[0][w] = ss;
            red[1][w] = attn;
            red[2][w] = mxd;
        }
        __syncthreads();
        if (tid == 0) {
            Partial p{0.0, 0.0, 0.0, 0.0};
            for (int i = 0; i < 8; i++) {
                p.sum_sq += red[0][i];
                p.attn_abs += red[1][i];
                p.max_abs = fmax(p.max_abs, red[2][i]);
            }
            partials[blockIdx.x] = p;
        }
    }
}

// Single CTA: fixed-order reduction of the per-tile partials, plus
// theoretical_max = max_d s_d / 2 (Eq. 9) and the element counts.
__global__ void __launch_bounds__(1024) reduce_partials_kernel(const Partial *__restrict__ partials, int64_t np,
                                                               const float *__restrict__ scales, int64_t D,
                                                               double n_elems, double n_scores, double *sums,
                                                               uint64_t *maxes, kvq_metrics *out) {
    pdl_wait();  // partials of the preceding tensor-core pass / split_combine
    pdl_trigger();
    // fixed-order two-level reduction (xor butterfly within each warp, then warp 0 over the 32 warp
    // results): deterministic, and 2 barriers instead of a 10-level shared-memory tree per quantity
    __shared__ double sh[4][32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    double ss = 0.0, at = 0.0, mx = 0.0, th = 0.0;
    for (int64_t i = tid; i < np; i += 1024) {
        ss += partials[i].sum_sq;
        at += partials[i].attn_abs;
        mx = fmax(mx, partials[i].max_abs);
    }
    if (scales)
        for (int64_t d = tid; d < D; d += 1024) th = fmax(th, (double)scales[d] / 2.0);
    for (int o = 16; o > 0; o >>= 1) {
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
        at += __shfl_xor_sync(0xffffffffu, at, o);
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        th = fmax(th, __shfl_xor_sync(0xffffffffu, th, o));
    }
    if (lane == 0) {
        sh[0][wid] = ss;
        sh[1][wid] = at;
        sh[2][wid] = mx;
        sh[3][wid] = th;
    }
    __syncthreads();
    if (wid != 0) return;
    ss = sh[0][lane];
    at = sh[1][lane];
    mx = sh[2][lane];
    th = sh[3][lane];
    for (int o = 16; o > 0; o >>= 1) {
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
        at += __shfl_xor_sync(0xffffffffu, at, o);
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        th = fmax(th, __shfl_xor_sync(0xffffffffu, th, o));
    }
    const double maxabs = fmax(mx, 0.0);
    if (tid == 0) {
        sums[0] = ss;
        sums[1] = at;
        sums[2] = n_elems;
        sums[3] = n_scores;
        maxes[0] = (uint64_t)__double_as_longlong(maxabs);
        maxes[1] = (uint64_t)__double_as_longlong(th);
        if (out) {  // single process: the final struct too (same arithmetic as metrics_finalize_kernel)
            kvq_metrics m;
            m.sum_sq = ss;
            m.attn_abs_sum = at;
            m.n_elems = (int64_t)n_elems;
            m.n_scores = (int64_t)n_scores;
            m.l2 = sqrt(ss);
            m.max_abs = maxabs;
            m.theoretical_max = th;
            m.attn_mean_abs = n_scores > 0.0 ? at / n_scores : 0.0;
            *out = m;
        }
    }
}

__global__ void metrics_finalize_kernel(const double *sums, const uint64_t *maxes, kvq_metrics *out) {
    pdl_wait();
    kvq_metrics m;
    m.sum_sq = sums[0];
    m.attn_abs_sum = sums[1];
    m.n_elems = (int64_t)sums[2];
    m.n_scores = (int64_t)sums[3];
    m.l2 = sqrt(sums[0]);
    m.max_abs = __longlong_as_double((long long)maxes[0]);
    m.theoretical_max = __longlong_as_double((long long)maxes[1]);
    m.attn_mean_abs = sums[3] > 0.0 ? sums[1] / sums[3] : 0.0;
    *out = m;
}

// ---------------------------------------------------------------------------- host side
static int64_t num_tiles(int64_t T) { return (T + kTileRows - 1) / kTileRows; }

bool force_simt() {
    const char *e = std::getenv("KVQ_FORCE_SIMT");
    return e && e[0] == '1';
}

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

// workspace: [partials (max(simt tiles, 1024 CTAs)) | Q split tiles | column constants | totals]
struct WsLayout {
    Partial *partials;
    void *qsplit;
    void *colq;
    void *split;  // tensor-core kernels: fp64 Delta of tiles split between CTAs
    double *sums;
    uint64_t *maxes;
    unsigned *ticket;  // the roundtrip pass's last-CTA reduction (attn_tc.cu last_cta_reduce)
};

static WsLayout ws_layout(void *ws, int64_t T, int64_t D) {
    const uintptr_t base = (reinterpret_cast<uintptr_t>(ws) + 255) & ~(uintptr_t)255;
    const size_t np = (size_t)metrics_partials_count(num_tiles(T));
    WsLayout L;
    uintptr_t off = base;
    L.partials = reinterpret_cast<Partial *>(off);
    off += al256(np * sizeof(Partial));
    L.qsplit = reinterpret_cast<void *>(off);
    off += al256(tc_qsplit_bytes(D));
    L.colq = reinterpret_cast<void *>(off);
    off += al256(tc_colq_bytes(D));
    L.split = reinterpret_cast<void *>(off);
    off += al256(tc_split_bytes(T, D));
    L.sums = reinterpret_cast<double *>(off);
    L.maxes = reinterpret_cast<uint64_t *>(L.sums + 4);
    L.ticket = reinterpret_cast<unsigned *>(L.maxes + 2);
    return L;
}

size_t metrics_workspace_size(int64_t T, int64_t D, int64_t nq) {
    (void)nq;
    const size_t np = (size_t)metrics_partials_count(num_tiles(T));
    return 256 + al256(np * sizeof(Partial)) + al256(tc_qsplit_bytes(D)) + al256(tc_colq_bytes(D)) +
           al256(tc_split_bytes(T, D)) + 4 * sizeof(double) + 2 * sizeof(uint64_t) + 2 * sizeof(unsigned);
}

static kvq_status reduce_partials(const WsLayout &L, int64_t nparts, const float *scales, int64_t T, int64_t D,
                                  int64_t nq, MetricTotals *totals, cudaStream_t s) {
    totals->sums = L.sums;
    totals->maxes = L.maxes;
    (void)launch_pdl(reduce_partials_kernel, dim3(1), dim3(1024), 0, s, L.partials, nparts, scales, D, (double)T * (double)D,
                                              (double)nq * (double)T, L.sums, L.maxes, totals->fused_out);
    return check_launch("metrics_reduce");
}

kvq_status launch_metrics_partials(const float *K, const float *K_hat, int64_t T, int64_t D, const float *Q,
                                   int64_t nq, const float *scales, void *ws, size_t ws_bytes,
                                   MetricTotals *totals, cudaStream_t s) {
    if (ws_bytes < metrics_workspace_size(T, D, nq))
        return fail(KVQ_ERR_INVALID_VALUE, "error_metrics: workspace too small");
    const WsLayout L = ws_layout(ws, T, D);
    int64_t nparts;
    if (!force_simt() && tc_eligible(K, K_hat, T, D, nq)) {
        int grid = 0;
        if (kvq_status st = launch_attn_tc(0, K, K_hat, T, D, Q, nq, L.qsplit, L.partials, &grid, nullptr, s, nullptr, nullptr,
                                                nullptr, nullptr, L.split);
            st != KVQ_OK)
            return st;
        nparts = grid;
    } else {
        nparts = num_tiles(T);
        attn_tile_kernel<0><<<(unsigned)nparts, 256, 0, s>>>(K, K_hat, Q, T, D, nq, L.partials, nullptr);
        if (kvq_status st = check_launch("metrics_tiles"); st != KVQ_OK) return st;
    }
    return reduce_partials(L, nparts, scales, T, D, nq, totals, s);
}

// kvq_step on an L2-resident K: a1 + a2 fused into the tensor-core roundtrip (one cooperative launch after the
// Q split), so the column-max pass, the scale finalize and the column-record prep are not separate kernels and
// the roundtrip re-reads K from L2.
size_t roundtrip_fused_a1_workspace_size(int64_t T, int64_t D, int64_t nq) {
    return metrics_workspace_size(T, D, nq) + 256 + al256((size_t)kSplitMaxCtas * (size_t)D * 4);
}

bool roundtrip_fused_a1_eligible(const float *K, const int8_t *Kq, const float *K_hat, int64_t T, int64_t D,
                                 int64_t nq, kvq_comm_t comm) {
    if (comm || force_simt() || !tc_roundtrip_eligible(K, Kq, K_hat, T, D, nq)) return false;
    const char *e = std::getenv("KVQ_STEP_FUSED");  // tests / experiments: 0 = never, 1 = whenever eligible
    if (e) return e[0] == '1';
    return T * D * 4 <= device_info().l2_bytes / 2;  // K stays in L2 between the column-max phase and the pass
}

kvq_status launch_roundtrip_fused_a1(const float *K, int64_t T, int64_t D, float *scales_out, int8_t *Kq,
                                     float *K_hat, const float *Q, int64_t nq, void *ws, size_t ws_bytes,
                                     MetricTotals *totals, cudaStream_t s) {
    if (ws_bytes < roundtrip_fused_a1_workspace_size(T, D, nq))
        return fail(KVQ_ERR_INVALID_VALUE, "kvq_step: workspace too small");
    const WsLayout L = ws_layout(ws, T, D);
    const uintptr_t pm = (reinterpret_cast<uintptr_t>(ws) + metrics_workspace_size(T, D, nq) + 255) & ~(uintptr_t)255;
    int grid = 0;
    totals->sums = L.sums;
    totals->maxes = L.maxes;
    bool reduced = false;  // whole tiles: the pass's last CTA reduces the partials itself
    if (kvq_status st = launch_attn_tc(2, K, nullptr, T, D, Q, nq, L.qsplit, L.partials, &grid, nullptr, s,
                                       scales_out, L.colq, Kq, K_hat, L.split, scales_out,
                                       reinterpret_cast<void *>(pm), totals, L.ticket, &reduced);
        st != KVQ_OK)
        return st;
    if (reduced) return KVQ_OK;
    return reduce_partials(L, grid, scales_out, T, D, nq, totals, s);
}

kvq_status launch_roundtrip_partials(const float *K, const float *scales, int64_t T, int64_t D, int8_t *Kq,
                                     float *K_hat, const float *Q, int64_t nq, void *ws, size_t ws_bytes,
                                     MetricTotals *totals, cudaStream_t s) {
    if (ws_bytes < metrics_workspace_size(T, D, nq))
        return fail(KVQ_ERR_INVALID_VALUE, "roundtrip: workspace too small");
    if (!force_simt() && tc_roundtrip_eligible(K, Kq, K_hat, T, D, nq)) {
        const WsLayout L = ws_layout(ws, T, D);
        int grid = 0;
        totals->sums = L.sums;
        totals->maxes = L.maxes;
        bool reduced = false;  // whole tiles: the pass's last CTA reduces the partials itself
        if (kvq_status st = launch_attn_tc(2, K, nullptr, T, D, Q, nq, L.qsplit, L.partials, &grid, nullptr, s,
                                           scales, L.colq, Kq, K_hat, L.split, nullptr, nullptr, totals, L.ticket,
                                           &reduced);
            st != KVQ_OK)
            return st;
        if (reduced) return KVQ_OK;
        return reduce_partials(L, grid, scales, T, D, nq, totals, s);
    }
    // not eligible for the single pass: fused quantize+dequantize, then the metrics pass
    if (kvq_status st = launch_quantize(K, scales, T, D, Kq, K_hat, s); st != KVQ_OK) return st;
    return launch_metrics_partials(K, K_hat, T, D, Q, nq, scales, ws, ws_bytes, totals, s);
}

kvq_status launch_metrics_finalize(const MetricTotals &t, kvq_metrics *out_dev, cudaStream_t s) {
    (void)launch_pdl(metrics_finalize_kernel, dim3(1), dim3(1), 0, s, (const double *)t.sums,
                     (const uint64_t *)t.maxes, out_dev);
    return check_launch("metrics_finalize");
}

size_t attention_scores_workspace_size(int64_t D, int64_t nq) {
    (void)nq;
    return tc_qsplit_bytes(D) + 256;
}

kvq_status launch_attention_scores(const float *Q, int64_t nq, const float *K, const float *K_hat, int64_t T,
                                   int64_t D, float *S, void *ws, size_t ws_bytes, cudaStream_t s) {
    const bool tc = ws && ws_bytes >= attention_scores_workspace_size(D, nq) && !force_simt() &&
                    tc_eligible(K, K_hat ? K_hat : K, T, D, nq);
    if (tc) {
        void *qsplit = reinterpret_cast<void *>((reinterpret_cast<uintptr_t>(ws) + 255) & ~(uintptr_t)255);
        return launch_attn_tc(1, K, K_hat, T, D, Q, nq, qsplit, nullptr, nullptr, S, s);
    }
    attn_tile_kernel<1><<<(unsigned)num_tiles(T), 256, 0, s>>>(K, K_hat, Q, T, D, nq, nullptr, S);
    return check_launch("attention_scores");
}

}  // namespace kvq
