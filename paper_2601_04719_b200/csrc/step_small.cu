// step_small.cu — the whole hot path (a1 column abs-max, a2 scales, a3 quantize, a4 dequantize,
// a5 L2 / max-abs, a6 attention-score error) in ONE cooperative launch for small problems
// (a persistent kernel for the launch-bound C1 step; PAPER.md:570 future work
// "persistent kernels").  The paper's steps run in its order (Alg. 1 then Eq. 7, Eq. 8, the checks of
// P:20-24), separated by grid-wide barriers instead of kernel boundaries:
//
//   phase A  each CTA: column max |K| over its row slab (abs bits, Eq. 6) -> its row of partial maxima;
//            Q staged in shared memory (fp64)
//   -- grid sync --
//   phase B  every CTA: m_d = max over the partial rows (order-free), s_d = fl32(m_d / 127) (Eq. 5/6,
//            IEEE division), RN(1/s_d) for the quantizer; CTA 0 stores the scales
//   phase C  each CTA, row chunks of its slab: q = clamp(rint(fl32(x/s))) (Eq. 7, provably exact fast
//            path + IEEE repair, device_common.cuh), x_hat = q s (Eq. 8), E = x - x_hat (exact);
//            sum E^2, max |E| (a5) and Delta[t][i] = sum_d Q[i][d] E[t][d] with exact fp64 products
//            and fp64 sums on the CUDA cores (a6; Q staged in shared memory)
//   -- grid sync --
//   phase D  CTA 0: the per-CTA partials in fixed order -> kvq_metrics (same fields and arithmetic as
//            reduce_partials_kernel)
//
// Deterministic (fixed partition and reduction order).  Codes, scales and K_hat are bit-identical to the
// streaming kernels; the metrics agree with them and with the oracle within rounding of the fp64 sums.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "device_common.cuh"
#include "kvq_internal.h"

namespace cg = cooperative_groups;

namespace kvq {

namespace {
constexpr int SS_THREADS = 256;
constexpr int SS_MAXD = 256;  // head dims the single launch takes (Q and a row chunk of E in shared memory)
constexpr int SS_MAXQ = 64;
constexpr int SS_ROWS = 8;          // rows of E per chunk
constexpr int64_t SS_MAXN = 1 << 20;  // elements: beyond this the streaming / tensor-core passes win

struct SmallLayout {
    uint32_t *pmax;  // [G][D] per-CTA column maxima (abs bits): no zeroing needed between calls
    Partial *part;   // [G]
};
size_t small_ws_bytes(int G, int64_t D) { return ((size_t)G * D * 4 + 255) / 256 * 256 + (size_t)G * sizeof(Partial); }
SmallLayout small_layout(void *ws, int G, int64_t D) {
    uint8_t *b = reinterpret_cast<uint8_t *>(ws);
    SmallLayout L;
    L.pmax = reinterpret_cast<uint32_t *>(b);
    L.part = reinterpret_cast<Partial *>(b + ((size_t)G * D * 4 + 255) / 256 * 256);
    return L;
}
// ~1024 elements per CTA (C1: 128 CTAs of 8 rows, one row chunk each), at most one wave
constexpr int64_t SS_ELEMS_PER_CTA = 1024;
int small_grid(int64_t T, int64_t D) {
    const int64_t g = std::max<int64_t>(1, std::min<int64_t>(T, (T * D) / SS_ELEMS_PER_CTA));
    return (int)std::min<int64_t>(device_info().num_sms, g);
}
}  // namespace

#ifdef KVQ_TRACE
__device__ unsigned long long g_step_trace[10];
#define SS_TR(k)                                                                                  \
    do {                                                                                          \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                                \
            unsigned long long t_;                                                                \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                \
            g_step_trace[k] = t_;                                                                 \
        }                                                                                         \
    } while (0)
#else
#define SS_TR(k) \
    do {         \
    } while (0)
#endif

__global__ void __launch_bounds__(SS_THREADS) step_small_kernel(const float *__restrict__ K, int64_t T, int D,
                                                                const float *__restrict__ Q, int nq,
                                                                float *__restrict__ scales, int8_t *__restrict__ Kq,
                                                                float *__restrict__ Kh, uint32_t *__restrict__ pmax,
                                                                Partial *__restrict__ part, kvq_metrics *out) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double smd[];
    const int QS = D + 1;                                // padded Q row stride: conflict-free column reads
    double *sd = smd;                                    // [4][SS_ROWS][SS_MAXQ] a6 partial sums per D-quarter
    double *sq = sd + 4 * SS_ROWS * SS_MAXQ;             // [nq][D + 1] Q in fp64 (exact), converted once
    double *se = sq + (size_t)SS_MAXQ * (SS_MAXD + 1);   // [D][SS_ROWS] E of the current row chunk, transposed
    float *ssc = reinterpret_cast<float *>(se + SS_ROWS * SS_MAXD);  // [D] s_d
    uint32_t *smax = reinterpret_cast<uint32_t *>(ssc + SS_MAXD);      // [D]
    __shared__ double red[3][SS_THREADS / 32];

    const int tid = threadIdx.x, b = blockIdx.x, G = gridDim.x;
    const int r0 = (int)(T * b / G), r1 = (int)(T * (b + 1) / G);  // this CTA's rows (T*D <= 2^20)
    const int nrows = r1 - r0;
    // column-owning threads: thread = (row phase ph, column col); rpp row phases cover the block
    const int rpp = SS_THREADS / D, col = tid % D, ph = tid / D;
    const bool active = ph < rpp;

    SS_TR(0);
    // ---- phase A: a1 over the slab (Alg. 1, Eq. 6): u32 max of |x| bits, order-free -> this CTA's row of
    // partial maxima.  Q is staged meanwhile (independent of a1).  Loads go out in batches of 16 per thread
    // (registers first, then shared memory) so their latencies overlap.
    for (int d = tid; d < D; d += SS_THREADS) smax[d] = 0u;
    __syncthreads();
    if (active) {
        constexpr int U = 16;
        uint32_t m = 0u;
        for (int r = ph; r < nrows; r += U * rpp) {
            float v[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int rr = r + u * rpp;
                v[u] = rr < nrows ? __ldg(K + (int64_t)(r0 + rr) * D + col) : 0.0f;
            }
#pragma unroll
            for (int u = 0; u < U; u++) m = max(m, absbits(v[u]));
        }
        constexpr int UQ = 32;  // C1: all of this thread's Q elements in flight at once
        for (int i = ph; i < nq; i += UQ * rpp) {
            float v[UQ];
#pragma unroll
            for (int u = 0; u < UQ; u++) {
                const int ii = i + u * rpp;
                v[u] = ii < nq ? __ldg(Q + (int64_t)ii * D + col) : 0.0f;
            }
#pragma unroll
            for (int u = 0; u < UQ; u++)
                if (i + u * rpp < nq) sq[(i + u * rpp) * QS + col] = (double)v[u];
        }
        if (m) atomicMax(&smax[col], m);
    }
    __syncthreads();
    for (int d = tid; d < D; d += SS_THREADS) pmax[(int64_t)b * D + d] = smax[d];
    SS_TR(1);
    grid.sync();
    SS_TR(2);

    // ---- phase B: a2 (Eq. 5/6): every CTA folds the G partial rows (batched loads) and forms
    // s_d = fl32(m_d / 127) with the IEEE division; CTA 0 publishes the scales
    for (int d = tid; d < D; d += SS_THREADS) smax[d] = 0u;
    __syncthreads();
    if (active) {
        constexpr int U = 64;  // C1: every partial row of this thread's column in flight at once
        uint32_t m = 0u;
        for (int c = ph; c < G; c += U * rpp) {
            uint32_t v[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int cc = c + u * rpp;
                v[u] = cc < G ? __ldcg(pmax + (int64_t)cc * D + col) : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; u++) m = max(m, v[u]);
        }
        if (m) atomicMax(&smax[col], m);
    }
    __syncthreads();
    for (int d = tid; d < D; d += SS_THREADS) {
        const float s = __fdiv_rn(__uint_as_float(smax[d]), 127.0f);
        ssc[d] = s;
        if (b == 0) scales[d] = s;
    }
    __syncthreads();

    SS_TR(3);
    // ---- phase C: a3 + a4 + a5 + a6, SS_ROWS rows at a time
    double ss = 0.0, attn = 0.0;
    float mx = 0.0f;
    const float s_col = active ? ssc[col] : 0.0f;
    const ColQ cq = make_colq(s_col);  // RN(1/s) once per thread (column-owning)
    // a6 mapping: thread = (query qi, quarter qd of the D columns); rows of the chunk in registers
    const int qi = tid % SS_MAXQ, qd = tid / SS_MAXQ;
    const int d0 = qd * D / 4, d1 = (qd + 1) * D / 4;
    for (int c0 = 0; c0 < nrows; c0 += SS_ROWS) {
        const int nr = min(SS_ROWS, nrows - c0);
        if (active) {
            for (int rr = ph; rr < nr; rr += rpp) {
                const int64_t idx = (int64_t)(r0 + c0 + rr) * D + col;
                const float x = __ldg(K + idx);
                int code;
                float xh;
                bool danger = false;
                const float v = quant_fast(x, cq, danger);
                if (danger || cq.exact) {  // near-tie quotient or subnormal scale: the IEEE quotient (Eq. 7)
                    code = quant_exact(x, s_col);
                    xh = __fmul_rn((float)code, s_col);
                } else {
                    code = (int)(int8_t)code_byte(v);
                    xh = __fmul_rn(__fsub_rn(v, kMagic), s_col);
                }
                Kq[idx] = (int8_t)code;
                Kh[idx] = xh;
                const float e = __fsub_rn(x, xh);  // exact
                ss += (double)e * (double)e;       // exact product in fp64
                mx = fmaxf(mx, fabsf(e));
                se[col * SS_ROWS + rr] = (double)e;
            }
        }
        __syncthreads();
        // a6: Delta[t][i] = sum_d Q[i][d] E[t][d] with exact fp64 products and fp64 sums (the oracle's
        // arithmetic class; also for subnormal E); a warp = 32 queries (one Q element each, padded rows:
        // conflict-free) x the chunk's rows (E transposed: one d's rows are two 16-byte broadcast loads per
        // pair of rows); the four D-quarters are added in fixed order below
        if (qi < nq) {
            double acc[SS_ROWS];
#pragma unroll
            for (int r = 0; r < SS_ROWS; r++) acc[r] = 0.0;
            const double *qr = sq + qi * QS;
            for (int d = d0; d < d1; d++) {
                const double qv = qr[d];
                const double2 *ed = reinterpret_cast<const double2 *>(se + d * SS_ROWS);
#pragma unroll
                for (int r = 0; r < SS_ROWS; r += 2) {
                    const double2 e2 = ed[r / 2];
                    acc[r] = fma(qv, e2.x, acc[r]);
                    acc[r + 1] = fma(qv, e2.y, acc[r + 1]);
                }
            }
#pragma unroll
            for (int r = 0; r < SS_ROWS; r++) sd[(qd * SS_ROWS + r) * SS_MAXQ + qi] = acc[r];
        }
        __syncthreads();
        for (int pi = tid; pi < nr * SS_MAXQ; pi += SS_THREADS) {
            const int i = pi % SS_MAXQ, r = pi / SS_MAXQ;
            if (i < nq)
                attn += fabs((sd[(0 * SS_ROWS + r) * SS_MAXQ + i] + sd[(1 * SS_ROWS + r) * SS_MAXQ + i]) +
                             (sd[(2 * SS_ROWS + r) * SS_MAXQ + i] + sd[(3 * SS_ROWS + r) * SS_MAXQ + i]));
        }
        __syncthreads();
    }
    // per-CTA partials (fixed order: warp butterfly, then warp 0)
    double mxd = (double)mx;
    for (int o = 16; o > 0; o >>= 1) {
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
        attn += __shfl_xor_sync(0xffffffffu, attn, o);
        mxd = fmax(mxd, __shfl_xor_sync(0xffffffffu, mxd, o));
    }
    if ((tid & 31) == 0) {
        red[0][tid >> 5] = ss;
        red[1][tid >> 5] = attn;
        red[2][tid >> 5] = mxd;
    }
    __syncthreads();
    if (tid == 0) {
        Partial p{0.0, 0.0, 0.0, 0.0};
        for (int w = 0; w < SS_THREADS / 32; w++) {
            p.sum_sq += red[0][w];
            p.attn_abs += red[1][w];
            p.max_abs = fmax(p.max_abs, red[2][w]);
        }
        part[b] = p;
    }
    SS_TR(4);
    grid.sync();
    SS_TR(5);

    // ---- phase D: CTA 0 reduces the partials in fixed order and writes the metrics
    if (b != 0) return;
    double s0 = 0.0, a0 = 0.0, m0 = 0.0, th = 0.0;
    for (int c = tid; c < G; c += SS_THREADS) {
        const double *pc = reinterpret_cast<const double *>(part + c);  // written by other CTAs: L2 loads
        s0 += __ldcg(pc + 0);
        a0 += __ldcg(pc + 1);
        m0 = fmax(m0, __ldcg(pc + 2));
    }
    for (int d = tid; d < D; d += SS_THREADS) th = fmax(th, (double)ssc[d] / 2.0);
    for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        a0 += __shfl_xor_sync(0xffffffffu, a0, o);
        m0 = fmax(m0, __shfl_xor_sync(0xffffffffu, m0, o));
        th = fmax(th, __shfl_xor_sync(0xffffffffu, th, o));
    }
    __shared__ double red2[4][SS_THREADS / 32];
    if ((tid & 31) == 0) {
        red2[0][tid >> 5] = s0;
        red2[1][tid >> 5] = a0;
        red2[2][tid >> 5] = m0;
        red2[3][tid >> 5] = th;
    }
    __syncthreads();
    if (tid == 0) {
        double S = 0.0, A = 0.0, M = 0.0, TH = 0.0;
        for (int w = 0; w < SS_THREADS / 32; w++) {
            S += red2[0][w];
            A += red2[1][w];
            M = fmax(M, red2[2][w]);
            TH = fmax(TH, red2[3][w]);
        }
        const double n_elems = (double)T * (double)D, n_scores = (double)nq * (double)T;
        kvq_metrics m;
        m.sum_sq = S;
        m.attn_abs_sum = A;
        m.n_elems = (int64_t)n_elems;
        m.n_scores = (int64_t)n_scores;
        m.l2 = sqrt(S);
        m.max_abs = fmax(M, 0.0);
        m.theoretical_max = TH;
        m.attn_mean_abs = n_scores > 0.0 ? A / n_scores : 0.0;
        *out = m;
        SS_TR(6);
    }
}

bool step_small_eligible(int64_t T, int64_t D, int64_t nq, kvq_comm_t comm) {
    if (comm || D > SS_MAXD || nq > SS_MAXQ || T * D > SS_MAXN) return false;
    const char *e = std::getenv("KVQ_STEP_SMALL");  // experiments / tests: 0 = never, 1 = whenever eligible
    return !(e && e[0] == '0');
}

size_t step_small_workspace_size(int64_t T, int64_t D) {
    if (D > SS_MAXD || T * D > SS_MAXN) return 0;
    return small_ws_bytes(small_grid(T, D), D) + 256;
}

kvq_status launch_step_small(const float *K, int64_t T, int64_t D, const float *Q, int64_t nq, float *scales,
                             int8_t *Kq, float *K_hat, void *ws, size_t ws_bytes, kvq_metrics *out_dev,
                             cudaStream_t s) {
    const int G = small_grid(T, D);
    uint8_t *w = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(ws) + 255) & ~(uintptr_t)255);
    if ((size_t)(w - reinterpret_cast<uint8_t *>(ws)) + small_ws_bytes(G, D) > ws_bytes)
        return fail(KVQ_ERR_INVALID_VALUE, "kvq_step: workspace too small");
    const SmallLayout L = small_layout(w, G, D);
    const size_t smem = ((size_t)4 * SS_ROWS * SS_MAXQ + (size_t)SS_MAXQ * (SS_MAXD + 1) + SS_ROWS * SS_MAXD) * 8 +
                        (size_t)2 * SS_MAXD * 4;
    ensure_max_smem<step_small_kernel>((int)smem);
    int Di = (int)D, nqi = (int)nq;
    const float *Qp = nq ? Q : nullptr;
    void *args[] = {(void *)&K, (void *)&T, (void *)&Di, (void *)&Qp, (void *)&nqi, (void *)&scales, (void *)&Kq,
                    (void *)&K_hat, (void *)&L.pmax, (void *)&L.part, (void *)&out_dev};
    (void)cudaLaunchCooperativeKernel((const void *)step_small_kernel, dim3(G), dim3(SS_THREADS), args, smem, s);
    return check_launch("step_small (cooperative)");
}

}  // namespace kvq

#ifdef KVQ_TRACE
extern "C" int kvq_debug_step_trace_read(void *host) {
    return (int)cudaMemcpyFromSymbol(host, kvq::g_step_trace, sizeof(kvq::g_step_trace));
}
#endif
