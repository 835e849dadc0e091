/*
 * kvq_oracle.c — CPU ORACLE for per-channel symmetric INT8 KV-key quantization
 * (arxiv 2601.04719). TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load this file's library.  The product path
 * (paper_2601_04719_b200/, libkvq.so) never links, includes or calls it, and
 * this file includes nothing from the product.  The two share no code.
 *
 * Plain C99, single-threaded, no intrinsics.  Build flags (see oracle/__init__.py):
 *   gcc -O2 -std=c99 -fno-fast-math -ffp-contract=off -shared -fPIC
 * -ffp-contract=off keeps every product and sum separately rounded as written.
 *
 * Citations: P:<line> = /root/reference/PAPER.md line, S:<line> = SPEC.md line.
 * Readings of silent/ambiguous passages are numbered Q1..Q16 as in SURVEY.md §8(c)
 * and listed in DESIGN.md §3.
 *
 * Parity status of each function (what pins it, see tests/test_oracle_*.py):
 *   kvqo_splitmix64 / kvqo_uniform   pinned: SURVEY §8(d) test vector + numpy re-implementation
 *   kvqo_compute_scales              pinned: hand examples S:121-132, numpy abs-max, invariants
 *   kvqo_absmax_rows                 pinned: equals kvqo_compute_scales on every shape tested
 *   kvqo_quantize                    pinned: hand examples S:180-181, tie example, numpy rint,
 *                                    brute force over all codes for fixed s
 *   kvqo_dequantize                  pinned: S:189-191, numpy product
 *   kvqo_recon_errors                pinned: identity, 3-4-5, closed form L2
 *   kvqo_scores / kvqo_attention_abs_sum
 *                                    pinned: [[1]] vs [[0.9]] -> 0.1, identity,
 *                                    numpy float64 matmul, closed form sqrt(2/pi) s sqrt(D/36)
 *   kvqo_e4m3_encode / _decode, kvqo_*_e4m3 (NEXT-1 FP8 variant)
 *                                    pinned: hand-worked E4M3 codes incl. ties and saturation,
 *                                    torch float8_e4m3fn on all 256 codes and exhaustively over
 *                                    every fp32 in [2^-12, 448), numpy abs-max / 448
 *   kvqo_scales_from_absmax_q, kvqo_quantize_q, kvqo_pack_codes / kvqo_unpack_codes
 *   (NEXT-3 INT4 / INT2)             pinned: hand-worked codes and packed bytes, numpy
 *                                    rint(fp32(K/s)) clip, exact-rational brute force, pack /
 *                                    unpack round trip vs numpy bit arithmetic, error bound s/2,
 *                                    qmax = 127 reduces to kvqo_quantize
 *   No function is "parity unpinned".
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>

/* ------------------------------------------------------------------------ */
/* Input generator; independent of the method's arithmetic.    */
/* ------------------------------------------------------------------------ */

/* splitmix64 keyed by (seed, global element index i), SURVEY §8(d). */
uint64_t kvqo_splitmix64(uint64_t seed, uint64_t i)
{
    uint64_t z = seed + (i + 1u) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* Uniform on the exact lattice k * 2^-23, k in [-2^23, 2^23): "values in
 * [-1, 1]", reading Q12. */
float kvqo_uniform(uint64_t seed, uint64_t i)
{
    int32_t k = (int32_t)(kvqo_splitmix64(seed, i) >> 40) - (int32_t)(1 << 23);
    return (float)k * 0x1p-23f; /* exact: |k| < 2^24 */
}

/* Fill rows [row0, row0+rows) of a T x D matrix (row-major, global index
 * t*D + d), so a shard generated alone equals the same rows of the full matrix.
 * dist 0: uniform lattice.
 * dist 1: outlier channels: column d scaled by 2^(e_d), e_d = (splitmix64(seed ^
 *         0xC0FFEE, d) mod 9) - 4 (motivates per-channel scales).
 * dist 2: on-grid: x = c * s_d with s_d = j_d * 2^-24, j_d odd < 2^17, code c
 *         uniform in [-127, 127] and row 0 forced to +-127.
 */
void kvqo_fill(float *out, int64_t row0, int64_t rows, int64_t D, uint64_t seed, int dist)
{
    for (int64_t r = 0; r < rows; r++) {
        int64_t t = row0 + r;
        for (int64_t d = 0; d < D; d++) {
            uint64_t gi = (uint64_t)t * (uint64_t)D + (uint64_t)d;
            float v;
            if (dist == 1) {
                int e = (int)(kvqo_splitmix64(seed ^ 0xC0FFEEull, (uint64_t)d) % 9u) - 4;
                v = ldexpf(kvqo_uniform(seed, gi), e);
            } else if (dist == 2) {
                uint64_t j = ((kvqo_splitmix64(seed ^ 0x5CA1Eull, (uint64_t)d) >> 47) | 1u);
                float s = (float)j * 0x1p-24f;
                int c;
                if (t == 0)
                    c = (kvqo_splitmix64(seed ^ 0x516Eull, (uint64_t)d) & 1u) ? 127 : -127;
                else
                    c = (int)(kvqo_splitmix64(seed, gi) % 255u) - 127;
                v = (float)c * s;
            } else {
                v = kvqo_uniform(seed, gi);
            }
            out[r * D + d] = v;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* The method.                                                                */
/* ------------------------------------------------------------------------ */

/* Alg. 1 "Compute Scales" = Listing 2, Eq. 6:
 *   for d: max_abs = 0; for t: if |K[t,d]| > max_abs then max_abs = |K[t,d]|;
 *          scales[d] = max_abs / 127          (fp32 division, reading Q3)      */
void kvqo_compute_scales(const float *K, int64_t T, int64_t D, float *scales)
{
    for (int64_t d = 0; d < D; d++) {
        float max_abs = 0.0f;
        for (int64_t t = 0; t < T; t++) {
            float val = fabsf(K[t * D + d]);
            if (val > max_abs)
                max_abs = val;
        }
        scales[d] = max_abs / 127.0f;
    }
}

/* The inner loop of Alg. 1 over a block of rows, carrying max_abs[d] across
 * calls, so a matrix too large for host RAM can be streamed in row blocks.
 * The max of Eq. 6 is over the set {|K[t,d]| : t}; it does not depend on the
 * order in which t is visited, so visiting rows block by block computes the
 * same max_abs as Alg. 1.  Caller zero-fills max_abs before the first block
 * and finishes with kvqo_scales_from_absmax. */
void kvqo_absmax_rows(const float *K, int64_t rows, int64_t D, float *max_abs)
{
    for (int64_t t = 0; t < rows; t++)
        for (int64_t d = 0; d < D; d++) {
            float val = fabsf(K[t * D + d]);
            if (val > max_abs[d])
                max_abs[d] = val;
        }
}

/* Alg. 1 line "scales[d] <- max_abs / 127". */
void kvqo_scales_from_absmax(const float *max_abs, int64_t D, float *scales)
{
    for (int64_t d = 0; d < D; d++)
        scales[d] = max_abs[d] / 127.0f;
}

/* Eq. 7 = Listing 3:
 *   q = round(K[t,d] / s_d), clamped to [-127, 127].
 * Readings: Q1 round = round-half-even (rintf under FE_TONEAREST, as the GPU
 * listings' __float2int_rn at P:272); Q2 the quotient is the fp32 IEEE quotient
 * rounded to fp32 before rounding to an integer; Q4 symmetric clamp;
 * Q5 s_d == 0 gives q = 0.  The clamp is applied to the rounded float before
 * the int conversion (same result as Listing 3 for every finite quotient,
 * and avoids converting out-of-range floats). */
void kvqo_quantize(const float *K, const float *scales, int64_t T, int64_t D, int8_t *Kq)
{
    for (int64_t t = 0; t < T; t++) {
        for (int64_t d = 0; d < D; d++) {
            float s = scales[d];
            int q;
            if (s == 0.0f) {
                q = 0;
            } else {
                float val = K[t * D + d];
                float v = val / s;
                float r = rintf(v);
                if (r > 127.0f)
                    r = 127.0f;
                if (r < -127.0f)
                    r = -127.0f;
                q = (int)r;
            }
            Kq[t * D + d] = (int8_t)q;
        }
    }
}

/* Eq. 8 = Listing 4: K_hat[t,d] = (float)q * s_d. */
void kvqo_dequantize(const int8_t *Kq, const float *scales, int64_t T, int64_t D, float *K_hat)
{
    for (int64_t t = 0; t < T; t++)
        for (int64_t d = 0; d < D; d++) {
            int8_t q = Kq[t * D + d];
            K_hat[t * D + d] = (float)q * scales[d];
        }
}

/* Reconstruction errors (reading Q9):
 *   sum_sq  += sum_i ((double)A_i - (double)B_i)^2   (L2 = sqrt(sum_sq))
 *   max_abs  = max(max_abs, |(double)A_i - (double)B_i|)
 * Accumulated sequentially in double; callers chain blocks through the
 * in/out arguments. */
void kvqo_recon_errors(const float *A, const float *B, int64_t n, double *sum_sq, double *max_abs)
{
    double ss = *sum_sq, mx = *max_abs;
    for (int64_t i = 0; i < n; i++) {
        double e = (double)A[i] - (double)B[i];
        ss += e * e;
        double ae = fabs(e);
        if (ae > mx)
            mx = ae;
    }
    *sum_sq = ss;
    *max_abs = mx;
}

/* Raw dot-product scores S[i][t] = sum_d Q[i][d] * K[t][d] in double
 * ("attention dot products"; reading Q10: no 1/sqrt(d_k), no softmax). */
void kvqo_scores(const float *Q, int64_t nq, const float *K, int64_t T, int64_t D, double *S)
{
    for (int64_t i = 0; i < nq; i++)
        for (int64_t t = 0; t < T; t++) {
            double acc = 0.0;
            for (int64_t d = 0; d < D; d++)
                acc += (double)Q[i * D + d] * (double)K[t * D + d];
            S[i * T + t] = acc;
        }
}

/* Attention-score error (readings Q10, Q11):
 *   returns sum_{i<nq, t<T} |S[i][t] - S'[i][t]|, S from K, S' from K_hat,
 * each dot product accumulated in double.  mean = return / (nq * T). */
double kvqo_attention_abs_sum(const float *Q, int64_t nq, const float *K, const float *K_hat,
                              int64_t T, int64_t D)
{
    double total = 0.0;
    for (int64_t i = 0; i < nq; i++)
        for (int64_t t = 0; t < T; t++) {
            double s = 0.0, sh = 0.0;
            for (int64_t d = 0; d < D; d++) {
                s += (double)Q[i * D + d] * (double)K[t * D + d];
                sh += (double)Q[i * D + d] * (double)K_hat[t * D + d];
            }
            total += fabs(s - sh);
        }
    return total;
}

/* Theoretical max error max_d s_d / 2 (Eq. 9). */
double kvqo_theoretical_max(const float *scales, int64_t D)
{
    double m = 0.0;
    for (int64_t d = 0; d < D; d++)
        if ((double)scales[d] / 2.0 > m)
            m = (double)scales[d] / 2.0;
    return m;
}

/* ------------------------------------------------------------------------ */
/* NEXT-1 (paper future work "FP8"): per-channel FP8   */
/* E4M3 variant.  Reading Q17: s_d = max_t |K[t,d]| / 448    */
/* (448 = largest finite E4M3), code = E4M3 round-to-nearest-even of the     */
/* fp32 IEEE quotient with saturation to +-448 (OCP "satfinite"), s_d == 0   */
/* gives code 0 (+0), K_hat = decode(code) * s_d in fp32.                   */
/* E4M3 (OCP FP8 "e4m3fn"): sign, 4 exponent bits (bias 7), 3 mantissa bits, */
/* no infinities, S.1111.111 = NaN; normal (1 + M/8) 2^(E-7), subnormal      */
/* (M/8) 2^-6.                                                               */
/* ------------------------------------------------------------------------ */

float kvqo_e4m3_decode(uint8_t c)
{
    int sgn = c >> 7, E = (c >> 3) & 15, M = c & 7;
    float v;
    if (E == 15 && M == 7)
        return NAN;
    if (E == 0)
        v = ldexpf((float)M / 8.0f, -6);
    else
        v = ldexpf(1.0f + (float)M / 8.0f, E - 7);
    return sgn ? -v : v;
}

uint8_t kvqo_e4m3_encode(float v)
{
    uint8_t sgn = signbit(v) ? 0x80 : 0x00;
    float a = fabsf(v);
    if (isnan(v))
        return 0x7F;
    if (a >= 448.0f) /* every value >= 448 rounds to 448 or beyond it: saturate */
        return sgn | 0x7E;
    if (a == 0.0f)
        return sgn;
    int e;
    frexpf(a, &e); /* a = m 2^e, m in [0.5, 1): floor(log2 a) = e - 1 */
    int E = e - 1;
    if (E < -6)
        E = -6; /* subnormals share the quantum of the 2^-6 binade */
    float quantum = ldexpf(1.0f, E - 3);
    float r = rintf(a / quantum); /* exact scaling by a power of two; half-even */
    float val = r * quantum;
    if (val == 0.0f)
        return sgn;
    if (val < 0x1p-6f) /* subnormal: M = val / 2^-9 in 1..7 */
        return sgn | (uint8_t)(val / 0x1p-9f);
    frexpf(val, &e);
    E = e - 1;
    int M = (int)(val / ldexpf(1.0f, E - 3)) - 8;
    return sgn | (uint8_t)(((E + 7) << 3) | M);
}

/* scales for E4M3: s_d = max_abs / 448 (fp32 division) */
void kvqo_scales_from_absmax_e4m3(const float *max_abs, int64_t D, float *scales)
{
    for (int64_t d = 0; d < D; d++)
        scales[d] = max_abs[d] / 448.0f;
}

void kvqo_quantize_e4m3(const float *K, const float *scales, int64_t T, int64_t D, uint8_t *Kq)
{
    for (int64_t t = 0; t < T; t++)
        for (int64_t d = 0; d < D; d++) {
            float s = scales[d];
            Kq[t * D + d] = (s == 0.0f) ? 0 : kvqo_e4m3_encode(K[t * D + d] / s);
        }
}

void kvqo_dequantize_e4m3(const uint8_t *Kq, const float *scales, int64_t T, int64_t D, float *K_hat)
{
    for (int64_t t = 0; t < T; t++)
        for (int64_t d = 0; d < D; d++)
            K_hat[t * D + d] = kvqo_e4m3_decode(Kq[t * D + d]) * scales[d];
}

/* ------------------------------------------------------------------------ */
/* NEXT-3: INT4 / INT2 per-channel variant (future work P:562; reading Q19).  */
/* The same method with a smaller symmetric code range [-qmax, qmax]:         */
/* qmax = 7 (4-bit) or 1 (2-bit); everything else as Eq. 6-8.                */
/* ------------------------------------------------------------------------ */

/* Alg. 1's last line with the divisor qmax: s_d = max_abs / qmax (fp32 division). */
void kvqo_scales_from_absmax_q(const float *max_abs, int64_t D, int qmax, float *scales)
{
    for (int64_t d = 0; d < D; d++)
        scales[d] = max_abs[d] / (float)qmax;
}

/* Eq. 7 with the clamp at +-qmax: q = clamp(rint(fl32(K/s)), -qmax, qmax), 0 where s == 0. */
void kvqo_quantize_q(const float *K, const float *scales, int64_t T, int64_t D, int qmax, int8_t *q)
{
    for (int64_t t = 0; t < T; t++) {
        for (int64_t d = 0; d < D; d++) {
            float s = scales[d];
            int c;
            if (s == 0.0f) {
                c = 0;
            } else {
                float v = K[t * D + d] / s;
                float r = rintf(v);
                if (r > (float)qmax)
                    r = (float)qmax;
                if (r < -(float)qmax)
                    r = -(float)qmax;
                c = (int)r;
            }
            q[t * D + d] = (int8_t)c;
        }
    }
}

/* Storage (reading Q19): each row packed on its own into ceil(D * bits / 8)
 * bytes; column d's code, in `bits`-bit two's complement, occupies bits
 * [bits * (d % per), bits * (d % per) + bits) of byte d / per, per = 8 / bits
 * (low bits first: column 2j in the low nibble for INT4); unused bits are 0. */
void kvqo_pack_codes(const int8_t *q, int64_t T, int64_t D, int bits, uint8_t *out)
{
    int per = 8 / bits;
    int64_t rb = (D + per - 1) / per;
    unsigned mask = (1u << bits) - 1u;
    for (int64_t t = 0; t < T; t++) {
        for (int64_t j = 0; j < rb; j++)
            out[t * rb + j] = 0;
        for (int64_t d = 0; d < D; d++) {
            unsigned field = ((unsigned)(int)q[t * D + d]) & mask;
            out[t * rb + d / per] |= (uint8_t)(field << (bits * (int)(d % per)));
        }
    }
}

void kvqo_unpack_codes(const uint8_t *in, int64_t T, int64_t D, int bits, int8_t *q)
{
    int per = 8 / bits;
    int64_t rb = (D + per - 1) / per;
    unsigned mask = (1u << bits) - 1u;
    for (int64_t t = 0; t < T; t++)
        for (int64_t d = 0; d < D; d++) {
            unsigned field = ((unsigned)in[t * rb + d / per] >> (bits * (int)(d % per))) & mask;
            int c = (field & (1u << (bits - 1))) ? (int)field - (1 << bits) : (int)field;
            q[t * D + d] = (int8_t)c;
        }
}
