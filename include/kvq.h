/*
 * kvq.h — C ABI of libkvq.so: per-channel symmetric INT8 quantization of an
 * FP32 KV-cache key matrix on NVIDIA B200 (sm_100a), after arxiv 2601.04719.
 *
 * Citations: P:<line> = PAPER.md, S:<line> = SPEC.md (read-only reference),
 * readings Q1..Q16 = DESIGN.md §3 (= SURVEY.md §8(c)).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Matrices are dense row-major [T][D]: K and K_hat are float32,
 *    Kq is int8; element (t, d) lives at index t*D + d.  T is tokens, D is the
 *    head dimension, one scale per column d.
 *  - Pointers are CUDA device pointers on the current device unless marked
 *    [host].  The caller owns every buffer; the library never allocates or
 *    frees caller memory.  Any alignment is accepted: 16-byte aligned bases
 *    with D % 4 == 0 take the 128-bit vector path, everything else an in-kernel
 *    scalar path with bit-identical results.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Every call is asynchronous on `stream` unless documented otherwise.
 *  - Argument errors are detected synchronously, return KVQ_ERR_INVALID_VALUE
 *    and touch no output.  Launch failures return KVQ_ERR_CUDA; NCCL failures
 *    KVQ_ERR_NCCL.  Device faults surface at the caller's next synchronization.
 *    kvq_last_error() gives a thread-local message for the last failure.
 *  - Input must be finite (reading Q7).  A column containing Inf/NaN
 *    yields an Inf/NaN scale (visible without a sync); its codes are unspecified.
 *  - Results are deterministic: codes, scales and K_hat are bit-identical run
 *    to run, across launch geometries and across 1..N token-sharded ranks.
 *  - There is no CPU fallback.  On a device other than sm_100 every compute
 *    entry point returns KVQ_ERR_UNSUPPORTED.
 */
#ifndef KVQ_H
#define KVQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVQ_ABI_VERSION 1

typedef enum {
    KVQ_OK = 0,
    KVQ_ERR_INVALID_VALUE = 1, /* NULL pointer, T < 1, D < 1, T*D > 2^62, nq < 0, aliasing, short workspace */
    KVQ_ERR_CUDA = 2,          /* CUDA runtime / launch error */
    KVQ_ERR_NCCL = 3,          /* NCCL error, or NCCL not loadable */
    KVQ_ERR_UNSUPPORTED = 4    /* current device is not sm_100 */
} kvq_status;

/* Code formats.  KVQ_FMT_INT8 is the paper's method; KVQ_FMT_E4M3 the FP8 variant
 * of its future work (reading Q17); KVQ_FMT_INT4 /
 * KVQ_FMT_INT2 the packed low-bit variants (NEXT-3; reading Q19). */
typedef enum { KVQ_FMT_INT8 = 0, KVQ_FMT_E4M3 = 1, KVQ_FMT_INT4 = 2, KVQ_FMT_INT2 = 3 } kvq_format;

/* Opaque multi-GPU communicator (wraps an ncclComm_t, or a kvq_peer_t via
 * kvq_comm_from_peer; NULL = single GPU).  Every rank must issue a communicator's
 * calls in the same order, and their exchanges must execute in that order: use one
 * stream per communicator (a second concurrent stream needs its own communicator). */
typedef struct kvq_comm_s *kvq_comm_t;

/* Opaque peer-memory exchange (library-owned device buffer shared over CUDA IPC). */
typedef struct kvq_peer_s *kvq_peer_t;

/* Result of the paper's fidelity checks. */
typedef struct {
    double l2;              /* sqrt(sum (K - K_hat)^2), unnormalised Frobenius norm (reading Q9) */
    double max_abs;         /* max |K - K_hat| */
    double attn_mean_abs;   /* mean_{i<nq,t<T} |Q_i.K_t - Q_i.K_hat_t|, raw dot products (Q10/Q11); 0 if nq == 0 */
    double theoretical_max; /* max_d s_d / 2 (Eq. 9); 0 if scales == NULL */
    double sum_sq;          /* sum (K - K_hat)^2 (l2^2, kept for combination across calls) */
    double attn_abs_sum;    /* sum_{i,t} |Q_i.K_t - Q_i.K_hat_t| */
    int64_t n_elems;        /* T*D over all ranks */
    int64_t n_scores;       /* nq*T over all ranks */
} kvq_metrics;

/* ---------------------------------------------------------------- utilities */
int kvq_abi_version(void);
const char *kvq_status_string(kvq_status s);
/* Thread-local detail for the last non-OK status returned on this thread. */
const char *kvq_last_error(void);
/* KVQ_OK iff the current CUDA device is sm_100 (B200) and a kernel image loads. */
kvq_status kvq_device_check(void);

/* ---------------------------------------------------------------- multi-GPU */
/* [host] out: 128 bytes (an ncclUniqueId).  Call on one rank, broadcast the bytes. */
kvq_status kvq_comm_unique_id(void *out_id128);
/* Collective over `nranks` processes (one GPU each, current device).  id: [host] 128 B. */
kvq_status kvq_comm_init(kvq_comm_t *out, const void *id128, int nranks, int rank);
kvq_status kvq_comm_destroy(kvq_comm_t comm);

/* ---------------------------------------------------------------- the hot path */
/* a1+a2(+a7): per-channel scales, Alg. 1, Eq. 6:
 *   scales[d] = (max_t |K[t,d]|) / 127.0f       (fp32 IEEE division, reading Q3)
 * K: [T][D] float32 in.  scales: [D] float32 out (also used as uint32 scratch
 * while the max is formed; must not alias K).
 * comm != NULL: K is this rank's token shard (rows of the global matrix); the
 * column max is all-reduced (MAX) over ranks before the division, so scales
 * come out global and identical on all ranks.  Must then be called by every
 * rank of `comm` in the same order (NCCL rule). */
kvq_status kvq_compute_scales(const float *K, int64_t T, int64_t D, float *scales,
                              kvq_comm_t comm, void *stream);

/* Same as kvq_compute_scales with the divisor of `fmt`: 127 (KVQ_FMT_INT8),
 * 448 (KVQ_FMT_E4M3, the largest finite E4M3 value), 7 (KVQ_FMT_INT4) or 1
 * (KVQ_FMT_INT2).  Unknown fmt: KVQ_ERR_INVALID_VALUE. */
kvq_status kvq_compute_scales_fmt(const float *K, int64_t T, int64_t D, float *scales, int fmt,
                                  kvq_comm_t comm, void *stream);

/* a3: Eq. 7 / Listing 3:
 *   Kq[t,d] = clamp(round_half_even(fl32(K[t,d] / scales[d])), -127, 127),
 *   and 0 where scales[d] == 0                   (readings Q1, Q2, Q4, Q5)
 * K: [T][D] float32 in; scales: [D] in; Kq: [T][D] int8 out (may not alias K). */
kvq_status kvq_quantize(const float *K, const float *scales, int64_t T, int64_t D,
                        int8_t *Kq, void *stream);

/* a4: Eq. 8 / Listing 4:
 *   K_hat[t,d] = (float)Kq[t,d] * scales[d]      (one fp32 multiply; never -0)
 * Kq: [T][D] int8 in; scales: [D] in; K_hat: [T][D] float32 out (may not alias Kq). */
kvq_status kvq_dequantize(const int8_t *Kq, const float *scales, int64_t T, int64_t D,
                          float *K_hat, void *stream);

/* FP8 E4M3 variant of a3 (+a4) (P:570 future work; reading Q17):
 *   Kq8[t,d] = E4M3_RN_satfinite(fl32(K[t,d] / scales[d]))  (0x00 where scales[d] == 0)
 *   K_hat[t,d] = decode(Kq8[t,d]) * scales[d]               (if K_hat != NULL)
 * Codes are OCP E4M3 ("e4m3fn") bytes; scales from kvq_compute_scales_fmt(KVQ_FMT_E4M3).
 * Bit-identical to the oracle's kvqo_quantize_e4m3 / kvqo_dequantize_e4m3. */
kvq_status kvq_quantize_e4m3(const float *K, const float *scales, int64_t T, int64_t D,
                             uint8_t *Kq8, float *K_hat, void *stream);
kvq_status kvq_dequantize_e4m3(const uint8_t *Kq8, const float *scales, int64_t T, int64_t D,
                               float *K_hat, void *stream);

/* INT4 / INT2 packed variant of a3 (+a4) (P:562 future work; SURVEY §8(f) NEXT-3;
 * reading Q19), bits = 4 (qmax 7) or 2 (qmax 1):
 *   q[t,d]     = clamp(round_half_even(fl32(K[t,d] / scales[d])), -qmax, qmax), 0 where scales[d] == 0
 *   K_hat[t,d] = q[t,d] * scales[d]                          (if K_hat != NULL; one fp32 multiply)
 * Kp: [T][kvq_packed_row_bytes(D, bits)] bytes out; each row packed on its own,
 * column d's code in bits-bit two's complement at bits [bits*(d % p), +bits) of
 * byte d / p, p = 8 / bits (low bits first); unused bits are 0.  Scales from
 * kvq_compute_scales_fmt(KVQ_FMT_INT4 / KVQ_FMT_INT2).  Bit-identical to the
 * oracle's kvqo_quantize_q + kvqo_pack_codes / kvqo_unpack_codes + Eq. 8.
 * bits not in {4, 2}, NULL or aliasing buffers: KVQ_ERR_INVALID_VALUE. */
int64_t kvq_packed_row_bytes(int64_t D, int bits); /* ceil(D * bits / 8); -1 for bad arguments */
kvq_status kvq_quantize_packed(const float *K, const float *scales, int64_t T, int64_t D, int bits,
                               uint8_t *Kp, float *K_hat, void *stream);
kvq_status kvq_dequantize_packed(const uint8_t *Kp, const float *scales, int64_t T, int64_t D, int bits,
                                 float *K_hat, void *stream);

/* NEXT-4 (P:564 dynamic quantization, P:570 persistent kernels;
 * reading Q20): append n_new tokens to a growing key cache with dynamic
 * per-channel scales, keeping streaming == batch BIT FOR BIT:
 *   after the call, scales == kvq_compute_scales(K[0:T_new]) and
 *   Kq[0:T_new] (and K_hat[0:T_new]) == kvq_quantize(_dequantize)(K[0:T_new], scales),
 *   T_new = T_old + n_new.
 * K:      [T_new][D] fp32 [device], the retained full-precision cache; rows
 *         [T_old, T_new) hold the new tokens (written by the caller).  Read only.
 * absmax: [D] uint32 [device] running column abs-max (IEEE bits of |x|), and
 * scales: [D] fp32 [device] running scales: both zero-filled by the caller
 *         before the first append, then owned by this call.
 * Kq:     [T_new][D] int8 [device]; K_hat: [T_new][D] fp32 [device] or NULL.
 * Codes of old rows are rewritten only in columns whose scale changed
 * ("re-quantize when a scale grows").  n_new may be 0 and T_old may be 0 (an
 * empty append still takes part in the all-reduce when comm != NULL).
 * comm != NULL: token-sharded cache; every rank calls with its own shard and
 * its own n_new (0 allowed); the running max is all-reduced (MAX) each call,
 * so scales stay global.  Decode-sized appends (n_new <= 256, comm == NULL)
 * run as ONE cooperative launch.  workspace: kvq_append_workspace_size(D)
 * bytes [device], not shared by concurrent calls. */
size_t kvq_append_workspace_size(int64_t D);
kvq_status kvq_append(const float *K, int64_t T_old, int64_t n_new, int64_t D, uint32_t *absmax,
                      float *scales, int8_t *Kq, float *K_hat, void *workspace, size_t workspace_bytes,
                      kvq_comm_t comm, void *stream);

/* a3+a4 fused in one pass over K (9 B/elem instead of 10): writes both Kq and
 * K_hat, bit-identical to kvq_quantize followed by kvq_dequantize. */
kvq_status kvq_quantize_dequantize(const float *K, const float *scales, int64_t T, int64_t D,
                                   int8_t *Kq, float *K_hat, void *stream);

/* a1+a2+a3+a4 in ONE cooperative launch (single GPU, D % 4 == 0, aligned): the
 * column max pass pulls K into the 126 MB L2, a grid-wide barrier, then each
 * thread forms its own columns' scales and quantizes + dequantizes the same
 * elements from L2.  Results are bit-identical to
 * kvq_compute_scales + kvq_quantize_dequantize, which is what runs otherwise
 * (K larger than 3/4 of the L2 or D < 256 -- where the two streaming passes are
 * faster, measured crossover in profiles/r01/sweep_c5.md --, comm != NULL,
 * unaligned, or no co-resident grid).  workspace: device scratch
 * of kvq_quantize_fused_workspace_size(T, D) bytes.  *single_pass_out [host,
 * nullable] reports which path ran. */
size_t kvq_quantize_fused_workspace_size(int64_t T, int64_t D);
kvq_status kvq_quantize_fused(const float *K, int64_t T, int64_t D, float *scales, int8_t *Kq,
                              float *K_hat, void *workspace, size_t workspace_bytes, kvq_comm_t comm,
                              int *single_pass_out, void *stream);

/* a1 + a7 + a2 in ONE kernel over peer memory, without NCCL (
 * the all-reduce MAX of the column maxima).  Setup, once per rank:
 *   kvq_peer_init(&p, nranks, rank, D, handle)  allocates this rank's exchange buffer
 *     (library-owned, 2 x nranks x D u32 + flags) and writes its CUDA IPC handle
 *     (kvq_peer_handle_bytes() bytes, [host]) for the caller to all-gather;
 *   kvq_peer_open(p, handles)  maps every other rank's buffer ([host] nranks handles
 *     in rank order; needs peer access between the GPUs, or one GPU).
 * kvq_compute_scales_peer: K is this rank's token shard [T][D] (T may be 0), D % 4 == 0,
 * K and scales 16-byte aligned.  Each CTA reduces its share into `scales` (abs bits);
 * the last CTA pushes the local D-vector into every rank's buffer (P2P stores), raises
 * an epoch flag in each (system-scope release), waits for all ranks' flags, takes the
 * max over ranks and writes scales[d] = fl32(m_d / 127) (Eq. 5/6).  Scales are
 * global and bit-identical to kvq_compute_scales over the whole matrix.  Every rank
 * must make the same sequence of calls, and the ranks' kernels must be able to run
 * concurrently (the last CTA waits for its peers).  kvq_peer_destroy: after all ranks'
 * last call has completed (collective, like ncclCommDestroy).
 * Argument checks are rank-local: a call that returns an error on one rank enqueues nothing
 * there, so its peers' exchange kernels wait for a flag that never comes.  The wait is
 * bounded (KVQ_PEER_TIMEOUT_S, default 120 s): the waiting kernel traps and the peers'
 * next synchronization reports a launch failure instead of hanging the GPU.  Validate
 * arguments identically on every rank. */
size_t kvq_peer_handle_bytes(void);
/* A communicator whose collectives (the a7 MAX in kvq_compute_scales[_fmt] -- fused into
 * the column-max kernel when D % 4 == 0 and K / scales are 16-byte aligned --, the metric
 * SUM/MAX of kvq_error_metrics / kvq_roundtrip, the running-max MAX of kvq_append and the
 * host pipeline) all go through the peer's memory instead of NCCL.  The fp64 metric sums
 * are added in rank order (deterministic, identical on every rank).  `p` stays owned by
 * the caller and must outlive the communicator (kvq_comm_destroy first). */
kvq_status kvq_comm_from_peer(kvq_comm_t *out, kvq_peer_t p);
kvq_status kvq_peer_init(kvq_peer_t *out, int nranks, int rank, int64_t D, void *handle_out);
kvq_status kvq_peer_open(kvq_peer_t p, const void *handles);
kvq_status kvq_peer_destroy(kvq_peer_t p);

/* NVLS (NVLink SHARP) for the peer's a7 exchange (multi-GPU is the
 * paper's future work).  With NVLS active, the last CTA of the fused column-max kernel
 * stores the rank's D column maxima into its OWN copy of a multicast-bound buffer and, after
 * the epoch flags, reads m_d with one multimem.ld_reduce.max.u32 per column: the NVSwitch reads
 * every rank's copy and returns the max (order-free, so scales stay bit-identical).  Setup is
 * collective and staged so that no rank blocks on a rank that failed:
 *   rank 0:     kvq_peer_nvls_create(p, blob)  multicast object for nranks devices; [host] blob
 *               of kvq_peer_nvls_handle_bytes() bytes to broadcast (a fabric handle, or the tag
 *               of a unix socket on which rank 0's process hands out a POSIX fd for it)
 *   every rank: kvq_peer_nvls_join(p, blob)    import + cuMulticastAddDevice
 *   (all joined) kvq_peer_nvls_map(p)          own memory, bind, multicast + unicast mappings
 *   (all mapped) kvq_peer_nvls_enable(p, 1)    or (p, 0) on every rank to release and keep P2P
 * Errors: KVQ_ERR_UNSUPPORTED when the device, driver or handle exchange cannot do multicast
 * (resources released; the P2P exchange keeps working).  p must be open (kvq_peer_open). */
size_t kvq_peer_nvls_handle_bytes(void);
kvq_status kvq_peer_nvls_create(kvq_peer_t p, void *blob_out);
kvq_status kvq_peer_nvls_join(kvq_peer_t p, const void *blob);
kvq_status kvq_peer_nvls_map(kvq_peer_t p);
kvq_status kvq_peer_nvls_enable(kvq_peer_t p, int on);
int kvq_peer_nvls_active(kvq_peer_t p);
kvq_status kvq_compute_scales_peer(const float *K, int64_t T, int64_t D, float *scales, kvq_peer_t p, void *stream);

/* a5+a6: the paper's fidelity checks.
 * K, K_hat: [T][D] float32 in.  Q: [nq][D] float32 queries or NULL (nq == 0).
 * scales: [D] or NULL (only used for theoretical_max).  workspace: device
 * scratch of at least kvq_error_metrics_workspace_size(T, D, nq) bytes.
 * out_dev: DEVICE pointer to one kvq_metrics, written asynchronously.
 * comm != NULL: K/K_hat are this rank's token shard; sums and maxima are
 * all-reduced so every rank receives the global metrics.
 * a6 runs on the tcgen05 tensor cores (3xTF32) when 1 <= nq <= 64, D % 4 == 0
 * and K/K_hat are 16-byte aligned, else on the CUDA cores.  Sums are carried in
 * fp64 and reduced with a fixed tree (deterministic run to run).  The workspace
 * holds per-CTA partials, the split Q tiles, per-K-block column records and, for
 * tiles the tensor-core pass splits between CTAs, up to 160 x 128 KB of fp64
 * partial scores (the size function accounts for all of it). */
size_t kvq_error_metrics_workspace_size(int64_t T, int64_t D, int64_t nq);
kvq_status kvq_error_metrics_async(const float *K, const float *K_hat, int64_t T, int64_t D,
                                   const float *Q, int64_t nq, const float *scales,
                                   void *workspace, size_t workspace_bytes, kvq_comm_t comm,
                                   kvq_metrics *out_dev, void *stream);
/* Same, but out_host is [host] memory and the call synchronizes `stream`. */
kvq_status kvq_error_metrics(const float *K, const float *K_hat, int64_t T, int64_t D,
                             const float *Q, int64_t nq, const float *scales,
                             void *workspace, size_t workspace_bytes, kvq_comm_t comm,
                             kvq_metrics *out_host, void *stream);

/* a3+a4+a5+a6 in ONE pass over K (the B200 single-pass path; 9 B/elem of HBM
 * traffic instead of 5 + 5 + 8): quantize (Eq. 7) and dequantize (Eq. 8) each
 * K tile while it is on chip, write Kq and K_hat, and contract E = K - K_hat
 * with Q on the tensor cores for the fidelity checks.  Kq and K_hat are
 * bit-identical to kvq_quantize + kvq_dequantize; the metrics equal
 * kvq_error_metrics on (K, K_hat) within 1e-5 (fp64 sums in another order).
 * Single pass when 1 <= nq <= 64, D % 16 == 0 and K, Kq, K_hat are 16-byte
 * aligned; otherwise the same results from the separate kernels.
 * scales: [D] from kvq_compute_scales.  out_dev: DEVICE kvq_metrics, async.
 * workspace: kvq_roundtrip_workspace_size(T, D, nq) bytes [device], not shared by
 * calls in flight at the same time (it holds the per-CTA partials and the ticket
 * with which the pass's last CTA reduces them when its tiles are whole).  comm as
 * in kvq_error_metrics_async. */
size_t kvq_roundtrip_workspace_size(int64_t T, int64_t D, int64_t nq);
kvq_status kvq_roundtrip(const float *K, const float *scales, int64_t T, int64_t D, int8_t *Kq,
                         float *K_hat, const float *Q, int64_t nq, void *workspace,
                         size_t workspace_bytes, kvq_comm_t comm, kvq_metrics *out_dev, void *stream);

/* The whole hot path on device buffers in one call (a1 column abs-max over K, a7
 * the all-reduce MAX of the column maxima over the token shards when comm != NULL,
 * a2 scales, then a3-a6 as kvq_roundtrip): kvq_compute_scales + kvq_roundtrip.
 * Alg. 1, Eq. 7/8, fidelity checks P:20-24.
 * K: [T][D] (this rank's token shard when comm != NULL); Q: [nq][D] or NULL;
 * outputs scales [D] (global, identical on every rank), Kq [T][D], K_hat [T][D] and
 * out_dev (DEVICE kvq_metrics), all caller-owned, written asynchronously on `stream`.
 * Small single-GPU problems (comm == NULL, D <= 256, nq <= 64, T*D <= 2^20, e.g.
 * BASELINE C1) run as ONE cooperative launch (grid-wide barriers between the
 * paper's steps; a6 with exact fp64 products and sums on the CUDA cores); everything else
 * runs the streaming column max and the single-pass tensor-core roundtrip.  Both
 * give bit-identical scales, codes and K_hat; metrics within rounding of fp64 sums.
 * workspace: kvq_step_workspace_size(T, D, nq) bytes, any alignment; not shared by
 * concurrent calls.  Errors as kvq_roundtrip (KVQ_ERR_INVALID_VALUE on NULL/alias/
 * small workspace before anything is enqueued). */
size_t kvq_step_workspace_size(int64_t T, int64_t D, int64_t nq);
kvq_status kvq_step(const float *K, int64_t T, int64_t D, const float *Q, int64_t nq, float *scales,
                    int8_t *Kq, float *K_hat, void *workspace, size_t workspace_bytes, kvq_comm_t comm,
                    kvq_metrics *out_dev, void *stream);

/* Raw attention scores for parity checks of a6 (reading Q10):
 *   K_hat == NULL:  S[i][t] = sum_d Q[i][d] * K[t][d]
 *   K_hat != NULL:  S[i][t] = sum_d Q[i][d] * (K[t][d] - K_hat[t][d])   (= S - S')
 * Q: [nq][D], K/K_hat: [T][D], S: [nq][T] float32 out.
 * With a workspace of kvq_attention_scores_workspace_size(D, nq) bytes, nq <= 64,
 * D % 4 == 0 and 16-byte aligned K/K_hat the contraction runs on the tcgen05
 * tensor cores (3xTF32 split, fp32 accumulation in TMEM); otherwise (or with
 * workspace == NULL) on the CUDA cores (fp32 products, 32-term fp32 partial
 * sums carried in fp64).  Both are GPU paths. */
size_t kvq_attention_scores_workspace_size(int64_t D, int64_t nq);
kvq_status kvq_attention_scores(const float *Q, int64_t nq, const float *K, const float *K_hat,
                                int64_t T, int64_t D, float *S, void *workspace, size_t workspace_bytes,
                                void *stream);

/* NEXT-2: raw attention scores computed directly from the
 * compressed cache, without materialising K_hat ("dequantize them back ...
 * when needed for attention"; P:24 raw dot products, reading Q10):
 *   S[i][t] = sum_d Q[i][d] * (Kq[t][d] * scales[d])
 * Q: [nq][D] fp32, Kq: [T][D] int8 codes, scales: [D], S: [nq][T] fp32 out.
 * With a workspace of kvq_scores_from_codes_workspace_size(D, nq) bytes,
 * 1 <= nq <= 64, D % 16 == 0, D <= 264208 and 16-byte aligned Kq this runs on
 * the tcgen05 INTEGER tensor cores (kind::i8, CTA pairs): the codes are the A
 * operand as stored; W = fl32(Q*s) is written as 4 signed base-2^7 digits per
 * query row under a per-row exponent (truncation |e| < 2^-27 max_d |W[i][d]|),
 * s8 x s8 products accumulate EXACTLY in s32 and are recombined in fp64, reading
 * 1 byte per key element.  Rows of Q with a non-finite W take an fp64
 * per-element path (inf/nan propagate as in the definition).  Otherwise a
 * CUDA-core kernel (fp64 sums).  Within 1e-5 of sum_d Q[i][d]*K_hat[t][d]
 * relative to sum_d |Q[i][d]*K_hat[t][d]|; exact (before the final fp32
 * rounding) when every W[i][d] is a multiple of 2^(E_i - 28).  Enqueues 3
 * kernels on `stream`; the workspace must not be shared by concurrent calls. */
size_t kvq_scores_from_codes_workspace_size(int64_t D, int64_t nq);
kvq_status kvq_scores_from_codes(const float *Q, int64_t nq, const int8_t *Kq, const float *scales,
                                 int64_t T, int64_t D, float *S, void *workspace, size_t workspace_bytes,
                                 void *stream);

/* ---------------------------------------------------------------- host-buffer pipeline */
/* The whole path from HOST memory (the end-to-end call a user makes):
 * H2D of K (row blocks, overlapped with the column-max kernel), scales,
 * fused quantize+dequantize, metrics, then D2H of scales, codes and metrics
 * (and K_hat if K_hat_host != NULL).  Synchronizes `stream`.
 * K_host [T][D], Q_host [nq][D] or NULL, scales_host [D], Kq_host [T][D]:
 * [host] buffers, pinned (cudaHostAlloc / torch pin_memory) for full speed.
 * dev_workspace: device scratch of kvq_roundtrip_host_workspace_size() bytes. */
size_t kvq_roundtrip_host_workspace_size(int64_t T, int64_t D, int64_t nq);
kvq_status kvq_roundtrip_host(const float *K_host, int64_t T, int64_t D,
                              const float *Q_host, int64_t nq,
                              float *scales_host, int8_t *Kq_host, float *K_hat_host,
                              kvq_metrics *metrics_host,
                              void *dev_workspace, size_t workspace_bytes,
                              kvq_comm_t comm, void *stream);
/* Same, asynchronous: returns after enqueueing; all host outputs (including
 * metrics_host) must be pinned and are valid once `stream` has been
 * synchronized.  The copies run on library-owned H2D / D2H streams, so calls on
 * two caller streams with two workspaces pipeline: call i's device-to-host
 * results travel while call i+1's inputs arrive. */
kvq_status kvq_roundtrip_host_async(const float *K_host, int64_t T, int64_t D,
                                    const float *Q_host, int64_t nq,
                                    float *scales_host, int8_t *Kq_host, float *K_hat_host,
                                    kvq_metrics *metrics_host,
                                    void *dev_workspace, size_t workspace_bytes,
                                    kvq_comm_t comm, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* KVQ_H */
