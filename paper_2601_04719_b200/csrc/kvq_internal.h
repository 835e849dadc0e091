// kvq_internal.h — internal (non-ABI) declarations shared by the libkvq.so
// translation units.  Nothing here is exported; the ABI is include/kvq.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <utility>

#include "../../include/kvq.h"

#include <nvtx3/nvToolsExt.h>

namespace kvq {

// NVTX range around every C-ABI call (header-only NVTX v3: a no-op unless a profiler injects itself), so
// nsys / ncu timelines show which ABI call enqueued which kernels.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};
#define KVQ_NVTX(name) ::kvq::NvtxRange kvq_nvtx_range_(name)

// Thread-local last-error message (kvq_last_error).
void set_error(const std::string &msg);
kvq_status fail(kvq_status st, const std::string &msg);
kvq_status check_launch(const char *what);
kvq_status device_ok();  // cached sm_100 check for the current device

struct DeviceInfo {
    int device;
    int num_sms;
    int cc_major, cc_minor;
    int64_t l2_bytes;
};
const DeviceInfo &device_info();

// Launch-geometry plan for the column-owning streaming kernels: G threads in
// total, G a multiple of `cols` (element groups per row) so that every thread
// owns fixed columns for the whole grid-stride loop (its scale and reciprocal
// are loaded once; SURVEY §7 hard part (i)).
struct StreamPlan {
    int64_t G;        // total active threads (multiple of cols)
    unsigned blocks;  // ceil(G / kThreads)
};
constexpr int kThreads = 256;
StreamPlan plan_stream(int64_t rows, int64_t cols, int threads_per_sm);

// ---- quantization kernels (quant_kernels.cu)
kvq_status launch_colmax(const float *K, int64_t T, int64_t D, uint32_t *mbits, cudaStream_t s);
kvq_status launch_finalize(uint32_t *mbits_to_scales, int64_t D, cudaStream_t s, float divisor = 127.0f);
// ---- FP8 E4M3 variant (fp8_kernels.cu)
kvq_status launch_quantize_e4m3(const float *K, const float *scales, int64_t T, int64_t D, uint8_t *Kq,
                                float *K_hat /* nullable */, cudaStream_t s);
kvq_status launch_dequantize_e4m3(const uint8_t *Kq, const float *scales, int64_t T, int64_t D, float *K_hat,
                                  cudaStream_t s);
// ---- streaming append with dynamic scales (append_kernels.cu, NEXT-4)
size_t append_workspace_size(int64_t D);
kvq_status launch_append(const float *K, int64_t T_old, int64_t n_new, int64_t D, uint32_t *absmax, float *scales,
                         int8_t *Kq, float *K_hat, void *ws, kvq_comm_t comm, cudaStream_t s);
// ---- INT4 / INT2 packed variant (lowbit_kernels.cu)
int64_t packed_row_bytes(int64_t D, int bits);
kvq_status launch_quantize_packed(const float *K, const float *scales, int64_t T, int64_t D, int bits, uint8_t *Kp,
                                  float *K_hat /* nullable */, cudaStream_t s);
kvq_status launch_dequantize_packed(const uint8_t *Kp, const float *scales, int64_t T, int64_t D, int bits,
                                    float *K_hat, cudaStream_t s);
kvq_status launch_quantize(const float *K, const float *scales, int64_t T, int64_t D, int8_t *Kq,
                           float *K_hat /* nullable: fused a3+a4 */, cudaStream_t s);
kvq_status launch_dequantize(const int8_t *Kq, const float *scales, int64_t T, int64_t D, float *K_hat,
                             cudaStream_t s);

size_t single_pass_workspace_size(int64_t D);
kvq_status launch_single_pass(const float *K, int64_t T, int64_t D, float *scales, int8_t *Kq, float *K_hat,
                              void *ws, cudaStream_t s);

// ---- metrics kernels (metrics_kernels.cu, attn_tc.cu)
// Writes per-rank totals {sum_sq, attn_abs_sum, n_elems, n_scores} (double[4]) and
// {max_abs_bits, theo_max_bits} (uint64[2]) into the workspace tail; returns
// pointers to them so the comm layer can all-reduce in place.
struct MetricTotals {
    double *sums;      // [4] device
    uint64_t *maxes;   // [2] device
    kvq_metrics *fused_out = nullptr;  // set by the caller when no exchange follows: the reduction kernel
                                       // then also writes the final struct (no metrics_finalize launch)
};
struct Partial {  // per-CTA partial sums of a5/a6
    double sum_sq, attn_abs, max_abs, pad;
};
bool tc_eligible(const float *K, const float *K_hat, int64_t T, int64_t D, int64_t nq);
size_t tc_qsplit_bytes(int64_t D);
// mode 0: write per-CTA Partials (grid returned in *grid_out); mode 1: write S [nq][T].
bool tc_roundtrip_eligible(const float *K, const int8_t *Kq, const float *K_hat, int64_t T, int64_t D, int64_t nq);
size_t tc_colq_bytes(int64_t D);
// mode 2: fused a3+a4+a5+a6 (needs scales, colq workspace, Kq/Kh outputs).
kvq_status launch_attn_tc(int mode, const float *K, const float *K_hat, int64_t T, int64_t D, const float *Q,
                          int64_t nq, void *ws_q, void *partials, int *grid_out, float *S, cudaStream_t s,
                          const float *scales = nullptr, void *ws_colq = nullptr, int8_t *Kq_out = nullptr,
                          float *Kh_out = nullptr, void *ws_split = nullptr, float *scales_out = nullptr,
                          void *ws_pmax = nullptr, const MetricTotals *fin = nullptr, unsigned *ticket = nullptr,
                          bool *reduced = nullptr);
// mode 2 with a1 + a2 fused in front (scales_out, ws_pmax set; cooperative launch): the kvq_step path for an
// L2-resident K (the pmax workspace holds kSplitMaxCtas x D u32, the largest grid).
kvq_status launch_roundtrip_fused_a1(const float *K, int64_t T, int64_t D, float *scales_out, int8_t *Kq,
                                     float *K_hat, const float *Q, int64_t nq, void *ws, size_t ws_bytes,
                                     MetricTotals *totals, cudaStream_t s);
size_t roundtrip_fused_a1_workspace_size(int64_t T, int64_t D, int64_t nq);
bool roundtrip_fused_a1_eligible(const float *K, const int8_t *Kq, const float *K_hat, int64_t T, int64_t D,
                                 int64_t nq, kvq_comm_t comm);
// modes 0/2: fp64 Delta slots for the pieces of a split tail (at most kSplitMaxPieces pieces, grid <= kSplitMaxCtas)
constexpr int kSplitMaxCtas = 160;
constexpr int kSplitMaxPieces = 640;
size_t tc_split_bytes(int64_t T, int64_t D);
struct TailPlan {
    int grid, whole, rt, pieces;
    bool split;
};
TailPlan tc_plan_tail(int ntiles, int ngrp, int nsm, int force);
// the partials array of the metric reductions: per-CTA partials + COMBINE_JQ per tail tile
inline int64_t metrics_partials_count(int64_t ntiles) {
    const int64_t a = kSplitMaxCtas + 4 * ntiles;
    return a > 1024 ? a : 1024;
}
// a3+a4+a5+a6 in one pass when eligible, else quantize_dequantize + metrics kernels.
kvq_status launch_roundtrip_partials(const float *K, const float *scales, int64_t T, int64_t D, int8_t *Kq,
                                     float *K_hat, const float *Q, int64_t nq, void *ws, size_t ws_bytes,
                                     MetricTotals *totals, cudaStream_t s);
bool force_simt();  // KVQ_FORCE_SIMT=1: use the CUDA-core attention kernel (tests compare the two)
size_t metrics_workspace_size(int64_t T, int64_t D, int64_t nq);
kvq_status launch_metrics_partials(const float *K, const float *K_hat, int64_t T, int64_t D, const float *Q,
                                   int64_t nq, const float *scales, void *ws, size_t ws_bytes,
                                   MetricTotals *totals, cudaStream_t s);
kvq_status launch_metrics_finalize(const MetricTotals &totals, kvq_metrics *out_dev, cudaStream_t s);
size_t attention_scores_workspace_size(int64_t D, int64_t nq);
kvq_status launch_attention_scores(const float *Q, int64_t nq, const float *K, const float *K_hat, int64_t T,
                                   int64_t D, float *S, void *ws, size_t ws_bytes, cudaStream_t s);

// ---- the whole step in one cooperative launch for small problems (step_small.cu, NEXT-4)
bool step_small_eligible(int64_t T, int64_t D, int64_t nq, kvq_comm_t comm);
size_t step_small_workspace_size(int64_t T, int64_t D);
kvq_status launch_step_small(const float *K, int64_t T, int64_t D, const float *Q, int64_t nq, float *scales,
                             int8_t *Kq, float *K_hat, void *ws, size_t ws_bytes, kvq_metrics *out_dev,
                             cudaStream_t s);

// ---- scores from codes (scores_codes.cu, NEXT-2)
size_t scores_codes_workspace_size(int64_t D);
kvq_status launch_scores_codes(const float *Q, int64_t nq, const int8_t *Kq, const float *scales, int64_t T,
                               int64_t D, float *S, void *ws, size_t ws_bytes, cudaStream_t s);

// ---- comm (comm.cpp)
// peer-memory exchanges (peer.cu); a kvq_comm_t made with kvq_comm_from_peer routes its collectives here
int peer_nranks(kvq_peer_t p);
int peer_rank(kvq_peer_t p);
bool peer_ready(kvq_peer_t p);
kvq_status peer_allreduce_max_u32(kvq_peer_t p, uint32_t *buf, size_t count, cudaStream_t s);
kvq_status peer_allreduce_metrics(kvq_peer_t p, double *sums, size_t nsum, uint64_t *maxes, size_t nmax,
                                  cudaStream_t s);
kvq_status peer_compute_scales(const float *K, int64_t T, int64_t D, float *scales, float divisor, kvq_peer_t p,
                               cudaStream_t s);
kvq_peer_t comm_peer(kvq_comm_t comm);  // the peer behind a peer-backed communicator, else nullptr
kvq_status comm_allreduce_max_u32(kvq_comm_t comm, uint32_t *buf, size_t count, cudaStream_t s);
kvq_status comm_allreduce_sum_f64(kvq_comm_t comm, double *buf, size_t count, cudaStream_t s);
kvq_status comm_allreduce_max_u64(kvq_comm_t comm, uint64_t *buf, size_t count, cudaStream_t s);
kvq_status comm_allreduce_metrics(kvq_comm_t comm, double *sums, size_t nsum, uint64_t *maxes, size_t nmax,
                                  cudaStream_t s);

// Programmatic dependent launch for the step's chained kernels (finalize, prep/qsplit, the tensor-core
// pass, split_combine, the partials reduction, metrics_finalize): the launch of kernel i+1 and its prologue
// overlap kernel i's tail; every such kernel executes griddepcontrol.wait (pdl_wait) before its first
// global-memory access, which returns once all prerequisite grids have completed and their writes are
// visible, so the stream order of memory effects is unchanged.  Each kernel triggers its dependents only
// after its own wait, so a grid never launches before its predecessor's predecessor has completed (no two
// tensor-core grids ever hold TMEM on one SM).  The column-max kernel does not trigger early: finalize
// blocks resident during its stream cost 5-7 us at the 4/8-rank shard sizes (profiles/r01/s4/pdl_ab.txt).
// KVQ_PDL=0 launches them plainly (A/B).
bool pdl_enabled();
template <typename... Exp, typename... Act>
cudaError_t launch_pdl(void (*kernel)(Exp...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Act &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Act>(args)...);
}

// The dynamic shared-memory opt-in of a kernel, once per device (cudaFuncSetAttribute acts on the current
// device, so a process driving several GPUs needs it on each).  One set of flags per kernel (K is the kernel).
constexpr int kMaxDevices = 64;
template <auto K>
inline void ensure_max_smem(int bytes) {
    static std::once_flag flags[kMaxDevices];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
        cudaGetLastError();
        (void)cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        return;
    }
    std::call_once(flags[dev], [&] { (void)cudaFuncSetAttribute(K, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes); });
}

}  // namespace kvq
