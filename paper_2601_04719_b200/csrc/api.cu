// api.cu — the extern "C" entry points of libkvq.so (include/kvq.h):
// argument validation, launch sequencing on the caller's stream, error mapping.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "kvq_internal.h"

namespace kvq {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

kvq_status fail(kvq_status st, const std::string &msg) {
    set_error(msg);
    return st;
}

bool pdl_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("KVQ_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

kvq_status check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(KVQ_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return KVQ_OK;
}

static kvq_status cuda_check(cudaError_t e, const char *what) {
    if (e != cudaSuccess) return fail(KVQ_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return KVQ_OK;
}

__global__ void probe_kernel() {}

namespace {
std::mutex g_mu;
int g_state[kMaxDevices];  // 0 unknown, 1 ok, 2 unsupported
DeviceInfo g_info[kMaxDevices];
cudaStream_t g_copy_stream[kMaxDevices][2];
}  // namespace

kvq_status device_ok() {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(KVQ_ERR_CUDA, std::string("no usable CUDA device: ") + cudaGetErrorString(e));
    }
    if (dev < 0 || dev >= kMaxDevices) return fail(KVQ_ERR_UNSUPPORTED, "device index out of range");
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_state[dev] == 0) {
        cudaDeviceProp p;
        if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) {
            cudaGetLastError();
            return fail(KVQ_ERR_CUDA, "cudaGetDeviceProperties failed");
        }
        g_info[dev] = DeviceInfo{dev, p.multiProcessorCount, p.major, p.minor, (int64_t)p.l2CacheSize};
        cudaFuncAttributes fa;
        bool image = cudaFuncGetAttributes(&fa, probe_kernel) == cudaSuccess;
        cudaGetLastError();
        g_state[dev] = (p.major == 10 && p.minor == 0 && image) ? 1 : 2;
    }
    if (g_state[dev] != 1)
        return fail(KVQ_ERR_UNSUPPORTED, "libkvq.so is built for sm_100a (B200) only; current device cc " +
                                             std::to_string(g_info[dev].cc_major) + "." +
                                             std::to_string(g_info[dev].cc_minor));
    return KVQ_OK;
}

const DeviceInfo &device_info() {
    int dev = 0;
    cudaGetDevice(&dev);
    return g_info[dev];
}

// Library-owned copy streams per device: 0 = host-to-device, 1 = device-to-host.
static cudaStream_t copy_stream(int which) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_copy_stream[dev][which]) cudaStreamCreateWithFlags(&g_copy_stream[dev][which], cudaStreamNonBlocking);
    return g_copy_stream[dev][which];
}

}  // namespace kvq

using namespace kvq;

// ------------------------------------------------------------------------------ validation helpers
static bool bad_dims(int64_t T, int64_t D) { return T < 1 || D < 1 || T > (int64_t(1) << 62) / D; }

static bool overlap(const void *a, size_t na, const void *b, size_t nb) {
    if (!a || !b) return false;
    uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return x < y + nb && y < x + na;
}

#define KVQ_REQUIRE(cond, msg) \
    do {                       \
        if (!(cond)) return fail(KVQ_ERR_INVALID_VALUE, msg); \
    } while (0)

#define KVQ_TRY(expr)                       \
    do {                                    \
        kvq_status _st = (expr);            \
        if (_st != KVQ_OK) return _st;      \
    } while (0)

// ------------------------------------------------------------------------------ utilities
extern "C" int kvq_abi_version(void) { return KVQ_ABI_VERSION; }

extern "C" const char *kvq_status_string(kvq_status s) {
    switch (s) {
        case KVQ_OK: return "KVQ_OK";
        case KVQ_ERR_INVALID_VALUE: return "KVQ_ERR_INVALID_VALUE";
        case KVQ_ERR_CUDA: return "KVQ_ERR_CUDA";
        case KVQ_ERR_NCCL: return "KVQ_ERR_NCCL";
        case KVQ_ERR_UNSUPPORTED: return "KVQ_ERR_UNSUPPORTED";
    }
    return "KVQ_ERR_UNKNOWN";
}

extern "C" const char *kvq_last_error(void) { return g_last_error.c_str(); }

extern "C" kvq_status kvq_device_check(void) {
    KVQ_NVTX("kvq_device_check");
    return device_ok();
}

// ------------------------------------------------------------------------------ a1 + a2 (+ a7)
extern "C" kvq_status kvq_compute_scales_fmt(const float *K, int64_t T, int64_t D, float *scales, int fmt,
                                             kvq_comm_t comm, void *stream) {
    KVQ_NVTX("kvq_compute_scales_fmt");
    KVQ_REQUIRE(K && scales, "kvq_compute_scales: NULL pointer");
    KVQ_REQUIRE(!bad_dims(T, D), "kvq_compute_scales: need T >= 1, D >= 1, T*D <= 2^62");
    KVQ_REQUIRE(fmt == KVQ_FMT_INT8 || fmt == KVQ_FMT_E4M3 || fmt == KVQ_FMT_INT4 || fmt == KVQ_FMT_INT2,
                "kvq_compute_scales: unknown format");
    KVQ_REQUIRE(!overlap(K, (size_t)(T * D) * 4, scales, (size_t)D * 4), "kvq_compute_scales: scales aliases K");
    KVQ_TRY(device_ok());
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t *bits = reinterpret_cast<uint32_t *>(scales);
    const float divisor = fmt == KVQ_FMT_E4M3 ? 448.0f : fmt == KVQ_FMT_INT4 ? 7.0f : fmt == KVQ_FMT_INT2 ? 1.0f : 127.0f;
    if (kvq_peer_t p = comm_peer(comm)) {
        // peer-backed communicator: column max + exchange + finalize in one kernel when aligned
        const kvq_status st = peer_compute_scales(K, T, D, scales, divisor, p, s);
        if (st != KVQ_ERR_UNSUPPORTED) return st;
    }
    KVQ_TRY(cuda_check(cudaMemsetAsync(bits, 0, (size_t)D * 4, s), "memset scales"));
    KVQ_TRY(launch_colmax(K, T, D, bits, s));
    if (comm) KVQ_TRY(comm_allreduce_max_u32(comm, bits, (size_t)D, s));
    return launch_finalize(bits, D, s, divisor);
}

extern "C" kvq_status kvq_compute_scales(const float *K, int64_t T, int64_t D, float *scales, kvq_comm_t comm,
                                         void *stream) {
    KVQ_NVTX("kvq_compute_scales");
    return kvq_compute_scales_fmt(K, T, D, scales, KVQ_FMT_INT8, comm, stream);
}

// ------------------------------------------------------------------------------ FP8 E4M3 variant (NEXT-1)
extern "C" kvq_status kvq_quantize_e4m3(const float *K, const float *scales, int64_t T, int64_t D, uint8_t *Kq8,
                                        float *K_hat, void *stream) {
    KVQ_NVTX("kvq_quantize_e4m3");
    KVQ_REQUIRE(K && scales && Kq8, "kvq_quantize_e4m3: NULL pointer");
    KVQ_REQUIRE(!bad_dims(T, D), "kvq_quantize_e4m3: need T >= 1, D >= 1, T*D <= 2^62");
    const size_t n = (size_t)(T * D);
    KVQ_REQUIRE(!overlap(K, n * 4, Kq8, n) && !overlap(scales, (size_t)D * 4, Kq8, n),
                "kvq_quantize_e4m3: Kq8 aliases an input");
    if (K_hat)
        KVQ_REQUIRE(!overlap(K_hat, n * 4, K, n * 4) && !overlap(K_hat, n * 4, Kq8, n) &&
                        !overlap(K_hat, n * 4, scales, (size_t)D * 4),
                    "kvq_quantize_e4m3: K_hat aliases an input");
    KVQ_TRY(device_ok());
    return launch_quantize_e4m3(K, scales, T, D, Kq8, K_hat, (cudaStream_t)stream);
}

extern "C" kvq_status kvq_dequantize_e4m3(const uint8_t *Kq8, const float *scales, int64_t T, int64_t D,
                                          float *K_hat, void *stream) {
    KVQ_NVTX("kvq_dequantize_e4m3");
    KVQ_REQUIRE(Kq8 && scales && K_hat, "kvq_dequantize_e4m3: NULL pointer");
    KVQ_REQUIRE(!bad_dims(T, D), "kvq_dequantize_e4m3: need T >= 1, D >= 1, T*D <= 2^62");
    const size_t n = (size_t)(T * D);
    KVQ_REQUIRE(!overlap(K_hat, n * 4, Kq8, n) && !overlap(K_hat, n * 4, scales, (size_t)D * 4),
                "kvq_dequantize_e4m3: K_hat aliases an input");
    KVQ_TRY(device_ok());
    return launch_dequantize_e4m3(Kq8, scales, T, D, K_hat, (cudaStream_t)stream);
}

// ------------------------------------------------------------------------------ streaming append (NEXT-4)
extern "C" size_t kvq_append_workspace_size(int64_t D) { return D < 1 ? 0 : append_workspace_size(D); }

extern "C" kvq_status kvq_append(const float *K, int64_t T_old, int64_t n_new, int64_t D, uint32_t *absmax,
                                 float *scales, int8_t *Kq, float *K_hat, void *workspace, size_t workspace_bytes,
                                 kvq_comm_t comm, void *stream) {
    KVQ_NVTX("kvq_append");
    KVQ_REQUIRE(K && absmax && scales && Kq && workspace, "kvq_append: NULL pointer");
    KVQ_REQUIRE(T_old >= 0 && n_new >= 0 && D >= 1, "kvq_append: need T_old >= 0, n_new >= 0, D >= 1");
    const int64_t T = T_old + n_new;
    KVQ_REQUIRE(T == 0 || !bad_dims(T, D), "kvq_append: need (T_old + n_new) * D <= 2^62");
    KVQ_REQUIRE(workspace_bytes >= append_workspace_size(D), "kvq_append: workspace too small");
    const size_t n = (size_t)(T * D), d4 = (size_t)D * 4;
    KVQ_REQUIRE(!overlap(K, n * 4, Kq, n) && !overlap(K, n * 4, absmax, d4) && !overlap(K, n * 4, scales, d4) &&
                    !overlap(absmax, d4, scales, d4) && !overlap(Kq, n, scales, d4) && !overlap(Kq, n, absmax, d4),
                "kvq_append: buffers alias");
    if (K_hat)
        KVQ_REQUIRE(!overlap(K_hat, n * 4, K, n * 4) && !overlap(K_hat, n * 4, Kq, n) &&
                        !overlap(K_hat, n * 4, scales, d4) && !overlap(K_hat, n * 4, absmax, d4) &&
                        !overlap(workspace, workspace_bytes, K_hat, n * 4),
                    "kvq_append: K_hat aliases an input");
    KVQ_REQUIRE(!overlap(workspace, workspace_bytes, K, n * 4) && !overlap(workspace, workspace_bytes, Kq, n) &&
                    !overlap(workspace, workspace_bytes, scales, d4) && !overlap(workspace, workspace_bytes, absmax, d4),
                "kvq_append: workspace aliases a buffer");
    KVQ_TRY(device_ok());
    return launch_append(K, T_old, n_new, D, absmax, scales, Kq, K_hat, workspace, comm, (cudaStream_t)stream);
}

// ------------------------------------------------------------------------------ INT4 / INT2 packed (NEXT-3)
extern "C" int64_t kvq_packed_row_bytes(int64_t D, int bits) {
    if (D < 1 || (bits != 4 && bits != 2)) return -1;
    return packed_row_bytes(D, bits);
}

extern "C" kvq_status kvq_quantize_packed(const float *K, const float *scales, int64_t T, int64_t D, int bits,
                                          uint8_t *Kp, float *K_hat, void *stream) {
    KVQ_NVTX("kvq_quantize_packed");
    KVQ_REQUIRE(K && scales && Kp, "kvq_quantize_packed: NULL pointer");
    KVQ_REQUIRE(bits == 4 || bits == 2, "kvq_quantize_packed: bits must be 4 or 2");
    KVQ_REQUIRE(!bad_dims(T, D), "kvq_quantize_packed: need T >= 1, D >= 1, T*D <= 2^62");
    const size_t n = (size_t)(T * D), np = (size_t)(T * packed_row_bytes(D, bits));
    KVQ_REQUIRE(!overlap(K, n * 4, Kp, np) && !overlap(scales, (size_t)D * 4, Kp, np),
                "kvq_quantize_packed: Kp aliases an input");
    if (K_hat)
        KVQ_REQUIRE(!overlap(K_hat, n * 4, K, n * 4) && !overlap(K_hat, n * 4, Kp, np) &&
                        !overlap(K_hat, n * 4, scales, (size_t)D * 4),
                    "kvq_quantize_packed: K_hat aliases an input");
    KVQ_TRY(device_ok());
    return launch_quantize_packed(K, scales, T, D, bits, Kp, K_hat, (cudaStream_t)stream);
}

extern "C" kvq_status kvq_dequantize_packed(const uint8_t *Kp, const float *scales, int64_t T, int64_t D, int bits,
                                            float *K_hat, void *stream) {
    KVQ_NVTX("kvq_dequantize_packed");
    KVQ_REQUIRE(Kp && scales && K_hat, "kvq_dequantize_packed: NULL pointer");
    KVQ_REQUIRE(bits == 4 || bits == 2, "kvq_dequantize_packed: bits must be 4 or 2");
    KVQ_REQUIRE(!bad_dims(T, D), "kvq_dequantize_packed: need T >= 1, D >= 1, T*D <= 2^62");
    const size_t n = (size_t)(T * D), np = (size_t)(T * packed_row_bytes(D, bits));
    KVQ_REQUIRE(!overlap(K_hat, n * 4, Kp, np) && !overlap(K_hat, n * 4, scales, (size_t)D * 4),
                "kvq_dequantize_packed: K_hat aliases an input");
    KVQ_TRY(device_ok());
    return launch_dequantize_packed(Kp, scales, T, D, bits, K_hat, (cudaStream_t)stream);
}

// ------------------------------------------------------------------------------ a3, a4
static kvq_status quant_common(const float *K, const float *scales, int64_t T, int64_t D, int8_t *Kq, float *K_hat,
                               void *stream, const char *name) {
    KVQ_REQUIRE(K && scales && Kq, std::string(name) + ": NULL pointer");
    KVQ_REQUIRE(!bad_dims(T, D), std::string(name) + ": need T >= 1, D >= 1, T*D <= 2^62");
    const size_t n = (size_t)(T * D);
    KVQ_REQUIRE(!overlap(K, n * 4, Kq, n), std::string(name) + ": Kq aliases K");
    KVQ_REQUIRE(!overlap(scales, (size_t)D * 4, Kq, n), std::string(name) + ": Kq aliases scales");
    if (K_hat) {
        KVQ_REQUIRE(!overlap(K_hat, n * 4, K, n * 4) && !overlap(K_hat, n * 4, Kq, n) &&
                        !overlap(K_hat, n * 4, scales, (size_t)D * 4),
                    std::string(name) + ": K_hat aliases an input");
    }
    KVQ_TRY(device_ok());
    return launch_quantize(K, scales, T, D, Kq, K_hat, (cudaStream_t)stream);
}

extern "C" kvq_status kvq_quantize(const float *K, const float *scales, int64_t T, int64_t D, int8_t *Kq,
                                   void *stream) {
    KVQ_NVTX("kvq_quantize");
    return quant_common(K, scales, T, D, Kq, nullptr, stream, "kvq_quantize");
}

extern "C" kvq_status kvq_quantize_dequantize(const float *K, const float *scales, int64_t T, int64_t D, int8_t *Kq,
                                              float *K_hat, void *stream) {
    KVQ_NVTX("kvq_quantize_dequantize");
    KVQ_REQUIRE(K_hat, "kvq_quantize_dequantize: NULL K_hat");
    return quant_common(K, scales, T, D, Kq, K_hat, stream, "kvq_quantize_dequantize");
}

extern "C" kvq_status kvq_dequantize(const int8_t *Kq, const float *scales, int64_t T, int64_t D, float *K_hat,
                                     void *stream) {
    KVQ_NVTX("kvq_dequantize");
    KVQ_REQUIRE(Kq && scales && K_hat, "kvq_dequantize: NULL pointer");
    KVQ_REQUIRE(!bad_dims(T, D), "kvq_dequantize: need T >= 1, D >= 1, T*D <= 2^62");
    const size_t n = (size_t)(T * D);
    KVQ_REQUIRE(!overlap(K_hat, n * 4, Kq, n) && !overlap(K_hat, n * 4, scales, (size_t)D * 4),
                "kvq_dequantize: K_hat aliases an input");
    KVQ_TRY(device_ok());
    return launch_dequantize(Kq, scales, T, D, K_hat, (cudaStream_t)stream);
}

// ------------------------------------------------------------------------------ a1..a4 in one launch
extern "C" size_t kvq_quantize_fused_workspace_size(int64_t T, int64_t D) {
    if (bad_dims(T, D)) return 0;
    return single_pass_workspace_size(D);
}

extern "C" kvq_status kvq_quantize_fused(const float *K, int64_t T, int64_t D, float *scales, int8_t *Kq,
                                         float *K_hat, void *workspace, size_t workspace_bytes, kvq_comm_t comm,
                                         int *single_pass_out, void *stream) {
    KVQ_NVTX("kvq_quantize_fused");
    KVQ_REQUIRE(K && scales && Kq && K_hat && workspace, "kvq_quantize_fused: NULL pointer");
    KVQ_REQUIRE(!bad_dims(T, D), "kvq_quantize_fused: need T >= 1, D >= 1, T*D <= 2^62");
    KVQ_REQUIRE(workspace_bytes >= single_pass_workspace_size(D), "kvq_quantize_fused: workspace too small");
    const size_t n = (size_t)(T * D);
    KVQ_REQUIRE(!overlap(K, n * 4, Kq, n) && !overlap(K_hat, n * 4, K, n * 4) && !overlap(K_hat, n * 4, Kq, n) &&
                    !overlap(scales, (size_t)D * 4, K, n * 4) && !overlap(scales, (size_t)D * 4, Kq, n) &&
                    !overlap(scales, (size_t)D * 4, K_hat, n * 4) &&
                    !overlap(workspace, workspace_bytes, K, n * 4) && !overlap(workspace, workspace_bytes, Kq, n) &&
                    !overlap(workspace, workspace_bytes, K_hat, n * 4) &&
                    !overlap(workspace, workspace_bytes, scales, (size_t)D * 4),
                "kvq_quantize_fused: buffers alias");
    KVQ_TRY(device_ok());
    cudaStream_t s = (cudaStream_t)stream;
    if (single_pass_out) *single_pass_out = 0;
    // The single pass pays off only while its second phase re-reads K from L2: measured crossover
    // (C5 sweep, profiles/r01/sweep_c5.md) between 0.5 and 1 L2 of K for D >= 1024, never for D = 128.  Beyond
    // that the two streaming passes (row-slab quantize+dequantize) are faster.  KVQ_FUSED_FORCE_SINGLE=1
    // (tests only) keeps the single pass for every shape it supports.
    const char *force_env = std::getenv("KVQ_FUSED_FORCE_SINGLE");
    const bool force_single = force_env && std::atoi(force_env) == 1;
    const bool l2_resident = D >= 256 && (int64_t)n * 4 <= device_info().l2_bytes / 4 * 3;
    if (!comm && (l2_resident || force_single)) {
        kvq_status st = launch_single_pass(K, T, D, scales, Kq, K_hat, workspace, s);
        if (st == KVQ_OK) {
            if (single_pass_out) *single_pass_out = 1;
            return KVQ_OK;
        }
        if (st != KVQ_ERR_UNSUPPORTED) return st;
    }
    // two passes (sharded input, K not L2-resident, D < 256, too large for one co-resident grid, or unaligned)
    KVQ_TRY(kvq_compute_scales(K, T, D, scales, comm, stream));
    return launch_quantize(K, scales, T, D, Kq, K_hat, s);
}

// ------------------------------------------------------------------------------ a5 + a6
extern "C" size_t kvq_error_metrics_workspace_size(int64_t T, int64_t D, int64_t nq) {
    if (bad_dims(T, D) || nq < 0) return 0;
    return metrics_workspace_size(T, D, nq) + 512;  // +512: device copy of the result for kvq_error_metrics
}

extern "C" kvq_status kvq_error_metrics_async(const float *K, const float *K_hat, int64_t T, int64_t D,
                                              const float *Q, int64_t nq, const float *scales, void *workspace,
                                              size_t workspace_bytes, kvq_comm_t comm, kvq_metrics *out_dev,
                                              void *stream) {
    KVQ_NVTX("kvq_error_metrics_async");
    KVQ_REQUIRE(K && K_hat && workspace && out_dev, "kvq_error_metrics: NULL pointer");
    KVQ_REQUIRE(!bad_dims(T, D), "kvq_error_metrics: need T >= 1, D >= 1, T*D <= 2^62");
    KVQ_REQUIRE(nq >= 0 && (nq == 0 || Q), "kvq_error_metrics: need nq >= 0 and Q when nq > 0");
    KVQ_REQUIRE(nq <= (int64_t(1) << 62) / D && nq <= (int64_t(1) << 62) / T, "kvq_error_metrics: nq too large");
    KVQ_REQUIRE(workspace_bytes >= metrics_workspace_size(T, D, nq), "kvq_error_metrics: workspace too small");
    KVQ_TRY(device_ok());
    cudaStream_t s = (cudaStream_t)stream;
    MetricTotals tot;
    if (!comm) tot.fused_out = out_dev;  // nothing to exchange: the reduction writes the result
    KVQ_TRY(launch_metrics_partials(K, K_hat, T, D, nq ? Q : nullptr, nq, scales, workspace, workspace_bytes, &tot,
                                    s));
    if (!comm) return KVQ_OK;
    KVQ_TRY(comm_allreduce_metrics(comm, tot.sums, 4, tot.maxes, 2, s));
    return launch_metrics_finalize(tot, out_dev, s);
}

extern "C" kvq_status kvq_error_metrics(const float *K, const float *K_hat, int64_t T, int64_t D, const float *Q,
                                        int64_t nq, const float *scales, void *workspace, size_t workspace_bytes,
                                        kvq_comm_t comm, kvq_metrics *out_host, void *stream) {
    KVQ_NVTX("kvq_error_metrics");
    KVQ_REQUIRE(out_host, "kvq_error_metrics: NULL out_host");
    KVQ_REQUIRE(workspace && workspace_bytes >= 512 + 64, "kvq_error_metrics: workspace too small");
    // The device copy of the result lives in the last 512 bytes of the workspace.
    uintptr_t tail = ((uintptr_t)workspace + workspace_bytes - 512 + 63) & ~(uintptr_t)63;
    kvq_metrics *dev_out = reinterpret_cast<kvq_metrics *>(tail);
    KVQ_TRY(kvq_error_metrics_async(K, K_hat, T, D, Q, nq, scales, workspace, workspace_bytes - 512, comm, dev_out,
                                    stream));
    cudaStream_t s = (cudaStream_t)stream;
    KVQ_TRY(cuda_check(cudaMemcpyAsync(out_host, dev_out, sizeof(kvq_metrics), cudaMemcpyDeviceToHost, s),
                       "copy metrics"));
    return cuda_check(cudaStreamSynchronize(s), "sync metrics");
}

extern "C" size_t kvq_roundtrip_workspace_size(int64_t T, int64_t D, int64_t nq) {
    return kvq_error_metrics_workspace_size(T, D, nq);
}

extern "C" kvq_status kvq_roundtrip(const float *K, const float *scales, int64_t T, int64_t D, int8_t *Kq,
                                    float *K_hat, const float *Q, int64_t nq, void *workspace, size_t workspace_bytes,
                                    kvq_comm_t comm, kvq_metrics *out_dev, void *stream) {
    KVQ_NVTX("kvq_roundtrip");
    KVQ_REQUIRE(K && scales && Kq && K_hat && workspace && out_dev, "kvq_roundtrip: NULL pointer");
    KVQ_REQUIRE(!bad_dims(T, D), "kvq_roundtrip: need T >= 1, D >= 1, T*D <= 2^62");
    KVQ_REQUIRE(nq >= 0 && (nq == 0 || Q), "kvq_roundtrip: need nq >= 0 and Q when nq > 0");
    KVQ_REQUIRE(nq <= (int64_t(1) << 62) / D && nq <= (int64_t(1) << 62) / T, "kvq_roundtrip: nq too large");
    const size_t n = (size_t)(T * D);
    KVQ_REQUIRE(!overlap(K, n * 4, Kq, n) && !overlap(K_hat, n * 4, K, n * 4) && !overlap(K_hat, n * 4, Kq, n) &&
                    !overlap(scales, (size_t)D * 4, Kq, n) && !overlap(scales, (size_t)D * 4, K_hat, n * 4),
                "kvq_roundtrip: outputs alias inputs");
    KVQ_REQUIRE(workspace_bytes >= metrics_workspace_size(T, D, nq), "kvq_roundtrip: workspace too small");
    KVQ_TRY(device_ok());
    cudaStream_t s = (cudaStream_t)stream;
    MetricTotals tot;
    if (!comm) tot.fused_out = out_dev;  // nothing to exchange: the reduction writes the result
    KVQ_TRY(launch_roundtrip_partials(K, scales, T, D, Kq, K_hat, nq ? Q : nullptr, nq, workspace, workspace_bytes,
                                      &tot, s));
    if (!comm) return KVQ_OK;
    KVQ_TRY(comm_allreduce_metrics(comm, tot.sums, 4, tot.maxes, 2, s));
    return launch_metrics_finalize(tot, out_dev, s);
}

extern "C" size_t kvq_step_workspace_size(int64_t T, int64_t D, int64_t nq) {
    if (bad_dims(T, D) || nq < 0) return 0;
    return std::max({kvq_roundtrip_workspace_size(T, D, nq), step_small_workspace_size(T, D),
                     roundtrip_fused_a1_workspace_size(T, D, nq)});
}

extern "C" kvq_status kvq_step(const float *K, int64_t T, int64_t D, const float *Q, int64_t nq, float *scales,
                               int8_t *Kq, float *K_hat, void *workspace, size_t workspace_bytes, kvq_comm_t comm,
                               kvq_metrics *out_dev, void *stream) {
    KVQ_NVTX("kvq_step");
    KVQ_REQUIRE(K && scales && Kq && K_hat && workspace && out_dev, "kvq_step: NULL pointer");
    KVQ_REQUIRE(!bad_dims(T, D), "kvq_step: need T >= 1, D >= 1, T*D <= 2^62");
    KVQ_REQUIRE(nq >= 0 && (nq == 0 || Q), "kvq_step: need nq >= 0 and Q when nq > 0");
    KVQ_REQUIRE(nq <= (int64_t(1) << 62) / D && nq <= (int64_t(1) << 62) / T, "kvq_step: nq too large");
    const size_t n = (size_t)(T * D);
    KVQ_REQUIRE(!overlap(K, n * 4, Kq, n) && !overlap(K_hat, n * 4, K, n * 4) && !overlap(K_hat, n * 4, Kq, n) &&
                    !overlap(scales, (size_t)D * 4, K, n * 4) && !overlap(scales, (size_t)D * 4, Kq, n) &&
                    !overlap(scales, (size_t)D * 4, K_hat, n * 4),
                "kvq_step: outputs alias inputs");
    KVQ_REQUIRE(!overlap(workspace, workspace_bytes, Kq, n) && !overlap(workspace, workspace_bytes, K_hat, n * 4) &&
                    !overlap(workspace, workspace_bytes, scales, (size_t)D * 4),
                "kvq_step: workspace aliases an output");
    KVQ_REQUIRE(workspace_bytes >= kvq_step_workspace_size(T, D, nq), "kvq_step: workspace too small");
    KVQ_TRY(device_ok());
    cudaStream_t s = (cudaStream_t)stream;
    if (step_small_eligible(T, D, nq, comm))
        return launch_step_small(K, T, D, nq ? Q : nullptr, nq, scales, Kq, K_hat, workspace, workspace_bytes,
                                 out_dev, s);
    if (roundtrip_fused_a1_eligible(K, Kq, K_hat, T, D, nq, comm)) {  // L2-resident K: one cooperative pass
        MetricTotals tot;
        tot.fused_out = out_dev;
        return launch_roundtrip_fused_a1(K, T, D, scales, Kq, K_hat, nq ? Q : nullptr, nq, workspace,
                                         workspace_bytes, &tot, s);
    }
    KVQ_TRY(kvq_compute_scales(K, T, D, scales, comm, stream));
    return kvq_roundtrip(K, scales, T, D, Kq, K_hat, Q, nq, workspace, workspace_bytes, comm, out_dev, stream);
}

extern "C" size_t kvq_attention_scores_workspace_size(int64_t D, int64_t nq) {
    if (D < 1 || nq < 1) return 0;
    return attention_scores_workspace_size(D, nq);
}

extern "C" kvq_status kvq_attention_scores(const float *Q, int64_t nq, const float *K, const float *K_hat, int64_t T,
                                           int64_t D, float *S, void *workspace, size_t workspace_bytes,
                                           void *stream) {
    KVQ_NVTX("kvq_attention_scores");
    KVQ_REQUIRE(Q && K && S, "kvq_attention_scores: NULL pointer");
    KVQ_REQUIRE(!bad_dims(T, D) && nq >= 1 && nq <= (int64_t(1) << 62) / T, "kvq_attention_scores: bad sizes");
    KVQ_TRY(device_ok());
    return launch_attention_scores(Q, nq, K, K_hat, T, D, S, workspace, workspace_bytes, (cudaStream_t)stream);
}

// ------------------------------------------------------------------------------ NEXT-2: scores from codes
extern "C" size_t kvq_scores_from_codes_workspace_size(int64_t D, int64_t nq) {
    if (D < 1 || nq < 1) return 0;
    return scores_codes_workspace_size(D);
}

extern "C" kvq_status kvq_scores_from_codes(const float *Q, int64_t nq, const int8_t *Kq, const float *scales,
                                            int64_t T, int64_t D, float *S, void *workspace, size_t workspace_bytes,
                                            void *stream) {
    KVQ_NVTX("kvq_scores_from_codes");
    KVQ_REQUIRE(Q && Kq && scales && S, "kvq_scores_from_codes: NULL pointer");
    KVQ_REQUIRE(!bad_dims(T, D) && nq >= 1 && nq <= (int64_t(1) << 62) / T && nq <= (int64_t(1) << 62) / D,
                "kvq_scores_from_codes: bad sizes");
    KVQ_REQUIRE(!overlap(S, (size_t)(nq * T) * 4, Kq, (size_t)(T * D)) &&
                    !overlap(S, (size_t)(nq * T) * 4, Q, (size_t)(nq * D) * 4),
                "kvq_scores_from_codes: S aliases an input");
    KVQ_TRY(device_ok());
    return launch_scores_codes(Q, nq, Kq, scales, T, D, S, workspace, workspace_bytes, (cudaStream_t)stream);
}

// ------------------------------------------------------------------------------ host-buffer pipeline
namespace {
struct HostLayout {
    size_t K, Kh, Kq, scales, Q, mws, mout, total;
};
size_t al(size_t x) { return (x + 255) & ~(size_t)255; }
HostLayout host_layout(int64_t T, int64_t D, int64_t nq) {
    HostLayout L;
    const size_t n = (size_t)(T * D);
    size_t off = 0;
    L.K = off; off += al(n * 4);
    L.Kh = off; off += al(n * 4);
    L.Kq = off; off += al(n);
    L.scales = off; off += al((size_t)D * 4);
    L.Q = off; off += al((size_t)(nq * D) * 4);
    L.mws = off; off += al(metrics_workspace_size(T, D, nq));
    L.mout = off; off += al(sizeof(kvq_metrics));
    L.total = off + 256;  // base alignment slack
    return L;
}
}  // namespace

extern "C" size_t kvq_roundtrip_host_workspace_size(int64_t T, int64_t D, int64_t nq) {
    if (bad_dims(T, D) || nq < 0) return 0;
    return host_layout(T, D, nq).total;
}

// Enqueue the whole host-buffer pipeline.  Three streams: the caller's `stream`
// runs the kernels; library-owned H2D and D2H streams drive the two copy engines,
// so consecutive calls on different caller streams overlap call i's D2H with
// call i+1's H2D (PCIe is full duplex).  The caller's stream finally waits for
// the D2H stream, so synchronizing `stream` covers everything.
static kvq_status roundtrip_host_enqueue(const float *K_host, int64_t T, int64_t D, const float *Q_host, int64_t nq,
                                         float *scales_host, int8_t *Kq_host, float *K_hat_host,
                                         kvq_metrics *metrics_host, void *dev_workspace, size_t workspace_bytes,
                                         kvq_comm_t comm, void *stream, const char *name) {
    KVQ_REQUIRE(K_host && scales_host && Kq_host && metrics_host && dev_workspace, std::string(name) + ": NULL pointer");
    KVQ_REQUIRE(!bad_dims(T, D), std::string(name) + ": need T >= 1, D >= 1, T*D <= 2^62");
    KVQ_REQUIRE(nq >= 0 && (nq == 0 || Q_host), std::string(name) + ": need nq >= 0 and Q when nq > 0");
    const HostLayout L = host_layout(T, D, nq);
    KVQ_REQUIRE(workspace_bytes >= L.total, std::string(name) + ": workspace too small");
    KVQ_TRY(device_ok());
    cudaStream_t s = (cudaStream_t)stream;
    cudaStream_t hs = copy_stream(0), ds = copy_stream(1);
    char *base = reinterpret_cast<char *>(((uintptr_t)dev_workspace + 255) & ~(uintptr_t)255);
    float *K = reinterpret_cast<float *>(base + L.K);
    float *Kh = reinterpret_cast<float *>(base + L.Kh);
    int8_t *Kq = reinterpret_cast<int8_t *>(base + L.Kq);
    float *sc = reinterpret_cast<float *>(base + L.scales);
    float *Q = reinterpret_cast<float *>(base + L.Q);
    kvq_metrics *mout = reinterpret_cast<kvq_metrics *>(base + L.mout);
    uint32_t *bits = reinterpret_cast<uint32_t *>(sc);

    // Row blocks of ~64 MB: block b's column-max kernel runs while block b+1 is on the copy engine.
    const size_t row_bytes = (size_t)D * 4;
    int64_t rows_per = std::max<int64_t>(1, (int64_t)((64u << 20) / row_bytes));
    int64_t nblk = (T + rows_per - 1) / rows_per;
    if (nblk > 64) {
        rows_per = (T + 63) / 64;
        nblk = (T + rows_per - 1) / rows_per;
    }
    // events: [0, nblk) H2D blocks, nblk start, nblk+1 Q, nblk+2 compute done, nblk+3 D2H done
    std::vector<cudaEvent_t> ev(nblk + 4);
    for (auto &e : ev) KVQ_TRY(cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create"));
    kvq_status st = KVQ_OK;
    auto ck = [&](cudaError_t e, const char *what) {
        if (st == KVQ_OK) st = cuda_check(e, what);
        return st == KVQ_OK;
    };
    do {
        // the workspace is free once earlier work on `s` is done
        if (!ck(cudaEventRecord(ev[nblk], s), "record") || !ck(cudaStreamWaitEvent(hs, ev[nblk], 0), "wait")) break;
        if (!ck(cudaMemsetAsync(bits, 0, (size_t)D * 4, s), "memset")) break;
        if (nq) {
            if (!ck(cudaMemcpyAsync(Q, Q_host, (size_t)(nq * D) * 4, cudaMemcpyHostToDevice, hs), "H2D Q") ||
                !ck(cudaEventRecord(ev[nblk + 1], hs), "record"))
                break;
        }
        for (int64_t b = 0; b < nblk && st == KVQ_OK; b++) {
            const int64_t r0 = b * rows_per, nr = std::min(rows_per, T - r0);
            if (!ck(cudaMemcpyAsync(K + r0 * D, K_host + r0 * D, (size_t)(nr * D) * 4, cudaMemcpyHostToDevice, hs),
                    "H2D K") ||
                !ck(cudaEventRecord(ev[b], hs), "record") || !ck(cudaStreamWaitEvent(s, ev[b], 0), "wait"))
                break;
            st = launch_colmax(K + r0 * D, nr, D, bits, s);
        }
        if (st != KVQ_OK) break;
        if (nq && !ck(cudaStreamWaitEvent(s, ev[nblk + 1], 0), "wait")) break;
        if (comm && (st = comm_allreduce_max_u32(comm, bits, (size_t)D, s)) != KVQ_OK) break;
        if ((st = launch_finalize(bits, D, s)) != KVQ_OK) break;
        MetricTotals tot;
        if ((st = launch_roundtrip_partials(K, sc, T, D, Kq, Kh, nq ? Q : nullptr, nq, base + L.mws,
                                            metrics_workspace_size(T, D, nq), &tot, s)) != KVQ_OK)
            break;
        if (comm) {
            if ((st = comm_allreduce_metrics(comm, tot.sums, 4, tot.maxes, 2, s)) != KVQ_OK) break;
        }
        if ((st = launch_metrics_finalize(tot, mout, s)) != KVQ_OK) break;
        // results back on the D2H copy engine
        if (!ck(cudaEventRecord(ev[nblk + 2], s), "record") || !ck(cudaStreamWaitEvent(ds, ev[nblk + 2], 0), "wait"))
            break;
        if (!ck(cudaMemcpyAsync(Kq_host, Kq, (size_t)(T * D), cudaMemcpyDeviceToHost, ds), "D2H Kq") ||
            !ck(cudaMemcpyAsync(scales_host, sc, (size_t)D * 4, cudaMemcpyDeviceToHost, ds), "D2H scales") ||
            !ck(cudaMemcpyAsync(metrics_host, mout, sizeof(kvq_metrics), cudaMemcpyDeviceToHost, ds), "D2H metrics"))
            break;
        if (K_hat_host &&
            !ck(cudaMemcpyAsync(K_hat_host, Kh, (size_t)(T * D) * 4, cudaMemcpyDeviceToHost, ds), "D2H K_hat"))
            break;
        if (!ck(cudaEventRecord(ev[nblk + 3], ds), "record") || !ck(cudaStreamWaitEvent(s, ev[nblk + 3], 0), "wait"))
            break;
    } while (0);
    for (auto &e : ev) cudaEventDestroy(e);  // released once the pending work completes
    return st;
}

extern "C" kvq_status kvq_roundtrip_host_async(const float *K_host, int64_t T, int64_t D, const float *Q_host,
                                               int64_t nq, float *scales_host, int8_t *Kq_host, float *K_hat_host,
                                               kvq_metrics *metrics_host, void *dev_workspace, size_t workspace_bytes,
                                               kvq_comm_t comm, void *stream) {
    KVQ_NVTX("kvq_roundtrip_host_async");
    return roundtrip_host_enqueue(K_host, T, D, Q_host, nq, scales_host, Kq_host, K_hat_host, metrics_host,
                                  dev_workspace, workspace_bytes, comm, stream, "kvq_roundtrip_host_async");
}

extern "C" kvq_status kvq_roundtrip_host(const float *K_host, int64_t T, int64_t D, const float *Q_host, int64_t nq,
                                         float *scales_host, int8_t *Kq_host, float *K_hat_host,
                                         kvq_metrics *metrics_host, void *dev_workspace, size_t workspace_bytes,
                                         kvq_comm_t comm, void *stream) {
    KVQ_NVTX("kvq_roundtrip_host");
    KVQ_TRY(roundtrip_host_enqueue(K_host, T, D, Q_host, nq, scales_host, Kq_host, K_hat_host, metrics_host,
                                   dev_workspace, workspace_bytes, comm, stream, "kvq_roundtrip_host"));
    return cuda_check(cudaStreamSynchronize((cudaStream_t)stream), "sync stream");
}
