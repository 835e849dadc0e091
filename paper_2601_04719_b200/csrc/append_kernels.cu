// append_kernels.cu — NEXT-4: streaming append with dynamic
// per-channel scales (P:564 dynamic quantization, P:570 persistent kernels;
// reading Q20 in DESIGN.md §3).
//
// A growing key cache K[0:T][D] (fp32, retained) with its INT8 codes and scales.
// Appending rows [T_old, T_old + n_new) keeps the invariant
//     scales == Alg.1 / Eq.6 over K[0:T_new],  Kq / K_hat == Eq.7 / Eq.8 of K[0:T_new]
// bit for bit (streaming == batch), by
//   A  running column max m_d <- max(m_d, max over the new rows |K[t,d]|)
//      (uint32 abs-bit max, order-free; all-reduced (MAX) over ranks when the
//      cache is token-sharded);
//   B  s'_d = fl32(m_d / 127); a column whose scale changed is "grown";
//   C  quantize (+dequantize) the new rows with s', and RE-quantize the old rows
//      of every grown column from the retained K (a code depends only on x and s_d).
// For i.i.d. keys a column's max grows with probability ~n_new / T, so after the
// first tokens step C touches ~D * n_new / T old columns per append.
//
// Decode-sized appends (n_new <= kSmallAppend, single GPU) run A, B and C in ONE
// cooperative launch with grid-wide syncs (launch latency dominates these steps;
// one launch instead of four).  Prefill-sized appends, and every append on a
// token-sharded cache (the NCCL all-reduce sits between A and B), run the
// streaming kernels of quant_kernels.cu for the new rows plus the small kernels
// below.  Quantization uses the IEEE quotient (quant_exact) in the small kernels
// and the reciprocal+repair path of quant_kernels.cu for prefill; both are exact.
#include <cooperative_groups.h>

#include <algorithm>

#include "device_common.cuh"
#include "kvq_internal.h"

namespace cg = cooperative_groups;

namespace kvq {

constexpr int64_t kSmallAppend = 256;  // rows: cooperative single-launch path at or below this
constexpr int kAppendThreads = 256;

struct AppendParams {
    const float *K;  // [T_old + n_new][D]
    int64_t T_old, n_new, D;
    uint32_t *absmax;  // [D] running abs-bit max
    float *scales;     // [D] running scales
    int8_t *Kq;        // [T_old + n_new][D]
    float *K_hat;      // nullable
    int *grown;        // [D] list of grown columns (workspace)
    int *n_grown;      // [1] (workspace)
};

constexpr int kMaxRows = 8;  // rows folded per thread before the atomic in phase A

__device__ __forceinline__ void phase_max(const AppendParams &p, int64_t tid, int64_t nthreads) {
    // item = (row group of kMaxRows new rows, column d): coalesced across threads,
    // one atomicMax per item (order-free uint32 max of the abs bits)
    const int64_t groups = (p.n_new + kMaxRows - 1) / kMaxRows, items = groups * p.D;
    for (int64_t o = tid; o < items; o += nthreads) {
        const int64_t d = o % p.D, t0 = p.T_old + (o / p.D) * kMaxRows;
        const int64_t t1 = min(t0 + kMaxRows, p.T_old + p.n_new);
        uint32_t m = 0;
#pragma unroll 4
        for (int64_t t = t0; t < t1; t++) m = max(m, absbits(__ldg(p.K + t * p.D + d)));
        if (m) atomicMax(p.absmax + d, m);
    }
}

__device__ __forceinline__ void phase_scales(const AppendParams &p, int64_t tid, int64_t nthreads) {
    for (int64_t d = tid; d < p.D; d += nthreads) {
        const float s = __fdiv_rn(__uint_as_float(p.absmax[d]), 127.0f);
        if (__float_as_uint(s) != __float_as_uint(p.scales[d])) {
            p.scales[d] = s;
            p.grown[atomicAdd(p.n_grown, 1)] = (int)d;
        }
    }
}

__device__ __forceinline__ void quant_one(const AppendParams &p, int64_t t, int64_t d, float s) {
    const int64_t i = t * p.D + d;
    const int q = quant_exact(p.K[i], s);
    p.Kq[i] = (int8_t)q;
    if (p.K_hat) p.K_hat[i] = __fmul_rn((float)q, s);
}

// new rows (if `new_rows`) and the old rows of the grown columns
__device__ __forceinline__ void phase_quant(const AppendParams &p, bool new_rows, int64_t tid, int64_t nthreads) {
    if (new_rows) {
        const int64_t n = p.n_new * p.D;
        for (int64_t o = tid; o < n; o += nthreads) {
            const int64_t d = o % p.D;
            quant_one(p, p.T_old + o / p.D, d, p.scales[d]);
        }
    }
    const int64_t ng = *reinterpret_cast<volatile int *>(p.n_grown);
    const int64_t m = ng * p.T_old;
    for (int64_t o = tid; o < m; o += nthreads) {
        const int64_t d = p.grown[o % ng];
        quant_one(p, o / ng, d, p.scales[d]);
    }
}

// ---- decode-sized appends: one cooperative launch
__global__ void __launch_bounds__(kAppendThreads) append_coop_kernel(AppendParams p) {
    cg::grid_group grid = cg::this_grid();
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    if (tid == 0) *p.n_grown = 0;
    phase_max(p, tid, nth);
    grid.sync();
    phase_scales(p, tid, nth);
    grid.sync();
    phase_quant(p, true, tid, nth);
}

// ---- general path: separate kernels
__global__ void append_max_kernel(AppendParams p) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    if (tid == 0) *p.n_grown = 0;
    phase_max(p, tid, nth);
}
__global__ void append_reset_kernel(int *n_grown) { *n_grown = 0; }
__global__ void append_scales_kernel(AppendParams p) {
    phase_scales(p, (int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
}
__global__ void append_quant_kernel(AppendParams p, int new_rows) {
    phase_quant(p, new_rows != 0, (int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
}

// [n_grown (4 B) | pad to 256 | grown[D] ints] at a 256-byte aligned offset of any caller pointer
size_t append_workspace_size(int64_t D) { return (size_t)D * sizeof(int) + 256 + 255; }

kvq_status launch_append(const float *K, int64_t T_old, int64_t n_new, int64_t D, uint32_t *absmax, float *scales,
                         int8_t *Kq, float *K_hat, void *ws, kvq_comm_t comm, cudaStream_t s) {
    AppendParams p{K, T_old, n_new, D, absmax, scales, Kq, K_hat, nullptr, nullptr};
    char *w = reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(ws) + 255) & ~(uintptr_t)255);
    p.n_grown = reinterpret_cast<int *>(w);  // atomicAdd target: aligned whatever the caller's pointer
    p.grown = reinterpret_cast<int *>(w + 256);
    const int sms = device_info().num_sms;
    if (!comm && n_new <= kSmallAppend) {
        static int per_sm = [] {
            int nb = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, append_coop_kernel, kAppendThreads, 0) !=
                    cudaSuccess ||
                nb < 1) {
                cudaGetLastError();
                nb = 1;
            }
            return nb;
        }();
        // enough threads for the widest phase, never more than co-resident
        const int64_t work = std::max<int64_t>(D, n_new * D);
        const int blocks = (int)std::min<int64_t>((int64_t)sms * per_sm,
                                                  std::max<int64_t>(1, (work + kAppendThreads - 1) / kAppendThreads));
        void *args[] = {&p};
        const cudaError_t e = cudaLaunchCooperativeKernel((const void *)append_coop_kernel, dim3(blocks),
                                                          dim3(kAppendThreads), args, 0, s);
        if (e != cudaSuccess) {
            cudaGetLastError();
            return fail(KVQ_ERR_CUDA, std::string("append cooperative launch: ") + cudaGetErrorString(e));
        }
        return check_launch("append_coop");
    }
    // A: running max over the new rows (this rank's), then the all-reduce
    if (n_new > kSmallAppend) {
        append_reset_kernel<<<1, 1, 0, s>>>(p.n_grown);
        if (kvq_status st = check_launch("append_reset"); st != KVQ_OK) return st;
        if (kvq_status st = launch_colmax(K + T_old * D, n_new, D, absmax, s); st != KVQ_OK) return st;
    } else {
        append_max_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((D + 255) / 256, 4 * sms)), 256, 0, s>>>(
            p);
        if (kvq_status st = check_launch("append_max"); st != KVQ_OK) return st;
    }
    if (comm)
        if (kvq_status st = comm_allreduce_max_u32(comm, absmax, (size_t)D, s); st != KVQ_OK) return st;
    // B: new scales, grown columns
    append_scales_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((D + 255) / 256, 4 * sms)), 256, 0, s>>>(
        p);
    if (kvq_status st = check_launch("append_scales"); st != KVQ_OK) return st;
    // C: new rows (streaming kernel for prefill-sized appends), old rows of grown columns
    const bool big = n_new > kSmallAppend;
    if (big && n_new > 0) {
        if (kvq_status st = launch_quantize(K + T_old * D, scales, n_new, D, Kq + T_old * D,
                                            K_hat ? K_hat + T_old * D : nullptr, s);
            st != KVQ_OK)
            return st;
    }
    append_quant_kernel<<<(unsigned)(4 * sms), 256, 0, s>>>(p, big ? 0 : 1);
    return check_launch("append_quant");
}

}  // namespace kvq
