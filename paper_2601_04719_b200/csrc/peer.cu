// peer.cu — a1 + a7 + a2 in ONE kernel over peer memory (the
// scale all-reduce without NCCL).
//
// Token-sharded ranks (one GPU each) need the global column max m_d = MAX_r m_d^(r)
// (Eq. 6 over the whole matrix; the max is order-free) before
// any rank can form s_d = m_d / 127 (Eq. 5/6).  Instead of column-max kernel
// -> ncclAllReduce(MAX) -> finalize kernel, each rank runs one kernel:
//   1. every CTA reduces its share of the local shard into `bits` (the same
//      column-owning 128-bit streaming loop as colmax_v4_kernel, atomicMax of the
//      abs bits);
//   2. the LAST CTA to finish (grid-wide ticket) pushes the local D-vector straight
//      into slot `rank` of every rank's exchange buffer (P2P stores over NVLink into
//      buffers mapped with CUDA IPC), publishes an epoch flag in every rank's buffer
//      (system-scope release), waits for the flags of all ranks (system-scope
//      acquire), then takes the max over the R slots of its own buffer and writes
//      s_d = fl32(m_d / divisor) for all d.
// No host round trip and no collective library call: the exchange (R x D x 4 bytes
// per rank, 32 KB per peer at D = 8192) overlaps the tail of the column-max pass of
// the slower ranks.  Slots are double-buffered by epoch parity: a fast rank can be
// at most one epoch ahead (it needs every rank's flag of epoch e to finish e), so
// epoch e+1 never overwrites the slots a slow rank is still reading for epoch e.
//
// Bit-exact with kvq_compute_scales (+NCCL) and the oracle: max is exact in any
// order.  Every rank must call kvq_compute_scales_peer the same number of times in
// the same order (like NCCL), and the ranks' kernels must be able to run
// concurrently (one GPU per rank, or time-sliced processes on one GPU in tests).
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <random>
#include <string>
#include <thread>

#include "device_common.cuh"
#include "kvq_internal.h"

constexpr int kPeerMax = 16;

struct PeerArgs {
    uint32_t *bufs[kPeerMax];  // every rank's exchange buffer (bufs[rank] = this rank's own)
    uint32_t *mc;              // NVLS: multicast mapping of the column slots (nullptr: P2P slot stores)
    uint32_t *uc;              // NVLS: this rank's own physical copy of them (unicast mapping)
    unsigned *ticket;          // grid-wide ticket (this rank's buffer)
    int nranks, rank;
    int64_t D, slot_stride;    // u32 per slot (D rounded up to 64)
    uint64_t epoch;
    float divisor;
    uint64_t timeout_ns;       // a peer that has not arrived by then failed or died: trap instead of hanging
};

// exchange buffer layout (u32 units): [flags: kPeerMax x u64 = 32 u32][ticket: 1 u32, pad to 64]
// [metric slots: 2 parities x kPeerMax x 8 u64 = 512 u32][column slots: 2 parities x R x S u32]
// One epoch counter and one flag per rank serve both kinds of exchange: every rank performs the same sequence
// of exchanges, so epoch e means the same exchange everywhere.
constexpr int64_t kFlagsU32 = 2 * kPeerMax, kMetU32 = 64, kMetSlotU64 = 8,
                  kHdrU32 = kMetU32 + 2 * kPeerMax * kMetSlotU64 * 2;

struct kvq_peer_s {
    int nranks, rank, device;
    int64_t D;
    uint32_t *local;                 // library-owned (cudaMalloc), shared with the peers over CUDA IPC
    uint32_t *mapped[kPeerMax];      // peer buffers opened with cudaIpcOpenMemHandle (own slot: nullptr)
    uint32_t *bufs[kPeerMax];
    uint64_t epoch;
    bool open;
    // NVLS (NVLink SHARP multicast): the a7 column maxima reduced inside the NVSwitch
    struct {
        bool joined = false, mapped = false, active = false;
        unsigned long long mc = 0, mem = 0;  // CUmemGenericAllocationHandle of the multicast object / own memory
        unsigned long long mc_va = 0, uc_va = 0;
        size_t bytes = 0;
        int device = -1;
        std::thread server;  // POSIX-fd export: hands the fd to the other ranks over a unix socket
        int listen_fd = -1, export_fd = -1;
    } nv;
};

namespace kvq {

__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// The calling CTA's slot stores are done (before a __syncthreads): publish epoch `pa.epoch` in every rank's
// buffer, then wait until every rank has published it in ours.  Release/acquire at system scope.
// (fence.acq_rel.sys, not the sequentially consistent fence.sc.sys of __threadfence_system: the release store
// is cumulative over the CTA's slot stores ordered before it by bar.sync.)
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void peer_signal_wait(const PeerArgs &pa) {
    __syncthreads();
    if (threadIdx.x == 0) {
        fence_acq_rel_sys();  // the slot stores are visible to every GPU before the flags
        for (int r = 0; r < pa.nranks; r++)
            st_release_sys(reinterpret_cast<uint64_t *>(pa.bufs[r]) + pa.rank, pa.epoch);
    }
    const uint64_t *flags = reinterpret_cast<const uint64_t *>(pa.bufs[pa.rank]);
    if ((int)threadIdx.x < pa.nranks) {
        uint64_t t0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        while (ld_acquire_sys(flags + threadIdx.x) < pa.epoch) {
            __nanosleep(32);
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            // Bounded wait: a rank that returned an error before its exchange (argument checks are
            // rank-local) or died never raises its flag.  Fail loudly (the caller's next synchronization
            // reports a launch failure) instead of spinning forever.
            if (t - t0 > pa.timeout_ns) __trap();
        }
    }
    __syncthreads();
    fence_acq_rel_sys();
}

// All-reduce MAX of `count` (<= D) u32 in place, one CTA.
__global__ void __launch_bounds__(kThreads) peer_max_u32_kernel(uint32_t *buf, int64_t count,
                                                                const __grid_constant__ PeerArgs pa) {
    const int par = (int)(pa.epoch & 1);
    const int64_t base = kHdrU32 + (int64_t)par * pa.nranks * pa.slot_stride;
    for (int64_t i = threadIdx.x; i < count; i += kThreads) {
        const uint32_t v = buf[i];
        for (int r = 0; r < pa.nranks; r++) pa.bufs[r][base + (int64_t)pa.rank * pa.slot_stride + i] = v;
    }
    peer_signal_wait(pa);
    const uint32_t *own = pa.bufs[pa.rank] + base;
    for (int64_t i = threadIdx.x; i < count; i += kThreads) {
        uint32_t m = 0;
        for (int r = 0; r < pa.nranks; r++) m = max(m, __ldcv(own + (int64_t)r * pa.slot_stride + i));
        buf[i] = m;
    }
}

// The metric partials: nsum fp64 sums (added in rank order: deterministic and identical on every rank) and nmax
// u64 bit-pattern maxima, in place, one CTA.
__global__ void peer_metrics_kernel(double *sums, int nsum, uint64_t *maxes, int nmax,
                                    const __grid_constant__ PeerArgs pa) {
    const int par = (int)(pa.epoch & 1);
    const int64_t base = kMetU32 + (int64_t)par * kPeerMax * kMetSlotU64 * 2;  // u32 units
    const int t = threadIdx.x;
    if (t < nsum + nmax) {
        const uint64_t v = t < nsum ? (uint64_t)__double_as_longlong(sums[t]) : maxes[t - nsum];
        for (int r = 0; r < pa.nranks; r++)
            reinterpret_cast<uint64_t *>(pa.bufs[r] + base)[pa.rank * kMetSlotU64 + t] = v;
    }
    peer_signal_wait(pa);
    const uint64_t *own = reinterpret_cast<const uint64_t *>(pa.bufs[pa.rank] + base);
    if (t < nsum) {
        double acc = 0.0;
        for (int r = 0; r < pa.nranks; r++) acc += __longlong_as_double((long long)__ldcv(own + r * kMetSlotU64 + t));
        sums[t] = acc;
    } else if (t < nsum + nmax) {
        uint64_t m = 0;
        for (int r = 0; r < pa.nranks; r++) m = max(m, __ldcv(own + r * kMetSlotU64 + t));
        maxes[t - nsum] = m;
    }
}

template <int U>
__global__ void __launch_bounds__(kThreads, 6) colmax_peer_kernel(const float4 *__restrict__ K, int64_t n4,
                                                               int64_t cols4, int64_t G, uint32_t *bits,
                                                               const __grid_constant__ PeerArgs pa) {
    // ---- 1. local column max of this rank's shard (colmax_v4_kernel's loop: a CTA-level smem max first when
    //         the columns fit, so narrow heads do not funnel every thread's atomics into D addresses)
    extern __shared__ uint32_t smax[];  // [4 * cols4] when cols4 <= kThreads
    const bool share = cols4 <= kThreads;
    const int64_t g = (int64_t)blockIdx.x * kThreads + threadIdx.x;
    if (share) {
        for (int i = threadIdx.x; i < 4 * cols4; i += kThreads) smax[i] = 0u;
        __syncthreads();
    }
    uint32_t m0 = 0, m1 = 0, m2 = 0, m3 = 0;
    int64_t c4 = 0;
    if (g < G) {
        c4 = g % cols4;
        int64_t i = g;
        for (; i + (U - 1) * G < n4; i += U * G) {
            float4 v[U];
#pragma unroll
            for (int k = 0; k < U; k++) v[k] = KVQ_COLMAX_LD(K + i + k * G);
#pragma unroll
            for (int k = 0; k < U; k++) {
                m0 = max(m0, absbits(v[k].x));
                m1 = max(m1, absbits(v[k].y));
                m2 = max(m2, absbits(v[k].z));
                m3 = max(m3, absbits(v[k].w));
            }
        }
        for (; i < n4; i += G) {
            const float4 v = KVQ_COLMAX_LD(K + i);
            m0 = max(m0, absbits(v.x));
            m1 = max(m1, absbits(v.y));
            m2 = max(m2, absbits(v.z));
            m3 = max(m3, absbits(v.w));
        }
    }
    if (share) {
        if (g < G) {
            atomicMax(&smax[4 * c4 + 0], m0);
            atomicMax(&smax[4 * c4 + 1], m1);
            atomicMax(&smax[4 * c4 + 2], m2);
            atomicMax(&smax[4 * c4 + 3], m3);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < 4 * cols4; i += kThreads)
            if (smax[i]) atomicMax(&bits[i], smax[i]);
    } else if (g < G) {
        if (m0) atomicMax(&bits[4 * c4 + 0], m0);
        if (m1) atomicMax(&bits[4 * c4 + 1], m1);
        if (m2) atomicMax(&bits[4 * c4 + 2], m2);
        if (m3) atomicMax(&bits[4 * c4 + 3], m3);
    }
    // ---- 2. the last CTA exchanges and finalizes
    __shared__ unsigned last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(pa.ticket, 1u) == gridDim.x - 1 ? 1u : 0u;
    __syncthreads();
    if (!last) return;
    __threadfence();  // every CTA's atomics on `bits` are visible
    const int64_t D = pa.D;
    const int par = (int)(pa.epoch & 1);
    const int64_t D4 = D / 4;
    if (pa.mc) {
        // NVLS: every rank stores its D-vector into its OWN copy of the parity's slot; after the flags, one
        // multimem.ld_reduce.max per column makes the NVSwitch read all ranks' copies and return their max
        uint4 *mine = reinterpret_cast<uint4 *>(pa.uc + (int64_t)par * pa.slot_stride);
        for (int64_t i = threadIdx.x; i < D4; i += kThreads) mine[i] = __ldcg(reinterpret_cast<const uint4 *>(bits) + i);
        if (threadIdx.x == 0) *pa.ticket = 0u;
        peer_signal_wait(pa);
        const uint32_t *mc = pa.mc + (int64_t)par * pa.slot_stride;
        for (int64_t d = threadIdx.x; d < D; d += kThreads) {
            uint32_t m;
            asm volatile("multimem.ld_reduce.relaxed.sys.global.max.u32 %0, [%1];" : "=r"(m) : "l"(mc + d) : "memory");
            reinterpret_cast<float *>(bits)[d] = __fdiv_rn(__uint_as_float(m), pa.divisor);  // Eq. 5/6, reading Q3
        }
        return;
    }
    const int64_t my_slot = kHdrU32 + ((int64_t)par * pa.nranks + pa.rank) * pa.slot_stride;
    // 16-byte accesses (D % 4 == 0; slots are 256-byte aligned), independent iterations
    for (int64_t i = threadIdx.x; i < D4; i += kThreads) {
        const uint4 v = __ldcg(reinterpret_cast<const uint4 *>(bits) + i);
        for (int r = 0; r < pa.nranks; r++)
            reinterpret_cast<uint4 *>(pa.bufs[r] + my_slot)[i] = v;  // P2P stores (own buffer for r == rank)
    }
    if (threadIdx.x == 0) *pa.ticket = 0u;  // ready for the next call (stream order separates the launches)
    peer_signal_wait(pa);
    const uint32_t *own = pa.bufs[pa.rank] + kHdrU32 + (int64_t)par * pa.nranks * pa.slot_stride;
    float4 *scales4 = reinterpret_cast<float4 *>(bits);
    for (int64_t i = threadIdx.x; i < D4; i += kThreads) {
        uint4 m = make_uint4(0u, 0u, 0u, 0u);
        for (int r = 0; r < pa.nranks; r++) {
            const uint4 v = __ldcv(reinterpret_cast<const uint4 *>(own + (int64_t)r * pa.slot_stride) + i);
            m.x = max(m.x, v.x);
            m.y = max(m.y, v.y);
            m.z = max(m.z, v.z);
            m.w = max(m.w, v.w);
        }
        // Eq. 5/6, reading Q3: IEEE division
        scales4[i] = make_float4(__fdiv_rn(__uint_as_float(m.x), pa.divisor), __fdiv_rn(__uint_as_float(m.y), pa.divisor),
                                 __fdiv_rn(__uint_as_float(m.z), pa.divisor), __fdiv_rn(__uint_as_float(m.w), pa.divisor));
    }
}

static int64_t slot_stride(int64_t D) { return (D + 63) / 64 * 64; }
static size_t peer_bytes(int64_t D, int nranks) {
    return (size_t)(kHdrU32 + 2 * (int64_t)nranks * slot_stride(D)) * 4;
}

}  // namespace kvq

using namespace kvq;

#define KVQ_REQUIRE(cond, msg)                                    \
    do {                                                          \
        if (!(cond)) return fail(KVQ_ERR_INVALID_VALUE, msg);     \
    } while (0)
#define KVQ_TRY(expr)                  \
    do {                               \
        kvq_status _st = (expr);       \
        if (_st != KVQ_OK) return _st; \
    } while (0)


extern "C" size_t kvq_peer_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

extern "C" kvq_status kvq_peer_init(kvq_peer_t *out, int nranks, int rank, int64_t D, void *handle_out) {
    KVQ_NVTX("kvq_peer_init");
    KVQ_REQUIRE(out && handle_out, "kvq_peer_init: NULL pointer");
    KVQ_REQUIRE(nranks >= 1 && nranks <= kPeerMax && rank >= 0 && rank < nranks,
                "kvq_peer_init: need 1 <= nranks <= 16 and 0 <= rank < nranks");
    KVQ_REQUIRE(D >= 1 && D <= (int64_t(1) << 31), "kvq_peer_init: need 1 <= D <= 2^31");
    *out = nullptr;
    KVQ_TRY(device_ok());
    auto *p = new kvq_peer_s();
    p->nranks = nranks;
    p->rank = rank;
    p->D = D;
    p->epoch = 0;
    p->open = false;
    cudaGetDevice(&p->device);
    const size_t bytes = peer_bytes(D, nranks);
    if (cudaMalloc(&p->local, bytes) != cudaSuccess || cudaMemset(p->local, 0, bytes) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
        if (p->local) cudaFree(p->local);
        delete p;
        cudaGetLastError();
        return fail(KVQ_ERR_CUDA, "kvq_peer_init: exchange buffer allocation failed");
    }
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, p->local) != cudaSuccess) {
        cudaFree(p->local);
        delete p;
        cudaGetLastError();
        return fail(KVQ_ERR_CUDA, "kvq_peer_init: cudaIpcGetMemHandle failed");
    }
    std::memcpy(handle_out, &h, sizeof(h));
    *out = p;
    return KVQ_OK;
}

extern "C" kvq_status kvq_peer_open(kvq_peer_t p, const void *handles) {
    KVQ_NVTX("kvq_peer_open");
    KVQ_REQUIRE(p && handles, "kvq_peer_open: NULL pointer");
    KVQ_REQUIRE(!p->open, "kvq_peer_open: already open");
    for (int r = 0; r < p->nranks; r++) {
        if (r == p->rank) {
            p->bufs[r] = p->local;
            continue;
        }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, static_cast<const char *>(handles) + (size_t)r * sizeof(h), sizeof(h));
        void *ptr = nullptr;
        if (cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            const std::string e = cudaGetErrorString(cudaGetLastError());
            for (int q = 0; q < r; q++)
                if (p->mapped[q]) cudaIpcCloseMemHandle(p->mapped[q]), p->mapped[q] = nullptr;
            return fail(KVQ_ERR_CUDA, "kvq_peer_open: cudaIpcOpenMemHandle(rank " + std::to_string(r) + "): " + e);
        }
        p->mapped[r] = p->bufs[r] = static_cast<uint32_t *>(ptr);
    }
    p->open = true;
    return KVQ_OK;
}

static void nvls_release(kvq_peer_t p);

extern "C" kvq_status kvq_peer_destroy(kvq_peer_t p) {
    KVQ_NVTX("kvq_peer_destroy");
    if (!p) return KVQ_OK;
    cudaDeviceSynchronize();
    nvls_release(p);
    for (int r = 0; r < p->nranks; r++)
        if (p->mapped[r]) cudaIpcCloseMemHandle(p->mapped[r]);
    cudaFree(p->local);
    cudaGetLastError();
    delete p;
    return KVQ_OK;
}

static PeerArgs peer_args(kvq_peer_t p, float divisor) {
    PeerArgs pa{};
    if (p->nv.active) {
        pa.mc = reinterpret_cast<uint32_t *>(p->nv.mc_va);
        pa.uc = reinterpret_cast<uint32_t *>(p->nv.uc_va);
    }
    for (int r = 0; r < p->nranks; r++) pa.bufs[r] = p->bufs[r];
    pa.ticket = p->local + kFlagsU32;
    pa.nranks = p->nranks;
    pa.rank = p->rank;
    pa.D = p->D;
    pa.slot_stride = slot_stride(p->D);
    pa.epoch = ++p->epoch;
    pa.divisor = divisor;
    static const uint64_t timeout_ns = [] {
        const char *e = std::getenv("KVQ_PEER_TIMEOUT_S");  // default 120 s
        const double sec = e ? std::atof(e) : 120.0;
        return (uint64_t)((sec > 0 ? sec : 120.0) * 1e9);
    }();
    pa.timeout_ns = timeout_ns;
    return pa;
}

namespace kvq {

int peer_nranks(kvq_peer_t p) { return p->nranks; }
int peer_rank(kvq_peer_t p) { return p->rank; }
bool peer_ready(kvq_peer_t p) { return p && p->open; }

kvq_status peer_allreduce_max_u32(kvq_peer_t p, uint32_t *buf, size_t count, cudaStream_t s) {
    if (!peer_ready(p)) return fail(KVQ_ERR_INVALID_VALUE, "peer exchange: kvq_peer_open was not called");
    if ((int64_t)count > p->D) return fail(KVQ_ERR_INVALID_VALUE, "peer exchange: count exceeds the peer's D");
    const PeerArgs pa = peer_args(p, 1.0f);
    peer_max_u32_kernel<<<1, kThreads, 0, s>>>(buf, (int64_t)count, pa);
    return check_launch("peer_max_u32");
}

kvq_status peer_allreduce_metrics(kvq_peer_t p, double *sums, size_t nsum, uint64_t *maxes, size_t nmax,
                                  cudaStream_t s) {
    if (!peer_ready(p)) return fail(KVQ_ERR_INVALID_VALUE, "peer exchange: kvq_peer_open was not called");
    if (nsum + nmax > (size_t)kMetSlotU64) return fail(KVQ_ERR_INVALID_VALUE, "peer exchange: too many metrics");
    const PeerArgs pa = peer_args(p, 1.0f);
    peer_metrics_kernel<<<1, 32, 0, s>>>(sums, (int)nsum, maxes, (int)nmax, pa);
    return check_launch("peer_metrics");
}

// a1 + a7 + a2 in one kernel; KVQ_ERR_UNSUPPORTED when the shape/alignment needs the generic path.
kvq_status peer_compute_scales(const float *K, int64_t T, int64_t D, float *scales, float divisor, kvq_peer_t p,
                               cudaStream_t s) {
    if (!peer_ready(p)) return fail(KVQ_ERR_INVALID_VALUE, "peer exchange: kvq_peer_open was not called");
    if (D != p->D || D % 4 || reinterpret_cast<uintptr_t>(K) % 16 || reinterpret_cast<uintptr_t>(scales) % 16)
        return KVQ_ERR_UNSUPPORTED;
    uint32_t *bits = reinterpret_cast<uint32_t *>(scales);
    if (cudaMemsetAsync(bits, 0, (size_t)D * 4, s) != cudaSuccess) return check_launch("memset scales");
    const PeerArgs pa = peer_args(p, divisor);
    const int64_t cols4 = D / 4, n4 = T * cols4;
    // one full wave of resident CTAs (the streaming loop is sized like colmax_v4_kernel's)
    const size_t smem = cols4 <= kThreads ? (size_t)4 * cols4 * sizeof(uint32_t) : 0;
    static const int resident = [] {
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, colmax_peer_kernel<8>, kThreads,
                                                          4 * kThreads * sizeof(uint32_t)) != cudaSuccess ||
            nb < 1) {
            cudaGetLastError();
            nb = 1;
        }
        return nb * kThreads;
    }();
    // an empty shard still takes part in the exchange: one CTA with no rows
    StreamPlan plan = n4 > 0 ? plan_stream(T, cols4, resident) : StreamPlan{0, 1};
    if (plan.blocks < 1) plan.blocks = 1;
    colmax_peer_kernel<8><<<plan.blocks, kThreads, smem, s>>>(reinterpret_cast<const float4 *>(K), n4, cols4, plan.G,
                                                           bits, pa);
    return check_launch("colmax_peer");
}

}  // namespace kvq

extern "C" kvq_status kvq_compute_scales_peer(const float *K, int64_t T, int64_t D, float *scales, kvq_peer_t p,
                                              void *stream) {
    KVQ_NVTX("kvq_compute_scales_peer");
    KVQ_REQUIRE((K || T == 0) && scales && p, "kvq_compute_scales_peer: NULL pointer");
    KVQ_REQUIRE(p->open, "kvq_compute_scales_peer: call kvq_peer_open first");
    KVQ_REQUIRE(D == p->D, "kvq_compute_scales_peer: D differs from kvq_peer_init");
    KVQ_REQUIRE(T >= 0 && (T == 0 || T <= (int64_t(1) << 62) / D), "kvq_compute_scales_peer: need 0 <= T, T*D <= 2^62");
    KVQ_REQUIRE(D % 4 == 0 && reinterpret_cast<uintptr_t>(K) % 16 == 0 &&
                    reinterpret_cast<uintptr_t>(scales) % 16 == 0,
                "kvq_compute_scales_peer: needs D % 4 == 0 and 16-byte aligned K, scales");
    KVQ_TRY(device_ok());
    return peer_compute_scales(K, T, D, scales, 127.0f, p, (cudaStream_t)stream);
}

// ============================================================================ NVLS (multicast) setup
// Driver entry points (cuMulticast*, cuMem*) resolved through the runtime: no -lcuda link.
namespace {
struct Drv {
    decltype(&cuDeviceGetAttribute) devAttr = nullptr;
    decltype(&cuDeviceGet) devGet = nullptr;
    decltype(&cuMulticastCreate) mcCreate = nullptr;
    decltype(&cuMulticastAddDevice) mcAdd = nullptr;
    decltype(&cuMulticastGetGranularity) mcGran = nullptr;
    decltype(&cuMulticastBindMem) mcBind = nullptr;
    decltype(&cuMulticastUnbind) mcUnbind = nullptr;
    decltype(&cuMemCreate) memCreate = nullptr;
    decltype(&cuMemGetAllocationGranularity) memGran = nullptr;
    decltype(&cuMemAddressReserve) vaReserve = nullptr;
    decltype(&cuMemAddressFree) vaFree = nullptr;
    decltype(&cuMemMap) map = nullptr;
    decltype(&cuMemUnmap) unmap = nullptr;
    decltype(&cuMemSetAccess) setAccess = nullptr;
    decltype(&cuMemRelease) release = nullptr;
    decltype(&cuMemExportToShareableHandle) exportH = nullptr;
    decltype(&cuMemImportFromShareableHandle) importH = nullptr;
    bool ok = false;
};
template <typename F>
bool sym(const char *name, F &f) {
    void *ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &ptr, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) {
        cudaGetLastError();
        return false;
    }
    f = reinterpret_cast<F>(ptr);
    return true;
}
const Drv &drv() {
    static Drv d;
    static std::once_flag once;
    std::call_once(once, [] {
        d.ok = sym("cuDeviceGetAttribute", d.devAttr) && sym("cuDeviceGet", d.devGet) &&
               sym("cuMulticastCreate", d.mcCreate) && sym("cuMulticastAddDevice", d.mcAdd) &&
               sym("cuMulticastGetGranularity", d.mcGran) && sym("cuMulticastBindMem", d.mcBind) &&
               sym("cuMulticastUnbind", d.mcUnbind) && sym("cuMemCreate", d.memCreate) &&
               sym("cuMemGetAllocationGranularity", d.memGran) && sym("cuMemAddressReserve", d.vaReserve) &&
               sym("cuMemAddressFree", d.vaFree) && sym("cuMemMap", d.map) && sym("cuMemUnmap", d.unmap) &&
               sym("cuMemSetAccess", d.setAccess) && sym("cuMemRelease", d.release) &&
               sym("cuMemExportToShareableHandle", d.exportH) &&
               sym("cuMemImportFromShareableHandle", d.importH);
    });
    return d;
}

// The 128-byte handle blob rank 0 broadcasts: the multicast object as a fabric handle, or (kind 2) the tag
// of the abstract unix socket on which rank 0's process hands out a POSIX file descriptor for it.
struct NvlsBlob {
    uint32_t magic, kind;
    uint64_t size, tag;
    uint32_t nranks, pad;
    unsigned char fabric[64];
    unsigned char rest[128 - 96];
};
static_assert(sizeof(NvlsBlob) == 128, "blob");
constexpr uint32_t kNvlsMagic = 0x4b56514eu;  // "KVQN"

std::string sock_name(uint64_t tag) { return "kvq-nvls-" + std::to_string(tag); }
int make_listen(uint64_t tag) {
    int fd = socket(AF_UNIX, SOCK_STREAM, 0);
    if (fd < 0) return -1;
    sockaddr_un a{};
    a.sun_family = AF_UNIX;
    const std::string n = sock_name(tag);
    std::memcpy(a.sun_path + 1, n.data(), n.size());  // abstract namespace (leading NUL)
    const socklen_t len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n.size());
    if (bind(fd, reinterpret_cast<sockaddr *>(&a), len) != 0 || listen(fd, kPeerMax) != 0) {
        close(fd);
        return -1;
    }
    return fd;
}
bool send_fd(int sock, int fd) {
    char dummy = 'k';
    iovec iov{&dummy, 1};
    char ctrl[CMSG_SPACE(sizeof(int))] = {};
    msghdr m{};
    m.msg_iov = &iov;
    m.msg_iovlen = 1;
    m.msg_control = ctrl;
    m.msg_controllen = sizeof(ctrl);
    cmsghdr *c = CMSG_FIRSTHDR(&m);
    c->cmsg_level = SOL_SOCKET;
    c->cmsg_type = SCM_RIGHTS;
    c->cmsg_len = CMSG_LEN(sizeof(int));
    std::memcpy(CMSG_DATA(c), &fd, sizeof(int));
    return sendmsg(sock, &m, 0) == 1;
}
int recv_fd(uint64_t tag) {
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {  // rank 0 is already listening when the blob is broadcast; retry briefly anyway
        int s = socket(AF_UNIX, SOCK_STREAM, 0);
        if (s < 0) return -1;
        sockaddr_un a{};
        a.sun_family = AF_UNIX;
        const std::string n = sock_name(tag);
        std::memcpy(a.sun_path + 1, n.data(), n.size());
        const socklen_t len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n.size());
        if (connect(s, reinterpret_cast<sockaddr *>(&a), len) == 0) {
            char dummy;
            iovec iov{&dummy, 1};
            char ctrl[CMSG_SPACE(sizeof(int))] = {};
            msghdr m{};
            m.msg_iov = &iov;
            m.msg_iovlen = 1;
            m.msg_control = ctrl;
            m.msg_controllen = sizeof(ctrl);
            int fd = -1;
            if (recvmsg(s, &m, 0) == 1) {
                cmsghdr *c = CMSG_FIRSTHDR(&m);
                if (c && c->cmsg_type == SCM_RIGHTS) std::memcpy(&fd, CMSG_DATA(c), sizeof(int));
            }
            close(s);
            return fd;
        }
        close(s);
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(20)) return -1;
        std::this_thread::sleep_for(std::chrono::milliseconds(20));
    }
}
}  // namespace

static void nvls_release(kvq_peer_t p) {
    const Drv &d = drv();
    auto &nv = p->nv;
    nv.active = false;
    if (nv.server.joinable()) {
        if (nv.listen_fd >= 0) shutdown(nv.listen_fd, SHUT_RDWR);
        nv.server.join();
    }
    if (nv.listen_fd >= 0) close(nv.listen_fd), nv.listen_fd = -1;
    if (nv.export_fd >= 0) close(nv.export_fd), nv.export_fd = -1;
    if (!d.ok) return;
    if (nv.mc_va) d.unmap(nv.mc_va, nv.bytes), d.vaFree(nv.mc_va, nv.bytes), nv.mc_va = 0;
    if (nv.uc_va) d.unmap(nv.uc_va, nv.bytes), d.vaFree(nv.uc_va, nv.bytes), nv.uc_va = 0;
    if (nv.mapped && nv.mc) {
        CUdevice dev;
        if (d.devGet(&dev, nv.device) == CUDA_SUCCESS) d.mcUnbind(nv.mc, dev, 0, nv.bytes);
    }
    if (nv.mem) d.release(nv.mem), nv.mem = 0;
    if (nv.mc) d.release(nv.mc), nv.mc = 0;
    nv.mapped = nv.joined = false;
}

static kvq_status nvls_fail(kvq_peer_t p, const std::string &msg, CUresult r) {
    nvls_release(p);
    return fail(KVQ_ERR_UNSUPPORTED, msg + " (CUresult " + std::to_string((int)r) + ")");
}

extern "C" size_t kvq_peer_nvls_handle_bytes(void) { return sizeof(NvlsBlob); }

extern "C" kvq_status kvq_peer_nvls_create(kvq_peer_t p, void *handle_out) {
    KVQ_NVTX("kvq_peer_nvls_create");
    KVQ_REQUIRE(p && handle_out, "kvq_peer_nvls_create: NULL pointer");
    KVQ_REQUIRE(p->open && !p->nv.joined, "kvq_peer_nvls_create: needs an open peer without NVLS");
    const Drv &d = drv();
    if (!d.ok) return fail(KVQ_ERR_UNSUPPORTED, "kvq_peer_nvls_create: driver lacks the multicast API");
    CUdevice dev;
    int sup = 0;
    CUresult r = d.devGet(&dev, p->device);
    if (r == CUDA_SUCCESS) r = d.devAttr(&sup, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
    if (r != CUDA_SUCCESS || !sup) return fail(KVQ_ERR_UNSUPPORTED, "kvq_peer_nvls_create: device has no multicast support");
    CUmulticastObjectProp prop{};
    prop.numDevices = (unsigned)p->nranks;
    prop.size = (size_t)2 * slot_stride(p->D) * 4;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR | (p->nranks > 1 ? CU_MEM_HANDLE_TYPE_FABRIC : 0);
    size_t g = 0;
    if ((r = d.mcGran(&g, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED)) != CUDA_SUCCESS || g == 0)
        return nvls_fail(p, "cuMulticastGetGranularity", r);
    prop.size = (prop.size + g - 1) / g * g;
    if ((r = d.mcCreate(&p->nv.mc, &prop)) != CUDA_SUCCESS) {
        prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;  // no fabric handles here: fd only
        if ((r = d.mcCreate(&p->nv.mc, &prop)) != CUDA_SUCCESS) return nvls_fail(p, "cuMulticastCreate", r);
    }
    p->nv.bytes = prop.size;
    NvlsBlob b{};
    b.magic = kNvlsMagic;
    b.size = prop.size;
    b.nranks = (uint32_t)p->nranks;
    CUmemFabricHandle fh;
    if (p->nranks > 1 && (prop.handleTypes & CU_MEM_HANDLE_TYPE_FABRIC) &&
        d.exportH(&fh, p->nv.mc, CU_MEM_HANDLE_TYPE_FABRIC, 0) == CUDA_SUCCESS) {
        b.kind = 1;
        std::memcpy(b.fabric, &fh, sizeof(fh));
    } else if (p->nranks > 1) {
        int fd = -1;
        if ((r = d.exportH(&fd, p->nv.mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0)) != CUDA_SUCCESS)
            return nvls_fail(p, "cuMemExportToShareableHandle(fd)", r);
        p->nv.export_fd = fd;
        b.kind = 2;
        b.tag = std::random_device{}() ^ ((uint64_t)getpid() << 20) ^ ((uint64_t)std::random_device{}() << 32);
        p->nv.listen_fd = make_listen(b.tag);
        if (p->nv.listen_fd < 0) return nvls_fail(p, "abstract unix socket", CUDA_ERROR_UNKNOWN);
        const int lfd = p->nv.listen_fd, efd = fd, n = p->nranks - 1;
        p->nv.server = std::thread([lfd, efd, n] {
            for (int k = 0; k < n; k++) {
                const int c = accept(lfd, nullptr, nullptr);
                if (c < 0) return;
                send_fd(c, efd);
                close(c);
            }
        });
    } else {
        b.kind = 0;  // one rank: nothing to share
    }
    std::memcpy(handle_out, &b, sizeof(b));
    return KVQ_OK;
}

extern "C" kvq_status kvq_peer_nvls_join(kvq_peer_t p, const void *handle) {
    KVQ_NVTX("kvq_peer_nvls_join");
    KVQ_REQUIRE(p && handle, "kvq_peer_nvls_join: NULL pointer");
    KVQ_REQUIRE(p->open && !p->nv.joined, "kvq_peer_nvls_join: needs an open peer without NVLS");
    NvlsBlob b;
    std::memcpy(&b, handle, sizeof(b));
    KVQ_REQUIRE(b.magic == kNvlsMagic && b.nranks == (uint32_t)p->nranks, "kvq_peer_nvls_join: foreign handle");
    const Drv &d = drv();
    if (!d.ok) return fail(KVQ_ERR_UNSUPPORTED, "kvq_peer_nvls_join: driver lacks the multicast API");
    CUresult r;
    if (p->rank != 0) {
        if (b.kind == 1) {
            CUmemFabricHandle fh;
            std::memcpy(&fh, b.fabric, sizeof(fh));
            if ((r = d.importH(&p->nv.mc, &fh, CU_MEM_HANDLE_TYPE_FABRIC)) != CUDA_SUCCESS)
                return nvls_fail(p, "cuMemImportFromShareableHandle(fabric)", r);
        } else if (b.kind == 2) {
            const int fd = recv_fd(b.tag);
            if (fd < 0) return nvls_fail(p, "receiving the multicast fd", CUDA_ERROR_UNKNOWN);
            r = d.importH(&p->nv.mc, reinterpret_cast<void *>((uintptr_t)fd), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
            close(fd);
            if (r != CUDA_SUCCESS) return nvls_fail(p, "cuMemImportFromShareableHandle(fd)", r);
        } else {
            return fail(KVQ_ERR_INVALID_VALUE, "kvq_peer_nvls_join: handle kind");
        }
        p->nv.bytes = b.size;
    }
    CUdevice dev;
    if ((r = d.devGet(&dev, p->device)) != CUDA_SUCCESS) return nvls_fail(p, "cuDeviceGet", r);
    if ((r = d.mcAdd(p->nv.mc, dev)) != CUDA_SUCCESS) return nvls_fail(p, "cuMulticastAddDevice", r);
    p->nv.device = p->device;
    p->nv.joined = true;
    return KVQ_OK;
}

// Every rank, once every rank has joined (binding and mapping block until all devices are added).
extern "C" kvq_status kvq_peer_nvls_map(kvq_peer_t p) {
    KVQ_NVTX("kvq_peer_nvls_map");
    KVQ_REQUIRE(p && p->nv.joined && !p->nv.mapped, "kvq_peer_nvls_map: call kvq_peer_nvls_join first");
    const Drv &d = drv();
    auto &nv = p->nv;
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = nv.device;
    size_t g = 0;
    CUresult r = d.memGran(&g, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
    if (r != CUDA_SUCCESS || g == 0 || nv.bytes % g) return nvls_fail(p, "cuMemGetAllocationGranularity", r);
    if ((r = d.memCreate(&nv.mem, nv.bytes, &ap, 0)) != CUDA_SUCCESS) return nvls_fail(p, "cuMemCreate", r);
    if ((r = d.mcBind(nv.mc, 0, nv.mem, 0, nv.bytes, 0)) != CUDA_SUCCESS) return nvls_fail(p, "cuMulticastBindMem", r);
    nv.mapped = true;
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = nv.device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CUdeviceptr va = 0;
    if ((r = d.vaReserve(&va, nv.bytes, g, 0, 0)) != CUDA_SUCCESS) return nvls_fail(p, "cuMemAddressReserve(mc)", r);
    if ((r = d.map(va, nv.bytes, 0, nv.mc, 0)) != CUDA_SUCCESS) {
        d.vaFree(va, nv.bytes);
        return nvls_fail(p, "cuMemMap(mc)", r);
    }
    nv.mc_va = va;
    if ((r = d.setAccess(va, nv.bytes, &acc, 1)) != CUDA_SUCCESS) return nvls_fail(p, "cuMemSetAccess(mc)", r);
    va = 0;
    if ((r = d.vaReserve(&va, nv.bytes, g, 0, 0)) != CUDA_SUCCESS) return nvls_fail(p, "cuMemAddressReserve(uc)", r);
    if ((r = d.map(va, nv.bytes, 0, nv.mem, 0)) != CUDA_SUCCESS) {
        d.vaFree(va, nv.bytes);
        return nvls_fail(p, "cuMemMap(uc)", r);
    }
    nv.uc_va = va;
    if ((r = d.setAccess(va, nv.bytes, &acc, 1)) != CUDA_SUCCESS) return nvls_fail(p, "cuMemSetAccess(uc)", r);
    if (cudaMemset(reinterpret_cast<void *>(nv.uc_va), 0, nv.bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
        cudaGetLastError();
        return nvls_fail(p, "zeroing the multicast slots", CUDA_ERROR_UNKNOWN);
    }
    return KVQ_OK;
}

// Every rank, once every rank has mapped: on != 0 routes the a7 exchange through multimem.ld_reduce;
// on == 0 releases the multicast resources (the P2P slots take over).
extern "C" kvq_status kvq_peer_nvls_enable(kvq_peer_t p, int on) {
    KVQ_NVTX("kvq_peer_nvls_enable");
    KVQ_REQUIRE(p, "kvq_peer_nvls_enable: NULL pointer");
    if (!on) {
        cudaDeviceSynchronize();
        nvls_release(p);
        return KVQ_OK;
    }
    KVQ_REQUIRE(p->nv.mapped && p->nv.mc_va && p->nv.uc_va, "kvq_peer_nvls_enable: call kvq_peer_nvls_map first");
    p->nv.active = true;
    return KVQ_OK;
}

extern "C" int kvq_peer_nvls_active(kvq_peer_t p) { return p && p->nv.active ? 1 : 0; }
