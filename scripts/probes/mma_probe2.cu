// tcgen05.mma kind::tf32 throughput per SM for the roundtrip's contraction shapes:
// A from TMEM (.ts) vs smem (.ss), B SWIZZLE_128B vs SWIZZLE_NONE canonical layout,
// M = 128, N = 64 / 128 / 256, K = 8 per instruction; back to back, one CTA per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint64_t desc_none(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
    return pred;
}

// V: 0 = SS sw128/sw128, 1 = TS + B sw128, 2 = TS + B none (lbo 1024 sbo 128, the kernel's Q layout),
//    3 = SS with B none
template <int N, int V>
__global__ void __launch_bounds__(128, 1) probe(int iters, long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3f800000u;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t d = tbase, at = tbase + 256;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t a = desc_sw128(smem_u32(sm));
    const uint64_t b = (V == 2 || V == 3) ? desc_none(smem_u32(sm + 64 * 1024), 1024, 128) : desc_sw128(smem_u32(sm + 64 * 1024));
    long long t0 = 0, t1 = 0;
    if (warp == 0) {
        if (elect_one()) {
            t0 = clock64();
            for (int it = 0; it < iters; it++) {
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const uint64_t boff = (V == 2 || V == 3) ? (uint64_t)(j * 128) : (uint64_t)(2 * j);
                    if (V == 1 || V == 2)
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                                     "r"(at + 8 * j), "l"(b + boff), "r"(idesc), "r"(1));
                    else
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                                     "l"(a + 2 * j), "l"(b + boff), "r"(idesc), "r"(1));
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
            asm volatile("{\n\t.reg .pred P1;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(smem_u32(&bar)));
            t1 = clock64();
            if (blockIdx.x == 0) out[0] = t1 - t0;
        }
        __syncwarp();
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(d));
}

template <int N, int V>
void run(const char *name) {
    long long *o;
    cudaMalloc(&o, 8);
    cudaFuncSetAttribute(probe<N, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    const int iters = 4096;
    probe<N, V><<<148, 128, 160 * 1024>>>(iters, o);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<N, V><<<148, 128, 160 * 1024>>>(iters, o);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long cyc;
    cudaMemcpy(&cyc, o, 8, cudaMemcpyDeviceToHost);
    const double macs = 128.0 * N * 8 * 4 * iters * 148;
    printf("%-28s N=%3d: %6.1f cyc/MMA  %5.0f TFLOPS tf32  err=%s\n", name, N, (double)cyc / (4.0 * iters),
           2 * macs / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    run<64, 0>("SS  A sw128 B sw128");
    run<128, 0>("SS  A sw128 B sw128");
    run<256, 0>("SS  A sw128 B sw128");
    run<64, 1>("TS  A tmem  B sw128");
    run<128, 1>("TS  A tmem  B sw128");
    run<256, 1>("TS  A tmem  B sw128");
    run<64, 2>("TS  A tmem  B none (kernel)");
    run<128, 2>("TS  A tmem  B none");
    run<64, 3>("SS  A sw128 B none");
    return 0;
}
