// Microbenchmark: back-to-back tcgen05.mma throughput per SM (one CTA per SM,
// operands resident in smem, no barriers in the loop).  Prints cycles/MMA for
// kind::i8 / kind::f16, SS operands, cta_group::1, M=128, several N.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
    return pred;
}

template <int KIND, int N, int VAR>
__global__ void __launch_bounds__(128, 1) probe(int iters, long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar, bar2[2], bar3;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x01010101u * (i & 3);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2[1])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar3)));
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar3)));  // phase 0 complete
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
    const uint32_t d = tbase;
    // kind::i8: D s32, A/B s8; kind::f16: D f32, A/B bf16
    const uint32_t idesc = (KIND == 0 ? (2u << 4) | (1u << 7) | (1u << 10) : (1u << 4) | (1u << 7) | (1u << 10)) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t a = desc_sw128(smem_u32(sm)), b = desc_sw128(smem_u32(sm + 64 * 1024));  // A: 64 KB, B: 96 KB
    long long t0 = 0, t1 = 0;
    if (warp == 0) {
        if (elect_one()) {
            t0 = clock64();
            for (int it = 0; it < iters; it++) {
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const uint64_t ao = (VAR & 8) ? (uint64_t)((it % 4) * 1024) : 0;   // 16 KB stages, 4 of them
                    const uint64_t bo = (VAR & 8) ? (uint64_t)((it % 3) * 2048) : 0;   // 32 KB stages, 3 of them
                    if (KIND == 0)
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                                     "l"(a + ao + 2 * j), "l"(b + bo + 2 * j), "r"(idesc), "r"(1));
                    else
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                                     "l"(a + 2 * j), "l"(b + 2 * j), "r"(idesc), "r"(1));
                }
                if (VAR & 1)  // commit per K-block
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2[it & 1])));
                if (VAR & 2)  // second commit
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2[(it + 1) & 1])));
                if (VAR & 4) {  // try_wait on an already-complete barrier + fence
                    asm volatile("{\n\t.reg .pred P1;\n\tW2: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W2;\n\t}" ::"r"(smem_u32(&bar3)));
                    asm volatile("tcgen05.fence::after_thread_sync;");
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

template <int KIND, int N, int VAR = 0>
void run(const char *name) {
    long long *o;
    cudaMalloc(&o, 8);
    cudaFuncSetAttribute(probe<KIND, N, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    const int iters = 4096;
    for (int grid : {1, 148}) {
        probe<KIND, N, VAR><<<grid, 128, 160 * 1024>>>(iters, o);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        probe<KIND, N, VAR><<<grid, 128, 160 * 1024>>>(iters, o);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        long long cyc;
        cudaMemcpy(&cyc, o, 8, cudaMemcpyDeviceToHost);
        const double macs = 128.0 * N * (KIND == 0 ? 32 : 16) * 4 * iters * grid;
        printf("var%d %-10s N=%3d grid=%3d: %.1f cyc/MMA  (%.0f T MAC-ops/s x2 = %.0f TOPS)  err=%s\n", VAR, name, N, grid,
               (double)cyc / (4.0 * iters), macs / (ms * 1e-3) / 1e12, 2 * macs / (ms * 1e-3) / 1e12,
               cudaGetErrorString(cudaGetLastError()));
    }
}

int main() {
    run<0, 256, 0>("i8");
    run<0, 256, 8>("i8");
    run<0, 128, 8>("i8");
    run<1, 256, 8>("bf16");
    return 0;
}
