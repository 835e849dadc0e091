// HBM ceiling for the roundtrip's traffic mix: read 4 B/elem, write 4 B (+1 B) /elem.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int WK, int WC>  // write K_hat?  write codes (bytes per elem x4)?
__global__ void __launch_bounds__(256) mix(const float4 *__restrict__ in, float4 *__restrict__ outk,
                                           uint32_t *__restrict__ outc, int64_t n4) {
    const int64_t G = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += 4 * G) {
        float4 v[4];
#pragma unroll
        for (int k = 0; k < 4; k++)
            if (i + k * G < n4)
                asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                             : "=f"(v[k].x), "=f"(v[k].y), "=f"(v[k].z), "=f"(v[k].w) : "l"(in + i + k * G));
#pragma unroll
        for (int k = 0; k < 4; k++)
            if (i + k * G < n4) {
                if (WK) asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(outk + i + k * G), "f"(v[k].x),
                                     "f"(v[k].y), "f"(v[k].z), "f"(v[k].w) : "memory");
                if (WC) asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(outc + i + k * G),
                                     "r"(__float_as_uint(v[k].x) ^ __float_as_uint(v[k].w)) : "memory");
                if (!WK && !WC && v[k].x == 1.2345f) outc[0] = 1;
            }
    }
}

template <int WK, int WC>
void run(const char *name, const float4 *in, float4 *ok, uint32_t *oc, int64_t n4, double bpe) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, mix<WK, WC>, 256, 0);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * nb;
    for (int w = 0; w < 3; w++) mix<WK, WC><<<grid, 256>>>(in, ok, oc, n4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9;
    for (int r = 0; r < 10; r++) {
        cudaEventRecord(a);
        mix<WK, WC><<<grid, 256>>>(in, ok, oc, n4);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    printf("%-22s %.3f ms  %.0f GB/s (%.1f B/elem)\n", name, best, bpe * n4 * 4 / (best * 1e-3) / 1e9, bpe);
}

int main() {
    const int64_t n = 131072LL * 8192, n4 = n / 4;
    float4 *in, *ok;
    uint32_t *oc;
    cudaMalloc(&in, n * 4);
    cudaMalloc(&ok, n * 4);
    cudaMalloc(&oc, n);
    cudaMemset(in, 0, n * 4);
    run<0, 0>("read only", in, ok, oc, n4, 4);
    run<1, 0>("R4 W4 (copy)", in, ok, oc, n4, 8);
    run<0, 1>("R4 W1", in, ok, oc, n4, 5);
    run<1, 1>("R4 W4+1 (roundtrip)", in, ok, oc, n4, 9);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
