// HBM probe: does writing each row's K_hat as a 1 KB BURST (8 consecutive 128 B pieces from one thread, from
// registers) instead of one 128 B piece per K-block (~1 us apart, the roundtrip kernel's TMA box stores)
// recover the linear-stream write bandwidth for a 128-row tile?
// Traffic of the roundtrip at C4: read K (TMA [128 x 32] fp32 boxes, 8-stage ring), write K_hat 4 B/elem and
// codes 1 B/elem ([128 x 128 B] TMA box per 4 K-blocks).  No arithmetic.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2601_04719_b200/csrc bw_burst.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

using namespace kvq::tc;

static const int64_t T = 131072, D = 8192, N = T * D;
constexpr int ST = 8;
constexpr uint32_t BOX = 128u * 32 * 4;

// GW = K-blocks per burst group (1 = the roundtrip's pattern through registers, 8 = 1 KB bursts)
template <int GW, int STORE_TMA>
__global__ void __launch_bounds__(192, 1) burst(const __grid_constant__ CUtensorMap mi,
                                                const __grid_constant__ CUtensorMap mo,
                                                const __grid_constant__ CUtensorMap mc, float *out, int ntiles,
                                                int nkb) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + ST * BOX + 16384);
    uint64_t *empty = full + ST;
    uint64_t *grp = empty + ST;  // [2] group progress (consumer -> store warps)
    uint64_t *grp_free = grp + 2;  // [2] store warps -> consumer
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < ST; i++) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(&grp[0], 1);
        mbar_init(&grp[1], 1);
        mbar_init(&grp_free[0], 4);
        mbar_init(&grp_free[1], 4);
        mbar_fence_init();
    }
    __syncthreads();
    const uint64_t pol = policy_evict_first();
    const int ngrp = nkb / GW;
    if (warp == 0 && lane == 0) {
        uint32_t g = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
            for (int kb = 0; kb < nkb; kb++, g++) {
                const int sk = g % ST;
                mbar_wait(&empty[sk], ((g / ST) & 1) ^ 1);
                mbar_arrive_tx(&full[sk], BOX);
                tma_load_2d(sm + sk * BOX, &mi, &full[sk], kb * 32, tile * 128, pol);
            }
    } else if (warp == 1 && lane == 0) {
        // consumer: frees stages as they land (the converters' read), reports group progress, stores codes
        uint32_t g = 0, gg = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
            for (int kb = 0; kb < nkb; kb++, g++) {
                const int sk = g % ST;
                mbar_wait(&full[sk], (g / ST) & 1);
                if (STORE_TMA) tma_store_2d(&mo, sm + sk * BOX, kb * 32, tile * 128, pol);
                if ((kb & 3) == 3) tma_store_2d(&mc, sm + ST * BOX, (kb / 4) * 128, tile * 128, pol);
                bulk_commit();
                bulk_wait_read<0>();
                mbar_arrive(&empty[sk]);
                if (!STORE_TMA && (kb % GW) == GW - 1) {
                    mbar_wait(&grp_free[gg & 1], ((gg >> 1) & 1) ^ 1);
                    mbar_arrive(&grp[gg & 1]);
                    gg++;
                }
            }
        bulk_wait<0>();
    } else if (warp >= 2 && !STORE_TMA) {
        // 4 store warps: thread = row (warp quarter q covers rows 32q..32q+31); per group, each thread writes its
        // row's GW x 128 B back to back (16-byte stores from registers)
        const int q = warp - 2, r = 32 * q + lane;
        uint32_t gg = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
            for (int G = 0; G < ngrp; G++, gg++) {
                mbar_wait_sleep(&grp[gg & 1], (gg >> 1) & 1);
                float4 *row = reinterpret_cast<float4 *>(out + ((int64_t)tile * 128 + r) * D + (int64_t)G * GW * 32);
#pragma unroll 8
                for (int c = 0; c < GW * 8; c++) __stcs(row + c, make_float4(1.f, 2.f, 3.f, (float)c));
                __syncwarp();
                if (lane == 0) mbar_arrive(&grp_free[gg & 1]);
            }
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *ptr = nullptr;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}
static CUtensorMap map2d(void *base, CUtensorMapDataType ty, int elem, int box_cols) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)T};
    cuuint64_t strides[1] = {(cuuint64_t)D * elem};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, 128};
    cuuint32_t estr[2] = {1, 1};
    enc()(&m, ty, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return m;
}

template <typename F>
static void timeit(const char *name, F launch) {
    for (int w = 0; w < 3; w++) launch();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    std::vector<float> ts;
    for (int r = 0; r < 10; r++) {
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    printf("%-44s best %.3f ms  med %.3f ms  %5.0f GB/s (9 B/elem, best)  %s\n", name, ts[0], ts[5],
           9.0 * N / (ts[0] * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *in, *out;
    uint8_t *oc;
    cudaMalloc(&in, N * 4);
    cudaMalloc(&out, N * 4);
    cudaMalloc(&oc, N);
    cudaMemset(in, 0, N * 4);
    CUtensorMap mi = map2d(in, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 32);
    CUtensorMap mo = map2d(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 32);
    CUtensorMap mc = map2d(oc, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, 128);
    const size_t smem = ST * BOX + 16384 + 1024;
    const int ntiles = (int)(T / 128), nkb = (int)(D / 32);
#define RUN(GW, TMA, name)                                                                                 \
    cudaFuncSetAttribute(burst<GW, TMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);         \
    timeit(name, [&] { burst<GW, TMA><<<sms, 192, smem>>>(mi, mo, mc, out, ntiles, nkb); });
    RUN(1, 1, "TMA box store per K-block (roundtrip pattern)");
    RUN(1, 0, "register stores, 128 B per row per K-block");
    RUN(2, 0, "register stores, 256 B bursts per row");
    RUN(4, 0, "register stores, 512 B bursts per row");
    RUN(8, 0, "register stores, 1 KB bursts per row");
    RUN(16, 0, "register stores, 2 KB bursts per row");
    RUN(32, 0, "register stores, 4 KB bursts per row");
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
