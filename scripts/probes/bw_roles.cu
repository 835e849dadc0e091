// HBM probe: does running the next batch's column-max read stream (R4) CONCURRENTLY
// with this batch's roundtrip traffic (R4 W5 in 128-row tiles) beat running them one
// after the other?  One kernel, two CTA roles split by SM: CTAs [0, NR) stream buffer B
// (1-D bulk loads, read only), CTAs [NR, 148) walk 128-row tiles of A with [128 x 32]
// fp32 TMA boxes (load K, store K_hat box + one [128 x 128 B] code box per 4 K-blocks),
// the roundtrip kernel's pattern.  No arithmetic.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2601_04719_b200/csrc bw_roles.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "tc_common.cuh"

using namespace kvq::tc;

static const int64_t T = 131072, D = 8192, N = T * D;
constexpr int ST = 8;
constexpr uint32_t BOX = 128u * 32 * 4;  // 16 KB
constexpr uint32_t RCH = 16384;          // read-role bulk chunk

__global__ void __launch_bounds__(64, 1) roles(const __grid_constant__ CUtensorMap mi,
                                               const __grid_constant__ CUtensorMap mo,
                                               const __grid_constant__ CUtensorMap mc, const uint8_t *inB,
                                               int NR, int tiles_lo, int tiles_hi, int64_t rch_lo, int64_t rch_hi) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + ST * BOX + 16384);
    uint64_t *empty = full + ST;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < ST; i++) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const uint64_t pol = policy_evict_first();
    const int nkb = (int)(D / 32);
    if ((int)blockIdx.x < NR) {
        // ---- read role: chunks rch_lo + blockIdx.x + i * NR
        if (warp == 0 && lane == 0) {
            uint32_t g = 0;
            for (int64_t c = rch_lo + blockIdx.x; c < rch_hi; c += NR, g++) {
                const int sk = g % ST;
                mbar_wait(&empty[sk], ((g / ST) & 1) ^ 1);
                mbar_arrive_tx(&full[sk], RCH);
                bulk_load(sm + sk * BOX, inB + c * RCH, RCH, &full[sk], pol);
            }
        } else if (warp == 1 && lane == 0) {
            uint32_t g = 0;
            for (int64_t c = rch_lo + blockIdx.x; c < rch_hi; c += NR, g++) {
                const int sk = g % ST;
                mbar_wait(&full[sk], (g / ST) & 1);
                mbar_arrive(&empty[sk]);
            }
        }
        return;
    }
    const int b = blockIdx.x - NR, nb = gridDim.x - NR;
    if (warp == 0 && lane == 0) {
        uint32_t g = 0;
        for (int tile = tiles_lo + b; tile < tiles_hi; tile += nb)
            for (int kb = 0; kb < nkb; kb++, g++) {
                const int sk = g % ST;
                mbar_wait(&empty[sk], ((g / ST) & 1) ^ 1);
                mbar_arrive_tx(&full[sk], BOX);
                tma_load_2d(sm + sk * BOX, &mi, &full[sk], kb * 32, tile * 128, pol);
            }
    } else if (warp == 1 && lane == 0) {
        uint32_t g = 0;
        for (int tile = tiles_lo + b; tile < tiles_hi; tile += nb)
            for (int kb = 0; kb < nkb; kb++, g++) {
                const int sk = g % ST;
                mbar_wait(&full[sk], (g / ST) & 1);
                tma_store_2d(&mo, sm + sk * BOX, kb * 32, tile * 128, pol);
                if ((kb & 3) == 3) tma_store_2d(&mc, sm + ST * BOX, (kb / 4) * 128, tile * 128, pol);
                bulk_commit();
                if (g > 0) {
                    bulk_wait_read<1>();
                    mbar_arrive(&empty[(g - 1) % ST]);
                }
            }
        bulk_wait<0>();
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
static float timeit(F launch) {
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
    return ts[ts.size() / 2];
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *A, *O, *B;
    uint8_t *C;
    cudaMalloc(&A, N * 4);
    cudaMalloc(&O, N * 4);
    cudaMalloc(&B, N * 4);
    cudaMalloc(&C, N);
    cudaMemset(A, 0, N * 4);
    cudaMemset(B, 0, N * 4);
    CUtensorMap mi = map2d(A, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 32);
    CUtensorMap mo = map2d(O, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 32);
    CUtensorMap mc = map2d(C, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, 128);
    const size_t smem = ST * BOX + 16384 + 1024;
    cudaFuncSetAttribute(roles, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int ntiles = (int)(T / 128);
    const int64_t nrch = N * 4 / RCH;
    const auto *Bb = reinterpret_cast<const uint8_t *>(B);
    const float t_tile = timeit([&] { roles<<<sms, 64, smem>>>(mi, mo, mc, Bb, 0, 0, ntiles, 0, 0); });
    const float t_read = timeit([&] { roles<<<sms, 64, smem>>>(mi, mo, mc, Bb, sms, 0, 0, 0, nrch); });
    printf("tile R4W5 alone (148 SMs): %.3f ms   read R4 alone (148 SMs): %.3f ms   sequential sum %.3f ms\n", t_tile,
           t_read, t_tile + t_read);
    for (int NR : {16, 24, 28, 32, 36, 40, 48}) {
        const float t = timeit([&] { roles<<<sms, 64, smem>>>(mi, mo, mc, Bb, NR, 0, ntiles, 0, nrch); });
        // each role alone at this split, to see which one set the combined time
        const float tt = timeit([&] { roles<<<sms, 64, smem>>>(mi, mo, mc, Bb, NR, 0, ntiles, 0, 0); });
        const float tr = timeit([&] { roles<<<sms, 64, smem>>>(mi, mo, mc, Bb, NR, 0, 0, 0, nrch); });
        printf("NR=%3d  combined %.3f ms (%.1f%% of sequential)   tile role alone %.3f   read role alone %.3f\n", NR, t,
               100.0 * t / (t_tile + t_read), tt, tr);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
