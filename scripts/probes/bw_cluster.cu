// HBM write-pattern probe (no arithmetic), C4 size: the roundtrip's traffic (read K 4 B/elem, write K_hat 4 +
// codes 1 B/elem) in [128 x 32] fp32 TMA boxes, with G CTAs of a thread-block cluster sharing one 128-row tile:
// CTA j of the cluster takes K-blocks kb = k G + j, and the store warps of the cluster move in LOCKSTEP (a
// cluster-wide barrier of mbarriers, one remote arrival per CTA per step), so at any moment the cluster writes G
// adjacent 128-byte pieces of each of its 128 rows (G x 128 B contiguous per row).  Question: does keeping the
// pieces adjacent in time move the write-pattern floor (1.72 ms for whole tiles per CTA, 1.40 ms linear)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2601_04719_b200/csrc bw_cluster.cu
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

template <int G, int LOCK>
__global__ void __launch_bounds__(64, 1) tile_clu(const __grid_constant__ CUtensorMap mi,
                                                  const __grid_constant__ CUtensorMap mo,
                                                  const __grid_constant__ CUtensorMap mc, int ntiles, int nkb) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + ST * BOX + 16384);
    uint64_t *empty = full + ST;
    uint64_t *stepb = empty + ST;  // [2] cluster lockstep barriers (count G), double-buffered by step parity
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int j = G > 1 ? (int)cluster_rank() : 0;
    const int c = blockIdx.x / G, nclu = gridDim.x / G;
    if (threadIdx.x == 0) {
        for (int i = 0; i < ST; i++) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(&stepb[0], G);
        mbar_init(&stepb[1], G);
        mbar_fence_init();
    }
    if (G > 1) cluster_sync(); else __syncthreads();
    const uint64_t pin = policy_evict_first(), pout = policy_evict_first();
    const int my_kb = nkb / G;
    if (warp == 0 && lane == 0) {
        uint32_t g = 0;
        for (int tile = c; tile < ntiles; tile += nclu)
            for (int k = 0; k < my_kb; k++, g++) {
                const int kb = k * G + j;
                const int sk = g % ST;
                mbar_wait(&empty[sk], ((g / ST) & 1) ^ 1);
                mbar_arrive_tx(&full[sk], BOX);
                tma_load_2d(sm + sk * BOX, &mi, &full[sk], kb * 32, tile * 128, pin);
            }
    } else if (warp == 1 && lane == 0) {
        uint32_t g = 0;
        for (int tile = c; tile < ntiles; tile += nclu)
            for (int k = 0; k < my_kb; k++, g++) {
                const int kb = k * G + j;
                const int sk = g % ST;
                mbar_wait(&full[sk], (g / ST) & 1);
                if (G > 1 && LOCK) {  // lockstep: every CTA of the cluster has block g loaded before anyone stores it
                    const uint32_t mine = smem_u32(&stepb[g & 1]);
                    for (int r = 0; r < G; r++) mbar_arrive_cluster(mapa(mine, (uint32_t)r));
                    mbar_wait(&stepb[g & 1], (g >> 1) & 1);
                }
                tma_store_2d(&mo, sm + sk * BOX, kb * 32, tile * 128, pout);
                tma_store_2d(&mc, sm + ST * BOX, kb * 32, tile * 128, pout);  // 32 codes per row
                bulk_commit();
                if (g > 0) {
                    bulk_wait_read<1>();
                    mbar_arrive(&empty[(g - 1) % ST]);
                }
            }
        bulk_wait<0>();
    }
    __syncwarp();
    if (G > 1) cluster_sync();  // no CTA exits while a peer may still arrive on its barriers
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
static CUtensorMap map2d(void *base, CUtensorMapDataType ty, int elem, int box_cols, bool swz) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)T};
    cuuint64_t strides[1] = {(cuuint64_t)D * elem};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, 128u};
    cuuint32_t estr[2] = {1, 1};
    enc()(&m, ty, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
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
    const cudaError_t e = cudaGetLastError();
    printf("%-36s best %.3f ms  med %.3f ms  %6.0f GB/s (med) %s\n", name, ts[0], ts[ts.size() / 2],
           9.0 * N / (ts[ts.size() / 2] * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

template <int G, int LOCK>
static void run(const char *name, const CUtensorMap &mi, const CUtensorMap &mo, const CUtensorMap &mc, int sms) {
    const size_t smem = ST * BOX + 16384 + 1024;
    cudaFuncSetAttribute(tile_clu<G, LOCK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (G > 1) cudaFuncSetAttribute(tile_clu<G, LOCK>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int grid = (sms / G) * G;
    if (G > 1) {  // as many whole clusters as can be co-resident
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(64);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = G;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = 0;
        cudaOccupancyMaxActiveClusters(&ncl, (void *)tile_clu<G, LOCK>, &cfg);
        if (ncl > 0) grid = std::min(grid, ncl * G);
        cfg.gridDim = dim3(grid);
        printf("G=%d: %d clusters co-resident -> grid %d\n", G, ncl, grid);
        timeit(name, [&] {
            cudaLaunchKernelEx(&cfg, tile_clu<G, LOCK>, mi, mo, mc, (int)(T / 128), (int)(D / 32));
        });
    } else {
        timeit(name, [&] { tile_clu<G, LOCK><<<grid, 64, smem>>>(mi, mo, mc, (int)(T / 128), (int)(D / 32)); });
    }
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *in, *ok;
    uint8_t *oc;
    cudaMalloc(&in, N * 4);
    cudaMalloc(&ok, N * 4);
    cudaMalloc(&oc, N);
    cudaMemset(in, 0, N * 4);
    CUtensorMap mi = map2d(in, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 32, true);
    CUtensorMap mo = map2d(ok, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 32, true);
    CUtensorMap mc = map2d(oc, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, 32, false);
    run<1, 0>("G1  (whole tile per CTA)", mi, mo, mc, sms);
    run<2, 0>("G2  free-running", mi, mo, mc, sms);
    run<2, 1>("G2  lockstep", mi, mo, mc, sms);
    run<4, 0>("G4  free-running", mi, mo, mc, sms);
    run<4, 1>("G4  lockstep", mi, mo, mc, sms);
    run<8, 0>("G8  free-running", mi, mo, mc, sms);
    run<8, 1>("G8  lockstep", mi, mo, mc, sms);
    run<16, 1>("G16 lockstep", mi, mo, mc, sms);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
