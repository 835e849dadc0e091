// synth.cu — device implementation of the seeded input generator
// (include/kvq_synth.h).  Input generation only: none of
// the method's arithmetic lives here.  The CPU oracle has its own independent
// implementation; both are pinned to the same test vector.
#include "../../include/kvq_synth.h"
#include "kvq_internal.h"

namespace kvq {

__device__ __forceinline__ uint64_t splitmix64(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1ull) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ float lattice_uniform(uint64_t seed, uint64_t i) {
    int32_t k = (int32_t)(splitmix64(seed, i) >> 40) - (int32_t)(1 << 23);
    return __fmul_rn((float)k, 0x1p-23f);  // exact
}

__global__ void synth_kernel(float *__restrict__ out, int64_t row0, int64_t n, int64_t D, uint64_t seed,
                             int dist) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        const int64_t r = j / D, d = j - r * D;
        const int64_t t = row0 + r;
        const uint64_t gi = (uint64_t)t * (uint64_t)D + (uint64_t)d;
        float v;
        if (dist == KVQ_DIST_OUTLIER) {
            int e = (int)(splitmix64(seed ^ 0xC0FFEEull, (uint64_t)d) % 9ull) - 4;
            v = ldexpf(lattice_uniform(seed, gi), e);
        } else if (dist == KVQ_DIST_ONGRID) {
            uint64_t jd = (splitmix64(seed ^ 0x5CA1Eull, (uint64_t)d) >> 47) | 1ull;
            float s = __fmul_rn((float)jd, 0x1p-24f);
            int c;
            if (t == 0)
                c = (splitmix64(seed ^ 0x516Eull, (uint64_t)d) & 1ull) ? 127 : -127;
            else
                c = (int)(splitmix64(seed, gi) % 255ull) - 127;
            v = __fmul_rn((float)c, s);
        } else {
            v = lattice_uniform(seed, gi);
        }
        out[j] = v;
    }
}

}  // namespace kvq

extern "C" kvq_status kvq_synth_fill(float *out, int64_t row0, int64_t rows, int64_t D, uint64_t seed, int dist,
                                     void *stream) {
    KVQ_NVTX("kvq_synth_fill");
    using namespace kvq;
    if (!out || rows < 1 || D < 1 || row0 < 0 || dist < 0 || dist > 2)
        return fail(KVQ_ERR_INVALID_VALUE, "kvq_synth_fill: invalid argument");
    if (rows > (int64_t(1) << 62) / D) return fail(KVQ_ERR_INVALID_VALUE, "kvq_synth_fill: rows*D too large");
    if (kvq_status st = device_ok(); st != KVQ_OK) return st;
    const int64_t n = rows * D;
    const DeviceInfo &di = device_info();
    int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)di.num_sms * 16);
    synth_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(out, row0, n, D, seed, dist);
    return check_launch("synth_fill");
}
