// In-run L2 roofline probes: the hash gather/scatter is bounded by L2,
// whose bandwidth is not in MEASURED_PEAKS.json, so bench.py measures it in the same
// job with two kernels over a buffer the size of the real working set:
//   * a 16-B-vector read sweep, repeated so the buffer stays L2-resident;
//   * random-address float2 REDs (RED.E.ADD.F32x2), the scatter's instruction.
#include "common.cuh"

namespace ns2b {

__global__ void l2_read_kernel(const float4 *__restrict__ buf, int64_t n4, int iters,
                               float *__restrict__ sink) {
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
             i += (int64_t)gridDim.x * blockDim.x) {
            float4 v = __ldcg(buf + i);  // cache-global: bypass L1, hit L2
            acc += v.x + v.y + v.z + v.w;
        }
    }
    if (acc == 123456.f) sink[0] = acc;  // keep the loads alive
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

__global__ void red_kernel(float *__restrict__ buf, uint32_t nrows, int64_t nops, uint32_t seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nops;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t r = hash32(static_cast<uint32_t>(i) ^ seed) % nrows;
        red_add_f32x2(buf + 2 * static_cast<int64_t>(r), 1e-9f, 1e-9f);
    }
}

}  // namespace ns2b

using namespace ns2b;

extern "C" {

int ns2b_bench_l2_read(const float *buf, int64_t nfloats, int32_t iters, float *sink, void *stream) {
    NS2B_REQUIRE(nfloats % 4 == 0 && iters >= 1, "bench_l2_read: nfloats % 4 == 0, iters >= 1");
    l2_read_kernel<<<kNumSMs * 8, 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const float4 *>(buf), nfloats / 4, iters, sink);
    return check_launch("bench_l2_read");
}

int ns2b_bench_red(float *buf, int64_t nrows, int64_t nops, uint32_t seed, void *stream) {
    NS2B_REQUIRE(nrows >= 1 && nrows < (1ll << 32), "bench_red: row count");
    red_kernel<<<kNumSMs * 8, 256, 0, as_stream(stream)>>>(buf, static_cast<uint32_t>(nrows), nops,
                                                           seed);
    return check_launch("bench_red");
}

}  // extern "C"
