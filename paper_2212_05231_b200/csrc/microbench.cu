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

// Random 8-B gathers: the hash-grid gather's access pattern (one float2 row per lane,
// rows uniformly random over a table-sized buffer, 8 independent loads in flight per
// thread like one level's 8 corners).  Useful bytes = 8 per load.
__global__ void gather_kernel(const float2 *__restrict__ buf, uint32_t nrows, int64_t nloads, uint32_t seed,
                              float *__restrict__ sink) {
    float acc = 0.f;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 8; i < nloads; i += stride) {
        float2 v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = __ldg(buf + hash32(static_cast<uint32_t>(i + c) ^ seed) % nrows);
#pragma unroll
        for (int c = 0; c < 8; ++c) acc += v[c].x + v[c].y;
    }
    if (acc == 123456.f) sink[0] = acc;
}

// Coalesced float2 REDs (lane k of a warp adds to row base + k): the L2 atomic units'
// throughput with full sectors, the ceiling for the table scatter's REDs.
__global__ void red_coalesced_kernel(float *__restrict__ buf, uint32_t nrows, int64_t nops, uint32_t seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nops;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t warp_base = (hash32(static_cast<uint32_t>(i >> 5) ^ seed) % (nrows / 32)) * 32;
        red_add_f32x2(buf + 2 * static_cast<int64_t>(warp_base + (i & 31)), 1e-9f, 1e-9f);
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

int ns2b_bench_gather(const float *buf, int64_t nrows, int64_t nloads, uint32_t seed, float *sink, void *stream) {
    NS2B_REQUIRE(nrows >= 1 && nrows < (1ll << 32), "bench_gather: row count");
    gather_kernel<<<kNumSMs * 16, 128, 0, as_stream(stream)>>>(reinterpret_cast<const float2 *>(buf),
                                                               static_cast<uint32_t>(nrows), nloads, seed, sink);
    return check_launch("bench_gather");
}

int ns2b_bench_red_coalesced(float *buf, int64_t nrows, int64_t nops, uint32_t seed, void *stream) {
    NS2B_REQUIRE(nrows >= 32 && nrows < (1ll << 32), "bench_red_coalesced: row count");
    red_coalesced_kernel<<<kNumSMs * 8, 256, 0, as_stream(stream)>>>(buf, static_cast<uint32_t>(nrows), nops, seed);
    return check_launch("bench_red_coalesced");
}

}  // extern "C"
