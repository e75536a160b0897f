// tcgen05 issue-rate probe for the MLP kernels' GEMM shapes (profiling aid): one CTA,
// one thread issues `iters` kind::f16 MMAs of a given shape from zeroed shared memory and
// waits for their commit; the result is clock64 cycles for the batch.
//   shape 0: M=128 N=64  A K-major  B MN-major (chain GEMM, K = features)
//   shape 1: M=64  N=16  A MN-major B MN-major (weight-gradient GEMM, K = samples)
//   shape 2: M=64  N=64  A MN-major B MN-major
//   shape 3: M=128 N=16  A K-major  B K-major
//   shape 4: M=64  N=8   A MN-major B MN-major
//   shape 5: M=128 N=64  A K-major  B K-major
// variant: number of independent accumulators the MMAs rotate over (1, 2, 4).
#include "common.cuh"
#include "umma.cuh"

namespace ns2b {

__global__ void __launch_bounds__(128) umma_rate_kernel(int shape, int iters, int nacc, long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tbase;
    const int t = threadIdx.x;
    for (int i = t; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (t == 0) {
        umma::mbar_init(&mbar, 1);
        umma::fence_barrier_init();
    }
    if (t < 32) umma::tmem_alloc(&tbase, 512);
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    if (t < 32 && nacc == 2 && iters % 12 == 0) {  // warp-converged elect issue (gemm3w)
        const int M = (shape == 1 || shape == 2 || shape == 4) ? 64 : 128;
        const int N = (shape == 0 || shape == 2 || shape == 5) ? 64 : (shape == 4 ? 8 : 16);
        const bool a_mn = (shape == 1 || shape == 2 || shape == 4);
        const bool b_mn = (shape != 3 && shape != 5);
        const uint32_t idesc = umma::make_idesc(M, N, 0, a_mn, b_mn);
        const umma::Operand A = a_mn ? umma::mnmajor(sm, sm + 16384, 64) : umma::kmajor(sm, sm + 16384, 64);
        const umma::Operand B = b_mn ? umma::mnmajor(sm + 32768, sm + 49152, 64)
                                     : umma::kmajor(sm + 32768, sm + 49152, 64);
        __syncwarp();
        const long long c0 = clock64();
        for (int i = 0; i < iters / 12; ++i) umma::gemm3w<4>(tbase, A, B, idesc, i > 0);
        umma::commit_elect(&mbar);
        if (shape == 5) umma::mbar_wait_spin(&mbar, 0);  // shape 5: compare the plain spin wait
        else umma::mbar_wait(&mbar, 0);
        if (t == 0) out[0] = clock64() - c0;
    } else if (t == 0) {
        const int M = (shape == 1 || shape == 2 || shape == 4) ? 64 : 128;
        const int N = (shape == 0 || shape == 2 || shape == 5) ? 64 : (shape == 4 ? 8 : 16);
        const bool a_mn = (shape == 1 || shape == 2 || shape == 4);
        const bool b_mn = (shape != 3 && shape != 5);
        const uint32_t idesc = umma::make_idesc(M, N, 0, a_mn, b_mn);
        const umma::Operand A = a_mn ? umma::mnmajor(sm, sm + 16384, 64) : umma::kmajor(sm, sm + 16384, 64);
        const umma::Operand B = b_mn ? umma::mnmajor(sm + 32768, sm + 49152, 64)
                                     : umma::kmajor(sm + 32768, sm + 49152, 64);
        const long long c0 = clock64();
        if (nacc == 4 && iters % 12 == 0) {  // unrolled gemm3u, one accumulator
            for (int i = 0; i < iters / 12; ++i) umma::gemm3u<4>(tbase, A, B, idesc, i > 0);
        } else if (iters % 12 == 0) {  // through gemm3 (3-term split, 4 K steps), as the kernels issue
            for (int i = 0; i < iters / 12; ++i)
                umma::gemm3(tbase + static_cast<uint32_t>((i % nacc) * 64), A, B, 4, idesc, i >= nacc);
        } else {
            for (int i = 0; i < iters; ++i) {
                const int k = i & 3;
                const uint32_t d = tbase + static_cast<uint32_t>((i % nacc) * 64);
                umma::mma_f16(d, A.desc_hi(k), B.desc_hi(k), idesc, i >= nacc ? 1u : 0u);
            }
        }
        umma::commit(&mbar);
        umma::mbar_wait(&mbar, 0);
        out[0] = clock64() - c0;
    }
    umma::fence_before_sync();
    __syncthreads();
    if (t < 32) umma::tmem_dealloc(tbase, 512);
}

}  // namespace ns2b

using namespace ns2b;

extern "C" int ns2b_bench_umma(int32_t shape, int32_t iters, int32_t nacc, long long *cycles, void *stream) {
    NS2B_REQUIRE(shape >= 0 && shape <= 5 && iters > 0 && (nacc == 1 || nacc == 2 || nacc == 4) && cycles,
                 "bench_umma: shape 0..5, iters > 0, nacc 1|2|4");
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(umma_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        attr = true;
    }
    umma_rate_kernel<<<1, 128, 65536, as_stream(stream)>>>(shape, iters, nacc, cycles);
    return check_launch("bench_umma");
}
