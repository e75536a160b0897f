// Self-test of the tcgen05 building blocks (umma.cuh): one CTA computes a small
// GEMM with the three-term 16-bit split and writes D to global memory, so the
// descriptor encodings (K-major / MN-major views of the same tile layout, M = 128
// and M = 64 accumulator layouts, F16 and BF16) are validated on the device against
// a host fp64 reference (tests/test_gpu_umma.py).
#include "common.cuh"
#include "umma.cuh"

namespace ns2b {

// mode 0: D[128x64] = A[128x48] * B[64x48]^T          f16, A K-major, B K-major
// mode 1: D[128x64] = A[128x48] * B[48x64]            f16, A K-major, B MN-major
// mode 2: D[64x48]  = U[128x64]^T * V[128x48]         bf16, A MN-major, B MN-major (M=64)
// mode 3: as mode 0 with bf16
// mode 4: as mode 1 with A in tensor memory (tcgen05.st of the packed hi / lo halves)
__global__ void __launch_bounds__(128) umma_selftest_kernel(const float *__restrict__ A,
                                                            const float *__restrict__ B,
                                                            float *__restrict__ D, int mode) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base;
    uint8_t *a_hi = sm, *a_lo = sm + 16384, *b_hi = sm + 32768, *b_lo = sm + 49152;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    float row[64];
    // stage A (row t)
    if (mode == 2) {
        for (int i = 0; i < 64; ++i) row[i] = A[t * 64 + i];
        umma::stage_row<1, 64>(a_hi, a_lo, t, row);
        for (int i = 0; i < 48; ++i) row[i] = B[t * 48 + i];
        umma::stage_row<1, 48>(b_hi, b_lo, t, row);
    } else if (mode == 4) {
        if (t < 48) {
            for (int i = 0; i < 64; ++i) row[i] = B[t * 64 + i];
            umma::stage_row<0, 64>(b_hi, b_lo, t, row);
        }
    } else {
        for (int i = 0; i < 48; ++i) row[i] = A[t * 48 + i];
        if (mode == 3) umma::stage_row<1, 48>(a_hi, a_lo, t, row);
        else umma::stage_row<0, 48>(a_hi, a_lo, t, row);
        if (mode == 0 || mode == 3) {
            if (t < 64) {
                for (int i = 0; i < 48; ++i) row[i] = B[t * 48 + i];
                if (mode == 3) umma::stage_row<1, 48>(b_hi, b_lo, t, row);
                else umma::stage_row<0, 48>(b_hi, b_lo, t, row);
            }
        } else if (t < 48) {
            for (int i = 0; i < 64; ++i) row[i] = B[t * 64 + i];
            umma::stage_row<0, 64>(b_hi, b_lo, t, row);
        }
    }
    umma::fence_async_smem();
    if (t == 0) {
        umma::mbar_init(&mbar, 1);
        umma::fence_barrier_init();
    }
    if (warp == 0) umma::tmem_alloc(&tmem_base, 128);
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tb = tmem_base;
    constexpr uint32_t kAH = 64, kAL = 96;  // mode 4: A hi / lo columns
    if (mode == 4) {  // row t -> lane t: 8 K elements (4 columns) per store
        const uint32_t la = tb + ((static_cast<uint32_t>(warp) * 32u) << 16);
        for (int kb = 0; kb < 6; ++kb) {
            uint4 h, l;
            umma::split2<0>(A[t * 48 + 8 * kb + 0], A[t * 48 + 8 * kb + 1], h.x, l.x);
            umma::split2<0>(A[t * 48 + 8 * kb + 2], A[t * 48 + 8 * kb + 3], h.y, l.y);
            umma::split2<0>(A[t * 48 + 8 * kb + 4], A[t * 48 + 8 * kb + 5], h.z, l.z);
            umma::split2<0>(A[t * 48 + 8 * kb + 6], A[t * 48 + 8 * kb + 7], h.w, l.w);
            umma::tmem_st4u(la + kAH + 4 * kb, h);
            umma::tmem_st4u(la + kAL + 4 * kb, l);
        }
        umma::tmem_st_wait();
        umma::fence_before_sync();
        __syncthreads();
        umma::fence_after_sync();
    }
    if (t == 0) {
        if (mode == 0 || mode == 3) {
            const int fmt = mode == 3 ? 1 : 0;
            umma::gemm3(tb, umma::kmajor(a_hi, a_lo, 48), umma::kmajor(b_hi, b_lo, 48), 3,
                        umma::make_idesc(128, 64, fmt, 0, 0), false);
        } else if (mode == 1) {
            umma::gemm3(tb, umma::kmajor(a_hi, a_lo, 48), umma::mnmajor(b_hi, b_lo, 64), 3,
                        umma::make_idesc(128, 64, 0, 0, 1), false);
        } else if (mode == 2) {
            umma::gemm3(tb, umma::mnmajor(a_hi, a_lo, 64), umma::mnmajor(b_hi, b_lo, 48), 8,
                        umma::make_idesc(64, 48, 1, 1, 1), false);
        }
        if (mode != 4) umma::commit(&mbar);
    }
    if (mode == 4 && warp == 0) {
        umma::gemm3t<3>(tb, tb + kAH, tb + kAL, umma::mnmajor(b_hi, b_lo, 64), umma::make_idesc(128, 64, 0, 0, 1),
                        false);
        umma::commit_elect(&mbar);
    }
    umma::mbar_wait(&mbar, 0);
    umma::fence_after_sync();
    const uint32_t lane_addr = tb + ((static_cast<uint32_t>(warp) * 32u) << 16);
    if (mode != 2) {
        for (int c = 0; c < 64; c += 16) {
            float v[16];
            umma::tmem_ld16(lane_addr + c, v);
            for (int i = 0; i < 16; ++i) D[t * 64 + c + i] = v[i];
        }
    } else {
        for (int c = 0; c < 48; c += 16) {
            float v[16];
            umma::tmem_ld16(lane_addr + c, v);
            if (lane < 16)
                for (int i = 0; i < 16; ++i) D[(warp * 16 + lane) * 48 + c + i] = v[i];
        }
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tb, 128);
}

}  // namespace ns2b

using namespace ns2b;

extern "C" {

int ns2b_selftest_umma(const float *A, const float *B, float *D, int32_t mode, void *stream) {
    NS2B_REQUIRE(mode >= 0 && mode <= 4, "selftest mode 0..4");
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(umma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        if (e != cudaSuccess) return set_error(NS2B_ECUDA, "selftest attr: %s", cudaGetErrorString(e));
        attr = true;
    }
    umma_selftest_kernel<<<1, 128, 65536, as_stream(stream)>>>(A, B, D, mode);
    return check_launch("selftest_umma");
}

}  // extern "C"
