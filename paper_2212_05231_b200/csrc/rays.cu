// Device ray-batch generation (scene_io.py:98-116,129-172): the pixel
// picks come from the reference's own draws (rng.integers on the host, identical
// stream), everything else -- pool lookup, pinhole rays, targets image * mask -- runs
// here from images, masks and pixel pools resident in HBM.
//
// Arithmetic follows numpy op for op (fp64, explicit round-to-nearest, no contraction
// except where numpy's matmul itself fuses):
//   d_cam = ((px + 0.5 - cx) / fx, (py + 0.5 - cy) / fy, 1)
//   d     = d_cam @ R^T    (one BLAS dgemm order: fma(d2, R2, fma(d1, R1, d0 * R0));
//                           another host BLAS may sum differently: within 2 ulp)
//   d    /= sqrt((d0^2 + d1^2) + d2^2)          (np.linalg.norm, pairwise add)
//   target = (u8 / 255.0) * mask
#include "common.cuh"

namespace ns2b {

__global__ void rays_kernel(const int64_t *__restrict__ picks, int64_t n, int64_t n_first,
                            const int32_t *__restrict__ pool_a, const int32_t *__restrict__ pool_b,
                            const double *__restrict__ frames, int32_t width, int32_t height,
                            const uint8_t *__restrict__ images, const uint8_t *__restrict__ masks,
                            double *__restrict__ origins, double *__restrict__ dirs,
                            double *__restrict__ targets) {
    const int64_t hw = static_cast<int64_t>(width) * height;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t pick = picks[i];
        const int64_t flat = (i < n_first ? pool_a : pool_b)[pick];
        const int64_t k = flat / hw;
        const int64_t rem = flat - k * hw;
        const int y = static_cast<int>(rem / width), x = static_cast<int>(rem - static_cast<int64_t>(y) * width);
        const double *fr = frames + 16 * k;  // R (row-major 3x3) | t (3) | fx fy cx cy
        const double px = static_cast<double>(x), py = static_cast<double>(y);
        const double c0 = __ddiv_rn(__dadd_rn(__dadd_rn(px, 0.5), -fr[14]), fr[12]);
        const double c1 = __ddiv_rn(__dadd_rn(__dadd_rn(py, 0.5), -fr[15]), fr[13]);
        double d[3];
#pragma unroll
        for (int j = 0; j < 3; ++j)
            d[j] = __fma_rn(1.0, fr[3 * j + 2], __fma_rn(c1, fr[3 * j + 1], __dmul_rn(c0, fr[3 * j])));
        const double nrm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])),
                                                __dmul_rn(d[2], d[2])));
        const uint8_t *im = images + 3 * (k * hw + rem);
        const double mk = static_cast<double>(masks[k * hw + rem]);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            origins[3 * i + j] = fr[9 + j];
            dirs[3 * i + j] = __ddiv_rn(d[j], nrm);
            targets[3 * i + j] = __dmul_rn(__ddiv_rn(static_cast<double>(im[j]), 255.0), mk);
        }
    }
}

}  // namespace ns2b

using namespace ns2b;

extern "C" int ns2b_rays_from_picks(const int64_t *picks, int64_t n, int64_t n_first, const int32_t *pool_first,
                                    const int32_t *pool_rest, const double *frames, int32_t width, int32_t height,
                                    const uint8_t *images, const uint8_t *masks, double *origins, double *dirs,
                                    double *targets, void *stream) {
    NS2B_REQUIRE(n >= 0 && n_first >= 0 && n_first <= n, "rays_from_picks: bad counts");
    NS2B_REQUIRE(width > 0 && height > 0, "rays_from_picks: bad image size");
    NS2B_REQUIRE(picks && pool_first && pool_rest && frames && images && masks && origins && dirs && targets,
                 "rays_from_picks: null pointer");
    if (n == 0) return NS2B_OK;
    rays_kernel<<<grid_for(n, 256, kNumSMs * 8), 256, 0, as_stream(stream)>>>(
        picks, n, n_first, pool_first, pool_rest, frames, width, height, images, masks, origins, dirs, targets);
    return check_launch("rays_from_picks");
}
