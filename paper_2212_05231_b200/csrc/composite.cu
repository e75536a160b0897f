// K3/K4: per-ray NeuS compositing, Huber colour loss and the compositing backward
// (renderer.py:35-56, 217-291, 303-358; trainer.py:96-112, 215-221).  Warp per ray;
// a ray's kept samples are contiguous (ray-major marching), so every load is
// coalesced.  Intervals are consecutive kept samples (i, i+1) of the ray.
//
// Forward: alpha from the logistic CDF (fp64), log-transmittance by a warp scan
// with a carry across 32-interval chunks, w = T*alpha, C = sum w c.
// Backward: walks the chunks back to front with a reverse warp scan for the
// suffix sum_{k>i} w_k a_dot_k; each lane writes dL/dsdf of sample i+1 =
// (interval i's dalpha/df_{i+1} term) + (interval i+1's dalpha/df_{i+1} term),
// so no atomics are needed.  Compiled with -fmad=false (no contraction) to stay
// op-for-op with the reference's numpy.
#include "common.cuh"

namespace ns2b {

constexpr double kAlphaMax = 1.0 - 1e-7;
constexpr int CBLOCK = 256;

__device__ __forceinline__ double logistic_cdf(double s, double f) {
    // sdf_transforms (renderer.py:35-49): Phi = sigma(clip(s f, +-80)), two branches
    double z = s * f;
    z = fmin(fmax(z, -80.0), 80.0);
    if (z >= 0.0) return 1.0 / (1.0 + exp(-z));
    double ez = exp(z);
    return ez / (1.0 + ez);
}

__device__ __forceinline__ double huber(double r, double delta) {
    double a = fabs(r);
    return a <= delta ? 0.5 * r * r / delta : a - 0.5 * delta;
}
__device__ __forceinline__ double huber_grad(double r, double delta) {
    if (fabs(r) <= delta) return r / delta;
    return r > 0.0 ? 1.0 : (r < 0.0 ? -1.0 : 0.0);
}

__device__ __forceinline__ double warp_incl_scan(double v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        double t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}
__device__ __forceinline__ double warp_incl_suffix(double v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        double t = __shfl_down_sync(0xffffffffu, v, o);
        if (lane + o < 32) v += t;
    }
    return v;
}

// mode bits
constexpr int kFwd = 1;       // compute alphas/weights/T and rendered colour
constexpr int kLoss = 2;      // Huber loss + per-ray cotangent from targets
constexpr int kBwd = 4;       // compositing backward

template <int kMode>
__global__ void __launch_bounds__(CBLOCK)
composite_kernel(const int32_t *__restrict__ offsets, int64_t nrays, const float *__restrict__ sdf,
                 const float *__restrict__ colors, double s, const double *__restrict__ targets,
                 double delta, double m_total, const double *__restrict__ dl_dray_in,
                 double *__restrict__ rendered, double *__restrict__ resid_t, double *__restrict__ alphas,
                 double *__restrict__ weights, double *__restrict__ tb, float *__restrict__ dl_dc,
                 float *__restrict__ dl_dsdf, double *__restrict__ sums) {
    __shared__ double red[3][CBLOCK / 32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double acc_loss = 0.0, acc_ds = 0.0, acc_sq = 0.0;
    const int64_t nw = ((int64_t)gridDim.x * CBLOCK) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * CBLOCK + threadIdx.x) >> 5; r < nrays; r += nw) {
        const int64_t start = offsets[r];
        const int n = offsets[r + 1] - static_cast<int>(start);
        const int nint = n > 1 ? n - 1 : 0;
        double C0 = 0.0, C1 = 0.0, C2 = 0.0;
        if (kMode & kFwd) {
            double carry = 0.0;
            // Phi of each sample is computed once: lane l holds sample b + l of the current
            // 32-sample window; interval i's cj is the next lane's value (lane 31: the next
            // window's first)
            double phi = (nint > 0 && lane < n) ? logistic_cdf(s, static_cast<double>(sdf[start + lane])) : 0.0;
            for (int b = 0; b < nint; b += 32) {
                const int i = b + lane;
                const int nx = b + 32 + lane;
                const double phi_next = nx < n ? logistic_cdf(s, static_cast<double>(sdf[start + nx])) : 0.0;
                double up = __shfl_down_sync(0xffffffffu, phi, 1);
                const double first_next = __shfl_sync(0xffffffffu, phi_next, 0);
                if (lane == 31) up = first_next;
                double a = 0.0, lg = 0.0;
                if (i < nint) {
                    const double ci = phi;
                    const double cj = up;
                    a = (ci - cj) / ci;
                    a = fmin(fmax(a, 0.0), kAlphaMax);
                    lg = log1p(-a);
                }
                const double incl = warp_incl_scan(lg, lane);
                if (i < nint) {
                    const double T = exp(carry + (incl - lg));
                    const double w = T * a;
                    const int64_t q = start + i;
                    C0 += w * static_cast<double>(colors[3 * q]);
                    C1 += w * static_cast<double>(colors[3 * q + 1]);
                    C2 += w * static_cast<double>(colors[3 * q + 2]);
                    alphas[q] = a;
                    weights[q] = w;
                    tb[q] = T;
                }
                carry += __shfl_sync(0xffffffffu, incl, 31);
                phi = phi_next;
            }
            C0 = warp_sum(C0);
            C1 = warp_sum(C1);
            C2 = warp_sum(C2);
            if (lane == 0) {
                rendered[3 * r] = C0;
                rendered[3 * r + 1] = C1;
                rendered[3 * r + 2] = C2;
                if (resid_t) resid_t[r] = exp(carry);
            }
        }
        double g0, g1, g2;
        if (kMode & kLoss) {
            const double e0 = C0 - targets[3 * r], e1 = C1 - targets[3 * r + 1], e2 = C2 - targets[3 * r + 2];
            if (lane == 0) {
                acc_loss += huber(e0, delta) + huber(e1, delta) + huber(e2, delta);
                acc_sq += e0 * e0 + e1 * e1 + e2 * e2;
            }
            g0 = huber_grad(e0, delta) / m_total;
            g1 = huber_grad(e1, delta) / m_total;
            g2 = huber_grad(e2, delta) / m_total;
        } else if (kMode & kBwd) {
            g0 = dl_dray_in[3 * r];
            g1 = dl_dray_in[3 * r + 1];
            g2 = dl_dray_in[3 * r + 2];
        }
        if (kMode & kBwd) {
            if (n == 1 && lane == 0) {
                dl_dsdf[start] = 0.f;
                dl_dc[3 * start] = dl_dc[3 * start + 1] = dl_dc[3 * start + 2] = 0.f;
            }
            double suffix = 0.0;   // sum over intervals of later chunks
            double next_ci = 0.0;  // interval (b+32)'s dalpha/df_i term, for lane 31
            const int nchunks = (nint + 31) >> 5;
            // Phi once per sample again, windows walked back to front (phi_w: the window
            // after the current chunk, whose lane 0 is lane 31's cj)
            double phi_w = 0.0;
            if (nint > 0) {
                const int w0 = nchunks * 32 + lane;
                phi_w = w0 < n ? logistic_cdf(s, static_cast<double>(sdf[start + w0])) : 0.0;
            }
            for (int ch = nchunks - 1; ch >= 0; --ch) {
                const int i = ch * 32 + lane;
                const bool ok = i < nint;
                const double phi_c = i < n ? logistic_cdf(s, static_cast<double>(sdf[start + i])) : 0.0;
                double phi_up = __shfl_down_sync(0xffffffffu, phi_c, 1);
                const double first_w = __shfl_sync(0xffffffffu, phi_w, 0);
                if (lane == 31) phi_up = first_w;
                phi_w = phi_c;
                double wa = 0.0, a = 0.0, w = 0.0, T = 0.0, adot = 0.0;
                if (ok) {
                    const int64_t q = start + i;
                    a = alphas[q];
                    w = weights[q];
                    T = tb[q];
                    adot = static_cast<double>(colors[3 * q]) * g0 + static_cast<double>(colors[3 * q + 1]) * g1 +
                           static_cast<double>(colors[3 * q + 2]) * g2;
                    wa = w * adot;
                }
                const double incl = warp_incl_suffix(wa, lane);  // sum_{k>=i} in chunk
                double t_ci = 0.0, t_cj = 0.0;
                if (ok) {
                    const double S = suffix + (incl - wa);
                    const double dl_da = T * adot - S / (1.0 - a);
                    const int64_t q = start + i;
                    const double fi = static_cast<double>(sdf[q]), fj = static_cast<double>(sdf[q + 1]);
                    const double ci = phi_c, cj = phi_up;
                    const double raw = (ci - cj) / ci;
                    if (raw > 0.0 && raw < kAlphaMax) {
                        const double dpi = s * ci * (1.0 - ci);
                        const double dpj = s * cj * (1.0 - cj);
                        const double ci2 = ci * ci;
                        t_ci = dl_da * (cj / ci2 * dpi);
                        t_cj = dl_da * (-dpj / ci);
                        const double dads = cj / ci2 * fi * ci * (1.0 - ci) - fj * cj * (1.0 - cj) / ci;
                        acc_ds += dl_da * dads;
                    }
                    dl_dc[3 * q] = static_cast<float>(w * g0);
                    dl_dc[3 * q + 1] = static_cast<float>(w * g1);
                    dl_dc[3 * q + 2] = static_cast<float>(w * g2);
                }
                // sample i+1 gets t_cj(i) + t_ci(i+1)
                double up = __shfl_down_sync(0xffffffffu, t_ci, 1);
                if (lane == 31) up = next_ci;
                if (ok) {
                    const int64_t q1 = start + i + 1;
                    const double ci_next = (i + 1 < nint) ? up : 0.0;
                    dl_dsdf[q1] = static_cast<float>(t_cj + ci_next);
                    if (i + 1 == nint) {  // last sample: no interval starts there
                        dl_dc[3 * q1] = dl_dc[3 * q1 + 1] = dl_dc[3 * q1 + 2] = 0.f;
                    }
                }
                if (ch == 0 && lane == 0 && ok) dl_dsdf[start] = static_cast<float>(t_ci);
                next_ci = __shfl_sync(0xffffffffu, t_ci, 0);
                suffix += __shfl_sync(0xffffffffu, incl, 0);
            }
        }
    }
    if (sums) {
        acc_loss = warp_sum(acc_loss);
        acc_ds = warp_sum(acc_ds);
        acc_sq = warp_sum(acc_sq);
        if (lane == 0) {
            red[0][wib] = acc_loss;
            red[1][wib] = acc_ds;
            red[2][wib] = acc_sq;
        }
        __syncthreads();
        if (threadIdx.x < 3) {
            double v = 0.0;
            for (int k = 0; k < CBLOCK / 32; ++k) v += red[threadIdx.x][k];
            if (v != 0.0) atomicAdd(sums + threadIdx.x, v);
        }
    }
}

}  // namespace ns2b

using namespace ns2b;

extern "C" {

int ns2b_composite(const int32_t *offsets, int64_t nrays, const float *sdf, const float *colors,
                   double sharpness, const double *targets, double huber_delta,
                   double num_rays_total, double *rendered, double *resid_trans, double *alphas,
                   double *weights, double *trans_before, float *dl_dc, float *dl_dsdf,
                   double *sums, void *stream) {
    NS2B_REQUIRE(rendered && alphas && weights && trans_before, "composite: output buffers required");
    if (nrays == 0) return NS2B_OK;
    const int blocks = grid_for(nrays * 32, CBLOCK, kNumSMs * 16);
    cudaStream_t st = as_stream(stream);
    if (targets) {
        NS2B_REQUIRE(dl_dc && dl_dsdf && sums, "composite: cotangent buffers required with targets");
        NS2B_REQUIRE(num_rays_total >= 1.0, "need at least one ray");
        composite_kernel<kFwd | kLoss | kBwd><<<blocks, CBLOCK, 0, st>>>(
            offsets, nrays, sdf, colors, sharpness, targets, huber_delta, num_rays_total, nullptr,
            rendered, resid_trans, alphas, weights, trans_before, dl_dc, dl_dsdf, sums);
    } else {
        composite_kernel<kFwd><<<blocks, CBLOCK, 0, st>>>(
            offsets, nrays, sdf, colors, sharpness, nullptr, 0.0, 1.0, nullptr, rendered,
            resid_trans, alphas, weights, trans_before, nullptr, nullptr, nullptr);
    }
    return check_launch("composite");
}

int ns2b_composite_backward(const int32_t *offsets, int64_t nrays, const float *sdf,
                            const float *colors, double sharpness, const double *alphas,
                            const double *weights, const double *trans_before,
                            const double *dl_dray, float *dl_dc, float *dl_dsdf, double *sums,
                            void *stream) {
    NS2B_REQUIRE(alphas && weights && trans_before && dl_dray && dl_dc && dl_dsdf,
                 "composite_backward: null buffer");
    if (nrays == 0) return NS2B_OK;
    const int blocks = grid_for(nrays * 32, CBLOCK, kNumSMs * 16);
    composite_kernel<kBwd><<<blocks, CBLOCK, 0, as_stream(stream)>>>(
        offsets, nrays, sdf, colors, sharpness, nullptr, 0.0, 1.0, dl_dray, nullptr, nullptr,
        const_cast<double *>(alphas), const_cast<double *>(weights), const_cast<double *>(trans_before),
        dl_dc, dl_dsdf, sums);
    return check_launch("composite_backward");
}

}  // extern "C"
