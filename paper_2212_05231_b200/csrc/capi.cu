// Error plumbing and the array-level drop-ins for hashsdf/_kernels.py
// (interp_features, interp_full, scatter_first, scatter_second, adam_step).
#include <stdarg.h>
#include <stdio.h>

#include <atomic>

#include "common.cuh"

namespace ns2b {

static thread_local char g_err[512] = "";
static std::atomic<uint64_t> g_launches{0};

int set_error(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int check_launch(const char *what) {
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(NS2B_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return NS2B_OK;
}

// ------------------------------------------------------------------------
// Array-level kernels.  Thread per point; the 8 corner loads of a level are
// issued back to back (independent) so each thread keeps 8 L2 requests in flight.
struct GridArgs {
    int nlev, n_active;
    int64_t tsize;
    LevelInfo lv[NS2B_MAX_LEVELS];
    float sx[NS2B_MAX_LEVELS], sy[NS2B_MAX_LEVELS], sz[NS2B_MAX_LEVELS];
};

static int make_grid_args(GridArgs &g, int64_t nlev, int64_t tsize, int64_t nfeat,
                          const int64_t *res_host, int64_t n_active, const float *inv_ext_host) {
    NS2B_REQUIRE(nlev >= 1 && nlev <= NS2B_MAX_LEVELS, "shape error: 1..16 levels supported");
    NS2B_REQUIRE(nfeat == 2, "shape error: features_per_level must be 2");
    NS2B_REQUIRE(tsize >= 1 && tsize <= (1ll << 31), "shape error: table size out of range");
    NS2B_REQUIRE(n_active >= 0 && n_active <= nlev, "n_active out of range");
    g.nlev = static_cast<int>(nlev);
    g.n_active = static_cast<int>(n_active);
    g.tsize = tsize;
    for (int l = 0; l < nlev; ++l) {
        g.lv[l] = make_level(static_cast<int>(res_host[l]), tsize);
        if (inv_ext_host) {
            g.sx[l] = static_cast<float>(static_cast<double>(res_host[l]) * inv_ext_host[0]);
            g.sy[l] = static_cast<float>(static_cast<double>(res_host[l]) * inv_ext_host[1]);
            g.sz[l] = static_cast<float>(static_cast<double>(res_host[l]) * inv_ext_host[2]);
        }
    }
    return NS2B_OK;
}

template <bool kFull>
__global__ void interp_kernel(const float *__restrict__ xn, int64_t npts,
                              const float *__restrict__ tables, GridArgs g, float *__restrict__ feats,
                              float *__restrict__ jac, int64_t *__restrict__ cidx,
                              float *__restrict__ cw, float *__restrict__ cdw) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npts;
         p += (int64_t)gridDim.x * blockDim.x) {
        float x = xn[3 * p], y = xn[3 * p + 1], z = xn[3 * p + 2];
        for (int l = 0; l < g.nlev; ++l) {
            const int a0 = 2 * l;
            float f0 = 0.f, f1 = 0.f, j0[3] = {0.f, 0.f, 0.f}, j1[3] = {0.f, 0.f, 0.f};
            if (l < g.n_active) {
                const LevelInfo lv = g.lv[l];
                int cx, cy, cz;
                float fx, fy, fz;
                cell_frac(x, lv.n, cx, fx);
                cell_frac(y, lv.n, cy, fy);
                cell_frac(z, lv.n, cz, fz);
                const float2 *tab = reinterpret_cast<const float2 *>(tables + l * g.tsize * 2);
                uint32_t rows[8];
                float2 val[8];
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    rows[c] = corner_row(lv, cx + ((c >> 2) & 1), cy + ((c >> 1) & 1), cz + (c & 1));
#pragma unroll
                for (int c = 0; c < 8; ++c) val[c] = __ldg(tab + rows[c]);
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const int ox = (c >> 2) & 1, oy = (c >> 1) & 1, oz = c & 1;
                    float wx = ox ? fx : 1.f - fx, wy = oy ? fy : 1.f - fy, wz = oz ? fz : 1.f - fz;
                    float w = wx * wy * wz;
                    f0 = fmaf(w, val[c].x, f0);
                    f1 = fmaf(w, val[c].y, f1);
                    if (kFull) {
                        float dwx = (ox ? 1.f : -1.f) * wy * wz * g.sx[l];
                        float dwy = (oy ? 1.f : -1.f) * wx * wz * g.sy[l];
                        float dwz = (oz ? 1.f : -1.f) * wx * wy * g.sz[l];
                        j0[0] = fmaf(dwx, val[c].x, j0[0]);
                        j0[1] = fmaf(dwy, val[c].x, j0[1]);
                        j0[2] = fmaf(dwz, val[c].x, j0[2]);
                        j1[0] = fmaf(dwx, val[c].y, j1[0]);
                        j1[1] = fmaf(dwy, val[c].y, j1[1]);
                        j1[2] = fmaf(dwz, val[c].y, j1[2]);
                        int64_t r = (p * g.nlev + l) * 8 + c;
                        cidx[r] = rows[c];
                        cw[r] = w;
                        cdw[3 * r] = dwx;
                        cdw[3 * r + 1] = dwy;
                        cdw[3 * r + 2] = dwz;
                    }
                }
            } else if (kFull) {
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    int64_t r = (p * g.nlev + l) * 8 + c;
                    cidx[r] = 0;
                    cw[r] = 0.f;
                    cdw[3 * r] = cdw[3 * r + 1] = cdw[3 * r + 2] = 0.f;
                }
            }
            int64_t fo = p * g.nlev * 2 + a0;
            feats[fo] = f0;
            feats[fo + 1] = f1;
            if (kFull) {
                for (int k = 0; k < 3; ++k) {
                    jac[3 * fo + k] = j0[k];
                    jac[3 * (fo + 1) + k] = j1[k];
                }
            }
        }
    }
}

// hessian_contract (_kernels.py:159-206): (P,3,3) fp32, zero diagonal.
__global__ void hessian_kernel(const float *__restrict__ xn, int64_t npts, const float *__restrict__ tables,
                               GridArgs g, double ix, double iy, double iz, const float *__restrict__ coeff,
                               float *__restrict__ out) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npts;
         p += (int64_t)gridDim.x * blockDim.x) {
        const float u0 = xn[3 * p], u1 = xn[3 * p + 1], u2 = xn[3 * p + 2];
        float oxy = 0.f, oxz = 0.f, oyz = 0.f;
        for (int l = 0; l < g.n_active; ++l) {
            const LevelInfo lv = g.lv[l];
            const float2 *tab = reinterpret_cast<const float2 *>(tables + l * g.tsize * 2);
            const float *cf = coeff + (p * g.nlev + l) * 2;
            double hxy, hxz, hyz;
            hess_level(tab, lv, u0, u1, u2, cf[0], cf[1], hxy, hxz, hyz);
            const double n = static_cast<double>(lv.n);
            const double sx = n * ix, sy = n * iy, sz = n * iz;
            oxy = hess_acc(oxy, hxy, sx, sy);
            oxz = hess_acc(oxz, hxz, sx, sz);
            oyz = hess_acc(oyz, hyz, sy, sz);
        }
        float *o = out + 9 * p;
        o[0] = 0.f;
        o[1] = oxy;
        o[2] = oxz;
        o[3] = oxy;
        o[4] = 0.f;
        o[5] = oyz;
        o[6] = oxz;
        o[7] = oyz;
        o[8] = 0.f;
    }
}

__global__ void scatter_kernel(float *__restrict__ grad, int nlev, int64_t tsize,
                               const int64_t *__restrict__ cidx, const float *__restrict__ cw,
                               const float *__restrict__ cdw, const float *__restrict__ dl,
                               int64_t npts, int n_active, bool second) {
    // one thread per (point, level): 8 corners x float2 RED
    int64_t n = npts * n_active;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = i / n_active;
        int l = static_cast<int>(i - p * n_active);
        int64_t fo = p * nlev * 2 + 2 * l;
        float *g = grad + l * tsize * 2;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            int64_t r = (p * nlev + l) * 8 + c;
            float a, b;
            if (!second) {
                float w = cw[r];
                a = w * dl[fo];
                b = w * dl[fo + 1];
            } else {
                const float *d = cdw + 3 * r;
                const float *u0 = dl + 3 * fo, *u1 = dl + 3 * (fo + 1);
                a = u0[0] * d[0] + u0[1] * d[1] + u0[2] * d[2];
                b = u1[0] * d[0] + u1[1] * d[1] + u1[2] * d[2];
            }
            red_add_f32x2(g + 2 * cidx[r], a, b);
        }
    }
}

// adam_step (_kernels.py:209-218): fp64 math, moments stored in the param dtype,
// the parameter update re-reads the stored (rounded) moments as numba does.
template <typename T>
__global__ void adam_kernel(T *__restrict__ param, const T *__restrict__ grad, T *__restrict__ m,
                            T *__restrict__ v, int64_t n, double lr, double b1, double b2,
                            double eps, double c1, double c2) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double g = static_cast<double>(grad[i]);
        T mi = static_cast<T>(__dadd_rn(__dmul_rn(b1, static_cast<double>(m[i])), __dmul_rn(1.0 - b1, g)));
        T vi = static_cast<T>(__dadd_rn(__dmul_rn(b2, static_cast<double>(v[i])),
                                        __dmul_rn(__dmul_rn(1.0 - b2, g), g)));
        m[i] = mi;
        v[i] = vi;
        double step = __ddiv_rn(__dmul_rn(lr, __ddiv_rn(static_cast<double>(mi), c1)),
                                __dadd_rn(sqrt(__ddiv_rn(static_cast<double>(vi), c2)), eps));
        param[i] = static_cast<T>(__dsub_rn(static_cast<double>(param[i]), step));
    }
}

double int_pow(double a, int64_t e) {
    // float ** int as numba lowers it (binary exponentiation)
    bool inv = e < 0;
    uint64_t k = inv ? static_cast<uint64_t>(-e) : static_cast<uint64_t>(e);
    double r = 1.0;
    while (k) {
        if (k & 1) r *= a;
        k >>= 1;
        if (k) a *= a;
    }
    return inv ? 1.0 / r : r;
}

}  // namespace ns2b

using namespace ns2b;

extern "C" {

const char *ns2b_last_error(void) { return g_err; }
int ns2b_abi_version(void) { return NS2B_ABI_VERSION; }
uint64_t ns2b_launch_count(void) { return g_launches.load(); }

static int copy_res(const int64_t *res_dev, int64_t nlev, int64_t *res_host, cudaStream_t st) {
    // resolutions are tiny; the shim passes a device copy like every other argument.
    cudaError_t e = cudaMemcpyAsync(res_host, res_dev, nlev * sizeof(int64_t), cudaMemcpyDefault, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return set_error(NS2B_ECUDA, "resolutions copy: %s", cudaGetErrorString(e));
    return NS2B_OK;
}

int ns2b_interp_features(const float *xn, int64_t npts, const float *tables, int64_t nlev,
                         int64_t tsize, int64_t nfeat, const int64_t *resolutions,
                         int64_t n_active, float *out, void *stream) {
    cudaStream_t st = as_stream(stream);
    NS2B_REQUIRE(nlev >= 1 && nlev <= NS2B_MAX_LEVELS, "shape error: 1..16 levels supported");
    int64_t res[NS2B_MAX_LEVELS];
    int rc = copy_res(resolutions, nlev, res, st);
    if (rc) return rc;
    GridArgs g;
    if ((rc = make_grid_args(g, nlev, tsize, nfeat, res, n_active, nullptr))) return rc;
    if (npts == 0) return NS2B_OK;
    interp_kernel<false><<<grid_for(npts, 128), 128, 0, st>>>(xn, npts, tables, g, out, nullptr,
                                                              nullptr, nullptr, nullptr);
    return check_launch("interp_features");
}

int ns2b_interp_full(const float *xn, int64_t npts, const float *tables, int64_t nlev,
                     int64_t tsize, int64_t nfeat, const int64_t *resolutions, int64_t n_active,
                     const float *inv_extent, float *feats, float *jac, int64_t *cidx, float *cw,
                     float *cdw, void *stream) {
    cudaStream_t st = as_stream(stream);
    NS2B_REQUIRE(nlev >= 1 && nlev <= NS2B_MAX_LEVELS, "shape error: 1..16 levels supported");
    int64_t res[NS2B_MAX_LEVELS];
    float inv[3];
    int rc = copy_res(resolutions, nlev, res, st);
    if (rc) return rc;
    cudaError_t e = cudaMemcpyAsync(inv, inv_extent, sizeof(inv), cudaMemcpyDefault, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return set_error(NS2B_ECUDA, "inv_extent copy: %s", cudaGetErrorString(e));
    GridArgs g;
    if ((rc = make_grid_args(g, nlev, tsize, nfeat, res, n_active, inv))) return rc;
    if (npts == 0) return NS2B_OK;
    interp_kernel<true><<<grid_for(npts, 128), 128, 0, st>>>(xn, npts, tables, g, feats, jac, cidx,
                                                             cw, cdw);
    return check_launch("interp_full");
}

int ns2b_hessian_contract(const float *xn, int64_t npts, const float *tables, int64_t nlev, int64_t tsize,
                          int64_t nfeat, const int64_t *resolutions, int64_t n_active, const float *inv_extent,
                          const float *coeff, float *out, void *stream) {
    cudaStream_t st = as_stream(stream);
    NS2B_REQUIRE(nlev >= 1 && nlev <= NS2B_MAX_LEVELS, "shape error: 1..16 levels supported");
    int64_t res[NS2B_MAX_LEVELS];
    float inv[3];
    int rc = copy_res(resolutions, nlev, res, st);
    if (rc) return rc;
    cudaError_t e = cudaMemcpyAsync(inv, inv_extent, sizeof(inv), cudaMemcpyDefault, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return set_error(NS2B_ECUDA, "inv_extent copy: %s", cudaGetErrorString(e));
    GridArgs g;
    if ((rc = make_grid_args(g, nlev, tsize, nfeat, res, n_active, inv))) return rc;
    if (npts == 0) return NS2B_OK;
    hessian_kernel<<<grid_for(npts, 128), 128, 0, st>>>(xn, npts, tables, g, inv[0], inv[1], inv[2], coeff,
                                                         out);
    return check_launch("hessian_contract");
}

static int scatter_common(float *grad, int64_t nlev, int64_t tsize, int64_t nfeat,
                          const int64_t *cidx, const float *cw, const float *cdw, const float *dl,
                          int64_t npts, int64_t n_active, bool second, void *stream) {
    NS2B_REQUIRE(nlev >= 1 && nlev <= NS2B_MAX_LEVELS, "shape error: 1..16 levels supported");
    NS2B_REQUIRE(nfeat == 2, "shape error: features_per_level must be 2");
    NS2B_REQUIRE(n_active >= 0 && n_active <= nlev, "n_active out of range");
    if (npts == 0 || n_active == 0) return NS2B_OK;
    scatter_kernel<<<grid_for(npts * n_active, 256), 256, 0, as_stream(stream)>>>(
        grad, static_cast<int>(nlev), tsize, cidx, cw, cdw, dl, npts, static_cast<int>(n_active),
        second);
    return check_launch(second ? "scatter_second" : "scatter_first");
}

int ns2b_scatter_first(float *grad, int64_t nlev, int64_t tsize, int64_t nfeat,
                       const int64_t *cidx, const float *cw, const float *dl_dfeat, int64_t npts,
                       int64_t n_active, void *stream) {
    return scatter_common(grad, nlev, tsize, nfeat, cidx, cw, nullptr, dl_dfeat, npts, n_active,
                          false, stream);
}

int ns2b_scatter_second(float *grad, int64_t nlev, int64_t tsize, int64_t nfeat,
                        const int64_t *cidx, const float *cdw, const float *u, int64_t npts,
                        int64_t n_active, void *stream) {
    return scatter_common(grad, nlev, tsize, nfeat, cidx, nullptr, cdw, u, npts, n_active, true,
                          stream);
}

int ns2b_adam_step_f32(float *param, const float *grad, float *m, float *v, int64_t n, int64_t t,
                       double lr, double beta1, double beta2, double eps, void *stream) {
    if (n == 0) return NS2B_OK;
    double c1 = 1.0 - int_pow(beta1, t), c2 = 1.0 - int_pow(beta2, t);
    adam_kernel<float><<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(param, grad, m, v, n, lr,
                                                                        beta1, beta2, eps, c1, c2);
    return check_launch("adam_step_f32");
}

int ns2b_adam_step_f64(double *param, const double *grad, double *m, double *v, int64_t n,
                       int64_t t, double lr, double beta1, double beta2, double eps,
                       void *stream) {
    if (n == 0) return NS2B_OK;
    double c1 = 1.0 - int_pow(beta1, t), c2 = 1.0 - int_pow(beta2, t);
    adam_kernel<double><<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(param, grad, m, v, n, lr,
                                                                         beta1, beta2, eps, c1, c2);
    return check_launch("adam_step_f64");
}

}  // extern "C"
