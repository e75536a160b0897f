/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's compiled
 * hash-grid / Adam loops, used as the parity checker and as the timed CPU
 * baseline.  Never linked into the product library.
 *
 * Restates hashsdf/_kernels.py (numba, fastmath=False, single-threaded):
 *   cell/frac           _kernels.py:20-29   (lower-cell convention)
 *   corner index        _kernels.py:32-37   (dense iff (n+1)^3 <= T, else xor-prime
 *                                             hash; numba widens the uint32 products to
 *                                             64 bits before the xor and the modulo)
 *   interp_features     _kernels.py:40-64
 *   interp_full         _kernels.py:67-119
 *   scatter_first       _kernels.py:122-133
 *   scatter_second      _kernels.py:136-156
 *   hessian_contract    _kernels.py:159-206 (cv = sum_f f32(coeff*table) in fp64,
 *                                             per-level fp64 h, out re-rounded to fp32)
 *   adam_step           _kernels.py:209-218
 *
 * Numeric contract kept from numba's typing: positions are float32, t = x*n and the
 * trilinear weights are float64, feature/jacobian accumulators are float32 arrays that
 * are re-rounded after every corner (out = f32(f64(out) + w*v)); the scatters are pure
 * float32 arithmetic in (point, level, corner, feature) order.  Compiled with
 * -ffp-contract=off so no multiply-add is fused (numba/LLVM does not fuse either).
 * The gathers may run point-parallel (each point writes only its own rows, so the
 * result is thread-count independent); the scatters stay sequential.
 */
#include <math.h>
#include <stdint.h>

static inline void cell_frac(double t, int64_t n, int64_t *c, double *frac)
{
    int64_t ci = (int64_t)ceil(t) - 1;
    if (ci < 0)
        ci = 0;
    else if (ci > n - 1)
        ci = n - 1;
    *c = ci;
    *frac = t - (double)ci;
}

static inline int64_t corner_row(int64_t cx, int64_t cy, int64_t cz, int64_t n, int64_t tsize)
{
    if ((n + 1) * (n + 1) * (n + 1) <= tsize)
        return cx + (n + 1) * (cy + (n + 1) * cz);
    uint64_t h = ((uint64_t)(uint32_t)cx * 1ull) ^ ((uint64_t)(uint32_t)cy * 2654435761ull) ^
                 ((uint64_t)(uint32_t)cz * 805459861ull);
    return (int64_t)(h % (uint64_t)(uint32_t)tsize);
}

void orc_interp_features(const float *xn, int64_t npts, const float *tables, int64_t nlev,
                         int64_t tsize, int64_t nfeat, const int64_t *res, int64_t n_active,
                         float *out, int nthreads)
{
    (void)nlev;
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (int64_t p = 0; p < npts; ++p) {
        float *row = out + p * nlev * nfeat;
        for (int64_t l = 0; l < n_active; ++l) {
            int64_t n = res[l];
            int64_t cx, cy, cz;
            double fx, fy, fz;
            cell_frac((double)xn[3 * p + 0] * (double)n, n, &cx, &fx);
            cell_frac((double)xn[3 * p + 1] * (double)n, n, &cy, &fy);
            cell_frac((double)xn[3 * p + 2] * (double)n, n, &cz, &fz);
            const float *tab = tables + l * tsize * nfeat;
            for (int c = 0; c < 8; ++c) {
                int ox = (c >> 2) & 1, oy = (c >> 1) & 1, oz = c & 1;
                double w = (ox ? fx : 1.0 - fx) * (oy ? fy : 1.0 - fy);
                w = w * (oz ? fz : 1.0 - fz);
                int64_t r = corner_row(cx + ox, cy + oy, cz + oz, n, tsize);
                for (int64_t f = 0; f < nfeat; ++f) {
                    float *o = row + l * nfeat + f;
                    *o = (float)((double)*o + w * (double)tab[r * nfeat + f]);
                }
            }
        }
    }
}

void orc_interp_full(const float *xn, int64_t npts, const float *tables, int64_t nlev,
                     int64_t tsize, int64_t nfeat, const int64_t *res, int64_t n_active,
                     const float *inv_extent, float *feats, float *jac, int64_t *cidx,
                     float *cw, float *cdw, int nthreads)
{
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (int64_t p = 0; p < npts; ++p) {
        for (int64_t l = 0; l < n_active; ++l) {
            int64_t n = res[l];
            double sx = (double)n * (double)inv_extent[0];
            double sy = (double)n * (double)inv_extent[1];
            double sz = (double)n * (double)inv_extent[2];
            int64_t cx, cy, cz;
            double fx, fy, fz;
            cell_frac((double)xn[3 * p + 0] * (double)n, n, &cx, &fx);
            cell_frac((double)xn[3 * p + 1] * (double)n, n, &cy, &fy);
            cell_frac((double)xn[3 * p + 2] * (double)n, n, &cz, &fz);
            const float *tab = tables + l * tsize * nfeat;
            int64_t rec = (p * nlev + l) * 8;
            for (int c = 0; c < 8; ++c) {
                int ox = (c >> 2) & 1, oy = (c >> 1) & 1, oz = c & 1;
                double wx = ox ? fx : 1.0 - fx;
                double wy = oy ? fy : 1.0 - fy;
                double wz = oz ? fz : 1.0 - fz;
                double w = wx * wy * wz;
                double dwx = ox ? (wy * wz * sx) : (-wy * wz * sx);
                double dwy = oy ? (wx * wz * sy) : (-wx * wz * sy);
                double dwz = oz ? (wx * wy * sz) : (-wx * wy * sz);
                int64_t r = corner_row(cx + ox, cy + oy, cz + oz, n, tsize);
                cidx[rec + c] = r;
                cw[rec + c] = (float)w;
                cdw[(rec + c) * 3 + 0] = (float)dwx;
                cdw[(rec + c) * 3 + 1] = (float)dwy;
                cdw[(rec + c) * 3 + 2] = (float)dwz;
                for (int64_t f = 0; f < nfeat; ++f) {
                    double v = (double)tab[r * nfeat + f];
                    int64_t a = p * nlev * nfeat + l * nfeat + f;
                    feats[a] = (float)((double)feats[a] + w * v);
                    jac[3 * a + 0] = (float)((double)jac[3 * a + 0] + dwx * v);
                    jac[3 * a + 1] = (float)((double)jac[3 * a + 1] + dwy * v);
                    jac[3 * a + 2] = (float)((double)jac[3 * a + 2] + dwz * v);
                }
            }
        }
    }
}

void orc_scatter_first(float *grad, int64_t nlev, int64_t tsize, int64_t nfeat,
                       const int64_t *cidx, const float *cw, const float *dl_dfeat, int64_t npts,
                       int64_t n_active)
{
    for (int64_t p = 0; p < npts; ++p)
        for (int64_t l = 0; l < n_active; ++l)
            for (int c = 0; c < 8; ++c) {
                int64_t rec = (p * nlev + l) * 8 + c;
                float w = cw[rec];
                float *g = grad + (l * tsize + cidx[rec]) * nfeat;
                for (int64_t f = 0; f < nfeat; ++f) {
                    float prod = w * dl_dfeat[p * nlev * nfeat + l * nfeat + f];
                    g[f] = g[f] + prod;
                }
            }
}

void orc_scatter_second(float *grad, int64_t nlev, int64_t tsize, int64_t nfeat,
                        const int64_t *cidx, const float *cdw, const float *u, int64_t npts,
                        int64_t n_active)
{
    for (int64_t p = 0; p < npts; ++p)
        for (int64_t l = 0; l < n_active; ++l)
            for (int c = 0; c < 8; ++c) {
                int64_t rec = (p * nlev + l) * 8 + c;
                const float *dw = cdw + rec * 3;
                float *g = grad + (l * tsize + cidx[rec]) * nfeat;
                for (int64_t f = 0; f < nfeat; ++f) {
                    const float *uu = u + (p * nlev * nfeat + l * nfeat + f) * 3;
                    float a0 = uu[0] * dw[0];
                    float a1 = uu[1] * dw[1];
                    float a2 = uu[2] * dw[2];
                    float acc = (a0 + a1) + a2;
                    g[f] = g[f] + acc;
                }
            }
}

/* float ** int as numba lowers it: binary exponentiation in float64. */
void orc_hessian_contract(const float *xn, int64_t npts, const float *tables, int64_t nlev,
                          int64_t tsize, int64_t nfeat, const int64_t *res, int64_t n_active,
                          const float *inv_extent, const float *coeff, float *out, int nthreads)
{
#pragma omp parallel for schedule(static) num_threads(nthreads)
    for (int64_t p = 0; p < npts; ++p) {
        float *o = out + 9 * p;
        for (int k = 0; k < 9; ++k)
            o[k] = 0.0f;
        for (int64_t l = 0; l < n_active; ++l) {
            int64_t n = res[l];
            double sx = (double)n * (double)inv_extent[0];
            double sy = (double)n * (double)inv_extent[1];
            double sz = (double)n * (double)inv_extent[2];
            int64_t cx, cy, cz;
            double fx, fy, fz;
            cell_frac((double)xn[3 * p + 0] * (double)n, n, &cx, &fx);
            cell_frac((double)xn[3 * p + 1] * (double)n, n, &cy, &fy);
            cell_frac((double)xn[3 * p + 2] * (double)n, n, &cz, &fz);
            const float *tab = tables + l * tsize * nfeat;
            double hxy = 0.0, hxz = 0.0, hyz = 0.0;
            for (int c = 0; c < 8; ++c) {
                int ox = (c >> 2) & 1, oy = (c >> 1) & 1, oz = c & 1;
                double wx = ox ? fx : 1.0 - fx, wy = oy ? fy : 1.0 - fy, wz = oz ? fz : 1.0 - fz;
                double gx = ox ? 1.0 : -1.0, gy = oy ? 1.0 : -1.0, gz = oz ? 1.0 : -1.0;
                int64_t r = corner_row(cx + ox, cy + oy, cz + oz, n, tsize);
                double cv = 0.0;
                for (int64_t f = 0; f < nfeat; ++f) {
                    float prod = coeff[(p * nlev + l) * nfeat + f] * tab[r * nfeat + f];
                    cv += (double)prod;
                }
                hxy += cv * gx * gy * wz;
                hxz += cv * gx * gz * wy;
                hyz += cv * gy * gz * wx;
            }
            o[1] = (float)((double)o[1] + hxy * sx * sy);
            o[3] = (float)((double)o[3] + hxy * sx * sy);
            o[2] = (float)((double)o[2] + hxz * sx * sz);
            o[6] = (float)((double)o[6] + hxz * sx * sz);
            o[5] = (float)((double)o[5] + hyz * sy * sz);
            o[7] = (float)((double)o[7] + hyz * sy * sz);
        }
    }
}

static double int_pow(double a, int64_t e)
{
    int invert = e < 0;
    uint64_t k = invert ? (uint64_t)(-e) : (uint64_t)e;
    double r = 1.0;
    while (k) {
        if (k & 1)
            r *= a;
        k >>= 1;
        if (k)
            a *= a;
    }
    return invert ? 1.0 / r : r;
}

void orc_adam_step_f32(float *param, const float *grad, float *m, float *v, int64_t n, int64_t t,
                       double lr, double beta1, double beta2, double eps)
{
    double c1 = 1.0 - int_pow(beta1, t);
    double c2 = 1.0 - int_pow(beta2, t);
    for (int64_t i = 0; i < n; ++i) {
        double g = (double)grad[i];
        m[i] = (float)(beta1 * (double)m[i] + (1.0 - beta1) * g);
        v[i] = (float)(beta2 * (double)v[i] + (1.0 - beta2) * g * g);
        double step = lr * ((double)m[i] / c1) / (sqrt((double)v[i] / c2) + eps);
        param[i] = (float)((double)param[i] - step);
    }
}

void orc_adam_step_f64(double *param, const double *grad, double *m, double *v, int64_t n,
                       int64_t t, double lr, double beta1, double beta2, double eps)
{
    double c1 = 1.0 - int_pow(beta1, t);
    double c2 = 1.0 - int_pow(beta2, t);
    for (int64_t i = 0; i < n; ++i) {
        double g = grad[i];
        m[i] = beta1 * m[i] + (1.0 - beta1) * g;
        v[i] = beta2 * v[i] + (1.0 - beta2) * g * g;
        param[i] = param[i] - lr * (m[i] / c1) / (sqrt(v[i] / c2) + eps);
    }
}
