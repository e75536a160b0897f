// SDF-only field queries (renderer.py:108-142): the lean SDF evaluation and the
// occupancy refresh, thread per point (SIMT; no per-sample state is kept).  The
// training-step field kernels (gather, tcgen05 MLP forward / backward, table scatter)
// live in field_tc.cu; this file also holds their C-ABI entry points.
//
// Layout.  The SDF path works in a padded "36-wide" encoding space regardless of L:
// e_aug = [x(3), level features (32, zero beyond 2L), const 1], so one compiled kernel
// serves 1..16 levels; the block prologue copies the SDF weights into shared memory.
#include "common.cuh"

#include <stdlib.h>
#include <string.h>

#include "field_common.cuh"

namespace ns2b {

// ------------------------------------------------------------ forward -----
constexpr int FWD_BLOCK = 128;

// -------------------------------------------------------- SDF only --------
__global__ void __launch_bounds__(FWD_BLOCK)
field_sdf_kernel(FieldDev f, const float *__restrict__ pos, int64_t npts, float *__restrict__ sdf) {
    extern __shared__ float4 smem4[];
    float *sw = reinterpret_cast<float *>(smem4);
    load_weights(sw, f);
    __syncthreads();
    for (int64_t p = blockIdx.x * (int64_t)FWD_BLOCK + threadIdx.x; p < npts;
         p += (int64_t)gridDim.x * FWD_BLOCK) {
        float e[EP];
        e[0] = pos[3 * p];
        e[1] = pos[3 * p + 1];
        e[2] = pos[3 * p + 2];
        e[EC] = 1.f;
        gather_features(f, e[0], e[1], e[2], e);
        float y[NOUT], jd[EP];
        uint32_t mlo, mhi;
        sdf_forward<false>(sw, e, y, jd, mlo, mhi);
        sdf[p] = y[0];
    }
}

// Logistic density of one cell (renderer.py:35-49 sdf_transforms, fp64, stable
// branches), max-decay EMA and threshold (renderer.py:125-127).
__device__ __forceinline__ void occupancy_cell(float d, double sharp, double step, double thresh, double *ema,
                                               uint8_t *bit) {
    double z = sharp * static_cast<double>(d);
    z = fmin(fmax(z, -80.0), 80.0);
    double cdf;
    if (z >= 0.0) {
        cdf = 1.0 / (1.0 + exp(-z));
    } else {
        double ez = exp(z);
        cdf = ez / (1.0 + ez);
    }
    double dens = __dmul_rn(__dmul_rn(sharp, cdf), 1.0 - cdf);
    double prev = __dmul_rn(0.95, *ema);
    double v = fmax(dens, prev);
    *ema = v;
    *bit = __dmul_rn(v, step) > thresh ? 1 : 0;
}

// update_occupancy (renderer.py:108-128): centres lo + (i+0.5)*ext/G per axis (fp64),
// cast to fp32 for the field, logistic density in fp64, max-decay EMA, threshold.
__global__ void __launch_bounds__(FWD_BLOCK)
occupancy_kernel(FieldDev f, int G, double lo0, double lo1, double lo2, double e0, double e1,
                 double e2, double sharp, double step, double thresh, double *__restrict__ ema,
                 uint8_t *__restrict__ bits) {
    extern __shared__ float4 smem4[];
    float *sw = reinterpret_cast<float *>(smem4);
    load_weights(sw, f);
    __syncthreads();
    const int64_t n = (int64_t)G * G * G;
    for (int64_t c = blockIdx.x * (int64_t)FWD_BLOCK + threadIdx.x; c < n;
         c += (int64_t)gridDim.x * FWD_BLOCK) {
        const int ix = static_cast<int>(c / ((int64_t)G * G));
        const int iy = static_cast<int>((c / G) % G);
        const int iz = static_cast<int>(c % G);
        const double gd = static_cast<double>(G);
        double cx = __dadd_rn(lo0, __ddiv_rn(__dmul_rn(ix + 0.5, e0), gd));
        double cy = __dadd_rn(lo1, __ddiv_rn(__dmul_rn(iy + 0.5, e1), gd));
        double cz = __dadd_rn(lo2, __ddiv_rn(__dmul_rn(iz + 0.5, e2), gd));
        float e[EP];
        e[0] = static_cast<float>(cx);
        e[1] = static_cast<float>(cy);
        e[2] = static_cast<float>(cz);
        e[EC] = 1.f;
        gather_features(f, e[0], e[1], e[2], e);
        float y[NOUT], jd[EP];
        uint32_t mlo, mhi;
        sdf_forward<false>(sw, e, y, jd, mlo, mhi);
        occupancy_cell(y[0], sharp, step, thresh, ema + c, bits + c);
    }
}

// Same EMA / threshold from given SDF values (update_occupancy with a point_transform:
// the centres are moved on the host side of the API and queried with field_sdf).
__global__ void occupancy_from_sdf_kernel(const float *__restrict__ sdf, int64_t n, double sharp, double step,
                                          double thresh, double *__restrict__ ema, uint8_t *__restrict__ bits) {
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x)
        occupancy_cell(sdf[c], sharp, step, thresh, ema + c, bits + c);
}

// field_backward(need_input_grads=True) position / view cotangents (field.py:332-349),
// thread per sample, for the dynamic-scene transform optimiser.  Inputs are the
// forward's per-sample outputs (sdf, geo, normals, colors: the colour-net input is
// rebuilt from them exactly as eval_field formed it) and the three cotangents; the
// colour and SDF masks are recomputed from the weights (the nets are piecewise
// linear, so masks and weights are all the backward needs):
//   dcin = C1^T (m1 . C2^T (m2 . C3^T dlogits)),  dlogits = dl_dc c (1-c)
//   q = dl_dn + dcin[3:6],  dd = dl_dd + dcin[9],  dg = dcin[10:25]
//   de = H1^T (m . H2^T [dd, dg])          (= dd j_d + dg jg, field.py:336-341)
//   dl_dx = dcin[0:3] + de[:E] J + q Hess(j_d[3:E]),  dl_dv = dcin[6:9]
// de[:E] J = dd n + dg (jg J): the reference's two terms in one contraction.
__global__ void __launch_bounds__(FWD_BLOCK)
field_input_grads_kernel(FieldDev f, const float *__restrict__ pos, const int32_t *__restrict__ ray_ids,
                         const double *__restrict__ dirs, int64_t npts, const float *__restrict__ sdf,
                         const float *__restrict__ geo, const float *__restrict__ normals,
                         const float *__restrict__ colors, const float *__restrict__ dl_dc,
                         const float *__restrict__ dl_dd, const float *__restrict__ dl_dn, double ix, double iy,
                         double iz, float *__restrict__ dl_dx, float *__restrict__ dl_dv) {
    extern __shared__ float4 smem4[];
    float *sw = reinterpret_cast<float *>(smem4);
    load_weights(sw, f);
    __syncthreads();
    for (int64_t p = blockIdx.x * (int64_t)FWD_BLOCK + threadIdx.x; p < npts;
         p += (int64_t)gridDim.x * FWD_BLOCK) {
        const float x0 = pos[3 * p], x1 = pos[3 * p + 1], x2 = pos[3 * p + 2];
        float q0 = 0.f, q1 = 0.f, q2 = 0.f, dd = 0.f;
        if (dl_dn) {
            q0 = dl_dn[3 * p];
            q1 = dl_dn[3 * p + 1];
            q2 = dl_dn[3 * p + 2];
        }
        if (dl_dd) dd = dl_dd[p];
        float gx0 = 0.f, gx1 = 0.f, gx2 = 0.f, gv0 = 0.f, gv1 = 0.f, gv2 = 0.f;
        float dy[NOUT];
#pragma unroll
        for (int o = 0; o < NOUT; ++o) dy[o] = 0.f;
        if (dl_dc) {
            float cin[CINP];
            cin[0] = x0;
            cin[1] = x1;
            cin[2] = x2;
            cin[3] = normals[3 * p];
            cin[4] = normals[3 * p + 1];
            cin[5] = normals[3 * p + 2];
            const double *v = dirs + 3 * (int64_t)ray_ids[p];
            cin[6] = static_cast<float>(v[0]);
            cin[7] = static_cast<float>(v[1]);
            cin[8] = static_cast<float>(v[2]);
            cin[9] = sdf[p];
#pragma unroll
            for (int k = 0; k < NOUT - 1; ++k) cin[10 + k] = geo[(NOUT - 1) * p + k];
            cin[25] = cin[26] = cin[27] = 0.f;
            float a[H];
            uint32_t m1lo, m1hi, m2lo = 0u, m2hi = 0u;
            color_layer1(sw, cin, a, m1lo, m1hi);
#pragma unroll 1
            for (int j = 0; j < H; ++j) {
                if (dot64(sw + OFF_C2 + j * H, a) > 0.f) {
                    if (j < 32) m2lo |= 1u << j;
                    else m2hi |= 1u << (j - 32);
                }
            }
            float dl[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const float c = colors[3 * p + k];
                dl[k] = __fmul_rn(__fmul_rn(dl_dc[3 * p + k], c), __fsub_rn(1.f, c));
            }
#pragma unroll
            for (int i = 0; i < H; ++i) a[i] = 0.f;
#pragma unroll 1
            for (int j = 0; j < H; ++j) {
                if (!mask_bit(m2lo, m2hi, j)) continue;
                const float s = sw[OFF_C3 + j] * dl[0] + sw[OFF_C3 + H + j] * dl[1] + sw[OFF_C3 + 2 * H + j] * dl[2];
                const float *c2 = sw + OFF_C2 + j * H;
#pragma unroll
                for (int i = 0; i < H; i += 4) {
                    float4 w = lds4(c2 + i);
                    a[i] = fmaf(s, w.x, a[i]);
                    a[i + 1] = fmaf(s, w.y, a[i + 1]);
                    a[i + 2] = fmaf(s, w.z, a[i + 2]);
                    a[i + 3] = fmaf(s, w.w, a[i + 3]);
                }
            }
            float dc[CINP];
#pragma unroll
            for (int c = 0; c < CINP; ++c) dc[c] = 0.f;
#pragma unroll 1
            for (int j = 0; j < H; ++j) {
                const float s = mask_bit(m1lo, m1hi, j) ? a[j] : 0.f;
                const float *c1 = sw + OFF_C1 + j * CINP;
#pragma unroll
                for (int c = 0; c < CINP; c += 4) {
                    float4 w = lds4(c1 + c);
                    dc[c] = fmaf(s, w.x, dc[c]);
                    dc[c + 1] = fmaf(s, w.y, dc[c + 1]);
                    dc[c + 2] = fmaf(s, w.z, dc[c + 2]);
                    dc[c + 3] = fmaf(s, w.w, dc[c + 3]);
                }
            }
            gx0 = dc[0];
            gx1 = dc[1];
            gx2 = dc[2];
            q0 += dc[3];
            q1 += dc[4];
            q2 += dc[5];
            gv0 = dc[6];
            gv1 = dc[7];
            gv2 = dc[8];
            dd += dc[9];
#pragma unroll
            for (int k = 1; k < NOUT; ++k) dy[k] = dc[9 + k];
        }
        dy[0] = dd;
        // SDF forward (features, mask, j_d), then de = H1^T (m . H2^T dy)
        const float u0 = normalize_coord(x0, f.lo[0], f.ext[0]);
        const float u1 = normalize_coord(x1, f.lo[1], f.ext[1]);
        const float u2 = normalize_coord(x2, f.lo[2], f.ext[2]);
        // features, 4 levels (32 independent loads) in flight per thread, via shared memory
        float *fs = sw + W_FLOATS + threadIdx.x;
#pragma unroll 1
        for (int g = 0; g < f.n_active; g += 4) {
            float2 v[4][8];
            float fr[4][3];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int l = g + i;
                if (l < f.n_active) {
                    const LevelInfo lv = f.lv[l];
                    int cx, cy, cz;
                    cell_frac(u0, lv.n, cx, fr[i][0]);
                    cell_frac(u1, lv.n, cy, fr[i][1]);
                    cell_frac(u2, lv.n, cz, fr[i][2]);
                    const float2 *tab = reinterpret_cast<const float2 *>(f.tables) + l * f.T;
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        v[i][c] = __ldg(tab + corner_row(lv, cx + ((c >> 2) & 1), cy + ((c >> 1) & 1), cz + (c & 1)));
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int l = g + i;
                if (l < f.n_active) {
                    float f0 = 0.f, f1 = 0.f;
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const int ox = (c >> 2) & 1, oy = (c >> 1) & 1, oz = c & 1;
                        const float w = (ox ? fr[i][0] : 1.f - fr[i][0]) * (oy ? fr[i][1] : 1.f - fr[i][1]) *
                                        (oz ? fr[i][2] : 1.f - fr[i][2]);
                        f0 = fmaf(w, v[i][c].x, f0);
                        f1 = fmaf(w, v[i][c].y, f1);
                    }
                    fs[(2 * l) * FWD_BLOCK] = f0;
                    fs[(2 * l + 1) * FWD_BLOCK] = f1;
                }
            }
        }
        float e[EP];
        e[0] = x0;
        e[1] = x1;
        e[2] = x2;
        e[EC] = 1.f;
#pragma unroll
        for (int a = 0; a < 2 * NS2B_MAX_LEVELS; ++a) e[3 + a] = a < 2 * f.n_active ? fs[a * FWD_BLOCK] : 0.f;
        float y[NOUT], jd[EP];
        uint32_t mlo, mhi;
        sdf_forward<true>(sw, e, y, jd, mlo, mhi);
#pragma unroll
        for (int i = 0; i < EP; ++i) e[i] = 0.f;
#pragma unroll 1
        for (int j = 0; j < H; ++j) {
            if (!mask_bit(mlo, mhi, j)) continue;
            const float *h2t = sw + OFF_H2T + j * NOUT;
            float s = 0.f;
#pragma unroll
            for (int o = 0; o < NOUT; ++o) s = fmaf(h2t[o], dy[o], s);
            const float *h1 = sw + OFF_H1 + j * EP;
#pragma unroll
            for (int i = 0; i < EP; i += 4) {
                float4 w = lds4(h1 + i);
                e[i] = fmaf(s, w.x, e[i]);
                e[i + 1] = fmaf(s, w.y, e[i + 1]);
                e[i + 2] = fmaf(s, w.z, e[i + 2]);
                e[i + 3] = fmaf(s, w.w, e[i + 3]);
            }
        }
        gx0 += e[0];
        gx1 += e[1];
        gx2 += e[2];
        // per level: de . d feat/dx and the curvature term q Hess(j_d features); two levels
        // (16 independent loads) per iteration, one set of corner values for both terms
        float hxy = 0.f, hxz = 0.f, hyz = 0.f;
#pragma unroll 1
        for (int g = 0; g < f.n_active; g += 2) {
            float2 v[2][8];
            double fr[2][3];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int l = g + i;
                if (l < f.n_active) {
                    const LevelInfo lv = f.lv[l];
                    int cx, cy, cz;
                    cell_frac_d(u0, lv.n, cx, fr[i][0]);
                    cell_frac_d(u1, lv.n, cy, fr[i][1]);
                    cell_frac_d(u2, lv.n, cz, fr[i][2]);
                    const float2 *tab = reinterpret_cast<const float2 *>(f.tables) + l * f.T;
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        v[i][c] = __ldg(tab + corner_row(lv, cx + ((c >> 2) & 1), cy + ((c >> 1) & 1), cz + (c & 1)));
                }
            }
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int l = g + i;
                if (l < f.n_active) {
                    const float fx = static_cast<float>(fr[i][0]), fy = static_cast<float>(fr[i][1]),
                                fz = static_cast<float>(fr[i][2]);
                    const float sx = f.sx[l], sy = f.sy[l], sz = f.sz[l];
                    const float d0 = e[3 + 2 * l], d1 = e[4 + 2 * l];
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const int ox = (c >> 2) & 1, oy = (c >> 1) & 1, oz = c & 1;
                        const float wx = ox ? fx : 1.f - fx, wy = oy ? fy : 1.f - fy, wz = oz ? fz : 1.f - fz;
                        const float t = fmaf(d0, v[i][c].x, d1 * v[i][c].y);
                        gx0 = fmaf((ox ? sx : -sx) * (wy * wz), t, gx0);
                        gx1 = fmaf((oy ? sy : -sy) * (wx * wz), t, gx1);
                        gx2 = fmaf((oz ? sz : -sz) * (wx * wy), t, gx2);
                    }
                    double h01, h02, h12;
                    hess_from_corners(v[i], fr[i][0], fr[i][1], fr[i][2], jd[3 + 2 * l], jd[4 + 2 * l], h01, h02,
                                      h12);
                    const double n = static_cast<double>(f.lv[l].n);
                    const double dsx = n * ix, dsy = n * iy, dsz = n * iz;
                    hxy = hess_acc(hxy, h01, dsx, dsy);
                    hxz = hess_acc(hxz, h02, dsx, dsz);
                    hyz = hess_acc(hyz, h12, dsy, dsz);
                }
            }
        }
        dl_dx[3 * p] = gx0 + (q1 * hxy + q2 * hxz);
        dl_dx[3 * p + 1] = gx1 + (q0 * hxy + q2 * hyz);
        dl_dx[3 * p + 2] = gx2 + (q0 * hxz + q1 * hyz);
        dl_dv[3 * p] = gv0;
        dl_dv[3 * p + 1] = gv1;
        dl_dv[3 * p + 2] = gv2;
    }
}

constexpr size_t SDF_SMEM = W_FLOATS * sizeof(float);
constexpr size_t IG_SMEM = SDF_SMEM + 2 * NS2B_MAX_LEVELS * FWD_BLOCK * sizeof(float);  // + per-thread features

static int g_attr_done = 0;
static int ensure_attrs() {
    if (g_attr_done) return NS2B_OK;
    cudaError_t e = cudaFuncSetAttribute(field_sdf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(SDF_SMEM));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(field_input_grads_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(IG_SMEM));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(occupancy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(SDF_SMEM));
    if (e != cudaSuccess) return set_error(NS2B_ECUDA, "smem attribute: %s", cudaGetErrorString(e));
    g_attr_done = 1;
    return NS2B_OK;
}

}  // namespace ns2b

namespace ns2b {
int field_workspace_bytes(int64_t capacity, size_t *bytes);
int field_stage_tc(int which, const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids,
                   const double *dirs, const int32_t *count, int64_t capacity, float *sdf, float *colors,
                   float *normals, float *geo, double *eik_sum, const float *dl_dc, const float *dl_dsdf,
                   const float *dl_dn_extra, double eik_weight, const int64_t *eik_count, float *grad_sdf,
                   float *grad_color, float *grad_tables, void *workspace, cudaStream_t st);
int field_forward_tc(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids, const double *dirs,
                     const int32_t *count, int64_t capacity, float *sdf, float *colors, float *normals, float *geo,
                     double *eik_sum, void *workspace, cudaStream_t st);
int field_backward_tc(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids, const double *dirs,
                      const int32_t *count, int64_t capacity, const float *dl_dc, const float *dl_dsdf,
                      const float *dl_dn_extra, double eik_weight, const int64_t *eik_count, float *grad_sdf,
                      float *grad_color, float *grad_tables, void *workspace, cudaStream_t st);

}  // namespace ns2b

using namespace ns2b;

extern "C" {

int ns2b_field_forward(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids,
                       const double *dirs, const int32_t *count, int64_t capacity, float *sdf,
                       float *colors, float *normals, float *geo, double *eik_sum, void *workspace,
                       void *stream) {
    return field_forward_tc(field, pos32, ray_ids, dirs, count, capacity, sdf, colors, normals, geo, eik_sum,
                            workspace, as_stream(stream));
}

int ns2b_field_workspace_bytes(int64_t capacity, size_t *bytes) {
    return field_workspace_bytes(capacity, bytes);
}

int ns2b_field_gather(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids, const double *dirs,
                      const int32_t *count, int64_t capacity, void *workspace, void *stream) {
    NS2B_REQUIRE(pos32 && ray_ids && dirs && count, "field_gather: null input");
    return field_stage_tc(0, field, pos32, ray_ids, dirs, count, capacity, nullptr, nullptr, nullptr, nullptr,
                          nullptr, nullptr, nullptr, nullptr, 0.0, nullptr, nullptr, nullptr, nullptr, workspace,
                          as_stream(stream));
}

int ns2b_field_mlp_forward(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids,
                           const double *dirs, const int32_t *count, int64_t capacity, float *sdf,
                           float *colors, float *normals, float *geo, double *eik_sum, void *workspace,
                           void *stream) {
    return field_stage_tc(1, field, pos32, ray_ids, dirs, count, capacity, sdf, colors, normals, geo, eik_sum,
                          nullptr, nullptr, nullptr, 0.0, nullptr, nullptr, nullptr, nullptr, workspace,
                          as_stream(stream));
}

int ns2b_field_mlp_backward(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids,
                            const double *dirs, const int32_t *count, int64_t capacity, const float *dl_dc,
                            const float *dl_dsdf, const float *dl_dn_extra, double eik_weight,
                            const int64_t *eik_count, float *grad_sdf, float *grad_color, void *workspace,
                            void *stream) {
    return field_stage_tc(2, field, pos32, ray_ids, dirs, count, capacity, nullptr, nullptr, nullptr, nullptr,
                          nullptr, dl_dc, dl_dsdf, dl_dn_extra, eik_weight, eik_count, grad_sdf, grad_color,
                          nullptr, workspace, as_stream(stream));
}

int ns2b_field_scatter(const ns2b_field_t *field, const float *pos32, const int32_t *count, int64_t capacity,
                       float *grad_tables, void *workspace, void *stream) {
    return field_stage_tc(3, field, pos32, nullptr, nullptr, count, capacity, nullptr, nullptr, nullptr, nullptr,
                          nullptr, nullptr, nullptr, nullptr, 0.0, nullptr, nullptr, nullptr, grad_tables,
                          workspace, as_stream(stream));
}

int ns2b_field_sdf(const ns2b_field_t *field, const float *pos32, int64_t npts, float *sdf,
                   void *stream) {
    FieldDev f;
    int rc = make_field_dev(field, f);
    if (rc) return rc;
    if ((rc = ensure_attrs())) return rc;
    if (npts <= 0) return NS2B_OK;
    field_sdf_kernel<<<grid_for(npts, FWD_BLOCK, kNumSMs * 8), FWD_BLOCK, SDF_SMEM, as_stream(stream)>>>(
        f, pos32, npts, sdf);
    return check_launch("field_sdf");
}

int ns2b_occupancy_update(const ns2b_field_t *field, const ns2b_occ_t *occ, double sharpness,
                          double threshold, double *ema, uint8_t *bits, void *stream) {
    FieldDev f;
    int rc = make_field_dev(field, f);
    if (rc) return rc;
    if ((rc = ensure_attrs())) return rc;
    NS2B_REQUIRE(occ && occ->resolution > 0, "invalid occupancy grid");
    const int G = occ->resolution;
    int64_t n = (int64_t)G * G * G;
    occupancy_kernel<<<grid_for(n, FWD_BLOCK, kNumSMs * 8), FWD_BLOCK, SDF_SMEM, as_stream(stream)>>>(
        f, G, occ->lo[0], occ->lo[1], occ->lo[2], occ->hi[0] - occ->lo[0], occ->hi[1] - occ->lo[1],
        occ->hi[2] - occ->lo[2], sharpness, occ->step_size, threshold, ema, bits);
    return check_launch("occupancy_update");
}

int ns2b_occupancy_from_sdf(const float *sdf, int64_t ncells, double sharpness, double step_size,
                            double threshold, double *ema, uint8_t *bits, void *stream) {
    NS2B_REQUIRE(sdf && ema && bits, "occupancy_from_sdf: null argument");
    if (ncells <= 0) return NS2B_OK;
    occupancy_from_sdf_kernel<<<grid_for(ncells, 256), 256, 0, as_stream(stream)>>>(sdf, ncells, sharpness,
                                                                                   step_size, threshold, ema, bits);
    return check_launch("occupancy_from_sdf");
}

int ns2b_field_input_grads(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids,
                           const double *dirs, int64_t npts, const float *sdf, const float *geo,
                           const float *normals, const float *colors, const float *dl_dc, const float *dl_dd,
                           const float *dl_dn, float *dl_dx, float *dl_dv, void *stream) {
    FieldDev f;
    int rc = make_field_dev(field, f);
    if (rc) return rc;
    if ((rc = ensure_attrs())) return rc;
    NS2B_REQUIRE(pos32 && sdf && geo && normals && dl_dx && dl_dv, "field_input_grads: null argument");
    NS2B_REQUIRE(!dl_dc || (colors && ray_ids && dirs), "stale sample");
    if (npts <= 0) return NS2B_OK;
    field_input_grads_kernel<<<grid_for(npts, FWD_BLOCK, kNumSMs * 8), FWD_BLOCK, IG_SMEM,
                               as_stream(stream)>>>(f, pos32, ray_ids, dirs, npts, sdf, geo, normals, colors, dl_dc,
                                                    dl_dd, dl_dn, field->inv_extent[0], field->inv_extent[1],
                                                    field->inv_extent[2], dl_dx, dl_dv);
    return check_launch("field_input_grads");
}

int ns2b_field_backward(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids,
                        const double *dirs, const int32_t *count, int64_t capacity,
                        const float *dl_dc, const float *dl_dsdf, const float *dl_dn_extra,
                        double eik_weight, const int64_t *eik_count, float *grad_sdf,
                        float *grad_color, float *grad_tables, void *workspace, void *stream) {
    return field_backward_tc(field, pos32, ray_ids, dirs, count, capacity, dl_dc, dl_dsdf, dl_dn_extra, eik_weight,
                             eik_count, grad_sdf, grad_color, grad_tables, workspace, as_stream(stream));
}

}  // extern "C"
