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

constexpr size_t SDF_SMEM = W_FLOATS * sizeof(float);

static int g_attr_done = 0;
static int ensure_attrs() {
    if (g_attr_done) return NS2B_OK;
    cudaError_t e = cudaFuncSetAttribute(field_sdf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(SDF_SMEM));
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
                      float *grad_color, float *grad_tables, void *workspace, cudaStream_t st,
                      float *dl_dx = nullptr, float *dl_dv = nullptr);

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

int ns2b_field_mlp_forward_eik(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids,
                               const double *dirs, const int32_t *count, int64_t capacity, float *sdf,
                               float *colors, float *normals, float *geo, double *eik_sum, double eik_weight,
                               const int64_t *eik_count, void *workspace, void *stream) {
    return field_stage_tc(4, field, pos32, ray_ids, dirs, count, capacity, sdf, colors, normals, geo, eik_sum,
                          nullptr, nullptr, nullptr, eik_weight, eik_count, nullptr, nullptr, nullptr, workspace,
                          as_stream(stream));
}

int ns2b_field_forward_fused_eik(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids,
                                 const double *dirs, const int32_t *count, int64_t capacity, float *sdf,
                                 float *colors, float *normals, float *geo, double *eik_sum, double eik_weight,
                                 const int64_t *eik_count, void *workspace, void *stream) {
    return field_stage_tc(5, field, pos32, ray_ids, dirs, count, capacity, sdf, colors, normals, geo, eik_sum,
                          nullptr, nullptr, nullptr, eik_weight, eik_count, nullptr, nullptr, nullptr, workspace,
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

int ns2b_field_backward_inputs(const ns2b_field_t *field, const int32_t *count, int64_t capacity,
                               const float *dl_dc, const float *dl_dsdf, const float *dl_dn_extra, double eik_weight,
                               const int64_t *eik_count, float *grad_sdf, float *grad_color, float *dl_dx,
                               float *dl_dv, void *workspace, void *stream) {
    NS2B_REQUIRE(dl_dx && dl_dv, "field_backward_inputs: dl_dx / dl_dv required");
    return field_backward_tc(field, nullptr, nullptr, nullptr, count, capacity, dl_dc, dl_dsdf, dl_dn_extra,
                             eik_weight, eik_count, grad_sdf, grad_color, nullptr, workspace, as_stream(stream), dl_dx,
                             dl_dv);
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
