/*
 * ns2b.h — C ABI of the B200-native NeuS2 training hot path (libns2b.so).
 *
 * Plain pointers, sizes and scalars only; every pointer is a DEVICE pointer
 * (cudaMalloc / torch CUDA storage) unless stated otherwise, and every call is
 * asynchronous on the caller's `stream` (a cudaStream_t passed as void*).
 * Buffers are caller-owned; the library allocates nothing persistent.
 * Every entry point returns 0 on success or a negative NS2B_E* code; the
 * message of the last failure on the calling thread is ns2b_last_error().
 *
 * The entry points replace the reference package's two FFI seams
 * (reference = /root/reference/pkg/src/hashsdf):
 *   (1) the compiled array kernels of _kernels.py (numba) — same argument
 *       meaning, outputs written to caller buffers instead of returned;
 *   (2) the module-level renderer / field / trainer calls that train_step
 *       makes (renderer.py, field.py, trainer.py), as fused device kernels.
 * Citations are file:line into that package.
 */
#ifndef NS2B_H
#define NS2B_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define NS2B_API __attribute__((visibility("default")))
#else
#define NS2B_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define NS2B_ABI_VERSION 1

#define NS2B_OK 0
#define NS2B_EINVAL (-1)      /* bad argument / shape: the shim raises ValueError/ShapeError */
#define NS2B_ECUDA (-2)       /* CUDA runtime error (launch or earlier async fault)          */
#define NS2B_EUNSUPPORTED (-3) /* configuration outside the compiled kernels' envelope       */
#define NS2B_ENOSPACE (-4)    /* sample capacity exceeded (caller must grow its buffers)     */

#define NS2B_MAX_LEVELS 16
#define NS2B_HIDDEN 64
#define NS2B_GEO_DIM 15
#define NS2B_COLOR_IN 25

/* Hash-grid + MLP description shared by the field kernels.
 * tables: (L, T, 2) fp32, row-major (hash_encoding.py:48-109).
 * sdf_w:  H1 (64, E+1) then H2 (16, 64), E = 3 + 2L, row-major (field.py:92-95).
 * color_w: C1 (64, 25), C2 (64, 64), C3 (3, 64) (field.py:96).               */
typedef struct {
    int32_t num_levels;          /* L <= 16 */
    int32_t table_size;          /* T */
    int32_t features_per_level;  /* must be 2 */
    int32_t n_active;            /* active_level_count(max_level) (hash_encoding.py:132-138) */
    int32_t resolutions[NS2B_MAX_LEVELS];
    float aabb_min[3];           /* fp32 copies, as grid.normalize casts (hash_encoding.py:102-106) */
    float aabb_extent[3];
    float inv_extent[3];         /* fp32(1/extent) (hash_encoding.py:189) */
    int32_t hidden_width;        /* must be 64 */
    const float *tables;
    const float *sdf_w;
    const float *color_w;
} ns2b_field_t;

/* ---------------------------------------------------------------- errors -- */
NS2B_API const char *ns2b_last_error(void);
NS2B_API int ns2b_abi_version(void);
/* Number of kernel launches issued by this library since load (telemetry). */
NS2B_API uint64_t ns2b_launch_count(void);

/* ------------------------------------------- seam (1): _kernels.py arrays -- */
/* _kernels.interp_features (_kernels.py:40-64): out (P, L*2) fully written,
 * inactive levels zero. xn (P,3) fp32 in [0,1]; resolutions int64 (L,). */
NS2B_API int ns2b_interp_features(const float *xn, int64_t npts, const float *tables, int64_t nlev,
                         int64_t tsize, int64_t nfeat, const int64_t *resolutions,
                         int64_t n_active, float *out, void *stream);

/* _kernels.interp_full (_kernels.py:67-119): feats (P,L*2), jac (P,L*2,3),
 * cidx (P,L,8) int64, cw (P,L,8), cdw (P,L,8,3); all fully written. */
NS2B_API int ns2b_interp_full(const float *xn, int64_t npts, const float *tables, int64_t nlev,
                     int64_t tsize, int64_t nfeat, const int64_t *resolutions, int64_t n_active,
                     const float *inv_extent, float *feats, float *jac, int64_t *cidx, float *cw,
                     float *cdw, void *stream);

/* _kernels.scatter_first (_kernels.py:122-133): grad (L,T,2) += w * dL/dfeat. */
/* _kernels.hessian_contract (_kernels.py:159-206; hash_encoding.py:240-254): out (P,3,3)
 * fp32 = sum over active feature rows a of coeff[p,a] d2 e_a / dx dx, zero diagonal.
 * coeff (P, nlev*nfeat) fp32; xn normalised positions as for interp_full. */
NS2B_API int ns2b_hessian_contract(const float *xn, int64_t npts, const float *tables, int64_t nlev,
                                   int64_t tsize, int64_t nfeat, const int64_t *resolutions,
                                   int64_t n_active, const float *inv_extent, const float *coeff,
                                   float *out, void *stream);

NS2B_API int ns2b_scatter_first(float *grad, int64_t nlev, int64_t tsize, int64_t nfeat,
                       const int64_t *cidx, const float *cw, const float *dl_dfeat, int64_t npts,
                       int64_t n_active, void *stream);

/* _kernels.scatter_second (_kernels.py:136-156): grad += sum_k u[..,k] * cdw[..,k]. */
NS2B_API int ns2b_scatter_second(float *grad, int64_t nlev, int64_t tsize, int64_t nfeat,
                        const int64_t *cidx, const float *cdw, const float *u, int64_t npts,
                        int64_t n_active, void *stream);

/* _kernels.adam_step (_kernels.py:209-218) on flat views; fp64 math. */
NS2B_API int ns2b_adam_step_f32(float *param, const float *grad, float *m, float *v, int64_t n, int64_t t,
                       double lr, double beta1, double beta2, double eps, void *stream);
NS2B_API int ns2b_adam_step_f64(double *param, const double *grad, double *m, double *v, int64_t n,
                       int64_t t, double lr, double beta1, double beta2, double eps,
                       void *stream);

/* ------------------------------------ seam (2): renderer.py / field.py ---- */
/* Occupancy grid: bits uint8 (G,G,G) [x][y][z]; lo/hi fp64 aabb; step = ||hi-lo||/512
 * (renderer.py:72-105). */
typedef struct {
    int32_t resolution;
    double lo[3];
    double hi[3];
    double step_size;
    const uint8_t *bits;
} ns2b_occ_t;

/* Ray batch from pixel picks (scene_io.py:98-116,129-172).  picks[i] indexes
 * pool_first for i < n_first and pool_rest otherwise (the reference's foreground /
 * background draws); a pool entry is frame * H * W + y * W + x.  frames: per frame 16
 * doubles = R (row-major 3x3) | camera centre (3) | fx fy cx cy.  images (F,H,W,3) and
 * masks (F,H,W) uint8 (image = u8 / 255, mask 0/1).  Out (n,3) fp64: origins, unit
 * directions, targets image * mask. */
NS2B_API int ns2b_rays_from_picks(const int64_t *picks, int64_t n, int64_t n_first,
                                  const int32_t *pool_first, const int32_t *pool_rest,
                                  const double *frames, int32_t width, int32_t height,
                                  const uint8_t *images, const uint8_t *masks, double *origins,
                                  double *dirs, double *targets, void *stream);

/* march_rays pass 1 (renderer.py:153-192): kept-sample count per ray (fp64 slab test,
 * fixed-stride midpoints, <=512 candidates, occupancy bit test). */
NS2B_API int ns2b_march_count(const double *origins, const double *dirs, int64_t nrays,
                     const ns2b_occ_t *occ, int32_t *counts, void *stream);

/* Pass 1 that also records each ray's kept candidates (keep_mask: nrays x 16 uint32, bit
 * k of word w = candidate 32w + k), so ns2b_march_fill_masked computes the positions of
 * the kept candidates only.  Same counts as ns2b_march_count. */
NS2B_API int ns2b_march_count_masked(const double *origins, const double *dirs, int64_t nrays,
                                     const ns2b_occ_t *occ, int32_t *counts, uint32_t *keep_mask,
                                     void *stream);

/* Exclusive scan of counts -> offsets (nrays+1); offsets[nrays] = P.  Workspace
 * query: pass ws == NULL to receive the byte size in *ws_bytes. */
NS2B_API int ns2b_scan_offsets(const int32_t *counts, int64_t nrays, int32_t *offsets, void *ws,
                      size_t *ws_bytes, void *stream);

/* march_rays pass 2: ray-major, t-ascending samples.  t (fp64) and pos64 may be NULL;
 * pos32 = float32(position) is what the field consumes (field.py:216). */
NS2B_API int ns2b_march_fill(const double *origins, const double *dirs, int64_t nrays,
                    const ns2b_occ_t *occ, const int32_t *offsets, int32_t *ray_ids, double *t,
                    double *pos64, float *pos32, void *stream);

/* Pass 2 from pass 1's keep masks (same outputs as ns2b_march_fill, bit for bit). */
NS2B_API int ns2b_march_fill_masked(const double *origins, const double *dirs, int64_t nrays,
                                    const ns2b_occ_t *occ, const int32_t *offsets, const uint32_t *keep_mask,
                                    int32_t *ray_ids, double *t, double *pos64, float *pos32, void *stream);

/* eval_field forward (field.py:208-244) over the samples [0, *count): sdf d (P),
 * colors (P,3) and optionally normals (P,3), geometry feature g (P,15).  View directions
 * are dirs[ray_ids] cast to fp32.  eik_sum (fp64 scalar, accumulated) receives
 * sum_p (||n_p|| - 1)^2 (trainer.py:227-229); may be NULL.  count is a device int32. */
NS2B_API int ns2b_field_forward(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids,
                       const double *dirs, const int32_t *count, int64_t capacity, float *sdf,
                       float *colors, float *normals, float *geo, double *eik_sum, void *workspace,
                       void *stream);

/* Device workspace (bytes) the field kernels need for `capacity` samples: the gather
 * pass's pre-staged encoding tiles and d feature/dx, and the backward's scatter inputs.
 * ns2b_field_backward must get the workspace its matching ns2b_field_forward filled. */
NS2B_API int ns2b_field_workspace_bytes(int64_t capacity, size_t *bytes);

/* The four kernels ns2b_field_forward / ns2b_field_backward chain, as separate entry
 * points (same arguments): gather (features + d feature/dx, positions and fp32 view
 * directions -> workspace), the tcgen05 MLP forward, the tcgen05 MLP backward (weight
 * gradients + per-sample scatter inputs -> workspace) and the table-gradient scatter
 * (Eq. 9, warp-aggregated float2 REDs).  The MLP kernels take their per-sample inputs
 * from the workspace the gather filled (pos32/ray_ids/dirs are kept in their signatures
 * for the fused entry points). */
NS2B_API int ns2b_field_gather(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids,
                               const double *dirs, const int32_t *count, int64_t capacity,
                               void *workspace, void *stream);
NS2B_API int ns2b_field_mlp_forward(const ns2b_field_t *field, const float *pos32,
                                    const int32_t *ray_ids, const double *dirs,
                                    const int32_t *count, int64_t capacity, float *sdf,
                                    float *colors, float *normals, float *geo, double *eik_sum,
                                    void *workspace, void *stream);
/* ns2b_field_mlp_forward with the training step's Eikonal cotangent fused
 * (trainer.py:229-235: eik_weight 2 (|n| - 1) / max(|n|, 1e-12) n / *eik_count, fp32 in
 * numpy's order) where the normal is computed; the workspace then carries it in place of
 * the normal and ns2b_field_mlp_backward uses it instead of recomputing (its own
 * eik_weight / eik_count are then ignored).  The one-tile forward (NS2B_FWD=1) does not
 * fuse and the backward computes the term itself; the result is the same. */
NS2B_API int ns2b_field_mlp_forward_eik(const ns2b_field_t *field, const float *pos32,
                                        const int32_t *ray_ids, const double *dirs,
                                        const int32_t *count, int64_t capacity, float *sdf,
                                        float *colors, float *normals, float *geo, double *eik_sum,
                                        double eik_weight, const int64_t *eik_count,
                                        void *workspace, void *stream);
/* ns2b_field_gather + ns2b_field_mlp_forward_eik in one call.  With NS2B_FWD=3 in the
 * environment it is one kernel (field_fwd2_kernel<true>: the hash-grid gather inside the
 * two-tile MLP forward; E, d feature/dx, x and v still reach the workspace for the
 * backward) -- measured slower than the two kernels, so the default (and NS2B_FWD=1|2)
 * launches the gather kernel and then the one-tile | two-tile forward.  eik_count may be
 * NULL (no Eikonal fusion).  Results agree to the order of fp32 sums. */
NS2B_API int ns2b_field_forward_fused_eik(const ns2b_field_t *field, const float *pos32,
                                          const int32_t *ray_ids, const double *dirs,
                                          const int32_t *count, int64_t capacity, float *sdf,
                                          float *colors, float *normals, float *geo, double *eik_sum,
                                          double eik_weight, const int64_t *eik_count,
                                          void *workspace, void *stream);
NS2B_API int ns2b_field_mlp_backward(const ns2b_field_t *field, const float *pos32,
                                     const int32_t *ray_ids, const double *dirs,
                                     const int32_t *count, int64_t capacity, const float *dl_dc,
                                     const float *dl_dsdf, const float *dl_dn_extra,
                                     double eik_weight, const int64_t *eik_count,
                                     float *grad_sdf, float *grad_color, void *workspace,
                                     void *stream);
NS2B_API int ns2b_field_scatter(const ns2b_field_t *field, const float *pos32, const int32_t *count,
                                int64_t capacity, float *grad_tables, void *workspace,
                                void *stream);

/* field_backward(need_input_grads=True) (field.py:332-349) on the forward's workspace:
 * the tcgen05 MLP backward (weight gradients accumulated into grad_sdf / grad_color, as
 * ns2b_field_mlp_backward) additionally leaves each sample's colour-input x / v
 * cotangents and de_aug's position rows in the workspace, then one pass over the levels
 * gives dl_dx = dcin_x + de_x + sum_a de_a J_a + q Hess(j_d) (hessian_contract's
 * curvature) and dl_dv = dcin_v, (P,3) fp32 each.  No table gradients: run
 * ns2b_field_scatter on the same workspace for those. */
NS2B_API int ns2b_field_backward_inputs(const ns2b_field_t *field, const int32_t *count, int64_t capacity,
                                        const float *dl_dc, const float *dl_dsdf, const float *dl_dn_extra,
                                        double eik_weight, const int64_t *eik_count, float *grad_sdf,
                                        float *grad_color, float *dl_dx, float *dl_dv, void *workspace,
                                        void *stream);

/* Lean SDF-only query (renderer.py:131-142) on fp32 positions; d (P). */
NS2B_API int ns2b_field_sdf(const ns2b_field_t *field, const float *pos32, int64_t npts, float *sdf,
                   void *stream);

/* update_occupancy (renderer.py:108-128): SDF at every cell centre, logistic density,
 * ema = max(density, 0.95 ema), bits = ema*step > threshold.  ema fp64 (G^3). */
NS2B_API int ns2b_occupancy_update(const ns2b_field_t *field, const ns2b_occ_t *occ, double sharpness,
                          double threshold, double *ema, uint8_t *bits, void *stream);

/* The density / EMA / threshold half of update_occupancy from given per-cell SDF values
 * (ncells = G^3, C order), for update_occupancy(point_transform=...) where the caller
 * moves the cell centres and queries ns2b_field_sdf itself. */
NS2B_API int ns2b_occupancy_from_sdf(const float *sdf, int64_t ncells, double sharpness, double step_size,
                                     double threshold, double *ema, uint8_t *bits, void *stream);

/* Per-ray compositing (renderer.py:234-291) fused with the Huber colour loss and
 * its cotangent (trainer.py:96-112,215-221) and the compositing backward
 * (renderer.py:303-358).  Per sample: sdf, colors in; alphas/weights/trans_before
 * (fp64, per interval-first sample; NULL allowed), dl_dc (P,3) fp32 and dl_dsdf (P)
 * fp32 out.  Per ray: rendered (m,3) fp64, residual transmittance (m) fp64 (NULL ok).
 * targets may be NULL (forward only: no loss, no backward).
 * sums (fp64, accumulated): [0] sum_rays huber, [1] sum dL/dalpha*dalpha/ds, [2] sum of
 * squared colour error (for PSNR).  num_rays_total = global m: dL/dC = huber'(r)/m
 * (trainer.py:221). */
NS2B_API int ns2b_composite(const int32_t *offsets, int64_t nrays, const float *sdf, const float *colors,
                   double sharpness, const double *targets, double huber_delta,
                   double num_rays_total,
                   double *rendered, double *resid_trans, double *alphas, double *weights,
                   double *trans_before, float *dl_dc, float *dl_dsdf, double *sums,
                   void *stream);

/* Standalone backward_cotangents (renderer.py:303-358) from a given per-ray colour
 * cotangent dl_dray (m,3) fp64 and stored alphas/weights/trans_before. */
NS2B_API int ns2b_composite_backward(const int32_t *offsets, int64_t nrays, const float *sdf,
                            const float *colors, double sharpness, const double *alphas,
                            const double *weights, const double *trans_before,
                            const double *dl_dray, float *dl_dc, float *dl_dsdf, double *sums,
                            void *stream);

/* field_backward (field.py:272-331) fused with the Eikonal cotangent
 * (trainer.py:229-235): recomputes the forward per sample, then colour bwd, SDF
 * first-order bwd, Eq. 9 table scatter and the Theorem-1 (Eq. 10) SDF weight
 * gradients.  Accumulates into grad_sdf (H1|H2 layout), grad_color (C1|C2|C3),
 * grad_tables (L,T,2).  dl_dn_extra (P,3, may be NULL) is added to the Eikonal
 * normal cotangent; eik_weight/eik_count give dL/dn = w*2(|n|-1)/max(|n|,1e-12)*n/P
 * with P = *eik_count (device int64, the GLOBAL sample count); eik_weight = 0
 * disables the term. */
NS2B_API int ns2b_field_backward(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids,
                        const double *dirs, const int32_t *count, int64_t capacity,
                        const float *dl_dc, const float *dl_dsdf, const float *dl_dn_extra,
                        double eik_weight, const int64_t *eik_count, float *grad_sdf,
                        float *grad_color, float *grad_tables, void *workspace, void *stream);

/* Finite check over flat fp32 segments: flag |= 1<<seg for non-finite gradients
 * (trainer.py:158-159).  seg_off/seg_len are HOST arrays of nseg entries. */
NS2B_API int ns2b_check_finite(const float *grad, const int64_t *seg_off, const int64_t *seg_len,
                      int32_t nseg, int32_t *flag, void *stream);

/* Multi-group Adam (trainer.py:243-278 / _kernels.py:209-218) over one flat fp32
 * parameter buffer: segment s covers [off[s], off[s]+len[s]) with its own lr and
 * group step t[s].  Skips everything if *flag != 0 (divergence). Host arrays. */
NS2B_API int ns2b_adam_multi(float *param, const float *grad, float *m, float *v, const int64_t *seg_off,
                    const int64_t *seg_len, const double *seg_lr, const int64_t *seg_t,
                    int32_t nseg, double beta1, double beta2, double eps, const int32_t *flag,
                    void *stream);

/* Adam for the fp64 sharpness_log scalar: grad = raw_grad[0] * grad_scale
 * (renderer.py:358 returns sum * s).  A non-finite grad sets flag_out |= 1<<flag_bit and
 * skips; a nonzero *flag (earlier check) also skips.  Launch it before ns2b_adam_multi
 * with flag_out == flag so no group is updated when any gradient diverged. */
NS2B_API int ns2b_adam_scalar_f64(double *param, const double *raw_grad, double grad_scale, double *m,
                         double *v, int64_t t, double lr, double beta1, double beta2, double eps,
                         const int32_t *flag, int32_t *flag_out, int32_t flag_bit, void *stream);

/* ------------------------------------------------ in-run roofline probes -- */
/* L2 read sweep: `iters` passes of 16-B ld.global.cg over buf (nfloats % 4 == 0). */
NS2B_API int ns2b_bench_l2_read(const float *buf, int64_t nfloats, int32_t iters, float *sink,
                                void *stream);
/* nops random float2 REDs over nrows 8-B rows of buf (the scatter's access pattern). */
NS2B_API int ns2b_bench_red(float *buf, int64_t nrows, int64_t nops, uint32_t seed, void *stream);
/* nloads random 8-B row loads (ld.global.nc) over nrows rows of buf, 8 in flight per
 * thread: the hash gather's access pattern (useful bytes = 8 per load). */
NS2B_API int ns2b_bench_gather(const float *buf, int64_t nrows, int64_t nloads, uint32_t seed,
                               float *sink, void *stream);
/* nops float2 REDs, lane k of each warp on row base + k (full sectors): the L2 atomic
 * units' ceiling for the scatter. */
NS2B_API int ns2b_bench_red_coalesced(float *buf, int64_t nrows, int64_t nops, uint32_t seed,
                                      void *stream);

/* tcgen05 issue-rate probe (profiling aid, one CTA): `iters` kind::f16 MMAs of one of the
 * MLP kernels' shapes (0: M128 N64 K/MN, 1: M64 N16 MN/MN, 2: M64 N64 MN/MN, 3: M128
 * N16 K/K, 4: M64 N8 MN/MN, 5: M128 N64 K/K) rotating over nacc (1|2|4) accumulators;
 * *cycles (device int64) = clock64 cycles from first issue to commit completion. */
NS2B_API int ns2b_bench_umma(int32_t shape, int32_t iters, int32_t nacc, long long *cycles, void *stream);

/* tcgen05 building-block self-test (one CTA): mode 0: D[128x64] = A[128x48] B[64x48]^T
 * (f16 split, K-major/K-major); 1: D = A[128x48] B[48x64] (B MN-major); 2: D[64x48] =
 * U[128x64]^T V[128x48] (bf16, M=64, MN-major both); 3: mode 0 in bf16. fp32 in/out. */
NS2B_API int ns2b_selftest_umma(const float *A, const float *B, float *D, int32_t mode,
                                void *stream);

#ifdef __cplusplus
}
#endif
#endif /* NS2B_H */
