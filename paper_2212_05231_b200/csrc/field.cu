// K2/K5: fused neural-field forward and backward (field.py:208-331), plus the lean
// SDF-only query and the occupancy refresh (renderer.py:108-142).
//
// Layout.  Every kernel works in a padded "36-wide" encoding space regardless of L:
// e_aug = [x(3), level features (32, zero beyond 2L), const 1], so one compiled kernel
// serves 1..16 levels.  The block prologue copies the MLP weights into shared memory
// in that padded layout (H1p 64x36, H2 16x64 + its transpose, C1p 64x28, C2 64x64,
// C3p 4x64); every per-sample mat-vec then reads weights as warp-broadcast LDS.128.
//
// Forward: thread per sample.  The hash gather writes the 32x3 feature Jacobian to
// shared memory (needed once the SDF net has produced j_d, for the normal).
// Backward: thread per sample, warps own 32-sample chunks of a persistent loop.  The
// forward is recomputed (no per-sample activations are stored between the passes),
// then colour bwd -> SDF first-order bwd -> fused first+second-order table scatter
// (one float2 RED per corner) -> Theorem-1 vectors.  The weight gradients are
// sum-over-samples outer products: each warp stages the per-sample vectors of its
// 32 samples in shared memory and reduces them as a 32-deep rank-k update into
// block-shared fp32 accumulators; the block flushes them with one global RED per
// element at exit.
#include "common.cuh"

#include <stdlib.h>
#include <string.h>

#include "field_common.cuh"

namespace ns2b {

// ------------------------------------------------------------ forward -----
constexpr int FWD_BLOCK = 128;

__global__ void __launch_bounds__(FWD_BLOCK)
field_forward_kernel(FieldDev f, const float *__restrict__ pos, const int32_t *__restrict__ ray_ids,
                     const double *__restrict__ dirs, const int32_t *__restrict__ count,
                     float *__restrict__ sdf, float *__restrict__ colors, float *__restrict__ normals,
                     float *__restrict__ geo, double *__restrict__ eik_sum) {
    extern __shared__ float4 smem4[];
    float *sw = reinterpret_cast<float *>(smem4);
    float *Js = sw + W_FLOATS;  // 96 x FWD_BLOCK
    load_weights(sw, f);
    __syncthreads();
    const int P = *count;
    float eik = 0.f;
    for (int64_t base = (int64_t)blockIdx.x * FWD_BLOCK; base < P; base += (int64_t)gridDim.x * FWD_BLOCK) {
        const int64_t p = base + threadIdx.x;
        if (p >= P) break;
        const float x0 = pos[3 * p], x1 = pos[3 * p + 1], x2 = pos[3 * p + 2];
        float e[EP];
        e[0] = x0;
        e[1] = x1;
        e[2] = x2;
        e[EC] = 1.f;
        float *jt = Js + threadIdx.x;
        gather_full(f, x0, x1, x2, e, jt, FWD_BLOCK);
        float y[NOUT], jd[EP];
        uint32_t mlo, mhi;
        sdf_forward<true>(sw, e, y, jd, mlo, mhi);
        float n0, n1, n2;
        normal_from(jd, jt, FWD_BLOCK, f.n_active, n0, n1, n2);
        const int r = ray_ids[p];
        float cin[CINP];
        cin[0] = x0;
        cin[1] = x1;
        cin[2] = x2;
        cin[3] = n0;
        cin[4] = n1;
        cin[5] = n2;
        cin[6] = static_cast<float>(dirs[3 * r]);
        cin[7] = static_cast<float>(dirs[3 * r + 1]);
        cin[8] = static_cast<float>(dirs[3 * r + 2]);
#pragma unroll
        for (int o = 0; o < NOUT; ++o) cin[9 + o] = y[o];
        cin[25] = cin[26] = cin[27] = 0.f;
        float a1[H];
        uint32_t clo, chi;
        color_layer1(sw, cin, a1, clo, chi);
        float l0 = 0.f, l1 = 0.f, l2 = 0.f;
#pragma unroll 4
        for (int k = 0; k < H; ++k) {
            float z = dot64(sw + OFF_C2 + k * H, a1);
            float a = z > 0.f ? z : 0.f;
            l0 = fmaf(sw[OFF_C3 + k], a, l0);
            l1 = fmaf(sw[OFF_C3 + H + k], a, l1);
            l2 = fmaf(sw[OFF_C3 + 2 * H + k], a, l2);
        }
        sdf[p] = y[0];
        colors[3 * p] = sigmoid_f(l0);
        colors[3 * p + 1] = sigmoid_f(l1);
        colors[3 * p + 2] = sigmoid_f(l2);
        if (normals) {
            normals[3 * p] = n0;
            normals[3 * p + 1] = n1;
            normals[3 * p + 2] = n2;
        }
        if (geo) {
#pragma unroll
            for (int o = 1; o < NOUT; ++o) geo[15 * p + o - 1] = y[o];
        }
        const float nn = sqrtf(n0 * n0 + n1 * n1 + n2 * n2) - 1.f;
        eik += nn * nn;
    }
    if (eik_sum) {
        double v = warp_sum(static_cast<double>(eik));
        if ((threadIdx.x & 31) == 0 && v != 0.0) atomicAdd(eik_sum, v);
    }
}

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
        double z = sharp * static_cast<double>(y[0]);
        z = fmin(fmax(z, -80.0), 80.0);
        double cdf;
        if (z >= 0.0) {
            cdf = 1.0 / (1.0 + exp(-z));
        } else {
            double ez = exp(z);
            cdf = ez / (1.0 + ez);
        }
        double dens = __dmul_rn(__dmul_rn(sharp, cdf), 1.0 - cdf);
        double prev = __dmul_rn(0.95, ema[c]);
        double v = fmax(dens, prev);
        ema[c] = v;
        bits[c] = __dmul_rn(v, step) > thresh ? 1 : 0;
    }
}

// ----------------------------------------------------------- backward -----
constexpr int BWD_BLOCK = 128;
constexpr int BWD_WARPS = BWD_BLOCK / 32;
constexpr int SROW = 132;  // staging row stride (floats): 4 * odd -> conflict-free LDS.128 rows

// acc[M x N] (row stride ldc) += sum_{s<32} A[s][a_off+m] * B[s][b_off+n]
// over the warp's 32 staged sample rows; M, N multiples of 4.  4x4 micro-tile per
// lane per step, accumulators folded into block shared memory with RED.shared.
__device__ __forceinline__ void warp_rank32(float *acc, int ldc, int M, int N, const float *stage,
                                            int a_off, int b_off, int lane) {
    const int tn = N >> 2;
    const int tiles = (M >> 2) * tn;
    for (int t = lane; t < tiles; t += 32) {
        const int m0 = (t / tn) << 2, n0 = (t % tn) << 2;
        float c[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) c[i][j] = 0.f;
#pragma unroll 8
        for (int s = 0; s < 32; ++s) {
            const float4 a = lds4(stage + s * SROW + a_off + m0);
            const float4 b = lds4(stage + s * SROW + b_off + n0);
            const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) c[i][j] = fmaf(av[i], bv[j], c[i][j]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (c[i][j] != 0.f) atomicAdd(acc + (m0 + i) * ldc + n0 + j, c[i][j]);
    }
}

__global__ void __launch_bounds__(BWD_BLOCK, 1)
field_backward_kernel(FieldDev f, const float *__restrict__ pos, const int32_t *__restrict__ ray_ids,
                      const double *__restrict__ dirs, const int32_t *__restrict__ count,
                      const float *__restrict__ dl_dc, const float *__restrict__ dl_dsdf,
                      const float *__restrict__ dl_dn_extra, float eik_w,
                      const int64_t *__restrict__ eik_count, float *__restrict__ g_sdf,
                      float *__restrict__ g_color, float *__restrict__ g_tab) {
    extern __shared__ float4 smem4[];
    float *sw = reinterpret_cast<float *>(smem4);
    float *gacc = sw + W_FLOATS;                 // G_FLOATS
    float *Js = gacc + G_FLOATS;                 // 96 x BWD_BLOCK
    float *Es = Js + 96 * BWD_BLOCK;             // EP x BWD_BLOCK (e_aug, column-major per thread)
    float *stage_all = Es + EP * BWD_BLOCK;      // BWD_WARPS x 32 x SROW
    load_weights(sw, f);
    for (int i = threadIdx.x; i < G_FLOATS; i += BWD_BLOCK) gacc[i] = 0.f;
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float *stage = stage_all + warp * 32 * SROW;
    float *my = stage + lane * SROW;  // this lane's staging row
    float *jt = Js + threadIdx.x;
    float *et = Es + threadIdx.x;
    const int P = *count;
    const float inv_p = eik_count ? 1.f / static_cast<float>(*eik_count) : 0.f;
    const float Pf = eik_count ? static_cast<float>(*eik_count) : 1.f;
    (void)inv_p;
    const int64_t stride = (int64_t)gridDim.x * BWD_BLOCK;

    for (int64_t base = (int64_t)blockIdx.x * BWD_BLOCK + warp * 32; base < P; base += stride) {
        const int64_t p = base + lane;
        const bool valid = p < P;
        float x0 = 0.f, x1 = 0.f, x2 = 0.f, v0 = 0.f, v1 = 0.f, v2 = 0.f;
        float gc0 = 0.f, gc1 = 0.f, gc2 = 0.f, gd = 0.f, gn0 = 0.f, gn1 = 0.f, gn2 = 0.f;
        if (valid) {
            x0 = pos[3 * p];
            x1 = pos[3 * p + 1];
            x2 = pos[3 * p + 2];
            const int r = ray_ids[p];
            v0 = static_cast<float>(dirs[3 * r]);
            v1 = static_cast<float>(dirs[3 * r + 1]);
            v2 = static_cast<float>(dirs[3 * r + 2]);
            gc0 = dl_dc[3 * p];
            gc1 = dl_dc[3 * p + 1];
            gc2 = dl_dc[3 * p + 2];
            gd = dl_dsdf[p];
            if (dl_dn_extra) {
                gn0 = dl_dn_extra[3 * p];
                gn1 = dl_dn_extra[3 * p + 1];
                gn2 = dl_dn_extra[3 * p + 2];
            }
        }
        // ---- recompute forward ----
        float e[EP];
        e[0] = x0;
        e[1] = x1;
        e[2] = x2;
        e[EC] = 1.f;
        gather_full(f, x0, x1, x2, e, jt, BWD_BLOCK);
#pragma unroll
        for (int i = 0; i < EP; ++i) et[i * BWD_BLOCK] = e[i];
        float y[NOUT], jd[EP];
        uint32_t mlo, mhi;
        sdf_forward<true>(sw, e, y, jd, mlo, mhi);
        float n0, n1, n2;
        normal_from(jd, jt, BWD_BLOCK, f.n_active, n0, n1, n2);
        // Eikonal cotangent (trainer.py:229-235), fp32 as numpy evaluates it.
        if (valid && eik_w != 0.f) {
            const float nn = sqrtf(n0 * n0 + n1 * n1 + n2 * n2);
            const float coef = eik_w * (2.f * (nn - 1.f) / fmaxf(nn, 1e-12f));
            gn0 += coef * n0 / Pf;
            gn1 += coef * n1 / Pf;
            gn2 += coef * n2 / Pf;
        }
        float cin[CINP];
        cin[0] = x0;
        cin[1] = x1;
        cin[2] = x2;
        cin[3] = n0;
        cin[4] = n1;
        cin[5] = n2;
        cin[6] = v0;
        cin[7] = v1;
        cin[8] = v2;
#pragma unroll
        for (int o = 0; o < NOUT; ++o) cin[9 + o] = y[o];
        cin[25] = cin[26] = cin[27] = 0.f;
        float dlg0, dlg1, dlg2;
        uint32_t clo, chi, c2lo = 0u, c2hi = 0u;
        {
            float a1[H];
            color_layer1(sw, cin, a1, clo, chi);
            float l0 = 0.f, l1 = 0.f, l2 = 0.f;
            __syncwarp();
#pragma unroll 4
            for (int k = 0; k < H; ++k) {
                const float z = dot64(sw + OFF_C2 + k * H, a1);
                const bool on = z > 0.f;
                const float a = on ? z : 0.f;
                if (on) {
                    if (k < 32) c2lo |= 1u << k;
                    else c2hi |= 1u << (k - 32);
                }
                l0 = fmaf(sw[OFF_C3 + k], a, l0);
                l1 = fmaf(sw[OFF_C3 + H + k], a, l1);
                l2 = fmaf(sw[OFF_C3 + 2 * H + k], a, l2);
                my[64 + k] = a;  // AC2 -> slot B
            }
            // dlogits = dl_dc * c * (1 - c) (field.py:304)
            const float c0 = sigmoid_f(l0), c1 = sigmoid_f(l1), c2 = sigmoid_f(l2);
            dlg0 = gc0 * c0 * (1.f - c0);
            dlg1 = gc1 * c1 * (1.f - c1);
            dlg2 = gc2 * c2 * (1.f - c2);
            my[0] = dlg0;
            my[1] = dlg1;
            my[2] = dlg2;
            my[3] = 0.f;
            __syncwarp();
            warp_rank32(gacc + G_C3, H, 4, H, stage, 0, 64, lane);  // dC3 += dlogits^T AC2
            __syncwarp();
            // u2 = (C3^T dlogits) . m2  -> slot B ; AC1 -> slot A
#pragma unroll
            for (int k = 0; k < H; ++k) {
                const float u = sw[OFF_C3 + k] * dlg0 + sw[OFF_C3 + H + k] * dlg1 + sw[OFF_C3 + 2 * H + k] * dlg2;
                my[64 + k] = mask_bit(c2lo, c2hi, k) ? u : 0.f;
                my[k] = a1[k];
            }
        }
        __syncwarp();
        warp_rank32(gacc + G_C2, H, H, H, stage, 64, 0, lane);  // dC2 += U2^T AC1
        __syncwarp();
        // u1 = (C2^T u2) . m1c
        float u1[H];
#pragma unroll
        for (int j = 0; j < H; ++j) u1[j] = 0.f;
#pragma unroll 2
        for (int k4 = 0; k4 < H; k4 += 4) {
            const float4 u2 = lds4(my + 64 + k4);
            const float uv[4] = {u2.x, u2.y, u2.z, u2.w};
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const float *c2 = sw + OFF_C2 + (k4 + kk) * H;
#pragma unroll
                for (int j = 0; j < H; j += 4) {
                    const float4 w = lds4(c2 + j);
                    u1[j] = fmaf(w.x, uv[kk], u1[j]);
                    u1[j + 1] = fmaf(w.y, uv[kk], u1[j + 1]);
                    u1[j + 2] = fmaf(w.z, uv[kk], u1[j + 2]);
                    u1[j + 3] = fmaf(w.w, uv[kk], u1[j + 3]);
                }
            }
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < H; ++j) {
            u1[j] = mask_bit(clo, chi, j) ? u1[j] : 0.f;
            my[64 + j] = u1[j];
        }
#pragma unroll
        for (int i = 0; i < CINP; ++i) my[i] = cin[i];
        __syncwarp();
        warp_rank32(gacc + G_C1, CINP, H, CINP, stage, 64, 0, lane);  // dC1 += U1^T CIN
        // dcin = C1^T u1
        float dcin[CINP];
#pragma unroll
        for (int i = 0; i < CINP; ++i) dcin[i] = 0.f;
#pragma unroll 4
        for (int j = 0; j < H; ++j) {
            const float *c1 = sw + OFF_C1 + j * CINP;
#pragma unroll
            for (int i = 0; i < CINP; i += 4) {
                const float4 w = lds4(c1 + i);
                dcin[i] = fmaf(w.x, u1[j], dcin[i]);
                dcin[i + 1] = fmaf(w.y, u1[j], dcin[i + 1]);
                dcin[i + 2] = fmaf(w.z, u1[j], dcin[i + 2]);
                dcin[i + 3] = fmaf(w.w, u1[j], dcin[i + 3]);
            }
        }
        // total normal / sdf / geometry cotangents (field.py:308-314)
        const float q0 = gn0 + dcin[3], q1 = gn1 + dcin[4], q2 = gn2 + dcin[5];
        float dly[NOUT];
        dly[0] = gd + dcin[9];
#pragma unroll
        for (int o = 1; o < NOUT; ++o) dly[o] = dcin[9 + o];
        // SDF first-order: u = (H2^T dl_dy) . m1 ; de = H1^T u
        float de[EP];
#pragma unroll
        for (int i = 0; i < EP; ++i) de[i] = 0.f;
        __syncwarp();
#pragma unroll 2
        for (int j = 0; j < H; ++j) {
            const float *h2t = sw + OFF_H2T + j * NOUT;
            float u = 0.f;
#pragma unroll
            for (int o = 0; o < NOUT; o += 4) {
                const float4 w = lds4(h2t + o);
                u = fmaf(w.x, dly[o], u);
                u = fmaf(w.y, dly[o + 1], u);
                u = fmaf(w.z, dly[o + 2], u);
                u = fmaf(w.w, dly[o + 3], u);
            }
            u = mask_bit(mlo, mhi, j) ? u : 0.f;
            my[j] = u;  // U -> slot A
            const float *h1 = sw + OFF_H1 + j * EP;
#pragma unroll
            for (int i = 0; i < EP; i += 4) {
                const float4 w = lds4(h1 + i);
                de[i] = fmaf(w.x, u, de[i]);
                de[i + 1] = fmaf(w.y, u, de[i + 1]);
                de[i + 2] = fmaf(w.z, u, de[i + 2]);
                de[i + 3] = fmaf(w.w, u, de[i + 3]);
            }
        }
        // mvec = [q, J q, 0] (field.py:326-327)
        float mv[EP];
        mv[0] = q0;
        mv[1] = q1;
        mv[2] = q2;
#pragma unroll
        for (int a = 0; a < 2 * NS2B_MAX_LEVELS; ++a) {
            const float *jr = jt + a * 3 * BWD_BLOCK;
            mv[3 + a] = (a < 2 * f.n_active) ? (jr[0] * q0 + jr[BWD_BLOCK] * q1 + jr[2 * BWD_BLOCK] * q2) : 0.f;
        }
        mv[EC] = 0.f;
        // ---- fused first + second order table scatter (Eq. 9) ----
        if (valid) {
            const float u0 = normalize_coord(x0, f.lo[0], f.ext[0]);
            const float uu1 = normalize_coord(x1, f.lo[1], f.ext[1]);
            const float u2 = normalize_coord(x2, f.lo[2], f.ext[2]);
#pragma unroll
            for (int l = 0; l < NS2B_MAX_LEVELS; ++l) {
                if (l < f.n_active) {
                    const LevelInfo lv = f.lv[l];
                    int cx, cy, cz;
                    float fx, fy, fz;
                    cell_frac(u0, lv.n, cx, fx);
                    cell_frac(uu1, lv.n, cy, fy);
                    cell_frac(u2, lv.n, cz, fz);
                    const float sx = f.sx[l], sy = f.sy[l], sz = f.sz[l];
                    const float de0 = de[3 + 2 * l], de1 = de[4 + 2 * l];
                    const float jd0 = jd[3 + 2 * l], jd1 = jd[4 + 2 * l];
                    float *gt = g_tab + l * f.T * 2;
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const int ox = (c >> 2) & 1, oy = (c >> 1) & 1, oz = c & 1;
                        const float wx = ox ? fx : 1.f - fx, wy = oy ? fy : 1.f - fy, wz = oz ? fz : 1.f - fz;
                        const float w = wx * wy * wz;
                        const float dwx = (ox ? sx : -sx) * (wy * wz);
                        const float dwy = (oy ? sy : -sy) * (wx * wz);
                        const float dwz = (oz ? sz : -sz) * (wx * wy);
                        const float qd = dwx * q0 + dwy * q1 + dwz * q2;
                        const uint32_t row = corner_row(lv, cx + ox, cy + oy, cz + oz);
                        red_add_f32x2(gt + 2 * row, fmaf(w, de0, jd0 * qd), fmaf(w, de1, jd1 * qd));
                    }
                }
            }
        }
        // ---- SDF weight gradients ----
        // slot B <- e_aug ; dH1 += U^T E
#pragma unroll
        for (int i = 0; i < EP; ++i) my[64 + i] = et[i * BWD_BLOCK];
        __syncwarp();
        warp_rank32(gacc + G_H1, EP, H, EP, stage, 0, 64, lane);
        __syncwarp();
        // slot A <- s1 = H2[0] . m1 ; slot B <- mvec ; dH1 += S1^T MV  (Theorem 1, l = 1)
#pragma unroll
        for (int j = 0; j < H; ++j) my[j] = mask_bit(mlo, mhi, j) ? sw[OFF_H2 + j] : 0.f;
#pragma unroll
        for (int i = 0; i < EP; ++i) my[64 + i] = mv[i];
        __syncwarp();
        warp_rank32(gacc + G_H1, EP, H, EP, stage, 0, 64, lane);
        __syncwarp();
        // slot A <- dl_dy (16) ; slot B <- a1 (recomputed from e_aug) ; dH2 += DLY^T A1
        float e2[EP];
#pragma unroll
        for (int i = 0; i < EP; ++i) e2[i] = et[i * BWD_BLOCK];
#pragma unroll
        for (int o = 0; o < NOUT; ++o) my[o] = dly[o];
#pragma unroll 2
        for (int j = 0; j < H; ++j) {
            const float *h1 = sw + OFF_H1 + j * EP;
            float z = 0.f;
#pragma unroll
            for (int i = 0; i < EP; i += 4) {
                const float4 w = lds4(h1 + i);
                z = fmaf(w.x, e2[i], z);
                z = fmaf(w.y, e2[i + 1], z);
                z = fmaf(w.z, e2[i + 2], z);
                z = fmaf(w.w, e2[i + 3], z);
            }
            my[64 + j] = mask_bit(mlo, mhi, j) ? z : 0.f;
        }
        __syncwarp();
        warp_rank32(gacc + G_H2, H, NOUT, H, stage, 0, 64, lane);
        __syncwarp();
        // Theorem 1, layer 2 (row 0 only): dH2[0] += pvec = (H1 mvec) . m1,
        // staged against the one-hot row e_0
        my[0] = 1.f;
        my[1] = my[2] = my[3] = 0.f;
#pragma unroll 2
        for (int j = 0; j < H; ++j) {
            const float *h1 = sw + OFF_H1 + j * EP;
            float zp = 0.f;
#pragma unroll
            for (int i = 0; i < EP; i += 4) {
                const float4 w = lds4(h1 + i);
                zp = fmaf(w.x, mv[i], zp);
                zp = fmaf(w.y, mv[i + 1], zp);
                zp = fmaf(w.z, mv[i + 2], zp);
                zp = fmaf(w.w, mv[i + 3], zp);
            }
            my[64 + j] = mask_bit(mlo, mhi, j) ? zp : 0.f;
        }
        __syncwarp();
        warp_rank32(gacc + G_H2, H, 4, H, stage, 0, 64, lane);
        __syncwarp();
    }
    __syncthreads();
    // flush block accumulators to the real (unpadded) gradient layouts
    const int E = 3 + 2 * f.L;
    for (int i = threadIdx.x; i < G_FLOATS; i += BWD_BLOCK) {
        const float v = gacc[i];
        if (v == 0.f) continue;
        if (i < G_H2) {
            const int j = i / EP, c = i % EP;
            const int dst = c < E ? c : (c == EC ? E : -1);
            if (dst >= 0) atomicAdd(g_sdf + j * (E + 1) + dst, v);
        } else if (i < G_C1) {
            atomicAdd(g_sdf + H * (E + 1) + (i - G_H2), v);
        } else if (i < G_C2) {
            const int r = i - G_C1, j = r / CINP, c = r % CINP;
            if (c < CIN) atomicAdd(g_color + j * CIN + c, v);
        } else if (i < G_C3) {
            atomicAdd(g_color + H * CIN + (i - G_C2), v);
        } else {
            const int r = i - G_C3;
            if (r < 3 * H) atomicAdd(g_color + H * CIN + H * H + r, v);
        }
    }
}

constexpr size_t FWD_SMEM = (W_FLOATS + 96 * FWD_BLOCK) * sizeof(float);
constexpr size_t SDF_SMEM = W_FLOATS * sizeof(float);
constexpr size_t BWD_SMEM =
    (W_FLOATS + G_FLOATS + 96 * BWD_BLOCK + EP * BWD_BLOCK + BWD_WARPS * 32 * SROW) * sizeof(float);

static int g_attr_done = 0;
static int ensure_attrs() {
    if (g_attr_done) return NS2B_OK;
    cudaError_t e = cudaFuncSetAttribute(field_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(FWD_SMEM));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(field_backward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(BWD_SMEM));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(field_sdf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
                      float *grad_color, float *grad_tables, void *workspace, cudaStream_t st);

// NS2B_FIELD_IMPL=simt selects the round-1 SIMT kernels for both passes (A/B
// comparison; default tcgen05); NS2B_FIELD_FWD / NS2B_FIELD_BWD override per pass.
static bool env_is_simt(const char *name) {
    const char *e = getenv(name);
    return e && strcmp(e, "simt") == 0;
}
static bool use_simt(bool bwd) {
    static int v[2] = {-1, -1};
    if (v[bwd] < 0) {
        const char *specific = bwd ? "NS2B_FIELD_BWD" : "NS2B_FIELD_FWD";
        const char *e = getenv(specific);
        v[bwd] = e ? (strcmp(e, "simt") == 0) : env_is_simt("NS2B_FIELD_IMPL");
    }
    return v[bwd] == 1;
}
}  // namespace ns2b

using namespace ns2b;

extern "C" {

int ns2b_field_forward(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids,
                       const double *dirs, const int32_t *count, int64_t capacity, float *sdf,
                       float *colors, float *normals, float *geo, double *eik_sum, void *workspace,
                       void *stream) {
    if (!use_simt(false))
        return field_forward_tc(field, pos32, ray_ids, dirs, count, capacity, sdf, colors, normals, geo, eik_sum,
                                workspace, as_stream(stream));
    FieldDev f;
    int rc = make_field_dev(field, f);
    if (rc) return rc;
    if ((rc = ensure_attrs())) return rc;
    if (capacity <= 0) return NS2B_OK;
    int blocks = grid_for(capacity, FWD_BLOCK, kNumSMs * 2);
    field_forward_kernel<<<blocks, FWD_BLOCK, FWD_SMEM, as_stream(stream)>>>(
        f, pos32, ray_ids, dirs, count, sdf, colors, normals, geo, eik_sum);
    return check_launch("field_forward");
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

int ns2b_field_backward(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids,
                        const double *dirs, const int32_t *count, int64_t capacity,
                        const float *dl_dc, const float *dl_dsdf, const float *dl_dn_extra,
                        double eik_weight, const int64_t *eik_count, float *grad_sdf,
                        float *grad_color, float *grad_tables, void *workspace, void *stream) {
    if (!use_simt(true))
        return field_backward_tc(field, pos32, ray_ids, dirs, count, capacity, dl_dc, dl_dsdf, dl_dn_extra,
                                 eik_weight, eik_count, grad_sdf, grad_color, grad_tables, workspace,
                                 as_stream(stream));
    FieldDev f;
    int rc = make_field_dev(field, f);
    if (rc) return rc;
    if ((rc = ensure_attrs())) return rc;
    NS2B_REQUIRE(eik_weight == 0.0 || eik_count != nullptr, "eik_count required with eik_weight");
    if (capacity <= 0) return NS2B_OK;
    int blocks = grid_for(capacity, BWD_BLOCK, kNumSMs);
    field_backward_kernel<<<blocks, BWD_BLOCK, BWD_SMEM, as_stream(stream)>>>(
        f, pos32, ray_ids, dirs, count, dl_dc, dl_dsdf, dl_dn_extra, static_cast<float>(eik_weight),
        eik_count, grad_sdf, grad_color, grad_tables);
    return check_launch("field_backward");
}

}  // extern "C"
