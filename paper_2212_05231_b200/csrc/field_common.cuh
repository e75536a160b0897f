// Shared device code of the field kernels (SIMT SDF queries: field.cu, tcgen05: field_tc.cu).
#pragma once

#include "common.cuh"

namespace ns2b {

constexpr int H = 64;        // hidden width
constexpr int EP = 36;       // padded e_aug width (3 + 32 + 1)
constexpr int EC = 35;       // const-channel column in the padded layout
constexpr int CIN = 25;      // colour-net input
constexpr int NOUT = 16;     // sdf-net outputs (d + 15 geometry features)

// shared-memory weight block of the SIMT SDF kernels (floats)
constexpr int OFF_H1 = 0;                       // 64 x 36
constexpr int OFF_H2 = OFF_H1 + H * EP;         // 16 x 64
constexpr int OFF_H2T = OFF_H2 + NOUT * H;      // 64 x 16
constexpr int W_FLOATS = OFF_H2T + H * NOUT;    // 4352

struct FieldDev {
    int L, n_active;
    int64_t T;
    LevelInfo lv[NS2B_MAX_LEVELS];
    float sx[NS2B_MAX_LEVELS], sy[NS2B_MAX_LEVELS], sz[NS2B_MAX_LEVELS];
    float lo[3], ext[3];
    const float *tables, *sdf_w, *color_w;
};

static inline int make_field_dev(const ns2b_field_t *f, FieldDev &d) {
    NS2B_REQUIRE(f != nullptr, "null field");
    NS2B_REQUIRE(f->num_levels >= 1 && f->num_levels <= NS2B_MAX_LEVELS,
                 "shape error: 1..16 levels supported (got %d)", f->num_levels);
    NS2B_REQUIRE(f->features_per_level == 2, "shape error: features_per_level must be 2");
    if (f->hidden_width != NS2B_HIDDEN)
        return set_error(NS2B_EUNSUPPORTED, "hidden_width %d unsupported (kernels are built for 64)",
                         f->hidden_width);
    NS2B_REQUIRE(f->n_active >= 0 && f->n_active <= f->num_levels, "n_active out of range");
    NS2B_REQUIRE(f->table_size >= 1, "table size must be positive");
    NS2B_REQUIRE(f->tables && f->sdf_w && f->color_w, "null parameter pointer");
    d.L = f->num_levels;
    d.n_active = f->n_active;
    d.T = f->table_size;
    for (int l = 0; l < NS2B_MAX_LEVELS; ++l) {
        int n = l < d.L ? f->resolutions[l] : 1;
        d.lv[l] = make_level(n, d.T);
        d.sx[l] = static_cast<float>(static_cast<double>(n) * f->inv_extent[0]);
        d.sy[l] = static_cast<float>(static_cast<double>(n) * f->inv_extent[1]);
        d.sz[l] = static_cast<float>(static_cast<double>(n) * f->inv_extent[2]);
    }
    for (int k = 0; k < 3; ++k) {
        d.lo[k] = f->aabb_min[k];
        d.ext[k] = f->aabb_extent[k];
    }
    d.tables = f->tables;
    d.sdf_w = f->sdf_w;
    d.color_w = f->color_w;
    return NS2B_OK;
}

// ------------------------------------------------------------ prologue ----
static __device__ void load_weights(float *sw, const FieldDev &f) {
    const int E = 3 + 2 * f.L;  // real encoding dim; H1 is (64, E+1)
    for (int i = threadIdx.x; i < W_FLOATS; i += blockDim.x) {
        float v = 0.f;
        if (i < OFF_H2) {
            int j = i / EP, c = i % EP;
            int src = c < E ? c : (c == EC ? E : -1);
            if (src >= 0) v = f.sdf_w[j * (E + 1) + src];
        } else if (i < OFF_H2T) {
            v = f.sdf_w[H * (E + 1) + (i - OFF_H2)];
        } else {
            int r = i - OFF_H2T, j = r / NOUT, o = r % NOUT;  // H2T[j][o] = H2[o][j]
            v = f.sdf_w[H * (E + 1) + o * H + j];
        }
        sw[i] = v;
    }
}

__device__ __forceinline__ float4 lds4(const float *p) { return *reinterpret_cast<const float4 *>(p); }

__device__ __forceinline__ float sigmoid_f(float z) {
    // two-branch logistic (field.py:40-46)
    if (z >= 0.f) return 1.f / (1.f + expf(-z));
    float ez = expf(z);
    return ez / (1.f + ez);
}

// ------------------------------------------------------------- gather -----
// Trilinear features of all active levels (_kernels.py:40-64); e[3..34] receives them.
__device__ __forceinline__ void gather_features(const FieldDev &f, float x0, float x1, float x2,
                                                float (&e)[EP]) {
    const float u0 = normalize_coord(x0, f.lo[0], f.ext[0]);
    const float u1 = normalize_coord(x1, f.lo[1], f.ext[1]);
    const float u2 = normalize_coord(x2, f.lo[2], f.ext[2]);
#pragma unroll
    for (int l = 0; l < NS2B_MAX_LEVELS; ++l) {
        float f0 = 0.f, f1 = 0.f;
        if (l < f.n_active) {
            const LevelInfo lv = f.lv[l];
            int cx, cy, cz;
            float fx, fy, fz;
            cell_frac(u0, lv.n, cx, fx);
            cell_frac(u1, lv.n, cy, fy);
            cell_frac(u2, lv.n, cz, fz);
            const float2 *tab = reinterpret_cast<const float2 *>(f.tables) + l * f.T;
            float2 v[8];
#pragma unroll
            for (int c = 0; c < 8; ++c)
                v[c] = __ldg(tab + corner_row(lv, cx + ((c >> 2) & 1), cy + ((c >> 1) & 1), cz + (c & 1)));
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int ox = (c >> 2) & 1, oy = (c >> 1) & 1, oz = c & 1;
                const float w = (ox ? fx : 1.f - fx) * (oy ? fy : 1.f - fy) * (oz ? fz : 1.f - fz);
                f0 = fmaf(w, v[c].x, f0);
                f1 = fmaf(w, v[c].y, f1);
            }
        }
        e[3 + 2 * l] = f0;
        e[4 + 2 * l] = f1;
    }
}

// -------------------------------------------------------- SDF forward -----
// y = H2 relu(H1 e_aug); j_d = (H2[0] . m1) H1  (relu_mlp.py:94-129, field.py:218-219).
// Returns the hidden mask as two 32-bit words.
template <bool kJd>
__device__ __forceinline__ void sdf_forward(const float *sw, const float (&e)[EP], float (&y)[NOUT],
                                            float (&jd)[EP], uint32_t &mlo, uint32_t &mhi) {
#pragma unroll
    for (int o = 0; o < NOUT; ++o) y[o] = 0.f;
    if (kJd) {
#pragma unroll
        for (int i = 0; i < EP; ++i) jd[i] = 0.f;
    }
    mlo = mhi = 0u;
#pragma unroll 2
    for (int j = 0; j < H; ++j) {
        const float *h1 = sw + OFF_H1 + j * EP;
        float z = 0.f;
#pragma unroll
        for (int i = 0; i < EP; i += 4) {
            float4 w = lds4(h1 + i);
            z = fmaf(w.x, e[i], z);
            z = fmaf(w.y, e[i + 1], z);
            z = fmaf(w.z, e[i + 2], z);
            z = fmaf(w.w, e[i + 3], z);
        }
        const bool on = z > 0.f;
        const float a = on ? z : 0.f;
        if (on) {
            if (j < 32) mlo |= 1u << j;
            else mhi |= 1u << (j - 32);
        }
        const float *h2t = sw + OFF_H2T + j * NOUT;
#pragma unroll
        for (int o = 0; o < NOUT; o += 4) {
            float4 w = lds4(h2t + o);
            y[o] = fmaf(w.x, a, y[o]);
            y[o + 1] = fmaf(w.y, a, y[o + 1]);
            y[o + 2] = fmaf(w.z, a, y[o + 2]);
            y[o + 3] = fmaf(w.w, a, y[o + 3]);
        }
        if (kJd) {
            const float s = on ? sw[OFF_H2 + j] : 0.f;  // H2[0][j] * m_j
#pragma unroll
            for (int i = 0; i < EP; i += 4) {
                float4 w = lds4(h1 + i);
                jd[i] = fmaf(s, w.x, jd[i]);
                jd[i + 1] = fmaf(s, w.y, jd[i + 1]);
                jd[i + 2] = fmaf(s, w.z, jd[i + 2]);
                jd[i + 3] = fmaf(s, w.w, jd[i + 3]);
            }
        }
    }
}

}  // namespace ns2b
