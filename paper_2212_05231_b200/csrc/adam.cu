// K6: divergence check + multi-group fused Adam over one flat fp32 parameter buffer
// (trainer.py:152-172, 243-278; _kernels.py:209-218).  fp64 math, fp32 storage,
// moments re-read after rounding exactly like the numba loop.
#include "common.cuh"

namespace ns2b {

constexpr int kMaxSeg = 16;

struct Segs {
    int n;
    int64_t off[kMaxSeg + 1];  // prefix of lengths (flattened index space)
    int64_t base[kMaxSeg];     // offset of the segment in the buffer
    double lr[kMaxSeg], c1[kMaxSeg], c2[kMaxSeg];
};

__global__ void finite_kernel(const float *__restrict__ g, Segs s, int32_t *__restrict__ flag) {
    const int64_t total = s.off[s.n];
    uint32_t bad = 0u;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        int k = 0;
        while (k + 1 < s.n && i >= s.off[k + 1]) ++k;
        const float v = g[s.base[k] + (i - s.off[k])];
        if (!isfinite(v)) bad |= 1u << k;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    if ((threadIdx.x & 31) == 0 && bad) atomicOr(flag, static_cast<int32_t>(bad));
}

// one element (the numba loop's arithmetic, op for op)
__device__ __forceinline__ void adam_elem(float &p, float g32, float &m, float &v, double lr, double c1, double c2,
                                          double b1, double b2, double eps) {
    const double g = static_cast<double>(g32);
    const float mi = static_cast<float>(__dadd_rn(__dmul_rn(b1, static_cast<double>(m)), __dmul_rn(1.0 - b1, g)));
    const float vi = static_cast<float>(
        __dadd_rn(__dmul_rn(b2, static_cast<double>(v)), __dmul_rn(__dmul_rn(1.0 - b2, g), g)));
    m = mi;
    v = vi;
    const double step = __ddiv_rn(__dmul_rn(lr, __ddiv_rn(static_cast<double>(mi), c1)),
                                  __dadd_rn(sqrt(__ddiv_rn(static_cast<double>(vi), c2)), eps));
    p = static_cast<float>(__dsub_rn(static_cast<double>(p), step));
}

// With 16-B aligned buffers, segments whose buffer offset is a multiple of 4 are walked 4 elements per thread with
// 16-B loads and stores (the table segment: all but ~9k of the parameters); the rest,
// and every segment's tail, element by element.  Same per-element arithmetic either way.
__global__ void adam_multi_kernel(float *__restrict__ param, const float *__restrict__ grad,
                                  float *__restrict__ m, float *__restrict__ v, Segs s, double b1,
                                  double b2, double eps, const int32_t *__restrict__ flag, bool vec_ok) {
    if (flag && *flag) return;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
    for (int k = 0; k < s.n; ++k) {
        const int64_t len = s.off[k + 1] - s.off[k], base = s.base[k];
        const double lr = s.lr[k], c1 = s.c1[k], c2 = s.c2[k];
        int64_t done = 0;
        if (vec_ok && (base & 3) == 0) {
            const int64_t n4 = len >> 2;
            float4 *p4 = reinterpret_cast<float4 *>(param + base);
            const float4 *g4 = reinterpret_cast<const float4 *>(grad + base);
            float4 *m4 = reinterpret_cast<float4 *>(m + base);
            float4 *v4 = reinterpret_cast<float4 *>(v + base);
            for (int64_t i = tid; i < n4; i += nth) {
                float4 pp = p4[i], mm = m4[i], vv = v4[i];
                const float4 gg = g4[i];
                adam_elem(pp.x, gg.x, mm.x, vv.x, lr, c1, c2, b1, b2, eps);
                adam_elem(pp.y, gg.y, mm.y, vv.y, lr, c1, c2, b1, b2, eps);
                adam_elem(pp.z, gg.z, mm.z, vv.z, lr, c1, c2, b1, b2, eps);
                adam_elem(pp.w, gg.w, mm.w, vv.w, lr, c1, c2, b1, b2, eps);
                p4[i] = pp;
                m4[i] = mm;
                v4[i] = vv;
            }
            done = n4 << 2;
        }
        for (int64_t i = done + tid; i < len; i += nth) {
            const int64_t j = base + i;
            float pp = param[j], mm = m[j], vv = v[j];
            adam_elem(pp, grad[j], mm, vv, lr, c1, c2, b1, b2, eps);
            param[j] = pp;
            m[j] = mm;
            v[j] = vv;
        }
    }
}

// sharpness_log (fp64 scalar): grad = raw * scale (renderer.py:358 multiplies by s)
__global__ void adam_scalar_kernel(double *p, const double *raw, double scale, double *m, double *v,
                                   double lr, double b1, double b2, double eps, double c1, double c2,
                                   const int32_t *flag, int32_t *flag_out, int bit) {
    const double g = raw[0] * scale;
    if (!isfinite(g)) {
        if (flag_out) atomicOr(flag_out, 1 << bit);
        return;
    }
    if (flag && *flag) return;
    const double mi = __dadd_rn(__dmul_rn(b1, m[0]), __dmul_rn(1.0 - b1, g));
    const double vi = __dadd_rn(__dmul_rn(b2, v[0]), __dmul_rn(__dmul_rn(1.0 - b2, g), g));
    m[0] = mi;
    v[0] = vi;
    p[0] = __dsub_rn(p[0], __ddiv_rn(__dmul_rn(lr, __ddiv_rn(mi, c1)), __dadd_rn(sqrt(__ddiv_rn(vi, c2)), eps)));
}

double int_pow(double a, int64_t e);

static int build_segs(Segs &s, const int64_t *off, const int64_t *len, int nseg) {
    NS2B_REQUIRE(nseg >= 1 && nseg <= kMaxSeg, "1..16 segments supported");
    s.n = nseg;
    s.off[0] = 0;
    for (int k = 0; k < nseg; ++k) {
        NS2B_REQUIRE(len[k] >= 0 && off[k] >= 0, "negative segment");
        s.base[k] = off[k];
        s.off[k + 1] = s.off[k] + len[k];
    }
    return NS2B_OK;
}

}  // namespace ns2b

using namespace ns2b;

extern "C" {

int ns2b_check_finite(const float *grad, const int64_t *seg_off, const int64_t *seg_len,
                      int32_t nseg, int32_t *flag, void *stream) {
    Segs s;
    int rc = build_segs(s, seg_off, seg_len, nseg);
    if (rc) return rc;
    if (s.off[s.n] == 0) return NS2B_OK;
    finite_kernel<<<grid_for(s.off[s.n], 256, kNumSMs * 8), 256, 0, as_stream(stream)>>>(grad, s, flag);
    return check_launch("check_finite");
}

int ns2b_adam_multi(float *param, const float *grad, float *m, float *v, const int64_t *seg_off,
                    const int64_t *seg_len, const double *seg_lr, const int64_t *seg_t,
                    int32_t nseg, double beta1, double beta2, double eps, const int32_t *flag,
                    void *stream) {
    Segs s;
    int rc = build_segs(s, seg_off, seg_len, nseg);
    if (rc) return rc;
    for (int k = 0; k < nseg; ++k) {
        NS2B_REQUIRE(seg_t[k] >= 1, "adam step counter must be >= 1");
        s.lr[k] = seg_lr[k];
        s.c1[k] = 1.0 - int_pow(beta1, seg_t[k]);
        s.c2[k] = 1.0 - int_pow(beta2, seg_t[k]);
    }
    if (s.off[s.n] == 0) return NS2B_OK;
    adam_multi_kernel<<<grid_for(s.off[s.n], 256, kNumSMs * 8), 256, 0, as_stream(stream)>>>(
        param, grad, m, v, s, beta1, beta2, eps, flag,
        ((reinterpret_cast<uintptr_t>(param) | reinterpret_cast<uintptr_t>(grad) | reinterpret_cast<uintptr_t>(m) |
          reinterpret_cast<uintptr_t>(v)) & 15u) == 0);
    return check_launch("adam_multi");
}

int ns2b_adam_scalar_f64(double *param, const double *raw_grad, double grad_scale, double *m,
                         double *v, int64_t t, double lr, double beta1, double beta2, double eps,
                         const int32_t *flag, int32_t *flag_out, int32_t flag_bit, void *stream) {
    NS2B_REQUIRE(t >= 1, "adam step counter must be >= 1");
    double c1 = 1.0 - int_pow(beta1, t), c2 = 1.0 - int_pow(beta2, t);
    adam_scalar_kernel<<<1, 1, 0, as_stream(stream)>>>(param, raw_grad, grad_scale, m, v, lr, beta1,
                                                        beta2, eps, c1, c2, flag, flag_out, flag_bit);
    return check_launch("adam_scalar");
}

}  // extern "C"
