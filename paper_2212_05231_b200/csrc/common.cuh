// Shared device helpers for libns2b (sm_100a).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/ns2b.h"

namespace ns2b {

// ---------------------------------------------------------------- errors --
int set_error(int code, const char *fmt, ...);
int check_launch(const char *what);
void count_launch();

#define NS2B_REQUIRE(cond, ...)                                     \
    do {                                                            \
        if (!(cond)) return ::ns2b::set_error(NS2B_EINVAL, __VA_ARGS__); \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kNumSMs = 148;

inline int grid_for(int64_t n, int block, int max_blocks = kNumSMs * 32) {
    int64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return static_cast<int>(g);
}

// ------------------------------------------------------- hash grid math ----
// Lower-cell convention (_kernels.py:20-29): c = ceil(t)-1 clamped to [0, n-1],
// frac = t - c.  t = x*n is formed in fp64, where it is exact (24-bit x times
// n <= 2^12), so ceil() is the same integer the reference computes.
__device__ __forceinline__ void cell_frac(float xn, int n, int &c, float &frac) {
    double t = static_cast<double>(xn) * static_cast<double>(n);
    int ci = static_cast<int>(ceil(t)) - 1;
    ci = ci < 0 ? 0 : (ci > n - 1 ? n - 1 : ci);
    c = ci;
    frac = static_cast<float>(t - static_cast<double>(ci));
}

// Corner row (_kernels.py:32-37): dense row-major iff (n+1)^3 <= T, else the
// xor of the coordinates times (1, 2654435761, 805459861) with 64-bit products
// (numba widens uint32*uint32 to 64 bits) reduced modulo T.  For power-of-two T the
// low bits of the 64-bit products equal the 32-bit ones, so a 32-bit xor + mask is
// bit-identical.
struct LevelInfo {
    int n;        // resolution
    int dense;    // 1 if dense indexing
    uint32_t T;   // table size
    uint32_t mask;  // T-1 when power of two, else 0
};

__device__ __forceinline__ uint32_t corner_row(const LevelInfo &lv, int cx, int cy, int cz) {
    if (lv.dense) {
        uint32_t s = static_cast<uint32_t>(lv.n + 1);
        return static_cast<uint32_t>(cx) + s * (static_cast<uint32_t>(cy) + s * static_cast<uint32_t>(cz));
    }
    if (lv.mask) {
        uint32_t h = static_cast<uint32_t>(cx) ^ (static_cast<uint32_t>(cy) * 2654435761u) ^
                     (static_cast<uint32_t>(cz) * 805459861u);
        return h & lv.mask;
    }
    uint64_t h = static_cast<uint64_t>(static_cast<uint32_t>(cx)) ^
                 (static_cast<uint64_t>(static_cast<uint32_t>(cy)) * 2654435761ull) ^
                 (static_cast<uint64_t>(static_cast<uint32_t>(cz)) * 805459861ull);
    return static_cast<uint32_t>(h % static_cast<uint64_t>(lv.T));
}

__host__ __device__ inline LevelInfo make_level(int n, int64_t T) {
    LevelInfo lv;
    lv.n = n;
    int64_t s = static_cast<int64_t>(n) + 1;
    lv.dense = (s * s * s <= T) ? 1 : 0;
    lv.T = static_cast<uint32_t>(T);
    lv.mask = ((T & (T - 1)) == 0) ? static_cast<uint32_t>(T - 1) : 0u;
    return lv;
}

// grid.normalize (hash_encoding.py:102-106): fp32 IEEE sub / div, clip to [0,1].
__device__ __forceinline__ float normalize_coord(float x, float lo, float ext) {
    float v = __fdiv_rn(__fsub_rn(x, lo), ext);
    return fminf(fmaxf(v, 0.0f), 1.0f);
}

// Interpolation curvature of one level (_kernels.py:159-206): trilinear interpolation
// is linear per axis, so d2 feat/dx dx has a zero diagonal and mixed entries that are
// constant per cell.  With cv = sum_f coeff_f * corner_f (fp32 products summed in
// fp64, as numba types them), h_xy = sum_c cv * gx * gy * wz etc. in fp64 with fp64
// fractions; the caller scales by n*inv_extent and rounds into its fp32 output.
__device__ __forceinline__ void cell_frac_d(float xn, int n, int &c, double &frac) {
    double t = static_cast<double>(xn) * static_cast<double>(n);
    int ci = static_cast<int>(ceil(t)) - 1;
    ci = ci < 0 ? 0 : (ci > n - 1 ? n - 1 : ci);
    c = ci;
    frac = t - static_cast<double>(ci);
}

__device__ __forceinline__ void hess_from_corners(const float2 (&v)[8], double fx, double fy, double fz, float c0,
                                                  float c1, double &hxy, double &hxz, double &hyz) {
    hxy = hxz = hyz = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const int ox = (c >> 2) & 1, oy = (c >> 1) & 1, oz = c & 1;
        const double wx = ox ? fx : 1.0 - fx, wy = oy ? fy : 1.0 - fy, wz = oz ? fz : 1.0 - fz;
        const double cv = __dadd_rn(static_cast<double>(__fmul_rn(c0, v[c].x)),
                                    static_cast<double>(__fmul_rn(c1, v[c].y)));
        // gx*gy etc. are +-1: exact sign flips
        const double sxy = (ox ^ oy) ? -cv : cv, sxz = (ox ^ oz) ? -cv : cv, syz = (oy ^ oz) ? -cv : cv;
        hxy = __dadd_rn(hxy, __dmul_rn(sxy, wz));
        hxz = __dadd_rn(hxz, __dmul_rn(sxz, wy));
        hyz = __dadd_rn(hyz, __dmul_rn(syz, wx));
    }
}

__device__ __forceinline__ void hess_level(const float2 *__restrict__ tab, const LevelInfo &lv, float u0,
                                           float u1, float u2, float c0, float c1, double &hxy,
                                           double &hxz, double &hyz) {
    int cx, cy, cz;
    double fx, fy, fz;
    cell_frac_d(u0, lv.n, cx, fx);
    cell_frac_d(u1, lv.n, cy, fy);
    cell_frac_d(u2, lv.n, cz, fz);
    float2 v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c)
        v[c] = __ldg(tab + corner_row(lv, cx + ((c >> 2) & 1), cy + ((c >> 1) & 1), cz + (c & 1)));
    hess_from_corners(v, fx, fy, fz, c0, c1, hxy, hxz, hyz);
}

// out += h * s_a * s_b, the fp64 term rounded into the fp32 accumulator.
__device__ __forceinline__ float hess_acc(float out, double h, double sa, double sb) {
    return static_cast<float>(__dadd_rn(static_cast<double>(out), __dmul_rn(__dmul_rn(h, sa), sb)));
}

// ---------------------------------------------------------- misc device ----
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ void red_add_f32x2(float *addr, float a, float b) {
    atomicAdd(reinterpret_cast<float2 *>(addr), make_float2(a, b));
}

}  // namespace ns2b
