// K1: occupancy-grid ray marching (renderer.py:153-192), warp per ray.
//
// Bit-exactness: every fp64 operation of intersect_aabb / march_rays / bits_at is
// issued with an explicit round-to-nearest intrinsic so nvcc cannot contract a
// multiply-add into an FMA (the reference's numpy never fuses).  Counts, sample
// order and kept sets therefore equal the oracle's given the same occupancy bits.
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace ns2b {

struct OccArgs {
    int G;
    double lo[3], hi[3], ext[3], step;
    double scale[3];  // G / ext: the fast path of the cell index (see candidate)
    const uint8_t *bits;
};

static OccArgs make_occ(const ns2b_occ_t *o) {
    OccArgs a;
    a.G = o->resolution;
    for (int k = 0; k < 3; ++k) {
        a.lo[k] = o->lo[k];
        a.hi[k] = o->hi[k];
        a.ext[k] = o->hi[k] - o->lo[k];
        a.scale[k] = static_cast<double>(o->resolution) / a.ext[k];
    }
    a.step = o->step_size;
    a.bits = o->bits;
    return a;
}

// intersect_aabb (renderer.py:153-168) + candidate count (renderer.py:181-182).
__device__ __forceinline__ void ray_span(const OccArgs &g, const double *o, const double *d,
                                         double &t_enter, int &count) {
    double tn = -INFINITY, tf = INFINITY;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        double nk, fk;
        if (fabs(d[k]) < 1e-12) {
            bool inside = (o[k] >= g.lo[k]) && (o[k] <= g.hi[k]);
            nk = inside ? -INFINITY : INFINITY;
            fk = inside ? INFINITY : -INFINITY;
        } else {
            double inv = __ddiv_rn(1.0, d[k]);
            double a = __dmul_rn(__dsub_rn(g.lo[k], o[k]), inv);
            double b = __dmul_rn(__dsub_rn(g.hi[k], o[k]), inv);
            nk = fmin(a, b);
            fk = fmax(a, b);
        }
        tn = fmax(tn, nk);
        tf = fmin(tf, fk);
    }
    t_enter = fmax(tn, 0.0);
    double span = fmax(__dsub_rn(tf, t_enter), 0.0);
    double c = ceil(__ddiv_rn(span, g.step));
    count = c > 512.0 ? 512 : static_cast<int>(c);
}

// Candidate k: t = t_enter + (k+0.5)*dt, pos = o + t*d, cell = trunc((pos-lo)/ext*G)
// clipped (renderer.py:188-191, 98-102).
__device__ __forceinline__ bool candidate(const OccArgs &g, const double *o, const double *d,
                                          double t_enter, int k, double &t, double *pos) {
    t = __dadd_rn(t_enter, __dmul_rn(__dadd_rn(static_cast<double>(k), 0.5), g.step));
    int cell[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        pos[a] = __dadd_rn(o[a], __dmul_rn(t, d[a]));
        // the reference's cell index is trunc(((pos - lo) / ext) * G); (pos - lo) * (G / ext)
        // is within a few ulp of it (|u| <~ G: ~1e-13 absolute), so away from an integer
        // boundary its truncation is the same and the fp64 division is skipped
        const double du = __dsub_rn(pos[a], g.lo[a]);
        const double ua = __dmul_rn(du, g.scale[a]);
        const double fa = floor(ua);
        const double fr = __dsub_rn(ua, fa);
        long long ci;
        if (fr > 1e-9 && fr < 1.0 - 1e-9) {
            ci = static_cast<long long>(fa);  // == trunc(u) for u >= 0; u < 0 clamps to 0 either way
        } else {
            const double u = __dmul_rn(__ddiv_rn(du, g.ext[a]), static_cast<double>(g.G));
            ci = static_cast<long long>(u);  // astype(int64): truncation toward zero
        }
        ci = ci < 0 ? 0 : (ci > g.G - 1 ? g.G - 1 : ci);
        cell[a] = static_cast<int>(ci);
    }
    return g.bits[(static_cast<int64_t>(cell[0]) * g.G + cell[1]) * g.G + cell[2]] != 0;
}

// keep masks (optional): 16 words per ray, bit k of word w = candidate 32 w + k kept, so the
// fill pass computes positions for the kept candidates only (no second occupancy test)
constexpr int kMaskWords = 16;

__global__ void march_count_kernel(const double *__restrict__ origins, const double *__restrict__ dirs,
                                   int64_t nrays, OccArgs g, int32_t *__restrict__ counts,
                                   uint32_t *__restrict__ keep_mask) {
    const int lane = threadIdx.x & 31;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < nrays; r += nwarps) {
        double o[3] = {origins[3 * r], origins[3 * r + 1], origins[3 * r + 2]};
        double d[3] = {dirs[3 * r], dirs[3 * r + 1], dirs[3 * r + 2]};
        double t0;
        int n;
        ray_span(g, o, d, t0, n);
        int kept = 0;
        for (int base = 0; base < n; base += 32) {
            int k = base + lane;
            bool keep = false;
            if (k < n) {
                double t, pos[3];
                keep = candidate(g, o, d, t0, k, t, pos);
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, keep);
            if (keep_mask && lane == 0) keep_mask[r * kMaskWords + (base >> 5)] = bal;
            kept += __popc(bal);
        }
        if (lane == 0) counts[r] = kept;
    }
}

__global__ void march_fill_kernel(const double *__restrict__ origins, const double *__restrict__ dirs,
                                  int64_t nrays, OccArgs g, const int32_t *__restrict__ offsets,
                                  const uint32_t *__restrict__ keep_mask, int32_t *__restrict__ ray_ids,
                                  double *__restrict__ tout,
                                  double *__restrict__ pos64, float *__restrict__ pos32) {
    const int lane = threadIdx.x & 31;
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = warp; r < nrays; r += nwarps) {
        double o[3] = {origins[3 * r], origins[3 * r + 1], origins[3 * r + 2]};
        double d[3] = {dirs[3 * r], dirs[3 * r + 1], dirs[3 * r + 2]};
        double t0;
        int n;
        ray_span(g, o, d, t0, n);
        int64_t out = offsets[r];
        for (int base = 0; base < n; base += 32) {
            int k = base + lane;
            bool keep = false;
            double t = 0.0, pos[3] = {0.0, 0.0, 0.0};
            unsigned bal;
            if (keep_mask) {  // the count pass's verdicts: t and the position of kept candidates only
                bal = keep_mask[r * kMaskWords + (base >> 5)];
                keep = (bal >> lane) & 1u;
                if (keep) {
                    t = __dadd_rn(t0, __dmul_rn(__dadd_rn(static_cast<double>(k), 0.5), g.step));
#pragma unroll
                    for (int a = 0; a < 3; ++a) pos[a] = __dadd_rn(o[a], __dmul_rn(t, d[a]));
                }
            } else {
                if (k < n) keep = candidate(g, o, d, t0, k, t, pos);
                bal = __ballot_sync(0xffffffffu, keep);
            }
            if (keep) {
                int64_t s = out + __popc(bal & ((1u << lane) - 1u));
                ray_ids[s] = static_cast<int32_t>(r);
                if (tout) tout[s] = t;
                if (pos64) {
                    pos64[3 * s] = pos[0];
                    pos64[3 * s + 1] = pos[1];
                    pos64[3 * s + 2] = pos[2];
                }
                pos32[3 * s] = static_cast<float>(pos[0]);
                pos32[3 * s + 1] = static_cast<float>(pos[1]);
                pos32[3 * s + 2] = static_cast<float>(pos[2]);
            }
            out += __popc(bal);
        }
    }
}

}  // namespace ns2b

using namespace ns2b;

extern "C" {

int ns2b_march_count_masked(const double *origins, const double *dirs, int64_t nrays,
                            const ns2b_occ_t *occ, int32_t *counts, uint32_t *keep_mask, void *stream) {
    NS2B_REQUIRE(occ && occ->bits && occ->resolution > 0, "invalid occupancy grid");
    if (nrays == 0) return NS2B_OK;
    OccArgs g = make_occ(occ);
    int blocks = grid_for(nrays * 32, 256, kNumSMs * 16);
    march_count_kernel<<<blocks, 256, 0, as_stream(stream)>>>(origins, dirs, nrays, g, counts, keep_mask);
    return check_launch("march_count");
}

int ns2b_march_count(const double *origins, const double *dirs, int64_t nrays,
                     const ns2b_occ_t *occ, int32_t *counts, void *stream) {
    return ns2b_march_count_masked(origins, dirs, nrays, occ, counts, nullptr, stream);
}

int ns2b_scan_offsets(const int32_t *counts, int64_t nrays, int32_t *offsets, void *ws,
                      size_t *ws_bytes, void *stream) {
    NS2B_REQUIRE(ws_bytes != nullptr, "ws_bytes required");
    size_t need = 0;
    // inclusive scan into offsets[1..n]; offsets[0] = 0
    cudaError_t e = cub::DeviceScan::InclusiveSum(nullptr, need, counts, offsets + 1,
                                                  static_cast<int>(nrays), as_stream(stream));
    if (e != cudaSuccess) return set_error(NS2B_ECUDA, "scan sizing: %s", cudaGetErrorString(e));
    if (ws == nullptr) {
        *ws_bytes = need;
        return NS2B_OK;
    }
    NS2B_REQUIRE(*ws_bytes >= need, "scan workspace too small");
    e = cudaMemsetAsync(offsets, 0, sizeof(int32_t), as_stream(stream));
    if (e == cudaSuccess && nrays > 0)
        e = cub::DeviceScan::InclusiveSum(ws, need, counts, offsets + 1, static_cast<int>(nrays),
                                          as_stream(stream));
    count_launch();
    if (e != cudaSuccess) return set_error(NS2B_ECUDA, "scan: %s", cudaGetErrorString(e));
    return NS2B_OK;
}

int ns2b_march_fill_masked(const double *origins, const double *dirs, int64_t nrays,
                           const ns2b_occ_t *occ, const int32_t *offsets, const uint32_t *keep_mask,
                           int32_t *ray_ids, double *t, double *pos64, float *pos32, void *stream) {
    NS2B_REQUIRE(occ && occ->bits && occ->resolution > 0, "invalid occupancy grid");
    if (nrays == 0) return NS2B_OK;
    OccArgs g = make_occ(occ);
    int blocks = grid_for(nrays * 32, 256, kNumSMs * 16);
    march_fill_kernel<<<blocks, 256, 0, as_stream(stream)>>>(origins, dirs, nrays, g, offsets, keep_mask,
                                                             ray_ids, t, pos64, pos32);
    return check_launch("march_fill");
}

int ns2b_march_fill(const double *origins, const double *dirs, int64_t nrays,
                    const ns2b_occ_t *occ, const int32_t *offsets, int32_t *ray_ids, double *t,
                    double *pos64, float *pos32, void *stream) {
    return ns2b_march_fill_masked(origins, dirs, nrays, occ, offsets, nullptr, ray_ids, t, pos64, pos32,
                                  stream);
}

}  // extern "C"
