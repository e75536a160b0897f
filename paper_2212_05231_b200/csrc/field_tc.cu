// K2/K5 on the 5th-gen tensor cores: fused field forward / backward with tcgen05.
//
// One CTA = 128 threads = one 128-sample tile at a time (persistent loop); thread t
// owns sample t of the tile AND TMEM lane t, so every per-sample epilogue (ReLU,
// masks, normals, sigmoid, losses, scatter) is plain per-thread code on the rows that
// tcgen05.ld returns.  Every dense contraction is a UMMA issued by thread 0:
//
//   chain GEMMs (M = 128 samples):  operand tiles [sample][feature] (K-major A) x the
//     weights (K-major for W^T, MN-major view of the same tile for W), fp16 with the
//     three-term hi/lo split (A_hi B_hi + A_lo B_hi + A_hi B_lo, fp32 accumulation
//     in TMEM) -> fp32-level accuracy.
//   weight-gradient GEMMs (M = 64 weight rows, K = the 128 samples): MN-major views
//     of the same per-sample tiles; accumulated per tile in TMEM and folded into an
//     fp32 shared-memory accumulator (one global RED per element per CTA at exit).
//
// Cotangents span many binades (dL/dc ~ 1/m), so every cotangent tile is staged
// scaled by an exact per-tile power of two (the tile max lands in [2^13, 2^14)) and
// the GEMM results are multiplied back: exact, keeps fp16 hi/lo parts normal.
//
// Algorithm per tile (field.py:208-331, relu_mlp.py:94-216):
//   P0 gather features + d feature/dx (J -> TMEM);  Z1 = E H1^T
//   P1 a1 = relu(Z1), s1 = H2[0].m1;  Y = A1 H2^T,  JD = S1 H1          (j_d)
//   P2 n = j_d J; cin = [x,n,v,y];  Zc1 = CIN C1^T
//   P3 Zc2 = A1c C2^T;  P4 LOG = A2c C3^T;  P5 c = sigmoid  (forward ends here)
//   P5 dlogits -> U2 = DLOG C3,  dC3 += A2c^T DLOG
//   P6 u2 -> U1 = U2 C2,         dC2 += U2^T A1c
//   P7 u1 -> DCIN = U1 C1,       dC1 += U1^T CIN
//   P8 q, dly -> U = DLY H2,     dH2 += A1^T DLY
//   P9 u, mvec=[q,Jq,0] -> DE = U H1, PV = MV H1^T,  dH1 += U^T E + S1^T MV  (Thm 1)
//   P10 dH2[0] += sum pv (PV^T ONES);  fused first+second-order table scatter (Eq. 9)
//   P11 fold the per-tile weight gradients into shared fp32
#include "field_common.cuh"
#include "umma.cuh"

namespace ns2b {
namespace tc {

constexpr int TILE = 128;

// shared memory map (bytes); every tile is hi part then lo part
constexpr uint32_t WH1 = 0;                          // 64 x 48 f16
constexpr uint32_t WH1B = 64 * 48 * 2;
constexpr uint32_t WH2 = WH1 + 2 * WH1B;              // 16 x 64
constexpr uint32_t WH2B = 16 * 64 * 2;
constexpr uint32_t WC1 = WH2 + 2 * WH2B;              // 64 x 32
constexpr uint32_t WC1B = 64 * 32 * 2;
constexpr uint32_t WC2 = WC1 + 2 * WC1B;              // 64 x 64
constexpr uint32_t WC2B = 64 * 64 * 2;
constexpr uint32_t WC3 = WC2 + 2 * WC2B;              // 16 x 64
constexpr uint32_t WC3B = 16 * 64 * 2;
constexpr uint32_t TE = WC3 + 2 * WC3B;               // 128 x 48
constexpr uint32_t TEB = TILE * 48 * 2;
constexpr uint32_t TX = TE + 2 * TEB;                 // 128 x 64
constexpr uint32_t T64B = TILE * 64 * 2;
constexpr uint32_t TY = TX + 2 * T64B;
constexpr uint32_t TZ = TY + 2 * T64B;
constexpr uint32_t TC = TZ + 2 * T64B;                // 128 x 32
constexpr uint32_t TCB = TILE * 32 * 2;
constexpr uint32_t TD = TC + 2 * TCB;                 // 128 x 16
constexpr uint32_t TDB = TILE * 16 * 2;
constexpr uint32_t TEND = TD + 2 * TDB;
constexpr uint32_t GACC = TEND;                       // fp32 gradient accumulator (bwd)
constexpr int GACC_FLOATS = 9216;                     // 64*36 + 16*64 + 64*25 + 64*64 + 3*64
constexpr uint32_t SMEM_FWD = TEND;
constexpr uint32_t SMEM_BWD = GACC + GACC_FLOATS * 4;

// TMEM columns (512 allocated)
constexpr uint32_t TM_DC2 = 0, TM_DC1 = 64, TM_DC3 = 96, TM_DH2 = 112, TM_DH1 = 128;
constexpr uint32_t TM_J = 176, TM_Z1 = 272, TM_JD = 336, TM_SA = 384, TM_SB = 448;

// instruction descriptors
// Cotangent tiles are staged as v * 2^(kHead - G), G = exponent of the tile max, so the
// largest element lands in [2^13, 2^14) (< 65504) and small elements keep normal fp16
// hi/lo parts; results are multiplied back by 2^(G - kHead).
constexpr int kHead = 14;

constexpr uint32_t ID_KK(int N) { return umma::make_idesc(128, N, 0, 0, 0); }
constexpr uint32_t ID_KM(int N) { return umma::make_idesc(128, N, 0, 0, 1); }
constexpr uint32_t ID_WG(int N) { return umma::make_idesc(64, N, 0, 1, 1); }

__device__ __forceinline__ float pow2i(int e) {
    e = e < -120 ? -120 : (e > 120 ? 120 : e);
    return __int_as_float((127 + e) << 23);
}

struct Smem {
    uint8_t *base;
    __device__ uint8_t *p(uint32_t off) const { return base + off; }
    __device__ umma::Operand K(uint32_t off, uint32_t part, int C) const {
        return umma::kmajor(base + off, base + off + part, C);
    }
    __device__ umma::Operand MN(uint32_t off, uint32_t part, int C) const {
        return umma::mnmajor(base + off, base + off + part, C);
    }
};

template <int C>
__device__ __forceinline__ void stage(const Smem &s, uint32_t off, uint32_t part, int r, const float *v) {
    umma::stage_row<0, C>(s.p(off), s.p(off + part), r, v);
}

// weights -> fp16 hi/lo tiles in the padded 36-wide encoding layout (see field.cu)
__device__ void load_weight_tiles(const Smem &s, const FieldDev &f) {
    const int E = 3 + 2 * f.L;
    for (int r = threadIdx.x; r < 64 + 16 + 64 + 64 + 16; r += blockDim.x) {
        float row[64];
        if (r < 64) {
            for (int c = 0; c < 48; ++c) {
                int src = c < E ? c : (c == EC ? E : -1);
                row[c] = (c < EP && src >= 0) ? f.sdf_w[r * (E + 1) + src] : 0.f;
            }
            stage<48>(s, WH1, WH1B, r, row);
        } else if (r < 80) {
            const int o = r - 64;
            for (int c = 0; c < 64; ++c) row[c] = f.sdf_w[H * (E + 1) + o * H + c];
            stage<64>(s, WH2, WH2B, o, row);
        } else if (r < 144) {
            const int j = r - 80;
            for (int c = 0; c < 32; ++c) row[c] = c < CIN ? f.color_w[j * CIN + c] : 0.f;
            stage<32>(s, WC1, WC1B, j, row);
        } else if (r < 208) {
            const int k = r - 144;
            for (int c = 0; c < 64; ++c) row[c] = f.color_w[H * CIN + k * H + c];
            stage<64>(s, WC2, WC2B, k, row);
        } else {
            const int o = r - 208;
            for (int c = 0; c < 64; ++c) row[c] = o < 3 ? f.color_w[H * CIN + H * H + o * H + c] : 0.f;
            stage<64>(s, WC3, WC3B, o, row);
        }
    }
}

// gather (features into e, jacobian rows into J[96])
__device__ __forceinline__ void gather_regs(const FieldDev &f, float x0, float x1, float x2, float (&e)[EP],
                                            float (&J)[96]) {
    const float u0 = normalize_coord(x0, f.lo[0], f.ext[0]);
    const float u1 = normalize_coord(x1, f.lo[1], f.ext[1]);
    const float u2 = normalize_coord(x2, f.lo[2], f.ext[2]);
#pragma unroll
    for (int l = 0; l < NS2B_MAX_LEVELS; ++l) {
        float f0 = 0.f, f1 = 0.f, j00 = 0.f, j01 = 0.f, j02 = 0.f, j10 = 0.f, j11 = 0.f, j12 = 0.f;
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
            const float sx = f.sx[l], sy = f.sy[l], sz = f.sz[l];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int ox = (c >> 2) & 1, oy = (c >> 1) & 1, oz = c & 1;
                const float wx = ox ? fx : 1.f - fx, wy = oy ? fy : 1.f - fy, wz = oz ? fz : 1.f - fz;
                const float w = wx * wy * wz;
                const float dwx = (ox ? sx : -sx) * (wy * wz);
                const float dwy = (oy ? sy : -sy) * (wx * wz);
                const float dwz = (oz ? sz : -sz) * (wx * wy);
                f0 = fmaf(w, v[c].x, f0);
                f1 = fmaf(w, v[c].y, f1);
                j00 = fmaf(dwx, v[c].x, j00);
                j01 = fmaf(dwy, v[c].x, j01);
                j02 = fmaf(dwz, v[c].x, j02);
                j10 = fmaf(dwx, v[c].y, j10);
                j11 = fmaf(dwy, v[c].y, j11);
                j12 = fmaf(dwz, v[c].y, j12);
            }
        }
        e[3 + 2 * l] = f0;
        e[4 + 2 * l] = f1;
        J[6 * l + 0] = j00;
        J[6 * l + 1] = j01;
        J[6 * l + 2] = j02;
        J[6 * l + 3] = j10;
        J[6 * l + 4] = j11;
        J[6 * l + 5] = j12;
    }
}

__device__ __forceinline__ void block_sync_tc() {
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
}

// make this thread's staged smem visible to the tensor core and rendezvous
__device__ __forceinline__ void publish() {
    umma::fence_async_smem();
    block_sync_tc();
}

__device__ __forceinline__ void wait_mma(uint64_t *mbar, uint32_t &phase) {
    umma::mbar_wait(mbar, phase);
    phase ^= 1u;
    umma::fence_after_sync();
}

// exponent G of the tile-wide max |v| (max in [2^(G-1), 2^G)); all threads call it
__device__ __forceinline__ int tile_exponent(float rowmax, uint32_t *red) {
    uint32_t b = __reduce_max_sync(0xffffffffu, __float_as_uint(fabsf(rowmax)));
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) red[warp] = b;
    __syncthreads();
    uint32_t m = max(max(red[0], red[1]), max(red[2], red[3]));
    __syncthreads();
    float mv = __uint_as_float(m);
    int e = 0;
    if (mv > 0.f && mv < INFINITY) frexpf(mv, &e);
    return e;
}

template <int N>
__device__ __forceinline__ float absmax(const float *v) {
    float m = 0.f;
#pragma unroll
    for (int i = 0; i < N; ++i) m = fmaxf(m, fabsf(v[i]));
    return m;
}

template <bool kBwd>
__global__ void __launch_bounds__(TILE, 1)
field_tc_kernel(FieldDev f, const float *__restrict__ pos, const int32_t *__restrict__ ray_ids,
                const double *__restrict__ dirs, const int32_t *__restrict__ count,
                float *__restrict__ sdf_out, float *__restrict__ col_out, float *__restrict__ nrm_out,
                float *__restrict__ geo_out, double *__restrict__ eik_sum,
                const float *__restrict__ dl_dc, const float *__restrict__ dl_dsdf,
                const float *__restrict__ dl_dn_extra, float eik_w, const int64_t *__restrict__ eik_count,
                float *__restrict__ g_sdf, float *__restrict__ g_color, float *__restrict__ g_tab) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base_s;
    __shared__ uint32_t red[4];
    __shared__ float h2row0[H];
    const Smem S{smem_raw};
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int E = 3 + 2 * f.L;

    load_weight_tiles(S, f);
    if (t < H) h2row0[t] = f.sdf_w[H * (E + 1) + t];
    float *gacc = reinterpret_cast<float *>(S.p(GACC));
    if (kBwd)
        for (int i = t; i < GACC_FLOATS; i += TILE) gacc[i] = 0.f;
    if (t == 0) {
        umma::mbar_init(&mbar, 1);
        umma::fence_barrier_init();
    }
    if (warp == 0) umma::tmem_alloc(&tmem_base_s, 512);
    publish();
    const uint32_t tb = tmem_base_s;
    const uint32_t my = tb + (static_cast<uint32_t>(warp * 32) << 16);  // this warp's lane quadrant
    uint32_t phase = 0;
    const int P = *count;
    const float Pf = (kBwd && eik_count) ? static_cast<float>(*eik_count) : 1.f;
    // gradient layout offsets inside gacc (= the flat parameter layout's MLP prefix)
    const int G_H1r = 0, G_H2r = H * (E + 1), G_C1r = G_H2r + NOUT * H, G_C2r = G_C1r + H * CIN,
              G_C3r = G_C2r + H * H;
    float eik = 0.f;

    for (int64_t base = static_cast<int64_t>(blockIdx.x) * TILE; base < P;
         base += static_cast<int64_t>(gridDim.x) * TILE) {
        const int64_t p = base + t;
        const bool valid = p < P;
        float x0 = 0.f, x1 = 0.f, x2 = 0.f, v0 = 0.f, v1 = 0.f, v2 = 0.f;
        if (valid) {
            x0 = pos[3 * p];
            x1 = pos[3 * p + 1];
            x2 = pos[3 * p + 2];
            const int r = ray_ids[p];
            v0 = static_cast<float>(dirs[3 * r]);
            v1 = static_cast<float>(dirs[3 * r + 1]);
            v2 = static_cast<float>(dirs[3 * r + 2]);
        }
        // ------------------------------------------------ P0: gather, Z1
        {
            float e[EP], J[96];
            gather_regs(f, x0, x1, x2, e, J);
            e[0] = x0;
            e[1] = x1;
            e[2] = x2;
            e[EC] = 1.f;
            float row[48];
#pragma unroll
            for (int i = 0; i < 48; ++i) row[i] = i < EP ? e[i] : 0.f;
            stage<48>(S, TE, TEB, t, row);
#pragma unroll
            for (int c = 0; c < 96; c += 16) umma::tmem_st16(my + TM_J + c, J + c);
            umma::tmem_st_wait();
        }
        publish();
        if (t == 0) {
            umma::gemm3(tb + TM_Z1, S.K(TE, TEB, 48), S.K(WH1, WH1B, 48), 3, ID_KK(64), false);
            umma::commit(&mbar);
        }
        wait_mma(&mbar, phase);
        // ------------------------------------------------ P1: a1, s1 -> Y, JD
        uint32_t mlo = 0u, mhi = 0u;
        {
            float z[64];
            umma::tmem_ld<64>(my + TM_Z1, z);
            float a[64], s1[64];
#pragma unroll
            for (int j = 0; j < 64; ++j) {
                const bool on = z[j] > 0.f;
                if (on) {
                    if (j < 32) mlo |= 1u << j;
                    else mhi |= 1u << (j - 32);
                }
                a[j] = on ? z[j] : 0.f;
                s1[j] = on ? h2row0[j] : 0.f;
            }
            stage<64>(S, TX, T64B, t, a);
            stage<64>(S, TY, T64B, t, s1);
        }
        publish();
        if (t == 0) {
            umma::gemm3(tb + TM_SB, S.K(TX, T64B, 64), S.K(WH2, WH2B, 64), 4, ID_KK(16), false);
            umma::gemm3(tb + TM_JD, S.K(TY, T64B, 64), S.MN(WH1, WH1B, 48), 4, ID_KM(48), false);
            umma::commit(&mbar);
        }
        wait_mma(&mbar, phase);
        // ------------------------------------------------ P2: normal, cin -> Zc1
        float y[16], n0, n1, n2;
        float gn0 = 0.f, gn1 = 0.f, gn2 = 0.f;
        {
            umma::tmem_ld<16>(my + TM_SB, y);
            float jd[48], J[96];
            umma::tmem_ld<48>(my + TM_JD, jd);
            umma::tmem_ld<96>(my + TM_J, J);
            n0 = jd[0];
            n1 = jd[1];
            n2 = jd[2];
#pragma unroll
            for (int a = 0; a < 2 * NS2B_MAX_LEVELS; ++a) {
                if (a < 2 * f.n_active) {
                    n0 = fmaf(jd[3 + a], J[3 * a], n0);
                    n1 = fmaf(jd[3 + a], J[3 * a + 1], n1);
                    n2 = fmaf(jd[3 + a], J[3 * a + 2], n2);
                }
            }
            const float nn = sqrtf(n0 * n0 + n1 * n1 + n2 * n2);
            if (valid) eik += (nn - 1.f) * (nn - 1.f);
            if (kBwd && valid) {
                if (dl_dn_extra) {
                    gn0 = dl_dn_extra[3 * p];
                    gn1 = dl_dn_extra[3 * p + 1];
                    gn2 = dl_dn_extra[3 * p + 2];
                }
                if (eik_w != 0.f) {  // trainer.py:229-235 (fp32, numpy's order)
                    const float coef = eik_w * (2.f * (nn - 1.f) / fmaxf(nn, 1e-12f));
                    gn0 += coef * n0 / Pf;
                    gn1 += coef * n1 / Pf;
                    gn2 += coef * n2 / Pf;
                }
            }
            float cin[32];
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
            for (int o = 0; o < 16; ++o) cin[9 + o] = y[o];
#pragma unroll
            for (int i = 25; i < 32; ++i) cin[i] = 0.f;
            stage<32>(S, TC, TCB, t, cin);
        }
        publish();
        if (t == 0) {
            umma::gemm3(tb + TM_SA, S.K(TC, TCB, 32), S.K(WC1, WC1B, 32), 2, ID_KK(64), false);
            umma::commit(&mbar);
        }
        wait_mma(&mbar, phase);
        // ------------------------------------------------ P3: a1c -> Zc2
        uint32_t c1lo = 0u, c1hi = 0u, c2lo = 0u, c2hi = 0u;
        {
            float z[64];
            umma::tmem_ld<64>(my + TM_SA, z);
#pragma unroll
            for (int j = 0; j < 64; ++j) {
                const bool on = z[j] > 0.f;
                if (on) {
                    if (j < 32) c1lo |= 1u << j;
                    else c1hi |= 1u << (j - 32);
                }
                z[j] = on ? z[j] : 0.f;
            }
            stage<64>(S, TZ, T64B, t, z);
        }
        publish();
        if (t == 0) {
            umma::gemm3(tb + TM_SB, S.K(TZ, T64B, 64), S.K(WC2, WC2B, 64), 4, ID_KK(64), false);
            umma::commit(&mbar);
        }
        wait_mma(&mbar, phase);
        // ------------------------------------------------ P4: a2c -> LOG
        {
            float z[64];
            umma::tmem_ld<64>(my + TM_SB, z);
#pragma unroll
            for (int j = 0; j < 64; ++j) {
                const bool on = z[j] > 0.f;
                if (on) {
                    if (j < 32) c2lo |= 1u << j;
                    else c2hi |= 1u << (j - 32);
                }
                z[j] = on ? z[j] : 0.f;
            }
            stage<64>(S, TX, T64B, t, z);
        }
        publish();
        if (t == 0) {
            umma::gemm3(tb + TM_SA, S.K(TX, T64B, 64), S.K(WC3, WC3B, 64), 4, ID_KK(16), false);
            umma::commit(&mbar);
        }
        wait_mma(&mbar, phase);
        // ------------------------------------------------ P5: colours (+ backward start)
        float cc0, cc1, cc2;
        {
            float lg[16];
            umma::tmem_ld<16>(my + TM_SA, lg);
            cc0 = sigmoid_f(lg[0]);
            cc1 = sigmoid_f(lg[1]);
            cc2 = sigmoid_f(lg[2]);
        }
        if (!kBwd) {
            if (valid) {
                sdf_out[p] = y[0];
                col_out[3 * p] = cc0;
                col_out[3 * p + 1] = cc1;
                col_out[3 * p + 2] = cc2;
                if (nrm_out) {
                    nrm_out[3 * p] = n0;
                    nrm_out[3 * p + 1] = n1;
                    nrm_out[3 * p + 2] = n2;
                }
                if (geo_out)
#pragma unroll
                    for (int o = 1; o < 16; ++o) geo_out[15 * p + o - 1] = y[o];
            }
            continue;
        }
        float gc0 = 0.f, gc1 = 0.f, gc2 = 0.f, gd = 0.f;
        if (valid) {
            gc0 = dl_dc[3 * p];
            gc1 = dl_dc[3 * p + 1];
            gc2 = dl_dc[3 * p + 2];
            gd = dl_dsdf[p];
        }
        int G1;
        {
            float dlog[16];
            dlog[0] = gc0 * cc0 * (1.f - cc0);  // field.py:304
            dlog[1] = gc1 * cc1 * (1.f - cc1);
            dlog[2] = gc2 * cc2 * (1.f - cc2);
#pragma unroll
            for (int i = 3; i < 16; ++i) dlog[i] = 0.f;
            G1 = tile_exponent(absmax<3>(dlog), red);
            const float sc = pow2i(kHead - G1);
#pragma unroll
            for (int i = 0; i < 3; ++i) dlog[i] *= sc;
            stage<16>(S, TD, TDB, t, dlog);
        }
        publish();
        if (t == 0) {
            umma::gemm3(tb + TM_SA, S.K(TD, TDB, 16), S.MN(WC3, WC3B, 64), 1, ID_KM(64), false);
            umma::gemm3(tb + TM_DC3, S.MN(TX, T64B, 64), S.MN(TD, TDB, 16), 8, ID_WG(16), false);
            umma::commit(&mbar);
        }
        wait_mma(&mbar, phase);
        // ------------------------------------------------ P6: u2 -> U1, dC2 (+ flush dC3)
        int G2;
        {
            float d[16];
            umma::tmem_ld<16>(my + TM_DC3, d);
            if (lane < 16) {
                const int j = warp * 16 + lane;
                const float sc = pow2i(G1 - kHead);
#pragma unroll
                for (int o = 0; o < 3; ++o) gacc[G_C3r + o * H + j] += d[o] * sc;
            }
            float u[64];
            umma::tmem_ld<64>(my + TM_SA, u);
            const float sc1 = pow2i(G1 - kHead);
#pragma unroll
            for (int k = 0; k < 64; ++k) u[k] = mask_bit(c2lo, c2hi, k) ? u[k] * sc1 : 0.f;
            G2 = tile_exponent(absmax<64>(u), red);
            const float sc = pow2i(kHead - G2);
#pragma unroll
            for (int k = 0; k < 64; ++k) u[k] *= sc;
            stage<64>(S, TY, T64B, t, u);
        }
        publish();
        if (t == 0) {
            umma::gemm3(tb + TM_SB, S.K(TY, T64B, 64), S.MN(WC2, WC2B, 64), 4, ID_KM(64), false);
            umma::gemm3(tb + TM_DC2, S.MN(TY, T64B, 64), S.MN(TZ, T64B, 64), 8, ID_WG(64), false);
            umma::commit(&mbar);
        }
        wait_mma(&mbar, phase);
        // ------------------------------------------------ P7: u1 -> DCIN, dC1
        int G3;
        {
            float u[64];
            umma::tmem_ld<64>(my + TM_SB, u);
            const float sc2 = pow2i(G2 - kHead);
#pragma unroll
            for (int j = 0; j < 64; ++j) u[j] = mask_bit(c1lo, c1hi, j) ? u[j] * sc2 : 0.f;
            G3 = tile_exponent(absmax<64>(u), red);
            const float sc = pow2i(kHead - G3);
#pragma unroll
            for (int j = 0; j < 64; ++j) u[j] *= sc;
            stage<64>(S, TX, T64B, t, u);
        }
        publish();
        if (t == 0) {
            umma::gemm3(tb + TM_SA, S.K(TX, T64B, 64), S.MN(WC1, WC1B, 32), 4, ID_KM(32), false);
            umma::gemm3(tb + TM_DC1, S.MN(TX, T64B, 64), S.MN(TC, TCB, 32), 8, ID_WG(32), false);
            umma::commit(&mbar);
        }
        wait_mma(&mbar, phase);
        // ------------------------------------------------ P8: q, dly -> U, dH2
        float q0, q1, q2;
        int G4;
        {
            float dcin[32];
            umma::tmem_ld<32>(my + TM_SA, dcin);
            const float sc3 = pow2i(G3 - kHead);
            q0 = gn0 + dcin[3] * sc3;  // field.py:308-312
            q1 = gn1 + dcin[4] * sc3;
            q2 = gn2 + dcin[5] * sc3;
            float dly[16];
            dly[0] = gd + dcin[9] * sc3;
#pragma unroll
            for (int o = 1; o < 16; ++o) dly[o] = dcin[9 + o] * sc3;
            G4 = tile_exponent(absmax<16>(dly), red);
            const float sc = pow2i(kHead - G4);
#pragma unroll
            for (int o = 0; o < 16; ++o) dly[o] *= sc;
            stage<16>(S, TD, TDB, t, dly);
            float z[64];
            umma::tmem_ld<64>(my + TM_Z1, z);
#pragma unroll
            for (int j = 0; j < 64; ++j) z[j] = z[j] > 0.f ? z[j] : 0.f;
            stage<64>(S, TY, T64B, t, z);
        }
        publish();
        if (t == 0) {
            umma::gemm3(tb + TM_SB, S.K(TD, TDB, 16), S.MN(WH2, WH2B, 64), 1, ID_KM(64), false);
            umma::gemm3(tb + TM_DH2, S.MN(TY, T64B, 64), S.MN(TD, TDB, 16), 8, ID_WG(16), false);
            umma::commit(&mbar);
        }
        wait_mma(&mbar, phase);
        // ------------------------------------------------ P9: u, mvec -> DE, PV, dH1
        int G56;
        {
            float u[64];
            umma::tmem_ld<64>(my + TM_SB, u);
            const float sc4 = pow2i(G4 - kHead);
#pragma unroll
            for (int j = 0; j < 64; ++j) u[j] = mask_bit(mlo, mhi, j) ? u[j] * sc4 : 0.f;
            float J[96];
            umma::tmem_ld<96>(my + TM_J, J);
            float mv[48];
            mv[0] = q0;
            mv[1] = q1;
            mv[2] = q2;
#pragma unroll
            for (int a = 0; a < 32; ++a)
                mv[3 + a] = (a < 2 * f.n_active) ? (J[3 * a] * q0 + J[3 * a + 1] * q1 + J[3 * a + 2] * q2) : 0.f;
#pragma unroll
            for (int i = 35; i < 48; ++i) mv[i] = 0.f;
            G56 = tile_exponent(fmaxf(absmax<64>(u), absmax<48>(mv)), red);
            const float sc = pow2i(kHead - G56);
#pragma unroll
            for (int j = 0; j < 64; ++j) u[j] *= sc;
#pragma unroll
            for (int i = 0; i < 48; ++i) mv[i] *= sc;
            stage<64>(S, TX, T64B, t, u);
            stage<48>(S, TZ, T64B, t, mv);
            float s1[64];
#pragma unroll
            for (int j = 0; j < 64; ++j) s1[j] = mask_bit(mlo, mhi, j) ? h2row0[j] : 0.f;
            stage<64>(S, TY, T64B, t, s1);
        }
        publish();
        if (t == 0) {
            umma::gemm3(tb + TM_SA, S.K(TX, T64B, 64), S.MN(WH1, WH1B, 48), 4, ID_KM(48), false);
            umma::gemm3(tb + TM_SB, S.K(TZ, T64B, 48), S.K(WH1, WH1B, 48), 3, ID_KK(64), false);
            umma::gemm3(tb + TM_DH1, S.MN(TX, T64B, 64), S.MN(TE, TEB, 48), 8, ID_WG(48), false);
            umma::gemm3(tb + TM_DH1, S.MN(TY, T64B, 64), S.MN(TZ, T64B, 48), 8, ID_WG(48), true);
            umma::commit(&mbar);
        }
        wait_mma(&mbar, phase);
        // ------------------------------------------------ P10: pvec, scatter
        int G7;
        float de[48], jd[48];
        {
            umma::tmem_ld<48>(my + TM_SA, de);
            const float sc56 = pow2i(G56 - kHead);
#pragma unroll
            for (int i = 0; i < 48; ++i) de[i] *= sc56;
            float pv[64];
            umma::tmem_ld<64>(my + TM_SB, pv);
#pragma unroll
            for (int j = 0; j < 64; ++j) pv[j] = mask_bit(mlo, mhi, j) ? pv[j] * sc56 : 0.f;
            G7 = tile_exponent(absmax<64>(pv), red);
            const float sc = pow2i(kHead - G7);
#pragma unroll
            for (int j = 0; j < 64; ++j) pv[j] *= sc;
            stage<64>(S, TX, T64B, t, pv);
            float ones[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) ones[i] = i == 0 ? 1.f : 0.f;
            stage<16>(S, TD, TDB, t, ones);
            umma::tmem_ld<48>(my + TM_JD, jd);
        }
        publish();
        if (t == 0) {
            umma::gemm3(tb + TM_DC3, S.MN(TX, T64B, 64), S.MN(TD, TDB, 16), 8, ID_WG(16), false);
            umma::commit(&mbar);
        }
        // fused first + second order table scatter while the last MMA runs (Eq. 9):
        // grad += w * dL/dfeat + j_d[feat] * (q . dw)   (one float2 RED per corner)
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
        wait_mma(&mbar, phase);
        // ------------------------------------------------ P11: fold weight gradients
        {
            const int j = warp * 16 + lane;  // weight row held by lanes 0..15 (M=64 layout)
            float d[64];
            umma::tmem_ld<64>(my + TM_DC2, d);
            if (lane < 16) {
                const float sc = pow2i(G2 - kHead);
#pragma unroll
                for (int c = 0; c < 64; ++c) gacc[G_C2r + j * H + c] += d[c] * sc;
            }
            umma::tmem_ld<32>(my + TM_DC1, d);
            if (lane < 16) {
                const float sc = pow2i(G3 - kHead);
#pragma unroll
                for (int c = 0; c < CIN; ++c) gacc[G_C1r + j * CIN + c] += d[c] * sc;
            }
            umma::tmem_ld<16>(my + TM_DH2, d);
            float dp[16];
            umma::tmem_ld<16>(my + TM_DC3, dp);
            if (lane < 16) {
                const float sc = pow2i(G4 - kHead);
#pragma unroll
                for (int o = 0; o < 16; ++o) gacc[G_H2r + o * H + j] += d[o] * sc;
                gacc[G_H2r + j] += dp[0] * pow2i(G7 - kHead);
            }
            umma::tmem_ld<48>(my + TM_DH1, d);
            if (lane < 16) {
                const float sc = pow2i(G56 - kHead);
#pragma unroll
                for (int c = 0; c < EP; ++c) {
                    const int dst = c < E ? c : (c == EC ? E : -1);
                    if (dst >= 0) gacc[G_H1r + j * (E + 1) + dst] += d[c] * sc;
                }
            }
        }
    }
    if (eik_sum) {
        double v = warp_sum(static_cast<double>(eik));
        if (lane == 0 && v != 0.0) atomicAdd(eik_sum, v);
    }
    umma::fence_before_sync();
    __syncthreads();
    if (kBwd) {
        const int nsdf = H * (E + 1) + NOUT * H;
        for (int i = t; i < GACC_FLOATS; i += TILE) {
            const float v = gacc[i];
            if (i < nsdf) {
                if (v != 0.f) atomicAdd(g_sdf + i, v);
            } else if (i < G_C3r + 3 * H) {
                if (v != 0.f) atomicAdd(g_color + (i - nsdf), v);
            }
        }
    }
    if (warp == 0) umma::tmem_dealloc(tb, 512);
}

static int g_tc_attr = 0;
static int ensure_tc_attrs() {
    if (g_tc_attr) return NS2B_OK;
    cudaError_t e = cudaFuncSetAttribute(field_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(SMEM_FWD));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(field_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(SMEM_BWD));
    if (e != cudaSuccess) return set_error(NS2B_ECUDA, "tc smem attribute: %s", cudaGetErrorString(e));
    g_tc_attr = 1;
    return NS2B_OK;
}

}  // namespace tc

int field_forward_tc(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids, const double *dirs,
                     const int32_t *count, int64_t capacity, float *sdf, float *colors, float *normals, float *geo,
                     double *eik_sum, cudaStream_t st) {
    FieldDev f;
    int rc = make_field_dev(field, f);
    if (rc) return rc;
    if ((rc = tc::ensure_tc_attrs())) return rc;
    if (capacity <= 0) return NS2B_OK;
    const int blocks = grid_for(capacity, tc::TILE, kNumSMs);
    tc::field_tc_kernel<false><<<blocks, tc::TILE, tc::SMEM_FWD, st>>>(
        f, pos32, ray_ids, dirs, count, sdf, colors, normals, geo, eik_sum, nullptr, nullptr, nullptr, 0.f,
        nullptr, nullptr, nullptr, nullptr);
    return check_launch("field_forward_tc");
}

int field_backward_tc(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids, const double *dirs,
                      const int32_t *count, int64_t capacity, const float *dl_dc, const float *dl_dsdf,
                      const float *dl_dn_extra, double eik_weight, const int64_t *eik_count, float *grad_sdf,
                      float *grad_color, float *grad_tables, cudaStream_t st) {
    FieldDev f;
    int rc = make_field_dev(field, f);
    if (rc) return rc;
    if ((rc = tc::ensure_tc_attrs())) return rc;
    NS2B_REQUIRE(eik_weight == 0.0 || eik_count != nullptr, "eik_count required with eik_weight");
    if (capacity <= 0) return NS2B_OK;
    const int blocks = grid_for(capacity, tc::TILE, kNumSMs);
    tc::field_tc_kernel<true><<<blocks, tc::TILE, tc::SMEM_BWD, st>>>(
        f, pos32, ray_ids, dirs, count, nullptr, nullptr, nullptr, nullptr, nullptr, dl_dc, dl_dsdf, dl_dn_extra,
        static_cast<float>(eik_weight), eik_count, grad_sdf, grad_color, grad_tables);
    return check_launch("field_backward_tc");
}

}  // namespace ns2b
