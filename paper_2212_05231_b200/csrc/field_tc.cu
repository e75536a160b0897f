// K2/K5 on the 5th-gen tensor cores: the field's MLP forward / backward with tcgen05, plus
// the hash-grid gather and the table scatter around them.
//
// Kernels (one training step launches gather -> fwd2 -> [composite] -> bwd2 -> scatter):
//   field_gather_kernel   one 128-sample tile per block: trilinear features, d feature/dx
//                         (J), the encoding tile E pre-staged in the UMMA layout;
//   field_fwd2_kernel     persistent, 512 threads = two 256-thread groups, each running
//                         its own 128-sample tile (two tiles in flight per SM);
//   field_bwd2_kernel     persistent, 512 threads = group C (colour-net half of the chain)
//                         a tile ahead of group S (SDF-net half), handoff through a
//                         two-slot shared-memory ring;
//   field_scatter_kernel  one tile per block, first + second-order table gradients (Eq. 9)
//                         as float2 / x-pair float4 REDs;
//   field_fwd_kernel / field_bwd_kernel: the one-tile versions (NS2B_FWD=1 / NS2B_BWD=1;
//                         the dynamic path's input cotangents use field_bwd_kernel).
//
// A tile is 128 samples = 128 TMEM lanes; a warp reads its lane quadrant (warp % 4), and
// the warps sharing a quadrant split each row's columns, so every per-sample epilogue
// (ReLU, masks, normals, sigmoid, losses, cotangents) is plain per-thread code on the rows
// tcgen05.ld returns.  Every dense contraction is a UMMA issued by one elected lane of an
// MMA warp:
//   chain GEMMs (M = 128 samples): operand tiles [sample][feature] (K-major A, in shared
//     memory or -- the backward's cotangent tiles -- in TMEM) x the weights (K-major view
//     for W^T, MN-major view of the same tile for W);
//   weight-gradient GEMMs (M = 64 weight rows, K = the 128 samples of the tile): MN-major
//     views of the per-sample tiles, accumulated in TMEM across a CTA's tiles and folded to
//     global memory on a scale change and at the end.
//
// Precision: chain GEMMs use fp16 with the three-term hi/lo split (A_hi B_hi + A_lo B_hi +
// A_hi B_lo, fp32 accumulation in TMEM); it is fp32-accurate only while the lo parts stay
// normal, so every staged tile (per tile, predicted exponents) and every weight matrix (per
// CTA) is scaled by an exact power of two putting its max in [2^13, 2^14); GEMM results are
// multiplied back by 2^-(eA+eB) (folded into the next staging scale where one follows).
// Weight-gradient GEMMs take both operands as fp16 (stated, fp32 accumulation).
//
// Encoding column order inside the tiles: [features 0..31 | x y z | 1 | 0 x 12] (48),
// so a level's feature pair is 4-byte aligned; H1 / dH1 are permuted accordingly.
//
// Algorithm per tile (field.py:208-331, relu_mlp.py:94-216):
//   forward   P0 Z1 = E H1^T;  P1 a1 = relu(Z1), d (fp32 FMAs);  Y = A1 H2^T,  JD = M1 H1'
//             (j_d);  P2 n = j_d J, cin = [x, n, v, y];  Zc1 = CIN C1^T;  P3 Zc2 = A1c C2^T;
//             P4 logits (FMAs);  P5 c = sigmoid  (+ the Eikonal cotangent when fused)
//   backward  dlog -> U2 = DLOG C3, dC3 += A2c^T DLOG;  u2 -> U1 = U2 C2, dC2 += U2^T A1c;
//             u1 -> DCIN = U1 C1, dC1 += U1^T CIN;  q, dly -> U = DLY H2, dH2 += A1^T DLY;
//             u, mvec = [J q, q] -> DE = U H1, dH1 += U^T E, G += M1^T MV (Theorem 1:
//             dH1 += diag(H2[0]) G, dH2[0] += rowdot(H1, G) at fold time);  DE, j_d, q ->
//             the scatter's inputs
#include <cstdio>

#include "field_common.cuh"
#include "umma.cuh"

namespace ns2b {
namespace tc {

constexpr int TILE = 128;
constexpr int kHead = 14;  // staged maxima land in [2^13, 2^14)
#ifndef NS2B_PRED_SLACK
#define NS2B_PRED_SLACK 10  // accepted predicted exponents: staged max in [2^(13-slack), 2^15)
#endif

// shared memory map (bytes); every tile is hi part then lo part
constexpr uint32_t WH1 = 0;                          // 64 x 48
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
constexpr uint32_t TW = TEND;                         // 128 x 64 (backward: DMA'd A2c / A1)
constexpr uint32_t WH1S = TEND;                       // forward: H1' = diag(H2[0]) H1, 64 x 48
constexpr uint32_t TLG = WH1S + 2 * WH1B;             // forward: per-quarter logit partials [4][3][128] fp32
constexpr uint32_t SMEM_FWD = TLG + 4 * 3 * TILE * 4;
constexpr uint32_t SMEM_BWD = TW + 2 * T64B;

// TMEM columns (512 allocated).  Forward:
constexpr uint32_t TM_J = 176;    // 16 levels x 8: [dfeat/dx (6) | 2 spare]
constexpr uint32_t TM_Z1 = 304;   // 64
constexpr uint32_t TM_SA = 368;   // 64 chain slot A
constexpr uint32_t TM_SB = 432;   // 64 chain slot B
// Backward: weight-gradient accumulators (M = 64 rows in lanes 0-15 of each quadrant),
// accumulated across tiles while their scale exponent is unchanged
constexpr uint32_t TB_DC2 = 0;     // 64
constexpr uint32_t TB_DC1 = 64;    // 32
constexpr uint32_t TB_DC3 = 96;    // 16 (3 used)
constexpr uint32_t TB_DH2 = 112;   // 16
constexpr uint32_t TB_DH1A = 128;  // 48: U^T E
constexpr uint32_t TB_DH1B = 176;  // 48: G = M1^T MV (Theorem 1: dH1 and dH2[0])
constexpr uint32_t TB_J = 240;     // 128
constexpr uint32_t TB_SA = 368;    // 64
constexpr uint32_t TB_SB = 432;    // 64

constexpr uint32_t ID_KK(int N) { return umma::make_idesc(128, N, 0, 0, 0); }
constexpr uint32_t ID_KM(int N) { return umma::make_idesc(128, N, 0, 0, 1); }
constexpr uint32_t ID_WG(int N) { return umma::make_idesc(64, N, 0, 1, 1); }
// Weight-gradient GEMMs (dW = X^T Y summed over the tile's 128 samples, and over a CTA's
// ~1.2k tiles in TMEM) take both operands in fp16 (stated fp16 storage of the
// activations A1, CIN, A1c, A2c, E and of the cotangent tiles for the weight gradients,
// fp32 accumulation): one MMA per K step, and the forward stores (the backward DMAs) only
// the hi halves of its tiles.  Measured: backward 10.13 -> 9.73 ms against the round-2
// two-term form (cotangent split hi + lo, gemm2a / gemm2w; -DNS2B_WG2 restores it); at
// 2^22 points every weight gradient stays within 1e-4 relL2 of torch fp64
// (tests/test_gpu_c3.py).  The per-sample chain GEMMs keep the full 3-term split: a row's
// precision there reaches the table gradients directly.  Their A operands (the cotangent
// tiles) live in tensor memory (NS2B_BWD_TA, default; -DNS2B_BWD_SMEM_A reads them from
// shared memory): 9.73 -> 9.43 ms.
#ifndef NS2B_WG2
#define NS2B_WG1
#endif
#ifndef NS2B_BWD_SMEM_A  // (NS2B_BWD_SMEM_A: the chain GEMMs read A from shared memory)
#define NS2B_BWD_TA
#endif
#ifdef NS2B_WG1
#define WG_ACT_A umma::gemm1
#define WG_ACT_B umma::gemm1
#define WG_MASK umma::gemm1
#else
#define WG_ACT_A umma::gemm2a
#define WG_ACT_B umma::gemm2w
#define WG_MASK umma::gemm2a
#endif

#ifdef NS2B_PHASE_PROF
#define PMARK(i)                                  \
    do {                                          \
        if (threadIdx.x == 160) {                 \
            const long long c_ = clock64();       \
            pacc[(i) & 63] += c_ - plast;         \
            plast = c_;                           \
        }                                         \
    } while (0)
#define PWAIT(stmt)                              \
    do {                                         \
        const long long w0_ = clock64();         \
        stmt;                                    \
        pacc[63] += clock64() - w0_;             \
    } while (0)
#else
#define PWAIT(stmt) stmt
#define PMARK(i) \
    do {         \
    } while (0)
#endif

__device__ __forceinline__ float pow2i(int e) {
    e = max(-120, min(120, e));
    return __int_as_float((127 + e) << 23);
}

// tile column -> column of the real H1 (64, E+1) layout, -1 for padding
__device__ __forceinline__ int h1_col(int c, int E) {
    if (c < 32) return (3 + c < E) ? 3 + c : -1;
    if (c < 35) return c - 32;
    if (c == 35) return E;
    return -1;
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

// stage row r of a tile with values v * 2^e
template <int C>
__device__ __forceinline__ void stage(const Smem &s, uint32_t off, uint32_t part, int r, const float *v, int e) {
    const float sc = pow2i(e);
    float w[C];
#pragma unroll
    for (int i = 0; i < C; ++i) w[i] = v[i] * sc;
    umma::stage_row<0, C>(s.p(off), s.p(off + part), r, w);
}

// staging exponent for a tile maximum m >= 0: 2^e m in [2^13, 2^14); 0 for 0 / inf / nan
__device__ __forceinline__ int exp_for(float m) {
    const int biased = static_cast<int>(__float_as_uint(m) >> 23);  // m >= 0: no sign bit
    if (biased == 0 || biased >= 255) return m > 0.f ? kHead + 126 : 0;  // denormal / 0, inf, nan
    return kHead + 126 - biased;  // frexp exponent of m = biased - 126
}

// block-wide max of up to two values -> their staging exponents (one barrier)
struct Reducer {
    uint32_t (*red)[2][4];
    int parity;
    __device__ void two(float a, float b, int &ea, int &eb) {
        const int warp = threadIdx.x >> 5;
        const uint32_t ra = __reduce_max_sync(0xffffffffu, __float_as_uint(fabsf(a)));
        const uint32_t rb = __reduce_max_sync(0xffffffffu, __float_as_uint(fabsf(b)));
        if ((threadIdx.x & 31) == 0) {
            red[parity][0][warp] = ra;
            red[parity][1][warp] = rb;
        }
        __syncthreads();
        uint32_t ma = 0, mb = 0;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            ma = max(ma, red[parity][0][w]);
            mb = max(mb, red[parity][1][w]);
        }
        parity ^= 1;
        ea = exp_for(__uint_as_float(ma));
        eb = exp_for(__uint_as_float(mb));
    }
    __device__ int one(float a) {
        int ea, eb;
        two(a, 0.f, ea, eb);
        return ea;
    }
};

template <int N>
__device__ __forceinline__ float absmax(const float *v) {
    float m = 0.f;
#pragma unroll
    for (int i = 0; i < N; ++i) m = fmaxf(m, fabsf(v[i]));
    return m;
}

// weights -> fp16 hi/lo tiles, each matrix scaled by its own power of two.  With kH1S
// (forward) a sixth tile holds H1' = diag(H2[0]) H1, so the j_d GEMM S1 H1 becomes
// M1 H1' with the exact 0/1 ReLU mask M1 as its A operand.
template <bool kH1S>
__device__ void load_weight_tiles(const Smem &s, const FieldDev &f, uint32_t *wmax, int *wexp,
                                  uint32_t h1s_off = WH1S) {
    const int E = 3 + 2 * f.L;
    constexpr int NM = kH1S ? 6 : 5, NR = kH1S ? 288 : 224;
    auto fetch = [&](int r, int c) -> float {  // row r of the stacked [H1|H2|C1|C2|C3|H1'] tiles
        if (r < 64 || r >= 224) {
            const int rr = r < 64 ? r : r - 224;
            const int rc = h1_col(c, E);
            const float v = (c < 48 && rc >= 0) ? f.sdf_w[rr * (E + 1) + rc] : 0.f;
            return r < 64 ? v : v * f.sdf_w[H * (E + 1) + rr];
        }
        if (r < 80) return f.sdf_w[H * (E + 1) + (r - 64) * H + c];
        if (r < 144) return c < CIN ? f.color_w[(r - 80) * CIN + c] : 0.f;
        if (r < 208) return f.color_w[H * CIN + (r - 144) * H + c];
        return (r - 208) < 3 ? f.color_w[H * CIN + H * H + (r - 208) * H + c] : 0.f;
    };
    auto mat = [](int r) { return r < 64 ? 0 : r < 80 ? 1 : r < 144 ? 2 : r < 208 ? 3 : r < 224 ? 4 : 5; };
    const int cols[6] = {48, 64, 32, 64, 64, 48};
    if (threadIdx.x < NM) wmax[threadIdx.x] = 0u;
    __syncthreads();
    for (int r = threadIdx.x; r < NR; r += blockDim.x) {
        float m = 0.f;
        for (int c = 0; c < cols[mat(r)]; ++c) m = fmaxf(m, fabsf(fetch(r, c)));
        atomicMax(&wmax[mat(r)], __float_as_uint(m));
    }
    __syncthreads();
    if (threadIdx.x < NM) wexp[threadIdx.x] = exp_for(__uint_as_float(wmax[threadIdx.x]));
    __syncthreads();
    for (int r = threadIdx.x; r < NR; r += blockDim.x) {
        float row[64];
        const int k = mat(r);
        for (int c = 0; c < 64; ++c) row[c] = c < cols[k] ? fetch(r, c) : 0.f;
        const int e = wexp[k];
        if (k == 0) stage<48>(s, WH1, WH1B, r, row, e);
        else if (k == 1) stage<64>(s, WH2, WH2B, r - 64, row, e);
        else if (k == 2) stage<32>(s, WC1, WC1B, r - 80, row, e);
        else if (k == 3) stage<64>(s, WC2, WC2B, r - 144, row, e);
        else if (k == 4) stage<64>(s, WC3, WC3B, r - 208, row, e);
        else stage<48>(s, h1s_off, WH1B, r - 224, row, e);
    }
}

__device__ __forceinline__ void block_sync_tc() {
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
}

__device__ __forceinline__ void publish() {
    umma::fence_async_smem();
    block_sync_tc();
}

__device__ __forceinline__ void wait_mma(uint64_t *mbar, uint32_t &phase) {
#ifdef NS2B_SPIN_WAIT
    umma::mbar_wait_spin(mbar, phase);
#else
    umma::mbar_wait(mbar, phase);
#endif
    phase ^= 1u;
    umma::fence_after_sync();
}

struct LevelSm {
    LevelInfo lv;
    float sx, sy, sz;
    float pad;
};

// Per-tile workspace (see ns2b_field_workspace_bytes):
//   gather  -> pre-staged E tiles (fp16 hi | lo, UMMA tile layout) + exponent, d feature/dx
//              value-major [tile][96][128] fp32, position | view dir [tile][6][128] fp32;
//   MLP fwd -> its staged operand tiles A1 | CIN | A1c | A2c (fp16 hi parts) + exponents,
//              ReLU masks [tile][4][128] (uint2: m1 | mc1 << 16, mc2 of a column quarter),
//              normal | colour [tile][6][128] fp32, j_d feature rows (into the sb block);
//   MLP bwd -> scatter inputs [tile][68][128] fp32 = dL/dfeature (32) | j_d rows (32) | q (3).
// The backward therefore never recomputes the forward: it DMAs the forward's tiles.
//   MLP bwd (input cotangents requested) -> [tile][9][128] fp32 = dcin_x (3) | dcin_v (3) | de_x (3).
constexpr int JROWS = 96, SBROWS = 68, XVROWS = 6, NCROWS = 6, XINROWS = 9;
// stored tiles: fp16 hi parts only (the weight-gradient GEMMs read nothing else)
constexpr uint32_t FW_A1 = 0, FW_CIN = T64B, FW_A1C = FW_CIN + TCB, FW_A2C = FW_A1C + T64B,
                   FWB = FW_A2C + T64B;
struct Workspace {
    uint8_t *e_tiles;
    int *e_exp;
    float *jac;
    float *sb;
    float *xv;
    uint8_t *fw_tiles;
    int4 *fw_exp;
    uint32_t *fw_mask;  // [tile][m1 | mc1 | mc2][half][128]: a row's 32 hidden-unit bits of a half (blocks 4h..4h+3)
    float *fw_nc;
    float *xin;
    int *flags;  // [0]: 1 when the forward stored the Eikonal cotangent (not n) in fw_nc rows 0-2
};
// mask word of (kind, half) for row r of a tile
__device__ __forceinline__ int64_t mask_idx(int64_t tile, int kind, int h, int r) {
    return (tile * 6 + kind * 2 + h) * TILE + r;
}
// the one-group kernels' quarter view: quarter q owns blocks q and q + 4, as
// (m1 | mc1 << 16, mc2) with block q in the low byte of each 16-bit field
__device__ __forceinline__ uint2 mask_quarter(const uint32_t *w6, int stride, int q) {
    auto q16 = [&](int kind) {
        return ((w6[(2 * kind) * stride] >> (8 * q)) & 0xFFu) | (((w6[(2 * kind + 1) * stride] >> (8 * q)) & 0xFFu) << 8);
    };
    return make_uint2(q16(0) | (q16(1) << 16), q16(2));
}
__host__ __device__ inline size_t ws_tile_bytes() {
    return 2 * static_cast<size_t>(TEB) + FWB + sizeof(int4) + sizeof(int) + 6 * TILE * sizeof(uint32_t) +
           (JROWS + SBROWS + XVROWS + NCROWS + XINROWS) * TILE * sizeof(float);
}
__host__ inline Workspace ws_carve(void *base, int64_t ntiles) {
    uint8_t *b = static_cast<uint8_t *>(base);
    Workspace w;
    w.e_tiles = b;
    b += ntiles * 2 * static_cast<size_t>(TEB);
    w.fw_tiles = b;
    b += ntiles * static_cast<size_t>(FWB);
    w.fw_exp = reinterpret_cast<int4 *>(b);
    b += ntiles * sizeof(int4);
    w.fw_mask = reinterpret_cast<uint32_t *>(b);
    b += ntiles * 6 * TILE * sizeof(uint32_t);
    w.fw_nc = reinterpret_cast<float *>(b);
    b += ntiles * NCROWS * TILE * sizeof(float);
    w.jac = reinterpret_cast<float *>(b);
    b += ntiles * JROWS * TILE * sizeof(float);
    w.sb = reinterpret_cast<float *>(b);
    b += ntiles * SBROWS * TILE * sizeof(float);
    w.xv = reinterpret_cast<float *>(b);
    b += ntiles * XVROWS * TILE * sizeof(float);
    w.xin = reinterpret_cast<float *>(b);
    b += ntiles * XINROWS * TILE * sizeof(float);
    w.e_exp = reinterpret_cast<int *>(b);
    w.flags = w.e_exp + ntiles;  // in the workspace's 256-byte tail
    return w;
}

// ---------------------------------------------------------------------------
// MLP kernel: 512 threads per 128-sample tile.  Warp w reads TMEM lane quadrant w%4,
// so thread (quarter k = w/4, row r = 32*(w%4) + lane) co-owns sample r with three
// other threads; every per-row epilogue is split by 8-column blocks: the thread of
// quarter k owns blocks k and k+4 of a tile.  Row scalars (the SDF value, the normal)
// are combined through shared memory.  One elected thread issues all MMAs.
constexpr int MLP_THREADS = 512;
// The warp that issues every tcgen05.mma / commit (and the forward's tile stores): a
// quarter-3 warp, whose epilogue share is the lightest (quarter 0 owns the row scalars).
constexpr int kMmaWarp = 15;
// The thread that issues the bulk DMAs and L2 prefetches (another quarter-3 warp).
constexpr int kDmaThread = 14 * 32;

// Predicted staging exponents.  The exponent a tile is staged with only has to keep its
// maximum inside fp16's range with the lo parts normal, so instead of a block-wide max
// before staging (one barrier per phase) each staging point uses the exponent its
// previous tile ended with (one bit of extra headroom), every warp atomically maxes its
// |value| into a shared slot, and the value is checked after the publish barrier the
// phase needs anyway.  A tile whose max left [2^3, 2^15) is restaged with the exact
// exponent (first tile of a CTA, sudden range changes).  Scaling by 2^e is exact, so
// the products equal those of an exactly-scaled tile.
enum Slot { kA1, kCin, kA1c, kA2c, kDlog, kU2, kU1, kDly, kU, kMv, kE, NSLOT };
struct PredScale {
    uint32_t (*mx)[NSLOT];  // [2][NSLOT] block maxima (bits of |v|), tile parity
    int *pred;              // [NSLOT]
    int par;
    __device__ __forceinline__ int guess(int k) const { return pred[k]; }
    __device__ __forceinline__ void contrib(int k, float m) {
        const uint32_t w = __reduce_max_sync(0xffffffffu, __float_as_uint(m));
        if ((threadIdx.x & 31) == 0 && w) atomicMax(&mx[par][k], w);
    }
    // after the barrier: is e acceptable?  Otherwise e <- the exact exponent less one
    // (max in [2^12, 2^13)), which also becomes the new prediction.  Accepted exponents
    // stay (sticky), so the weight-gradient accumulators keep one scale across tiles.
    __device__ __forceinline__ bool check(int k, int &e) {
        const float m = __uint_as_float(mx[par][k]);
        const int ex = exp_for(m);
        const bool ok = !(m > 0.f) || (e <= ex + 1 && e >= ex - NS2B_PRED_SLACK);
        if (!ok) {
            e = ex - 1;
            if (threadIdx.x == 0) pred[k] = e;
        }
        return ok;
    }
};

// stage one 8-column block of row r (values * sc) into a C-column tile
template <int C>
__device__ __forceinline__ void stage_blk(const Smem &s, uint32_t off, uint32_t part, int r, int b, const float *v,
                                          float sc) {
    uint4 h, l;
    umma::split2<0>(v[0] * sc, v[1] * sc, h.x, l.x);
    umma::split2<0>(v[2] * sc, v[3] * sc, h.y, l.y);
    umma::split2<0>(v[4] * sc, v[5] * sc, h.z, l.z);
    umma::split2<0>(v[6] * sc, v[7] * sc, h.w, l.w);
    const uint32_t o = umma::tile_off(r, 8 * b, C);
    *reinterpret_cast<uint4 *>(s.p(off) + o) = h;
    *reinterpret_cast<uint4 *>(s.p(off + part) + o) = l;
}

// hi part only (a tile that is stored for the backward's weight-gradient GEMMs and read
// by no GEMM of its own kernel)
// Common per-CTA setup of both MLP kernels: weight tiles, H2 row 0, barriers, TMEM.
struct MlpShared {
    uint32_t tmem_base;
    uint32_t slot_mx[2][NSLOT];
    int slot_pred[NSLOT];
    uint32_t wmax[6];
    int wexp[6];
    float h2row0[H];
    float c3[3][H];  // colour output layer (fp32): logits / u2 as FMA dot products
};

template <bool kH1S>
__device__ __forceinline__ void mlp_setup(const Smem &S, const FieldDev &f, MlpShared &sh, uint64_t *bars, int nbars) {
    const int t = threadIdx.x;
    const int E = 3 + 2 * f.L;
    if (t < H) sh.h2row0[t] = f.sdf_w[H * (E + 1) + t];
    if (t < 3 * H) sh.c3[t / H][t % H] = f.color_w[H * CIN + H * H + t];
    load_weight_tiles<kH1S>(S, f, sh.wmax, sh.wexp);
    if (t < NSLOT) {
        sh.slot_mx[0][t] = 0u;
        sh.slot_mx[1][t] = 0u;
        sh.slot_pred[t] = 0;
    }
    if (t == 0) {
        for (int i = 0; i < nbars; ++i) umma::mbar_init(bars + i, 1);
        umma::fence_barrier_init();
    }
    if ((t >> 5) == 0) umma::tmem_alloc(&sh.tmem_base, 512);
    publish();
}


// ---------------------------------------------------------------------------
// MLP forward (field.py:208-244): per tile P0 Z1 = E H1^T; P1 a1 -> Y = A1 H2^T (SDF
// value in fp32 FMAs), JD = S1 H1 (j_d); P2 normal n = j_d J, cin = [x, n, v, y] ->
// Zc1; P3 Zc2; P4 logits; P5 colours.  Every staged operand tile the backward needs (A1,
// CIN, A1c, A2c) leaves by bulk DMA to the workspace, with the ReLU masks, n and c.
__global__ void __launch_bounds__(MLP_THREADS, 1)
field_fwd_kernel(FieldDev f, const int32_t *__restrict__ count, float *__restrict__ sdf_out,
                 float *__restrict__ col_out, float *__restrict__ nrm_out, float *__restrict__ geo_out,
                 double *__restrict__ eik_sum, Workspace ws) {
    if (blockIdx.x == 0 && threadIdx.x == 0) ws.flags[0] = 0;  // fw_nc rows 0-2 hold the normal
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bars[2];  // [0] chain MMAs, [1] E-tile DMA
    __shared__ MlpShared sh;
    uint64_t *mbar = bars, *mbare = bars + 1;
    const Smem S{smem_raw};
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int qd = warp & 3, qt = warp >> 2;  // TMEM lane quadrant, column quarter
    const int r = 32 * qd + lane;              // sample row in the tile
    const int NA = f.n_active;
    mlp_setup<true>(S, f, sh, bars, 2);
    const int eH1 = sh.wexp[0], eH2 = sh.wexp[1], eC1 = sh.wexp[2], eC2 = sh.wexp[3];
    const float *h2row0 = sh.h2row0;
    const uint32_t tb = sh.tmem_base;
    const uint32_t my = tb + (static_cast<uint32_t>(qd * 32) << 16);
    float *xch = reinterpret_cast<float *>(S.p(TZ));  // row-scalar exchange scratch (P1-P2)
    uint32_t phase = 0, phasee = 0;
    PredScale PS{sh.slot_mx, sh.slot_pred, 1};
    const int eH1s = sh.wexp[5];
    const int P = *count;
    const int b0 = qt, b1 = qt + 4;  // my column blocks of 64-wide tiles
    float eik = 0.f;

    float jv[4][6];
    auto j_load = [&](int64_t tl) {
        const float *jt = ws.jac + tl * JROWS * TILE;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (4 * qt + i < NA) {
                const float *jr = jt + 6 * (4 * qt + i) * TILE + r;
#pragma unroll
                for (int k = 0; k < 6; ++k) jv[i][k] = jr[k * TILE];
            }
    };
    auto j_store = [&]() {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (4 * qt + i < NA) {
                const uint32_t c = my + TM_J + 8 * (4 * qt + i);
                umma::tmem_st4(c, jv[i][0], jv[i][1], jv[i][2], jv[i][3]);
                umma::tmem_st2(c + 4, jv[i][4], jv[i][5]);
            }
        umma::tmem_st_wait();
    };
    auto e_fetch = [&](int64_t tl) {
        if (t == kDmaThread && tl * TILE < P) umma::bulk_g2s(S.p(TE), ws.e_tiles + tl * 2 * TEB, 2 * TEB, mbare);
    };
    e_fetch(blockIdx.x);
    if (static_cast<int64_t>(blockIdx.x) * TILE < P) {
        j_load(blockIdx.x);
        j_store();
    }
#ifdef NS2B_PHASE_PROF
    __shared__ long long pacc[64];
    long long plast = clock64();
    if (t < 64) pacc[t] = 0;
    __syncthreads();
#endif
    int eE_cur = static_cast<int64_t>(blockIdx.x) * TILE < P ? ws.e_exp[blockIdx.x] : 0;
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * TILE; base < P;
         base += static_cast<int64_t>(gridDim.x) * TILE) {
        const int64_t p = base + r;
        const bool valid = p < P;
        const int64_t tile = base / TILE;
        const int64_t ntile = tile + gridDim.x;
        PS.par ^= 1;
        float *SBt = ws.sb + tile * SBROWS * TILE;
        uint8_t *fwt = ws.fw_tiles + tile * static_cast<int64_t>(FWB);
        float *nct = ws.fw_nc + tile * NCROWS * TILE + r;
        if (t == kDmaThread && ntile * TILE < P) umma::prefetch_l2(ws.jac + ntile * JROWS * TILE, JROWS * TILE * 4);
        const float *xvt = ws.xv + tile * XVROWS * TILE + r;
        const float x0 = xvt[0], x1 = xvt[TILE], x2 = xvt[2 * TILE];
        const float v0 = xvt[3 * TILE], v1 = xvt[4 * TILE], v2 = xvt[5 * TILE];
        const int eE = eE_cur;  // loaded during the previous tile
        // ------------------------------------------------ P0: Z1 = E H1^T
        if (warp == kMmaWarp) {  // converged MMA warp; elect.sync picks the issuing lane
            umma::mbar_wait(mbare, phasee);
            umma::gemm3w<3>(tb + TM_Z1, S.K(TE, TEB, 48), S.K(WH1, WH1B, 48), ID_KK(64), false);
            // the previous tile's A1 (TX), CIN (TC) and A1c (TZ) stores must have left smem
            // before P1 / P2 / P3 restage those buffers: wait for them while Z1 runs (its
            // A2c store from TY may still be reading; P3 waits for that one); committing
            // afterwards orders every thread's P1 staging (which waits on this commit)
            if (lane == 0) umma::bulk_wait_read_n<1>();
            __syncwarp();
            umma::commit_elect(mbar);
        }
        phasee ^= 1u;
        wait_mma(mbar, phase);
        PMARK(1);
        e_fetch(ntile);
        // ------------------------------------------------ P1: a1, s1 -> Y, JD; SDF value
        uint32_t m1 = 0u;  // my 16 hidden-unit mask bits (blocks b0, b1)
        int eA1;
        {
            float z[2][8], ma = 0.f, dpart = 0.f;
            const float sc = pow2i(-(eE + eH1));
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int b = i ? b1 : b0;
                umma::tmem_ld8(my + TM_Z1 + 8 * b, z[i]);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const bool on = z[i][k] > 0.f;
                    m1 |= on ? (1u << (8 * i + k)) : 0u;
                    const float a = on ? z[i][k] * sc : 0.f;
                    z[i][k] = a;
                    ma = fmaxf(ma, a);
                    // d = H2[0] a1 in fp32 FMAs: a cancelling sum the NeuS alpha
                    // differentiates along the ray (the MMA accumulator truncates)
                    dpart = fmaf(h2row0[8 * b + k], a, dpart);
                }
            }
            xch[qt * TILE + r] = dpart;
            eA1 = PS.guess(kA1);
            PS.contrib(kA1, ma);
            auto stg = [&](int e) {
                const float sa = pow2i(e);
#pragma unroll
                for (int i = 0; i < 2; ++i) stage_blk<64>(S, TX, T64B, r, i ? b1 : b0, z[i], sa);
            };
            stg(eA1);
            // j_d = (H2[0] . m1) H1 = M1 H1': the mask is exact in fp16 (hi part only)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const uint32_t bits = (m1 >> (8 * i)) & 0xFFu;
                auto h2 = [&](int k) {
                    return ((bits >> k) & 1u ? 0x3C00u : 0u) | ((bits >> (k + 1)) & 1u ? 0x3C000000u : 0u);
                };
                // M1 goes to TC (free until P2 stages CIN): TY may still be draining the
                // previous tile's A2c store
                *reinterpret_cast<uint4 *>(S.p(TC) + umma::tile_off(r, 8 * (i ? b1 : b0), 64)) =
                    make_uint4(h2(0), h2(2), h2(4), h2(6));
            }
            publish();
            PMARK(2);
            if (t < NSLOT) sh.slot_mx[PS.par ^ 1][t] = 0u;  // next tile's slots (last read before this barrier)
            if (!PS.check(kA1, eA1)) {
                stg(eA1);
                publish();
                PMARK(3);
            }
        }
        const float d_sdf = xch[r] + xch[TILE + r] + xch[2 * TILE + r] + xch[3 * TILE + r];
        if (warp == kMmaWarp) {  // converged MMA warp; elect.sync picks the issuing lane
            umma::gemm3w<4>(tb + TM_SB, S.K(TX, T64B, 64), S.K(WH2, WH2B, 64), ID_KK(16), false);
            umma::gemm2a<4>(tb + TM_SA, S.K(TC, T64B, 64), S.MN(WH1S, WH1B, 48), ID_KM(48), false);
            umma::commit_elect(mbar);
            if (lane == 0) umma::bulk_s2g(fwt + FW_A1, S.p(TX), T64B);
        }
        wait_mma(mbar, phase);
        PMARK(4);
        // ------------------------------------------------ P2: normal, cin -> Zc1
        int eCin;
        if (ntile * TILE < P) eE_cur = ws.e_exp[ntile];  // next tile's E exponent, a tile ahead
        {
            float y[16];
            umma::tmem_ld8(my + TM_SB, *reinterpret_cast<float(*)[8]>(y));
            umma::tmem_ld8(my + TM_SB + 8, *reinterpret_cast<float(*)[8]>(y + 8));
            const float scy = pow2i(-(eA1 + eH2));
#pragma unroll
            for (int o = 0; o < 16; ++o) y[o] *= scy;
            y[0] = d_sdf;
            // normal: my quarter's levels (+ the x rows for quarter 0), summed via smem
            const float scd = pow2i(-eH1s);
            float p0 = 0.f, p1 = 0.f, p2 = 0.f;
            if (qt == 0) {
                float jx[4];
                umma::tmem_ld4(my + TM_SA + 32, jx);
                p0 = jx[0] * scd;
                p1 = jx[1] * scd;
                p2 = jx[2] * scd;
            }
#pragma unroll 1
            for (int l = 4 * qt; l < min(NA, 4 * qt + 4); ++l) {
                float d0, d1;
                umma::tmem_ld2(my + TM_SA + 2 * l, d0, d1);
                d0 *= scd;
                d1 *= scd;
                float jl[8];
                umma::tmem_ld8(my + TM_J + 8 * l, jl);
                __stcs(SBt + (32 + 2 * l) * TILE + r, d0);  // j_d feature rows for the scatter (Eq. 9)
                __stcs(SBt + (33 + 2 * l) * TILE + r, d1);
                p0 = fmaf(d0, jl[0], fmaf(d1, jl[3], p0));
                p1 = fmaf(d0, jl[1], fmaf(d1, jl[4], p1));
                p2 = fmaf(d0, jl[2], fmaf(d1, jl[5], p2));
            }
            // normal partials in rows 4..15 of the scratch (P1's d partials, rows 0..3, may
            // still be being read: no barrier needed before these writes)
            float *xn = xch + 4 * TILE;
            xn[(3 * qt + 0) * TILE + r] = p0;
            xn[(3 * qt + 1) * TILE + r] = p1;
            xn[(3 * qt + 2) * TILE + r] = p2;
            __syncthreads();
            const float n0 = xn[r] + xn[3 * TILE + r] + xn[6 * TILE + r] + xn[9 * TILE + r];
            const float n1 = xn[TILE + r] + xn[4 * TILE + r] + xn[7 * TILE + r] + xn[10 * TILE + r];
            const float n2 = xn[2 * TILE + r] + xn[5 * TILE + r] + xn[8 * TILE + r] + xn[11 * TILE + r];
            const float nn = sqrtf(n0 * n0 + n1 * n1 + n2 * n2);
            if (valid && qt == 0) eik += (nn - 1.f) * (nn - 1.f);
            // cin = [x, n, v, y] (field.py:237-239); quarter k stages block k of the 32
            float blk[8];
            float mc = 0.f;
            if (qt == 0) {
                blk[0] = x0; blk[1] = x1; blk[2] = x2; blk[3] = n0;
                blk[4] = n1; blk[5] = n2; blk[6] = v0; blk[7] = v1;
                nct[0] = n0;
                nct[TILE] = n1;
                nct[2 * TILE] = n2;
            } else if (qt == 1) {
                blk[0] = v2;
#pragma unroll
                for (int k = 1; k < 8; ++k) blk[k] = y[k - 1];
            } else if (qt == 2) {
#pragma unroll
                for (int k = 0; k < 8; ++k) blk[k] = y[7 + k];
            } else {
                blk[0] = y[15];
#pragma unroll
                for (int k = 1; k < 8; ++k) blk[k] = 0.f;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) mc = fmaxf(mc, fabsf(blk[k]));
            eCin = PS.guess(kCin);
            PS.contrib(kCin, mc);
            stage_blk<32>(S, TC, TCB, r, qt, blk, pow2i(eCin));
            if (valid && qt == 0) {
                sdf_out[p] = d_sdf;
                if (nrm_out) {
                    nrm_out[3 * p] = n0;
                    nrm_out[3 * p + 1] = n1;
                    nrm_out[3 * p + 2] = n2;
                }
                if (geo_out)
#pragma unroll
                    for (int o = 1; o < 16; ++o) geo_out[15 * p + o - 1] = y[o];
            }
            publish();
            PMARK(5);
            if (!PS.check(kCin, eCin)) {
                stage_blk<32>(S, TC, TCB, r, qt, blk, pow2i(eCin));
                publish();
                PMARK(6);
            }
        }
        if (warp == kMmaWarp) {  // converged MMA warp; elect.sync picks the issuing lane
            umma::gemm3w<2>(tb + TM_SA, S.K(TC, TCB, 32), S.K(WC1, WC1B, 32), ID_KK(64), false);
            umma::commit_elect(mbar);
            if (lane == 0) umma::bulk_s2g(fwt + FW_CIN, S.p(TC), TCB);
        }
        const bool jnext = ntile * TILE < P;
        if (jnext) j_load(ntile);  // next tile's d feature/dx: its latency hides under the Zc1 GEMM
        wait_mma(mbar, phase);
        PMARK(7);
        // ------------------------------------------------ P3: a1c -> Zc2
        uint32_t mc1 = 0u, mc2 = 0u;
        int eA1c, eA2c;
        {
            float z[2][8], m = 0.f;
            const float sc = pow2i(-(eCin + eC1));
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                umma::tmem_ld8(my + TM_SA + 8 * (i ? b1 : b0), z[i]);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const bool on = z[i][k] > 0.f;
                    mc1 |= on ? (1u << (8 * i + k)) : 0u;
                    z[i][k] = on ? z[i][k] * sc : 0.f;
                    m = fmaxf(m, z[i][k]);
                }
            }
            eA1c = PS.guess(kA1c);
            PS.contrib(kA1c, m);
            if (jnext) j_store();
            auto stg = [&](int e) {
                const float s = pow2i(e);
#pragma unroll
                for (int i = 0; i < 2; ++i) stage_blk<64>(S, TZ, T64B, r, i ? b1 : b0, z[i], s);
            };
            #pragma unroll 1
            for (int pass = 0;; ++pass) {  // stage; restage once if the predicted exponent missed
                stg(eA1c);
                publish();
                if (pass) break;
                PMARK(8);
                if (PS.check(kA1c, eA1c)) break;
            }
        }
        if (warp == kMmaWarp) {  // converged MMA warp; elect.sync picks the issuing lane
            umma::gemm3w<4>(tb + TM_SB, S.K(TZ, T64B, 64), S.K(WC2, WC2B, 64), ID_KK(64), false);
            // the previous tile's A2c store (TY) must be done before P4 restages TY: all but
            // this tile's A1 and CIN stores; the commit orders P4's staging after it
            if (lane == 0) umma::bulk_wait_read_n<2>();
            __syncwarp();
            umma::commit_elect(mbar);
            if (lane == 0) umma::bulk_s2g(fwt + FW_A1C, S.p(TZ), T64B);
        }
        wait_mma(mbar, phase);
        PMARK(10);
        // ------------------------------------------------ P4: a2c -> LOG
        {
            float z[2][8], m = 0.f;
            const float sc = pow2i(-(eA1c + eC2));
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                umma::tmem_ld8(my + TM_SB + 8 * (i ? b1 : b0), z[i]);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const bool on = z[i][k] > 0.f;
                    mc2 |= on ? (1u << (8 * i + k)) : 0u;
                    z[i][k] = on ? z[i][k] * sc : 0.f;
                    m = fmaxf(m, z[i][k]);
                }
            }
            eA2c = PS.guess(kA2c);
            PS.contrib(kA2c, m);
            // logits = C3 a2c (3 outputs): fp32 FMA partials over my 16 hidden units,
            // summed across the four quarter-threads of the row after the barrier
            {
                float lp0 = 0.f, lp1 = 0.f, lp2 = 0.f;
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int b = i ? b1 : b0;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        lp0 = fmaf(sh.c3[0][8 * b + k], z[i][k], lp0);
                        lp1 = fmaf(sh.c3[1][8 * b + k], z[i][k], lp1);
                        lp2 = fmaf(sh.c3[2][8 * b + k], z[i][k], lp2);
                    }
                }
                float *lg = reinterpret_cast<float *>(S.p(TLG)) + 3 * qt * TILE + r;
                lg[0] = lp0;
                lg[TILE] = lp1;
                lg[2 * TILE] = lp2;
            }
            auto stg = [&](int e) {
                const float s = pow2i(e);
#pragma unroll
                for (int i = 0; i < 2; ++i) stage_blk<64>(S, TY, T64B, r, i ? b1 : b0, z[i], s);
            };
            #pragma unroll 1
            for (int pass = 0;; ++pass) {  // stage; restage once if the predicted exponent missed
                stg(eA2c);  // into TY (the mask tile is dead): TX's A1 store may still be reading
                publish();
                if (pass) break;
                PMARK(11);
                if (PS.check(kA2c, eA2c)) break;
            }
        }
        if (t == kMmaWarp * 32) {  // the thread that issues (and drains) the tile stores
            umma::bulk_s2g(fwt + FW_A2C, S.p(TY), T64B);
            ws.fw_exp[tile] = make_int4(eA1, eCin, eA1c, eA2c);
        }
        {  // this quarter's two blocks: byte qt of the half-0 word (block qt) and of the half-1 word
            uint8_t *mb = reinterpret_cast<uint8_t *>(ws.fw_mask);
            const uint32_t qw[3] = {m1, mc1, mc2};
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                mb[4 * mask_idx(tile, k, 0, r) + qt] = static_cast<uint8_t>(qw[k]);
                mb[4 * mask_idx(tile, k, 1, r) + qt] = static_cast<uint8_t>(qw[k] >> 8);
            }
        }
        // ------------------------------------------------ P5: colours
        {
            if (qt == 0) {
                const float *lg = reinterpret_cast<const float *>(S.p(TLG)) + r;
                float l0 = 0.f, l1 = 0.f, l2 = 0.f;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    l0 += lg[3 * q * TILE];
                    l1 += lg[(3 * q + 1) * TILE];
                    l2 += lg[(3 * q + 2) * TILE];
                }
                const float cc0 = sigmoid_f(l0), cc1 = sigmoid_f(l1), cc2 = sigmoid_f(l2);
                nct[3 * TILE] = cc0;
                nct[4 * TILE] = cc1;
                nct[5 * TILE] = cc2;
                if (valid) {
                    col_out[3 * p] = cc0;
                    col_out[3 * p + 1] = cc1;
                    col_out[3 * p + 2] = cc2;
                }
            }
        }
    }
#ifdef NS2B_PHASE_PROF
    __syncthreads();
    if (blockIdx.x == 0 && t == 0) {
        printf("PHASEPROF fwd");
        for (int i = 0; i < 64; ++i)
            if (pacc[i]) printf(" %d:%lld", i, pacc[i]);
        printf("\n");
    }
#endif
    if (eik_sum) {
        double v = warp_sum(static_cast<double>(eik));
        if (lane == 0 && v != 0.0) atomicAdd(eik_sum, v);
    }
    if (t == kMmaWarp * 32) umma::bulk_wait_all();
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tb, 512);
}

// ---------------------------------------------------------------------------
// MLP forward, two tiles in flight (field_fwd2_kernel): the 512 threads form two
// independent 256-thread groups, each running the forward above on its own tiles (the
// CTA's even / odd tiles) with its own shared buffers, TMEM columns, mbarriers, named
// barrier and MMA-issuing warp, so one group's epilogue overlaps the other's MMAs,
// DMAs and barrier waits.  Per group:
//   threads: warp w (0..7) reads TMEM lane quadrant w % 4 and owns column blocks
//            4 (w / 4) .. 4 (w / 4) + 3 of every 64-wide row (32 columns);
//   TMEM:    two 64-column chain slots (Z1 -> A, Y -> B, JD -> A, Zc1 -> A, Zc2 -> B);
//   smem:    EB (24 KB): E (P0) -> M1 (P1) -> CIN (P2) -> the next tile's E (DMA'd in P3);
//            AB (32 KB): A1 (P1) -> A1c (P3) -> A2c hi (P4, store only);  plus row-scalar
//            exchange scratch.
// d feature/dx (J) is read straight from global memory in P2 (prefetched to L2 a tile
// ahead): it only enters the normal, so it needs neither registers a tile ahead nor TMEM.
// Results equal field_fwd_kernel's up to the order of the per-row partial sums.
constexpr uint32_t F2_H1S = TE;                       // H1' right after the weights
constexpr uint32_t F2_G0 = F2_H1S + 2 * WH1B;         // group 0 buffers
constexpr uint32_t F2_EB = 0, F2_AB = 2 * TEB, F2_XCH = F2_AB + 2 * T64B,  // offsets in a group block
                   F2_LG = F2_XCH + 8 * TILE * 4, F2_MK = F2_LG + 6 * TILE * 4, F2_FS = F2_MK + 24 * TILE,
                   F2_GB = F2_FS, F2_GBG = F2_FS + 32 * TILE * 4;  // F2_FS (kG): raw features [32][128]
constexpr uint32_t SMEM_FWD2 = F2_G0 + 2 * F2_GB, SMEM_FWD2G = F2_G0 + 2 * F2_GBG;
static_assert(SMEM_FWD2G <= 227 * 1024, "fwd2 shared memory");

__device__ __forceinline__ void group_sync(int g) { asm volatile("bar.sync %0, 256;" ::"r"(g + 1) : "memory"); }
__device__ __forceinline__ void group_publish(int g) {
    umma::fence_async_smem();
    umma::fence_before_sync();
    group_sync(g);
    umma::fence_after_sync();
}

// PredScale for a 256-thread group (the leader thread owns the prediction slot)
struct PredScaleG {
    uint32_t (*mx)[NSLOT];
    int *pred;
    int par;
    bool leader;
    __device__ __forceinline__ int guess(int k) const { return pred[k]; }
    __device__ __forceinline__ void contrib(int k, float m) {
        const uint32_t w = __reduce_max_sync(0xffffffffu, __float_as_uint(m));
        if ((threadIdx.x & 31) == 0 && w) atomicMax(&mx[par][k], w);
    }
    __device__ __forceinline__ bool check(int k, int &e) {
        const float m = __uint_as_float(mx[par][k]);
        const int ex = exp_for(m);
        const bool ok = !(m > 0.f) || (e <= ex + 1 && e >= ex - NS2B_PRED_SLACK);
        if (!ok) {
            e = ex - 1;
            if (leader) pred[k] = e;
        }
        return ok;
    }
};

// A 0/1 mask byte as 8 fp16 values (1.0 = 0x3C00): entry b of a 256-entry table, so a
// thread stages its 32 mask bits with four shared-memory loads instead of ~80 ALU ops
__device__ __forceinline__ void mask_lut_init(uint4 *lut) {
    for (int b = threadIdx.x; b < 256; b += blockDim.x) {
        auto h2 = [&](int k) {
            return ((b >> k) & 1 ? 0x3C00u : 0u) | ((b >> (k + 1)) & 1 ? 0x3C000000u : 0u);
        };
        lut[b] = make_uint4(h2(0), h2(2), h2(4), h2(6));
    }
}

__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}

// kG: the hash-grid gather runs inside the kernel (phase G, before P0): each thread
// interpolates its 8 levels of its sample, stages the encoding tile E straight into EB,
// keeps d feature/dx (J) in TMEM for P2's normal and writes J, E's hi part, x and v to
// the workspace for the backward -- the separate gather kernel and the E / J / x round
// trip through HBM disappear.
template <bool kG>
__global__ void __launch_bounds__(MLP_THREADS, 1)
field_fwd2_kernel(FieldDev f, const int32_t *__restrict__ count, float *__restrict__ sdf_out,
                  float *__restrict__ col_out, float *__restrict__ nrm_out, float *__restrict__ geo_out,
                  double *__restrict__ eik_sum, Workspace ws, float eik_w, const int64_t *__restrict__ eik_count,
                  const float *__restrict__ pos, const int32_t *__restrict__ ray_ids,
                  const double *__restrict__ dirs) {
    // with eik_count the Eikonal cotangent (trainer.py:229-235) is fused here, where the
    // normal is computed, and stored in place of the normal for the backward
    const bool fuse_eik = eik_count != nullptr;
    const float Pf = fuse_eik ? static_cast<float>(*eik_count) : 1.f;
    if (blockIdx.x == 0 && threadIdx.x == 0) ws.flags[0] = fuse_eik ? 1 : 0;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bars[4];  // [2g] chain MMAs, [2g+1] E-tile DMA
    __shared__ uint32_t wmax[6];
    __shared__ int wexp[6];
    __shared__ float h2row0[H];
    __shared__ float c3w[3][H];
    __shared__ uint32_t tmem_base_sh;
    __shared__ uint32_t gmx[2][2][NSLOT];
    __shared__ int gpred[2][NSLOT];
    __shared__ LevelSm lvs[NS2B_MAX_LEVELS];
    __shared__ uint4 m1lut[256];
    mask_lut_init(m1lut);
    const Smem S{smem_raw};
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int g = warp >> 3, gw = warp & 7, tg = t & 255;
    const int qd = gw & 3, qh = gw >> 2;
    const int r = 32 * qd + lane;
    const int NA = f.n_active;
    const int E = 3 + 2 * f.L;
    // ---- setup (all 512 threads)
    if (t < H) h2row0[t] = f.sdf_w[H * (E + 1) + t];
    if (t < 3 * H) c3w[t / H][t % H] = f.color_w[H * CIN + H * H + t];
    load_weight_tiles<true>(S, f, wmax, wexp, F2_H1S);
    if (t < 2 * NSLOT) {
        gmx[t / NSLOT][0][t % NSLOT] = 0u;
        gmx[t / NSLOT][1][t % NSLOT] = 0u;
        gpred[t / NSLOT][t % NSLOT] = 0;
    }
    if (t == 0) {
        for (int i = 0; i < 4; ++i) umma::mbar_init(bars + i, 1);
        umma::fence_barrier_init();
    }
    if (kG && t < NS2B_MAX_LEVELS) {
        lvs[t].lv = f.lv[t];
        lvs[t].sx = f.sx[t];
        lvs[t].sy = f.sy[t];
        lvs[t].sz = f.sz[t];
    }
    if (warp == 0) umma::tmem_alloc(&tmem_base_sh, kG ? 512 : 256);
    publish();
    const int eH1 = wexp[0], eH2 = wexp[1], eC1 = wexp[2], eC2 = wexp[3], eH1s = wexp[5];
    uint64_t *mbar = bars + 2 * g, *mbare = bars + 2 * g + 1;
    const uint32_t gbase = F2_G0 + g * (kG ? F2_GBG : F2_GB);
    const uint32_t EB = gbase + F2_EB, AB = gbase + F2_AB;
    float *xch = reinterpret_cast<float *>(S.p(gbase + F2_XCH));  // [2][128] d | [2][3][128] normal
    float *lgx = reinterpret_cast<float *>(S.p(gbase + F2_LG));   // [2][3][128] logit partials
    const uint32_t tb = tmem_base_sh + g * (kG ? 256 : 128);
    const uint32_t my = tb + (static_cast<uint32_t>(qd * 32) << 16);
    const uint32_t SA = 0, SB = 64, TJ = 128;  // TJ (kG): 16 levels x 8 columns of J
    float *fsx = reinterpret_cast<float *>(S.p(gbase + F2_FS));  // kG: raw features [32][128]
    const bool io = (gw == 7 && lane == 0);  // stores, DMAs, prefetches of the group
    PredScaleG PS{gmx[g], gpred[g], 1, tg == 0};
    uint32_t phase = 0, phasee = 0;
    const int P = *count;
    // The CTA's tiles are b, b + G, b + 2G, ... (the backward's order); group 0 takes the
    // first half of that list, group 1 the second, so the staging exponents the backward
    // reads change at most once per CTA (each group's predictions are sticky; alternating
    // groups would make the backward fold its TMEM accumulators on every tile)
    const int64_t G = gridDim.x;
    const int64_t ntl_all = (static_cast<int64_t>(P) + TILE - 1) / TILE;
    const int64_t ntl = blockIdx.x < ntl_all ? (ntl_all - blockIdx.x + G - 1) / G : 0;
    const int64_t half = (ntl + 1) / 2;
    const int64_t i_end = g == 0 ? half : ntl;
    const int64_t stride = G;
    const int64_t t0 = blockIdx.x + (g == 0 ? 0 : half) * G;
    const int64_t t_end = blockIdx.x + i_end * G;  // exclusive
    float eik = 0.f;
#ifdef NS2B_PHASE_PROF
    __shared__ long long pacc[64];
    long long plast = clock64();
    if (t < 64) pacc[t] = 0;
    __syncthreads();
#endif
    if (!kG && io && t0 < t_end) umma::bulk_g2s(S.p(EB), ws.e_tiles + t0 * 2 * TEB, 2 * TEB, mbare);
    int eE_cur = (!kG && t0 < t_end) ? ws.e_exp[t0] : 0;
    for (int64_t tile = t0; tile < t_end; tile += stride) {
        const int64_t p = tile * TILE + r;
        const bool valid = p < P;
        const int64_t ntile = tile + stride;
        const bool has_next = ntile < t_end;
        PS.par ^= 1;
        uint8_t *fwt = ws.fw_tiles + tile * static_cast<int64_t>(FWB);
        float *SBt = ws.sb + tile * SBROWS * TILE;
        float *nct = ws.fw_nc + tile * NCROWS * TILE + r;
        float x0, x1, x2, v0, v1, v2;
        int eE;
        if constexpr (!kG) {
            if (io && has_next) umma::prefetch_l2(ws.jac + ntile * JROWS * TILE, JROWS * TILE * 4);
            const float *xvt = ws.xv + tile * XVROWS * TILE + r;
            x0 = xvt[0];
            x1 = xvt[TILE];
            x2 = xvt[2 * TILE];
            v0 = xvt[3 * TILE];
            v1 = xvt[4 * TILE];
            v2 = xvt[5 * TILE];
            eE = eE_cur;
        } else {
            // ------------------------------------------ G: gather (_kernels.py:67-119) -> E, J
            x0 = x1 = x2 = v0 = v1 = v2 = 0.f;
            if (valid) {
                x0 = pos[3 * p];
                x1 = pos[3 * p + 1];
                x2 = pos[3 * p + 2];
                if (qh == 0) {
                    const int rr = ray_ids[p];
                    v0 = static_cast<float>(dirs[3 * rr]);  // field.py:216 (fp32 view dirs)
                    v1 = static_cast<float>(dirs[3 * rr + 1]);
                    v2 = static_cast<float>(dirs[3 * rr + 2]);
                }
            }
            const float un0 = normalize_coord(x0, f.lo[0], f.ext[0]);
            const float un1 = normalize_coord(x1, f.lo[1], f.ext[1]);
            const float un2 = normalize_coord(x2, f.lo[2], f.ext[2]);
            float fmax_ = qh == 0 ? fmaxf(fmaxf(fabsf(x0), fabsf(x1)), fmaxf(fabsf(x2), 1.f)) : 0.f;
            float *Jt = ws.jac + tile * JROWS * TILE + r;
#pragma unroll 1
            for (int lb = 0; lb < 8; lb += 2) {  // 2 levels (16 float2 loads) in flight
                float2 v[2][8];
                float fr[2][3];
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int l = 8 * qh + lb + i;
                    if (l < NA) {
                        const LevelInfo lv = lvs[l].lv;
                        int cx, cy, cz;
                        cell_frac(un0, lv.n, cx, fr[i][0]);
                        cell_frac(un1, lv.n, cy, fr[i][1]);
                        cell_frac(un2, lv.n, cz, fr[i][2]);
                        const float2 *tab = reinterpret_cast<const float2 *>(f.tables) + l * f.T;
#pragma unroll
                        for (int c = 0; c < 8; ++c)
                            v[i][c] = __ldg(tab + corner_row(lv, cx + ((c >> 2) & 1), cy + ((c >> 1) & 1), cz + (c & 1)));
                    }
                }
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const int l = 8 * qh + lb + i;
                    float f0 = 0.f, f1 = 0.f;
                    if (l < NA) {
                        const float fx = fr[i][0], fy = fr[i][1], fz = fr[i][2];
                        const float sx = lvs[l].sx, sy = lvs[l].sy, sz = lvs[l].sz;
                        float j00 = 0.f, j01 = 0.f, j02 = 0.f, j10 = 0.f, j11 = 0.f, j12 = 0.f;
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            const int ox = (c >> 2) & 1, oy = (c >> 1) & 1, oz = c & 1;
                            const float wx = ox ? fx : 1.f - fx, wy = oy ? fy : 1.f - fy, wz = oz ? fz : 1.f - fz;
                            const float w = wx * wy * wz;
                            const float dwx = (ox ? sx : -sx) * (wy * wz);
                            const float dwy = (oy ? sy : -sy) * (wx * wz);
                            const float dwz = (oz ? sz : -sz) * (wx * wy);
                            f0 = fmaf(w, v[i][c].x, f0);
                            f1 = fmaf(w, v[i][c].y, f1);
                            j00 = fmaf(dwx, v[i][c].x, j00);
                            j01 = fmaf(dwy, v[i][c].x, j01);
                            j02 = fmaf(dwz, v[i][c].x, j02);
                            j10 = fmaf(dwx, v[i][c].y, j10);
                            j11 = fmaf(dwy, v[i][c].y, j11);
                            j12 = fmaf(dwz, v[i][c].y, j12);
                        }
                        fmax_ = fmaxf(fmax_, fmaxf(fabsf(f0), fabsf(f1)));
                        float *jr = Jt + 6 * l * TILE;  // for the backward (evict-first)
                        __stcs(jr, j00);
                        __stcs(jr + TILE, j01);
                        __stcs(jr + 2 * TILE, j02);
                        __stcs(jr + 3 * TILE, j10);
                        __stcs(jr + 4 * TILE, j11);
                        __stcs(jr + 5 * TILE, j12);
                        const uint32_t c = my + TJ + 8 * l;  // for P2's normal
                        umma::tmem_st4(c, j00, j01, j02, j10);
                        umma::tmem_st2(c + 4, j11, j12);
                    }
                    fsx[(2 * l) * TILE + r] = f0;  // E feature columns 2l, 2l + 1
                    fsx[(2 * l + 1) * TILE + r] = f1;
                }
            }
            umma::tmem_st_wait();
            if (qh == 0 && valid) {  // x, v for the input-gradient pass (dynamic scenes)
                float *xvt = ws.xv + tile * XVROWS * TILE + r;
                __stcs(xvt, x0);
                __stcs(xvt + TILE, x1);
                __stcs(xvt + 2 * TILE, x2);
                __stcs(xvt + 3 * TILE, v0);
                __stcs(xvt + 4 * TILE, v1);
                __stcs(xvt + 5 * TILE, v2);
            }
            // E = [features 0..31 | x y z | 1 | 0 x 12]: half qh stages blocks 2qh, 2qh+1 (its
            // 8 levels) and block 4 + qh (x, 1 / zeros)
            int e = PS.guess(kE);
            PS.contrib(kE, fmax_);
            auto stg = [&](int ee) {
                const float sc = pow2i(ee);
                float blk[8];
#pragma unroll
                for (int bb = 0; bb < 2; ++bb) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) blk[k] = fsx[(16 * qh + 8 * bb + k) * TILE + r];
                    stage_blk<48>(S, EB, TEB, r, 2 * qh + bb, blk, sc);
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) blk[k] = 0.f;
                if (qh == 0) {
                    blk[0] = x0;
                    blk[1] = x1;
                    blk[2] = x2;
                    blk[3] = 1.f;
                }
                stage_blk<48>(S, EB, TEB, r, 4 + qh, blk, sc);
            };
            stg(e);  // EB: the previous tile's CIN store and Zc1 GEMM have finished with it
            group_publish(g);
            if (tg < NSLOT) gmx[g][PS.par ^ 1][tg] = 0u;  // (the slot reset moves here from P1)
            if (!PS.check(kE, e)) {
                stg(e);
                group_publish(g);
            }
            eE = e;
            PMARK(13);
            if (io) {  // E's hi part for the backward's dH1 GEMM
                umma::bulk_s2g(ws.e_tiles + tile * 2 * TEB, S.p(EB), TEB);
                ws.e_exp[tile] = e;
            }
        }
        // ------------------------------------------------ P0: Z1 = E H1^T -> A
        if (gw == 7) {
            if (!kG) umma::mbar_wait(mbare, phasee);
            umma::gemm3w<3>(tb + SA, S.K(EB, TEB, 48), S.K(WH1, WH1B, 48), ID_KK(64), false);
            if (lane == 0) umma::bulk_wait_read_n<0>();  // the previous tile's A1c store has left AB
            __syncwarp();
            umma::commit_elect(mbar);
        }
        phasee ^= 1u;
        wait_mma(mbar, phase);
        PMARK(1);
        // ------------------------------------------------ P1: a1 -> AB, M1 -> EB; d
        uint32_t m1 = 0u;  // my 32 hidden-unit bits (blocks 4qh..4qh+3)
        int eA1;
        float d_sdf;
        {
            // raw accumulator values; the result scale 2^-(eE + eH1) (a power of two: exact) is
            // applied to the partial SDF sum once and folded into the staging scale
            float z[4][8], ma = 0.f, dpart = 0.f;
            const int esc = -(eE + eH1);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int b = 4 * qh + i;
                umma::tmem_ld8(my + SA + 8 * b, z[i]);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const bool on = z[i][k] > 0.f;
                    m1 |= on ? (1u << (8 * i + k)) : 0u;
                    const float a = on ? z[i][k] : 0.f;
                    z[i][k] = a;
                    ma = fmaxf(ma, a);
                    dpart = fmaf(h2row0[8 * b + k], a, dpart);
                }
            }
            xch[qh * TILE + r] = dpart * pow2i(esc);
            eA1 = PS.guess(kA1);
            PS.contrib(kA1, ma * pow2i(esc));
            auto stg = [&](int e) {
                const float sa = pow2i(e + esc);
#pragma unroll
                for (int i = 0; i < 4; ++i) stage_blk<64>(S, AB, T64B, r, 4 * qh + i, z[i], sa);
            };
            stg(eA1);
#pragma unroll
            for (int i = 0; i < 4; ++i)  // M1 (exact in fp16: hi part only) into EB (E is dead)
                *reinterpret_cast<uint4 *>(S.p(EB) + umma::tile_off(r, 8 * (4 * qh + i), 64)) =
                    m1lut[(m1 >> (8 * i)) & 0xFFu];
            group_publish(g);
            PMARK(2);
            if (!kG && tg < NSLOT) gmx[g][PS.par ^ 1][tg] = 0u;
            if (!PS.check(kA1, eA1)) {
                stg(eA1);
                group_publish(g);
            }
            d_sdf = xch[r] + xch[TILE + r];
        }
        if (gw == 7) {
            umma::gemm3w<4>(tb + SB, S.K(AB, T64B, 64), S.K(WH2, WH2B, 64), ID_KK(16), false);
            umma::gemm2a<4>(tb + SA, S.K(EB, T64B, 64), S.MN(F2_H1S, WH1B, 48), ID_KM(48), false);
            umma::commit_elect(mbar);
            if (lane == 0) umma::bulk_s2g(fwt + FW_A1, S.p(AB), T64B);
        }
        // the first 4 levels of this thread's d feature/dx: their L2 latency hides under the
        // Y / JD GEMMs
        const float *jt = ws.jac + tile * JROWS * TILE + r;
        float jv0[4][6];
        if constexpr (!kG) {
            const float *jt0 = jt + 48 * qh * TILE;  // this half's 8 levels
            if (8 * qh + 8 <= NA) {  // all active (the common case): plain loads
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int k = 0; k < 6; ++k) jv0[i][k] = __ldcs(jt0 + (6 * i + k) * TILE);
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int k = 0; k < 6; ++k) jv0[i][k] = 8 * qh + i < NA ? __ldcs(jt0 + (6 * i + k) * TILE) : 0.f;
            }
        }
        wait_mma(mbar, phase);
        PMARK(4);
        // ------------------------------------------------ P2: normal, cin -> EB; Zc1 -> A
        int eCin;
        {
            float y[16];
            umma::tmem_ld8(my + SB, *reinterpret_cast<float(*)[8]>(y));
            umma::tmem_ld8(my + SB + 8, *reinterpret_cast<float(*)[8]>(y + 8));
            const float scy = pow2i(-(eA1 + eH2));
#pragma unroll
            for (int o = 0; o < 16; ++o) y[o] *= scy;
            y[0] = d_sdf;
            const float scd = pow2i(-eH1s);
            float p0 = 0.f, p1 = 0.f, p2 = 0.f;
            if (qh == 0) {
                float jx[4];
                umma::tmem_ld4(my + SA + 32, jx);
                p0 = jx[0] * scd;
                p1 = jx[1] * scd;
                p2 = jx[2] * scd;
            }
            // 4 levels per batch: the j_d feature rows go to the scatter's inputs, the normal
            // accumulates d . J
            // this half's 8 levels of j_d (16 columns) in one TMEM load
            float jda[16];
            umma::tmem_ld16(my + SA + 16 * qh, jda);
            auto batch = [&](int l0, int jo, const float (&jv)[4][6]) {  // jo: 0 / 4, a literal
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int l = l0 + i;
                    if (l < NA) {
                        const float d0 = jda[2 * (jo + i)] * scd, d1 = jda[2 * (jo + i) + 1] * scd;
                        __stcs(SBt + (32 + 2 * l) * TILE + r, d0);  // j_d feature rows for the scatter (Eq. 9)
                        __stcs(SBt + (33 + 2 * l) * TILE + r, d1);
                        p0 = fmaf(d0, jv[i][0], fmaf(d1, jv[i][3], p0));
                        p1 = fmaf(d0, jv[i][1], fmaf(d1, jv[i][4], p1));
                        p2 = fmaf(d0, jv[i][2], fmaf(d1, jv[i][5], p2));
                    }
                }
            };
            if constexpr (kG) {  // J from TMEM (the G phase put it there)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int l0 = 8 * qh + 4 * h;
                    if (l0 >= NA) break;
                    float jv[4][6];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        float jl[8];
                        umma::tmem_ld8(my + TJ + 8 * (l0 + i), jl);
#pragma unroll
                        for (int k = 0; k < 6; ++k) jv[i][k] = jl[k];
                    }
                    batch(l0, 4 * h, jv);
                }
            } else {
                // the first batch was loaded during P1's GEMMs; the second's 24 loads
                // (L2-resident) are issued before the first batch is consumed
                const int l1 = 8 * qh + 4;
                float jv1[4][6];
                const float *jt1 = jt + 6 * l1 * TILE;
                if (8 * qh + 8 <= NA) {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int k = 0; k < 6; ++k) jv1[i][k] = __ldcs(jt1 + (6 * i + k) * TILE);
                } else {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int k = 0; k < 6; ++k) jv1[i][k] = l1 + i < NA ? __ldcs(jt1 + (6 * i + k) * TILE) : 0.f;
                }
                if (8 * qh < NA) batch(8 * qh, 0, jv0);
                if (l1 < NA) batch(l1, 4, jv1);
            }
            float *xn = xch + 2 * TILE;  // [2][3][128]
            xn[(3 * qh + 0) * TILE + r] = p0;
            xn[(3 * qh + 1) * TILE + r] = p1;
            xn[(3 * qh + 2) * TILE + r] = p2;
            PMARK(5);
            group_sync(g);
            PMARK(6);
            const float n0 = xn[r] + xn[3 * TILE + r];
            const float n1 = xn[TILE + r] + xn[4 * TILE + r];
            const float n2 = xn[2 * TILE + r] + xn[5 * TILE + r];
            const float nn = sqrtf(n0 * n0 + n1 * n1 + n2 * n2);
            if (valid && qh == 0) eik += (nn - 1.f) * (nn - 1.f);
            // cin = [x, n, v, y] (field.py:237-239): half 0 stages blocks 0, 1; half 1 blocks 2, 3
            float blk[2][8];
            if (qh == 0) {
                blk[0][0] = x0; blk[0][1] = x1; blk[0][2] = x2; blk[0][3] = n0;
                blk[0][4] = n1; blk[0][5] = n2; blk[0][6] = v0; blk[0][7] = v1;
                blk[1][0] = v2;
#pragma unroll
                for (int k = 1; k < 8; ++k) blk[1][k] = y[k - 1];
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) blk[0][k] = y[7 + k];
                blk[1][0] = y[15];
#pragma unroll
                for (int k = 1; k < 8; ++k) blk[1][k] = 0.f;
            }
            float mc = 0.f;
#pragma unroll
            for (int k = 0; k < 8; ++k) mc = fmaxf(mc, fmaxf(fabsf(blk[0][k]), fabsf(blk[1][k])));
            eCin = PS.guess(kCin);
            PS.contrib(kCin, mc);
            auto stg = [&](int e) {
                const float sc = pow2i(e);
                stage_blk<32>(S, EB, TCB, r, 2 * qh, blk[0], sc);
                stage_blk<32>(S, EB, TCB, r, 2 * qh + 1, blk[1], sc);
            };
            stg(eCin);  // EB: the JD GEMM (M1) completed
            if (valid && qh == 0) {
                sdf_out[p] = d_sdf;
                if (fuse_eik) {  // trainer.py:229-235 (fp32, numpy's order): dL/dn of the Eikonal term
                    const float coef = eik_w * (2.f * (nn - 1.f) / fmaxf(nn, 1e-12f));
                    nct[0] = coef * n0 / Pf;
                    nct[TILE] = coef * n1 / Pf;
                    nct[2 * TILE] = coef * n2 / Pf;
                } else {
                    nct[0] = n0;
                    nct[TILE] = n1;
                    nct[2 * TILE] = n2;
                }
                if (nrm_out) {
                    nrm_out[3 * p] = n0;
                    nrm_out[3 * p + 1] = n1;
                    nrm_out[3 * p + 2] = n2;
                }
                if (geo_out)
#pragma unroll
                    for (int o = 1; o < 16; ++o) geo_out[15 * p + o - 1] = y[o];
            }
            group_publish(g);
            if (!PS.check(kCin, eCin)) {
                stg(eCin);
                group_publish(g);
            }
        }
        if (gw == 7) {
            umma::gemm3w<2>(tb + SA, S.K(EB, TCB, 32), S.K(WC1, WC1B, 32), ID_KK(64), false);
            if (lane == 0) umma::bulk_wait_read_n<0>();  // A1's store has left AB before P3 restages it
            __syncwarp();
            umma::commit_elect(mbar);
            if (lane == 0) umma::bulk_s2g(fwt + FW_CIN, S.p(EB), TCB);
        }
        PMARK(7);
        wait_mma(mbar, phase);
        PMARK(8);
        // ------------------------------------------------ P3: a1c -> AB; Zc2 -> B
        uint32_t mc1 = 0u, mc2 = 0u;
        int eA1c, eA2c;
        {
            // raw accumulator values: the result scale 2^-(eCin + eC1) is folded into the
            // staging scale (one multiply per element; powers of two, exact)
            float z[4][8], m = 0.f;
            const int esc = -(eCin + eC1);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                umma::tmem_ld8(my + SA + 8 * (4 * qh + i), z[i]);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const bool on = z[i][k] > 0.f;
                    mc1 |= on ? (1u << (8 * i + k)) : 0u;
                    z[i][k] = on ? z[i][k] : 0.f;
                    m = fmaxf(m, z[i][k]);
                }
            }
            eA1c = PS.guess(kA1c);
            PS.contrib(kA1c, m * pow2i(esc));
            auto stg = [&](int e) {
                const float s = pow2i(e + esc);
#pragma unroll
                for (int i = 0; i < 4; ++i) stage_blk<64>(S, AB, T64B, r, 4 * qh + i, z[i], s);
            };
#pragma unroll 1
            for (int pass = 0;; ++pass) {
                stg(eA1c);
                group_publish(g);
                if (pass) break;
                if (PS.check(kA1c, eA1c)) break;
            }
        }
        if (gw == 7) {
            umma::gemm3w<4>(tb + SB, S.K(AB, T64B, 64), S.K(WC2, WC2B, 64), ID_KK(64), false);
            if (lane == 0) {
                // A1c's store reads AB alongside the Zc2 GEMM; once it and CIN's store (EB) have
                // read their tiles, P4 may stage A2c into AB and EB can take the next E
                umma::bulk_s2g(fwt + FW_A1C, S.p(AB), T64B);
                umma::bulk_wait_read_n<0>();
                if (!kG && has_next) umma::bulk_g2s(S.p(EB), ws.e_tiles + ntile * 2 * TEB, 2 * TEB, mbare);
            }
            __syncwarp();
            umma::commit_elect(mbar);
        }
        PMARK(9);
        wait_mma(mbar, phase);
        PMARK(10);
        // ------------------------------------------------ P4: a2c (hi, store only) -> EB; logits
        {
            // raw accumulator values: the result scale 2^-(eA1c + eC2) is applied to the logit
            // partials once and folded into the staging scale (powers of two: exact)
            float z[4][8], m = 0.f;
            const int esc = -(eA1c + eC2);
            const float sc = pow2i(esc);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                umma::tmem_ld8(my + SB + 8 * (4 * qh + i), z[i]);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const bool on = z[i][k] > 0.f;
                    mc2 |= on ? (1u << (8 * i + k)) : 0u;
                    z[i][k] = on ? z[i][k] : 0.f;
                    m = fmaxf(m, z[i][k]);
                }
            }
            eA2c = PS.guess(kA2c);
            PS.contrib(kA2c, m * sc);
            float lp0 = 0.f, lp1 = 0.f, lp2 = 0.f;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int b = 4 * qh + i;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    lp0 = fmaf(c3w[0][8 * b + k], z[i][k], lp0);
                    lp1 = fmaf(c3w[1][8 * b + k], z[i][k], lp1);
                    lp2 = fmaf(c3w[2][8 * b + k], z[i][k], lp2);
                }
            }
            lgx[(3 * qh + 0) * TILE + r] = lp0 * sc;
            lgx[(3 * qh + 1) * TILE + r] = lp1 * sc;
            lgx[(3 * qh + 2) * TILE + r] = lp2 * sc;
            auto stg = [&](int e) {  // hi part only: the backward's weight-gradient GEMMs read nothing else
                const float s = pow2i(e + esc);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint4 h = make_uint4(pack_half2(z[i][0] * s, z[i][1] * s), pack_half2(z[i][2] * s, z[i][3] * s),
                                               pack_half2(z[i][4] * s, z[i][5] * s), pack_half2(z[i][6] * s, z[i][7] * s));
                    *reinterpret_cast<uint4 *>(S.p(AB) + umma::tile_off(r, 8 * (4 * qh + i), 64)) = h;
                }
            };
#pragma unroll 1
            for (int pass = 0;; ++pass) {
                stg(eA2c);
                group_publish(g);
                if (pass) break;
                if (PS.check(kA2c, eA2c)) break;
            }
        }
        if (io) {
            umma::bulk_s2g(fwt + FW_A2C, S.p(AB), T64B);  // (P0 waits for it before P1 restages AB)
            ws.fw_exp[tile] = make_int4(eA1, eCin, eA1c, eA2c);
        }
        if (!kG && has_next) eE_cur = ws.e_exp[ntile];
        PMARK(11);
        // ------------------------------------------------ P5: colours, masks
        if (qh == 0) {
            const float l0 = lgx[r] + lgx[3 * TILE + r];
            const float l1 = lgx[TILE + r] + lgx[4 * TILE + r];
            const float l2 = lgx[2 * TILE + r] + lgx[5 * TILE + r];
            const float cc0 = sigmoid_f(l0), cc1 = sigmoid_f(l1), cc2 = sigmoid_f(l2);
            nct[3 * TILE] = cc0;
            nct[4 * TILE] = cc1;
            nct[5 * TILE] = cc2;
            if (valid) {
                col_out[3 * p] = cc0;
                col_out[3 * p + 1] = cc1;
                col_out[3 * p + 2] = cc2;
            }
        }
        ws.fw_mask[mask_idx(tile, 0, qh, r)] = m1;  // this half's 32 hidden-unit bits
        ws.fw_mask[mask_idx(tile, 1, qh, r)] = mc1;
        ws.fw_mask[mask_idx(tile, 2, qh, r)] = mc2;
        PMARK(12);
    }
#ifdef NS2B_PHASE_PROF
    __syncthreads();
    if (blockIdx.x == 0 && t == 0) {
        printf("PHASEPROF fwd2");
        for (int i = 0; i < 64; ++i)
            if (pacc[i]) printf(" %d:%lld", i, pacc[i]);
        printf("\n");
    }
#endif
    if (eik_sum) {
        double v = warp_sum(static_cast<double>(eik));
        if (lane == 0 && v != 0.0) atomicAdd(eik_sum, v);
    }
    if (io) umma::bulk_wait_all();
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tmem_base_sh, kG ? 512 : 256);
}

// ---------------------------------------------------------------------------
// MLP backward (field.py:272-331, relu_mlp.py:132-216) from the forward's stored tiles:
//   B0 dlog = dL/dc c(1-c) -> U2 = DLOG C3,           dC3 += A2c^T DLOG
//   B1 u2 = U2 . mc2       -> U1 = U2 C2,             dC2 += U2^T A1c
//   B2 u1 = U1 . mc1       -> DCIN = U1 C1,           dC1 += U1^T CIN
//   B3 q, dly              -> U = DLY H2,             dH2 += A1^T DLY
//   B4 u = U . m1, mvec = [J q, q] -> DE = U H1, PV = MV H1^T;  dH1 += U^T E + S1^T MV
//   B5 dH2[0] += PV^T 1 (Theorem 1); DE and q -> the scatter's inputs.
// The forward's tiles arrive by bulk DMA (A2c, A1 -> TW; A1c -> TZ; CIN -> TC; E -> TE),
// each issued as soon as its buffer's last reader has retired.  Weight-gradient GEMMs
// run behind the chain GEMMs in the in-order MMA pipe; only B4's and B5's are awaited.  Weight gradients
// accumulate in TMEM across tiles while their operand exponents stay the same (sticky
// predictions), and are folded into global memory every kFoldTiles tiles, when an
// exponent changes, and at the end.
// Backward chain GEMMs with the A operand in tensor memory (NS2B_BWD_TA, needs NS2B_WG1):
// an epilogue block of 8 columns goes to the TMEM A region as packed hi and lo halves
// (tcgen05.st) and, as its hi half only, to the shared-memory tile the weight-gradient
// GEMMs read.  The chain GEMMs then read no shared memory for A (3 of the 4 operand
// streams of a split K step), and the smem tiles hold hi halves only.
#if defined(NS2B_BWD_TA) && !defined(NS2B_WG1)
#error "NS2B_BWD_TA needs NS2B_WG1 (the smem tiles carry hi halves only)"
#endif
template <int C>
__device__ __forceinline__ void stage_blk_ta(const Smem &s, uint32_t off, int r, int b, const float *v, float sc,
                                             uint32_t ta_hi, uint32_t ta_lo) {
    uint4 h, l;
    umma::split2<0>(v[0] * sc, v[1] * sc, h.x, l.x);
    umma::split2<0>(v[2] * sc, v[3] * sc, h.y, l.y);
    umma::split2<0>(v[4] * sc, v[5] * sc, h.z, l.z);
    umma::split2<0>(v[6] * sc, v[7] * sc, h.w, l.w);
    *reinterpret_cast<uint4 *>(s.p(off) + umma::tile_off(r, 8 * b, C)) = h;
    umma::tmem_st4u(ta_hi + 4 * b, h);
    umma::tmem_st4u(ta_lo + 4 * b, l);
}
// hi half only (an operand only weight-gradient GEMMs read, with NS2B_WG1)
template <int C>
__device__ __forceinline__ void stage_blk_hi(const Smem &s, uint32_t off, int r, int b, const float *v, float sc) {
    const uint4 h = make_uint4(pack_half2(v[0] * sc, v[1] * sc), pack_half2(v[2] * sc, v[3] * sc),
                               pack_half2(v[4] * sc, v[5] * sc), pack_half2(v[6] * sc, v[7] * sc));
    *reinterpret_cast<uint4 *>(s.p(off) + umma::tile_off(r, 8 * b, C)) = h;
}

enum Acc { aC3, aC2, aC1, aH2, aH1a, aH1b, NACC };

// Fold one TMEM weight-gradient accumulator (scaled by 2^-e) into global memory.  All
// threads call it; the accumulator's MMAs have completed.  Out of line: it runs only
// every kFoldTiles tiles or on a scale change, and inlining its 18 call sites made the
// backward kernel's code overflow the instruction cache.
__device__ __noinline__ void fold_acc(int j, int e, uint32_t my, int E, const float *__restrict__ h2row0,
                                      const float *__restrict__ sdf_w, float *__restrict__ g_sdf,
                                      float *__restrict__ g_color) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int qd = warp & 3, qt = warp >> 2;
    const int jrow = 16 * qd + lane;
    const int b0 = qt, b1 = qt + 4;
    {
        const float sc = pow2i(-e);
        float d[8];
        switch (j) {
        case aC3:  // dC3^T: row = hidden unit, col = output (3)
            umma::tmem_ld8(my + TB_DC3, d);
            if (lane < 16 && qt == 0)
                for (int o = 0; o < 3; ++o) atomicAdd(g_color + H * CIN + H * H + o * H + jrow, d[o] * sc);
            break;
        case aC2:
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int b = i ? b1 : b0;
                umma::tmem_ld8(my + TB_DC2 + 8 * b, d);
                if (lane < 16)
#pragma unroll
                    for (int k = 0; k < 8; ++k) atomicAdd(g_color + H * CIN + jrow * H + 8 * b + k, d[k] * sc);
            }
            break;
        case aC1:
            umma::tmem_ld8(my + TB_DC1 + 8 * qt, d);
            if (lane < 16)
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (8 * qt + k < CIN) atomicAdd(g_color + jrow * CIN + 8 * qt + k, d[k] * sc);
            break;
        case aH2:  // dH2^T: row = hidden unit, col = output unit
            umma::tmem_ld8(my + TB_DH2 + 8 * (qt & 1), d);
            if (lane < 16 && qt < 2)
#pragma unroll
                for (int k = 0; k < 8; ++k) atomicAdd(g_sdf + H * (E + 1) + (8 * qt + k) * H + jrow, d[k] * sc);
            break;
        case aH1a:
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int b = i ? b1 : b0;
                umma::tmem_ld8(my + TB_DH1A + 8 * (b < 6 ? b : 0), d);
                if (lane < 16 && b < 6)
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int rc = h1_col(8 * b + k, E);
                        if (rc >= 0) atomicAdd(g_sdf + jrow * (E + 1) + rc, d[k] * sc);
                    }
            }
            break;
        default: {  // G = M1^T MV: dH1 += H2[0][j] G[j],  dH2[0][j] += H1[j] . G[j]
            float dot = 0.f;
            const float h2j = lane < 16 ? h2row0[jrow] : 0.f;
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int b = i ? b1 : b0;
                umma::tmem_ld8(my + TB_DH1B + 8 * (b < 6 ? b : 0), d);
                if (lane < 16 && b < 6)
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int rc = h1_col(8 * b + k, E);
                        if (rc >= 0) {
                            atomicAdd(g_sdf + jrow * (E + 1) + rc, h2j * d[k] * sc);
                            dot = fmaf(sdf_w[jrow * (E + 1) + rc], d[k], dot);
                        }
                    }
            }
            if (lane < 16 && dot != 0.f) atomicAdd(g_sdf + H * (E + 1) + jrow, dot * sc);
            break;
        }
        }
    }
}

// Accumulators fold to global memory on a scale change and at the end only: periodic
// folds (every 32 / 128 tiles) cost 0.4 / 0.12 ms per launch -- all 148 CTAs fold at once
// and their float atomics collide -- while an fp32 TMEM run over a CTA's ~1.2k tiles is
// still ~1e-5 relative.
constexpr int kFoldTiles = 1 << 20;

__global__ void __launch_bounds__(MLP_THREADS, 1)
field_bwd_kernel(FieldDev f, const int32_t *__restrict__ count, const float *__restrict__ dl_dc,
                 const float *__restrict__ dl_dsdf, const float *__restrict__ dl_dn_extra, float eik_w,
                 const int64_t *__restrict__ eik_count, float *__restrict__ g_sdf, float *__restrict__ g_color,
                 Workspace ws, int want_xin) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // [0] chain MMAs, [1] weight-gradient MMAs, [2..6] DMA into TW (A2c), TZ (A1c), TC (CIN),
    // TE (E), TA1 (A1)
    __shared__ uint64_t bars[8];
    __shared__ MlpShared sh;
    uint64_t *mbar = bars, *mbarw = bars + 1, *mb_w = bars + 2, *mb_z = bars + 3, *mb_c = bars + 4,
             *mb_e = bars + 5, *mb_a = bars + 6, *mb_in = bars + 7;
    // the stored tiles arrive as fp16 hi parts only, so TW's second half holds A1: its
    // DMA no longer waits for dC3 to release TW
    constexpr uint32_t TA1 = TW + T64B;
    // ... and TE's second half (E also arrives as its hi part) holds a full tile's per-sample
    // inputs, DMA'd while the previous tile runs: masks [4][128] uint2 | n, c [6][128] |
    // dL/dc [128][3] | dL/dsdf [128] | the forward's exponents (int4)
    constexpr uint32_t TIN = TE + TEB, IN_MK = TIN, IN_NC = IN_MK + 6 * TILE * 4,
                       IN_DC = IN_NC + NCROWS * TILE * 4, IN_DS = IN_DC + 3 * TILE * 4, IN_EX = IN_DS + TILE * 4,
                       IN_BYTES = IN_EX + 16 - TIN;
    static_assert(IN_BYTES <= TEB, "per-tile inputs fit in TE's free half");
    const Smem S{smem_raw};
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
#ifdef NS2B_BWD_TA
    // the chain GEMMs' A operands in TMEM (the second chain slot: hi | lo), one result slot
    constexpr uint32_t TA_H = TB_SB, TA_L = TB_SB + 32, SLB = TB_SA;
#define STG_A(C, off, part, b, v, sc) stage_blk_ta<C>(S, off, r, b, v, sc, my + TA_H, my + TA_L)
#define PUB_A()              \
    do {                     \
        umma::tmem_st_wait(); \
        publish();           \
    } while (0)
#define CHAIN(NK, d, off, part, KC, bop, idesc) umma::gemm3t<NK>(d, tb + TA_H, tb + TA_L, bop, idesc, false)
#else
    constexpr uint32_t SLB = TB_SB;
#define STG_A(C, off, part, b, v, sc) stage_blk<C>(S, off, part, r, b, v, sc)
#define PUB_A() publish()
#define CHAIN(NK, d, off, part, KC, bop, idesc) umma::gemm3w<NK>(d, S.K(off, part, KC), bop, idesc, false)
#endif
#ifdef NS2B_WG1  // operands only the weight-gradient GEMMs read: hi halves
#define STG_W(C, off, part, b, v, sc) stage_blk_hi<C>(S, off, r, b, v, sc)
#else
#define STG_W(C, off, part, b, v, sc) stage_blk<C>(S, off, part, r, b, v, sc)
#endif
    const int qd = warp & 3, qt = warp >> 2;
    const int r = 32 * qd + lane;
    const int E = 3 + 2 * f.L;
    const int NA = f.n_active;
    mlp_setup<false>(S, f, sh, bars, 8);
    const int eH1 = sh.wexp[0], eH2 = sh.wexp[1], eC1 = sh.wexp[2], eC2 = sh.wexp[3], eC3 = sh.wexp[4];
    const float *h2row0 = sh.h2row0;
    const uint32_t tb = sh.tmem_base;
    const uint32_t my = tb + (static_cast<uint32_t>(qd * 32) << 16);
    uint32_t phase = 0, phasew = 0, ph_w = 0, ph_z = 0, ph_c = 0, ph_e = 0, ph_a = 0, ph_in = 0;
    PredScale PS{sh.slot_mx, sh.slot_pred, 1};
    const int P = *count;
    const float Pf = eik_count ? static_cast<float>(*eik_count) : 1.f;
    // the forward may already have turned the normal rows into the Eikonal cotangent
    const bool gn_fused = ws.flags[0] != 0;
    const int jrow = 16 * qd + lane;  // weight row (lanes 0..15) of the M=64 accumulators
    const int b0 = qt, b1 = qt + 4;
    const int nsdf = H * (E + 1) + NOUT * H;

    // ---- weight-gradient accumulators (TMEM) and their folds into global memory
    int acc_e[NACC];
    bool acc_live[NACC];
#pragma unroll
    for (int j = 0; j < NACC; ++j) {
        acc_e[j] = 0;
        acc_live[j] = false;
    }
    auto fold = [&](int j) {
        fold_acc(j, acc_e[j], my, E, h2row0, f.sdf_w, g_sdf, g_color);
        acc_live[j] = false;
    };
    // before a weight-gradient GEMM into j with operand exponent sum e: fold on a scale
    // change; returns the accumulate flag
    auto acc_begin = [&](int j, int e) -> bool {
        if (acc_live[j] && acc_e[j] != e) {
            fold(j);
            block_sync_tc();
        }
        const bool accumulate = acc_live[j];
        acc_e[j] = e;
        acc_live[j] = true;
        return accumulate;
    };
    (void)nsdf;

    float jv[4][6];
    auto j_load = [&](int64_t tl) {
        const float *jt = ws.jac + tl * JROWS * TILE;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (4 * qt + i < NA) {
                const float *jr = jt + 6 * (4 * qt + i) * TILE + r;
#pragma unroll
                for (int k = 0; k < 6; ++k) jv[i][k] = __ldcs(jr + k * TILE);
            }
    };
    auto j_store = [&]() {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (4 * qt + i < NA) {
                const uint32_t c = my + TB_J + 8 * (4 * qt + i);
                umma::tmem_st4(c, jv[i][0], jv[i][1], jv[i][2], jv[i][3]);
                umma::tmem_st2(c + 4, jv[i][4], jv[i][5]);
            }
        umma::tmem_st_wait();
    };
    auto fwt = [&](int64_t tl) { return ws.fw_tiles + tl * static_cast<int64_t>(FWB); };
    auto dma = [&](uint32_t soff, const uint8_t *g, uint32_t bytes, uint64_t *mb) {
        umma::bulk_g2s<true>(S.p(soff), g, bytes, mb);
    };
    {
        const int64_t t0 = blockIdx.x;
        if (t0 * TILE < P) {
            if (t == kDmaThread) {
                dma(TW, fwt(t0) + FW_A2C, T64B, mb_w);
                dma(TA1, fwt(t0) + FW_A1, T64B, mb_a);
                dma(TZ, fwt(t0) + FW_A1C, T64B, mb_z);
                dma(TC, fwt(t0) + FW_CIN, TCB, mb_c);
                dma(TE, ws.e_tiles + t0 * 2 * TEB, TEB, mb_e);  // E hi part (weight gradient)
            }
            j_load(t0);
            j_store();
        }
    }
    // per-sample inputs of a tile, loaded a tile ahead (their latency then hides behind
    // the previous tile's last phase instead of stalling B0)
    struct BwdIn {
        float gc0, gc1, gc2, cc0, cc1, cc2, gd, n0, n1, n2;
        uint2 mk;
    };
    // per-sample inputs of a tile: full tiles arrive by one batched bulk DMA into TIN (issued
    // during the previous tile's B1); the partial last tile (and misaligned caller
    // buffers) read global memory directly
    const bool in_dma_ok = ((reinterpret_cast<uintptr_t>(dl_dc) | reinterpret_cast<uintptr_t>(dl_dsdf)) & 15u) == 0;
    auto in_full = [&](int64_t tl) { return in_dma_ok && (tl + 1) * TILE <= P; };
    auto in_dma = [&](int64_t tl) {  // one thread
        umma::mbar_expect_tx(mb_in, IN_BYTES);
        umma::bulk_g2s_tx(S.p(IN_MK), ws.fw_mask + tl * 6 * TILE, 6 * TILE * 4, mb_in);
        umma::bulk_g2s_tx(S.p(IN_NC), ws.fw_nc + tl * NCROWS * TILE, NCROWS * TILE * 4, mb_in);
        umma::bulk_g2s_tx(S.p(IN_DC), dl_dc + 3 * tl * TILE, 3 * TILE * 4, mb_in);
        umma::bulk_g2s_tx(S.p(IN_DS), dl_dsdf + tl * TILE, TILE * 4, mb_in);
        umma::bulk_g2s_tx(S.p(IN_EX), ws.fw_exp + tl, 16, mb_in);
    };
    auto read_in = [&](int64_t tl, int4 &fe) {
        BwdIn v{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, make_uint2(0u, 0u)};
        if (in_full(tl)) {
            umma::mbar_wait(mb_in, ph_in);
            ph_in ^= 1u;
            v.mk = mask_quarter(reinterpret_cast<const uint32_t *>(S.p(IN_MK)) + r, TILE, qt);
            const float *nc = reinterpret_cast<const float *>(S.p(IN_NC)) + r;
            if (qt == 0) {
                const float *dc = reinterpret_cast<const float *>(S.p(IN_DC)) + 3 * r;
                v.gc0 = dc[0];
                v.gc1 = dc[1];
                v.gc2 = dc[2];
                v.cc0 = nc[3 * TILE];
                v.cc1 = nc[4 * TILE];
                v.cc2 = nc[5 * TILE];
                v.gd = reinterpret_cast<const float *>(S.p(IN_DS))[r];
            }
            v.n0 = nc[0];
            v.n1 = nc[TILE];
            v.n2 = nc[2 * TILE];
            fe = *reinterpret_cast<const int4 *>(S.p(IN_EX));
            return v;
        }
        const int64_t pp = tl * TILE + r;
        v.mk = mask_quarter(ws.fw_mask + mask_idx(tl, 0, 0, r), TILE, qt);
        fe = ws.fw_exp[tl];
        if (pp < P) {
            const float *nc = ws.fw_nc + tl * NCROWS * TILE + r;
            if (qt == 0) {
                v.gc0 = dl_dc[3 * pp];
                v.gc1 = dl_dc[3 * pp + 1];
                v.gc2 = dl_dc[3 * pp + 2];
                v.cc0 = nc[3 * TILE];
                v.cc1 = nc[4 * TILE];
                v.cc2 = nc[5 * TILE];
                v.gd = dl_dsdf[pp];
            }
            v.n0 = nc[0];
            v.n1 = nc[TILE];
            v.n2 = nc[2 * TILE];
        }
        return v;
    };
    if (t == kDmaThread && in_full(blockIdx.x)) in_dma(blockIdx.x);
    int eE_cur = static_cast<int64_t>(blockIdx.x) * TILE < P ? ws.e_exp[blockIdx.x] : 0;
    // each tile's per-sample inputs are read at the end of the previous tile (its B5)
    int4 fe_nx = make_int4(0, 0, 0, 0);
    BwdIn in_nx{};
    if (static_cast<int64_t>(blockIdx.x) * TILE < P) in_nx = read_in(blockIdx.x, fe_nx);
    int ntiles_done = 0;
#ifdef NS2B_PHASE_PROF
    __shared__ long long pacc[64];
    long long plast = clock64();
    if (t < 64) pacc[t] = 0;
    __syncthreads();
#endif
    for (int64_t base = static_cast<int64_t>(blockIdx.x) * TILE; base < P;
         base += static_cast<int64_t>(gridDim.x) * TILE) {
        const int64_t p = base + r;
        const bool valid = p < P;
        const int64_t tile = base / TILE;
        const int64_t ntile = tile + gridDim.x;
        const bool has_next = ntile * TILE < P;
        PS.par ^= 1;
        float *SBt = ws.sb + tile * SBROWS * TILE;
        if (t == kDmaThread && has_next) {  // next tile's inputs -> L2 while this one runs
            umma::prefetch_l2(fwt(ntile), FWB);
            umma::prefetch_l2(ws.jac + ntile * JROWS * TILE, JROWS * TILE * 4);
            umma::prefetch_l2(ws.e_tiles + ntile * 2 * TEB, TEB);
        }
        // per-sample inputs (DMA'd during the previous tile)
        const int4 fe = fe_nx;  // read at the end of the previous tile
        const BwdIn in = in_nx;
        PMARK(19);
        const uint32_t m1 = in.mk.x & 0xFFFFu, mc1 = in.mk.x >> 16, mc2 = in.mk.y;
        const int eA1 = fe.x, eCin = fe.y, eA1c = fe.z, eA2c = fe.w;
        const int eE = eE_cur;  // loaded during the previous tile
        const float gc0 = in.gc0, gc1 = in.gc1, gc2 = in.gc2, gd = in.gd;
        const float cc0 = in.cc0, cc1 = in.cc1, cc2 = in.cc2;
        float gn0 = 0.f, gn1 = 0.f, gn2 = 0.f;
        if (valid) {
            const float n0 = in.n0, n1 = in.n1, n2 = in.n2;
            if (dl_dn_extra) {
                gn0 = dl_dn_extra[3 * p];
                gn1 = dl_dn_extra[3 * p + 1];
                gn2 = dl_dn_extra[3 * p + 2];
            }
            if (gn_fused) {  // fused by the forward (same arithmetic)
                gn0 += n0;
                gn1 += n1;
                gn2 += n2;
            } else if (eik_w != 0.f) {  // trainer.py:229-235 (fp32, numpy's order)
                const float nn = sqrtf(n0 * n0 + n1 * n1 + n2 * n2);
                const float coef = eik_w * (2.f * (nn - 1.f) / fmaxf(nn, 1e-12f));
                gn0 += coef * n0 / Pf;
                gn1 += coef * n1 / Pf;
                gn2 += coef * n2 / Pf;
            }
        }
        // ------------------------------------------------ B0: dlog -> U2, dC3
        int eD;
        {
            float dlog[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) dlog[k] = 0.f;
            if (qt == 0) {  // field.py:304
                dlog[0] = gc0 * cc0 * (1.f - cc0);
                dlog[1] = gc1 * cc1 * (1.f - cc1);
                dlog[2] = gc2 * cc2 * (1.f - cc2);
            }
            eD = PS.guess(kDlog);
            PS.contrib(kDlog, fmaxf(fabsf(dlog[0]), fmaxf(fabsf(dlog[1]), fabsf(dlog[2]))));
            PMARK(20);
            #pragma unroll 1
            for (int pass = 0;; ++pass) {  // stage; restage once if the predicted exponent missed
                if (qt < 2) STG_A(16, TD, TDB, qt, dlog, pow2i(eD));
                PUB_A();
                if (pass) break;
                PMARK(1);
                if (t < NSLOT) sh.slot_mx[PS.par ^ 1][t] = 0u;
                if (PS.check(kDlog, eD)) break;
            }
        }
        {
            const bool acc = acc_begin(aC3, eA2c + eD);
            if (warp == kMmaWarp) {  // converged MMA warp; elect.sync picks the issuing lane
                CHAIN(1, tb + TB_SA, TD, TDB, 16, S.MN(WC3, WC3B, 64), ID_KM(64));
                umma::commit_elect(mbar);
                PWAIT(umma::mbar_wait(mb_w, ph_w));
                WG_ACT_A<8>(tb + TB_DC3, S.MN(TW, T64B, 64), S.MN(TD, TDB, 16), ID_WG(16), acc);
            }
            ph_w ^= 1u;
        }
        wait_mma(mbar, phase);
        PMARK(3);
        // ------------------------------------------------ B1: u2 -> U1, dC2
        // every thread read this tile's inputs from TIN before B0's barrier: next tile's
        if (t == kDmaThread && has_next && in_full(ntile)) in_dma(ntile);
        if (has_next) eE_cur = ws.e_exp[ntile];
        int eU2;
        {
            float u[2][8], m = 0.f;
            const float sc = pow2i(-(eD + eC3));
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                umma::tmem_ld8(my + TB_SA + 8 * (i ? b1 : b0), u[i]);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    u[i][k] = ((mc2 >> (8 * i + k)) & 1u) ? u[i][k] * sc : 0.f;
                    m = fmaxf(m, fabsf(u[i][k]));
                }
            }
            eU2 = PS.guess(kU2);
            PS.contrib(kU2, m);
            auto stg = [&](int e) {
                const float s = pow2i(e);
#pragma unroll
                for (int i = 0; i < 2; ++i) STG_A(64, TY, T64B, i ? b1 : b0, u[i], s);
            };
            #pragma unroll 1
            for (int pass = 0;; ++pass) {  // stage; restage once if the predicted exponent missed
                stg(eU2);
                publish();
                if (pass) break;
                PMARK(4);
                if (PS.check(kU2, eU2)) break;
            }
        }
        {
            const bool acc = acc_begin(aC2, eU2 + eA1c);
            if (warp == kMmaWarp) {  // converged MMA warp; elect.sync picks the issuing lane
                CHAIN(4, tb + SLB, TY, T64B, 64, S.MN(WC2, WC2B, 64), ID_KM(64));
                umma::commit_elect(mbar);
                PWAIT(umma::mbar_wait(mb_z, ph_z));
                WG_ACT_B<8>(tb + TB_DC2, S.MN(TY, T64B, 64), S.MN(TZ, T64B, 64), ID_WG(64), acc);
            }
            ph_z ^= 1u;
        }
        wait_mma(mbar, phase);
        PMARK(6);
        // ------------------------------------------------ B2: u1 -> DCIN, dC1
        int eU1;
        {
            float u[2][8], m = 0.f;
            const float sc = pow2i(-(eU2 + eC2));
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                umma::tmem_ld8(my + SLB + 8 * (i ? b1 : b0), u[i]);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    u[i][k] = ((mc1 >> (8 * i + k)) & 1u) ? u[i][k] * sc : 0.f;
                    m = fmaxf(m, fabsf(u[i][k]));
                }
            }
            eU1 = PS.guess(kU1);
            PS.contrib(kU1, m);
            auto stg = [&](int e) {
                const float s = pow2i(e);
#pragma unroll
                for (int i = 0; i < 2; ++i) STG_A(64, TX, T64B, i ? b1 : b0, u[i], s);
            };
            #pragma unroll 1
            for (int pass = 0;; ++pass) {  // stage; restage once if the predicted exponent missed
                stg(eU1);
                publish();
                if (pass) break;
                PMARK(7);
                if (PS.check(kU1, eU1)) break;
            }
        }
        {
            const bool acc = acc_begin(aC1, eU1 + eCin);
            if (warp == kMmaWarp) {  // converged MMA warp; elect.sync picks the issuing lane
                CHAIN(4, tb + TB_SA, TX, T64B, 64, S.MN(WC1, WC1B, 32), ID_KM(32));
                umma::commit_elect(mbar);
                // TW is free (dC3 of B0 completed before B1's chain GEMM did): next tile's A2c
                if (lane == 0 && has_next) dma(TW, fwt(ntile) + FW_A2C, T64B, mb_w);
                PWAIT(umma::mbar_wait(mb_c, ph_c));
                WG_ACT_B<8>(tb + TB_DC1, S.MN(TX, T64B, 64), S.MN(TC, TCB, 32), ID_WG(32), acc);
            }
            ph_c ^= 1u;
        }
        wait_mma(mbar, phase);
        PMARK(9);
        // ------------------------------------------------ B3: q, dly -> U, dH2
        float q0, q1, q2;
        int eDLY;
        {
            const float sc3 = pow2i(-(eU1 + eC1));
            float c0[8], c1[8], c2[8], c3[8];
            umma::tmem_ld8(my + TB_SA, c0);
            umma::tmem_ld8(my + TB_SA + 8, c1);
            umma::tmem_ld8(my + TB_SA + 16, c2);
            umma::tmem_ld8(my + TB_SA + 24, c3);
            q0 = gn0 + c0[3] * sc3;  // field.py:308-312
            q1 = gn1 + c0[4] * sc3;
            q2 = gn2 + c0[5] * sc3;
            if (want_xin && qt == 2 && valid) {  // dl_dx / dl_dv colour-input parts (field.py:307,309)
                float *xi = ws.xin + tile * XINROWS * TILE + r;
                xi[0] = c0[0] * sc3;
                xi[TILE] = c0[1] * sc3;
                xi[2 * TILE] = c0[2] * sc3;
                xi[3 * TILE] = c0[6] * sc3;
                xi[4 * TILE] = c0[7] * sc3;
                xi[5 * TILE] = c1[0] * sc3;
            }
            // dly = [dd + dcin[9], dcin[10..24]]: block 0 (quarter 0), block 1 (quarter 1)
            float blk[8];
            if (qt == 0) {
                blk[0] = gd + c1[1] * sc3;
#pragma unroll
                for (int k = 1; k < 7; ++k) blk[k] = c1[1 + k] * sc3;
                blk[7] = c2[0] * sc3;
            } else if (qt == 1) {
#pragma unroll
                for (int k = 0; k < 7; ++k) blk[k] = c2[1 + k] * sc3;
                blk[7] = c3[0] * sc3;
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) blk[k] = 0.f;
            }
            float m = 0.f;
#pragma unroll
            for (int k = 0; k < 8; ++k) m = fmaxf(m, fabsf(blk[k]));
            eDLY = PS.guess(kDly);
            PS.contrib(kDly, m);
            #pragma unroll 1
            for (int pass = 0;; ++pass) {  // stage; restage once if the predicted exponent missed
                if (qt < 2) STG_A(16, TD, TDB, qt, blk, pow2i(eDLY));
                PUB_A();
                if (pass) break;
                PMARK(10);
                if (PS.check(kDly, eDLY)) break;
            }
        }
        {
            const bool acc = acc_begin(aH2, eA1 + eDLY);
            if (warp == kMmaWarp) {  // converged MMA warp; elect.sync picks the issuing lane
                CHAIN(1, tb + SLB, TD, TDB, 16, S.MN(WH2, WH2B, 64), ID_KM(64));
                umma::commit_elect(mbar);
                PWAIT(umma::mbar_wait(mb_a, ph_a));
                WG_ACT_A<8>(tb + TB_DH2, S.MN(TA1, T64B, 64), S.MN(TD, TDB, 16), ID_WG(16), acc);
            }
            ph_a ^= 1u;
        }
        // While U = DLY H2 runs: mvec = [J q (features), q, 0] (field.py:326-327) -> MV (TZ)
        // and the ReLU mask M1 -> TY (exact in fp16: hi part only), both for B4's
        // G = M1^T MV.  TZ / TY are free (A1c / U2 were last read by B1's GEMMs).
        // Quarter k stages block k (levels 4k..4k+3) and block k+4 (block 4 holds q).
        auto mv_stage = [&](int emv) -> float {
            float mv[2][8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                mv[0][k] = 0.f;
                mv[1][k] = 0.f;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int l = 4 * qt + i;
                float jl[8];
                umma::tmem_ld8(my + TB_J + 8 * l, jl);
                if (l < NA) {
                    mv[0][2 * i] = jl[0] * q0 + jl[1] * q1 + jl[2] * q2;
                    mv[0][2 * i + 1] = jl[3] * q0 + jl[4] * q1 + jl[5] * q2;
                }
            }
            if (qt == 0) {
                mv[1][0] = q0;
                mv[1][1] = q1;
                mv[1][2] = q2;
            }
            float mm = 0.f;
#pragma unroll
            for (int k = 0; k < 8; ++k) mm = fmaxf(mm, fmaxf(fabsf(mv[0][k]), fabsf(mv[1][k])));
            const float sm = pow2i(emv);
            STG_W(48, TZ, T64B, qt, mv[0], sm);
            if (qt < 2) STG_W(48, TZ, T64B, qt + 4, mv[1], sm);
            return mm;
        };
        int eMV = PS.guess(kMv);
        PS.contrib(kMv, mv_stage(eMV));
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const uint32_t bits = (m1 >> (8 * i)) & 0xFFu;
            auto h2 = [&](int k) {
                return ((bits >> k) & 1u ? 0x3C00u : 0u) | ((bits >> (k + 1)) & 1u ? 0x3C000000u : 0u);
            };
            *reinterpret_cast<uint4 *>(S.p(TY) + umma::tile_off(r, 8 * (i ? b1 : b0), 64)) =
                make_uint4(h2(0), h2(2), h2(4), h2(6));
        }
        wait_mma(mbar, phase);
        PMARK(12);
        // ------------------------------------------------ B4: u -> DE, dH1, G
        // TC is free (dC1 of B2 completed before B3's chain GEMM): next tile's CIN
        if (t == kDmaThread && has_next) dma(TC, fwt(ntile) + FW_CIN, TCB, mb_c);
        int eU;
        {
            float u[2][8], mu = 0.f;
            const float sc4 = pow2i(-(eDLY + eH2));
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                umma::tmem_ld8(my + SLB + 8 * (i ? b1 : b0), u[i]);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    u[i][k] = ((m1 >> (8 * i + k)) & 1u) ? u[i][k] * sc4 : 0.f;
                    mu = fmaxf(mu, fabsf(u[i][k]));
                }
            }
            eU = PS.guess(kU);
            PS.contrib(kU, mu);
            auto stg = [&](int eu) {
                const float su = pow2i(eu);
#pragma unroll
                for (int i = 0; i < 2; ++i) STG_A(64, TX, T64B, i ? b1 : b0, u[i], su);
            };
            stg(eU);
            PUB_A();
            PMARK(13);
            const bool oku = PS.check(kU, eU);
            const bool okm = PS.check(kMv, eMV);
            if (!(oku && okm)) {  // (uniform) restage whichever missed its exponent window
                if (!oku) stg(eU);
                if (!okm) mv_stage(eMV);
                PUB_A();
                PMARK(14);
            }
        }
        {
            // Theorem 1 through one accumulator: with G = M1^T MV (64 x 48),
            //   dH1 += diag(H2[0]) G   and   dH2[0][j] += sum_c H1[j][c] G[j][c]
            // (both applied when G is folded), so pvec = m1 . (H1 mvec) never materialises.
            const bool acca = acc_begin(aH1a, eU + eE);
            const bool accb = acc_begin(aH1b, eMV);
            if (warp == kMmaWarp) {  // converged MMA warp; elect.sync picks the issuing lane
                CHAIN(4, tb + TB_SA, TX, T64B, 64, S.MN(WH1, WH1B, 48), ID_KM(48));
                umma::commit_elect(mbar);
                PWAIT(umma::mbar_wait(mb_e, ph_e));
                WG_ACT_B<8>(tb + TB_DH1A, S.MN(TX, T64B, 64), S.MN(TE, TEB, 48), ID_WG(48), acca);
                WG_MASK<8>(tb + TB_DH1B, S.MN(TY, T64B, 64), S.MN(TZ, T64B, 48), ID_WG(48), accb);
                umma::commit_elect(mbarw);
            }
            ph_e ^= 1u;
        }
        if (has_next) j_load(ntile);  // registers only (TMEM J is rewritten in B5): hides under B4's GEMM
        wait_mma(mbar, phase);
        PMARK(15);
        // ------------------------------------------------ B5: scatter inputs; next tile's DMAs
        // TA1 is free (dH2 of B3 completed before B4's chain GEMM): next tile's A1
        if (t == kDmaThread && has_next) dma(TA1, fwt(ntile) + FW_A1, T64B, mb_a);
        {
            // dL/dfeature pairs (DE) and q for the scatter kernel
            const float sde = pow2i(-(eU + eH1));
            float de[8];
            umma::tmem_ld8(my + TB_SA + 8 * qt, de);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (8 * qt + k < 2 * NA) __stcs(SBt + (8 * qt + k) * TILE + r, de[k] * sde);
            if (qt == 0) {
                __stcs(SBt + 64 * TILE + r, q0);
                __stcs(SBt + 65 * TILE + r, q1);
                __stcs(SBt + 66 * TILE + r, q2);
            }
            if (want_xin && qt == 3) {  // de_aug's position rows (E columns 32..34)
                float dx[8];
                umma::tmem_ld8(my + TB_SA + 32, dx);
                if (valid) {
                    float *xi = ws.xin + tile * XINROWS * TILE + r;
                    xi[6 * TILE] = dx[0] * sde;
                    xi[7 * TILE] = dx[1] * sde;
                    xi[8 * TILE] = dx[2] * sde;
                }
            }
            wait_mma(mbarw, phasew);  // B4's weight-gradient GEMMs: TX, TY, TZ, TE free
            PMARK(16);
            if (t == kDmaThread && has_next) {
                dma(TE, ws.e_tiles + ntile * 2 * TEB, TEB, mb_e);
                dma(TZ, fwt(ntile) + FW_A1C, T64B, mb_z);
            }
            if (has_next) j_store();
            if (has_next) in_nx = read_in(ntile, fe_nx);  // TIN landed during B1
            PMARK(17);
        }
        // Tile boundary barrier: without it a warp can run into the next tile while another
        // is still in B5; observed to deadlock on the c1 field (mbarw never completing),
        // so warps leave the tile together.
        publish();
        PMARK(18);
        if (++ntiles_done == kFoldTiles) {  // bound the TMEM accumulation run (all MMAs done)
            ntiles_done = 0;
#pragma unroll  // compile-time j: acc_e / acc_live stay in registers
            for (int j = 0; j < NACC; ++j)
                if (acc_live[j]) fold(j);
            block_sync_tc();
        }
    }
    if (warp == 0) umma::commit_elect(mbarw);
    wait_mma(mbarw, phasew);
#pragma unroll
    for (int j = 0; j < NACC; ++j)
        if (acc_live[j]) fold(j);
#ifdef NS2B_PHASE_PROF
    __syncthreads();
    if (blockIdx.x == 0 && t == 0) {
        printf("PHASEPROF bwd");
        for (int i = 0; i < 64; ++i)
            if (pacc[i]) printf(" %d:%lld", i, pacc[i]);
        printf("\n");
    }
#endif
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc(tb, 512);
}
#undef STG_A
#undef PUB_A
#undef CHAIN
#undef STG_W

// ---------------------------------------------------------------------------
// MLP backward, pipelined across two thread groups (field_bwd2_kernel, the default; NS2B_BWD=1
// selects field_bwd_kernel above).  The backward of a tile is a strict chain of five
// MMA round trips, so one tile in flight leaves the SM idle while each phase waits on its
// GEMM.  Here the colour-net half of the chain (group C, warps 0-7) runs one tile ahead of
// the SDF-net half (group S, warps 8-15):
//   C0 dlog -> U2 = DLOG C3,      dC3 += A2c^T DLOG
//   C1 u2   -> U1 = U2 C2,        dC2 += U2^T A1c
//   C2 u1   -> DCIN = U1 C1,      dC1 += U1^T CIN
//   C3 q, dly (and the m1 mask words) -> a two-slot handoff ring in shared memory
//   S0 dly  -> U = DLY H2,        dH2 += A1^T DLY;   MV = [J q, q] and M1 staged
//   S1 u    -> DE = U H1,         dH1 += U^T E,  G += M1^T MV   (Theorem 1, as field_bwd_kernel)
//   S2 DE, q -> the scatter's inputs
// so while one group waits on its GEMM the other runs its epilogue.  Each group has its
// own named barrier (256 threads), MMA-issuing warp, DMA thread, mbarriers, staging-exponent
// predictions and weight-gradient accumulators; a thread owns 32 columns of its row (half
// qh = blocks 4qh..4qh+3 of a 64-wide tile).  Chain GEMMs read A from tensor memory (each
// group has its own A region), weight-gradient GEMMs take fp16 x fp16 operands (NS2B_WG1).
// J is read from L2 by group S (prefetched a tile ahead), not kept in TMEM.
// Shared memory: weights 44 KB | C: DLOG 4 | A2c 16 | A1c 16 | U2/U1 16 | CIN 8 | inputs 2 x 9.2 |
// S: DLY 4 | A1 16 | U 16 | M1 16 | MV 12 | E 12 | handoff 2 x 10.75  (~220 KB).
// TMEM: C dC2 64 | dC1 32 | dC3 16 | slot 64 | A 64;  S dH2 16 | dH1a 48 | G 48 | slot 64 | A 64.
namespace b2 {
constexpr uint32_t TDC = TE;                    // DLOG hi   128 x 16
constexpr uint32_t TWC = TDC + TDB;             // A2c hi    128 x 64
constexpr uint32_t TZC = TWC + T64B;            // A1c hi
constexpr uint32_t TYC = TZC + T64B;            // U2 hi -> U1 hi
constexpr uint32_t TCC = TYC + T64B;            // CIN hi    128 x 32
constexpr uint32_t IN_MK = 0, IN_NC = IN_MK + 6 * TILE * 4, IN_DC = IN_NC + NCROWS * TILE * 4,
                   IN_DS = IN_DC + 3 * TILE * 4, IN_EX = IN_DS + TILE * 4, IN_BYTES = IN_EX + 16;
constexpr uint32_t IN_STRIDE = (IN_BYTES + 127) / 128 * 128;
constexpr uint32_t TIN0 = TCC + TCB;            // per-tile inputs, two slots
constexpr uint32_t TDS = TIN0 + 2 * IN_STRIDE;  // DLY hi    128 x 16
constexpr uint32_t TA1S = TDS + TDB;            // A1 hi
constexpr uint32_t TXS = TA1S + T64B;           // U hi
constexpr uint32_t TYS = TXS + T64B;            // M1
constexpr uint32_t TMV = TYS + T64B;            // MV hi     128 x 48
constexpr uint32_t TES = TMV + TEB;             // E hi      128 x 48
constexpr uint32_t H_Q = 0, H_DLY = H_Q + 3 * TILE * 4, H_M1 = H_DLY + 16 * TILE * 4, H_BYTES = H_M1 + 2 * TILE * 4;
constexpr uint32_t TH0 = TES + TEB;             // handoff ring, two slots
constexpr uint32_t SMEM = TH0 + 2 * H_BYTES;
static_assert(SMEM <= 220 * 1024, "bwd2 shared memory");
// TMEM columns
constexpr uint32_t C_DC2 = 0, C_DC1 = 64, C_DC3 = 96, C_SL = 112, C_AH = 176, C_AL = 208;
constexpr uint32_t S_DH2 = 240, S_DH1A = 256, S_G = 304, S_SL = 352, S_AH = 416, S_AL = 448;
}  // namespace b2

// Fold one weight-gradient accumulator (scaled by 2^-e) into global memory: the 8 warps of
// a group (lane quadrant qd, half qh) read lanes 0-15 of their quadrant (M = 64 rows).
__device__ __noinline__ void fold_acc2(int j, int e, uint32_t my, int qh, int E, const float *__restrict__ h2row0,
                                       const float *__restrict__ sdf_w, float *__restrict__ g_sdf,
                                       float *__restrict__ g_color) {
    using namespace b2;
    const int lane = threadIdx.x & 31, qd = (threadIdx.x >> 5) & 3;
    const int jrow = 16 * qd + lane;
    const float sc = pow2i(-e);
    float d[8];
    switch (j) {
    case aC3:  // dC3^T: row = hidden unit, col = output (3)
        umma::tmem_ld8(my + C_DC3, d);
        if (lane < 16 && qh == 0)
            for (int o = 0; o < 3; ++o) atomicAdd(g_color + H * CIN + H * H + o * H + jrow, d[o] * sc);
        break;
    case aC2:
        for (int b = qh; b < 8; b += 2) {
            umma::tmem_ld8(my + C_DC2 + 8 * b, d);
            if (lane < 16)
#pragma unroll
                for (int k = 0; k < 8; ++k) atomicAdd(g_color + H * CIN + jrow * H + 8 * b + k, d[k] * sc);
        }
        break;
    case aC1:
        for (int b = qh; b < 4; b += 2) {
            umma::tmem_ld8(my + C_DC1 + 8 * b, d);
            if (lane < 16)
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if (8 * b + k < CIN) atomicAdd(g_color + jrow * CIN + 8 * b + k, d[k] * sc);
        }
        break;
    case aH2:  // dH2^T: row = hidden unit, col = output unit
        umma::tmem_ld8(my + S_DH2 + 8 * qh, d);
        if (lane < 16)
#pragma unroll
            for (int k = 0; k < 8; ++k) atomicAdd(g_sdf + H * (E + 1) + (8 * qh + k) * H + jrow, d[k] * sc);
        break;
    case aH1a:
        for (int b = qh; b < 6; b += 2) {
            umma::tmem_ld8(my + S_DH1A + 8 * b, d);
            if (lane < 16)
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int rc = h1_col(8 * b + k, E);
                    if (rc >= 0) atomicAdd(g_sdf + jrow * (E + 1) + rc, d[k] * sc);
                }
        }
        break;
    default: {  // G = M1^T MV: dH1 += H2[0][j] G[j],  dH2[0][j] += H1[j] . G[j]
        float dot = 0.f;
        const float h2j = lane < 16 ? h2row0[jrow] : 0.f;
        for (int b = qh; b < 6; b += 2) {
            umma::tmem_ld8(my + S_G + 8 * b, d);
            if (lane < 16)
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int rc = h1_col(8 * b + k, E);
                    if (rc >= 0) {
                        atomicAdd(g_sdf + jrow * (E + 1) + rc, h2j * d[k] * sc);
                        dot = fmaf(sdf_w[jrow * (E + 1) + rc], d[k], dot);
                    }
                }
        }
        if (lane < 16 && dot != 0.f) atomicAdd(g_sdf + H * (E + 1) + jrow, dot * sc);
        break;
    }
    }
}

__global__ void __launch_bounds__(MLP_THREADS, 1)
field_bwd2_kernel(FieldDev f, const int32_t *__restrict__ count, const float *__restrict__ dl_dc,
                  const float *__restrict__ dl_dsdf, const float *__restrict__ dl_dn_extra, float eik_w,
                  const int64_t *__restrict__ eik_count, float *__restrict__ g_sdf, float *__restrict__ g_color,
                  Workspace ws) {
    using namespace b2;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // C: [0] chain, [1] dC2 done, [2] dC1 done, [3] A2c, [4] A1c, [5] CIN, [6..7] inputs;
    // S: [8] chain, [9] WG, [10] A1, [11] E;  handoff: [12..13] full, [14..15] empty
    __shared__ uint64_t bars[16];
    __shared__ uint32_t wmax[6];
    __shared__ int wexp[6];
    __shared__ float h2row0[H];
    __shared__ uint32_t tmem_base_sh;
    __shared__ uint32_t gmx[2][2][NSLOT];
    __shared__ int gpred[2][NSLOT];
    __shared__ uint4 m1lut[256];
    mask_lut_init(m1lut);
    const Smem S{smem_raw};
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int g = warp >> 3, gw = warp & 7, tg = t & 255;
#ifdef NS2B_PHASE_PROF  // cycles group C waits for a free handoff slot [0], S for a full one [1], loop totals [2, 3]
    __shared__ long long bpw[4];
    if (t < 4) bpw[t] = 0;
#define BPW(i, stmt)                                      \
    do {                                                  \
        const long long w0_ = clock64();                  \
        stmt;                                             \
        if (tg == 0) bpw[i] += clock64() - w0_;           \
    } while (0)
#else
#define BPW(i, stmt) stmt
#endif
    const int qd = gw & 3, qh = gw >> 2;
    const int r = 32 * qd + lane;
    const int E = 3 + 2 * f.L;
    const int NA = f.n_active;
    // ---- setup (all 512 threads)
    if (t < H) h2row0[t] = f.sdf_w[H * (E + 1) + t];
    load_weight_tiles<false>(S, f, wmax, wexp);
    if (t < 2 * NSLOT) {
        gmx[t / NSLOT][0][t % NSLOT] = 0u;
        gmx[t / NSLOT][1][t % NSLOT] = 0u;
        gpred[t / NSLOT][t % NSLOT] = 0;
    }
    if (t == 0) {
        for (int i = 0; i < 12; ++i) umma::mbar_init(bars + i, 1);
        for (int i = 12; i < 16; ++i) umma::mbar_init(bars + i, 256);
        umma::fence_barrier_init();
    }
    if (warp == 0) umma::tmem_alloc(&tmem_base_sh, 512);
    publish();
    const int eH1 = wexp[0], eH2 = wexp[1], eC1 = wexp[2], eC2 = wexp[3], eC3 = wexp[4];
    const uint32_t tb = tmem_base_sh;
    const uint32_t my = tb + (static_cast<uint32_t>(qd * 32) << 16);
    PredScaleG PS{gmx[g], gpred[g], 1, tg == 0};
    const int P = *count;
    const float Pf = eik_count ? static_cast<float>(*eik_count) : 1.f;
    const bool gn_fused = ws.flags[0] != 0;
    const bool mma_w = gw == 7;                 // the group's MMA-issuing warp
    const bool dma_t = gw == 6 && lane == 0;    // the group's DMA thread
    const int64_t G = gridDim.x;
    auto fwt = [&](int64_t tl) { return ws.fw_tiles + tl * static_cast<int64_t>(FWB); };
    auto dma = [&](uint32_t soff, const uint8_t *gp, uint32_t bytes, uint64_t *mb) {
        umma::bulk_g2s<true>(S.p(soff), gp, bytes, mb);
    };
    int acc_e[3];
    bool acc_live[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        acc_e[j] = 0;
        acc_live[j] = false;
    }
    const int acc0 = g == 0 ? aC3 : aH2;  // this group's accumulators: acc0 .. acc0 + 2
    auto fold = [&](int jj) {
        fold_acc2(acc0 + jj, acc_e[jj], my, qh, E, h2row0, f.sdf_w, g_sdf, g_color);
        acc_live[jj] = false;
    };
    auto acc_begin = [&](int jj, int e) -> bool {  // group-uniform
        if (acc_live[jj] && acc_e[jj] != e) {
            fold(jj);
            umma::fence_before_sync();
            group_sync(g);
            umma::fence_after_sync();
        }
        const bool accumulate = acc_live[jj];
        acc_e[jj] = e;
        acc_live[jj] = true;
        return accumulate;
    };
    if (g == 0) {
        // =============================================== group C: colour-net backward
        uint64_t *mbar = bars, *mbar2 = bars + 1, *mbar3 = bars + 2, *mb_w = bars + 3, *mb_z = bars + 4,
                 *mb_c = bars + 5, *mb_in = bars + 6, *hfull = bars + 12, *hempty = bars + 14;
        uint32_t ph = 0, ph2 = 0, ph3 = 0, ph_w = 0, ph_z = 0, ph_c = 0, ph_in[2] = {0, 0}, ph_he[2] = {0, 0};
        const bool in_dma_ok =
            ((reinterpret_cast<uintptr_t>(dl_dc) | reinterpret_cast<uintptr_t>(dl_dsdf)) & 15u) == 0;
        auto in_full = [&](int64_t tl) { return in_dma_ok && (tl + 1) * TILE <= P; };
        auto in_dma = [&](int64_t tl, int s) {  // one thread
            const uint32_t base = TIN0 + s * IN_STRIDE;
            umma::mbar_expect_tx(mb_in + s, IN_BYTES);
            umma::bulk_g2s_tx(S.p(base + IN_MK), ws.fw_mask + tl * 6 * TILE, 6 * TILE * 4, mb_in + s);
            umma::bulk_g2s_tx(S.p(base + IN_NC), ws.fw_nc + tl * NCROWS * TILE, NCROWS * TILE * 4, mb_in + s);
            umma::bulk_g2s_tx(S.p(base + IN_DC), dl_dc + 3 * tl * TILE, 3 * TILE * 4, mb_in + s);
            umma::bulk_g2s_tx(S.p(base + IN_DS), dl_dsdf + tl * TILE, TILE * 4, mb_in + s);
            umma::bulk_g2s_tx(S.p(base + IN_EX), ws.fw_exp + tl, 16, mb_in + s);
        };
        const int64_t t0 = blockIdx.x;
        if (dma_t && t0 * TILE < P) {
            dma(TWC, fwt(t0) + FW_A2C, T64B, mb_w);
            dma(TZC, fwt(t0) + FW_A1C, T64B, mb_z);
            dma(TCC, fwt(t0) + FW_CIN, TCB, mb_c);
            if (in_full(t0)) in_dma(t0, 0);
        }
        int it = 0;
        for (int64_t tile = t0; tile * TILE < P; tile += G, ++it) {
            const int64_t p = tile * TILE + r;
            const bool valid = p < P;
            const int64_t ntile = tile + G;
            const bool has_next = ntile * TILE < P;
            const int s = it & 1;
            PS.par ^= 1;
            if (dma_t && has_next) {
                umma::prefetch_l2(fwt(ntile), FWB);
                if (in_full(ntile)) in_dma(ntile, s ^ 1);  // slot s^1 was read during the previous tile
            }
            // ---- per-sample inputs: masks (byte qh of each quarter word = blocks 4qh..4qh+3), dL/dc,
            // c, dL/dsdf, normal / Eikonal cotangent, the forward's exponents
            uint32_t m1 = 0u, mc1 = 0u, mc2 = 0u;
            float gc0 = 0.f, gc1 = 0.f, gc2 = 0.f, cc0 = 0.f, cc1 = 0.f, cc2 = 0.f, gd = 0.f, n0 = 0.f, n1 = 0.f,
                  n2 = 0.f;
            int4 fe;
            if (in_full(tile)) {
                umma::mbar_wait(mb_in + s, ph_in[s]);
                ph_in[s] ^= 1u;
                const uint8_t *base = S.p(TIN0 + s * IN_STRIDE);
                const uint32_t *mw = reinterpret_cast<const uint32_t *>(base + IN_MK) + qh * TILE + r;
                m1 = mw[0];  // this half's 32 hidden-unit bits of each mask
                mc1 = mw[2 * TILE];
                mc2 = mw[4 * TILE];
                const float *nc = reinterpret_cast<const float *>(base + IN_NC) + r;
                const float *dc = reinterpret_cast<const float *>(base + IN_DC) + 3 * r;
                gc0 = dc[0];
                gc1 = dc[1];
                gc2 = dc[2];
                cc0 = nc[3 * TILE];
                cc1 = nc[4 * TILE];
                cc2 = nc[5 * TILE];
                gd = reinterpret_cast<const float *>(base + IN_DS)[r];
                n0 = nc[0];
                n1 = nc[TILE];
                n2 = nc[2 * TILE];
                fe = *reinterpret_cast<const int4 *>(base + IN_EX);
            } else {
                m1 = ws.fw_mask[mask_idx(tile, 0, qh, r)];
                mc1 = ws.fw_mask[mask_idx(tile, 1, qh, r)];
                mc2 = ws.fw_mask[mask_idx(tile, 2, qh, r)];
                fe = ws.fw_exp[tile];
                if (valid) {
                    const float *nc = ws.fw_nc + tile * NCROWS * TILE + r;
                    gc0 = dl_dc[3 * p];
                    gc1 = dl_dc[3 * p + 1];
                    gc2 = dl_dc[3 * p + 2];
                    cc0 = nc[3 * TILE];
                    cc1 = nc[4 * TILE];
                    cc2 = nc[5 * TILE];
                    gd = dl_dsdf[p];
                    n0 = nc[0];
                    n1 = nc[TILE];
                    n2 = nc[2 * TILE];
                }
            }
            const int eA1c = fe.z, eA2c = fe.w, eCin = fe.y;
            float gn0 = 0.f, gn1 = 0.f, gn2 = 0.f;
            if (valid) {
                if (dl_dn_extra) {
                    gn0 = dl_dn_extra[3 * p];
                    gn1 = dl_dn_extra[3 * p + 1];
                    gn2 = dl_dn_extra[3 * p + 2];
                }
                if (gn_fused) {  // fused by the forward (same arithmetic)
                    gn0 += n0;
                    gn1 += n1;
                    gn2 += n2;
                } else if (eik_w != 0.f) {  // trainer.py:229-235 (fp32, numpy's order)
                    const float nn = sqrtf(n0 * n0 + n1 * n1 + n2 * n2);
                    const float coef = eik_w * (2.f * (nn - 1.f) / fmaxf(nn, 1e-12f));
                    gn0 += coef * n0 / Pf;
                    gn1 += coef * n1 / Pf;
                    gn2 += coef * n2 / Pf;
                }
            }
            // ------------------------------------------- C0: dlog -> U2, dC3
            int eD;
            {
                float dlog[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) dlog[k] = 0.f;
                if (qh == 0) {  // field.py:304
                    dlog[0] = gc0 * cc0 * (1.f - cc0);
                    dlog[1] = gc1 * cc1 * (1.f - cc1);
                    dlog[2] = gc2 * cc2 * (1.f - cc2);
                }
                eD = PS.guess(kDlog);
                PS.contrib(kDlog, fmaxf(fabsf(dlog[0]), fmaxf(fabsf(dlog[1]), fabsf(dlog[2]))));
#pragma unroll 1
                for (int pass = 0;; ++pass) {
                    stage_blk_ta<16>(S, TDC, r, qh, dlog, pow2i(eD), my + C_AH, my + C_AL);
                    umma::tmem_st_wait();
                    group_publish(0);
                    if (pass) break;
                    if (tg < NSLOT) gmx[0][PS.par ^ 1][tg] = 0u;
                    if (PS.check(kDlog, eD)) break;
                }
            }
            {
                const bool acc = acc_begin(0, eA2c + eD);
                if (mma_w) {
                    umma::gemm3t<1>(tb + C_SL, tb + C_AH, tb + C_AL, S.MN(WC3, WC3B, 64), ID_KM(64), false);
                    umma::commit_elect(mbar);
                    umma::mbar_wait(mb_w, ph_w);
                    umma::gemm1<8>(tb + C_DC3, S.MN(TWC, T64B, 64), S.MN(TDC, TDB, 16), ID_WG(16), acc);
                }
                ph_w ^= 1u;
            }
            wait_mma(mbar, ph);
            // ------------------------------------------- C1: u2 -> U1, dC2
            // the previous tile's dC1 ran before this tile's U2 GEMM in the MMA pipe: TC takes
            // this tile's CIN (needed by C2's dC1), with no wait on the issuing thread
            if (dma_t && it > 0) dma(TCC, fwt(tile) + FW_CIN, TCB, mb_c);
            int eU2;
            {
                // raw accumulator values: the result scale 2^-(eD + eC3) is folded into the
                // staging scale (one multiply per element; powers of two, exact)
                float u[4][8], m = 0.f;
                const int esc = -(eD + eC3);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    umma::tmem_ld8(my + C_SL + 8 * (4 * qh + i), u[i]);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        u[i][k] = ((mc2 >> (8 * i + k)) & 1u) ? u[i][k] : 0.f;
                        m = fmaxf(m, fabsf(u[i][k]));
                    }
                }
                eU2 = PS.guess(kU2);
                PS.contrib(kU2, m * pow2i(esc));
#pragma unroll 1
                for (int pass = 0;; ++pass) {
                    const float s2 = pow2i(eU2 + esc);
#pragma unroll
                    for (int i = 0; i < 4; ++i) stage_blk_ta<64>(S, TYC, r, 4 * qh + i, u[i], s2, my + C_AH, my + C_AL);
                    umma::tmem_st_wait();
                    group_publish(0);
                    if (pass) break;
                    if (PS.check(kU2, eU2)) break;
                }
            }
            {
                const bool acc = acc_begin(1, eU2 + eA1c);
                if (mma_w) {
                    umma::gemm3t<4>(tb + C_SL, tb + C_AH, tb + C_AL, S.MN(WC2, WC2B, 64), ID_KM(64), false);
                    umma::commit_elect(mbar);
                    umma::mbar_wait(mb_z, ph_z);
                    umma::gemm1<8>(tb + C_DC2, S.MN(TYC, T64B, 64), S.MN(TZC, T64B, 64), ID_WG(64), acc);
                    umma::commit_elect(mbar2);  // dC2 has read U2 (TY) and A1c (TZ)
                }
                ph_z ^= 1u;
            }
            wait_mma(mbar, ph);
            // ------------------------------------------- C2: u1 -> DCIN, dC1
            int eU1;
            {
                float u[4][8], m = 0.f;
                const int esc = -(eU2 + eC2);  // folded into the staging scale (see C1)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    umma::tmem_ld8(my + C_SL + 8 * (4 * qh + i), u[i]);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        u[i][k] = ((mc1 >> (8 * i + k)) & 1u) ? u[i][k] : 0.f;
                        m = fmaxf(m, fabsf(u[i][k]));
                    }
                }
                eU1 = PS.guess(kU1);
                PS.contrib(kU1, m * pow2i(esc));
                wait_mma(mbar2, ph2);  // U1 restages TY
                if (dma_t && has_next) {  // dC3 (before U1's GEMM) and dC2 are done: next A2c, A1c
                    dma(TWC, fwt(ntile) + FW_A2C, T64B, mb_w);
                    dma(TZC, fwt(ntile) + FW_A1C, T64B, mb_z);
                }
#pragma unroll 1
                for (int pass = 0;; ++pass) {
                    const float s1 = pow2i(eU1 + esc);
#pragma unroll
                    for (int i = 0; i < 4; ++i) stage_blk_ta<64>(S, TYC, r, 4 * qh + i, u[i], s1, my + C_AH, my + C_AL);
                    umma::tmem_st_wait();
                    group_publish(0);
                    if (pass) break;
                    if (PS.check(kU1, eU1)) break;
                }
            }
            {
                const bool acc = acc_begin(2, eU1 + eCin);
                if (mma_w) {
                    umma::gemm3t<4>(tb + C_SL, tb + C_AH, tb + C_AL, S.MN(WC1, WC1B, 32), ID_KM(32), false);
                    umma::commit_elect(mbar);
                    umma::mbar_wait(mb_c, ph_c);
                    umma::gemm1<8>(tb + C_DC1, S.MN(TYC, T64B, 64), S.MN(TCC, TCB, 32), ID_WG(32), acc);
                    umma::commit_elect(mbar3);  // dC1 has read U1 (TY) and CIN (TC)
                }
                ph_c ^= 1u;
            }
            wait_mma(mbar, ph);
            // ------------------------------------------- C3: q, dly, m1 -> the handoff ring
            {
                const float sc3 = pow2i(-(eU1 + eC1));
                float c0[8], c1[8];
                umma::tmem_ld8(my + C_SL + 16 * qh, c0);
                umma::tmem_ld8(my + C_SL + 16 * qh + 8, c1);
                const int hs = it & 1;
                if (it >= 2) {  // group S has read this slot (tile it - 2)
                    BPW(0, umma::mbar_wait(hempty + hs, ph_he[hs]));
                    ph_he[hs] ^= 1u;
                }
                float *hq = reinterpret_cast<float *>(S.p(TH0 + hs * H_BYTES + H_Q)) + r;
                float *hd = reinterpret_cast<float *>(S.p(TH0 + hs * H_BYTES + H_DLY)) + r;
                uint32_t *hm = reinterpret_cast<uint32_t *>(S.p(TH0 + hs * H_BYTES + H_M1)) + r;
                if (qh == 0) {  // field.py:308-312: q = dL/dn, dly = [dd + dcin[9], dcin[10..24]]
                    hq[0] = gn0 + c0[3] * sc3;
                    hq[TILE] = gn1 + c0[4] * sc3;
                    hq[2 * TILE] = gn2 + c0[5] * sc3;
                    hd[0] = gd + c1[1] * sc3;
#pragma unroll
                    for (int k = 1; k < 7; ++k) hd[k * TILE] = c1[1 + k] * sc3;
                } else {
#pragma unroll
                    for (int k = 0; k < 8; ++k) hd[(7 + k) * TILE] = c0[k] * sc3;
                    hd[15 * TILE] = c1[0] * sc3;
                }
                hm[qh * TILE] = m1;
                umma::mbar_arrive(hfull + hs);
            }
            ph3 ^= 1u;
        }
        // all of group C's MMAs have completed once the last tile's dC1 has
        if (it > 0) {
            ph3 ^= 1u;  // the last tile's dC1 phase
            wait_mma(mbar3, ph3);
        }
#pragma unroll
        for (int jj = 0; jj < 3; ++jj)
            if (acc_live[jj]) fold(jj);
    } else {
        // =============================================== group S: SDF-net backward
        uint64_t *mbar = bars + 8, *mbarw = bars + 9, *mb_a = bars + 10, *mb_e = bars + 11, *hfull = bars + 12,
                 *hempty = bars + 14;
        uint32_t ph = 0, phw = 0, ph_a = 0, ph_e = 0, ph_hf[2] = {0, 0};
        const int64_t t0 = blockIdx.x;
        if (dma_t && t0 * TILE < P) {
            dma(TA1S, fwt(t0) + FW_A1, T64B, mb_a);
            dma(TES, ws.e_tiles + t0 * 2 * TEB, TEB, mb_e);
        }
        bool wpend = false;
        int it = 0;
        for (int64_t tile = t0; tile * TILE < P; tile += G, ++it) {
            const int64_t ntile = tile + G;
            const bool has_next = ntile * TILE < P;
            PS.par ^= 1;
            float *SBt = ws.sb + tile * SBROWS * TILE;
            if (dma_t && has_next) {
                umma::prefetch_l2(fwt(ntile) + FW_A1, T64B);
                umma::prefetch_l2(ws.jac + ntile * JROWS * TILE, JROWS * TILE * 4);
                umma::prefetch_l2(ws.e_tiles + ntile * 2 * TEB, TEB);
            }
            const int eE = ws.e_exp[tile];
            const int eA1 = ws.fw_exp[tile].x;
            // d feature/dx of this thread's 8 levels (L2; the handoff wait hides their latency)
            const float *jt = ws.jac + tile * JROWS * TILE + r;
            float jv[8][6];
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int k = 0; k < 6; ++k) jv[i][k] = 8 * qh + i < NA ? __ldcs(jt + (6 * (8 * qh + i) + k) * TILE) : 0.f;
            // ------------------------------------------- S0: dly -> U, dH2; MV, M1
            const int hs = it & 1;
            BPW(1, umma::mbar_wait(hfull + hs, ph_hf[hs]));
            ph_hf[hs] ^= 1u;
            float q0, q1, q2, dly[8];
            uint32_t m1;
            {
                const float *hq = reinterpret_cast<const float *>(S.p(TH0 + hs * H_BYTES + H_Q)) + r;
                const float *hd = reinterpret_cast<const float *>(S.p(TH0 + hs * H_BYTES + H_DLY)) + r;
                q0 = hq[0];
                q1 = hq[TILE];
                q2 = hq[2 * TILE];
#pragma unroll
                for (int k = 0; k < 8; ++k) dly[k] = hd[(8 * qh + k) * TILE];
                m1 = reinterpret_cast<const uint32_t *>(S.p(TH0 + hs * H_BYTES + H_M1))[qh * TILE + r];
            }
            umma::mbar_arrive(hempty + hs);
            if (wpend) {  // the previous tile's dH1 / G GEMMs read U (TX), M1 (TY), MV, E
                wait_mma(mbarw, phw);
                wpend = false;
                if (dma_t) dma(TES, ws.e_tiles + tile * 2 * TEB, TEB, mb_e);
            }
            int eDLY, eMV;
            {
                float md = 0.f;
#pragma unroll
                for (int k = 0; k < 8; ++k) md = fmaxf(md, fabsf(dly[k]));
                eDLY = PS.guess(kDly);
                PS.contrib(kDly, md);
                // mvec = [J q (features), q, 0] (field.py:326-327): half qh holds levels 8qh..8qh+7
                // (blocks 2qh, 2qh+1) and block 4 + qh (q / zeros)
                float mv[3][8], mm = 0.f;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    mv[i >> 2][2 * (i & 3)] = jv[i][0] * q0 + jv[i][1] * q1 + jv[i][2] * q2;
                    mv[i >> 2][2 * (i & 3) + 1] = jv[i][3] * q0 + jv[i][4] * q1 + jv[i][5] * q2;
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) mv[2][k] = 0.f;
                if (qh == 0) {
                    mv[2][0] = q0;
                    mv[2][1] = q1;
                    mv[2][2] = q2;
                }
#pragma unroll
                for (int b = 0; b < 3; ++b)
#pragma unroll
                    for (int k = 0; k < 8; ++k) mm = fmaxf(mm, fabsf(mv[b][k]));
                eMV = PS.guess(kMv);
                PS.contrib(kMv, mm);
                // M1 (exact in fp16: hi part only) -> TY
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    *reinterpret_cast<uint4 *>(S.p(TYS) + umma::tile_off(r, 8 * (4 * qh + i), 64)) =
                        m1lut[(m1 >> (8 * i)) & 0xFFu];
#pragma unroll 1
                for (int pass = 0;; ++pass) {
                    stage_blk_ta<16>(S, TDS, r, qh, dly, pow2i(eDLY), my + S_AH, my + S_AL);
                    const float sm = pow2i(eMV);
                    stage_blk_hi<48>(S, TMV, r, 2 * qh, mv[0], sm);
                    stage_blk_hi<48>(S, TMV, r, 2 * qh + 1, mv[1], sm);
                    stage_blk_hi<48>(S, TMV, r, 4 + qh, mv[2], sm);
                    umma::tmem_st_wait();
                    group_publish(1);
                    if (pass) break;
                    if (tg < NSLOT) gmx[1][PS.par ^ 1][tg] = 0u;
                    const bool okd = PS.check(kDly, eDLY);
                    const bool okm = PS.check(kMv, eMV);
                    if (okd && okm) break;
                }
            }
            {
                const bool acc = acc_begin(0, eA1 + eDLY);
                if (mma_w) {
                    umma::gemm3t<1>(tb + S_SL, tb + S_AH, tb + S_AL, S.MN(WH2, WH2B, 64), ID_KM(64), false);
                    umma::commit_elect(mbar);
                    umma::mbar_wait(mb_a, ph_a);
                    umma::gemm1<8>(tb + S_DH2, S.MN(TA1S, T64B, 64), S.MN(TDS, TDB, 16), ID_WG(16), acc);
                }
                ph_a ^= 1u;
            }
            wait_mma(mbar, ph);
            // ------------------------------------------- S1: u -> DE, dH1, G
            int eU;
            {
                float u[4][8], mu = 0.f;
                const int esc = -(eDLY + eH2);  // folded into the staging scale (see C1)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    umma::tmem_ld8(my + S_SL + 8 * (4 * qh + i), u[i]);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        u[i][k] = ((m1 >> (8 * i + k)) & 1u) ? u[i][k] : 0.f;
                        mu = fmaxf(mu, fabsf(u[i][k]));
                    }
                }
                eU = PS.guess(kU);
                PS.contrib(kU, mu * pow2i(esc));
#pragma unroll 1
                for (int pass = 0;; ++pass) {
                    const float su = pow2i(eU + esc);
#pragma unroll
                    for (int i = 0; i < 4; ++i) stage_blk_ta<64>(S, TXS, r, 4 * qh + i, u[i], su, my + S_AH, my + S_AL);
                    umma::tmem_st_wait();
                    group_publish(1);
                    if (pass) break;
                    if (PS.check(kU, eU)) break;
                }
            }
            {
                // Theorem 1 through one accumulator (see field_bwd_kernel)
                const bool acca = acc_begin(1, eU + eE);
                const bool accb = acc_begin(2, eMV);
                if (mma_w) {
                    umma::gemm3t<4>(tb + S_SL, tb + S_AH, tb + S_AL, S.MN(WH1, WH1B, 48), ID_KM(48), false);
                    umma::commit_elect(mbar);
                    umma::mbar_wait(mb_e, ph_e);
                    umma::gemm1<8>(tb + S_DH1A, S.MN(TXS, T64B, 64), S.MN(TES, TEB, 48), ID_WG(48), acca);
                    umma::gemm1<8>(tb + S_G, S.MN(TYS, T64B, 64), S.MN(TMV, TEB, 48), ID_WG(48), accb);
                    umma::commit_elect(mbarw);
                }
                ph_e ^= 1u;
                wpend = true;
            }
            wait_mma(mbar, ph);
            // ------------------------------------------- S2: scatter inputs
            // dH2 (before the DE GEMM) is done: TA1 takes the next tile's A1
            if (dma_t && has_next) dma(TA1S, fwt(ntile) + FW_A1, T64B, mb_a);
            {
                const float sde = pow2i(-(eU + eH1));
                float de0[8], de1[8];
                umma::tmem_ld8(my + S_SL + 16 * qh, de0);
                umma::tmem_ld8(my + S_SL + 16 * qh + 8, de1);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (16 * qh + k < 2 * NA) __stcs(SBt + (16 * qh + k) * TILE + r, de0[k] * sde);
                    if (16 * qh + 8 + k < 2 * NA) __stcs(SBt + (16 * qh + 8 + k) * TILE + r, de1[k] * sde);
                }
                if (qh == 0) {
                    __stcs(SBt + 64 * TILE + r, q0);
                    __stcs(SBt + 65 * TILE + r, q1);
                    __stcs(SBt + 66 * TILE + r, q2);
                }
            }
            // the next tile's S0 waits on its handoff slot; the slot reset of the exponent maxima
            // happens after S0's barrier, so no tile-boundary barrier is needed
        }
        if (wpend) wait_mma(mbarw, phw);
#pragma unroll
        for (int jj = 0; jj < 3; ++jj)
            if (acc_live[jj]) fold(jj);
    }
    umma::fence_before_sync();
    __syncthreads();
#ifdef NS2B_PHASE_PROF
    if (blockIdx.x == 0 && t == 0) printf("PHASEPROF bwd2 C-waits-free %lld S-waits-full %lld\n", bpw[0], bpw[1]);
#endif
    if (warp == 0) umma::tmem_dealloc(tb, 512);
}
#undef BPW

// ---------------------------------------------------------------------------
// Gather kernel (one pass per step): per 128-sample tile, trilinear features and
// d feature/dx for the active levels (_kernels.py:67-119 without corner records),
// 4 levels (32 float2 loads) in flight per thread.  Features are staged straight into
// the fp16 hi/lo E-tile layout the MLP kernels DMA into shared memory.
constexpr int GATHER_BLOCK = TILE;

#ifdef NS2B_GATHER_MINB
__global__ void __launch_bounds__(GATHER_BLOCK, NS2B_GATHER_MINB)
#else
__global__ void __launch_bounds__(GATHER_BLOCK)
#endif
field_gather_kernel(FieldDev f, const float *__restrict__ pos, const int32_t *__restrict__ ray_ids,
                    const double *__restrict__ dirs, const int32_t *__restrict__ count, Workspace ws) {
    __shared__ float raw[32][TILE + 1];
    __shared__ LevelSm lvs[NS2B_MAX_LEVELS];
    __shared__ uint32_t red[2][2][4];
    const int t = threadIdx.x;
    if (t < NS2B_MAX_LEVELS) {
        lvs[t].lv = f.lv[t];
        lvs[t].sx = f.sx[t];
        lvs[t].sy = f.sy[t];
        lvs[t].sz = f.sz[t];
    }
    __syncthreads();
    Reducer R{red, 0};
    const int NA = f.n_active;
    const int P = *count;
    const int64_t ntiles = (static_cast<int64_t>(P) + TILE - 1) / TILE;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t p = tile * TILE + t;
        const bool valid = p < P;
        float x0 = 0.f, x1 = 0.f, x2 = 0.f, v0 = 0.f, v1 = 0.f, v2 = 0.f;
        if (valid) {
            x0 = pos[3 * p];
            x1 = pos[3 * p + 1];
            x2 = pos[3 * p + 2];
            const int rr = ray_ids[p];
            v0 = static_cast<float>(dirs[3 * rr]);  // field.py:216 (fp32 view dirs)
            v1 = static_cast<float>(dirs[3 * rr + 1]);
            v2 = static_cast<float>(dirs[3 * rr + 2]);
        }
        const float un0 = normalize_coord(x0, f.lo[0], f.ext[0]);
        const float un1 = normalize_coord(x1, f.lo[1], f.ext[1]);
        const float un2 = normalize_coord(x2, f.lo[2], f.ext[2]);
        float *Jt = ws.jac + tile * JROWS * TILE;
        float fmax_ = fmaxf(fmaxf(fabsf(x0), fabsf(x1)), fmaxf(fabsf(x2), 1.f));
#pragma unroll 1
        for (int g = 0; g < NS2B_MAX_LEVELS; g += 4) {
            if (g >= NA) break;
            float2 v[4][8];
            float fr[4][3];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int l = g + i;
                if (l < NA) {
                    const LevelInfo lv = lvs[l].lv;
                    int cx, cy, cz;
                    cell_frac(un0, lv.n, cx, fr[i][0]);
                    cell_frac(un1, lv.n, cy, fr[i][1]);
                    cell_frac(un2, lv.n, cz, fr[i][2]);
                    const float2 *tab = reinterpret_cast<const float2 *>(f.tables) + l * f.T;
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        v[i][c] = __ldg(tab + corner_row(lv, cx + ((c >> 2) & 1), cy + ((c >> 1) & 1), cz + (c & 1)));
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int l = g + i;
                if (l < NA) {
                    const float fx = fr[i][0], fy = fr[i][1], fz = fr[i][2];
                    const float sx = lvs[l].sx, sy = lvs[l].sy, sz = lvs[l].sz;
                    float f0 = 0.f, f1 = 0.f, j00 = 0.f, j01 = 0.f, j02 = 0.f, j10 = 0.f, j11 = 0.f, j12 = 0.f;
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const int ox = (c >> 2) & 1, oy = (c >> 1) & 1, oz = c & 1;
                        const float wx = ox ? fx : 1.f - fx, wy = oy ? fy : 1.f - fy, wz = oz ? fz : 1.f - fz;
                        const float w = wx * wy * wz;
                        const float dwx = (ox ? sx : -sx) * (wy * wz);
                        const float dwy = (oy ? sy : -sy) * (wx * wz);
                        const float dwz = (oz ? sz : -sz) * (wx * wy);
                        f0 = fmaf(w, v[i][c].x, f0);
                        f1 = fmaf(w, v[i][c].y, f1);
                        j00 = fmaf(dwx, v[i][c].x, j00);
                        j01 = fmaf(dwy, v[i][c].x, j01);
                        j02 = fmaf(dwz, v[i][c].x, j02);
                        j10 = fmaf(dwx, v[i][c].y, j10);
                        j11 = fmaf(dwy, v[i][c].y, j11);
                        j12 = fmaf(dwz, v[i][c].y, j12);
                    }
                    fmax_ = fmaxf(fmax_, fmaxf(fabsf(f0), fabsf(f1)));
                    raw[2 * l][t] = f0;
                    raw[2 * l + 1][t] = f1;
                    float *jr = Jt + 6 * l * TILE + t;  // streaming stores: keep the tables in L2
                    __stcs(jr, j00);
                    __stcs(jr + TILE, j01);
                    __stcs(jr + 2 * TILE, j02);
                    __stcs(jr + 3 * TILE, j10);
                    __stcs(jr + 4 * TILE, j11);
                    __stcs(jr + 5 * TILE, j12);
                }
            }
        }
        {  // (view-dir loads issued before the level loop)
            float *xvt = ws.xv + tile * XVROWS * TILE + t;
            __stcs(xvt, x0);
            __stcs(xvt + TILE, x1);
            __stcs(xvt + 2 * TILE, x2);
            __stcs(xvt + 3 * TILE, v0);
            __stcs(xvt + 4 * TILE, v1);
            __stcs(xvt + 5 * TILE, v2);
        }
        const int eE = R.one(fmax_);
        float row[48];
#pragma unroll
        for (int a = 0; a < 32; ++a) row[a] = (a < 2 * NA) ? raw[a][t] : 0.f;
        row[32] = x0;
        row[33] = x1;
        row[34] = x2;
        row[35] = 1.f;
#pragma unroll
        for (int i = 36; i < 48; ++i) row[i] = 0.f;
        const float sc = pow2i(eE);
#pragma unroll
        for (int i = 0; i < 48; ++i) row[i] *= sc;
        uint8_t *et = ws.e_tiles + tile * 2 * TEB;
        umma::stage_row<0, 48, true>(et, et + TEB, t, row);
        if (t == 0) ws.e_exp[tile] = eE;
        __syncthreads();  // raw[] reuse
    }
}

// ---------------------------------------------------------------------------
// field_backward(need_input_grads=True) (field.py:332-349) from the backward's outputs:
//   dl_dx = dcin_x + de_x + sum_a de_a J_a + q Hess(j_d features),  dl_dv = dcin_v,
// with de = dL/de_aug (= dd j_d + dg jg, so de J = dd n + dg (jg J)), J from the gather,
// and the encoding curvature (hessian_contract, _kernels.py:159-206) from a fresh corner
// gather, 4 levels (32 loads) in flight per thread.
__global__ void __launch_bounds__(TILE)
field_input_levels_kernel(FieldDev f, const int32_t *__restrict__ count, const Workspace ws, double ix,
                          double iy, double iz, float *__restrict__ dl_dx, float *__restrict__ dl_dv) {
    __shared__ LevelSm lvs[NS2B_MAX_LEVELS];
    const int t = threadIdx.x;
    if (t < NS2B_MAX_LEVELS) {
        lvs[t].lv = f.lv[t];
        lvs[t].sx = f.sx[t];
        lvs[t].sy = f.sy[t];
        lvs[t].sz = f.sz[t];
    }
    __syncthreads();
    const int NA = f.n_active;
    const int P = *count;
    const int64_t ntiles = (static_cast<int64_t>(P) + TILE - 1) / TILE;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t p = tile * TILE + t;
        if (p >= P) continue;
        const float *SBt = ws.sb + tile * SBROWS * TILE + t;
        const float *Jt = ws.jac + tile * JROWS * TILE + t;
        const float *xi = ws.xin + tile * XINROWS * TILE + t;
        const float *xv = ws.xv + tile * XVROWS * TILE + t;
        const float u0 = normalize_coord(xv[0], f.lo[0], f.ext[0]);
        const float u1 = normalize_coord(xv[TILE], f.lo[1], f.ext[1]);
        const float u2 = normalize_coord(xv[2 * TILE], f.lo[2], f.ext[2]);
        const float q0 = SBt[64 * TILE], q1 = SBt[65 * TILE], q2 = SBt[66 * TILE];
        float gx0 = xi[0] + xi[6 * TILE], gx1 = xi[TILE] + xi[7 * TILE], gx2 = xi[2 * TILE] + xi[8 * TILE];
        float hxy = 0.f, hxz = 0.f, hyz = 0.f;
#pragma unroll 1
        for (int g = 0; g < NA; g += 4) {
            float2 v[4][8];
            double fr[4][3];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int l = g + i;
                if (l < NA) {
                    const LevelInfo lv = lvs[l].lv;
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
            for (int i = 0; i < 4; ++i) {
                const int l = g + i;
                if (l < NA) {
                    const float de0 = SBt[(2 * l) * TILE], de1 = SBt[(2 * l + 1) * TILE];
                    const float jd0 = SBt[(32 + 2 * l) * TILE], jd1 = SBt[(33 + 2 * l) * TILE];
                    const float *jr = Jt + 6 * l * TILE;
                    gx0 = fmaf(de0, jr[0], fmaf(de1, jr[3 * TILE], gx0));
                    gx1 = fmaf(de0, jr[TILE], fmaf(de1, jr[4 * TILE], gx1));
                    gx2 = fmaf(de0, jr[2 * TILE], fmaf(de1, jr[5 * TILE], gx2));
                    double h01, h02, h12;
                    hess_from_corners(v[i], fr[i][0], fr[i][1], fr[i][2], jd0, jd1, h01, h02, h12);
                    const double n = static_cast<double>(lvs[l].lv.n);
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
        dl_dv[3 * p] = xi[3 * TILE];
        dl_dv[3 * p + 1] = xi[4 * TILE];
        dl_dv[3 * p + 2] = xi[5 * TILE];
    }
}

// ---------------------------------------------------------------------------
// Table-gradient scatter (Eq. 9 + first order, field.py:317-324): block = one tile at
// one level, thread = sample, 8 float2 REDs:  grad += w dL/dfeat + j_d (q . dw).
// Consecutive lanes are consecutive samples of a ray; on the coarse levels they often
// hit the same corner row, so runs of equal rows are pre-summed with a segmented
// shuffle reduction and only the run's last lane issues the RED.
constexpr int kAggLevels = 11;  // default (measured 9..16 at c2: 11 best by ~0.03 ms); NS2B_AGG_LEVELS overrides
static int agg_levels_env() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("NS2B_AGG_LEVELS");
        v = e ? atoi(e) : kAggLevels;
    }
    return v;
}

__device__ __forceinline__ void red_add_f32x4(float *addr, float a, float b, float c, float d) {
    atomicAdd(reinterpret_cast<float4 *>(addr), make_float4(a, b, c, d));
}

#ifndef NS2B_SCATTER_MINB
#define NS2B_SCATTER_MINB 6
#endif
__global__ void __launch_bounds__(TILE, NS2B_SCATTER_MINB)
field_scatter_kernel(FieldDev f, const float *__restrict__ pos, const int32_t *__restrict__ count,
                     const Workspace ws, float *__restrict__ g_tab, int agg_levels) {
    __shared__ LevelSm lvs[NS2B_MAX_LEVELS];
    const int t = threadIdx.x, lane = t & 31;
    if (t < NS2B_MAX_LEVELS) {
        lvs[t].lv = f.lv[t];
        lvs[t].sx = f.sx[t];
        lvs[t].sy = f.sy[t];
        lvs[t].sz = f.sz[t];
    }
    __syncthreads();
    const int NA = f.n_active;
    const int P = *count;
    const int64_t ntiles = (static_cast<int64_t>(P) + TILE - 1) / TILE;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t p = tile * TILE + t;
        const bool valid = p < P;
        const float *SBt = ws.sb + tile * SBROWS * TILE + t;
        float x0 = 0.f, x1 = 0.f, x2 = 0.f, q0 = 0.f, q1 = 0.f, q2 = 0.f;
        if (valid) {
            x0 = pos[3 * p];
            x1 = pos[3 * p + 1];
            x2 = pos[3 * p + 2];
            q0 = SBt[64 * TILE];
            q1 = SBt[65 * TILE];
            q2 = SBt[66 * TILE];
        }
        const float un0 = normalize_coord(x0, f.lo[0], f.ext[0]);
        const float un1 = normalize_coord(x1, f.lo[1], f.ext[1]);
        const float un2 = normalize_coord(x2, f.lo[2], f.ext[2]);
        // per-level inputs, loaded one level ahead
        float nde0 = 0.f, nde1 = 0.f, njd0 = 0.f, njd1 = 0.f;
        if (valid) {
            nde0 = SBt[0];
            nde1 = SBt[TILE];
            njd0 = SBt[32 * TILE];
            njd1 = SBt[33 * TILE];
        }
#pragma unroll 1
        for (int l = 0; l < NA; ++l) {
            const float de0 = nde0, de1 = nde1, jd0 = njd0, jd1 = njd1;
            if (valid && l + 1 < NA) {
                nde0 = SBt[(2 * l + 2) * TILE];
                nde1 = SBt[(2 * l + 3) * TILE];
                njd0 = SBt[(34 + 2 * l) * TILE];
                njd1 = SBt[(35 + 2 * l) * TILE];
            }
            const LevelInfo lv = lvs[l].lv;
            const float sx = lvs[l].sx, sy = lvs[l].sy, sz = lvs[l].sz;
            int cx, cy, cz;
            float fx, fy, fz;
            cell_frac(un0, lv.n, cx, fx);
            cell_frac(un1, lv.n, cy, fy);
            cell_frac(un2, lv.n, cz, fz);
            float *gt = g_tab + l * f.T * 2;
            // the 16-B x-pair RED needs a 16-B aligned level base: with an odd table size
            // every other level starts 8-B aligned, so those levels take two float2 REDs
            const bool pair16 = (reinterpret_cast<uintptr_t>(gt) & 15u) == 0;
            // runs of equal cells along the warp's samples (consecutive samples of a ray):
            // on the coarse levels all 8 corners of a run are pre-summed by one segmented
            // scan and only the run's last lane issues the REDs
            uint32_t heads = 0xFFFFFFFFu;
            if (l < agg_levels) {
                const uint64_t key = static_cast<uint64_t>(cx) | (static_cast<uint64_t>(cy) << 21) |
                                     (static_cast<uint64_t>(cz) << 42);
                const uint64_t prev = __shfl_up_sync(0xFFFFFFFFu, key, 1);
                heads = __ballot_sync(0xFFFFFFFFu, lane == 0 || prev != key);
            }
            // corner c = 4 ox + 2 oy + oz
            float a[8], b[8];
            uint32_t row[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int ox = (c >> 2) & 1, oy = (c >> 1) & 1, oz = c & 1;
                const float wx = ox ? fx : 1.f - fx, wy = oy ? fy : 1.f - fy, wz = oz ? fz : 1.f - fz;
                const float w = wx * wy * wz;
                const float dwx = (ox ? sx : -sx) * (wy * wz);
                const float dwy = (oy ? sy : -sy) * (wx * wz);
                const float dwz = (oz ? sz : -sz) * (wx * wy);
                const float qd = dwx * q0 + dwy * q1 + dwz * q2;
                a[c] = valid ? fmaf(w, de0, jd0 * qd) : 0.f;
                b[c] = valid ? fmaf(w, de1, jd1 * qd) : 0.f;
                row[c] = corner_row(lv, cx + ox, cy + oy, cz + oz);
            }
            if (heads != 0xFFFFFFFFu) {  // some run is longer than one sample (warp-uniform)
                const int seg_start = 31 - __clz(heads & ((2u << lane) - 1u));
                // only as many scan steps as the longest run needs
                const int maxrun = static_cast<int>(__reduce_max_sync(0xFFFFFFFFu, lane - seg_start + 1));
#pragma unroll 1
                for (int o = 1; o < maxrun; o <<= 1) {  // segmented inclusive scan of all 16 values
                    const bool take = lane - o >= seg_start;
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float pa = __shfl_up_sync(0xFFFFFFFFu, a[c], o);
                        const float pb = __shfl_up_sync(0xFFFFFFFFu, b[c], o);
                        if (take) {
                            a[c] += pa;
                            b[c] += pb;
                        }
                    }
                }
                if (!(lane == 31 || ((heads >> (lane + 1)) & 1u))) continue;  // not a run's last lane
            } else if (!valid) {
                continue;
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {  // x-pairs (c, c + 4): one 16-B RED when adjacent
                if (pair16 && (row[c] ^ row[c + 4]) == 1u) {
                    const bool sw = row[c] & 1u;
                    red_add_f32x4(gt + 2 * (row[c] & ~1u), sw ? a[c + 4] : a[c], sw ? b[c + 4] : b[c],
                                  sw ? a[c] : a[c + 4], sw ? b[c] : b[c + 4]);
                } else {
                    red_add_f32x2(gt + 2 * row[c], a[c], b[c]);
                    red_add_f32x2(gt + 2 * row[c + 4], a[c + 4], b[c + 4]);
                }
            }
        }
    }
}

static int g_tc_attr = 0;
static int ensure_tc_attrs() {
    if (g_tc_attr) return NS2B_OK;
    cudaError_t e = cudaFuncSetAttribute(field_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(SMEM_FWD));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(field_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(SMEM_BWD));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(field_bwd2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(b2::SMEM));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(field_fwd2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(SMEM_FWD2));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(field_fwd2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(SMEM_FWD2G));
    if (e != cudaSuccess) return set_error(NS2B_ECUDA, "tc smem attribute: %s", cudaGetErrorString(e));
    g_tc_attr = 1;
    return NS2B_OK;
}

// NS2B_FWD=1 selects the one-tile forward (field_fwd_kernel); the default is the
// two-tiles-in-flight field_fwd2_kernel
static bool use_fwd1() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("NS2B_FWD");
        v = (e && atoi(e) == 1) ? 1 : 0;
    }
    return v == 1;
}

static int fwd_mode();

// NS2B_BWD=1 selects the one-group backward (field_bwd_kernel); the default is the
// two-group pipelined field_bwd2_kernel (input cotangents, want_xin, always use the former)
static bool use_bwd1() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("NS2B_BWD");
        v = (e && atoi(e) == 1) ? 1 : 0;
    }
    return v == 1;
}

static void launch_bwd(const FieldDev &f, int64_t ntiles, const int32_t *count, const float *dl_dc,
                       const float *dl_dsdf, const float *dl_dn_extra, float eik_w, const int64_t *eik_count,
                       float *g_sdf, float *g_color, const Workspace &ws, int want_xin, cudaStream_t st) {
    if (want_xin || use_bwd1())
        field_bwd_kernel<<<grid_for(ntiles, 1, kNumSMs), MLP_THREADS, SMEM_BWD, st>>>(
            f, count, dl_dc, dl_dsdf, dl_dn_extra, eik_w, eik_count, g_sdf, g_color, ws, want_xin);
    else
        field_bwd2_kernel<<<grid_for(ntiles, 1, kNumSMs), MLP_THREADS, b2::SMEM, st>>>(
            f, count, dl_dc, dl_dsdf, dl_dn_extra, eik_w, eik_count, g_sdf, g_color, ws);
}

static void launch_fwd(const FieldDev &f, int64_t ntiles, const int32_t *count, float *sdf, float *colors,
                       float *normals, float *geo, double *eik_sum, const Workspace &ws, cudaStream_t st,
                       float eik_w = 0.f, const int64_t *eik_count = nullptr) {
    if (use_fwd1())  // (does not fuse the Eikonal cotangent: its flag tells the backward)
        field_fwd_kernel<<<grid_for(ntiles, 1, kNumSMs), MLP_THREADS, SMEM_FWD, st>>>(f, count, sdf, colors, normals,
                                                                                     geo, eik_sum, ws);
    else
        field_fwd2_kernel<false><<<grid_for(ntiles, 1, kNumSMs), MLP_THREADS, SMEM_FWD2, st>>>(
            f, count, sdf, colors, normals, geo, eik_sum, ws, eik_w, eik_count, nullptr, nullptr, nullptr);
}

// NS2B_FWD: 1 = gather kernel + one-tile forward, unset / 2 = gather kernel + two-tile
// forward (the default), 3 = the two-tile forward with the gather fused
// (field_fwd2_kernel<true>).  Measured at c2: 3 is slower (gather + forward 25.2 ms vs 6.35 +
// 7.3 ms): a tile's gather is bound by L1 wavefronts (~10k cycles of L1 per tile), and with
// two tiles per SM, each gathering before its MLP phases, the L1 idles while both groups
// run MMAs -- the separate gather kernel keeps four tiles per SM in flight on the L1.
static int fwd_mode() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("NS2B_FWD");
        v = e ? atoi(e) : 2;
    }
    return v;
}

}  // namespace tc

int field_workspace_bytes(int64_t capacity, size_t *bytes) {
    NS2B_REQUIRE(bytes != nullptr && capacity >= 0, "workspace query");
    const int64_t ntiles = (capacity + tc::TILE - 1) / tc::TILE;
    *bytes = static_cast<size_t>(ntiles) * tc::ws_tile_bytes() + 256;
    return NS2B_OK;
}

// split entry points (the trainer times each kernel; field_forward/backward chain them)
int field_stage_tc(int which, const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids,
                   const double *dirs, const int32_t *count, int64_t capacity, float *sdf, float *colors,
                   float *normals, float *geo, double *eik_sum, const float *dl_dc, const float *dl_dsdf,
                   const float *dl_dn_extra, double eik_weight, const int64_t *eik_count, float *grad_sdf,
                   float *grad_color, float *grad_tables, void *workspace, cudaStream_t st) {
    FieldDev f;
    int rc = make_field_dev(field, f);
    if (rc) return rc;
    if ((rc = tc::ensure_tc_attrs())) return rc;
    NS2B_REQUIRE(workspace != nullptr, "field kernels need the workspace (ns2b_field_workspace_bytes)");
    if (capacity <= 0) return NS2B_OK;
    const int64_t ntiles = (capacity + tc::TILE - 1) / tc::TILE;
    const tc::Workspace ws = tc::ws_carve(workspace, ntiles);
    switch (which) {
    case 0:
        tc::field_gather_kernel<<<grid_for(ntiles, 1, 1 << 30), tc::GATHER_BLOCK, 0, st>>>(f, pos32, ray_ids, dirs,
                                                                                         count, ws);
        return check_launch("field_gather");
    case 1:
        tc::launch_fwd(f, ntiles, count, sdf, colors, normals, geo, eik_sum, ws, st);
        return check_launch("field_mlp_forward");
    case 4:
        NS2B_REQUIRE(eik_count != nullptr, "field_mlp_forward_eik: eik_count required");
        tc::launch_fwd(f, ntiles, count, sdf, colors, normals, geo, eik_sum, ws, st, static_cast<float>(eik_weight),
                       eik_count);
        return check_launch("field_mlp_forward");
    case 5:  // gather + MLP forward (+ the Eikonal cotangent when eik_count)
        NS2B_REQUIRE(pos32 && ray_ids && dirs && count, "field_forward_fused: null input");
        if (tc::fwd_mode() == 3) {
            tc::field_fwd2_kernel<true><<<grid_for(ntiles, 1, kNumSMs), tc::MLP_THREADS, tc::SMEM_FWD2G, st>>>(
                f, count, sdf, colors, normals, geo, eik_sum, ws, static_cast<float>(eik_weight), eik_count, pos32,
                ray_ids, dirs);
            return check_launch("field_gather_mlp_forward");
        }
        tc::field_gather_kernel<<<grid_for(ntiles, 1, 1 << 30), tc::GATHER_BLOCK, 0, st>>>(f, pos32, ray_ids, dirs,
                                                                                             count, ws);
        if ((rc = check_launch("field_gather"))) return rc;
        tc::launch_fwd(f, ntiles, count, sdf, colors, normals, geo, eik_sum, ws, st, static_cast<float>(eik_weight),
                       eik_count);
        return check_launch("field_mlp_forward");
    case 2:
        NS2B_REQUIRE(eik_weight == 0.0 || eik_count != nullptr, "eik_count required with eik_weight");
        tc::launch_bwd(f, ntiles, count, dl_dc, dl_dsdf, dl_dn_extra, static_cast<float>(eik_weight), eik_count,
                       grad_sdf, grad_color, ws, 0, st);
        return check_launch("field_mlp_backward");
    default:
        tc::field_scatter_kernel<<<grid_for(ntiles, 1, 1 << 30), tc::TILE, 0, st>>>(f, pos32, count, ws,
                                                                                       grad_tables, tc::agg_levels_env());
        return check_launch("field_scatter");
    }
}

int field_forward_tc(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids, const double *dirs,
                     const int32_t *count, int64_t capacity, float *sdf, float *colors, float *normals, float *geo,
                     double *eik_sum, void *workspace, cudaStream_t st) {
    FieldDev f;
    int rc = make_field_dev(field, f);
    if (rc) return rc;
    if ((rc = tc::ensure_tc_attrs())) return rc;
    NS2B_REQUIRE(workspace != nullptr, "field_forward: workspace required (ns2b_field_workspace_bytes)");
    if (capacity <= 0) return NS2B_OK;
    const int64_t ntiles = (capacity + tc::TILE - 1) / tc::TILE;
    const tc::Workspace ws = tc::ws_carve(workspace, ntiles);
    if (tc::fwd_mode() == 3) {
        tc::field_fwd2_kernel<true><<<grid_for(ntiles, 1, kNumSMs), tc::MLP_THREADS, tc::SMEM_FWD2G, st>>>(
            f, count, sdf, colors, normals, geo, eik_sum, ws, 0.f, nullptr, pos32, ray_ids, dirs);
        return check_launch("field_forward_tc");
    }
    tc::field_gather_kernel<<<grid_for(ntiles, 1, 1 << 30), tc::GATHER_BLOCK, 0, st>>>(f, pos32, ray_ids, dirs,
                                                                                         count, ws);
    if ((rc = check_launch("field_gather"))) return rc;
    tc::launch_fwd(f, ntiles, count, sdf, colors, normals, geo, eik_sum, ws, st);
    return check_launch("field_forward_tc");
}

int field_backward_tc(const ns2b_field_t *field, const float *pos32, const int32_t *ray_ids, const double *dirs,
                      const int32_t *count, int64_t capacity, const float *dl_dc, const float *dl_dsdf,
                      const float *dl_dn_extra, double eik_weight, const int64_t *eik_count, float *grad_sdf,
                      float *grad_color, float *grad_tables, void *workspace, cudaStream_t st, float *dl_dx,
                      float *dl_dv) {
    FieldDev f;
    int rc = make_field_dev(field, f);
    if (rc) return rc;
    if ((rc = tc::ensure_tc_attrs())) return rc;
    NS2B_REQUIRE(eik_weight == 0.0 || eik_count != nullptr, "eik_count required with eik_weight");
    NS2B_REQUIRE(workspace != nullptr, "field_backward: workspace of the matching forward required");
    if (capacity <= 0) return NS2B_OK;
    const int64_t ntiles = (capacity + tc::TILE - 1) / tc::TILE;
    const tc::Workspace ws = tc::ws_carve(workspace, ntiles);
    tc::launch_bwd(f, ntiles, count, dl_dc, dl_dsdf, dl_dn_extra, static_cast<float>(eik_weight), eik_count,
                   grad_sdf, grad_color, ws, dl_dx != nullptr, st);
    if ((rc = check_launch("field_backward_tc"))) return rc;
    if (dl_dx != nullptr) {
        tc::field_input_levels_kernel<<<grid_for(ntiles, 1, kNumSMs * 8), tc::TILE, 0, st>>>(
            f, count, ws, field->inv_extent[0], field->inv_extent[1], field->inv_extent[2], dl_dx, dl_dv);
        if ((rc = check_launch("field_input_levels"))) return rc;
    }
    if (grad_tables == nullptr) return NS2B_OK;
    tc::field_scatter_kernel<<<grid_for(ntiles, 1, 1 << 30), tc::TILE, 0, st>>>(f, pos32, count, ws,
                                                                                   grad_tables, tc::agg_levels_env());
    return check_launch("field_scatter");
}

}  // namespace ns2b
