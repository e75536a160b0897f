// tcgen05 (5th-gen tensor core) building blocks for sm_100a: shared-memory matrix
// descriptors, instruction descriptors, MMA issue, commit/mbarrier, TMEM alloc/ld.
//
// Operand tiles use the SWIZZLE_NONE canonical layout made of 8-row x 16-byte "core
// matrices" (8 x 8 16-bit elements, 128 B contiguous).  A logical R x C tile (R rows,
// C columns, C % 8 == 0) is stored as core matrices [R/8][C/8], column-block fastest:
//     byte(r, c) = ((r/8) * (C/8) + c/8) * 128 + (r%8) * 16 + (c%8) * 2
// The same bytes serve two descriptor views:
//   * K-major   (rows = M or N, cols = K):  LBO = 128,           SBO = (C/8)*128
//   * MN-major  (rows = K, cols = M or N):  LBO = (C/8)*128,     SBO = 128
// so a per-sample tile [sample][feature] is both the A operand of a forward GEMM
// (K = features) and an operand of a weight-gradient GEMM (K = samples).  Every MMA
// consumes K = 16, i.e. two core-matrix steps along K, so the descriptor start
// address advances by 2*LBO per instruction in either view.
#pragma once

#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace ns2b {
namespace umma {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Shared-memory matrix descriptor (SmemDescriptor, version 1, SWIZZLE_NONE).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // version = 1 (sm100)
    // base_offset = 0, lbo_mode = 0, layout_type = 0 (SWIZZLE_NONE)
    return d;
}

// Instruction descriptor for kind::f16 with fp32 accumulation.
//   fmt: 0 = F16, 1 = BF16 (both operands);  a_mn/b_mn: 0 = K-major, 1 = MN-major
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int fmt, int a_mn, int b_mn) {
    return (1u << 4)                                   // c_format = F32
           | (static_cast<uint32_t>(fmt) << 7)         // a_format
           | (static_cast<uint32_t>(fmt) << 10)        // b_format
           | (static_cast<uint32_t>(a_mn) << 15)       // a_major
           | (static_cast<uint32_t>(b_mn) << 16)       // b_major
           | (static_cast<uint32_t>(N >> 3) << 17)     // n_dim
           | (static_cast<uint32_t>(M >> 4) << 24);    // m_dim
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

// Arrive on an mbarrier once all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void commit(uint64_t *mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(mbar)));
}

__device__ __forceinline__ void mbar_init(uint64_t *mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count));
}

// try_wait suspends the warp until the phase completes or this many ns pass, so the
// waiting warps do not spin on the issue slots the MMA-issuing warp needs.
constexpr uint32_t kSuspendNs = 1000000;
__device__ __forceinline__ void mbar_wait(uint64_t *mbar, uint32_t parity) {
    uint32_t addr = smem_u32(mbar);
#ifdef NS2B_DEBUG_HANG
    {
        const long long t0 = clock64();
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n\t.reg .pred P1;\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                "selp.u32 %0, 1, 0, P1;\n\t}\n"
                : "=r"(done)
                : "r"(addr), "r"(parity));
            if (!done && clock64() - t0 > 4000000000LL) {
                printf("HANG block %d thread %d mbar smem 0x%x parity %u\n", blockIdx.x, threadIdx.x, addr, parity);
                __trap();
            }
        }
        return;
    }
#endif
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n\t"
        "DONE:\n\t}\n" ::"r"(addr),
        "r"(parity), "r"(kSuspendNs));
}

// plain spin (no suspend hint), for latency comparisons
__device__ __forceinline__ void mbar_wait_spin(uint64_t *mbar, uint32_t parity) {
    uint32_t addr = smem_u32(mbar);
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n\t"
        "DONE:\n\t}\n" ::"r"(addr),
        "r"(parity));
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// Generic-proxy smem writes -> visible to the tensor core (async proxy).
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_before_sync() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after_sync() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// TMEM allocation (one warp; the base column address lands in *dst).
__device__ __forceinline__ void tmem_alloc(uint32_t *dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}

// 32 lanes x 32 bit, 16 consecutive columns: thread t of warp w gets lane 32w+t.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 32 bit, 16 consecutive columns from registers (thread t -> lane 32w+t).
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float *v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
        "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
        "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
        : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld2(uint32_t taddr, float &a, float &b) {
    uint32_t r0, r1;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    a = __uint_as_float(r0);
    b = __uint_as_float(r1);
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float (&v)[4]) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st2(uint32_t taddr, float a, float b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(taddr), "r"(__float_as_uint(a)),
                 "r"(__float_as_uint(b))
                 : "memory");
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, float a, float b, float c, float d) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(__float_as_uint(a)),
                 "r"(__float_as_uint(b)), "r"(__float_as_uint(c)), "r"(__float_as_uint(d))
                 : "memory");
}

// Load N (multiple of 16) consecutive columns of this thread's lane into v[0..N).
template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float *v) {
#pragma unroll
    for (int c = 0; c < N; c += 16) {
        float t[16];
        tmem_ld16(taddr + c, t);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[c + i] = t[i];
    }
}

// Bulk L2 prefetch (TMA engine) of a contiguous global range; bytes % 16 == 0.
__device__ __forceinline__ void prefetch_l2(const void *gptr, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gptr), "r"(bytes) : "memory");
}

// One-thread bulk DMA global -> shared (TMA engine, no registers); completion is
// signalled as transaction bytes on `mbar` (arrive + expect_tx by the same thread).
template <bool kEvictFirst = false>
__device__ __forceinline__ void bulk_g2s(void *sdst, const void *gsrc, uint32_t bytes, uint64_t *mbar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes)
                 : "memory");
    if (kEvictFirst) {  // data read exactly once: leave L2 to the prefetched next-tile inputs
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
            "%4;" ::"r"(smem_u32(sdst)),
            "l"(gsrc), "r"(bytes), "r"(smem_u32(mbar)), "l"(pol)
            : "memory");
    } else {
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(sdst)),
            "l"(gsrc), "r"(bytes), "r"(smem_u32(mbar))
            : "memory");
    }
}

// Plain arrive (release.cta): one of the barrier's expected arrivals.
__device__ __forceinline__ void mbar_arrive(uint64_t *mbar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(mbar)) : "memory");
}

// Several bulk copies completing one mbarrier phase: one arrive + expect_tx for the
// total, then the copies (complete_tx only).  Evict-first: data read exactly once.
__device__ __forceinline__ void mbar_expect_tx(uint64_t *mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s_tx(void *sdst, const void *gsrc, uint32_t bytes, uint64_t *mbar) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
        "%4;" ::"r"(smem_u32(sdst)),
        "l"(gsrc), "r"(bytes), "r"(smem_u32(mbar)), "l"(pol)
        : "memory");
}

// One-thread bulk DMA shared -> global (bulk-group completion; the source buffer may be
// rewritten after bulk_wait_read() returns in the issuing thread).
__device__ __forceinline__ void bulk_s2g(void *gdst, const void *ssrc, uint32_t bytes) {
    // evict-first in L2: the tiles are read back by a later kernel, long after this one
    // has streamed far more than L2 through; keep L2 for the prefetched next-tile inputs
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(gdst),
                 "r"(smem_u32(ssrc)), "r"(bytes), "l"(pol)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// all but the N most recent bulk groups of this thread have finished reading shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read_n() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// ---------------------------------------------------------------- staging --
// Byte offset of element (r, c) in a core-matrix tiled tile with C columns.
__host__ __device__ constexpr uint32_t tile_off(int r, int c, int C) {
    return static_cast<uint32_t>((((r >> 3) * (C >> 3) + (c >> 3)) << 7) + ((r & 7) << 4) + ((c & 7) << 1));
}
__host__ __device__ constexpr uint32_t tile_bytes(int R, int C) { return static_cast<uint32_t>(R * C * 2); }

// Split v into hi + lo 16-bit parts (hi = rn(v), lo = rn(v - hi)).
template <int kFmt>
__device__ __forceinline__ void split2(float a, float b, uint32_t &hi, uint32_t &lo) {
    if (kFmt == 0) {
        __half2 h = __floats2half2_rn(a, b);
        float2 hf = __half22float2(h);
        __half2 l = __floats2half2_rn(a - hf.x, b - hf.y);
        hi = *reinterpret_cast<uint32_t *>(&h);
        lo = *reinterpret_cast<uint32_t *>(&l);
    } else {
        __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        float2 hf = __bfloat1622float2(h);
        __nv_bfloat162 l = __floats2bfloat162_rn(a - hf.x, b - hf.y);
        hi = *reinterpret_cast<uint32_t *>(&h);
        lo = *reinterpret_cast<uint32_t *>(&l);
    }
}

// Write row r (C values, C % 8 == 0) of a tile as hi and lo parts: 16-B stores.
template <int kFmt, int C, bool kStream = false>
__device__ __forceinline__ void stage_row(uint8_t *hi_tile, uint8_t *lo_tile, int r, const float *v) {
#pragma unroll
    for (int cb = 0; cb < C; cb += 8) {
        uint4 h, l;
        split2<kFmt>(v[cb + 0], v[cb + 1], h.x, l.x);
        split2<kFmt>(v[cb + 2], v[cb + 3], h.y, l.y);
        split2<kFmt>(v[cb + 4], v[cb + 5], h.z, l.z);
        split2<kFmt>(v[cb + 6], v[cb + 7], h.w, l.w);
        const uint32_t off = tile_off(r, cb, C);
        if (kStream) {  // global destination written once, read by a later kernel
            __stcs(reinterpret_cast<uint4 *>(hi_tile + off), h);
            __stcs(reinterpret_cast<uint4 *>(lo_tile + off), l);
        } else {
            *reinterpret_cast<uint4 *>(hi_tile + off) = h;
            *reinterpret_cast<uint4 *>(lo_tile + off) = l;
        }
    }
}

// Views of a tile (byte address in shared space) as a GEMM operand.
struct Operand {
    uint32_t hi, lo;     // smem byte addresses of the hi / lo tiles
    uint32_t lbo, sbo;   // descriptor strides
    __device__ __forceinline__ uint64_t desc_hi(int kstep) const { return make_desc(hi + kstep * 2 * lbo, lbo, sbo); }
    __device__ __forceinline__ uint64_t desc_lo(int kstep) const { return make_desc(lo + kstep * 2 * lbo, lbo, sbo); }
};

// tile [rows][C] used with K = its columns (K-major)
__device__ __forceinline__ Operand kmajor(const void *hi, const void *lo, int C) {
    return Operand{smem_u32(hi), smem_u32(lo), 128u, static_cast<uint32_t>(C / 8 * 128)};
}
// tile [rows][C] used with K = its rows (MN-major, MN = columns)
__device__ __forceinline__ Operand mnmajor(const void *hi, const void *lo, int C) {
    return Operand{smem_u32(hi), smem_u32(lo), static_cast<uint32_t>(C / 8 * 128), 128u};
}
// Sub-view starting at column c0 (multiple of 8) of a tile with C columns.
__device__ __forceinline__ Operand col_offset(Operand o, int c0, bool k_major) {
    const uint32_t shift = k_major ? static_cast<uint32_t>(c0 / 8 * 128)   // along K
                                   : static_cast<uint32_t>(c0 / 8 * 128);  // along MN
    o.hi += shift;
    o.lo += shift;
    return o;
}

// D (tmem) (+)= A * B with the three-term split A_hi B_hi + A_lo B_hi + A_hi B_lo over
// nk K-steps of 16.  Issued by one thread.
__device__ __forceinline__ void gemm3(uint32_t tmem_d, const Operand &a, const Operand &b, int nk,
                                      uint32_t idesc, bool accumulate) {
    // descriptors built once; a K step only advances the 14-bit start-address field
    const uint64_t ah = make_desc(a.hi, a.lbo, a.sbo), al = make_desc(a.lo, a.lbo, a.sbo);
    const uint64_t bh = make_desc(b.hi, b.lbo, b.sbo), bl = make_desc(b.lo, b.lbo, b.sbo);
    const uint64_t sa = (2 * a.lbo) >> 4, sb = (2 * b.lbo) >> 4;
#pragma unroll 1
    for (int k = 0; k < nk; ++k) {
        const uint64_t oa = k * sa, ob = k * sb;
        mma_f16(tmem_d, ah + oa, bh + ob, idesc, (accumulate || k > 0) ? 1u : 0u);
        mma_f16(tmem_d, al + oa, bh + ob, idesc, 1u);
        mma_f16(tmem_d, ah + oa, bl + ob, idesc, 1u);
    }
}

// One K step of the 3-term split (A_hi B_hi [+acc], A_lo B_hi, A_hi B_lo) issued by the
// lane elect.sync picks: call from a converged warp.  Doing the election inside the asm
// lets ptxas emit the three UTCHMMAs back to back instead of a per-instruction
// single-thread loop.
__device__ __forceinline__ void mma3_elect(uint32_t tmem_d, uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl,
                                           uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %3, %5, p;\n\t"
        "setp.eq.b32 p, 1, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %3, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %4, %5, p;\n\t}\n" ::"r"(tmem_d),
        "l"(ah), "l"(al), "l"(bh), "l"(bl), "r"(idesc), "r"(accumulate));
}
template <int NK>
__device__ __forceinline__ void gemm3w(uint32_t tmem_d, const Operand &a, const Operand &b, uint32_t idesc,
                                       bool accumulate) {
    uint64_t ah = make_desc(a.hi, a.lbo, a.sbo), al = make_desc(a.lo, a.lbo, a.sbo);
    uint64_t bh = make_desc(b.hi, b.lbo, b.sbo), bl = make_desc(b.lo, b.lbo, b.sbo);
    const uint64_t sa = (2 * a.lbo) >> 4, sb = (2 * b.lbo) >> 4;
    mma3_elect(tmem_d, ah, al, bh, bl, idesc, accumulate ? 1u : 0u);
#pragma unroll 1
    for (int k = 1; k < NK; ++k) {  // running descriptors: four live 64-bit values
        ah += sa;
        al += sa;
        bh += sb;
        bl += sb;
        mma3_elect(tmem_d, ah, al, bh, bl, idesc, 1u);
    }
}
// Two-term split (A_hi B + A_lo B) for a B operand that is exact in fp16 (lo part zero):
// only b.hi is read.
__device__ __forceinline__ void mma2_elect(uint32_t tmem_d, uint64_t ah, uint64_t al, uint64_t bh, uint32_t idesc,
                                           uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %5, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %3, %4, p;\n\t"
        "setp.eq.b32 p, 1, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %3, %4, p;\n\t}\n" ::"r"(tmem_d),
        "l"(ah), "l"(al), "l"(bh), "r"(idesc), "r"(accumulate));
}
template <int NK>
__device__ __forceinline__ void gemm2w(uint32_t tmem_d, const Operand &a, const Operand &b, uint32_t idesc,
                                       bool accumulate) {
    uint64_t ah = make_desc(a.hi, a.lbo, a.sbo), al = make_desc(a.lo, a.lbo, a.sbo);
    uint64_t bh = make_desc(b.hi, b.lbo, b.sbo);
    const uint64_t sa = (2 * a.lbo) >> 4, sb = (2 * b.lbo) >> 4;
    mma2_elect(tmem_d, ah, al, bh, idesc, accumulate ? 1u : 0u);
#pragma unroll 1
    for (int k = 1; k < NK; ++k) {
        ah += sa;
        al += sa;
        bh += sb;
        mma2_elect(tmem_d, ah, al, bh, idesc, 1u);
    }
}

// Two-term split for an A operand that is exact in fp16 (lo part zero): A B_hi + A B_lo;
// only a.hi is read.
__device__ __forceinline__ void mma2a_elect(uint32_t tmem_d, uint64_t ah, uint64_t bh, uint64_t bl, uint32_t idesc,
                                            uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %5, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %4, p;\n\t"
        "setp.eq.b32 p, 1, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %3, %4, p;\n\t}\n" ::"r"(tmem_d),
        "l"(ah), "l"(bh), "l"(bl), "r"(idesc), "r"(accumulate));
}
template <int NK>
__device__ __forceinline__ void gemm2a(uint32_t tmem_d, const Operand &a, const Operand &b, uint32_t idesc,
                                       bool accumulate) {
    uint64_t ah = make_desc(a.hi, a.lbo, a.sbo);
    uint64_t bh = make_desc(b.hi, b.lbo, b.sbo), bl = make_desc(b.lo, b.lbo, b.sbo);
    const uint64_t sa = (2 * a.lbo) >> 4, sb = (2 * b.lbo) >> 4;
    mma2a_elect(tmem_d, ah, bh, bl, idesc, accumulate ? 1u : 0u);
#pragma unroll 1
    for (int k = 1; k < NK; ++k) {
        ah += sa;
        bh += sb;
        bl += sb;
        mma2a_elect(tmem_d, ah, bh, bl, idesc, 1u);
    }
}

// One term (A_hi B_hi): both operands taken as their fp16 hi parts.
__device__ __forceinline__ void mma1_elect(uint32_t tmem_d, uint64_t ah, uint64_t bh, uint32_t idesc,
                                           uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(ah), "l"(bh), "r"(idesc), "r"(accumulate));
}
template <int NK>
__device__ __forceinline__ void gemm1(uint32_t tmem_d, const Operand &a, const Operand &b, uint32_t idesc,
                                      bool accumulate) {
    uint64_t ah = make_desc(a.hi, a.lbo, a.sbo);
    uint64_t bh = make_desc(b.hi, b.lbo, b.sbo);
    const uint64_t sa = (2 * a.lbo) >> 4, sb = (2 * b.lbo) >> 4;
    mma1_elect(tmem_d, ah, bh, idesc, accumulate ? 1u : 0u);
#pragma unroll 1
    for (int k = 1; k < NK; ++k) {
        ah += sa;
        bh += sb;
        mma1_elect(tmem_d, ah, bh, idesc, 1u);
    }
}

// ---- A operand in tensor memory (the "TS" form): A is M x K fp16, row m in lane m, K
// elements packed two per 32-bit column (even k in the low half), K-major only.  A K step
// of 16 elements is 8 columns.  B stays a shared-memory descriptor.
__device__ __forceinline__ void tmem_st4u(uint32_t taddr, uint4 v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}
// three-term split, A from TMEM: [A_hi] B_hi + [A_lo] B_hi + [A_hi] B_lo
__device__ __forceinline__ void mma3t_elect(uint32_t tmem_d, uint32_t ah, uint32_t al, uint64_t bh, uint64_t bl,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %3, %5, p;\n\t"
        "setp.eq.b32 p, 1, 1;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %3, %5, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %4, %5, p;\n\t}\n" ::"r"(tmem_d),
        "r"(ah), "r"(al), "l"(bh), "l"(bl), "r"(idesc), "r"(accumulate));
}
template <int NK>
__device__ __forceinline__ void gemm3t(uint32_t tmem_d, uint32_t a_hi, uint32_t a_lo, const Operand &b,
                                       uint32_t idesc, bool accumulate) {
    uint64_t bh = make_desc(b.hi, b.lbo, b.sbo), bl = make_desc(b.lo, b.lbo, b.sbo);
    const uint64_t sb = (2 * b.lbo) >> 4;
    mma3t_elect(tmem_d, a_hi, a_lo, bh, bl, idesc, accumulate ? 1u : 0u);
#pragma unroll 1
    for (int k = 1; k < NK; ++k) {
        a_hi += 8;
        a_lo += 8;
        bh += sb;
        bl += sb;
        mma3t_elect(tmem_d, a_hi, a_lo, bh, bl, idesc, 1u);
    }
}

// commit by the elected lane (the one that issued the MMAs)
__device__ __forceinline__ void commit_elect(uint64_t *mbar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
            smem_u32(mbar)));
}

// Same with a compile-time K-step count: fully unrolled, so the issue loop is just the
// descriptor adds and the MMAs on the uniform datapath.
template <int NK>
__device__ __forceinline__ void gemm3u(uint32_t tmem_d, const Operand &a, const Operand &b, uint32_t idesc,
                                       bool accumulate) {
    const uint64_t ah = make_desc(a.hi, a.lbo, a.sbo), al = make_desc(a.lo, a.lbo, a.sbo);
    const uint64_t bh = make_desc(b.hi, b.lbo, b.sbo), bl = make_desc(b.lo, b.lbo, b.sbo);
    const uint64_t sa = (2 * a.lbo) >> 4, sb = (2 * b.lbo) >> 4;
#pragma unroll
    for (int k = 0; k < NK; ++k) {
        const uint64_t oa = k * sa, ob = k * sb;
        mma_f16(tmem_d, ah + oa, bh + ob, idesc, (accumulate || k > 0) ? 1u : 0u);
        mma_f16(tmem_d, al + oa, bh + ob, idesc, 1u);
        mma_f16(tmem_d, ah + oa, bl + ob, idesc, 1u);
    }
}

}  // namespace umma
}  // namespace ns2b
