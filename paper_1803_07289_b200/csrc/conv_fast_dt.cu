// conv_fast_dt.cu -- backward, forward-gather half, for the headline shape (c_in = c_out = 64,
// K = 8, Dp = 3): d_theta / d_theta_b and the centre role of d_locations.
//
//   d_theta[c', k] = sum_p g_p[c'] X_p[k]    (k = t*64 + c; _native.pyx:106-112)
//   Z_t[p, c']    = sum_c Xb_p[c] theta[c', c, t],  centre[p, t] = sum_c' g_p[c'] Z_t[p, c']
//                                               (the +dt terms of _native.pyx:121-127)
// Warp-specialised like conv_fast.cu:
//   * index warps (16..19): the forward neighbourhood's entries {j, l_p - l_j}, one tile
//     ahead, in a 2-stage shared-memory ring (identical to the forward kernel's producer);
//   * gather warps (0..15): a 16-point CHUNK is gathered by all 16 warps at once, one point
//     per warp (lane = 2 channels, one 256-byte neighbour row per warp load), so chunks
//     complete one after another and a 2-stage chunk ring suffices.  Each point's moment
//     row X_p (tf32 hi/lo, MN-major, 2 KB) and upstream row g_p (tf32 hi/lo) go to the
//     chunk, its bias moments Xb_p (fp16 hi/lo, per-row power-of-two scale) to the Z tile;
//   * MMA issue (warp 20, lane 0), strictly in chunk order (bitwise reproducible): per 8
//     points two kind::tf32 MMAs [G_hi; G_lo]^T . X_hi / X_lo with M = 128, N = 256 into a
//     CTA-resident accumulator (~130 cycles each, scripts/microbench/mma_lat.cu), and per
//     tile Z = Xb . [theta_0; theta_1; theta_2] as one N = 192 operand (3 fp16 MMAs per
//     k-step);
//   * Z epilogue (warps 20..23, TMEM lane quadrant = warp % 4) in 8 column slices
//     interleaved with the next tile's chunk MMAs; the d_theta accumulator is drained once
//     at the end as two per-CTA partial slices (hi / lo lanes), reduced in fixed order.
#include <cstdio>
#include <cstdlib>

#include "fast_common.cuh"

namespace fc {
using namespace sm100;

namespace fast {

constexpr int dGatherWarps = 16;
constexpr int dIdxWarp0 = 16;
constexpr int dIdxWarps = 4;
constexpr int dEpiWarp0 = 20;  // Z epilogue (+ warp 20 lane 0: MMA issue, TMEM owner)
constexpr int dEpiWarps = 4;
constexpr int dWarps = 24;
constexpr int dThreads = dWarps * 32;
constexpr int dChunk = 16;     // points per chunk (= gather warps)
constexpr int dK = 8;
// d_theta accumulation segment: tiles (128 points, 16 tf32 k-steps each) accumulated in TMEM
// before the index warps drain the accumulator (precision: see dt_drain)
constexpr int kSegTiles = 8;
// register split (setmaxnreg): control warps (index, epilogue) give registers to the gather
// warps, which hold a point's 8 rows and their offsets across the load latency;
// 8 x 32 x kCtlRegs + 16 x 32 x kGatherRegs <= 768 x 80 (the launch allocation)
constexpr int kCtlRegs = 64;
constexpr int kGatherRegs = 88;

struct DtL {
    static constexpr int XST = dChunk * 256 * 4;       // one tf32 X chunk image (16 KB)
    static constexpr int GST = dChunk * 64 * 4;        // one tf32 G chunk image (4 KB)
    static constexpr int STAGE = 2 * XST + 2 * GST;    // X_hi, X_lo, G_hi, G_lo (40 KB)
    static constexpr int XB = kTile * 64 * 2;          // fp16 bias-moment tile (16 KB)
    static constexpr int BZ = 64 * 128;                // one K-block of the forward image (8 KB)
    static constexpr int C_OFF = 0;                    // [2 stages]
    static constexpr int XB_OFF = C_OFF + 2 * STAGE;   // [2 bufs][hi, lo]
    static constexpr int BZ_OFF = XB_OFF + 2 * 2 * XB; // [hi K-blocks 0..2][lo K-blocks 0..2]
    static constexpr int E_STAGE = dK * kTile * 16;
    static constexpr int E_OFF = BZ_OFF + 2 * 3 * BZ;
    static constexpr int RS_OFF = E_OFF + 2 * E_STAGE;  // int8 [3 buf][128] (by tile % 3)
    static constexpr int BAR_OFF = RS_OFF + 3 * kTile;
    static constexpr int SMEM = BAR_OFF + 128;
    static constexpr int SMEM_ALLOC = SMEM + 1024;
    static_assert(SMEM_ALLOC <= 232448, "shared memory budget");
};

struct DtArgs2 {
    int64_t total, n;
    int64_t num_tiles;
    const float *feat, *loc, *g;
    const int32_t *nbr;
    const uint8_t *bimg;  // forward fp16 image (hi, lo); K-blocks 0..2 used
    const float *binv;
    float *partial;       // [gridDim.x][128 lanes][256 columns]: TMEM-native (c' hi | c' lo) x (t, c), zeroed
    float *centre;        // [total, 3]
    int dbg;                    // FC_DBG & 8: per-role wait-cycle counters
    unsigned long long *clk;    // [grid][24][4]
};

// per-role wait-cycle counters (FC_DBG & 8) exist only in builds with -DFC_DT_CLOCKS: the
// counters live across the hot loops and, in the register-capped roles, were spilled to local
// memory around every ring wait (measured: +0.4 ms per 7M-point call)
#ifdef FC_DT_CLOCKS
#define DT_CLK(slot, stmt)                                                  \
    do {                                                                    \
        long long _c0, _c1;                                                 \
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(_c0)::"memory");      \
        stmt;                                                               \
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(_c1)::"memory");      \
        ck[slot] += _c1 - _c0;                                              \
    } while (0)
#else
#define DT_CLK(slot, stmt) \
    do {                   \
        stmt;              \
    } while (0)
#endif

// tf32 hi part by truncation (the low 13 mantissa bits cleared); lo = x - hi is exact and
// carries the remaining 13 bits (read by the MMA as tf32: 2^-21 relative overall)
__device__ __forceinline__ uint32_t tf32_hi(float x) { return __float_as_uint(x) & 0xffffe000u; }
// byte offset of MN element mn in K-row r of an SW128_BASE32B MN-major image (16 K-rows per
// MN block of 32 elements): MN blocks 2 KB apart, 4-row K groups 512 B apart
__device__ __forceinline__ uint32_t mn32(int mn, int r) {
    return (uint32_t)((mn >> 5) * 2048 + (r >> 2) * 512 + (r & 3) * 128 + ((((mn & 31) >> 3) ^ (r & 3)) << 5) + (mn & 7) * 4);
}
__device__ __forceinline__ uint64_t desc_mn32(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
    d |= (uint64_t)((2048 >> 4) & 0x3FFF) << 16;  // LBO: MN blocks
    d |= (uint64_t)((512 >> 4) & 0x3FFF) << 32;   // SBO: 4-row K groups
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)1 << 61;  // SWIZZLE_128B_BASE32B
    return d;
}
__device__ __forceinline__ void mma_tf32_mn(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(
            d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void red_add_v4(float *p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
// Drain of a d_theta accumulation segment: add the 256 TMEM columns of this thread's lane into
// its CTA partial row with fp32 reductions at L2 (one thread per address, segments in order:
// deterministic).  Why segments: the tensor pipe's fp32 accumulation truncates -- measured
// on the B200, the d_theta error grows linearly with the number of accumulated k-steps and is
// biased toward zero (2.9e-5 at 886 steps, 1M points; scripts/dtheta_precision.py) -- so no
// accumulator runs longer than kSegTiles tiles (128 k-steps, ~5e-6).
__device__ __noinline__ void dt_drain(uint32_t taddr, float *part_row) {
#pragma unroll 1
    for (int n0 = 0; n0 < 256; n0 += 16) {
        float v[16];
        tmem_ld16(taddr + (uint32_t)n0, v);
#pragma unroll
        for (int q = 0; q < 16; q += 4) red_add_v4(part_row + n0 + q, v[q], v[q + 1], v[q + 2], v[q + 3]);
    }
}
// Segment drain of the c' hi rows (the rows whose accumulator is large): add the lane's 256
// columns into its partial row and zero them in TMEM, so the MMAs continue (accumulate = 1)
// from zero on these rows while the c' lo rows (2^-11 smaller, their truncation negligible)
// keep accumulating until the final drain.
__device__ __noinline__ void dt_drain_zero(uint32_t taddr, float *part_row) {
#pragma unroll 1
    for (int n0 = 0; n0 < 256; n0 += 16) {
        float v[16];
        tmem_ld16(taddr + (uint32_t)n0, v);
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                taddr + (uint32_t)n0),
            "r"(0u)
            : "memory");
#pragma unroll
        for (int q = 0; q < 16; q += 4) red_add_v4(part_row + n0 + q, v[q], v[q + 1], v[q + 2], v[q + 3]);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void named_bar_dt(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void sts64u(uint32_t addr, uint32_t a, uint32_t b) {
    asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void sts32u(uint32_t addr, uint32_t a) {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(a) : "memory");
}
__device__ __forceinline__ void ldg_nc8f(const float *p, float (&v)[8]) {
    asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
}
__device__ __forceinline__ float2 ldg_nc2(const float *p) {
    float2 v;
    asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return v;
}

__global__ void __launch_bounds__(dThreads, 1) tc_dt64_kernel(DtArgs2 a) {
    using L = DtL;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sb = smem_u32(smem);
    const uint32_t C0 = sb + L::C_OFF, XB0 = sb + L::XB_OFF, BZ0 = sb + L::BZ_OFF, E0 = sb + L::E_OFF;
    const uint32_t rs_s = sb + L::RS_OFF;
    const int8_t *rs = reinterpret_cast<const int8_t *>(smem + L::RS_OFF);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + L::BAR_OFF);
    uint64_t *e_full = bar + 0;       // [2] index warps
    uint64_t *e_empty = bar + 2;      // [2] gather warps
    uint64_t *c_full = bar + 4;       // [2] chunk stage written (gather warps)
    uint64_t *c_empty = bar + 6;      // [2] commit: chunk stage consumed
    uint64_t *z_done = bar + 8;       // commit: Z accumulator ready
    uint64_t *z_free = bar + 9;       // [2 by tile parity] epilogue warps: Z drained, rs read
    uint64_t *xb_free = bar + 11;     // [2] commit: Xb buffer consumed (Z MMAs of its tile done)
    uint64_t *dt_done = bar + 13;     // commit: d_theta accumulator final
    uint64_t *dt_seg = bar + 14;      // commit: a d_theta accumulation segment complete
    uint64_t *seg_drained = bar + 15; // index warps: the segment has been read out of TMEM
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bar + 16);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef FC_DT_CLOCKS
    long long ck[4] = {0, 0, 0, 0};
    long long ck_t0;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(ck_t0)::"memory");
#endif
    if (threadIdx.x == 0) {
        for (int q = 0; q < 2; ++q) {
            mbar_init(e_full + q, dIdxWarps);
            mbar_init(e_empty + q, dGatherWarps);
            mbar_init(c_full + q, dGatherWarps);
            mbar_init(c_empty + q, 1);
            mbar_init(xb_free + q, 1);
            mbar_init(z_free + q, dEpiWarps);
        }
        mbar_init(z_done, 1);
        mbar_init(dt_done, 1);
        mbar_init(dt_seg, 1);
        mbar_init(seg_drained, 2);
        fence_mbar_init();
    }
    if (warp == dEpiWarp0) tmem_alloc(tmem_holder, 512);
    {  // K-blocks 0..2 of the forward image (hi, then lo) -> resident B for Z
        const int img_b = 64 * 4 * 64 * 2;  // one full forward image
        for (int h = 0; h < 2; ++h) {
            const uint4 *src = reinterpret_cast<const uint4 *>(a.bimg + h * img_b);
            uint4 *dst = reinterpret_cast<uint4 *>(smem + L::BZ_OFF + h * 3 * L::BZ);
            smem_fill16(dst, src, 3 * L::BZ / 16);
        }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const int T = a.num_tiles > blockIdx.x ? (int)ceil_div(a.num_tiles - blockIdx.x, gridDim.x) : 0;

    if (warp >= dEpiWarp0) {
        // ------------------------------------------------------------ MMA issue + Z epilogue
        setmaxnreg_dec<kCtlRegs>();
        // TMEM: d_theta D columns 0..255 (lanes: c' hi 0..63, c' lo 64..127), Z 256..447
        const int ew = warp - dEpiWarp0;
        const int row = ew * 32 + lane;
        const float binv = a.binv[0];
        constexpr uint32_t idt = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(256 >> 3) << 17) |
                                 ((uint32_t)(kTile >> 4) << 24);
        constexpr uint32_t idz = idesc_f16(kTile, 192, 0);
        float c0 = 0.f, c1 = 0.f, c2 = 0.f;
        int64_t pz = 0;
        float inv = 1.f;
        // slice s of the Z epilogue of tile i: c' in [8s, 8s+8) for t = 0..2 (TMEM columns
        // 256 + 64t + 8s .. +7), g[p, 8s .. 8s+7] from global (L2)
        auto zslice = [&](int i, int s) {
            if (s == 0) {
                DT_CLK(1, mbar_wait_sleep(z_done, (uint32_t)(i & 1)));
                tc_fence_after();
                pz = (blockIdx.x + (int64_t)i * gridDim.x) * kTile + row;
                inv = exp2i(rs[(i % 3) * kTile + row]) * binv;
                c0 = c1 = c2 = 0.f;
            }
            const uint32_t tb = tmem_base + ((uint32_t)(ew * 32) << 16) + 256u + (uint32_t)(8 * s);
            float z0[8], z1[8], z2[8];
            tmem_ld8(tb, z0);
            tmem_ld8(tb + 64u, z1);
            tmem_ld8(tb + 128u, z2);
            float gv[8];
            if (pz < a.total) {
                ldg_nc8f(a.g + pz * 64 + 8 * s, gv);  // own row: one 32-byte load (one line touch)
            } else {
#pragma unroll
                for (int q = 0; q < 8; ++q) gv[q] = 0.f;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                c0 = fmaf(gv[q], z0[q], c0);
                c1 = fmaf(gv[q], z1[q], c1);
                c2 = fmaf(gv[q], z2[q], c2);
            }
            if (s == 7) {
                if (pz < a.total) {
                    a.centre[pz * 3 + 0] = c0 * inv;
                    a.centre[pz * 3 + 1] = c1 * inv;
                    a.centre[pz * 3 + 2] = c2 * inv;
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(z_free + (i & 1));
            }
        };
        // d_theta segments (see dt_drain_zero): every kSegTiles tiles (staggered by CTA) the
        // first MMA of a tile waits until index warps 16-17 have drained and zeroed the c' hi rows.
        for (int i = 0; i < T; ++i) {
            for (int c = 0; c < kTile / dChunk; ++c) {
                if (warp == dEpiWarp0) {
                    if (lane == 0) {
                        const int u = i * (kTile / dChunk) + c, st = u & 1;
                        // segment boundaries staggered by CTA (the drains' L2 reductions spread in time)
                        const int sg = i + (int)(blockIdx.x & (kSegTiles - 1));
                        if (c == 0 && i > 0 && (sg & (kSegTiles - 1)) == 0)
                            DT_CLK(0, mbar_wait(seg_drained, (uint32_t)(((sg / kSegTiles) - 1) & 1)));
                        DT_CLK(0, mbar_wait(c_full + st, (uint32_t)((u >> 1) & 1)));
                        tc_fence_after();
                        const uint32_t cs = C0 + (uint32_t)(st * L::STAGE);
                        const uint32_t xh = cs, xl = cs + L::XST, gh = cs + 2 * L::XST;
#pragma unroll
                        for (int ks = 0; ks < dChunk / 8; ++ks) {
                            const uint32_t ko = (uint32_t)(ks * 1024);
                            mma_tf32_mn(tmem_base, desc_mn32(gh + ko), desc_mn32(xh + ko), idt, (u == 0 && ks == 0) ? 0u : 1u);
                            mma_tf32_mn(tmem_base, desc_mn32(gh + ko), desc_mn32(xl + ko), idt, 1u);
                        }
                        mma_commit(c_empty + st);
                    }
                    __syncwarp();
                }
                if (i >= 1) zslice(i - 1, c);
            }
            // Z of tile i: single TMEM buffer, free once the epilogue of tile i-1 drained it
            if (warp == dEpiWarp0) {
                if (lane == 0) {
                    if (i >= 1) DT_CLK(2, mbar_wait(z_free + ((i - 1) & 1), (uint32_t)(((i - 1) >> 1) & 1)));
                    tc_fence_after();
                    const uint32_t ah = XB0 + (uint32_t)((i & 1) * 2 * L::XB), al = ah + L::XB;
                    const uint32_t bh = BZ0, bl = BZ0 + 3 * L::BZ;
                    const uint32_t z = tmem_base + 256u;
#pragma unroll
                    for (int s = 0; s < 4; ++s) {
                        const uint32_t o = (uint32_t)(s * 32);
                        mma_f16(z, desc_sw128(ah + o), desc_sw128(bh + o), idz, s > 0 ? 1u : 0u);
                        mma_f16(z, desc_sw128(ah + o), desc_sw128(bl + o), idz, 1u);
                        mma_f16(z, desc_sw128(al + o), desc_sw128(bh + o), idz, 1u);
                    }
                    mma_commit(z_done);
                    mma_commit(xb_free + (i & 1));
                    if (i == T - 1) mma_commit(dt_done);
                    else if (((i + 1 + (int)(blockIdx.x & (kSegTiles - 1))) & (kSegTiles - 1)) == 0) mma_commit(dt_seg);
                }
                __syncwarp();
            }
        }
        for (int s = 0; s < 8 && T > 0; ++s) zslice(T - 1, s);
        // ---- drain the d_theta accumulator: lane m = c' (hi part) or 64 + c' (lo part)
        if (T > 0) {
            mbar_wait(dt_done, 0);
            tc_fence_after();
        }
        if (T > 0) dt_drain(tmem_base + ((uint32_t)(ew * 32) << 16), a.partial + ((int64_t)blockIdx.x * 128 + row) * 256);
    } else if (warp >= dIdxWarp0) {
        // ------------------------------------------------------------ index producers
        setmaxnreg_dec<kCtlRegs>();
        const int t = (warp - dIdxWarp0) * 32 + lane;
        struct Nb {
            int32_t j[dK];
            bool v;
        };
        struct Pos {
            float c0, c1, c2;
            float q[dK][3];
        };
        auto load_nb = [&](int i, Nb &nb) {
            const int64_t p = (blockIdx.x + (int64_t)i * gridDim.x) * kTile + t;
            nb.v = p < a.total;
            int4 n0 = make_int4(0, 0, 0, 0), n1 = n0;
            int32_t base = 0;
            if (nb.v) {
                n0 = ldg_nc4i(a.nbr + p * dK);
                n1 = ldg_nc4i(a.nbr + p * dK + 4);
                if (p >= a.n) base = (int32_t)((p / a.n) * a.n);
            }
            nb.j[0] = n0.x, nb.j[1] = n0.y, nb.j[2] = n0.z, nb.j[3] = n0.w;
            nb.j[4] = n1.x, nb.j[5] = n1.y, nb.j[6] = n1.z, nb.j[7] = n1.w;
#pragma unroll
            for (int s2 = 0; s2 < dK; ++s2) nb.j[s2] = nb.v ? base + nb.j[s2] : 0;
        };
        auto load_pos = [&](int i, const Nb &nb, Pos &ps) {
            const int64_t p = (blockIdx.x + (int64_t)i * gridDim.x) * kTile + t;
            ps.c0 = ps.c1 = ps.c2 = 0.f;
            if (nb.v) {
                ps.c0 = __ldg(a.loc + p * 3 + 0);
                ps.c1 = __ldg(a.loc + p * 3 + 1);
                ps.c2 = __ldg(a.loc + p * 3 + 2);
            }
#pragma unroll
            for (int s2 = 0; s2 < dK; ++s2) {
                ps.q[s2][0] = nb.v ? __ldg(a.loc + (int64_t)nb.j[s2] * 3 + 0) : 0.f;
                ps.q[s2][1] = nb.v ? __ldg(a.loc + (int64_t)nb.j[s2] * 3 + 1) : 0.f;
                ps.q[s2][2] = nb.v ? __ldg(a.loc + (int64_t)nb.j[s2] * 3 + 2) : 0.f;
            }
        };
        auto store_e = [&](int i, const Nb &nb, const Pos &ps) {
            const int st = i & 1;
            if (i >= 2) mbar_wait_sleep(e_empty + st, (uint32_t)(((i >> 1) + 1) & 1));
            const uint32_t es = E0 + (uint32_t)(st * L::E_STAGE);
#pragma unroll
            for (int s2 = 0; s2 < dK; ++s2)
                sts128f(es + (uint32_t)((s2 * kTile + t) * 16), __int_as_float(nb.j[s2]), ps.c0 - ps.q[s2][0],
                        ps.c1 - ps.q[s2][1], ps.c2 - ps.q[s2][2]);
            __syncwarp();
            if (lane == 0) mbar_arrive(e_full + st);
        };
        Nb nb_next, nb_cur;
        Pos ps;
        if (T > 0) {
            load_nb(0, nb_cur);
            load_pos(0, nb_cur, ps);
            if (T > 1) load_nb(1, nb_next);
            store_e(0, nb_cur, ps);
        }
        for (int i = 0; i + 1 < T; ++i) {
            nb_cur = nb_next;
            load_pos(i + 1, nb_cur, ps);
            if (i + 2 < T) load_nb(i + 2, nb_next);
            store_e(i + 1, nb_cur, ps);
            const int sg = i + 1 + (int)(blockIdx.x & (kSegTiles - 1));
            if ((sg & (kSegTiles - 1)) == 0 && warp < dIdxWarp0 + 2) {
                // a d_theta segment is complete: the two warps on TMEM lane quadrants 0, 1 (the
                // c' hi rows) drain and zero them, then release the accumulator
                mbar_wait(dt_seg, (uint32_t)(((sg / kSegTiles) - 1) & 1));
                tc_fence_after();
                dt_drain_zero(tmem_base + ((uint32_t)(t & ~31) << 16), a.partial + ((int64_t)blockIdx.x * 128 + t) * 256);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(seg_drained);
            }
        }
    } else {
        // ------------------------------------------------------------ gather warps
        // chunk c of tile i: warp w owns point 16c + w (tile row); lane owns channels 2L, 2L+1
        setmaxnreg_inc<kGatherRegs>();
        const int cc = 2 * lane;
        const float *fsrc = a.feat + cc;
        float2 v[dK];
        float dx[dK], dy[dK], dz[dK];  // offsets l_p - l_j of the rows in v
        float2 gn;  // upstream row of the point whose rows are in v
        auto issue_loads = [&](int i, int c) {
            if (c == 0) DT_CLK(0, mbar_wait(e_full + (i & 1), (uint32_t)((i >> 1) & 1)));
            const int row = dChunk * c + warp;
            const int64_t p = (blockIdx.x + (int64_t)i * gridDim.x) * kTile + row;
            const uint32_t es = E0 + (uint32_t)((i & 1) * L::E_STAGE + row * 16);
            int32_t j[dK];
#pragma unroll
            for (int s2 = 0; s2 < dK; ++s2) {
                const float4 e = lds128f(es + (uint32_t)(s2 * kTile * 16));
                j[s2] = __float_as_int(e.x);
                dx[s2] = e.y, dy[s2] = e.z, dz[s2] = e.w;
            }
#pragma unroll
            for (int s2 = 0; s2 < dK; ++s2) v[s2] = ldg_nc2(fsrc + (int64_t)j[s2] * 64);
            gn = p < a.total ? ldg_nc2(a.g + p * 64 + cc) : make_float2(0.f, 0.f);
        };
        // The hand-off of a chunk stage (proxy fence = MEMBAR.CTA, which waits for all of the
        // thread's outstanding loads, + arrival) is deferred to the next chunk, at the point
        // where that chunk's rows have landed and the following rows are not yet issued.
        int pend = -1;
        auto handoff = [&]() {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(c_full + pend);
            pend = -1;
        };
        if (T > 0) issue_loads(0, 0);
        for (int i = 0; i < T; ++i) {
            const int64_t tile0 = (blockIdx.x + (int64_t)i * gridDim.x) * kTile;
#pragma unroll 1
            for (int c = 0; c < kTile / dChunk; ++c) {
                const int row = dChunk * c + warp;
                const int64_t p = tile0 + row;
                const bool pv = p < a.total;
                // moments: m[t] = (channel 2L, 2L+1) of component t
                float2 m0 = make_float2(0.f, 0.f), m1 = m0, m2 = m0, m3 = m0;
#pragma unroll
                for (int s2 = 0; s2 < dK; ++s2) {
                    m0 = ffma2(v[s2], make_float2(dx[s2], dx[s2]), m0);
                    m1 = ffma2(v[s2], make_float2(dy[s2], dy[s2]), m1);
                    m2 = ffma2(v[s2], make_float2(dz[s2], dz[s2]), m2);
                    m3 = fadd2(m3, v[s2]);
                }
                const float2 gv = gn;
                if (c == kTile / dChunk - 1) {  // E(i) no longer read by this warp
                    __syncwarp();
                    if (lane == 0) mbar_arrive(e_empty + (i & 1));
                }
                if (pend >= 0) handoff();
                if (c + 1 < kTile / dChunk) issue_loads(i, c + 1);
                else if (i + 1 < T) issue_loads(i + 1, 0);
                if (!pv) m0 = m1 = m2 = m3 = make_float2(0.f, 0.f);
                // ---- Xb row (fp16 hi/lo, per-row scale) -> Z tile row `row`
                // row max of |Xb|: non-negative floats order like their bit patterns -> one REDUX
                const float mx = __uint_as_float(
                    __reduce_max_sync(0xffffffffu, __float_as_uint(fmaxf(fabsf(m3.x), fabsf(m3.y)))));
                const int e = scale_exp(mx);
                if (c == 0 && i >= 2) {  // Xb buffer / rs slot of tile i-2 consumed (Z MMAs done, epilogue read rs)
                    DT_CLK(1, mbar_wait(xb_free + (i & 1), (uint32_t)(((i >> 1) + 1) & 1)));
                    // (no wait for the Z epilogue of tile i-2: the row scales it reads are
                    // triple-buffered by tile % 3, and the Xb buffer is released by xb_free)
                }
                {
                    uint32_t lo;
                    const uint32_t hi = split2(m3, exp2i(-e), lo);
                    const uint32_t xo = XB0 + (uint32_t)((i & 1) * 2 * L::XB) + sw128_offset(row, cc, kTile);
                    sts32u(xo, hi);
                    sts32u(xo + L::XB, lo);
                    if (lane == 0) sts8(rs_s + (uint32_t)((i % 3) * kTile + row), e);
                }
                // ---- X row (tf32 hi/lo) and G row into chunk stage u & 1
                const int u = i * (kTile / dChunk) + c, st = u & 1;
                if (u >= 2) DT_CLK(2, mbar_wait(c_empty + st, (uint32_t)(((u >> 1) + 1) & 1)));
                const uint32_t cs = C0 + (uint32_t)(st * L::STAGE);
                const float2 mm[4] = {m0, m1, m2, m3};
#pragma unroll
                for (int tt = 0; tt < 4; ++tt) {
                    const uint32_t off = mn32(tt * 64 + cc, warp);
                    const uint32_t h0 = tf32_hi(mm[tt].x), h1 = tf32_hi(mm[tt].y);
                    sts64u(cs + off, h0, h1);
                    sts64u(cs + L::XST + off, __float_as_uint(mm[tt].x - __uint_as_float(h0)),
                           __float_as_uint(mm[tt].y - __uint_as_float(h1)));
                }
                {
                    const uint32_t off = mn32(cc, warp);
                    const uint32_t h0 = tf32_hi(gv.x), h1 = tf32_hi(gv.y);
                    sts64u(cs + 2 * L::XST + off, h0, h1);
                    sts64u(cs + 2 * L::XST + L::GST + off, __float_as_uint(gv.x - __uint_as_float(h0)),
                           __float_as_uint(gv.y - __uint_as_float(h1)));
                }
                pend = st;
            }
        }
        if (pend >= 0) handoff();
    }
#ifdef FC_DT_CLOCKS
    if ((a.dbg & 8) && lane == 0) {
        long long t1;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1)::"memory");
        unsigned long long *o = a.clk + ((int64_t)blockIdx.x * 24 + warp) * 4;
        o[0] = ck[0], o[1] = ck[1], o[2] = ck[2], o[3] = t1 - ck_t0;
    }
#endif
    tc_fence_before();
    __syncthreads();
    if (warp == dEpiWarp0) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

}  // namespace fast

void launch_pack_b(bool split, int cin, int cout, const float *theta, const float *theta_b, int reverse, int nout,
                   int gc, uint8_t *img, float *binv, cudaStream_t st);
template <typename T>
int launch_dtheta_reduce(int chunks, int cin, int d, int cout, const T *partial, T *d_theta, T *d_theta_b,
                         cudaStream_t st, int tmajor = 0, int ld = 0);

// d_theta / d_theta_b (reduced in fixed order) and the centre role of d_locations for
// c_in = c_out = 64, k = 8, d = 3; centre may be null when d_locations is not wanted
int tc_fast_dtheta(int64_t total, int64_t n, const float *feat, const float *loc, const int32_t *nbr, const float *g,
                   const float *theta, const float *theta_b, float *d_theta, float *d_theta_b, float *centre,
                   cudaStream_t st) {
    using namespace fast;
    const size_t img_bytes = (size_t)64 * 4 * 64 * 2 * 2;
    const int64_t num_tiles = ceil_div(total, kTile);
    const int grid = (int)std::min<int64_t>(num_tiles, num_sms());
    uint8_t *img = (uint8_t *)scratch_alloc(img_bytes + 256, st);
    float *partial = (float *)scratch_alloc(sizeof(float) * 2 * grid * 64 * 64 * 4, st);
    if (partial) cudaMemsetAsync(partial, 0, sizeof(float) * 2 * grid * 64 * 64 * 4, st);
    float *cscratch = centre ? nullptr : (float *)scratch_alloc(sizeof(float) * total * 3, st);
    if (!img || !partial || (!centre && !cscratch)) return set_error(FC_ERR_CUDA, "scratch allocation failed (fast dtheta)");
    float *binv = reinterpret_cast<float *>(img + img_bytes);
    launch_pack_b(true, 64, 64, theta, theta_b, 0, 64, 64, img, binv, st);
    DtArgs2 a{};
    a.total = total;
    a.n = n;
    a.num_tiles = num_tiles;
    a.feat = feat;
    a.loc = loc;
    a.g = g;
    a.nbr = nbr;
    a.bimg = img;
    a.binv = binv;
    a.partial = partial;
    a.centre = centre ? centre : cscratch;
    {
        const char *e = getenv("FC_DBG");
        a.dbg = e ? atoi(e) : 0;
    }
    static unsigned long long *clk = nullptr;
    if (a.dbg & 8) {
        if (!clk) cudaMalloc(&clk, sizeof(unsigned long long) * 148 * 24 * 4);
        a.clk = clk;
    }
    static uint64_t attr = 0;
    if (first_use_on_device(attr)) {
        cudaFuncSetAttribute(tc_dt64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, DtL::SMEM_ALLOC);
    }
    prof_begin("tc_dtheta", st);
    tc_dt64_kernel<<<grid, dThreads, DtL::SMEM_ALLOC, st>>>(a);
    prof_end(st);
    count_launch();
    int rc = check_launch("tc_dt64_kernel");
    if (a.dbg & 8) {
        static unsigned long long h[148 * 24 * 4];
        cudaMemcpyAsync(h, clk, sizeof(unsigned long long) * grid * 24 * 4, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        const char *nm[3] = {"gather (e_full, xb/z_free, c_empty)", "index (-)", "mma/epi (c_full, z_done, z_free)"};
        for (int r = 0; r < 3; ++r) {
            const int w0 = r == 0 ? 0 : (r == 1 ? dIdxWarp0 : dEpiWarp0), w1 = r == 0 ? 16 : w0 + 4;
            for (int w = w0; w < w1; w += (r == 2 ? 1 : w1 - w0)) {
                double acc[4] = {};
                const int we = r == 2 ? w + 1 : w1;
                for (int b = 0; b < grid; ++b)
                    for (int ww = w; ww < we; ++ww)
                        for (int k = 0; k < 4; ++k) acc[k] += (double)h[((size_t)b * 24 + ww) * 4 + k] / (grid * (we - w));
                fprintf(stderr, "%s w%d: total %.0f  waits %.1f%% %.1f%% %.1f%%\n", nm[r], w, acc[3], 100 * acc[0] / acc[3],
                        100 * acc[1] / acc[3], 100 * acc[2] / acc[3]);
            }
        }
    }
    // per CTA: rows c' hi (64) then c' lo (64) = two partial slices in the t-major column order
    if (!rc && (d_theta || d_theta_b))
        rc = launch_dtheta_reduce<float>(2 * grid, 64, 3, 64, partial, d_theta, d_theta_b, st, 1);
    scratch_free(img, st);
    scratch_free(partial, st);
    scratch_free(cscratch, st);
    return rc;
}

}  // namespace fc
