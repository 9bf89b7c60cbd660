// conv_fast.cu -- the headline-shape flex_conv forward (c_in = c_out = 64, K = 8, Dp = 3)
// as a warp-specialised, channel-half-pipelined tcgen05 kernel.
//
// Same operator as tc_gmc_kernel (conv_tc.cu) -- out_p = sum_{t,c} X_p[t,c] B[t,c,:],
// X_p[t,c] = sum_s (l_p - l_{j_s})_t f_{j_s}[c] (t < 3), X_p[3,c] = sum_s f_{j_s}[c]
// (_native.pyx:52-66) -- restructured for the measured B200 costs:
//
//   * a tcgen05.mma kind::f16 with M = 128 costs ~88 cycles for any N <= 128 and ~130 at
//     N = 256 (scripts/microbench/mma_lat.cu), so the fp32-accurate split uses TWO N = 128
//     MMAs per k-step, A_hi x [B_hi; B_lo] and A_lo x [B_hi; B_lo] (D = (A_hi + A_lo)(B_hi +
//     B_lo), the two 64-column halves of D summed in the epilogue) instead of three N = 64
//     ones: 32 MMAs per 128-point tile instead of 48;
//   * index warps (4): one thread per tile row builds the 8 entries {j, l_p - l_j} of its
//     point one tile ahead into a 2-stage shared-memory ring E[stage][slot][row], so the
//     gather warps never touch indices or positions in global memory;
//   * gather warps (16): an item is 4 points x one channel HALF (32 channels = one 128-B
//     line per neighbour row), lane (pt, cl) owns 4 channels of one point; moments are
//     accumulated with packed FFMA2 in the reference's slot order and written as the UMMA
//     A operand (K-major, SW128) with a per-(point, half) power-of-two scale.  The rows of
//     the next item are loaded as soon as the current item's rows are consumed;
//   * each channel half is its own GEMM (own scale, own accumulator D[tile&1][half]), so
//     half 0 of tile i+1 is gathered while the MMAs of half 1 of tile i run: the 128 KB A
//     image is double-buffered by channel half.  A dedicated MMA warp issues them (the
//     tcgen05.mma issue blocks while the tensor pipe's queue is full, so it must not sit
//     in a gather warp);
//   * the index warps also run the epilogue (TMEM lane quadrant = warp % 4):
//     out = (D0[:, :64] + D0[:, 64:]) * s0 + (D1[:, :64] + D1[:, 64:]) * s1, 32-byte stores.
#include <cstdio>
#include <cstdlib>

#include "fast_common.cuh"

namespace fc {
using namespace sm100;

namespace fast {

constexpr int kK = 8;
constexpr int kGatherWarps = 16;
constexpr int kIdxWarp0 = 16;  // warps 16..19: index producers + epilogue (TMEM lane quadrant = warp % 4)
constexpr int kIdxWarps = 4;
constexpr int kEpiWarps = 4;
constexpr int kMmaWarp = 20;   // warp 20: TMEM owner and MMA issuer
constexpr int kWarps = 21;
constexpr int kThreads = kWarps * 32;  // <= 6 warps per SM sub-partition -> 80 registers

template <bool SPLIT>
struct FwdL {
    static constexpr int NS = SPLIT ? 2 : 1;          // A images (hi, lo)
    static constexpr int BN = SPLIT ? 128 : 64;       // B rows: [B_hi; B_lo] or B
    static constexpr int A_BYTES = kTile * 256 * 2;   // one A image: 4 K-blocks x 128 rows x 128 B
    static constexpr int B_BYTES = BN * 256 * 2;      // 4 K-blocks x BN rows x 128 B
    static constexpr int A_OFF = 0;
    static constexpr int B_OFF = A_OFF + NS * A_BYTES;
    static constexpr int E_STAGE = kK * kTile * 16;
    static constexpr int E_OFF = B_OFF + B_BYTES;
    static constexpr int RS_OFF = E_OFF + 2 * E_STAGE;  // int8 scale exponents [2 buf][2 half][128]
    static constexpr int BAR_OFF = RS_OFF + 2 * 2 * kTile;
    static constexpr int SMEM = BAR_OFF + 128;
    static constexpr int SMEM_ALLOC = SMEM + 1024;       // + base alignment slack
    static_assert(SMEM_ALLOC <= 232448, "shared memory budget");
};

struct FwdArgs {
    int64_t total, n;
    int64_t num_tiles;
    const float *feat;
    const float *loc;
    const int32_t *nbr;
    const uint8_t *bimg;
    const float *binv;
    float *out;
    // row-list mode (wide kernel): compute only the rows rows[0 .. nrows) (sorted, < total),
    // e.g. the interior rows of a shard while its halo is in flight; null = every row
    const int32_t *rows;
    int64_t nrows;
    // one 64 x 64 block of a wider conv (wide kernel): feature rows / output rows with these
    // strides, the block's product added to out (acc) -- the channel-blocked engine's passes
    int ld_feat, ld_out;  // (32-bit, as RevArgs: keeps the plain instance's register allocation)
    int acc;
    int dbg;                    // timing-probe variants (FC_DBG): 2 no MMA, 8 gather+index only, 32 CTA-0 trace
    unsigned long long *trace;  // [24 warps][kTraceN]
};

// B image for the forward: B[n][k], k = t*64 + c (theta[n', c, t], t < 3 | theta_b[n', c]),
// rows n < 64: hi (or bf16) of c' = n; rows 64..127 (split only): lo of c' = n - 64.
template <bool SPLIT>
__device__ __forceinline__ void fwd_pack_b_body(const float *__restrict__ theta, const float *__restrict__ theta_b,
                                                uint8_t *__restrict__ img, float *__restrict__ binv, int ld_cin, int bx,
                                                int gx) {
    // theta / theta_b: the 64 x 64 block's first (c', c) of a theta with ld_cin input channels;
    // (bx, gx): this CTA's slice of the image
    __shared__ float red[32];
    float m = 0.f;
#pragma unroll 4
    for (int i = threadIdx.x; i < 64 * 64 * 3; i += blockDim.x) {  // (unrolled: loads in flight)
        const int cp = i / 192, r = i % 192;
        m = fmaxf(m, fabsf(__ldg(theta + (int64_t)cp * ld_cin * 3 + r)));
    }
#pragma unroll 4
    for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) m = fmaxf(m, fabsf(__ldg(theta_b + (int64_t)(i >> 6) * ld_cin + (i & 63))));
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (threadIdx.x == 0) red[0] = m;
    }
    __syncthreads();
    int e = 0;
    if (SPLIT) e = scale_exp(red[0]);
    if (bx == 0 && threadIdx.x == 0) binv[0] = exp2i(e);
    const float sc = exp2i(-e);
    constexpr int BN = FwdL<SPLIT>::BN;
    // every block reduces the (L2-resident) max itself and packs its slice of the image
    for (int idx = bx * blockDim.x + threadIdx.x; idx < BN * 256; idx += gx * blockDim.x) {
        const int nn = idx >> 8, k = idx & 255;
        const int t = k >> 6, c = k & 63, cp = nn & 63;
        const float v = ((t < 3) ? theta[((int64_t)cp * ld_cin + c) * 3 + t] : theta_b[(int64_t)cp * ld_cin + c]) * sc;
        uint16_t bits;
        if (SPLIT) {
            const __half hh = __float2half_rn(v);
            bits = nn < 64 ? __half_as_ushort(hh) : __half_as_ushort(__float2half_rn(v - __half2float(hh)));
        } else {
            bits = __bfloat16_as_ushort(__float2bfloat16_rn(v));
        }
        *reinterpret_cast<uint16_t *>(img + sw128_offset(nn, k, BN)) = bits;
    }
}
template <bool SPLIT>
__global__ void __launch_bounds__(1024) fwd_pack_b_kernel(const float *__restrict__ theta,
                                                          const float *__restrict__ theta_b, uint8_t *__restrict__ img,
                                                          float *__restrict__ binv, int ld_cin) {
    fwd_pack_b_body<SPLIT>(theta, theta_b, img, binv, ld_cin, blockIdx.x, gridDim.x);
}
// the images of a channel-blocked forward's passes in one launch (blockIdx.y = pass): image j
// at img0 + j * stride, its 1 / scale right after the image bytes
constexpr int kFwdPackBatch = 32;
struct FwdPackJobs {
    const float *theta[kFwdPackBatch];
    const float *theta_b[kFwdPackBatch];
};
template <bool SPLIT>
__global__ void __launch_bounds__(1024) fwd_pack_b_batch_kernel(const __grid_constant__ FwdPackJobs jobs, int ld_cin,
                                                                uint8_t *__restrict__ img0, int64_t stride) {
    uint8_t *img = img0 + (int64_t)blockIdx.y * stride;
    fwd_pack_b_body<SPLIT>(jobs.theta[blockIdx.y], jobs.theta_b[blockIdx.y], img,
                           reinterpret_cast<float *>(img + FwdL<SPLIT>::B_BYTES), ld_cin, blockIdx.x, gridDim.x);
}

constexpr int kTraceN = 2048;
#define TRACE(ev, ti, tq)                                                                                  \
    do {                                                                                                   \
        if ((a.dbg & 32) && blockIdx.x == 0 && lane == 0 && ntr < kTraceN) {                               \
            long long _t;                                                                                  \
            asm volatile("mov.u64 %0, %%clock64;" : "=l"(_t)::"memory");                                  \
            a.trace[warp * kTraceN + ntr++] = ((unsigned long long)(_t - ck0) << 24) | ((unsigned)(ev) << 16) | \
                                              ((unsigned)(ti) << 4) | (unsigned)(tq);                      \
        }                                                                                                  \
    } while (0)

template <bool SPLIT>
__global__ void __launch_bounds__(kThreads, 1) tc_fwd64_kernel(FwdArgs a) {
    using L = FwdL<SPLIT>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sb = smem_u32(smem);
    const uint32_t A_hi = sb + L::A_OFF, A_lo = A_hi + L::A_BYTES;
    const uint32_t Bimg = sb + L::B_OFF;
    const uint32_t E0 = sb + L::E_OFF;
    const uint32_t rs_s = sb + L::RS_OFF;  // int8 [2 buf][2 half][128]
    const int8_t *rs = reinterpret_cast<const int8_t *>(smem + L::RS_OFF);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + L::BAR_OFF);
    uint64_t *e_full = bar + 0;                               // [2] index warps
    uint64_t *e_empty = bar + 2;                              // [2] gather warps
    uint64_t *a_full = bar + 4;                               // [2 halves] gather warps
    uint64_t *mma_done = bar + 6;                             // [2 halves] commit: A half free
    uint64_t *acc_full = bar + 8;                             // [2 bufs] commit: accumulators ready
    uint64_t *acc_free = bar + 10;                            // [2 bufs] epilogue warps
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bar + 12);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long ck0 = clock64();
    int ntr = 0;
    if (threadIdx.x == 0) {
        for (int q = 0; q < 2; ++q) {
            mbar_init(e_full + q, kIdxWarps);
            mbar_init(e_empty + q, kGatherWarps);
            mbar_init(acc_full + q, 1);
            mbar_init(acc_free + q, kEpiWarps);
            mbar_init(mma_done + q, 1);
            mbar_init(a_full + q, kGatherWarps);
        }
        fence_mbar_init();
    }
    if (warp == kMmaWarp) tmem_alloc(tmem_holder, 512);
    {  // resident B image
        const uint4 *src = reinterpret_cast<const uint4 *>(a.bimg);
        uint4 *dst = reinterpret_cast<uint4 *>(smem + L::B_OFF);
        for (int i = threadIdx.x; i < L::B_BYTES / 16; i += blockDim.x) dst[i] = src[i];  // (a cp.async fill measured 1-2 % slower here)
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const int T = a.num_tiles > blockIdx.x ? (int)ceil_div(a.num_tiles - blockIdx.x, gridDim.x) : 0;

    // MMAs of half-tile (i, h): D[i&1][h] = A_h . B_h over k = t*64 + 32h + {0, 16}, t = 0..3
    auto issue_mma = [&](int i, int h) {
        constexpr uint32_t idesc = idesc_f16(kTile, L::BN, SPLIT ? 0 : 1);
        const int b = i & 1;
        if (a.dbg & 2) {
            mbar_arrive(mma_done + h);
            if (h == 1) mbar_arrive(acc_full + b);
            return;
        }
        const uint32_t d = tmem_base + (uint32_t)((b * 2 + h) * 128);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            const int t = ks >> 1, kk = ks & 1;
            const uint32_t ko = (uint32_t)((32 * h + 16 * kk) * 2);
            const uint32_t ao = (uint32_t)t * (kTile * 128) + ko, bo = (uint32_t)t * (L::BN * 128) + ko;
            mma_f16(d, desc_sw128(A_hi + ao), desc_sw128(Bimg + bo), idesc, ks > 0 ? 1u : 0u);
            if (SPLIT) mma_f16(d, desc_sw128(A_lo + ao), desc_sw128(Bimg + bo), idesc, 1u);
        }
        mma_commit(mma_done + h);
        if (h == 1) mma_commit(acc_full + b);
    };

    if (warp == kMmaWarp) {
        // ------------------------------------------------------------ MMA issue
        if (lane == 0 && !(a.dbg & 8)) {
            for (int i = 0; i < T; ++i) {
                for (int h = 0; h < 2; ++h) {
                    mbar_wait(a_full + h, (uint32_t)(i & 1));
                    if (h == 0 && i >= 2) mbar_wait(acc_free + (i & 1), (uint32_t)(((i >> 1) + 1) & 1));
                    tc_fence_after();
                    issue_mma(i, h);
                    TRACE(4, i, h);
                }
            }
        }
        __syncwarp();
    } else if (warp >= kIdxWarp0) {
        // ------------------------------------------------------------ index producers + epilogue
        // one thread per tile row: neighbour rows of tile i+2 and positions of tile i+1 are
        // in flight before the entries of tile i+1 are stored (the stage frees when every
        // gather warp is done with tile i-1); then the epilogue of tile i-1.
        const int t = (warp - kIdxWarp0) * 32 + lane;
        const int ew = warp - kIdxWarp0;  // TMEM lane quadrant (warp % 4)
        const float binv = a.binv[0];
        auto epilogue = [&](int i) {
            if (a.dbg & 8) return;
            const int b = i & 1;
            mbar_wait_sleep(acc_full + b, (uint32_t)((i >> 1) & 1));
            TRACE(10, i, 0);
            tc_fence_after();
            const int64_t p = (blockIdx.x + (int64_t)i * gridDim.x) * kTile + t;
            const float s0 = exp2i(rs[(b * 2 + 0) * kTile + t]) * binv;
            const float s1 = exp2i(rs[(b * 2 + 1) * kTile + t]) * binv;
            const uint32_t tb = tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(b * 256);
            float *orow = a.out + p * 64;
#pragma unroll 1
            for (int c0 = 0; c0 < 64; c0 += 16) {
                float x0[16], x1[16], d[16];
                tmem_ld16(tb + (uint32_t)c0, x0);
                tmem_ld16(tb + 128u + (uint32_t)c0, x1);
                if (SPLIT) {
                    tmem_ld16(tb + 64u + (uint32_t)c0, d);
#pragma unroll
                    for (int c = 0; c < 16; ++c) x0[c] += d[c];
                    tmem_ld16(tb + 192u + (uint32_t)c0, d);
#pragma unroll
                    for (int c = 0; c < 16; ++c) x1[c] += d[c];
                }
                if (p < a.total && !(a.dbg & 64)) {
                    float o[16];
#pragma unroll
                    for (int c = 0; c < 16; ++c) o[c] = fmaf(x1[c], s1, x0[c] * s0);
                    stg256(orow + c0, o);       // full 32-byte sectors per thread
                    stg256(orow + c0 + 8, o + 8);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_free + b);
            TRACE(11, i, 0);
        };
        struct Nb {
            int32_t j[kK];
            bool v;
        };
        struct Pos {
            float c0, c1, c2;
            float q[kK][3];
        };
        auto load_nb = [&](int i, Nb &nb) {
            const int64_t p = (blockIdx.x + (int64_t)i * gridDim.x) * kTile + t;
            nb.v = p < a.total;
            int4 n0 = make_int4(0, 0, 0, 0), n1 = n0;
            int32_t base = 0;
            if (nb.v) {
                n0 = ldg_nc4i(a.nbr + p * kK);
                n1 = ldg_nc4i(a.nbr + p * kK + 4);
                if (p >= a.n) base = (int32_t)((p / a.n) * a.n);
            }
            nb.j[0] = n0.x, nb.j[1] = n0.y, nb.j[2] = n0.z, nb.j[3] = n0.w;
            nb.j[4] = n1.x, nb.j[5] = n1.y, nb.j[6] = n1.z, nb.j[7] = n1.w;
#pragma unroll
            for (int s2 = 0; s2 < kK; ++s2) nb.j[s2] = nb.v ? base + nb.j[s2] : 0;
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
            for (int s2 = 0; s2 < kK; ++s2) {
                ps.q[s2][0] = nb.v ? __ldg(a.loc + (int64_t)nb.j[s2] * 3 + 0) : 0.f;
                ps.q[s2][1] = nb.v ? __ldg(a.loc + (int64_t)nb.j[s2] * 3 + 1) : 0.f;
                ps.q[s2][2] = nb.v ? __ldg(a.loc + (int64_t)nb.j[s2] * 3 + 2) : 0.f;
            }
        };
        auto store_e = [&](int i, const Nb &nb, const Pos &ps) {
            const int st = i & 1;
            if (i >= 2) mbar_wait_sleep(e_empty + st, (uint32_t)(((i >> 1) + 1) & 1));
            TRACE(20, i, 0);
            const uint32_t es = E0 + (uint32_t)(st * L::E_STAGE);
#pragma unroll
            for (int s2 = 0; s2 < kK; ++s2)
                sts128f(es + (uint32_t)((s2 * kTile + t) * 16), __int_as_float(nb.j[s2]), ps.c0 - ps.q[s2][0],
                        ps.c1 - ps.q[s2][1], ps.c2 - ps.q[s2][2]);
            __syncwarp();
            if (lane == 0) mbar_arrive(e_full + st);
            TRACE(21, i, 0);
        };
        Nb nb_next, nb_cur;
        Pos ps;
        if (T > 0) {
            load_nb(0, nb_cur);
            load_pos(0, nb_cur, ps);
            if (T > 1) load_nb(1, nb_next);
            store_e(0, nb_cur, ps);
        }
        for (int i = 0; i < T; ++i) {
            if (i + 1 < T) {
                nb_cur = nb_next;
                load_pos(i + 1, nb_cur, ps);
                if (i + 2 < T) load_nb(i + 2, nb_next);
                store_e(i + 1, nb_cur, ps);
            }
            if (i >= 1) epilogue(i - 1);
        }
        if (T > 0) epilogue(T - 1);
    } else {
        // ------------------------------------------------------------ gather warps
        // Warp w handles items q = w and w + 16 of every half-tile (i, h).
        const int pt = lane >> 3, cl = lane & 7;
        float4 v[kK];
        auto issue_loads = [&](int i, int h, int k) {
            if (h == 0 && k == 0) mbar_wait(e_full + (i & 1), (uint32_t)((i >> 1) & 1));
            const int row = item_row(warp + 16 * k, pt);
            const uint32_t es = E0 + (uint32_t)((i & 1) * L::E_STAGE + row * 16);
            int32_t j[kK];
#pragma unroll
            for (int s2 = 0; s2 < kK; ++s2) j[s2] = lds32(es + (uint32_t)(s2 * kTile * 16));
            const float *src = a.feat + 32 * h + 4 * cl;
#pragma unroll
            for (int s2 = 0; s2 < kK; ++s2) v[s2] = ldg_nc4(src + (int64_t)j[s2] * 64);
        };
        // Hand-off of a finished half-tile to the MMA issuer: generic->async proxy fence
        // (MEMBAR.CTA + FENCE.VIEW.ASYNC, which also waits for this thread's outstanding
        // global loads), then the arrival count; the last of the 16 warps issues the MMAs.
        // Deferred to the point of the next item where its rows have landed and the
        // following rows are not yet issued, so the membar never drains the row prefetch.
        auto handoff = [&](int i, int h) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(a_full + h);
        };
        int pi = -1, ph = 0;  // half-tile whose hand-off is pending
        if (T > 0) issue_loads(0, 0, 0);
        for (int i = 0; i < T; ++i) {
            const bool tile_ok = true;
            const int64_t lim = (a.rows ? a.nrows : a.total) - ((int64_t)blockIdx.x + (int64_t)i * gridDim.x) * kTile;
#pragma unroll 1
            for (int hk = 0; hk < 4; ++hk) {
                const int h = hk >> 1, k = hk & 1;
                const int row = item_row(warp + 16 * k, pt);
                const uint32_t es = E0 + (uint32_t)((i & 1) * L::E_STAGE + row * 16);
                TRACE(1, i, hk);
                Mom4 x;
#pragma unroll
                for (int tt = 0; tt < 4; ++tt) x.m[tt][0] = x.m[tt][1] = make_float2(0.f, 0.f);
#pragma unroll
                for (int s2 = 0; s2 < kK; ++s2) {
                    const float4 e = lds128f(es + (uint32_t)(s2 * kTile * 16));
                    const float2 lo = make_float2(v[s2].x, v[s2].y), hi = make_float2(v[s2].z, v[s2].w);
                    const float2 w0 = make_float2(e.y, e.y), w1 = make_float2(e.z, e.z), w2 = make_float2(e.w, e.w);
                    x.m[0][0] = ffma2(lo, w0, x.m[0][0]);
                    x.m[0][1] = ffma2(hi, w0, x.m[0][1]);
                    x.m[1][0] = ffma2(lo, w1, x.m[1][0]);
                    x.m[1][1] = ffma2(hi, w1, x.m[1][1]);
                    x.m[2][0] = ffma2(lo, w2, x.m[2][0]);
                    x.m[2][1] = ffma2(hi, w2, x.m[2][1]);
                    x.m[3][0] = fadd2(x.m[3][0], lo);
                    x.m[3][1] = fadd2(x.m[3][1], hi);
                }
                TRACE(2, i, hk);
                if (hk == 3) {  // E(i) no longer read by this warp
                    __syncwarp();
                    if (lane == 0) mbar_arrive(e_empty + (i & 1));
                }
                if (pi >= 0 && !(a.dbg & 8)) {  // this item's rows have landed and the next ones are not issued
                    handoff(pi, ph);
                    pi = -1;
                }
                if (hk < 3) issue_loads(i, (hk + 1) >> 1, (hk + 1) & 1);
                else if (i + 1 < T) issue_loads(i + 1, 0, 0);
                // ---- per-(point, half) power-of-two scale, split, A-operand row
                int e = 0;
                float sc = 1.f;
                if (SPLIT) {
                    float m = 0.f;
#pragma unroll
                    for (int tt = 0; tt < 4; ++tt)
                        m = fmaxf(m, fmaxf(fmaxf(fabsf(x.m[tt][0].x), fabsf(x.m[tt][0].y)),
                                           fmaxf(fabsf(x.m[tt][1].x), fabsf(x.m[tt][1].y))));
                    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 4));
                    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
                    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
                    e = scale_exp(m);
                    sc = exp2i(-e);
                }
                if (!tile_ok || (int64_t)row >= lim) sc = 0.f;
                if (k == 0 && !(a.dbg & 8)) {
                    // A half h is free once the MMAs of tile i-1 half h completed; the scale
                    // slots rs[i&1] once the epilogue of tile i-2 has read them
                    if (i >= 1) mbar_wait(mma_done + h, (uint32_t)((i - 1) & 1));
                    if (h == 0 && i >= 2) mbar_wait(acc_free + (i & 1), (uint32_t)(((i >> 1) + 1) & 1));
                }
                TRACE(5, i, hk);
                // A row `row`, k = t*64 + 32h + 4cl .. +3 -> 8 bytes in 16-B chunk (4h + cl/2)
                const uint32_t rb = (uint32_t)(row >> 3) * 1024u + (uint32_t)(row & 7) * 128u +
                                    ((uint32_t)(((4 * h + (cl >> 1)) ^ (row & 7))) << 4) + (uint32_t)(cl & 1) * 8u;
#pragma unroll
                for (int tt = 0; tt < 4; ++tt) {
                    uint32_t h0, h1, l0 = 0, l1 = 0;
                    if (SPLIT) {
                        h0 = split2(x.m[tt][0], sc, l0);
                        h1 = split2(x.m[tt][1], sc, l1);
                    } else {
                        h0 = bf16x2(x.m[tt][0]);
                        h1 = bf16x2(x.m[tt][1]);
                    }
                    const uint32_t off = (uint32_t)tt * (kTile * 128) + rb;
                    sts64(A_hi + off, h0, h1);
                    if (SPLIT) sts64(A_lo + off, l0, l1);
                }
                if (cl == 0) sts8(rs_s + (uint32_t)(((i & 1) * 2 + h) * kTile + row), e);
                if (k == 1) {
                    pi = i;
                    ph = h;
                }
                TRACE(6, i, hk);
            }
        }
        if (pi >= 0 && !(a.dbg & 8)) handoff(pi, ph);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}


// =================================================================================
// Wide-lane variant: lane = 8 channels of one point (one 32-byte LDG.256 per neighbour
// slot), an item = 8 points x one channel half, 2 items per gather warp per tile.  Per
// point this halves the load, index-entry and bookkeeping instructions of the 4-channel
// lanes above.  20 warps (5 per SM sub-partition -> 96 registers): 16 gather warps and one
// control warpgroup that produces the index entries, runs the epilogue and (warp 16,
// lane 0) issues the MMAs.
// =================================================================================
constexpr int wGatherWarps = 16;
constexpr int wCtlWarp0 = 16;
constexpr int wThreads = 20 * 32;

__device__ __forceinline__ void ldg_nc8(const float *p, float (&v)[8]) {
    asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
}
__device__ __forceinline__ void sts128u(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

template <bool SPLIT, bool BLK = false>  // BLK: strided rows / out + accumulate (channel blocks)
__global__ void __launch_bounds__(wThreads, 1) tc_fwd64w_kernel(FwdArgs a) {
    using L = FwdL<SPLIT>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sb = smem_u32(smem);
    const uint32_t A_hi = sb + L::A_OFF, A_lo = A_hi + L::A_BYTES;
    const uint32_t Bimg = sb + L::B_OFF;
    const uint32_t E0 = sb + L::E_OFF;
    const uint32_t rs_s = sb + L::RS_OFF;  // int8 [2 buf][2 half][128]
    const int8_t *rs = reinterpret_cast<const int8_t *>(smem + L::RS_OFF);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + L::BAR_OFF);
    uint64_t *e_full = bar + 0;     // [2] control warps
    uint64_t *e_empty = bar + 2;    // [2] gather warps
    uint64_t *a_full = bar + 4;     // [2 halves] gather warps
    uint64_t *mma_done = bar + 6;   // [2 halves] commit: A half free
    uint64_t *acc_full = bar + 8;   // [2 bufs] commit after half 1
    uint64_t *acc_free = bar + 10;  // [2 bufs] control warps
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bar + 12);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int q = 0; q < 2; ++q) {
            mbar_init(e_full + q, 4);
            mbar_init(e_empty + q, wGatherWarps);
            mbar_init(a_full + q, wGatherWarps);
            mbar_init(mma_done + q, 1);
            mbar_init(acc_full + q, 1);
            mbar_init(acc_free + q, 4);
        }
        fence_mbar_init();
    }
    if (warp == wCtlWarp0) tmem_alloc(tmem_holder, 512);
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(a.bimg);
        uint4 *dst = reinterpret_cast<uint4 *>(smem + L::B_OFF);
        for (int i = threadIdx.x; i < L::B_BYTES / 16; i += blockDim.x) dst[i] = src[i];  // (a cp.async fill measured 1-2 % slower here)
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const int T = a.num_tiles > blockIdx.x ? (int)ceil_div(a.num_tiles - blockIdx.x, gridDim.x) : 0;
    // point of row t of tile `tile` (past the end: a.total, i.e. invalid)
    auto row_of = [&](int64_t tile, int t) -> int64_t {
        const int64_t q = tile * kTile + t;
        if (!a.rows) return q;
        return q < a.nrows ? (int64_t)__ldg(a.rows + q) : a.total;
    };

    if (warp >= wCtlWarp0) {
        // ------------------------------------------------------------ control warpgroup
        const int t = (warp - wCtlWarp0) * 32 + lane;  // tile row (index producer, epilogue)
        const int ew = warp - wCtlWarp0;               // TMEM lane quadrant
        const float binv = a.binv[0];
        auto issue_mma = [&](int i, int h) {
            constexpr uint32_t idesc = idesc_f16(kTile, L::BN, SPLIT ? 0 : 1);
            const int b = i & 1;
            mbar_wait(a_full + h, (uint32_t)(i & 1));
            if (h == 0 && i >= 2) mbar_wait(acc_free + b, (uint32_t)(((i >> 1) + 1) & 1));
            tc_fence_after();
            const uint32_t d = tmem_base + (uint32_t)((b * 2 + h) * 128);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int tt = ks >> 1, kk = ks & 1;
                const uint32_t ko = (uint32_t)((32 * h + 16 * kk) * 2);
                const uint32_t ao = (uint32_t)tt * (kTile * 128) + ko, bo = (uint32_t)tt * (L::BN * 128) + ko;
                mma_f16(d, desc_sw128(A_hi + ao), desc_sw128(Bimg + bo), idesc, ks > 0 ? 1u : 0u);
                if (SPLIT) mma_f16(d, desc_sw128(A_lo + ao), desc_sw128(Bimg + bo), idesc, 1u);
            }
            mma_commit(mma_done + h);
            if (h == 1) mma_commit(acc_full + b);
        };
        auto epilogue = [&](int i, int64_t p) {  // p: this thread's row of tile i (from produce)
            const int b = i & 1;
            mbar_wait_sleep(acc_full + b, (uint32_t)((i >> 1) & 1));
            tc_fence_after();
            const float s0 = exp2i(rs[(b * 2 + 0) * kTile + t]) * binv;
            const float s1 = exp2i(rs[(b * 2 + 1) * kTile + t]) * binv;
            const uint32_t tb = tmem_base + ((uint32_t)(ew * 32) << 16) + (uint32_t)(b * 256);
            float *orow = a.out + p * (BLK ? a.ld_out : 64);
#pragma unroll 1
            for (int c0 = 0; c0 < 64; c0 += 16) {
                float x0[16], x1[16], d[16];
                tmem_ld16(tb + (uint32_t)c0, x0);
                tmem_ld16(tb + 128u + (uint32_t)c0, x1);
                if (SPLIT) {
                    tmem_ld16(tb + 64u + (uint32_t)c0, d);
#pragma unroll
                    for (int c = 0; c < 16; ++c) x0[c] += d[c];
                    tmem_ld16(tb + 192u + (uint32_t)c0, d);
#pragma unroll
                    for (int c = 0; c < 16; ++c) x1[c] += d[c];
                }
                if (p < a.total) {
                    float o[16];
#pragma unroll
                    for (int c = 0; c < 16; ++c) o[c] = fmaf(x1[c], s1, x0[c] * s0);
                    if (BLK && a.acc) {  // block pass after the first: out += this block's product
#pragma unroll
                        for (int c = 0; c < 16; c += 4) {
                            const float4 q = *reinterpret_cast<const float4 *>(orow + c0 + c);
                            o[c] += q.x, o[c + 1] += q.y, o[c + 2] += q.z, o[c + 3] += q.w;
                        }
                    }
                    stg256(orow + c0, o);
                    stg256(orow + c0 + 8, o + 8);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_free + b);
        };
        auto produce = [&](int i, int64_t p) {  // entries of tile i (one thread per row p)
            const bool v = p < a.total;
            int4 n0 = make_int4(0, 0, 0, 0), n1 = n0;
            int32_t base = 0;
            float c0 = 0.f, c1 = 0.f, c2 = 0.f;
            if (v) {
                n0 = ldg_nc4i(a.nbr + p * kK);
                n1 = ldg_nc4i(a.nbr + p * kK + 4);
                c0 = __ldg(a.loc + p * 3 + 0);
                c1 = __ldg(a.loc + p * 3 + 1);
                c2 = __ldg(a.loc + p * 3 + 2);
                if (p >= a.n) base = (int32_t)((p / a.n) * a.n);
            }
            int32_t js[kK] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y, n1.z, n1.w};
            float q0[kK], q1[kK], q2[kK];
#pragma unroll
            for (int s2 = 0; s2 < kK; ++s2) {
                js[s2] = v ? base + js[s2] : 0;
                q0[s2] = v ? __ldg(a.loc + (int64_t)js[s2] * 3 + 0) : 0.f;
                q1[s2] = v ? __ldg(a.loc + (int64_t)js[s2] * 3 + 1) : 0.f;
                q2[s2] = v ? __ldg(a.loc + (int64_t)js[s2] * 3 + 2) : 0.f;
            }
            const int st = i & 1;
            if (i >= 2) mbar_wait_sleep(e_empty + st, (uint32_t)(((i >> 1) + 1) & 1));
            const uint32_t es = E0 + (uint32_t)(st * L::E_STAGE);
#pragma unroll
            for (int s2 = 0; s2 < kK; ++s2)
                sts128f(es + (uint32_t)((s2 * kTile + t) * 16), __int_as_float(js[s2]), c0 - q0[s2], c1 - q1[s2], c2 - q2[s2]);
            __syncwarp();
            if (lane == 0) mbar_arrive(e_full + st);
        };
        // row ids: in row-list mode a global load, issued two tiles ahead of its producer and
        // kept in registers for the epilogue (a dependent load there would sit on the path
        // that frees the accumulator; measured 2x slower forward before this)
        auto row_id = [&](int i) -> int64_t { return i < T ? row_of(blockIdx.x + (int64_t)i * gridDim.x, t) : 0; };
        int64_t pp = row_id(0), pp2 = row_id(1), pe_prev = 0, pe_cur = 0, pe_next = 0;
        if (T > 0) {
            produce(0, pp);
            pe_cur = pp;
            pp = pp2;
            pp2 = row_id(2);
        }
        for (int i = 0; i < T; ++i) {
            if (i + 1 < T) {
                produce(i + 1, pp);
                pe_next = pp;
                pp = pp2;
                pp2 = row_id(i + 3);
            }
            if (warp == wCtlWarp0) {
                if (lane == 0) issue_mma(i, 0);
                __syncwarp();
            }
            if (i >= 1) epilogue(i - 1, pe_prev);
            if (warp == wCtlWarp0) {
                if (lane == 0) issue_mma(i, 1);
                __syncwarp();
            }
            pe_prev = pe_cur;
            pe_cur = pe_next;
        }
        if (T > 0) epilogue(T - 1, pe_prev);
    } else {
        // ------------------------------------------------------------ gather warps
        // warp w: rows 8w .. 8w+7 of every tile, channel half h = 0 then 1.  Lane (pt, cl):
        // point row 8w + {0,4,1,5,2,6,3,7}[pt] (each quarter-warp's two rows store to disjoint
        // chunk sets), channels 32h + 8cl .. +7.
        const int pt = lane >> 2, cl = lane & 3;
        const int row = 8 * warp + ((pt & 1) << 2) + (pt >> 1);
        float v[4][8];
        auto load4 = [&](int i, int h, int b0) {
            const uint32_t es = E0 + (uint32_t)((i & 1) * L::E_STAGE + row * 16);
            const float *src = a.feat + 32 * h + 8 * cl;
            const int64_t ldf = BLK ? a.ld_feat : 64;
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
                const int32_t j = lds32(es + (uint32_t)((b0 + s2) * kTile * 16));
                ldg_nc8(src + (int64_t)j * ldf, v[s2]);
            }
        };
        // x[t][c]: 4 components x 8 channels as float2 pairs
        float2 x[4][4];
        auto fma4 = [&](int i, int b0) {
            const uint32_t es = E0 + (uint32_t)((i & 1) * L::E_STAGE + row * 16);
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
                const float4 e = lds128f(es + (uint32_t)((b0 + s2) * kTile * 16));
                const float2 w0 = make_float2(e.y, e.y), w1 = make_float2(e.z, e.z), w2 = make_float2(e.w, e.w);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float2 f = make_float2(v[s2][2 * c], v[s2][2 * c + 1]);
                    x[0][c] = ffma2(f, w0, x[0][c]);
                    x[1][c] = ffma2(f, w1, x[1][c]);
                    x[2][c] = ffma2(f, w2, x[2][c]);
                    x[3][c] = fadd2(x[3][c], f);
                }
            }
        };
        if (T > 0) {
            mbar_wait(e_full + 0, 0u);
            load4(0, 0, 0);
        }
        for (int i = 0; i < T; ++i) {
            const int64_t lim = (a.rows ? a.nrows : a.total) - ((int64_t)blockIdx.x + (int64_t)i * gridDim.x) * kTile;
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
#pragma unroll
                for (int tt = 0; tt < 4; ++tt)
#pragma unroll
                    for (int c = 0; c < 4; ++c) x[tt][c] = make_float2(0.f, 0.f);
                fma4(i, 0);
                load4(i, h, 4);
                fma4(i, 4);
                if (h == 1) {  // E(i) no longer read by this warp
                    __syncwarp();
                    if (lane == 0) mbar_arrive(e_empty + (i & 1));
                }
                // first batch of the next item
                if (h == 0) {
                    load4(i, 1, 0);
                } else if (i + 1 < T) {
                    mbar_wait(e_full + ((i + 1) & 1), (uint32_t)(((i + 1) >> 1) & 1));
                    load4(i + 1, 0, 0);
                }
                // ---- scale, split, A-operand row
                int e = 0;
                float sc = 1.f;
                if (SPLIT) {
                    float m = 0.f;
#pragma unroll
                    for (int tt = 0; tt < 4; ++tt)
#pragma unroll
                        for (int c = 0; c < 4; ++c) m = fmaxf(m, fmaxf(fabsf(x[tt][c].x), fabsf(x[tt][c].y)));
                    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
                    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
                    e = scale_exp(m);
                    sc = exp2i(-e);
                }
                if ((int64_t)row >= lim) sc = 0.f;
                if (i >= 1) mbar_wait(mma_done + h, (uint32_t)((i - 1) & 1));
                if (h == 0 && i >= 2) mbar_wait(acc_free + (i & 1), (uint32_t)(((i >> 1) + 1) & 1));
                // k = t*64 + 32h + 8cl .. +7: 16 bytes = chunk (4h + cl) of the row
                const uint32_t rb = (uint32_t)(row >> 3) * 1024u + (uint32_t)(row & 7) * 128u +
                                    ((uint32_t)(((4 * h + cl) ^ (row & 7))) << 4);
#pragma unroll
                for (int tt = 0; tt < 4; ++tt) {
                    uint32_t hv[4], lv[4] = {0, 0, 0, 0};
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        if (SPLIT) hv[c] = split2(x[tt][c], sc, lv[c]);
                        else hv[c] = bf16x2(x[tt][c]);
                    }
                    const uint32_t off = (uint32_t)tt * (kTile * 128) + rb;
                    sts128u(A_hi + off, hv[0], hv[1], hv[2], hv[3]);
                    if (SPLIT) sts128u(A_lo + off, lv[0], lv[1], lv[2], lv[3]);
                }
                if (cl == 0) sts8(rs_s + (uint32_t)(((i & 1) * 2 + h) * kTile + row), e);
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(a_full + h);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == wCtlWarp0) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

}  // namespace fast

// forward for c_in = c_out = 64, k = 8, d = 3 (the bench / C3 / C4 shape)
int tc_fast_forward_block(bool split, int64_t total, int64_t n, const float *feat, int64_t ld_feat, const float *loc,
                          const int32_t *nbr, const float *theta, const float *theta_b, int ld_cin, float *out,
                          int64_t ld_out, bool acc, cudaStream_t st, const int32_t *rows, int64_t nrows,
                          const uint8_t *pre_img = nullptr);

// bytes per pass image of pack_forward_blocks (image, 1 / scale, alignment)
int64_t fast_forward_image_stride(bool split) {
    using namespace fast;
    const int64_t b = split ? FwdL<true>::B_BYTES : FwdL<false>::B_BYTES;
    return (b + 256 + 1023) / 1024 * 1024;
}

// all passes' forward images of a channel-blocked forward in one launch (img0: njobs strides)
int pack_forward_blocks(bool split, int njobs, const float *const *th, const float *const *tb, int ld_cin,
                        uint8_t *img0, cudaStream_t st) {
    using namespace fast;
    const int64_t stride = fast_forward_image_stride(split);
    for (int j0 = 0; j0 < njobs; j0 += kFwdPackBatch) {
        const int nj = std::min(kFwdPackBatch, njobs - j0);
        FwdPackJobs jobs{};
        for (int j = 0; j < nj; ++j) jobs.theta[j] = th[j0 + j], jobs.theta_b[j] = tb[j0 + j];
        uint8_t *img = img0 + (int64_t)j0 * stride;
        if (split) fwd_pack_b_batch_kernel<true><<<dim3(FwdL<true>::BN * 256 / 1024, nj), 1024, 0, st>>>(jobs, ld_cin, img, stride);
        else fwd_pack_b_batch_kernel<false><<<dim3(FwdL<false>::BN * 256 / 1024, nj), 1024, 0, st>>>(jobs, ld_cin, img, stride);
        count_launch();
    }
    return check_launch("pack forward blocks");
}

int tc_fast_forward(bool split, int64_t total, int64_t n, const float *feat, const float *loc, const int32_t *nbr,
                    const float *theta, const float *theta_b, float *out, cudaStream_t st, const int32_t *rows,
                    int64_t nrows) {
    return tc_fast_forward_block(split, total, n, feat, 64, loc, nbr, theta, theta_b, 64, out, 64, false, st, rows, nrows);
}

// one 64 x 64 channel block of a wider forward (feat / out row strides ld_feat / ld_out, theta
// rows of ld_cin input channels; acc adds the block's product to out), or the whole 64 -> 64
// conv (strides 64, no acc)
int tc_fast_forward_block(bool split, int64_t total, int64_t n, const float *feat, int64_t ld_feat, const float *loc,
                          const int32_t *nbr, const float *theta, const float *theta_b, int ld_cin, float *out,
                          int64_t ld_out, bool acc, cudaStream_t st, const int32_t *rows, int64_t nrows,
                          const uint8_t *pre_img) {
    using namespace fast;
    const size_t bbytes = split ? FwdL<true>::B_BYTES : FwdL<false>::B_BYTES;
    uint8_t *img = pre_img ? const_cast<uint8_t *>(pre_img) : (uint8_t *)scratch_alloc(bbytes + 256, st);
    if (!img) return set_error(FC_ERR_CUDA, "scratch allocation failed (fast forward)");
    float *binv = reinterpret_cast<float *>(img + bbytes);
    if (!pre_img) {
        if (split) fwd_pack_b_kernel<true><<<FwdL<true>::BN * 256 / 1024, 1024, 0, st>>>(theta, theta_b, img, binv, ld_cin);
        else fwd_pack_b_kernel<false><<<FwdL<false>::BN * 256 / 1024, 1024, 0, st>>>(theta, theta_b, img, binv, ld_cin);
        count_launch();
    }
    FwdArgs a{};
    a.total = total;
    a.n = n;
    a.num_tiles = ceil_div(rows ? nrows : total, kTile);
    a.rows = rows;
    a.nrows = nrows;
    a.feat = feat;
    a.loc = loc;
    a.nbr = nbr;
    a.bimg = img;
    a.binv = binv;
    a.out = out;
    a.ld_feat = (int)ld_feat;
    a.ld_out = (int)ld_out;
    a.acc = acc ? 1 : 0;
    {
        const char *e = getenv("FC_DBG");
        a.dbg = e ? atoi(e) : 0;
    }
    const int grid = (int)std::min<int64_t>(a.num_tiles, num_sms());
    static unsigned long long *trace = nullptr;
    if (a.dbg & 32) {
        if (!trace) cudaMalloc(&trace, sizeof(unsigned long long) * kWarps * kTraceN);
        cudaMemsetAsync(trace, 0, sizeof(unsigned long long) * kWarps * kTraceN, st);
        a.trace = trace;
    }
    prof_begin("tc_forward", st);
    static int narrow = -1;
    if (narrow < 0) {
        const char *e = getenv("FC_FWD_NARROW");
        narrow = (e && e[0] == '1') ? 1 : 0;
    }
    if (narrow && (rows || ld_feat != 64 || ld_out != 64 || acc)) {
        prof_end(st);
        if (!pre_img) scratch_free(img, st);
        return set_error(FC_ERR_UNSUPPORTED, "row-list / channel-block forward needs the wide kernel");
    }
    if (a.num_tiles == 0) {
        prof_end(st);
        if (!pre_img) scratch_free(img, st);
        return FC_OK;
    }
    const bool blk = ld_feat != 64 || ld_out != 64 || acc;  // (a separate instance: the plain one keeps its registers)
    if (blk) {
        static uint64_t attr_t = 0, attr_f = 0;
        if (split) {
            if (first_use_on_device(attr_t))
                cudaFuncSetAttribute(tc_fwd64w_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdL<true>::SMEM_ALLOC);
            tc_fwd64w_kernel<true, true><<<grid, wThreads, FwdL<true>::SMEM_ALLOC, st>>>(a);
        } else {
            if (first_use_on_device(attr_f))
                cudaFuncSetAttribute(tc_fwd64w_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdL<false>::SMEM_ALLOC);
            tc_fwd64w_kernel<false, true><<<grid, wThreads, FwdL<false>::SMEM_ALLOC, st>>>(a);
        }
    } else if (!narrow) {
        if (split) {
            static uint64_t attr = 0;
            if (first_use_on_device(attr)) {
                cudaFuncSetAttribute(tc_fwd64w_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdL<true>::SMEM_ALLOC);
            }
            tc_fwd64w_kernel<true><<<grid, wThreads, FwdL<true>::SMEM_ALLOC, st>>>(a);
        } else {
            static uint64_t attr = 0;
            if (first_use_on_device(attr)) {
                cudaFuncSetAttribute(tc_fwd64w_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdL<false>::SMEM_ALLOC);
            }
            tc_fwd64w_kernel<false><<<grid, wThreads, FwdL<false>::SMEM_ALLOC, st>>>(a);
        }
    } else if (split) {
        static uint64_t attr = 0;
        if (first_use_on_device(attr)) {
            cudaFuncSetAttribute(tc_fwd64_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdL<true>::SMEM_ALLOC);
        }
        tc_fwd64_kernel<true><<<grid, kThreads, FwdL<true>::SMEM_ALLOC, st>>>(a);
    } else {
        static uint64_t attr = 0;
        if (first_use_on_device(attr)) {
            cudaFuncSetAttribute(tc_fwd64_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, FwdL<false>::SMEM_ALLOC);
        }
        tc_fwd64_kernel<false><<<grid, kThreads, FwdL<false>::SMEM_ALLOC, st>>>(a);
    }
    prof_end(st);
    count_launch();
    if (!pre_img) scratch_free(img, st);
    if (a.dbg & 32) {
        static unsigned long long h[kWarps * kTraceN];
        cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        FILE *f = fopen("gpurun_out/fwd_trace.txt", "w");
        if (f) {
            for (int w = 0; w < kWarps; ++w)
                for (int k = 0; k < kTraceN; ++k) {
                    const unsigned long long ev = h[w * kTraceN + k];
                    if (!ev) continue;
                    fprintf(f, "%d %llu %llu %llu %llu\n", w, ev >> 24, (ev >> 16) & 0xff, (ev >> 4) & 0xfff, ev & 0xf);
                }
            fclose(f);
        }
    }
    return check_launch("tc_fwd64_kernel");
}

}  // namespace fc
