// conv_tc.cu -- tcgen05 tensor-core flex-convolution: fused gather -> moments ->
// contraction, one persistent warp-specialised CTA per SM.
//
// Per tile of 128 centre points (UMMA M = 128):
//   gather warps (16): coalesced neighbour-row loads -- a lane group of GC/4 lanes owns
//     one point (float4 = 4 channels per lane), so a warp loads 2 (GC = 64) or 4 (GC = 32)
//     neighbour rows per instruction -- and the moments
//       X_p[t, c] = sum_s (l_p - l_j)_t f_j[c]  (t < 3),   X_p[3, c] = sum_s f_j[c]
//     accumulated in fp32 (packed FFMA2) in the reference's slot order
//     (_native.pyx:52-59), written to shared memory as the UMMA A operand (K-major,
//     128-byte swizzle, k = t*GC + c).  Index / position loads of the next group are
//     issued before the current group is accumulated (software pipelining).
//   MMA warp (1 elected thread): D[p, n] (+)= sum_k A[p, k] * B[n, k] into TMEM,
//     B = [theta; theta_b] resident in shared memory for the whole kernel.
//   epilogue warps (4): tcgen05.ld the accumulator rows, undo the operand scaling, store.
// Engines:
//   SPLIT (fp32-accurate): every fp32 operand v is scaled by a power of two s (per point
//     row for A, per tensor for B) so that max|v*s| is in [2^14, 2^15), and split into
//     fp16 hi = rn(v*s), lo = rn(v*s - hi): 22 significant bits, i.e. fp32-level accuracy
//     (the product hi*hi + hi*lo + lo*hi drops lo*lo ~ 2^-22 relative).  3 MMAs per k-step.
//   BF16: single bf16 MMA per k-step (stated 1e-2 relative tolerance).
// REVERSE = the same kernel over the reverse neighbourhood (d_features of the backward
// and flex_deconv): Y_j = sum_{(i,s) in R(j)} (l_i - l_j, 1) (x) g_i, out = Y_j . B_rev.
#include "fc_common.cuh"
#include "sm100.cuh"

namespace fc {
using namespace sm100;

constexpr int kTcM = 128;          // tile rows (points)
// 16 warps, all gather / moments producers; warps 0..3 also drain the accumulator (TMEM
// lane quadrants 0..3) and warp 15 also allocates TMEM and issues the MMAs.  16 warps =
// 4 per SM sub-partition -> up to 128 registers per thread.
constexpr int kGatherWarps = 16;
constexpr int kEpiWarps = 4;
constexpr int kMmaWarp = kGatherWarps - 1;
constexpr int kTcThreads = kGatherWarps * 32;
constexpr int kSlots = 8;          // neighbour slots per point per batch

struct TcArgs {
    int64_t total;  // points (B*N)
    int64_t n;      // points per cloud
    int k;          // forward neighbourhood size (slot divisor for reverse entries)
    const float *rows;
    const float *loc;
    const int32_t *nbr;
    Csr csr;
    const uint8_t *bimg;  // B operand image (hi [, lo]) in the exact smem layout
    const float *binv;    // 1 / (B scale)
    float *out;
    int64_t num_tiles;
};

template <bool SPLIT>
__device__ __forceinline__ uint16_t pack1(float a, uint16_t &lo_out) {
    if constexpr (SPLIT) {
        const __half ha = __float2half_rn(a);
        lo_out = __half_as_ushort(__float2half_rn(a - __half2float(ha)));
        return __half_as_ushort(ha);
    } else {
        lo_out = 0;
        return __bfloat16_as_ushort(__float2bfloat16_rn(a));
    }
}

// power-of-two scale putting max|v| into [2^14, 2^15); returns the scale, writes 1/scale
__device__ __forceinline__ float split_scale(float m, float &inv) {
    if (!(m > 0.f) || !isfinite(m)) {
        inv = 1.f;
        return 1.f;
    }
    int e = ilogbf(m);
    e = max(-100, min(100, e));
    inv = ldexpf(1.f, e - 14);
    return ldexpf(1.f, 14 - e);
}

template <int GC, int NOUT, bool SPLIT>
struct TcLayout {
    static constexpr int KT = 4 * GC;                      // K = (Dp + 1) * GC, Dp = 3
    static constexpr int A_BYTES = kTcM * KT * 2;          // one 16-bit A image
    static constexpr int B_BYTES = NOUT * KT * 2;          // one 16-bit B image
    static constexpr int NSPLIT = SPLIT ? 2 : 1;
    static constexpr int A_OFF = 0;
    static constexpr int B_OFF = A_OFF + A_BYTES * NSPLIT;
    static constexpr int RS_OFF = B_OFF + B_BYTES * NSPLIT;  // float rs[2][128]
    static constexpr int BAR_OFF = RS_OFF + 2 * kTcM * 4;    // 5 x uint64 + tmem holder
    static constexpr int SMEM = BAR_OFF + 64 + 1024;         // + alignment slack
    static constexpr int TMEM_COLS = (2 * NOUT <= 32) ? 32 : (2 * NOUT <= 64) ? 64 : (2 * NOUT <= 128) ? 128 : 256;
};

// ---------------------------------------------------------------------------------
// B image: B[n][k] = theta[c', c, t] (t < 3) | theta_b[c', c] (t == 3), k = t*GC + c.
//   forward: n = c' (rows = c_out), c = input channel   (GC = c_in)
//   reverse: n = c  (rows = c_in),  c' = gathered chan  (GC = c_out)
template <bool SPLIT>
__global__ void __launch_bounds__(1024)
    tc_pack_b_kernel(int cin, int cout, const float *__restrict__ theta, const float *__restrict__ theta_b,
                     int reverse, int nout, int gc, uint8_t *__restrict__ img, float *__restrict__ binv) {
    __shared__ float red[32];
    float m = 0.f;
    const int nth = cout * cin * 3, ntb = cout * cin;
    for (int i = threadIdx.x; i < nth; i += blockDim.x) m = fmaxf(m, fabsf(theta[i]));
    for (int i = threadIdx.x; i < ntb; i += blockDim.x) m = fmaxf(m, fabsf(theta_b[i]));
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (threadIdx.x == 0) red[0] = m;
    }
    __syncthreads();
    float inv = 1.f, s = 1.f;
    if (SPLIT) s = split_scale(red[0], inv);
    if (threadIdx.x == 0) binv[0] = inv;
    const int KT = 4 * gc;
    const int bbytes = nout * KT * 2;
    for (int idx = threadIdx.x; idx < nout * KT; idx += blockDim.x) {
        const int nn = idx / KT, k = idx % KT;
        const int t = k / gc, c = k % gc;
        const int cp = reverse ? c : nn;
        const int ci = reverse ? nn : c;
        const float v = (t < 3) ? theta[((int64_t)cp * cin + ci) * 3 + t] : theta_b[(int64_t)cp * cin + ci];
        uint16_t lo;
        const uint16_t hi = pack1<SPLIT>(v * s, lo);
        const uint32_t off = sw128_offset(nn, k, nout);
        *reinterpret_cast<uint16_t *>(img + off) = hi;
        if (SPLIT) *reinterpret_cast<uint16_t *>(img + bbytes + off) = lo;
    }
}

// ---------------------------------------------------------------------------------
// packed fp32x2 arithmetic (sm_100 FFMA2 / FADD2 / FMUL2): two independent IEEE
// operations per instruction, identical results to two scalar fmaf / add / mul.
__device__ __forceinline__ uint64_t as_u64(float2 a) { return *reinterpret_cast<uint64_t *>(&a); }
__device__ __forceinline__ float2 as_f2(uint64_t d) { return *reinterpret_cast<float2 *>(&d); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(as_u64(a)), "l"(as_u64(b)), "l"(as_u64(c)));
    return as_f2(d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(as_u64(a)), "l"(as_u64(b)));
    return as_f2(d);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(as_u64(a)), "l"(as_u64(b)));
    return as_f2(d);
}

__device__ __forceinline__ void sts64(uint32_t addr, uint32_t lo, uint32_t hi) {
    asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(lo), "r"(hi) : "memory");
}

// split (scaled fp16 hi + lo) or bf16 pack of a pair
template <bool SPLIT>
__device__ __forceinline__ uint32_t cvt_pair(float2 x, uint32_t &lo) {
    if constexpr (SPLIT) {
        const __half2 h = __floats2half2_rn(x.x, x.y);
        const float2 hb = __half22float2(h);
        const __half2 l = __floats2half2_rn(x.x - hb.x, x.y - hb.y);
        lo = *reinterpret_cast<const uint32_t *>(&l);
        return *reinterpret_cast<const uint32_t *>(&h);
    } else {
        lo = 0;
        const __nv_bfloat162 h = __floats2bfloat162_rn(x.x, x.y);
        return *reinterpret_cast<const uint32_t *>(&h);
    }
}

// Lane geometry: a group of LPR = GC/4 lanes owns one point (4 channels per lane);
// a warp covers PPI = 32/LPR points per "group".  Index work for a group is done by
// lane (ipt, slot) = (lane >> 3, lane & 7), ipt < PPI.
template <int GC>
struct Geo {
    static constexpr int LPR = GC / 4;
    static constexpr int PPI = 32 / LPR;
    static constexpr int GROUPS = kTcM / PPI;                // per tile
    static constexpr int GPW = GROUPS / kGatherWarps;        // per warp per tile
    static_assert(GC == 32 || GC == 64, "GC must be 32 or 64");
    static_assert(GPW * kGatherWarps == GROUPS, "groups must divide evenly");
};

// One point's moments held by one lane: m[t] = channels (4cl .. 4cl+3) at component t.
struct Mom {
    float2 m[4][2];
};

__device__ __forceinline__ void mom_zero(Mom &a) {
#pragma unroll
    for (int t = 0; t < 4; ++t) a.m[t][0] = a.m[t][1] = make_float2(0.f, 0.f);
}

__device__ __forceinline__ void mom_add(Mom &a, const float4 &v, float w0, float w1, float w2) {
    const float2 lo = make_float2(v.x, v.y), hi = make_float2(v.z, v.w);
    a.m[0][0] = ffma2(lo, make_float2(w0, w0), a.m[0][0]);
    a.m[0][1] = ffma2(hi, make_float2(w0, w0), a.m[0][1]);
    a.m[1][0] = ffma2(lo, make_float2(w1, w1), a.m[1][0]);
    a.m[1][1] = ffma2(hi, make_float2(w1, w1), a.m[1][1]);
    a.m[2][0] = ffma2(lo, make_float2(w2, w2), a.m[2][0]);
    a.m[2][1] = ffma2(hi, make_float2(w2, w2), a.m[2][1]);
    a.m[3][0] = fadd2(a.m[3][0], lo);
    a.m[3][1] = fadd2(a.m[3][1], hi);
}

// Write one point's (scaled) moments as A-operand row `row` (k = t*GC + c): the lane's
// 4 channels are 4 consecutive fp16 of K-block (t*GC)/64 -> one 8-byte store per t.
template <int GC, bool SPLIT>
__device__ __forceinline__ void store_row(uint32_t a_hi, uint32_t a_lo, int row, int cl, const Mom &x,
                                          float sc) {
    constexpr uint32_t KBLK = kTcM * 128;
    const uint32_t rbase = (uint32_t)(row >> 3) * 1024u + (uint32_t)(row & 7) * 128u;
    const float2 s2 = make_float2(sc, sc);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int k = t * GC + 4 * cl;
        const int kb = k >> 6, kin = k & 63;
        const uint32_t off = (uint32_t)kb * KBLK + rbase + ((uint32_t)((kin >> 3) ^ (row & 7)) << 4) +
                             (uint32_t)(kin & 7) * 2u;
        uint32_t l0, l1;
        const uint32_t h0 = cvt_pair<SPLIT>(fmul2(x.m[t][0], s2), l0);
        const uint32_t h1 = cvt_pair<SPLIT>(fmul2(x.m[t][1], s2), l1);
        sts64(a_hi + off, h0, h1);
        if (SPLIT) sts64(a_lo + off, l0, l1);
    }
}

__device__ __forceinline__ float group_absmax(const Mom &x, int lpr) {
    float v = 0.f;
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int h = 0; h < 2; ++h) v = fmaxf(v, fmaxf(fabsf(x.m[t][h].x), fabsf(x.m[t][h].y)));
    for (int o = lpr >> 1; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Index state of one neighbour slot (held by index lane (ipt, slot)).
struct Idx {
    int32_t j;             // global neighbour / source point index (0 when invalid)
    float o0, o1, o2;      // offset components
};

// ---------------------------------------------------------------------------------
template <int GC, int NOUT, bool SPLIT, bool REVERSE, int KFIX>
__global__ void __launch_bounds__(kTcThreads, 1) tc_gmc_kernel(TcArgs a) {
    using L = TcLayout<GC, NOUT, SPLIT>;
    using G = Geo<GC>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t *A_hi = smem + L::A_OFF;
    uint8_t *A_lo = A_hi + L::A_BYTES;
    uint8_t *B_hi = smem + L::B_OFF;
    uint8_t *B_lo = B_hi + L::B_BYTES;
    float *rs = reinterpret_cast<float *>(smem + L::RS_OFF);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + L::BAR_OFF);
    uint64_t *full = bar + 0;
    uint64_t *mma_done = bar + 1;  // [2]
    uint64_t *d_free = bar + 3;    // [2]
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bar + 5);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        mbar_init(full, kGatherWarps);
        mbar_init(mma_done + 0, 1);
        mbar_init(mma_done + 1, 1);
        mbar_init(d_free + 0, kEpiWarps);
        mbar_init(d_free + 1, kEpiWarps);
        fence_mbar_init();
    }
    if (warp == kMmaWarp) tmem_alloc(tmem_holder, L::TMEM_COLS);
    {  // resident B operand image(s)
        const uint4 *src = reinterpret_cast<const uint4 *>(a.bimg);
        uint4 *dst = reinterpret_cast<uint4 *>(B_hi);
        const int nvec = L::B_BYTES * L::NSPLIT / 16;
        for (int i = threadIdx.x; i < nvec; i += blockDim.x) dst[i] = src[i];
    }
    const float binv = a.binv[0];
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    // ---------------------------------------------------------------- MMA issue (warp kMmaWarp, lane 0)
    // tile i: wait until every gather warp wrote A (full) and the epilogue of tile i-2 freed
    // accumulator buffer i&1, then issue the K loop and commit to mma_done[i&1].
    auto issue_mma = [&](int i) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_f16(kTcM, NOUT, SPLIT ? 0 : 1);
            const uint32_t a_hi = smem_u32(A_hi), a_lo = smem_u32(A_lo);
            const uint32_t b_hi = smem_u32(B_hi), b_lo = smem_u32(B_lo);
            mbar_wait(full, i & 1);
            if (i >= 2) mbar_wait(d_free + (i & 1), ((i >> 1) + 1) & 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + (uint32_t)((i & 1) * NOUT);
#pragma unroll
            for (int s = 0; s < L::KT / 16; ++s) {
                const uint32_t aoff = (uint32_t)((s >> 2) * kTcM * 128 + (s & 3) * 32);
                const uint32_t boff = (uint32_t)((s >> 2) * NOUT * 128 + (s & 3) * 32);
                mma_f16(d_tmem, desc_sw128(a_hi + aoff), desc_sw128(b_hi + boff), idesc, s > 0 ? 1u : 0u);
                if (SPLIT) {
                    mma_f16(d_tmem, desc_sw128(a_hi + aoff), desc_sw128(b_lo + boff), idesc, 1u);
                    mma_f16(d_tmem, desc_sw128(a_lo + aoff), desc_sw128(b_hi + boff), idesc, 1u);
                }
            }
            mma_commit(mma_done + (i & 1));
        }
        __syncwarp();
    };
    // ---------------------------------------------------------------- epilogue (warps 0..3)
    // warp q owns TMEM lanes / tile rows 32q .. 32q+31; one thread per output row.
    auto epilogue = [&](int i) {
        const int64_t tile = blockIdx.x + (int64_t)i * gridDim.x;
        const int row = warp * 32 + lane;
        mbar_wait(mma_done + (i & 1), (i >> 1) & 1);
        tc_fence_after();
        const int64_t p = tile * kTcM + row;
        const float inv = rs[(i & 1) * kTcM + row];
        float *orow = a.out + p * NOUT;
#pragma unroll
        for (int c0 = 0; c0 < NOUT; c0 += 16) {
            float v[16];
            tmem_ld16(tmem_base + ((uint32_t)(warp * 32) << 16) + (uint32_t)((i & 1) * NOUT + c0), v);
            if (p < a.total) {
#pragma unroll
                for (int q = 0; q < 16; q += 4) {
                    float4 w = make_float4(v[q] * inv, v[q + 1] * inv, v[q + 2] * inv, v[q + 3] * inv);
                    *reinterpret_cast<float4 *>(orow + c0 + q) = w;
                }
            }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(d_free + (i & 1));
    };

    {
        // ------------------------------------------------------------ gather producers (all warps)
        const int gw = warp;
        const uint32_t a_hi_u = smem_u32(A_hi), a_lo_u = smem_u32(A_lo);
        const int pt = lane / G::LPR, cl = lane % G::LPR;  // accumulation role
        const int ipt = lane >> 3, slot = lane & 7;         // index-work role
        const int64_t tiles_mine = a.num_tiles > blockIdx.x ? ceil_div(a.num_tiles - blockIdx.x, gridDim.x) : 0;
        const int64_t items = tiles_mine * G::GPW;
        auto item_p0 = [&](int64_t w) -> int64_t {
            const int64_t tile = blockIdx.x + (w / G::GPW) * gridDim.x;
            const int grp = gw + (int)(w % G::GPW) * kGatherWarps;
            return tile * kTcM + (int64_t)grp * G::PPI;
        };
        // index lanes: issue the loads describing slot `b0 + slot` of point p0 + ipt
        auto idx_load = [&](int64_t p0, int b0, Idx &x, int &cnt) {
            const int64_t myp = p0 + ipt;
            x.j = 0;
            x.o0 = x.o1 = x.o2 = 0.f;
            cnt = 0;
            if (ipt < G::PPI && myp < a.total) {
                int64_t q0;
                if (REVERSE) {
                    q0 = a.csr.off[myp];
                    cnt = a.csr.off[myp + 1] - (int)q0;
                } else {
                    q0 = myp * (KFIX ? KFIX : a.k);
                    cnt = KFIX ? KFIX : a.k;
                }
                if (b0 + slot < cnt) {
                    const float lp0 = a.loc[myp * 3 + 0], lp1 = a.loc[myp * 3 + 1], lp2 = a.loc[myp * 3 + 2];
                    if (REVERSE) {
                        x.j = a.csr.ent[q0 + b0 + slot] / a.k;
                    } else {
                        x.j = (int32_t)((myp / a.n) * a.n) + a.nbr[q0 + b0 + slot];
                    }
                    const float l0 = a.loc[(int64_t)x.j * 3 + 0], l1 = a.loc[(int64_t)x.j * 3 + 1],
                                l2 = a.loc[(int64_t)x.j * 3 + 2];
                    if (REVERSE) {
                        x.o0 = l0 - lp0;
                        x.o1 = l1 - lp1;
                        x.o2 = l2 - lp2;
                    } else {
                        x.o0 = lp0 - l0;
                        x.o1 = lp1 - l1;
                        x.o2 = lp2 - l2;
                    }
                }
            }
        };
        // one batch of 8 slots: all row loads first, then the slot-ordered accumulation
        auto batch_load = [&](const Idx &x, int mycnt_b, float4 (&v)[kSlots]) {
#pragma unroll
            for (int s = 0; s < kSlots; ++s) {
                const int32_t jj = __shfl_sync(0xffffffffu, x.j, pt * 8 + s);
                v[s] = (KFIX || s < mycnt_b)
                           ? __ldg(reinterpret_cast<const float4 *>(a.rows + (int64_t)jj * GC) + cl)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        };
        auto batch_acc = [&](const Idx &x, int mycnt_b, const float4 (&v)[kSlots], Mom &acc) {
#pragma unroll
            for (int s = 0; s < kSlots; ++s) {
                const float w0 = __shfl_sync(0xffffffffu, x.o0, pt * 8 + s);
                const float w1 = __shfl_sync(0xffffffffu, x.o1, pt * 8 + s);
                const float w2 = __shfl_sync(0xffffffffu, x.o2, pt * 8 + s);
                if (KFIX || s < mycnt_b) mom_add(acc, v[s], w0, w1, w2);
            }
        };
        auto batch = [&](const Idx &x, int mycnt_b, Mom &acc) {
            float4 v[kSlots];
            batch_load(x, mycnt_b, v);
            batch_acc(x, mycnt_b, v, acc);
        };
        auto finish = [&](int64_t w, int64_t p0, const Mom &acc) {
            const int i = (int)(w / G::GPW);
            if (w % G::GPW == 0) {
                // the previous tile's MMA must have consumed A (and the epilogue two tiles
                // back must have read rs[i & 1]) before this tile's first shared-memory write
                if (i >= 1) mbar_wait(mma_done + ((i - 1) & 1), ((i - 1) >> 1) & 1);
                if (i >= 2) mbar_wait(d_free + (i & 1), ((i >> 1) + 1) & 1);
            }
            const int row = (int)(p0 - (blockIdx.x + (int64_t)i * gridDim.x) * kTcM) + pt;
            float inv = 1.f, sc = 1.f;
            if (SPLIT) sc = split_scale(group_absmax(acc, G::LPR), inv);
            if (p0 + pt >= a.total) sc = 0.f;
            store_row<GC, SPLIT>(a_hi_u, a_lo_u, row, cl, acc, sc);
            if (cl == 0) rs[(i & 1) * kTcM + row] = inv * binv;
            if (w % G::GPW == G::GPW - 1) {
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(full);
                // tile i is complete for this warp: drain the previous tile's accumulator
                // (warps 0..3) / issue this tile's MMAs (warp kMmaWarp)
                if (warp < kEpiWarps && i >= 1) epilogue(i - 1);
                if (warp == kMmaWarp) issue_mma(i);
            }
        };

        if (KFIX == kSlots && !REVERSE) {
            // fixed k = 8: one batch per group; the next group's index/position loads are
            // in flight while the current group's rows are loaded and accumulated
            // index lane state of the NEXT group, split into stages so that no load result
            // is consumed before the current group's rows are in flight
            // Three-deep software pipeline over this warp's groups g:
            //   raw index + centre position of g+2 issued during g,
            //   neighbour position of g+1 issued (and its rows prefetched to L2) during g,
            //   rows of g loaded and accumulated during g.
            // (the loaded values are only consumed one iteration later)
            struct Raw {
                int32_t nb, base;  // cloud-local neighbour index, cloud base
                float l0, l1, l2;
                bool v;
                __device__ int32_t j() const { return base + nb; }
            };
            auto raw_load = [&](int64_t w) {
                Raw r{0, 0, 0.f, 0.f, 0.f, false};
                if (w < items) {
                    const int64_t myp = item_p0(w) + ipt;
                    r.v = ipt < G::PPI && myp < a.total;
                    if (r.v) {
                        r.base = myp < a.n ? 0 : (int32_t)((myp / a.n) * a.n);
                        r.nb = __ldg(a.nbr + myp * kSlots + slot);
                        r.l0 = __ldg(a.loc + myp * 3 + 0);
                        r.l1 = __ldg(a.loc + myp * 3 + 1);
                        r.l2 = __ldg(a.loc + myp * 3 + 2);
                    }
                }
                return r;
            };
            Idx cur;
            int cdummy;
            if (items > 0) idx_load(item_p0(0), 0, cur, cdummy);
            Raw r1 = raw_load(1);
            for (int64_t w = 0; w < items; ++w) {
                const int64_t p0 = item_p0(w);
                float4 v[kSlots];
                batch_load(cur, kSlots, v);
                // g+1: neighbour positions, and its rows into L2
                const int32_t j1 = r1.j();
                float nl0 = 0.f, nl1 = 0.f, nl2 = 0.f;
                if (r1.v) {
                    nl0 = __ldg(a.loc + (int64_t)j1 * 3 + 0);
                    nl1 = __ldg(a.loc + (int64_t)j1 * 3 + 1);
                    nl2 = __ldg(a.loc + (int64_t)j1 * 3 + 2);
                    const float *rp = a.rows + (int64_t)j1 * GC;
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(rp));
                    if (GC * 4 > 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + 32));
                }
                // g+2: raw indices
                const Raw r2 = raw_load(w + 2);
                Mom acc;
                mom_zero(acc);
                batch_acc(cur, kSlots, v, acc);
                finish(w, p0, acc);
                // offsets of g+1
                cur.j = j1;
                cur.o0 = r1.v ? r1.l0 - nl0 : 0.f;
                cur.o1 = r1.v ? r1.l1 - nl1 : 0.f;
                cur.o2 = r1.v ? r1.l2 - nl2 : 0.f;
                r1 = r2;
            }
        } else {
            for (int64_t w = 0; w < items; ++w) {
                const int64_t p0 = item_p0(w);
                Mom acc;
                mom_zero(acc);
                Idx x;
                int cnt;
                idx_load(p0, 0, x, cnt);
                const int mycnt = __shfl_sync(0xffffffffu, cnt, pt * 8);
                int maxcnt = cnt;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) maxcnt = max(maxcnt, __shfl_xor_sync(0xffffffffu, maxcnt, o));
                for (int b0 = 0; b0 < maxcnt; b0 += kSlots) {
                    if (b0 > 0) idx_load(p0, b0, x, cnt);
                    batch(x, mycnt - b0, acc);
                }
                finish(w, p0, acc);
            }
        }
        if (warp < kEpiWarps && tiles_mine > 0) epilogue((int)tiles_mine - 1);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
        tc_fence_after();
        tmem_dealloc(tmem_base, L::TMEM_COLS);
    }
}

// ---------------------------------------------------------------------------------
// host side
template <int GC, int NOUT, bool SPLIT, bool REVERSE, int KFIX>
static int launch_tc(const TcArgs &a0, int cin, int cout, const float *theta, const float *theta_b,
                     cudaStream_t st) {
    using L = TcLayout<GC, NOUT, SPLIT>;
    TcArgs a = a0;
    uint8_t *img = (uint8_t *)scratch_alloc((size_t)L::B_BYTES * L::NSPLIT + 256, st);
    if (!img) return set_error(FC_ERR_CUDA, "scratch allocation failed (tc)");
    float *binv = reinterpret_cast<float *>(img + (size_t)L::B_BYTES * L::NSPLIT);
    tc_pack_b_kernel<SPLIT><<<1, 1024, 0, st>>>(cin, cout, theta, theta_b, REVERSE ? 1 : 0, NOUT, GC, img, binv);
    count_launch();
    a.bimg = img;
    a.binv = binv;
    a.num_tiles = ceil_div(a.total, kTcM);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(tc_gmc_kernel<GC, NOUT, SPLIT, REVERSE, KFIX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             L::SMEM);
        attr = true;
    }
    const int grid = (int)std::min<int64_t>(a.num_tiles, num_sms());
    tc_gmc_kernel<GC, NOUT, SPLIT, REVERSE, KFIX><<<grid, kTcThreads, L::SMEM, st>>>(a);
    count_launch();
    scratch_free(img, st);
    return check_launch("tc_gmc_kernel");
}

template <int GC, int NOUT, bool SPLIT, bool REVERSE>
static int launch_tc_k(const TcArgs &a, int cin, int cout, const float *theta, const float *theta_b,
                       cudaStream_t st) {
    if (!REVERSE && a.k == kSlots) return launch_tc<GC, NOUT, SPLIT, REVERSE, kSlots>(a, cin, cout, theta, theta_b, st);
    return launch_tc<GC, NOUT, SPLIT, REVERSE, 0>(a, cin, cout, theta, theta_b, st);
}

template <bool SPLIT, bool REVERSE>
static int dispatch_tc(int gc, int nout, const TcArgs &a, int cin, int cout, const float *theta,
                       const float *theta_b, cudaStream_t st) {
    if (gc == 64 && nout == 64) return launch_tc_k<64, 64, SPLIT, REVERSE>(a, cin, cout, theta, theta_b, st);
    if (gc == 64 && nout == 32) return launch_tc_k<64, 32, SPLIT, REVERSE>(a, cin, cout, theta, theta_b, st);
    if (gc == 32 && nout == 32) return launch_tc_k<32, 32, SPLIT, REVERSE>(a, cin, cout, theta, theta_b, st);
    if (gc == 32 && nout == 64) return launch_tc_k<32, 64, SPLIT, REVERSE>(a, cin, cout, theta, theta_b, st);
    if (gc == 32 && nout == 128) return launch_tc_k<32, 128, SPLIT, REVERSE>(a, cin, cout, theta, theta_b, st);
    if (!SPLIT && gc == 64 && nout == 128) return launch_tc_k<64, 128, false, REVERSE>(a, cin, cout, theta, theta_b, st);
    return set_error(FC_ERR_UNSUPPORTED, "no tensor-core instance for gathered=%d out=%d", gc, nout);
}

static bool tc_shape_ok(int mode, int gc, int d, int nout) {
    if (d != 3) return false;
    const bool split = mode != FC_MODE_TC_BF16;
    if (gc == 64 && (nout == 64 || nout == 32)) return true;
    if (gc == 32 && (nout == 32 || nout == 64 || nout == 128)) return true;
    if (!split && gc == 64 && nout == 128) return true;
    return false;
}

int tc_conv_forward_supported(int mode, int c_in, int d, int k, int c_out) {
    (void)k;
    return tc_shape_ok(mode, c_in, d, c_out) ? 1 : 0;
}

int tc_conv_forward(int mode, int64_t total, int64_t n, int c_in, int d, int k, int c_out, const float *feat,
                    const float *loc, const int32_t *nbr, const float *theta, const float *theta_b, float *out,
                    cudaStream_t st) {
    (void)d;
    TcArgs a{};
    a.total = total;
    a.n = n;
    a.k = k;
    a.rows = feat;
    a.loc = loc;
    a.nbr = nbr;
    a.out = out;
    if (mode == FC_MODE_TC_BF16) return dispatch_tc<false, false>(c_in, c_out, a, c_in, c_out, theta, theta_b, st);
    return dispatch_tc<true, false>(c_in, c_out, a, c_in, c_out, theta, theta_b, st);
}

int tc_reverse_supported(int mode, int gc, int d, int cout) { return tc_shape_ok(mode, gc, d, cout) ? 1 : 0; }

int tc_reverse_gmc(int mode, int64_t total, int64_t n, int gc, int d, int k, int cout, const float *rows,
                   const float *loc, Csr csr, const float *theta, const float *theta_b, float *out,
                   cudaStream_t st) {
    (void)d;
    TcArgs a{};
    a.total = total;
    a.n = n;
    a.k = k;
    a.rows = rows;
    a.loc = loc;
    a.csr = csr;
    a.out = out;
    // conv shapes: c_in = cout (output of this pass), c_out = gc (gathered rows)
    if (mode == FC_MODE_TC_BF16) return dispatch_tc<false, true>(gc, cout, a, cout, gc, theta, theta_b, st);
    return dispatch_tc<true, true>(gc, cout, a, cout, gc, theta, theta_b, st);
}

}  // namespace fc
