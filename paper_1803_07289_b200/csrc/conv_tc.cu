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
#include <vector>
#include <cstdlib>

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
    int no_pipe32;  // FC_NO_REVPIPE32=1: the unpipelined reverse gather for GC = 32 (A/B)
    const float *rows;
    const float *loc;
    const int32_t *nbr;
    Csr csr;
    const uint8_t *bimg;  // B operand image (hi [, lo]) in the exact smem layout
    const float *binv;    // 1 / (B scale)
    float *out;
    int64_t num_tiles;
    // REVERSE + DLOC only: location gradient d_loc[j] = centre[j] - sum_c f[j,c] U_j[c,:]
    const float *feat;    // [total, NOUT] conv input features
    const float *centre;  // [total, 3] centre-role term (tc_dtheta kernel)
    float *dloc;          // [total, 3]
    // channel blocks (wide shapes, tc_blocked_*): row strides of the gathered rows, of the
    // output and of feat (elements; the pointers address the block's first channel), and
    // acc = 1 to add into out (and subtract from dloc) instead of overwriting
    int64_t ld_rows, ld_out, ld_feat;
    int acc;       // out += block result
    int acc_dloc;  // dloc -= this block's neighbour term (else dloc = centre - term)
    // bimg == null: every CTA packs the B image itself from this block of theta (no separate
    // pack launch on the critical path of a small call)
    const float *pk_theta, *pk_theta_b;
    int pk_cin, pk_cout, pk_ld;
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

template <int GC, int NOUT, bool SPLIT, bool DLOC = false>
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
    // per accumulator buffer: D (NOUT columns) [+ U_0..U_2 (3 x NOUT) for DLOC]; 2 buffers
    static constexpr int CPB = NOUT * (DLOC ? 4 : 1);
    static constexpr int TMEM_COLS = (2 * CPB <= 32) ? 32 : (2 * CPB <= 64) ? 64 : (2 * CPB <= 128) ? 128 : (2 * CPB <= 256) ? 256 : 512;
};

// ---------------------------------------------------------------------------------
// B image: B[n][k] = theta[c', c, t] (t < 3) | theta_b[c', c] (t == 3), k = t*GC + c.
//   forward: n = c' (rows = c_out), c = input channel   (GC = c_in)
//   reverse: n = c  (rows = c_in),  c' = gathered chan  (GC = c_out)
template <bool SPLIT>
__device__ __forceinline__ void pack_b_body(int cin, int cout, int ld_cin, const float *__restrict__ theta,
                                            const float *__restrict__ theta_b, int reverse, int nout, int gc,
                                            uint8_t *__restrict__ img, float *__restrict__ binv, int bx, int gx) {
    // (cin, cout): the block of theta packed; ld_cin: theta's full c_in (row stride); theta /
    // theta_b point at the block's first (c', c); (bx, gx): this CTA's slice of the image
    __shared__ float red[32];
    float m = 0.f;
    const int ntb = cout * cin;
    // unrolled: the loads of several iterations in flight (the loop-carried max would otherwise
    // serialise one L2 round trip per iteration)
#pragma unroll 4
    for (int i = threadIdx.x; i < ntb; i += blockDim.x) {
        const int64_t e = (int64_t)(i / cin) * ld_cin + i % cin;
        m = fmaxf(m, fmaxf(fabsf(__ldg(theta_b + e)), fmaxf(fabsf(__ldg(theta + e * 3)), fmaxf(fabsf(__ldg(theta + e * 3 + 1)),
                                                                                          fabsf(__ldg(theta + e * 3 + 2))))));
    }
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
    if (bx == 0 && threadIdx.x == 0) binv[0] = inv;
    const int KT = 4 * gc;
    const int bbytes = nout * KT * 2;
    // every block reduces the (L2-resident) max itself and packs its slice of the image
    for (int idx = bx * blockDim.x + threadIdx.x; idx < nout * KT; idx += gx * blockDim.x) {
        const int nn = idx / KT, k = idx % KT;
        const int t = k / gc, c = k % gc;
        const int cp = reverse ? c : nn;
        const int ci = reverse ? nn : c;
        const float v = (t < 3) ? theta[((int64_t)cp * ld_cin + ci) * 3 + t] : theta_b[(int64_t)cp * ld_cin + ci];
        uint16_t lo;
        const uint16_t hi = pack1<SPLIT>(v * s, lo);
        const uint32_t off = sw128_offset(nn, k, nout);
        *reinterpret_cast<uint16_t *>(img + off) = hi;
        if (SPLIT) *reinterpret_cast<uint16_t *>(img + bbytes + off) = lo;
    }
}
template <bool SPLIT>
__global__ void __launch_bounds__(1024)
    tc_pack_b_kernel(int cin, int cout, int ld_cin, const float *__restrict__ theta, const float *__restrict__ theta_b,
                     int reverse, int nout, int gc, uint8_t *__restrict__ img, float *__restrict__ binv) {
    pack_b_body<SPLIT>(cin, cout, ld_cin, theta, theta_b, reverse, nout, gc, img, binv, blockIdx.x, gridDim.x);
}
// the B images of all passes of a channel-blocked call in ONE launch (blockIdx.y = pass),
// each identical to its own tc_pack_b_kernel launch: image j at img0 + j * stride, its
// 1 / scale right after the image bytes
constexpr int kPackBatch = 32;
struct PackBatch {
    const float *theta[kPackBatch];
    const float *theta_b[kPackBatch];
};
template <bool SPLIT>
__global__ void __launch_bounds__(1024)
    tc_pack_b_batch_kernel(int cin, int cout, int ld_cin, int reverse, int nout, int gc, uint8_t *__restrict__ img0,
                           int64_t stride, int64_t bbytes, const __grid_constant__ PackBatch jobs) {
    uint8_t *img = img0 + (int64_t)blockIdx.y * stride;
    pack_b_body<SPLIT>(cin, cout, ld_cin, jobs.theta[blockIdx.y], jobs.theta_b[blockIdx.y], reverse, nout, gc, img,
                       reinterpret_cast<float *>(img + bbytes), blockIdx.x, gridDim.x);
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
// Software-pipelined forward gather for k = 8 (one 8-slot batch per group).
// A warp walks its sequence of groups ("items"); item w covers points p0(w) .. p0(w)+PPI-1.
// Three-deep pipeline: raw index + centre position of item w+2 are issued during w, the
// neighbour positions of w+1 are issued (and its rows prefetched to L2) during w, and the
// rows of w are loaded and accumulated during w; no load result is consumed in the
// iteration that issues it.
struct GatherSrc {
    const float *rows, *loc;
    const int32_t *nbr;
    int64_t total, n;
    int64_t ld;  // row stride of `rows` (elements)
};
struct ItemMap {
    int ipt;         // items per tile for this warp
    int sub_base;    // first point of item 0 within its tile
    int sub_stride;  // points between consecutive items of one tile
    __device__ __forceinline__ int64_t p0(int64_t w) const {
        return ((int64_t)blockIdx.x + (w / ipt) * gridDim.x) * kTcM + sub_base + (w % ipt) * sub_stride;
    }
};

template <int GC>
struct FwdPipe8 {
    using G = Geo<GC>;
    struct Raw {
        int32_t nb, base;  // cloud-local neighbour index, cloud base
        float l0, l1, l2;
        bool v;
    };
    GatherSrc s;
    ItemMap im;
    int64_t items;
    int pt, cl, ipt, slot;
    Idx cur;
    Raw r1;
    int32_t j1;
    float nl0, nl1, nl2;

    __device__ __forceinline__ Raw raw_load(int64_t w) const {
        Raw r{0, 0, 0.f, 0.f, 0.f, false};
        if (w < items) {
            const int64_t myp = im.p0(w) + ipt;
            r.v = ipt < G::PPI && myp < s.total;
            if (r.v) {
                r.base = myp < s.n ? 0 : (int32_t)((myp / s.n) * s.n);
                r.nb = __ldg(s.nbr + myp * kSlots + slot);
                r.l0 = __ldg(s.loc + myp * 3 + 0);
                r.l1 = __ldg(s.loc + myp * 3 + 1);
                r.l2 = __ldg(s.loc + myp * 3 + 2);
            }
        }
        return r;
    }
    __device__ __forceinline__ void issue_pos(const Raw &r) {
        j1 = r.base + r.nb;
        nl0 = nl1 = nl2 = 0.f;
        if (r.v) {
            nl0 = __ldg(s.loc + (int64_t)j1 * 3 + 0);
            nl1 = __ldg(s.loc + (int64_t)j1 * 3 + 1);
            nl2 = __ldg(s.loc + (int64_t)j1 * 3 + 2);
        }
    }
    __device__ __forceinline__ void make_cur(const Raw &r) {
        cur.j = j1;
        cur.o0 = r.v ? r.l0 - nl0 : 0.f;
        cur.o1 = r.v ? r.l1 - nl1 : 0.f;
        cur.o2 = r.v ? r.l2 - nl2 : 0.f;
    }
    __device__ __forceinline__ void start(GatherSrc src, ItemMap map, int64_t n_items, int lane) {
        s = src;
        im = map;
        items = n_items;
        pt = lane / G::LPR;
        cl = lane % G::LPR;
        ipt = lane >> 3;
        slot = lane & 7;
        const Raw r0 = raw_load(0);
        issue_pos(r0);
        make_cur(r0);
        r1 = raw_load(1);
    }
    // moments of item w (issues the prefetches of w+1 and w+2)
    __device__ __forceinline__ void gather(int64_t w, Mom &acc) {
        float4 v[kSlots];
#pragma unroll
        for (int q = 0; q < kSlots; ++q) {
            const int32_t jj = __shfl_sync(0xffffffffu, cur.j, pt * 8 + q);
            v[q] = __ldg(reinterpret_cast<const float4 *>(s.rows + (int64_t)jj * s.ld) + cl);
        }
        issue_pos(r1);
        if (r1.v) {
            const float *rp = s.rows + (int64_t)j1 * s.ld;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(rp));
            if (GC * 4 > 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + 32));
        }
        r2_ = raw_load(w + 2);
        mom_zero(acc);
#pragma unroll
        for (int q = 0; q < kSlots; ++q) {
            const float w0 = __shfl_sync(0xffffffffu, cur.o0, pt * 8 + q);
            const float w1 = __shfl_sync(0xffffffffu, cur.o1, pt * 8 + q);
            const float w2 = __shfl_sync(0xffffffffu, cur.o2, pt * 8 + q);
            mom_add(acc, v[q], w0, w1, w2);
        }
    }
    // after the caller consumed item w: offsets of w+1 become current
    __device__ __forceinline__ void advance() {
        make_cur(r1);
        r1 = r2_;
    }
    Raw r2_;
};

// ---------------------------------------------------------------------------------
// Software-pipelined REVERSE gather (GC = 64: 2 points per item, 16 index slots per point,
// lane = point * 16 + slot).  The reverse list of point p is ent[off[p] .. off[p+1]) (flat
// forward slots e, source point i = e / k, offset l_i - l_p).  Four-deep pipeline:
// off[] of item w+3, ent[] (+ centre position) of w+2, source positions of w+1 are issued
// during w; rows of w are loaded in 8-slot sub-batches and accumulated in list order.
// Lists longer than 16 finish on a (rare) unpipelined tail.
struct RevPipe16 {
    static constexpr int GC = 64;
    const float *rows, *loc;
    int64_t ld;  // row stride of `rows` (elements)
    Csr csr;
    int64_t total;
    int k;
    ItemMap im;
    int64_t items;
    int pt, cl, ipt, slot;
    // stage "off" (item w+3): list range of the lane's point
    int32_t oq0_3, ocnt_3;
    // stage "ent" (item w+2)
    int32_t eq0_2, ecnt_2, ent_2;
    float lp0_2, lp1_2, lp2_2;
    // stage "pos" (item w+1)
    int32_t pq0_1, pcnt_1, j_1;
    float lp0_1, lp1_1, lp2_1, nl0_1, nl1_1, nl2_1;
    // current (item w)
    int32_t q0, cnt, j;
    float o0, o1, o2;

    __device__ __forceinline__ void load_off(int64_t w, int32_t &q0o, int32_t &cnto) const {
        q0o = 0;
        cnto = 0;
        if (w < items) {
            const int64_t myp = im.p0(w) + ipt;
            if (myp < total) {
                q0o = __ldg(csr.off + myp);
                cnto = __ldg(csr.off + myp + 1) - q0o;
            }
        }
    }
    __device__ __forceinline__ void load_ent(int64_t w, int32_t q0i, int32_t cnti) {
        eq0_2 = q0i;
        ecnt_2 = cnti;
        ent_2 = -1;
        lp0_2 = lp1_2 = lp2_2 = 0.f;
        if (w < items) {
            const int64_t myp = im.p0(w) + ipt;
            if (myp < total) {
                lp0_2 = __ldg(loc + myp * 3 + 0);
                lp1_2 = __ldg(loc + myp * 3 + 1);
                lp2_2 = __ldg(loc + myp * 3 + 2);
                if (slot < cnti) ent_2 = __ldg(csr.ent + q0i + slot);
            }
        }
    }
    __device__ __forceinline__ void load_pos() {
        pq0_1 = eq0_2;
        pcnt_1 = ecnt_2;
        lp0_1 = lp0_2, lp1_1 = lp1_2, lp2_1 = lp2_2;
        j_1 = ent_2 >= 0 ? ent_2 / k : 0;
        nl0_1 = nl1_1 = nl2_1 = 0.f;
        if (ent_2 >= 0) {
            nl0_1 = __ldg(loc + (int64_t)j_1 * 3 + 0);
            nl1_1 = __ldg(loc + (int64_t)j_1 * 3 + 1);
            nl2_1 = __ldg(loc + (int64_t)j_1 * 3 + 2);
        }
    }
    __device__ __forceinline__ void make_cur() {
        q0 = pq0_1;
        cnt = pcnt_1;
        j = j_1;
        const bool v = slot < pcnt_1;
        o0 = v ? nl0_1 - lp0_1 : 0.f;
        o1 = v ? nl1_1 - lp1_1 : 0.f;
        o2 = v ? nl2_1 - lp2_1 : 0.f;
    }
    __device__ __forceinline__ void start(const float *rows_, int64_t ld_, const float *loc_, Csr csr_, int64_t total_,
                                          int k_, ItemMap map, int64_t n_items, int lane) {
        rows = rows_;
        ld = ld_;
        loc = loc_;
        csr = csr_;
        total = total_;
        k = k_;
        im = map;
        items = n_items;
        pt = lane >> 4;
        cl = lane & 15;
        ipt = lane >> 4;
        slot = lane & 15;
        int32_t a0, c0;
        load_off(0, a0, c0);
        load_ent(0, a0, c0);
        load_pos();
        make_cur();  // item 0 (blocking, once)
        load_off(1, a0, c0);
        load_ent(1, a0, c0);
        load_off(2, oq0_3, ocnt_3);
    }
    __device__ __forceinline__ void sub_batch(int b0, int mycnt, Mom &acc) const {
        float4 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int32_t jj = __shfl_sync(0xffffffffu, j, pt * 16 + b0 + q);
            v[q] = (b0 + q < mycnt) ? __ldg(reinterpret_cast<const float4 *>(rows + (int64_t)jj * ld) + cl)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float w0 = __shfl_sync(0xffffffffu, o0, pt * 16 + b0 + q);
            const float w1 = __shfl_sync(0xffffffffu, o1, pt * 16 + b0 + q);
            const float w2 = __shfl_sync(0xffffffffu, o2, pt * 16 + b0 + q);
            if (b0 + q < mycnt) mom_add(acc, v[q], w0, w1, w2);
        }
    }
    // moments of item w; issues the loads of items w+1 .. w+3
    __device__ __forceinline__ void gather(int64_t w, Mom &acc) {
        const int mycnt = __shfl_sync(0xffffffffu, cnt, pt * 16);
        const int c0 = __shfl_sync(0xffffffffu, cnt, 0), c1 = __shfl_sync(0xffffffffu, cnt, 16);
        const int maxcnt = max(c0, c1);
        mom_zero(acc);
        // rows of the first 8 slots first, then the prefetches of later items
        float4 v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int32_t jj = __shfl_sync(0xffffffffu, j, pt * 16 + q);
            v[q] = (q < mycnt) ? __ldg(reinterpret_cast<const float4 *>(rows + (int64_t)jj * ld) + cl)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        load_pos();                    // item w+1: source positions
        load_ent(w + 2, oq0_3, ocnt_3);  // item w+2: list entries
        load_off(w + 3, oq0_3, ocnt_3);  // item w+3: list ranges
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float w0 = __shfl_sync(0xffffffffu, o0, pt * 16 + q);
            const float w1 = __shfl_sync(0xffffffffu, o1, pt * 16 + q);
            const float w2 = __shfl_sync(0xffffffffu, o2, pt * 16 + q);
            if (q < mycnt) mom_add(acc, v[q], w0, w1, w2);
        }
        if (maxcnt > 8) sub_batch(8, mycnt, acc);
        if (maxcnt > 16) {
            // tail: lists longer than 16 entries, unpipelined, still in list order
            const int64_t myp = im.p0(w) + ipt;
            const float lp0 = myp < total ? __ldg(loc + myp * 3 + 0) : 0.f;
            const float lp1 = myp < total ? __ldg(loc + myp * 3 + 1) : 0.f;
            const float lp2 = myp < total ? __ldg(loc + myp * 3 + 2) : 0.f;
            for (int b0 = 16; b0 < maxcnt; b0 += 16) {
                int32_t jt = 0;
                float t0 = 0.f, t1 = 0.f, t2 = 0.f;
                if (b0 + slot < cnt) {
                    jt = __ldg(csr.ent + q0 + b0 + slot) / k;
                    t0 = __ldg(loc + (int64_t)jt * 3 + 0) - lp0;
                    t1 = __ldg(loc + (int64_t)jt * 3 + 1) - lp1;
                    t2 = __ldg(loc + (int64_t)jt * 3 + 2) - lp2;
                }
                for (int q = 0; q < 16; ++q) {
                    const int32_t jj = __shfl_sync(0xffffffffu, jt, pt * 16 + q);
                    const float w0 = __shfl_sync(0xffffffffu, t0, pt * 16 + q);
                    const float w1 = __shfl_sync(0xffffffffu, t1, pt * 16 + q);
                    const float w2 = __shfl_sync(0xffffffffu, t2, pt * 16 + q);
                    if (b0 + q < mycnt) {
                        const float4 x = __ldg(reinterpret_cast<const float4 *>(rows + (int64_t)jj * ld) + cl);
                        mom_add(acc, x, w0, w1, w2);
                    }
                }
            }
        }
    }
    __device__ __forceinline__ void advance() { make_cur(); }
};

// Software-pipelined REVERSE gather for GC = 32: 4 points per item, 8 lanes per point
// (lane = point * 8 + slot), each index lane holding TWO list slots (slot, slot + 8), so the
// first 16 entries of every list are pipelined like RevPipe16's: off[] of item w+3, ent[]
// (+ centre position) of w+2, source positions of w+1 issued during w; rows of w loaded in
// 8-slot sub-batches and accumulated in list order; lists longer than 16 finish unpipelined.
struct RevPipe8x2 {
    static constexpr int GC = 32;
    const float *rows, *loc;
    int64_t ld;
    Csr csr;
    int64_t total;
    int k;
    ItemMap im;
    int64_t items;
    int pt, cl, slot;
    int32_t oq0_3, ocnt_3;                      // item w+3
    int32_t eq0_2, ecnt_2, ent_2[2];            // item w+2
    float lp0_2, lp1_2, lp2_2;
    int32_t pq0_1, pcnt_1, j_1[2];              // item w+1
    float lp0_1, lp1_1, lp2_1, nl_1[2][3];
    int32_t q0, cnt, j[2];                      // item w
    float o[2][3];

    __device__ __forceinline__ void load_off(int64_t w, int32_t &q0o, int32_t &cnto) const {
        q0o = 0;
        cnto = 0;
        if (w < items) {
            const int64_t myp = im.p0(w) + pt;
            if (myp < total) {
                q0o = __ldg(csr.off + myp);
                cnto = __ldg(csr.off + myp + 1) - q0o;
            }
        }
    }
    __device__ __forceinline__ void load_ent(int64_t w, int32_t q0i, int32_t cnti) {
        eq0_2 = q0i;
        ecnt_2 = cnti;
        ent_2[0] = ent_2[1] = -1;
        lp0_2 = lp1_2 = lp2_2 = 0.f;
        if (w < items) {
            const int64_t myp = im.p0(w) + pt;
            if (myp < total) {
                lp0_2 = __ldg(loc + myp * 3 + 0);
                lp1_2 = __ldg(loc + myp * 3 + 1);
                lp2_2 = __ldg(loc + myp * 3 + 2);
                if (slot < cnti) ent_2[0] = __ldg(csr.ent + q0i + slot);
                if (slot + 8 < cnti) ent_2[1] = __ldg(csr.ent + q0i + slot + 8);
            }
        }
    }
    __device__ __forceinline__ void load_pos() {
        pq0_1 = eq0_2;
        pcnt_1 = ecnt_2;
        lp0_1 = lp0_2, lp1_1 = lp1_2, lp2_1 = lp2_2;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            j_1[h] = ent_2[h] >= 0 ? ent_2[h] / k : 0;
            nl_1[h][0] = nl_1[h][1] = nl_1[h][2] = 0.f;
            if (ent_2[h] >= 0) {
                nl_1[h][0] = __ldg(loc + (int64_t)j_1[h] * 3 + 0);
                nl_1[h][1] = __ldg(loc + (int64_t)j_1[h] * 3 + 1);
                nl_1[h][2] = __ldg(loc + (int64_t)j_1[h] * 3 + 2);
            }
        }
    }
    __device__ __forceinline__ void make_cur() {
        q0 = pq0_1;
        cnt = pcnt_1;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            j[h] = j_1[h];
            const bool v = slot + 8 * h < pcnt_1;
            o[h][0] = v ? nl_1[h][0] - lp0_1 : 0.f;
            o[h][1] = v ? nl_1[h][1] - lp1_1 : 0.f;
            o[h][2] = v ? nl_1[h][2] - lp2_1 : 0.f;
        }
    }
    __device__ __forceinline__ void start(const float *rows_, int64_t ld_, const float *loc_, Csr csr_, int64_t total_,
                                          int k_, ItemMap map, int64_t n_items, int lane) {
        rows = rows_;
        ld = ld_;
        loc = loc_;
        csr = csr_;
        total = total_;
        k = k_;
        im = map;
        items = n_items;
        pt = lane >> 3;
        cl = lane & 7;
        slot = lane & 7;
        int32_t a0, c0;
        load_off(0, a0, c0);
        load_ent(0, a0, c0);
        load_pos();
        make_cur();  // item 0 (blocking, once)
        load_off(1, a0, c0);
        load_ent(1, a0, c0);
        load_off(2, oq0_3, ocnt_3);
    }
    template <int H>
    __device__ __forceinline__ void half_batch(int mycnt, Mom &acc, const float4 (&v)[8]) const {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float w0 = __shfl_sync(0xffffffffu, o[H][0], pt * 8 + q);
            const float w1 = __shfl_sync(0xffffffffu, o[H][1], pt * 8 + q);
            const float w2 = __shfl_sync(0xffffffffu, o[H][2], pt * 8 + q);
            if (8 * H + q < mycnt) mom_add(acc, v[q], w0, w1, w2);
        }
    }
    template <int H>
    __device__ __forceinline__ void load_rows(int mycnt, float4 (&v)[8]) const {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int32_t jj = __shfl_sync(0xffffffffu, j[H], pt * 8 + q);
            v[q] = (8 * H + q < mycnt) ? __ldg(reinterpret_cast<const float4 *>(rows + (int64_t)jj * ld) + cl)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    __device__ __forceinline__ void gather(int64_t w, Mom &acc) {
        const int mycnt = __shfl_sync(0xffffffffu, cnt, pt * 8);
        const int maxcnt = (int)__reduce_max_sync(0xffffffffu, (uint32_t)max(cnt, 0));
        mom_zero(acc);
        float4 v[8];
        load_rows<0>(mycnt, v);
        load_pos();                      // item w+1: source positions
        load_ent(w + 2, oq0_3, ocnt_3);  // item w+2: list entries
        load_off(w + 3, oq0_3, ocnt_3);  // item w+3: list ranges
        half_batch<0>(mycnt, acc, v);
        if (maxcnt > 8) {
            load_rows<1>(mycnt, v);
            half_batch<1>(mycnt, acc, v);
        }
        if (maxcnt > 16) {
            // tail: lists longer than 16 entries, unpipelined, still in list order
            const int64_t myp = im.p0(w) + pt;
            const float lp0 = myp < total ? __ldg(loc + myp * 3 + 0) : 0.f;
            const float lp1 = myp < total ? __ldg(loc + myp * 3 + 1) : 0.f;
            const float lp2 = myp < total ? __ldg(loc + myp * 3 + 2) : 0.f;
            for (int b0 = 16; b0 < maxcnt; b0 += 8) {
                int32_t jt = 0;
                float t0 = 0.f, t1 = 0.f, t2 = 0.f;
                if (b0 + slot < cnt) {
                    jt = __ldg(csr.ent + q0 + b0 + slot) / k;
                    t0 = __ldg(loc + (int64_t)jt * 3 + 0) - lp0;
                    t1 = __ldg(loc + (int64_t)jt * 3 + 1) - lp1;
                    t2 = __ldg(loc + (int64_t)jt * 3 + 2) - lp2;
                }
                for (int q = 0; q < 8; ++q) {
                    const int32_t jj = __shfl_sync(0xffffffffu, jt, pt * 8 + q);
                    const float w0 = __shfl_sync(0xffffffffu, t0, pt * 8 + q);
                    const float w1 = __shfl_sync(0xffffffffu, t1, pt * 8 + q);
                    const float w2 = __shfl_sync(0xffffffffu, t2, pt * 8 + q);
                    if (b0 + q < mycnt) {
                        const float4 x = __ldg(reinterpret_cast<const float4 *>(rows + (int64_t)jj * ld) + cl);
                        mom_add(acc, x, w0, w1, w2);
                    }
                }
            }
        }
    }
    __device__ __forceinline__ void advance() { make_cur(); }
};

// ---------------------------------------------------------------------------------
// Accumulator drain of tile i by one epilogue warp (TMEM lane quadrant = warp % 4): one
// thread per output row.  Kept out of line so that its registers do not add to the live
// set of the gather pipeline it interrupts.
template <int NOUT, bool DLOC, int CPB>
__device__ __noinline__ void tc_gmc_epilogue(const TcArgs &a, int i, int warp, int lane, uint32_t tmem_base,
                                             const float *rs, uint64_t *mma_done, uint64_t *d_free) {
    const int64_t tile = blockIdx.x + (int64_t)i * gridDim.x;
    const int row = warp * 32 + lane;
    mbar_wait(mma_done + (i & 1), (i >> 1) & 1);
    tc_fence_after();
    const int64_t p = tile * kTcM + row;
    const bool pv = p < a.total;
    const float inv = rs[(i & 1) * kTcM + row];
    float *orow = a.out + p * a.ld_out;
    const uint32_t tbase = tmem_base + ((uint32_t)(warp * 32) << 16) + (uint32_t)((i & 1) * CPB);
    float nb0 = 0.f, nb1 = 0.f, nb2 = 0.f;
#pragma unroll 1
    for (int c0 = 0; c0 < NOUT; c0 += 16) {
        float v[16];
        tmem_ld16(tbase + (uint32_t)c0, v);
        if (pv) {
#pragma unroll
            for (int q = 0; q < 16; q += 4) {
                float4 w = make_float4(v[q] * inv, v[q + 1] * inv, v[q + 2] * inv, v[q + 3] * inv);
                if (a.acc) {
                    const float4 o = *reinterpret_cast<const float4 *>(orow + c0 + q);
                    w.x += o.x, w.y += o.y, w.z += o.z, w.w += o.w;
                }
                *reinterpret_cast<float4 *>(orow + c0 + q) = w;
            }
        }
        if constexpr (DLOC) {
            // neighbour role: -sum_c f[p, c] U_t[p, c] (the -dt terms of _native.pyx:121-127)
            float f[16];
            if (pv) {
#pragma unroll
                for (int q = 0; q < 16; q += 4) {
                    const float4 x = __ldg(reinterpret_cast<const float4 *>(a.feat + p * a.ld_feat + c0 + q));
                    f[q] = x.x, f[q + 1] = x.y, f[q + 2] = x.z, f[q + 3] = x.w;
                }
            } else {
#pragma unroll
                for (int q = 0; q < 16; ++q) f[q] = 0.f;
            }
            float u[16];
            tmem_ld16(tbase + (uint32_t)(NOUT + c0), u);
#pragma unroll
            for (int q = 0; q < 16; ++q) nb0 = fmaf(f[q], u[q], nb0);
            tmem_ld16(tbase + (uint32_t)(2 * NOUT + c0), u);
#pragma unroll
            for (int q = 0; q < 16; ++q) nb1 = fmaf(f[q], u[q], nb1);
            tmem_ld16(tbase + (uint32_t)(3 * NOUT + c0), u);
#pragma unroll
            for (int q = 0; q < 16; ++q) nb2 = fmaf(f[q], u[q], nb2);
        }
    }
    if constexpr (DLOC) {
        if (pv) {
            const float *base = a.acc_dloc ? a.dloc : a.centre;  // blocks after the first subtract their part
            a.dloc[p * 3 + 0] = base[p * 3 + 0] - nb0 * inv;
            a.dloc[p * 3 + 1] = base[p * 3 + 1] - nb1 * inv;
            a.dloc[p * 3 + 2] = base[p * 3 + 2] - nb2 * inv;
        }
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(d_free + (i & 1));
}

template <int GC, int NOUT, bool SPLIT, bool REVERSE, int KFIX, bool DLOC = false>
__global__ void __launch_bounds__(kTcThreads, 1) tc_gmc_kernel(TcArgs a) {
    static_assert(!DLOC || REVERSE, "the location-gradient epilogue belongs to the reverse pass");
    using L = TcLayout<GC, NOUT, SPLIT, DLOC>;
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
    __shared__ float binv_s;
    {  // resident B operand image(s): the caller's packed image, or packed here from theta
        if (a.bimg) {
            const uint4 *src = reinterpret_cast<const uint4 *>(a.bimg);
            uint4 *dst = reinterpret_cast<uint4 *>(B_hi);
            const int nvec = L::B_BYTES * L::NSPLIT / 16;
            smem_fill16(dst, src, nvec);
        } else {
            pack_b_body<SPLIT>(a.pk_cin, a.pk_cout, a.pk_ld, a.pk_theta, a.pk_theta_b, REVERSE ? 1 : 0, NOUT, GC, B_hi,
                               &binv_s, 0, 1);
        }
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const float binv = a.bimg ? a.binv[0] : binv_s;
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
            const uint32_t d_tmem = tmem_base + (uint32_t)((i & 1) * L::CPB);
            // byte offset of 16-bit element k of a K-major SW128 operand with `rows` rows
            auto koff = [](int k, int rows) { return (uint32_t)((k >> 6) * rows * 128 + (k & 63) * 2); };
#pragma unroll
            for (int s = 0; s < L::KT / 16; ++s) {
                const uint32_t aoff = koff(16 * s, kTcM), boff = koff(16 * s, NOUT);
                mma_f16(d_tmem, desc_sw128(a_hi + aoff), desc_sw128(b_hi + boff), idesc, s > 0 ? 1u : 0u);
                if (SPLIT) {
                    mma_f16(d_tmem, desc_sw128(a_hi + aoff), desc_sw128(b_lo + boff), idesc, 1u);
                    mma_f16(d_tmem, desc_sw128(a_lo + aoff), desc_sw128(b_hi + boff), idesc, 1u);
                }
            }
            if constexpr (DLOC) {
                // U_t[p, c] = sum_c' Yb[p, c'] theta[c', c, t]: A = the bias-moment block
                // (k in [3GC, 4GC)), B = K-block t of the resident adjoint image B_rev.
#pragma unroll
                for (int t = 0; t < 3; ++t) {
                    const uint32_t u_tmem = d_tmem + (uint32_t)(NOUT * (1 + t));
#pragma unroll
                    for (int s = 0; s < GC / 16; ++s) {
                        const uint32_t aoff = koff(3 * GC + 16 * s, kTcM), boff = koff(t * GC + 16 * s, NOUT);
                        mma_f16(u_tmem, desc_sw128(a_hi + aoff), desc_sw128(b_hi + boff), idesc, s > 0 ? 1u : 0u);
                        if (SPLIT) {
                            mma_f16(u_tmem, desc_sw128(a_hi + aoff), desc_sw128(b_lo + boff), idesc, 1u);
                            mma_f16(u_tmem, desc_sw128(a_lo + aoff), desc_sw128(b_hi + boff), idesc, 1u);
                        }
                    }
                }
            }
            mma_commit(mma_done + (i & 1));
        }
        __syncwarp();
    };
    // ---------------------------------------------------------------- epilogue (warps 0..3)
    // warp q owns TMEM lanes / tile rows 32q .. 32q+31; one thread per output row.
    auto epilogue = [&](int i) {
        tc_gmc_epilogue<NOUT, DLOC, L::CPB>(a, i, warp, lane, tmem_base, rs, mma_done, d_free);
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
                           ? __ldg(reinterpret_cast<const float4 *>(a.rows + (int64_t)jj * a.ld_rows) + cl)
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
            FwdPipe8<GC> pipe;
            pipe.start(GatherSrc{a.rows, a.loc, a.nbr, a.total, a.n, a.ld_rows},
                       ItemMap{G::GPW, gw * G::PPI, kGatherWarps * G::PPI}, items, lane);
            for (int64_t w = 0; w < items; ++w) {
                Mom acc;
                pipe.gather(w, acc);
                finish(w, item_p0(w), acc);
                pipe.advance();
            }
        } else if (REVERSE && GC == 32 && !a.no_pipe32) {
            RevPipe8x2 pipe;
            pipe.start(a.rows, a.ld_rows, a.loc, a.csr, a.total, a.k, ItemMap{G::GPW, gw * G::PPI, kGatherWarps * G::PPI}, items,
                       lane);
            for (int64_t w = 0; w < items; ++w) {
                Mom acc;
                pipe.gather(w, acc);
                finish(w, item_p0(w), acc);
                pipe.advance();
            }
        } else if (REVERSE && GC == 64) {
            RevPipe16 pipe;
            pipe.start(a.rows, a.ld_rows, a.loc, a.csr, a.total, a.k, ItemMap{G::GPW, gw * G::PPI, kGatherWarps * G::PPI}, items,
                       lane);
            for (int64_t w = 0; w < items; ++w) {
                Mom acc;
                pipe.gather(w, acc);
                finish(w, item_p0(w), acc);
                pipe.advance();
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

// =================================================================================
// Backward, forward-gather half: d_theta / d_theta_b and the centre role of d_locations.
//
//   D[k, c'] = sum_p X_p[k] g_p[c']            (d_theta, k = t*64 + c;  _native.pyx:106-112)
//   Z_t[p, c'] = sum_c X_p[3, c] theta[c', c, t],  centre[p, t] = sum_c' g_p[c'] Z_t[p, c']
//                                               (the +dt terms of _native.pyx:121-127)
// d_theta reduces over POINTS, so it is fed point-chunk by point-chunk (16 points) through a
// 2-stage shared-memory ring as kind::tf32 MMAs with M = k (two halves of 128), N = c', K =
// points, both operands MN-major; tf32 hi/lo split (3 MMAs) keeps fp32 accuracy with no
// scaling, so the accumulator stays in TMEM across all tiles of the CTA (deterministic per
// CTA); the per-CTA partials are then reduced in fixed order (dtheta_reduce_kernel).
// Z is an fp16-split M = 128 (points) GEMM on the bias moments, B = K-blocks 0..2 of the
// forward image.  GC = c_in = 64 and CO = c_out = 64 (the headline shape).
// =================================================================================
constexpr int kDtChunk = 16;  // points per d_theta chunk (2 tf32 k-steps)

struct DtArgs {
    int64_t total, n;
    int k;
    const float *feat, *loc, *g;
    const int32_t *nbr;
    const uint8_t *bimg;  // forward fp16 image (hi, lo); K-blocks 0..2 used
    const float *binv;
    float *partial;       // [gridDim.x][2 (hi / lo lanes)][CO * 4 * GC], layout (c', c, t) like dtheta_partial_kernel
    float *centre;        // [total, 3]
    int64_t num_tiles;
    int64_t ld_feat, ld_g;  // row strides of feat / g (channel blocks of wide shapes)
    int acc;                // add into centre instead of overwriting (blocks after the first)
};

// MT = 64-channel c' tiles per pass (M-tiles of the d_theta MMA, each [c' hi; c' lo] = 128
// rows x N = 256 columns of TMEM): MT = 1 with the centre-role Z GEMM (TMEM 256 + 192), MT = 2
// without it (TMEM 2 x 256) -- a wide layer's 64-channel feature block is then gathered once
// per 128 upstream channels instead of once per 64.
template <int MT = 1>
struct DtLayoutT {
    static constexpr int GC = 64, CO = 64 * MT;
    static constexpr bool Z = MT == 1;
    static constexpr int XST = kDtChunk * 4 * GC * 4;   // one tf32 X chunk image (16 KB)
    static constexpr int GST = kDtChunk * 64 * 4;       // one tf32 G image of a c' tile (4 KB)
    static constexpr int XB = kTcM * GC * 2;            // fp16 bias-moment tile (16 KB)
    static constexpr int BZ = 64 * 128;                 // one K-block of the forward image (8 KB)
    static constexpr int X_OFF = 0;                     // [stage][hi, lo]
    static constexpr int G_OFF = X_OFF + 2 * 2 * XST;   // [stage][c' tile][hi, lo]
    static constexpr int XB_OFF = G_OFF + 2 * MT * 2 * GST;        // [buf][hi, lo]   (Z only)
    static constexpr int B_OFF = XB_OFF + (Z ? 2 * 2 * XB : 0);    // [hi K-blocks 0..2][lo] (Z only)
    static constexpr int RS_OFF = B_OFF + (Z ? 2 * 3 * BZ : 0);    // float rs[2][128]
    static constexpr int BAR_OFF = RS_OFF + 2 * kTcM * 4;
    static constexpr int SMEM = BAR_OFF + 128 + 1024;
    static constexpr int TMEM_COLS = 512;  // D: MT x 256 (M = [c' hi; c' lo], N = k) [+ Z: 192]
};
using DtLayout = DtLayoutT<1>;

__device__ __forceinline__ uint32_t f32_to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
// tf32 hi / lo of 4 values -> 16-byte stores at hi_addr and lo_addr
__device__ __forceinline__ void store_tf32x4(uint32_t hi_addr, uint32_t lo_addr, float2 a, float2 b) {
    const uint32_t h0 = f32_to_tf32(a.x), h1 = f32_to_tf32(a.y), h2 = f32_to_tf32(b.x), h3 = f32_to_tf32(b.y);
    sts128(hi_addr, h0, h1, h2, h3);
    sts128(lo_addr, __float_as_uint(a.x - __uint_as_float(h0)), __float_as_uint(a.y - __uint_as_float(h1)),
           __float_as_uint(b.x - __uint_as_float(h2)), __float_as_uint(b.y - __uint_as_float(h3)));
}

// MN-major tf32 operand descriptor.  The only MN-major smem layout the hardware takes for
// 32-bit elements is SWIZZLE_128B_BASE32B: atoms of 4 K-rows x 128 B (32 elements along
// MN), the 32-byte chunk index XOR-ed with (row % 4).  MN blocks of 128 B are LBO apart,
// 4-row K groups SBO apart.
__device__ __forceinline__ uint64_t desc_sw128b32_mn(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)1 << 61;  // SWIZZLE_128B_BASE32B
    return d;
}
// byte offset of 4 consecutive MN elements starting at mn (multiple of 4) in K-row r of an
// SW128_BASE32B MN-major chunk image with 16 K-rows per MN block
__device__ __forceinline__ uint32_t mn32_off(int mn, int r) {
    const int blk = mn >> 5, in = mn & 31;
    return (uint32_t)(blk * 2048 + (r >> 2) * 512 + (r & 3) * 128 + ((((in >> 3) ^ (r & 3))) << 5) + (in & 7) * 4);
}
__host__ __device__ constexpr uint32_t idesc_tf32_mn(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

template <int KFIX, int MT = 1>
__global__ void __launch_bounds__(kTcThreads, 1) tc_dtheta_kernel(DtArgs a) {
    using L = DtLayoutT<MT>;
    constexpr int GC = L::GC, CO = L::CO;
    using G = Geo<GC>;  // 16 lanes per point, 2 points per group
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t s_base = smem_u32(smem);
    float *rs = reinterpret_cast<float *>(smem + L::RS_OFF);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + L::BAR_OFF);
    uint64_t *chunk_full = bar + 0;   // [2] count 8 warps
    uint64_t *chunk_empty = bar + 2;  // [2] tcgen05.commit
    uint64_t *z_done = bar + 4;       // [2] tcgen05.commit
    uint64_t *z_free = bar + 6;       // [2] count 4 epilogue warps
    uint64_t *dt_done = bar + 8;      // tcgen05.commit
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bar + 9);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int q = 0; q < 2; ++q) {
            mbar_init(chunk_full + q, 8);
            mbar_init(chunk_empty + q, 1);
            mbar_init(z_done + q, 1);
            mbar_init(z_free + q, kEpiWarps);
        }
        mbar_init(dt_done, 1);
        fence_mbar_init();
    }
    if (warp == kMmaWarp) tmem_alloc(tmem_holder, L::TMEM_COLS);
    if (L::Z) {  // K-blocks 0..2 of the forward image (hi, then lo) -> resident B for Z
        const int img_b = CO * 4 * GC * 2;  // bytes of one full forward image
        for (int h = 0; h < 2; ++h) {
            const uint4 *src = reinterpret_cast<const uint4 *>(a.bimg + h * img_b);
            uint4 *dst = reinterpret_cast<uint4 *>(smem + L::B_OFF + h * 3 * L::BZ);
            smem_fill16(dst, src, 3 * L::BZ / 16);
        }
    }
    const float binv = L::Z ? a.binv[0] : 1.f;
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const int64_t tiles_mine = a.num_tiles > blockIdx.x ? ceil_div(a.num_tiles - blockIdx.x, gridDim.x) : 0;

    // ---------------------------------------------------------------- MMA issue (warp 15, lane 0)
    auto issue_chunk = [&](int64_t u_global) {
        // u_global = tile_local * 8 + c.  D[(c' | c'+64), k] += [G_hi; G_lo]^T . X_hi + [G_hi; G_lo]^T . X_lo:
        // M = 128 (upstream channel hi / lo parts), N = 256 (all moment columns), K = 8 points
        // per MMA -- a kind::tf32 MMA costs ~104 cycles up to N = 128 and ~130 at N = 256, so
        // this is 2 MMAs per 8 points instead of 6 (M = k halves, N = c' = 64).
        const int c = (int)(u_global & 7);
        const int st = c & 1;
        const int64_t u = u_global >> 1;  // completion index of stage st
        if (lane == 0) {
            mbar_wait(chunk_full + st, (uint32_t)(u & 1));
            tc_fence_after();
            constexpr uint32_t idesc = idesc_tf32_mn(kTcM, 4 * GC);
            const uint32_t xh = s_base + L::X_OFF + st * 2 * L::XST, xl = xh + L::XST;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                // c' tile mt: [G_hi | G_lo] = 4 MN blocks of 32
                const uint32_t gh = s_base + L::G_OFF + (st * MT + mt) * 2 * L::GST;
                const uint32_t dt = tmem_base + (uint32_t)(mt * 256);
#pragma unroll
                for (int ks = 0; ks < kDtChunk / 8; ++ks) {
                    const uint32_t ko = (uint32_t)(ks * 1024);
                    const uint32_t first = (u_global == 0 && ks == 0) ? 0u : 1u;
                    mma_tf32(dt, desc_sw128b32_mn(gh + ko, 2048, 512), desc_sw128b32_mn(xh + ko, 2048, 512), idesc, first);
                    mma_tf32(dt, desc_sw128b32_mn(gh + ko, 2048, 512), desc_sw128b32_mn(xl + ko, 2048, 512), idesc, 1u);
                }
            }
            mma_commit(chunk_empty + st);
        }
        __syncwarp();
    };
    auto issue_z = [&](int i) {
        // Z[p, (t, c')] = Xb[p, :] . theta[c', :, t] for t = 0..2 as ONE N = 192 operand: the
        // K-blocks 0..2 of the forward image are 64-row blocks 8 KB apart, i.e. a 192-row
        // K-major SW128 operand.  Single TMEM buffer (columns 256..447): wait until the
        // epilogue of tile i-1 has drained it.
        if (lane == 0) {
            if (i >= 1) mbar_wait(z_free + ((i - 1) & 1), (uint32_t)(((i - 1) >> 1) & 1));
            tc_fence_after();
            constexpr uint32_t idesc = idesc_f16(kTcM, 3 * CO, 0);
            const uint32_t ah = s_base + L::XB_OFF + (i & 1) * 2 * L::XB, al = ah + L::XB;
            const uint32_t bh = s_base + L::B_OFF, bl = bh + 3 * L::BZ;
            const uint32_t z = tmem_base + 256u;
#pragma unroll
            for (int s = 0; s < GC / 16; ++s) {
                const uint32_t ao = (uint32_t)(s * 32), bo = (uint32_t)(s * 32);
                mma_f16(z, desc_sw128(ah + ao), desc_sw128(bh + bo), idesc, s > 0 ? 1u : 0u);
                mma_f16(z, desc_sw128(ah + ao), desc_sw128(bl + bo), idesc, 1u);
                mma_f16(z, desc_sw128(al + ao), desc_sw128(bh + bo), idesc, 1u);
            }
            mma_commit(z_done + (i & 1));
        }
        __syncwarp();
    };
    // ---------------------------------------------------------------- Z epilogue (warps 0..3)
    auto epilogue_z = [&](int i) {
        const int64_t tile = blockIdx.x + (int64_t)i * gridDim.x;
        const int row = warp * 32 + lane;
        const int64_t p = tile * kTcM + row;
        mbar_wait(z_done + (i & 1), (i >> 1) & 1);
        tc_fence_after();
        const float inv = rs[(i & 1) * kTcM + row];
        const uint32_t tb = tmem_base + ((uint32_t)(warp * 32) << 16) + 256u;
        float c0 = 0.f, c1 = 0.f, c2 = 0.f;
#pragma unroll
        for (int q0 = 0; q0 < CO; q0 += 16) {
            float gv[16];
            if (p < a.total) {
#pragma unroll
                for (int q = 0; q < 16; q += 4) {
                    const float4 x = __ldg(reinterpret_cast<const float4 *>(a.g + p * a.ld_g + q0 + q));
                    gv[q] = x.x, gv[q + 1] = x.y, gv[q + 2] = x.z, gv[q + 3] = x.w;
                }
            } else {
#pragma unroll
                for (int q = 0; q < 16; ++q) gv[q] = 0.f;
            }
            float z[16];
            tmem_ld16(tb + (uint32_t)q0, z);
#pragma unroll
            for (int q = 0; q < 16; ++q) c0 = fmaf(gv[q], z[q], c0);
            tmem_ld16(tb + (uint32_t)(CO + q0), z);
#pragma unroll
            for (int q = 0; q < 16; ++q) c1 = fmaf(gv[q], z[q], c1);
            tmem_ld16(tb + (uint32_t)(2 * CO + q0), z);
#pragma unroll
            for (int q = 0; q < 16; ++q) c2 = fmaf(gv[q], z[q], c2);
        }
        if (p < a.total && a.centre) {
            const float b0 = a.acc ? a.centre[p * 3 + 0] : 0.f;
            const float b1 = a.acc ? a.centre[p * 3 + 1] : 0.f;
            const float b2 = a.acc ? a.centre[p * 3 + 2] : 0.f;
            a.centre[p * 3 + 0] = b0 + c0 * inv;
            a.centre[p * 3 + 1] = b1 + c1 * inv;
            a.centre[p * 3 + 2] = b2 + c2 * inv;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(z_free + (i & 1));
    };

    // ---------------------------------------------------------------- gather producers
    // warp w: parity q = w / 8 fills stage q of the chunks c = q, q+2, q+4, q+6 of each tile,
    // group r = w % 8 (points 2r, 2r+1 of the chunk).
    {
        const int q = warp >> 3, r = warp & 7;
        const int pt = lane / G::LPR, cl = lane % G::LPR;
        const int ipt = lane >> 3, slot = lane & 7;
        // items of this warp: (tile, chunk c = q + 2m), group r of the chunk
        const ItemMap im{4, q * kDtChunk + 2 * r, 2 * kDtChunk};
        FwdPipe8<GC> pipe;
        if (KFIX == kSlots) pipe.start(GatherSrc{a.feat, a.loc, a.nbr, a.total, a.n, a.ld_feat}, im, tiles_mine * 4, lane);
        for (int64_t tl = 0; tl < tiles_mine; ++tl) {
            const int i = (int)tl;
            const int64_t tile = blockIdx.x + tl * gridDim.x;
            for (int c = q; c < 8; c += 2) {
                const int64_t u = tl * 4 + (c >> 1);  // this stage's use count (= item index)
                const int64_t p0 = tile * kTcM + c * kDtChunk + 2 * r;
                // ---- moments of points p0, p0+1 (lane group pt)
                Mom acc;
                if (KFIX == kSlots) {
                    pipe.gather(u, acc);
                } else {
                    mom_zero(acc);
                    const int64_t myp = p0 + ipt;
                    const bool pv = ipt < 2 && myp < a.total;
                    const int cnt = a.k;
                    for (int b0 = 0; b0 < cnt; b0 += kSlots) {
                        int32_t j = 0;
                        float o0 = 0.f, o1 = 0.f, o2 = 0.f;
                        if (pv && b0 + slot < cnt) {
                            const int32_t base = myp < a.n ? 0 : (int32_t)((myp / a.n) * a.n);
                            j = base + __ldg(a.nbr + myp * cnt + b0 + slot);
                            o0 = __ldg(a.loc + myp * 3 + 0) - __ldg(a.loc + (int64_t)j * 3 + 0);
                            o1 = __ldg(a.loc + myp * 3 + 1) - __ldg(a.loc + (int64_t)j * 3 + 1);
                            o2 = __ldg(a.loc + myp * 3 + 2) - __ldg(a.loc + (int64_t)j * 3 + 2);
                        }
                        float4 v[kSlots];
#pragma unroll
                        for (int s = 0; s < kSlots; ++s) {
                            const int32_t jj = __shfl_sync(0xffffffffu, j, pt * 8 + s);
                            v[s] = (b0 + s < cnt) ? __ldg(reinterpret_cast<const float4 *>(a.feat + (int64_t)jj * a.ld_feat) + cl)
                                                  : make_float4(0.f, 0.f, 0.f, 0.f);
                        }
#pragma unroll
                        for (int s = 0; s < kSlots; ++s) {
                            const float w0 = __shfl_sync(0xffffffffu, o0, pt * 8 + s);
                            const float w1 = __shfl_sync(0xffffffffu, o1, pt * 8 + s);
                            const float w2 = __shfl_sync(0xffffffffu, o2, pt * 8 + s);
                            if (b0 + s < cnt) mom_add(acc, v[s], w0, w1, w2);
                        }
                    }
                }
                const int64_t pme = p0 + pt;
                const bool valid = pme < a.total;
                if (!valid) mom_zero(acc);
                float4 gvs[MT];
#pragma unroll
                for (int mt = 0; mt < MT; ++mt)
                    gvs[mt] = valid ? __ldg(reinterpret_cast<const float4 *>(a.g + pme * a.ld_g + 64 * mt) + cl)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                // ---- wait for the ring stage (and, at a tile's first chunk, the Xb/rs buffer)
                if (u >= 1) mbar_wait(chunk_empty + q, (uint32_t)((u - 1) & 1));
                if (L::Z && c == q && i >= 2) mbar_wait(z_free + (i & 1), ((i >> 1) + 1) & 1);
                // X chunk row (tf32 hi/lo, MN-major): row rr = 2r + pt of the chunk
                const int rr = 2 * r + pt;
                const uint32_t xh = s_base + L::X_OFF + q * 2 * L::XST, xl = xh + L::XST;
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const uint32_t off = mn32_off(t * GC + 4 * cl, rr);
                    store_tf32x4(xh + off, xl + off, acc.m[t][0], acc.m[t][1]);
                }
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {  // G chunk rows (tf32 hi/lo, MN-major over c'), per c' tile
                    const uint32_t gh = s_base + L::G_OFF + (q * MT + mt) * 2 * L::GST, gl = gh + L::GST;
                    const uint32_t off = mn32_off(4 * cl, rr);
                    store_tf32x4(gh + off, gl + off, make_float2(gvs[mt].x, gvs[mt].y), make_float2(gvs[mt].z, gvs[mt].w));
                }
                if (L::Z) {   // bias moments -> Xb tile row (fp16 hi/lo, per-row scale), K-major over c
                    float inv = 1.f;
                    float m = 0.f;
                    m = fmaxf(fmaxf(fabsf(acc.m[3][0].x), fabsf(acc.m[3][0].y)), fmaxf(fabsf(acc.m[3][1].x), fabsf(acc.m[3][1].y)));
                    for (int o = G::LPR >> 1; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
                    const float sc = split_scale(m, inv);
                    const int row = c * kDtChunk + rr;
                    const uint32_t ah = s_base + L::XB_OFF + (i & 1) * 2 * L::XB, al = ah + L::XB;
                    const int kin = 4 * cl;
                    const uint32_t off = (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + (((kin >> 3) ^ (row & 7)) << 4) + (kin & 7) * 2);
                    uint32_t l0, l1;
                    const uint32_t h0 = cvt_pair<true>(fmul2(acc.m[3][0], make_float2(sc, sc)), l0);
                    const uint32_t h1 = cvt_pair<true>(fmul2(acc.m[3][1], make_float2(sc, sc)), l1);
                    sts64(ah + off, h0, h1);
                    sts64(al + off, l0, l1);
                    if (cl == 0) rs[(i & 1) * kTcM + row] = inv * binv;
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(chunk_full + q);
                if (KFIX == kSlots) pipe.advance();
                if (warp == kMmaWarp) {
                    // warp 15 (odd chunks) issues the MMAs of this chunk and the even one before it
                    issue_chunk(tl * 8 + c - 1);
                    issue_chunk(tl * 8 + c);
                    if (L::Z && c == 7) issue_z(i);
                }
            }
            if (L::Z && warp < kEpiWarps && i >= 1) epilogue_z(i - 1);
        }
        if (warp == kMmaWarp && lane == 0) mma_commit(dt_done);
        __syncwarp();
        if (L::Z && warp < kEpiWarps && tiles_mine > 0) epilogue_z((int)tiles_mine - 1);
    }
    // ---------------------------------------------------------------- drain d_theta partials
    if (warp < kEpiWarps) {
        if (tiles_mine > 0) {
            mbar_wait(dt_done, 0);
            tc_fence_after();
        }
        // TMEM lane m = c' (hi part, warps 0-1) or 64 + c' (lo part, warps 2-3): two partial
        // slices per CTA, summed by dtheta_reduce_kernel with the other CTAs' (fixed order)
        const int m = warp * 32 + lane;
        float *part = a.partial + ((int64_t)blockIdx.x * 2 + (m >> 6)) * (CO * 4 * GC);
#pragma unroll 1
        for (int mt = 0; mt < MT; ++mt) {
            const int cp = 64 * mt + (m & 63);
#pragma unroll 1
            for (int n0 = 0; n0 < 4 * GC; n0 += 16) {
                float v[16];
                tmem_ld16(tmem_base + ((uint32_t)(warp * 32) << 16) + (uint32_t)(mt * 256 + n0), v);
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const int kx = n0 + q;  // k = t*64 + c
                    const int t = kx / GC, cc = kx % GC;
                    part[(int64_t)cp * (GC * 4) + cc * 4 + t] = tiles_mine > 0 ? v[q] : 0.f;
                }
            }
        }
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
template <int GC, int NOUT, bool SPLIT, bool REVERSE, int KFIX, bool DLOC = false>
static int launch_tc(const TcArgs &a0, int cin, int cout, const float *theta, const float *theta_b,
                     cudaStream_t st, int ld_cin = -1) {
    using L = TcLayout<GC, NOUT, SPLIT, DLOC>;
    TcArgs a = a0;
    uint8_t *img = nullptr;  // a0.bimg set: the caller packed this pass's image (pack_passes)
    static int pack_launch = -1;  // FC_PACK_KERNEL=1: a separate pack launch (A/B)
    if (pack_launch < 0) {
        const char *e = getenv("FC_PACK_KERNEL");
        pack_launch = (e && e[0] == '1') ? 1 : 0;
    }
    if (!a.bimg && !pack_launch) {  // each CTA packs the image in its prologue
        a.pk_theta = theta;
        a.pk_theta_b = theta_b;
        a.pk_cin = cin;
        a.pk_cout = cout;
        a.pk_ld = ld_cin > 0 ? ld_cin : cin;
    } else if (!a.bimg) {
        img = (uint8_t *)scratch_alloc((size_t)L::B_BYTES * L::NSPLIT + 256, st);
        if (!img) return set_error(FC_ERR_CUDA, "scratch allocation failed (tc)");
        float *binv = reinterpret_cast<float *>(img + (size_t)L::B_BYTES * L::NSPLIT);
        tc_pack_b_kernel<SPLIT><<<(unsigned)ceil_div(NOUT * 4 * GC, 1024), 1024, 0, st>>>(
            cin, cout, ld_cin > 0 ? ld_cin : cin, theta, theta_b, REVERSE ? 1 : 0, NOUT, GC, img, binv);
        count_launch();
        a.bimg = img;
        a.binv = binv;
    }
    a.num_tiles = ceil_div(a.total, kTcM);
    {
        static int off = -1;
        if (off < 0) {
            const char *e = getenv("FC_NO_REVPIPE32");
            off = (e && e[0] == '1') ? 1 : 0;
        }
        a.no_pipe32 = off;
    }
    static uint64_t attr = 0;
    if (first_use_on_device(attr)) {
        cudaFuncSetAttribute(tc_gmc_kernel<GC, NOUT, SPLIT, REVERSE, KFIX, DLOC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             L::SMEM);
    }
    const int grid = (int)std::min<int64_t>(a.num_tiles, num_sms());
    prof_begin(REVERSE ? (DLOC ? "tc_reverse_dloc" : "tc_reverse") : "tc_forward", st);
    tc_gmc_kernel<GC, NOUT, SPLIT, REVERSE, KFIX, DLOC><<<grid, kTcThreads, L::SMEM, st>>>(a);
    prof_end(st);
    count_launch();
    if (img) scratch_free(img, st);
    return check_launch("tc_gmc_kernel");
}

int tc_fast_reverse(bool split, int64_t total, int k, const float *rows, const float *loc, Csr csr, const float *theta,
                    const float *theta_b, float *out, const float *feat, const float *centre, float *dloc,
                    cudaStream_t st);
static bool fast_enabled();

template <int GC, int NOUT, bool SPLIT, bool REVERSE>
static int launch_tc_k(const TcArgs &a, int cin, int cout, const float *theta, const float *theta_b,
                       cudaStream_t st, int ld_cin) {
    const bool plain = a.ld_rows == GC && a.ld_out == NOUT && !a.acc && !a.acc_dloc && ld_cin == cin;
    if constexpr (REVERSE && GC == 64 && NOUT == 64) {
        if (fast_enabled() && plain && a.ld_feat == NOUT)
            return tc_fast_reverse(SPLIT, a.total, a.k, a.rows, a.loc, a.csr, theta, theta_b, a.out, a.feat, a.centre,
                                   a.dloc, st);
    }
    if (!REVERSE && a.k == kSlots)
        return launch_tc<GC, NOUT, SPLIT, REVERSE, kSlots>(a, cin, cout, theta, theta_b, st, ld_cin);
    if constexpr (REVERSE && NOUT <= 64) {
        if (a.dloc) return launch_tc<GC, NOUT, SPLIT, true, 0, true>(a, cin, cout, theta, theta_b, st, ld_cin);
    }
    if (REVERSE && a.dloc) return set_error(FC_ERR_UNSUPPORTED, "tensor-core location gradient needs c_in <= 64");
    return launch_tc<GC, NOUT, SPLIT, REVERSE, 0>(a, cin, cout, theta, theta_b, st, ld_cin);
}

template <bool SPLIT, bool REVERSE>
static int dispatch_tc(int gc, int nout, const TcArgs &a0, int cin, int cout, const float *theta,
                       const float *theta_b, cudaStream_t st, int ld_cin = -1) {
    TcArgs a = a0;  // unset strides = dense rows of the block's own width
    if (a.ld_rows == 0) a.ld_rows = gc;
    if (a.ld_out == 0) a.ld_out = nout;
    if (a.ld_feat == 0) a.ld_feat = nout;
    if (ld_cin <= 0) ld_cin = cin;
    if (gc == 64 && nout == 64) return launch_tc_k<64, 64, SPLIT, REVERSE>(a, cin, cout, theta, theta_b, st, ld_cin);
    if (gc == 64 && nout == 32) return launch_tc_k<64, 32, SPLIT, REVERSE>(a, cin, cout, theta, theta_b, st, ld_cin);
    if (gc == 32 && nout == 32) return launch_tc_k<32, 32, SPLIT, REVERSE>(a, cin, cout, theta, theta_b, st, ld_cin);
    if (gc == 32 && nout == 64) return launch_tc_k<32, 64, SPLIT, REVERSE>(a, cin, cout, theta, theta_b, st, ld_cin);
    if (gc == 32 && nout == 128) return launch_tc_k<32, 128, SPLIT, REVERSE>(a, cin, cout, theta, theta_b, st, ld_cin);
    if (gc == 32 && nout == 256) return launch_tc_k<32, 256, SPLIT, REVERSE>(a, cin, cout, theta, theta_b, st, ld_cin);
    if (!SPLIT && gc == 64 && nout == 128)
        return launch_tc_k<64, 128, false, REVERSE>(a, cin, cout, theta, theta_b, st, ld_cin);
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

void launch_pack_b_ld(bool split, int cin, int cout, int ld_cin, const float *theta, const float *theta_b, int reverse,
                      int nout, int gc, uint8_t *img, float *binv, cudaStream_t st) {
    const unsigned g = (unsigned)ceil_div((int64_t)nout * 4 * gc, 1024);
    if (split) tc_pack_b_kernel<true><<<g, 1024, 0, st>>>(cin, cout, ld_cin, theta, theta_b, reverse, nout, gc, img, binv);
    else tc_pack_b_kernel<false><<<g, 1024, 0, st>>>(cin, cout, ld_cin, theta, theta_b, reverse, nout, gc, img, binv);
    count_launch();
}
void launch_pack_b(bool split, int cin, int cout, const float *theta, const float *theta_b, int reverse, int nout,
                   int gc, uint8_t *img, float *binv, cudaStream_t st) {
    launch_pack_b_ld(split, cin, cout, cin, theta, theta_b, reverse, nout, gc, img, binv, st);
}

int tc_fast_forward(bool split, int64_t total, int64_t n, const float *feat, const float *loc, const int32_t *nbr,
                    const float *theta, const float *theta_b, float *out, cudaStream_t st,
                    const int32_t *rows = nullptr, int64_t nrows = 0);

static bool fast_enabled() {
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("FC_NO_FAST");
        on = (e && e[0] == '1') ? 0 : 1;
    }
    return on == 1;
}

int tc_conv_forward(int mode, int64_t total, int64_t n, int c_in, int d, int k, int c_out, const float *feat,
                    const float *loc, const int32_t *nbr, const float *theta, const float *theta_b, float *out,
                    cudaStream_t st) {
    (void)d;
    if (c_in == 64 && c_out == 64 && k == kSlots && fast_enabled())
        return tc_fast_forward(mode != FC_MODE_TC_BF16, total, n, feat, loc, nbr, theta, theta_b, out, st);
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

template <typename T>
int launch_dtheta_reduce(int chunks, int cin, int d, int cout, const T *partial, T *d_theta, T *d_theta_b,
                         cudaStream_t st, int tmajor = 0, int ld = 0);

// Full fp32 backward on the tensor cores (c_in = c_out = 64, d = 3):
//   tc_dtheta_kernel : d_theta partials + centre term of d_locations
//   dtheta_reduce    : fixed-order reduction of the per-CTA partials (fp64 accumulate)
//   tc_gmc (reverse) : d_features (+ neighbour term of d_locations)
// K != 8 (or FC_NO_FAST=1) would take tc_dtheta_kernel below, whose d_theta accumulates a
// CTA's whole point range in TMEM (the tensor pipe's fp32 accumulation truncates: error
// linear in the run length), so those shapes use the moments + GEMM route instead unless
// the A/B knob asks for the generic kernel, which then bounds the run per CTA by its grid.
int tc_backward_supported(int mode, int cin, int d, int k, int cout) {
    return (d == 3 && cin == 64 && cout == 64 && mode != FC_MODE_SIMT && (k == kSlots || !fast_enabled())) ? 1 : 0;
}

int tc_fast_dtheta(int64_t total, int64_t n, const float *feat, const float *loc, const int32_t *nbr, const float *g,
                   const float *theta, const float *theta_b, float *d_theta, float *d_theta_b, float *centre,
                   cudaStream_t st);

// d_theta / d_theta_b of one 64 x 64 channel block (c' block of g, c block of feat) and its
// centre-role location term, on tc_dtheta_kernel: feat / g / theta / theta_b / d_theta /
// d_theta_b point at the block's first channel; ld_* are the full row strides.  d_theta block
// rows are written with row stride ld_dt (full c_in); centre is written (acc_centre = false)
// or added to.
template <int MT = 1>
static int generic_dtheta_block(int64_t total, int64_t n, int k, const float *feat, int64_t ld_feat,
                                const float *loc, const int32_t *nbr, const float *g, int64_t ld_g,
                                const float *theta, const float *theta_b, int ld_cin, float *d_theta,
                                float *d_theta_b, int ld_dt, float *centre, bool acc_centre, cudaStream_t st,
                                const uint8_t *pimg = nullptr) {
    // pimg: this block's forward image already packed (pack_passes), else packed here
    using L = DtLayoutT<MT>;
    constexpr int cin = 64, cout = 64 * MT;  // MT c' tiles of 64 (the centre term needs MT = 1)
    if (MT > 1 && centre) return set_error(FC_ERR_UNSUPPORTED, "d_theta c' tiles > 1 without the centre term only");
    const int64_t num_tiles = ceil_div(total, kTcM);
    // at most 8 tiles (1024 points, 128 tf32 k-steps) accumulated in TMEM per CTA -- more
    // CTAs (waves) instead of a longer, truncating accumulation
    const int grid = (int)std::min<int64_t>(num_tiles, std::max<int64_t>(num_sms(), ceil_div(num_tiles, 8)));
    const size_t img_bytes = (size_t)cout * 4 * cin * 2 * 2;
    Scratch img_buf((L::Z && !pimg) ? img_bytes + 256 : 16, st);
    Scratch partial_buf(sizeof(float) * 2 * grid * cout * cin * 4, st);
    if (!img_buf.ok() || !partial_buf.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed (tc d_theta)");
    uint8_t *img = pimg ? const_cast<uint8_t *>(pimg) : img_buf.as<uint8_t>();
    float *binv = reinterpret_cast<float *>(img + img_bytes);
    if (L::Z && !pimg) {  // the forward image: B of the centre-role Z GEMM
        tc_pack_b_kernel<true><<<(unsigned)ceil_div((int64_t)cout * 4 * cin, 1024), 1024, 0, st>>>(
            cin, cout, ld_cin, theta, theta_b, 0, cout, cin, img, binv);
        count_launch();
    }
    DtArgs a{};
    a.total = total;
    a.n = n;
    a.k = k;
    a.feat = feat;
    a.loc = loc;
    a.g = g;
    a.nbr = nbr;
    a.bimg = img;
    a.binv = binv;
    a.partial = partial_buf.as<float>();
    a.centre = centre;
    a.num_tiles = num_tiles;
    a.ld_feat = ld_feat;
    a.ld_g = ld_g;
    a.acc = acc_centre ? 1 : 0;
    static uint64_t attr8 = 0, attr0 = 0;
    prof_begin("tc_dtheta", st);
    if (k == kSlots) {
        if (first_use_on_device(attr8))
            cudaFuncSetAttribute(tc_dtheta_kernel<kSlots, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
        tc_dtheta_kernel<kSlots, MT><<<grid, kTcThreads, L::SMEM, st>>>(a);
    } else {
        if (first_use_on_device(attr0))
            cudaFuncSetAttribute(tc_dtheta_kernel<0, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
        tc_dtheta_kernel<0, MT><<<grid, kTcThreads, L::SMEM, st>>>(a);
    }
    prof_end(st);
    count_launch();
    int rc = check_launch("tc_dtheta_kernel");
    if (rc || !(d_theta || d_theta_b)) return rc;
    // a block of a wider theta is written in place (row stride ld_dt)
    return launch_dtheta_reduce<float>(2 * grid, cin, 3, cout, a.partial, d_theta, d_theta_b, st, 0, ld_dt);
}

// Without the location gradient, d_theta and d_features of a backward are independent: the
// d_theta kernels go to a side stream while the reverse pass runs on the caller's, so one
// latency-bound kernel's tail overlaps the other's start (fork / join by events, so a graph
// capture of the caller's stream includes it; FC_NO_SIDE_BWD=1 runs them in sequence).
struct SideFork {
    cudaStream_t main, side;
    bool on;
    cudaEvent_t join_ev{};
    SideFork(cudaStream_t m, bool enable) : main(m), side(m), on(false) {
        static int off = -1;
        if (off < 0) {
            const char *e = getenv("FC_NO_SIDE_BWD");
            off = (e && e[0] == '1') ? 1 : 0;
        }
        if (!enable || off) return;
        static thread_local cudaStream_t ss[64];
        static thread_local cudaEvent_t ev[64][2];
        static thread_local uint64_t made = 0;
        const int dev = current_device() & 63;
        if (first_use_on_device(made)) {
            cudaStreamCreateWithFlags(&ss[dev], cudaStreamNonBlocking);
            cudaEventCreateWithFlags(&ev[dev][0], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&ev[dev][1], cudaEventDisableTiming);
        }
        on = true;
        side = ss[dev];
        join_ev = ev[dev][1];
        cudaEventRecord(ev[dev][0], m);
        cudaStreamWaitEvent(side, ev[dev][0], 0);
    }
    void join() {
        if (!on) return;
        cudaEventRecord(join_ev, side);
        cudaStreamWaitEvent(main, join_ev, 0);
        on = false;
    }
    ~SideFork() { join(); }
};

int tc_backward(int mode, int64_t total, int64_t n, int cin, int d, int k, int cout, const float *g,
                const float *feat, const float *loc, const int32_t *nbr, Csr csr, const float *theta,
                const float *theta_b, float *d_features, float *d_locations, float *d_theta, float *d_theta_b,
                cudaStream_t st) {
    (void)d;
    using L = DtLayout;
    // without d_locations the d_theta kernels run on a side stream beside the reverse pass
    SideFork sf(st, !d_locations && d_features && (d_theta || d_theta_b));
    const int64_t num_tiles = ceil_div(total, kTcM);
    // generic d_theta kernel: at most 8 tiles (1024 points, 128 tf32 k-steps) accumulated in
    // TMEM per CTA -- more CTAs (waves) instead of a longer truncating accumulation
    const int grid = (int)std::min<int64_t>(num_tiles, std::max<int64_t>(num_sms(), ceil_div(num_tiles, 8)));
    Scratch centre_buf;
    float *centre = nullptr;
    int rc = FC_OK;
    if ((d_theta || d_theta_b || d_locations) && k == kSlots && fast_enabled()) {
        if (d_locations) {
            centre_buf.alloc(sizeof(float) * total * 3, st);
            if (!centre_buf.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed (tc backward)");
            centre = centre_buf.as<float>();
        }
        rc = tc_fast_dtheta(total, n, feat, loc, nbr, g, theta, theta_b, d_theta, d_theta_b, centre, sf.side);
        if (rc) return rc;
    } else if (d_theta || d_theta_b || d_locations) {
        centre_buf.alloc(sizeof(float) * total * 3, sf.side);
        if (!centre_buf.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed (tc backward)");
        centre = centre_buf.as<float>();
        rc = generic_dtheta_block(total, n, k, feat, cin, loc, nbr, g, cout, theta, theta_b, cin, d_theta, d_theta_b,
                                  cin, centre, false, sf.side);
        if (rc) return rc;
    }
    if (d_features || d_locations) {
        float *df = d_features;
        Scratch df_buf;
        if (!df) {
            df_buf.alloc(sizeof(float) * total * cin, st);
            if (!df_buf.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed (tc backward)");
            df = df_buf.as<float>();
        }
        TcArgs a{};
        a.total = total;
        a.n = n;
        a.k = k;
        a.rows = g;
        a.loc = loc;
        a.csr = csr;
        a.out = df;
        a.feat = feat;
        a.centre = centre;
        a.dloc = d_locations;
        if (mode == FC_MODE_TC_BF16) rc = dispatch_tc<false, true>(cout, cin, a, cin, cout, theta, theta_b, st);
        else rc = dispatch_tc<true, true>(cout, cin, a, cin, cout, theta, theta_b, st);
    }
    return rc;
}

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


// ---------------------------------------------------------------------------------
// Wide shapes on the tensor cores (C2's 64 -> 128, the U-Net's 128 / 256 channels): the
// channels are cut into 64-wide blocks and every (gathered block, output block) pair runs
// the 64 x 64 engines above (the A tile of one block fits shared memory, the whole
// operand does not); the K-blocks of one output block accumulate in its epilogue (out +=,
// in ascending block order: deterministic), d_theta is assembled block by block, and the
// location gradient's two roles accumulate over all block pairs.  The gathers are repeated
// once per output block -- the price of keeping the moments on chip instead of writing
// [points, 4 C] moment rows to HBM for a library GEMM.
// ---- small clouds: the blocked passes run CONCURRENTLY on per-device side streams (each
// pass is one latency-bound wave on tiles <= a few dozen SMs, e.g. C2's 8 K points are 64
// tiles), every pass into its own buffer, then combined on the caller's stream in the same
// order as the sequential accumulation (identical results; fork / join by events, so a CUDA
// graph capture of the caller's stream includes them).
struct ForkJoin {
    cudaStream_t main;
    int n = 0;
    bool on = false;
    cudaStream_t s[4];
    cudaEvent_t fork_ev, join_ev[4];
    // pool: which set of side streams (two fork / joins in flight at once -- d_theta's passes
    // beside the reverse pass's -- must not share streams, or they would serialise)
    ForkJoin(cudaStream_t m, int jobs, bool enable, int pool = 0)
        : main(m), n(jobs), on(enable && jobs > 1 && jobs <= 4) {
        for (int j = 0; j < 4; ++j) s[j] = m;
        if (!on) return;
        // per host thread and device: two threads forking on one device must not share events
        static thread_local cudaStream_t aux[64][2][4];
        static thread_local cudaEvent_t evs[64][2][5];
        static thread_local uint64_t made = 0;
        const int dev = current_device() & 63;
        if (first_use_on_device(made)) {
            for (int q = 0; q < 2; ++q) {
                for (int j = 0; j < 4; ++j) cudaStreamCreateWithFlags(&aux[dev][q][j], cudaStreamNonBlocking);
                for (int j = 0; j < 5; ++j) cudaEventCreateWithFlags(&evs[dev][q][j], cudaEventDisableTiming);
            }
        }
        pool &= 1;
        fork_ev = evs[dev][pool][4];
        cudaEventRecord(fork_ev, m);
        for (int j = 0; j < n; ++j) {
            s[j] = aux[dev][pool][j];
            join_ev[j] = evs[dev][pool][j];
            cudaStreamWaitEvent(s[j], fork_ev, 0);
        }
    }
    cudaStream_t operator[](int j) const { return s[j]; }
    void join() {
        if (!on) return;
        for (int j = 0; j < n; ++j) {
            cudaEventRecord(join_ev[j], s[j]);
            cudaStreamWaitEvent(main, join_ev[j], 0);
        }
    }
};
static bool concurrent_passes(int64_t total, int passes) {
    static int off = -1;
    if (off < 0) {
        const char *e = getenv("FC_NO_CONCURRENT");
        off = (e && e[0] == '1') ? 1 : 0;
    }
    return !off && passes > 1 && passes <= 4 && ceil_div(total, kTcM) * passes <= 2 * num_sms();
}

// dst[p, 0:w] (row stride ldd) += src[p, 0:w] (row stride lds), p < rows
__global__ void add_rows_kernel(int64_t rows, int w, float *__restrict__ dst, int64_t ldd, const float *__restrict__ src,
                                int64_t lds) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * w; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = e / w;
        const int c = (int)(e - p * w);
        dst[p * ldd + c] += src[p * lds + c];
    }
}
static void add_rows(int64_t rows, int w, float *dst, int64_t ldd, const float *src, int64_t lds, cudaStream_t st) {
    add_rows_kernel<<<(unsigned)std::min<int64_t>(ceil_div(rows * w, 256), 4 * num_sms()), 256, 0, st>>>(rows, w, dst,
                                                                                                          ldd, src, lds);
    count_launch();
}

// The B images of a blocked call's passes (one shape, njobs blocks of theta) packed up front
// in one launch instead of one small, latency-bound launch ahead of every pass: image j at
// buf + j * stride, its 1 / scale right after its bytes.
static int pack_passes(bool split, int cin, int cout, int ld_cin, int reverse, int nout, int gc, int njobs,
                       const float *const *th, const float *const *tb, Scratch &buf, int64_t &stride, cudaStream_t st) {
    const int64_t bbytes = (int64_t)nout * 4 * gc * 2 * (split ? 2 : 1);
    stride = (bbytes + 256 + 1023) / 1024 * 1024;
    buf.alloc((size_t)(stride * njobs), st);
    if (!buf.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed (pass images)");
    const unsigned gx = (unsigned)ceil_div((int64_t)nout * 4 * gc, 1024);
    for (int j0 = 0; j0 < njobs; j0 += kPackBatch) {
        const int nj = std::min(kPackBatch, njobs - j0);
        PackBatch pb{};
        for (int j = 0; j < nj; ++j) {
            pb.theta[j] = th[j0 + j];
            pb.theta_b[j] = tb[j0 + j];
        }
        uint8_t *img0 = buf.as<uint8_t>() + (int64_t)j0 * stride;
        const dim3 grid(gx, (unsigned)nj);
        if (split) tc_pack_b_batch_kernel<true><<<grid, 1024, 0, st>>>(cin, cout, ld_cin, reverse, nout, gc, img0, stride, bbytes, pb);
        else tc_pack_b_batch_kernel<false><<<grid, 1024, 0, st>>>(cin, cout, ld_cin, reverse, nout, gc, img0, stride, bbytes, pb);
        count_launch();
    }
    return check_launch("pack passes");
}

// output channels per pass of the channel-blocked engines: all of them up to 256
static int blocked_out_block(int c) {
    if (c <= 256) return c % 64 == 0 && c != 192 ? c : 64;
    return c % 256 == 0 ? 256 : (c % 128 == 0 ? 128 : 64);
}

int tc_blocked_supported(int mode, int c_in, int d, int c_out) {
    return (d == 3 && mode != FC_MODE_SIMT && c_in % 64 == 0 && c_out % 64 == 0 && (c_in > 64 || c_out > 64)) ? 1 : 0;
}

int tc_fast_forward_block(bool split, int64_t total, int64_t n, const float *feat, int64_t ld_feat, const float *loc,
                          const int32_t *nbr, const float *theta, const float *theta_b, int ld_cin, float *out,
                          int64_t ld_out, bool acc, cudaStream_t st, const int32_t *rows, int64_t nrows,
                          const uint8_t *pre_img);
int64_t fast_forward_image_stride(bool split);
int pack_forward_blocks(bool split, int njobs, const float *const *th, const float *const *tb, int ld_cin,
                        uint8_t *img0, cudaStream_t st);

// Channel blocks on the 64 -> 64 K = 8 headline kernels (warp-specialised gather, 8-channel
// lanes): for clouds large enough to fill the GPU with one pass, each of the
// (c_in / 64) x (c_out / 64) block pairs is one fast pass, the input blocks of an output
// block accumulated in ascending order in the epilogue.  FC_BLOCK_FAST=0 keeps the generic
// 32-channel-gather engine below for A/B.
static bool block_fast(int64_t total, int k, int c_in, int c_out) {
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("FC_BLOCK_FAST");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on && fast_enabled() && k == kSlots && c_in % 64 == 0 && c_out % 64 == 0 &&
           ceil_div(total, kTcM) >= num_sms();
}

int tc_blocked_forward(int mode, int64_t total, int64_t n, int c_in, int k, int c_out, const float *feat,
                       const float *loc, const int32_t *nbr, const float *theta, const float *theta_b, float *out,
                       cudaStream_t st) {
    if (block_fast(total, k, c_in, c_out)) {
        const bool split = mode != FC_MODE_TC_BF16;
        std::vector<const float *> th, tb;  // all passes' images packed up front, one launch
        for (int o0 = 0; o0 < c_out; o0 += 64)
            for (int i0 = 0; i0 < c_in; i0 += 64) {
                th.push_back(theta + ((int64_t)o0 * c_in + i0) * 3);
                tb.push_back(theta_b + (int64_t)o0 * c_in + i0);
            }
        const int64_t stride = fast_forward_image_stride(split);
        Scratch imgs((size_t)stride * th.size(), st);
        if (!imgs.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed (block images)");
        int rc = pack_forward_blocks(split, (int)th.size(), th.data(), tb.data(), c_in, imgs.as<uint8_t>(), st);
        int pass = 0;
        for (int o0 = 0; o0 < c_out && rc == FC_OK; o0 += 64)
            for (int i0 = 0; i0 < c_in && rc == FC_OK; i0 += 64, ++pass)
                rc = tc_fast_forward_block(split, total, n, feat + i0, c_in, loc, nbr, th[pass], tb[pass], c_in, out + o0,
                                           c_out, i0 > 0, st, nullptr, 0, imgs.as<uint8_t>() + pass * stride);
        return rc;
    }
    // each 32-channel block of the input is gathered ONCE and contracted against all (up to
    // 256) output channels in one pass (N = 128 / 256 accumulators), the blocks' products
    // summed in the epilogue (acc): the gather -- the kernel's cost -- is not repeated per
    // output block
    const int ob = blocked_out_block(c_out);
    const int gb = ob > 64 ? 32 : 64;  // 64-channel gathers where the output block is 64 wide
    const int nin = (int)ceil_div(c_in, gb), nout = (int)ceil_div(c_out, ob);
    const bool conc = nout == 1 && concurrent_passes(total, nin);
    Scratch tmp;
    if (conc) {  // passes 1.. write [total, ob] partials, added to out in pass order afterwards
        tmp.alloc(sizeof(float) * (size_t)(nin - 1) * total * ob, st);
        if (!tmp.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed (blocked forward)");
    }
    Scratch imgs;
    int64_t istride = 0;
    {
        std::vector<const float *> th, tb;
        for (int o0 = 0; o0 < c_out; o0 += ob)
            for (int i0 = 0; i0 < c_in; i0 += gb) {
                th.push_back(theta + ((int64_t)o0 * c_in + i0) * 3);
                tb.push_back(theta_b + (int64_t)o0 * c_in + i0);
            }
        const int rc0 = pack_passes(mode != FC_MODE_TC_BF16, gb, ob, c_in, 0, ob, gb, (int)th.size(), th.data(), tb.data(),
                                    imgs, istride, st);
        if (rc0) return rc0;
    }
    ForkJoin fj(st, nin, conc);
    int rc = FC_OK;
    int pass = 0;
    for (int o0 = 0; o0 < c_out && rc == FC_OK; o0 += ob) {
        for (int i0 = 0, b = 0; i0 < c_in; i0 += gb, ++b) {
            TcArgs a{};
            a.total = total;
            a.n = n;
            a.k = k;
            a.rows = feat + i0;
            a.ld_rows = c_in;
            a.loc = loc;
            a.nbr = nbr;
            a.out = (conc && b > 0) ? tmp.as<float>() + (size_t)(b - 1) * total * ob : out + o0;
            a.ld_out = (conc && b > 0) ? ob : c_out;
            a.acc = !conc && i0 > 0;
            a.bimg = imgs.as<uint8_t>() + pass * istride;
            a.binv = reinterpret_cast<const float *>(a.bimg + (ob * 4 * gb * 2 * (mode != FC_MODE_TC_BF16 ? 2 : 1)));
            ++pass;
            const float *th = theta + ((int64_t)o0 * c_in + i0) * 3, *tb = theta_b + (int64_t)o0 * c_in + i0;
            const cudaStream_t sj = conc ? fj[b] : st;
            rc = mode == FC_MODE_TC_BF16 ? dispatch_tc<false, false>(gb, ob, a, gb, ob, th, tb, sj, c_in)
                                         : dispatch_tc<true, false>(gb, ob, a, gb, ob, th, tb, sj, c_in);
            if (rc) break;
        }
    }
    fj.join();
    if (rc) return rc;
    for (int b = 1; conc && b < nin; ++b) add_rows(total, ob, out, c_out, tmp.as<float>() + (size_t)(b - 1) * total * ob, ob, st);
    return check_launch("blocked forward");
}

// Reverse pass over blocks: out [total, c_in] = sum over gathered c' blocks of the block
// products (d_features of the backward, or flex_deconv); with dloc, the neighbour role of
// the location gradient (dloc = centre - sum of the blocks' terms).
int tc_fast_reverse_block(bool split, int64_t total, int k, const float *rows, int64_t ld_rows, const float *loc,
                          Csr csr, const float *theta, const float *theta_b, int ld_cin, float *out, int64_t ld_out,
                          bool acc, cudaStream_t st, const uint8_t *pre_img, const float *pre_zero);

// late_centre (with dloc): the centre term is still being computed on late_join's side
// stream; every pass runs against a zero centre and the centre is added after the join,
// right after pass 0's term and before the later passes' (so the additions are the sequential
// order's: (c - t0) - t1 ... = ((0 - t0) + c) + (0 - t1) ...).  Needs the concurrent-pass form
// (or one pass); the caller checks blocked_reverse_late_ok.
static int tc_blocked_reverse(int mode, int64_t total, int64_t n, int c_in, int k, int c_out, const float *rows,
                              const float *loc, Csr csr, const float *theta, const float *theta_b, float *out,
                              const float *feat, const float *centre, float *dloc, cudaStream_t st,
                              const float *late_centre = nullptr, SideFork *late_join = nullptr) {
    if (!dloc && block_fast(total, k, c_in, c_out)) {  // 64 x 64 blocks on the headline reverse kernel
        const bool split = mode != FC_MODE_TC_BF16;
        std::vector<const float *> th, tb;  // all passes' images packed up front, one launch
        for (int i0 = 0; i0 < c_in; i0 += 64)
            for (int j0 = 0; j0 < c_out; j0 += 64) {
                th.push_back(theta + ((int64_t)j0 * c_in + i0) * 3);
                tb.push_back(theta_b + (int64_t)j0 * c_in + i0);
            }
        Scratch imgs, zero(256, st);
        int64_t stride = 0;
        int rc = zero.ok() ? pack_passes(split, 64, 64, c_in, 1, 64, 64, (int)th.size(), th.data(), tb.data(), imgs, stride, st)
                           : set_error(FC_ERR_CUDA, "scratch allocation failed (block images)");
        if (rc == FC_OK) cudaMemsetAsync(zero.p, 0, 256, st);
        int pass = 0;
        for (int i0 = 0; i0 < c_in && rc == FC_OK; i0 += 64)
            for (int j0 = 0; j0 < c_out && rc == FC_OK; j0 += 64, ++pass)
                rc = tc_fast_reverse_block(split, total, k, rows + j0, c_out, loc, csr, th[pass], tb[pass], c_in, out + i0,
                                           c_in, j0 > 0, st, imgs.as<uint8_t>() + pass * stride, zero.as<float>());
        return rc;
    }
    // gathered (c') blocks of 32 channels, each gathered once per output block of up to 256
    // channels (64-channel gathers for a 64-wide output block, e.g. with the location-gradient
    // epilogue, whose U accumulators need 4x the columns)
    const int ob = dloc ? 64 : blocked_out_block(c_in);
    const int gb = ob > 64 ? 32 : 64;
    const int nj = (int)ceil_div(c_out, gb), ni = (int)ceil_div(c_in, ob);
    const bool conc = ni == 1 && concurrent_passes(total, nj);
    const bool late = dloc && late_centre;
    if (late && !(conc || (ni == 1 && nj == 1))) return set_error(FC_ERR_CONFIG, "late centre needs one block row");
    Scratch tmp, tdl, zero3;
    if (conc) {  // passes 1.. write their d_features part and (-) location term to side buffers
        tmp.alloc(sizeof(float) * (size_t)(nj - 1) * total * ob, st);
        if (dloc) tdl.alloc(sizeof(float) * (size_t)(nj - 1) * total * 3, st);
        if (!tmp.ok() || (dloc && !tdl.ok())) return set_error(FC_ERR_CUDA, "scratch allocation failed (blocked reverse)");
    }
    if (dloc && (conc || late)) {
        zero3.alloc(sizeof(float) * (size_t)total * 3, st);
        if (!zero3.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed (blocked reverse)");
        cudaMemsetAsync(zero3.p, 0, sizeof(float) * total * 3, st);
    }
    Scratch imgs;
    int64_t istride = 0;
    {
        std::vector<const float *> th, tb;
        for (int i0 = 0; i0 < c_in; i0 += ob)
            for (int j0 = 0; j0 < c_out; j0 += gb) {
                th.push_back(theta + ((int64_t)j0 * c_in + i0) * 3);
                tb.push_back(theta_b + (int64_t)j0 * c_in + i0);
            }
        const int rc0 = pack_passes(mode != FC_MODE_TC_BF16, ob, gb, c_in, 1, ob, gb, (int)th.size(), th.data(), tb.data(),
                                    imgs, istride, st);
        if (rc0) return rc0;
    }
    ForkJoin fj(st, nj, conc);
    int rc = FC_OK;
    int pass = 0;
    for (int i0 = 0; i0 < c_in && rc == FC_OK; i0 += ob) {
        for (int j0 = 0, b = 0; j0 < c_out; j0 += gb, ++b) {
            const bool side = conc && b > 0;
            TcArgs a{};
            a.total = total;
            a.n = n;
            a.k = k;
            a.rows = rows + j0;
            a.ld_rows = c_out;
            a.loc = loc;
            a.csr = csr;
            a.out = side ? tmp.as<float>() + (size_t)(b - 1) * total * ob : out + i0;
            a.ld_out = side ? ob : c_in;
            a.acc = !conc && j0 > 0;
            if (dloc) {
                a.feat = feat + i0;
                a.ld_feat = c_in;
                // side passes: dloc_b = 0 - term_b (exact negation), added below: (c - t0) - t1
                a.centre = (side || late) ? zero3.as<float>() : centre;
                a.dloc = side ? tdl.as<float>() + (size_t)(b - 1) * total * 3 : dloc;
                a.acc_dloc = !conc && (i0 > 0 || j0 > 0);
            }
            a.bimg = imgs.as<uint8_t>() + pass * istride;
            a.binv = reinterpret_cast<const float *>(a.bimg + (ob * 4 * gb * 2 * (mode != FC_MODE_TC_BF16 ? 2 : 1)));
            ++pass;
            const float *th = theta + ((int64_t)j0 * c_in + i0) * 3, *tb = theta_b + (int64_t)j0 * c_in + i0;
            const cudaStream_t sj = conc ? fj[b] : st;
            rc = mode == FC_MODE_TC_BF16 ? dispatch_tc<false, true>(gb, ob, a, ob, gb, th, tb, sj, c_in)
                                         : dispatch_tc<true, true>(gb, ob, a, ob, gb, th, tb, sj, c_in);
            if (rc) break;
        }
    }
    fj.join();
    if (late) {  // the centre term: pass 0's (0 - t0) + c
        late_join->join();
        if (rc == FC_OK) add_rows(total, 3, dloc, 3, late_centre, 3, st);
    }
    if (rc) return rc;
    for (int b = 1; conc && b < nj; ++b) {
        add_rows(total, ob, out, c_in, tmp.as<float>() + (size_t)(b - 1) * total * ob, ob, st);
        if (dloc) add_rows(total, 3, dloc, 3, tdl.as<float>() + (size_t)(b - 1) * total * 3, 3, st);
    }
    return check_launch("blocked reverse");
}

int tc_blocked_deconv(int mode, int64_t total, int64_t n, int c_in, int k, int c_out, const float *x,
                      const float *loc, Csr csr, const float *theta, const float *theta_b, float *y, cudaStream_t st) {
    return tc_blocked_reverse(mode, total, n, c_in, k, c_out, x, loc, csr, theta, theta_b, y, nullptr, nullptr,
                              nullptr, st);
}

int tc_blocked_backward(int mode, int64_t total, int64_t n, int c_in, int k, int c_out, const float *g,
                        const float *feat, const float *loc, const int32_t *nbr, Csr csr, const float *theta,
                        const float *theta_b, float *d_features, float *d_locations, float *d_theta,
                        float *d_theta_b, cudaStream_t st0) {
    // without the location gradient, c' tiles of 128 (each 64-channel feature block is
    // gathered once per 128 upstream channels)
    const int jb = (!d_locations && c_out % 128 == 0) ? 128 : 64;
    const int npass = (int)(ceil_div(c_out, jb) * ceil_div(c_in, 64));
    const bool conc = concurrent_passes(total, npass);
    // small clouds with the location gradient: the reverse pass need not wait for the centre
    // term (tc_blocked_reverse's late centre), so d_theta runs beside it there too
    const int rni = (int)ceil_div(c_in, 64), rnj = (int)ceil_div(c_out, 64);
    const bool late = d_locations && d_features && conc && rni == 1 && (rnj == 1 || concurrent_passes(total, rnj));
    Scratch centre_buf;  // (allocated before the fork: the side stream writes it)
    if (d_locations) {
        centre_buf.alloc(sizeof(float) * total * 3, st0);
        if (!centre_buf.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed (blocked backward)");
    }
    SideFork sf(st0, (!d_locations && d_features && (d_theta || d_theta_b)) || late);
    const cudaStream_t st = sf.side;  // d_theta section (the caller's stream unless forked)
    if (d_theta || d_theta_b || d_locations) {
        Scratch cside;  // concurrent passes 1..: their own centre terms, added in pass order below
        if (conc && d_locations) {
            cside.alloc(sizeof(float) * (size_t)(npass - 1) * total * 3, st);
            if (!cside.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed (blocked backward)");
        }
        Scratch imgs;  // the forward images of the centre-role Z GEMMs (64-wide c' tiles only)
        int64_t istride = 0;
        if (jb == 64) {
            std::vector<const float *> th, tb;
            for (int j0 = 0; j0 < c_out; j0 += jb)
                for (int i0 = 0; i0 < c_in; i0 += 64) {
                    th.push_back(theta + ((int64_t)j0 * c_in + i0) * 3);
                    tb.push_back(theta_b + (int64_t)j0 * c_in + i0);
                }
            const int rc0 = pack_passes(true, 64, 64, c_in, 0, 64, 64, (int)th.size(), th.data(), tb.data(), imgs, istride, st);
            if (rc0) return rc0;
        }
        ForkJoin fj(st, npass, conc, sf.on ? 1 : 0);  // (its own side streams beside the reverse pass's)
        int rc = FC_OK;
        int b = 0;
        for (int j0 = 0; j0 < c_out && rc == FC_OK; j0 += jb) {
            for (int i0 = 0; i0 < c_in; i0 += 64, ++b) {
                // the centre term needs every block pair; d_theta blocks are independent
                const int64_t e0 = (int64_t)j0 * c_in + i0;
                float *dtp = d_theta ? d_theta + e0 * 3 : nullptr, *dtbp = d_theta_b ? d_theta_b + e0 : nullptr;
                const cudaStream_t sj = conc ? fj[b] : st;
                float *cen = !d_locations ? nullptr
                             : (conc && b > 0) ? cside.as<float>() + (size_t)(b - 1) * total * 3 : centre_buf.as<float>();
                rc = jb == 128 ? generic_dtheta_block<2>(total, n, k, feat + i0, c_in, loc, nbr, g + j0, c_out,
                                                         theta + e0 * 3, theta_b + e0, c_in, dtp, dtbp, c_in, nullptr,
                                                         false, sj)
                               : generic_dtheta_block<1>(total, n, k, feat + i0, c_in, loc, nbr, g + j0, c_out,
                                                         theta + e0 * 3, theta_b + e0, c_in, dtp, dtbp, c_in, cen,
                                                         !conc && (j0 > 0 || i0 > 0), sj, imgs.as<uint8_t>() + b * istride);
                if (rc) break;
            }
        }
        fj.join();
        if (rc) return rc;
        for (int q = 1; conc && d_locations && q < npass; ++q)
            add_rows(total, 3, centre_buf.as<float>(), 3, cside.as<float>() + (size_t)(q - 1) * total * 3, 3, st);
    }
    if (d_features || d_locations) {
        Scratch df_buf;
        float *df = d_features;
        if (!df) {
            df_buf.alloc(sizeof(float) * total * c_in, st0);
            if (!df_buf.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed (blocked backward)");
            df = df_buf.as<float>();
        }
        const int rc = tc_blocked_reverse(mode, total, n, c_in, k, c_out, g, loc, csr, theta, theta_b, df, feat,
                                          centre_buf.as<float>(), d_locations, st0, late ? centre_buf.as<float>() : nullptr,
                                          late ? &sf : nullptr);
        sf.join();
        return rc;
    }
    return FC_OK;
}

}  // namespace fc
