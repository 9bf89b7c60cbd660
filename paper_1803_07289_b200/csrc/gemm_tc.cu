// gemm_tc.cu -- the pointwise (1x1) convolutions of the U-Net / classifier step (SURVEY.md
// §8(f)-1; reference flexops.py:206-226 pointwise_conv, network.py:94-122 _Pointwise and the
// concatenations feeding them, network.py:180-246) as fp32-accurate tcgen05 GEMMs.
//
//   rows:  Y[p, :] = bias + [A_0 | A_1 | ...][p, :] . B^T      (forward: B = W; d_input:
//          A_0 = G (optionally masked by a saved pre-activation, G * (Z > 0)), B = W^T)
//   wgrad: dW = G^T [X_0 | X_1 | ...], db = sum_p G[p, :]        (SIMT, fixed-order partials)
//
// The concatenation [A_0 | A_1 | ...] (features | skip | coordinates) is never built: each
// operand contributes its own 32-column K-blocks.  Precision: kind::tf32 with a hi/lo split of
// both operands (A_hi = the fp32 value, which the tensor core truncates to tf32; A_lo = the
// exact remainder), D = A_hi.[B_hi; B_lo] + A_lo.[B_hi; B_lo] as two MMAs of N = 2 nc per
// 8-wide k-step, the halves of D summed in the epilogue: ~2^-21 relative per product, no
// per-row scaling (tf32 keeps the fp32 exponent range) -- so any row / operand mix works.
// Epilogue: + bias, the result to up to four column ranges (per-operand d_input outputs) and
// optionally ReLU(result) to a second buffer (the ResBlock's r and relu(r) in one pass).
#include <cstdio>
#include <cstdlib>

#include "fast_common.cuh"

namespace fc {
using namespace sm100;

namespace gemm {
using fast::ldg_nc4;
using fast::sts128f;
using fast::lds128f;
using fast::ffma2;

constexpr int kMaxOps = 4;
constexpr int kMaxOuts = 4;
constexpr int kThreads = 256;
constexpr int kTileM = 128;
constexpr int kA = kTileM * 128;  // one fp32 K-block image: 128 rows x 32 columns (16 KB)

struct Op {
    const float *a;
    int64_t lda;
    int k;    // columns of this operand
    int kb0;  // first K-block (rows) / first concatenated column (wgrad)
};
struct Out {
    float *p;
    int64_t ld;
    int c0, c1;  // output columns [c0, c1) -> p[:, 0 .. c1 - c0)
};
struct Args {
    int64_t n;
    int nops;
    Op ops[kMaxOps];
    int kblocks;
    const float *mask;  // operand 0 *= (mask > 0) (nullable)
    int64_t mask_ld;
    const uint8_t *bimg;
    int nc, nchunks, ncols;
    const float *bias;
    int nouts;
    Out outs[kMaxOuts];
    float *relu;
    int64_t relu_ld;
};

__host__ __device__ inline int chunk_cols(int ncols) { return std::min(128, (int)((ncols + 15) / 16 * 16)); }
__host__ __device__ inline int64_t image_bytes(int ncols, int kblocks) {
    const int nc = chunk_cols(ncols);
    return (int64_t)ceil_div(ncols, nc) * kblocks * 2 * nc * 128;
}

// kind::tf32, fp32 accumulate, both operands K-major
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(
            d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ float tf32_lo(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xffffe000u); }
// byte offset of 16-byte chunk c (0..7) of row r in a 128-byte-row SW128 K-major image
__device__ __forceinline__ uint32_t sw_chunk(int r, int c) {
    return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4));
}

// B image: chunk ch (nc output columns) x K-block kb -> [2 nc rows: hi then lo] x 128 B.
// Element (row n, column k) of B: transpose ? w[k * ldw + n] : w[n * ldw + k], where the
// K axis is the concatenation of segments (src column / row offset, width), each padded to
// whole 32-column K-blocks.
struct PackArgs {
    const float *w;
    int64_t ldw;
    int transpose;
    int nrows, nc, kblocks;
    int nseg;
    int seg_src[kMaxOps], seg_k[kMaxOps], seg_kb0[kMaxOps];
    uint8_t *img;
};
__global__ void pack_b_kernel(PackArgs a) {
    const int64_t total = (int64_t)ceil_div(a.nrows, a.nc) * a.kblocks * a.nc * 32;  // (row, k) pairs
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int kk = (int)(idx & 31);
        const int64_t r1 = idx >> 5;
        const int rr = (int)(r1 % a.nc);
        const int64_t r2 = r1 / a.nc;
        const int kb = (int)(r2 % a.kblocks);
        const int ch = (int)(r2 / a.kblocks);
        const int n = ch * a.nc + rr;
        float v = 0.f;
        if (n < a.nrows) {
#pragma unroll
            for (int s = 0; s < kMaxOps; ++s) {  // (compile-time indices: the segment table stays in registers)
                if (s >= a.nseg) break;
                const int kl = (kb - a.seg_kb0[s]) * 32 + kk;
                if (kb >= a.seg_kb0[s] && kl < a.seg_k[s]) {
                    const int kc = a.seg_src[s] + kl;
                    v = a.transpose ? a.w[(int64_t)kc * a.ldw + n] : a.w[(int64_t)n * a.ldw + kc];
                }
            }
        }
        const float hi = __uint_as_float(__float_as_uint(v) & 0xffffe000u);
        uint8_t *blk = a.img + ((int64_t)ch * a.kblocks + kb) * (2 * a.nc * 128);
        const uint32_t o = sw_chunk(rr, kk >> 2) + (uint32_t)(kk & 3) * 4u;
        *reinterpret_cast<float *>(blk + o) = v;  // hi: the tensor core reads the tf32 part
        *reinterpret_cast<float *>(blk + sw_chunk(a.nc + rr, kk >> 2) + (uint32_t)(kk & 3) * 4u) = v - hi;
    }
}

__device__ __forceinline__ void cpa16(uint32_t dst, const void *src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cpa4(uint32_t dst, const void *src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Pipeline: iteration j = (tile, chunk, K-block) of this CTA; the raw fp32 A block (= the hi
// operand: the tensor core reads its tf32 part) and the packed B block are copied with
// cp.async kStages - 1 iterations ahead (zero-filled past the rows / columns); a short pass
// over the landed block writes the lo operand (and applies the ReLU mask); one thread issues
// the MMAs.  K-block partials accumulate in two alternating TMEM accumulators and are summed
// in fp32 registers (round-to-nearest): the tensor pipe's fp32 accumulation truncates, so a
// long K in one accumulator drifts (~2^-24 per MMA, biased; measured 3.5x the SGEMM error on
// the U-Net's 387-wide merge GEMM before this change).
// kStages: cp.async stages; 3 (1 CTA / SM, TMEM 512) or, for nc <= 64 (2 x 2nc <= 256 TMEM
// columns), 2 (two CTAs / SM: twice the warps to hide the per-K-block dependency chain)
template <int kStages>
__global__ void __launch_bounds__(kThreads, kStages == 2 ? 2 : 1) gemm_rows_kernel(Args a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sb = smem_u32(smem);
    const int bstage = 2 * a.nc * 128;
    const int stage = 2 * kA + bstage;
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + kStages * stage);
    uint64_t *mma_done = bar;         // [kStages]
    uint64_t *dfull = bar + kStages;  // [2] K-block accumulator ready
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bar + kStages + 2);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(mma_done + s, 1);
        mbar_init(dfull, 1);
        mbar_init(dfull + 1, 1);
        fence_mbar_init();
    }
    constexpr uint32_t kCols = kStages == 3 ? 512 : 256;
    if (warp == 0) tmem_alloc(tmem_holder, kCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    const int64_t tiles = ceil_div(a.n, kTileM);
    const int64_t my_tiles = tiles > blockIdx.x ? ceil_div(tiles - blockIdx.x, gridDim.x) : 0;
    const int per_tile = a.nchunks * a.kblocks;
    const int64_t total = my_tiles * per_tile;
    const uint32_t idesc = idesc_tf32(kTileM, 2 * a.nc);
    const int r = tid >> 1, hf = tid & 1;  // A rows: row r, columns 16 hf .. +15 of the K-block

    auto issue = [&](int64_t j) {  // cp.async of iteration j into stage j % kStages
        if (j < total) {
            const int64_t tile = blockIdx.x + (j / per_tile) * gridDim.x;
            const int rem = (int)(j % per_tile), ch = rem / a.kblocks, kb = rem % a.kblocks;
            const uint32_t As = sb + (uint32_t)((j % kStages) * stage), Bs = As + 2 * kA;
            int q = 0;
            while (q + 1 < a.nops && kb >= a.ops[q + 1].kb0) ++q;
            const Op op = a.ops[q];
            const int col0 = (kb - op.kb0) * 32 + 16 * hf;
            const int64_t p = tile * kTileM + r;
            const bool pv = p < a.n;
            const float *src = op.a + (pv ? p : 0) * op.lda + col0;
            if (((op.lda & 3) == 0) && ((reinterpret_cast<uintptr_t>(op.a) & 15) == 0) && (op.k & 3) == 0) {
#pragma unroll
                for (int c = 0; c < 4; ++c) cpa16(As + sw_chunk(r, 4 * hf + c), src + 4 * c, pv && col0 + 4 * c < op.k);
            } else {
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    cpa4(As + sw_chunk(r, 4 * hf + (e >> 2)) + (uint32_t)(e & 3) * 4u, src + e, pv && col0 + e < op.k);
            }
            const uint8_t *bsrc = a.bimg + ((int64_t)ch * a.kblocks + kb) * bstage;
            for (int v = tid; v < bstage / 16; v += kThreads) cpa16(Bs + (uint32_t)(v * 16), bsrc + v * 16, true);
        }
        cpa_commit();
    };

    float acc[4][16];
    const uint32_t tb = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    auto drain = [&](int64_t jt) {  // add accumulator (jt & 1) of iteration jt into acc
        mbar_wait(dfull + (jt & 1), (uint32_t)((jt >> 1) & 1));
        tc_fence_after();
        const uint32_t db = tb + (uint32_t)((jt & 1) * 2 * a.nc);
#pragma unroll
        for (int jb = 0; jb < 4; ++jb) {
            const int c0 = 16 * (warp >> 2) + 32 * jb;
            if (c0 < a.nc) {
                float d0[16], d1[16];
                tmem_ld16(db + (uint32_t)c0, d0);
                tmem_ld16(db + (uint32_t)(a.nc + c0), d1);
#pragma unroll
                for (int c = 0; c < 16; ++c) acc[jb][c] += d0[c] + d1[c];
            }
        }
        tc_fence_before();
    };

    for (int j = 0; j < kStages - 1; ++j) issue(j);
    for (int64_t it = 0; it < total; ++it) {
        const int s = (int)(it % kStages);
        const int64_t tile = blockIdx.x + (it / per_tile) * gridDim.x;
        const int rem = (int)(it % per_tile), ch = rem / a.kblocks, kb = rem % a.kblocks;
        if (kb == 0) {
#pragma unroll
            for (int jb = 0; jb < 4; ++jb)
#pragma unroll
                for (int c = 0; c < 16; ++c) acc[jb][c] = 0.f;
        }
        cpa_wait<kStages - 2>();  // this thread's copies of iteration it have landed
        __syncthreads();
        // ---- lo operand (+ the ReLU mask on operand 0) for this thread's 16 columns
        const uint32_t As = sb + (uint32_t)(s * stage), Al = As + kA, Bs = As + 2 * kA;
        {
            const int64_t p = tile * kTileM + r;
            const bool masked = a.mask != nullptr && kb < a.ops[a.nops > 1 ? 1 : 0].kb0 + (a.nops > 1 ? 0 : a.kblocks) &&
                                p < a.n;
            const int col0 = kb * 32 + 16 * hf;  // operand 0 starts at K-block 0
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const uint32_t o = sw_chunk(r, 4 * hf + c);
                float4 v = lds128f(As + o);
                if (masked) {
                    const float *mk = a.mask + p * a.mask_ld + col0 + 4 * c;
                    const int k0 = a.ops[0].k;
                    if (col0 + 4 * c + 0 < k0 && !(__ldg(mk + 0) > 0.f)) v.x = 0.f;
                    if (col0 + 4 * c + 1 < k0 && !(__ldg(mk + 1) > 0.f)) v.y = 0.f;
                    if (col0 + 4 * c + 2 < k0 && !(__ldg(mk + 2) > 0.f)) v.z = 0.f;
                    if (col0 + 4 * c + 3 < k0 && !(__ldg(mk + 3) > 0.f)) v.w = 0.f;
                    sts128f(As + o, v.x, v.y, v.z, v.w);
                }
                sts128f(Al + o, tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
            }
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const uint32_t d = tmem + (uint32_t)((it & 1) * 2 * a.nc);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const uint32_t ko = (uint32_t)(ks * 32);
                const uint64_t bd = desc_sw128(Bs + ko);
                mma_tf32(d, desc_sw128(As + ko), bd, idesc, ks > 0 ? 1u : 0u);
                mma_tf32(d, desc_sw128(Al + ko), bd, idesc, 1u);
            }
            mma_commit(mma_done + s);
            mma_commit(dfull + (it & 1));
        }
        if (kb > 0) drain(it - 1);  // overlaps this K-block's MMAs
        // refill the stage of iteration it - 1 (its MMAs are done) with iteration it + kStages - 1
        if (it >= 1 && it + kStages - 1 < total)
            mbar_wait(mma_done + ((it - 1) % kStages), (uint32_t)((((it - 1) / kStages)) & 1));
        issue(it + kStages - 1);
        if (kb == a.kblocks - 1) {
            drain(it);
            // ---- epilogue of (tile, chunk): warp w holds TMEM lane quadrant w % 4, 16-column
            // blocks starting at 16 (w / 4), stride 32
            const int row = (warp & 3) * 32 + lane;
            const int64_t pe = tile * kTileM + row;
            if (pe < a.n) {
#pragma unroll
                for (int jb = 0; jb < 4; ++jb) {
                    const int c0 = 16 * (warp >> 2) + 32 * jb;
                    if (c0 >= a.nc) continue;
                    const int g0 = ch * a.nc + c0;
                    float y[16];
#pragma unroll
                    for (int c = 0; c < 16; ++c) y[c] = acc[jb][c] + ((a.bias && g0 + c < a.ncols) ? __ldg(a.bias + g0 + c) : 0.f);
                    for (int o = 0; o < a.nouts; ++o) {
                        const Out ou = a.outs[o];
                        float *dst = ou.p + pe * ou.ld + (g0 - ou.c0);
                        if (g0 >= ou.c0 && g0 + 16 <= ou.c1 && ((ou.ld & 3) == 0) && (((g0 - ou.c0) & 3) == 0) &&
                            ((reinterpret_cast<uintptr_t>(ou.p) & 15) == 0)) {
#pragma unroll
                            for (int c = 0; c < 16; c += 4)
                                *reinterpret_cast<float4 *>(dst + c) = make_float4(y[c], y[c + 1], y[c + 2], y[c + 3]);
                        } else {
#pragma unroll
                            for (int c = 0; c < 16; ++c)
                                if (g0 + c >= ou.c0 && g0 + c < ou.c1) dst[c] = y[c];
                        }
                    }
                    if (a.relu) {
                        float *dst = a.relu + pe * a.relu_ld + g0;
                        if (g0 + 16 <= a.ncols && ((a.relu_ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.relu) & 15) == 0)) {
#pragma unroll
                            for (int c = 0; c < 16; c += 4)
                                *reinterpret_cast<float4 *>(dst + c) = make_float4(fmaxf(y[c], 0.f), fmaxf(y[c + 1], 0.f),
                                                                                   fmaxf(y[c + 2], 0.f), fmaxf(y[c + 3], 0.f));
                        } else {
#pragma unroll
                            for (int c = 0; c < 16; ++c)
                                if (g0 + c < a.ncols) dst[c] = fmaxf(y[c], 0.f);
                        }
                    }
                }
            }
        }
    }
    cpa_wait<0>();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, kCols);
    }
}

// ---------------------------------------------------------------- weight gradient (SIMT)
struct WArgs {
    int64_t n, chunk;
    const float *g;
    int64_t ldg;
    const float *mask;
    int64_t mask_ld;
    int co;
    int nops;
    Op ops[kMaxOps];  // kb0 = first concatenated column of the operand
    int ci;           // concatenated columns; column ci = the bias (ones)
    float *part;      // [nchunk][co][ci + 1]
};
// CTA (64 threads): 64 (co) x 64 (ci) outputs over one point chunk; thread: 8 x 8 outputs
// (4 shared loads per 32 FFMA2).  32-point slabs of G, X (and the ReLU mask) arrive by 4-byte
// cp.async into a double-buffered shared tile, one slab ahead of the FMAs (no registers held
// across the load latency).  Partial sums per chunk, reduced in fixed order (deterministic).
// TAIL: the last ci tile also carries up to 8 more columns (64 + 3 coordinates + the bias
// column of a ResBlock is one tile plus a 4-column tail, not two tiles): thread (ty, tx) adds
// co 8 ty .. +7 x tail column tx.
template <bool MASKED, bool TAIL>
struct WgradSmem {
    static constexpr int XW = TAIL ? 72 : 64;
    float Gs[2][32][64];
    float Xs[2][32][XW];
    float Ms[MASKED ? 2 : 1][MASKED ? 32 : 1][MASKED ? 64 : 4];
};
template <bool MASKED, bool TAIL>
__global__ void __launch_bounds__(64) wgrad_kernel(WArgs a) {
    extern __shared__ __align__(16) uint8_t wg_smem[];
    auto &sm = *reinterpret_cast<WgradSmem<MASKED, TAIL> *>(wg_smem);
    auto &Gs = sm.Gs;
    auto &Xs = sm.Xs;
    auto &Ms = sm.Ms;
    const int tid = threadIdx.x, ty = tid >> 3, tx = tid & 7;
    const int co0 = blockIdx.x * 64, ci0 = blockIdx.y * 64;
    const int64_t p0 = (int64_t)blockIdx.z * a.chunk, p1 = std::min<int64_t>(a.n, p0 + a.chunk);
    // loader: thread tid copies the column quad qd = tid & 15 (columns 4 qd .. +3) of rows
    // rg + 4 k (rg = tid >> 4, k < 8) of every slab -- one 16-byte copy where the quad lies in
    // one 16-byte-aligned operand row, else four 4-byte copies; the tail columns 64 + tx
    // (tx = tid & 7 < ntail) of rows (tid >> 3) + 8 k (k < 4)
    const int qd = tid & 15, rg = tid >> 4;
    const int gc4 = co0 + 4 * qd;
    const bool gvec = (a.ldg & 3) == 0 && (reinterpret_cast<uintptr_t>(a.g) & 15) == 0 && gc4 + 4 <= a.co;
    const bool mvec = MASKED && (a.mask_ld & 3) == 0 && (reinterpret_cast<uintptr_t>(a.mask) & 15) == 0 && gc4 + 4 <= a.co;
    auto col_src = [&](int col, int64_t &ld) -> const float * {  // operand column (null: bias / past ci)
        ld = 0;
        if (col >= a.ci) return nullptr;
        for (int q = 0; q < a.nops; ++q)
            if (col >= a.ops[q].kb0 && col < a.ops[q].kb0 + a.ops[q].k) {
                ld = a.ops[q].lda;
                return a.ops[q].a + (col - a.ops[q].kb0);
            }
        return nullptr;
    };
    const int xc4 = ci0 + 4 * qd;
    const float *xe[4];
    int64_t xl[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) xe[e] = col_src(xc4 + e, xl[e]);
    const bool xvec = xe[0] && xe[3] == xe[0] + 3 && xl[3] == xl[0] && (xl[0] & 3) == 0 &&
                      (reinterpret_cast<uintptr_t>(xe[0]) & 15) == 0;
    const int ntail = (TAIL && blockIdx.y == gridDim.y - 1) ? a.ci + 1 - (ci0 + 64) : 0;
    const int tcol = ci0 + 64 + tx;
    const bool tload = tx < ntail;
    int64_t tld = 0;
    const float *tp = tload ? col_src(tcol, tld) : nullptr;
    const bool tones = tload && tcol == a.ci;
    auto issue = [&](int64_t pb, int buf) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int rr = rg + 4 * k;
            const int64_t p = pb + rr;
            const bool pv = p < p1;
            const uint32_t gs = smem_u32(&Gs[buf][rr][4 * qd]), xs = smem_u32(&Xs[buf][rr][4 * qd]);
            if (gvec) {
                cpa16(gs, pv ? a.g + p * a.ldg + gc4 : a.g, pv);
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const bool v = pv && gc4 + e < a.co;
                    cpa4(gs + 4u * e, v ? a.g + p * a.ldg + gc4 + e : a.g, v);
                }
            }
            if (xvec) {
                cpa16(xs, pv ? xe[0] + p * xl[0] : a.g, pv);
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (xc4 + e == a.ci)
                        Xs[buf][rr][4 * qd + e] = pv ? 1.f : 0.f;  // the bias column (no async write pending here)
                    else
                        cpa4(xs + 4u * e, xe[e] && pv ? xe[e] + p * xl[e] : a.g, xe[e] != nullptr && pv);
                }
            }
            if constexpr (MASKED) {
                const uint32_t ms = smem_u32(&Ms[buf][rr][4 * qd]);
                if (mvec) {
                    cpa16(ms, pv ? a.mask + p * a.mask_ld + gc4 : a.mask, pv);
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const bool v = pv && gc4 + e < a.co;
                        cpa4(ms + 4u * e, v ? a.mask + p * a.mask_ld + gc4 + e : a.mask, v);
                    }
                }
            }
        }
        if constexpr (TAIL) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int rr = (tid >> 3) + 8 * k;
                const int64_t p = pb + rr;
                const bool pv = p < p1;
                if (tones)
                    Xs[buf][rr][64 + tx] = pv ? 1.f : 0.f;
                else if (tload)
                    cpa4(smem_u32(&Xs[buf][rr][64 + tx]), tp && pv ? tp + p * tld : a.g, tp != nullptr && pv);
            }
        }
        cpa_commit();
    };
    float2 acc[8][4], acct[4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < 4; ++i) acct[i] = make_float2(0.f, 0.f);
    int buf = 0;
    if (p0 < p1) issue(p0, 0);
    for (int64_t pb = p0; pb < p1; pb += 32, buf ^= 1) {
        if (pb + 32 < p1) {
            issue(pb + 32, buf ^ 1);
            cpa_wait<1>();
        } else {
            cpa_wait<0>();
        }
        __syncthreads();
#pragma unroll 4
        for (int rr = 0; rr < 32; ++rr) {
            float4 g0 = *reinterpret_cast<const float4 *>(&Gs[buf][rr][8 * ty]);
            float4 g1 = *reinterpret_cast<const float4 *>(&Gs[buf][rr][8 * ty + 4]);
            if constexpr (MASKED) {
                const float4 m0 = *reinterpret_cast<const float4 *>(&Ms[buf][rr][8 * ty]);
                const float4 m1 = *reinterpret_cast<const float4 *>(&Ms[buf][rr][8 * ty + 4]);
                g0.x = m0.x > 0.f ? g0.x : 0.f, g0.y = m0.y > 0.f ? g0.y : 0.f, g0.z = m0.z > 0.f ? g0.z : 0.f,
                g0.w = m0.w > 0.f ? g0.w : 0.f;
                g1.x = m1.x > 0.f ? g1.x : 0.f, g1.y = m1.y > 0.f ? g1.y : 0.f, g1.z = m1.z > 0.f ? g1.z : 0.f,
                g1.w = m1.w > 0.f ? g1.w : 0.f;
            }
            const float4 x0 = *reinterpret_cast<const float4 *>(&Xs[buf][rr][8 * tx]);
            const float4 x1 = *reinterpret_cast<const float4 *>(&Xs[buf][rr][8 * tx + 4]);
            const float g8[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
            const float2 x2[4] = {make_float2(x0.x, x0.y), make_float2(x0.z, x0.w), make_float2(x1.x, x1.y),
                                  make_float2(x1.z, x1.w)};
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = ffma2(make_float2(g8[i], g8[i]), x2[j], acc[i][j]);
            if constexpr (TAIL) {
                const float xt = Xs[buf][rr][64 + tx];  // (columns past the tail: never written out)
#pragma unroll
                for (int i = 0; i < 4; ++i) acct[i] = ffma2(make_float2(g8[2 * i], g8[2 * i + 1]), make_float2(xt, xt), acct[i]);
            }
        }
        __syncthreads();  // buffer buf is refilled by the next iteration's issue
    }
    const int ldp = a.ci + 1;
    float *out = a.part + (int64_t)blockIdx.z * a.co * ldp;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int o = co0 + 8 * ty + i, c = ci0 + 8 * tx + j;
            if (o < a.co && c <= a.ci) out[(int64_t)o * ldp + c] = (j & 1) ? acc[i][j >> 1].y : acc[i][j >> 1].x;
        }
    if (TAIL && tx < ntail) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int o = co0 + 8 * ty + i;
            if (o < a.co) out[(int64_t)o * ldp + ci0 + 64 + tx] = (i & 1) ? acct[i >> 1].y : acct[i >> 1].x;
        }
    }
}
// fixed-order chunk reduction (fp64): a CTA owns 32 consecutive outputs, warp w adds the
// chunks of its contiguous block in ascending order, the 8 block sums are added in warp order
__global__ void __launch_bounds__(256) wgrad_reduce_kernel(const float *__restrict__ part, int nchunk, int co, int ci,
                                                           float *__restrict__ dw, float *__restrict__ db) {
    constexpr int W = 8;
    __shared__ double red[W][32];
    const int ldp = ci + 1;
    const int64_t E = (int64_t)co * ldp;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int per = (nchunk + W - 1) / W;
    const int z0 = min(nchunk, w * per), z1 = min(nchunk, z0 + per);
    for (int64_t e0 = (int64_t)blockIdx.x * 32; e0 < E; e0 += (int64_t)gridDim.x * 32) {
        const int64_t idx = e0 + lane;
        double s = 0.0;
        if (idx < E) {
            int z = z0;
            for (; z + 4 <= z1; z += 4) {
                const float v0 = part[(int64_t)z * E + idx], v1 = part[(int64_t)(z + 1) * E + idx];
                const float v2 = part[(int64_t)(z + 2) * E + idx], v3 = part[(int64_t)(z + 3) * E + idx];
                s += (double)v0;
                s += (double)v1;
                s += (double)v2;
                s += (double)v3;
            }
            for (; z < z1; ++z) s += (double)part[(int64_t)z * E + idx];
        }
        red[w][lane] = s;
        __syncthreads();
        if (w == 0 && idx < E) {
            double t = red[0][lane];
#pragma unroll
            for (int q = 1; q < W; ++q) t += red[q][lane];
            const int o = (int)(idx / ldp), c = (int)(idx % ldp);
            if (c < ci) {
                if (dw) dw[(int64_t)o * ci + c] = (float)t;
            } else if (db) {
                db[o] = (float)t;
            }
        }
        __syncthreads();
    }
}

}  // namespace gemm
}  // namespace fc

using namespace fc;

static bool gemm_one_cta() {  // FC_GEMM_ONE_CTA=1: always the 3-stage, one-CTA-per-SM kernel (A/B)
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("FC_GEMM_ONE_CTA");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v == 1;
}

extern "C" int64_t fc_gemm_image_bytes(int ncols, int kblocks) { return gemm::image_bytes(ncols, kblocks); }

extern "C" int fc_gemm_pack_b(int transpose, int nrows, int nseg, const int *seg_src, const int *seg_k,
                              const float *w, int64_t ldw, uint8_t *img, void *stream) {
    if (nseg < 1 || nseg > gemm::kMaxOps || nrows < 1) return set_error(FC_ERR_CONFIG, "gemm_pack_b: bad segments");
    gemm::PackArgs a{};
    a.w = w;
    a.ldw = ldw;
    a.transpose = transpose;
    a.nrows = nrows;
    a.nc = gemm::chunk_cols(nrows);
    a.nseg = nseg;
    int kb = 0;
    for (int s = 0; s < nseg; ++s) {
        if (seg_k[s] < 1) return set_error(FC_ERR_CONFIG, "gemm_pack_b: empty segment");
        a.seg_src[s] = seg_src[s];
        a.seg_k[s] = seg_k[s];
        a.seg_kb0[s] = kb;
        kb += (int)ceil_div(seg_k[s], 32);
    }
    a.kblocks = kb;
    a.img = img;
    const int64_t total = ceil_div(nrows, a.nc) * kb * a.nc * 32;
    const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 4 * num_sms());
    gemm::pack_b_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(a);
    count_launch();
    return check_launch("gemm_pack_b");
}

extern "C" int fc_gemm_rows(int64_t n, int nops, const float *const *a_ptr, const int64_t *lda, const int *ka,
                            const float *mask, int64_t mask_ld, const uint8_t *img, int ncols, const float *bias,
                            int nouts, float *const *out, const int64_t *ld, const int *c0, const int *c1,
                            float *relu_out, int64_t relu_ld, void *stream) {
    if (nops < 1 || nops > gemm::kMaxOps || nouts < 0 || nouts > gemm::kMaxOuts || ncols < 1)
        return set_error(FC_ERR_CONFIG, "gemm_rows: bad operand / output count");
    if (n <= 0) return FC_OK;
    gemm::Args a{};
    a.n = n;
    a.nops = nops;
    int kb = 0;
    for (int q = 0; q < nops; ++q) {
        if (ka[q] < 1 || lda[q] < ka[q]) return set_error(FC_ERR_SHAPE, "gemm_rows: operand %d shape", q);
        a.ops[q] = gemm::Op{a_ptr[q], lda[q], ka[q], kb};
        kb += (int)ceil_div(ka[q], 32);
    }
    a.kblocks = kb;
    a.mask = mask;
    a.mask_ld = mask_ld;
    a.bimg = img;
    a.nc = gemm::chunk_cols(ncols);
    a.nchunks = (int)ceil_div(ncols, a.nc);
    a.ncols = ncols;
    a.bias = bias;
    a.nouts = nouts;
    for (int o = 0; o < nouts; ++o) {
        if (c0[o] < 0 || c1[o] > ncols || c0[o] >= c1[o] || ld[o] < c1[o] - c0[o])
            return set_error(FC_ERR_SHAPE, "gemm_rows: output %d columns", o);
        a.outs[o] = gemm::Out{out[o], ld[o], c0[o], c1[o]};
    }
    a.relu = relu_out;
    a.relu_ld = relu_ld;
    const bool two = a.nc <= 64 && !gemm_one_cta();  // 2 stages, TMEM 256: two CTAs per SM
    const int stages = two ? 2 : 3;
    const int smem = stages * (2 * gemm::kA + 2 * a.nc * 128) + 1024 + 64;
    static uint64_t attr = 0;
    if (first_use_on_device(attr)) {
        cudaFuncSetAttribute(gemm::gemm_rows_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             3 * (2 * gemm::kA + 2 * 128 * 128) + 1024 + 64);
        cudaFuncSetAttribute(gemm::gemm_rows_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             2 * (2 * gemm::kA + 2 * 64 * 128) + 1024 + 64);
    }
    const int grid = (int)std::min<int64_t>(ceil_div(n, gemm::kTileM), (two ? 2 : 1) * num_sms());
    prof_begin("tc_pointwise", (cudaStream_t)stream);
    if (two) gemm::gemm_rows_kernel<2><<<grid, gemm::kThreads, smem, (cudaStream_t)stream>>>(a);
    else gemm::gemm_rows_kernel<3><<<grid, gemm::kThreads, smem, (cudaStream_t)stream>>>(a);
    prof_end((cudaStream_t)stream);
    count_launch();
    return check_launch("gemm_rows");
}

extern "C" int fc_gemm_wgrad(int64_t n, const float *g, int64_t ldg, const float *mask, int64_t mask_ld, int co,
                             int nops, const float *const *x, const int64_t *ldx, const int *kx, float *dw, float *db,
                             void *stream) {
    if (nops < 0 || nops > gemm::kMaxOps || co < 1) return set_error(FC_ERR_CONFIG, "gemm_wgrad: bad operands");
    cudaStream_t st = (cudaStream_t)stream;
    gemm::WArgs a{};
    a.n = n;
    a.g = g;
    a.ldg = ldg;
    a.mask = mask;
    a.mask_ld = mask_ld;
    a.co = co;
    a.nops = nops;
    int ci = 0;
    for (int q = 0; q < nops; ++q) {
        a.ops[q] = gemm::Op{x[q], ldx[q], kx[q], ci};
        ci += kx[q];
    }
    a.ci = ci;
    // ci + 1 columns (the bias last) in tiles of 64; a remainder of <= 8 rides on the last tile
    const int nfull = (ci + 1) / 64, rem = (ci + 1) % 64;
    const bool tail = nfull >= 1 && rem > 0 && rem <= 8;
    const int gx = (int)ceil_div(co, 64), gy = tail ? nfull : (int)ceil_div(ci + 1, 64);
    // point chunks: one full wave of resident CTAs (the kernel is latency-bound; partials
    // are reduced in fixed order afterwards), at least 64 and at most 4096 points per chunk
    size_t smem_b = 0;
    const void *kfn = nullptr;
    if (mask) {
        smem_b = tail ? sizeof(gemm::WgradSmem<true, true>) : sizeof(gemm::WgradSmem<true, false>);
        kfn = tail ? (const void *)gemm::wgrad_kernel<true, true> : (const void *)gemm::wgrad_kernel<true, false>;
    } else {
        smem_b = tail ? sizeof(gemm::WgradSmem<false, true>) : sizeof(gemm::WgradSmem<false, false>);
        kfn = tail ? (const void *)gemm::wgrad_kernel<false, true> : (const void *)gemm::wgrad_kernel<false, false>;
    }
    static uint64_t wattr = 0;
    if (first_use_on_device(wattr)) {  // the masked tail variant needs > 48 KB
        cudaFuncSetAttribute(gemm::wgrad_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(gemm::WgradSmem<true, true>));
        cudaFuncSetAttribute(gemm::wgrad_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)sizeof(gemm::WgradSmem<true, false>));
    }
    static int occ_cache[4] = {0, 0, 0, 0};  // resident CTAs per SM of each variant
    int &occ = occ_cache[(mask ? 2 : 0) + (tail ? 1 : 0)];
    if (occ < 1 && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, 64, smem_b) != cudaSuccess || occ < 1)) occ = 1;
    const int64_t nn = std::max<int64_t>(n, 1), tiles = (int64_t)gx * gy;
    int64_t nchunk = std::max<int64_t>(1, (int64_t)occ * num_sms() / tiles);
    nchunk = std::min<int64_t>(std::max<int64_t>(nchunk, ceil_div(nn, 4096)), ceil_div(nn, 64));
    a.chunk = ceil_div(nn, nchunk);
    nchunk = ceil_div(nn, a.chunk);
    Scratch part((size_t)nchunk * co * (ci + 1) * sizeof(float), st);
    if (!part.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed (gemm_wgrad)");
    a.part = part.as<float>();
    prof_begin("pointwise_wgrad", st);
    const dim3 grid(gx, gy, (unsigned)nchunk);
    if (mask) {
        if (tail) gemm::wgrad_kernel<true, true><<<grid, 64, sizeof(gemm::WgradSmem<true, true>), st>>>(a);
        else gemm::wgrad_kernel<true, false><<<grid, 64, sizeof(gemm::WgradSmem<true, false>), st>>>(a);
    } else {
        if (tail) gemm::wgrad_kernel<false, true><<<grid, 64, sizeof(gemm::WgradSmem<false, true>), st>>>(a);
        else gemm::wgrad_kernel<false, false><<<grid, 64, sizeof(gemm::WgradSmem<false, false>), st>>>(a);
    }
    count_launch();
    gemm::wgrad_reduce_kernel<<<(unsigned)ceil_div((int64_t)co * (ci + 1), 32), 256, 0, st>>>(
        a.part, (int)nchunk, co, ci, dw, db);
    count_launch();
    prof_end(st);
    return check_launch("gemm_wgrad");
}
