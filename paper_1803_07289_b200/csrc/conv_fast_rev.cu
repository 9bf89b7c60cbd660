// conv_fast_rev.cu -- the reverse (adjoint) flex-convolution for the headline shape
// (c_in = c_out = 64, Dp = 3): d_features of flex_conv's backward together with the
// neighbour-role location gradient, and flex_deconv.
//
// For point j and its reverse list R(j) = {(i, s): nbr[i][s] = j} (CSR, ascending = the
// reference's serial (i, s) order, _native.pyx:93-127):
//   Y_j[t, c'] = sum_{(i,s)} (l_i - l_j)_t g_i[c'] (t < 3),  Y_j[3, c'] = sum_{(i,s)} g_i[c']
//   d_f[j, c]  = sum_{t, c'} Y_j[t, c'] B_rev[(t, c'), c],  B_rev = [theta_0; theta_1; theta_2; theta_b]
//   U_t[j, c]  = sum_c' Y_j[3, c'] theta[c', c, t],  d_l[j, t] = centre[j, t] - sum_c f[j, c] U_t[j, c]
// Same machinery as conv_fast.cu (channel halves, per-(point, half) power-of-two scales,
// fp16 hi/lo split, dedicated MMA warp), adapted to variable-length lists:
//   * index warps (4, also the epilogue) stage each 64-row group's list entries {i, l_i - l_j}
//     contiguously (a group's CSR entries are contiguous) in a 3-stage ring, software-
//     pipelined over groups (row offsets two groups ahead, entries one group ahead,
//     positions for the current group); rows with more than 16 entries or past the stage
//     capacity are marked "direct" and gathered straight from the CSR (rare);
//   * gather warps walk each point's entries in 8-slot batches (warp-uniform bound = the
//     longest of the item's 4 lists, shorter lists predicated off);
//   * per half h the MMA warp issues the d_f product (3 fp16 MMAs of N = 64 per k-step: the
//     TMEM budget -- D 2 x 64 + U 2 x 192 columns -- rules out the N = 128 hi/lo-concatenated
//     form of the forward) and, with the location gradient, U_h = Yb_h . [theta_0; theta_1;
//     theta_2] as ONE N = 192 operand (K-blocks 0..2 of the B_rev image, 8 KB apart).
// Accumulators are single-buffered: the MMAs of tile i+1 wait for the epilogue of tile i.
#include <cstdio>
#include <cstdlib>

#include "fast_common.cuh"

namespace fc {
using namespace sm100;

namespace fast {

constexpr int rGatherWarps = 16;
constexpr int rEpiWarp0 = 16;  // warps 16..19: epilogue (TMEM quadrant = warp % 4); warp 16 also
constexpr int rEpiWarps = 4;   //   owns TMEM and issues the MMAs
constexpr int rMmaWarp = 16;
constexpr int rIdxWarp0 = 20;  // warps 20..23: index producer
constexpr int rWarps = 24;
constexpr int rThreads = rWarps * 32;
constexpr int rCap = 680;      // staged entries per 64-row group (mean 512 at K = 8)
constexpr int rStages = 3;
constexpr int rMaxRow = 16;    // staged entries per row; longer lists take the direct path
constexpr uint32_t rDirect = 0xffffu;
// wide-lane variant: 12 gather warps (8 channels per lane), 4 epilogue / MMA, 4 index
constexpr int wrGatherWarps = 12;
constexpr int wrEpiWarp0 = 12;
constexpr int wrMmaWarp = 12;
constexpr int wrIdxWarp0 = 16;
constexpr int wrThreads = 20 * 32;

template <bool SPLIT>
struct RevL {
    static constexpr int NS = SPLIT ? 2 : 1;
    static constexpr int A_BYTES = kTile * 256 * 2;  // 4 K-blocks x 128 rows x 128 B
    static constexpr int B_BYTES = 64 * 256 * 2;     // 4 K-blocks x 64 rows x 128 B
    static constexpr int A_OFF = 0;
    static constexpr int B_OFF = A_OFF + NS * A_BYTES;
    static constexpr int E_STAGE = (rCap + 1) * 16;  // + the zero entry (index rCap)
    static constexpr int E_OFF = B_OFF + NS * B_BYTES;
    static constexpr int R_OFF = E_OFF + rStages * E_STAGE;  // per row: start << 16 | count
    static constexpr int RS_OFF = R_OFF + rStages * 64 * 4;  // int8 [2 buf][2 half][128]
    static constexpr int SC_OFF = RS_OFF + 2 * 2 * kTile;    // int [4] index-warp scan scratch
    static constexpr int BAR_OFF = SC_OFF + 32;
    static constexpr int SMEM = BAR_OFF + 128;
    static constexpr int SMEM_ALLOC = SMEM + 1024;
    static_assert(SMEM_ALLOC <= 232448, "shared memory budget");
};

struct RevArgs {
    int64_t total;
    int64_t num_tiles;
    int k;                // forward neighbourhood size (entry e = i * k + s)
    const float *rows;    // gathered rows (upstream gradient g, or deconv input) [total, 64]
    const float *zero;    // 64 zero floats (the row of slots past a list's end)
    const float *loc;     // [total, 3]
    Csr csr;
    const uint8_t *bimg;  // B_rev image (hi [, lo])
    const float *binv;
    float *out;           // [total, 64]
    const float *feat;    // location gradient only: conv input features [total, 64]
    const float *centre;  // centre-role term [total, 3]
    float *dloc;          // [total, 3] or null
    int dbg;              // timing probes (FC_DBG): 2 no MMA, 8 gather + index only, 16 first 8 slots only (wrong results)
    int ld_rows, ld_out;  // wide kernel, BLK instance: row strides of rows / out (a 64 x 64 channel block;
                          // 32-bit: with 64-bit fields here ptxas spills one more register in the plain instance)
    int acc;                  // wide kernel, BLK instance: out += this block's product
};

__device__ __forceinline__ void ldg_nc8r(const float *p, float (&v)[8]) {
    asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
}
// predicated form: lanes whose slot is past their list's end issue no load (no L1 wavefronts)
// and read zeros
__device__ __forceinline__ void ldg_nc8r_if(const float *p, float (&v)[8], bool ok) {
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.b32 q, %9, 0;\n"
        " mov.b32 %0, 0;\n mov.b32 %1, 0;\n mov.b32 %2, 0;\n mov.b32 %3, 0;\n"
        " mov.b32 %4, 0;\n mov.b32 %5, 0;\n mov.b32 %6, 0;\n mov.b32 %7, 0;\n"
        " @q ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n}"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
        : "l"(p), "r"((int)ok));
}
__device__ __forceinline__ void sts128r(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <bool SPLIT, bool DLOC>
__global__ void __launch_bounds__(rThreads, 1) tc_rev64_kernel(RevArgs a) {
    using L = RevL<SPLIT>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sb = smem_u32(smem);
    const uint32_t A_hi = sb + L::A_OFF, A_lo = A_hi + L::A_BYTES;
    const uint32_t B_hi = sb + L::B_OFF, B_lo = B_hi + L::B_BYTES;
    const uint32_t E0 = sb + L::E_OFF, R0 = sb + L::R_OFF, rs_s = sb + L::RS_OFF;
    const int8_t *rs = reinterpret_cast<const int8_t *>(smem + L::RS_OFF);
    int *scan = reinterpret_cast<int *>(smem + L::SC_OFF);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + L::BAR_OFF);
    uint64_t *e_full = bar + 0;    // [3] index warps
    uint64_t *e_empty = bar + 3;   // [3] gather warps
    uint64_t *a_full = bar + 6;    // [2 halves] gather warps
    uint64_t *mma_done = bar + 8;  // [2 halves] commit
    uint64_t *acc_full = bar + 10;
    uint64_t *acc_free = bar + 11;
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bar + 12);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int q = 0; q < rStages; ++q) {
            mbar_init(e_full + q, 4);
            mbar_init(e_empty + q, rGatherWarps);
        }
        for (int q = 0; q < 2; ++q) {
            mbar_init(a_full + q, rGatherWarps);
            mbar_init(mma_done + q, 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_free, rEpiWarps);
        fence_mbar_init();
    }
    if (warp == rMmaWarp) tmem_alloc(tmem_holder, 512);
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(a.bimg);
        uint4 *dst = reinterpret_cast<uint4 *>(smem + L::B_OFF);
        smem_fill16(dst, src, L::NS * L::B_BYTES / 16);
    }
    if (threadIdx.x < rStages) {  // zero entries: row 0 of the zero row, zero offsets
        float4 *z = reinterpret_cast<float4 *>(smem + L::E_OFF + threadIdx.x * L::E_STAGE + rCap * 16);
        *z = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const int T = a.num_tiles > blockIdx.x ? (int)ceil_div(a.num_tiles - blockIdx.x, gridDim.x) : 0;
    const int K = a.k;

    if (warp >= rEpiWarp0 && warp < rEpiWarp0 + rEpiWarps && (a.dbg & 8)) {
        // probe: no MMA / epilogue
    } else if (warp >= rEpiWarp0 && warp < rEpiWarp0 + rEpiWarps) {
        // ------------------------------------------------------------ MMA issue (warp 16, lane 0) + epilogue
        // TMEM columns: D_0 0..63, D_1 64..127, U_0 128..319, U_1 320..511 (single-buffered)
        const int ew = warp - rEpiWarp0;  // TMEM lane quadrant
        const float binv = a.binv[0];
        auto issue = [&](int i, int h) {
            constexpr uint32_t idn = idesc_f16(kTile, 64, SPLIT ? 0 : 1);
            constexpr uint32_t idu = idesc_f16(kTile, 192, SPLIT ? 0 : 1);
            mbar_wait(a_full + h, (uint32_t)(i & 1));
            if (h == 0 && i >= 1) mbar_wait(acc_free, (uint32_t)((i - 1) & 1));
            tc_fence_after();
            if (a.dbg & 2) {
                mbar_arrive(mma_done + h);
                if (h == 1) mbar_arrive(acc_full);
                return;
            }
            const uint32_t d = tmem_base + (uint32_t)(h * 64);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int t = ks >> 1, kk = ks & 1;
                const uint32_t ko = (uint32_t)((32 * h + 16 * kk) * 2);
                const uint32_t ao = (uint32_t)t * (kTile * 128) + ko, bo = (uint32_t)t * (64 * 128) + ko;
                mma_f16(d, desc_sw128(A_hi + ao), desc_sw128(B_hi + bo), idn, ks > 0 ? 1u : 0u);
                if (SPLIT) {
                    mma_f16(d, desc_sw128(A_hi + ao), desc_sw128(B_lo + bo), idn, 1u);
                    mma_f16(d, desc_sw128(A_lo + ao), desc_sw128(B_hi + bo), idn, 1u);
                }
            }
            if (DLOC) {
                const uint32_t u = tmem_base + 128u + (uint32_t)(h * 192);
#pragma unroll
                for (int kk = 0; kk < 2; ++kk) {
                    const uint32_t ko = (uint32_t)((32 * h + 16 * kk) * 2);
                    const uint32_t ao = 3u * (kTile * 128) + ko;
                    mma_f16(u, desc_sw128(A_hi + ao), desc_sw128(B_hi + ko), idu, kk > 0 ? 1u : 0u);
                    if (SPLIT) {
                        mma_f16(u, desc_sw128(A_hi + ao), desc_sw128(B_lo + ko), idu, 1u);
                        mma_f16(u, desc_sw128(A_lo + ao), desc_sw128(B_hi + ko), idu, 1u);
                    }
                }
            }
            mma_commit(mma_done + h);
            if (h == 1) mma_commit(acc_full);
        };
        auto epilogue = [&](int i) {
            mbar_wait_sleep(acc_full, (uint32_t)(i & 1));
            tc_fence_after();
            const int b = i & 1;
            const int tr = ew * 32 + lane;
            const int64_t p = (blockIdx.x + (int64_t)i * gridDim.x) * kTile + tr;
            const float s0 = exp2i(rs[(b * 2 + 0) * kTile + tr]) * binv;
            const float s1 = exp2i(rs[(b * 2 + 1) * kTile + tr]) * binv;
            const uint32_t tb = tmem_base + ((uint32_t)(ew * 32) << 16);
            const bool pv = p < a.total;
            float *orow = a.out + p * 64;
#pragma unroll 1
            for (int c0 = 0; c0 < 64; c0 += 16) {
                float x0[16], x1[16];
                tmem_ld16(tb + (uint32_t)c0, x0);
                tmem_ld16(tb + 64u + (uint32_t)c0, x1);
                if (pv) {
                    float o[16];
#pragma unroll
                    for (int c = 0; c < 16; ++c) o[c] = fmaf(x1[c], s1, x0[c] * s0);
                    stg256(orow + c0, o);
                    stg256(orow + c0 + 8, o + 8);
                }
            }
            if (DLOC) {
                float nb0 = 0.f, nb1 = 0.f, nb2 = 0.f;
#pragma unroll 1
                for (int c0 = 0; c0 < 64; c0 += 16) {
                    // own row, 32 bytes per lane per load (LDG.256): one line touch per 8 channels
                    float f[16], f8[8];
                    if (pv) {
                        ldg_nc8r(a.feat + p * 64 + c0, f8);
#pragma unroll
                        for (int q = 0; q < 8; ++q) f[q] = f8[q];
                        ldg_nc8r(a.feat + p * 64 + c0 + 8, f8);
#pragma unroll
                        for (int q = 0; q < 8; ++q) f[8 + q] = f8[q];
                    } else {
#pragma unroll
                        for (int q = 0; q < 16; ++q) f[q] = 0.f;
                    }
#pragma unroll
                    for (int tt = 0; tt < 3; ++tt) {
                        float u0[16], u1[16];
                        tmem_ld16(tb + 128u + (uint32_t)(64 * tt + c0), u0);
                        tmem_ld16(tb + 320u + (uint32_t)(64 * tt + c0), u1);
                        float acc = 0.f;
#pragma unroll
                        for (int c = 0; c < 16; ++c) acc = fmaf(f[c], fmaf(u1[c], s1, u0[c] * s0), acc);
                        if (tt == 0) nb0 += acc;
                        if (tt == 1) nb1 += acc;
                        if (tt == 2) nb2 += acc;
                    }
                }
                if (pv) {
                    a.dloc[p * 3 + 0] = a.centre[p * 3 + 0] - nb0;
                    a.dloc[p * 3 + 1] = a.centre[p * 3 + 1] - nb1;
                    a.dloc[p * 3 + 2] = a.centre[p * 3 + 2] - nb2;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_free);
        };
        for (int i = 0; i < T; ++i) {
            if (warp == rMmaWarp) {
                if (lane == 0) {
                    issue(i, 0);
                    issue(i, 1);
                }
                __syncwarp();
            }
            epilogue(i);
        }
    } else if (warp >= rIdxWarp0) {
        // ------------------------------------------------------------ index producer + epilogue
        const int t = (warp - rIdxWarp0) * 32 + lane;  // 0..127
        const int r = t >> 1, par = t & 1;             // row of the group, entry parity
        const int G = 2 * T;                           // 64-row groups of this CTA
        auto grow = [&](int gg) -> int64_t {           // global index of row r of group gg
            return (blockIdx.x + (int64_t)(gg >> 1) * gridDim.x) * kTile + (gg & 1) * 64 + r;
        };
        // pipeline registers: offsets of group gg+2, entries (source rows) of gg+1, positions of gg
        int32_t o2_lo = 0, o2_hi = 0;   // row range, group gg+2
        int32_t o1_lo = 0, o1_hi = 0;   // row range, group gg+1
        int32_t src1[rMaxRow / 2];      // source rows i of group gg+1 (this thread's parity)
        int32_t src0[rMaxRow / 2];
        int32_t o0_lo = 0, o0_hi = 0;
        auto load_off = [&](int gg, int32_t &lo, int32_t &hi) {
            lo = hi = 0;
            if (gg < G) {
                const int64_t j = grow(gg);
                if (j < a.total) {
                    lo = __ldg(a.csr.off + j);
                    hi = __ldg(a.csr.off + j + 1);
                }
            }
        };
        auto load_src = [&](int32_t lo, int32_t hi, int32_t (&src)[rMaxRow / 2]) {
            const int cnt = min(hi - lo, rMaxRow);
#pragma unroll
            for (int q = 0; q < rMaxRow / 2; ++q) {
                const int s2 = 2 * q + par;
                src[q] = s2 < cnt ? __ldg(a.csr.ent + lo + s2) / K : 0;
            }
        };
        // prologue: offsets of groups 0, 1; sources of group 0
        load_off(0, o0_lo, o0_hi);
        load_off(1, o1_lo, o1_hi);
        load_src(o0_lo, o0_hi, src0);
        for (int gg = 0; gg < G; ++gg) {
            // positions of group gg (sources loaded last iteration), sources of gg+1, offsets of gg+2
            const int64_t j = grow(gg);
            const bool jv = gg < G && j < a.total;
            float lj0 = 0.f, lj1 = 0.f, lj2 = 0.f;
            if (jv) {
                lj0 = __ldg(a.loc + j * 3 + 0);
                lj1 = __ldg(a.loc + j * 3 + 1);
                lj2 = __ldg(a.loc + j * 3 + 2);
            }
            const int cnt = jv ? o0_hi - o0_lo : 0;
            float q0[rMaxRow / 2], q1[rMaxRow / 2], q2[rMaxRow / 2];
#pragma unroll
            for (int q = 0; q < rMaxRow / 2; ++q) {
                const bool v = 2 * q + par < min(cnt, rMaxRow);
                q0[q] = v ? __ldg(a.loc + (int64_t)src0[q] * 3 + 0) : 0.f;
                q1[q] = v ? __ldg(a.loc + (int64_t)src0[q] * 3 + 1) : 0.f;
                q2[q] = v ? __ldg(a.loc + (int64_t)src0[q] * 3 + 2) : 0.f;
            }
            load_src(o1_lo, o1_hi, src1);
            load_off(gg + 2, o2_lo, o2_hi);
            // row starts within the stage: exclusive scan of the staged counts over the 64 rows
            const bool direct_row = cnt > rMaxRow;
            const int staged = direct_row ? 0 : cnt;
            int incl = par == 0 ? staged : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            named_bar(1, 128);
            if (lane == 31) scan[warp - rIdxWarp0] = incl;
            named_bar(1, 128);
            int base = 0;
            for (int w = 0; w < warp - rIdxWarp0; ++w) base += scan[w];
            const int start = base + incl - staged;  // incl of both threads of a row covers the row
            const bool direct = direct_row || start + staged > rCap;
            // store
            const int st = gg % rStages;
            if (gg >= rStages) mbar_wait_sleep(e_empty + st, (uint32_t)(((gg / rStages) + 1) & 1));
            const uint32_t es = E0 + (uint32_t)(st * L::E_STAGE);
            if (!direct) {
#pragma unroll
                for (int q = 0; q < rMaxRow / 2; ++q) {
                    const int s2 = 2 * q + par;
                    if (s2 < staged)
                        sts128f(es + (uint32_t)((start + s2) * 16), __int_as_float(src0[q]), q0[q] - lj0, q1[q] - lj1,
                                q2[q] - lj2);
                }
            }
            if (par == 0) {
                const uint32_t rec = direct ? ((rDirect << 16) | (uint32_t)min(cnt, 0xffff)) : (((uint32_t)start << 16) | (uint32_t)cnt);
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(R0 + (uint32_t)((st * 64 + r) * 4)), "r"(rec) : "memory");
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(e_full + st);
            // rotate the pipeline
            o0_lo = o1_lo, o0_hi = o1_hi;
            o1_lo = o2_lo, o1_hi = o2_hi;
#pragma unroll
            for (int q = 0; q < rMaxRow / 2; ++q) src0[q] = src1[q];
        }
    } else {
        // ------------------------------------------------------------ gather warps
        // warp w: items q = w (rows 0..63, group 0) and w + 16 (group 1) of each half, in the
        // order (h0 g0) (h0 g1) (h1 g0) (h1 g1).  Each item's 4 lists are walked in 8-slot
        // batches up to the longest of them; slots past a list's end read the stage's zero
        // entry and the zero row (no predication in the hot loop).  The first batch of the
        // next item is in flight while the current item is finished.  Items containing a
        // "direct" row (list not staged) take a separate, simple path.
        const int pt = lane >> 3, cl = lane & 7;
        float4 v[8];
        struct Item {
            uint32_t es;     // stage entry base
            int cnt, start;  // list length, staged start (rDirect: direct path)
            int mx;          // longest list of the item (warp-uniform)
            bool direct;     // any direct row in the item (warp-uniform)
            int64_t p;       // global row
        };
        auto open_item = [&](int i, int hk, Item &it) {
            const int g = hk & 1;
            const int gg = 2 * i + g, st = gg % rStages;
            if (hk < 2) mbar_wait(e_full + st, (uint32_t)((gg / rStages) & 1));
            const int row = item_row(warp + 16 * g, pt);
            it.es = E0 + (uint32_t)(st * L::E_STAGE);
            const uint32_t rec = (uint32_t)lds32(R0 + (uint32_t)((st * 64 + (row & 63)) * 4));
            it.cnt = (int)(rec & 0xffffu);
            it.start = (int)(rec >> 16);
            it.p = (blockIdx.x + (int64_t)i * gridDim.x) * kTile + row;
            const bool dr = it.start == (int)rDirect;
            if (dr && it.p < a.total) it.cnt = __ldg(a.csr.off + it.p + 1) - __ldg(a.csr.off + it.p);
            it.direct = __any_sync(0xffffffffu, dr);
            it.mx = (int)__reduce_max_sync(0xffffffffu, (uint32_t)it.cnt);
            if (a.dbg & 16) it.mx = min(it.mx, 8);
        };
        // staged path: entry index of slot sl (the stage's zero entry rCap past the end)
        auto load8 = [&](const Item &it, int h, int b0) {
            const float *src = a.rows + 32 * h + 4 * cl;
            const float *zsrc = a.zero + 4 * cl;
#pragma unroll
            for (int s2 = 0; s2 < 8; ++s2) {
                const int sl = b0 + s2;
                const bool ok = sl < it.cnt;
                const int32_t jr = lds32(it.es + (uint32_t)((ok ? it.start + sl : rCap) * 16));
                v[s2] = ldg_nc4(ok ? src + (int64_t)jr * 64 : zsrc);
            }
        };
        auto load4 = [&](const Item &it, int h, int b0) {
            const float *src = a.rows + 32 * h + 4 * cl;
            const float *zsrc = a.zero + 4 * cl;
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
                const int sl = b0 + s2;
                const bool ok = sl < it.cnt;
                const int32_t jr = lds32(it.es + (uint32_t)((ok ? it.start + sl : rCap) * 16));
                v[s2] = ldg_nc4(ok ? src + (int64_t)jr * 64 : zsrc);
            }
        };
        auto fma4 = [&](const Item &it, int b0, Mom4 &x) {
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
                const int sl = b0 + s2;
                const float4 e = lds128f(it.es + (uint32_t)((sl < it.cnt ? it.start + sl : rCap) * 16));
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
        };
        auto fma8 = [&](const Item &it, int b0, Mom4 &x) {
#pragma unroll
            for (int s2 = 0; s2 < 8; ++s2) {
                const int sl = b0 + s2;
                const float4 e = lds128f(it.es + (uint32_t)((sl < it.cnt ? it.start + sl : rCap) * 16));
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
        };
        // direct path (rare): every lane walks its point's list from the CSR
        auto direct_item = [&](const Item &it, int h, Mom4 &x) {
            const bool staged = it.start != (int)rDirect;
            const int32_t o0 = it.p < a.total ? __ldg(a.csr.off + it.p) : 0;
            const float lp0 = it.p < a.total ? __ldg(a.loc + it.p * 3 + 0) : 0.f;
            const float lp1 = it.p < a.total ? __ldg(a.loc + it.p * 3 + 1) : 0.f;
            const float lp2 = it.p < a.total ? __ldg(a.loc + it.p * 3 + 2) : 0.f;
            const float *src = a.rows + 32 * h + 4 * cl;
            for (int sl = 0; sl < it.mx; ++sl) {
                if (sl < it.cnt) {
                    float4 e;
                    if (staged) {
                        e = lds128f(it.es + (uint32_t)((it.start + sl) * 16));
                    } else {
                        const int32_t jr = __ldg(a.csr.ent + o0 + sl) / K;
                        e = make_float4(__int_as_float(jr), __ldg(a.loc + (int64_t)jr * 3 + 0) - lp0,
                                        __ldg(a.loc + (int64_t)jr * 3 + 1) - lp1, __ldg(a.loc + (int64_t)jr * 3 + 2) - lp2);
                    }
                    const float4 r = ldg_nc4(src + (int64_t)__float_as_int(e.x) * 64);
                    const float2 lo = make_float2(r.x, r.y), hi = make_float2(r.z, r.w);
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
            }
        };
        auto handoff = [&](int h) {
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(a_full + h);
        };
        int pend = -1;  // half whose hand-off is pending
        Item cur;
        if (T > 0) {
            open_item(0, 0, cur);
            if (!cur.direct) load8(cur, 0, 0);
        }
        for (int i = 0; i < T; ++i) {
            const int64_t lim = a.total - ((int64_t)blockIdx.x + (int64_t)i * gridDim.x) * kTile;
#pragma unroll 1
            for (int hk = 0; hk < 4; ++hk) {
                const int h = hk >> 1, g = hk & 1;
                const int row = item_row(warp + 16 * g, pt);
                Mom4 x;
#pragma unroll
                for (int tt = 0; tt < 4; ++tt) x.m[tt][0] = x.m[tt][1] = make_float2(0.f, 0.f);
                if (cur.direct) {
                    direct_item(cur, h, x);
                } else {
                    if (cur.mx > 0) fma8(cur, 0, x);
                    for (int b0 = 8; b0 < cur.mx; b0 += 4) {  // tails in 4-slot batches
                        load4(cur, h, b0);
                        fma4(cur, b0, x);
                    }
                }
                if (hk >= 2) {  // last use of the group's stage by this warp
                    __syncwarp();
                    if (lane == 0) mbar_arrive(e_empty + (2 * i + g) % rStages);
                }
                if (pend >= 0) {  // no row loads in flight here
                    if (!(a.dbg & 8)) handoff(pend);
                    pend = -1;
                }
                if (hk < 3 || i + 1 < T) {  // first batch of the next item
                    const int ni = hk < 3 ? i : i + 1, nhk = hk < 3 ? hk + 1 : 0;
                    open_item(ni, nhk, cur);
                    if (!cur.direct && cur.mx > 0) load8(cur, nhk >> 1, 0);
                }
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
                if ((int64_t)row >= lim) sc = 0.f;
                if (g == 0 && i >= 1 && !(a.dbg & 8)) mbar_wait(mma_done + h, (uint32_t)((i - 1) & 1));
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
                if (g == 1) pend = h;
            }
        }
        if (pend >= 0 && !(a.dbg & 8)) handoff(pend);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == rMmaWarp) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

template <bool SPLIT, bool DLOC, bool BLK = false>  // BLK: strided rows / out + accumulate (channel blocks)
__global__ void __launch_bounds__(wrThreads, 1) tc_rev64w_kernel(RevArgs a) {
    using L = RevL<SPLIT>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sb = smem_u32(smem);
    const uint32_t A_hi = sb + L::A_OFF, A_lo = A_hi + L::A_BYTES;
    const uint32_t B_hi = sb + L::B_OFF, B_lo = B_hi + L::B_BYTES;
    const uint32_t E0 = sb + L::E_OFF, R0 = sb + L::R_OFF, rs_s = sb + L::RS_OFF;
    const int8_t *rs = reinterpret_cast<const int8_t *>(smem + L::RS_OFF);
    int *scan = reinterpret_cast<int *>(smem + L::SC_OFF);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + L::BAR_OFF);
    uint64_t *e_full = bar + 0;    // [3] index warps
    uint64_t *e_empty = bar + 3;   // [3] gather warps
    uint64_t *a_full = bar + 6;    // [2 halves] gather warps
    uint64_t *mma_done = bar + 8;  // [2 halves] commit
    uint64_t *acc_full = bar + 10;
    uint64_t *acc_free = bar + 11;
    uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bar + 12);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int q = 0; q < rStages; ++q) {
            mbar_init(e_full + q, 4);
            mbar_init(e_empty + q, wrGatherWarps);
        }
        for (int q = 0; q < 2; ++q) {
            mbar_init(a_full + q, wrGatherWarps);
            mbar_init(mma_done + q, 1);
        }
        mbar_init(acc_full, 1);
        mbar_init(acc_free, rEpiWarps);
        fence_mbar_init();
    }
    if (warp == wrMmaWarp) tmem_alloc(tmem_holder, 512);
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(a.bimg);
        uint4 *dst = reinterpret_cast<uint4 *>(smem + L::B_OFF);
        smem_fill16(dst, src, L::NS * L::B_BYTES / 16);
    }
    if (threadIdx.x < rStages) {  // zero entries: row 0 of the zero row, zero offsets
        float4 *z = reinterpret_cast<float4 *>(smem + L::E_OFF + threadIdx.x * L::E_STAGE + rCap * 16);
        *z = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const int T = a.num_tiles > blockIdx.x ? (int)ceil_div(a.num_tiles - blockIdx.x, gridDim.x) : 0;
    const int K = a.k;

    if (warp >= wrEpiWarp0 && warp < wrEpiWarp0 + rEpiWarps && (a.dbg & 8)) {
        // probe: no MMA / epilogue
    } else if (warp >= wrEpiWarp0 && warp < wrEpiWarp0 + rEpiWarps) {
        // ------------------------------------------------------------ MMA issue (warp 16, lane 0) + epilogue
        // TMEM columns: D_0 0..63, D_1 64..127, U_0 128..319, U_1 320..511 (single-buffered)
        const int ew = warp - wrEpiWarp0;  // TMEM lane quadrant
        const float binv = a.binv[0];
        auto issue = [&](int i, int h) {
            constexpr uint32_t idn = idesc_f16(kTile, 64, SPLIT ? 0 : 1);
            constexpr uint32_t idu = idesc_f16(kTile, 192, SPLIT ? 0 : 1);
            mbar_wait(a_full + h, (uint32_t)(i & 1));
            if (h == 0 && i >= 1) mbar_wait(acc_free, (uint32_t)((i - 1) & 1));
            tc_fence_after();
            if (a.dbg & 2) {
                mbar_arrive(mma_done + h);
                if (h == 1) mbar_arrive(acc_full);
                return;
            }
            const uint32_t d = tmem_base + (uint32_t)(h * 64);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int t = ks >> 1, kk = ks & 1;
                const uint32_t ko = (uint32_t)((32 * h + 16 * kk) * 2);
                const uint32_t ao = (uint32_t)t * (kTile * 128) + ko, bo = (uint32_t)t * (64 * 128) + ko;
                mma_f16(d, desc_sw128(A_hi + ao), desc_sw128(B_hi + bo), idn, ks > 0 ? 1u : 0u);
                if (SPLIT) {
                    mma_f16(d, desc_sw128(A_hi + ao), desc_sw128(B_lo + bo), idn, 1u);
                    mma_f16(d, desc_sw128(A_lo + ao), desc_sw128(B_hi + bo), idn, 1u);
                }
            }
            if (DLOC) {
                const uint32_t u = tmem_base + 128u + (uint32_t)(h * 192);
#pragma unroll
                for (int kk = 0; kk < 2; ++kk) {
                    const uint32_t ko = (uint32_t)((32 * h + 16 * kk) * 2);
                    const uint32_t ao = 3u * (kTile * 128) + ko;
                    mma_f16(u, desc_sw128(A_hi + ao), desc_sw128(B_hi + ko), idu, kk > 0 ? 1u : 0u);
                    if (SPLIT) {
                        mma_f16(u, desc_sw128(A_hi + ao), desc_sw128(B_lo + ko), idu, 1u);
                        mma_f16(u, desc_sw128(A_lo + ao), desc_sw128(B_hi + ko), idu, 1u);
                    }
                }
            }
            mma_commit(mma_done + h);
            if (h == 1) mma_commit(acc_full);
        };
        auto epilogue = [&](int i) {
            mbar_wait_sleep(acc_full, (uint32_t)(i & 1));
            tc_fence_after();
            const int b = i & 1;
            const int tr = ew * 32 + lane;
            const int64_t p = (blockIdx.x + (int64_t)i * gridDim.x) * kTile + tr;
            const float s0 = exp2i(rs[(b * 2 + 0) * kTile + tr]) * binv;
            const float s1 = exp2i(rs[(b * 2 + 1) * kTile + tr]) * binv;
            const uint32_t tb = tmem_base + ((uint32_t)(ew * 32) << 16);
            const bool pv = p < a.total;
            float *orow = a.out + p * (BLK ? a.ld_out : 64);
#pragma unroll 1
            for (int c0 = 0; c0 < 64; c0 += 16) {
                float x0[16], x1[16];
                tmem_ld16(tb + (uint32_t)c0, x0);
                tmem_ld16(tb + 64u + (uint32_t)c0, x1);
                if (pv) {
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
            if (DLOC) {
                float nb0 = 0.f, nb1 = 0.f, nb2 = 0.f;
#pragma unroll 1
                for (int c0 = 0; c0 < 64; c0 += 16) {
                    // own row, 32 bytes per lane per load (LDG.256): one line touch per 8 channels
                    float f[16], f8[8];
                    if (pv) {
                        ldg_nc8r(a.feat + p * 64 + c0, f8);
#pragma unroll
                        for (int q = 0; q < 8; ++q) f[q] = f8[q];
                        ldg_nc8r(a.feat + p * 64 + c0 + 8, f8);
#pragma unroll
                        for (int q = 0; q < 8; ++q) f[8 + q] = f8[q];
                    } else {
#pragma unroll
                        for (int q = 0; q < 16; ++q) f[q] = 0.f;
                    }
#pragma unroll
                    for (int tt = 0; tt < 3; ++tt) {
                        float u0[16], u1[16];
                        tmem_ld16(tb + 128u + (uint32_t)(64 * tt + c0), u0);
                        tmem_ld16(tb + 320u + (uint32_t)(64 * tt + c0), u1);
                        float acc = 0.f;
#pragma unroll
                        for (int c = 0; c < 16; ++c) acc = fmaf(f[c], fmaf(u1[c], s1, u0[c] * s0), acc);
                        if (tt == 0) nb0 += acc;
                        if (tt == 1) nb1 += acc;
                        if (tt == 2) nb2 += acc;
                    }
                }
                if (pv) {
                    a.dloc[p * 3 + 0] = a.centre[p * 3 + 0] - nb0;
                    a.dloc[p * 3 + 1] = a.centre[p * 3 + 1] - nb1;
                    a.dloc[p * 3 + 2] = a.centre[p * 3 + 2] - nb2;
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_free);
        };
        for (int i = 0; i < T; ++i) {
            if (warp == wrMmaWarp) {
                if (lane == 0) {
                    issue(i, 0);
                    issue(i, 1);
                }
                __syncwarp();
            }
            epilogue(i);
        }
    } else if (warp >= wrIdxWarp0) {
        // ------------------------------------------------------------ index producer + epilogue
        const int t = (warp - wrIdxWarp0) * 32 + lane;  // 0..127
        const int r = t >> 1, par = t & 1;             // row of the group, entry parity
        const int G = 2 * T;                           // 64-row groups of this CTA
        auto grow = [&](int gg) -> int64_t {           // global index of row r of group gg
            return (blockIdx.x + (int64_t)(gg >> 1) * gridDim.x) * kTile + (gg & 1) * 64 + r;
        };
        // pipeline registers: offsets of group gg+2, entries (source rows) of gg+1, positions of gg
        int32_t o2_lo = 0, o2_hi = 0;   // row range, group gg+2
        int32_t o1_lo = 0, o1_hi = 0;   // row range, group gg+1
        int32_t src1[rMaxRow / 2];      // source rows i of group gg+1 (this thread's parity)
        int32_t src0[rMaxRow / 2];
        int32_t o0_lo = 0, o0_hi = 0;
        auto load_off = [&](int gg, int32_t &lo, int32_t &hi) {
            lo = hi = 0;
            if (gg < G) {
                const int64_t j = grow(gg);
                if (j < a.total) {
                    lo = __ldg(a.csr.off + j);
                    hi = __ldg(a.csr.off + j + 1);
                }
            }
        };
        auto load_src = [&](int32_t lo, int32_t hi, int32_t (&src)[rMaxRow / 2]) {
            const int cnt = min(hi - lo, rMaxRow);
#pragma unroll
            for (int q = 0; q < rMaxRow / 2; ++q) {
                const int s2 = 2 * q + par;
                src[q] = s2 < cnt ? __ldg(a.csr.ent + lo + s2) / K : 0;
            }
        };
        // prologue: offsets of groups 0, 1; sources of group 0
        load_off(0, o0_lo, o0_hi);
        load_off(1, o1_lo, o1_hi);
        load_src(o0_lo, o0_hi, src0);
        for (int gg = 0; gg < G; ++gg) {
            // positions of group gg (sources loaded last iteration), sources of gg+1, offsets of gg+2
            const int64_t j = grow(gg);
            const bool jv = gg < G && j < a.total;
            float lj0 = 0.f, lj1 = 0.f, lj2 = 0.f;
            if (jv) {
                lj0 = __ldg(a.loc + j * 3 + 0);
                lj1 = __ldg(a.loc + j * 3 + 1);
                lj2 = __ldg(a.loc + j * 3 + 2);
            }
            const int cnt = jv ? o0_hi - o0_lo : 0;
            float q0[rMaxRow / 2], q1[rMaxRow / 2], q2[rMaxRow / 2];
#pragma unroll
            for (int q = 0; q < rMaxRow / 2; ++q) {
                const bool v = 2 * q + par < min(cnt, rMaxRow);
                q0[q] = v ? __ldg(a.loc + (int64_t)src0[q] * 3 + 0) : 0.f;
                q1[q] = v ? __ldg(a.loc + (int64_t)src0[q] * 3 + 1) : 0.f;
                q2[q] = v ? __ldg(a.loc + (int64_t)src0[q] * 3 + 2) : 0.f;
            }
            load_src(o1_lo, o1_hi, src1);
            load_off(gg + 2, o2_lo, o2_hi);
            // row starts within the stage: exclusive scan of the staged counts over the 64 rows
            const bool direct_row = cnt > rMaxRow;
            const int staged = direct_row ? 0 : cnt;
            int incl = par == 0 ? staged : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            named_bar(1, 128);
            if (lane == 31) scan[warp - wrIdxWarp0] = incl;
            named_bar(1, 128);
            int base = 0;
            for (int w = 0; w < warp - wrIdxWarp0; ++w) base += scan[w];
            const int start = base + incl - staged;  // incl of both threads of a row covers the row
            const bool direct = direct_row || start + staged > rCap;
            // store
            const int st = gg % rStages;
            if (gg >= rStages) mbar_wait_sleep(e_empty + st, (uint32_t)(((gg / rStages) + 1) & 1));
            const uint32_t es = E0 + (uint32_t)(st * L::E_STAGE);
            if (!direct) {
#pragma unroll
                for (int q = 0; q < rMaxRow / 2; ++q) {
                    const int s2 = 2 * q + par;
                    if (s2 < staged)
                        sts128f(es + (uint32_t)((start + s2) * 16), __int_as_float(src0[q]), q0[q] - lj0, q1[q] - lj1,
                                q2[q] - lj2);
                }
            }
            if (par == 0) {
                const uint32_t rec = direct ? ((rDirect << 16) | (uint32_t)min(cnt, 0xffff)) : (((uint32_t)start << 16) | (uint32_t)cnt);
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(R0 + (uint32_t)((st * 64 + r) * 4)), "r"(rec) : "memory");
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(e_full + st);
            // rotate the pipeline
            o0_lo = o1_lo, o0_hi = o1_hi;
            o1_lo = o2_lo, o1_hi = o2_hi;
#pragma unroll
            for (int q = 0; q < rMaxRow / 2; ++q) src0[q] = src1[q];
        }
    } else {
        // ------------------------------------------------------------ gather warps (wide lanes)
        // Item g = (tile i, half h, group of 8 rows q): i = g / 32, h = (g / 16) % 2, q = g % 16;
        // warp w takes g = w, w + 12, ...  Lane (pt, cl): row 8q + {0,4,1,5,2,6,3,7}[pt],
        // channels 32h + 8cl .. +7 (one 32-byte load per slot).  Lists are walked in 4-slot
        // batches up to the longest of the item's 8; past a list's end a slot reads the
        // stage's zero entry (row 0, offsets 0) with bias weight 0.
        const int pt = lane >> 2, cl = lane & 3;
        const int rowoff = ((pt & 1) << 2) + (pt >> 1);
        const int NI = T * 32;
        float v[4][8];
        float2 x[4][4];
        struct ItemW {
            uint32_t eb, ez;  // first staged entry of the row, the stage's zero entry
            int cnt, start;   // list length, staged start (rDirect: direct path)
            int nb;           // 4-slot batches (warp-uniform)
            bool direct;      // any direct row in the item (warp-uniform)
        };
        auto open_w = [&](int g, ItemW &it) {
            const int i = g >> 5, q = g & 15;
            const int gg = 2 * i + (q >> 3), st = gg % rStages;
            mbar_wait(e_full + st, (uint32_t)((gg / rStages) & 1));
            const int row = 8 * q + rowoff;
            const uint32_t es = E0 + (uint32_t)(st * L::E_STAGE);
            const uint32_t rec = (uint32_t)lds32(R0 + (uint32_t)((st * 64 + (row & 63)) * 4));
            it.cnt = (int)(rec & 0xffffu);
            it.start = (int)(rec >> 16);
            it.ez = es + (uint32_t)(rCap * 16);
            it.eb = es + (uint32_t)(it.start * 16);
            const bool dr = it.start == (int)rDirect;
            if (dr) {
                const int64_t p = (blockIdx.x + (int64_t)i * gridDim.x) * kTile + row;
                it.cnt = p < a.total ? __ldg(a.csr.off + p + 1) - __ldg(a.csr.off + p) : 0;
            }
            it.direct = __any_sync(0xffffffffu, dr);
            it.nb = ((int)__reduce_max_sync(0xffffffffu, (uint32_t)it.cnt) + 3) >> 2;
        };
        auto load4w = [&](const ItemW &it, int h, int b0) {
            const float *src = a.rows + 32 * h + 8 * cl;
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
                const int sl = b0 + s2;
                const bool ok = sl < it.cnt;
                const int32_t j = lds32(ok ? it.eb + (uint32_t)(sl * 16) : it.ez);
                ldg_nc8r_if(src + (int64_t)j * (BLK ? a.ld_rows : 64), v[s2], ok);
            }
        };
        auto fma4w = [&](const ItemW &it, int b0) {
#pragma unroll
            for (int s2 = 0; s2 < 4; ++s2) {
                const int sl = b0 + s2;
                const bool ok = sl < it.cnt;
                const float4 e = lds128f(ok ? it.eb + (uint32_t)(sl * 16) : it.ez);
                const float wb = ok ? 1.f : 0.f;
                const float2 w0 = make_float2(e.y, e.y), w1 = make_float2(e.z, e.z), w2 = make_float2(e.w, e.w);
                const float2 w3 = make_float2(wb, wb);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float2 f = make_float2(v[s2][2 * c], v[s2][2 * c + 1]);
                    x[0][c] = ffma2(f, w0, x[0][c]);
                    x[1][c] = ffma2(f, w1, x[1][c]);
                    x[2][c] = ffma2(f, w2, x[2][c]);
                    x[3][c] = ffma2(f, w3, x[3][c]);
                }
            }
        };
        // direct path (rare): each lane walks its point's list from the CSR
        auto direct_w = [&](const ItemW &it, int g) {
            const int i = g >> 5, h = (g >> 4) & 1, q = g & 15;
            const int64_t p = (blockIdx.x + (int64_t)i * gridDim.x) * kTile + 8 * q + rowoff;
            const bool pv = p < a.total;
            const bool staged = it.start != (int)rDirect;
            const int32_t o0 = pv ? __ldg(a.csr.off + p) : 0;
            const float lp0 = pv ? __ldg(a.loc + p * 3 + 0) : 0.f;
            const float lp1 = pv ? __ldg(a.loc + p * 3 + 1) : 0.f;
            const float lp2 = pv ? __ldg(a.loc + p * 3 + 2) : 0.f;
            const float *src = a.rows + 32 * h + 8 * cl;
            const int mx = 4 * it.nb;
            for (int sl = 0; sl < mx; ++sl) {
                if (sl < it.cnt) {
                    float4 e;
                    if (staged) {
                        e = lds128f(it.eb + (uint32_t)(sl * 16));
                    } else {
                        const int32_t jr = __ldg(a.csr.ent + o0 + sl) / K;
                        e = make_float4(__int_as_float(jr), __ldg(a.loc + (int64_t)jr * 3 + 0) - lp0,
                                        __ldg(a.loc + (int64_t)jr * 3 + 1) - lp1, __ldg(a.loc + (int64_t)jr * 3 + 2) - lp2);
                    }
                    float r[8];
                    ldg_nc8r(src + (int64_t)__float_as_int(e.x) * (BLK ? a.ld_rows : 64), r);
                    const float2 w0 = make_float2(e.y, e.y), w1 = make_float2(e.z, e.z), w2 = make_float2(e.w, e.w);
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const float2 f = make_float2(r[2 * c], r[2 * c + 1]);
                        x[0][c] = ffma2(f, w0, x[0][c]);
                        x[1][c] = ffma2(f, w1, x[1][c]);
                        x[2][c] = ffma2(f, w2, x[2][c]);
                        x[3][c] = fadd2(x[3][c], f);
                    }
                }
            }
        };
        ItemW cur;
        if (warp < NI) {
            open_w(warp, cur);
            if (!cur.direct && cur.nb > 0) load4w(cur, 0, 0);
        }
        for (int g = warp; g < NI; g += wrGatherWarps) {
            const int i = g >> 5, h = (g >> 4) & 1, q = g & 15;
            const int row = 8 * q + rowoff;
            const int64_t p = (blockIdx.x + (int64_t)i * gridDim.x) * kTile + row;
#pragma unroll
            for (int tt = 0; tt < 4; ++tt)
#pragma unroll
                for (int c = 0; c < 4; ++c) x[tt][c] = make_float2(0.f, 0.f);
            if (cur.direct) {
                direct_w(cur, g);
            } else if (cur.nb > 0) {
                fma4w(cur, 0);
                for (int b = 1; b < cur.nb; ++b) {
                    load4w(cur, h, 4 * b);
                    fma4w(cur, 4 * b);
                }
            }
            const int gn = g + wrGatherWarps;
            if (gn >= NI || (gn >> 5) != i) {  // this warp's last item of tile i: release both stages
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(e_empty + (2 * i) % rStages);
                    mbar_arrive(e_empty + (2 * i + 1) % rStages);
                }
            }
            if (gn < NI) {  // first batch of the next item
                open_w(gn, cur);
                if (!cur.direct && cur.nb > 0) load4w(cur, (gn >> 4) & 1, 0);
            }
            // ---- per-(point, half) power-of-two scale, split, A-operand row
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
            if (p >= a.total) sc = 0.f;
            const bool first_in_half = g - wrGatherWarps < 0 || ((g - wrGatherWarps) >> 4) != (g >> 4);
            if (first_in_half && i >= 1) mbar_wait(mma_done + h, (uint32_t)((i - 1) & 1));
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
                sts128r(A_hi + off, hv[0], hv[1], hv[2], hv[3]);
                if (SPLIT) sts128r(A_lo + off, lv[0], lv[1], lv[2], lv[3]);
            }
            if (cl == 0) sts8(rs_s + (uint32_t)(((i & 1) * 2 + h) * kTile + row), e);
            if (gn >= NI || (gn >> 4) != (g >> 4)) {  // this warp's last rows of half-tile (i, h)
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(a_full + h);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == wrMmaWarp) {
        tc_fence_after();
        tmem_dealloc(tmem_base, 512);
    }
}

}  // namespace fast

void launch_pack_b_ld(bool split, int cin, int cout, int ld_cin, const float *theta, const float *theta_b, int reverse,
                      int nout, int gc, uint8_t *img, float *binv, cudaStream_t st);

static int fast_reverse_impl(bool split, int64_t total, int k, const float *rows, int64_t ld_rows, const float *loc,
                             Csr csr, const float *theta, const float *theta_b, int ld_cin, float *out, int64_t ld_out,
                             bool acc, const float *feat, const float *centre, float *dloc, cudaStream_t st,
                             const uint8_t *pre_img = nullptr, const float *pre_zero = nullptr);

// reverse pass for c_in = c_out = 64, d = 3: out = A(theta)^T rows (d_features / flex_deconv),
// plus the neighbour-role location gradient when dloc is non-null
int tc_fast_reverse(bool split, int64_t total, int k, const float *rows, const float *loc, Csr csr, const float *theta,
                    const float *theta_b, float *out, const float *feat, const float *centre, float *dloc,
                    cudaStream_t st) {
    return fast_reverse_impl(split, total, k, rows, 64, loc, csr, theta, theta_b, 64, out, 64, false, feat, centre, dloc,
                             st);
}

// one 64 x 64 channel block of a wider reverse pass (no location gradient): gathered rows /
// output rows with strides ld_rows / ld_out, theta rows of ld_cin input channels, the block's
// product added to out when acc
// (pre_img: this block's reverse image already packed -- tc_pack_b layout, 1 / scale after it --
// and pre_zero: 64 zero floats, both from the caller; null = packed / zeroed here)
int tc_fast_reverse_block(bool split, int64_t total, int k, const float *rows, int64_t ld_rows, const float *loc,
                          Csr csr, const float *theta, const float *theta_b, int ld_cin, float *out, int64_t ld_out,
                          bool acc, cudaStream_t st, const uint8_t *pre_img, const float *pre_zero) {
    return fast_reverse_impl(split, total, k, rows, ld_rows, loc, csr, theta, theta_b, ld_cin, out, ld_out, acc, nullptr,
                             nullptr, nullptr, st, pre_img, pre_zero);
}

static int fast_reverse_impl(bool split, int64_t total, int k, const float *rows, int64_t ld_rows, const float *loc,
                             Csr csr, const float *theta, const float *theta_b, int ld_cin, float *out, int64_t ld_out,
                             bool acc, const float *feat, const float *centre, float *dloc, cudaStream_t st,
                             const uint8_t *pre_img, const float *pre_zero) {
    using namespace fast;
    const size_t bbytes = (size_t)RevL<true>::B_BYTES * (split ? 2 : 1);
    const bool own = !(pre_img && pre_zero);
    uint8_t *img = own ? (uint8_t *)scratch_alloc(bbytes + 512, st) : const_cast<uint8_t *>(pre_img);
    if (!img) return set_error(FC_ERR_CUDA, "scratch allocation failed (fast reverse)");
    float *binv = reinterpret_cast<float *>(img + bbytes);
    float *zero = own ? reinterpret_cast<float *>(img + bbytes + 256) : const_cast<float *>(pre_zero);
    if (own) {
        cudaMemsetAsync(zero, 0, 256, st);
        launch_pack_b_ld(split, 64, 64, ld_cin, theta, theta_b, 1, 64, 64, img, binv, st);
    }
    RevArgs a{};
    a.total = total;
    a.num_tiles = ceil_div(total, kTile);
    a.k = k;
    a.rows = rows;
    a.zero = zero;
    a.loc = loc;
    a.csr = csr;
    a.bimg = img;
    a.binv = binv;
    a.out = out;
    a.feat = feat;
    a.centre = centre;
    a.dloc = dloc;
    a.ld_rows = (int)ld_rows;
    a.ld_out = (int)ld_out;
    a.acc = acc ? 1 : 0;
    {
        const char *e = getenv("FC_DBG");
        a.dbg = e ? atoi(e) : 0;
    }
    const int grid = (int)std::min<int64_t>(a.num_tiles, num_sms());
    prof_begin(dloc ? "tc_reverse_dloc" : "tc_reverse", st);
    static int narrow = -1;
    if (narrow < 0) {
        const char *e = getenv("FC_REV_NARROW");
        narrow = (e && e[0] == '1') ? 1 : 0;
    }
    if ((ld_rows != 64 || ld_out != 64 || acc) && (narrow || dloc)) {
        prof_end(st);
        if (own) scratch_free(img, st);
        return set_error(FC_ERR_UNSUPPORTED, "channel-block reverse needs the wide kernel without d_locations");
    }
#define FC_LAUNCH_REV(S, D)                                                                                     \
    do {                                                                                                        \
        if (narrow) {                                                                                           \
            static uint64_t attr = 0;                                                                           \
            if (first_use_on_device(attr)) {                                                                                        \
                cudaFuncSetAttribute(tc_rev64_kernel<S, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, RevL<S>::SMEM_ALLOC); \
            }                                                                                                   \
            tc_rev64_kernel<S, D><<<grid, rThreads, RevL<S>::SMEM_ALLOC, st>>>(a);                              \
        } else {                                                                                                \
            static uint64_t attr = 0;                                                                           \
            if (first_use_on_device(attr)) {                                                                                        \
                cudaFuncSetAttribute(tc_rev64w_kernel<S, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, RevL<S>::SMEM_ALLOC); \
            }                                                                                                   \
            tc_rev64w_kernel<S, D><<<grid, wrThreads, RevL<S>::SMEM_ALLOC, st>>>(a);                            \
        }                                                                                                       \
    } while (0)
    const bool blk = ld_rows != 64 || ld_out != 64 || acc;  // (a separate instance: the plain one keeps its registers)
    if (blk) {
        static uint64_t attr_t = 0, attr_f = 0;
        if (split) {
            if (first_use_on_device(attr_t))
                cudaFuncSetAttribute(tc_rev64w_kernel<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     RevL<true>::SMEM_ALLOC);
            tc_rev64w_kernel<true, false, true><<<grid, wrThreads, RevL<true>::SMEM_ALLOC, st>>>(a);
        } else {
            if (first_use_on_device(attr_f))
                cudaFuncSetAttribute(tc_rev64w_kernel<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     RevL<false>::SMEM_ALLOC);
            tc_rev64w_kernel<false, false, true><<<grid, wrThreads, RevL<false>::SMEM_ALLOC, st>>>(a);
        }
    } else if (split) {
        if (dloc) FC_LAUNCH_REV(true, true);
        else FC_LAUNCH_REV(true, false);
    } else {
        if (dloc) FC_LAUNCH_REV(false, true);
        else FC_LAUNCH_REV(false, false);
    }
#undef FC_LAUNCH_REV
    prof_end(st);
    count_launch();
    if (own) scratch_free(img, st);
    return check_launch("tc_rev64_kernel");
}

}  // namespace fc
