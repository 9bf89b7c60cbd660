// conv_simt.cu -- CUDA-core flex-convolution kernels (fp32 FMA and fp64 reference order).
//
// One "gather -> moments -> contraction" kernel serves three operators:
//   forward      : X_i = sum_{s} (l_i - l_j, 1) (x) f_j  over j = nbr[i, s]       (_native.pyx:47-59)
//                  out_i = [theta; theta_b] . X_i                                  (_native.pyx:60-66)
//   d_features / : Y_j = sum_{(i,s) in R(j)} (l_i - l_j, 1) (x) g_i  (reverse CSR)
//   flex_deconv    d_f_j = [theta; theta_b]^T . Y_j  -- the same sum as the reference's
//                  per-(i,s) scatter of W_i (_native.pyx:106-120), regrouped per target j.
// Every warp owns whole points (no cross-warp dependencies, no atomics): results are
// deterministic and independent of the launch configuration.
#include "fc_common.cuh"

namespace fc {

// wt[(c*(D+1)+t)*cout + cp] = theta[cp,c,t] (t < D) | theta_b[cp,c] (t == D)   forward packing
// wr[(cp*(D+1)+t)*cin + c]  = same value                                       adjoint packing
template <typename T>
__global__ void pack_weights_kernel(int cin, int d, int cout, const T *__restrict__ theta,
                                    const T *__restrict__ theta_b, T *__restrict__ wt,
                                    T *__restrict__ wr) {
    const int64_t total = (int64_t)cout * cin * (d + 1);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(q % (d + 1));
        const int64_t r = q / (d + 1);
        const int c = (int)(r % cin);
        const int cp = (int)(r / cin);
        const T v = (t < d) ? theta[((int64_t)cp * cin + c) * d + t] : theta_b[(int64_t)cp * cin + c];
        if (wt) wt[((int64_t)c * (d + 1) + t) * cout + cp] = v;
        if (wr) wr[((int64_t)cp * (d + 1) + t) * cin + c] = v;
    }
}

// Moments of one centre point, computed by one warp (lanes over channels), written
// c-major into xs[c*(DP+1) + t].  Per (c,t) the neighbour terms are added in slot
// order, exactly the reference's accumulation order (_native.pyx:52-59).
//   REVERSE = false: neighbours j = base + nbr[p*k + s], offset = l_p - l_j
//   REVERSE = true : (i, s) from the reverse CSR of p, i = e / k, offset = l_i - l_p
template <typename T, int DP, bool REVERSE>
__device__ __forceinline__ void warp_moments(const T *__restrict__ rows, int gc,
                                             const T *__restrict__ loc,
                                             const int32_t *__restrict__ nbr, int k, Csr csr,
                                             int64_t p, int64_t base, T *__restrict__ xs,
                                             int lane) {
    T lp[DP];
#pragma unroll
    for (int t = 0; t < DP; ++t) lp[t] = loc[p * DP + t];
    int64_t q0 = 0, q1 = k;
    if (REVERSE) {
        q0 = csr.off[p];
        q1 = csr.off[p + 1];
    }
    for (int c0 = 0; c0 < gc; c0 += 32) {
        const int c = c0 + lane;
        const bool ok = c < gc;
        T acc[DP + 1];
#pragma unroll
        for (int t = 0; t <= DP; ++t) acc[t] = T(0);
        for (int64_t q = q0; q < q1; ++q) {
            int64_t j;
            if (REVERSE)
                j = (int64_t)csr.ent[q] / k;
            else
                j = base + nbr[p * k + q];
            T o[DP];
#pragma unroll
            for (int t = 0; t < DP; ++t)
                o[t] = REVERSE ? Ar<T>::sub(loc[j * DP + t], lp[t]) : Ar<T>::sub(lp[t], loc[j * DP + t]);
            const T v = ok ? rows[j * gc + c] : T(0);
#pragma unroll
            for (int t = 0; t < DP; ++t) acc[t] = Ar<T>::madd(acc[t], v, o[t]);
            acc[DP] = Ar<T>::add(acc[DP], v);
        }
        if (ok) {
#pragma unroll
            for (int t = 0; t <= DP; ++t) xs[c * (DP + 1) + t] = acc[t];
        }
    }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Gather-moment-contract.  Each warp processes PPW points at a time (persistent loop).
//   out[p, cp] = sum_{c, t} w[(c*(DP+1)+t)*cout + cp] * M_p[c, t]   (c-major, t fastest =
//   the reference's contraction order, _native.pyx:60-66).
// Optional (REVERSE, dloc != nullptr): neighbour role of the location gradient,
//   dloc[j,t] = centre[j,t] - sum_c f[j,c] sum_cp theta[cp,c,t] * Y_j[cp, DP]
// (the -dt terms of _native.pyx:121-127 regrouped per j; `feat` rows have `cout` channels).
template <typename T, int DP, bool REVERSE, int PPW>
__global__ void __launch_bounds__(256)
    gmc_kernel(int64_t total, int64_t n, int gc, int k, int cout, const T *__restrict__ rows,
               const T *__restrict__ loc, const int32_t *__restrict__ nbr, Csr csr,
               const T *__restrict__ w, T *__restrict__ out, const T *__restrict__ feat,
               const T *__restrict__ theta, const T *__restrict__ centre, T *__restrict__ dloc) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ktot = gc * (DP + 1);
    T *xs = reinterpret_cast<T *>(smem_raw) + (int64_t)warp * PPW * ktot;
    const int64_t nwarps = (int64_t)gridDim.x * 8;
    for (int64_t g0 = ((int64_t)blockIdx.x * 8 + warp) * PPW; g0 < total; g0 += nwarps * PPW) {
#pragma unroll
        for (int q = 0; q < PPW; ++q) {
            const int64_t p = g0 + q;
            if (p < total)
                warp_moments<T, DP, REVERSE>(rows, gc, loc, nbr, k, csr, p, (p / n) * n,
                                             xs + q * ktot, lane);
        }
        __syncwarp();
        for (int cp0 = 0; cp0 < cout; cp0 += 32) {
            const int cp = cp0 + lane;
            if (cp < cout) {
                T acc[PPW];
#pragma unroll
                for (int q = 0; q < PPW; ++q) acc[q] = T(0);
                for (int kk = 0; kk < ktot; ++kk) {
                    const T wv = w[(int64_t)kk * cout + cp];
#pragma unroll
                    for (int q = 0; q < PPW; ++q) acc[q] = Ar<T>::madd(acc[q], wv, xs[q * ktot + kk]);
                }
#pragma unroll
                for (int q = 0; q < PPW; ++q)
                    if (g0 + q < total) out[(g0 + q) * cout + cp] = acc[q];
            }
        }
        if (REVERSE && dloc != nullptr) {
            // theta is the conv's [gc (= conv c_out), cout (= conv c_in), DP] tensor.
#pragma unroll
            for (int q = 0; q < PPW; ++q) {
                const int64_t p = g0 + q;
                if (p >= total) break;
                T part[DP];
#pragma unroll
                for (int t = 0; t < DP; ++t) part[t] = T(0);
                for (int c0 = 0; c0 < cout; c0 += 32) {
                    const int c = c0 + lane;
                    if (c < cout) {
                        T z[DP];
#pragma unroll
                        for (int t = 0; t < DP; ++t) z[t] = T(0);
                        for (int cp = 0; cp < gc; ++cp) {
                            const T yb = xs[q * ktot + cp * (DP + 1) + DP];
#pragma unroll
                            for (int t = 0; t < DP; ++t)
                                z[t] = Ar<T>::madd(z[t], theta[((int64_t)cp * cout + c) * DP + t], yb);
                        }
                        const T fv = feat[p * cout + c];
#pragma unroll
                        for (int t = 0; t < DP; ++t) part[t] = Ar<T>::madd(part[t], fv, z[t]);
                    }
                }
#pragma unroll
                for (int t = 0; t < DP; ++t) {
                    const T s = warp_sum(part[t]);
                    if (lane == 0) dloc[p * DP + t] = Ar<T>::sub(centre[p * DP + t], s);
                }
            }
        }
        __syncwarp();
    }
}

// Centre role of the location gradient:
//   centre[i,t] = sum_c (sum_s f[j_s, c]) * (sum_cp theta[cp,c,t] g[i,cp])
// (the +dt terms of _native.pyx:121-127 summed over s: sum_s f_j . W_i[:,t] = X_i[:,D] . W_i[:,t]).
template <typename T, int DP>
__global__ void __launch_bounds__(256)
    dloc_centre_kernel(int64_t total, int64_t n, int cin, int k, int cout,
                       const T *__restrict__ feat, const int32_t *__restrict__ nbr,
                       const T *__restrict__ g, const T *__restrict__ theta,
                       T *__restrict__ centre) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    T *gs = reinterpret_cast<T *>(smem_raw) + (int64_t)warp * cout;
    const int64_t nwarps = (int64_t)gridDim.x * 8;
    for (int64_t p = (int64_t)blockIdx.x * 8 + warp; p < total; p += nwarps) {
        const int64_t base = (p / n) * n;
        for (int cp = lane; cp < cout; cp += 32) gs[cp] = g[p * cout + cp];
        __syncwarp();
        T part[DP];
#pragma unroll
        for (int t = 0; t < DP; ++t) part[t] = T(0);
        for (int c0 = 0; c0 < cin; c0 += 32) {
            const int c = c0 + lane;
            if (c < cin) {
                T xb = T(0);
                for (int s = 0; s < k; ++s) xb = Ar<T>::add(xb, feat[(base + nbr[p * k + s]) * cin + c]);
                T z[DP];
#pragma unroll
                for (int t = 0; t < DP; ++t) z[t] = T(0);
                for (int cp = 0; cp < cout; ++cp) {
                    const T gv = gs[cp];
#pragma unroll
                    for (int t = 0; t < DP; ++t)
                        z[t] = Ar<T>::madd(z[t], theta[((int64_t)cp * cin + c) * DP + t], gv);
                }
#pragma unroll
                for (int t = 0; t < DP; ++t) part[t] = Ar<T>::madd(part[t], xb, z[t]);
            }
        }
#pragma unroll
        for (int t = 0; t < DP; ++t) {
            const T s = warp_sum(part[t]);
            if (lane == 0) centre[p * DP + t] = s;
        }
        __syncwarp();
    }
}

// d_theta partials: block (chunk, slice) accumulates, over its contiguous point chunk
// in ascending order, the entries e = slice*256*RPT + tid + 256*r of
//   P[cp, c, t] = sum_i g[i, cp] * X_i[c, t]        (_native.pyx:106-112)
// then writes them to partial[chunk][e]; dtheta_reduce sums chunks in fixed order.
template <typename T, int DP, int RPT>
__global__ void __launch_bounds__(256)
    dtheta_partial_kernel(int64_t total, int64_t n, int cin, int k, int cout,
                          const T *__restrict__ feat, const T *__restrict__ loc,
                          const int32_t *__restrict__ nbr, const T *__restrict__ g,
                          T *__restrict__ partial, int64_t chunk_pts, int tile) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ktot = cin * (DP + 1);
    const int64_t E = (int64_t)cout * ktot;
    T *xs = reinterpret_cast<T *>(smem_raw);
    T *gs = xs + (int64_t)tile * ktot;
    const int64_t p_begin = (int64_t)blockIdx.x * chunk_pts;
    const int64_t p_end = min(total, p_begin + chunk_pts);
    const int64_t e0 = (int64_t)blockIdx.y * 256 * RPT + threadIdx.x;
    int cps[RPT], kks[RPT];
    T acc[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int64_t e = e0 + 256 * r;
        cps[r] = (int)(e / ktot);
        kks[r] = (int)(e % ktot);
        acc[r] = T(0);
    }
    const int ppw = tile / 8;
    for (int64_t t0 = p_begin; t0 < p_end; t0 += tile) {
        for (int q = 0; q < ppw; ++q) {
            const int pl = warp * ppw + q;
            const int64_t p = t0 + pl;
            if (p < p_end) {
                warp_moments<T, DP, false>(feat, cin, loc, nbr, k, Csr{nullptr, nullptr}, p,
                                           (p / n) * n, xs + (int64_t)pl * ktot, lane);
                for (int cp = lane; cp < cout; cp += 32) gs[(int64_t)pl * cout + cp] = g[p * cout + cp];
            }
        }
        __syncthreads();
        const int np = (int)min((int64_t)tile, p_end - t0);
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            if (e0 + 256 * r < E) {
                T a = acc[r];
                for (int pl = 0; pl < np; ++pl)
                    a = Ar<T>::madd(a, gs[(int64_t)pl * cout + cps[r]], xs[(int64_t)pl * ktot + kks[r]]);
                acc[r] = a;
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int64_t e = e0 + 256 * r;
        if (e < E) partial[(int64_t)blockIdx.x * E + e] = acc[r];
    }
}

// Fixed-order (ascending chunk) reduction of the d_theta partials, accumulated in fp64.
// Partial layouts: tmajor = 0: element e = (c' * cin + c) * (d + 1) + t; tmajor = 1 (the
// tensor-core accumulators' column order): e = c' * cin * (d + 1) + t * cin + c.
template <typename T>
__global__ void __launch_bounds__(256) dtheta_reduce_kernel(int chunks, int cin, int d, int cout,
                                                            const T *__restrict__ partial, T *__restrict__ d_theta,
                                                            T *__restrict__ d_theta_b, int tmajor, int ld) {
    // a CTA owns 32 consecutive elements; warp w adds the chunks of its contiguous block in
    // ascending order (fp64, coalesced 32-element rows), the 8 block sums are then added in
    // warp order -- a fixed order (deterministic) with 8 warps of loads in flight per element
    constexpr int W = 8;
    __shared__ double red[W][32];
    const int64_t E = (int64_t)cout * cin * (d + 1);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int per = (chunks + W - 1) / W;
    const int c0 = min(chunks, w * per), c1 = min(chunks, c0 + per);
    for (int64_t e0 = (int64_t)blockIdx.x * 32; e0 < E; e0 += (int64_t)gridDim.x * 32) {
        const int64_t e = e0 + lane;
        double s = 0.0;
        if (e < E) {
            const T *src = partial + e;
            int ch = c0;
            for (; ch + 4 <= c1; ch += 4) {
                const T v0 = src[(int64_t)ch * E], v1 = src[(int64_t)(ch + 1) * E];
                const T v2 = src[(int64_t)(ch + 2) * E], v3 = src[(int64_t)(ch + 3) * E];
                s = __dadd_rn(s, (double)v0);
                s = __dadd_rn(s, (double)v1);
                s = __dadd_rn(s, (double)v2);
                s = __dadd_rn(s, (double)v3);
            }
            for (; ch < c1; ++ch) s = __dadd_rn(s, (double)src[(int64_t)ch * E]);
        }
        red[w][lane] = s;
        __syncthreads();
        if (w == 0 && e < E) {
            double t = red[0][lane];
#pragma unroll
            for (int q = 1; q < W; ++q) t = __dadd_rn(t, red[q][lane]);
            const int cp = (int)(e / (cin * (d + 1)));
            const int kk = (int)(e % (cin * (d + 1)));
            const int c = tmajor ? kk % cin : kk / (d + 1), tt = tmajor ? kk / cin : kk % (d + 1);
            if (tt < d) {
                if (d_theta) d_theta[((int64_t)cp * ld + c) * d + tt] = (T)t;
            } else if (d_theta_b) {
                d_theta_b[(int64_t)cp * ld + c] = (T)t;
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------
// host-side launchers
// ------------------------------------------------------------------------------------

template <typename F>
static void set_smem(F *kernel, size_t bytes) {
    if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

static int grid_for(int64_t work_items, int per_block) {
    int64_t g = ceil_div(work_items, per_block);
    const int64_t cap = (int64_t)num_sms() * 8;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

template <typename T>
void launch_pack(int cin, int d, int cout, const T *theta, const T *theta_b, T *wt, T *wr,
                 cudaStream_t st) {
    const int64_t total = (int64_t)cout * cin * (d + 1);
    pack_weights_kernel<T><<<grid_for(total, 256), 256, 0, st>>>(cin, d, cout, theta, theta_b, wt, wr);
    count_launch();
}

template <typename T, int DP, bool REV>
int launch_wide_gmc_dp(int64_t total, int64_t n, int gc, int k, int cout, const T *rows, const T *loc,
                       const int32_t *nbr, Csr csr, const T *w, T *out, const T *feat, const T *theta,
                       const T *centre, T *dloc, cudaStream_t st);
template <typename T, int DP>
int launch_dtheta_slice_dp(int64_t total, int64_t n, int cin, int k, int cout, const T *feat, const T *loc,
                           const int32_t *nbr, const T *g, T *d_theta, T *d_theta_b, cudaStream_t st);

template <int DP, bool REV>
int launch_gemm_gmc_dp(int64_t total, int64_t n, int gc, int k, int cout, const float *rows, const float *loc,
                       const int32_t *nbr, Csr csr, const float *w, float *out, cudaStream_t st);
template <int DP>
int launch_gemm_centre_dp(int64_t total, int64_t n, int cin, int k, int cout, const float *feat, const int32_t *nbr,
                          const float *g, const float *theta, float *centre, cudaStream_t st);
template <int DP>
int launch_gemm_rev_dloc_dp(int64_t total, int64_t n, int gc, int k, int cout, const float *rows, const float *loc,
                            Csr csr, const float *w, float *out, const float *feat, const float *theta,
                            const float *centre, float *dloc, cudaStream_t st);
template <int DP>
int launch_gemm_dtheta_dp(int64_t total, int64_t n, int cin, int k, int cout, const float *feat, const float *loc,
                          const int32_t *nbr, const float *g, float *d_theta, float *d_theta_b, cudaStream_t st);

// FC_NO_WIDE=1: keep the per-warp kernels below (A/B timing of conv_wide.cu)
static bool wide_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("FC_NO_WIDE");
        v = (e && e[0] == '1') ? 0 : 1;
    }
    return v == 1;
}

template <typename T, int DP, bool REV>
static int launch_gmc_dp(int64_t total, int64_t n, int gc, int k, int cout, const T *rows,
                         const T *loc, const int32_t *nbr, Csr csr, const T *w, T *out,
                         const T *feat, const T *theta, const T *centre, T *dloc, cudaStream_t st) {
    if constexpr (sizeof(T) == 4) {  // fp32, >= 96 gathered channels: moments + cuBLAS GEMM (conv_wide.cu)
        if (dloc == nullptr && wide_enabled()) {
            const int rc = launch_gemm_gmc_dp<DP, REV>(total, n, gc, k, cout, (const float *)rows, (const float *)loc,
                                                       nbr, csr, (const float *)w, (float *)out, st);
            if (rc != FC_ERR_UNSUPPORTED) return rc;
        }
        if constexpr (REV) {
            if (dloc != nullptr && wide_enabled()) {
                const int rc = launch_gemm_rev_dloc_dp<DP>(total, n, gc, k, cout, (const float *)rows,
                                                           (const float *)loc, csr, (const float *)w, (float *)out,
                                                           (const float *)feat, (const float *)theta,
                                                           (const float *)centre, (float *)dloc, st);
                if (rc != FC_ERR_UNSUPPORTED) return rc;
            }
        }
    }
    if (wide_enabled()) {  // conv_wide.cu: same sums, same order, CTA-tiled (+ the d_loc neighbour term)
        const int rc = launch_wide_gmc_dp<T, DP, REV>(total, n, gc, k, cout, rows, loc, nbr, csr, w, out, feat, theta,
                                                      centre, dloc, st);
        if (rc != FC_ERR_UNSUPPORTED) return rc;
    }
    const int ktot = gc * (DP + 1);
    const size_t per_point = (size_t)ktot * sizeof(T);
    int ppw = 4;
    while (ppw > 1 && per_point * ppw * 8 > 96 * 1024) ppw >>= 1;
    const size_t smem = per_point * ppw * 8;
    if (smem > 200 * 1024) return set_error(FC_ERR_UNSUPPORTED, "channel count too large for the SIMT engine (%d)", gc);
    const int grid = grid_for(ceil_div(total, 8 * ppw), 1);
    prof_begin(REV ? "simt_reverse" : "simt_forward", st);
    switch (ppw) {
        case 4:
            set_smem(gmc_kernel<T, DP, REV, 4>, smem);
            gmc_kernel<T, DP, REV, 4><<<grid, 256, smem, st>>>(total, n, gc, k, cout, rows, loc, nbr, csr, w, out, feat, theta, centre, dloc);
            break;
        case 2:
            set_smem(gmc_kernel<T, DP, REV, 2>, smem);
            gmc_kernel<T, DP, REV, 2><<<grid, 256, smem, st>>>(total, n, gc, k, cout, rows, loc, nbr, csr, w, out, feat, theta, centre, dloc);
            break;
        default:
            set_smem(gmc_kernel<T, DP, REV, 1>, smem);
            gmc_kernel<T, DP, REV, 1><<<grid, 256, smem, st>>>(total, n, gc, k, cout, rows, loc, nbr, csr, w, out, feat, theta, centre, dloc);
            break;
    }
    prof_end(st);
    count_launch();
    return check_launch("gmc_kernel");
}

#define FC_DP_SWITCH(d, CALL)                                        \
    switch (d) {                                                     \
        case 1: { constexpr int DPC = 1; return CALL; }               \
        case 2: { constexpr int DPC = 2; return CALL; }               \
        case 3: { constexpr int DPC = 3; return CALL; }               \
        case 4: { constexpr int DPC = 4; return CALL; }               \
        case 5: { constexpr int DPC = 5; return CALL; }               \
        case 6: { constexpr int DPC = 6; return CALL; }               \
        case 7: { constexpr int DPC = 7; return CALL; }               \
        case 8: { constexpr int DPC = 8; return CALL; }               \
        default: return set_error(FC_ERR_UNSUPPORTED, "spatial dimension d=%d outside [1, %d]", d, kMaxDp); \
    }

template <typename T>
int launch_gmc(bool reverse, int64_t total, int64_t n, int d, int gc, int k, int cout, const T *rows,
               const T *loc, const int32_t *nbr, Csr csr, const T *w, T *out, const T *feat,
               const T *theta, const T *centre, T *dloc, cudaStream_t st) {
    if (reverse) {
        FC_DP_SWITCH(d, (launch_gmc_dp<T, DPC, true>(total, n, gc, k, cout, rows, loc, nbr, csr, w, out, feat, theta, centre, dloc, st)));
    } else {
        FC_DP_SWITCH(d, (launch_gmc_dp<T, DPC, false>(total, n, gc, k, cout, rows, loc, nbr, csr, w, out, feat, theta, centre, dloc, st)));
    }
}

template <typename T, int DP>
static int launch_dloc_centre_dp(int64_t total, int64_t n, int cin, int k, int cout, const T *feat,
                                 const int32_t *nbr, const T *g, const T *theta, T *centre,
                                 cudaStream_t st) {
    if constexpr (sizeof(T) == 4) {  // fp32: Z = G . theta as one SGEMM + a row dot (conv_wide.cu)
        const int rc = launch_gemm_centre_dp<DP>(total, n, cin, k, cout, (const float *)feat, nbr, (const float *)g,
                                                 (const float *)theta, (float *)centre, st);
        if (rc != FC_ERR_UNSUPPORTED) return rc;
    }
    const size_t smem = (size_t)8 * cout * sizeof(T);
    set_smem(dloc_centre_kernel<T, DP>, smem);
    dloc_centre_kernel<T, DP><<<grid_for(ceil_div(total, 8), 1), 256, smem, st>>>(total, n, cin, k, cout, feat, nbr, g, theta, centre);
    count_launch();
    return check_launch("dloc_centre_kernel");
}

template <typename T>
int launch_dloc_centre(int64_t total, int64_t n, int d, int cin, int k, int cout, const T *feat,
                       const int32_t *nbr, const T *g, const T *theta, T *centre, cudaStream_t st) {
    FC_DP_SWITCH(d, (launch_dloc_centre_dp<T, DPC>(total, n, cin, k, cout, feat, nbr, g, theta, centre, st)));
}

template <typename T, int DP>
static int launch_dtheta_dp(int64_t total, int64_t n, int cin, int k, int cout, const T *feat,
                            const T *loc, const int32_t *nbr, const T *g, T *d_theta,
                            T *d_theta_b, cudaStream_t st) {
    if constexpr (sizeof(T) == 4) {
        if (wide_enabled()) {
            const int rc = launch_gemm_dtheta_dp<DP>(total, n, cin, k, cout, (const float *)feat, (const float *)loc,
                                                     nbr, (const float *)g, (float *)d_theta, (float *)d_theta_b, st);
            if (rc != FC_ERR_UNSUPPORTED) return rc;
        }
    }
    if (wide_enabled()) {  // conv_wide.cu: one gather per 16-channel slice
        const int rc = launch_dtheta_slice_dp<T, DP>(total, n, cin, k, cout, feat, loc, nbr, g, d_theta, d_theta_b, st);
        if (rc != FC_ERR_UNSUPPORTED) return rc;
    }
    constexpr int RPT = 8;
    const int ktot = cin * (DP + 1);
    const int64_t E = (int64_t)cout * ktot;
    const int slices = (int)ceil_div(E, 256 * RPT);
    int tile = 32;
    while (tile > 8 && (size_t)tile * (ktot + cout) * sizeof(T) > 96 * 1024) tile >>= 1;
    const size_t smem = (size_t)tile * (ktot + cout) * sizeof(T);
    if (smem > 200 * 1024) return set_error(FC_ERR_UNSUPPORTED, "channel count too large for the SIMT d_theta engine");
    int64_t want_blocks = (int64_t)num_sms() * 4;
    int64_t chunks = ceil_div(want_blocks, slices);
    chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, ceil_div(total, tile)));
    const int64_t chunk_pts = ceil_div(ceil_div(total, chunks), tile) * tile;
    chunks = ceil_div(total, chunk_pts);
    T *partial = (T *)scratch_alloc((size_t)chunks * E * sizeof(T), st);
    if (!partial) return set_error(FC_ERR_CUDA, "scratch allocation failed");
    set_smem(dtheta_partial_kernel<T, DP, RPT>, smem);
    dtheta_partial_kernel<T, DP, RPT><<<dim3((unsigned)chunks, (unsigned)slices), 256, smem, st>>>(
        total, n, cin, k, cout, feat, loc, nbr, g, partial, chunk_pts, tile);
    count_launch();
    dtheta_reduce_kernel<T><<<(unsigned)ceil_div(E, 32), 256, 0, st>>>((int)chunks, cin, DP, cout, partial, d_theta, d_theta_b, 0, cin);
    count_launch();
    scratch_free(partial, st);
    return check_launch("dtheta kernels");
}

template <typename T>
int launch_dtheta(int64_t total, int64_t n, int d, int cin, int k, int cout, const T *feat,
                  const T *loc, const int32_t *nbr, const T *g, T *d_theta, T *d_theta_b,
                  cudaStream_t st) {
    FC_DP_SWITCH(d, (launch_dtheta_dp<T, DPC>(total, n, cin, k, cout, feat, loc, nbr, g, d_theta, d_theta_b, st)));
}

template <typename T>
int launch_dtheta_reduce(int chunks, int cin, int d, int cout, const T *partial, T *d_theta, T *d_theta_b,
                         cudaStream_t st, int tmajor, int ld) {
    // ld: row stride (channels) of d_theta / d_theta_b, 0 = dense (cin); a block of a wider theta
    const int64_t E = (int64_t)cout * cin * (d + 1);
    dtheta_reduce_kernel<T><<<(unsigned)ceil_div(E, 32), 256, 0, st>>>(chunks, cin, d, cout, partial, d_theta, d_theta_b,
                                                                        tmajor, ld > 0 ? ld : cin);
    count_launch();
    return check_launch("dtheta_reduce_kernel");
}
template int launch_dtheta_reduce<float>(int, int, int, int, const float *, float *, float *, cudaStream_t, int, int);
template int launch_dtheta_reduce<double>(int, int, int, int, const double *, double *, double *, cudaStream_t, int, int);

#define FC_INST(T)                                                                                   \
    template void launch_pack<T>(int, int, int, const T *, const T *, T *, T *, cudaStream_t);      \
    template int launch_gmc<T>(bool, int64_t, int64_t, int, int, int, int, const T *, const T *,    \
                               const int32_t *, Csr, const T *, T *, const T *, const T *,          \
                               const T *, T *, cudaStream_t);                                       \
    template int launch_dloc_centre<T>(int64_t, int64_t, int, int, int, int, const T *,             \
                                       const int32_t *, const T *, const T *, T *, cudaStream_t);  \
    template int launch_dtheta<T>(int64_t, int64_t, int, int, int, int, const T *, const T *,       \
                                  const int32_t *, const T *, T *, T *, cudaStream_t);
FC_INST(float)
FC_INST(double)

}  // namespace fc
