// conv_wide.cu -- CUDA-core engines for the channel counts the tensor-core kernels do not
// cover (the U-Net's 128 -> 128 and 256 -> 256 levels, the classifier's 64 -> 128, any d),
// in fp32 (FMA) and fp64 (the reference's operation order).
//
// wide_gmc_kernel : gather -> moments -> contraction (forward, and the reverse role that
//                   serves d_features / flex_deconv), the same sums as gmc_kernel
//                   (conv_simt.cu) in the same order, restructured as a CTA-wide tile:
//                   phase 1 gathers the moments of P points into shared memory (one warp per
//                   point, lanes over channels, slot order = _native.pyx:52-59), phase 2
//                   contracts them against the packed weights staged chunk by chunk in shared
//                   memory, lanes over points and 16 output channels per thread (the weights
//                   are warp-uniform broadcasts, the moments a conflict-free odd-stride read).
//                   Per (point, c') the sum still runs over kk = c*(d+1)+t ascending with one
//                   accumulator (_native.pyx:60-66): fp64 results equal gmc_kernel's bitwise.
// dtheta_slice_kernel : d_theta partials P[c', c, t] = sum_i g[i, c'] X_i[c, t]
//                   (_native.pyx:106-112).  A CTA owns a 16-channel slice of the moments and ALL
//                   output channels, over a contiguous point chunk: each neighbour row is
//                   gathered once per slice (64-byte segments), never once per output tile.
//                   Partials per chunk are reduced in fixed order by dtheta_reduce_kernel.
#include "fc_common.cuh"


#include <cstdlib>

namespace fc {

template <typename T>
int launch_dtheta_reduce(int chunks, int cin, int d, int cout, const T *partial, T *d_theta, T *d_theta_b,
                         cudaStream_t st, int tmajor = 0, int ld = 0);

namespace {

constexpr int kWideThreads = 256;
constexpr int kGroup = 16;       // output channels per thread in the contraction
constexpr int kChunkCh = 8;      // input channels per staged weight chunk
constexpr int kPassCp = 8 * kGroup;  // output channels per CTA pass (8 warps x 16)

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

// Stage w[(c0..c0+7) x (d+1)][pass's 128 output channels] into shared memory (zero padded):
// 16-byte cp.async when the weight rows are 16-byte aligned (no wait here), else plain copies.
template <typename T, int DP>
__device__ __forceinline__ void stage_weights(T *dst, const T *__restrict__ w, int c0, int pass, int ktot, int cout,
                                              bool async_ok) {
    constexpr int KC = kChunkCh * (DP + 1);
    if (async_ok) {
        constexpr int V = 16 / sizeof(T);
        for (int e = threadIdx.x; e < KC * kPassCp / V; e += kWideThreads) {
            const int kl = e / (kPassCp / V), cl = (e % (kPassCp / V)) * V;
            const int kk = c0 * (DP + 1) + kl;
            const int cp = pass * kPassCp + cl;
            const bool ok = kk < ktot && cp < cout;
            cp_async16(dst + kl * kPassCp + cl, ok ? (const void *)(w + (int64_t)kk * cout + cp) : (const void *)w, ok);
        }
    } else {
        for (int e = threadIdx.x; e < KC * kPassCp; e += kWideThreads) {
            const int kl = e / kPassCp, cl = e % kPassCp;
            const int kk = c0 * (DP + 1) + kl;
            const int cp = pass * kPassCp + cl;
            dst[e] = (kk < ktot && cp < cout) ? w[(int64_t)kk * cout + cp] : T(0);
        }
    }
}

// Moments of point p (one warp; lane = VEC consecutive channels, one 16-byte load per
// neighbour row when VEC > 1) stored t-major into xs[t*gc + c].  The neighbour rows of a
// batch of 8 slots are all loaded before any is accumulated (memory-level parallelism);
// per (c, t) the terms are still added in slot order with the reference's operations
// (warp_moments in conv_simt.cu, _native.pyx:52-59).
template <typename T, int VEC>
struct VecLd;
template <typename T>
struct VecLd<T, 1> {
    static __device__ __forceinline__ void ld(const T *p, T *v) { v[0] = __ldg(p); }
};
template <>
struct VecLd<float, 4> {
    static __device__ __forceinline__ void ld(const float *p, float *v) {
        const float4 x = __ldg(reinterpret_cast<const float4 *>(p));
        v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
    }
};
template <>
struct VecLd<double, 2> {
    static __device__ __forceinline__ void ld(const double *p, double *v) {
        const double2 x = __ldg(reinterpret_cast<const double2 *>(p));
        v[0] = x.x, v[1] = x.y;
    }
};

template <typename T, int DP, bool REVERSE, int VEC>
__device__ __forceinline__ void wide_moments(const T *__restrict__ rows, int gc, const T *__restrict__ loc,
                                             const int32_t *__restrict__ nbr, int k, Csr csr, int64_t p,
                                             int64_t base, T *__restrict__ xs, int lane) {
    constexpr int UB = 8;  // slots in flight
    T lp[DP];
#pragma unroll
    for (int t = 0; t < DP; ++t) lp[t] = loc[p * DP + t];
    int64_t q0 = 0, q1 = k;
    if (REVERSE) {
        q0 = csr.off[p];
        q1 = csr.off[p + 1];
    }
    for (int c0 = 0; c0 < gc; c0 += 32 * VEC) {
        const int c = c0 + lane * VEC;
        const bool ok = c < gc;  // gc % VEC == 0 when VEC > 1
        T acc[VEC][DP + 1];
#pragma unroll
        for (int e = 0; e < VEC; ++e)
#pragma unroll
            for (int t = 0; t <= DP; ++t) acc[e][t] = T(0);
        for (int64_t qb = q0; qb < q1; qb += UB) {
            int64_t jj[UB];
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const int64_t q = qb + u < q1 ? qb + u : q1 - 1;
                jj[u] = REVERSE ? (int64_t)csr.ent[q] / k : base + nbr[p * k + q];
            }
            T v[UB][VEC], o[UB][DP];
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                if (ok) {
                    VecLd<T, VEC>::ld(rows + jj[u] * gc + c, v[u]);
                } else {
#pragma unroll
                    for (int e = 0; e < VEC; ++e) v[u][e] = T(0);
                }
#pragma unroll
                for (int t = 0; t < DP; ++t)
                    o[u][t] = REVERSE ? Ar<T>::sub(loc[jj[u] * DP + t], lp[t]) : Ar<T>::sub(lp[t], loc[jj[u] * DP + t]);
            }
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                if (qb + u < q1) {
#pragma unroll
                    for (int e = 0; e < VEC; ++e) {
#pragma unroll
                        for (int t = 0; t < DP; ++t) acc[e][t] = Ar<T>::madd(acc[e][t], v[u][e], o[u][t]);
                        acc[e][DP] = Ar<T>::add(acc[e][DP], v[u][e]);
                    }
                }
            }
        }
        if (ok) {
#pragma unroll
            for (int t = 0; t <= DP; ++t)
#pragma unroll
                for (int e = 0; e < VEC; ++e) xs[t * gc + c + e] = acc[e][t];
        }
    }
}

// out[p, cp] = sum_{c, t} w[(c*(DP+1)+t)*cout + cp] * M_p[c, t]   (w = forward or adjoint packing)
// Neighbour role of the location gradient (REVERSE only; dloc == nullptr: skipped):
//   dloc[j, t] = centre[j, t] - sum_c f[j, c] sum_c' theta[c', c, t] Y_j[DP, c']
// (the -dt terms of _native.pyx:121-127 regrouped per j; Y_j[DP, :] = the bias moment row,
// already in shared memory).  w3 = theta repacked as [DP][gc][cout].
template <typename T>
struct WideDloc {
    const T *w3;
    const T *feat;    // [total, cout]
    const T *centre;  // [total, DP]
    T *dloc;          // [total, DP] or null
};

template <typename T, int DP, bool REVERSE, int PPL, int VEC>
__global__ void __launch_bounds__(kWideThreads)
    wide_gmc_kernel(int64_t total, int64_t n, int gc, int k, int cout, const T *__restrict__ rows,
                    const T *__restrict__ loc, const int32_t *__restrict__ nbr, Csr csr, const T *__restrict__ w,
                    T *__restrict__ out, WideDloc<T> dl) {
    constexpr int P = 32 * PPL;
    constexpr int KC = kChunkCh * (DP + 1);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int ktot = gc * (DP + 1);
    const int S = ktot | 1;  // odd row stride: lanes (= points) hit distinct banks
    T *xs = reinterpret_cast<T *>(smem_raw);
    constexpr int V16 = 16 / sizeof(T);
    T *wc = xs + (P * S + V16 - 1) / V16 * V16;  // 16-byte aligned; stays a shared-space pointer (LDS)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int passes = (cout + kPassCp - 1) / kPassCp;
    const bool async_ok = (cout * sizeof(T)) % 16 == 0 && (reinterpret_cast<uintptr_t>(w) % 16) == 0;
    const int64_t tiles = ceil_div(total, P);
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int64_t p0 = tile * P;
        for (int q = warp; q < P; q += kWideThreads / 32) {
            const int64_t p = p0 + q;
            if (p < total) wide_moments<T, DP, REVERSE, VEC>(rows, gc, loc, nbr, k, csr, p, (p / n) * n, xs + q * S, lane);
        }
        __syncthreads();
        for (int pass = 0; pass < passes; ++pass) {
            const int cpw = pass * kPassCp + warp * kGroup;  // this warp's first output channel
            T acc[PPL][kGroup];
#pragma unroll
            for (int a = 0; a < PPL; ++a)
#pragma unroll
                for (int j = 0; j < kGroup; ++j) acc[a][j] = T(0);
            // weight chunks double-buffered: chunk ci+1 streams in (cp.async) while ci is used
            const int nchunks = (gc + kChunkCh - 1) / kChunkCh;
            stage_weights<T, DP>(wc, w, 0, pass, ktot, cout, async_ok);
            cp_async_commit();
            for (int ci = 0; ci < nchunks; ++ci) {
                const int c0 = ci * kChunkCh;
                if (ci + 1 < nchunks)
                    stage_weights<T, DP>(wc + ((ci + 1) & 1) * KC * kPassCp, w, c0 + kChunkCh, pass, ktot, cout, async_ok);
                cp_async_commit();
                cp_async_wait1();
                __syncthreads();
                const T *wcur = wc + (ci & 1) * KC * kPassCp;
                const int nch = min(kChunkCh, gc - c0);
                for (int cl = 0; cl < nch; ++cl) {
#pragma unroll
                    for (int t = 0; t <= DP; ++t) {
                        const T *wrow = wcur + (cl * (DP + 1) + t) * kPassCp + warp * kGroup;
                        T wv[kGroup];  // warp-uniform broadcast, 16-byte loads
#pragma unroll
                        for (int j = 0; j < kGroup; j += 16 / (int)sizeof(T)) {
                            if constexpr (sizeof(T) == 4) {
                                const float4 x = *reinterpret_cast<const float4 *>(wrow + j);
                                wv[j] = x.x, wv[j + 1] = x.y, wv[j + 2] = x.z, wv[j + 3] = x.w;
                            } else {
                                const double2 x = *reinterpret_cast<const double2 *>(wrow + j);
                                wv[j] = x.x, wv[j + 1] = x.y;
                            }
                        }
#pragma unroll
                        for (int a = 0; a < PPL; ++a) {
                            const T xv = xs[(lane + 32 * a) * S + t * gc + c0 + cl];
#pragma unroll
                            for (int j = 0; j < kGroup; ++j) acc[a][j] = Ar<T>::madd(acc[a][j], wv[j], xv);
                        }
                    }
                }
                __syncthreads();
            }
#pragma unroll
            for (int a = 0; a < PPL; ++a) {
                const int64_t p = p0 + lane + 32 * a;
                if (p < total && cpw < cout) {
                    T *o = out + p * cout + cpw;
                    if (cpw + kGroup <= cout && ((cout * sizeof(T)) % 16) == 0) {
#pragma unroll
                        for (int j = 0; j < kGroup; j += 16 / (int)sizeof(T)) {
                            if (sizeof(T) == 4)
                                *reinterpret_cast<float4 *>(o + j) =
                                    make_float4((float)acc[a][j], (float)acc[a][j + 1], (float)acc[a][j + 2],
                                                (float)acc[a][j + 3]);
                            else
                                *reinterpret_cast<double2 *>(o + j) = make_double2((double)acc[a][j], (double)acc[a][j + 1]);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < kGroup; ++j)
                            if (cpw + j < cout) o[j] = acc[a][j];
                    }
                }
            }
        }
        if (REVERSE && dl.dloc != nullptr) {
            // U_t[p, c] = sum_c' Yb_p[c'] theta[c', c, t] with the same chunked, double-buffered
            // weight staging as above (weights = theta_t, [gc][cout]); then each thread dots its
            // 16 channels with f[p, :] and the 8 warps' partials are added in warp order.
            T *red = wc + 2 * KC * kPassCp;  // [8 warps][DP][P]
            const bool async3 = (cout * sizeof(T)) % 16 == 0 && (reinterpret_cast<uintptr_t>(dl.w3) % 16) == 0;
            T part[PPL][DP > 0 ? DP : 1];
#pragma unroll
            for (int a = 0; a < PPL; ++a)
#pragma unroll
                for (int t = 0; t < DP; ++t) part[a][t] = T(0);
            for (int pass = 0; pass < passes; ++pass) {
                const int cpw = pass * kPassCp + warp * kGroup;
#pragma unroll 1
                for (int t = 0; t < DP; ++t) {
                    const T *wt = dl.w3 + (int64_t)t * gc * cout;
                    T acc[PPL][kGroup];
#pragma unroll
                    for (int a = 0; a < PPL; ++a)
#pragma unroll
                        for (int j = 0; j < kGroup; ++j) acc[a][j] = T(0);
                    const int nchunks = (gc + kChunkCh - 1) / kChunkCh;
                    stage_weights<T, 0>(wc, wt, 0, pass, gc, cout, async3);
                    cp_async_commit();
                    for (int ci = 0; ci < nchunks; ++ci) {
                        const int c0 = ci * kChunkCh;
                        if (ci + 1 < nchunks)
                            stage_weights<T, 0>(wc + ((ci + 1) & 1) * KC * kPassCp, wt, c0 + kChunkCh, pass, gc, cout,
                                                async3);
                        cp_async_commit();
                        cp_async_wait1();
                        __syncthreads();
                        const T *wcur = wc + (ci & 1) * KC * kPassCp;
                        const int nch = min(kChunkCh, gc - c0);
                        for (int cl = 0; cl < nch; ++cl) {
                            const T *wrow = wcur + cl * kPassCp + warp * kGroup;
                            T wv[kGroup];
#pragma unroll
                            for (int j = 0; j < kGroup; ++j) wv[j] = wrow[j];
#pragma unroll
                            for (int a = 0; a < PPL; ++a) {
                                const T yb = xs[(lane + 32 * a) * S + DP * gc + c0 + cl];
#pragma unroll
                                for (int j = 0; j < kGroup; ++j) acc[a][j] = Ar<T>::madd(acc[a][j], wv[j], yb);
                            }
                        }
                        __syncthreads();
                    }
#pragma unroll
                    for (int a = 0; a < PPL; ++a) {
                        const int64_t p = p0 + lane + 32 * a;
                        if (p < total && cpw < cout) {
                            const T *fr = dl.feat + p * cout + cpw;
#pragma unroll
                            for (int j = 0; j < kGroup; ++j)
                                if (cpw + j < cout) part[a][t] = Ar<T>::madd(part[a][t], __ldg(fr + j), acc[a][j]);
                        }
                    }
                }
            }
#pragma unroll
            for (int a = 0; a < PPL; ++a)
#pragma unroll
                for (int t = 0; t < DP; ++t) red[(warp * DP + t) * P + lane + 32 * a] = part[a][t];
            __syncthreads();
            for (int e = threadIdx.x; e < P * DP; e += kWideThreads) {
                const int pl = e / DP, t = e - (e / DP) * DP;
                const int64_t p = p0 + pl;
                if (p < total) {
                    T sum = T(0);
                    for (int w8 = 0; w8 < kWideThreads / 32; ++w8) sum = Ar<T>::add(sum, red[(w8 * DP + t) * P + pl]);
                    dl.dloc[p * DP + t] = Ar<T>::sub(dl.centre[p * DP + t], sum);
                }
            }
        }
        __syncthreads();  // xs is rewritten by the next tile's gathers
    }
}

template <typename T>
__global__ void pack_theta_t_kernel(int gc, int cout, int d, const T *__restrict__ theta, T *__restrict__ w3) {
    const int64_t total = (int64_t)gc * cout * d;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(e % d);
        const int64_t r = e / d;  // = cp * cout + c
        w3[(int64_t)t * gc * cout + r] = theta[e];
    }
}

// d_theta partials of one (16-channel slice, point chunk):
//   partial[chunk][cp * ktot + c*(DP+1) + t] = sum_{i in chunk, ascending} g[i, cp] * X_i[c, t]
template <typename T, int DP, int NI>
__global__ void __launch_bounds__(256)
    dtheta_slice_kernel(int64_t total, int64_t n, int cin, int k, int cout, const T *__restrict__ feat,
                        const T *__restrict__ loc, const int32_t *__restrict__ nbr, const T *__restrict__ g,
                        T *__restrict__ partial, int64_t chunk_pts) {
    constexpr int PT = 16;  // points per step
    constexpr int GW = 16 * NI;
    __shared__ __align__(16) T gs[PT][GW];
    __shared__ __align__(16) T xl[PT][16 * (DP + 1)];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int c0 = blockIdx.x * 16;
    const int ktot = cin * (DP + 1);
    const int64_t p_begin = (int64_t)blockIdx.y * chunk_pts;
    const int64_t p_end = min(total, p_begin + chunk_pts);
    const int ty = tid >> 4, tx = tid & 15;
    T acc[NI][DP + 1];
#pragma unroll
    for (int i = 0; i < NI; ++i)
#pragma unroll
        for (int t = 0; t <= DP; ++t) acc[i][t] = T(0);
    for (int64_t t0 = p_begin; t0 < p_end; t0 += PT) {
        for (int e = tid; e < PT * GW; e += 256) {
            const int pl = e / GW, cp = e % GW;
            const int64_t p = t0 + pl;
            gs[pl][cp] = (p < p_end && cp < cout) ? g[p * cout + cp] : T(0);
        }
        {  // moment slice: half-warp per point, lane = channel
            const int pl = warp * 2 + (lane >> 4), cl = lane & 15, c = c0 + cl;
            const int64_t p = t0 + pl;
            T a[DP + 1];
#pragma unroll
            for (int t = 0; t <= DP; ++t) a[t] = T(0);
            if (p < p_end) {
                const int64_t base = (p / n) * n;
                T lp[DP];
#pragma unroll
                for (int t = 0; t < DP; ++t) lp[t] = loc[p * DP + t];
                for (int s0 = 0; s0 < k; s0 += 8) {  // 8 slots in flight, accumulated in slot order
                    int64_t jj[8];
                    T v[8], o[8][DP];
#pragma unroll
                    for (int u = 0; u < 8; ++u) jj[u] = base + nbr[p * k + min(s0 + u, k - 1)];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        v[u] = c < cin ? __ldg(feat + jj[u] * cin + c) : T(0);
#pragma unroll
                        for (int t = 0; t < DP; ++t) o[u][t] = Ar<T>::sub(lp[t], loc[jj[u] * DP + t]);
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        if (s0 + u < k) {
#pragma unroll
                            for (int t = 0; t < DP; ++t) a[t] = Ar<T>::madd(a[t], v[u], o[u][t]);
                            a[DP] = Ar<T>::add(a[DP], v[u]);
                        }
                    }
                }
            }
#pragma unroll
            for (int t = 0; t <= DP; ++t) xl[pl][cl * (DP + 1) + t] = a[t];
        }
        __syncthreads();
        const int np = (int)min((int64_t)PT, p_end - t0);
        for (int pl = 0; pl < np; ++pl) {
            T xv[DP + 1];
            if constexpr (sizeof(T) == 4 && DP == 3) {
                const float4 x = *reinterpret_cast<const float4 *>(&xl[pl][tx * 4]);
                xv[0] = x.x, xv[1] = x.y, xv[2] = x.z, xv[3] = x.w;
            } else {
#pragma unroll
                for (int t = 0; t <= DP; ++t) xv[t] = xl[pl][tx * (DP + 1) + t];
            }
            T gv[NI];  // this thread's NI consecutive output channels, 16-byte loads
            if constexpr (sizeof(T) == 4 && NI % 4 == 0) {
#pragma unroll
                for (int i = 0; i < NI; i += 4) {
                    const float4 x = *reinterpret_cast<const float4 *>(&gs[pl][ty * NI + i]);
                    gv[i] = x.x, gv[i + 1] = x.y, gv[i + 2] = x.z, gv[i + 3] = x.w;
                }
            } else {
#pragma unroll
                for (int i = 0; i < NI; ++i) gv[i] = gs[pl][ty * NI + i];
            }
#pragma unroll
            for (int i = 0; i < NI; ++i) {
#pragma unroll
                for (int t = 0; t <= DP; ++t) acc[i][t] = Ar<T>::madd(acc[i][t], gv[i], xv[t]);
            }
        }
        __syncthreads();
    }
    const int c = c0 + tx;
    if (c < cin) {
        T *dst = partial + (int64_t)blockIdx.y * cout * ktot;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
            const int cp = ty * NI + i;
            if (cp < cout) {
#pragma unroll
                for (int t = 0; t <= DP; ++t) dst[(int64_t)cp * ktot + c * (DP + 1) + t] = acc[i][t];
            }
        }
    }
}

template <typename F>
void set_smem_attr(F *kernel, size_t bytes) {
    if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <typename T, int DP>
size_t wide_smem(int gc, int ppl) {
    const size_t ktot = (size_t)gc * (DP + 1);
    const size_t xs = (size_t)32 * ppl * (ktot | 1);
    return (xs * sizeof(T) + 16) + (size_t)2 * kChunkCh * (DP + 1) * kPassCp * sizeof(T) +
           (size_t)(kWideThreads / 32) * DP * 32 * ppl * sizeof(T);  // + the d_loc reduction buffer
}

}  // namespace

// Wide gather-moment-contract: returns FC_ERR_UNSUPPORTED (without launching) when the
// moment tile does not fit in shared memory; the caller then uses gmc_kernel.
template <typename T, int DP, bool REV>
int launch_wide_gmc_dp(int64_t total, int64_t n, int gc, int k, int cout, const T *rows, const T *loc,
                       const int32_t *nbr, Csr csr, const T *w, T *out, const T *feat, const T *theta,
                       const T *centre, T *dloc, cudaStream_t st) {
    constexpr size_t kMax = 200 * 1024, kTwoPerSm = 110 * 1024;
    // two points per lane for fp32 (32 FMAs per 6 shared loads) where two CTAs still fit per
    // SM (one CTA's gathers overlap the other's contraction); fp64 keeps one (register budget)
    int ppl = 1;
    if (sizeof(T) == 4 && wide_smem<T, DP>(gc, 2) <= kTwoPerSm) ppl = 2;
    else if (wide_smem<T, DP>(gc, 1) > kTwoPerSm && sizeof(T) == 4 && wide_smem<T, DP>(gc, 2) <= kMax) ppl = 2;
    const size_t smem = wide_smem<T, DP>(gc, ppl);
    if (smem > kMax) return FC_ERR_UNSUPPORTED;
    const int per_sm = smem <= kTwoPerSm ? 2 : 1;
    const int64_t tiles = ceil_div(total, 32 * ppl);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)num_sms() * per_sm));
    constexpr int V = 16 / sizeof(T);
    const bool vec = gc % V == 0 && (reinterpret_cast<uintptr_t>(rows) % 16) == 0;
    WideDloc<T> dl{nullptr, feat, centre, dloc};
    T *w3 = nullptr;
    if (REV && dloc) {
        w3 = (T *)scratch_alloc(sizeof(T) * (size_t)gc * cout * DP, st);
        if (!w3) return set_error(FC_ERR_CUDA, "scratch allocation failed");
        const int64_t e = (int64_t)gc * cout * DP;
        pack_theta_t_kernel<T><<<(unsigned)std::min<int64_t>(ceil_div(e, 256), 4096), 256, 0, st>>>(gc, cout, DP, theta, w3);
        count_launch();
        dl.w3 = w3;
    }
    prof_begin(REV ? (dloc ? "simt_reverse_dloc" : "simt_reverse") : "simt_forward", st);
#define FC_WIDE_LAUNCH(PPLV, VECV)                                                                              \
    do {                                                                                                        \
        set_smem_attr(wide_gmc_kernel<T, DP, REV, PPLV, VECV>, smem);                                           \
        wide_gmc_kernel<T, DP, REV, PPLV, VECV><<<grid, kWideThreads, smem, st>>>(total, n, gc, k, cout, rows, loc, \
                                                                                 nbr, csr, w, out, dl);          \
    } while (0)
    if (sizeof(T) == 4 && ppl == 2) {
        if (vec) FC_WIDE_LAUNCH(2, V); else FC_WIDE_LAUNCH(2, 1);
    } else {
        if (vec) FC_WIDE_LAUNCH(1, V); else FC_WIDE_LAUNCH(1, 1);
    }
#undef FC_WIDE_LAUNCH
    prof_end(st);
    count_launch();
    scratch_free(w3, st);
    return check_launch("wide_gmc_kernel");
}

template <typename T, int DP, int NI>
static int launch_slice(int64_t total, int64_t n, int cin, int k, int cout, const T *feat, const T *loc,
                        const int32_t *nbr, const T *g, T *d_theta, T *d_theta_b, cudaStream_t st) {
    const int slices = (int)ceil_div(cin, 16);
    const int64_t E = (int64_t)cout * cin * (DP + 1);
    int64_t chunks = std::max<int64_t>(1, ceil_div((int64_t)num_sms() * 3, slices));
    chunks = std::min<int64_t>(chunks, ceil_div(total, 16));
    const int64_t chunk_pts = ceil_div(ceil_div(total, chunks), 16) * 16;
    chunks = ceil_div(total, chunk_pts);
    T *partial = (T *)scratch_alloc((size_t)chunks * E * sizeof(T), st);
    if (!partial) return set_error(FC_ERR_CUDA, "scratch allocation failed");
    prof_begin("simt_dtheta", st);
    dtheta_slice_kernel<T, DP, NI><<<dim3((unsigned)slices, (unsigned)chunks), 256, 0, st>>>(
        total, n, cin, k, cout, feat, loc, nbr, g, partial, chunk_pts);
    count_launch();
    int rc = launch_dtheta_reduce<T>((int)chunks, cin, DP, cout, partial, d_theta, d_theta_b, st);
    prof_end(st);
    scratch_free(partial, st);
    if (rc) return rc;
    return check_launch("dtheta_slice_kernel");
}

// d_theta through the slice kernel (cout <= 256); FC_ERR_UNSUPPORTED -> caller falls back.
template <typename T, int DP>
int launch_dtheta_slice_dp(int64_t total, int64_t n, int cin, int k, int cout, const T *feat, const T *loc,
                           const int32_t *nbr, const T *g, T *d_theta, T *d_theta_b, cudaStream_t st) {
    if (cout <= 32) return launch_slice<T, DP, 2>(total, n, cin, k, cout, feat, loc, nbr, g, d_theta, d_theta_b, st);
    if (cout <= 64) return launch_slice<T, DP, 4>(total, n, cin, k, cout, feat, loc, nbr, g, d_theta, d_theta_b, st);
    if (cout <= 128) return launch_slice<T, DP, 8>(total, n, cin, k, cout, feat, loc, nbr, g, d_theta, d_theta_b, st);
    if constexpr (DP <= 3) {
        if (cout <= 256)
            return launch_slice<T, DP, 16>(total, n, cin, k, cout, feat, loc, nbr, g, d_theta, d_theta_b, st);
    }
    return FC_ERR_UNSUPPORTED;
}

// ---------------------------------------------------------------------------------------
// fp32 wide channel counts as moments + library GEMM.  The contraction of the gathered
// moments with the packed weights (and d_theta = G^T X) is a plain dense GEMM once the moment
// rows X [points, ktot] are materialised; it goes to cuBLAS (FP32, no TF32: default math
// mode), which runs it at several times the CTA-tiled FFMA rate.  The gather stays here.
namespace {

// X[p, c*(DP+1) + t] for points [p0, p0 + m): one warp per point, lanes over 4 channels
// (H = 2: two 4-channel groups 128 channels apart, so a 256-channel row is one pass with the
// neighbour indices and offsets loaded once), 8 (H = 2: 4) neighbour rows in flight, slot
// order per (c, t) (_native.pyx:52-59).
template <int DP, bool REVERSE, bool TMAJOR = false, int H = 1>
__global__ void __launch_bounds__(256)
    moments_rows_kernel(int64_t p0, int64_t m, int64_t n, int gc, int k, const float *__restrict__ rows,
                        const float *__restrict__ loc, const int32_t *__restrict__ nbr, Csr csr,
                        float *__restrict__ X) {
    constexpr int SB = H == 1 ? 8 : 4;  // slots per batch
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int ktot = gc * (DP + 1);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < m; r += nw) {
        const int64_t p = p0 + r;
        const int64_t base = (p / n) * n;
        float lp[DP];
#pragma unroll
        for (int t = 0; t < DP; ++t) lp[t] = loc[p * DP + t];
        int64_t q0 = 0, q1 = k;
        if (REVERSE) {
            q0 = csr.off[p];
            q1 = csr.off[p + 1];
        }
        float *xr = X + r * ktot;
        for (int c0 = 0; c0 < gc; c0 += 128 * H) {
            int cg[H];
            bool ok[H];
#pragma unroll
            for (int h = 0; h < H; ++h) {
                cg[h] = c0 + h * 128 + lane * 4;
                ok[h] = cg[h] < gc;
            }
            float acc[H][4][DP + 1];
#pragma unroll
            for (int h = 0; h < H; ++h)
#pragma unroll
                for (int e = 0; e < 4; ++e)
#pragma unroll
                    for (int t = 0; t <= DP; ++t) acc[h][e][t] = 0.f;
            for (int64_t qb = q0; qb < q1; qb += SB) {
                int64_t jj[SB];
#pragma unroll
                for (int u = 0; u < SB; ++u) {
                    const int64_t q = qb + u < q1 ? qb + u : q1 - 1;
                    jj[u] = REVERSE ? (int64_t)csr.ent[q] / k : base + nbr[p * k + q];
                }
                float4 v[SB][H];
                float o[SB][DP];
#pragma unroll
                for (int u = 0; u < SB; ++u) {
#pragma unroll
                    for (int h = 0; h < H; ++h)
                        v[u][h] = ok[h] ? __ldg(reinterpret_cast<const float4 *>(rows + jj[u] * gc + cg[h]))
                                        : make_float4(0, 0, 0, 0);
#pragma unroll
                    for (int t = 0; t < DP; ++t)
                        o[u][t] = REVERSE ? loc[jj[u] * DP + t] - lp[t] : lp[t] - loc[jj[u] * DP + t];
                }
#pragma unroll
                for (int u = 0; u < SB; ++u) {
                    if (qb + u < q1) {
#pragma unroll
                        for (int h = 0; h < H; ++h) {
                            const float ve[4] = {v[u][h].x, v[u][h].y, v[u][h].z, v[u][h].w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
#pragma unroll
                                for (int t = 0; t < DP; ++t) acc[h][e][t] = fmaf(ve[e], o[u][t], acc[h][e][t]);
                                acc[h][e][DP] += ve[e];
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int h = 0; h < H; ++h) {
                if (!ok[h]) continue;
                const int c = cg[h];
                if constexpr (TMAJOR) {  // X[p, t*gc + c]: one float4 per t
#pragma unroll
                    for (int t = 0; t <= DP; ++t)
                        *reinterpret_cast<float4 *>(xr + t * gc + c) =
                            make_float4(acc[h][0][t], acc[h][1][t], acc[h][2][t], acc[h][3][t]);
                } else {  // X[p, c*(DP+1) + t]: 4 channels x (DP+1) consecutive floats
#pragma unroll
                    for (int e = 0; e < 4; ++e)
#pragma unroll
                        for (int t = 0; t <= DP; ++t) xr[(c + e) * (DP + 1) + t] = acc[h][e][t];
                }
            }
        }
    }
}

// out [m, ncols] (row stride ldo) = A [m, k] (row stride lda) . B [k, ncols] (row-major, row
// stride ldb) on the hand-written tcgen05 GEMM (gemm_tc.cu: tf32 hi/lo split operands, fp32
// accumulation with K-block partials summed in registers); img: a packed image of B from
// pack_b_rm (reused across point chunks).
int pack_b_rm(const float *B, int64_t ldb, int k, int ncols, Scratch &img, cudaStream_t st) {
    img.alloc((size_t)fc_gemm_image_bytes(ncols, (int)ceil_div(k, 32)), st);
    if (!img.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed (GEMM image)");
    const int src = 0;
    return fc_gemm_pack_b(1, ncols, 1, &src, &k, B, ldb, img.as<uint8_t>(), st);
}
int tc_gemm(const float *A, int64_t lda, int k, int64_t m, const Scratch &img, int ncols, float *out, int64_t ldo,
            cudaStream_t st) {
    const float *a = A;
    float *o = out;
    int64_t la = lda, lo = ldo;
    int kk = k, c0 = 0, c1 = ncols;
    return fc_gemm_rows(m, 1, &a, &la, &kk, nullptr, 0, img.as<uint8_t>(), ncols, nullptr, 1, &o, &lo, &c0, &c1,
                        nullptr, 0, st);
}
__global__ void add_into_kernel(int64_t count, const float *__restrict__ src, float *__restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] += src[i];
}

bool gemm_route_enabled(int gc) {
    static int v = -1, gmin = 32;
    if (v < 0) {
        const char *e = getenv("FC_NO_GEMM");
        v = (e && e[0] == '1') ? 0 : 1;
        const char *m = getenv("FC_GEMM_MIN");  // smallest gathered channel count on the GEMM route
        if (m && atoi(m) > 0) gmin = atoi(m);
    }
    return v == 1 && gc >= gmin && gc % 4 == 0;
}

int64_t gemm_chunk(int64_t total, int ktot) {
    const int64_t cap = std::max<int64_t>(1024, ((int64_t)256 << 20) / ((int64_t)ktot * 4));
    return std::min<int64_t>(total, cap);
}

}  // namespace

// out [total, cout] = X [total, ktot] . w [ktot, cout]   (w: forward or adjoint packing)
template <int DP, bool REV>
int launch_gemm_gmc_dp(int64_t total, int64_t n, int gc, int k, int cout, const float *rows, const float *loc,
                       const int32_t *nbr, Csr csr, const float *w, float *out, cudaStream_t st) {
    if (!gemm_route_enabled(gc) || (reinterpret_cast<uintptr_t>(rows) % 16) != 0) return FC_ERR_UNSUPPORTED;
    const int ktot = gc * (DP + 1);
    const int64_t chunk = gemm_chunk(total, ktot);
    Scratch Xb(sizeof(float) * chunk * ktot, st), img;
    if (!Xb.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed");
    float *X = Xb.as<float>();
    if (int rc = pack_b_rm(w, cout, ktot, cout, img, st)) return rc;
    int rc = FC_OK;
    for (int64_t p0 = 0; p0 < total && rc == FC_OK; p0 += chunk) {
        const int64_t m = std::min(chunk, total - p0);
        const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(m, 8), (int64_t)num_sms() * 8);
        if (gc % 256 == 0) moments_rows_kernel<DP, REV, false, 2><<<grid, 256, 0, st>>>(p0, m, n, gc, k, rows, loc, nbr, csr, X);
        else moments_rows_kernel<DP, REV><<<grid, 256, 0, st>>>(p0, m, n, gc, k, rows, loc, nbr, csr, X);
        count_launch();
        rc = tc_gemm(X, ktot, ktot, m, img, cout, out + p0 * cout, cout, st);
    }
    if (rc) return rc;
    return check_launch("moments + GEMM");
}

// d_theta via P [cout, ktot] = sum over point chunks (fixed order) of G^T X, then the fp64
// fixed-order reduce kernel converts P into d_theta / d_theta_b.
template <int DP>
int launch_gemm_dtheta_dp(int64_t total, int64_t n, int cin, int k, int cout, const float *feat, const float *loc,
                          const int32_t *nbr, const float *g, float *d_theta, float *d_theta_b, cudaStream_t st) {
    if (!gemm_route_enabled(cin) || (reinterpret_cast<uintptr_t>(feat) % 16) != 0) return FC_ERR_UNSUPPORTED;
    const int ktot = cin * (DP + 1);
    const int64_t chunk = gemm_chunk(total, ktot);
    const bool chunked = chunk < total;
    Scratch Xb(sizeof(float) * chunk * ktot, st), Pb(sizeof(float) * (size_t)cout * ktot * (chunked ? 2 : 1), st);
    if (!Xb.ok() || !Pb.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed");
    float *X = Xb.as<float>(), *P = Pb.as<float>(), *Pc = chunked ? P + (size_t)cout * ktot : P;
    int rc = FC_OK;
    for (int64_t p0 = 0; p0 < total && rc == FC_OK; p0 += chunk) {
        const int64_t m = std::min(chunk, total - p0);
        const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(m, 8), (int64_t)num_sms() * 8);
        if (cin % 256 == 0)
            moments_rows_kernel<DP, false, false, 2><<<grid, 256, 0, st>>>(p0, m, n, cin, k, feat, loc, nbr, Csr{nullptr, nullptr}, X);
        else moments_rows_kernel<DP, false><<<grid, 256, 0, st>>>(p0, m, n, cin, k, feat, loc, nbr, Csr{nullptr, nullptr}, X);
        count_launch();
        // P [cout, ktot] = G^T X (fc_gemm_wgrad: fixed-order partial sums); chunks added in order
        const float *xo = X;
        int64_t lx = ktot;
        int kx = ktot;
        rc = fc_gemm_wgrad(m, g + p0 * cout, cout, nullptr, 0, cout, 1, &xo, &lx, &kx, p0 == 0 ? P : Pc, nullptr, st);
        if (rc == FC_OK && p0 > 0) {
            add_into_kernel<<<(unsigned)std::min<int64_t>(ceil_div((int64_t)cout * ktot, 256), 1024), 256, 0, st>>>(
                (int64_t)cout * ktot, Pc, P);
            count_launch();
        }
    }
    if (rc == FC_OK) rc = launch_dtheta_reduce<float>(1, cin, DP, cout, P, d_theta, d_theta_b, st);
    if (rc) return rc;
    return check_launch("moments + GEMM (d_theta)");
}

namespace {

// w_t[(t*gc + c)*cout + o] = w[(c*(DP+1) + t)*cout + o]   (c-major -> t-major packing)
__global__ void repack_tmajor_kernel(int gc, int dp1, int cout, const float *__restrict__ w, float *__restrict__ wt) {
    const int64_t total = (int64_t)gc * dp1 * cout;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int o = (int)(e % cout);
        const int64_t r = e / cout;  // = c*dp1 + t
        const int t = (int)(r % dp1), c = (int)(r / dp1);
        wt[((int64_t)t * gc + c) * cout + o] = w[e];
    }
}

// theta [gc][cout][d] -> tcat [gc][d*cout]: tcat[c'][t*cout + c] = theta[c', c, t]
__global__ void pack_theta_cat_kernel(int gc, int cout, int d, const float *__restrict__ theta,
                                      float *__restrict__ tcat) {
    const int64_t total = (int64_t)gc * cout * d;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(e % d);
        const int64_t r = e / d;  // = c' * cout + c
        const int c = (int)(r % cout), cp = (int)(r / cout);
        tcat[(int64_t)cp * d * cout + (int64_t)t * cout + c] = theta[e];
    }
}

// dloc[p, t] = centre[p, t] - sum_c f[p, c] U[p, t*cout + c]   (warp per point)
template <int DP>
__global__ void __launch_bounds__(256)
    dloc_nbr_kernel(int64_t p0, int64_t m, int cout, const float *__restrict__ feat, const float *__restrict__ U,
                    const float *__restrict__ centre, float *__restrict__ dloc) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < m; r += nw) {
        const int64_t p = p0 + r;
        float part[DP];
#pragma unroll
        for (int t = 0; t < DP; ++t) part[t] = 0.f;
        for (int c = lane; c < cout; c += 32) {
            const float f = feat[p * cout + c];
#pragma unroll
            for (int t = 0; t < DP; ++t) part[t] = fmaf(f, U[r * DP * cout + t * cout + c], part[t]);
        }
#pragma unroll
        for (int t = 0; t < DP; ++t) {
            float v = part[t];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) dloc[p * DP + t] = centre[p * DP + t] - v;
        }
    }
}

}  // namespace

// Reverse role with the location gradient: d_f = Y . W (t-major), U = Yb . [theta_0 .. theta_{d-1}]
// (one GEMM, N = d*cout), then the neighbour-role term dotted with f (dloc_nbr_kernel).
template <int DP>
int launch_gemm_rev_dloc_dp(int64_t total, int64_t n, int gc, int k, int cout, const float *rows, const float *loc,
                            Csr csr, const float *w, float *out, const float *feat, const float *theta,
                            const float *centre, float *dloc, cudaStream_t st) {
    if (!gemm_route_enabled(gc) || (reinterpret_cast<uintptr_t>(rows) % 16) != 0) return FC_ERR_UNSUPPORTED;
    const int ktot = gc * (DP + 1);
    const int64_t chunk = gemm_chunk(total, ktot + DP * cout);
    Scratch Xb(sizeof(float) * chunk * ktot, st), Ub(sizeof(float) * chunk * DP * cout, st);
    Scratch wtb(sizeof(float) * (size_t)ktot * cout, st), tcb(sizeof(float) * (size_t)gc * DP * cout, st);
    Scratch img_w, img_t;
    if (!Xb.ok() || !Ub.ok() || !wtb.ok() || !tcb.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed");
    float *X = Xb.as<float>(), *U = Ub.as<float>(), *wt = wtb.as<float>(), *tcat = tcb.as<float>();
    const unsigned pg = (unsigned)std::min<int64_t>(ceil_div((int64_t)ktot * cout, 256), 4096);
    repack_tmajor_kernel<<<pg, 256, 0, st>>>(gc, DP + 1, cout, w, wt);
    pack_theta_cat_kernel<<<pg, 256, 0, st>>>(gc, cout, DP, theta, tcat);
    count_launch();
    count_launch();
    if (int rc = pack_b_rm(wt, cout, ktot, cout, img_w, st)) return rc;
    if (int rc = pack_b_rm(tcat, DP * cout, gc, DP * cout, img_t, st)) return rc;
    int rc = FC_OK;
    for (int64_t p0 = 0; p0 < total && rc == FC_OK; p0 += chunk) {
        const int64_t m = std::min(chunk, total - p0);
        const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(m, 8), (int64_t)num_sms() * 8);
        if (gc % 256 == 0) moments_rows_kernel<DP, true, true, 2><<<grid, 256, 0, st>>>(p0, m, n, gc, k, rows, loc, nullptr, csr, X);
        else moments_rows_kernel<DP, true, true><<<grid, 256, 0, st>>>(p0, m, n, gc, k, rows, loc, nullptr, csr, X);
        count_launch();
        rc = tc_gemm(X, ktot, ktot, m, img_w, cout, out + p0 * cout, cout, st);
        // U = Yb . [theta_0 .. theta_{d-1}]: the bias-moment columns of X as the operand
        if (rc == FC_OK) rc = tc_gemm(X + DP * gc, ktot, gc, m, img_t, DP * cout, U, DP * cout, st);
        if (rc) break;
        dloc_nbr_kernel<DP><<<grid, 256, 0, st>>>(p0, m, cout, feat, U, centre, dloc);
        count_launch();
    }
    if (rc) return rc;
    return check_launch("moments + GEMM (reverse, d_loc)");
}

namespace {

// centre[p, t] = sum_c xbar[p, c] Z[p, t*cin + c],  xbar = sum_s f[j_s]  (warp per point)
template <int DP>
__global__ void __launch_bounds__(256)
    centre_dot_kernel(int64_t p0, int64_t m, int64_t n, int cin, int k, const float *__restrict__ feat,
                      const int32_t *__restrict__ nbr, const float *__restrict__ Z, float *__restrict__ centre) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < m; r += nw) {
        const int64_t p = p0 + r, base = (p / n) * n;
        float part[DP];
#pragma unroll
        for (int t = 0; t < DP; ++t) part[t] = 0.f;
        for (int c = lane; c < cin; c += 32) {
            float xb = 0.f;
            for (int s = 0; s < k; ++s) xb += feat[(base + nbr[p * k + s]) * cin + c];
#pragma unroll
            for (int t = 0; t < DP; ++t) part[t] = fmaf(xb, Z[r * DP * cin + t * cin + c], part[t]);
        }
#pragma unroll
        for (int t = 0; t < DP; ++t) {
            float v = part[t];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) centre[p * DP + t] = v;
        }
    }
}

}  // namespace

// Centre role of the location gradient: Z = G . [theta_0 .. theta_{d-1}] (one SGEMM,
// N = d*cin; theta_t is [cout][cin]), then centre = rowdot(xbar, Z_t).
template <int DP>
int launch_gemm_centre_dp(int64_t total, int64_t n, int cin, int k, int cout, const float *feat, const int32_t *nbr,
                          const float *g, const float *theta, float *centre, cudaStream_t st) {
    static const bool off = [] {
        const char *e = getenv("FC_NO_GEMM");
        return e && e[0] == '1';
    }();
    if (off || cout < 32 || (reinterpret_cast<uintptr_t>(g) % 16) != 0 || cout % 4 != 0) return FC_ERR_UNSUPPORTED;
    const int64_t chunk = gemm_chunk(total, DP * cin);
    Scratch Zb(sizeof(float) * chunk * DP * cin, st), tcb(sizeof(float) * (size_t)cout * DP * cin, st), img;
    if (!Zb.ok() || !tcb.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed");
    float *Z = Zb.as<float>(), *tcat = tcb.as<float>();
    const unsigned pg = (unsigned)std::min<int64_t>(ceil_div((int64_t)cout * cin * DP, 256), 4096);
    pack_theta_cat_kernel<<<pg, 256, 0, st>>>(cout, cin, DP, theta, tcat);  // tcat[c'][t*cin + c]
    count_launch();
    if (int rc = pack_b_rm(tcat, DP * cin, cout, DP * cin, img, st)) return rc;
    int rc = FC_OK;
    for (int64_t p0 = 0; p0 < total && rc == FC_OK; p0 += chunk) {
        const int64_t m = std::min(chunk, total - p0);
        rc = tc_gemm(g + p0 * cout, cout, cout, m, img, DP * cin, Z, DP * cin, st);  // Z = G . tcat
        if (rc) break;
        const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(m, 8), (int64_t)num_sms() * 8);
        centre_dot_kernel<DP><<<grid, 256, 0, st>>>(p0, m, n, cin, k, feat, nbr, Z, centre);
        count_launch();
    }
    if (rc) return rc;
    return check_launch("GEMM (d_loc centre)");
}

#define FC_GEMM_INST(DP)                                                                                          \
    template int launch_gemm_gmc_dp<DP, false>(int64_t, int64_t, int, int, int, const float *, const float *,     \
                                               const int32_t *, Csr, const float *, float *, cudaStream_t);       \
    template int launch_gemm_gmc_dp<DP, true>(int64_t, int64_t, int, int, int, const float *, const float *,      \
                                              const int32_t *, Csr, const float *, float *, cudaStream_t);        \
    template int launch_gemm_dtheta_dp<DP>(int64_t, int64_t, int, int, int, const float *, const float *,         \
                                           const int32_t *, const float *, float *, float *, cudaStream_t);       \
    template int launch_gemm_rev_dloc_dp<DP>(int64_t, int64_t, int, int, int, const float *, const float *, Csr,  \
                                             const float *, float *, const float *, const float *, const float *, \
                                             float *, cudaStream_t);                                              \
    template int launch_gemm_centre_dp<DP>(int64_t, int64_t, int, int, int, const float *, const int32_t *,      \
                                           const float *, const float *, float *, cudaStream_t);
FC_GEMM_INST(1)
FC_GEMM_INST(2)
FC_GEMM_INST(3)
FC_GEMM_INST(4)
FC_GEMM_INST(5)
FC_GEMM_INST(6)
FC_GEMM_INST(7)
FC_GEMM_INST(8)

#define FC_WIDE_INST(T, DP)                                                                                       \
    template int launch_wide_gmc_dp<T, DP, false>(int64_t, int64_t, int, int, int, const T *, const T *,       \
                                                  const int32_t *, Csr, const T *, T *, const T *, const T *,  \
                                                  const T *, T *, cudaStream_t);                               \
    template int launch_wide_gmc_dp<T, DP, true>(int64_t, int64_t, int, int, int, const T *, const T *,        \
                                                 const int32_t *, Csr, const T *, T *, const T *, const T *,   \
                                                 const T *, T *, cudaStream_t);                                \
    template int launch_dtheta_slice_dp<T, DP>(int64_t, int64_t, int, int, int, const T *, const T *,          \
                                               const int32_t *, const T *, T *, T *, cudaStream_t);
#define FC_WIDE_INST_T(T) \
    FC_WIDE_INST(T, 1) FC_WIDE_INST(T, 2) FC_WIDE_INST(T, 3) FC_WIDE_INST(T, 4) FC_WIDE_INST(T, 5) \
    FC_WIDE_INST(T, 6) FC_WIDE_INST(T, 7) FC_WIDE_INST(T, 8)
FC_WIDE_INST_T(float)
FC_WIDE_INST_T(double)

}  // namespace fc
