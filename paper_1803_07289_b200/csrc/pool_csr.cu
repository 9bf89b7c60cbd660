// pool_csr.cu -- flex_pool (neighbourhood max-pool) forward/backward, the reverse-CSR
// builder (a stable counting sort, no float atomics) and row gather/scatter.
#include "fc_common.cuh"

#include <cstdlib>
#include <initializer_list>

namespace fc {

static int grid_1d(int64_t items, int block = 256) {
    int64_t g = ceil_div(items, block);
    const int64_t cap = (int64_t)num_sms() * 16;
    if (g > cap) g = cap;
    return (int)std::max<int64_t>(g, 1);
}

// ---------------------------------------------------------------- flex_pool forward
// out[p,c] = max_s f[j_s, c]; argmax = winning cloud-local index, ties to the lower index
// (_native.pyx:144-155: start from slot 0, replace on v > best or (v == best and j < bj)).
template <typename T>
__global__ void pool_fwd_kernel(int64_t total, int64_t n, int c, int k, const T *__restrict__ feat,
                                const int32_t *__restrict__ nbr, T *__restrict__ out,
                                int32_t *__restrict__ argmax) {
    const int64_t items = total * c;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < items;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = idx / c;
        const int ch = (int)(idx - p * c);
        const int64_t base = (p / n) * n;
        const int32_t *row = nbr + p * k;
        int32_t bj = row[0];
        T bv = feat[(base + bj) * c + ch];
        for (int s = 1; s < k; ++s) {
            const int32_t j = row[s];
            const T v = feat[(base + j) * c + ch];
            if (v > bv || (v == bv && j < bj)) {
                bv = v;
                bj = j;
            }
        }
        out[idx] = bv;
        argmax[idx] = bj;
    }
}

// ---------------------------------------------------------------- flex_pool backward
// Through the reverse neighbourhood: the winner of (i, c) is a neighbour of i, so
// d_f[j,c] = sum over i in R(j) (ascending, each i once) of [argmax[i,c]==j] g[i,c]:
// the additions of _native.pyx:165-168 in the same order -> bitwise identical.
template <typename T>
__global__ void pool_bwd_kernel(int64_t total, int64_t n, int c, int k, const T *__restrict__ g,
                                const int32_t *__restrict__ argmax, Csr csr, T *__restrict__ df) {
    const int64_t items = total * c;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < items;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = idx / c;
        const int ch = (int)(idx - j * c);
        const int32_t jl = (int32_t)(j - (j / n) * n);
        T acc = T(0);
        int64_t prev = -1;
        for (int32_t q = csr.off[j]; q < csr.off[j + 1]; ++q) {
            const int64_t i = (int64_t)csr.ent[q] / k;
            if (i == prev) continue;  // row i lists j twice: its gradient is routed once
            prev = i;
            if (argmax[i * c + ch] == jl) acc = Ar<T>::add(acc, g[i * c + ch]);
        }
        df[idx] = acc;
    }
}

// ---------------------------------------------------------------- vectorised forms
// A thread owns (point, V channels) with V = 16 / sizeof(T) (one 16-byte load per neighbour
// row); the row's K indices are loaded first and up to 8 neighbour rows are in flight before
// the first comparison.  Same comparisons in the same slot order as pool_fwd_kernel, same
// additions in the same reverse-list order as pool_bwd_kernel -> identical results.
template <typename T>
struct Vec16;
template <>
struct Vec16<float> {
    using V = float4;
    using I = int4;
    static constexpr int N = 4;
};
template <>
struct Vec16<double> {
    using V = double2;
    using I = int2;
    static constexpr int N = 2;
};

template <typename T>
__device__ __forceinline__ T vget(const typename Vec16<T>::V &v, int e) {
    return reinterpret_cast<const T *>(&v)[e];
}
template <typename T>
__device__ __forceinline__ int32_t iget(const typename Vec16<T>::I &v, int e) {
    return reinterpret_cast<const int32_t *>(&v)[e];
}

template <typename T>
__global__ void __launch_bounds__(256)
    pool_fwd_vec_kernel(int64_t total, int64_t n, int c, int k, const T *__restrict__ feat,
                        const int32_t *__restrict__ nbr, T *__restrict__ out, int32_t *__restrict__ argmax) {
    using VT = typename Vec16<T>::V;
    using IT = typename Vec16<T>::I;
    constexpr int V = Vec16<T>::N;
    const int cv = c / V;
    const int64_t items = total * cv;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < items;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = idx / cv;
        const int ch = (int)(idx - p * cv) * V;
        const int64_t base = (p / n) * n;
        const int32_t *row = nbr + p * k;
        T bv[V];
        int32_t bj[V];
        for (int s0 = 0; s0 < k; s0 += 8) {
            int32_t jj[8];
            VT vv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) jj[u] = __ldg(row + min(s0 + u, k - 1));
#pragma unroll
            for (int u = 0; u < 8; ++u) vv[u] = __ldg(reinterpret_cast<const VT *>(feat + (base + jj[u]) * c + ch));
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int s = s0 + u;
                if (s < k) {
#pragma unroll
                    for (int e = 0; e < V; ++e) {
                        const T v = vget<T>(vv[u], e);
                        if (s == 0 || v > bv[e] || (v == bv[e] && jj[u] < bj[e])) {
                            bv[e] = v;
                            bj[e] = jj[u];
                        }
                    }
                }
            }
        }
        VT o;
        IT a;
#pragma unroll
        for (int e = 0; e < V; ++e) {
            reinterpret_cast<T *>(&o)[e] = bv[e];
            reinterpret_cast<int32_t *>(&a)[e] = bj[e];
        }
        *reinterpret_cast<VT *>(out + p * c + ch) = o;
        *reinterpret_cast<IT *>(argmax + p * c + ch) = a;
    }
}

// fp32, 8 channels per thread: one 32-byte load per neighbour row (ld.global.nc.v8), twice
// the bytes in flight per thread of pool_fwd_vec_kernel; same comparisons in the same order.
__device__ __forceinline__ void ldg8f(const float *p, float (&v)[8]) {
    asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "l"(p));
}

__global__ void __launch_bounds__(256)
    pool_fwd_w8_kernel(int64_t total, int64_t n, int c, int k, const float *__restrict__ feat,
                       const int32_t *__restrict__ nbr, float *__restrict__ out, int32_t *__restrict__ argmax) {
    const int cv = c / 8;
    const int64_t items = total * cv;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < items;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = idx / cv;
        const int ch = (int)(idx - p * cv) * 8;
        const int32_t base = (int32_t)((p / n) * n);  // (point indices fit int32: B*N*k < 2^31)
        const int32_t *row = nbr + p * k;
        const float *fch = feat + ch;
        float bv[8];
        int32_t bj[8];
        for (int s0 = 0; s0 < k; s0 += 8) {
            int32_t jj[8];
            float vv[8][8];
#pragma unroll
            for (int u = 0; u < 8; ++u) jj[u] = __ldg(row + min(s0 + u, k - 1));
#pragma unroll
            for (int u = 0; u < 8; ++u) ldg8f(fch + (int64_t)(base + jj[u]) * c, vv[u]);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int s = s0 + u;
                if (s < k) {
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const float v = vv[u][e];
                        if (s == 0 || v > bv[e] || (v == bv[e] && jj[u] < bj[e])) {
                            bv[e] = v;
                            bj[e] = jj[u];
                        }
                    }
                }
            }
        }
        float4 *o = reinterpret_cast<float4 *>(out + p * c + ch);
        int4 *a = reinterpret_cast<int4 *>(argmax + p * c + ch);
        o[0] = make_float4(bv[0], bv[1], bv[2], bv[3]);
        o[1] = make_float4(bv[4], bv[5], bv[6], bv[7]);
        a[0] = make_int4(bj[0], bj[1], bj[2], bj[3]);
        a[1] = make_int4(bj[4], bj[5], bj[6], bj[7]);
    }
}

template <typename T>
__global__ void __launch_bounds__(256)
    pool_bwd_vec_kernel(int64_t total, int64_t n, int c, int k, const T *__restrict__ g,
                        const int32_t *__restrict__ argmax, Csr csr, T *__restrict__ df) {
    using VT = typename Vec16<T>::V;
    using IT = typename Vec16<T>::I;
    constexpr int V = Vec16<T>::N;
    const int cv = c / V;
    const int64_t items = total * cv;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < items;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = idx / cv;
        const int ch = (int)(idx - j * cv) * V;
        const int32_t jl = (int32_t)(j - (j / n) * n);
        const int32_t q0 = __ldg(csr.off + j), q1 = __ldg(csr.off + j + 1);
        T acc[V];
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] = T(0);
        int64_t prev = -1;
        for (int32_t qb = q0; qb < q1; qb += 8) {
            int64_t ii[8];
            IT am[8];
            VT gv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) ii[u] = (int64_t)__ldg(csr.ent + min(qb + u, q1 - 1)) / k;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                am[u] = __ldg(reinterpret_cast<const IT *>(argmax + ii[u] * c + ch));
                gv[u] = __ldg(reinterpret_cast<const VT *>(g + ii[u] * c + ch));
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (qb + u < q1 && ii[u] != prev) {  // row i lists j twice: routed once
                    prev = ii[u];
#pragma unroll
                    for (int e = 0; e < V; ++e)
                        if (iget<T>(am[u], e) == jl) acc[e] = Ar<T>::add(acc[e], vget<T>(gv[u], e));
                }
            }
        }
        VT o;
#pragma unroll
        for (int e = 0; e < V; ++e) reinterpret_cast<T *>(&o)[e] = acc[e];
        *reinterpret_cast<VT *>(df + j * c + ch) = o;
    }
}

// fp32 backward, 8 channels per thread, 2 reverse entries in flight (32-byte argmax and
// upstream loads); same additions in the same order as pool_bwd_vec_kernel.
__device__ __forceinline__ void ldg8i(const int32_t *p, int32_t (&v)[8]) {
    asm volatile("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "l"(p));
}

constexpr int kPB = 2;  // reverse entries in flight per thread
__global__ void __launch_bounds__(256)
    pool_bwd_w8_kernel(int64_t total, int64_t n, int c, int k, const float *__restrict__ g,
                       const int32_t *__restrict__ argmax, Csr csr, float *__restrict__ df) {
    const int cv = c / 8;
    const int64_t items = total * cv;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < items;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = idx / cv;
        const int ch = (int)(idx - j * cv) * 8;
        const int32_t jl = (int32_t)(j - (j / n) * n);
        const int32_t q0 = __ldg(csr.off + j), q1 = __ldg(csr.off + j + 1);
        float acc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.f;
        int64_t prev = -1;
        for (int32_t qb = q0; qb < q1; qb += kPB) {
            int32_t ii[kPB];
            int32_t am[kPB][8];
            float gv[kPB][8];
#pragma unroll
            for (int u = 0; u < kPB; ++u) ii[u] = __ldg(csr.ent + min(qb + u, q1 - 1)) / k;
#pragma unroll
            for (int u = 0; u < kPB; ++u) {
                ldg8i(argmax + (int64_t)ii[u] * c + ch, am[u]);
                ldg8f(g + (int64_t)ii[u] * c + ch, gv[u]);
            }
#pragma unroll
            for (int u = 0; u < kPB; ++u) {
                if (qb + u < q1 && ii[u] != prev) {  // row i lists j twice: routed once
                    prev = ii[u];
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        if (am[u][e] == jl) acc[e] += gv[u][e];
                }
            }
        }
        float4 *o = reinterpret_cast<float4 *>(df + j * c + ch);
        o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
        o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
}

template <typename T>
static bool vec16_ok(int c, std::initializer_list<const void *> ptrs) {
    if (c % (16 / (int)sizeof(T)) != 0) return false;
    for (const void *q : ptrs)
        if (reinterpret_cast<uintptr_t>(q) % 16 != 0) return false;
    return true;
}

// ---------------------------------------------------------------- fused down/upsample pooling
// (network.py:248-280, flexops.py:168-203) without the fine-level intermediate tensors.
// V channels per thread (V = 16 / sizeof(T) when the rows are 16-byte aligned, else 1).
template <typename T, int V>
__device__ __forceinline__ void ldvec(const T *p, T (&v)[V]) {
    if constexpr (V == 1) {
        v[0] = __ldg(p);
    } else if constexpr (V == 8 && sizeof(T) == 4) {  // fp32, 32-byte load
        asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                     : "l"(p));
    } else {
        using VT = typename Vec16<T>::V;
        const VT x = __ldg(reinterpret_cast<const VT *>(p));
#pragma unroll
        for (int e = 0; e < V; ++e) v[e] = reinterpret_cast<const T *>(&x)[e];
    }
}

// out row r pools fine row p = rows ? rows[r] : r; neighbour j's value is
// owner ? (owner[j] >= 0 ? feat[owner[j]] : 0) : feat[j]; winners hold the fine index j.
// B slots in flight per batch (fp32 x 8 channels: 4 in the forward, 2 in the backward -- 78 registers, three 256-thread blocks per SM -- so that the loaded rows stay within
// ~128 registers and two or more 256-thread blocks fit an SM: these are latency-bound)
template <typename T, int V, int B = (V == 8 ? 4 : 8)>
__global__ void __launch_bounds__(256)
    pool_select_fwd_kernel(int64_t m, int c, int k, const T *__restrict__ feat, const int32_t *__restrict__ nbr,
                           const int32_t *__restrict__ rows, const int32_t *__restrict__ owner, T *__restrict__ out,
                           int32_t *__restrict__ winners) {
    const int cv = c / V;
    const int64_t items = m * cv;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < items;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / cv;
        const int ch = (int)(idx - r * cv) * V;
        const int64_t p = rows ? (int64_t)__ldg(rows + r) : r;
        const int32_t *row = nbr + p * k;
        T bv[V];
        int32_t bj[V];
        for (int s0 = 0; s0 < k; s0 += B) {
            int32_t jj[B];
            T vv[B][V];
#pragma unroll
            for (int u = 0; u < B; ++u) jj[u] = __ldg(row + min(s0 + u, k - 1));
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const int64_t src = owner ? (int64_t)__ldg(owner + jj[u]) : (int64_t)jj[u];
                if (src >= 0) {
                    ldvec<T, V>(feat + src * c + ch, vv[u]);
                } else {
#pragma unroll
                    for (int e = 0; e < V; ++e) vv[u][e] = T(0);
                }
            }
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const int sl = s0 + u;
                if (sl < k) {
#pragma unroll
                    for (int e = 0; e < V; ++e) {
                        const T v = vv[u][e];
                        if (sl == 0 || v > bv[e] || (v == bv[e] && jj[u] < bj[e])) {
                            bv[e] = v;
                            bj[e] = jj[u];
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int e = 0; e < V; ++e) {
            out[r * c + ch + e] = bv[e];
            winners[r * c + ch + e] = bj[e];
        }
    }
}

// out row r is fine row j = rows ? rows[r] : r; sums upstream[q, ch] over j's reverse entries
// (i, s) ascending, each i once, with q = owner ? owner[i] : i (skipped when < 0) and
// winners[q, ch] == j -- the additions of _native.pyx:165-168 restricted to the rows that can
// be non-zero (dropping additions of +0.0 cannot change an accumulator that starts at +0.0).
template <typename T, int V, int B = (V == 8 ? 2 : 8)>
__global__ void __launch_bounds__(256)
    pool_select_bwd_kernel(int64_t m, int c, int k, const T *__restrict__ g, const int32_t *__restrict__ winners,
                           Csr csr, const int32_t *__restrict__ rows, const int32_t *__restrict__ owner,
                           T *__restrict__ df) {
    const int cv = c / V;
    const int64_t items = m * cv;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < items;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / cv;
        const int ch = (int)(idx - r * cv) * V;
        const int32_t j = rows ? __ldg(rows + r) : (int32_t)r;
        const int32_t q0 = __ldg(csr.off + j), q1 = __ldg(csr.off + j + 1);
        T acc[V];
#pragma unroll
        for (int e = 0; e < V; ++e) acc[e] = T(0);
        int64_t prev = -1;
        for (int32_t qb = q0; qb < q1; qb += B) {
            int32_t ii[B], src[B];
#pragma unroll
            for (int u = 0; u < B; ++u) {
                ii[u] = __ldg(csr.ent + min(qb + u, q1 - 1)) / k;
                src[u] = owner ? __ldg(owner + ii[u]) : ii[u];
            }
            int32_t am[B][V];
            T gv[B][V];
#pragma unroll
            for (int u = 0; u < B; ++u) {
                if (src[u] >= 0) {
                    if constexpr (V == 8) {
                        asm volatile("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                                     : "=r"(am[u][0]), "=r"(am[u][1]), "=r"(am[u][2]), "=r"(am[u][3]), "=r"(am[u][4]),
                                       "=r"(am[u][5]), "=r"(am[u][6]), "=r"(am[u][7])
                                     : "l"(winners + (int64_t)src[u] * c + ch));
                    } else {
#pragma unroll
                        for (int e = 0; e < V; ++e) am[u][e] = __ldg(winners + (int64_t)src[u] * c + ch + e);
                    }
                    ldvec<T, V>(g + (int64_t)src[u] * c + ch, gv[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < B; ++u) {
                if (qb + u < q1 && ii[u] != prev) {
                    prev = ii[u];
                    if (src[u] >= 0) {
#pragma unroll
                        for (int e = 0; e < V; ++e)
                            if (am[u][e] == j) acc[e] = Ar<T>::add(acc[e], gv[u][e]);
                    }
                }
            }
        }
#pragma unroll
        for (int e = 0; e < V; ++e) df[r * c + ch + e] = acc[e];
    }
}

// Record-only backward (flexops.py:154-165): buckets (row, channel) of the record.
template <typename T>
__global__ void pool_bwd_record_kernel(int64_t n_rows, int c, const T *__restrict__ g,
                                       const int32_t *__restrict__ off,
                                       const int32_t *__restrict__ ent, T *__restrict__ df) {
    const int64_t items = n_rows * c;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < items;
         idx += (int64_t)gridDim.x * blockDim.x) {
        T acc = T(0);
        for (int32_t q = off[idx]; q < off[idx + 1]; ++q) acc = Ar<T>::add(acc, g[ent[q]]);
        df[idx] = acc;
    }
}

// ---------------------------------------------------------------- counting-sort CSR
// (bucket functions: BucketFn in fc_common.cuh)

__global__ void csr_count_kernel(const int32_t *__restrict__ keys, int64_t count, BucketFn bf,
                                 int32_t *__restrict__ counts, int32_t *__restrict__ bad) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int32_t key = keys[e];
        if (key < 0 || key >= bf.n) {
            atomicAdd(bad, 1);
            continue;
        }
        atomicAdd(&counts[bf(e, key)], 1);
    }
}

__global__ void csr_fill_kernel(const int32_t *__restrict__ keys, int64_t count, BucketFn bf,
                                int32_t *__restrict__ cursor, int32_t *__restrict__ ent) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int32_t key = keys[e];
        if (key < 0 || key >= bf.n) continue;
        const int32_t pos = atomicAdd(&cursor[bf(e, key)], 1);
        ent[pos] = (int32_t)e;
    }
}

// The fill order inside a bucket is arbitrary; sorting each segment makes the result a
// deterministic, stable counting sort.  Segments of up to 16 entries (the usual case: the
// mean reverse-list length is k) are sorted here in registers; longer ones (hubs: duplicate
// points, clustered scans) are queued in long_list for csr_sort_long_kernel.
constexpr int kShortSeg = 16;

__global__ void csr_sort_segments_kernel(int64_t buckets, const int32_t *__restrict__ off,
                                         int32_t *__restrict__ ent, int32_t *__restrict__ long_list,
                                         int32_t *__restrict__ long_count) {
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < buckets;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int32_t lo = off[b], hi = off[b + 1];
        if (hi - lo <= 1) continue;
        if (hi - lo == 2) {
            const int32_t x = ent[lo], y = ent[lo + 1];
            if (x > y) {
                ent[lo] = y;
                ent[lo + 1] = x;
            }
            continue;
        }
        if (hi - lo <= kShortSeg) {  // sort in registers (bounded insertion network)
            constexpr int32_t kBig = 0x7fffffff;
            int32_t v[kShortSeg];
#pragma unroll
            for (int q = 0; q < kShortSeg; ++q) v[q] = lo + q < hi ? ent[lo + q] : kBig;
#pragma unroll
            for (int a = 1; a < kShortSeg; ++a) {
#pragma unroll
                for (int q = a; q > 0; --q) {
                    const int32_t x = v[q - 1], y = v[q];
                    v[q - 1] = min(x, y);
                    v[q] = max(x, y);
                }
            }
#pragma unroll
            for (int q = 0; q < kShortSeg; ++q)
                if (lo + q < hi) ent[lo + q] = v[q];
            continue;
        }
        long_list[atomicAdd(long_count, 1)] = (int32_t)b;
    }
}

// One CTA per long segment (grid-strided over the queue, so the launch needs no host read
// of the queue length): an ascending bitonic network over the next power of two, with the
// virtual padding slots >= m treated as +inf.  In this network form (the first stage of each
// merge compares i with i ^ (size - 1), later stages i with i ^ stride) every
// compare-exchange puts the minimum at the lower index, so padding never moves into range
// and comparisons with a partner >= m are skipped.  O(m log^2 m / threads) per segment;
// segments of up to kLongSmem entries are sorted in shared memory.
constexpr int kLongSmem = 8192;

__device__ __forceinline__ void bitonic_ascending(int32_t *v, int32_t m) {
    int32_t p2 = 1;
    while (p2 < m) p2 <<= 1;
    for (int32_t size = 2; size <= p2; size <<= 1) {
        for (int32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (int32_t i = threadIdx.x; i < p2; i += blockDim.x) {
                const int32_t j = stride == (size >> 1) ? (i ^ (size - 1)) : (i ^ stride);
                if (j > i && j < m) {
                    const int32_t x = v[i], y = v[j];
                    if (x > y) {
                        v[i] = y;
                        v[j] = x;
                    }
                }
            }
            __syncthreads();
        }
    }
}

__global__ void __launch_bounds__(256) csr_sort_long_kernel(const int32_t *__restrict__ off, int32_t *ent,
                                                            const int32_t *__restrict__ long_list,
                                                            const int32_t *__restrict__ long_count) {
    __shared__ int32_t sv[kLongSmem];
    const int32_t nl = *long_count;
    for (int32_t q = blockIdx.x; q < nl; q += gridDim.x) {
        const int32_t b = long_list[q];
        const int32_t lo = off[b], m = off[b + 1] - lo;
        if (m <= kLongSmem) {
            for (int32_t i = threadIdx.x; i < m; i += blockDim.x) sv[i] = ent[lo + i];
            __syncthreads();
            bitonic_ascending(sv, m);
            for (int32_t i = threadIdx.x; i < m; i += blockDim.x) ent[lo + i] = sv[i];
        } else {
            bitonic_ascending(ent + lo, m);  // in place in global memory (__syncthreads between stages)
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- exclusive scan (int32)
constexpr int kScanTile = 4096;  // 1024 threads x 4 items

__global__ void __launch_bounds__(1024)
    scan_block_kernel(const int32_t *__restrict__ in, int32_t *__restrict__ out, int64_t n,
                      int32_t *__restrict__ block_sums) {
    __shared__ int32_t warp_tot[32];
    const int64_t base = (int64_t)blockIdx.x * kScanTile + threadIdx.x * 4;
    int32_t v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = (base + i < n) ? in[base + i] : 0;
    const int32_t tsum = v[0] + v[1] + v[2] + v[3];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t inc = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) warp_tot[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        int32_t w = warp_tot[lane];
        int32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        warp_tot[lane] = wi - w;  // exclusive
        if (lane == 31 && block_sums) block_sums[blockIdx.x] = wi;
    }
    __syncthreads();
    int32_t run = warp_tot[warp] + inc - tsum;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
}

__global__ void scan_add_kernel(int32_t *__restrict__ out, int64_t n, const int32_t *__restrict__ add) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] += add[i / kScanTile];
}

// out[i] = sum_{q<i} in[q] for i in [0, n).
static void exclusive_scan(const int32_t *in, int32_t *out, int64_t n, cudaStream_t st) {
    const int64_t blocks = ceil_div(n, kScanTile);
    if (blocks <= 1) {
        scan_block_kernel<<<1, 1024, 0, st>>>(in, out, n, nullptr);
        count_launch();
        return;
    }
    int32_t *sums = (int32_t *)scratch_alloc(sizeof(int32_t) * blocks * 2, st);
    int32_t *sums_scan = sums + blocks;
    scan_block_kernel<<<(unsigned)blocks, 1024, 0, st>>>(in, out, n, sums);
    count_launch();
    exclusive_scan(sums, sums_scan, blocks, st);
    scan_add_kernel<<<grid_1d(n), 256, 0, st>>>(out, n, sums_scan);
    count_launch();
    scratch_free(sums, st);
}

// Generic stable CSR build: offsets [buckets+1], entries [count].  Returns the number
// of out-of-range keys through *bad_host if non-null (synchronising), else leaves the
// device counter in *bad_dev.
int build_csr(const int32_t *keys, int64_t count, BucketFn bf, int64_t buckets, int32_t *off,
              int32_t *ent, int32_t *bad_dev, cudaStream_t st) {
    int32_t *counts = (int32_t *)scratch_alloc(sizeof(int32_t) * (buckets + 1) * 2, st);
    if (!counts) return set_error(FC_ERR_CUDA, "scratch allocation failed (csr)");
    int32_t *cursor = counts + buckets + 1;
    cudaMemsetAsync(counts, 0, sizeof(int32_t) * (buckets + 1), st);
    csr_count_kernel<<<grid_1d(count), 256, 0, st>>>(keys, count, bf, counts, bad_dev);
    count_launch();
    exclusive_scan(counts, off, buckets + 1, st);
    cudaMemcpyAsync(cursor, off, sizeof(int32_t) * (buckets + 1), cudaMemcpyDeviceToDevice, st);
    csr_fill_kernel<<<grid_1d(count), 256, 0, st>>>(keys, count, bf, cursor, ent);
    count_launch();
    // long-segment queue: [0] = queue length, [1..] = bucket ids (at most
    // count / (kShortSeg + 1) segments can be longer than kShortSeg)
    int32_t *long_count = (int32_t *)scratch_alloc(sizeof(int32_t) * (count / (kShortSeg + 1) + 2), st);
    if (!long_count) {
        scratch_free(counts, st);
        return set_error(FC_ERR_CUDA, "scratch allocation failed (csr)");
    }
    int32_t *long_list = long_count + 1;
    cudaMemsetAsync(long_count, 0, sizeof(int32_t), st);
    csr_sort_segments_kernel<<<grid_1d(buckets), 256, 0, st>>>(buckets, off, ent, long_list, long_count);
    count_launch();
    csr_sort_long_kernel<<<(unsigned)num_sms() * 2, 256, 0, st>>>(off, ent, long_list, long_count);
    count_launch();
    scratch_free(long_count, st);
    scratch_free(counts, st);
    return check_launch("build_csr");
}

// ---------------------------------------------------------------- rows
template <typename T>
__global__ void gather_rows_kernel(int64_t rows_out, int c, const T *__restrict__ in,
                                   const int32_t *__restrict__ sel, T *__restrict__ out) {
    const int64_t items = rows_out * c;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < items;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / c;
        out[idx] = in[(int64_t)sel[r] * c + (idx - r * c)];
    }
}

__global__ void scatter_owner_kernel(int64_t rows_in, const int32_t *__restrict__ sel,
                                     int32_t *__restrict__ owner) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows_in;
         r += (int64_t)gridDim.x * blockDim.x)
        atomicMax(&owner[sel[r]], (int32_t)r);
}

template <typename T>
__global__ void scatter_rows_kernel(int64_t rows_out, int c, const T *__restrict__ in,
                                    const int32_t *__restrict__ owner, T *__restrict__ out) {
    const int64_t items = rows_out * c;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < items;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / c;
        const int32_t o = owner[r];
        out[idx] = o >= 0 ? in[(int64_t)o * c + (idx - r * c)] : T(0);
    }
}

__global__ void fill_i32_kernel(int32_t *p, int64_t n, int32_t v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void narrow_indices_kernel(const int64_t *__restrict__ in, int32_t *__restrict__ out,
                                      int64_t count, int64_t hi, int32_t *__restrict__ bad) {
    int32_t local_bad = 0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = in[e];
        if (v < 0 || v >= hi) {
            ++local_bad;
            out[e] = 0;
        } else {
            out[e] = (int32_t)v;
        }
    }
    if (local_bad) atomicAdd(bad, local_bad);
}

__global__ void check_indices_kernel(const int32_t *__restrict__ in, int64_t count, int64_t hi,
                                     int32_t *__restrict__ bad) {
    int32_t local_bad = 0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = in[e];
        if (v < 0 || v >= hi) ++local_bad;
    }
    if (local_bad) atomicAdd(bad, local_bad);
}

// Non-finite entries of a float tensor: *bad += count (16-byte loads where aligned).  Used for
// the network's per-layer gradient checks (network.py:391-392) without a reduction library.
template <typename T>
__global__ void __launch_bounds__(256) count_nonfinite_kernel(const T *__restrict__ x, int64_t count,
                                                              int32_t *__restrict__ bad) {
    int32_t local = 0;
    constexpr int V = 16 / sizeof(T);
    const bool vec = (reinterpret_cast<uintptr_t>(x) % 16) == 0;
    const int64_t nv = vec ? count / V : 0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nv; e += (int64_t)gridDim.x * blockDim.x) {
        typename Vec16<T>::V v = __ldg(reinterpret_cast<const typename Vec16<T>::V *>(x) + e);
#pragma unroll
        for (int q = 0; q < V; ++q) local += isfinite(reinterpret_cast<const T *>(&v)[q]) ? 0 : 1;
    }
    for (int64_t e = nv * V + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
         e += (int64_t)gridDim.x * blockDim.x)
        local += isfinite(x[e]) ? 0 : 1;
    if (__any_sync(0xffffffffu, local != 0)) {
        for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
        if ((threadIdx.x & 31) == 0 && local) atomicAdd(bad, local);
    }
}

// ---------------------------------------------------------------- launchers
template <typename T>
int launch_pool_fwd(int64_t total, int64_t n, int c, int k, const T *feat, const int32_t *nbr,
                    T *out, int32_t *argmax, cudaStream_t st) {
    if (vec16_ok<T>(c, {feat, out, argmax}))
    {
        static const bool v4 = [] {  // FC_POOL_V4=1: 4-channel lanes (A/B)
            const char *e = getenv("FC_POOL_V4");
            return e && e[0] == '1';
        }();
        if constexpr (sizeof(T) == 4) {
            if (!v4 && c % 8 == 0 && reinterpret_cast<uintptr_t>(feat) % 32 == 0) {
                static const int bs = [] {  // (FC_POOL_FWD_BLOCK for A/B)
                    const char *e = getenv("FC_POOL_FWD_BLOCK");
                    return e ? atoi(e) : 256;
                }();
                pool_fwd_w8_kernel<<<grid_1d(total * (c / 8), bs), bs, 0, st>>>(total, n, c, k, (const float *)feat, nbr,
                                                                                (float *)out, argmax);
                count_launch();
                return check_launch("pool_fwd_w8_kernel");
            }
        }
        pool_fwd_vec_kernel<T><<<grid_1d(total * (c / (16 / (int)sizeof(T)))), 256, 0, st>>>(total, n, c, k, feat, nbr,
                                                                                          out, argmax);
    }
    else
        pool_fwd_kernel<T><<<grid_1d(total * c), 256, 0, st>>>(total, n, c, k, feat, nbr, out, argmax);
    count_launch();
    return check_launch("pool_fwd_kernel");
}
template <typename T>
int launch_pool_bwd(int64_t total, int64_t n, int c, int k, const T *g, const int32_t *argmax,
                    Csr csr, T *df, cudaStream_t st) {
    if constexpr (sizeof(T) == 4) {
        static const bool v4 = [] {
            const char *e = getenv("FC_POOL_V4");
            return e && e[0] == '1';
        }();
        if (!v4 && c % 8 == 0 && reinterpret_cast<uintptr_t>(g) % 32 == 0 &&
            reinterpret_cast<uintptr_t>(argmax) % 32 == 0 && reinterpret_cast<uintptr_t>(df) % 16 == 0) {
            // latency-bound: with 2 reverse entries in flight the kernel needs 58 registers, so
            // four 256-thread blocks fill an SM (32 warps); 7 M x 64 ch 2.76 ms (4 entries, 92
            // registers, 128-thread blocks) -> 2.29 ms (FC_POOL_BWD_BLOCK for A/B)
            static const int bs = [] {
                const char *e = getenv("FC_POOL_BWD_BLOCK");
                return e ? atoi(e) : 256;
            }();
            pool_bwd_w8_kernel<<<grid_1d(total * (c / 8), bs), bs, 0, st>>>(total, n, c, k, (const float *)g, argmax, csr,
                                                                          (float *)df);
            count_launch();
            return check_launch("pool_bwd_w8_kernel");
        }
    }
    if (vec16_ok<T>(c, {g, argmax, df}))
        pool_bwd_vec_kernel<T><<<grid_1d(total * (c / (16 / (int)sizeof(T)))), 256, 0, st>>>(total, n, c, k, g, argmax,
                                                                                          csr, df);
    else
        pool_bwd_kernel<T><<<grid_1d(total * c), 256, 0, st>>>(total, n, c, k, g, argmax, csr, df);
    count_launch();
    return check_launch("pool_bwd_kernel");
}
template <typename T>
int launch_pool_bwd_record(int64_t n_rows, int c, const T *g, const int32_t *off,
                           const int32_t *ent, T *df, cudaStream_t st) {
    pool_bwd_record_kernel<T><<<grid_1d(n_rows * c), 256, 0, st>>>(n_rows, c, g, off, ent, df);
    count_launch();
    return check_launch("pool_bwd_record_kernel");
}
template <typename T>
int launch_gather_rows(int64_t rows_out, int c, const T *in, const int32_t *sel, T *out,
                       cudaStream_t st) {
    gather_rows_kernel<T><<<grid_1d(rows_out * c), 256, 0, st>>>(rows_out, c, in, sel, out);
    count_launch();
    return check_launch("gather_rows_kernel");
}
template <typename T>
int launch_scatter_rows(int64_t rows_in, int64_t rows_out, int c, const T *in, const int32_t *sel,
                        T *out, cudaStream_t st) {
    int32_t *owner = (int32_t *)scratch_alloc(sizeof(int32_t) * std::max<int64_t>(rows_out, 1), st);
    fill_i32_kernel<<<grid_1d(rows_out), 256, 0, st>>>(owner, rows_out, -1);
    count_launch();
    scatter_owner_kernel<<<grid_1d(rows_in), 256, 0, st>>>(rows_in, sel, owner);
    count_launch();
    scatter_rows_kernel<T><<<grid_1d(rows_out * c), 256, 0, st>>>(rows_out, c, in, owner, out);
    count_launch();
    scratch_free(owner, st);
    return check_launch("scatter_rows");
}

int launch_selection_owner(int64_t m, int64_t n, const int32_t *sel, int32_t *owner, cudaStream_t st) {
    fill_i32_kernel<<<grid_1d(n), 256, 0, st>>>(owner, n, -1);
    count_launch();
    if (m > 0) {
        scatter_owner_kernel<<<grid_1d(m), 256, 0, st>>>(m, sel, owner);
        count_launch();
    }
    return check_launch("selection_owner");
}

template <typename T>
int launch_pool_select_fwd(int64_t m, int c, int k, const T *feat, const int32_t *nbr, const int32_t *rows,
                           const int32_t *owner, T *out, int32_t *winners, cudaStream_t st) {
    constexpr int V = 16 / sizeof(T);
    if constexpr (sizeof(T) == 4) {  // fp32: 8 channels per thread, 32-byte loads
        if (c % 8 == 0 && reinterpret_cast<uintptr_t>(feat) % 32 == 0 && reinterpret_cast<uintptr_t>(out) % 32 == 0 &&
            reinterpret_cast<uintptr_t>(winners) % 32 == 0) {
            static const int bs = [] {  // 128-thread blocks: 5 resident per SM at 89 registers (FC_POOL_SEL_BLOCK: A/B)
                const char *e = getenv("FC_POOL_SEL_BLOCK");
                return e ? atoi(e) : 128;
            }();
            pool_select_fwd_kernel<T, 8><<<grid_1d(m * (c / 8), bs), bs, 0, st>>>(m, c, k, feat, nbr, rows, owner, out,
                                                                                  winners);
            count_launch();
            return check_launch("pool_select_fwd_kernel");
        }
    }
    if (vec16_ok<T>(c, {feat, out, winners}))
        pool_select_fwd_kernel<T, V><<<grid_1d(m * (c / V)), 256, 0, st>>>(m, c, k, feat, nbr, rows, owner, out, winners);
    else
        pool_select_fwd_kernel<T, 1><<<grid_1d(m * c), 256, 0, st>>>(m, c, k, feat, nbr, rows, owner, out, winners);
    count_launch();
    return check_launch("pool_select_fwd_kernel");
}

template <typename T>
int launch_pool_select_bwd(int64_t m, int c, int k, const T *g, const int32_t *winners, Csr csr,
                           const int32_t *rows, const int32_t *owner, T *df, cudaStream_t st) {
    constexpr int V = 16 / sizeof(T);
    if constexpr (sizeof(T) == 4) {
        if (c % 8 == 0 && reinterpret_cast<uintptr_t>(g) % 32 == 0 && reinterpret_cast<uintptr_t>(winners) % 32 == 0 &&
            reinterpret_cast<uintptr_t>(df) % 32 == 0) {
            pool_select_bwd_kernel<T, 8><<<grid_1d(m * (c / 8)), 256, 0, st>>>(m, c, k, g, winners, csr, rows, owner,
                                                                                df);
            count_launch();
            return check_launch("pool_select_bwd_kernel");
        }
    }
    if (vec16_ok<T>(c, {g, winners, df}))
        pool_select_bwd_kernel<T, V><<<grid_1d(m * (c / V)), 256, 0, st>>>(m, c, k, g, winners, csr, rows, owner, df);
    else
        pool_select_bwd_kernel<T, 1><<<grid_1d(m * c), 256, 0, st>>>(m, c, k, g, winners, csr, rows, owner, df);
    count_launch();
    return check_launch("pool_select_bwd_kernel");
}

int launch_narrow_indices(const int64_t *in, int32_t *out, int64_t count, int64_t hi, int32_t *bad,
                          cudaStream_t st) {
    narrow_indices_kernel<<<grid_1d(count), 256, 0, st>>>(in, out, count, hi, bad);
    count_launch();
    return check_launch("narrow_indices_kernel");
}
int launch_count_nonfinite(int dtype, const void *x, int64_t count, int32_t *bad, cudaStream_t st) {
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(count, 256 * 4), (int64_t)num_sms() * 8));
    if (dtype == FC_F32) count_nonfinite_kernel<float><<<g, 256, 0, st>>>((const float *)x, count, bad);
    else count_nonfinite_kernel<double><<<g, 256, 0, st>>>((const double *)x, count, bad);
    count_launch();
    return check_launch("count_nonfinite_kernel");
}
int launch_check_indices(const int32_t *in, int64_t count, int64_t hi, int32_t *bad, cudaStream_t st) {
    check_indices_kernel<<<grid_1d(count), 256, 0, st>>>(in, count, hi, bad);
    count_launch();
    return check_launch("check_indices_kernel");
}

#define FC_POOL_INST(T)                                                                          \
    template int launch_pool_fwd<T>(int64_t, int64_t, int, int, const T *, const int32_t *, T *,  \
                                    int32_t *, cudaStream_t);                                    \
    template int launch_pool_bwd<T>(int64_t, int64_t, int, int, const T *, const int32_t *, Csr,  \
                                    T *, cudaStream_t);                                          \
    template int launch_pool_bwd_record<T>(int64_t, int, const T *, const int32_t *,             \
                                           const int32_t *, T *, cudaStream_t);                  \
    template int launch_gather_rows<T>(int64_t, int, const T *, const int32_t *, T *,            \
                                       cudaStream_t);                                            \
    template int launch_scatter_rows<T>(int64_t, int64_t, int, const T *, const int32_t *, T *,  \
                                        cudaStream_t);                                           \
    template int launch_pool_select_fwd<T>(int64_t, int, int, const T *, const int32_t *,        \
                                           const int32_t *, const int32_t *, T *, int32_t *,     \
                                           cudaStream_t);                                        \
    template int launch_pool_select_bwd<T>(int64_t, int, int, const T *, const int32_t *, Csr,   \
                                           const int32_t *, const int32_t *, T *, cudaStream_t);
FC_POOL_INST(float)
FC_POOL_INST(double)

}  // namespace fc
