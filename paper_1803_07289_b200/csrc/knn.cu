// knn.cu -- exact self-kNN neighbourhood builder.
//
// Contract (neighborhood.py:1-8, :149-187; _native.pyx:171-255): row i is
// [i, the k-1 nearest OTHER points by (squared distance, index)], the distance
// accumulated in fp64 left to right over the coordinates, each term (p_i - p_j)^2
// separately rounded (no FMA) -- so equal inputs give bit-identical rows.
//  * brute : tiled all-pairs scan (candidates in ascending index, so an equal
//            distance never displaces an earlier index);
//  * grid  : cell-binned search in Chebyshev shells around the query cell, stopped
//            only when the k-1-th distance is strictly below the distance to every
//            unscanned cell (with a conservative margin) -- exact, not approximate.
#include <cfloat>
#include <climits>
#include <cmath>
#include <vector>

#include "fc_common.cuh"

namespace fc {


__device__ __forceinline__ bool key_less(double d1, int32_t j1, double d2, int32_t j2) {
    return d1 < d2 || (d1 == d2 && j1 < j2);
}

template <int KK>
__device__ __forceinline__ void topk_insert(double (&bd)[KK], int32_t (&bi)[KK], double dist, int32_t j) {
    if (!key_less(dist, j, bd[KK - 1], bi[KK - 1])) return;
#pragma unroll
    for (int q = KK - 1; q > 0; --q) {
        if (key_less(dist, j, bd[q], bi[q])) {
            const bool sh = key_less(dist, j, bd[q - 1], bi[q - 1]);
            bd[q] = sh ? bd[q - 1] : dist;
            bi[q] = sh ? bi[q - 1] : j;
        }
    }
    if (key_less(dist, j, bd[0], bi[0])) {
        bd[0] = dist;
        bi[0] = j;
    }
}

template <typename PT>
__device__ __forceinline__ double coord(const PT *p, int64_t i, int d, int t) {
    return (double)p[i * d + t];
}

// ------------------------------------------------------------------------ brute force
template <typename PT, int KK>
__global__ void __launch_bounds__(128)
    knn_brute_kernel(int64_t n, int d, int k, const PT *__restrict__ pts, int32_t *__restrict__ out) {
    __shared__ double tile[128 * kMaxDp];
    const int64_t base = (int64_t)blockIdx.y * n;
    const int64_t i = (int64_t)blockIdx.x * 128 + threadIdx.x;
    double pi[kMaxDp];
#pragma unroll
    for (int t = 0; t < kMaxDp; ++t) pi[t] = (i < n && t < d) ? coord(pts, base + i, d, t) : 0.0;
    double bd[KK];
    int32_t bi[KK];
#pragma unroll
    for (int q = 0; q < KK; ++q) {
        bd[q] = DBL_MAX;
        bi[q] = INT_MAX;
    }
    for (int64_t t0 = 0; t0 < n; t0 += 128) {
        const int64_t jl = t0 + threadIdx.x;
        if (jl < n)
            for (int t = 0; t < d; ++t) tile[threadIdx.x * kMaxDp + t] = coord(pts, base + jl, d, t);
        __syncthreads();
        const int m = (int)min((int64_t)128, n - t0);
        if (i < n) {
            for (int jj = 0; jj < m; ++jj) {
                const int32_t j = (int32_t)(t0 + jj);
                if (j == i) continue;
                double dist = 0.0;
#pragma unroll
                for (int t = 0; t < kMaxDp; ++t) {
                    if (t < d) {
                        const double dv = __dsub_rn(pi[t], tile[jj * kMaxDp + t]);
                        dist = __dadd_rn(dist, __dmul_rn(dv, dv));
                    }
                }
                topk_insert<KK>(bd, bi, dist, j);
            }
        }
        __syncthreads();
    }
    if (i < n) {
        int32_t *row = out + (base + i) * k;
        row[0] = (int32_t)i;
#pragma unroll
        for (int q = 0; q < KK; ++q)
            if (q < k - 1) row[1 + q] = bi[q];
    }
}

// Generic (large k) variant: the candidate list lives in local memory.
template <typename PT>
__global__ void __launch_bounds__(128)
    knn_brute_big_kernel(int64_t n, int d, int k, const PT *__restrict__ pts, double *__restrict__ wd,
                         int32_t *__restrict__ out) {
    const int64_t base = (int64_t)blockIdx.y * n;
    const int64_t i = (int64_t)blockIdx.x * 128 + threadIdx.x;
    if (i >= n) return;
    const int kk = k - 1;
    int32_t *row = out + (base + i) * k;
    double *bd = wd + (base + i) * (int64_t)kk;  // scratch distances, indices go to row[1..]
    int32_t *bi = row + 1;
    row[0] = (int32_t)i;
    int cnt = 0;
    for (int64_t jl = 0; jl < n; ++jl) {
        if (jl == i) continue;
        double dist = 0.0;
        for (int t = 0; t < d; ++t) {
            const double dv = __dsub_rn(coord(pts, base + i, d, t), coord(pts, base + jl, d, t));
            dist = __dadd_rn(dist, __dmul_rn(dv, dv));
        }
        int m;
        if (cnt == kk) {
            if (!(dist < bd[kk - 1])) continue;
            m = kk - 1;
        } else {
            m = cnt;
        }
        int q = m;
        while (q > 0 && bd[q - 1] > dist) {
            bd[q] = bd[q - 1];
            bi[q] = bi[q - 1];
            --q;
        }
        bd[q] = dist;
        bi[q] = (int32_t)jl;
        if (cnt < kk) ++cnt;
    }
}

// ------------------------------------------------------------------------ grid
struct GridParams {
    double lo[3];
    double h;
    int G[3];
    int bits[3];
    int d;
    int rowmajor;  // cell keys: 0 = Morton interleave (spatial order), 1 = x-fastest rows (kNN)
};

__device__ __forceinline__ int64_t interleave_cell(const GridParams &gp, int cx, int cy, int cz) {
    int64_t code = 0;
    int pos = 0;
    const int c[3] = {cx, cy, cz};
    const int maxb = max(gp.bits[0], max(gp.bits[1], gp.bits[2]));
    for (int l = 0; l < maxb; ++l)
        for (int t = 0; t < 3; ++t)
            if (l < gp.bits[t]) code |= (int64_t)((c[t] >> l) & 1) << (pos++);
    return code;
}

// cell key of the cell CSR: Morton code (spatial_order: 3-D-local runs for the conv tiles) or
// x-fastest row-major (kNN: a row of cells along x is one contiguous bucket range, scanned
// as one run of points instead of cell by cell)
__device__ __forceinline__ int64_t cell_key(const GridParams &gp, int cx, int cy, int cz) {
    if (gp.rowmajor) return ((int64_t)cz * gp.G[1] + cy) * gp.G[0] + cx;
    return interleave_cell(gp, cx, cy, cz);
}

__device__ __forceinline__ int cell_coord(const GridParams &gp, double x, int t) {
    if (t >= gp.d) return 0;
    double f = floor(__ddiv_rn(__dsub_rn(x, gp.lo[t]), gp.h));
    int c = (int)f;
    if (f < 0) c = 0;
    if (f >= gp.G[t]) c = gp.G[t] - 1;
    return c;
}

// Bounding box in two passes: each block reduces a grid-stride share to partial[block][6]
// (min x,y,z, max x,y,z); bbox_final_kernel (one block) reduces the partials.
template <typename PT>
__global__ void __launch_bounds__(256)
    bbox_partial_kernel(int64_t n, int d, const PT *__restrict__ pts, double *__restrict__ partial) {
    __shared__ double smin[3][8], smax[3][8];
    double mn[3] = {DBL_MAX, DBL_MAX, DBL_MAX}, mx[3] = {-DBL_MAX, -DBL_MAX, -DBL_MAX};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
        for (int t = 0; t < 3; ++t)
            if (t < d) {
                const double v = coord(pts, i, d, t);
                mn[t] = fmin(mn[t], v);
                mx[t] = fmax(mx[t], v);
            }
#pragma unroll
    for (int t = 0; t < 3; ++t) {
        for (int o = 16; o > 0; o >>= 1) {
            mn[t] = fmin(mn[t], __shfl_xor_sync(0xffffffffu, mn[t], o));
            mx[t] = fmax(mx[t], __shfl_xor_sync(0xffffffffu, mx[t], o));
        }
        if ((threadIdx.x & 31) == 0) {
            smin[t][threadIdx.x >> 5] = mn[t];
            smax[t][threadIdx.x >> 5] = mx[t];
        }
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        const int t = threadIdx.x;
        double a = DBL_MAX, b = -DBL_MAX;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            a = fmin(a, smin[t][w]);
            b = fmax(b, smax[t][w]);
        }
        partial[(int64_t)blockIdx.x * 6 + t] = a;
        partial[(int64_t)blockIdx.x * 6 + 3 + t] = b;
    }
}

__global__ void bbox_final_kernel(int parts, const double *__restrict__ partial, double *__restrict__ box) {
    // warp t reduces component t (0..2: min, 3..5: max) over the block partials
    const int t = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (t >= 6) return;
    double v = t < 3 ? DBL_MAX : -DBL_MAX;
    for (int q = lane; q < parts; q += 32) v = t < 3 ? fmin(v, partial[q * 6 + t]) : fmax(v, partial[q * 6 + t]);
    for (int o = 16; o > 0; o >>= 1) {
        const double w = __shfl_xor_sync(0xffffffffu, v, o);
        v = t < 3 ? fmin(v, w) : fmax(v, w);
    }
    if (lane == 0) box[t] = v;
}

// Grid parameters from the bounding box, on the device (no host read-back: the kNN and the
// spatial order are stream-ordered and CUDA-graph capturable).  Cell edge h targets `ppc`
// points per cell; per-axis resolution is clamped to 1024 cells; the Morton bucket space
// 2^(sum of per-axis bits) must fit the caller's capacity `cap` (sized on the host from n
// alone), else h grows until it does.  Any h > 0 gives the same (exact) neighbour rows.
__global__ void grid_params_kernel(const double *__restrict__ box, int64_t n, int d, double ppc, int64_t cap,
                                   int rowmajor, GridParams *__restrict__ gp_out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    GridParams gp{};
    gp.d = d;
    gp.rowmajor = rowmajor;
    double ext[3];
    int deff = 0;
    double vol = 1.0;
    for (int t = 0; t < 3; ++t) {
        ext[t] = t < d ? box[3 + t] - box[t] : 0.0;
        gp.lo[t] = t < d ? box[t] : 0.0;
        if (ext[t] > 0) {
            ++deff;
            vol *= ext[t];
        }
    }
    const double target_cells = fmax(1.0, (double)n / ppc);
    double h = deff > 0 ? pow(vol / target_cells, 1.0 / deff) : 1.0;
    if (!(h > 0) || !isfinite(h)) h = 1.0;
    for (int t = 0; t < 3; ++t)
        if (ext[t] > 0 && ext[t] / h > 1024.0) h = ext[t] / 1024.0;
    for (;;) {
        int total_bits = 0;
        for (int t = 0; t < 3; ++t) {
            gp.G[t] = ext[t] > 0 ? (int)fmin(1024.0, floor(ext[t] / h) + 1.0) : 1;
            int b = 0;
            while ((1 << b) < gp.G[t]) ++b;
            gp.bits[t] = b;
            total_bits += b;
        }
        const int64_t space = rowmajor ? (int64_t)gp.G[0] * gp.G[1] * gp.G[2] : ((int64_t)1 << total_bits);
        if (space <= cap) break;
        h *= 1.25;
    }
    gp.h = h;
    *gp_out = gp;
}

template <typename PT>
__global__ void cell_bucket_kernel(int64_t n, int d, const PT *__restrict__ pts, const GridParams *__restrict__ gpp,
                                   int32_t *__restrict__ bucket) {
    const GridParams gp = *gpp;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int c[3] = {0, 0, 0};
        for (int t = 0; t < d && t < 3; ++t) c[t] = cell_coord(gp, coord(pts, i, d, t), t);
        bucket[i] = (int32_t)cell_key(gp, c[0], c[1], c[2]);
    }
}

template <typename PT>
__global__ void sorted_points_kernel(int64_t n, int d, const PT *__restrict__ pts,
                                     const int32_t *__restrict__ ent, double4 *__restrict__ sp) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = ent[q];
        double4 v;
        v.x = coord(pts, i, d, 0);
        v.y = d > 1 ? coord(pts, i, d, 1) : 0.0;
        v.z = d > 2 ? coord(pts, i, d, 2) : 0.0;
        // the point's index rides along as raw bits (one 32-byte load per candidate; no
        // F2I conversion in the query loop -- it was 13 % of the query kernel's stalls)
        v.w = __hiloint2double(0, (int)i);
        sp[q] = v;
    }
}

// squared gap between coordinate x and cell c of axis t (0 inside; the first / last cell of
// an axis extends to infinity outward, since cell_coord clamps)
__device__ __forceinline__ double cell_gap2(const GridParams &gp, double x, int c, int t) {
    if (t >= gp.d) return 0.0;
    const double lo = gp.lo[t] + (double)c * gp.h, hi = lo + gp.h;
    double g = 0.0;
    if (c > 0 && x < lo) g = lo - x;
    else if (c < gp.G[t] - 1 && x > hi) g = x - hi;
    return g * g;
}

// candidates of a contiguous bucket range (a forced-inline function, not a lambda: the
// lambda was outlined as a call, which put the top-k arrays in local memory)
template <int KK>
__device__ __forceinline__ void knn_scan(int32_t s0, int32_t s1, const double4 *__restrict__ sp, int32_t i,
                                         const double4 &pi, int d, double (&bd)[KK], int32_t (&bi)[KK]) {
    for (int32_t s = s0; s < s1; ++s) {
        const double4 pj = sp[s];
        const int32_t j = __double2loint(pj.w);
        if (j == i) continue;
        double dist = 0.0, dv;
        dv = __dsub_rn(pi.x, pj.x);
        dist = __dadd_rn(dist, __dmul_rn(dv, dv));
        if (d > 1) {
            dv = __dsub_rn(pi.y, pj.y);
            dist = __dadd_rn(dist, __dmul_rn(dv, dv));
        }
        if (d > 2) {
            dv = __dsub_rn(pi.z, pj.z);
            dist = __dadd_rn(dist, __dmul_rn(dv, dv));
        }
        topk_insert<KK>(bd, bi, dist, j);
    }
}

template <int KK>
__global__ void __launch_bounds__(128)
    knn_grid_query_kernel(int64_t n, int k, const double4 *__restrict__ sp,
                          const int32_t *__restrict__ ent, const int32_t *__restrict__ off,
                          const GridParams *__restrict__ gpp, int32_t *__restrict__ out) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const GridParams gp = *gpp;
    const int32_t i = ent[q];
    const double4 pi = sp[q];
    const double px[3] = {pi.x, pi.y, pi.z};
    int c[3];
    for (int t = 0; t < 3; ++t) c[t] = cell_coord(gp, px[t], t);
    double bd[KK];
    int32_t bi[KK];
#pragma unroll
    for (int a = 0; a < KK; ++a) {
        bd[a] = DBL_MAX;
        bi[a] = INT_MAX;
    }
    const int kk = k - 1;
    const int rmax = max(gp.G[0], max(gp.G[1], gp.G[2]));
    const double margin = gp.h * 1e-7;
    const double prune_margin = gp.h * gp.h * 1e-6;
    for (int r = 0;; ++r) {
        for (int dz = -r; dz <= r; ++dz) {
            const int z = c[2] + dz;
            if (z < 0 || z >= gp.G[2]) continue;
            for (int dy = -r; dy <= r; ++dy) {
                const int y = c[1] + dy;
                if (y < 0 || y >= gp.G[1]) continue;
                const bool full = (dz == -r || dz == r || dy == -r || dy == r);
                // lower bound of the squared distance to any point of a cell of row (y, z):
                // cells farther than the current k-1-th distance cannot contribute (exact:
                // boundary cells are unbounded outward, and a small margin covers rounding)
                // the k-1-th distance, by register selects (an index by the runtime kk would put
                // the top-k arrays in local memory)
                double worst = bd[0];
#pragma unroll
                for (int a = 1; a < KK; ++a) worst = a <= kk - 1 ? bd[a] : worst;
                const double gyz = cell_gap2(gp, px[1], y, 1) + cell_gap2(gp, px[2], z, 2);
                if (worst < DBL_MAX && gyz - prune_margin > worst) continue;  // the whole row
                const int64_t rb = ((int64_t)z * gp.G[1] + y) * gp.G[0];
                if (full) {
                    // the row's cells x0 .. x1 are one contiguous bucket range; trim pruned ends
                    int x0 = max(c[0] - r, 0), x1 = min(c[0] + r, gp.G[0] - 1);
                    if (worst < DBL_MAX) {
                        while (x0 <= x1 && gyz + cell_gap2(gp, px[0], x0, 0) - prune_margin > worst) ++x0;
                        while (x1 >= x0 && gyz + cell_gap2(gp, px[0], x1, 0) - prune_margin > worst) --x1;
                    }
                    if (x0 <= x1) knn_scan<KK>(off[rb + x0], off[rb + x1 + 1], sp, i, pi, gp.d, bd, bi);
                } else {
                    for (int dx = -r; dx <= r; dx += 2 * r) {
                        const int x = c[0] + dx;
                        if (x < 0 || x >= gp.G[0]) continue;
                        if (worst < DBL_MAX && gyz + cell_gap2(gp, px[0], x, 0) - prune_margin > worst) continue;
                        knn_scan<KK>(off[rb + x], off[rb + x + 1], sp, i, pi, gp.d, bd, bi);
                    }
                }
            }
        }
        if (r >= rmax) break;
        // distance from the query to the nearest face of the scanned block beyond which
        // unscanned points may exist
        double dmin = DBL_MAX;
        for (int t = 0; t < 3; ++t) {
            if (c[t] - r > 0) dmin = fmin(dmin, px[t] - (gp.lo[t] + (double)(c[t] - r) * gp.h));
            if (c[t] + r < gp.G[t] - 1) dmin = fmin(dmin, (gp.lo[t] + (double)(c[t] + r + 1) * gp.h) - px[t]);
        }
        if (dmin == DBL_MAX) break;  // the block covers the whole grid
        dmin -= margin;
        double worst = bd[0];
#pragma unroll
        for (int a = 1; a < KK; ++a) worst = a <= kk - 1 ? bd[a] : worst;
        if (dmin > 0.0 && worst < dmin * dmin) break;
    }
    int32_t *row = out + (int64_t)i * k;
    row[0] = i;
#pragma unroll
    for (int a = 0; a < KK; ++a)
        if (a < kk) row[1 + a] = bi[a];
}

// ------------------------------------------------------------------------ host side
static int grid_1d(int64_t items, int block = 256) {
    int64_t g = ceil_div(items, block);
    const int64_t cap = (int64_t)num_sms() * 16;
    if (g > cap) g = cap;
    return (int)std::max<int64_t>(g, 1);
}

template <typename PT>
static int knn_brute(int64_t batch, int64_t n, int d, int k, const PT *pts, int32_t *out, cudaStream_t st) {
    const dim3 grid((unsigned)ceil_div(n, 128), (unsigned)batch);
    const int kk = k - 1;
    // exact-size instances for the configs' k = 8 / 16: the insertion's early-out compares with
    // the LAST slot, which must be the (k-1)-th neighbour, not an unused DBL_MAX slot
    if (kk <= 4) knn_brute_kernel<PT, 4><<<grid, 128, 0, st>>>(n, d, k, pts, out);
    else if (kk == 7) knn_brute_kernel<PT, 7><<<grid, 128, 0, st>>>(n, d, k, pts, out);
    else if (kk <= 8) knn_brute_kernel<PT, 8><<<grid, 128, 0, st>>>(n, d, k, pts, out);
    else if (kk == 15) knn_brute_kernel<PT, 15><<<grid, 128, 0, st>>>(n, d, k, pts, out);
    else if (kk <= 16) knn_brute_kernel<PT, 16><<<grid, 128, 0, st>>>(n, d, k, pts, out);
    else if (kk <= 32) knn_brute_kernel<PT, 32><<<grid, 128, 0, st>>>(n, d, k, pts, out);
    else {
        double *wd = (double *)scratch_alloc(sizeof(double) * batch * n * kk, st);
        if (!wd) return set_error(FC_ERR_CUDA, "scratch allocation failed (knn)");
        knn_brute_big_kernel<PT><<<grid, 128, 0, st>>>(n, d, k, pts, wd, out);
        scratch_free(wd, st);
    }
    count_launch();
    return check_launch("knn_brute");
}

// Bucket capacity of the cell CSR of an n-point cloud: the Morton space 2^(bits) of a grid
// with ~n/ppc cells, each axis rounded up to a power of two (grid_params_kernel keeps the
// actual space within it).
static int64_t cell_capacity(int64_t n, double ppc) {
    const double target = std::max(1.0, (double)n / ppc);
    int64_t cap = 64;
    while ((double)cap < 4.0 * target) cap <<= 1;
    return std::min<int64_t>(cap, (int64_t)1 << 30);
}

// Build the cell CSR of one cloud, entirely stream-ordered: bounding box -> grid parameters
// (device) -> cell keys -> stable counting sort.  gp_d (device), off [cap+1], ent [n].
template <typename PT>
static int cell_csr(int64_t n, int d, const PT *pts, GridParams *gp_d, int32_t **off_out, int32_t **ent_out,
                    int64_t *buckets_out, cudaStream_t st, double ppc_default = 2.0, int rowmajor = 0) {
    static const double ppc_env = [] {  // points per cell override (FC_KNN_PPC, for tuning)
        const char *e = getenv("FC_KNN_PPC");
        return e ? atof(e) : 0.0;
    }();
    const double ppc = ppc_env > 0.0 ? ppc_env : ppc_default;
    const int64_t cap = cell_capacity(n, ppc);
    {
        const int parts = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), (int64_t)num_sms() * 4));
        Scratch partial(sizeof(double) * 6 * parts, st), box(6 * sizeof(double), st);
        if (!partial.ok() || !box.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed (bbox)");
        bbox_partial_kernel<PT><<<parts, 256, 0, st>>>(n, d, pts, partial.as<double>());
        bbox_final_kernel<<<1, 192, 0, st>>>(parts, partial.as<double>(), box.as<double>());
        grid_params_kernel<<<1, 32, 0, st>>>(box.as<double>(), n, d, ppc, cap, rowmajor, gp_d);
        count_launch();
        count_launch();
        count_launch();
    }
    if (int rc = check_launch("bbox")) return rc;
    Scratch bucket(sizeof(int32_t) * n, st), bad(sizeof(int32_t), st);
    int32_t *off = (int32_t *)scratch_alloc(sizeof(int32_t) * (cap + 1), st);
    int32_t *ent = (int32_t *)scratch_alloc(sizeof(int32_t) * n, st);
    if (!bucket.ok() || !off || !ent || !bad.ok()) {
        scratch_free(off, st);
        scratch_free(ent, st);
        return set_error(FC_ERR_CUDA, "scratch allocation failed (grid)");
    }
    cudaMemsetAsync(bad.p, 0, sizeof(int32_t), st);
    cell_bucket_kernel<PT><<<grid_1d(n), 256, 0, st>>>(n, d, pts, gp_d, bucket.as<int32_t>());
    count_launch();
    int rc = build_csr(bucket.as<int32_t>(), n, BucketFn{2, cap, 1}, cap, off, ent, bad.as<int32_t>(), st);
    if (rc) {
        scratch_free(off, st);
        scratch_free(ent, st);
        return rc;
    }
    *off_out = off;
    *ent_out = ent;
    *buckets_out = cap;
    return FC_OK;
}

template <typename PT>
static int knn_grid(int64_t batch, int64_t n, int d, int k, const PT *pts, int32_t *out, cudaStream_t st) {
    if (d > 3) return set_error(FC_ERR_UNSUPPORTED, "grid kNN supports d <= 3");
    const int kk = k - 1;
    if (kk > 32) return set_error(FC_ERR_UNSUPPORTED, "grid kNN supports k <= 33");
    Scratch gp(sizeof(GridParams), st);
    if (!gp.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed (grid params)");
    for (int64_t b = 0; b < batch; ++b) {
        const PT *p = pts + b * n * d;
        int32_t *o = out + b * n * k;
        int32_t *off = nullptr, *ent = nullptr;
        int64_t buckets = 0;
        // kNN grid: ~3 points per cell at K <= 9 (measured 1M points: 1 -> 2.23, 2 -> 1.94,
        // 3 -> 1.82, 4 -> 1.83, 6 -> 1.93 ms), about K / 3 beyond
        if (int rc = cell_csr<PT>(n, d, p, gp.as<GridParams>(), &off, &ent, &buckets, st, std::max(3.0, k / 3.0), 1))
            return rc;
        Scratch sp(sizeof(double4) * n, st);
        if (!sp.ok()) {
            scratch_free(off, st);
            scratch_free(ent, st);
            return set_error(FC_ERR_CUDA, "scratch allocation failed (knn)");
        }
        sorted_points_kernel<PT><<<grid_1d(n), 256, 0, st>>>(n, d, p, ent, sp.as<double4>());
        count_launch();
        const unsigned g = (unsigned)ceil_div(n, 128);
        const GridParams *gpd = gp.as<GridParams>();
        const double4 *spd = sp.as<double4>();
        prof_begin("knn_grid_query", st);
        // exact-size instances for k = 8 / 16 (see knn_brute): with an unused DBL_MAX last slot
        // every candidate took the full insertion (73 % of candidates, measured)
        if (kk <= 4) knn_grid_query_kernel<4><<<g, 128, 0, st>>>(n, k, spd, ent, off, gpd, o);
        else if (kk == 7) knn_grid_query_kernel<7><<<g, 128, 0, st>>>(n, k, spd, ent, off, gpd, o);
        else if (kk <= 8) knn_grid_query_kernel<8><<<g, 128, 0, st>>>(n, k, spd, ent, off, gpd, o);
        else if (kk == 15) knn_grid_query_kernel<15><<<g, 128, 0, st>>>(n, k, spd, ent, off, gpd, o);
        else if (kk <= 16) knn_grid_query_kernel<16><<<g, 128, 0, st>>>(n, k, spd, ent, off, gpd, o);
        else knn_grid_query_kernel<32><<<g, 128, 0, st>>>(n, k, spd, ent, off, gpd, o);
        prof_end(st);
        count_launch();
        scratch_free(off, st);
        scratch_free(ent, st);
        if (int rc = check_launch("knn_grid")) return rc;
    }
    return FC_OK;
}

template <typename PT>
int launch_knn(int64_t batch, int64_t n, int d, int k, const PT *pts, int32_t *out, int algo, cudaStream_t st) {
    if (algo == FC_KNN_AUTO) algo = (n > 8192 && d <= 3 && k <= 33) ? FC_KNN_GRID : FC_KNN_BRUTE;
    if (algo == FC_KNN_GRID) return knn_grid<PT>(batch, n, d, k, pts, out, st);
    return knn_brute<PT>(batch, n, d, k, pts, out, st);
}

template <typename PT>
int launch_spatial_order(int64_t n, int d, const PT *pts, int32_t *order, cudaStream_t st) {
    if (d > 3) return set_error(FC_ERR_UNSUPPORTED, "spatial order supports d <= 3");
    Scratch gp(sizeof(GridParams), st);
    if (!gp.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed (grid params)");
    int32_t *off = nullptr, *ent = nullptr;
    int64_t buckets = 0;
    if (int rc = cell_csr<PT>(n, d, pts, gp.as<GridParams>(), &off, &ent, &buckets, st)) return rc;
    cudaMemcpyAsync(order, ent, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st);
    scratch_free(off, st);
    scratch_free(ent, st);
    return check_launch("spatial_order");
}

// ---- inverse density (sampling.py:33-48): phi[i] = sum_j |l_i - l_j| over the neighbour
// row, in the reference's numpy order: per pair ((0 + dx^2) + dy^2) + ..., sqrt, then the
// row sum as numpy's pairwise reduction (n < 8: sequential from 0; 8 <= n <= 128: eight
// running partials combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the tail).
// Plain IEEE fp64 mul/add/sqrt (no FMA contraction): bitwise equal to the reference.
__device__ __forceinline__ double pair_dist(const double *__restrict__ pts, int d, int64_t i, int64_t j) {
    double s = 0.0;
    for (int t = 0; t < d; ++t) {
        const double df = __dsub_rn(pts[i * d + t], pts[j * d + t]);
        s = __dadd_rn(s, __dmul_rn(df, df));
    }
    return __dsqrt_rn(s);
}
__global__ void inverse_density_kernel(int64_t n, int d, int k, const double *__restrict__ pts,
                                       const int32_t *__restrict__ nbr, double *__restrict__ phi) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t *row = nbr + i * k;
        double res;
        if (k < 8) {
            res = 0.0;
            for (int q = 0; q < k; ++q) res = __dadd_rn(res, pair_dist(pts, d, i, row[q]));
        } else {
            double r[8];
            for (int q = 0; q < 8; ++q) r[q] = pair_dist(pts, d, i, row[q]);
            int q = 8;
            for (; q + 8 <= k; q += 8)
                for (int u = 0; u < 8; ++u) r[u] = __dadd_rn(r[u], pair_dist(pts, d, i, row[q + u]));
            res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                            __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
            for (; q < k; ++q) res = __dadd_rn(res, pair_dist(pts, d, i, row[q]));
        }
        phi[i] = res;
    }
}

int launch_inverse_density(int64_t n, int d, int k, const double *pts, const int32_t *nbr, double *phi,
                           cudaStream_t st) {
    if (k > 128) return set_error(FC_ERR_UNSUPPORTED, "inverse density: k > 128 (numpy pairwise blocks)");
    const int grid = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)num_sms() * 8);
    inverse_density_kernel<<<grid, 256, 0, st>>>(n, d, k, pts, nbr, phi);
    count_launch();
    return check_launch("inverse_density");
}

template int launch_knn<float>(int64_t, int64_t, int, int, const float *, int32_t *, int, cudaStream_t);
template int launch_knn<double>(int64_t, int64_t, int, int, const double *, int32_t *, int, cudaStream_t);
template int launch_spatial_order<float>(int64_t, int, const float *, int32_t *, cudaStream_t);
template int launch_spatial_order<double>(int64_t, int, const double *, int32_t *, cudaStream_t);

}  // namespace fc
