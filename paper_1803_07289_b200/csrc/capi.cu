// capi.cu -- the extern "C" boundary (include/flexconv_b200.h): argument validation,
// dtype/engine dispatch, stream-ordered scratch, error reporting, launch accounting.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <unordered_map>

#include "fc_common.cuh"

namespace fc {

static thread_local char g_err[512] = "";
static std::atomic<uint64_t> g_launches{0};

int set_error(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int check_launch(const char *what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(FC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return FC_OK;
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// ---- optional per-kernel event timing (fc_profile_*): CUDA events recorded on the
// launching stream around the main kernels, read back after the caller synchronises.
struct ProfRec {
    const char *name;
    cudaEvent_t a, b;
};
static std::atomic<int> g_prof_on{0};
static ProfRec g_prof[4096];
static std::atomic<int> g_prof_n{0};
static ProfRec *g_prof_open = nullptr;

void prof_begin(const char *name, cudaStream_t st) {
    if (!g_prof_on.load()) return;
    const int i = g_prof_n.fetch_add(1);
    if (i >= 4096) return;
    ProfRec &r = g_prof[i];
    r.name = name;
    cudaEventCreate(&r.a);
    cudaEventCreate(&r.b);
    cudaEventRecord(r.a, st);
    g_prof_open = &r;
}
void prof_end(cudaStream_t st) {
    if (!g_prof_on.load() || !g_prof_open) return;
    cudaEventRecord(g_prof_open->b, st);
    g_prof_open = nullptr;
}

// Stream-ordered scratch from the device's default memory pool (kept resident: the
// release threshold is raised once so repeated calls do not return memory to the OS).
// device scratch accounting (this thread): bytes live and the high-water mark since the last
// fc_scratch_peak_reset() -- the workspace an entry point took from the pool
static thread_local int64_t g_scratch_live = 0, g_scratch_peak = 0;
static std::unordered_map<void *, size_t> &scratch_sizes() {
    static thread_local std::unordered_map<void *, size_t> m;
    return m;
}

void *scratch_alloc(size_t bytes, cudaStream_t st) {
    static uint64_t configured = 0;
    if (first_use_on_device(configured)) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, current_device()) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    void *p = nullptr;
    if (bytes == 0) bytes = 16;
    if (cudaMallocAsync(&p, bytes, st) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    scratch_sizes()[p] = bytes;
    g_scratch_live += (int64_t)bytes;
    g_scratch_peak = std::max(g_scratch_peak, g_scratch_live);
    return p;
}
void scratch_free(void *p, cudaStream_t st) {
    if (!p) return;
    auto it = scratch_sizes().find(p);
    if (it != scratch_sizes().end()) {
        g_scratch_live -= (int64_t)it->second;
        scratch_sizes().erase(it);
    }
    cudaFreeAsync(p, st);
}

// conv_simt.cu
template <typename T>
void launch_pack(int cin, int d, int cout, const T *theta, const T *theta_b, T *wt, T *wr, cudaStream_t st);
template <typename T>
int launch_gmc(bool reverse, int64_t total, int64_t n, int d, int gc, int k, int cout, const T *rows,
               const T *loc, const int32_t *nbr, Csr csr, const T *w, T *out, const T *feat,
               const T *theta, const T *centre, T *dloc, cudaStream_t st);
template <typename T>
int launch_dloc_centre(int64_t total, int64_t n, int d, int cin, int k, int cout, const T *feat,
                       const int32_t *nbr, const T *g, const T *theta, T *centre, cudaStream_t st);
template <typename T>
int launch_dtheta(int64_t total, int64_t n, int d, int cin, int k, int cout, const T *feat,
                  const T *loc, const int32_t *nbr, const T *g, T *d_theta, T *d_theta_b, cudaStream_t st);
// conv_tc.cu
int tc_conv_forward_supported(int mode, int c_in, int d, int k, int c_out);
int tc_conv_forward(int mode, int64_t total, int64_t n, int c_in, int d, int k, int c_out,
                    const float *feat, const float *loc, const int32_t *nbr, const float *theta,
                    const float *theta_b, float *out, cudaStream_t st);
int tc_reverse_supported(int mode, int gc, int d, int cout);
int tc_backward_supported(int mode, int cin, int d, int k, int cout);
int tc_backward(int mode, int64_t total, int64_t n, int cin, int d, int k, int cout, const float *g,
                const float *feat, const float *loc, const int32_t *nbr, Csr csr, const float *theta,
                const float *theta_b, float *d_features, float *d_locations, float *d_theta, float *d_theta_b,
                cudaStream_t st);
int tc_reverse_gmc(int mode, int64_t total, int64_t n, int gc, int d, int k, int cout,
                   const float *rows, const float *loc, Csr csr, const float *theta,
                   const float *theta_b, float *out, cudaStream_t st);
int tc_blocked_supported(int mode, int c_in, int d, int c_out);
int tc_blocked_forward(int mode, int64_t total, int64_t n, int c_in, int k, int c_out, const float *feat,
                       const float *loc, const int32_t *nbr, const float *theta, const float *theta_b, float *out,
                       cudaStream_t st);
int tc_blocked_deconv(int mode, int64_t total, int64_t n, int c_in, int k, int c_out, const float *x,
                      const float *loc, Csr csr, const float *theta, const float *theta_b, float *y, cudaStream_t st);
int tc_blocked_backward(int mode, int64_t total, int64_t n, int c_in, int k, int c_out, const float *g,
                        const float *feat, const float *loc, const int32_t *nbr, Csr csr, const float *theta,
                        const float *theta_b, float *d_features, float *d_locations, float *d_theta,
                        float *d_theta_b, cudaStream_t st);
// pool_csr.cu
template <typename T>
int launch_pool_fwd(int64_t total, int64_t n, int c, int k, const T *feat, const int32_t *nbr, T *out,
                    int32_t *argmax, cudaStream_t st);
template <typename T>
int launch_pool_bwd(int64_t total, int64_t n, int c, int k, const T *g, const int32_t *argmax, Csr csr,
                    T *df, cudaStream_t st);
template <typename T>
int launch_pool_bwd_record(int64_t n_rows, int c, const T *g, const int32_t *off, const int32_t *ent,
                           T *df, cudaStream_t st);
template <typename T>
int launch_gather_rows(int64_t rows_out, int c, const T *in, const int32_t *sel, T *out, cudaStream_t st);
template <typename T>
int launch_scatter_rows(int64_t rows_in, int64_t rows_out, int c, const T *in, const int32_t *sel, T *out,
                        cudaStream_t st);
int launch_selection_owner(int64_t m, int64_t n, const int32_t *sel, int32_t *owner, cudaStream_t st);
int launch_count_nonfinite(int dtype, const void *x, int64_t count, int32_t *bad, cudaStream_t st);
template <typename T>
int launch_pool_select_fwd(int64_t m, int c, int k, const T *feat, const int32_t *nbr, const int32_t *rows,
                           const int32_t *owner, T *out, int32_t *winners, cudaStream_t st);
template <typename T>
int launch_pool_select_bwd(int64_t m, int c, int k, const T *g, const int32_t *winners, Csr csr,
                           const int32_t *rows, const int32_t *owner, T *df, cudaStream_t st);
int launch_narrow_indices(const int64_t *in, int32_t *out, int64_t count, int64_t hi, int32_t *bad,
                          cudaStream_t st);
int launch_check_indices(const int32_t *in, int64_t count, int64_t hi, int32_t *bad, cudaStream_t st);
// knn.cu
template <typename PT>
int launch_knn(int64_t batch, int64_t n, int d, int k, const PT *pts, int32_t *out, int algo, cudaStream_t st);
template <typename PT>
int launch_spatial_order(int64_t n, int d, const PT *pts, int32_t *order, cudaStream_t st);
int launch_inverse_density(int64_t n, int d, int k, const double *pts, const int32_t *nbr, double *phi,
                           cudaStream_t st);

}  // namespace fc

namespace fc {
int tc_fast_forward(bool split, int64_t total, int64_t n, const float *feat, const float *loc, const int32_t *nbr,
                    const float *theta, const float *theta_b, float *out, cudaStream_t st, const int32_t *rows,
                    int64_t nrows);
}

using namespace fc;

#define ST(s) (reinterpret_cast<cudaStream_t>(s))

// Wide fp32 shapes: the channel-blocked tensor-core engines (gather -> tcgen05, nothing in HBM
// between).  FC_GEMM_ROUTE=1 selects moments rows + the hand-written tcgen05 GEMM instead (A/B
// timing; measured on C2's 8192 points: forward 0.056 vs 0.070 ms, backward 0.297 vs 0.226 ms --
// both routes are one latency-bound wave at that size).
// Wide fp32 shapes: the channel-blocked gather -> tcgen05 engines, except (mode "auto") for
// clouds of less than one wave of tiles with >= 256 channels on both sides (the U-Net's
// 16 K-point level): there each blocked pass is a single latency-bound tile per CTA repeated
// 8 times, and the moments rows + one tcgen05 GEMM route measures ~20 % faster (16 K x 256:
// fwd 0.33 -> 0.26, deconv 0.35 -> 0.28, bwd 0.77 -> 0.66 ms).  FC_GEMM_ROUTE=1 / 0 forces
// the GEMM / blocked route for every wide shape.
static bool blocked_route(int mode, int64_t total, int c_in, int d, int c_out) {
    static int gemm = -2;
    if (gemm == -2) {
        const char *e = getenv("FC_GEMM_ROUTE");
        gemm = e ? (e[0] == '1' ? 1 : 0) : -1;
    }
    if (gemm == 1 || !tc_blocked_supported(mode, c_in, d, c_out)) return false;
    if (gemm == -1 && mode == FC_MODE_AUTO && ceil_div(total, (int64_t)128) < num_sms() && c_in >= 256 && c_out >= 256)
        return false;
    return true;
}

static int check_dtype(int dtype) {
    if (dtype != FC_F32 && dtype != FC_F64) return set_error(FC_ERR_CONFIG, "unknown dtype %d", dtype);
    return FC_OK;
}

static int check_conv_shape(int64_t batch, int64_t n, int c_in, int d, int k, int c_out) {
    if (batch < 1 || n < 1) return set_error(FC_ERR_EMPTY, "empty input (batch=%lld, n=%lld)", (long long)batch, (long long)n);
    if (c_in < 1 || c_out < 1) return set_error(FC_ERR_SHAPE, "channel counts must be >= 1 (c_in=%d, c_out=%d)", c_in, c_out);
    if (d < 1 || d > kMaxDp) return set_error(FC_ERR_UNSUPPORTED, "spatial dimension d=%d outside [1, %d]", d, kMaxDp);
    if (k < 1) return set_error(FC_ERR_SHAPE, "neighbourhood size k must be >= 1 (got %d)", k);
    if (batch * n * (int64_t)k >= (int64_t)INT32_MAX) return set_error(FC_ERR_UNSUPPORTED, "B*N*k exceeds the int32 slot space");
    return FC_OK;
}

extern "C" {

int fc_abi_version(void) { return FC_ABI_VERSION; }
const char *fc_last_error(void) { return g_err; }
uint64_t fc_launch_count(void) { return g_launches.load(); }

void fc_profile_enable(int on) { g_prof_on.store(on ? 1 : 0); }
void fc_profile_reset(void) {
    const int n = std::min(g_prof_n.load(), 4096);
    for (int i = 0; i < n; ++i) {
        cudaEventDestroy(g_prof[i].a);
        cudaEventDestroy(g_prof[i].b);
    }
    g_prof_n.store(0);
}
int fc_profile_count(void) { return std::min(g_prof_n.load(), 4096); }
const char *fc_profile_name(int i) { return (i >= 0 && i < fc_profile_count()) ? g_prof[i].name : ""; }
float fc_profile_ms(int i) {
    if (i < 0 || i >= fc_profile_count()) return -1.f;
    float ms = -1.f;
    if (cudaEventElapsedTime(&ms, g_prof[i].a, g_prof[i].b) != cudaSuccess) {
        cudaGetLastError();
        return -1.f;
    }
    return ms;
}

// Forward of a subset of the rows of one cloud (the interior rows of a point-chunk shard while
// its halo rows are in flight, then the boundary rows): fp32 split engine, the headline shape.
int fc_conv_forward_rows(int64_t n, int c_in, int d, int k, int c_out, const void *features, const void *locations,
                         const int32_t *neighbors, const void *theta, const void *theta_b, const int32_t *rows,
                         int64_t nrows, void *out, void *stream) {
    if (int rc = check_conv_shape(1, n, c_in, d, k, c_out)) return rc;
    if (!(c_in == 64 && c_out == 64 && d == 3 && k == 8))
        return set_error(FC_ERR_UNSUPPORTED, "row-list forward covers c_in = c_out = 64, d = 3, k = 8");
    if (nrows < 0 || nrows > n) return set_error(FC_ERR_SHAPE, "nrows %lld outside [0, %lld]", (long long)nrows, (long long)n);
    if (nrows == 0) return FC_OK;  // (an empty list's pointer may be null, which means "every row" below)
    if (!rows) return set_error(FC_ERR_CONFIG, "row list is null");
    return fc::tc_fast_forward(true, n, n, (const float *)features, (const float *)locations, neighbors, (const float *)theta,
                           (const float *)theta_b, (float *)out, ST(stream), rows, nrows);
}

int fc_conv_forward(int dtype, int mode, int64_t batch, int64_t n, int c_in, int d, int k, int c_out,
                    const void *features, const void *locations, const int32_t *neighbors,
                    const void *theta, const void *theta_b, void *out, void *stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (int rc = check_conv_shape(batch, n, c_in, d, k, c_out)) return rc;
    cudaStream_t st = ST(stream);
    const int64_t total = batch * n;
    if (dtype == FC_F32 && mode != FC_MODE_SIMT) {
        if (tc_conv_forward_supported(mode, c_in, d, k, c_out))
            return tc_conv_forward(mode, total, n, c_in, d, k, c_out, (const float *)features,
                                   (const float *)locations, neighbors, (const float *)theta,
                                   (const float *)theta_b, (float *)out, st);
        if (blocked_route(mode, total, c_in, d, c_out))
            return tc_blocked_forward(mode, total, n, c_in, k, c_out, (const float *)features,
                                      (const float *)locations, neighbors, (const float *)theta,
                                      (const float *)theta_b, (float *)out, st);
        if (mode != FC_MODE_AUTO)
            return set_error(FC_ERR_UNSUPPORTED, "tensor-core engine %d does not cover c_in=%d d=%d c_out=%d", mode, c_in, d, c_out);
    }
    auto run = [&](auto tag) -> int {
        using T = decltype(tag);
        const size_t wbytes = (size_t)c_out * c_in * (d + 1) * sizeof(T);
        T *wt = (T *)scratch_alloc(wbytes, st);
        if (!wt) return set_error(FC_ERR_CUDA, "scratch allocation failed");
        launch_pack<T>(c_in, d, c_out, (const T *)theta, (const T *)theta_b, wt, nullptr, st);
        int rc = launch_gmc<T>(false, total, n, d, c_in, k, c_out, (const T *)features, (const T *)locations,
                               neighbors, Csr{nullptr, nullptr}, wt, (T *)out, nullptr, nullptr, nullptr, nullptr, st);
        scratch_free(wt, st);
        return rc;
    };
    return dtype == FC_F32 ? run(float{}) : run(double{});
}

int fc_conv_backward(int dtype, int mode, int64_t batch, int64_t n, int c_in, int d, int k, int c_out,
                     const void *upstream, const void *features, const void *locations,
                     const int32_t *neighbors, const int32_t *rev_offsets, const int32_t *rev_entries,
                     const void *theta, const void *theta_b, void *d_features, void *d_locations,
                     void *d_theta, void *d_theta_b, void *stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (int rc = check_conv_shape(batch, n, c_in, d, k, c_out)) return rc;
    if ((d_features || d_locations) && (!rev_offsets || !rev_entries))
        return set_error(FC_ERR_CONFIG, "d_features/d_locations need the reverse neighbourhood (fc_csr_build)");
    cudaStream_t st = ST(stream);
    const int64_t total = batch * n;
    if (dtype == FC_F32 && mode != FC_MODE_SIMT && tc_backward_supported(mode, c_in, d, k, c_out))
        return tc_backward(mode, total, n, c_in, d, k, c_out, (const float *)upstream, (const float *)features,
                           (const float *)locations, neighbors, Csr{rev_offsets, rev_entries}, (const float *)theta,
                           (const float *)theta_b, (float *)d_features, (float *)d_locations, (float *)d_theta,
                           (float *)d_theta_b, st);
    if (dtype == FC_F32 && mode != FC_MODE_SIMT && blocked_route(mode, total, c_in, d, c_out))
        return tc_blocked_backward(mode, total, n, c_in, k, c_out, (const float *)upstream, (const float *)features,
                                   (const float *)locations, neighbors, Csr{rev_offsets, rev_entries},
                                   (const float *)theta, (const float *)theta_b, (float *)d_features,
                                   (float *)d_locations, (float *)d_theta, (float *)d_theta_b, st);
    auto run = [&](auto tag) -> int {
        using T = decltype(tag);
        const T *g = (const T *)upstream;
        const T *f = (const T *)features;
        const T *l = (const T *)locations;
        const T *th = (const T *)theta;
        int rc = FC_OK;
        if (d_theta || d_theta_b) {
            rc = launch_dtheta<T>(total, n, d, c_in, k, c_out, f, l, neighbors, g, (T *)d_theta, (T *)d_theta_b, st);
            if (rc) return rc;
        }
        if (d_features || d_locations) {
            Scratch centre_buf;
            if (d_locations) {
                centre_buf.alloc(sizeof(T) * total * d, st);
                if (!centre_buf.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed");
                rc = launch_dloc_centre<T>(total, n, d, c_in, k, c_out, f, neighbors, g, th, centre_buf.as<T>(), st);
                if (rc) return rc;
            }
            T *centre = centre_buf.as<T>();
            T *df = (T *)d_features;
            Scratch df_buf;
            if (!df) {
                df_buf.alloc(sizeof(T) * total * c_in, st);
                if (!df_buf.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed");
                df = df_buf.as<T>();
            }
            const bool tc = dtype == FC_F32 && mode != FC_MODE_SIMT && !d_locations &&
                            tc_reverse_supported(mode, c_out, d, c_in);
            if (tc) {
                rc = tc_reverse_gmc(mode, total, n, c_out, d, k, c_in, (const float *)g, (const float *)l,
                                    Csr{rev_offsets, rev_entries}, (const float *)th, (const float *)theta_b,
                                    (float *)df, st);
            } else {
                Scratch wr((size_t)c_out * c_in * (d + 1) * sizeof(T), st);
                if (!wr.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed");
                launch_pack<T>(c_in, d, c_out, th, (const T *)theta_b, nullptr, wr.as<T>(), st);
                rc = launch_gmc<T>(true, total, n, d, c_out, k, c_in, g, l, neighbors, Csr{rev_offsets, rev_entries},
                                   wr.as<T>(), df, f, th, centre, (T *)d_locations, st);
            }
        }
        return rc;
    };
    return dtype == FC_F32 ? run(float{}) : run(double{});
}

int fc_deconv_forward(int dtype, int mode, int64_t batch, int64_t n, int c_in, int d, int k, int c_out,
                      const void *x, const void *locations, const int32_t *rev_offsets,
                      const int32_t *rev_entries, const void *theta, const void *theta_b, void *y,
                      void *stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (int rc = check_conv_shape(batch, n, c_in, d, k, c_out)) return rc;
    if (!rev_offsets || !rev_entries) return set_error(FC_ERR_CONFIG, "flex_deconv needs the reverse neighbourhood");
    cudaStream_t st = ST(stream);
    const int64_t total = batch * n;
    if (dtype == FC_F32 && mode != FC_MODE_SIMT) {
        if (tc_reverse_supported(mode, c_out, d, c_in))
            return tc_reverse_gmc(mode, total, n, c_out, d, k, c_in, (const float *)x, (const float *)locations,
                                  Csr{rev_offsets, rev_entries}, (const float *)theta, (const float *)theta_b,
                                  (float *)y, st);
        if (blocked_route(mode, total, c_in, d, c_out))
            return tc_blocked_deconv(mode, total, n, c_in, k, c_out, (const float *)x, (const float *)locations,
                                     Csr{rev_offsets, rev_entries}, (const float *)theta, (const float *)theta_b,
                                     (float *)y, st);
        if (mode != FC_MODE_AUTO)
            return set_error(FC_ERR_UNSUPPORTED, "tensor-core engine %d does not cover this deconv shape", mode);
    }
    auto run = [&](auto tag) -> int {
        using T = decltype(tag);
        T *wr = (T *)scratch_alloc((size_t)c_out * c_in * (d + 1) * sizeof(T), st);
        if (!wr) return set_error(FC_ERR_CUDA, "scratch allocation failed");
        launch_pack<T>(c_in, d, c_out, (const T *)theta, (const T *)theta_b, nullptr, wr, st);
        int rc = launch_gmc<T>(true, total, n, d, c_out, k, c_in, (const T *)x, (const T *)locations, nullptr,
                               Csr{rev_offsets, rev_entries}, wr, (T *)y, nullptr, nullptr, nullptr, nullptr, st);
        scratch_free(wr, st);
        return rc;
    };
    return dtype == FC_F32 ? run(float{}) : run(double{});
}

int fc_csr_build(int64_t batch, int64_t n, int k, const int32_t *neighbors, int32_t *offsets,
                 int32_t *entries, void *stream) {
    if (batch < 1 || n < 1 || k < 1) return set_error(FC_ERR_EMPTY, "empty neighbourhood");
    if (batch * n * (int64_t)k >= (int64_t)INT32_MAX) return set_error(FC_ERR_UNSUPPORTED, "B*N*k exceeds int32");
    cudaStream_t st = ST(stream);
    Scratch bad(sizeof(int32_t), st);
    if (!bad.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed (csr)");
    cudaMemsetAsync(bad.p, 0, sizeof(int32_t), st);
    int rc = build_csr(neighbors, batch * n * k, BucketFn{0, n, k}, batch * n, offsets, entries, bad.as<int32_t>(), st);
    int32_t bad_h = 0;
    cudaMemcpyAsync(&bad_h, bad.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (rc) return rc;
    if (int rc2 = check_launch("fc_csr_build")) return rc2;
    if (bad_h) return set_error(FC_ERR_INDEX, "neighbor index out of [0, n) (%d entries)", bad_h);
    return FC_OK;
}

int fc_csr_build_async(int64_t batch, int64_t n, int k, const int32_t *neighbors, int32_t *offsets,
                       int32_t *entries, int32_t *bad, void *stream) {
    if (batch < 1 || n < 1 || k < 1) return set_error(FC_ERR_EMPTY, "empty neighbourhood");
    if (batch * n * (int64_t)k >= (int64_t)INT32_MAX) return set_error(FC_ERR_UNSUPPORTED, "B*N*k exceeds int32");
    if (!bad) return set_error(FC_ERR_CONFIG, "fc_csr_build_async needs a device counter for bad indices");
    return build_csr(neighbors, batch * n * k, BucketFn{0, n, k}, batch * n, offsets, entries, bad, ST(stream));
}

int fc_pool_forward(int dtype, int64_t batch, int64_t n, int c, int k, const void *features,
                    const int32_t *neighbors, void *out, int32_t *argmax, void *stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (batch < 1 || n < 1) return set_error(FC_ERR_EMPTY, "empty input");
    if (c < 1 || k < 1) return set_error(FC_ERR_SHAPE, "c and k must be >= 1");
    cudaStream_t st = ST(stream);
    if (dtype == FC_F32)
        return launch_pool_fwd<float>(batch * n, n, c, k, (const float *)features, neighbors, (float *)out, argmax, st);
    return launch_pool_fwd<double>(batch * n, n, c, k, (const double *)features, neighbors, (double *)out, argmax, st);
}

int fc_pool_backward(int dtype, int64_t batch, int64_t n, int c, int k, const void *upstream,
                     const int32_t *argmax, const int32_t *rev_offsets, const int32_t *rev_entries,
                     void *d_features, void *stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (batch < 1 || n < 1) return set_error(FC_ERR_EMPTY, "empty input");
    if (!rev_offsets || !rev_entries) return set_error(FC_ERR_CONFIG, "pool backward needs the reverse neighbourhood");
    cudaStream_t st = ST(stream);
    Csr csr{rev_offsets, rev_entries};
    if (dtype == FC_F32)
        return launch_pool_bwd<float>(batch * n, n, c, k, (const float *)upstream, argmax, csr, (float *)d_features, st);
    return launch_pool_bwd<double>(batch * n, n, c, k, (const double *)upstream, argmax, csr, (double *)d_features, st);
}

int fc_record_csr_build(int64_t n_up, int64_t n_rows, int c, const int32_t *record, int32_t *offsets,
                        int32_t *entries, void *stream) {
    if (n_rows < 1 || c < 1) return set_error(FC_ERR_EMPTY, "empty record");
    if (n_up * (int64_t)c >= (int64_t)INT32_MAX || n_rows * (int64_t)c >= (int64_t)INT32_MAX)
        return set_error(FC_ERR_UNSUPPORTED, "record too large for int32 slots");
    cudaStream_t st = ST(stream);
    Scratch bad(sizeof(int32_t), st);
    if (!bad.ok()) return set_error(FC_ERR_CUDA, "scratch allocation failed (record csr)");
    cudaMemsetAsync(bad.p, 0, sizeof(int32_t), st);
    int rc = build_csr(record, n_up * c, BucketFn{1, n_rows, c}, n_rows * c, offsets, entries, bad.as<int32_t>(), st);
    int32_t bad_h = 0;
    cudaMemcpyAsync(&bad_h, bad.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (rc) return rc;
    if (bad_h) return set_error(FC_ERR_INDEX, "corrupt pool record: winner index out of range");
    return check_launch("fc_record_csr_build");
}

int fc_pool_backward_record(int dtype, int64_t n_up, int64_t n_rows, int c, const void *upstream,
                            const int32_t *offsets, const int32_t *entries, void *d_features, void *stream) {
    if (int rc = check_dtype(dtype)) return rc;
    (void)n_up;
    cudaStream_t st = ST(stream);
    if (dtype == FC_F32)
        return launch_pool_bwd_record<float>(n_rows, c, (const float *)upstream, offsets, entries, (float *)d_features, st);
    return launch_pool_bwd_record<double>(n_rows, c, (const double *)upstream, offsets, entries, (double *)d_features, st);
}

__global__ static void self_rows_kernel(int64_t total, int64_t n, int32_t *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)(i % n);
}

int fc_knn(int dtype, int64_t batch, int64_t n, int d, int k, const void *points, int32_t *out, int algo,
           void *stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (batch < 1 || n < 1) return set_error(FC_ERR_EMPTY, "no points to index");
    if (d < 1 || d > kMaxDp) return set_error(FC_ERR_UNSUPPORTED, "kNN supports 1 <= d <= %d", kMaxDp);
    if (k < 1 || k > n) return set_error(FC_ERR_CONFIG, "k must satisfy 1 <= k <= %lld, got %d", (long long)n, k);
    if (n >= (int64_t)INT32_MAX) return set_error(FC_ERR_UNSUPPORTED, "cloud too large for int32 indices");
    cudaStream_t st = ST(stream);
    if (k == 1) {
        self_rows_kernel<<<(unsigned)std::min<int64_t>(ceil_div(batch * n, 256), 4096), 256, 0, st>>>(batch * n, n, out);
        count_launch();
        return check_launch("self_rows_kernel");
    }
    if (dtype == FC_F32) return launch_knn<float>(batch, n, d, k, (const float *)points, out, algo, st);
    return launch_knn<double>(batch, n, d, k, (const double *)points, out, algo, st);
}

int fc_spatial_order(int dtype, int64_t n, int d, const void *points, int32_t *order, void *stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (n < 1) return set_error(FC_ERR_EMPTY, "no points");
    cudaStream_t st = ST(stream);
    if (dtype == FC_F32) return launch_spatial_order<float>(n, d, (const float *)points, order, st);
    return launch_spatial_order<double>(n, d, (const double *)points, order, st);
}

int fc_inverse_density(int64_t n, int d, int k, const double *points, const int32_t *neighbors, double *phi,
                       void *stream) {
    if (n < 1) return set_error(FC_ERR_EMPTY, "no points");
    if (d < 1 || k < 1) return set_error(FC_ERR_SHAPE, "d and k must be >= 1");
    return launch_inverse_density(n, d, k, points, neighbors, phi, ST(stream));
}

int fc_gather_rows(int dtype, int64_t rows_out, int c, const void *in, const int32_t *sel, void *out, void *stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (rows_out == 0) return FC_OK;
    cudaStream_t st = ST(stream);
    if (dtype == FC_F32) return launch_gather_rows<float>(rows_out, c, (const float *)in, sel, (float *)out, st);
    return launch_gather_rows<double>(rows_out, c, (const double *)in, sel, (double *)out, st);
}

int fc_scatter_rows(int dtype, int64_t rows_in, int64_t rows_out, int c, const void *in, const int32_t *sel,
                    void *out, void *stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (rows_out == 0) return FC_OK;
    cudaStream_t st = ST(stream);
    if (dtype == FC_F32) return launch_scatter_rows<float>(rows_in, rows_out, c, (const float *)in, sel, (float *)out, st);
    return launch_scatter_rows<double>(rows_in, rows_out, c, (const double *)in, sel, (double *)out, st);
}

int fc_selection_owner(int64_t m, int64_t n, const int32_t *sel, int32_t *owner, void *stream) {
    if (n < 1) return set_error(FC_ERR_EMPTY, "empty fine level");
    if (m < 0) return set_error(FC_ERR_SHAPE, "negative selection size");
    return launch_selection_owner(m, n, sel, owner, ST(stream));
}

int fc_pool_select_forward(int dtype, int64_t m, int64_t n, int c, int k, const void *features,
                           const int32_t *neighbors, const int32_t *rows, const int32_t *owner, void *out,
                           int32_t *winners, void *stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (n < 1) return set_error(FC_ERR_EMPTY, "empty fine level");
    if (c < 1 || k < 1 || m < 0) return set_error(FC_ERR_SHAPE, "c and k must be >= 1, m >= 0");
    if (m == 0) return FC_OK;
    cudaStream_t st = ST(stream);
    if (dtype == FC_F32)
        return launch_pool_select_fwd<float>(m, c, k, (const float *)features, neighbors, rows, owner, (float *)out,
                                             winners, st);
    return launch_pool_select_fwd<double>(m, c, k, (const double *)features, neighbors, rows, owner, (double *)out,
                                          winners, st);
}

int fc_pool_select_backward(int dtype, int64_t m, int64_t n, int c, int k, const void *upstream,
                            const int32_t *winners, const int32_t *rev_offsets, const int32_t *rev_entries,
                            const int32_t *rows, const int32_t *owner, void *d_features, void *stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (n < 1) return set_error(FC_ERR_EMPTY, "empty fine level");
    if (c < 1 || k < 1 || m < 0) return set_error(FC_ERR_SHAPE, "c and k must be >= 1, m >= 0");
    if (!rev_offsets || !rev_entries) return set_error(FC_ERR_CONFIG, "pool backward needs the reverse neighbourhood");
    if (m == 0) return FC_OK;
    cudaStream_t st = ST(stream);
    const Csr csr{rev_offsets, rev_entries};
    if (dtype == FC_F32)
        return launch_pool_select_bwd<float>(m, c, k, (const float *)upstream, winners, csr, rows, owner,
                                             (float *)d_features, st);
    return launch_pool_select_bwd<double>(m, c, k, (const double *)upstream, winners, csr, rows, owner,
                                          (double *)d_features, st);
}

int fc_indices_to_i32(const int64_t *in, int32_t *out, int64_t count, int64_t hi, int32_t *bad, void *stream) {
    if (count == 0) return FC_OK;
    return launch_narrow_indices(in, out, count, hi, bad, ST(stream));
}

int fc_count_nonfinite(int dtype, const void *x, int64_t count, int32_t *bad, void *stream) {
    if (int rc = check_dtype(dtype)) return rc;
    if (count == 0) return FC_OK;
    return fc::launch_count_nonfinite(dtype, x, count, bad, ST(stream));
}

int fc_check_indices(const int32_t *idx, int64_t count, int64_t hi, int32_t *bad, void *stream) {
    if (count == 0) return FC_OK;
    return launch_check_indices(idx, count, hi, bad, ST(stream));
}


// Workspace query: the peak device scratch (bytes, stream-ordered pool) the
// entry points called on this thread took since the last reset -- run an op once on the
// shape of interest after fc_scratch_peak_reset() to size a pool.
int64_t fc_scratch_peak_bytes(void) { return g_scratch_peak; }
void fc_scratch_peak_reset(void) { g_scratch_peak = g_scratch_live; }

// flex_deconv backward: y = A(theta)^T x, so with upstream gy = dL/dy:
//   d_x = A(theta) gy (flex_conv forward of gy), and theta / theta_b / location gradients are
//   flex_conv's backward with upstream = x and features = gy (<A^T x, gy> = <x, A gy>).
int fc_deconv_backward(int dtype, int mode, int64_t batch, int64_t n, int c_in, int d, int k, int c_out,
                       const void *upstream, const void *x, const void *locations, const int32_t *neighbors,
                       const int32_t *rev_offsets, const int32_t *rev_entries, const void *theta,
                       const void *theta_b, void *d_x, void *d_locations, void *d_theta, void *d_theta_b,
                       void *stream) {
    if (d_x) {
        if (int rc = fc_conv_forward(dtype, mode, batch, n, c_in, d, k, c_out, upstream, locations, neighbors, theta,
                                     theta_b, d_x, stream))
            return rc;
    }
    if (d_locations || d_theta || d_theta_b)
        return fc_conv_backward(dtype, mode, batch, n, c_in, d, k, c_out, x, upstream, locations, neighbors,
                                rev_offsets, rev_entries, theta, theta_b, nullptr, d_locations, d_theta, d_theta_b,
                                stream);
    return FC_OK;
}

}  // extern "C"
