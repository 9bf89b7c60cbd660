/*
 * flexconv_b200.h -- C ABI of the B200-native flex-convolution hot path.
 *
 * The drop-in boundary: plain pointers, sizes and a cudaStream_t (passed as void*),
 * int status codes, caller-allocated outputs, no torch types.  Each entry point names
 * the reference interface it replaces.  The reference's kernel slot is the module ABI
 * shared by flexconv._native and flexconv._reference (identical signatures,
 * /root/reference/pkg/src/flexconv/_reference.py:3-4) selected by backend.active()
 * (/root/reference/pkg/src/flexconv/backend.py:34-36); its callers are the flexops /
 * neighborhood wrappers.  INTEGRATION.md shows the binding a maintainer would add.
 *
 * Conventions (all entry points)
 *  - Device pointers.  Point-major layouts: features [B*N, C], locations [B*N, d],
 *    neighbours [B*N, k] int32 with CLOUD-LOCAL indices (row i of cloud b lists
 *    indices in [0, N)); B clouds of N points stacked along the point axis.
 *    The reference has no batch axis: B = 1 reproduces it exactly.
 *  - theta [c_out, c_in, d], theta_b [c_out, c_in] -- the reference's FlexConvParams
 *    shapes (flexops.py:22-51).  Offsets are centre - neighbour (l_i - l_j,
 *    _native.pyx:55).
 *  - dtype: FC_F32 or FC_F64 for every floating tensor of the call.  FC_F64 runs
 *    the reference's arithmetic (fp64, same operation order; forward and pooling
 *    are bitwise identical to _native).
 *  - Outputs are OVERWRITTEN (the reference zero-fills then accumulates,
 *    flexops.py:123-126 -- same result).  Nullable outputs are skipped.
 *  - Work is enqueued on `stream` (cudaStream_t; NULL = legacy default stream);
 *    no entry point synchronises the host except the validating reverse-CSR builders
 *    (fc_csr_build, fc_record_csr_build: they report bad indices as a status code, like the
 *    reference's range checks); fc_csr_build_async is their stream-ordered form.
 *  - Return FC_OK or an FC_ERR_* code; fc_last_error() holds the message (thread-local).
 */
#ifndef FLEXCONV_B200_H
#define FLEXCONV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FC_ABI_VERSION 1

/* Status codes map 1:1 onto the reference's EngineError kinds (errors.py:8-35). */
enum {
    FC_OK = 0,
    FC_ERR_SHAPE = 1,      /* ShapeMismatchError  */
    FC_ERR_INDEX = 2,      /* IndexOutOfRangeError */
    FC_ERR_NONFINITE = 3,  /* NonFiniteError       */
    FC_ERR_EMPTY = 4,      /* EmptyInputError      */
    FC_ERR_CONFIG = 5,     /* ConfigInvalidError   */
    FC_ERR_CUDA = 6,       /* CUDA runtime failure */
    FC_ERR_UNSUPPORTED = 7 /* shape not covered by the requested engine */
};

enum { FC_F32 = 0, FC_F64 = 1 };

/* Contraction engine for FC_F32 (ignored for FC_F64, which is always SIMT fp64). */
enum {
    FC_MODE_AUTO = 0,     /* tensor-core split engine where the shape is covered, else SIMT */
    FC_MODE_SIMT = 1,     /* CUDA-core fp32 FMA                                             */
    FC_MODE_TC_SPLIT = 2, /* tcgen05 kind::f16: each fp32 operand split into fp16 hi + lo    */
                          /* with power-of-two scaling, 3 MMAs (hi*hi + hi*lo + lo*hi),      */
                          /* fp32 accumulate -- fp32-level accuracy (1e-4 rel / 1e-5 abs)    */
    FC_MODE_TC_BF16 = 3   /* tcgen05 kind::f16, bf16 operands, 1 MMA, fp32 accumulate (1e-2) */
};

/* kNN algorithm selector. */
enum { FC_KNN_AUTO = 0, FC_KNN_BRUTE = 1, FC_KNN_GRID = 2 };

int fc_abi_version(void);
const char *fc_last_error(void);
/* Number of kernel launches this library has issued (process-wide counter). */
uint64_t fc_launch_count(void);

/* Optional per-kernel timing: while enabled, CUDA events are recorded on the launching
 * stream around each main kernel; after synchronising, fc_profile_ms(i) is the device time
 * of record i (fc_profile_name(i) names the kernel).  Used by bench.py's roofline. */
void fc_profile_enable(int on);
void fc_profile_reset(void);
int fc_profile_count(void);
const char *fc_profile_name(int i);
float fc_profile_ms(int i);

/* ---- flex_conv -------------------------------------------------------------------
 * Replaces _native.flex_conv_forward(features, locations, neighbors, theta, theta_b,
 * out, num_threads) (_native.pyx:25-28), called by flexops.flex_conv_forward
 * (flexops.py:97-110).  out [B*N, c_out]. */
int fc_conv_forward(int dtype, int mode, int64_t batch, int64_t n, int c_in, int d, int k,
                    int c_out, const void *features, const void *locations,
                    const int32_t *neighbors, const void *theta, const void *theta_b,
                    void *out, void *stream);

/* Replaces _native.flex_conv_backward(upstream, features, locations, neighbors, theta,
 * theta_b, d_features, d_locations, d_theta, d_theta_b, with_locations)
 * (_native.pyx:69-74), called by flexops.flex_conv_backward (flexops.py:113-132).
 * rev_offsets/rev_entries: the reverse neighbourhood from fc_csr_build (needed when
 * d_features or d_locations is requested).  d_locations == NULL <=> with_locations=False.
 * Deterministic: no floating-point atomics; bitwise reproducible run to run. */
int fc_conv_backward(int dtype, int mode, int64_t batch, int64_t n, int c_in, int d, int k,
                     int c_out, const void *upstream, const void *features,
                     const void *locations, const int32_t *neighbors,
                     const int32_t *rev_offsets, const int32_t *rev_entries,
                     const void *theta, const void *theta_b, void *d_features,
                     void *d_locations, void *d_theta, void *d_theta_b, void *stream);

/* ---- flex_deconv (transposed flex_conv) --------------------------------------------
 * No reference function (the reference drops it); defined as the adjoint
 * y = A(theta)^T x of flex_conv with the SAME theta shapes.  Exact reference equivalent:
 * flex_conv_backward(upstream=x, ...).d_features (_native.pyx:106-120).
 * x [B*N, c_out] -> y [B*N, c_in].  Needs the reverse neighbourhood. */
/* Forward of the rows rows[0 .. nrows) only (sorted int32 row ids of one cloud of n points;
 * the other rows of `out` are untouched): a point-chunk shard computes its interior rows while
 * the halo exchange is in flight, then its boundary rows.  fp32, c_in = c_out = 64, d = 3,
 * k = 8 (the tensor-core split engine); else FC_ERR_UNSUPPORTED.  Replaces nothing in the
 * reference (single-process); the rows it computes equal fc_conv_forward's. */
int fc_conv_forward_rows(int64_t n, int c_in, int d, int k, int c_out, const void *features,
                         const void *locations, const int32_t *neighbors, const void *theta,
                         const void *theta_b, const int32_t *rows, int64_t nrows, void *out,
                         void *stream);
int fc_deconv_forward(int dtype, int mode, int64_t batch, int64_t n, int c_in, int d, int k,
                      int c_out, const void *x, const void *locations,
                      const int32_t *rev_offsets, const int32_t *rev_entries,
                      const void *theta, const void *theta_b, void *y, void *stream);

/* ---- reverse neighbourhood ---------------------------------------------------------
 * Bucket g = b*N + neighbors[e] collects the forward slots e = p*k + s, ascending
 * (the fixed i-order of the reference's serial scatter, _native.pyx:93-127).
 * offsets [B*N + 1], entries [B*N*k].  Validates indices (FC_ERR_INDEX). */
int fc_csr_build(int64_t batch, int64_t n, int k, const int32_t *neighbors,
                 int32_t *offsets, int32_t *entries, void *stream);
/* The same build without the host synchronisation of the index check: *bad (device int32,
 * caller-zeroed) receives the number of out-of-range entries.  Stream-ordered and
 * CUDA-graph capturable; used where the table is valid by construction (fc_knn output) or
 * was range-checked already (fc_check_indices when the neighbourhood was created). */
int fc_csr_build_async(int64_t batch, int64_t n, int k, const int32_t *neighbors,
                       int32_t *offsets, int32_t *entries, int32_t *bad, void *stream);

/* ---- flex_pool (neighbourhood max-pool) --------------------------------------------
 * Replaces _native.max_pool_forward (_native.pyx:130-155) behind flexops.flex_max_pool
 * (flexops.py:135-151).  argmax [B*N, c] holds the winning CLOUD-LOCAL index; ties go to
 * the lowest index (_native.pyx:151). */
int fc_pool_forward(int dtype, int64_t batch, int64_t n, int c, int k, const void *features,
                    const int32_t *neighbors, void *out, int32_t *argmax, void *stream);

/* Pool backward through the reverse neighbourhood (argmax always lies in N(i)):
 * d_f[j,c] = sum over i in R(j), ascending, of [argmax[i,c]==j] * g[i,c] -- the same
 * additions in the same order as _native.max_pool_backward (_native.pyx:158-168). */
int fc_pool_backward(int dtype, int64_t batch, int64_t n, int c, int k, const void *upstream,
                     const int32_t *argmax, const int32_t *rev_offsets,
                     const int32_t *rev_entries, void *d_features, void *stream);

/* Record-only pool backward, the exact flexops.flex_max_pool_backward(upstream, record, n)
 * contract (flexops.py:154-165): record [n_up, c] indexes rows [0, n_rows).
 * fc_record_csr_build groups slots e = i*c + ch by (record[e], ch): offsets
 * [n_rows*c + 1], entries [n_up*c]; fc_pool_backward_record then sums in ascending i. */
int fc_record_csr_build(int64_t n_up, int64_t n_rows, int c, const int32_t *record,
                        int32_t *offsets, int32_t *entries, void *stream);
int fc_pool_backward_record(int dtype, int64_t n_up, int64_t n_rows, int c,
                            const void *upstream, const int32_t *offsets,
                            const int32_t *entries, void *d_features, void *stream);

/* ---- kNN neighbourhood builder ------------------------------------------------------
 * Exact self-kNN: row i = [i, the k-1 nearest other points ordered by (d^2, index)],
 * d^2 evaluated in fp64 left-to-right over the d coordinates without FMA -- the
 * contract of knn_query / knn_brute_force (neighborhood.py:149-187, _native.pyx:171-255).
 * points [B*N, d] (dtype), out [B*N, k] int32 cloud-local.  algo: FC_KNN_*.
 * The grid path (d <= 3) reads each cloud's bounding box to the host once. */
int fc_knn(int dtype, int64_t batch, int64_t n, int d, int k, const void *points,
           int32_t *out, int algo, void *stream);

/* Cell-ordered (spatially coherent) permutation of one cloud: order[q] = point index.
 * Permutation equivariance (tests/test_flexops.py:263-276) makes any relabelling legal. */
int fc_spatial_order(int dtype, int64_t n, int d, const void *points, int32_t *order,
                     void *stream);

/* Inverse density of the IDISS sampler: phi[i] = sum over neighbour row i of |l_i - l_j|
 * (sampling.py:33-48), fp64 in the reference's numpy evaluation order (bitwise equal).
 * points [n, d] fp64, neighbors [n, k] int32 (k <= 128), phi [n] fp64. */
int fc_inverse_density(int64_t n, int d, int k, const double *points, const int32_t *neighbors,
                       double *phi, void *stream);

/* ---- row movement used by the pooling stage (flexops.py:168-203) --------------------- */
/* out[r] = in[sel[r]] -- downsample_gather (flexops.py:168-175). */
int fc_gather_rows(int dtype, int64_t rows_out, int c, const void *in, const int32_t *sel,
                   void *out, void *stream);
/* out = 0; out[sel[r]] = in[r], last writer wins on duplicate targets -- scatter_to_fine
 * (flexops.py:178-190). */
int fc_scatter_rows(int dtype, int64_t rows_in, int64_t rows_out, int c, const void *in,
                    const int32_t *sel, void *out, void *stream);

/* ---- fused downsample / upsample pooling (network.py:248-280 _PoolDown / _Upsample,
 * flexops.py:168-203 downsample_gather / flex_upsample), one cloud, without the fine-level
 * intermediates (the pooled map of every fine point, the zero-filled scattered map):
 * fc_selection_owner     owner[0..n) = -1, then owner[sel[r]] = r (largest r on duplicate
 *                        targets: scatter_to_fine's last-writer rule).
 * fc_pool_select_forward out row r (of m) pools fine row p = rows ? rows[r] : r over its
 *                        neighbours j = neighbors[p*k + s]; neighbour j's value is
 *                        owner ? (owner[j] >= 0 ? features[owner[j]] : 0) : features[j];
 *                        winners [m, c] = the fine index j, ties to the lower j (_native.pyx:151).
 *                        PoolDown: rows = selection, owner = NULL.  Upsample: rows = NULL, owner = map.
 * fc_pool_select_backward d_features row r (of m) is fine row j = rows ? rows[r] : r: the sum,
 *                        over j's reverse entries (i, s) ascending (each i once), of
 *                        upstream[q, ch] with q = owner ? owner[i] : i (none if q < 0) and
 *                        winners[q, ch] == j -- flexops.flex_max_pool_backward's additions
 *                        (_native.pyx:165-168) restricted to rows that can be non-zero.
 *                        PoolDown: rows = NULL, owner = map.  Upsample: rows = selection, owner = NULL. */
int fc_selection_owner(int64_t m, int64_t n, const int32_t *sel, int32_t *owner, void *stream);
int fc_pool_select_forward(int dtype, int64_t m, int64_t n, int c, int k, const void *features,
                           const int32_t *neighbors, const int32_t *rows, const int32_t *owner,
                           void *out, int32_t *winners, void *stream);
int fc_pool_select_backward(int dtype, int64_t m, int64_t n, int c, int k, const void *upstream,
                            const int32_t *winners, const int32_t *rev_offsets,
                            const int32_t *rev_entries, const int32_t *rows, const int32_t *owner,
                            void *d_features, void *stream);

/* ---- index plumbing --------------------------------------------------------------------
 * int64 -> int32 narrowing with a device-side range check: *bad (device int32) receives
 * the number of entries outside [0, hi) (the reference's idx.min()/max() scan,
 * flexops.py:92-93).  fc_check_indices does the same on an int32 table.  If `row_len` > 0
 * the bound is per cloud: entry e belongs to cloud e / (n_per_cloud*row_len). */
int fc_indices_to_i32(const int64_t *in, int32_t *out, int64_t count, int64_t hi,
                      int32_t *bad, void *stream);
/* *bad (device int32, caller-zeroed) += number of NaN / +-inf entries of x[0..count): the
 * reference's np.isfinite(...).all() checks (network.py:391-396, flexops.py:38-39) on the device. */
int fc_count_nonfinite(int dtype, const void *x, int64_t count, int32_t *bad, void *stream);
int fc_check_indices(const int32_t *idx, int64_t count, int64_t hi, int32_t *bad,
                     void *stream);

/* flex_deconv backward (gradient of y = A(theta)^T x): upstream gy [B*N, c_in] ->
 * d_x = A(theta) gy [B*N, c_out] (a flex_conv forward), d_theta / d_theta_b / d_locations =
 * flex_conv backward with upstream = x and features = gy.  Nullable outputs are skipped.
 * (The reference has no flex_deconv; this is the adjoint's exact gradient.) */
int fc_deconv_backward(int dtype, int mode, int64_t batch, int64_t n, int c_in, int d, int k,
                       int c_out, const void *upstream, const void *x, const void *locations,
                       const int32_t *neighbors, const int32_t *rev_offsets,
                       const int32_t *rev_entries, const void *theta, const void *theta_b,
                       void *d_x, void *d_locations, void *d_theta, void *d_theta_b, void *stream);

/* Workspace (SURVEY.md §8(b) workspace_bytes): every entry point takes its scratch from the
 * device's stream-ordered memory pool; fc_scratch_peak_bytes() is the high-water mark (bytes)
 * of that scratch for calls made on this host thread since fc_scratch_peak_reset(). */
int64_t fc_scratch_peak_bytes(void);
void fc_scratch_peak_reset(void);

/* ---- pointwise (1x1) convolutions of the U-Net step: replace the
 * reference's pointwise_conv (flexops.py:206-226) and the concatenations that feed it
 * (network.py:94-122, 180-246).  fp32, tcgen05 kind::tf32 with hi/lo split operands.
 *
 * fc_gemm_pack_b: pack B [nrows x K] (K = the concatenation of nseg column segments
 *   (seg_src[s] .. + seg_k[s]) of w, each padded to 32 columns; transpose = 1 reads w^T)
 *   into the tensor-core image `img` of fc_gemm_image_bytes(nrows, kblocks) bytes,
 *   kblocks = sum ceil(seg_k / 32).
 * fc_gemm_rows: Y = bias + [A_0 | ... | A_{nops-1}] . B^T for n rows; A_q row-major
 *   [n x ka[q]] (row stride lda[q]); operand 0 optionally masked by (mask > 0) (the
 *   ReLU of a saved pre-activation); column range [c0[o], c1[o]) of Y written to out[o]
 *   (row stride ld[o]); relu_out (nullable) receives max(Y, 0).
 * fc_gemm_wgrad: dw [co x sum kx] = G^T [X_0 | ...], db [co] = column sums of G (G
 *   optionally masked); deterministic (fixed-order partial sums).  dw / db nullable. */
int64_t fc_gemm_image_bytes(int ncols, int kblocks);
int fc_gemm_pack_b(int transpose, int nrows, int nseg, const int *seg_src, const int *seg_k,
                   const float *w, int64_t ldw, uint8_t *img, void *stream);
int fc_gemm_rows(int64_t n, int nops, const float *const *a, const int64_t *lda, const int *ka,
                 const float *mask, int64_t mask_ld, const uint8_t *img, int ncols,
                 const float *bias, int nouts, float *const *out, const int64_t *ld,
                 const int *c0, const int *c1, float *relu_out, int64_t relu_ld, void *stream);
int fc_gemm_wgrad(int64_t n, const float *g, int64_t ldg, const float *mask, int64_t mask_ld,
                  int co, int nops, const float *const *x, const int64_t *ldx, const int *kx,
                  float *dw, float *db, void *stream);

/* ---- ReLU gradient of the U-Net blocks (the reference's tf.nn.relu inside its residual and
 * merge blocks, network.py:404-416 / :261-280) in one pass: out[i] = g[i] * (z[i] > 0 ? 1 : 0)
 * (+ add[i] when add is non-null) -- the arithmetic of `g * (z > 0) + add`; n elements of
 * dtype FC_F32 / FC_F64; out may alias g. */
int fc_relu_backward(int dtype, int64_t n, const void *g, const void *z, const void *add, void *out,
                     void *stream);

#ifdef __cplusplus
}
#endif

#endif /* FLEXCONV_B200_H */
