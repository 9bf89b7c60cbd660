// fc_common.cuh -- shared helpers for the flex-convolution sm_100a kernels.
//
// Layout contract: every tensor is point-major
// ([B*N, D] row-major, one point's D channels contiguous), B clouds of N points
// each stacked along the point axis; neighbour tables are [B*N, K] int32 holding
// CLOUD-LOCAL indices (the reference's NeighborIndex rows, neighborhood.py:54-71),
// so global row = b*N + local.  Offsets are centre - neighbour (l_i - l_j), as the
// reference computes them (_native.pyx:55).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "../../include/flexconv_b200.h"

namespace fc {

int set_error(int code, const char *fmt, ...);
int check_launch(const char *what);

constexpr int kMaxDp = 8;  // spatial dimensions handled by the templated kernels

// Arithmetic policy per scalar type.
//  float : fused multiply-add (the fast fp32 path; parity is tolerance-based).
//  double: separately rounded multiply and add, the same operations in the same
//          order as the reference's non-contracted C (gcc -O3, x86-64, no FMA), so
//          the fp64 forward/pool results are bitwise identical to _native.
template <typename T>
struct Ar;
template <>
struct Ar<float> {
    static __device__ __forceinline__ float madd(float acc, float a, float b) { return fmaf(a, b, acc); }
    static __device__ __forceinline__ float add(float a, float b) { return a + b; }
    static __device__ __forceinline__ float sub(float a, float b) { return a - b; }
    static __device__ __forceinline__ float mul(float a, float b) { return a * b; }
};
template <>
struct Ar<double> {
    static __device__ __forceinline__ double madd(double acc, double a, double b) {
        return __dadd_rn(acc, __dmul_rn(a, b));
    }
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
};

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

inline int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

// Per-device one-time set-up (kernel attributes, pool configuration): `mask` holds one bit
// per device ordinal; returns true the first time it is called on the current device.
// (Launches go to the caller's current device, so per-process flags would leave a second
// GPU driven from the same process without its >48 KB shared-memory attributes.)
inline bool first_use_on_device(uint64_t &mask) {
    const int dev = current_device() & 63;
    const uint64_t bit = 1ull << dev;
    if (__atomic_fetch_or(&mask, bit, __ATOMIC_ACQ_REL) & bit) return false;
    return true;
}

inline int num_sms() {
    static int sms[64] = {0};
    const int dev = current_device() & 63;
    if (sms[dev] <= 0) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
        sms[dev] = v;
    }
    return sms[dev];
}

// Reverse (transposed) neighbourhood in CSR form: for global point j,
// entries[off[j] .. off[j+1]) hold flat forward slots e = p*K + s with
// nbr[e] == j (cloud-local), sorted ascending -> ascending (i, s), the order in
// which the reference's serial backward visits them (_native.pyx:93-120).
struct Csr {
    const int32_t *off;
    const int32_t *ent;
};

// Bucket function of the stable counting-sort CSR builder (pool_csr.cu):
// mode 0 (NBR)   : key = neighbour table entry, bucket = (e / (n*k)) * n + key, key < n
// mode 1 (RECORD): key = record entry,          bucket = key * k + e % k,        key < n
// mode 2 (DIRECT): key is the bucket id,                                          key < n
struct BucketFn {
    int mode;
    int64_t n;
    int k;
    __device__ __forceinline__ int64_t operator()(int64_t e, int32_t key) const {
        if (mode == 0) return (e / (n * k)) * n + key;
        if (mode == 1) return (int64_t)key * k + (e % k);
        return key;
    }
};

int build_csr(const int32_t *keys, int64_t count, BucketFn bf, int64_t buckets, int32_t *off,
              int32_t *ent, int32_t *bad_dev, cudaStream_t st);
void *scratch_alloc(size_t bytes, cudaStream_t st);
void scratch_free(void *p, cudaStream_t st);

// RAII stream-ordered scratch: released (stream-ordered) on every return path, so an early
// error return can neither leak nor hand a kernel a null pointer unnoticed (check `ok()`).
struct Scratch {
    void *p = nullptr;
    cudaStream_t st = nullptr;
    Scratch() = default;
    Scratch(size_t bytes, cudaStream_t s) : p(scratch_alloc(bytes, s)), st(s) {}
    ~Scratch() { scratch_free(p, st); }
    Scratch(const Scratch &) = delete;
    Scratch &operator=(const Scratch &) = delete;
    void alloc(size_t bytes, cudaStream_t s) {
        scratch_free(p, st);
        st = s;
        p = scratch_alloc(bytes, s);
    }
    template <typename T>
    T *as() const { return static_cast<T *>(p); }
    bool ok() const { return p != nullptr; }
};
void count_launch();
// per-kernel event timing (fc_profile_*); no-ops unless enabled
void prof_begin(const char *name, cudaStream_t st);
void prof_end(cudaStream_t st);

}  // namespace fc
