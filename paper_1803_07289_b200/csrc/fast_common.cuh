// fast_common.cuh -- device helpers shared by the warp-specialised flex-conv kernels
// (conv_fast.cu forward, conv_fast_rev.cu reverse / adjoint): packed fp32x2 arithmetic,
// shared / global vector accesses, the fp32-accurate fp16 hi/lo split, row scales.
#pragma once

#include "fc_common.cuh"
#include "sm100.cuh"

namespace fc {
namespace fast {
using namespace sm100;

constexpr int kTile = 128;

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
// 32 lanes x 8 columns of 32-bit (thread t <- TMEM lane quadrant*32 + t)
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
// 32-byte (one sector) store per thread: STG.E.ENL2.256
__device__ __forceinline__ void stg256(float *p, const float *v) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]),
                 "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}
__device__ __forceinline__ void sts64(uint32_t addr, uint32_t lo, uint32_t hi) {
    asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(lo), "r"(hi) : "memory");
}
__device__ __forceinline__ void sts128f(uint32_t addr, float a, float b, float c, float d) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
__device__ __forceinline__ void sts8(uint32_t addr, int v) {
    asm volatile("st.shared.b8 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t lds32(uint32_t addr) {
    int32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ float4 lds128f(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ float4 ldg_nc4(const float *p) {
    float4 v;
    asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ int4 ldg_nc4i(const int32_t *p) {
    int4 v;
    asm volatile("ld.global.nc.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// fp32-accurate split of a scaled pair into fp16 hi + lo (block floating point): with
// |v*sc| < 2^15, hi = v*sc rounded to a multiple of 16 (exact in fp16: <= 11 significant
// bits) via the 1.5*2^27 magic constant, lo = v*sc - hi (exact in fp32, |lo| <= 8) rounded
// to fp16: |error| <= 2^-9 against a row maximum >= 2^14, i.e. 2^-23 of the row scale.
__device__ __forceinline__ uint32_t split2(float2 v, float sc, uint32_t &lo_out) {
    const float2 s2 = make_float2(sc, sc);
    const float2 C = make_float2(201326592.f, 201326592.f), nC = make_float2(-201326592.f, -201326592.f);
    const float2 hi = fadd2(ffma2(v, s2, C), nC);
    const float2 lo = ffma2(v, s2, make_float2(-hi.x, -hi.y));
    const __half2 H = __floats2half2_rn(hi.x, hi.y);
    const __half2 Lh = __floats2half2_rn(lo.x, lo.y);
    lo_out = *reinterpret_cast<const uint32_t *>(&Lh);
    return *reinterpret_cast<const uint32_t *>(&H);
}
__device__ __forceinline__ uint32_t bf16x2(float2 v) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(v.x, v.y);
    return *reinterpret_cast<const uint32_t *>(&h);
}

// exponent e of a power-of-two row scale: scale = 2^-e puts max|v| into [2^14, 2^15)
// (e clamped to [-114, 86] so 2^e and 2^-e stay normal; 0 for an all-zero row)
__device__ __forceinline__ int scale_exp(float m) {
    const int b = (__float_as_int(m) >> 23) & 0xff;  // m >= 0
    if (b == 0 || b == 0xff) return 0;                // zero / subnormal max / inf-nan: no scaling
    return max(-114, min(86, b - 127 - 14));
}
__device__ __forceinline__ float exp2i(int e) { return __int_as_float((127 + e) << 23); }

// One lane's moments: 4 channels x 4 components (m[t][0] = channels 0,1; m[t][1] = 2,3).
struct Mom4 {
    float2 m[4][2];
};

// row of tile item q (0..31), lane group pt: rows {a, a+4, a+1, a+5} (a = 8(q/2) + 2(q%2))
// so that the two points of each half-warp store to disjoint 16-byte chunk sets of the
// SW128 atom
__device__ __forceinline__ int item_row(int q, int pt) { return 8 * (q >> 1) + 2 * (q & 1) + (pt >> 1) + 4 * (pt & 1); }

}  // namespace fast
}  // namespace fc
