// Groundwork: tcgen05.mma kind::f16 with the A operand in TENSOR MEMORY
// (the "TS" form) -- checks the TMEM layout of A: row m in TMEM lane m, K packed two fp16 per
// 32-bit column (element k in column k/2, low half = even k), 8 columns per K = 16 step --
// against a host GEMM.  M = 128, N = 64, K = 64; A written with tcgen05.st by the thread that
// owns the lane (warp w -> lanes 32w..32w+31), B K-major SW128 in shared memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o mma_ts_check mma_ts_check.cu && ./mma_ts_check
#include <cuda_fp16.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../../paper_1803_07289_b200/csrc/sm100.cuh"
using namespace fc::sm100;

constexpr int M = 128, N = 64, K = 64;

__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                       uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
        : "memory");
}

__global__ void k(const __half *A, const __half *B, float *D, int swap_halves) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t *sm = (uint8_t *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *Bs = sm;  // N rows x 128 B (one K-block of 64)
    uint64_t *bar = (uint64_t *)(sm + N * 128);
    uint32_t *holder = (uint32_t *)(bar + 1);
    for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
        const int n = e / K, kk = e % K;
        *(__half *)(Bs + sw128_offset(n, kk, N)) = B[n * K + kk];
    }
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) tmem_alloc(holder, 128);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = *holder;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = warp * 32 + lane;
    // A row m -> TMEM lane m, columns 0..31 (two fp16 per column)
    uint32_t r[32];
    for (int c = 0; c < 32; ++c) {
        const uint16_t lo = __half_as_ushort(A[m * K + 2 * c]), hi = __half_as_ushort(A[m * K + 2 * c + 1]);
        r[c] = swap_halves ? ((uint32_t)lo << 16 | hi) : ((uint32_t)hi << 16 | lo);
    }
    const uint32_t a_taddr = tb + ((uint32_t)(warp * 32) << 16);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(a_taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t d_tmem = tb + 64;  // columns 64..127
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = idesc_f16(M, N, 0);
        for (int s = 0; s < K / 16; ++s)
            mma_ts(d_tmem, tb + 8 * s, desc_sw128(smem_u32(Bs) + 32 * s), idesc, s > 0 ? 1u : 0u);
        mma_commit(bar);
    }
    mbar_wait(bar, 0);
    tc_fence_after();
    for (int c0 = 0; c0 < N; c0 += 16) {
        float v[16];
        tmem_ld16(d_tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
        for (int j = 0; j < 16; ++j) D[m * N + c0 + j] = v[j];
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tb, 128);
}

int main() {
    __half *hA = (__half *)malloc(M * K * 2), *hB = (__half *)malloc(N * K * 2);
    float *ref = (float *)malloc(M * N * 4), *hD = (float *)malloc(M * N * 4);
    srand(1);
    float fa[M * K], fb[N * K];
    for (int i = 0; i < M * K; ++i) fa[i] = (float)(rand() % 17 - 8), hA[i] = __float2half(fa[i]);
    for (int i = 0; i < N * K; ++i) fb[i] = (float)(rand() % 13 - 6), hB[i] = __float2half(fb[i]);
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int kk = 0; kk < K; ++kk) s += (double)fa[m * K + kk] * fb[n * K + kk];
            ref[m * N + n] = (float)s;
        }
    __half *dA, *dB;
    float *dD;
    cudaMalloc(&dA, M * K * 2);
    cudaMalloc(&dB, N * K * 2);
    cudaMalloc(&dD, M * N * 4);
    cudaMemcpy(dA, hA, M * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, N * K * 2, cudaMemcpyHostToDevice);
    const int smem = N * 128 + 64 + 1024;
    for (int swap = 0; swap < 2; ++swap) {
        cudaMemset(dD, 0, M * N * 4);
        k<<<1, 128, smem>>>(dA, dB, dD, swap);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
        double err = 0;
        for (int i = 0; i < M * N; ++i) err = fmax(err, fabs(hD[i] - ref[i]));
        printf("A-in-TMEM layout %s (k even in the %s half): max |D - ref| = %g  [%s]\n",
               swap ? "swapped" : "natural", swap ? "high" : "low", err, cudaGetErrorString(e));
    }
    return 0;
}
