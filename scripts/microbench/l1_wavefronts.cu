// L1TEX data-pipe cost of the gather access shapes used by the kernels (one CTA per SM, an
// L1-resident 16 KB table, loads summed into a sink).  Run under
//   ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_lgds.sum,smsp__inst_executed_op_global_ld.sum
// and divide: wavefronts per load instruction for each mode.
//   mode 0: LDG.256 per lane, 4 lanes per 128-B line, 8 lines per instruction (wide-lane gather)
//   mode 1: LDG.64 per lane, a warp reads one contiguous 256-B row (d_theta gather)
//   mode 2: LDG.128 per lane, 8 lanes per line, 4 lines per instruction
//   mode 3: LDG.32 per lane, 32 lanes scattered over 32 lines (scattered positions)
//   mode 4: LDG.256 per lane, every lane its own line (own-row epilogue access)
//   mode 5: LDS.128 per lane, 8 lanes per 128 B (shared-memory gather for comparison)
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(const float *__restrict__ tab, float *sink, int mode, int iters) {
    __shared__ float sm[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = tab[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float acc = 0.f;
#pragma unroll 8
    for (int it = 0; it < iters; ++it) {
        const int base = ((it * 7 + w * 3) & 15) * 256;  // 16 rows of 256 floats (1 KB each)
        if (mode == 0) {
            const float *p = tab + base + (lane >> 2) * 32 + (lane & 3) * 8;  // 8 lines x 128 B
            float v0, v1, v2, v3, v4, v5, v6, v7;
            asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=f"(v0), "=f"(v1), "=f"(v2), "=f"(v3), "=f"(v4), "=f"(v5), "=f"(v6), "=f"(v7) : "l"(p));
            acc += v0 + v1 + v2 + v3 + v4 + v5 + v6 + v7;
        } else if (mode == 1) {
            const float *p = tab + base + lane * 2;
            float2 v;
            asm volatile("ld.global.nc.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
            acc += v.x + v.y;
        } else if (mode == 2) {
            const float *p = tab + base + lane * 4;
            float4 v;
            asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
            acc += v.x + v.y + v.z + v.w;
        } else if (mode == 3) {
            const float *p = tab + ((base + lane * 32) & 4095);
            float v;
            asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p));
            acc += v;
        } else if (mode == 4) {
            const float *p = tab + ((base + lane * 32) & 4095);
            float v0, v1, v2, v3, v4, v5, v6, v7;
            asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=f"(v0), "=f"(v1), "=f"(v2), "=f"(v3), "=f"(v4), "=f"(v5), "=f"(v6), "=f"(v7) : "l"(p));
            acc += v0 + v1 + v2 + v3 + v4 + v5 + v6 + v7;
        } else {
            const float4 v = reinterpret_cast<const float4 *>(sm)[((base + lane * 4) & 4095) >> 2];
            acc += v.x + v.y + v.z + v.w;
        }
    }
    if (acc == 123.456f) sink[threadIdx.x] = acc;
}

int main() {
    float *tab, *sink;
    cudaMalloc(&tab, 4096 * 4);
    cudaMalloc(&sink, 4096 * 4);
    cudaMemset(tab, 0, 4096 * 4);
    for (int mode = 0; mode < 6; ++mode) {
        k<<<148, 1024>>>(tab, sink, mode, 4096);
        cudaDeviceSynchronize();
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        k<<<148, 1024>>>(tab, sink, mode, 4096);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double instr = 148.0 * 32 * 4096;  // warp-level load instructions
        printf("mode %d: %.3f ms, %.2f SM-cycles per warp load instruction (at 1.965 GHz)\n", mode, ms,
               ms * 1e-3 * 1.965e9 * 148 / instr);
    }
    return 0;
}
