// Does the proxy fence (fence.proxy.async.shared::cta -> MEMBAR.ALL.CTA + FENCE.VIEW.ASYNC.S)
// wait for the thread's OUTSTANDING GLOBAL LOADS?  Issue 8 independent L2-missing loads, then
// (mode 1) the fence or (mode 0) nothing, read the clock, then consume the loads.  If the fence
// drains loads, the clock read after it includes the load latency.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o membar_loads membar_loads.cu && ./membar_loads
#include <cstdio>
#include <cstdint>

__global__ void k(const float *__restrict__ big, int stride, int mode, long long *out, float *sink) {
    const float *p = big + (size_t)(blockIdx.x * 32 + threadIdx.x) * 64;
    float v[8], s0;
    long long t0 = clock64();
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(p + (size_t)u * stride);
    __shared__ float sh[64];
    if (mode == 1) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (mode == 2) asm volatile("membar.cta;" ::: "memory");
    sh[threadIdx.x] = 1.f;  // a later memory instruction: blocked if the fence waits for the loads
    long long t1 = clock64();
    s0 = sh[(threadIdx.x + 1) & 31];
    float s = s0;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
    long long t2 = clock64();
    if (threadIdx.x == 0) {
        out[blockIdx.x * 2] = t1 - t0;
        out[blockIdx.x * 2 + 1] = t2 - t0;
    }
    sink[blockIdx.x * 32 + threadIdx.x] = s;
}

int main() {
    const size_t n = (size_t)1 << 28;  // 1 GB: beyond L2
    float *big, *sink;
    long long *out, h[2];
    cudaMalloc(&big, n * 4);
    cudaMemset(big, 0, n * 4);
    cudaMalloc(&sink, 1 << 20);
    cudaMalloc(&out, 1 << 20);
    const char *names[3] = {"no fence", "fence.proxy.async", "membar.cta"};
    for (int mode = 0; mode < 3; ++mode) {
        double a = 0, b = 0;
        for (int rep = 0; rep < 20; ++rep) {
            k<<<1, 32>>>(big + (size_t)rep * (1 << 22), 1 << 20, mode, out, sink);
            cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
            a += h[0];
            b += h[1];
        }
        printf("%-18s  clocks to after-fence: %7.0f   to loads consumed: %7.0f\n", names[mode], a / 20, b / 20);
    }
    return 0;
}
