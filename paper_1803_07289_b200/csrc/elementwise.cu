// ReLU gradient of the U-Net blocks in one pass (the gradient of the reference's tf.nn.relu
// inside its residual / merge blocks, network.py:404-416 and :261-280):
//   out = g * (z > 0 ? 1 : 0) [+ add]
// exactly the arithmetic of `g * (z > 0)` followed by `+ add` (a multiply by 1 or 0, so
// NaN / -0 propagate as they do there), replacing a compare, a multiply and an add pass
// (and a bool temporary) over [points, channels] tensors.  out may alias g.
#include <cstdint>

#include "fc_common.cuh"

namespace fc {
namespace {

template <typename T>
__device__ __forceinline__ T relu_grad1(T g, T z, const T *add, int64_t i) {
    T v = g * (z > T(0) ? T(1) : T(0));
    if (add) v = v + add[i];
    return v;
}

template <typename T>
__global__ void relu_grad_kernel(int64_t n, const T *__restrict__ g, const T *__restrict__ z,
                                 const T *__restrict__ add, T *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = relu_grad1(g[i], z[i], add, i);
}

// fp32, every pointer 16-byte aligned: four elements per thread and load
__global__ void relu_grad4_kernel(int64_t n4, const float4 *__restrict__ g, const float4 *__restrict__ z,
                                  const float4 *__restrict__ add, float4 *out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 gv = g[i], zv = z[i];
        float4 v = make_float4(gv.x * (zv.x > 0.f ? 1.f : 0.f), gv.y * (zv.y > 0.f ? 1.f : 0.f),
                               gv.z * (zv.z > 0.f ? 1.f : 0.f), gv.w * (zv.w > 0.f ? 1.f : 0.f));
        if (add) {
            const float4 a = add[i];
            v = make_float4(v.x + a.x, v.y + a.y, v.z + a.z, v.w + a.w);
        }
        out[i] = v;
    }
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace
}  // namespace fc

using namespace fc;

extern "C" int fc_relu_backward(int dtype, int64_t n, const void *g, const void *z, const void *add, void *out,
                                void *stream) {
    if (n < 0) return set_error(FC_ERR_SHAPE, "relu_backward: n < 0");
    if (n == 0) return FC_OK;
    if (!g || !z || !out) return set_error(FC_ERR_CONFIG, "relu_backward: null tensor");
    cudaStream_t st = (cudaStream_t)stream;
    const int threads = 256;
    if (dtype == FC_F32) {
        const bool vec = (n & 3) == 0 && aligned16(g) && aligned16(z) && aligned16(out) && (!add || aligned16(add));
        if (vec) {
            const int64_t n4 = n >> 2;
            const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(n4, threads), 8 * num_sms());
            relu_grad4_kernel<<<blocks, threads, 0, st>>>(n4, (const float4 *)g, (const float4 *)z, (const float4 *)add,
                                                          (float4 *)out);
        } else {
            const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(n, threads), 8 * num_sms());
            relu_grad_kernel<float><<<blocks, threads, 0, st>>>(n, (const float *)g, (const float *)z, (const float *)add,
                                                                (float *)out);
        }
    } else if (dtype == FC_F64) {
        const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(n, threads), 8 * num_sms());
        relu_grad_kernel<double><<<blocks, threads, 0, st>>>(n, (const double *)g, (const double *)z,
                                                             (const double *)add, (double *)out);
    } else {
        return set_error(FC_ERR_CONFIG, "relu_backward: bad dtype %d", dtype);
    }
    count_launch();
    return check_launch("relu_backward");
}
