// conv_tc.cu -- tcgen05 tensor-core engines (placeholder until the TC kernels land).
#include "fc_common.cuh"

namespace fc {

int tc_conv_forward_supported(int, int, int, int, int) { return 0; }
int tc_conv_forward(int, int64_t, int64_t, int, int, int, int, const float *, const float *,
                    const int32_t *, const float *, const float *, float *, cudaStream_t) {
    return set_error(FC_ERR_UNSUPPORTED, "tensor-core forward not built");
}
int tc_reverse_supported(int, int, int, int) { return 0; }
int tc_reverse_gmc(int, int64_t, int64_t, int, int, int, int, const float *, const float *, Csr,
                   const float *, const float *, float *, cudaStream_t) {
    return set_error(FC_ERR_UNSUPPORTED, "tensor-core reverse not built");
}

}  // namespace fc
