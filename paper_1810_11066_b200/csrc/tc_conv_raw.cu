// tc_conv_raw.cu — tensor-core bitserial conv2d / dense on PACKED weight planes (the
// three-call boundary's path: bs_bitserial_conv2d_nhwc / bs_bitserial_dense): the producer
// warps expand each weight chunk into its shared-memory B slot (tc_conv_impl.cuh, RAW).
#include "tc_conv_impl.cuh"

namespace bs {

cudaError_t launch_tc_conv_raw(const ConvProblem& p, cudaStream_t stream) {
  if (!tc_supported(p.a_bits, p.w_bits) || p.bipolar > 1 || p.a_enc != 0) return cudaErrorNotSupported;
#define BS_TC(A, W, CALL) \
  if (p.a_bits == A && p.w_bits == W) return tc::launch_raw_aw<A, W>(p, stream);
  BS_TC_DISPATCH(0)
#undef BS_TC
  return cudaErrorNotSupported;
}

}  // namespace bs
