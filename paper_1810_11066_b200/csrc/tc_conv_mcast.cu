// tc_conv_mcast.cu — the tensor-core dense / conv with the NVLS multicast epilogue (the fused
// all-gather's multimem.st form; kernel variant kVarMcast in tc_conv_impl.cuh).
#include "tc_conv_impl.cuh"

namespace bs {

cudaError_t launch_tc_conv_mcast(const ConvProblem& p, const int8_t* wexp, cudaStream_t stream, int32_t* mcast) {
  if (!tc_supported(p.a_bits, p.w_bits)) return cudaErrorNotSupported;
#define BS_TC(A, W, CALL) \
  if (p.a_bits == A && p.w_bits == W) return tc::launch_mcast_aw<A, W>(p, wexp, stream, mcast);
  BS_TC_DISPATCH(0)
#undef BS_TC
  return cudaErrorNotSupported;
}

}  // namespace bs
