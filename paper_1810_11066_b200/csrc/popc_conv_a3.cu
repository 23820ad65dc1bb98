// popc_conv_a3.cu — instantiations of the AND+POPC conv kernel for a_bits = 3
// (split per a_bits so nvcc compiles them in parallel; see popc_conv_impl.cuh).
#include "popc_conv_impl.cuh"

namespace bs {

cudaError_t popc_conv_a3(const ConvProblem& p, bool lit, cudaStream_t s) {
  switch (p.w_bits) {
    case 1: return lit ? cudaErrorNotSupported : popc_detail::launch_tile<3, 1, false>(p, s);
    case 2: return lit ? cudaErrorNotSupported : popc_detail::launch_tile<3, 2, false>(p, s);
    case 3: return lit ? cudaErrorNotSupported : popc_detail::launch_tile<3, 3, false>(p, s);
    case 4: return lit ? cudaErrorNotSupported : popc_detail::launch_tile<3, 4, false>(p, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace bs
