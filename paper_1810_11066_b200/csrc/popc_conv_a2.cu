// popc_conv_a2.cu — instantiations of the AND+POPC conv kernel for a_bits = 2
// (split per a_bits so nvcc compiles them in parallel; see popc_conv_impl.cuh).
#include "popc_conv_impl.cuh"

namespace bs {

cudaError_t popc_conv_a2(const ConvProblem& p, bool lit, cudaStream_t s) {
  switch (p.w_bits) {
    case 1: return lit ? popc_detail::launch_tile<2, 1, true>(p, s) : popc_detail::launch_tile<2, 1, false>(p, s);
    case 2: return lit ? popc_detail::launch_tile<2, 2, true>(p, s) : popc_detail::launch_tile<2, 2, false>(p, s);
    case 3: return lit ? cudaErrorNotSupported : popc_detail::launch_tile<2, 3, false>(p, s);
    case 4: return lit ? cudaErrorNotSupported : popc_detail::launch_tile<2, 4, false>(p, s);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace bs
