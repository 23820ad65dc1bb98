// popc_conv.cu — dispatch of the tiled AND+POPC implicit-GEMM conv/dense kernel
// (kernel: popc_conv_impl.cuh) over bit widths and encodings.
//
// Compile-time widths cover the limit-study grid A, W in 1..4;
// the literal two-popcount bipolar variant is built for the BASELINE widths (A1W1,
// A2W1, A2W2); every other combination runs the runtime-width instantiation.
#include "popc_conv_impl.cuh"

namespace bs {

cudaError_t popc_conv_a1(const ConvProblem& p, bool lit, cudaStream_t s);
cudaError_t popc_conv_a2(const ConvProblem& p, bool lit, cudaStream_t s);
cudaError_t popc_conv_a3(const ConvProblem& p, bool lit, cudaStream_t s);
cudaError_t popc_conv_a4(const ConvProblem& p, bool lit, cudaStream_t s);

cudaError_t launch_popc_conv(const ConvProblem& p, Algo algo, cudaStream_t stream) {
  const bool lit = algo == Algo::PopcLit && p.bipolar;
  if (p.w_bits >= 1 && p.w_bits <= 4) {
    cudaError_t e = cudaErrorNotSupported;
    switch (p.a_bits) {
      case 1: e = popc_conv_a1(p, lit, stream); break;
      case 2: e = popc_conv_a2(p, lit, stream); break;
      case 3: e = popc_conv_a3(p, lit, stream); break;
      case 4: e = popc_conv_a4(p, lit, stream); break;
      default: break;
    }
    if (e != cudaErrorNotSupported) return e;
  }
  return lit ? popc_detail::launch_tile<0, 0, true>(p, stream) : popc_detail::launch_tile<0, 0, false>(p, stream);
}

}  // namespace bs
