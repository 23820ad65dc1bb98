// tc_conv_group.cu — several tensor-core bitserial convolutions of one precision in one
// persistent launch (bs_bitserial_conv2d_nhwc_tc_group; kernel in tc_conv_impl.cuh).
#include "tc_conv_impl.cuh"

namespace bs {

cudaError_t launch_tc_conv_group(const ConvProblem* ps, const int8_t* const* wexps, int count, int fmt,
                                 cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  const int a_bits = ps[0].a_bits, w_bits = ps[0].w_bits;
  if (!tc_supported(a_bits, w_bits)) return cudaErrorNotSupported;
  for (int q = 1; q < count; ++q)
    if (ps[q].a_bits != a_bits || ps[q].w_bits != w_bits) return cudaErrorInvalidValue;
  const bool f4 = tc_resolve_format(fmt) == kTcF4;
  // members whose filters fit a 64-wide tile run in BN = 64 groups, the rest in BN = 128
  // groups (the tile width pick_bn makes for a single launch)
  for (int wide = 1; wide >= 0; --wide) {
    ConvProblem gp[tc::kGroupMax];
    const int8_t* gw[tc::kGroupMax];
    int cnt = 0;
    for (int q = 0; q <= count; ++q) {
      if (q < count && (tc::pick_bn(ps[q]) == 128) == bool(wide)) {
        gp[cnt] = ps[q];
        gw[cnt++] = wexps[q];
      }
      if (cnt == tc::kGroupMax || (q == count && cnt > 0)) {
        cudaError_t e = cudaErrorNotSupported;
#define BS_TC(A, W, CALL)                                                                          \
  if (a_bits == A && w_bits == W)                                                                  \
    e = wide ? (f4 ? tc::launch_group_aw<A, W, 128, true>(gp, gw, cnt, stream)                     \
                   : tc::launch_group_aw<A, W, 128, false>(gp, gw, cnt, stream))                   \
             : (f4 ? tc::launch_group_aw<A, W, 64, true>(gp, gw, cnt, stream)                      \
                   : tc::launch_group_aw<A, W, 64, false>(gp, gw, cnt, stream));
        BS_TC_DISPATCH(0)
#undef BS_TC
        if (e != cudaSuccess) return e;
        cnt = 0;
      }
    }
  }
  return cudaSuccess;
}
}  // namespace bs
