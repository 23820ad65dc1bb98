// tc_conv.cu — tensor-core bitserial conv2d / dense: single prepared-weight launches, the
// offline weight expansion and the format helpers (kernel template in tc_conv_impl.cuh).
#include "tc_conv_impl.cuh"

namespace bs {
namespace tc {


__global__ void __launch_bounds__(256) expand_weights_kernel(const uint32_t* __restrict__ w_packed,
                                                             int8_t* __restrict__ wexp, int w_bits, int n,
                                                             int64_t kp, int64_t kpad, int w_enc, int c_tap,
                                                             int kw_tap) {
  const int64_t words = int64_t(w_bits) * n * kpad;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < words; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t kk = t % kpad, rest = t / kpad;
    const int64_t row = rest % n, j = rest / n;
    const uint32_t valid = tap_word_mask(kk, kp, c_tap, kw_tap);
    const uint32_t w = kk < kp ? w_packed[(j * n + row) * kp + kk] : 0u;
    const int32_t mag = (1 << j) * plane_sign(int(j), w_bits, w_enc);
    uint32_t out[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {  // byte r of expanded word q = element 8r + q (see expand_word)
      uint32_t v = 0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int e = 8 * r + q;
        const int b = (w >> e) & 1;
        const int32_t val = !((valid >> e) & 1) ? 0 : (w_enc == 1 ? (b ? mag : -mag) : (b ? mag : 0));
        v |= (uint32_t(val) & 0xFFu) << (8 * r);
      }
      out[q] = v;
    }
    uint4* dst = reinterpret_cast<uint4*>(wexp + (j * int64_t(n) + row) * kpad * 32 + kk * 32);
    dst[0] = make_uint4(out[0], out[1], out[2], out[3]);
    dst[1] = make_uint4(out[4], out[5], out[6], out[7]);
  }
}

// FP4 layout: w_packed [W][N][kp] words -> wexp [WD][N][kpad*16] bytes, WD = ceil(W/2)
// radix-4 digits (planes 2e, 2e+1; see digit_nibbles), 16 bytes (4 expanded words of 8
// nibbles) per packed word in the order of expand_word_f4; padding elements are 0;
// digit scale 2^(2e+1) at run time.
__global__ void __launch_bounds__(256) expand_weights_f4_kernel(const uint32_t* __restrict__ w_packed,
                                                                uint8_t* __restrict__ wexp, int w_bits, int n,
                                                                int64_t kp, int64_t kpad, int w_enc, int c_tap,
                                                                int kw_tap) {
  const int wd = (w_bits + 1) / 2;
  const int64_t words = int64_t(wd) * n * kpad;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < words; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t kk = t % kpad, rest = t / kpad;
    const int64_t row = rest % n, e = rest / n;
    const uint32_t valid = tap_word_mask(kk, kp, c_tap, kw_tap);
    const int jlo = int(2 * e), jhi = jlo + 1;
    const bool has_hi = jhi < w_bits;
    const uint32_t wl = kk < kp ? w_packed[(jlo * int64_t(n) + row) * kp + kk] : 0u;
    const uint32_t wh = (has_hi && kk < kp) ? w_packed[(jhi * int64_t(n) + row) * kp + kk] : 0u;
    // mode: 1 bipolar; 2 the digit holding the signed top plane (W-1); else 0
    const int mode = w_enc == 1 ? 1 : (w_enc == 2 && (has_hi ? jhi : jlo) == w_bits - 1 ? 2 : 0);
    uint32_t out[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // nibble r of expanded word q = element 4r + q
      uint32_t L = 0, H = 0, V = 0;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int el = 4 * r + q;
        L |= ((wl >> el) & 1u) << (4 * r);
        H |= ((wh >> el) & 1u) << (4 * r);
        V |= ((valid >> el) & 1u) ? 0xFu << (4 * r) : 0u;
      }
      out[q] = (has_hi ? digit_nibbles<true>(L, H, mode) : digit_nibbles<false>(L, H, mode)) & V;
    }
    *reinterpret_cast<uint4*>(wexp + (e * int64_t(n) + row) * kpad * 16 + kk * 16) =
        make_uint4(out[0], out[1], out[2], out[3]);
  }
}

}  // namespace tc

int tc_resolve_format(int fmt) {
  return fmt == kTcI8 || fmt == kTcF4 ? fmt : kTcDefault;
}

int64_t tc_kpad(int64_t kp, int fmt) {
  const int64_t cw = tc::chunk_words(tc_resolve_format(fmt) == kTcF4);
  return (kp + cw - 1) / cw * cw;
}

int64_t tc_weight_bytes(int64_t n, int64_t kp, int w_bits, int fmt) {
  const bool f4 = tc_resolve_format(fmt) == kTcF4;  // F4: ceil(W/2) radix-4 digits of 16 B per word
  return int64_t(f4 ? (w_bits + 1) / 2 : w_bits) * n * tc_kpad(kp, fmt) * (f4 ? 16 : 32);
}

bool tc_supported(int a_bits, int w_bits) { return a_bits >= 1 && a_bits <= 4 && w_bits >= 1 && w_bits <= 4; }

cudaError_t launch_tc_expand_weights(const uint32_t* w_packed, int w_bits, int w_enc, int64_t n, int64_t kp,
                                     int c_tap, int kw_tap, int8_t* wexp, int fmt, cudaStream_t stream) {
  const int64_t kpad = tc_kpad(kp, fmt);
  const int64_t words = int64_t(w_bits) * n * kpad;
  int64_t blocks = (words + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  if (tc_resolve_format(fmt) == kTcF4)
    tc::expand_weights_f4_kernel<<<unsigned(blocks), 256, 0, stream>>>(w_packed, reinterpret_cast<uint8_t*>(wexp),
                                                                       w_bits, int(n), kp, kpad, w_enc, c_tap,
                                                                       kw_tap);
  else
    tc::expand_weights_kernel<<<unsigned(blocks), 256, 0, stream>>>(w_packed, wexp, w_bits, int(n), kp, kpad,
                                                                    w_enc, c_tap, kw_tap);
  note_launch();
  return cudaPeekAtLastError();
}

cudaError_t launch_tc_conv_prepared(const ConvProblem& p, const int8_t* wexp, int fmt, cudaStream_t stream,
                                    int32_t* const* peers, int npeer, int32_t* mcast) {
  if (!tc_supported(p.a_bits, p.w_bits)) return cudaErrorNotSupported;
  const bool f4 = tc_resolve_format(fmt) == kTcF4;
  if (mcast) return f4 ? launch_tc_conv_mcast(p, wexp, stream, mcast) : cudaErrorNotSupported;
#define BS_TC(A, W, CALL)                                                                 \
  if (p.a_bits == A && p.w_bits == W)                                                     \
    return f4 ? tc::launch_aw<A, W, true>(p, wexp, stream, peers, npeer)                  \
              : tc::launch_aw<A, W, false>(p, wexp, stream, peers, npeer);
  BS_TC_DISPATCH(0)
#undef BS_TC
  return cudaErrorNotSupported;
}


cudaError_t launch_tc_conv(const ConvProblem& p, int8_t* wexp_ws, int fmt, cudaStream_t stream) {
  if (!tc_supported(p.a_bits, p.w_bits)) return cudaErrorNotSupported;
  const int c_tap = p.c_tap, kw_tap = p.kw_a;
  cudaError_t e = launch_tc_expand_weights(p.wt, p.w_bits, p.bipolar, p.oc, p.kp, c_tap, kw_tap, wexp_ws, fmt, stream);
  if (e != cudaSuccess) return e;
  return launch_tc_conv_prepared(p, wexp_ws, fmt, stream);
}

}  // namespace bs
