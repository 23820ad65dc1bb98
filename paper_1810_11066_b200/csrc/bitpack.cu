// bitpack.cu — bit-plane packing kernel.
//
// PAPER.md:519-523 (Sec. 2.2): "splitting input vectors into individual bitplanes
// ... The binary vectors are then packed data into a larger storage type such as a
// uint32"; PAPER.md:555-567 (Sec. 3.1): d-dim tensor -> (d+1)-dim packed tensor with
// a new bit axis, packed along the reduction axis; layout BMK' (bit axis outermost).
//
// in  : uint8 codes [rows][k] (row-major; reduction axis innermost)
// out : uint32 [bits][rows][kwp], kwp = bs_packed_row_words(k); bit t of word j of
//       plane b = bit b of in[r][32 j + t]; bits at index >= k are 0.
//
// One thread produces word j of every plane for one row: it reads the 32 codes of
// that word (two 16-byte loads on the aligned path, so a warp streams 1 KiB of
// contiguous input) and writes `bits` words, each store coalesced across the warp.
// HBM-bound: 1 byte read + bits/8 bytes written per element.
#include "common.cuh"
#include "kernels.h"

namespace bs {

template <int BITS>
__global__ void __launch_bounds__(256) bitpack_kernel(const uint8_t* __restrict__ in, uint32_t* __restrict__ out,
                                                      int64_t rows, int64_t k, int64_t kwp, int bits_rt,
                                                      bool aligned16) {
  const int bits = BITS > 0 ? BITS : bits_rt;
  const int64_t tasks = rows * kwp;
  const int64_t plane_stride = rows * kwp;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tasks; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / kwp, j = t - r * kwp;
    const int64_t e0 = 32 * j;  // first element of this word
    uint32_t v[8];
    const uint8_t* src = in + r * k + e0;
    if (aligned16 && e0 + 32 <= k) {
      uint4 lo = __ldg(reinterpret_cast<const uint4*>(src));
      uint4 hi = __ldg(reinterpret_cast<const uint4*>(src) + 1);
      v[0] = lo.x; v[1] = lo.y; v[2] = lo.z; v[3] = lo.w;
      v[4] = hi.x; v[5] = hi.y; v[6] = hi.z; v[7] = hi.w;
    } else if (aligned16 && e0 + 16 == k) {  // k % 32 == 16: last word half full
      uint4 lo = __ldg(reinterpret_cast<const uint4*>(src));
      v[0] = lo.x; v[1] = lo.y; v[2] = lo.z; v[3] = lo.w;
      v[4] = v[5] = v[6] = v[7] = 0u;
    } else {  // ragged / unaligned rows, pad words: byte loads with bounds
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint32_t x = 0;
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          int64_t e = e0 + 4 * q + rr;
          if (e < k) x |= uint32_t(__ldg(src + 4 * q + rr)) << (8 * rr);
        }
        v[q] = x;
      }
    }
    uint32_t* dst = out + r * kwp + j;
#pragma unroll
    for (int b = 0; b < (BITS > 0 ? BITS : 8); ++b) {
      if (BITS == 0 && b >= bits) break;
      dst[b * plane_stride] = plane_word(v, b);
    }
  }
}

cudaError_t launch_bitpack(const uint8_t* in, uint32_t* out, int64_t rows, int64_t k, int64_t kwp, int bits,
                           cudaStream_t stream) {
  const int64_t tasks = rows * kwp;
  const int threads = 256;
  int64_t blocks = (tasks + threads - 1) / threads;
  const int64_t max_blocks = int64_t(kNumSMs) * 8 * 4;  // grid-stride beyond 4 waves of 8 CTAs/SM
  if (blocks > max_blocks) blocks = max_blocks;
  const bool aligned16 = (reinterpret_cast<uintptr_t>(in) % 16 == 0) && (k % 16 == 0);
  switch (bits) {
    case 1: bitpack_kernel<1><<<blocks, threads, 0, stream>>>(in, out, rows, k, kwp, bits, aligned16); break;
    case 2: bitpack_kernel<2><<<blocks, threads, 0, stream>>>(in, out, rows, k, kwp, bits, aligned16); break;
    case 3: bitpack_kernel<3><<<blocks, threads, 0, stream>>>(in, out, rows, k, kwp, bits, aligned16); break;
    case 4: bitpack_kernel<4><<<blocks, threads, 0, stream>>>(in, out, rows, k, kwp, bits, aligned16); break;
    default: bitpack_kernel<0><<<blocks, threads, 0, stream>>>(in, out, rows, k, kwp, bits, aligned16); break;
  }
  note_launch();
  return cudaPeekAtLastError();
}

}  // namespace bs
