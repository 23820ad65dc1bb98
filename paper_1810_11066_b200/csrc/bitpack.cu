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
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace bs {

template <int B, int BITS>
__device__ __forceinline__ void store_planes(uint32_t* dst, int64_t plane_stride, const uint32_t (&v)[8]) {
  if constexpr (B < BITS) {
    dst[B * plane_stride] = plane_word_c<B>(v);
    store_planes<B + 1, BITS>(dst, plane_stride, v);
  }
}

// One (row, word) task: 32 codes -> one word per plane.
template <int BITS>
__device__ __forceinline__ void pack_word(const uint8_t* __restrict__ in, uint32_t* __restrict__ out, int64_t r,
                                          int64_t j, int64_t k, int64_t kwp, int64_t plane_stride, int bits,
                                          bool aligned16) {
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
  if constexpr (BITS > 0) {
    store_planes<0, BITS>(dst, plane_stride, v);
  } else {
    for (int b = 0; b < bits; ++b) dst[b * plane_stride] = plane_word(v, b);
  }
}

// POW2: kwp is a power of two (every ResNet channel count and the dense K of the
// configs) -> the (row, word) split is a shift instead of a 64-bit division.
// FAST: k % 32 == 0 and 16-byte aligned rows — every task is two full 16-byte loads;
// each thread keeps kBatch tasks (kBatch x 32 bytes) in flight, so the kernel reaches
// HBM speed with few resident threads (it overlaps the tensor-core conv of another layer,
// which leaves room for one 256-thread CTA per SM).
template <int BITS, bool POW2, bool FAST>
__global__ void __launch_bounds__(256) bitpack_kernel(const uint8_t* __restrict__ in, uint32_t* __restrict__ out,
                                                      int64_t rows, int64_t k, int64_t kwp, int kwp_shift,
                                                      int bits_rt, bool aligned16) {
  const int bits = BITS > 0 ? BITS : bits_rt;
  const int64_t tasks = rows * kwp;
  const int64_t plane_stride = rows * kwp;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if constexpr (FAST && BITS > 0) {
    constexpr int kBatch = 4;
    for (; t + (kBatch - 1) * stride < tasks; t += kBatch * stride) {
      uint4 lo[kBatch], hi[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {  // all loads first
        const int64_t tt = t + u * stride;
        const int64_t r = POW2 ? (tt >> kwp_shift) : tt / kwp;
        const int64_t j = tt - r * kwp;
        const uint4* src = reinterpret_cast<const uint4*>(in + r * k + 32 * j);
        lo[u] = __ldg(src);
        hi[u] = __ldg(src + 1);
      }
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int64_t tt = t + u * stride;
        const uint32_t v[8] = {lo[u].x, lo[u].y, lo[u].z, lo[u].w, hi[u].x, hi[u].y, hi[u].z, hi[u].w};
        store_planes<0, BITS>(out + tt, plane_stride, v);  // (row, word) = tt in [rows][kwp]
      }
    }
  }
  for (; t < tasks; t += stride) {
    const int64_t r = POW2 ? (t >> kwp_shift) : t / kwp;
    pack_word<BITS>(in, out, r, t - r * kwp, k, kwp, plane_stride, bits, aligned16);
  }
}

cudaError_t launch_bitpack(const uint8_t* in, uint32_t* out, int64_t rows, int64_t k, int64_t kwp, int bits,
                           cudaStream_t stream, int max_ctas) {
  const int64_t tasks = rows * kwp;
  const int threads = 256;
  int64_t blocks = (tasks + threads - 1) / threads;
  const int64_t max_blocks = int64_t(kNumSMs) * 8 * 4;  // grid-stride beyond 4 waves of 8 CTAs/SM
  if (blocks > max_blocks) blocks = max_blocks;
  if (max_ctas > 0 && blocks > max_ctas) blocks = max_ctas;  // leave SM room for a concurrent kernel
  const bool aligned16 = (reinterpret_cast<uintptr_t>(in) % 16 == 0) && (k % 16 == 0);
  const bool pow2 = (kwp & (kwp - 1)) == 0;
  const bool fast = aligned16 && (k % 32) == 0 && kwp * 32 == k;  // every word full, no pad words
  int shift = 0;
  while ((int64_t(1) << shift) < kwp) ++shift;
#define BS_PACK(BITS)                                                                                          \
  if (fast && pow2)                                                                                            \
    bitpack_kernel<BITS, true, true><<<blocks, threads, 0, stream>>>(in, out, rows, k, kwp, shift, bits, aligned16); \
  else if (pow2)                                                                                               \
    bitpack_kernel<BITS, true, false><<<blocks, threads, 0, stream>>>(in, out, rows, k, kwp, shift, bits, aligned16); \
  else                                                                                                         \
    bitpack_kernel<BITS, false, false><<<blocks, threads, 0, stream>>>(in, out, rows, k, kwp, shift, bits, aligned16);
  switch (bits) {
    case 1: BS_PACK(1) break;
    case 2: BS_PACK(2) break;
    case 3: BS_PACK(3) break;
    case 4: BS_PACK(4) break;
    default: BS_PACK(0) break;
  }
#undef BS_PACK
  note_launch();
  return cudaPeekAtLastError();
}

// ------------------------------------------------------------------ grouped packing
// Several packing problems of one bit width in one launch: the (row, word) tasks of all
// segments form one sequence (segment s owns [task0_s, task0_{s+1})) walked with a grid
// stride, so a thread's segment index only grows.  Removes the per-launch cost of the
// small layers' packs (a ResNet-18 step packs ten activation tensors of 6-51 MB).
template <int BITS>
__global__ void __launch_bounds__(256) bitpack_group_kernel(const __grid_constant__ PackGroupArgs a) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int s = 0;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < a.tasks; t += stride) {
    while (s + 1 < a.nseg && t >= a.seg[s + 1].task0) ++s;
    const PackSeg& g = a.seg[s];
    const int64_t lt = t - g.task0;
    const int64_t r = g.shift >= 0 ? (lt >> g.shift) : lt / g.kwp;
    pack_word<BITS>(g.in, g.out, r, lt - r * g.kwp, g.k, g.kwp, g.rows * g.kwp, BITS, g.aligned16);
  }
}

cudaError_t launch_bitpack_group(const PackSeg* segs, int count, int bits, cudaStream_t stream, int max_ctas) {
  for (int q0 = 0; q0 < count; q0 += kPackGroupMax) {
    PackGroupArgs a;
    memset(&a, 0, sizeof(a));
    a.nseg = count - q0 < kPackGroupMax ? count - q0 : kPackGroupMax;
    int64_t tasks = 0;
    for (int q = 0; q < a.nseg; ++q) {
      PackSeg g = segs[q0 + q];
      g.task0 = tasks;
      g.shift = -1;
      for (int sh = 0; sh < 62; ++sh)
        if ((int64_t(1) << sh) == g.kwp) g.shift = sh;
      g.aligned16 = (reinterpret_cast<uintptr_t>(g.in) % 16 == 0) && (g.k % 16 == 0);
      tasks += g.rows * g.kwp;
      a.seg[q] = g;
    }
    a.tasks = tasks;
    // 128-thread CTAs (4 K registers each): one fits beside a persistent tensor-core conv CTA
    // (832 threads x 72 registers leave 5.6 K of the SM's 64 K), so packing the later layers
    // can run on the SMs while an earlier layer's conv occupies them
    constexpr int kThr = 128;
    int64_t blocks = (tasks + kThr - 1) / kThr;
    const int64_t max_blocks = int64_t(kNumSMs) * 16 * 4;
    if (blocks > max_blocks) blocks = max_blocks;
    if (max_ctas > 0 && blocks > max_ctas) blocks = max_ctas;
    if (blocks < 1) continue;
    switch (bits) {
      case 1: bitpack_group_kernel<1><<<blocks, kThr, 0, stream>>>(a); break;
      case 2: bitpack_group_kernel<2><<<blocks, kThr, 0, stream>>>(a); break;
      case 3: bitpack_group_kernel<3><<<blocks, kThr, 0, stream>>>(a); break;
      case 4: bitpack_group_kernel<4><<<blocks, kThr, 0, stream>>>(a); break;
      case 5: bitpack_group_kernel<5><<<blocks, kThr, 0, stream>>>(a); break;
      case 6: bitpack_group_kernel<6><<<blocks, kThr, 0, stream>>>(a); break;
      case 7: bitpack_group_kernel<7><<<blocks, kThr, 0, stream>>>(a); break;
      default: bitpack_group_kernel<8><<<blocks, kThr, 0, stream>>>(a); break;
    }
    note_launch();
    if (cudaError_t e = cudaPeekAtLastError()) return e;
  }
  return cudaSuccess;
}

}  // namespace bs
