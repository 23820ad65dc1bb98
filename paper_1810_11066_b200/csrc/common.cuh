// common.cuh — device helpers shared by the bitserial kernels (sm_100a).
// Nothing here is shared with oracle/ (the oracle is independent test code).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bs {

constexpr int kNumSMs = 148;  // B200; the host side queries the real count

// ---------------------------------------------------------------------------
// Bit-plane extraction used by every packer (Sec. 2.2:
// "splitting input vectors into individual bitplanes ... packed into a larger
// storage type such as a uint32").
// v holds 4 codes (byte q = element q).  Returns the 4 bits "bit b of element q"
// at bit positions q (LSB-first).  (v >> b) & 0x01010101 leaves one bit per byte at
// positions 0, 8, 16, 24; multiplying by 2^21 + 2^14 + 2^7 + 1 moves them to bits
// 21, 22, 23, 24 with no carries (all partial-product bits land on distinct
// positions), so one IMAD gathers the nibble.
__device__ __forceinline__ uint32_t plane_nibble(uint32_t v, int b) {
  uint32_t t = (v >> b) & 0x01010101u;
  return ((t * 0x00204081u) >> 21) & 0xFu;
}

// 32 codes in 8 words (element 4q+r in byte r of v[q]) -> packed word of plane b.
__device__ __forceinline__ uint32_t plane_word(const uint32_t (&v)[8], int b) {
  uint32_t w = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) w |= plane_nibble(v[q], b) << (4 * q);
  return w;
}

// Same result with compile-time plane B: mask the plane's bits in place (LOP3 with an
// immediate), gather them with one IMAD (bits land at 21+B..24+B), move the nibble
// to 4q with one funnel shift and merge with LOP3 — 4 integer ops per 4 codes.
template <int B>
__device__ __forceinline__ uint32_t plane_word_c(const uint32_t (&v)[8]) {
  uint32_t w = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint32_t prod = (v[q] & (0x01010101u << B)) * 0x00204081u;
    const int sh = 21 + B - 4 * q;  // compile-time after unrolling
    const uint32_t nib = sh >= 0 ? (prod >> sh) : (prod << (-sh));
    w |= nib & (0xFu << (4 * q));
  }
  return w;
}

// ---------------------------------------------------------------------------
// cp.async (LDGSTS) helpers: 8- and 16-byte copies with zero fill (src_size = 0).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];\n" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// Plain (compiler-scheduled) shared-memory vector loads through generic pointers
// into the dynamic smem array.
__device__ __forceinline__ uint4 lds128p(const uint32_t* p) { return *reinterpret_cast<const uint4*>(p); }
__device__ __forceinline__ uint2 lds64p(const uint32_t* p) { return *reinterpret_cast<const uint2*>(p); }

// n / d for 0 <= n < 2^31 with a precomputed multiplier (round-up method):
// q = (umulhi(n, mul) + n) >> shr, shr = ceil(log2 d), mul = floor(2^32 (2^shr - d) / d) + 1.
struct FastDiv {
  uint32_t d, mul, shr;
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, mul) + n) >> shr; }
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f{d, 0, 0};
  if (d > 1) {
    uint32_t p = 0;
    while ((uint64_t(1) << p) < d) ++p;
    f.shr = p;
    f.mul = uint32_t(((uint64_t(1) << 32) * ((uint64_t(1) << p) - d)) / d + 1);
  }
  return f;
}

}  // namespace bs
