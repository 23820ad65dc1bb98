// digit.cu — digit packing: the bit-packing step emitting the
// operand format of the TMA-fed tensor-core kernel (tcd_conv.cu).
//
// PAPER.md:519-523 (Sec. 2.2) splits the codes into bit planes and packs them along the
// reduction axis; PAPER.md:555-567 (Sec. 3.1) adds a bit axis to the packed tensor.  Eq. 2
// is a sum over plane pairs, so planes (2d, 2d+1) may be grouped into one
// radix-4 digit d of weight 4^d (reading R21).  The digit-packed tensor keeps
// the bit-plane layout with its bit axis split into (digit, bit-in-digit) and the
// bit-in-digit axis innermost: element t of a row stores its two plane bits of digit d in
// one 4-bit field, as the E2M1 value 0.5 * digit (reading R24):
//
//   out [D][rows][row_bytes]  uint8, D = ceil(bits / 2), row_bytes = 16 * bs_packed_row_words(k)
//   byte b of a row holds elements 2b (low nibble) and 2b+1 (high nibble); elements >= k are 0
//   nibble of a digit value v in {-3..3}: (v < 0 ? 8 : 0) | |v|   (E2M1: 0.5 * |v|, sign bit 3)
//
// digit value of digit d (planes lo = 2d, hi = 2d+1 when 2d+1 < bits):
//   unsigned  b_lo + 2 b_hi                       (the code's radix-4 digit)
//   bipolar   (2 b_lo - 1) + 2 (2 b_hi - 1)       (each plane a +/-1 digit, reading R2/R20)
//   signed    the digit holding plane bits-1: b_lo - 2 b_hi (or -b_lo alone), others unsigned
//             (two's complement, reading R19)
// so sum_d 4^d * value_d is the code's value in its encoding (pinned by tests).
//
// The packer is HBM-bound: 1 byte read + D/2 bytes written per element.
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace bs {

// byte c of the result = nibble of the digit whose plane bits are c (bit 0 lo, bit 1 hi)
uint32_t digit_lut(int bits, int enc, int d) {
  const bool has_hi = 2 * d + 1 < bits, top = 2 * d + 2 >= bits;
  uint32_t lut = 0;
  for (int c = 0; c < (has_hi ? 4 : 2); ++c) {
    const int lo = c & 1, hi = (c >> 1) & 1;
    int v;
    if (enc == 1)
      v = has_hi ? (2 * lo - 1) + 2 * (2 * hi - 1) : 2 * lo - 1;
    else if (enc == 2 && top)
      v = has_hi ? lo - 2 * hi : -lo;
    else
      v = lo + 2 * hi;
    const uint32_t nib = uint32_t((v < 0 ? 8 : 0) | (v < 0 ? -v : v));
    lut |= nib << (8 * c);
  }
  return lut;
}

namespace {

// 32 codes (element 4q+r in byte r of v[q]) -> the 16 digit bytes of digit D.  Two words (8 elements) at a
// time: y = x | x >> 4 leaves the nibble pairs of elements (0,1) and (2,3) in bytes 0 and 2, and one PRMT
// gathers those bytes of both words (the window pack had been ALU-bound at ~175 instructions per task with
// a per-word compress: ncu, profiles/r02zn_ncu_full_winpack.json).
template <int D, int BITS>
__device__ __forceinline__ uint4 digit_row16(const uint32_t (&v)[8], uint32_t lut, bool ident) {
  constexpr bool kHi = 2 * D + 1 < BITS;
  constexpr uint32_t kMask = kHi ? 0x03030303u : 0x01010101u;
  uint32_t o[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t x0 = (v[2 * q] >> (2 * D)) & kMask, x1 = (v[2 * q + 1] >> (2 * D)) & kMask;  // byte r = plane bits
    const uint32_t nib = __byte_perm(x0 | (x0 >> 4), x1 | (x1 >> 4), 0x6420);  // nibble e = plane bits of element e
    if (ident) {
      o[q] = nib;
    } else {  // nibbles as byte selectors into the digit table, then compressed the same way
      const uint32_t r0 = __byte_perm(lut, 0u, nib), r1 = __byte_perm(lut, 0u, nib >> 16);
      o[q] = __byte_perm(r0 | (r0 >> 4), r1 | (r1 >> 4), 0x6420);
    }
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}

// nvalid < 32: elements past the row end are value 0 whatever the encoding (a bipolar code 0
// would otherwise become -1.5)
__device__ __forceinline__ uint4 keep_nibbles(uint4 x, int nvalid) {
  uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int nv = nvalid - 8 * i;
    w[i] = nv >= 8 ? w[i] : (nv <= 0 ? 0u : w[i] & ((1u << (4 * nv)) - 1u));
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

template <int D, int BITS>
__device__ __forceinline__ void store_digits(uint8_t* dst, int64_t plane_stride, const uint32_t (&v)[8],
                                             const uint32_t (&lut)[2], bool ident, int nvalid = 32) {
  if constexpr (2 * D < BITS) {
    uint4 o = digit_row16<D, BITS>(v, lut[D], ident);
    if (nvalid < 32) o = keep_nibbles(o, nvalid);
    *reinterpret_cast<uint4*>(dst + D * plane_stride) = o;
    store_digits<D + 1, BITS>(dst, plane_stride, v, lut, ident, nvalid);
  }
}

// the 32 codes of task (row r, word j); zeros past k
__device__ __forceinline__ void load32(const uint8_t* __restrict__ in, int64_t r, int64_t j, int64_t k, bool aligned16,
                                       uint32_t (&v)[8]) {
  const int64_t e0 = 32 * j;
  const uint8_t* src = in + r * k + e0;
  if (aligned16 && e0 + 32 <= k) {
    const uint4 lo = __ldg(reinterpret_cast<const uint4*>(src));
    const uint4 hi = __ldg(reinterpret_cast<const uint4*>(src) + 1);
    v[0] = lo.x; v[1] = lo.y; v[2] = lo.z; v[3] = lo.w;
    v[4] = hi.x; v[5] = hi.y; v[6] = hi.z; v[7] = hi.w;
  } else if (aligned16 && e0 + 16 == k) {
    const uint4 lo = __ldg(reinterpret_cast<const uint4*>(src));
    v[0] = lo.x; v[1] = lo.y; v[2] = lo.z; v[3] = lo.w;
    v[4] = v[5] = v[6] = v[7] = 0u;
  } else {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t x = 0;
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        const int64_t e = e0 + 4 * q + rr;
        if (e < k) x |= uint32_t(__ldg(src + 4 * q + rr)) << (8 * rr);
      }
      v[q] = x;
    }
  }
}

// Grouped digit packing: the (row, word) tasks of all segments form one sequence walked
// with a grid stride (as bitpack_group_kernel); one task = 32 codes -> 16 bytes per digit.
// FAST segments (k % 32 == 0, 16-byte rows, no pad words) keep 4 tasks' loads in flight.
template <int BITS>
__global__ void __launch_bounds__(256) digitpack_group_kernel(const __grid_constant__ DigitPackArgs a) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int s = 0;
  int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  constexpr int kBatch = 4;
  for (; t < a.tasks; t += stride) {
    while (s + 1 < a.nseg && t >= a.seg[s + 1].task0) ++s;
    const DigitSeg& g = a.seg[s];
    const int64_t end = s + 1 < a.nseg ? a.seg[s + 1].task0 : a.tasks;
    if (g.fast && t + (kBatch - 1) * stride < end) {  // kBatch tasks of this segment, loads first
      uint4 lo[kBatch], hi[kBatch];
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int64_t lt = t + u * stride - g.task0;
        const int64_t r = lt >> g.shift, j = lt - (r << g.shift);
        const uint4* src = reinterpret_cast<const uint4*>(g.in + r * g.k + 32 * j);
        lo[u] = __ldg(src);
        hi[u] = __ldg(src + 1);
      }
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int64_t lt = t + u * stride - g.task0;
        const uint32_t v[8] = {lo[u].x, lo[u].y, lo[u].z, lo[u].w, hi[u].x, hi[u].y, hi[u].z, hi[u].w};
        store_digits<0, BITS>(g.out + lt * 16, g.plane_bytes, v, g.lut, g.ident);
      }
      t += (kBatch - 1) * stride;
      continue;
    }
    const int64_t lt = t - g.task0;
    const int64_t r = g.shift >= 0 ? (lt >> g.shift) : lt / g.kwp;
    const int64_t j = lt - r * g.kwp;
    uint32_t v[8];
    load32(g.in, r, j, g.k, g.aligned16, v);
    const int64_t left = g.k - 32 * j;
    store_digits<0, BITS>(g.out + lt * 16, g.plane_bytes, v, g.lut, g.ident, left >= 32 ? 32 : int(left < 0 ? 0 : left));
  }
}

}  // namespace

int64_t digit_row_bytes(int64_t k) {
  const int64_t w = (k + 31) / 32;
  return k <= 0 ? 0 : 16 * (w + (w & 1));
}

cudaError_t launch_digitpack_group(const DigitSeg* segs, int count, int bits, int enc, cudaStream_t stream) {
  for (int q0 = 0; q0 < count; q0 += kPackGroupMax) {
    DigitPackArgs a;
    memset(&a, 0, sizeof(a));
    a.nseg = count - q0 < kPackGroupMax ? count - q0 : kPackGroupMax;
    int64_t tasks = 0;
    for (int q = 0; q < a.nseg; ++q) {
      DigitSeg g = segs[q0 + q];
      g.kwp = digit_row_bytes(g.k) / 16;
      g.task0 = tasks;
      g.plane_bytes = g.rows * g.kwp * 16;
      g.shift = -1;
      for (int sh = 0; sh < 62; ++sh)
        if ((int64_t(1) << sh) == g.kwp) g.shift = sh;
      g.aligned16 = (reinterpret_cast<uintptr_t>(g.in) % 16 == 0) && (g.k % 16 == 0);
      g.fast = g.aligned16 && g.k % 32 == 0 && g.kwp * 32 == g.k && g.shift >= 0;
      g.lut[0] = digit_lut(bits, enc, 0);
      g.lut[1] = digit_lut(bits, enc, 1);
      g.ident = enc == 0;
      tasks += g.rows * g.kwp;
      a.seg[q] = g;
    }
    a.tasks = tasks;
    int64_t blocks = (tasks + 255) / 256;
    const int64_t max_blocks = int64_t(device_sms()) * 8 * 2;
    if (blocks > max_blocks) blocks = max_blocks;
    if (blocks < 1) continue;
    switch (bits) {
      case 1: digitpack_group_kernel<1><<<blocks, 256, 0, stream>>>(a); break;
      case 2: digitpack_group_kernel<2><<<blocks, 256, 0, stream>>>(a); break;
      case 3: digitpack_group_kernel<3><<<blocks, 256, 0, stream>>>(a); break;
      default: digitpack_group_kernel<4><<<blocks, 256, 0, stream>>>(a); break;
    }
    note_launch();
    if (cudaError_t e = cudaPeekAtLastError()) return e;
  }
  return cudaSuccess;
}

// ------------------------------------------------------------------ window layout (R26)
// One task = one 16-byte half of a 32-byte row (one 32-channel slab, all digits) of the window
// layout [D][nph][cw/2][pstride][32]: task index lt = ((slot * pairs + pair) * pstride + q) * 2 + j,
// so consecutive threads write consecutive 16-byte pieces (coalesced) and read the 32-channel
// halves of consecutive phase-grid pixels.  Half j of row q lands in position j ^ (bit 2 of q)
// (the 32-byte shared-memory swizzle).  Padding, grid positions past the image and the tail are
// written as 0 (value 0 in every encoding, R20) on every call: no separate clearing.
namespace {
template <int BITS>
__global__ void __launch_bounds__(256) digitpack_win_kernel(const __grid_constant__ WinPackArgs a) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int s = 0;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < a.tasks; t += stride) {
    while (s + 1 < a.nseg && t >= a.seg[s + 1].task0) ++s;
    const WinSeg& g = a.seg[s];
    const uint32_t lt = uint32_t(t - g.task0);
    const uint32_t j = lt & 1u, row = lt >> 1;  // row = (slot * pairs + pair) * pstride + q
    const uint32_t fp = g.div_ps.div(row);
    const uint32_t q = row - fp * g.div_ps.d;
    const uint32_t f = g.div_pairs.div(fp), cs = 2 * (fp - f * g.div_pairs.d) + j;
    bool ok = int64_t(q) < g.gpix && int64_t(cs) * 32 < g.c;
    int64_t pix = 0;
    if (ok) {
      const uint32_t img = g.div_img.div(q), rem = q - img * g.div_img.d;
      const uint32_t gy = g.div_wg.div(rem), gx = rem - gy * g.div_wg.d;
      const int y = int(gy) * g.s + g.py[f] - g.ph, x = int(gx) * g.s + g.px[f] - g.pw;
      ok = unsigned(y) < unsigned(g.h) && unsigned(x) < unsigned(g.w);
      pix = (int64_t(img) * g.h + y) * g.w + x;
    }
    uint8_t* dst = g.out + int64_t(row) * 32 + ((j ^ ((q >> 2) & 1u)) << 4);
    if (!ok) {
#pragma unroll
      for (int d = 0; 2 * d < BITS; ++d) *reinterpret_cast<uint4*>(dst + d * g.dstride) = make_uint4(0u, 0u, 0u, 0u);
      continue;
    }
    uint32_t v[8];
    load32(g.in, pix, cs, g.c, g.aligned16, v);
    const int64_t left = g.c - 32 * int64_t(cs);
    store_digits<0, BITS>(dst, g.dstride, v, g.lut, g.ident, left >= 32 ? 32 : int(left));
  }
}
}  // namespace

cudaError_t launch_digitpack_win_group(const WinSeg* segs, int count, int bits, int enc, cudaStream_t stream) {
  for (int q0 = 0; q0 < count; q0 += kPackGroupMax) {
    WinPackArgs a;
    memset(&a, 0, sizeof(a));
    a.nseg = count - q0 < kPackGroupMax ? count - q0 : kPackGroupMax;
    int64_t tasks = 0;
    for (int q = 0; q < a.nseg; ++q) {
      WinSeg g = segs[q0 + q];
      TcwGeom G;
      if (!tcw_geom(g.n, g.h, g.w, g.c, 1, g.kh, g.kw, g.s, g.s, g.ph, g.pw, G)) return cudaErrorNotSupported;
      g.hg = G.hg;
      g.wg = G.wg;
      g.cw = G.cw;
      g.gpix = G.gpix;
      g.dstride = G.digit_bytes;
      for (int f = 0; f < 4; ++f) {
        g.py[f] = f < G.nph ? G.phase[f] / G.s : 0;
        g.px[f] = f < G.nph ? G.phase[f] % G.s : 0;
      }
      g.tasks = int64_t(G.nph) * G.cw * G.pstride;
      g.task0 = tasks;
      g.div_ps = make_fastdiv(uint32_t(G.pstride));
      g.div_pairs = make_fastdiv(uint32_t(G.cw / 2));
      g.div_img = make_fastdiv(uint32_t(G.hg) * uint32_t(G.wg));
      g.div_wg = make_fastdiv(uint32_t(G.wg));
      g.aligned16 = (reinterpret_cast<uintptr_t>(g.in) % 16 == 0) && (g.c % 16 == 0);
      g.lut[0] = digit_lut(bits, enc, 0);
      g.lut[1] = digit_lut(bits, enc, 1);
      g.ident = enc == 0;
      tasks += g.tasks;
      a.seg[q] = g;
    }
    a.tasks = tasks;
    int64_t blocks = (tasks + 255) / 256;
    const int64_t max_blocks = int64_t(device_sms()) * 8;
    if (blocks > max_blocks) blocks = max_blocks;
    if (blocks < 1) continue;
    switch (bits) {
      case 1: digitpack_win_kernel<1><<<blocks, 256, 0, stream>>>(a); break;
      case 2: digitpack_win_kernel<2><<<blocks, 256, 0, stream>>>(a); break;
      case 3: digitpack_win_kernel<3><<<blocks, 256, 0, stream>>>(a); break;
      default: digitpack_win_kernel<4><<<blocks, 256, 0, stream>>>(a); break;
    }
    note_launch();
    if (cudaError_t e = cudaPeekAtLastError()) return e;
  }
  return cudaSuccess;
}

// Window-path weight digits [nblk][cw/2][Dw][taps][bn][32] from packed planes [W][oc][taps*cw]
// (the stage's weights of one 64-channel slab pair are one contiguous block: one bulk copy);
// half j of filter row r lands in position j ^ (bit 2 of r) (the 32-byte smem swizzle);
// filters past oc and channels past c are 0.
namespace {
__global__ void tcw_weight_kernel(const uint32_t* __restrict__ wp, int w_bits, int oc, int taps, int cw, int c, int bn,
                                  int nblk, uint32_t lut0, uint32_t lut1, uint8_t* __restrict__ out) {
  const int P = (w_bits + 1) / 2, pairs = cw / 2;
  const int64_t total = int64_t(nblk) * pairs * P * taps * bn * 2;
  const int64_t kp = int64_t(taps) * cw;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    int64_t x = idx;
    const int j = int(x % 2);
    x /= 2;
    const int r = int(x % bn);
    const int64_t rowi = x;  // ((((nb * pairs + p) * P + e) * taps + t) * bn + r)
    x /= bn;
    const int t = int(x % taps);
    x /= taps;
    const int e = int(x % P);
    x /= P;
    const int p = int(x % pairs);
    const int nb = int(x / pairs);
    const int o = nb * bn + r, cs = 2 * p + j;
    uint32_t w4[4] = {0u, 0u, 0u, 0u};
    if (o < oc) {
      const int64_t rk = int64_t(o) * kp + int64_t(t) * cw + cs;
      const bool has_hi = 2 * e + 1 < w_bits;
      const uint32_t lo = wp[int64_t(2 * e) * oc * kp + rk];
      const uint32_t hi = has_hi ? wp[int64_t(2 * e + 1) * oc * kp + rk] : 0u;
      const uint32_t lut = e == 0 ? lut0 : lut1;
      for (int b = 0; b < 32; ++b) {
        if (cs * 32 + b >= c) break;  // channel padding: value 0
        const uint32_t cc = ((lo >> b) & 1u) | (((hi >> b) & 1u) << 1);
        w4[b >> 3] |= ((lut >> (8 * cc)) & 0xFu) << (4 * (b & 7));
      }
    }
    *reinterpret_cast<uint4*>(out + rowi * 32 + ((j ^ ((r >> 2) & 1)) << 4)) = make_uint4(w4[0], w4[1], w4[2], w4[3]);
  }
}
}  // namespace

cudaError_t launch_tcw_weights(const uint32_t* w_packed, int w_bits, int w_enc, int oc, int kh, int kw, int c,
                               uint8_t* out, cudaStream_t stream) {
  const int64_t bytes = tcw_weight_bytes(oc, kh, kw, c, w_bits);
  if (bytes <= 0) return cudaErrorInvalidValue;
  const int cw = int(digit_row_bytes(c) / 16), bn = oc <= 64 ? 64 : 128;
  int64_t blocks = (bytes / 16 + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  tcw_weight_kernel<<<blocks, 256, 0, stream>>>(w_packed, w_bits, oc, kh * kw, cw, c, bn, (oc + bn - 1) / bn,
                                                digit_lut(w_bits, w_enc, 0), digit_lut(w_bits, w_enc, 1), out);
  note_launch();
  return cudaPeekAtLastError();
}

// ------------------------------------------------------------------ weight digits
// Packed weight planes [W][n][kp] words (filter rows of `taps` taps of kw_tap words, c_tap
// elements per tap) -> digit rows [P][n][tcd_wrow_bytes(kp)] bytes, P = ceil(W/2), in the same
// element order as the activation digits; positions past c_tap inside a tap (padding) and the
// row tail up to the next 128-byte multiple are 0 (the kernel's weight boxes are 128 bytes
// wide and never leave the tensor: TMA boxes reaching past a row end measured several times
// slower).
namespace {
__global__ void weight_digits_kernel(const uint32_t* __restrict__ wp, int w_bits, int64_t n, int64_t kp, int c_tap,
                                     int kw_tap, uint32_t lut0, uint32_t lut1, int64_t wrow, uint8_t* __restrict__ out) {
  const int P = (w_bits + 1) / 2;
  const int64_t total = int64_t(P) * n * kp;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int e = int(t / (n * kp));
    const int64_t rk = t - e * n * kp;  // row * kp + kk
    const int64_t kk = rk % kp;
    const bool has_hi = 2 * e + 1 < w_bits;
    const uint32_t lo = wp[int64_t(2 * e) * n * kp + rk];
    const uint32_t hi = has_hi ? wp[int64_t(2 * e + 1) * n * kp + rk] : 0u;
    const int wt = int(kk % kw_tap), base = wt * 32;
    const uint32_t lut = e == 0 ? lut0 : lut1;
    uint32_t o[4] = {0u, 0u, 0u, 0u};
    for (int b = 0; b < 32; ++b) {
      if (base + b >= c_tap) break;  // tap padding: value 0
      const uint32_t c = ((lo >> b) & 1u) | (((hi >> b) & 1u) << 1);
      const uint32_t nib = (lut >> (8 * c)) & 0xFu;
      o[b >> 3] |= nib << (4 * (b & 7));
    }
    *reinterpret_cast<uint4*>(out + (int64_t(e) * n + rk / kp) * wrow + kk * 16) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}
}  // namespace

int64_t tcd_wrow_bytes(int64_t kp) { return (kp * 16 + 127) / 128 * 128; }
int64_t tcd_weight_bytes(int64_t n, int64_t kp, int w_bits) { return int64_t((w_bits + 1) / 2) * n * tcd_wrow_bytes(kp); }

cudaError_t launch_weight_digits(const uint32_t* w_packed, int w_bits, int w_enc, int64_t n, int64_t kp, int c_tap,
                                 int kw_tap, uint8_t* out, cudaStream_t stream) {
  const int64_t total = int64_t((w_bits + 1) / 2) * n * kp;
  if (total == 0) return cudaSuccess;
  if (cudaError_t e = cudaMemsetAsync(out, 0, size_t(tcd_weight_bytes(n, kp, w_bits)), stream)) return e;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  weight_digits_kernel<<<blocks, 256, 0, stream>>>(w_packed, w_bits, n, kp, c_tap, kw_tap, digit_lut(w_bits, w_enc, 0),
                                                   digit_lut(w_bits, w_enc, 1), tcd_wrow_bytes(kp), out);
  note_launch();
  return cudaPeekAtLastError();
}

}  // namespace bs
