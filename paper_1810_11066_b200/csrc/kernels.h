// kernels.h — internal (C++) launch interface between abi.cu and the kernels.
// Not part of the C ABI; see include/bitserial.h for the public boundary.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace bs {

// Implicit-GEMM problem.  A dense product is the 1x1 convolution of M "pixels"
// (n = 1, h = M, w = 1, c = K), so one description serves both operators.
//   act : packed activations, plane stride act_plane = rows_a * kw_a words,
//         row (pixel) r at act + r * kw_a;            rows_a = n*h*w
//   wt  : packed weights [w_bits][oc][kp], kp = taps * kw_a words per filter
//   out : int32 [M][oc], M = n*oh*ow
struct ConvProblem {
  const uint32_t* act;
  const uint32_t* wt;
  int32_t* out;
  int n, h, w, kw_a;        // input geometry, words per pixel per plane (Cw_pad)
  int oc, kh, kwid;         // filters, kernel height/width
  int sh, sw, ph, pw;       // stride, padding
  int oh, ow;               // output extent
  int a_bits, w_bits;
  int bipolar;              // weight encoding (0 unipolar, 1 bipolar, 2 signed)
  int a_enc;                // activation encoding (0 unsigned, 1 bipolar, 2 signed; tensor-core FP4 path)
  int c_tap;                // channels (elements) per tap: c for conv, k for dense
  int64_t act_plane;        // rows_a * kw_a
  int64_t M;                // n*oh*ow
  int64_t kp;               // taps * kw_a
  int one;                  // always 1: opaque to the compiler (keeps plane weights in registers)
  int ksplit;               // K slices across blockIdx.z (set by the launcher)
};

// Count of kernels this library has launched (host-side, incremented per launch).
void note_launch();
int64_t launch_count();

// Process-wide tuning knobs (bs_set_tuning; atomics, read per launch; 0 = library choice).
enum TuneKnob : int {
  kTuneTileN = 0, kTuneEpilogue = 1, kTuneGroupSplit = 2, kTuneBSlots = 3, kTuneSmallKs = 4, kTuneTcdASrc = 5,
  kTuneTcdBStream = 6, kTuneTcdMcast = 7, kTuneCount = 8
};
int tuning(int knob);
// SM count of the current device (cached per device).
int device_sms();

enum class Algo : int { Auto = 0, Popc = 1, PopcLit = 2, Gemv = 3 };

cudaError_t launch_bitpack(const uint8_t* in, uint32_t* out, int64_t rows, int64_t k, int64_t kwp, int bits,
                           cudaStream_t stream, int max_ctas = 0);

// One segment of a grouped pack (in/out/rows/k/kwp set by the caller; the rest by the launcher).
struct PackSeg {
  const uint8_t* in;
  uint32_t* out;
  int64_t rows, k, kwp, task0;
  int shift;      // log2(kwp) or -1
  int aligned16;  // 16-byte aligned rows
};
constexpr int kPackGroupMax = 16;
struct PackGroupArgs {
  int nseg;
  int64_t tasks;
  PackSeg seg[kPackGroupMax];
};
cudaError_t launch_bitpack_group(const PackSeg* segs, int count, int bits, cudaStream_t stream, int max_ctas = 0);

// Tiled AND+POPC implicit-GEMM kernel (conv and dense); returns cudaErrorNotSupported
// when no instantiation covers (a_bits, w_bits, algo).
cudaError_t launch_popc_conv(const ConvProblem& p, Algo algo, cudaStream_t stream);

// Tensor-core (tcgen05, kind::i8) bitserial kernel: one MMA per activation/weight
// plane pair on expanded bit-planes (tc_conv.cu).  `wexp_ws` receives the expanded
// weight planes (tc_weight_bytes bytes); cudaErrorNotSupported outside A<=4, W<=2.
// Operand formats of the tensor-core path: kind::i8 bytes, or kind::mxf4 packed E2M1
// nibbles with per-plane UE8M0 scales (tc_conv.cu).  kTcDefault is what format 0 means.
constexpr int kTcI8 = 1, kTcF4 = 2;
constexpr int kTcDefault = kTcF4;
int tc_resolve_format(int fmt);
int64_t tc_kpad(int64_t kp, int fmt);  // K words rounded to the format's chunk (I8 4, FP4 8)
int64_t tc_weight_bytes(int64_t n, int64_t kp, int w_bits, int fmt);
bool tc_supported(int a_bits, int w_bits);
// expanded ("prepared") weights: [w_bits][n][tc_kpad(kp)*(32 | 16)] bytes, offline like packing
// w_enc: 0 unipolar, 1 bipolar, 2 signed; c_tap elements in each kw_tap-word tap (padding -> 0)
cudaError_t launch_tc_expand_weights(const uint32_t* w_packed, int w_bits, int w_enc, int64_t n, int64_t kp,
                                     int c_tap, int kw_tap, int8_t* wexp, int fmt, cudaStream_t stream);
// peers (npeer <= 8): the output is also stored, box by box from the same staged tile, to
// these [M][oc] blocks (other ranks' gathered buffers mapped over NVLink): a fused all-gather.
// mcast: the multicast (NVLS) address of the output instead: one multimem store per staged
// row segment reaches every device bound to the multicast object (fused all-gather, §8 f2).
cudaError_t launch_tc_conv_prepared(const ConvProblem& p, const int8_t* wexp, int fmt, cudaStream_t stream,
                                    int32_t* const* peers = nullptr, int npeer = 0, int32_t* mcast = nullptr);
cudaError_t launch_tc_conv(const ConvProblem& p, int8_t* wexp_ws, int fmt, cudaStream_t stream);
// FP4 prepared-weight launch whose epilogue stores through the multicast address `mcast`.
cudaError_t launch_tc_conv_mcast(const ConvProblem& p, const int8_t* wexp, cudaStream_t stream, int32_t* mcast);
// FP4 tensor-core conv / dense on the PACKED weight planes (no prepared copy): the producer
// warps expand each weight chunk in shared memory (unipolar / bipolar weights, unsigned
// activations; FP4 exactness bound applies).  The three-call boundary's tensor-core path.
cudaError_t launch_tc_conv_raw(const ConvProblem& p, cudaStream_t stream);
// Several problems of one (a_bits, w_bits) in one persistent launch per 16 problems.
cudaError_t launch_tc_conv_group(const ConvProblem* ps, const int8_t* const* wexps, int count, int fmt,
                                 cudaStream_t stream);

// Small problems in ONE launch (small_conv.cu): activation packing fused, AND+POPC, K split
// across a thread-block cluster and reduced through distributed shared memory.
// a_bits in [1,4], w_bits in [1,2], unipolar / bipolar weights; up to kSmallMax problems.
constexpr int kSmallMax = 16;
struct SmallConv {
  ConvProblem p;        // geometry, packed weights (p.wt), output (p.out); p.act unused
  const uint8_t* act;   // uint8 NHWC activation codes
};
bool small_supported(int a_bits, int w_bits);
cudaError_t launch_small_conv(const SmallConv* ps, int count, int a_bits, int w_bits, cudaStream_t stream);

// ---- digit-packed operands and the TMA-fed tensor-core kernel (digit.cu, tcd_conv.cu)
// Digit packing: [rows][k] codes -> [ceil(bits/2)][rows][digit_row_bytes(k)] E2M1 digit
// nibbles (two bit planes per 4-bit field; R24).  One segment per tensor.
struct DigitSeg {
  const uint8_t* in;  // [rows][k] codes
  uint8_t* out;       // [D][rows][digit_row_bytes(k)]
  int64_t rows, k;    // set by the caller; the rest by the launcher
  int64_t kwp, task0, plane_bytes;
  int shift, aligned16, fast, ident;
  uint32_t lut[2];
};
struct DigitPackArgs {
  int nseg;
  int64_t tasks;
  DigitSeg seg[kPackGroupMax];
};
int64_t digit_row_bytes(int64_t k);  // 16 * packed row words
uint32_t digit_lut(int bits, int enc, int d);
cudaError_t launch_digitpack_group(const DigitSeg* segs, int count, int bits, int enc, cudaStream_t stream);
// prepared weight digits [ceil(w_bits/2)][n][tcd_wrow_bytes(kp)] bytes from packed planes
// [w_bits][n][kp]: each row 16 kp bytes of digits, zero-padded to a multiple of 128 bytes
int64_t tcd_wrow_bytes(int64_t kp);
int64_t tcd_weight_bytes(int64_t n, int64_t kp, int w_bits);
cudaError_t launch_weight_digits(const uint32_t* w_packed, int w_bits, int w_enc, int64_t n, int64_t kp, int c_tap,
                                 int kw_tap, uint8_t* out, cudaStream_t stream);
// One problem of the TMA-fed kernel: activation digits (conv: [DA][n][h][w][row_bytes(c)];
// dense, kh = kw = h = w = 1 and c = k with `dense` set: [DA][n][row_bytes(k)]), weight digits
// [DW][oc][kh*kw*row_bytes(c)], int32 output [n*oh*ow][oc].
struct TcdProblem {
  const uint8_t* act;
  const uint8_t* wdig;
  int32_t* out;
  int n, h, w, c, oc, kh, kw, sh, sw, ph, pw, oh, ow;
  int a_digits, w_digits;
  int dense;  // 1: tiled 2-D operand map over [DA*n][row_bytes] (no im2col)
};
cudaError_t launch_tcd_group(const TcdProblem* ps, int count, cudaStream_t stream);

// ---- window layout and the windowed tensor-core conv (digit.cu, tcw_conv.cu; R26)
// The conv's zero-padded input split into its stride phases on a phase grid of hg x wg pixels
// per image; per (digit, phase slot, 32-channel slab) one contiguous array of pstride pixels x
// 16 bytes (digit-packed, R24).  Output (oy, ox) with tap (ky, kx) reads phase
// (ky % s, kx % s) at grid position q_out + (ky / s) * wg + kx / s, q_out = (img*hg + oy)*wg + ox,
// so a 128-row tile of consecutive grid positions reads every tap's A operand from ONE
// contiguous window per (phase, slab): a shifted shared-memory view, no gather.
constexpr int kTcwBM = 128;
struct TcwGeom {
  int s, oh, ow, hg, wg, nph, cw, taps, maxoff, lwin, R, ow8, bn, nblk;
  int phase[4];    // slot -> phase py*s + px
  int slot_of[4];  // phase -> slot (-1: not stored)
  int64_t gpix, pstride, digit_bytes;  // digit_bytes = nph * cw * pstride * 16
};
// false: outside the windowed kernel's domain (sh != sw, stride > 2, grid rows wider than a
// 128-row tile, 32-bit index limits)
bool tcw_geom(int n, int h, int w, int c, int oc, int kh, int kw, int sh, int sw, int ph, int pw, TcwGeom& g);
// prepared weights [nblk][cw/2][Dw][kh*kw][bn][32] bytes (bn = 64 if oc <= 64 else 128), rows
// with bit 2 set hold their 16-byte halves exchanged (the 32-byte smem swizzle)
int64_t tcw_weight_bytes(int oc, int kh, int kw, int c, int w_bits);
struct WinSeg {
  const uint8_t* in;  // [n][h][w][c] codes
  uint8_t* out;       // [D][nph][cw/2][pstride][32], halves exchanged on rows with bit 2 set
  int n, h, w, c, kh, kw, s, ph, pw;
  // set by the launcher
  int64_t task0, tasks, dstride;
  int hg, wg, cw, aligned16, ident;
  int py[4], px[4];
  int64_t gpix;
  FastDiv div_ps, div_pairs, div_img, div_wg;
  uint32_t lut[2];
};
struct WinPackArgs {
  int nseg;
  int64_t tasks;
  WinSeg seg[kPackGroupMax];
};
cudaError_t launch_digitpack_win_group(const WinSeg* segs, int count, int bits, int enc, cudaStream_t stream);
cudaError_t launch_tcw_weights(const uint32_t* w_packed, int w_bits, int w_enc, int oc, int kh, int kw, int c,
                               uint8_t* out, cudaStream_t stream);
struct TcwProblem {
  const uint8_t* act;  // window layout (launch_digitpack_win_group)
  const uint8_t* wt;   // launch_tcw_weights
  int32_t* out;        // int32 [n][oh][ow][oc]
  int n, h, w, c, oc, kh, kw, sh, sw, ph, pw;
  int a_digits, w_digits;
};
cudaError_t launch_tcw_group(const TcwProblem* ps, int count, cudaStream_t stream);

// Matrix-vector kernel for m <= 8 dense products.
//   a_packed : packed [a_bits][m][kwp] (or nullptr when a_codes is given)
//   a_codes  : uint8 [m][k] raw codes to pack in-kernel (fused; nullptr otherwise)
cudaError_t launch_gemv(const uint32_t* a_packed, const uint8_t* a_codes, int a_bits,
                        const uint32_t* w_packed, int w_bits, int bipolar,
                        int32_t* out, int64_t m, int64_t n, int64_t k, int64_t kwp, cudaStream_t stream);
bool gemv_supported(int64_t m, int64_t k, int a_bits, int w_bits);

}  // namespace bs
