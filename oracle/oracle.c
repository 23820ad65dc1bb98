/*
 * oracle.c — CPU oracle for the bitserial hot path of arXiv 1810.11066.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  The
 * product path (paper_1810_11066_b200/) never links, imports or calls it, and
 * this file shares no code, header, table or constant with the CUDA path.
 *
 * What it computes: the plain integer definitions that the bitserial method
 * reaches exactly (Eq. 1, Eq. 2 are identities over
 * integers, so the method's result IS the integer dot product / convolution):
 *
 *   oracle_weight_value  value of one weight code (unipolar / bipolar)
 *   oracle_dense         out[m][n] = sum_k a[m][k] * value(w[n][k])
 *   oracle_conv2d_nhwc   NHWC cross-correlation with zero padding, OHWI weights
 *   oracle_code_value    value of one code in any encoding (unsigned / bipolar / signed)
 *   oracle_dense_enc, oracle_conv2d_nhwc_enc
 *                        the same products with an encoding for each operand
 *                        (both-bipolar XNOR form; signed
 *                        two's-complement data)
 *   oracle_bitpack       the packed bit-plane layout of the C ABI (defines it)
 *   oracle_digitpack     the digit-packed layout of the C ABI (defines it): bit planes
 *                        (2d, 2d+1) of each element as one radix-4 digit (Eq. 2 regrouped,
 *                        PAPER.md:512; R21/R24) stored as a 4-bit E2M1 field
 *
 * No bit-planes, no popcount, no blocking or reordering: straight loops over the
 * decoded integer values in the order of the definitions.  The only parallelism is
 * an OpenMP split of the outermost output loop (each output is still one
 * sequential sum), used so the CPU baseline is timed on all host cores.
 *
 * Pinned by tests/test_oracle_pins.py (brute-force Eq. 2 over bit-planes,
 * torch float64 mm / conv2d, closed forms, invariants, tests/golden/ fixtures).
 * Readings of the paper this file relies on are listed in DESIGN.md §3.
 *
 * Return codes: 0 = ok, -1 = invalid argument (codes out of range, bad shape,
 * accumulator bound exceeded).  Outputs are int32 as on the GPU; every call checks
 * that the largest possible |output| fits (bound check, not saturation).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Value of one weight code (readings R1-R3).
 * Unipolar: the code itself (Eq. 2, weights are unsigned M-bit ints).
 * Bipolar : each bit-plane is a +/-1 digit ("bipolar format (-1 and 1)";
 *           north_star: per plane pair popc(a & w) - popc(a & ~w)), so bit b_j set
 *           contributes +2^j and clear contributes -2^j:  value = sum_j 2^j (2 b_j - 1). */
int64_t oracle_weight_value(int code, int bits, int bipolar) {
  if (!bipolar) return code;
  int64_t v = 0;
  for (int j = 0; j < bits; ++j) {
    int b = (code >> j) & 1;
    v += (b ? 1 : -1) * ((int64_t)1 << j);
  }
  return v;
}

static int codes_in_range(const uint8_t* x, int64_t n, int bits) {
  for (int64_t i = 0; i < n; ++i)
    if (x[i] >= (1u << bits)) return 0;
  return 1;
}

/* largest |value| a weight code can take */
static int64_t max_abs_weight(int bits) { return ((int64_t)1 << bits) - 1; }

/* Dense / matrix multiply: a [m][k] activation codes
 * (unsigned, a_bits), w [n][k] weight codes (w_bits, unipolar or bipolar),
 * out [m][n] int32 row-major. */
int oracle_dense(const uint8_t* a, int a_bits, const uint8_t* w, int w_bits, int bipolar,
                 int32_t* out, int64_t m, int64_t n, int64_t k) {
  if (m <= 0 || n <= 0 || k <= 0 || a_bits < 1 || a_bits > 8 || w_bits < 1 || w_bits > 8) return -1;
  if (!codes_in_range(a, m * k, a_bits) || !codes_in_range(w, n * k, w_bits)) return -1;
  if ((double)k * (double)(((int64_t)1 << a_bits) - 1) * (double)max_abs_weight(w_bits) >= 2147483648.0) return -1;
  int32_t* wv = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n * k));
  if (!wv) return -1;
  for (int64_t i = 0; i < n * k; ++i) wv[i] = (int32_t)oracle_weight_value(w[i], w_bits, bipolar);
#pragma omp parallel for schedule(static)
  for (int64_t mi = 0; mi < m; ++mi) {
    for (int64_t ni = 0; ni < n; ++ni) {
      int32_t acc = 0;
      for (int64_t ki = 0; ki < k; ++ki) acc += (int32_t)a[mi * k + ki] * wv[ni * k + ki];
      out[mi * n + ni] = acc;
    }
  }
  free(wv);
  return 0;
}

/* Output extent of a convolution along one axis: floor((in + 2p - r) / s) + 1. */
int64_t oracle_conv_out_extent(int64_t in, int64_t r, int64_t s, int64_t p) {
  int64_t span = in + 2 * p - r;
  if (span < 0 || s < 1) return 0;
  return span / s + 1;
}

/* 2-D convolution, NHWC activations, OHWI weights ("NHWC", Table 1
 * PAPER.md:733-746 geometry): cross-correlation (no kernel flip) with zero padding
 * (pad positions are activation code 0), out int32 NHWC [n][oh][ow][oc]. */
int oracle_conv2d_nhwc(const uint8_t* act, int a_bits, const uint8_t* wt, int w_bits, int bipolar,
                       int32_t* out, int n, int h, int w, int c, int oc, int kh, int kw,
                       int sh, int sw, int ph, int pw) {
  if (n <= 0 || h <= 0 || w <= 0 || c <= 0 || oc <= 0 || kh <= 0 || kw <= 0) return -1;
  if (sh < 1 || sw < 1 || ph < 0 || pw < 0) return -1;
  if (a_bits < 1 || a_bits > 8 || w_bits < 1 || w_bits > 8) return -1;
  int64_t oh = oracle_conv_out_extent(h, kh, sh, ph), ow = oracle_conv_out_extent(w, kw, sw, pw);
  if (oh <= 0 || ow <= 0) return -1;
  int64_t K = (int64_t)kh * kw * c;
  if (!codes_in_range(act, (int64_t)n * h * w * c, a_bits) || !codes_in_range(wt, (int64_t)oc * K, w_bits)) return -1;
  if ((double)K * (double)(((int64_t)1 << a_bits) - 1) * (double)max_abs_weight(w_bits) >= 2147483648.0) return -1;
  int32_t* wv = (int32_t*)malloc(sizeof(int32_t) * (size_t)(oc * K));
  if (!wv) return -1;
  for (int64_t i = 0; i < oc * K; ++i) wv[i] = (int32_t)oracle_weight_value(wt[i], w_bits, bipolar);
  int64_t rows = (int64_t)n * oh * ow;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    int64_t b = r / (oh * ow), oy = (r / ow) % oh, ox = r % ow;
    for (int o = 0; o < oc; ++o) {
      int32_t acc = 0;
      for (int ky = 0; ky < kh; ++ky) {
        int64_t iy = oy * sh + ky - ph;
        if (iy < 0 || iy >= h) continue; /* zero padding contributes 0 */
        for (int kx = 0; kx < kw; ++kx) {
          int64_t ix = ox * sw + kx - pw;
          if (ix < 0 || ix >= w) continue;
          const uint8_t* ap = act + ((b * h + iy) * w + ix) * c;
          const int32_t* wp = wv + (((int64_t)o * kh + ky) * kw + kx) * c;
          for (int ci = 0; ci < c; ++ci) acc += (int32_t)ap[ci] * wp[ci];
        }
      }
      out[r * oc + o] = acc;
    }
  }
  free(wv);
  return 0;
}

/* Value of one code in encoding enc:
 *   0 unsigned / unipolar : the code (Eq. 2);
 *   1 bipolar             : every bit-plane a +/-1 digit, sum_j 2^j (2 b_j - 1)
 *                           ("bipolar format (-1 and 1)");
 *   2 signed              : two's complement, the top plane weighted -2^(bits-1)
 *                           ("weighting binary dotproducts by their sign"). */
int64_t oracle_code_value(int code, int bits, int enc) {
  if (enc == 1) return oracle_weight_value(code, bits, 1);
  if (enc == 2) return code >= (1 << (bits - 1)) ? (int64_t)code - ((int64_t)1 << bits) : code;
  return code;
}

static int64_t max_abs_value(int bits, int enc) {
  if (enc == 2) return (int64_t)1 << (bits - 1);
  return ((int64_t)1 << bits) - 1;
}

static int enc_ok(int enc) { return enc >= 0 && enc <= 2; }

/* out[m][n] = sum_k value(a[m][k]) * value(w[n][k]) with per-operand encodings. */
int oracle_dense_enc(const uint8_t* a, int a_bits, int a_enc, const uint8_t* w, int w_bits, int w_enc,
                     int32_t* out, int64_t m, int64_t n, int64_t k) {
  if (m <= 0 || n <= 0 || k <= 0 || a_bits < 1 || a_bits > 8 || w_bits < 1 || w_bits > 8) return -1;
  if (!enc_ok(a_enc) || !enc_ok(w_enc)) return -1;
  if (!codes_in_range(a, m * k, a_bits) || !codes_in_range(w, n * k, w_bits)) return -1;
  if ((double)k * (double)max_abs_value(a_bits, a_enc) * (double)max_abs_value(w_bits, w_enc) >= 2147483648.0)
    return -1;
  int32_t* av = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m * k));
  int32_t* wv = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n * k));
  if (!av || !wv) {
    free(av);
    free(wv);
    return -1;
  }
  for (int64_t i = 0; i < m * k; ++i) av[i] = (int32_t)oracle_code_value(a[i], a_bits, a_enc);
  for (int64_t i = 0; i < n * k; ++i) wv[i] = (int32_t)oracle_code_value(w[i], w_bits, w_enc);
#pragma omp parallel for schedule(static)
  for (int64_t mi = 0; mi < m; ++mi) {
    for (int64_t ni = 0; ni < n; ++ni) {
      int32_t acc = 0;
      for (int64_t ki = 0; ki < k; ++ki) acc += av[mi * k + ki] * wv[ni * k + ki];
      out[mi * n + ni] = acc;
    }
  }
  free(av);
  free(wv);
  return 0;
}

/* NHWC cross-correlation with per-operand encodings; zero padding: a padded position
 * contributes 0 (value 0, whatever the activation encoding). */
int oracle_conv2d_nhwc_enc(const uint8_t* act, int a_bits, int a_enc, const uint8_t* wt, int w_bits, int w_enc,
                           int32_t* out, int n, int h, int w, int c, int oc, int kh, int kw,
                           int sh, int sw, int ph, int pw) {
  if (n <= 0 || h <= 0 || w <= 0 || c <= 0 || oc <= 0 || kh <= 0 || kw <= 0) return -1;
  if (sh < 1 || sw < 1 || ph < 0 || pw < 0) return -1;
  if (a_bits < 1 || a_bits > 8 || w_bits < 1 || w_bits > 8 || !enc_ok(a_enc) || !enc_ok(w_enc)) return -1;
  int64_t oh = oracle_conv_out_extent(h, kh, sh, ph), ow = oracle_conv_out_extent(w, kw, sw, pw);
  if (oh <= 0 || ow <= 0) return -1;
  int64_t K = (int64_t)kh * kw * c;
  int64_t na = (int64_t)n * h * w * c;
  if (!codes_in_range(act, na, a_bits) || !codes_in_range(wt, (int64_t)oc * K, w_bits)) return -1;
  if ((double)K * (double)max_abs_value(a_bits, a_enc) * (double)max_abs_value(w_bits, w_enc) >= 2147483648.0)
    return -1;
  int32_t* av = (int32_t*)malloc(sizeof(int32_t) * (size_t)na);
  int32_t* wv = (int32_t*)malloc(sizeof(int32_t) * (size_t)(oc * K));
  if (!av || !wv) {
    free(av);
    free(wv);
    return -1;
  }
  for (int64_t i = 0; i < na; ++i) av[i] = (int32_t)oracle_code_value(act[i], a_bits, a_enc);
  for (int64_t i = 0; i < oc * K; ++i) wv[i] = (int32_t)oracle_code_value(wt[i], w_bits, w_enc);
  int64_t rows = (int64_t)n * oh * ow;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    int64_t b = r / (oh * ow), oy = (r / ow) % oh, ox = r % ow;
    for (int o = 0; o < oc; ++o) {
      int32_t acc = 0;
      for (int ky = 0; ky < kh; ++ky) {
        int64_t iy = oy * sh + ky - ph;
        if (iy < 0 || iy >= h) continue; /* zero padding contributes 0 */
        for (int kx = 0; kx < kw; ++kx) {
          int64_t ix = ox * sw + kx - pw;
          if (ix < 0 || ix >= w) continue;
          const int32_t* ap = av + ((b * h + iy) * w + ix) * c;
          const int32_t* wp = wv + (((int64_t)o * kh + ky) * kw + kx) * c;
          for (int ci = 0; ci < c; ++ci) acc += ap[ci] * wp[ci];
        }
      }
      out[r * oc + o] = acc;
    }
  }
  free(av);
  free(wv);
  return 0;
}

/* Words per packed row: ceil(k/32) rounded up to an even count (8-byte rows). */
int64_t oracle_packed_row_words(int64_t k) {
  int64_t kw = (k + 31) / 32;
  return kw + (kw & 1);
}

/* Bit-packing: split codes into bit-planes and pack
 * along the reduction axis into uint32 words.  Layout BMK' (bit axis outermost,
 * PAPER.md:564-567): out[b][r][j], bit t of word j = bit b of in[r][32j + t]
 * (LSB-first, reading R7); bits past k are 0. */
int oracle_bitpack(const uint8_t* in, uint32_t* out, int64_t rows, int64_t k, int bits) {
  if (rows <= 0 || k <= 0 || bits < 1 || bits > 8) return -1;
  if (!codes_in_range(in, rows * k, bits)) return -1;
  int64_t kwp = oracle_packed_row_words(k);
  for (int b = 0; b < bits; ++b)
    for (int64_t r = 0; r < rows; ++r)
      for (int64_t j = 0; j < kwp; ++j) {
        uint32_t word = 0;
        for (int t = 0; t < 32; ++t) {
          int64_t ki = 32 * j + t;
          if (ki < k && ((in[r * k + ki] >> b) & 1)) word |= (uint32_t)1 << t;
        }
        out[(b * rows + r) * kwp + j] = word;
      }
  return 0;
}

/* E2M1 (4-bit float: sign bit 3, exponent bits 2..1 with bias 1, mantissa bit 0) value of
 * a 4-bit field, times 2 (an integer): e == 0 -> 0.5 * m (subnormal), else 2^(e-1) (1 + m/2). */
int oracle_e2m1_twice(int nib) {
  const int s = (nib >> 3) & 1, e = (nib >> 1) & 3, m = nib & 1;
  const int twice = e == 0 ? m : (1 << (e - 1)) * (2 + m);
  return s ? -twice : twice;
}

/* Digit value of digit d of a code (R21/R24): planes lo = 2d and hi = 2d+1 (hi
 * only when 2d+1 < bits).  Unsigned: b_lo + 2 b_hi.  Bipolar: each plane a +/-1 digit
 * (reading R2/R20): (2 b_lo - 1) + 2 (2 b_hi - 1).  Signed (PAPER.md:517,
 * reading R19): the digit holding plane bits-1 weighs that plane -2^(bits-1), i.e.
 * b_lo - 2 b_hi (or -b_lo when the top plane is the digit's lo plane); lower digits as
 * unsigned.  sum_d 4^d value = oracle_code_value (pinned). */
int oracle_digit_value(int code, int bits, int enc, int d) {
  const int lo = (code >> (2 * d)) & 1;
  const int has_hi = 2 * d + 1 < bits;
  const int hi = has_hi ? (code >> (2 * d + 1)) & 1 : 0;
  const int top = 2 * d + 2 >= bits;
  if (enc == 1) return has_hi ? (2 * lo - 1) + 2 * (2 * hi - 1) : 2 * lo - 1;
  if (enc == 2 && top) return has_hi ? lo - 2 * hi : -lo;
  return lo + 2 * hi;
}

/* Digit packing: out [D][rows][16 * packed_row_words(k)] bytes, D = ceil(bits/2); element t
 * of row r is the 4-bit field t % 2 (low nibble first) of byte t / 2; the field holds the
 * E2M1 code whose value is 0.5 * digit value (found by decoding every code, so this follows
 * the format definition directly); elements >= k are 0. */
int oracle_digitpack(const uint8_t* in, uint8_t* out, int64_t rows, int64_t k, int bits, int enc) {
  if (rows <= 0 || k <= 0 || bits < 1 || bits > 4 || !enc_ok(enc)) return -1;
  if (!codes_in_range(in, rows * k, bits)) return -1;
  const int64_t rb = 16 * oracle_packed_row_words(k);
  const int D = (bits + 1) / 2;
  memset(out, 0, (size_t)(D * rows * rb));
  for (int d = 0; d < D; ++d)
    for (int64_t r = 0; r < rows; ++r)
      for (int64_t t = 0; t < k; ++t) {
        const int v = oracle_digit_value(in[r * k + t], bits, enc, d);
        int nib = -1;
        for (int x = 0; x < 16 && nib < 0; ++x)
          if (oracle_e2m1_twice(x) == v && !(v == 0 && x != 0)) nib = x;  /* +0 for zero */
        if (nib < 0) return -1;
        out[(d * rows + r) * rb + t / 2] |= (uint8_t)(nib << (4 * (t % 2)));
      }
  return 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
