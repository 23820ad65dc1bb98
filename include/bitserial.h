/*
 * bitserial.h — C ABI of the B200 (sm_100a) bitserial hot path of arXiv 1810.11066,
 * "Automating Generation of Low Precision Deep Learning Operators".
 *
 * The library (paper_1810_11066_b200/libbitserial.so) exports exactly the functions
 * below.  Citations are PAPER.md line numbers (/root/reference/PAPER.md, assembled
 * copy lines 416-831) and the section/equation they fall in.
 *
 * The operation (Sec. 2.2, Eq. 1 and Eq. 2):
 *     x . y = sum_{n<N} sum_{m<M} popcount(x_n & y_m) * 2^(m+n)
 * over bit-planes x_n of the activations and y_m of the weights, packed into 32-bit
 * words.  Bipolar weights (north_star) take each
 * weight bit-plane as a +/-1 digit: per plane pair popc(a & w) - popc(a & ~w).
 * Results are exact int32 ("a higher machine supported precision").
 *
 * ---------------------------------------------------------------------------
 * Conventions shared by every entry point
 * ---------------------------------------------------------------------------
 * Codes.     Activation and weight codes are unsigned integers in [0, 2^bits),
 *            one per uint8_t, bits in [1, 8].  Activations are unsigned; the weight
 *            encoding is BS_UNIPOLAR (value = code) or BS_BIPOLAR
 *            (value = sum_j 2^j (2 b_j - 1) = 2 code - (2^bits - 1): W1 -> {-1,+1},
 *            W2 -> {-3,-1,+1,+3}).  Codes outside [0, 2^bits) are a precondition
 *            violation: the packer uses only the low `bits` bits.
 * Packed.    "Packed" tensors use layout BMK' (bit axis outermost):
 *            uint32 [bits][rows][Kw_pad], Kw_pad = bs_packed_row_words(K); bit t of
 *            word j of plane b is bit b of code [row][32 j + t] (LSB-first); bits at
 *            reduction index >= K are 0.
 * Pointers.  All tensor pointers are DEVICE pointers (cudaMalloc / torch CUDA
 *            storage) unless the name ends in _host.  Tensor base pointers must be
 *            16-byte aligned.  The caller owns every buffer; the library never
 *            allocates or frees device memory and keeps no per-call state except a
 *            thread-local error string.
 * Streams.   `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *            stream).  Every call except *_host is asynchronous and stream-ordered:
 *            it validates, launches and returns without synchronizing.
 * Errors.    Every function validates all arguments BEFORE launching; on a non-OK
 *            status nothing was launched and no output was written.  BS_ERR_CUDA
 *            reports a launch failure (cudaPeekAtLastError / cudaGetLastError after
 *            launch); faults of a running kernel surface at the caller's next
 *            synchronization, as usual in CUDA.  bs_last_error() returns a
 *            thread-local message for the last non-OK status.  No C++ exception
 *            crosses this boundary.
 * Accumulator bound.  K * (2^a_bits - 1) * (2^w_bits - 1) must be < 2^31
 *            (BS_ERR_OVERFLOW otherwise) so every output is exact in int32.
 */
#ifndef BITSERIAL_H_
#define BITSERIAL_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BS_ABI_VERSION 1

typedef enum {
  BS_OK = 0,
  BS_ERR_NULL = 1,          /* a required pointer is NULL */
  BS_ERR_INVALID_ARG = 2,   /* bits not in [1,8], stride < 1, pad < 0, bad encoding/algo */
  BS_ERR_UNSUPPORTED = 3,   /* valid but not implemented (e.g. algo not built for bits) */
  BS_ERR_SHAPE = 4,         /* non-positive extent, or empty convolution output */
  BS_ERR_ALIGN = 5,         /* a tensor pointer is not 16-byte aligned */
  BS_ERR_OVERFLOW = 6,      /* K * (2^A-1) * (2^W-1) >= 2^31 */
  BS_ERR_CUDA = 7,          /* CUDA runtime error at launch / copy */
  BS_ERR_WORKSPACE = 8      /* workspace missing or smaller than *_workspace_bytes() */
} bs_status;

/* Weight encoding.  BS_SIGNED (two's complement, the top bit-plane weighs -2^(W-1):
 * "weighting binary dotproducts by their sign") is accepted by the
 * tensor-core entries only. */
typedef enum { BS_UNIPOLAR = 0, BS_BIPOLAR = 1, BS_SIGNED = 2 } bs_encoding;

/* Activation encoding (tensor-core entries, FP4 format).  BS_A_BIPOLAR: every plane a
 * +/-1 digit (value 2 code - (2^A - 1)); with bipolar weights this is the XNOR form of
 * PAPER.md:503.  BS_A_SIGNED: two's complement.  Zero padding and the
 * reduction-axis tail contribute 0 in every encoding. */
typedef enum { BS_A_UNSIGNED = 0, BS_A_BIPOLAR = 1, BS_A_SIGNED = 2 } bs_a_encoding;

/* Kernel family for the *_ex entry points.
 *   AUTO     : what bs_bitserial_dense / bs_bitserial_conv2d_nhwc run:
 *                dense with m <= 8 (A in {1,2,4}, W in {1,2})  -> GEMV;
 *                otherwise, when A <= 4, W <= 4 and K*(2^A-1)*(2^W-1) < 2^22 -> TC;
 *                otherwise -> POPC.
 *   TC       : the tensor-core kernel (tcgen05.mma kind::mxf4, radix-4 digits of two bit
 *              planes, FP32 accumulation exact below the bound above) on the PACKED weight
 *              planes: its producer warps expand each weight chunk into shared memory
 *              (no prepared copy, no workspace; weights stay resident per N block when
 *              their K chunks fit).  BS_ERR_UNSUPPORTED outside A, W <= 4 / the bound.
 *   POPC     : AND + POPC per word pair (Eq. 1 inside Eq. 2) on the integer pipes;
 *              bipolar applied as the exact identity 2*U - (2^W-1)*sum(a).
 *   POPC_LIT : as POPC but bipolar evaluated literally, popc(a&w) - popc(a&~w) per
 *              plane pair (north_star form; twice the POPC work; unipolar = POPC).
 *   GEMV     : warp-per-rows matrix-vector kernel with butterfly multi-row reduction
 *              (PAPER.md:694-705 micro-kernel ideas), for m <= 8 (dense only).
 * The prepared-weight tensor-core entries below (bs_*_tc_prepared, *_tc_group) skip the
 * in-kernel weight expansion: the fastest form for weights reused across calls. */
typedef enum {
  BS_ALGO_AUTO = 0,
  BS_ALGO_POPC = 1,
  BS_ALGO_POPC_LIT = 2,
  BS_ALGO_GEMV = 3,
  BS_ALGO_TC = 4
} bs_algo;

int bs_abi_version(void);
const char* bs_status_string(int status);
const char* bs_last_error(void);

/* Number of kernels this library has launched in this process (host-side count,
 * incremented per launch call; graph replays of captured launches are not counted).
 * Used by bench.py to report how many of the library's kernels a step runs. */
int64_t bs_kernel_launches(void);

/* Tuning knobs of the tensor-core path, process-wide (atomic; every later launch on any
 * thread sees the new value).  They never change results, only the launch configuration;
 * 0 is the library's choice.  For tests and experiments:
 *   BS_TUNE_TC_TILE_N      : output tile width 64 or 128 (default: 64 when oc <= 64, else 128);
 *                            224: the digit path's single-problem launches (default for dense
 *                            products with n >= 1024)
 *   BS_TUNE_TC_EPILOGUE    : 1 = direct 16-byte global stores instead of TMA stores
 *   BS_TUNE_TC_GROUP_SPLIT : 1 = grouped launches interleave long-K and short-K members' tiles
 *   BS_TUNE_TC_B_SLOTS     : cap on the weight chunk slots in shared memory (2..32): fewer slots
 *                            than a tile's K chunks make its weights stream instead of staying
 *                            resident
 *   BS_TUNE_SMALL_KSPLIT   : K slices (= cluster size) of the one-launch small-problem path
 *                            (bs_bitserial_conv2d_nhwc_i8_group): 1, 2, 4 or 8
 *   BS_TUNE_TCD_A_SRC      : digit-path conv activations: 1 = TMA im2col loads, 2 = cp.async
 *                            gathers by producer warps (the default)
 *   BS_TUNE_TCD_B_STREAM   : 1 = digit-path weights always streamed per stage (default: a weight
 *                            block of up to 96 KB stays resident per N block)
 *   BS_TUNE_TCD_MCAST      : 2-CTA clusters that each load half of every streamed weight chunk and
 *                            multicast it to both (dense, even number of M blocks): 1 = never,
 *                            2 = always, 0 = at >= 128 M blocks or several digits
 * bs_set_tuning returns BS_ERR_INVALID_ARG for an unknown knob or value; bs_get_tuning returns
 * the current value (0 for an unknown knob). */
typedef enum {
  BS_TUNE_TC_TILE_N = 0,
  BS_TUNE_TC_EPILOGUE = 1,
  BS_TUNE_TC_GROUP_SPLIT = 2,
  BS_TUNE_TC_B_SLOTS = 3,
  BS_TUNE_SMALL_KSPLIT = 4,
  BS_TUNE_TCD_A_SRC = 5,
  BS_TUNE_TCD_B_STREAM = 6,
  BS_TUNE_TCD_MCAST = 7
} bs_tune_knob;
int bs_set_tuning(int knob, int value);
int bs_get_tuning(int knob);

/* Words per packed row for reduction length k: ceil(k/32) rounded up to an even
 * number (8-byte rows).  Returns 0 for k <= 0. */
int64_t bs_packed_row_words(int64_t k);

/* ---------------------------------------------------------------------------
 * Bit-packing (Sec. 3.1; timed for activations, not
 * for weights).
 *   in   : device uint8 codes [rows][k], row-major.
 *   out  : device uint32 [bits][rows][bs_packed_row_words(k)], written entirely
 *          (pad words/bits are written as 0).
 *   rows >= 1, k >= 1, bits in [1,8].  For conv activations rows = N*H*W, k = C
 *   (NHWC); for conv weights rows = OC*KH*KW, k = C (OHWI); for dense rows = M or N.
 */
int bs_bitpack(const uint8_t* in, uint32_t* out, int64_t rows, int64_t k, int bits, void* stream);

/* As bs_bitpack, with at most max_ctas thread blocks (0 = library choice).  A small
 * grid (e.g. one block per SM) leaves the SMs room for a kernel running concurrently on
 * another stream — the packing of one layer overlapping the tensor-core conv of another;
 * each thread keeps several 32-byte groups in flight, so the pack stays near HBM speed. */
int bs_bitpack_ex(const uint8_t* in, uint32_t* out, int64_t rows, int64_t k, int bits, int max_ctas, void* stream);

/* Several bs_bitpack problems of one bit width in ONE launch (per 16 descriptors): the
 * activation packing of every layer of a network step (PAPER.md:715 times activation
 * packing per layer) without a launch per tensor.  Each descriptor means exactly what
 * the bs_bitpack arguments mean; outputs must not overlap any input or each other.  All
 * descriptors are validated before anything is launched; count = 0 is a no-op. */
typedef struct bs_pack_desc {
  const uint8_t* in; /* [rows][k] uint8 codes */
  uint32_t* out;     /* [bits][rows][bs_packed_row_words(k)] */
  int64_t rows, k;
} bs_pack_desc;
int bs_bitpack_group(const bs_pack_desc* descs, int count, int bits, void* stream);
/* As bs_bitpack_group with the grid capped at max_ctas 128-thread CTAs (0 = library choice): a
 * capped pack fits beside a running persistent tensor-core conv (one CTA per SM), so later
 * layers can be packed while an earlier layer's conv runs. */
int bs_bitpack_group_ex(const bs_pack_desc* descs, int count, int bits, int max_ctas, void* stream);

/* ---------------------------------------------------------------------------
 * Bitserial dense / matrix multiply (Sec. 3.2 and 6.2.1).
 *   out[m][n] = sum_{k<K} a[m][k] * value(w[n][k])          (int32 [m][n] row-major)
 *   a_packed : device, bs_bitpack of the [m][k] activation codes at a_bits.
 *   w_packed : device, bs_bitpack of the [n][k] weight codes at w_bits.
 *   Both must be packed with the same k.
 */
int bs_bitserial_dense(const uint32_t* a_packed, int a_bits,
                       const uint32_t* w_packed, int w_bits, int w_enc,
                       int32_t* out, int64_t m, int64_t n, int64_t k, void* stream);

int bs_bitserial_dense_ex(const uint32_t* a_packed, int a_bits,
                          const uint32_t* w_packed, int w_bits, int w_enc,
                          int32_t* out, int64_t m, int64_t n, int64_t k,
                          int algo, void* stream);

/* ---------------------------------------------------------------------------
 * Bitserial 2-D convolution, NHWC ("NHWC ... efficient in place
 * convolution", geometry of Table 1).  Cross-correlation (no
 * kernel flip) with zero padding (pad positions are activation code 0, exact in
 * both encodings):
 *   out[b][oy][ox][o] = sum_{ky,kx,c} act[b][oy*sh+ky-ph][ox*sw+kx-pw][c] * value(wt[o][ky][kx][c])
 *   oh = floor((h + 2 ph - kh) / sh) + 1,  ow = floor((w + 2 pw - kw) / sw) + 1.
 *   act_packed : device, bs_bitpack of the NHWC codes viewed as [n*h*w][c].
 *   w_packed   : device, bs_bitpack of the OHWI codes viewed as [oc*kh*kw][c].
 *   out        : device int32 NHWC [n][oh][ow][oc].
 * The convolution is implicit-GEMM (M = n*oh*ow, N = oc, K = kh*kw*c): no lowered
 * (im2col) copy is materialized.
 */
int bs_bitserial_conv2d_nhwc(const uint32_t* act_packed, int a_bits,
                             const uint32_t* w_packed, int w_bits, int w_enc,
                             int32_t* out, int n, int h, int w, int c, int oc, int kh, int kw,
                             int stride_h, int stride_w, int pad_h, int pad_w, void* stream);

int bs_bitserial_conv2d_nhwc_ex(const uint32_t* act_packed, int a_bits,
                                const uint32_t* w_packed, int w_bits, int w_enc,
                                int32_t* out, int n, int h, int w, int c, int oc, int kh, int kw,
                                int stride_h, int stride_w, int pad_h, int pad_w,
                                int algo, void* stream);

/* ---------------------------------------------------------------------------
 * Entries that include activation packing — what the paper times (PAPER.md:715:
 * "we include the cost of bitpacking activations ... but not ... weights").
 * The activation operand is raw uint8 codes (device); the packed activations go to
 * a caller-supplied device workspace of at least *_workspace_bytes() bytes.
 */
int64_t bs_dense_workspace_bytes(int64_t m, int64_t k, int a_bits);
int bs_bitserial_dense_i8(const uint8_t* a, int a_bits,
                          const uint32_t* w_packed, int w_bits, int w_enc,
                          int32_t* out, int64_t m, int64_t n, int64_t k,
                          void* workspace, int64_t workspace_bytes, void* stream);

int64_t bs_conv2d_workspace_bytes(int n, int h, int w, int c, int a_bits);
int bs_bitserial_conv2d_nhwc_i8(const uint8_t* act, int a_bits,
                                const uint32_t* w_packed, int w_bits, int w_enc,
                                int32_t* out, int n, int h, int w, int c, int oc, int kh, int kw,
                                int stride_h, int stride_w, int pad_h, int pad_w,
                                void* workspace, int64_t workspace_bytes, void* stream);

/* Several convolutions from RAW uint8 codes in ONE launch: the batch-1 latency path
 * (small layers "can't amortize the bit-packing costs"; packing is timed,
 * PAPER.md:715).  Each CTA packs the activation codes of its implicit-im2col slab in shared
 * memory (nothing packed is written to HBM), runs AND + POPC per word pair (Eq. 1 inside
 * Eq. 2, bipolar through the exact identity), and the K slices of a tile — the CTAs of one
 * thread-block cluster — are summed through distributed shared memory.  Each descriptor
 * means what the bs_bitserial_conv2d_nhwc_i8 arguments mean (a dense layer is n = 1,
 * h = m, w = 1, c = k, kh = kw = 1); no workspace.  a_bits in [1,4], w_bits in [1,2],
 * unipolar / bipolar weights (BS_ERR_UNSUPPORTED otherwise).  Up to 16 descriptors per
 * launch (more: consecutive launches).  All descriptors are validated first; count = 0 is
 * a no-op.  bs_bitserial_conv2d_nhwc_i8 and bs_bitserial_dense_i8 (m > 8) take this path
 * by themselves for problems of at most 2^24 word-level AND+POPC pairs
 * (M * OC * K_words * A * W). */
typedef struct bs_conv_i8_desc {
  const uint8_t* act;        /* [n][h][w][c] uint8 codes (device) */
  const uint32_t* w_packed;  /* [w_bits][oc*kh*kw][bs_packed_row_words(c)] (bs_bitpack of OHWI) */
  int32_t* out;              /* [n][oh][ow][oc] */
  int w_enc;                 /* BS_UNIPOLAR / BS_BIPOLAR */
  int n, h, w, c, oc, kh, kw, stride_h, stride_w, pad_h, pad_w;
} bs_conv_i8_desc;
int bs_bitserial_conv2d_nhwc_i8_group(const bs_conv_i8_desc* descs, int count, int a_bits, int w_bits, void* stream);

/* ---------------------------------------------------------------------------
 * Tensor-core bitserial (tcgen05.mma on sm_100a, format BS_TC_DEFAULT).  Same operation and
 * operands as bs_bitserial_conv2d_nhwc / bs_bitserial_dense.  The packed activation and
 * weight planes are expanded inside the kernel (weights: by a first kernel into
 * `workspace`) into tensor-core operands whose exact products are the binary dot products
 * popcount(a_i AND w_j) = sum_k a_i[k] w_j[k] (Eq. 1) weighted 2^(i+j)
 * (Eq. 2): per plane pair (BS_TC_I8) or per pair of radix-4 digits of two
 * planes each (BS_TC_F4, see bs_tc_format).
 * Supported: a_bits in [1,4], w_bits in [1,4] (BS_ERR_UNSUPPORTED otherwise).
 * workspace: device, >= *_tc_workspace_bytes() (the larger, I8, size), 16-byte aligned,
 * overwritten.
 */
int64_t bs_conv2d_tc_workspace_bytes(int oc, int kh, int kw, int c, int w_bits);
int bs_bitserial_conv2d_nhwc_tc(const uint32_t* act_packed, int a_bits,
                                const uint32_t* w_packed, int w_bits, int w_enc,
                                int32_t* out, int n, int h, int w, int c, int oc, int kh, int kw,
                                int stride_h, int stride_w, int pad_h, int pad_w,
                                void* workspace, int64_t workspace_bytes, void* stream);
int64_t bs_dense_tc_workspace_bytes(int64_t n, int64_t k, int w_bits);
int bs_bitserial_dense_tc(const uint32_t* a_packed, int a_bits,
                          const uint32_t* w_packed, int w_bits, int w_enc,
                          int32_t* out, int64_t m, int64_t n, int64_t k,
                          void* workspace, int64_t workspace_bytes, void* stream);

/* Operand format of the tensor-core path (same results, bit-exact; different speed):
 *   BS_TC_I8  : every plane pair as tcgen05.mma.kind::i8 on bytes 2^i*a_i (u8) and
 *               2^j*b_j or 2^j*(2b_j-1) (s8), int32 accumulation; 128-element K chunks.
 *   BS_TC_F4  : tcgen05.mma.kind::mxf4 (block-scaled FP4): planes (2d, 2d+1) form one
 *               radix-4 digit, an E2M1 nibble 0.5 * {0..3} (bipolar +-0.5 / +-1.5, the
 *               signed top digit b_lo - 2 b_hi), the digit weights 4^d as UE8M0 block
 *               scales 2^(2d+1): ceil(A/2)*ceil(W/2) MMAs per K step instead of A*W;
 *               FP32 accumulation; 256-element K chunks.  Every product and partial sum
 *               is an integer far below 2^24, so the FP32 result is exact and is
 *               converted to int32 (tools/mxf4_probe.cu checks exactness up to |sum| >
 *               the 737,280 accumulator bound of the configs).
 *   BS_TC_DEFAULT (0): the library's choice (BS_TC_F4).
 * Prepared weights are format-specific: prepare and run with the same format. */
typedef enum { BS_TC_DEFAULT = 0, BS_TC_I8 = 1, BS_TC_F4 = 2 } bs_tc_format;

/* Prepared weights for the tensor-core path.  Weight packing is done ahead of time
 * and is not timed; the expansion of the packed weight planes into the
 * tensor-core operand layout is part of that offline step:
 *   w_tc : device [P][oc][Kpad*B] bytes (dense: [P][n][Kpad*B]); I8: P = w_bits planes,
 *          B = 32 bytes per packed word, Kpad = K words (kh*kw*bs_packed_row_words(c),
 *          dense bs_packed_row_words(k)) rounded up to a multiple of 4; F4: P = ceil(w_bits/2)
 *          radix-4 digits, B = 16, Kpad rounded up to a multiple of 8; the encoding
 *          (unipolar / bipolar / signed) is baked into w_tc.
 *   w_tc_bytes >= bs_conv2d_tc_weight_bytes() / bs_dense_tc_weight_bytes() (0 on bad
 *   arguments).
 */
int64_t bs_conv2d_tc_weight_bytes(int oc, int kh, int kw, int c, int w_bits, int tc_format);
int64_t bs_dense_tc_weight_bytes(int64_t n, int64_t k, int w_bits, int tc_format);
int bs_conv2d_tc_prepare_weights(const uint32_t* w_packed, int w_bits, int w_enc, int oc, int kh, int kw, int c,
                                 int tc_format, int8_t* w_tc, int64_t w_tc_bytes, void* stream);  /* w_enc 0..2 */
int bs_dense_tc_prepare_weights(const uint32_t* w_packed, int w_bits, int w_enc, int64_t n, int64_t k,
                                int tc_format, int8_t* w_tc, int64_t w_tc_bytes, void* stream);

/* Tensor-core conv / dense on prepared weights (one launch: the persistent tcgen05
 * kernel; out as in bs_bitserial_conv2d_nhwc / bs_bitserial_dense, with the value of
 * each code given by a_enc (bs_a_encoding) and w_enc (bs_encoding, the encoding the
 * weights were prepared with)).  a_enc != BS_A_UNSIGNED needs the FP4 format
 * (BS_ERR_UNSUPPORTED on I8). */
int bs_bitserial_conv2d_nhwc_tc_prepared(const uint32_t* act_packed, int a_bits, int a_enc, const int8_t* w_tc,
                                         int w_bits, int w_enc, int tc_format, int32_t* out, int n, int h, int w,
                                         int c, int oc, int kh, int kw, int stride_h, int stride_w, int pad_h,
                                         int pad_w, void* stream);
int bs_bitserial_dense_tc_prepared(const uint32_t* a_packed, int a_bits, int a_enc, const int8_t* w_tc, int w_bits,
                                   int w_enc, int tc_format, int32_t* out, int64_t m, int64_t n, int64_t k,
                                   void* stream);

/* Row-sharded dense with the all-gather FUSED into the epilogue (the
 * multi-GPU GEMM of BASELINE configs[4]): this rank computes its [m][n] row block of C
 * (as bs_bitserial_dense_tc_prepared) and every staged 32x32 output box is stored to
 * `out` AND to each out_peers[d] — device pointers, valid in this process, to this
 * rank's row block inside the other ranks' gathered C buffers (peer memory mapped over
 * NVLink, e.g. torch symmetric memory or CUDA IPC handles).  The transfer overlaps the
 * math tile by tile; no separate collective runs.  The caller orders the exchange: all
 * ranks' launches must complete (a barrier on every rank after the call) before C is
 * read.  npeers in [0, 8]; npeers > 0 needs n % 4 == 0.  npeers = 0 is exactly
 * bs_bitserial_dense_tc_prepared. */
int bs_bitserial_dense_tc_prepared_gather(const uint32_t* a_packed, int a_bits, int a_enc, const int8_t* w_tc,
                                          int w_bits, int w_enc, int tc_format, int32_t* out,
                                          int32_t* const* out_peers, int npeers, int64_t m, int64_t n, int64_t k,
                                          void* stream);

/* The fused all-gather in its NVLS form: as above, but every staged output
 * row segment is stored ONCE, with multimem.st, to out_mc — the MULTICAST address (NVLink
 * SHARP / NVLS multicast object, e.g. torch symmetric memory's multicast_ptr) of this rank's
 * [m][n] row block of the gathered C — and the switch replicates it into every rank's copy
 * (this rank's included).  Egress per rank is its own block once instead of once per peer.
 * The caller creates the multicast mapping, checks that the device supports multicast
 * (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED) and orders the exchange (a barrier on every rank
 * after the call).  n % 4 == 0. */
int bs_bitserial_dense_tc_prepared_multicast(const uint32_t* a_packed, int a_bits, int a_enc, const int8_t* w_tc,
                                             int w_bits, int w_enc, int tc_format, int32_t* out_mc, int64_t m,
                                             int64_t n, int64_t k, void* stream);

/* Several tensor-core convolutions of one precision in ONE persistent launch (per 16
 * problems): the tiles of all problems form one sequence that the SM-resident CTAs walk,
 * so the per-launch prologue, the pipeline fill and the last-wave tail are paid once
 * for the group instead of once per layer (the paper times each layer of ResNet-18,
 * PAPER.md:715-731, Table 1; a network runs them back to back).  Each descriptor is one
 * bs_bitserial_conv2d_nhwc_tc_prepared call (same meaning, layout and ownership of
 * act_packed / w_tc / out; a dense layer is n = 1, h = m, w = 1, c = k, kh = kw = 1).
 * All members share a_bits, w_bits and tc_format; outputs must not overlap inputs or
 * each other.  Every descriptor is validated before anything is launched (the first
 * failing one is reported; nothing runs).  count = 0 is a no-op. */
typedef struct bs_tc_conv_desc {
  const uint32_t* act_packed; /* [a_bits][n*h*w][bs_packed_row_words(c)] (bs_bitpack) */
  const int8_t* w_tc;         /* prepared weights (bs_conv2d_tc_prepare_weights) */
  int32_t* out;               /* [n][oh][ow][oc] */
  int a_enc, w_enc;           /* bs_a_encoding, bs_encoding */
  int n, h, w, c, oc, kh, kw, stride_h, stride_w, pad_h, pad_w;
} bs_tc_conv_desc;
int bs_bitserial_conv2d_nhwc_tc_group(const bs_tc_conv_desc* descs, int count, int a_bits, int w_bits,
                                      int tc_format, void* stream);

/* End-to-end from HOST buffers for several layers, pipelined: per layer the upload of
 * the uint8 NHWC activations (act_host -> act_dev), bit-packing (act_dev -> packed_dev,
 * bs_conv2d_workspace_bytes bytes), the tensor-core conv on prepared weights (-> out_dev)
 * and the download of the int32 output (out_dev -> out_host) — uploads, compute and
 * downloads run on three streams so a layer's download overlaps the next layers'
 * uploads and compute (PCIe is full duplex).  Host buffers should be pinned for the
 * copies to overlap.  Every buffer is the caller's and distinct per layer.  Returns when
 * every output is on the host; validation of all descriptors precedes any copy. */
typedef struct bs_tc_host_desc {
  const uint8_t* act_host; /* [n][h][w][c] uint8 codes (host, pinned) */
  int32_t* out_host;       /* [n][oh][ow][oc] (host, pinned) */
  uint8_t* act_dev;        /* device copy of act_host */
  uint32_t* packed_dev;    /* device workspace for the packed activations */
  int32_t* out_dev;        /* device output */
  const int8_t* w_tc;      /* prepared weights (bs_conv2d_tc_prepare_weights) */
  int a_enc, w_enc;
  int n, h, w, c, oc, kh, kw, stride_h, stride_w, pad_h, pad_w;
} bs_tc_host_desc;
int bs_bitserial_conv2d_nhwc_tc_host_group(const bs_tc_host_desc* descs, int count, int a_bits, int w_bits,
                                           int tc_format, void* stream);

/* The timed step of the paper on the tensor-core path: activation
 * bit-packing (raw uint8 codes -> workspace of *_workspace_bytes() bytes) followed by
 * the tensor-core conv / dense on prepared weights.  Two launches. */
int bs_bitserial_conv2d_nhwc_tc_i8(const uint8_t* act, int a_bits, int a_enc, const int8_t* w_tc, int w_bits,
                                   int w_enc, int tc_format, int32_t* out, int n, int h, int w, int c, int oc,
                                   int kh, int kw, int stride_h, int stride_w, int pad_h, int pad_w,
                                   void* workspace, int64_t workspace_bytes, void* stream);
int bs_bitserial_dense_tc_i8(const uint8_t* a, int a_bits, int a_enc, const int8_t* w_tc, int w_bits, int w_enc,
                             int tc_format, int32_t* out, int64_t m, int64_t n, int64_t k, void* workspace,
                             int64_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * End-to-end entry with HOST activations and HOST output (used for the bench's
 * e2e number).  Copies act_host (uint8 NHWC, pinned or pageable) into the device
 * buffer act_dev, packs it into workspace, convolves into out_dev, copies out_dev
 * into out_host, and synchronizes `stream` before returning (out_host is valid on
 * return).  act_dev must hold n*h*w*c bytes and out_dev n*oh*ow*oc int32.
 */
int bs_bitserial_conv2d_nhwc_host(const uint8_t* act_host, int a_bits,
                                  const uint32_t* w_packed, int w_bits, int w_enc,
                                  int32_t* out_host, int n, int h, int w, int c, int oc, int kh, int kw,
                                  int stride_h, int stride_w, int pad_h, int pad_w,
                                  uint8_t* act_dev, int32_t* out_dev,
                                  void* workspace, int64_t workspace_bytes, void* stream);

/* As above on the tensor-core path with prepared weights (bs_bitserial_conv2d_nhwc_tc_i8). */
int bs_bitserial_conv2d_nhwc_tc_host(const uint8_t* act_host, int a_bits, int a_enc, const int8_t* w_tc, int w_bits,
                                     int w_enc, int tc_format, int32_t* out_host, int n, int h, int w, int c, int oc, int kh, int kw,
                                     int stride_h, int stride_w, int pad_h, int pad_w,
                                     uint8_t* act_dev, int32_t* out_dev,
                                     void* workspace, int64_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Digit-packed operands and the TMA-fed tensor-core kernel (the product path of the
 * timed step).  Eq. 2 is a sum over plane pairs; grouping planes
 * (2d, 2d+1) into radix-4 digits (R21) and storing each element's digit as one
 * 4-bit E2M1 field (value 0.5 * digit) makes the packed tensor a tensor-core operand that
 * TMA moves into shared memory unchanged (R24) — no expansion inside the conv.
 *
 * Digit-packed layout ("digits"): uint8 [D][rows][bs_digit_row_bytes(k)], D = ceil(bits/2),
 * row bytes = 16 * bs_packed_row_words(k) (the bit-plane row length, 4 bits per element
 * per digit); byte b of a row holds elements 2b (low nibble) and 2b+1 (high nibble);
 * elements >= k are 0.  Nibble of digit value v in {-3..3}: (v < 0 ? 8 : 0) | |v|.  Digit
 * d holds planes lo = 2d and hi = 2d+1 (when 2d+1 < bits):
 *     BS_A_UNSIGNED / BS_UNIPOLAR : v = b_lo + 2 b_hi
 *     BS_A_BIPOLAR  / BS_BIPOLAR  : v = (2 b_lo - 1) + 2 (2 b_hi - 1)      (alone: 2 b_lo - 1)
 *     BS_A_SIGNED   / BS_SIGNED   : the digit holding plane bits-1: b_lo - 2 b_hi (alone: -b_lo);
 *                                   lower digits as unsigned
 * so that sum_d 4^d v_d is the code's value.  Activations: bs_digitpack of the [rows][k]
 * codes (conv: rows = n*h*w pixels, k = c).  Weights: bs_*_tcd_prepare_weights of the
 * packed weight planes (untimed, like the weight packing).
 * Supported: bits in [1,4] for both operands; the FP4 exactness bound
 * K * max|a| * max|w| < 2^22 (BS_ERR_OVERFLOW); conv geometry that the TMA im2col mode
 * encodes: pad <= 128, stride <= 8, (out-1)*stride - pad - (in-1) in [-128, 127]
 * (BS_ERR_UNSUPPORTED otherwise).  All pointers device, 16-byte aligned.
 */
int64_t bs_digit_row_bytes(int64_t k);
/* in [rows][k] uint8 codes -> out [ceil(bits/2)][rows][bs_digit_row_bytes(k)]; enc is a
 * bs_a_encoding (or the same value of a bs_encoding for weight codes).  HBM-bound: 1 byte
 * read + ceil(bits/2)/2 bytes written per element. */
int bs_digitpack(const uint8_t* in, uint8_t* out, int64_t rows, int64_t k, int bits, int enc, void* stream);
typedef struct bs_digit_pack_desc {
  const uint8_t* in; /* [rows][k] codes */
  uint8_t* out;      /* [ceil(bits/2)][rows][bs_digit_row_bytes(k)] */
  int64_t rows, k;
} bs_digit_pack_desc;
/* Several tensors of one bit width and encoding in ONE launch (the bench step's packing). */
int bs_digitpack_group(const bs_digit_pack_desc* descs, int count, int bits, int enc, void* stream);

/* Weight digits from PACKED weight planes (bs_bitpack of OHWI codes, or of [n][k] for dense):
 * [ceil(w_bits/2)][oc][R] bytes, each row R = kh*kw*bs_digit_row_bytes(c) bytes of digits
 * (dense: bs_digit_row_bytes(k)) zero-padded to the next multiple of 128 bytes; channel padding
 * inside each tap is 0. */
int64_t bs_conv2d_tcd_weight_bytes(int oc, int kh, int kw, int c, int w_bits);
int64_t bs_dense_tcd_weight_bytes(int64_t n, int64_t k, int w_bits);
int bs_conv2d_tcd_prepare_weights(const uint32_t* w_packed, int w_bits, int w_enc, int oc, int kh, int kw, int c,
                                  uint8_t* w_dig, int64_t w_dig_bytes, void* stream);
int bs_dense_tcd_prepare_weights(const uint32_t* w_packed, int w_bits, int w_enc, int64_t n, int64_t k,
                                 uint8_t* w_dig, int64_t w_dig_bytes, void* stream);

/* Conv2d NHWC / dense on digit-packed activations and prepared weight digits: one
 * persistent warp-specialized launch; TMA im2col (conv) or tiled (dense) loads of the
 * activation digits, TMA loads of the weight digits, tcgen05.mma kind::mxf4 with the digit
 * weights 4^d as UE8M0 block scales, FP32 accumulation in TMEM (exact below 2^22), F2I,
 * TMA-store epilogue.  a_enc / w_enc are the encodings the operands were packed with (they
 * set the exactness bound).  out: int32 [n][oh][ow][oc] / [m][n]. */
int bs_bitserial_conv2d_nhwc_tcd(const uint8_t* act_dig, int a_bits, int a_enc, const uint8_t* w_dig, int w_bits,
                                 int w_enc, int32_t* out, int n, int h, int w, int c, int oc, int kh, int kw,
                                 int stride_h, int stride_w, int pad_h, int pad_w, void* stream);
int bs_bitserial_dense_tcd(const uint8_t* a_dig, int a_bits, int a_enc, const uint8_t* w_dig, int w_bits, int w_enc,
                           int32_t* out, int64_t m, int64_t n, int64_t k, void* stream);
typedef struct bs_tcd_conv_desc {
  const uint8_t* act_dig; /* [ceil(a_bits/2)][n*h*w][bs_digit_row_bytes(c)] */
  const uint8_t* w_dig;   /* bs_conv2d_tcd_prepare_weights */
  int32_t* out;           /* [n][oh][ow][oc] */
  int a_enc, w_enc;
  int n, h, w, c, oc, kh, kw, stride_h, stride_w, pad_h, pad_w;
} bs_tcd_conv_desc;
/* Several convolutions of one (a_bits, w_bits) in one launch per 16 (tiles concatenated). */
int bs_bitserial_conv2d_nhwc_tcd_group(const bs_tcd_conv_desc* descs, int count, int a_bits, int w_bits,
                                       void* stream);

/* ---------------------------------------------------------------------------
 * Window layout and the windowed tensor-core conv (reading R26).  The conv's
 * zero-padded input (padding = value 0, R20) is split into the stride's phases
 * (py, px) that its taps read, each on a phase grid of hg x wg pixels per image:
 *   s = stride (stride_h == stride_w, 1 or 2), oh/ow the output extent,
 *   hg = oh + (kh-1)/s, wg = ow + (kw-1)/s; phase pixel (gy, gx) = padded pixel
 *   (gy*s + py, gx*s + px); q = (img*hg + gy)*wg + gx; output (oy, ox) with tap (ky, kx)
 *   reads phase (ky%s, kx%s) at q_out + (ky/s)*wg + kx/s, q_out = (img*hg + oy)*wg + ox.
 * Layout ("windows"): uint8 [D][nph][cw/2][pstride][32], D = ceil(bits/2), nph = the phases
 * some tap reads (ascending py*s+px), cw = bs_packed_row_words(c) 32-channel slabs taken in
 * pairs, pstride = ceil8(n*hg*wg + ceil8(128 + (kh-1)/s*wg + (kw-1)/s + 8)) grid positions (a
 * zero tail); 32-byte row (d, phase, pair p, q) holds the digit-packed bytes (R24) of channels
 * [64p, 64p+32) then [64p+32, 64p+64) of the input pixel the position maps to — the two 16-byte
 * halves exchanged when bit 2 of q is set (the 32-byte shared-memory swizzle the tensor core
 * reads) — and zeros for padding, grid positions past the image and the tail.
 * Because a 128-row tile of consecutive grid positions reads every tap's operand from one
 * contiguous window per (digit, phase, slab), the conv kernel moves the operands with plain
 * bulk copies and the tensor core reads each tap as a shifted view (no im2col, no gather).
 * The packing is the timed activation-packing step emitting this layout.
 * Supported: stride_h == stride_w in {1, 2}; wg <= 128; oc % 4 == 0;
 * bits in [1,4]; the FP4 exactness bound (BS_ERR_OVERFLOW); one pipeline stage (every activation
 * digit's windows of a 64-channel slab pair, plus the streamed weight digits of every tap when the
 * filter block does not stay resident) must fit shared memory — with three or four bits on both
 * operands a wide stride-2 or many-channel layer can exceed it; BS_ERR_UNSUPPORTED otherwise.
 */
int64_t bs_tcw_act_bytes(int n, int h, int w, int c, int kh, int kw, int stride, int pad_h, int pad_w, int bits);
/* in: uint8 codes [n][h][w][c]; out: the window layout (out_bytes >= bs_tcw_act_bytes); every
 * byte of it is written (no clearing needed). */
int bs_digitpack_win(const uint8_t* in, uint8_t* out, int64_t out_bytes, int n, int h, int w, int c, int kh, int kw,
                     int stride, int pad_h, int pad_w, int bits, int enc, void* stream);
typedef struct bs_win_pack_desc {
  const uint8_t* in; /* [n][h][w][c] codes */
  uint8_t* out;      /* window layout of the conv below */
  int64_t out_bytes;
  int n, h, w, c, kh, kw, stride, pad_h, pad_w;
} bs_win_pack_desc;
/* Several tensors of one bit width and encoding in ONE launch (the bench step's packing). */
int bs_digitpack_win_group(const bs_win_pack_desc* descs, int count, int bits, int enc, void* stream);
/* Window-path weight digits from PACKED OHWI weight planes (bs_bitpack of [oc*kh*kw][c]):
 * [nblk][cw/2][ceil(w_bits/2)][kh*kw][bn][32] bytes, bn = 64 if oc <= 64 else 128,
 * nblk = ceil(oc/bn): one 64-channel slab pair of one filter block is contiguous; filter row r's
 * two 16-byte halves are exchanged when bit 2 of r is set; filters past oc and channels past c
 * are 0.  Untimed, like the weight packing. */
int64_t bs_conv2d_tcw_weight_bytes(int oc, int kh, int kw, int c, int w_bits);
int bs_conv2d_tcw_prepare_weights(const uint32_t* w_packed, int w_bits, int w_enc, int oc, int kh, int kw, int c,
                                  uint8_t* w_win, int64_t w_win_bytes, void* stream);
/* Conv2d NHWC on window-layout activations and window-path weights: one persistent
 * warp-specialized launch (bulk copies of the windows and weights, tcgen05.mma kind::mxf4 on
 * shifted shared-memory views, FP32 accumulation in TMEM, F2I, one TMA store per valid output
 * row segment).  out: int32 [n][oh][ow][oc]. */
int bs_bitserial_conv2d_nhwc_tcw(const uint8_t* act_win, int a_bits, int a_enc, const uint8_t* w_win, int w_bits,
                                 int w_enc, int32_t* out, int n, int h, int w, int c, int oc, int kh, int kw,
                                 int stride_h, int stride_w, int pad_h, int pad_w, void* stream);
typedef struct bs_tcw_conv_desc {
  const uint8_t* act_win; /* bs_digitpack_win */
  const uint8_t* w_win;   /* bs_conv2d_tcw_prepare_weights */
  int32_t* out;           /* [n][oh][ow][oc] */
  int a_enc, w_enc;
  int n, h, w, c, oc, kh, kw, stride_h, stride_w, pad_h, pad_w;
} bs_tcw_conv_desc;
/* Several convolutions of one (a_bits, w_bits) in one launch per 16 (tiles concatenated). */
int bs_bitserial_conv2d_nhwc_tcw_group(const bs_tcw_conv_desc* descs, int count, int a_bits, int w_bits,
                                       void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BITSERIAL_H_ */
