// abi.cu — the C ABI declared in include/bitserial.h: argument validation (all of it
// before any launch), kernel selection, launch on the caller's stream.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/bitserial.h"
#include "kernels.h"

namespace bs {
static std::atomic<int64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
int64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

std::atomic<int> g_tune[kTuneCount];
int tuning(int knob) { return knob >= 0 && knob < kTuneCount ? g_tune[knob].load(std::memory_order_relaxed) : 0; }

constexpr int kMaxDevices = 64;
std::atomic<int> g_sms[kMaxDevices];
int device_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) dev = 0;
  if (dev < kMaxDevices)
    if (int n = g_sms[dev].load(std::memory_order_relaxed)) return n;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;  // B200
  if (dev < kMaxDevices) g_sms[dev].store(n, std::memory_order_relaxed);
  return n;
}
}  // namespace bs

namespace {

thread_local char g_last_error[512] = "";

int fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return status;
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return BS_OK;
  if (e == cudaErrorNotSupported) return fail(BS_ERR_UNSUPPORTED, "%s: no kernel instantiation for these arguments", where);
  return fail(BS_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int64_t row_words(int64_t k) {
  if (k <= 0) return 0;
  const int64_t kw = (k + 31) / 32;
  return kw + (kw & 1);
}

int check_bits(int a_bits, int w_bits, int w_enc, const char* fn) {
  if (a_bits < 1 || a_bits > 8) return fail(BS_ERR_INVALID_ARG, "%s: a_bits=%d not in [1,8]", fn, a_bits);
  if (w_bits < 1 || w_bits > 8) return fail(BS_ERR_INVALID_ARG, "%s: w_bits=%d not in [1,8]", fn, w_bits);
  if (w_enc != BS_UNIPOLAR && w_enc != BS_BIPOLAR) return fail(BS_ERR_INVALID_ARG, "%s: bad encoding %d", fn, w_enc);
  return BS_OK;
}

int check_bound(int64_t k, int a_bits, int w_bits, const char* fn) {
  const double bound = double(k) * double((1 << a_bits) - 1) * double((1 << w_bits) - 1);
  if (bound >= 2147483648.0) return fail(BS_ERR_OVERFLOW, "%s: K*(2^A-1)*(2^W-1) = %.0f >= 2^31", fn, bound);
  return BS_OK;
}

// Tensor-core path encodings: weights unipolar / bipolar / signed (prepared offline);
// activations unsigned / bipolar / signed on the FP4 format (the I8 format's A operand
// is unsigned u8: unsigned activations only).
int check_tc_enc(int a_enc, int w_enc, int tc_format, const char* fn) {
  if (a_enc < BS_A_UNSIGNED || a_enc > BS_A_SIGNED) return fail(BS_ERR_INVALID_ARG, "%s: bad a_enc %d", fn, a_enc);
  if (w_enc < BS_UNIPOLAR || w_enc > BS_SIGNED) return fail(BS_ERR_INVALID_ARG, "%s: bad w_enc %d", fn, w_enc);
  if (a_enc != BS_A_UNSIGNED && bs::tc_resolve_format(tc_format) != bs::kTcF4)
    return fail(BS_ERR_UNSUPPORTED, "%s: bipolar / signed activations need the FP4 tensor-core format", fn);
  return BS_OK;
}

int64_t max_abs_code(int bits, int enc) {  // largest |value| of a code (signed: -2^(bits-1))
  return enc == 2 ? (int64_t(1) << (bits - 1)) : (int64_t(1) << bits) - 1;
}

int check_format(int tc_format, const char* fn) {
  if (tc_format < BS_TC_DEFAULT || tc_format > BS_TC_F4)
    return fail(BS_ERR_INVALID_ARG, "%s: bad tensor-core format %d", fn, tc_format);
  return BS_OK;
}

// The FP4 tensor-core format accumulates in FP32 and converts with the 1.5*2^23 trick:
// exact while |out| < 2^22 (bound below); the I8 format is exact to the int32 bound.
int check_tc_bound(int64_t k, int a_bits, int w_bits, int tc_format, const char* fn, int a_enc = 0, int w_enc = 0) {
  if (bs::tc_resolve_format(tc_format) != bs::kTcF4) return BS_OK;
  const double bound = double(k) * double(max_abs_code(a_bits, a_enc)) * double(max_abs_code(w_bits, w_enc));
  if (bound >= 4194304.0)
    return fail(BS_ERR_OVERFLOW, "%s: K*(2^A-1)*(2^W-1) = %.0f >= 2^22 (FP4 format exactness bound; use BS_TC_I8)",
                fn, bound);
  return BS_OK;
}

int check_algo(int algo, const char* fn) {
  if (algo < BS_ALGO_AUTO || algo > BS_ALGO_TC) return fail(BS_ERR_INVALID_ARG, "%s: bad algo %d", fn, algo);
  return BS_OK;
}

constexpr int64_t kMaxRows = (int64_t(1) << 31) - 257;  // output rows (M) a launch may index

struct ConvArgs {
  int n, h, w, c, oc, kh, kw, sh, sw, ph, pw;
};

int conv_out(int in, int k, int s, int p) {
  const int span = in + 2 * p - k;
  return span < 0 ? 0 : span / s + 1;
}

int check_conv(const ConvArgs& g, int a_bits, int w_bits, int w_enc, const char* fn) {
  if (int s = check_bits(a_bits, w_bits, w_enc, fn)) return s;
  if (g.n <= 0 || g.h <= 0 || g.w <= 0 || g.c <= 0 || g.oc <= 0 || g.kh <= 0 || g.kw <= 0)
    return fail(BS_ERR_SHAPE, "%s: non-positive extent", fn);
  if (g.sh < 1 || g.sw < 1) return fail(BS_ERR_INVALID_ARG, "%s: stride < 1", fn);
  if (g.ph < 0 || g.pw < 0) return fail(BS_ERR_INVALID_ARG, "%s: pad < 0", fn);
  if (conv_out(g.h, g.kh, g.sh, g.ph) <= 0 || conv_out(g.w, g.kw, g.sw, g.pw) <= 0)
    return fail(BS_ERR_SHAPE, "%s: empty output (kernel larger than padded input)", fn);
  if (int64_t(g.n) * g.h * g.w > (int64_t(1) << 31) - 1) return fail(BS_ERR_SHAPE, "%s: too many pixels", fn);
  // output rows M = n*oh*ow index the kernels' 32-bit row arithmetic (fast division, TMA
  // coordinates) up to a tile past the end; oh, ow can exceed h, w when padded
  if (int64_t(g.n) * conv_out(g.h, g.kh, g.sh, g.ph) * conv_out(g.w, g.kw, g.sw, g.pw) > kMaxRows)
    return fail(BS_ERR_SHAPE, "%s: more than 2^31 - 257 output pixels", fn);
  if (int64_t(g.kh) * g.kw * row_words(g.c) > (int64_t(1) << 30)) return fail(BS_ERR_SHAPE, "%s: reduction too long", fn);
  return check_bound(int64_t(g.kh) * g.kw * g.c, a_bits, w_bits, fn);
}

bs::ConvProblem make_conv(const uint32_t* act, int a_bits, const uint32_t* wt, int w_bits, int w_enc, int32_t* out,
                          const ConvArgs& g) {
  bs::ConvProblem p{};
  p.act = act; p.wt = wt; p.out = out;
  p.n = g.n; p.h = g.h; p.w = g.w; p.kw_a = int(row_words(g.c));
  p.oc = g.oc; p.kh = g.kh; p.kwid = g.kw;
  p.sh = g.sh; p.sw = g.sw; p.ph = g.ph; p.pw = g.pw;
  p.oh = conv_out(g.h, g.kh, g.sh, g.ph); p.ow = conv_out(g.w, g.kw, g.sw, g.pw);
  p.a_bits = a_bits; p.w_bits = w_bits; p.bipolar = w_enc == BS_BIPOLAR;
  p.a_enc = BS_A_UNSIGNED;
  p.c_tap = g.c;
  p.act_plane = int64_t(g.n) * g.h * g.w * p.kw_a;
  p.M = int64_t(g.n) * p.oh * p.ow;
  p.kp = int64_t(g.kh) * g.kw * p.kw_a;
  p.one = 1;
  p.ksplit = 1;
  return p;
}

// The tensor-core path for the packed-weight entries (three-call boundary): FP4 digits with
// the weight planes expanded inside the kernel; needs A, W <= 4, unipolar / bipolar weights
// and the FP4 format's exactness bound K * (2^A - 1) * (2^W - 1) < 2^22.
bool tc_auto_ok(const bs::ConvProblem& p) {
  const int64_t k = int64_t(p.kh) * p.kwid * p.c_tap;
  return bs::tc_supported(p.a_bits, p.w_bits) && p.bipolar <= 1 &&
         double(k) * double((1 << p.a_bits) - 1) * double((1 << p.w_bits) - 1) < 4194304.0;
}

int launch_conv(const bs::ConvProblem& p, int algo, cudaStream_t s, const char* fn) {
  if (algo == BS_ALGO_GEMV) return fail(BS_ERR_UNSUPPORTED, "%s: GEMV algo applies to dense only", fn);
  if (algo == BS_ALGO_TC || (algo == BS_ALGO_AUTO && tc_auto_ok(p))) {
    if (!tc_auto_ok(p))
      return fail(BS_ERR_UNSUPPORTED, "%s: tensor-core path needs A, W <= 4, unipolar/bipolar weights and "
                  "K*(2^A-1)*(2^W-1) < 2^22", fn);
    return cuda_status(bs::launch_tc_conv_raw(p, s), fn);
  }
  const bs::Algo a = algo == BS_ALGO_POPC_LIT ? bs::Algo::PopcLit : bs::Algo::Popc;
  return cuda_status(bs::launch_popc_conv(p, a, s), fn);
}

// Small problems (batch-1 layers) run as ONE launch with the activation packing fused
// (small_conv.cu): below ~16 M word-level AND+POPC pairs a persistent tensor-core launch
// plus a separate pack launch costs more than the whole problem on the integer pipes.
constexpr int64_t kSmallWordOps = int64_t(16) << 20;
bool use_small(const bs::ConvProblem& p) {
  return bs::small_supported(p.a_bits, p.w_bits) && p.bipolar != 2 && p.kh * p.kwid <= 64 &&
         p.M * p.oc * p.kp * p.a_bits * p.w_bits <= kSmallWordOps;
}

int dense_core(const uint32_t* a_packed, const uint8_t* a_codes, int a_bits, const uint32_t* w_packed, int w_bits,
               int w_enc, int32_t* out, int64_t m, int64_t n, int64_t k, int algo, cudaStream_t s, const char* fn) {
  const int64_t kwp = row_words(k);
  const bool gemv_ok = bs::gemv_supported(m, k, a_bits, w_bits);
  if (algo == BS_ALGO_GEMV && !gemv_ok) return fail(BS_ERR_UNSUPPORTED, "%s: GEMV needs m <= 8 and A in {1,2,4}, W in {1,2}", fn);
  if (algo == BS_ALGO_GEMV || (algo == BS_ALGO_AUTO && gemv_ok))
    return cuda_status(bs::launch_gemv(a_packed, a_codes, a_bits, w_packed, w_bits, w_enc == BS_BIPOLAR, out, m, n, k,
                                       kwp, s), fn);
  if (a_codes) return fail(BS_ERR_UNSUPPORTED, "%s: internal: codes path needs GEMV", fn);
  if (m > kMaxRows || n > (int64_t(1) << 31) - 1) return fail(BS_ERR_SHAPE, "%s: m or n too large", fn);
  ConvArgs g{1, int(m), 1, int(k), int(n), 1, 1, 1, 1, 0, 0};  // dense = 1x1 conv over m "pixels"
  bs::ConvProblem p = make_conv(a_packed, a_bits, w_packed, w_bits, w_enc, out, g);
  return launch_conv(p, algo, s, fn);
}

int check_dense(const void* a, const uint32_t* w, const int32_t* out, int a_bits, int w_bits, int w_enc, int64_t m,
                int64_t n, int64_t k, const char* fn) {
  if (!a || !w || !out) return fail(BS_ERR_NULL, "%s: NULL tensor pointer", fn);
  if (int st = check_bits(a_bits, w_bits, w_enc, fn)) return st;
  if (m <= 0 || n <= 0 || k <= 0) return fail(BS_ERR_SHAPE, "%s: m, n, k must be >= 1", fn);
  if (!aligned16(a) || !aligned16(w) || !aligned16(out)) return fail(BS_ERR_ALIGN, "%s: pointers must be 16-byte aligned", fn);
  return check_bound(k, a_bits, w_bits, fn);
}

// Side streams and events of the pipelined host-buffer entry, kept per thread (created on
// first use, re-created when the thread's current device changes, grown to the largest
// event count seen) instead of being created and destroyed on every call.
struct HostPipe {
  int dev = -1;
  cudaStream_t in = nullptr, out = nullptr;
  std::vector<cudaEvent_t> ev;
  void release() {
    for (auto& x : ev)
      if (x) cudaEventDestroy(x);
    ev.clear();
    if (in) cudaStreamDestroy(in);
    if (out) cudaStreamDestroy(out);
    in = out = nullptr;
    dev = -1;
  }
  cudaError_t prepare(size_t events) {
    int d = 0;
    if (cudaError_t e = cudaGetDevice(&d)) return e;
    if (d != dev) {
      release();
      if (cudaError_t e = cudaStreamCreateWithFlags(&in, cudaStreamNonBlocking)) return e;
      if (cudaError_t e = cudaStreamCreateWithFlags(&out, cudaStreamNonBlocking)) return e;
      dev = d;
    }
    while (ev.size() < events) {
      cudaEvent_t x = nullptr;
      if (cudaError_t e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming)) return e;
      ev.push_back(x);
    }
    return cudaSuccess;
  }
  ~HostPipe() { release(); }
};
HostPipe& host_pipe() {
  thread_local HostPipe p;
  return p;
}


// ---- digit path (digit.cu, tcd_conv.cu)
// TMA im2col limits: padding corners in [-128, 127], traversal stride <= 8.
int check_tcd_conv(const ConvArgs& g, int a_bits, int w_bits, int a_enc, int w_enc, const char* fn) {
  if (int st = check_tc_enc(a_enc, w_enc, BS_TC_F4, fn)) return st;
  if (int st = check_conv(g, a_bits, w_bits, BS_UNIPOLAR, fn)) return st;
  if (int st = check_tc_bound(int64_t(g.kh) * g.kw * g.c, a_bits, w_bits, BS_TC_F4, fn, a_enc, w_enc)) return st;
  if (!bs::tc_supported(a_bits, w_bits)) return fail(BS_ERR_UNSUPPORTED, "%s: a_bits in [1,4], w_bits in [1,4]", fn);
  const int oh = conv_out(g.h, g.kh, g.sh, g.ph), ow = conv_out(g.w, g.kw, g.sw, g.pw);
  const int up_w = (ow - 1) * g.sw - g.pw - (g.w - 1), up_h = (oh - 1) * g.sh - g.ph - (g.h - 1);
  if (g.ph > 128 || g.pw > 128 || up_w < -128 || up_w > 127 || up_h < -128 || up_h > 127 || g.sh > 8 || g.sw > 8)
    return fail(BS_ERR_UNSUPPORTED, "%s: TMA im2col needs padding <= 128, stride <= 8 and kernel extent <= pad + 129",
                fn);
  return BS_OK;
}

bs::TcdProblem make_tcd(const uint8_t* act, const uint8_t* wdig, int32_t* out, int a_bits, int w_bits,
                        const ConvArgs& g) {
  bs::TcdProblem p{};
  p.act = act; p.wdig = wdig; p.out = out;
  p.n = g.n; p.h = g.h; p.w = g.w; p.c = g.c; p.oc = g.oc; p.kh = g.kh; p.kw = g.kw;
  p.sh = g.sh; p.sw = g.sw; p.ph = g.ph; p.pw = g.pw;
  p.oh = conv_out(g.h, g.kh, g.sh, g.ph); p.ow = conv_out(g.w, g.kw, g.sw, g.pw);
  p.a_digits = (a_bits + 1) / 2; p.w_digits = (w_bits + 1) / 2;
  p.dense = 0;
  return p;
}

// ---- window path (digit.cu, tcw_conv.cu)
int check_tcw_geom(const ConvArgs& g, int oc, bs::TcwGeom& G, const char* fn) {
  if (!bs::tcw_geom(g.n, g.h, g.w, g.c, oc, g.kh, g.kw, g.sh, g.sw, g.ph, g.pw, G))
    return fail(BS_ERR_UNSUPPORTED,
                "%s: the window layout needs stride_h == stride_w in {1,2} and output rows of at most 128 grid "
                "positions", fn);
  return BS_OK;
}

int check_tcw_conv(const ConvArgs& g, int a_bits, int w_bits, int a_enc, int w_enc, const char* fn) {
  if (int st = check_tc_enc(a_enc, w_enc, BS_TC_F4, fn)) return st;
  if (int st = check_conv(g, a_bits, w_bits, BS_UNIPOLAR, fn)) return st;
  if (int st = check_tc_bound(int64_t(g.kh) * g.kw * g.c, a_bits, w_bits, BS_TC_F4, fn, a_enc, w_enc)) return st;
  if (!bs::tc_supported(a_bits, w_bits)) return fail(BS_ERR_UNSUPPORTED, "%s: a_bits in [1,4], w_bits in [1,4]", fn);
  bs::TcwGeom G;
  if (int st = check_tcw_geom(g, g.oc, G, fn)) return st;
  if (g.oc % 4 != 0) return fail(BS_ERR_UNSUPPORTED, "%s: oc must be a multiple of 4", fn);
  return BS_OK;
}

// The window-path launcher refuses (cudaErrorNotSupported) only when one pipeline stage does not
// fit shared memory (the arguments were validated before).
int tcw_status(cudaError_t e, const char* fn) {
  if (e == cudaErrorNotSupported)
    return fail(BS_ERR_UNSUPPORTED,
                "%s: one window-path stage (every digit's windows of a 64-channel slab pair and the streamed "
                "weight digits of every tap) exceeds shared memory for these bit widths and geometry", fn);
  return cuda_status(e, fn);
}

bs::TcwProblem make_tcw(const uint8_t* act, const uint8_t* wt, int32_t* out, int a_bits, int w_bits,
                        const ConvArgs& g) {
  bs::TcwProblem p{};
  p.act = act; p.wt = wt; p.out = out;
  p.n = g.n; p.h = g.h; p.w = g.w; p.c = g.c; p.oc = g.oc; p.kh = g.kh; p.kw = g.kw;
  p.sh = g.sh; p.sw = g.sw; p.ph = g.ph; p.pw = g.pw;
  p.a_digits = (a_bits + 1) / 2; p.w_digits = (w_bits + 1) / 2;
  return p;
}

}  // namespace

extern "C" {

int bs_abi_version(void) { return BS_ABI_VERSION; }

const char* bs_status_string(int status) {
  switch (status) {
    case BS_OK: return "BS_OK";
    case BS_ERR_NULL: return "BS_ERR_NULL";
    case BS_ERR_INVALID_ARG: return "BS_ERR_INVALID_ARG";
    case BS_ERR_UNSUPPORTED: return "BS_ERR_UNSUPPORTED";
    case BS_ERR_SHAPE: return "BS_ERR_SHAPE";
    case BS_ERR_ALIGN: return "BS_ERR_ALIGN";
    case BS_ERR_OVERFLOW: return "BS_ERR_OVERFLOW";
    case BS_ERR_CUDA: return "BS_ERR_CUDA";
    case BS_ERR_WORKSPACE: return "BS_ERR_WORKSPACE";
    default: return "BS_ERR_UNKNOWN";
  }
}

const char* bs_last_error(void) { return g_last_error; }

int64_t bs_packed_row_words(int64_t k) { return row_words(k); }

int64_t bs_kernel_launches(void) { return bs::launch_count(); }

int bs_set_tuning(int knob, int value) {
  const char* fn = "bs_set_tuning";
  switch (knob) {
    case BS_TUNE_TC_TILE_N:
      if (value != 0 && value != 64 && value != 128 && value != 224)
        return fail(BS_ERR_INVALID_ARG, "%s: tile width %d", fn, value);
      break;
    case BS_TUNE_TC_EPILOGUE:
    case BS_TUNE_TC_GROUP_SPLIT:
      if (value != 0 && value != 1) return fail(BS_ERR_INVALID_ARG, "%s: value %d not 0 or 1", fn, value);
      break;
    case BS_TUNE_TC_B_SLOTS:
      if (value != 0 && (value < 2 || value > 32)) return fail(BS_ERR_INVALID_ARG, "%s: B slots %d", fn, value);
      break;
    case BS_TUNE_TCD_A_SRC:
      if (value < 0 || value > 2) return fail(BS_ERR_INVALID_ARG, "%s: value %d not in {0,1,2}", fn, value);
      break;
    case BS_TUNE_TCD_MCAST:
      if (value < 0 || value > 2) return fail(BS_ERR_INVALID_ARG, "%s: value %d not in {0,1,2}", fn, value);
      break;
    case BS_TUNE_TCD_B_STREAM:
      if (value != 0 && value != 1) return fail(BS_ERR_INVALID_ARG, "%s: value %d not 0 or 1", fn, value);
      break;
    case BS_TUNE_SMALL_KSPLIT:
      if (value != 0 && value != 1 && value != 2 && value != 4 && value != 8)
        return fail(BS_ERR_INVALID_ARG, "%s: K split %d not in {1,2,4,8}", fn, value);
      break;
    default:
      return fail(BS_ERR_INVALID_ARG, "%s: unknown knob %d", fn, knob);
  }
  bs::g_tune[knob].store(value, std::memory_order_relaxed);
  return BS_OK;
}

int bs_get_tuning(int knob) { return bs::tuning(knob); }

int bs_bitpack(const uint8_t* in, uint32_t* out, int64_t rows, int64_t k, int bits, void* stream) {
  return bs_bitpack_ex(in, out, rows, k, bits, 0, stream);
}

int bs_bitpack_ex(const uint8_t* in, uint32_t* out, int64_t rows, int64_t k, int bits, int max_ctas, void* stream) {
  const char* fn = "bs_bitpack";
  if (!in || !out) return fail(BS_ERR_NULL, "%s: NULL tensor pointer", fn);
  if (bits < 1 || bits > 8) return fail(BS_ERR_INVALID_ARG, "%s: bits=%d not in [1,8]", fn, bits);
  if (rows <= 0 || k <= 0) return fail(BS_ERR_SHAPE, "%s: rows and k must be >= 1", fn);
  if (!aligned16(in) || !aligned16(out)) return fail(BS_ERR_ALIGN, "%s: pointers must be 16-byte aligned", fn);
  if (max_ctas < 0) return fail(BS_ERR_INVALID_ARG, "%s: max_ctas < 0", fn);
  return cuda_status(bs::launch_bitpack(in, out, rows, k, row_words(k), bits, static_cast<cudaStream_t>(stream),
                                        max_ctas), fn);
}

int bs_bitpack_group(const bs_pack_desc* descs, int count, int bits, void* stream) {
  return bs_bitpack_group_ex(descs, count, bits, 0, stream);
}

int bs_bitpack_group_ex(const bs_pack_desc* descs, int count, int bits, int max_ctas, void* stream) {
  const char* fn = "bs_bitpack_group";
  if (max_ctas < 0) return fail(BS_ERR_INVALID_ARG, "%s: max_ctas < 0", fn);
  if (count < 0 || count > (1 << 20)) return fail(BS_ERR_SHAPE, "%s: count out of range", fn);
  if (count == 0) return BS_OK;
  if (!descs) return fail(BS_ERR_NULL, "%s: NULL descriptor array", fn);
  if (bits < 1 || bits > 8) return fail(BS_ERR_INVALID_ARG, "%s: bits=%d not in [1,8]", fn, bits);
  std::vector<bs::PackSeg> segs(static_cast<size_t>(count));
  for (int q = 0; q < count; ++q) {
    const bs_pack_desc& d = descs[q];
    if (!d.in || !d.out) return fail(BS_ERR_NULL, "%s: NULL tensor pointer in descriptor %d", fn, q);
    if (d.rows <= 0 || d.k <= 0) return fail(BS_ERR_SHAPE, "%s: descriptor %d: rows and k must be >= 1", fn, q);
    if (!aligned16(d.in) || !aligned16(d.out))
      return fail(BS_ERR_ALIGN, "%s: descriptor %d: pointers must be 16-byte aligned", fn, q);
    segs[q] = bs::PackSeg{d.in, d.out, d.rows, d.k, row_words(d.k), 0, -1, 0};
  }
  return cuda_status(bs::launch_bitpack_group(segs.data(), count, bits, static_cast<cudaStream_t>(stream), max_ctas),
                     fn);
}

int bs_bitserial_dense_ex(const uint32_t* a_packed, int a_bits, const uint32_t* w_packed, int w_bits, int w_enc,
                          int32_t* out, int64_t m, int64_t n, int64_t k, int algo, void* stream) {
  const char* fn = "bs_bitserial_dense";
  if (int st = check_dense(a_packed, w_packed, out, a_bits, w_bits, w_enc, m, n, k, fn)) return st;
  if (int st = check_algo(algo, fn)) return st;
  return dense_core(a_packed, nullptr, a_bits, w_packed, w_bits, w_enc, out, m, n, k, algo,
                    static_cast<cudaStream_t>(stream), fn);
}

int bs_bitserial_dense(const uint32_t* a_packed, int a_bits, const uint32_t* w_packed, int w_bits, int w_enc,
                       int32_t* out, int64_t m, int64_t n, int64_t k, void* stream) {
  return bs_bitserial_dense_ex(a_packed, a_bits, w_packed, w_bits, w_enc, out, m, n, k, BS_ALGO_AUTO, stream);
}

int64_t bs_dense_workspace_bytes(int64_t m, int64_t k, int a_bits) {
  if (m <= 0 || k <= 0 || a_bits < 1 || a_bits > 8) return 0;
  return int64_t(a_bits) * m * row_words(k) * 4;
}

int bs_bitserial_dense_i8(const uint8_t* a, int a_bits, const uint32_t* w_packed, int w_bits, int w_enc, int32_t* out,
                          int64_t m, int64_t n, int64_t k, void* workspace, int64_t workspace_bytes, void* stream) {
  const char* fn = "bs_bitserial_dense_i8";
  if (int st = check_dense(a, w_packed, out, a_bits, w_bits, w_enc, m, n, k, fn)) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (bs::gemv_supported(m, k, a_bits, w_bits))  // one fused launch: pack in-kernel + GEMV
    return dense_core(nullptr, a, a_bits, w_packed, w_bits, w_enc, out, m, n, k, BS_ALGO_GEMV, s, fn);
  if (m <= kMaxRows && n <= (int64_t(1) << 31) - 1 && k <= (int64_t(1) << 31) - 1) {
    const ConvArgs g{1, int(m), 1, int(k), int(n), 1, 1, 1, 1, 0, 0};  // dense = 1x1 conv over m "pixels"
    bs::SmallConv sc{make_conv(nullptr, a_bits, w_packed, w_bits, w_enc, out, g), a};
    if (use_small(sc.p)) return cuda_status(bs::launch_small_conv(&sc, 1, a_bits, w_bits, s), fn);
  }
  const int64_t need = bs_dense_workspace_bytes(m, k, a_bits);
  if (!workspace || workspace_bytes < need) return fail(BS_ERR_WORKSPACE, "%s: workspace needs %lld bytes", fn, (long long)need);
  if (!aligned16(workspace)) return fail(BS_ERR_ALIGN, "%s: workspace must be 16-byte aligned", fn);
  uint32_t* ap = static_cast<uint32_t*>(workspace);
  if (int st = cuda_status(bs::launch_bitpack(a, ap, m, k, row_words(k), a_bits, s), fn)) return st;
  return dense_core(ap, nullptr, a_bits, w_packed, w_bits, w_enc, out, m, n, k, BS_ALGO_AUTO, s, fn);
}

int bs_bitserial_conv2d_nhwc_ex(const uint32_t* act_packed, int a_bits, const uint32_t* w_packed, int w_bits,
                                int w_enc, int32_t* out, int n, int h, int w, int c, int oc, int kh, int kw,
                                int stride_h, int stride_w, int pad_h, int pad_w, int algo, void* stream) {
  const char* fn = "bs_bitserial_conv2d_nhwc";
  const ConvArgs g{n, h, w, c, oc, kh, kw, stride_h, stride_w, pad_h, pad_w};
  if (int st = check_conv(g, a_bits, w_bits, w_enc, fn)) return st;
  if (!act_packed || !w_packed || !out) return fail(BS_ERR_NULL, "%s: NULL tensor pointer", fn);
  if (int st = check_algo(algo, fn)) return st;
  if (!aligned16(act_packed) || !aligned16(w_packed) || !aligned16(out))
    return fail(BS_ERR_ALIGN, "%s: pointers must be 16-byte aligned", fn);
  bs::ConvProblem p = make_conv(act_packed, a_bits, w_packed, w_bits, w_enc, out, g);
  return launch_conv(p, algo, static_cast<cudaStream_t>(stream), fn);
}

int bs_bitserial_conv2d_nhwc(const uint32_t* act_packed, int a_bits, const uint32_t* w_packed, int w_bits, int w_enc,
                             int32_t* out, int n, int h, int w, int c, int oc, int kh, int kw, int stride_h,
                             int stride_w, int pad_h, int pad_w, void* stream) {
  return bs_bitserial_conv2d_nhwc_ex(act_packed, a_bits, w_packed, w_bits, w_enc, out, n, h, w, c, oc, kh, kw,
                                     stride_h, stride_w, pad_h, pad_w, BS_ALGO_AUTO, stream);
}

int64_t bs_conv2d_workspace_bytes(int n, int h, int w, int c, int a_bits) {
  if (n <= 0 || h <= 0 || w <= 0 || c <= 0 || a_bits < 1 || a_bits > 8) return 0;
  return int64_t(a_bits) * n * h * w * row_words(c) * 4;
}

int bs_bitserial_conv2d_nhwc_i8(const uint8_t* act, int a_bits, const uint32_t* w_packed, int w_bits, int w_enc,
                                int32_t* out, int n, int h, int w, int c, int oc, int kh, int kw, int stride_h,
                                int stride_w, int pad_h, int pad_w, void* workspace, int64_t workspace_bytes,
                                void* stream) {
  const char* fn = "bs_bitserial_conv2d_nhwc_i8";
  const ConvArgs g{n, h, w, c, oc, kh, kw, stride_h, stride_w, pad_h, pad_w};
  if (int st = check_conv(g, a_bits, w_bits, w_enc, fn)) return st;
  if (!act || !w_packed || !out) return fail(BS_ERR_NULL, "%s: NULL tensor pointer", fn);
  const int64_t need = bs_conv2d_workspace_bytes(n, h, w, c, a_bits);
  if (!workspace || workspace_bytes < need) return fail(BS_ERR_WORKSPACE, "%s: workspace needs %lld bytes", fn, (long long)need);
  if (!aligned16(act) || !aligned16(w_packed) || !aligned16(out) || !aligned16(workspace))
    return fail(BS_ERR_ALIGN, "%s: pointers must be 16-byte aligned", fn);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t* ap = static_cast<uint32_t*>(workspace);
  bs::ConvProblem p = make_conv(ap, a_bits, w_packed, w_bits, w_enc, out, g);
  if (use_small(p)) {  // one launch, packing fused (the workspace is not touched)
    const bs::SmallConv sc{p, act};
    return cuda_status(bs::launch_small_conv(&sc, 1, a_bits, w_bits, s), fn);
  }
  if (int st = cuda_status(bs::launch_bitpack(act, ap, int64_t(n) * h * w, c, row_words(c), a_bits, s), fn)) return st;
  return launch_conv(p, BS_ALGO_AUTO, s, fn);
}

int bs_bitserial_conv2d_nhwc_i8_group(const bs_conv_i8_desc* descs, int count, int a_bits, int w_bits, void* stream) {
  const char* fn = "bs_bitserial_conv2d_nhwc_i8_group";
  if (count < 0 || count > (1 << 20)) return fail(BS_ERR_SHAPE, "%s: count out of range", fn);
  if (count == 0) return BS_OK;
  if (!descs) return fail(BS_ERR_NULL, "%s: NULL descriptor array", fn);
  if (!bs::small_supported(a_bits, w_bits))
    return fail(BS_ERR_UNSUPPORTED, "%s: a_bits in [1,4], w_bits in [1,2]", fn);
  std::vector<bs::SmallConv> ps(static_cast<size_t>(count));
  for (int q = 0; q < count; ++q) {
    const bs_conv_i8_desc& d = descs[q];
    const ConvArgs g{d.n, d.h, d.w, d.c, d.oc, d.kh, d.kw, d.stride_h, d.stride_w, d.pad_h, d.pad_w};
    if (int st = check_conv(g, a_bits, w_bits, d.w_enc, fn)) return st;
    if (d.w_enc == BS_SIGNED) return fail(BS_ERR_UNSUPPORTED, "%s: descriptor %d: signed weights", fn, q);
    if (int64_t(d.kh) * d.kw > 64) return fail(BS_ERR_UNSUPPORTED, "%s: descriptor %d: more than 64 filter taps", fn, q);
    if (!d.act || !d.w_packed || !d.out) return fail(BS_ERR_NULL, "%s: NULL pointer in descriptor %d", fn, q);
    if (!aligned16(d.act) || !aligned16(d.w_packed) || !aligned16(d.out))
      return fail(BS_ERR_ALIGN, "%s: descriptor %d: pointers must be 16-byte aligned", fn, q);
    if (int64_t(d.n) * d.h * d.w * d.c > (int64_t(1) << 40)) return fail(BS_ERR_SHAPE, "%s: descriptor %d too large", fn, q);
    ps[q] = bs::SmallConv{make_conv(nullptr, a_bits, d.w_packed, w_bits, d.w_enc, d.out, g), d.act};
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int q0 = 0; q0 < count; q0 += bs::kSmallMax) {
    const int cnt = count - q0 < bs::kSmallMax ? count - q0 : bs::kSmallMax;
    if (int st = cuda_status(bs::launch_small_conv(ps.data() + q0, cnt, a_bits, w_bits, s), fn)) return st;
  }
  return BS_OK;
}

int64_t bs_conv2d_tc_workspace_bytes(int oc, int kh, int kw, int c, int w_bits) {
  if (oc <= 0 || kh <= 0 || kw <= 0 || c <= 0 || w_bits < 1 || w_bits > 8) return 0;
  const int64_t kp = int64_t(kh) * kw * row_words(c);  // either format fits
  const int64_t i8 = bs::tc_weight_bytes(oc, kp, w_bits, bs::kTcI8), f4 = bs::tc_weight_bytes(oc, kp, w_bits, bs::kTcF4);
  return i8 > f4 ? i8 : f4;
}

int64_t bs_dense_tc_workspace_bytes(int64_t n, int64_t k, int w_bits) {
  if (n <= 0 || k <= 0 || w_bits < 1 || w_bits > 8) return 0;
  const int64_t i8 = bs::tc_weight_bytes(n, row_words(k), w_bits, bs::kTcI8);
  const int64_t f4 = bs::tc_weight_bytes(n, row_words(k), w_bits, bs::kTcF4);
  return i8 > f4 ? i8 : f4;  // either format fits
}

int bs_bitserial_conv2d_nhwc_tc(const uint32_t* act_packed, int a_bits, const uint32_t* w_packed, int w_bits,
                                int w_enc, int32_t* out, int n, int h, int w, int c, int oc, int kh, int kw,
                                int stride_h, int stride_w, int pad_h, int pad_w, void* workspace,
                                int64_t workspace_bytes, void* stream) {
  const char* fn = "bs_bitserial_conv2d_nhwc_tc";
  const ConvArgs g{n, h, w, c, oc, kh, kw, stride_h, stride_w, pad_h, pad_w};
  if (int st = check_conv(g, a_bits, w_bits, w_enc, fn)) return st;
  if (int st = check_tc_bound(int64_t(kh) * kw * c, a_bits, w_bits, BS_TC_DEFAULT, fn)) return st;
  if (!bs::tc_supported(a_bits, w_bits)) return fail(BS_ERR_UNSUPPORTED, "%s: a_bits in [1,4], w_bits in [1,4]", fn);
  if (!act_packed || !w_packed || !out || !workspace) return fail(BS_ERR_NULL, "%s: NULL pointer", fn);
  const int64_t need = bs_conv2d_tc_workspace_bytes(oc, kh, kw, c, w_bits);
  if (workspace_bytes < need) return fail(BS_ERR_WORKSPACE, "%s: workspace needs %lld bytes", fn, (long long)need);
  if (!aligned16(act_packed) || !aligned16(w_packed) || !aligned16(out) || !aligned16(workspace))
    return fail(BS_ERR_ALIGN, "%s: pointers must be 16-byte aligned", fn);
  bs::ConvProblem p = make_conv(act_packed, a_bits, w_packed, w_bits, w_enc, out, g);
  return cuda_status(bs::launch_tc_conv(p, static_cast<int8_t*>(workspace), 0, static_cast<cudaStream_t>(stream)), fn);
}

int bs_bitserial_dense_tc(const uint32_t* a_packed, int a_bits, const uint32_t* w_packed, int w_bits, int w_enc,
                          int32_t* out, int64_t m, int64_t n, int64_t k, void* workspace, int64_t workspace_bytes,
                          void* stream) {
  const char* fn = "bs_bitserial_dense_tc";
  if (int st = check_dense(a_packed, w_packed, out, a_bits, w_bits, w_enc, m, n, k, fn)) return st;
  if (int st = check_tc_bound(k, a_bits, w_bits, BS_TC_DEFAULT, fn)) return st;
  if (!bs::tc_supported(a_bits, w_bits)) return fail(BS_ERR_UNSUPPORTED, "%s: a_bits in [1,4], w_bits in [1,4]", fn);
  if (m > kMaxRows || n > (int64_t(1) << 31) - 1) return fail(BS_ERR_SHAPE, "%s: m or n too large", fn);
  const int64_t need = bs_dense_tc_workspace_bytes(n, k, w_bits);
  if (!workspace || workspace_bytes < need) return fail(BS_ERR_WORKSPACE, "%s: workspace needs %lld bytes", fn, (long long)need);
  if (!aligned16(workspace)) return fail(BS_ERR_ALIGN, "%s: workspace must be 16-byte aligned", fn);
  ConvArgs g{1, int(m), 1, int(k), int(n), 1, 1, 1, 1, 0, 0};
  bs::ConvProblem p = make_conv(a_packed, a_bits, w_packed, w_bits, w_enc, out, g);
  return cuda_status(bs::launch_tc_conv(p, static_cast<int8_t*>(workspace), 0, static_cast<cudaStream_t>(stream)), fn);
}

int64_t bs_conv2d_tc_weight_bytes(int oc, int kh, int kw, int c, int w_bits, int tc_format) {
  if (oc <= 0 || kh <= 0 || kw <= 0 || c <= 0 || w_bits < 1 || w_bits > 8) return 0;
  if (tc_format < BS_TC_DEFAULT || tc_format > BS_TC_F4) return 0;
  return bs::tc_weight_bytes(oc, int64_t(kh) * kw * row_words(c), w_bits, tc_format);
}

int64_t bs_dense_tc_weight_bytes(int64_t n, int64_t k, int w_bits, int tc_format) {
  if (n <= 0 || k <= 0 || w_bits < 1 || w_bits > 8) return 0;
  if (tc_format < BS_TC_DEFAULT || tc_format > BS_TC_F4) return 0;
  return bs::tc_weight_bytes(n, row_words(k), w_bits, tc_format);
}

int bs_conv2d_tc_prepare_weights(const uint32_t* w_packed, int w_bits, int w_enc, int oc, int kh, int kw, int c,
                                 int tc_format, int8_t* w_tc, int64_t w_tc_bytes, void* stream) {
  const char* fn = "bs_conv2d_tc_prepare_weights";
  if (int st = check_format(tc_format, fn)) return st;
  if (!w_packed || !w_tc) return fail(BS_ERR_NULL, "%s: NULL pointer", fn);
  if (int st = check_bits(1, w_bits, BS_UNIPOLAR, fn)) return st;
  if (int st = check_tc_enc(BS_A_UNSIGNED, w_enc, tc_format, fn)) return st;
  if (!bs::tc_supported(1, w_bits)) return fail(BS_ERR_UNSUPPORTED, "%s: w_bits in [1,4]", fn);
  if (oc <= 0 || kh <= 0 || kw <= 0 || c <= 0) return fail(BS_ERR_SHAPE, "%s: non-positive extent", fn);
  const int64_t need = bs_conv2d_tc_weight_bytes(oc, kh, kw, c, w_bits, tc_format);
  if (w_tc_bytes < need) return fail(BS_ERR_WORKSPACE, "%s: w_tc needs %lld bytes", fn, (long long)need);
  if (!aligned16(w_packed) || !aligned16(w_tc)) return fail(BS_ERR_ALIGN, "%s: pointers must be 16-byte aligned", fn);
  return cuda_status(bs::launch_tc_expand_weights(w_packed, w_bits, w_enc, oc, int64_t(kh) * kw * row_words(c), c,
                                                  int(row_words(c)), w_tc, tc_format,
                                                  static_cast<cudaStream_t>(stream)), fn);
}

int bs_dense_tc_prepare_weights(const uint32_t* w_packed, int w_bits, int w_enc, int64_t n, int64_t k, int tc_format,
                                int8_t* w_tc, int64_t w_tc_bytes, void* stream) {
  const char* fn = "bs_dense_tc_prepare_weights";
  if (int st = check_format(tc_format, fn)) return st;
  if (!w_packed || !w_tc) return fail(BS_ERR_NULL, "%s: NULL pointer", fn);
  if (int st = check_bits(1, w_bits, BS_UNIPOLAR, fn)) return st;
  if (int st = check_tc_enc(BS_A_UNSIGNED, w_enc, tc_format, fn)) return st;
  if (!bs::tc_supported(1, w_bits)) return fail(BS_ERR_UNSUPPORTED, "%s: w_bits in [1,4]", fn);
  if (n <= 0 || k <= 0 || n > (int64_t(1) << 31) - 1) return fail(BS_ERR_SHAPE, "%s: bad n or k", fn);
  const int64_t need = bs_dense_tc_weight_bytes(n, k, w_bits, tc_format);
  if (w_tc_bytes < need) return fail(BS_ERR_WORKSPACE, "%s: w_tc needs %lld bytes", fn, (long long)need);
  if (!aligned16(w_packed) || !aligned16(w_tc)) return fail(BS_ERR_ALIGN, "%s: pointers must be 16-byte aligned", fn);
  if (k > (int64_t(1) << 31) - 1) return fail(BS_ERR_SHAPE, "%s: k too large", fn);
  return cuda_status(bs::launch_tc_expand_weights(w_packed, w_bits, w_enc, n, row_words(k), int(k),
                                                  int(row_words(k)), w_tc, tc_format,
                                                  static_cast<cudaStream_t>(stream)), fn);
}

int bs_bitserial_conv2d_nhwc_tc_prepared(const uint32_t* act_packed, int a_bits, int a_enc, const int8_t* w_tc,
                                         int w_bits, int w_enc, int tc_format, int32_t* out, int n, int h, int w,
                                         int c, int oc, int kh, int kw, int stride_h, int stride_w, int pad_h,
                                         int pad_w, void* stream) {
  const char* fn = "bs_bitserial_conv2d_nhwc_tc_prepared";
  if (int st = check_format(tc_format, fn)) return st;
  if (int st = check_tc_enc(a_enc, w_enc, tc_format, fn)) return st;
  const ConvArgs g{n, h, w, c, oc, kh, kw, stride_h, stride_w, pad_h, pad_w};
  if (int st = check_conv(g, a_bits, w_bits, BS_UNIPOLAR, fn)) return st;
  if (int st = check_tc_bound(int64_t(kh) * kw * c, a_bits, w_bits, tc_format, fn, a_enc, w_enc)) return st;
  if (!bs::tc_supported(a_bits, w_bits)) return fail(BS_ERR_UNSUPPORTED, "%s: a_bits in [1,4], w_bits in [1,4]", fn);
  if (!act_packed || !w_tc || !out) return fail(BS_ERR_NULL, "%s: NULL pointer", fn);
  if (!aligned16(act_packed) || !aligned16(w_tc) || !aligned16(out))
    return fail(BS_ERR_ALIGN, "%s: pointers must be 16-byte aligned", fn);
  bs::ConvProblem p = make_conv(act_packed, a_bits, nullptr, w_bits, BS_UNIPOLAR, out, g);
  p.a_enc = a_enc;
  return cuda_status(bs::launch_tc_conv_prepared(p, w_tc, tc_format, static_cast<cudaStream_t>(stream)), fn);
}

int bs_bitserial_conv2d_nhwc_tc_group(const bs_tc_conv_desc* descs, int count, int a_bits, int w_bits,
                                      int tc_format, void* stream) {
  const char* fn = "bs_bitserial_conv2d_nhwc_tc_group";
  if (count < 0 || count > (1 << 20)) return fail(BS_ERR_SHAPE, "%s: count out of range", fn);
  if (count == 0) return BS_OK;
  if (!descs) return fail(BS_ERR_NULL, "%s: NULL descriptor array", fn);
  if (int st = check_format(tc_format, fn)) return st;
  if (!bs::tc_supported(a_bits, w_bits)) return fail(BS_ERR_UNSUPPORTED, "%s: a_bits in [1,4], w_bits in [1,4]", fn);
  std::vector<bs::ConvProblem> ps(static_cast<size_t>(count));
  std::vector<const int8_t*> ws(static_cast<size_t>(count));
  for (int q = 0; q < count; ++q) {
    const bs_tc_conv_desc& d = descs[q];
    if (int st = check_tc_enc(d.a_enc, d.w_enc, tc_format, fn)) return st;
    const ConvArgs g{d.n, d.h, d.w, d.c, d.oc, d.kh, d.kw, d.stride_h, d.stride_w, d.pad_h, d.pad_w};
    if (int st = check_conv(g, a_bits, w_bits, BS_UNIPOLAR, fn)) return st;
    if (int st = check_tc_bound(int64_t(d.kh) * d.kw * d.c, a_bits, w_bits, tc_format, fn, d.a_enc, d.w_enc))
      return st;
    if (!d.act_packed || !d.w_tc || !d.out) return fail(BS_ERR_NULL, "%s: NULL pointer in descriptor %d", fn, q);
    if (!aligned16(d.act_packed) || !aligned16(d.w_tc) || !aligned16(d.out))
      return fail(BS_ERR_ALIGN, "%s: descriptor %d: pointers must be 16-byte aligned", fn, q);
    ps[q] = make_conv(d.act_packed, a_bits, nullptr, w_bits, BS_UNIPOLAR, d.out, g);
    ps[q].a_enc = d.a_enc;
    ws[q] = d.w_tc;
  }
  return cuda_status(bs::launch_tc_conv_group(ps.data(), ws.data(), count, tc_format,
                                              static_cast<cudaStream_t>(stream)), fn);
}

int bs_bitserial_conv2d_nhwc_tc_i8(const uint8_t* act, int a_bits, int a_enc, const int8_t* w_tc, int w_bits,
                                   int w_enc, int tc_format, int32_t* out, int n, int h, int w, int c, int oc, int kh,
                                   int kw, int stride_h, int stride_w, int pad_h, int pad_w, void* workspace,
                                   int64_t workspace_bytes, void* stream) {
  const char* fn = "bs_bitserial_conv2d_nhwc_tc_i8";
  if (int st = check_format(tc_format, fn)) return st;
  if (int st = check_tc_enc(a_enc, w_enc, tc_format, fn)) return st;
  const ConvArgs g{n, h, w, c, oc, kh, kw, stride_h, stride_w, pad_h, pad_w};
  if (int st = check_conv(g, a_bits, w_bits, BS_UNIPOLAR, fn)) return st;
  if (int st = check_tc_bound(int64_t(kh) * kw * c, a_bits, w_bits, tc_format, fn, a_enc, w_enc)) return st;
  if (!bs::tc_supported(a_bits, w_bits)) return fail(BS_ERR_UNSUPPORTED, "%s: a_bits in [1,4], w_bits in [1,4]", fn);
  if (!act || !w_tc || !out) return fail(BS_ERR_NULL, "%s: NULL pointer", fn);
  const int64_t need = bs_conv2d_workspace_bytes(n, h, w, c, a_bits);
  if (!workspace || workspace_bytes < need) return fail(BS_ERR_WORKSPACE, "%s: workspace needs %lld bytes", fn, (long long)need);
  if (!aligned16(act) || !aligned16(w_tc) || !aligned16(out) || !aligned16(workspace))
    return fail(BS_ERR_ALIGN, "%s: pointers must be 16-byte aligned", fn);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t* ap = static_cast<uint32_t*>(workspace);
  if (int st = cuda_status(bs::launch_bitpack(act, ap, int64_t(n) * h * w, c, row_words(c), a_bits, s), fn)) return st;
  bs::ConvProblem p = make_conv(ap, a_bits, nullptr, w_bits, BS_UNIPOLAR, out, g);
  p.a_enc = a_enc;
  return cuda_status(bs::launch_tc_conv_prepared(p, w_tc, tc_format, s), fn);
}

int bs_bitserial_dense_tc_prepared(const uint32_t* a_packed, int a_bits, int a_enc, const int8_t* w_tc, int w_bits,
                                   int w_enc, int tc_format, int32_t* out, int64_t m, int64_t n, int64_t k,
                                   void* stream) {
  const char* fn = "bs_bitserial_dense_tc_prepared";
  if (int st = check_format(tc_format, fn)) return st;
  if (int st = check_tc_enc(a_enc, w_enc, tc_format, fn)) return st;
  if (int st = check_dense(a_packed, reinterpret_cast<const uint32_t*>(w_tc), out, a_bits, w_bits, BS_UNIPOLAR, m, n,
                           k, fn))
    return st;
  if (int st = check_tc_bound(k, a_bits, w_bits, tc_format, fn, a_enc, w_enc)) return st;
  if (!bs::tc_supported(a_bits, w_bits)) return fail(BS_ERR_UNSUPPORTED, "%s: a_bits in [1,4], w_bits in [1,4]", fn);
  if (m > kMaxRows || n > (int64_t(1) << 31) - 1) return fail(BS_ERR_SHAPE, "%s: m or n too large", fn);
  ConvArgs g{1, int(m), 1, int(k), int(n), 1, 1, 1, 1, 0, 0};
  bs::ConvProblem p = make_conv(a_packed, a_bits, nullptr, w_bits, BS_UNIPOLAR, out, g);
  p.a_enc = a_enc;
  return cuda_status(bs::launch_tc_conv_prepared(p, w_tc, tc_format, static_cast<cudaStream_t>(stream)), fn);
}

int bs_bitserial_dense_tc_prepared_gather(const uint32_t* a_packed, int a_bits, int a_enc, const int8_t* w_tc,
                                          int w_bits, int w_enc, int tc_format, int32_t* out,
                                          int32_t* const* out_peers, int npeers, int64_t m, int64_t n, int64_t k,
                                          void* stream) {
  const char* fn = "bs_bitserial_dense_tc_prepared_gather";
  if (int st = check_format(tc_format, fn)) return st;
  if (int st = check_tc_enc(a_enc, w_enc, tc_format, fn)) return st;
  if (int st = check_dense(a_packed, reinterpret_cast<const uint32_t*>(w_tc), out, a_bits, w_bits, BS_UNIPOLAR, m, n,
                           k, fn))
    return st;
  if (int st = check_tc_bound(k, a_bits, w_bits, tc_format, fn, a_enc, w_enc)) return st;
  if (!bs::tc_supported(a_bits, w_bits)) return fail(BS_ERR_UNSUPPORTED, "%s: a_bits in [1,4], w_bits in [1,4]", fn);
  if (m > kMaxRows || n > (int64_t(1) << 31) - 1) return fail(BS_ERR_SHAPE, "%s: m or n too large", fn);
  if (npeers < 0 || npeers > 8) return fail(BS_ERR_INVALID_ARG, "%s: npeers=%d not in [0,8]", fn, npeers);
  if (npeers > 0 && !out_peers) return fail(BS_ERR_NULL, "%s: NULL out_peers", fn);
  if (npeers > 0 && n % 4 != 0) return fail(BS_ERR_UNSUPPORTED, "%s: the fused gather needs n %% 4 == 0", fn);
  for (int d = 0; d < npeers; ++d) {
    if (!out_peers[d]) return fail(BS_ERR_NULL, "%s: NULL out_peers[%d]", fn, d);
    if (!aligned16(out_peers[d])) return fail(BS_ERR_ALIGN, "%s: out_peers[%d] must be 16-byte aligned", fn, d);
  }
  ConvArgs g{1, int(m), 1, int(k), int(n), 1, 1, 1, 1, 0, 0};
  bs::ConvProblem p = make_conv(a_packed, a_bits, nullptr, w_bits, BS_UNIPOLAR, out, g);
  p.a_enc = a_enc;
  return cuda_status(bs::launch_tc_conv_prepared(p, w_tc, tc_format, static_cast<cudaStream_t>(stream), out_peers,
                                                 npeers), fn);
}

int bs_bitserial_dense_tc_prepared_multicast(const uint32_t* a_packed, int a_bits, int a_enc, const int8_t* w_tc,
                                             int w_bits, int w_enc, int tc_format, int32_t* out_mc, int64_t m,
                                             int64_t n, int64_t k, void* stream) {
  const char* fn = "bs_bitserial_dense_tc_prepared_multicast";
  if (int st = check_format(tc_format, fn)) return st;
  if (int st = check_tc_enc(a_enc, w_enc, tc_format, fn)) return st;
  if (int st = check_dense(a_packed, reinterpret_cast<const uint32_t*>(w_tc), out_mc, a_bits, w_bits, BS_UNIPOLAR, m,
                           n, k, fn))
    return st;
  if (int st = check_tc_bound(k, a_bits, w_bits, tc_format, fn, a_enc, w_enc)) return st;
  if (!bs::tc_supported(a_bits, w_bits)) return fail(BS_ERR_UNSUPPORTED, "%s: a_bits in [1,4], w_bits in [1,4]", fn);
  if (m > kMaxRows || n > (int64_t(1) << 31) - 1) return fail(BS_ERR_SHAPE, "%s: m or n too large", fn);
  if (n % 4 != 0) return fail(BS_ERR_UNSUPPORTED, "%s: the multicast epilogue needs n %% 4 == 0", fn);
  ConvArgs g{1, int(m), 1, int(k), int(n), 1, 1, 1, 1, 0, 0};
  bs::ConvProblem p = make_conv(a_packed, a_bits, nullptr, w_bits, BS_UNIPOLAR, out_mc, g);
  p.a_enc = a_enc;
  return cuda_status(bs::launch_tc_conv_prepared(p, w_tc, tc_format, static_cast<cudaStream_t>(stream), nullptr, 0,
                                                 out_mc), fn);
}

int bs_bitserial_dense_tc_i8(const uint8_t* a, int a_bits, int a_enc, const int8_t* w_tc, int w_bits, int w_enc,
                             int tc_format, int32_t* out, int64_t m, int64_t n, int64_t k, void* workspace,
                             int64_t workspace_bytes, void* stream) {
  const char* fn = "bs_bitserial_dense_tc_i8";
  if (int st = check_format(tc_format, fn)) return st;
  if (int st = check_tc_enc(a_enc, w_enc, tc_format, fn)) return st;
  if (int st = check_dense(a, reinterpret_cast<const uint32_t*>(w_tc), out, a_bits, w_bits, BS_UNIPOLAR, m, n, k, fn))
    return st;
  if (int st = check_tc_bound(k, a_bits, w_bits, tc_format, fn, a_enc, w_enc)) return st;
  if (!bs::tc_supported(a_bits, w_bits)) return fail(BS_ERR_UNSUPPORTED, "%s: a_bits in [1,4], w_bits in [1,4]", fn);
  if (m > kMaxRows || n > (int64_t(1) << 31) - 1) return fail(BS_ERR_SHAPE, "%s: m or n too large", fn);
  const int64_t need = bs_dense_workspace_bytes(m, k, a_bits);
  if (!workspace || workspace_bytes < need) return fail(BS_ERR_WORKSPACE, "%s: workspace needs %lld bytes", fn, (long long)need);
  if (!aligned16(workspace)) return fail(BS_ERR_ALIGN, "%s: workspace must be 16-byte aligned", fn);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t* ap = static_cast<uint32_t*>(workspace);
  if (int st = cuda_status(bs::launch_bitpack(a, ap, m, k, row_words(k), a_bits, s), fn)) return st;
  ConvArgs g{1, int(m), 1, int(k), int(n), 1, 1, 1, 1, 0, 0};
  bs::ConvProblem p = make_conv(ap, a_bits, nullptr, w_bits, BS_UNIPOLAR, out, g);
  p.a_enc = a_enc;
  return cuda_status(bs::launch_tc_conv_prepared(p, w_tc, tc_format, s), fn);
}

int bs_bitserial_conv2d_nhwc_tc_host(const uint8_t* act_host, int a_bits, int a_enc, const int8_t* w_tc, int w_bits,
                                     int w_enc, int tc_format, int32_t* out_host, int n, int h, int w, int c, int oc, int kh, int kw,
                                     int stride_h, int stride_w, int pad_h, int pad_w, uint8_t* act_dev,
                                     int32_t* out_dev, void* workspace, int64_t workspace_bytes, void* stream) {
  const char* fn = "bs_bitserial_conv2d_nhwc_tc_host";
  if (!act_host || !out_host || !act_dev || !out_dev) return fail(BS_ERR_NULL, "%s: NULL buffer pointer", fn);
  const ConvArgs g{n, h, w, c, oc, kh, kw, stride_h, stride_w, pad_h, pad_w};
  if (int st = check_conv(g, a_bits, w_bits, BS_UNIPOLAR, fn)) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t in_bytes = size_t(n) * h * w * c;
  const size_t out_bytes = size_t(n) * conv_out(h, kh, stride_h, pad_h) * conv_out(w, kw, stride_w, pad_w) * oc * 4;
  if (int st = cuda_status(cudaMemcpyAsync(act_dev, act_host, in_bytes, cudaMemcpyHostToDevice, s), fn)) return st;
  if (int st = bs_bitserial_conv2d_nhwc_tc_i8(act_dev, a_bits, a_enc, w_tc, w_bits, w_enc, tc_format, out_dev, n, h, w, c, oc, kh, kw,
                                              stride_h, stride_w, pad_h, pad_w, workspace, workspace_bytes, stream))
    return st;
  if (int st = cuda_status(cudaMemcpyAsync(out_host, out_dev, out_bytes, cudaMemcpyDeviceToHost, s), fn)) return st;
  return cuda_status(cudaStreamSynchronize(s), fn);
}

int bs_bitserial_conv2d_nhwc_tc_host_group(const bs_tc_host_desc* descs, int count, int a_bits, int w_bits,
                                           int tc_format, void* stream) {
  const char* fn = "bs_bitserial_conv2d_nhwc_tc_host_group";
  if (count < 0 || count > (1 << 16)) return fail(BS_ERR_SHAPE, "%s: count out of range", fn);
  if (count == 0) return BS_OK;
  if (!descs) return fail(BS_ERR_NULL, "%s: NULL descriptor array", fn);
  if (int st = check_format(tc_format, fn)) return st;
  if (!bs::tc_supported(a_bits, w_bits)) return fail(BS_ERR_UNSUPPORTED, "%s: a_bits in [1,4], w_bits in [1,4]", fn);
  std::vector<bs::ConvProblem> ps(static_cast<size_t>(count));
  for (int q = 0; q < count; ++q) {
    const bs_tc_host_desc& d = descs[q];
    if (int st = check_tc_enc(d.a_enc, d.w_enc, tc_format, fn)) return st;
    const ConvArgs g{d.n, d.h, d.w, d.c, d.oc, d.kh, d.kw, d.stride_h, d.stride_w, d.pad_h, d.pad_w};
    if (int st = check_conv(g, a_bits, w_bits, BS_UNIPOLAR, fn)) return st;
    if (int st = check_tc_bound(int64_t(d.kh) * d.kw * d.c, a_bits, w_bits, tc_format, fn, d.a_enc, d.w_enc))
      return st;
    if (!d.act_host || !d.out_host || !d.act_dev || !d.packed_dev || !d.out_dev || !d.w_tc)
      return fail(BS_ERR_NULL, "%s: NULL pointer in descriptor %d", fn, q);
    if (!aligned16(d.act_dev) || !aligned16(d.packed_dev) || !aligned16(d.out_dev) || !aligned16(d.w_tc))
      return fail(BS_ERR_ALIGN, "%s: descriptor %d: device pointers must be 16-byte aligned", fn, q);
    ps[q] = make_conv(d.packed_dev, a_bits, nullptr, w_bits, BS_UNIPOLAR, d.out_dev, g);
    ps[q].a_enc = d.a_enc;
  }
  // three-stage pipeline: uploads on one stream, pack + conv on the caller's stream,
  // downloads on a third; layer q's download overlaps layer q+1's upload and compute.
  // The side streams and events are this thread's, created once per device (HostPipe).
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  HostPipe& hp = host_pipe();
  cudaError_t e = hp.prepare(2 * count + 2);
  cudaStream_t s_in = hp.in, s_out = hp.out;
  const std::vector<cudaEvent_t>& ev = hp.ev;
  cudaEvent_t start = e == cudaSuccess ? ev[0] : nullptr, end = e == cudaSuccess ? ev[1] : nullptr;
  if (e == cudaSuccess) e = cudaEventRecord(start, s);  // nothing starts before the caller's prior work
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s_in, start, 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s_out, start, 0);
  for (int q = 0; q < count && e == cudaSuccess; ++q) {
    const bs_tc_host_desc& d = descs[q];
    const bs::ConvProblem& p = ps[q];
    cudaEvent_t in = ev[2 + 2 * q], done = ev[3 + 2 * q];
    const size_t in_bytes = size_t(d.n) * d.h * d.w * d.c;
    const size_t out_bytes = size_t(p.M) * d.oc * 4;
    e = cudaMemcpyAsync(d.act_dev, d.act_host, in_bytes, cudaMemcpyHostToDevice, s_in);
    if (e == cudaSuccess) e = cudaEventRecord(in, s_in);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, in, 0);
    if (e == cudaSuccess) e = bs::launch_bitpack(d.act_dev, d.packed_dev, int64_t(d.n) * d.h * d.w, d.c, row_words(d.c),
                                               a_bits, s);
    if (e == cudaSuccess) e = bs::launch_tc_conv_prepared(p, d.w_tc, tc_format, s);
    if (e == cudaSuccess) e = cudaEventRecord(done, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s_out, done, 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d.out_host, d.out_dev, out_bytes, cudaMemcpyDeviceToHost, s_out);
  }
  if (e == cudaSuccess) e = cudaEventRecord(end, s_out);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(s, end, 0);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (s_in) cudaStreamSynchronize(s_in);
  if (s_out) cudaStreamSynchronize(s_out);
  return cuda_status(e, fn);
}

int bs_bitserial_conv2d_nhwc_host(const uint8_t* act_host, int a_bits, const uint32_t* w_packed, int w_bits,
                                  int w_enc, int32_t* out_host, int n, int h, int w, int c, int oc, int kh, int kw,
                                  int stride_h, int stride_w, int pad_h, int pad_w, uint8_t* act_dev,
                                  int32_t* out_dev, void* workspace, int64_t workspace_bytes, void* stream) {
  const char* fn = "bs_bitserial_conv2d_nhwc_host";
  if (!act_host || !out_host || !act_dev || !out_dev) return fail(BS_ERR_NULL, "%s: NULL buffer pointer", fn);
  const ConvArgs g{n, h, w, c, oc, kh, kw, stride_h, stride_w, pad_h, pad_w};
  if (int st = check_conv(g, a_bits, w_bits, w_enc, fn)) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t in_bytes = size_t(n) * h * w * c;
  const size_t out_bytes = size_t(n) * conv_out(h, kh, stride_h, pad_h) * conv_out(w, kw, stride_w, pad_w) * oc * 4;
  if (int st = cuda_status(cudaMemcpyAsync(act_dev, act_host, in_bytes, cudaMemcpyHostToDevice, s), fn)) return st;
  if (int st = bs_bitserial_conv2d_nhwc_i8(act_dev, a_bits, w_packed, w_bits, w_enc, out_dev, n, h, w, c, oc, kh, kw,
                                           stride_h, stride_w, pad_h, pad_w, workspace, workspace_bytes, stream))
    return st;
  if (int st = cuda_status(cudaMemcpyAsync(out_host, out_dev, out_bytes, cudaMemcpyDeviceToHost, s), fn)) return st;
  return cuda_status(cudaStreamSynchronize(s), fn);
}

// ------------------------------------------------------------------ digit path
int64_t bs_digit_row_bytes(int64_t k) { return bs::digit_row_bytes(k); }

int bs_digitpack_group(const bs_digit_pack_desc* descs, int count, int bits, int enc, void* stream) {
  const char* fn = "bs_digitpack_group";
  if (count < 0 || count > (1 << 20)) return fail(BS_ERR_SHAPE, "%s: count out of range", fn);
  if (count == 0) return BS_OK;
  if (!descs) return fail(BS_ERR_NULL, "%s: NULL descriptor array", fn);
  if (bits < 1 || bits > 4) return fail(BS_ERR_INVALID_ARG, "%s: bits=%d not in [1,4]", fn, bits);
  if (enc < BS_A_UNSIGNED || enc > BS_A_SIGNED) return fail(BS_ERR_INVALID_ARG, "%s: bad encoding %d", fn, enc);
  std::vector<bs::DigitSeg> segs(static_cast<size_t>(count));
  for (int q = 0; q < count; ++q) {
    const bs_digit_pack_desc& d = descs[q];
    if (!d.in || !d.out) return fail(BS_ERR_NULL, "%s: NULL pointer in descriptor %d", fn, q);
    if (d.rows <= 0 || d.k <= 0) return fail(BS_ERR_SHAPE, "%s: descriptor %d: rows and k must be >= 1", fn, q);
    if (!aligned16(d.out)) return fail(BS_ERR_ALIGN, "%s: descriptor %d: out must be 16-byte aligned", fn, q);
    bs::DigitSeg g{};
    g.in = d.in;
    g.out = d.out;
    g.rows = d.rows;
    g.k = d.k;
    segs[q] = g;
  }
  return cuda_status(bs::launch_digitpack_group(segs.data(), count, bits, enc, static_cast<cudaStream_t>(stream)), fn);
}

int bs_digitpack(const uint8_t* in, uint8_t* out, int64_t rows, int64_t k, int bits, int enc, void* stream) {
  const bs_digit_pack_desc d{in, out, rows, k};
  const int st = bs_digitpack_group(&d, 1, bits, enc, stream);
  if (st != BS_OK) {  // name the single-tensor entry in the message
    char tmp[512];
    snprintf(tmp, sizeof(tmp), "%s", g_last_error);
    const char* rest = strncmp(tmp, "bs_digitpack_group", 18) == 0 ? tmp + 18 : tmp;
    fail(st, "bs_digitpack%s", rest);
  }
  return st;
}

int64_t bs_conv2d_tcd_weight_bytes(int oc, int kh, int kw, int c, int w_bits) {
  if (oc <= 0 || kh <= 0 || kw <= 0 || c <= 0 || w_bits < 1 || w_bits > 4) return 0;
  return bs::tcd_weight_bytes(oc, int64_t(kh) * kw * row_words(c), w_bits);
}

int64_t bs_dense_tcd_weight_bytes(int64_t n, int64_t k, int w_bits) {
  if (n <= 0 || k <= 0 || w_bits < 1 || w_bits > 4) return 0;
  return bs::tcd_weight_bytes(n, row_words(k), w_bits);
}

int bs_conv2d_tcd_prepare_weights(const uint32_t* w_packed, int w_bits, int w_enc, int oc, int kh, int kw, int c,
                                  uint8_t* w_dig, int64_t w_dig_bytes, void* stream) {
  const char* fn = "bs_conv2d_tcd_prepare_weights";
  if (!w_packed || !w_dig) return fail(BS_ERR_NULL, "%s: NULL pointer", fn);
  if (w_bits < 1 || w_bits > 4) return fail(BS_ERR_UNSUPPORTED, "%s: w_bits=%d not in [1,4]", fn, w_bits);
  if (w_enc < BS_UNIPOLAR || w_enc > BS_SIGNED) return fail(BS_ERR_INVALID_ARG, "%s: bad w_enc %d", fn, w_enc);
  if (oc <= 0 || kh <= 0 || kw <= 0 || c <= 0) return fail(BS_ERR_SHAPE, "%s: non-positive extent", fn);
  const int64_t need = bs_conv2d_tcd_weight_bytes(oc, kh, kw, c, w_bits);
  if (w_dig_bytes < need) return fail(BS_ERR_WORKSPACE, "%s: w_dig needs %lld bytes", fn, (long long)need);
  if (!aligned16(w_packed) || !aligned16(w_dig)) return fail(BS_ERR_ALIGN, "%s: pointers must be 16-byte aligned", fn);
  return cuda_status(bs::launch_weight_digits(w_packed, w_bits, w_enc, oc, int64_t(kh) * kw * row_words(c), c,
                                              int(row_words(c)), w_dig, static_cast<cudaStream_t>(stream)), fn);
}

int bs_dense_tcd_prepare_weights(const uint32_t* w_packed, int w_bits, int w_enc, int64_t n, int64_t k, uint8_t* w_dig,
                                 int64_t w_dig_bytes, void* stream) {
  const char* fn = "bs_dense_tcd_prepare_weights";
  if (!w_packed || !w_dig) return fail(BS_ERR_NULL, "%s: NULL pointer", fn);
  if (w_bits < 1 || w_bits > 4) return fail(BS_ERR_UNSUPPORTED, "%s: w_bits=%d not in [1,4]", fn, w_bits);
  if (w_enc < BS_UNIPOLAR || w_enc > BS_SIGNED) return fail(BS_ERR_INVALID_ARG, "%s: bad w_enc %d", fn, w_enc);
  if (n <= 0 || k <= 0 || n > (int64_t(1) << 31) - 1 || k > (int64_t(1) << 31) - 1)
    return fail(BS_ERR_SHAPE, "%s: bad n or k", fn);
  const int64_t need = bs_dense_tcd_weight_bytes(n, k, w_bits);
  if (w_dig_bytes < need) return fail(BS_ERR_WORKSPACE, "%s: w_dig needs %lld bytes", fn, (long long)need);
  if (!aligned16(w_packed) || !aligned16(w_dig)) return fail(BS_ERR_ALIGN, "%s: pointers must be 16-byte aligned", fn);
  return cuda_status(bs::launch_weight_digits(w_packed, w_bits, w_enc, n, row_words(k), int(k), int(row_words(k)),
                                              w_dig, static_cast<cudaStream_t>(stream)), fn);
}

int bs_bitserial_conv2d_nhwc_tcd_group(const bs_tcd_conv_desc* descs, int count, int a_bits, int w_bits,
                                       void* stream) {
  const char* fn = "bs_bitserial_conv2d_nhwc_tcd_group";
  if (count < 0 || count > (1 << 20)) return fail(BS_ERR_SHAPE, "%s: count out of range", fn);
  if (count == 0) return BS_OK;
  if (!descs) return fail(BS_ERR_NULL, "%s: NULL descriptor array", fn);
  std::vector<bs::TcdProblem> ps(static_cast<size_t>(count));
  for (int q = 0; q < count; ++q) {
    const bs_tcd_conv_desc& d = descs[q];
    const ConvArgs g{d.n, d.h, d.w, d.c, d.oc, d.kh, d.kw, d.stride_h, d.stride_w, d.pad_h, d.pad_w};
    if (int st = check_tcd_conv(g, a_bits, w_bits, d.a_enc, d.w_enc, fn)) return st;
    if (!d.act_dig || !d.w_dig || !d.out) return fail(BS_ERR_NULL, "%s: NULL pointer in descriptor %d", fn, q);
    if (!aligned16(d.act_dig) || !aligned16(d.w_dig) || !aligned16(d.out))
      return fail(BS_ERR_ALIGN, "%s: descriptor %d: pointers must be 16-byte aligned", fn, q);
    ps[q] = make_tcd(d.act_dig, d.w_dig, d.out, a_bits, w_bits, g);
  }
  return cuda_status(bs::launch_tcd_group(ps.data(), count, static_cast<cudaStream_t>(stream)), fn);
}

int bs_bitserial_conv2d_nhwc_tcd(const uint8_t* act_dig, int a_bits, int a_enc, const uint8_t* w_dig, int w_bits,
                                 int w_enc, int32_t* out, int n, int h, int w, int c, int oc, int kh, int kw,
                                 int stride_h, int stride_w, int pad_h, int pad_w, void* stream) {
  const char* fn = "bs_bitserial_conv2d_nhwc_tcd";
  const ConvArgs g{n, h, w, c, oc, kh, kw, stride_h, stride_w, pad_h, pad_w};
  if (int st = check_tcd_conv(g, a_bits, w_bits, a_enc, w_enc, fn)) return st;
  if (!act_dig || !w_dig || !out) return fail(BS_ERR_NULL, "%s: NULL pointer", fn);
  if (!aligned16(act_dig) || !aligned16(w_dig) || !aligned16(out))
    return fail(BS_ERR_ALIGN, "%s: pointers must be 16-byte aligned", fn);
  const bs::TcdProblem p = make_tcd(act_dig, w_dig, out, a_bits, w_bits, g);
  return cuda_status(bs::launch_tcd_group(&p, 1, static_cast<cudaStream_t>(stream)), fn);
}

int bs_bitserial_dense_tcd(const uint8_t* a_dig, int a_bits, int a_enc, const uint8_t* w_dig, int w_bits, int w_enc,
                           int32_t* out, int64_t m, int64_t n, int64_t k, void* stream) {
  const char* fn = "bs_bitserial_dense_tcd";
  if (int st = check_tc_enc(a_enc, w_enc, BS_TC_F4, fn)) return st;
  if (int st = check_dense(a_dig, reinterpret_cast<const uint32_t*>(w_dig), out, a_bits, w_bits, BS_UNIPOLAR, m, n,
                           k, fn))
    return st;
  if (int st = check_tc_bound(k, a_bits, w_bits, BS_TC_F4, fn, a_enc, w_enc)) return st;
  if (!bs::tc_supported(a_bits, w_bits)) return fail(BS_ERR_UNSUPPORTED, "%s: a_bits in [1,4], w_bits in [1,4]", fn);
  if (m > kMaxRows || n > (int64_t(1) << 31) - 1 || k > (int64_t(1) << 31) - 1)
    return fail(BS_ERR_SHAPE, "%s: m, n or k too large", fn);
  const ConvArgs g{int(m), 1, 1, int(k), int(n), 1, 1, 1, 1, 0, 0};
  bs::TcdProblem p = make_tcd(a_dig, w_dig, out, a_bits, w_bits, g);
  p.dense = 1;
  return cuda_status(bs::launch_tcd_group(&p, 1, static_cast<cudaStream_t>(stream)), fn);
}

// ------------------------------------------------------------------ window path
int64_t bs_tcw_act_bytes(int n, int h, int w, int c, int kh, int kw, int stride, int pad_h, int pad_w, int bits) {
  bs::TcwGeom G;
  if (bits < 1 || bits > 4 || pad_h < 0 || pad_w < 0 ||
      !bs::tcw_geom(n, h, w, c, 1, kh, kw, stride, stride, pad_h, pad_w, G))
    return 0;
  return int64_t((bits + 1) / 2) * G.digit_bytes;
}

int bs_digitpack_win_group(const bs_win_pack_desc* descs, int count, int bits, int enc, void* stream) {
  const char* fn = "bs_digitpack_win_group";
  if (count < 0 || count > (1 << 20)) return fail(BS_ERR_SHAPE, "%s: count out of range", fn);
  if (count == 0) return BS_OK;
  if (!descs) return fail(BS_ERR_NULL, "%s: NULL descriptor array", fn);
  if (bits < 1 || bits > 4) return fail(BS_ERR_INVALID_ARG, "%s: bits=%d not in [1,4]", fn, bits);
  if (enc < BS_A_UNSIGNED || enc > BS_A_SIGNED) return fail(BS_ERR_INVALID_ARG, "%s: bad encoding %d", fn, enc);
  std::vector<bs::WinSeg> segs(static_cast<size_t>(count));
  for (int q = 0; q < count; ++q) {
    const bs_win_pack_desc& d = descs[q];
    if (!d.in || !d.out) return fail(BS_ERR_NULL, "%s: NULL pointer in descriptor %d", fn, q);
    const ConvArgs g{d.n, d.h, d.w, d.c, 1, d.kh, d.kw, d.stride, d.stride, d.pad_h, d.pad_w};
    if (int st = check_conv(g, 1, 1, BS_UNIPOLAR, fn)) return st;
    bs::TcwGeom G;
    if (int st = check_tcw_geom(g, 1, G, fn)) return st;
    const int64_t need = int64_t((bits + 1) / 2) * G.digit_bytes;
    if (d.out_bytes < need) return fail(BS_ERR_WORKSPACE, "%s: descriptor %d: out needs %lld bytes", fn, q,
                                        (long long)need);
    if (!aligned16(d.out)) return fail(BS_ERR_ALIGN, "%s: descriptor %d: out must be 16-byte aligned", fn, q);
    bs::WinSeg s{};
    s.in = d.in;
    s.out = d.out;
    s.n = d.n; s.h = d.h; s.w = d.w; s.c = d.c; s.kh = d.kh; s.kw = d.kw; s.s = d.stride;
    s.ph = d.pad_h; s.pw = d.pad_w;
    segs[q] = s;
  }
  return cuda_status(bs::launch_digitpack_win_group(segs.data(), count, bits, enc, static_cast<cudaStream_t>(stream)),
                     fn);
}

int bs_digitpack_win(const uint8_t* in, uint8_t* out, int64_t out_bytes, int n, int h, int w, int c, int kh, int kw,
                     int stride, int pad_h, int pad_w, int bits, int enc, void* stream) {
  const bs_win_pack_desc d{in, out, out_bytes, n, h, w, c, kh, kw, stride, pad_h, pad_w};
  const int st = bs_digitpack_win_group(&d, 1, bits, enc, stream);
  if (st != BS_OK) {
    char tmp[512];
    snprintf(tmp, sizeof(tmp), "%s", g_last_error);
    const char* rest = strncmp(tmp, "bs_digitpack_win_group", 22) == 0 ? tmp + 22 : tmp;
    fail(st, "bs_digitpack_win%s", rest);
  }
  return st;
}

int64_t bs_conv2d_tcw_weight_bytes(int oc, int kh, int kw, int c, int w_bits) {
  return bs::tcw_weight_bytes(oc, kh, kw, c, w_bits);
}

int bs_conv2d_tcw_prepare_weights(const uint32_t* w_packed, int w_bits, int w_enc, int oc, int kh, int kw, int c,
                                  uint8_t* w_win, int64_t w_win_bytes, void* stream) {
  const char* fn = "bs_conv2d_tcw_prepare_weights";
  if (!w_packed || !w_win) return fail(BS_ERR_NULL, "%s: NULL pointer", fn);
  if (w_bits < 1 || w_bits > 4) return fail(BS_ERR_UNSUPPORTED, "%s: w_bits=%d not in [1,4]", fn, w_bits);
  if (w_enc < BS_UNIPOLAR || w_enc > BS_SIGNED) return fail(BS_ERR_INVALID_ARG, "%s: bad w_enc %d", fn, w_enc);
  if (oc <= 0 || kh <= 0 || kw <= 0 || c <= 0) return fail(BS_ERR_SHAPE, "%s: non-positive extent", fn);
  const int64_t need = bs_conv2d_tcw_weight_bytes(oc, kh, kw, c, w_bits);
  if (w_win_bytes < need) return fail(BS_ERR_WORKSPACE, "%s: w_win needs %lld bytes", fn, (long long)need);
  if (!aligned16(w_packed) || !aligned16(w_win)) return fail(BS_ERR_ALIGN, "%s: pointers must be 16-byte aligned", fn);
  return cuda_status(bs::launch_tcw_weights(w_packed, w_bits, w_enc, oc, kh, kw, c, w_win,
                                            static_cast<cudaStream_t>(stream)), fn);
}

int bs_bitserial_conv2d_nhwc_tcw_group(const bs_tcw_conv_desc* descs, int count, int a_bits, int w_bits,
                                       void* stream) {
  const char* fn = "bs_bitserial_conv2d_nhwc_tcw_group";
  if (count < 0 || count > (1 << 20)) return fail(BS_ERR_SHAPE, "%s: count out of range", fn);
  if (count == 0) return BS_OK;
  if (!descs) return fail(BS_ERR_NULL, "%s: NULL descriptor array", fn);
  std::vector<bs::TcwProblem> ps(static_cast<size_t>(count));
  for (int q = 0; q < count; ++q) {
    const bs_tcw_conv_desc& d = descs[q];
    const ConvArgs g{d.n, d.h, d.w, d.c, d.oc, d.kh, d.kw, d.stride_h, d.stride_w, d.pad_h, d.pad_w};
    if (int st = check_tcw_conv(g, a_bits, w_bits, d.a_enc, d.w_enc, fn)) return st;
    if (!d.act_win || !d.w_win || !d.out) return fail(BS_ERR_NULL, "%s: NULL pointer in descriptor %d", fn, q);
    if (!aligned16(d.act_win) || !aligned16(d.w_win) || !aligned16(d.out))
      return fail(BS_ERR_ALIGN, "%s: descriptor %d: pointers must be 16-byte aligned", fn, q);
    ps[q] = make_tcw(d.act_win, d.w_win, d.out, a_bits, w_bits, g);
  }
  return tcw_status(bs::launch_tcw_group(ps.data(), count, static_cast<cudaStream_t>(stream)), fn);
}

int bs_bitserial_conv2d_nhwc_tcw(const uint8_t* act_win, int a_bits, int a_enc, const uint8_t* w_win, int w_bits,
                                 int w_enc, int32_t* out, int n, int h, int w, int c, int oc, int kh, int kw,
                                 int stride_h, int stride_w, int pad_h, int pad_w, void* stream) {
  const char* fn = "bs_bitserial_conv2d_nhwc_tcw";
  const ConvArgs g{n, h, w, c, oc, kh, kw, stride_h, stride_w, pad_h, pad_w};
  if (int st = check_tcw_conv(g, a_bits, w_bits, a_enc, w_enc, fn)) return st;
  if (!act_win || !w_win || !out) return fail(BS_ERR_NULL, "%s: NULL pointer", fn);
  if (!aligned16(act_win) || !aligned16(w_win) || !aligned16(out))
    return fail(BS_ERR_ALIGN, "%s: pointers must be 16-byte aligned", fn);
  const bs::TcwProblem p = make_tcw(act_win, w_win, out, a_bits, w_bits, g);
  return tcw_status(bs::launch_tcw_group(&p, 1, static_cast<cudaStream_t>(stream)), fn);
}

}  // extern "C"
