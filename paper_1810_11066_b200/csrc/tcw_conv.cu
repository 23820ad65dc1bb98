// tcw_conv.cu — the windowed tensor-core bitserial conv2d: implicit GEMM whose A operand for
// every filter tap is a SHIFTED VIEW of one contiguous window in shared memory.
//
// Eq. 2 regrouped by radix-4 digits (R21), every inner sum one exact
// kind::mxf4 contraction (E2M1 digits, UE8M0 digit scales 2^(2d+1), FP32 accumulation exact
// below 2^22, R17).  The activations arrive in the window layout (digit.cu, R26):
// the conv's zero-padded input split into its stride phases on an hg x wg phase grid, one
// contiguous [pstride][16 B] array per (digit, phase, 32-channel slab).  Output (oy, ox) at
// grid position q = (img*hg + oy)*wg + ox reads tap (ky, kx) at q + (ky/s)*wg + kx/s of phase
// (ky%s, kx%s), so for a tile of 128 consecutive grid positions q0.. every tap's A operand
// is rows [q0 + off, q0 + off + 128) of the same window: the MMA's shared-memory descriptor
// (K-major, no swizzle: 8-row x 16-byte core matrices, SBO = 128 B, LBO = the slab stride)
// simply starts off*16 bytes later.  The windows arrive by 1-D bulk copies (contiguous
// bytes, no per-row TMA cost — the im2col TMA path is row-bound), each
// window serves every tap, and no thread touches the operands.
//
// Tiles: R whole grid rows (R*wg <= 128 MMA rows; rows past R*wg and junk grid positions
// (x >= ow, y >= oh) are computed and discarded) x BN filters (64 or 128).  K loop: one stage
// per 64-channel slab pair: the windows of both slabs (every phase, activation digit) and —
// unless the whole filter block is resident — that pair's weights for every tap; per stage
// taps x DA x DW MMAs of 128 x BN x 64.
//
// Kernel structure (persistent, warp-specialized, one CTA per SM, 6 warps):
//   warp 0     bulk-copy producer (one lane): windows (+ streamed weights) of each stage onto
//              full[stage]; resident weight blocks onto b_full.
//   warp 1     MMA issuer (one elected lane); double-buffered TMEM accumulators (2 x 128 cols).
//   warps 2-5  epilogue (TMEM lane quarters): tcgen05.ld -> F2I -> staging of the tile's valid
//              rows at their compacted positions (they are consecutive NHWC output rows) ->
//              one TMA store of 64 columns x 2^k rows per set bit k of the valid-row count.
#include "tc_conv_impl.cuh"

namespace bs {

namespace {
int64_t ceil_to(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
int out_extent(int in, int k, int s, int p) {
  const int span = in + 2 * p - k;
  return span < 0 ? 0 : span / s + 1;
}
}  // namespace

bool tcw_geom(int n, int h, int w, int c, int oc, int kh, int kw, int sh, int sw, int ph, int pw, TcwGeom& g) {
  memset(&g, 0, sizeof(g));
  if (sh != sw || sh < 1 || sh > 2 || n <= 0 || h <= 0 || w <= 0 || c <= 0 || oc <= 0 || kh <= 0 || kw <= 0)
    return false;
  const int s = sh;
  g.s = s;
  g.oh = out_extent(h, kh, s, ph);
  g.ow = out_extent(w, kw, s, pw);
  if (g.oh <= 0 || g.ow <= 0) return false;
  g.hg = g.oh + (kh - 1) / s;
  g.wg = g.ow + (kw - 1) / s;
  for (int f = 0; f < 4; ++f) g.slot_of[f] = -1;
  for (int ky = 0; ky < kh; ++ky)
    for (int kx = 0; kx < kw; ++kx) g.slot_of[(ky % s) * s + kx % s] = 0;
  for (int f = 0; f < s * s; ++f)
    if (g.slot_of[f] == 0) {
      g.slot_of[f] = g.nph;
      g.phase[g.nph++] = f;
    }
  g.maxoff = ((kh - 1) / s) * g.wg + (kw - 1) / s;
  g.lwin = int(ceil_to(kTcwBM + int64_t(g.maxoff) + 8, 8));  // from an 8-row boundary
  g.ow8 = int(ceil_to(g.ow, 8));
  g.R = kTcwBM / g.wg;  // whole grid rows per 128-row tile
  if (g.R < 1 || g.lwin > 8192) return false;
  g.gpix = int64_t(n) * g.hg * g.wg;
  g.pstride = ceil_to(g.gpix + g.lwin, 8);
  g.cw = int(digit_row_bytes(c) / 16);
  g.taps = kh * kw;
  g.bn = oc <= 64 ? 64 : 128;
  g.nblk = (oc + g.bn - 1) / g.bn;
  g.digit_bytes = int64_t(g.nph) * g.cw * g.pstride * 16;
  if (int64_t(g.nph) * g.cw * g.pstride >= (int64_t(1) << 31) || int64_t(n) * g.hg >= (int64_t(1) << 30)) return false;
  return true;
}

int64_t tcw_weight_bytes(int oc, int kh, int kw, int c, int w_bits) {
  if (oc <= 0 || kh <= 0 || kw <= 0 || c <= 0 || w_bits < 1 || w_bits > 4) return 0;
  const int64_t bn = oc <= 64 ? 64 : 128, nblk = (oc + bn - 1) / bn;
  return nblk * bn * int64_t((w_bits + 1) / 2) * kh * kw * digit_row_bytes(c);
}

namespace tcw {

#ifndef BS_TCW_EPI_WARPS
#define BS_TCW_EPI_WARPS 8  // epilogue warps (a multiple of 4: warp % 4 = TMEM lane quarter)
#endif
#ifndef BS_TCW_EPI_BUFS_MIN
#define BS_TCW_EPI_BUFS_MIN 2
#endif

constexpr int kTmaWarp = 0, kMmaWarp = 1, kEpiWarp0 = 2, kEpiWarps = BS_TCW_EPI_WARPS;
constexpr int kThreads = (kEpiWarp0 + kEpiWarps) * 32;
constexpr int kStageBuf = 32 * 128;  // per-warp epilogue staging: 32 compacted rows x 32 int32 (dense)
constexpr int kEpiBufsMin = BS_TCW_EPI_BUFS_MIN, kEpiBufsMax = 4;  // staging buffers per epilogue warp: runtime
constexpr int kBoxMaps = 6;  // output maps with boxes of 32 columns x 1, 2, 4, ..., 32 rows
constexpr int kBarBytes = 512;
constexpr int kSmemLimit = 222 * 1024;  // dynamic; + static problem records (NP x ~180 B) <= 227 KB
constexpr int kMinSmem = 116 * 1024;  // > half the SM: one CTA per SM (it owns all of TMEM)
constexpr int kGroupMax = 16;
constexpr int kMaxStages = 12;
constexpr int kBResMax = 100 * 1024;  // largest filter block kept resident
constexpr int kAccCols = 128;         // TMEM columns per accumulator buffer (BN <= 128)
constexpr int kSF0 = 2 * kAccCols;    // scale factors: SFA 4 columns per digit, SFB 8 per digit

struct TwProb {
  const uint8_t* act;
  const uint8_t* wt;
  int32_t* out;
  int64_t slab_bytes;   // pstride * 32: one (digit, phase, slab pair) array of 32-byte rows
  int64_t digit_bytes;  // one activation digit of the layout
  int tile0, nmb, bn, pairs, taps, kh, kw, s, wg, hg, oh, ow, ow8, R, nph, lwin, G, oc;
  int slot_of[4];
  uint32_t idesc;
  int b_res;
  uint32_t bslot;   // bytes of one slab pair's weights (DW * taps * 2 * bn * 16)
  uint32_t abytes;  // bytes of one stage's windows (DA * nph * 2 * lwin * 16)
  FastDiv div_nm, div_wg, div_hg;
};
template <int NP>
struct TwArgs {
  int nprob, ntiles, stages;
  int astage, bstride;  // A ring stage bytes; streamed weight slot bytes
  int a_off, epi_off, bar_off;
  int ebufs;  // epilogue staging buffers (kEpiBufsMin .. kEpiBufsMax)
  TwProb prob[NP];
};
template <int NP>
struct TwMaps {
  CUtensorMap out[NP][kBoxMaps];  // [problem][k]: box of 32 columns x 2^k rows, no swizzle
};

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}
__device__ __forceinline__ void spin_wait(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile(
      "{.reg .pred e; .reg .b32 x;\n"
      "elect.sync x|e, 0xffffffff;\n"
      "selp.u32 %0, 1, 0, e;\n}"
      : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ void mma_f4_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa,
                                          uint32_t sfb, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %6, 0;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(sfa), "r"(sfb), "r"(accumulate));
}
// One MMA from one elected lane of a warp that executes the call uniformly: the descriptor
// arithmetic around it stays on the uniform datapath (no per-MMA register -> uniform moves).
__device__ __forceinline__ void mma_f4_ss_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa,
                                                uint32_t sfb, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p, e;\n.reg .b32 x;\n"
      "elect.sync x|e, 0xffffffff;\n"
      "setp.ne.b32 p, %6, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(sfa), "r"(sfb), "r"(accumulate));
}
// All nine MMAs of a 3x3 filter from one elected lane: row r's three taps read A at ar, ar + da1r,
// ar + da2 (da1 of rows 0 and 2 is da1e, of row 1 da1o: the phase of an odd kernel row differs at
// stride 2) and B at b + t * db for tap t = 3r + c; one register -> uniform move per operand and
// stage instead of per MMA.
__device__ __forceinline__ void mma9_f4(uint32_t d, uint64_t a0, uint64_t a1, uint64_t a2, uint64_t b,
                                       uint64_t da1e, uint64_t da1o, uint64_t da2, uint64_t db, uint32_t idesc,
                                       uint32_t sfa, uint32_t sfb, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p, e;\n.reg .b32 x;\n.reg .b64 t, bb;\n"
      "elect.sync x|e, 0xffffffff;\n"
      "setp.ne.b32 p, %12, 0;\n"
      "@!e bra SKIP%=;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %4, %9, [%10], [%11], p;\n"
      "add.s64 t, %1, %5;\nadd.s64 bb, %4, %8;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], t, bb, %9, [%10], [%11], 1;\n"
      "add.s64 t, %1, %7;\nadd.s64 bb, bb, %8;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], t, bb, %9, [%10], [%11], 1;\n"
      "add.s64 bb, bb, %8;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %2, bb, %9, [%10], [%11], 1;\n"
      "add.s64 t, %2, %6;\nadd.s64 bb, bb, %8;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], t, bb, %9, [%10], [%11], 1;\n"
      "add.s64 t, %2, %7;\nadd.s64 bb, bb, %8;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], t, bb, %9, [%10], [%11], 1;\n"
      "add.s64 bb, bb, %8;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %3, bb, %9, [%10], [%11], 1;\n"
      "add.s64 t, %3, %5;\nadd.s64 bb, bb, %8;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], t, bb, %9, [%10], [%11], 1;\n"
      "add.s64 t, %3, %7;\nadd.s64 bb, bb, %8;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], t, bb, %9, [%10], [%11], 1;\n"
      "SKIP%=:\n}" ::"r"(d),
      "l"(a0), "l"(a1), "l"(a2), "l"(b), "l"(da1e), "l"(da1o), "l"(da2), "l"(db), "r"(idesc), "r"(sfa), "r"(sfb),
      "r"(accumulate));
}
// K-major shared-memory descriptor, 32-byte swizzle (SM100, version 1, layout code 6): rows of
// 32 bytes (one 64-element MMA K step), 8-row atoms of 256 B (SBO), the two 16-byte halves of
// a row exchanged when address bit 7 (row bit 2) is set — the layout the packer wrote (R26).
// A tap's operand starts `off` rows into the window, usually inside an atom: the swizzle
// follows the absolute address bits, so the matrix base offset stays 0 (measured: setting it
// to (start >> 7) & 7 gives wrong results).  LBO is unused for swizzled K-major layouts (1).
__device__ __forceinline__ uint64_t sdesc32(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(1) << 16) | (uint64_t(256 >> 4) << 32) | (uint64_t(1) << 46) |
         (uint64_t(6) << 61);
}
// The MMAs of one filter row (3 taps) from one elected lane of a warp that calls this uniformly:
// A at a, a + da1, a + da2 and B at b, b + db, b + 2 db (descriptor units of 16 bytes); the
// descriptor adds stay inside the asm block (uniform datapath, one register -> uniform move per
// row instead of per MMA).
__device__ __forceinline__ void mma3_f4(uint32_t d, uint64_t a, uint64_t b, uint64_t da1, uint64_t da2, uint64_t db,
                                       uint32_t idesc, uint32_t sfa, uint32_t sfb, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p, e;\n.reg .b32 x;\n.reg .b64 a1, a2, b1, b2;\n"
      "elect.sync x|e, 0xffffffff;\n"
      "setp.ne.b32 p, %9, 0;\n"
      "@!e bra SKIP%=;\n"
      "add.s64 a1, %1, %3;\nadd.s64 a2, %1, %4;\nadd.s64 b1, %2, %5;\nadd.s64 b2, b1, %5;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %6, [%7], [%8], p;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], a1, b1, %6, [%7], [%8], 1;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], a2, b2, %6, [%7], [%8], 1;\n"
      "SKIP%=:\n}" ::"r"(d),
      "l"(a), "l"(b), "l"(da1), "l"(da2), "l"(db), "r"(idesc), "r"(sfa), "r"(sfb), "r"(accumulate));
}
// wait until at most n - 1 bulk store groups still read shared memory
__device__ __forceinline__ void bulk_wait_read_n(int n) {
  switch (n) {
    case 1: tc::bulk_wait_read<0>(); break;
    case 2: tc::bulk_wait_read<1>(); break;
    case 3: tc::bulk_wait_read<2>(); break;
    case 4: tc::bulk_wait_read<3>(); break;
    case 5: tc::bulk_wait_read<4>(); break;
    default: tc::bulk_wait_read<5>(); break;
  }
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}

// Per-role cycle accounting of CTA 0 (experiment builds with -DBS_TCW_PROFILE only).
#ifdef BS_TCW_PROFILE
#define PROF_T0() const long long _t0 = clock64()
#define PROF_ADD(acc) (acc) += clock64() - _t0
#else
#define PROF_T0()
#define PROF_ADD(acc)
#endif

// ------------------------------------------------------------------ kernel
template <int DA, int DW, int NP>
__global__ void __launch_bounds__(kThreads, 1)
    tcw_conv_kernel(const __grid_constant__ TwArgs<NP> args, const __grid_constant__ TwMaps<NP> maps) {
  const int S = args.stages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* s_b = smem;                    // resident filter block, or streamed weight slots
  uint8_t* s_a = smem + args.a_off;       // window ring
  uint8_t* s_epi = smem + args.epi_off;   // epilogue staging (1024-aligned)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + args.bar_off);
  uint64_t* full = bars;
  uint64_t* empty = bars + kMaxStages;
  uint64_t* acc_full = bars + 2 * kMaxStages;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* b_full = acc_empty + 2;
  uint64_t* b_empty = b_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(b_empty + 1);
  static_assert(8 * (2 * kMaxStages + 6) + 4 <= kBarBytes, "barrier region");

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // per-problem records in shared memory: every role reads them per tile (parameter-space
  // loads with a runtime problem index are slow constant-cache lookups)
  __shared__ __align__(16) TwProb sprob[NP];
  {
    constexpr int kWords = int(sizeof(TwProb) / 4);
    static_assert(sizeof(TwProb) % 4 == 0, "record size");
    const uint32_t* src = reinterpret_cast<const uint32_t*>(args.prob);
    uint32_t* dst = reinterpret_cast<uint32_t*>(sprob);
    for (int i = tid; i < args.nprob * kWords; i += kThreads) dst[i] = src[i];
  }
#ifdef BS_TCW_PROFILE
  long long pw_empty = 0, pm_acc = 0, pm_full = 0, pe_acc = 0, pe_bar = 0, pm_issue = 0, pm_commit = 0, pe_ld = 0, pe_cvt = 0, pe_sts = 0, pe_st = 0, pe_wr = 0, pm_top = 0,
            pm_loop = 0;
  const long long p_start = clock64();
#endif
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(smem_u32(full + s), 1);
      tc::mbar_init(smem_u32(empty + s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(smem_u32(acc_full + a), 1);
      tc::mbar_init(smem_u32(acc_empty + a), kEpiWarps);
    }
    tc::mbar_init(smem_u32(b_full), 1);
    tc::mbar_init(smem_u32(b_empty), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == kTmaWarp && lane < args.nprob)
    for (int k = 0; k < kBoxMaps; ++k)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.out[lane][k])) : "memory");
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (*tmem_slot != 0u) asm volatile("trap;");  // all 512 columns, from column 0
  constexpr uint32_t tmem = 0;
  constexpr int kSFCols = 16 + 8 * DW;
  if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {  // uniform UE8M0 scales (one warp per lane quarter): SFA digit d = 2^(2d+1), SFB digit e = 2^(2e+1)
#pragma unroll
    for (int c0 = 0; c0 < kSFCols; c0 += 16) {
      uint32_t v[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const int col = c0 + c;
        v[c] = 0x01010101u * uint32_t(col < 16 ? 128 + 2 * (col >> 2) : 128 + 2 * ((col - 16) >> 3));
      }
      tc::tmem_st16(tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(kSF0 + c0), v);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();

  auto tile_mn = [&](const TwProb& P, int tile, uint32_t& mblk, uint32_t& nblk) {
    const uint32_t tl = uint32_t(tile - P.tile0);
    nblk = P.div_nm.div(tl);
    mblk = tl - nblk * P.div_nm.d;
  };
  auto next_prob = [&](int tile, int& pi) {
    while (pi + 1 < args.nprob && tile >= sprob[pi + 1].tile0) ++pi;
  };
  auto bkey = [&](const TwProb& P, int pi, uint32_t nb) { return P.b_res ? (pi << 16) | int(nb) : -2; };

  if (warp == kTmaWarp) {
    if (lane == 0) {
      int stage = 0, pi = 0, key = -1;
      uint32_t phase = 0, bpar = 1;  // b_empty: the first wait passes
      for (int tile = blockIdx.x; tile < args.ntiles; tile += gridDim.x) {
        next_prob(tile, pi);
        const TwProb& P = sprob[pi];
        uint32_t mb, nb;
        tile_mn(P, tile, mb, nb);
        const int k = bkey(P, pi, nb);
        if (k != key) {  // the weights change: wait until no MMA reads the B region
          tc::mbar_wait_sleep(smem_u32(b_empty), bpar);
          bpar ^= 1u;
          key = k;
          if (P.b_res) {
            const uint32_t fb = smem_u32(b_full);
            tc::mbar_expect_tx(fb, uint32_t(P.pairs) * P.bslot);
            const uint8_t* src = P.wt + int64_t(nb) * P.pairs * P.bslot;
            for (int p = 0; p < P.pairs; ++p)
              bulk_load(smem_u32(s_b) + uint32_t(p) * P.bslot, src + int64_t(p) * P.bslot, P.bslot, fb);
          }
        }
        // windows start at the 8-row boundary below the tile's first grid position: rows keep
        // their 32-byte swizzle phase (bit 2 of the row index) in shared memory
        const int64_t q0 = (int64_t(mb) * P.R * P.wg) & ~int64_t(7);
        const uint32_t wbytes = uint32_t(P.lwin) * 32u;
        for (int p = 0; p < P.pairs; ++p) {
          { PROF_T0();
          tc::mbar_wait_sleep(smem_u32(empty + stage), phase ^ 1u);
          PROF_ADD(pw_empty); }
          const uint32_t fb = smem_u32(full + stage);
#ifdef BS_TCW_NOLOAD  // experiment builds only: no window / streamed-weight copies (stale operands)
          tc::mbar_arrive(fb);
          if (++stage == S) {
            stage = 0;
            phase ^= 1u;
          }
          continue;
#endif
          tc::mbar_expect_tx(fb, P.abytes + (P.b_res ? 0u : P.bslot));
          if (!P.b_res)
            bulk_load(smem_u32(s_b) + uint32_t(stage * args.bstride),
                      P.wt + (int64_t(nb) * P.pairs + p) * P.bslot, P.bslot, fb);
          const uint32_t sA = smem_u32(s_a) + uint32_t(stage * args.astage);
#pragma unroll
          for (int d = 0; d < DA; ++d)
            for (int f = 0; f < P.nph; ++f)
              bulk_load(sA + uint32_t(d * P.nph + f) * wbytes,
                        P.act + d * P.digit_bytes + (int64_t(f) * P.pairs + p) * P.slab_bytes + q0 * 32, wbytes, fb);
          if (++stage == S) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    int stage = 0, acc = 0, pi = 0, key = -1;
    uint32_t phase = 0, acc_phase = 0, bfpar = 0;
    const uint32_t sa0 = smem_u32(s_a), sb0 = smem_u32(s_b);
    // the current problem's fields in registers, reloaded only when the tile sequence enters the
    // next problem (per-tile shared-memory reads of the record were ~40% of the MMA warp's time
    // on single-stage tiles)
    int cpi = -1, c_tile0 = 0, c_next0 = 0, c_pairs = 0, c_kh = 0, c_kw = 0, c_wg = 0, c_nph = 0, c_taps = 0, c_sl = 0,
        c_R = 0;
    uint32_t c_idesc = 0, c_wrows = 0, c_bn = 0, c_s0 = 0, c_s1 = 0, c_s2 = 0, c_s3 = 0, c_bslot = 0;
    uint32_t c_a0off0 = 0, c_a0off1 = 0;  // kw == 3 rows: first tap's phase offset, per row parity
    uint64_t c_da10 = 0, c_da11 = 0, c_da2 = 0;
    bool c_bres = false;
    FastDiv c_divnm{1u, 0u, 0u};
    auto load_prob = [&](int q) {
      const TwProb& P = sprob[q];
      cpi = q;
      c_tile0 = P.tile0;
      c_next0 = q + 1 < args.nprob ? sprob[q + 1].tile0 : args.ntiles;
      c_pairs = P.pairs; c_kh = P.kh; c_kw = P.kw; c_wg = P.wg; c_nph = P.nph; c_taps = P.taps; c_sl = P.s - 1;
      c_R = P.R;
      c_idesc = P.idesc; c_wrows = uint32_t(P.lwin); c_bn = uint32_t(P.bn);
      c_s0 = uint32_t(P.slot_of[0]); c_s1 = uint32_t(P.slot_of[1]); c_s2 = uint32_t(P.slot_of[2]);
      c_s3 = uint32_t(P.slot_of[3]);
      c_bslot = P.bslot; c_bres = P.b_res != 0; c_divnm = P.div_nm;
      c_a0off0 = c_s0 * c_wrows * 32u;
      c_a0off1 = c_s2 * c_wrows * 32u;
      c_da10 = uint64_t(((c_s1 * c_wrows + uint32_t(1 >> c_sl)) * 32u - c_a0off0) >> 4);
      c_da11 = uint64_t(((c_s3 * c_wrows + uint32_t(1 >> c_sl)) * 32u - c_a0off1) >> 4);
      c_da2 = uint64_t((uint32_t(2 >> c_sl) * 32u) >> 4);
    };
#ifdef BS_TCW_PROFILE
    long long t_tile = clock64();
#endif
    for (int tile = blockIdx.x; tile < args.ntiles; tile += gridDim.x) {
#ifdef BS_TCW_PROFILE
      pm_loop += clock64() - t_tile;  // previous tile's tail (acc commit, next-tile check, loop)
      const long long t_top = clock64();
#endif
      if (cpi < 0 || tile >= c_next0) {
        next_prob(tile, pi);
        load_prob(pi);
      }
      const uint32_t tl = uint32_t(tile - c_tile0);
      const uint32_t nb = c_divnm.div(tl), mb = tl - nb * c_divnm.d;
      const int k = c_bres ? (pi << 16) | int(nb) : -2;
      if (k != key) {
        key = k;
        if (c_bres) {
          spin_wait(smem_u32(b_full), bfpar);
          bfpar ^= 1u;
        }
      }
      const uint32_t delta = (mb * uint32_t(c_R) * uint32_t(c_wg)) & 7u;  // tile start inside the window's first 8 rows
#ifdef BS_TCW_PROFILE
      pm_top += clock64() - t_top;
#endif
      { PROF_T0();
      spin_wait(smem_u32(acc_empty + acc), acc_phase ^ 1u);
      PROF_ADD(pm_acc); }
      tc::tc_fence_after();
      const uint32_t tacc = uint32_t(acc * kAccCols);
      for (int p = 0; p < c_pairs; ++p) {
        { PROF_T0();
        spin_wait(smem_u32(full + stage), phase);
        PROF_ADD(pm_full); }
        tc::tc_fence_after();
        const uint32_t sA = sa0 + uint32_t(stage * args.astage);
        const uint32_t sB = c_bres ? sb0 + uint32_t(p) * c_bslot : sb0 + uint32_t(stage * args.bstride);
#ifdef BS_TCW_NOMMA  // experiment builds only: no MMAs (the pipeline's barriers still run)
        if (false) {
#else
        {  // the whole warp walks the taps; one elected lane issues each MMA
#endif
          PROF_T0();
#pragma unroll
          for (int e = 0; e < DW; ++e)
#pragma unroll
            for (int d = 0; d < DA; ++d) {
              const uint32_t ad0 = sA + (uint32_t(d * c_nph) * c_wrows + delta) * 32u;
              uint32_t bd = sB + uint32_t(e * c_taps) * c_bn * 32u;
              if (c_kw == 3 && c_kh == 3) {  // all nine taps in one issue block
                const uint32_t a0 = ad0 + c_a0off0;
                const uint32_t a1 = ad0 + uint32_t((1 >> c_sl) * c_wg) * 32u + (c_sl ? c_a0off1 : c_a0off0);
                const uint32_t a2 = ad0 + uint32_t((2 >> c_sl) * c_wg) * 32u + c_a0off0;
                mma9_f4(tacc, sdesc32(a0), sdesc32(a1), sdesc32(a2), sdesc32(bd), c_da10, c_sl ? c_da11 : c_da10, c_da2,
                        uint64_t(c_bn * 2u), c_idesc, uint32_t(kSF0 + 4 * d), uint32_t(kSF0 + 16 + 8 * e),
                        (p | e | d) != 0);
                continue;
              }
              if (c_kw == 3) {  // three taps per row, one issue block
                for (int ky = 0, t = 0; ky < c_kh; ++ky, t += 3, bd += 3u * c_bn * 32u) {
                  const bool oy = (ky & c_sl) != 0;
                  const uint32_t a0 = ad0 + uint32_t((ky >> c_sl) * c_wg) * 32u + (oy ? c_a0off1 : c_a0off0);
                  mma3_f4(tacc, sdesc32(a0), sdesc32(bd), oy ? c_da11 : c_da10, c_da2, uint64_t(c_bn * 2u), c_idesc,
                          uint32_t(kSF0 + 4 * d), uint32_t(kSF0 + 16 + 8 * e), (p | e | d | t) != 0);
                }
                continue;
              }
              int t = 0;
              for (int ky = 0; ky < c_kh; ++ky) {
                const uint32_t rowoff = ad0 + uint32_t((ky >> c_sl) * c_wg) * 32u;
                const bool oy = (ky & c_sl) != 0;
                const uint32_t fe = oy ? c_s2 : c_s0, fo = oy ? c_s3 : c_s1;  // phase slots of even / odd kx
                for (int kx = 0; kx < c_kw; ++kx, ++t, bd += c_bn * 32u) {
                  const uint32_t f = (kx & c_sl) ? fo : fe;
                  const uint32_t a = rowoff + (f * c_wrows + uint32_t(kx >> c_sl)) * 32u;
                  mma_f4_ss_elect(tacc, sdesc32(a), sdesc32(bd), c_idesc, uint32_t(kSF0 + 4 * d),
                                  uint32_t(kSF0 + 16 + 8 * e), (p | e | d | t) != 0);
                }
              }
            }
          PROF_ADD(pm_issue);
        }
        {
          PROF_T0();
          __syncwarp();
          tc::mma_commit_elect(smem_u32(empty + stage));
          PROF_ADD(pm_commit);
        }
        if (++stage == S) {
          stage = 0;
          phase ^= 1u;
        }
      }
#ifdef BS_TCW_PROFILE
      t_tile = clock64();
#endif
      tc::mma_commit_elect(smem_u32(acc_full + acc));
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
      const int nt = tile + int(gridDim.x);  // release the weights when the next tile reads others
      if (nt < args.ntiles) {
        int k2;
        if (nt < c_next0) {
          const uint32_t tl2 = uint32_t(nt - c_tile0);
          k2 = c_bres ? (pi << 16) | int(c_divnm.div(tl2)) : -2;
        } else {
          int npi = pi;
          next_prob(nt, npi);
          uint32_t mb2, nb2;
          tile_mn(sprob[npi], nt, mb2, nb2);
          k2 = bkey(sprob[npi], npi, nb2);
        }
        if (k2 != key) tc::mma_commit_elect(smem_u32(b_empty));
      }
    }
  } else {
    // ================= epilogue: 8 warps, two per TMEM lane quarter (warp % 4 = quarter = tile
    // rows 32q .. 32q+31), splitting the 32-column blocks.  Each warp works on its own: the valid
    // rows among its 32 (grid positions inside the image) are consecutive NHWC output rows
    // m_w .. m_w + nv - 1 in grid order, so each valid lane stages its 32 outputs at its
    // compacted position (rank among the valid lanes; 128-byte rows, 128-byte swizzle by address
    // bits: conflict-free, and TMA boxes may start inside a swizzle atom) and lane 0 stores the
    // block with at most two TMA boxes of 32 columns x 2^k rows — no barrier between warps.
    const int q4 = warp & 3, ew = warp - kEpiWarp0, cb0 = ew >> 2;
    constexpr int kCbStep = kEpiWarps / 4;
    const int ebufs = args.ebufs;
    uint8_t* const s_w = s_epi + ew * ebufs * kStageBuf;
    int acc = 0, buf = 0, pi = 0;
    uint32_t acc_phase = 0;
    // the current problem's fields (and this lane's tile-row coordinates) in registers, reloaded
    // only when the tile sequence enters the next problem
    int cpi = -1, c_tile0 = 0, c_next0 = 0, c_bn = 0, c_oc = 0, c_R = 0, c_G = 0, c_oh = 0, c_ow = 0, c_hg = 0;
    uint32_t c_gr = 0, c_gx = 0;
    bool c_lane_ok = false;
    FastDiv c_divnm{1u, 0u, 0u}, c_divhg{1u, 0u, 0u};
    for (int tile = blockIdx.x; tile < args.ntiles; tile += gridDim.x) {
      if (cpi < 0 || tile >= c_next0) {
        next_prob(tile, pi);
        const TwProb& P = sprob[pi];
        cpi = pi;
        c_tile0 = P.tile0;
        c_next0 = pi + 1 < args.nprob ? sprob[pi + 1].tile0 : args.ntiles;
        c_bn = P.bn; c_oc = P.oc; c_R = P.R; c_G = P.G; c_oh = P.oh; c_ow = P.ow; c_hg = P.hg;
        c_divnm = P.div_nm;
        c_divhg = P.div_hg;
        const uint32_t l = uint32_t(q4 * 32 + lane);  // this lane's tile row: grid row gr, column gx
        c_gr = P.div_wg.div(l);
        c_gx = l - c_gr * uint32_t(P.wg);
        c_lane_ok = int(c_gr) < P.R && int(c_gx) < P.ow;
      }
      const uint32_t tl = uint32_t(tile - c_tile0);
      const uint32_t nb = c_divnm.div(tl), mb = tl - nb * c_divnm.d;
      const int n0 = int(nb) * c_bn, g0 = int(mb) * c_R;
      const int ncb = (min(c_bn, c_oc - n0) + 31) / 32;
      const uint32_t gx = c_gx;
      const uint32_t g = uint32_t(g0) + c_gr;
      const uint32_t img = c_divhg.div(g), gy = g - img * uint32_t(c_hg);
      const bool valid = c_lane_ok && int(g) < c_G && int(gy) < c_oh;
      const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
      const int nv = __popc(vmask);
      const int rank = __popc(vmask & ((1u << lane) - 1u));
      const int m = valid ? (int(img) * c_oh + int(gy)) * c_ow + int(gx) : 0;
      const int m_w = __shfl_sync(0xffffffffu, m, nv ? __ffs(vmask) - 1 : 0);  // first valid row
      { PROF_T0();
      tc::mbar_wait_sleep(smem_u32(acc_full + acc), acc_phase);
      PROF_ADD(pe_acc); }
      tc::tc_fence_after();
      bool released = false;
      for (int cb = cb0; cb < ncb; cb += kCbStep) {
        uint32_t r[32];
        {
          PROF_T0();
          tc::tmem_ld32(tmem + (uint32_t(q4 * 32) << 16) + uint32_t(acc * kAccCols + cb * 32), r);
          PROF_ADD(pe_ld);
        }
        if (cb + kCbStep >= ncb) {
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(smem_u32(acc_empty + acc));
          released = true;
        }
        if (nv == 0) continue;
        PROF_T0();
        // FP32 -> int32 of an exact integer |v| < 2^22 (R17): v + 1.5 * 2^23 has v in its low
        // mantissa bits (FADD + IADD on the full-rate pipes instead of the quarter-rate F2I)
#pragma unroll
        for (int c = 0; c < 32; ++c) r[c] = uint32_t(__float_as_int(__uint_as_float(r[c]) + 12582912.0f) - 0x4B400000);
        PROF_ADD(pe_cvt);
        uint8_t* sb = s_w + buf * kStageBuf;
        {
          PROF_T0();
          if (lane == 0) bulk_wait_read_n(ebufs);  // this buffer's previous stores have read it
          __syncwarp();
          if (valid) {
            const uint32_t row = smem_u32(sb) + uint32_t(rank * 128);
            const uint32_t sw = uint32_t(rank & 7);  // 128-byte swizzle by the row's address bits (as the TMA map)
#pragma unroll
            for (int i = 0; i < 8; ++i)
              sts128(row + ((uint32_t(i) ^ sw) << 4), r[4 * i], r[4 * i + 1], r[4 * i + 2], r[4 * i + 3]);
          }
          tc::fence_proxy_async();
          __syncwarp();
          PROF_ADD(pe_sts);
        }
#ifndef BS_TCW_NOSTORE
        if (lane == 0) {
          PROF_T0();
          // at most two boxes: the largest power of two <= nv at 0, and the smallest power of two
          // >= the remainder ending at nv (rows both cover are written twice with the same values,
          // all inside this warp's rows; fewer than the remainder)
          const int k = 31 - __clz(nv), rem = nv - (1 << k);
          tc::tma_store_2d(&maps.out[pi][k], n0 + cb * 32, m_w, smem_u32(sb));
          if (rem) {
            const int j = 32 - __clz(rem - 1), box = 1 << j;  // ceil(log2(rem)) (0 for rem = 1)
            tc::tma_store_2d(&maps.out[pi][j], n0 + cb * 32, m_w + nv - box, smem_u32(sb) + uint32_t((nv - box) * 128));
          }
          tc::bulk_commit();
          PROF_ADD(pe_st);
        }
#endif
        buf = buf + 1 == ebufs ? 0 : buf + 1;
      }
      if (!released) {
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(smem_u32(acc_empty + acc));
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
    }
    if (lane == 0) tc::bulk_wait_all();
  }

#ifdef BS_TCW_PROFILE
  if (blockIdx.x == 0 && lane == 0) {
    const long long tot = clock64() - p_start;
    if (warp == kTmaWarp) printf("tcw prof: tma   total %lld wait_empty %lld\n", tot, pw_empty);
    if (warp == kMmaWarp) printf("tcw prof: mma   total %lld wait_full %lld wait_acc %lld issue %lld commit %lld top %lld tail %lld\n", tot, pm_full, pm_acc, pm_issue, pm_commit, pm_top, pm_loop);
    if (warp >= kEpiWarp0) printf("tcw prof: epi%d  total %lld wait_acc %lld bar %lld ld %lld cvt %lld sts %lld st %lld wr %lld\n", warp, tot, pe_acc, pe_bar, pe_ld, pe_cvt, pe_sts, pe_st, pe_wr);
  }
#endif
  tc::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ------------------------------------------------------------------ host side
template <int DA, int DW, int NP>
cudaError_t launch(const TcwProblem* ps, int count, cudaStream_t stream) {
  auto kern = tcw_conv_kernel<DA, DW, NP>;
  static std::atomic<uint64_t> configured{0};  // per-device smem opt-in
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  const uint64_t bit = dev < 64 ? uint64_t(1) << dev : 0;
  if (!bit || !(configured.load(std::memory_order_acquire) & bit)) {
    if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit)) return e;
    configured.fetch_or(bit, std::memory_order_release);
  }
  TwArgs<NP> a;
  TwMaps<NP> maps;
  memset(&a, 0, sizeof(a));
  memset(&maps, 0, sizeof(maps));
  a.nprob = count;
  int64_t total = 0;
  int amax = 0, bstream = 0, bres = 0;
  for (int q = 0; q < count; ++q) {
    const TcwProblem& p = ps[q];
    TcwGeom G;
    if (!tcw_geom(p.n, p.h, p.w, p.c, p.oc, p.kh, p.kw, p.sh, p.sw, p.ph, p.pw, G)) return cudaErrorNotSupported;
    if (p.oc % 4 != 0) return cudaErrorNotSupported;  // TMA-store epilogue: 16-byte output rows
    TwProb& P = a.prob[q];
    P.act = p.act;
    P.wt = p.wt;
    P.out = p.out;
    P.slab_bytes = G.pstride * 32;
    P.digit_bytes = G.digit_bytes;
    P.nmb = int((int64_t(p.n) * G.hg + G.R - 1) / G.R);
    P.tile0 = int(total);
    P.bn = G.bn;
    P.pairs = G.cw / 2;
    P.taps = G.taps;
    P.kh = p.kh;
    P.kw = p.kw;
    P.s = G.s;
    P.wg = G.wg;
    P.hg = G.hg;
    P.oh = G.oh;
    P.ow = G.ow;
    P.ow8 = G.ow8;
    P.R = G.R;
    P.nph = G.nph;
    P.lwin = G.lwin;
    P.G = p.n * G.hg;
    P.oc = p.oc;
    for (int f = 0; f < 4; ++f) P.slot_of[f] = G.slot_of[f] < 0 ? 0 : G.slot_of[f];
    P.idesc = tc::idesc_mxf4(G.bn);
    P.bslot = uint32_t(DW) * G.taps * G.bn * 32;
    P.abytes = uint32_t(DA) * G.nph * G.lwin * 32;
    P.b_res = int64_t(P.pairs) * P.bslot <= kBResMax;
    P.div_nm = make_fastdiv(uint32_t(P.nmb));
    P.div_wg = make_fastdiv(uint32_t(G.wg));
    P.div_hg = make_fastdiv(uint32_t(G.hg));
    amax = std::max(amax, int(P.abytes));
    if (P.b_res)
      bres = std::max(bres, int(P.pairs * P.bslot));
    else
      bstream = std::max(bstream, int(P.bslot));
    total += int64_t(P.nmb) * G.nblk;
    if (total > (int64_t(1) << 31) - 1) return cudaErrorInvalidValue;
    const int64_t M = int64_t(p.n) * G.oh * G.ow;
    for (int k = 0; k < kBoxMaps; ++k)
      if (!tc::encode_2d(&maps.out[q][k], CU_TENSOR_MAP_DATA_TYPE_INT32, p.out, uint64_t(p.oc), uint64_t(M),
                         uint64_t(p.oc) * 4, 32, 1u << k, CU_TENSOR_MAP_SWIZZLE_128B))
        return cudaErrorInvalidValue;
  }
  if (total == 0) return cudaSuccess;
  a.ntiles = int(total);
  a.astage = int(ceil_to(amax, 1024));
  a.bstride = int(ceil_to(bstream, 1024));
  // shared memory: [B region][window ring: S stages][epilogue staging: E buffers][barriers].  The ring
  // takes up to kMaxStages stages with the minimum staging; what is left goes to staging buffers (more
  // output bytes in flight: the TMA stores' reads complete only as the stores drain).
  const int budget = kSmemLimit - 1024 - kBarBytes;
  auto need = [&](int s, int e) {
    return ceil_to(std::max(bres, s * a.bstride), 1024) + ceil_to(int64_t(s) * a.astage, 1024) +
           int64_t(e) * kEpiWarps * kStageBuf;
  };
  int S = kMaxStages;
  while (S > 2 && need(S, kEpiBufsMin) > budget) --S;
  if (need(S, kEpiBufsMin) > budget) return cudaErrorNotSupported;
  int E = kEpiBufsMax;
  while (E > kEpiBufsMin && need(S, E) > budget) --E;
  a.stages = S;
  a.ebufs = E;
  a.a_off = int(ceil_to(std::max(bres, S * a.bstride), 1024));
  a.epi_off = int(a.a_off + ceil_to(int64_t(S) * a.astage, 1024));
  a.bar_off = a.epi_off + E * kEpiWarps * kStageBuf;
  int smem = 1024 + a.bar_off + kBarBytes;
  if (smem < kMinSmem) smem = kMinSmem;
  if (smem > kSmemLimit) return cudaErrorNotSupported;
  const int grid = a.ntiles < device_sms() ? a.ntiles : device_sms();
  kern<<<grid, kThreads, smem, stream>>>(a, maps);
  note_launch();
  return cudaPeekAtLastError();
}

template <int DA, int DW>
cudaError_t launch_dd(const TcwProblem* ps, int count, cudaStream_t stream) {
  if (count == 1) return launch<DA, DW, 1>(ps, 1, stream);
  return launch<DA, DW, kGroupMax>(ps, count, stream);
}

}  // namespace tcw

// Up to 16 problems of one (digits) precision per launch, ordered by decreasing K so the
// cheapest tiles form the tail of every CTA's sequence.
cudaError_t launch_tcw_group(const TcwProblem* ps, int count, cudaStream_t stream) {
  for (int q0 = 0; q0 < count; q0 += tcw::kGroupMax) {
    const int cnt = count - q0 < tcw::kGroupMax ? count - q0 : tcw::kGroupMax;
    TcwProblem sp[tcw::kGroupMax];
    for (int q = 0; q < cnt; ++q) sp[q] = ps[q0 + q];
    std::stable_sort(sp, sp + cnt, [](const TcwProblem& x, const TcwProblem& y) {
      return int64_t(x.kh) * x.kw * x.c > int64_t(y.kh) * y.kw * y.c;
    });
    const int da = sp[0].a_digits, dw = sp[0].w_digits;
    for (int q = 1; q < cnt; ++q)
      if (sp[q].a_digits != da || sp[q].w_digits != dw) return cudaErrorInvalidValue;
    cudaError_t e = cudaErrorNotSupported;
    if (da == 1 && dw == 1) e = tcw::launch_dd<1, 1>(sp, cnt, stream);
    else if (da == 2 && dw == 1) e = tcw::launch_dd<2, 1>(sp, cnt, stream);
    else if (da == 1 && dw == 2) e = tcw::launch_dd<1, 2>(sp, cnt, stream);
    else if (da == 2 && dw == 2) e = tcw::launch_dd<2, 2>(sp, cnt, stream);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace bs
