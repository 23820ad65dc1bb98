// tcd_conv.cu — the TMA-fed tensor-core bitserial conv2d / dense on DIGIT-PACKED operands
// (digit.cu): the product path of the timed step.
//
// Eq. 2, regrouped by radix-4 digits of two bit planes (R21):
//   out = sum_{d,e} 4^(d+e) sum_k a_{k,d} w_{k,e},
// every inner sum one exact small-integer contraction on the tensor core
// (tcgen05.mma kind::mxf4: E2M1 digit operands 0.5*{0,+-1,+-2,+-3}, UE8M0 block scales
// 2^(2d+1) / 2^(2e+1) = the digit weights, FP32 accumulation exact below 2^22, R17).
// Because the packer already stores each element's digit as an E2M1 nibble (R24), the
// operands reach shared memory by TMA alone — no producer warps, no per-element work in
// this kernel:
//   * A (activations): conv — one TMA im2col load (cp.async.bulk.tensor.4d.im2col) per
//     (filter tap, channel block, digit): 128 output pixels x cb bytes, traversal stride =
//     conv stride, spatial zero padding = the TMA's out-of-bounds fill (value 0, R20);
//     dense — one tiled 128 x 128-byte box per K chunk and digit;
//   * B (weight digits, prepared once like the weight packing): one 128-byte
//     wide box per stage and digit (the stage's K range is contiguous in a filter row).
// A stage holds 256 K elements (128 bytes per row and digit) — four K=64 MMAs per digit
// pair — in 128 x cb sub-tiles whose swizzle (32/64/128 B) matches cb.
//
// Kernel structure (persistent, warp-specialized, one CTA per SM, 10 warps):
//   warp 0     TMA producer (one lane): A and B boxes of each stage onto full[stage].
//   warp 1     MMA issuer (one elected lane): per stage up to 4 x DA x DW MMAs, A and B
//              from shared memory, accumulator double-buffered in TMEM (2 x BN columns);
//              tcgen05.commit frees the stage / publishes the accumulator.
//   warps 2-9  epilogue (two per TMEM lane quarter): tcgen05.ld -> F2I (exact: the FP32
//              accumulator holds an integer below 2^22) -> 128B-swizzled smem -> TMA store
//              of 32 x 32 int32 boxes (clipped at ragged M / OC), overlapping the next
//              tile's MMAs.
// Tiles: 128 output rows x BN filters, N-major order (CTAs working at the same time share
// a weight block); grouped launches concatenate the tiles of up to 16 problems.
#include "tc_conv_impl.cuh"

namespace bs {
namespace tcd {

using tc::FastDiv;
using tc::make_fastdiv;

constexpr int BM = 128;
constexpr int kTmaWarp = 0, kMmaWarp = 1, kEpiWarp0 = 2, kEpiWarps = 8;
constexpr int kThreads = (kEpiWarp0 + kEpiWarps) * 32;
constexpr int kEpiBufBytes = 32 * 128;  // one 32 x 32 int32 box
constexpr int kEpiBufs = 2;
constexpr int kEpiBytes = kEpiWarps * kEpiBufs * kEpiBufBytes;
constexpr int kBarBytes = 512;
constexpr int kSmemLimit = 226 * 1024;
constexpr int kMinSmem = 116 * 1024;  // > half the SM: one CTA per SM (it owns all of TMEM)
constexpr int kGroupMax = 16;
constexpr int kMaxStages = 8;
constexpr int kStageK = 128;  // bytes of K per stage row and digit (256 E2M1 elements)

template <int DA, int DW, int BN>
struct Cfg {
  static constexpr int kABytes = BM * kStageK;   // per digit
  static constexpr int kBBytes = BN * kStageK;   // per weight digit
  static constexpr int kStageBytes = DA * kABytes + DW * kBBytes;
  static constexpr int kFit = (kSmemLimit - 1024 - kEpiBytes - kBarBytes) / kStageBytes;
  static constexpr int kStages = kFit > kMaxStages ? kMaxStages : kFit;
  static constexpr int kUsed = 1024 + kStages * kStageBytes + kEpiBytes + kBarBytes;
  static constexpr int kBytes = kUsed < kMinSmem ? kMinSmem : kUsed;
  static constexpr int kSF0 = 2 * BN;  // scale factors: SFA 4 columns per digit (16), SFB 8 per digit
  static constexpr int kSFCols = 16 + 8 * DW;
  static_assert(2 * BN + kSFCols <= 512, "tensor memory");
};

struct TdProb {
  int32_t* out;
  int64_t M;
  int oc, epi;
  uint32_t idesc;
  int nmb, tile0, npieces, nstages;
  int cb_log;     // log2 of the piece width in bytes (5, 6, 7)
  uint64_t alay;  // A sub-tile descriptor bits: SBO and swizzle layout code (lay_of)
  int dense;
  int arows;      // rows (dense) or images (conv) per activation digit in the operand map
  int ow, sh, sw, ph, pw, kwid;
  FastDiv div_nm, div_hw, div_ow, div_cpt, div_kwid;
};
template <int NP>
struct TdArgs {
  int nprob, ntiles;
  TdProb prob[NP];
};
template <int NP>
struct TdMaps {
  CUtensorMap a[NP], w[NP], out[NP];
};

// ------------------------------------------------------------------ PTX
__device__ __forceinline__ void tma_load_im2col(uint32_t dst, const CUtensorMap* map, int c, int w, int h, int n,
                                                uint16_t offw, uint16_t offh, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5}], [%6], {%7, %8};" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c), "r"(w), "r"(h), "r"(n), "r"(mbar), "h"(offw), "h"(offh)
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

// K-major shared-memory descriptor (SM100): start >> 4, LBO 1 (unused when swizzled), SBO, version 1,
// layout code (2 = 128B, 4 = 64B, 6 = 32B swizzle); `lay` holds SBO>>4 << 32 | code << 61.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint64_t lay) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(1) << 16) | (uint64_t(1) << 46) | lay;
}
inline uint64_t lay_of(int cb_log) {
  const int code = cb_log == 7 ? 2 : (cb_log == 6 ? 4 : 6);
  const uint64_t sbo = uint64_t(8) << cb_log;  // 8 rows x cb bytes
  return ((sbo >> 4) << 32) | (uint64_t(code) << 61);
}

// ------------------------------------------------------------------ kernel
template <int DA, int DW, int BN, int NP>
__global__ void __launch_bounds__(kThreads, 1)
    tcd_conv_kernel(const __grid_constant__ TdArgs<NP> args, const __grid_constant__ TdMaps<NP> maps) {
  using C = Cfg<DA, DW, BN>;
  constexpr int S = C::kStages;
  static_assert(S >= 2, "two stages");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* s_stage = smem;
  uint8_t* s_epi = smem + S * C::kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_epi + kEpiBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* acc_full = bars + 2 * S;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  static_assert(8 * (2 * kMaxStages + 4) + 4 <= kBarBytes, "barrier region");

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(smem_u32(full + s), 1);
      tc::mbar_init(smem_u32(empty + s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(smem_u32(acc_full + a), 1);
      tc::mbar_init(smem_u32(acc_empty + a), kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == kTmaWarp && lane < args.nprob) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.a[lane])) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.w[lane])) : "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (*tmem_slot != 0u) asm volatile("trap;");  // all 512 columns, from column 0
  constexpr uint32_t tmem = 0;
  // uniform UE8M0 scale factors: SFA digit d (4 columns) = 2^(2d+1), SFB digit e (8 columns) = 2^(2e+1)
  if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
#pragma unroll
    for (int c0 = 0; c0 < C::kSFCols; c0 += 16) {
      uint32_t v[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const int col = c0 + c;
        v[c] = 0x01010101u * uint32_t(col < 16 ? 128 + 2 * (col >> 2) : 128 + 2 * ((col - 16) >> 3));
      }
      tc::tmem_st16(tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(C::kSF0 + c0), v);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();

  auto tile_mn = [&](const TdProb& P, int tile, uint32_t& mblk, uint32_t& nblk) {
    const uint32_t tl = uint32_t(tile - P.tile0);
    nblk = P.div_nm.div(tl);
    mblk = tl - nblk * P.div_nm.d;
  };
  auto next_prob = [&](int tile, int& pi) {
    while (pi + 1 < args.nprob && tile >= args.prob[pi + 1].tile0) ++pi;
  };

  if (warp == kTmaWarp) {
    if (lane == 0) {
      int stage = 0, pi = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < args.ntiles; tile += gridDim.x) {
        next_prob(tile, pi);
        const TdProb& P = args.prob[pi];
        uint32_t mb, nb;
        tile_mn(P, tile, mb, nb);
        const int m0 = int(mb) * BM, n0 = int(nb) * BN;
        int img = 0, wc = 0, hc = 0;
        if (!P.dense) {
          const uint32_t b = P.div_hw.div(uint32_t(m0)), rem = uint32_t(m0) - b * P.div_hw.d;
          const uint32_t oy = P.div_ow.div(rem), ox = rem - oy * P.div_ow.d;
          img = int(b);
          wc = int(ox) * P.sw - P.pw;
          hc = int(oy) * P.sh - P.ph;
        }
        const int cb = 1 << P.cb_log, pps = kStageK >> P.cb_log;
        for (int s = 0; s < P.nstages; ++s) {
          tc::mbar_wait_sleep(smem_u32(empty + stage), phase ^ 1u);
          const int p0 = s * pps;
          const int npc = min(pps, P.npieces - p0);
          const uint32_t fb = smem_u32(full + stage);
          tc::mbar_expect_tx(fb, uint32_t(npc * DA * BM * cb + DW * C::kBBytes));
          const uint32_t sA = smem_u32(s_stage + stage * C::kStageBytes);
          const uint32_t sB = sA + DA * C::kABytes;
#pragma unroll
          for (int e = 0; e < DW; ++e) tc::tma_load_2d(sB + e * C::kBBytes, &maps.w[pi], p0 * cb, e * P.oc + n0, fb);
          for (int pc = 0; pc < npc; ++pc) {
            const int p = p0 + pc;
            if (P.dense) {
#pragma unroll
              for (int d = 0; d < DA; ++d)
                tc::tma_load_2d(sA + d * C::kABytes + pc * (BM << P.cb_log), &maps.a[pi], p * cb, d * P.arows + m0, fb);
            } else {
              const int tap = int(P.div_cpt.div(uint32_t(p))), cbi = p - tap * int(P.div_cpt.d);
              const int ky = int(P.div_kwid.div(uint32_t(tap))), kx = tap - ky * P.kwid;
#pragma unroll
              for (int d = 0; d < DA; ++d)
                tma_load_im2col(sA + d * C::kABytes + pc * (BM << P.cb_log), &maps.a[pi], cbi * cb, wc, hc,
                                img + d * P.arows, uint16_t(kx), uint16_t(ky), fb);
            }
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    int stage = 0, acc = 0, pi = 0;
    uint32_t phase = 0, acc_phase = 0;
    const uint32_t sbase = smem_u32(s_stage);
    for (int tile = blockIdx.x; tile < args.ntiles; tile += gridDim.x) {
      next_prob(tile, pi);
      const TdProb& P = args.prob[pi];
      constexpr uint32_t kIdesc = NP == 1 ? tc::idesc_mxf4(BN) : 0u;
      const uint32_t idesc = NP == 1 ? kIdesc : P.idesc;
      const uint64_t alay = P.alay;
      const uint64_t blay = tc::smem_desc_sw128(0) & ~uint64_t(0x3FFF);
      const int cb_log = P.cb_log, kpp_log = cb_log - 5;  // MMA K-steps (32 bytes) per piece
      tc::mbar_wait(smem_u32(acc_empty + acc), acc_phase ^ 1u);
      tc::tc_fence_after();
      const uint32_t tacc = uint32_t(acc * BN);
      for (int s = 0; s < P.nstages; ++s) {
        tc::mbar_wait(smem_u32(full + stage), phase);
        tc::tc_fence_after();
        const int npc = min(kStageK >> cb_log, P.npieces - s * (kStageK >> cb_log));
        const int nsteps = npc << kpp_log;
        const uint32_t sA = sbase + stage * C::kStageBytes;
        const uint32_t sB = sA + DA * C::kABytes;
        if (elect_one()) {
          for (int u = 0; u < nsteps; ++u) {
            const uint32_t aoff = uint32_t(((u >> kpp_log) << (7 + cb_log)) + ((u & ((1 << kpp_log) - 1)) << 5));
#pragma unroll
            for (int d = 0; d < DA; ++d)
#pragma unroll
              for (int e = 0; e < DW; ++e)
                mma_f4_ss(tacc, sdesc(sA + d * C::kABytes + aoff, alay), sdesc(sB + e * C::kBBytes + 32 * u, blay),
                          idesc, uint32_t(C::kSF0 + 4 * d), uint32_t(C::kSF0 + 16 + 8 * e), (s | u | d | e) != 0);
          }
        }
        __syncwarp();
        tc::mma_commit_elect(smem_u32(empty + stage));
        if (++stage == S) {
          stage = 0;
          phase ^= 1u;
        }
      }
      tc::mma_commit_elect(smem_u32(acc_full + acc));
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
    }
  } else {
    // epilogue: warp % 4 = TMEM lane quarter; the two warps of a quarter split the 32-column blocks
    const int q = warp & 3;
    const int ew = warp - kEpiWarp0, cb0 = ew >> 2;
    constexpr int kCbStep = kEpiWarps / 4;
    uint8_t* ebuf = s_epi + ew * (kEpiBufs * kEpiBufBytes);
    int acc = 0, buf = 0, pi = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < args.ntiles; tile += gridDim.x) {
      next_prob(tile, pi);
      const TdProb& P = args.prob[pi];
      uint32_t mb, nb;
      tile_mn(P, tile, mb, nb);
      const int64_t m0 = int64_t(mb) * BM;
      const int n0 = int(nb) * BN, oc = P.oc;
      const int ncb = min(BN, oc - n0 + 31) / 32;
      tc::mbar_wait_sleep(smem_u32(acc_full + acc), acc_phase);
      tc::tc_fence_after();
      bool released = false;
      for (int cbk = cb0; cbk < ncb; cbk += kCbStep) {
        uint32_t r[32];
        tc::tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(acc * BN + cbk * 32), r);
#pragma unroll
        for (int c = 0; c < 32; ++c) r[c] = uint32_t(__float2int_rz(__uint_as_float(r[c])));
        if (cbk + kCbStep >= ncb) {
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(smem_u32(acc_empty + acc));
          released = true;
        }
        if (P.epi == tc::kEpiTma) {
          if (lane == 0) tc::bulk_wait_read<kEpiBufs - 1>();
          __syncwarp();
          uint8_t* sb = ebuf + buf * kEpiBufBytes + lane * 128;
          const uint32_t swz = uint32_t(lane & 7);
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<uint4*>(sb + ((uint32_t(c) ^ swz) << 4)) =
                make_uint4(r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);
          tc::fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            tc::tma_store_2d(&maps.out[pi], n0 + cbk * 32, int(m0) + q * 32, smem_u32(ebuf + buf * kEpiBufBytes));
            tc::bulk_commit();
          }
          buf = buf + 1 == kEpiBufs ? 0 : buf + 1;
        } else {  // oc % 4 != 0: bounded scalar stores
          const int64_t row = m0 + q * 32 + lane;
          if (row < P.M) {
            int32_t* dst = P.out + row * oc;
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              const int col = n0 + cbk * 32 + c;
              if (col < oc) dst[col] = int32_t(r[c]);
            }
          }
        }
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

  tc::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ------------------------------------------------------------------ host side
inline PFN_cuTensorMapEncodeIm2col_v12000 encode_im2col_fn() {
  static PFN_cuTensorMapEncodeIm2col_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(f);
    return static_cast<PFN_cuTensorMapEncodeIm2col_v12000>(nullptr);
  }();
  return fn;
}

inline CUtensorMapSwizzle swz_of(int cb_log) {
  return cb_log == 7 ? CU_TENSOR_MAP_SWIZZLE_128B : (cb_log == 6 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
}

// Fill one problem's record and tensor maps.  cudaErrorNotSupported: geometry outside what
// the TMA im2col mode encodes (padding corners beyond [-128, 127], stride > 8).
inline cudaError_t make_prob(TdProb& P, CUtensorMap& ta, CUtensorMap& tw, CUtensorMap& to, const TcdProblem& p,
                             int tile0, int bn, int64_t& tiles) {
  memset(&P, 0, sizeof(P));
  const int64_t cbytes = digit_row_bytes(p.c);  // bytes per pixel (row) and digit
  const int taps = p.kh * p.kw;
  P.out = p.out;
  P.M = int64_t(p.n) * p.oh * p.ow;
  P.oc = p.oc;
  P.epi = p.oc % 4 == 0 ? tc::kEpiTma : tc::kEpiScalar;
  P.idesc = tc::idesc_mxf4(p.oc <= 64 ? 64 : bn);
  P.nmb = int((P.M + BM - 1) / BM);
  const int ntn = (p.oc + bn - 1) / bn;
  tiles = int64_t(P.nmb) * ntn;
  P.tile0 = tile0;
  P.div_nm = make_fastdiv(uint32_t(P.nmb));
  P.dense = p.dense;
  P.cb_log = p.dense ? 7 : (cbytes % 128 == 0 ? 7 : (cbytes % 64 == 0 ? 6 : 5));
  const int cb = 1 << P.cb_log;
  const int64_t cpt = p.dense ? (cbytes + 127) / 128 : cbytes / cb;  // pieces per tap
  P.npieces = int(taps * cpt);
  const int pps = kStageK / cb;
  P.nstages = (P.npieces + pps - 1) / pps;
  P.alay = lay_of(P.cb_log);
  P.ow = p.ow;
  P.sh = p.sh;
  P.sw = p.sw;
  P.ph = p.ph;
  P.pw = p.pw;
  P.kwid = p.kw;
  P.div_hw = make_fastdiv(uint32_t(p.oh) * uint32_t(p.ow));
  P.div_ow = make_fastdiv(uint32_t(p.ow));
  P.div_cpt = make_fastdiv(uint32_t(cpt));
  P.div_kwid = make_fastdiv(uint32_t(p.kw));
  const int64_t wrow = int64_t(taps) * cbytes;  // weight-digit row bytes
  if (!tc::encode_2d(&tw, CU_TENSOR_MAP_DATA_TYPE_UINT8, p.wdig, uint64_t(wrow), uint64_t(p.w_digits) * p.oc,
                     uint64_t(wrow), kStageK, bn, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  if (p.dense) {
    P.arows = p.n;
    if (!tc::encode_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, p.act, uint64_t(cbytes), uint64_t(p.a_digits) * p.n,
                       uint64_t(cbytes), kStageK, BM, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  } else {
    P.arows = p.n;
    const int lower[2] = {-p.pw, -p.ph};
    const int upper[2] = {(p.ow - 1) * p.sw - p.pw - (p.w - 1), (p.oh - 1) * p.sh - p.ph - (p.h - 1)};
    for (int i = 0; i < 2; ++i)
      if (lower[i] < -128 || lower[i] > 127 || upper[i] < -128 || upper[i] > 127) return cudaErrorNotSupported;
    if (p.sh > 8 || p.sw > 8 || p.kh > 65536 || p.kw > 65536) return cudaErrorNotSupported;
    auto enc = encode_im2col_fn();
    if (!enc) return cudaErrorNotSupported;
    const cuuint64_t dims[4] = {cuuint64_t(cbytes), cuuint64_t(p.w), cuuint64_t(p.h), cuuint64_t(p.a_digits) * p.n};
    const cuuint64_t strides[3] = {cuuint64_t(cbytes), cuuint64_t(cbytes) * p.w, cuuint64_t(cbytes) * p.w * p.h};
    const cuuint32_t estr[4] = {1, cuuint32_t(p.sw), cuuint32_t(p.sh), 1};
    if (enc(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<uint8_t*>(p.act), dims, strides, lower, upper,
            cuuint32_t(cb), cuuint32_t(BM), estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz_of(P.cb_log),
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  if (P.epi == tc::kEpiTma)
    return tc::encode_2d(&to, CU_TENSOR_MAP_DATA_TYPE_INT32, p.out, uint64_t(p.oc), uint64_t(P.M), uint64_t(p.oc) * 4,
                         32, 32, CU_TENSOR_MAP_SWIZZLE_128B)
               ? cudaSuccess
               : cudaErrorInvalidValue;
  to = tw;  // unused
  return cudaSuccess;
}

template <int DA, int DW, int BN, int NP>
cudaError_t launch(const TcdProblem* ps, int count, cudaStream_t stream) {
  using C = Cfg<DA, DW, BN>;
  auto kern = tcd_conv_kernel<DA, DW, BN, NP>;
  static std::atomic<uint64_t> configured{0};  // per-device smem opt-in
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  const uint64_t bit = dev < 64 ? uint64_t(1) << dev : 0;
  if (!bit || !(configured.load(std::memory_order_acquire) & bit)) {
    if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kBytes)) return e;
    configured.fetch_or(bit, std::memory_order_release);
  }
  TdArgs<NP> a;
  TdMaps<NP> maps;
  memset(&a, 0, sizeof(a));
  memset(&maps, 0, sizeof(maps));
  a.nprob = count;
  int64_t total = 0;
  for (int q = 0; q < count; ++q) {
    int64_t tiles = 0;
    if (cudaError_t e = make_prob(a.prob[q], maps.a[q], maps.w[q], maps.out[q], ps[q], int(total), BN, tiles)) return e;
    total += tiles;
    if (total > (int64_t(1) << 31) - 1) return cudaErrorInvalidValue;
  }
  if (total == 0) return cudaSuccess;
  a.ntiles = int(total);
  const int grid = a.ntiles < device_sms() ? a.ntiles : device_sms();
  kern<<<grid, kThreads, C::kBytes, stream>>>(a, maps);
  note_launch();
  return cudaPeekAtLastError();
}

template <int DA, int DW>
cudaError_t launch_dd(const TcdProblem* ps, int count, cudaStream_t stream) {
  bool wide = false;
  for (int q = 0; q < count; ++q) wide |= ps[q].oc > 64;
  if (const int v = tuning(kTuneTileN)) wide = v > 64;
  if (count == 1) return wide ? launch<DA, DW, 128, 1>(ps, 1, stream) : launch<DA, DW, 64, 1>(ps, 1, stream);
  return wide ? launch<DA, DW, 128, kGroupMax>(ps, count, stream) : launch<DA, DW, 64, kGroupMax>(ps, count, stream);
}

}  // namespace tcd

// Up to 16 problems of one (digits) precision per launch, ordered by decreasing K so the
// cheapest tiles form the tail of every CTA's sequence.
cudaError_t launch_tcd_group(const TcdProblem* ps, int count, cudaStream_t stream) {
  for (int q0 = 0; q0 < count; q0 += tcd::kGroupMax) {
    const int cnt = count - q0 < tcd::kGroupMax ? count - q0 : tcd::kGroupMax;
    TcdProblem sp[tcd::kGroupMax];
    for (int q = 0; q < cnt; ++q) sp[q] = ps[q0 + q];
    std::stable_sort(sp, sp + cnt, [](const TcdProblem& x, const TcdProblem& y) {
      return int64_t(x.kh) * x.kw * x.c > int64_t(y.kh) * y.kw * y.c;
    });
    const int da = sp[0].a_digits, dw = sp[0].w_digits;
    for (int q = 1; q < cnt; ++q)
      if (sp[q].a_digits != da || sp[q].w_digits != dw) return cudaErrorInvalidValue;
    cudaError_t e = cudaErrorNotSupported;
    if (da == 1 && dw == 1) e = tcd::launch_dd<1, 1>(sp, cnt, stream);
    else if (da == 2 && dw == 1) e = tcd::launch_dd<2, 1>(sp, cnt, stream);
    else if (da == 1 && dw == 2) e = tcd::launch_dd<1, 2>(sp, cnt, stream);
    else if (da == 2 && dw == 2) e = tcd::launch_dd<2, 2>(sp, cnt, stream);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace bs
