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
constexpr int kTmaWarp = 0, kMmaWarp = 1, kEpiWarp0 = 2, kEpiWarps = 8, kProdWarp0 = 10, kProdWarps = 4;
constexpr int kThreads = (kProdWarp0 + kProdWarps) * 32;
constexpr int kEpiBufBytes = 32 * 128;  // one 32 x 32 int32 box
// staging buffers per epilogue warp: 2 (a store in flight while the next box is staged); the
// 224-wide GEMM tiles keep 1 so a fourth operand stage fits
constexpr int epi_bufs(int bn) { return bn >= 224 ? 1 : 2; }
constexpr int epi_bytes(int bn) { return kEpiWarps * epi_bufs(bn) * kEpiBufBytes; }
constexpr int kBarBytes = 512;
constexpr int kSmemLimit = 226 * 1024;
constexpr int kMinSmem = 116 * 1024;  // > half the SM: one CTA per SM (it owns all of TMEM)
constexpr int kGroupMax = 16;
constexpr int kMaxStages = 12;
constexpr int kStageK = 128;          // bytes of K per stage row and digit (256 E2M1 elements)
constexpr int kBResMax = 96 * 1024;   // largest weight block kept resident in shared memory
constexpr int kProdLag = 3;           // stages a producer thread keeps in flight before it signals one
constexpr int budget(int bn) { return kSmemLimit - 1024 - epi_bytes(bn) - kBarBytes; }  // B region + A ring

template <int DA, int DW, int BN>
struct Cfg {
  static constexpr int kABytes = BM * kStageK;   // A stage bytes per digit
  static constexpr int kBBytes = BN * kStageK;   // one 128-byte K chunk of one weight digit
  static constexpr int kAStage = DA * kABytes;
  static constexpr int kBSlot = DW * kBBytes;    // streamed weights: one stage's chunk, every digit
  static constexpr int kSF0 = 2 * BN;  // scale factors: SFA 4 columns per digit (16), SFB 8 per digit
  static constexpr int kSFCols = 16 + 8 * DW;
  static_assert(2 * BN + kSFCols <= 512, "tensor memory");
  static constexpr int kEpiBufs = epi_bufs(BN), kEpiBytes = epi_bytes(BN), kBudget = budget(BN);
  static constexpr bool kFits = kBudget >= 2 * (kAStage + kBSlot);  // two streamed stages
};

struct TdProb {
  int32_t* out;
  const uint8_t* act;  // activation digits (cp.async producers)
  int64_t M, plane_bytes;  // output rows; bytes per activation digit plane
  int oc, epi;
  uint32_t idesc;
  int nmb, tile0, npieces, nstages;
  int cb_log;      // log2 of the piece width in bytes (5, 6, 7)
  uint64_t alay;   // A sub-tile descriptor bits: SBO and swizzle layout code (lay_of)
  int dense;
  int a_tma;       // 1: A by TMA (tiled for dense, im2col for conv); 0: cp.async by the producer warps
  int b_res;       // 1: the whole weight block of an N block resident in the B region
  int nchk;        // 128-byte chunks per weight row
  int bres_bytes;  // resident block bytes (DW * nchk * BN * 128)
  int arows;       // rows (dense) or images (conv) per activation digit in the operand map
  int h, w, cbytes, ow, sh, sw, ph, pw, kwid;
  FastDiv div_nm, div_hw, div_ow, div_cpt, div_kwid;
};
template <int NP>
struct TdArgs {
  int nprob, ntiles;
  int stages;      // A ring stages (runtime: depends on the B region)
  int b_region;    // bytes of the B region (resident blocks, or streamed chunk slots)
  int gather;      // the producer warps gather every problem's activations (else all come by TMA)
  int mc;          // clusters of 2 CTAs on adjacent tiles of one N block: each CTA loads half of every weight
                   // chunk and multicasts it to both (dense, streamed weights, even tile counts)
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

// Busy wait (try_wait without a suspend-time hint) for the MMA warp, the only warp of its role.
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

__device__ __forceinline__ void tma_load_2d_mc(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t mbar,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(mbar), "h"(mask)
      : "memory");
}
// tcgen05.commit arriving on the barrier at this shared-memory offset in every CTA of `mask`
__device__ __forceinline__ void mma_commit_mc_elect(uint32_t mbar, uint16_t mask) {
  asm volatile(
      "{.reg .pred e; .reg .b32 x; elect.sync x|e, 0xffffffff;\n"
      "@!e bra SKIP%=;\n"
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
      "SKIP%=:\n}" ::"r"(mbar),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
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

__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}

// Which weights a tile's MMAs read: a resident block (problem, N block) or the streamed slots.
__device__ __forceinline__ int bkey(const TdProb& P, int pi, uint32_t nb) { return P.b_res ? (pi << 16) | int(nb) : -2; }

// ------------------------------------------------------------------ kernel
template <int DA, int DW, int BN, int NP>
__global__ void __launch_bounds__(kThreads, 1)
    tcd_conv_kernel(const __grid_constant__ TdArgs<NP> args, const __grid_constant__ TdMaps<NP> maps) {
  using C = Cfg<DA, DW, BN>;
  static_assert(C::kFits, "two streamed stages");
  const int S = args.stages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* s_b = smem;                          // B region: resident block or streamed chunk slots
  uint8_t* s_a = smem + args.b_region;          // A ring
  uint8_t* s_epi = s_a + S * C::kAStage;
  constexpr int kEpiBufs = C::kEpiBufs;
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_epi + C::kEpiBytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kMaxStages;
  uint64_t* acc_full = bars + 2 * kMaxStages;
  uint64_t* acc_empty = acc_full + 2;
  uint64_t* b_full = acc_empty + 2;
  uint64_t* b_empty = b_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(b_empty + 1);
  static_assert(8 * (2 * kMaxStages + 6) + 4 <= kBarBytes, "barrier region");

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(smem_u32(full + s), args.gather ? 1 + kProdWarps : 1);  // TMA thread (+ each producer warp)
      tc::mbar_init(smem_u32(empty + s), args.mc ? 2 : 1);  // (multicast: both CTAs' MMAs release a stage)
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
  if (warp == kTmaWarp && lane < args.nprob) {
    if (args.prob[lane].a_tma)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.a[lane])) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.w[lane])) : "memory");
    if (args.prob[lane].epi == tc::kEpiTma)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.out[lane])) : "memory");
  }
  tc::tc_fence_before();
  __syncthreads();
  if (args.mc) cluster_sync();  // the peer's multicasts and commits target these barriers
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
    // ================= TMA: weights (a resident block per (problem, N block), reloaded only when
    // it changes, after the MMA warp released the previous one; or one streamed chunk per stage),
    // and the activations of TMA-sourced problems (dense tiles, or conv im2col)
    if (lane == 0) {
      int stage = 0, pi = 0, key = -1;
      uint32_t phase = 0, bpar = 1;  // b_empty: the first wait passes (nothing loaded yet)
      for (int tile = blockIdx.x; tile < args.ntiles; tile += gridDim.x) {
        next_prob(tile, pi);
        const TdProb& P = args.prob[pi];
        uint32_t mb, nb;
        tile_mn(P, tile, mb, nb);
        const int m0 = int(mb) * BM, n0 = int(nb) * BN;
        const int k = bkey(P, pi, nb);
        if (k != key) {  // the weights this tile reads change: wait until no MMA reads the B region
          tc::mbar_wait_sleep(smem_u32(b_empty), bpar);
          bpar ^= 1u;
          key = k;
          if (P.b_res) {
            const uint32_t fb = smem_u32(b_full);
            tc::mbar_expect_tx(fb, uint32_t(P.bres_bytes));
            for (int e = 0; e < DW; ++e)
              for (int c = 0; c < P.nchk; ++c)
                tc::tma_load_2d(smem_u32(s_b) + uint32_t((e * P.nchk + c) * C::kBBytes), &maps.w[pi], c * kStageK,
                                e * P.oc + n0, fb);
          }
        }
        int img = 0, wc = 0, hc = 0;
        if (!P.dense && P.a_tma) {
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
          tc::mbar_expect_tx(fb, uint32_t((P.a_tma ? npc * DA * BM * cb : 0) + (P.b_res ? 0 : C::kBSlot)));
          const uint32_t sA = smem_u32(s_a + stage * C::kAStage);
          if (!P.b_res) {
            const uint32_t sB = smem_u32(s_b + stage * C::kBSlot);
#pragma unroll
            for (int e = 0; e < DW; ++e) {
              if (args.mc) {  // this CTA's half of the rows, into both CTAs' slots
                const int half = BN / 2, cr = int(cluster_rank());
                tma_load_2d_mc(sB + e * C::kBBytes + uint32_t(cr * half * kStageK), &maps.w[pi], p0 * cb,
                               e * P.oc + n0 + cr * half, fb, uint16_t(3));
              } else {
                tc::tma_load_2d(sB + e * C::kBBytes, &maps.w[pi], p0 * cb, e * P.oc + n0, fb);
              }
            }
          }
          if (P.a_tma) {
            for (int pc = 0; pc < npc; ++pc) {
              const int p = p0 + pc;
              if (P.dense) {
#pragma unroll
                for (int d = 0; d < DA; ++d)
                  tc::tma_load_2d(sA + d * C::kABytes + pc * (BM << P.cb_log), &maps.a[pi], p * cb, d * P.arows + m0,
                                  fb);
              } else {
                const int tap = int(P.div_cpt.div(uint32_t(p))), cbi = p - tap * int(P.div_cpt.d);
                const int ky = int(P.div_kwid.div(uint32_t(tap))), kx = tap - ky * P.kwid;
#pragma unroll
                for (int d = 0; d < DA; ++d)
                  tma_load_im2col(sA + d * C::kABytes + pc * (BM << P.cb_log), &maps.a[pi], cbi * cb, wc, hc,
                                  img + d * P.arows, uint16_t(kx), uint16_t(ky), fb);
              }
            }
          }
          if (++stage == S) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp >= kProdWarp0 && !args.gather) {
    // every operand of this launch comes by TMA: the producer warps have nothing to do
  } else if (warp >= kProdWarp0) {
    // ================= activation producers (cp.async): thread r gathers output row r's
    // receptive-field pixels, piece by piece, 16 bytes per copy into the 32/64/128-byte swizzled
    // A sub-tiles (zero fill = padding); a stage is signalled kProdLag stages later, once the
    // thread's copies of it have landed (cp.async.wait_group, then a proxy fence: the tensor
    // core reads shared memory through the async proxy).
    const int r = tid - kProdWarp0 * 32;  // tile row
    const int lag = S - 1 < kProdLag ? S - 1 : kProdLag;  // < S: the oldest signalled stage frees the next wait
    int stage = 0, pi = 0, pend = 0, sig = 0;
    uint32_t phase = 0;
    auto signal = [&]() {  // oldest un-signalled stage: this warp's copies landed
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(smem_u32(full + sig));
      if (++sig == S) sig = 0;
    };
    for (int tile = blockIdx.x; tile < args.ntiles; tile += gridDim.x) {
      next_prob(tile, pi);
      const TdProb& P = args.prob[pi];
      const bool gather = !P.a_tma;
      const uint8_t* base = P.act;
      int iy0 = 0, ix0 = 0;
      bool rok = false;
      if (gather) {
        uint32_t mb, nb;
        tile_mn(P, tile, mb, nb);
        const int64_t m = int64_t(mb) * BM + r;
        rok = m < P.M;
        const uint32_t mm = rok ? uint32_t(m) : 0u;
        const uint32_t b = P.div_hw.div(mm), rem = mm - b * P.div_hw.d;
        const uint32_t oy = P.div_ow.div(rem), ox = rem - oy * P.div_ow.d;
        iy0 = int(oy) * P.sh - P.ph;
        ix0 = int(ox) * P.sw - P.pw;
        base = P.act + int64_t(b) * P.h * P.w * P.cbytes;
      }
      const int cb_log = P.cb_log, cb = 1 << cb_log, pps = kStageK >> cb_log;
      const int nch = cb >> 4;                               // 16-byte chunks per piece row
      const uint32_t swz = uint32_t((r << cb_log) >> 7) & uint32_t(nch - 1);
      for (int s = 0; s < P.nstages; ++s) {
        tc::mbar_wait_sleep(smem_u32(empty + stage), phase ^ 1u);
        if (gather) {
          const int p0 = s * pps;
          const int npc = min(pps, P.npieces - p0);
          const uint32_t sA = smem_u32(s_a + stage * C::kAStage) + uint32_t(r << cb_log);
          for (int pc = 0; pc < npc; ++pc) {
            const int p = p0 + pc;
            const int tap = int(P.div_cpt.div(uint32_t(p))), cbi = p - tap * int(P.div_cpt.d);
            const int ky = int(P.div_kwid.div(uint32_t(tap))), kx = tap - ky * P.kwid;
            const int iy = iy0 + ky, ix = ix0 + kx;
            const bool ok = rok && unsigned(iy) < unsigned(P.h) && unsigned(ix) < unsigned(P.w);
            const uint8_t* src = base + (ok ? (int64_t(iy) * P.w + ix) * P.cbytes + (cbi << cb_log) : 0);
            const uint32_t dst = sA + uint32_t(pc * (BM << cb_log));
#pragma unroll
            for (int d = 0; d < DA; ++d)
              for (int j = 0; j < nch; ++j)
                cp_async16_zfill(dst + uint32_t(d * C::kABytes) + ((uint32_t(j) ^ swz) << 4), src + d * P.plane_bytes + 16 * j,
                                 ok);
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (pend == lag) {
          if (lag == 3)
            asm volatile("cp.async.wait_group 3;" ::: "memory");
          else if (lag == 2)
            asm volatile("cp.async.wait_group 2;" ::: "memory");
          else
            asm volatile("cp.async.wait_group 1;" ::: "memory");
          signal();
        } else {
          ++pend;
        }
        if (++stage == S) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    for (; pend > 0; --pend) signal();
  } else if (warp == kMmaWarp) {
    int stage = 0, acc = 0, pi = 0, key = -1;
    uint32_t phase = 0, acc_phase = 0, bfpar = 0;
    const uint32_t sa0 = smem_u32(s_a), sb0 = smem_u32(s_b);
    const uint64_t blay = tc::smem_desc_sw128(0) & ~uint64_t(0x3FFF);
    for (int tile = blockIdx.x; tile < args.ntiles; tile += gridDim.x) {
      next_prob(tile, pi);
      const TdProb& P = args.prob[pi];
      uint32_t mb, nb;
      tile_mn(P, tile, mb, nb);
      const int k = bkey(P, pi, nb);
      if (k != key) {  // (the previous block was released after the previous tile)
        key = k;
        if (P.b_res) {
          spin_wait(smem_u32(b_full), bfpar);
          bfpar ^= 1u;
        }
      }
      constexpr uint32_t kIdesc = NP == 1 ? tc::idesc_mxf4(BN) : 0u;
      const uint32_t idesc = NP == 1 ? kIdesc : P.idesc;
      const uint64_t alay = P.alay;
      const int cb_log = P.cb_log, kpp_log = cb_log - 5;  // MMA K-steps (32 bytes) per piece
      spin_wait(smem_u32(acc_empty + acc), acc_phase ^ 1u);
      tc::tc_fence_after();
      const uint32_t tacc = uint32_t(acc * BN);
      for (int s = 0; s < P.nstages; ++s) {
        spin_wait(smem_u32(full + stage), phase);
        tc::tc_fence_after();
        const int npc = min(kStageK >> cb_log, P.npieces - s * (kStageK >> cb_log));
        const int nsteps = npc << kpp_log;
        const uint32_t sA = sa0 + stage * C::kAStage;
        // this stage's 128-byte weight chunk: chunk s of the resident block, or the stage's slot
        const uint32_t sB = P.b_res ? sb0 + uint32_t(s * C::kBBytes) : sb0 + uint32_t(stage * C::kBSlot);
        const uint32_t bstep = P.b_res ? uint32_t(P.nchk * C::kBBytes) : uint32_t(C::kBBytes);  // per weight digit
        if (elect_one()) {
          for (int u = 0; u < nsteps; ++u) {
            const uint32_t aoff = uint32_t(((u >> kpp_log) << (7 + cb_log)) + ((u & ((1 << kpp_log) - 1)) << 5));
#pragma unroll
            for (int d = 0; d < DA; ++d)
#pragma unroll
              for (int e = 0; e < DW; ++e)
                mma_f4_ss(tacc, sdesc(sA + d * C::kABytes + aoff, alay), sdesc(sB + e * bstep + 32 * u, blay),
                          idesc, uint32_t(C::kSF0 + 4 * d), uint32_t(C::kSF0 + 16 + 8 * e), (s | u | d | e) != 0);
          }
        }
        __syncwarp();
        if (args.mc)
          mma_commit_mc_elect(smem_u32(empty + stage), uint16_t(3));
        else
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
      // release the weights when the next tile reads other ones (tcgen05.commit: arrives once
      // every MMA issued so far has completed)
      const int nt = tile + int(gridDim.x);
      if (nt < args.ntiles) {
        int npi = pi;
        next_prob(nt, npi);
        uint32_t mb2, nb2;
        tile_mn(args.prob[npi], nt, mb2, nb2);
        if (bkey(args.prob[npi], npi, nb2) != key) tc::mma_commit_elect(smem_u32(b_empty));
      }
    }
  } else {
    // ================= epilogue: warp % 4 = TMEM lane quarter; the two warps of a quarter split
    // the 32-column blocks
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
#ifdef BS_TCD_NOSTORE  // experiment builds only: the epilogue drains TMEM but stores nothing
        if (r[0] == 0x9e3779b9u && r[31] == 0x7f4a7c15u) asm volatile("trap;");
        continue;
#endif
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
        } else if (P.epi == tc::kEpiDirect) {  // staged box re-read row-contiguously: 4 rows x 128 B per store
          uint8_t* b0 = ebuf + buf * kEpiBufBytes;
          const uint32_t swz = uint32_t(lane & 7);
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<uint4*>(b0 + lane * 128 + ((uint32_t(c) ^ swz) << 4)) =
                make_uint4(r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = i * 4 + (lane >> 3), ch = lane & 7;
            const uint4 v = *reinterpret_cast<const uint4*>(b0 + rr * 128 + ((uint32_t(ch) ^ uint32_t(rr & 7)) << 4));
            const int64_t grow = m0 + q * 32 + rr;
            const int col = n0 + cbk * 32 + ch * 4;
            if (grow < P.M && col < oc) *reinterpret_cast<uint4*>(P.out + grow * oc + col) = v;
          }
          __syncwarp();
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
  if (args.mc) cluster_sync();  // no CTA leaves while its peer may still signal it
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
  // knobs (tests / measurements): BS_TUNE_TCD_A_SRC 1 = TMA im2col, 2 = cp.async producers for conv
  // activations (default: producers; dense always TMA); BS_TUNE_TCD_B_STREAM 1 = never resident weights
  memset(&P, 0, sizeof(P));
  const int64_t cbytes = digit_row_bytes(p.c);  // bytes per pixel (row) and digit
  const int taps = p.kh * p.kw;
  P.out = p.out;
  P.M = int64_t(p.n) * p.oh * p.ow;
  P.oc = p.oc;
  P.epi = p.oc % 4 != 0 ? tc::kEpiScalar : (tuning(kTuneEpilogue) == 1 ? tc::kEpiDirect : tc::kEpiTma);
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
  P.act = p.act;
  P.h = p.h;
  P.w = p.w;
  P.cbytes = int(cbytes);
  P.plane_bytes = int64_t(p.n) * p.h * p.w * cbytes;
  P.a_tma = p.dense || tuning(kTuneTcdASrc) == 1;
  const int64_t wrow = tcd_wrow_bytes(int64_t(taps) * cbytes / 16);  // weight-digit row bytes (128-byte multiple)
  P.nchk = int(wrow / kStageK);
  const int64_t bres = int64_t(p.w_digits) * P.nchk * bn * kStageK;
  P.b_res = bres <= kBResMax && tuning(kTuneTcdBStream) != 1;
  P.bres_bytes = P.b_res ? int(bres) : 0;
  if (!tc::encode_2d(&tw, CU_TENSOR_MAP_DATA_TYPE_UINT8, p.wdig, uint64_t(wrow), uint64_t(p.w_digits) * p.oc,
                     uint64_t(wrow), kStageK, bn, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  if (p.dense) {
    P.arows = p.n;
    if (!tc::encode_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, p.act, uint64_t(cbytes), uint64_t(p.a_digits) * p.n,
                       uint64_t(cbytes), kStageK, BM, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  } else if (P.a_tma) {
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
    if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit)) return e;
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
  // shared memory: [B region][A ring][epilogue staging][barriers]; the B region holds the largest
  // resident weight block and, when a member streams its weights, one chunk slot per stage
  int res = 0;
  bool stream_b = false;
  for (int q = 0; q < count; ++q) {
    res = std::max(res, a.prob[q].bres_bytes);
    stream_b |= !a.prob[q].b_res;
  }
  a.gather = 1;
  for (int q = 0; q < count; ++q) a.gather &= !a.prob[q].a_tma;
  for (int q = 0; q < count; ++q)  // one source per launch (a group is all-conv under one knob)
    if (!a.gather && !a.prob[q].a_tma) return cudaErrorInvalidValue;
  int S = kMaxStages;
  while (S > 2 && std::max(res, stream_b ? S * C::kBSlot : 0) + S * C::kAStage > C::kBudget) --S;
  a.stages = S;
  a.b_region = std::max(res, stream_b ? S * C::kBSlot : 0);
  if (a.b_region + S * C::kAStage > C::kBudget) return cudaErrorInvalidValue;
  int smem = 1024 + a.b_region + S * C::kAStage + C::kEpiBytes + kBarBytes;
  if (smem < kMinSmem) smem = kMinSmem;
  // clusters of two on adjacent tiles of one N block multicast the weight chunks (dense, streamed
  // weights): each CTA loads half of every chunk's rows, so per CTA the operand bytes per stage drop
  // from A + B to A + B/2
  const TdProb& P0 = a.prob[0];
  // (measured, profiles/r02h_tcd_probe_mc.json: +3-4% at 16384^3 and A4W2, -4% at 8192^3 A2W1, where the
  // pairs' lock-step release of each stage costs more than the halved weight bytes save)
  const int mknob = tuning(kTuneTcdMcast);
  a.mc = count == 1 && P0.dense && !P0.b_res && P0.nmb % 2 == 0 && a.ntiles >= 4 && BN % 16 == 0 && mknob != 1 &&
         (mknob == 2 || P0.nmb >= 128 || DA * DW > 1);
  int grid = a.ntiles < device_sms() ? a.ntiles : device_sms();
  if (a.mc) {
    static std::atomic<int> max_clusters[64];  // co-resident 2-CTA clusters, per device (persistent grid)
    int mcl = dev < 64 ? max_clusters[dev].load(std::memory_order_relaxed) : 0;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = size_t(smem);
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (mcl == 0) {
      cfg.gridDim = dim3(unsigned(device_sms() / 2 * 2));
      if (cudaOccupancyMaxActiveClusters(&mcl, kern, &cfg) != cudaSuccess || mcl < 1) {
        cudaGetLastError();
        mcl = -1;
      }
      if (dev < 64) max_clusters[dev].store(mcl, std::memory_order_relaxed);
    }
    if (mcl > 0) {
      grid = std::min(grid, 2 * mcl) / 2 * 2;
      // the weight map's box: half of the tile's rows per CTA
      const TcdProblem& p = ps[0];
      const int64_t wrow = tcd_wrow_bytes(digit_row_bytes(p.c) / 16);
      if (!tc::encode_2d(&maps.w[0], CU_TENSOR_MAP_DATA_TYPE_UINT8, p.wdig, uint64_t(wrow),
                         uint64_t(p.w_digits) * p.oc, uint64_t(wrow), kStageK, BN / 2, CU_TENSOR_MAP_SWIZZLE_128B))
        return cudaErrorInvalidValue;
      cfg.gridDim = dim3(unsigned(grid));
      if (cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a, maps)) return e;
      note_launch();
      return cudaPeekAtLastError();
    }
    a.mc = 0;
  }
  kern<<<grid, kThreads, smem, stream>>>(a, maps);
  note_launch();
  return cudaPeekAtLastError();
}

template <int DA, int DW>
cudaError_t launch_dd(const TcdProblem* ps, int count, cudaStream_t stream) {
  bool wide = false;
  for (int q = 0; q < count; ++q) wide |= ps[q].oc > 64;
  // large dense products: 128 x 224 tiles (two 224-column accumulators + scale factors fill the
  // 512 TMEM columns) load 1.3x fewer operand rows per MMA than 128 x 128
  bool x224 = count == 1 && ps[0].dense && ps[0].oc >= 1024;
  if (const int v = tuning(kTuneTileN)) {
    wide = v > 64;
    x224 = count == 1 && v == 224;
  }
  if constexpr (Cfg<DA, DW, 224>::kFits) {
    if (x224) return launch<DA, DW, 224, 1>(ps, 1, stream);
  }
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
