#pragma once
// popc_conv_impl.cuh — tiled AND+POPC implicit-GEMM kernel for bitserial conv2d (NHWC)
// and dense.
//
// Per output (Eq. 2):
//     out[m][n] = sum_{i<A} sum_{j<W} 2^(i+j) * sum_kw popc(a_i[m][kw] & w_j[n][kw])
// with the bipolar weight form either literal (north_star: popc(a&w) - popc(a&~w)
// per plane pair, LIT=true) or through the exact identity
//     bipolar = 2 * unipolar - (2^W - 1) * sum_k a[m][k]
// (sum over the receptive field, padding contributes 0; DESIGN.md §3 reading R2).
//
// Design (B200):
//  * CTA tile BM x BN outputs, 256 threads in a 16 x 16 grid, each thread TM x TN
//    outputs held in registers (register blocking, PAPER.md:635-640 tiling).
//  * The K loop runs over packed words; K is (tap, channel-word) for conv, so the
//    A tile of a stage is gathered straight from the NHWC packed activations with
//    8-byte cp.async (implicit im2col: no lowered copy), out-of-image
//    taps zero-filled by the copy engine (src-size 0) = zero padding (a3).
//  * 3-stage cp.async ring (LDGSTS) so global latency hides behind the compute.
//  * Inner loop (a4/a5), two variants:
//      G == 0 : per word pair one LOP3 (AND) + one POPC + shift-add — POPC-bound,
//               since POPC issues at 16/clk/SM vs 64/clk/SM for LOP3/IMAD
//               (profiles/r01_int_pipe_rates.json);
//      G >= 1 : groups of 2G k-words; per output the A*W*2G AND words go through a
//               carry-save tree (csa.cuh) that trades POPCs for LOP3s and
//               accumulates on the FMA pipe, balancing the three integer pipes.
//  * Epilogue: bipolar correction with the per-row activation sums the CTA computed
//    from its own staged A tiles, int32 stores (a6).
#include "common.cuh"
#include "csa.cuh"
#include "kernels.h"

namespace bs {
namespace popc_detail {

constexpr int kThreads = 256;
constexpr int kThrN = 16;     // thread grid is kThrM x kThrN = 16 x 16
constexpr int kThrM = 16;
#ifndef BS_KSTRIDE
#define BS_KSTRIDE 14
#endif
constexpr int kStride = BS_KSTRIDE;  // smem words per staged row (>= BK max, 8-byte rows): 14r mod 32
                                     // gives 16 distinct even banks for 16 rows -> LDS.64 conflict-free
constexpr int kBKMax = kStride >= 16 ? 16 : 12;  // k-words per stage (runtime BK <= kBKMax)
constexpr int kStages = 3;
#ifndef BS_MINB2
#define BS_MINB2 2
#endif

template <int BM, int BN>
struct SmemLayout {
  // per stage: A planes x BM rows x kStride words, then W planes x BN rows x kStride
  __host__ __device__ static int stage_words(int a_bits, int w_bits) {
    return (a_bits * BM + w_bits * BN) * kStride;
  }
  __host__ static size_t bytes(int a_bits, int w_bits) {
    return size_t(kStages) * stage_words(a_bits, w_bits) * 4;
  }
};

// Registers a thread holds in the carry-save loop: the W words of its TN columns for
// one group, the A words of one row, the AND/full-adder slots of one output and the
// TM x TN accumulators.
constexpr int csa_regs(int A, int W, int G, int TM, int TN) {
  return TN * W * 2 * G + A * 2 * G + TM * TN + A * W * 2 * G;
}

// Plans whose register estimate stays <= 112 fit in 128 registers: pin 2 CTAs (16 warps)
// per SM so ptxas does not trade that occupancy away; larger plans run one CTA per SM.
constexpr int min_ctas(int A, int W, int G, int TM, int TN) {
  return (G == 0 || csa_regs(A, W, G, TM, TN) <= 112) ? BS_MINB2 : 1;
}

// One group of 2*GG k-words starting at word kw of the stage: for every output of the
// thread, acc += carry-save dot of its A row and W column over those words.
template <int A, int W, int GG, int TM, int TN, int BM, int BN>
__device__ __forceinline__ void csa_group(int32_t (&acc)[TM][TN], const uint32_t* pA, const uint32_t* pW, int kw,
                                          int tm, int tn, const int (&wgt)[A + W + 6]) {
  uint32_t wv[TN][W][2 * GG];
#pragma unroll
  for (int j = 0; j < TN; ++j)
#pragma unroll
    for (int q = 0; q < W; ++q)
#pragma unroll
      for (int g = 0; g < GG; ++g) {
        const uint2 x = lds64p(pW + (q * BN + tn + j * kThrN) * kStride + kw + 2 * g);
        wv[j][q][2 * g] = x.x;
        wv[j][q][2 * g + 1] = x.y;
      }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    uint32_t av[A][2 * GG];
#pragma unroll
    for (int pl = 0; pl < A; ++pl)
#pragma unroll
      for (int g = 0; g < GG; ++g) {
        const uint2 x = lds64p(pA + (pl * BM + tm + i * kThrM) * kStride + kw + 2 * g);
        av[pl][2 * g] = x.x;
        av[pl][2 * g + 1] = x.y;
      }
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = csa_dot<A, W, GG>(acc[i][j], av, wv[j], wgt);
  }
}

// A_T / W_T > 0: compile-time bit widths (fully unrolled plane loops, PAPER.md:644-645
// "apply [unroll] to small dimensions such as the bit axis");  0: runtime widths.
// G: carry-save group size in k-word pairs (0 = direct AND+POPC loop).
template <int A_T, int W_T, int BM, int BN, bool LIT, int G>
__global__ void __launch_bounds__(kThreads, min_ctas(A_T > 0 ? A_T : 1, W_T > 0 ? W_T : 1, G, BM / kThrM, BN / kThrN)) popc_conv_kernel(const ConvProblem p, const int BK) {
  constexpr int TM = BM / kThrM, TN = BN / kThrN;
  constexpr int TPR_A = kThreads / BM;   // threads per A row in the loader / row-sum
  constexpr int TPR_W = kThreads / BN;
  static_assert(kThreads % BM == 0 && kThreads % BN == 0, "tile rows must divide the CTA");
  static_assert(G == 0 || (A_T > 0 && W_T > 0 && !LIT), "carry-save path needs compile-time widths");
  extern __shared__ __align__(16) uint32_t smem[];

  const int a_bits = A_T > 0 ? A_T : p.a_bits;
  const int w_bits = W_T > 0 ? W_T : p.w_bits;
  const int KQ = BK >> 1;  // 8-byte chunks per row per stage
  const int tid = threadIdx.x;
  const int tn = tid % kThrN, tm = tid / kThrN;
  const int64_t m0 = int64_t(blockIdx.x) * BM;
  const int n0 = blockIdx.y * BN;
  const int stage_words = SmemLayout<BM, BN>::stage_words(a_bits, w_bits);
  const int a_words = a_bits * BM * kStride;

  // ---- loader state: this thread stages A row `la_row` and W row `lw_row`
  const int la_row = tid % BM, la_part = tid / BM;
  const int lw_row = tid % BN, lw_part = tid / BN;
  const int64_t m_load = m0 + la_row;
  const bool a_row_ok = m_load < p.M;
  int iy0 = 0, ix0 = 0;
  int64_t img_base = 0;
  {
    const int64_t mm = a_row_ok ? m_load : 0;
    const int64_t hw_out = int64_t(p.oh) * p.ow;
    const int64_t b = mm / hw_out, rem = mm - b * hw_out;
    const int oy = int(rem / p.ow), ox = int(rem - int64_t(oy) * p.ow);
    iy0 = oy * p.sh - p.ph;
    ix0 = ox * p.sw - p.pw;
    img_base = b * int64_t(p.h) * p.w;
  }
  const bool w_row_ok = (n0 + lw_row) < p.oc;
  const uint32_t* w_row_ptr = p.wt + int64_t(w_row_ok ? n0 + lw_row : 0) * p.kp;
  const int64_t w_plane = int64_t(p.oc) * p.kp;
  const int kp = int(p.kp);
  const uint32_t smem_base = smem_u32(smem);

  auto load_stage = [&](int stage, int k0) {
    const uint32_t sA = smem_base + uint32_t(stage * stage_words) * 4u;
    const uint32_t sW = sA + uint32_t(a_words) * 4u;
    for (int kq = la_part; kq < KQ; kq += TPR_A) {
      const int kk = k0 + 2 * kq;
      const int tap = kk / p.kw_a;
      const int cw = kk - tap * p.kw_a;
      const int ky = tap / p.kwid, kx = tap - ky * p.kwid;
      const int iy = iy0 + ky, ix = ix0 + kx;
      const bool ok = a_row_ok && kk < kp && iy >= 0 && iy < p.h && ix >= 0 && ix < p.w;
      const uint32_t* src = ok ? p.act + (img_base + int64_t(iy) * p.w + ix) * p.kw_a + cw : p.act;
#pragma unroll
      for (int pl = 0; pl < (A_T > 0 ? A_T : 8); ++pl) {
        if (A_T == 0 && pl >= a_bits) break;
        cp_async8(sA + uint32_t((pl * BM + la_row) * kStride + 2 * kq) * 4u, ok ? src + pl * p.act_plane : src, ok);
      }
    }
    for (int kq = lw_part; kq < KQ; kq += TPR_W) {
      const int kk = k0 + 2 * kq;
      const bool ok = w_row_ok && kk < kp;
      const uint32_t* src = ok ? w_row_ptr + kk : p.wt;
#pragma unroll
      for (int pl = 0; pl < (W_T > 0 ? W_T : 8); ++pl) {
        if (W_T == 0 && pl >= w_bits) break;
        cp_async8(sW + uint32_t((pl * BN + lw_row) * kStride + 2 * kq) * 4u, ok ? src + pl * w_plane : src, ok);
      }
    }
  };

  int32_t acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0;
  int32_t rowsum = 0;  // partial sum_k a[la_row][k] (identity-form bipolar only)
  const bool need_rowsum = p.bipolar && !LIT;

  // plane weights 2^l in registers the compiler cannot fold (kernel argument), so the
  // carry-save accumulations stay IMADs on the FMA pipe (csa.cuh)
  int wgt[(A_T > 0 ? A_T : 1) + (W_T > 0 ? W_T : 1) + 6];
#pragma unroll
  for (int l = 0; l < int(sizeof(wgt) / sizeof(int)); ++l) wgt[l] = p.one << l;

  // split-K (small M*N, e.g. batch-1 layers): blockIdx.z owns k-tiles [kt0, kt0 + ktiles)
  const int ktiles_all = (kp + BK - 1) / BK;
  const int kt0 = int(int64_t(ktiles_all) * blockIdx.z / p.ksplit);
  const int ktiles = int(int64_t(ktiles_all) * (blockIdx.z + 1) / p.ksplit) - kt0;
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < ktiles) load_stage(s, (kt0 + s) * BK);
    cp_async_commit();
  }

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    {
      const int nk = kt + kStages - 1;
      if (nk < ktiles) load_stage(nk % kStages, (kt0 + nk) * BK);
      cp_async_commit();
    }
    const int stage = kt % kStages;
    const uint32_t* pA = smem + stage * stage_words;
    const uint32_t* pW = pA + a_words;

    if (need_rowsum) {
      for (int kq = la_part; kq < KQ; kq += TPR_A) {
#pragma unroll
        for (int pl = 0; pl < (A_T > 0 ? A_T : 8); ++pl) {
          if (A_T == 0 && pl >= a_bits) break;
          const uint2 v = lds64p(pA + (pl * BM + la_row) * kStride + 2 * kq);
          rowsum += (__popc(v.x) + __popc(v.y)) << pl;
        }
      }
    }

    if constexpr (G > 0) {
      constexpr int AA = A_T > 0 ? A_T : 1, WW = W_T > 0 ? W_T : 1;
      int kw = 0;
      for (; kw + 2 * G <= BK; kw += 2 * G)
        csa_group<AA, WW, G, TM, TN, BM, BN>(acc, pA, pW, kw, tm, tn, wgt);
      for (; kw < BK; kw += 2)  // trailing pairs when BK is not a multiple of 2G
        csa_group<AA, WW, 1, TM, TN, BM, BN>(acc, pA, pW, kw, tm, tn, wgt);
    } else {
      for (int kq = 0; kq < KQ; ++kq) {
        if constexpr (A_T > 0 && W_T > 0) {
          uint2 wv[W_T][TN];
#pragma unroll
          for (int q = 0; q < W_T; ++q)
#pragma unroll
            for (int j = 0; j < TN; ++j) wv[q][j] = lds64p(pW + (q * BN + tn + j * kThrN) * kStride + 2 * kq);
#pragma unroll
          for (int pl = 0; pl < A_T; ++pl) {
            uint2 av[TM];
#pragma unroll
            for (int i = 0; i < TM; ++i) av[i] = lds64p(pA + (pl * BM + tm + i * kThrM) * kStride + 2 * kq);
#pragma unroll
            for (int q = 0; q < W_T; ++q)
#pragma unroll
              for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) {
                  int d = __popc(av[i].x & wv[q][j].x) + __popc(av[i].y & wv[q][j].y);
                  if (LIT) d -= __popc(av[i].x & ~wv[q][j].x) + __popc(av[i].y & ~wv[q][j].y);
                  acc[i][j] += d << (pl + q);
                }
          }
        } else {  // runtime bit widths: planes looped, operands reloaded per plane pair
          for (int q = 0; q < w_bits; ++q) {
            uint2 wv[TN];
#pragma unroll
            for (int j = 0; j < TN; ++j) wv[j] = lds64p(pW + (q * BN + tn + j * kThrN) * kStride + 2 * kq);
            for (int pl = 0; pl < a_bits; ++pl) {
#pragma unroll
              for (int i = 0; i < TM; ++i) {
                const uint2 av = lds64p(pA + (pl * BM + tm + i * kThrM) * kStride + 2 * kq);
#pragma unroll
                for (int j = 0; j < TN; ++j) {
                  int d = __popc(av.x & wv[j].x) + __popc(av.y & wv[j].y);
                  if (LIT) d -= __popc(av.x & ~wv[j].x) + __popc(av.y & ~wv[j].y);
                  acc[i][j] += d << (pl + q);
                }
              }
            }
          }
        }
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // ---- epilogue (a5/a6): bipolar identity correction, int32 store
  int* s_rowsum = reinterpret_cast<int*>(smem);  // [TPR_A][BM], reuses the ring
  if (need_rowsum) {
    s_rowsum[la_part * BM + la_row] = rowsum;
    __syncthreads();
  }
  const int wmax = (1 << w_bits) - 1;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int ml = tm + i * kThrM;
    const int64_t m = m0 + ml;
    if (m >= p.M) continue;
    int corr = 0;
    if (need_rowsum) {
      int s = 0;
#pragma unroll
      for (int t = 0; t < TPR_A; ++t) s += s_rowsum[t * BM + ml];
      corr = wmax * s;
    }
    int32_t* orow = p.out + m * p.oc;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + tn + j * kThrN;
      if (n < p.oc) {
        const int32_t v = need_rowsum ? 2 * acc[i][j] - corr : acc[i][j];
        if (p.ksplit > 1)
          atomicAdd(orow + n, v);  // partial over this K slice; int32 addition is exact in any order
        else
          orow[n] = v;
      }
    }
  }
}

template <int A_T, int W_T, int BM, int BN, bool LIT, int G>
cudaError_t launch_cfg(const ConvProblem& p, int BK, cudaStream_t stream) {
  const size_t smem = SmemLayout<BM, BN>::bytes(p.a_bits, p.w_bits);
  auto kern = popc_conv_kernel<A_T, W_T, BM, BN, LIT, G>;
  // the dynamic shared-memory opt-in is per device and per size: set it on every launch
  // (a host-side attribute write; this is not the hot path)
  if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem))) return e;
  // Split K across CTAs when the M x N tiles cannot fill the 148 SMs twice (batch-1
  // layers): keep >= 2 k-tiles per slice; partials are summed with int32 atomics into
  // a zeroed output (exact: integer addition is associative).
  const int64_t tiles = ((p.M + BM - 1) / BM) * ((p.oc + BN - 1) / BN);
  const int ktiles = int((p.kp + BK - 1) / BK);
  int ksplit = 1;
  if (tiles < 2 * kNumSMs) {
    ksplit = int((2 * kNumSMs + tiles - 1) / tiles);
    if (ksplit > ktiles / 2) ksplit = ktiles / 2;
    if (ksplit < 1) ksplit = 1;
  }
  ConvProblem q = p;
  q.ksplit = ksplit;
  if (ksplit > 1) {
    cudaError_t e = cudaMemsetAsync(p.out, 0, size_t(p.M) * p.oc * sizeof(int32_t), stream);
    if (e != cudaSuccess) return e;
  }
  dim3 grid(unsigned((p.M + BM - 1) / BM), unsigned((p.oc + BN - 1) / BN), unsigned(ksplit));
  kern<<<grid, kThreads, smem, stream>>>(q, BK);
  note_launch();
  return cudaPeekAtLastError();
}

// Choose BK in {12,8,6,4,2}: minimise stages x (per-stage compute + 1 unit of barrier /
// loader overhead); a stage of BK words costs floor(BK/2G) groups of cost_g plus
// the remaining word pairs at cost_1 each (costs in cycles per group, cost model above).
inline int choose_bk(int kp, int g, double cost_g, double cost_1, double overhead) {
  int best = 8;
  double best_cost = -1.0;
  for (int bk : {16, 12, 8, 6, 4, 2}) {
    if (bk > kBKMax) continue;
    const int stages = (kp + bk - 1) / bk;
    const int groups = g > 0 ? bk / (2 * g) : 0;
    const int pairs = g > 0 ? (bk - groups * 2 * g) / 2 : bk / 2;
    const double cost = stages * (groups * cost_g + pairs * cost_1 + overhead);
    if (best_cost < 0 || cost < best_cost - 1e-9) { best = bk; best_cost = cost; }
  }
  return best;
}

// Group cost in SMSP cycles (cost model of csa.cuh).  Measured on B200 (tools/
// layer_sweep.py, profiles/r01_csa_group_sweep.jsonl): plans whose register estimate
// exceeds ~112 end up above 128 registers (one CTA of 8 warps per SM) and run ~25%
// above their model, so they are charged that much.
template <int A, int W, int G, int TM, int TN>
constexpr double group_cost() {
  return csa_cycles_per_word_pair<A, W, G>() * (A * W * 2 * G) * (csa_regs(A, W, G, TM, TN) > 112 ? 1.25 : 1.0);
}

template <int A_T, int W_T, int BM, int BN, int G>
cudaError_t launch_csa_g(const ConvProblem& p, cudaStream_t stream, int bk) {
  return launch_cfg<A_T, W_T, BM, BN, false, G>(p, bk, stream);
}

// Pick the carry-save group size (2 or 3 k-word pairs, whichever fits the register
// budget) and the stage depth BK that minimise the modelled cost for this K; the
// per-stage overhead (barrier + loader) is charged as 4*A*W cycles.
template <int A_T, int W_T, int BM, int BN>
cudaError_t launch_csa(const ConvProblem& p, cudaStream_t stream) {
  constexpr int TM = BM / kThrM, TN = BN / kThrN;
  constexpr bool g4_ok = csa_regs(A_T, W_T, 4, TM, TN) <= 150;
  constexpr bool g3_ok = csa_regs(A_T, W_T, 3, TM, TN) <= 150;
  constexpr bool g2_ok = csa_regs(A_T, W_T, 2, TM, TN) <= 150;
  const int kp = int(p.kp);
  const double ovh = 4.0 * A_T * W_T, c1 = group_cost<A_T, W_T, 1, TM, TN>();
  auto plan_cost = [&](int g, double cg, int* bk_out) {
    const int bk = choose_bk(kp, g, cg, c1, ovh);
    const int stages = (kp + bk - 1) / bk, groups = bk / (2 * g), pairs = (bk - groups * 2 * g) / 2;
    *bk_out = bk;
    return stages * (groups * cg + pairs * c1 + ovh);
  };
#ifdef BS_FORCE_G
  constexpr int GF = BS_FORCE_G > 0 ? BS_FORCE_G : 1;
  int bkf = 0;
  plan_cost(GF, group_cost<A_T, W_T, GF, TM, TN>(), &bkf);
  return launch_cfg<A_T, W_T, BM, BN, false, BS_FORCE_G>(p, bkf, stream);
#else
  int bk1 = 0, bk2 = 0, bk3 = 0, bk4 = 0;
  const double cost1 = plan_cost(1, c1, &bk1);
  const double cost2 = g2_ok ? plan_cost(2, group_cost<A_T, W_T, 2, TM, TN>(), &bk2) : 1e30;
  const double cost3 = g3_ok ? plan_cost(3, group_cost<A_T, W_T, 3, TM, TN>(), &bk3) : 1e30;
  const double cost4 = g4_ok ? plan_cost(4, group_cost<A_T, W_T, 4, TM, TN>(), &bk4) : 1e30;
  if constexpr (g4_ok) {
    if (cost4 < cost3 && cost4 < cost2 && cost4 < cost1) return launch_cfg<A_T, W_T, BM, BN, false, 4>(p, bk4, stream);
  }
  if constexpr (g3_ok) {
    if (cost3 < cost2 && cost3 < cost1) return launch_cfg<A_T, W_T, BM, BN, false, 3>(p, bk3, stream);
  }
  if constexpr (g2_ok) {
    if (cost2 <= cost1) return launch_cfg<A_T, W_T, BM, BN, false, 2>(p, bk2, stream);
  }
  return launch_cfg<A_T, W_T, BM, BN, false, 1>(p, bk1, stream);
#endif
}

template <int A_T, int W_T, bool LIT>
cudaError_t launch_tile(const ConvProblem& p, cudaStream_t stream) {
  // Tile choice: biggest tile that still gives >= 2 CTAs per SM (148 SMs), else smaller.
  auto ctas = [&](int bm, int bn) { return ((p.M + bm - 1) / bm) * ((p.oc + bn - 1) / bn); };
  if constexpr (A_T == 0 || W_T == 0 || LIT) {
    const int direct = (A_T > 0 ? A_T : p.a_bits) * (W_T > 0 ? W_T : p.w_bits) * (LIT ? 2 : 1);
    const int bk = choose_bk(int(p.kp), 0, 0.0, 8.0 * direct, 4.0 * direct);
    if constexpr (A_T > 0 && W_T > 0) {
      if (p.oc >= 128 && ctas(128, 128) >= 2 * kNumSMs) return launch_cfg<A_T, W_T, 128, 128, LIT, 0>(p, bk, stream);
      if (ctas(128, 64) >= 2 * kNumSMs) return launch_cfg<A_T, W_T, 128, 64, LIT, 0>(p, bk, stream);
    }
    return launch_cfg<A_T, W_T, 64, 64, LIT, 0>(p, bk, stream);
  } else {
    if (p.oc >= 128 && ctas(128, 128) >= 2 * kNumSMs) return launch_csa<A_T, W_T, 128, 128>(p, stream);
    if (ctas(128, 64) >= 2 * kNumSMs) return launch_csa<A_T, W_T, 128, 64>(p, stream);
    return launch_csa<A_T, W_T, 64, 64>(p, stream);
  }
}

}  // namespace popc_detail
}  // namespace bs
