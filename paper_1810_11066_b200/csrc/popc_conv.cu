// popc_conv.cu — tiled AND+POPC implicit-GEMM kernel for bitserial conv2d (NHWC)
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
//  * 3-stage cp.async ring (LDGSTS) so global latency hides behind the popcounts.
//  * Inner loop: LDS.64 of two k-words per operand row, then per word pair one LOP3
//    (AND), one POPC and one IADD/IMAD (a4/a5).  POPC issues at 16/clk/SM on B200
//    (profiles/r01_int_pipe_rates.json) vs 64/clk/SM for LOP3/IADD3/IMAD, so the
//    loop is POPC-bound by design and the roofline is R_popc.
//  * Plane weighting 2^(i+j) is applied per popcount pair as a shift-add (IMAD/LEA on
//    the FMA/ALU pipes, which have 4x the POPC rate), accumulators int32 (a5).
//  * Epilogue: bipolar correction with the per-row activation sums the CTA computed
//    from its own staged A tiles, int32 stores (a6).
#include <cstdio>

#include "common.cuh"
#include "kernels.h"

namespace bs {

namespace {

constexpr int kThreads = 256;
constexpr int kThrN = 16;     // thread grid is kThrM x kThrN = 16 x 16
constexpr int kThrM = 16;
constexpr int kBKMax = 8;     // k-words per stage (runtime BK in {2,4,6,8})
constexpr int kStride = 10;   // smem words per staged row: BK max + 2 (LDS.64 conflict-free)
constexpr int kStages = 3;

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

// A_T / W_T > 0: compile-time bit widths (fully unrolled plane loops, PAPER.md:644-645
// "apply [unroll] to small dimensions such as the bit axis");  0: runtime widths.
template <int A_T, int W_T, int BM, int BN, bool LIT>
__global__ void __launch_bounds__(kThreads) popc_conv_kernel(const ConvProblem p, const int BK) {
  constexpr int TM = BM / kThrM, TN = BN / kThrN;
  constexpr int TPR_A = kThreads / BM;   // threads per A row in the loader / row-sum
  constexpr int TPR_W = kThreads / BN;
  static_assert(kThreads % BM == 0 && kThreads % BN == 0, "tile rows must divide the CTA");
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
  const uint32_t smem_base = smem_u32(smem);

  auto load_stage = [&](int stage, int64_t k0) {
    const uint32_t sA = smem_base + uint32_t(stage * stage_words) * 4u;
    const uint32_t sW = sA + uint32_t(a_words) * 4u;
    for (int kq = la_part; kq < KQ; kq += TPR_A) {
      const int64_t kk = k0 + 2 * kq;
      const int tap = int(kk / p.kw_a);
      const int cw = int(kk - int64_t(tap) * p.kw_a);
      const int ky = tap / p.kwid, kx = tap - ky * p.kwid;
      const int iy = iy0 + ky, ix = ix0 + kx;
      const bool ok = a_row_ok && kk < p.kp && iy >= 0 && iy < p.h && ix >= 0 && ix < p.w;
      const uint32_t* src = ok ? p.act + (img_base + int64_t(iy) * p.w + ix) * p.kw_a + cw : p.act;
#pragma unroll
      for (int pl = 0; pl < (A_T > 0 ? A_T : 8); ++pl) {
        if (A_T == 0 && pl >= a_bits) break;
        cp_async8(sA + uint32_t((pl * BM + la_row) * kStride + 2 * kq) * 4u, ok ? src + pl * p.act_plane : src, ok);
      }
    }
    for (int kq = lw_part; kq < KQ; kq += TPR_W) {
      const int64_t kk = k0 + 2 * kq;
      const bool ok = w_row_ok && kk < p.kp;
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

  const int64_t ktiles = (p.kp + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < ktiles) load_stage(s, int64_t(s) * BK);
    cp_async_commit();
  }

  for (int64_t kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    {
      const int64_t nk = kt + kStages - 1;
      if (nk < ktiles) load_stage(int(nk % kStages), nk * BK);
      cp_async_commit();
    }
    const int stage = int(kt % kStages);
    const uint32_t sA = smem_base + uint32_t(stage * stage_words) * 4u;
    const uint32_t sW = sA + uint32_t(a_words) * 4u;

    if (need_rowsum) {
      for (int kq = la_part; kq < KQ; kq += TPR_A) {
#pragma unroll
        for (int pl = 0; pl < (A_T > 0 ? A_T : 8); ++pl) {
          if (A_T == 0 && pl >= a_bits) break;
          const uint2 v = lds64(sA + uint32_t((pl * BM + la_row) * kStride + 2 * kq) * 4u);
          rowsum += (__popc(v.x) + __popc(v.y)) << pl;
        }
      }
    }

    for (int kq = 0; kq < KQ; ++kq) {
      if constexpr (A_T > 0 && W_T > 0) {
        uint2 wv[W_T][TN];
#pragma unroll
        for (int q = 0; q < W_T; ++q)
#pragma unroll
          for (int j = 0; j < TN; ++j)
            wv[q][j] = lds64(sW + uint32_t((q * BN + tn + j * kThrN) * kStride + 2 * kq) * 4u);
#pragma unroll
        for (int pl = 0; pl < A_T; ++pl) {
          uint2 av[TM];
#pragma unroll
          for (int i = 0; i < TM; ++i)
            av[i] = lds64(sA + uint32_t((pl * BM + tm + i * kThrM) * kStride + 2 * kq) * 4u);
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
          for (int j = 0; j < TN; ++j)
            wv[j] = lds64(sW + uint32_t((q * BN + tn + j * kThrN) * kStride + 2 * kq) * 4u);
          for (int pl = 0; pl < a_bits; ++pl) {
#pragma unroll
            for (int i = 0; i < TM; ++i) {
              const uint2 av = lds64(sA + uint32_t((pl * BM + tm + i * kThrM) * kStride + 2 * kq) * 4u);
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
      if (n < p.oc) orow[n] = need_rowsum ? 2 * acc[i][j] - corr : acc[i][j];
    }
  }
}

template <int A_T, int W_T, int BM, int BN, bool LIT>
cudaError_t launch_cfg(const ConvProblem& p, int BK, cudaStream_t stream) {
  const size_t smem = SmemLayout<BM, BN>::bytes(p.a_bits, p.w_bits);
  auto kern = popc_conv_kernel<A_T, W_T, BM, BN, LIT>;
  static int configured_bytes = 0;  // per instantiation; attribute only grows
  if (int(smem) > configured_bytes) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    configured_bytes = int(smem);
  }
  dim3 grid(unsigned((p.M + BM - 1) / BM), unsigned((p.oc + BN - 1) / BN));
  kern<<<grid, kThreads, smem, stream>>>(p, BK);
  note_launch();
  return cudaPeekAtLastError();
}

// Choose BK in {8,6,4,2} minimising padded K work, ties to the larger BK.
int choose_bk(int64_t kp) {
  int best = 8;
  int64_t best_work = ((kp + 7) / 8) * 8;
  for (int bk : {6, 4, 2}) {
    const int64_t work = ((kp + bk - 1) / bk) * bk;
    if (work < best_work) { best = bk; best_work = work; }
  }
  return best;
}

template <int A_T, int W_T, bool LIT>
cudaError_t launch_tile(const ConvProblem& p, cudaStream_t stream) {
  const int bk = choose_bk(p.kp);
  // Tile choice: biggest tile that still gives >= 2 CTAs per SM (148 SMs), else smaller.
  auto ctas = [&](int bm, int bn) { return ((p.M + bm - 1) / bm) * ((p.oc + bn - 1) / bn); };
  if constexpr (A_T == 0 || W_T == 0) {
    return launch_cfg<A_T, W_T, 64, 64, LIT>(p, bk, stream);
  } else {
    if (p.oc >= 128 && ctas(128, 128) >= 2 * kNumSMs) return launch_cfg<A_T, W_T, 128, 128, LIT>(p, bk, stream);
    if (ctas(128, 64) >= 2 * kNumSMs) return launch_cfg<A_T, W_T, 128, 64, LIT>(p, bk, stream);
    return launch_cfg<A_T, W_T, 64, 64, LIT>(p, bk, stream);
  }
}

// Compile-time widths for the limit-study grid A, W in 1..4;
// the literal bipolar variant only for the BASELINE widths; everything else runs the
// runtime-width instantiation.
cudaError_t dispatch_uni(const ConvProblem& p, cudaStream_t stream) {
#define BS_CASE(A, W) \
  if (p.a_bits == A && p.w_bits == W) return launch_tile<A, W, false>(p, stream);
  BS_CASE(1, 1) BS_CASE(2, 1) BS_CASE(2, 2) BS_CASE(1, 2) BS_CASE(4, 1) BS_CASE(4, 2)
  BS_CASE(3, 1) BS_CASE(1, 3) BS_CASE(1, 4) BS_CASE(2, 3) BS_CASE(3, 2) BS_CASE(2, 4)
  BS_CASE(3, 3) BS_CASE(3, 4) BS_CASE(4, 3) BS_CASE(4, 4)
#undef BS_CASE
  return launch_tile<0, 0, false>(p, stream);
}

cudaError_t dispatch_lit(const ConvProblem& p, cudaStream_t stream) {
  if (p.a_bits == 1 && p.w_bits == 1) return launch_tile<1, 1, true>(p, stream);
  if (p.a_bits == 2 && p.w_bits == 1) return launch_tile<2, 1, true>(p, stream);
  if (p.a_bits == 2 && p.w_bits == 2) return launch_tile<2, 2, true>(p, stream);
  return launch_tile<0, 0, true>(p, stream);
}

}  // namespace

cudaError_t launch_popc_conv(const ConvProblem& p, Algo algo, cudaStream_t stream) {
  if (algo == Algo::PopcLit && p.bipolar) return dispatch_lit(p, stream);
  return dispatch_uni(p, stream);
}

}  // namespace bs
