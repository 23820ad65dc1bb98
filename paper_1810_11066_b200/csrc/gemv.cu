// gemv.cu — bitserial matrix-vector kernel (m <= 8 rows of activations), BASELINE
// config 2 (K = N = 4096, A2W1 bipolar, batch 1).
//
// The B200 analogue of the paper's tensorized ARM micro-kernel (PAPER.md:694-705,
// Sec. 5.2): "4 bitserial dot products ... accumulation and write back steps in a
// tree reduction fashion allowing for vectorized loads and stores on all tensors".
//  * The (tiny) activation operand is staged once per CTA in shared memory —
//    either copied pre-packed, or packed in-kernel from uint8 codes (FUSED: the
//    whole batch-1 dense op is one launch, the timed activation packing of
//    PAPER.md:715 included).
//  * Each warp owns R = 8 weight rows; every lane streams 16-byte (or 8-byte)
//    chunks of all R rows, so R independent LDG.128 per lane are in flight.
//  * The R x m per-lane partial sums are reduced with a transposed butterfly
//    (log2(32) levels, halving the values exchanged at each level: 4+2+1+1+1
//    shuffles for R = 8 instead of 8 x 5), after which lane 4r holds row r — the
//    "tree reduction" of PAPER.md:698/705 — and the 8 results go out as one segment.
//  * HBM-bound at large N*K (weights are read once: W*N*K/8 bytes), latency-bound
//    at config 2's 2 MiB.
#include <atomic>
#include "common.cuh"
#include "kernels.h"

namespace bs {

namespace {

constexpr int kGemvThreads = 64;   // 2 warps per CTA: 16 weight rows, 256 CTAs for n = 4096 (> 148 SMs)
constexpr int kR = 8;              // weight rows per warp
constexpr int kMaxM = 8;
constexpr size_t kMaxSmem = 96 * 1024;

template <int A, int W, int VEC, bool FUSED>
__global__ void __launch_bounds__(kGemvThreads) gemv_kernel(const uint32_t* __restrict__ a_packed,
                                                             const uint8_t* __restrict__ a_codes,
                                                             const uint32_t* __restrict__ w_packed,
                                                             int32_t* __restrict__ out, int m, int64_t n,
                                                             int64_t k, int kwp, int bipolar) {
  extern __shared__ __align__(16) uint32_t s_act[];  // [A][m][kwp], then per-warp row sums [warps][m]
  int* s_part = reinterpret_cast<int*>(s_act + A * m * kwp);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n0 = (int64_t(blockIdx.x) * (kGemvThreads / 32) + warp) * kR;
  const int64_t w_plane = n * kwp;
  const int nchunks = kwp / VEC;
  auto load_w = [&](int c, uint32_t (&wv)[W][kR][VEC]) {
#pragma unroll
    for (int q = 0; q < W; ++q)
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        const int64_t row = n0 + r < n ? n0 + r : n - 1;
        const uint32_t* src = w_packed + q * w_plane + row * kwp + c * VEC;
        if constexpr (VEC == 4) {
          const uint4 x = __ldg(reinterpret_cast<const uint4*>(src));
          wv[q][r][0] = x.x; wv[q][r][1] = x.y; wv[q][r][2] = x.z; wv[q][r][3] = x.w;
        } else {
          const uint2 x = __ldg(reinterpret_cast<const uint2*>(src));
          wv[q][r][0] = x.x; wv[q][r][1] = x.y;
        }
      }
  };
  // Weight loads of the first chunk are issued before the activation is staged, so
  // the HBM latency of the (dominant) weight stream overlaps the staging.
  uint32_t wv0[W][kR][VEC];
  const bool prefetched = n0 < n && lane < nchunks;
  if (prefetched) load_w(lane, wv0);

  // ---- stage the activation operand (packed) in shared memory; bipolar: the row sums
  // sum_k a[r][k] = sum_b 2^b popc(plane b) are gathered on the way (per warp, no second
  // pass and no second barrier)
  int rs[kMaxM];
#pragma unroll
  for (int r = 0; r < kMaxM; ++r) rs[r] = 0;
  if (FUSED) {
    const bool al16 = (reinterpret_cast<uintptr_t>(a_codes) % 16 == 0) && (k % 16 == 0);
    // two words per thread per pass, both words' codes loaded before either is packed (the
    // loads are the latency of this phase)
    for (int t0 = tid; t0 < m * kwp; t0 += 2 * kGemvThreads) {
      uint32_t v[2][8];
      int rr_[2], jj[2];
      bool ok[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int t = t0 + u * kGemvThreads;
        ok[u] = t < m * kwp;
        const int r = ok[u] ? t / kwp : 0, j = ok[u] ? t - r * kwp : 0;
        rr_[u] = r;
        jj[u] = j;
        const int64_t e0 = 32 * int64_t(j);
        const uint8_t* src = a_codes + r * k + e0;
        if (!ok[u]) {
#pragma unroll
          for (int q = 0; q < 8; ++q) v[u][q] = 0;
        } else if (al16 && e0 + 32 <= k) {
          const uint4 lo = __ldg(reinterpret_cast<const uint4*>(src)), hi = __ldg(reinterpret_cast<const uint4*>(src) + 1);
          v[u][0] = lo.x; v[u][1] = lo.y; v[u][2] = lo.z; v[u][3] = lo.w;
          v[u][4] = hi.x; v[u][5] = hi.y; v[u][6] = hi.z; v[u][7] = hi.w;
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            uint32_t x = 0;
#pragma unroll
            for (int rr = 0; rr < 4; ++rr)
              if (e0 + 4 * q + rr < k) x |= uint32_t(__ldg(src + 4 * q + rr)) << (8 * rr);
            v[u][q] = x;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (!ok[u]) continue;
        int s = 0;
#pragma unroll
        for (int b = 0; b < A; ++b) {
          const uint32_t wd = plane_word(v[u], b);
          s_act[(b * m + rr_[u]) * kwp + jj[u]] = wd;
          s += __popc(wd) << b;
        }
#pragma unroll
        for (int rr = 0; rr < kMaxM; ++rr) rs[rr] += rr == rr_[u] ? s : 0;
      }
    }
  } else {
    for (int t = tid; t < A * m * kwp; t += kGemvThreads) {
      const uint32_t wd = __ldg(a_packed + t);
      s_act[t] = wd;
      const int b = t / (m * kwp), r = (t / kwp) % m;
#pragma unroll
      for (int rr = 0; rr < kMaxM; ++rr) rs[rr] += rr == r ? (__popc(wd) << b) : 0;
    }
  }
  if (bipolar) {
    for (int r = 0; r < m; ++r) {
      const int s = __reduce_add_sync(0xffffffffu, rs[r]);
      if (lane == 0) s_part[warp * kMaxM + r] = s;
    }
  }
  __syncthreads();
  int rowsum[kMaxM];
#pragma unroll
  for (int r = 0; r < kMaxM; ++r) {
    rowsum[r] = 0;
    if (bipolar && r < m)
#pragma unroll
      for (int w2 = 0; w2 < kGemvThreads / 32; ++w2) rowsum[r] += s_part[w2 * kMaxM + r];
  }

  if (n0 >= n) return;
  for (int mi = 0; mi < m; ++mi) {
    int part[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) part[r] = 0;
    for (int c = lane; c < nchunks; c += 32) {
      uint32_t wv[W][kR][VEC];
      if (mi == 0 && c == lane) {
#pragma unroll
        for (int q = 0; q < W; ++q)
#pragma unroll
          for (int r = 0; r < kR; ++r)
#pragma unroll
            for (int v = 0; v < VEC; ++v) wv[q][r][v] = wv0[q][r][v];
      } else {
        load_w(c, wv);
      }
#pragma unroll
      for (int b = 0; b < A; ++b) {
        uint32_t av[VEC];
        const uint32_t* ap = s_act + (b * m + mi) * kwp + c * VEC;
        if constexpr (VEC == 4) {
          const uint4 x = *reinterpret_cast<const uint4*>(ap);
          av[0] = x.x; av[1] = x.y; av[2] = x.z; av[3] = x.w;
        } else {
          const uint2 x = *reinterpret_cast<const uint2*>(ap);
          av[0] = x.x; av[1] = x.y;
        }
#pragma unroll
        for (int q = 0; q < W; ++q)
#pragma unroll
          for (int r = 0; r < kR; ++r) {
            int d = 0;
#pragma unroll
            for (int v = 0; v < VEC; ++v) d += __popc(av[v] & wv[q][r][v]);
            part[r] += d << (b + q);
          }
      }
    }
    // transposed butterfly: 8 values/lane -> lane (4*r') holds row r'
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool up = lane & 16;
      const int send = up ? part[i] : part[i + 4];
      const int keep = up ? part[i + 4] : part[i];
      part[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const bool up = lane & 8;
      const int send = up ? part[i] : part[i + 2];
      const int keep = up ? part[i + 2] : part[i];
      part[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    {
      const bool up = lane & 4;
      const int send = up ? part[0] : part[1];
      const int keep = up ? part[1] : part[0];
      part[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    part[0] += __shfl_xor_sync(0xffffffffu, part[0], 2);
    part[0] += __shfl_xor_sync(0xffffffffu, part[0], 1);
    if ((lane & 3) == 0) {
      const int r = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
      if (n0 + r < n) {
        const int u = part[0];
        int rsum = 0;
#pragma unroll
        for (int rr = 0; rr < kMaxM; ++rr) rsum = rr == mi ? rowsum[rr] : rsum;
        out[int64_t(mi) * n + n0 + r] = bipolar ? 2 * u - ((1 << W) - 1) * rsum : u;
      }
    }
  }
}

template <int A, int W>
cudaError_t launch_aw(const uint32_t* a_packed, const uint8_t* a_codes, const uint32_t* w_packed, int bipolar,
                      int32_t* out, int64_t m, int64_t n, int64_t k, int64_t kwp, cudaStream_t stream) {
  const size_t smem = size_t(A) * m * kwp * 4 + (kGemvThreads / 32) * kMaxM * 4;
  const int64_t warps = (n + kR - 1) / kR;
  const unsigned grid = unsigned((warps + kGemvThreads / 32 - 1) / (kGemvThreads / 32));
  const bool vec4 = (kwp % 4 == 0) && (reinterpret_cast<uintptr_t>(w_packed) % 16 == 0);
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  const uint64_t dev_bit = dev < 64 ? uint64_t(1) << dev : 0;
#define BS_GEMV(VEC, FUSED)                                                                            \
  {                                                                                                    \
    auto kern = gemv_kernel<A, W, VEC, FUSED>;                                                         \
    static std::atomic<uint64_t> configured{0}; /* per device: opt-in to kMaxSmem once */           \
    if (!dev_bit || !(configured.load(std::memory_order_acquire) & dev_bit)) {                         \
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kMaxSmem)); \
      if (e != cudaSuccess) return e;                                                                  \
      configured.fetch_or(dev_bit, std::memory_order_release);                                         \
    }                                                                                                  \
    kern<<<grid, kGemvThreads, smem, stream>>>(a_packed, a_codes, w_packed, out, int(m), n, k, int(kwp), bipolar); \
  }
  if (a_codes) {
    if (vec4) BS_GEMV(4, true) else BS_GEMV(2, true)
  } else {
    if (vec4) BS_GEMV(4, false) else BS_GEMV(2, false)
  }
#undef BS_GEMV
  note_launch();
  return cudaPeekAtLastError();
}

}  // namespace

bool gemv_supported(int64_t m, int64_t k, int a_bits, int w_bits) {
  const bool bits_ok = (a_bits == 1 || a_bits == 2 || a_bits == 4) && (w_bits == 1 || w_bits == 2);
  const int64_t kwp = ((k + 31) / 32 + 1) / 2 * 2;
  return bits_ok && m >= 1 && m <= kMaxM && size_t(a_bits) * m * kwp * 4 + (kGemvThreads / 32) * kMaxM * 4 <= kMaxSmem;
}

cudaError_t launch_gemv(const uint32_t* a_packed, const uint8_t* a_codes, int a_bits, const uint32_t* w_packed,
                        int w_bits, int bipolar, int32_t* out, int64_t m, int64_t n, int64_t k, int64_t kwp,
                        cudaStream_t stream) {
#define BS_CASE(A, W) \
  if (a_bits == A && w_bits == W) return launch_aw<A, W>(a_packed, a_codes, w_packed, bipolar, out, m, n, k, kwp, stream);
  BS_CASE(1, 1) BS_CASE(2, 1) BS_CASE(2, 2) BS_CASE(1, 2) BS_CASE(4, 1) BS_CASE(4, 2)
#undef BS_CASE
  return cudaErrorNotSupported;
}

}  // namespace bs
