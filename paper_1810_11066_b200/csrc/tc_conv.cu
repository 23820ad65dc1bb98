// tc_conv.cu — bitserial conv2d / dense on the 5th-generation tensor cores (tcgen05).
//
// Eq. 2: out = sum_{i<A} sum_{j<W} 2^(i+j) * popcount(a_i AND w_j).
// For 0/1 vectors popcount(a_i AND w_j) = sum_k a_i[k] * w_j[k] (Eq. 1),
// a dense contraction, so every plane pair (i, j) is one binary dot product that the
// tensor core can evaluate exactly in int8 x int8 -> int32:
//   * activation plane i is expanded from its packed uint32 words into bytes 2^i * a_i
//     (u8) inside shared memory — operands stay bit-packed in HBM (A/8 bytes per
//     element, the point of bit-packing);
//   * weight plane j is expanded once per call into bytes 2^j * b_j (unipolar) or
//     2^j * (2 b_j - 1) (bipolar: each weight bit-plane a +/-1 digit, reading R2);
//   * the A*W plane-pair products are accumulated into one TMEM int32 accumulator with
//     tcgen05.mma.kind::i8 (bipolar needs no correction term in this form).
// The cost still grows with A*W (one MMA per plane pair), so this is the
// bitserial method with its binary dot products on the tensor cores instead of the
// integer pipes.
//
// Structure (one CTA = 128 output rows x BN output channels, 128 threads):
//   per K-chunk of 128 reduction elements (4 packed words per plane per row):
//     - all threads: B tile (expanded weights) -> swizzled smem with 16-byte cp.async,
//       A rows gathered (implicit im2col, zero padding) from the packed activations and
//       expanded to bytes straight into the 128B-swizzled K-major smem layout;
//     - fence.proxy.async + barrier; one thread issues A*W*4 tcgen05.mma (K = 32 each)
//       and commits them to the stage's mbarrier, releasing the buffers;
//   epilogue: tcgen05.ld 32x32b (warp w owns TMEM lanes 32w..32w+31 = rows), int32 store.
#include <cstdio>

#include "common.cuh"
#include "kernels.h"

namespace bs {
namespace tc {

constexpr int kThreads = 256;  // 8 warps: two threads per A row; warps w and w+4 share TMEM lanes
constexpr int BM = 128;          // UMMA M (cta_group::1)
constexpr int BKB = 128;         // K bytes per stage = one 128B swizzle row
constexpr int kWordsPerStage = BKB / 32;  // 4 packed words per plane per row

__device__ __forceinline__ void mbar_init(uint32_t addr, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(phase));
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// 128B-swizzled K-major UMMA shared-memory descriptor (SM100 layout, version 1):
// start address >> 4, LBO (unused for swizzled K-major) = 1, SBO = 1024 B (8 rows x
// 128 B) >> 4, layout type 2 = SWIZZLE_128B.  The tile base must be 1024-byte aligned;
// stepping K by 32 bytes inside the swizzle row is a +2 on the start field.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;  // version
  d |= uint64_t(2) << 61;  // SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::i8: D = S32, A = u8 (activation planes, 0 or 2^i),
// B = s8 (weight planes, +/-2^j or 0/2^j), both K-major, M = 128, N = BN.
template <int BN>
constexpr uint32_t idesc_i8() {
  return (2u << 4) | (0u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar) : "memory");
}

// Spread the 4 bits of a nibble (already isolated in the low bits of n) into bytes:
// n * (0x00204081 << i) puts bit r at 8r + i (other partial products elsewhere) and the
// mask keeps exactly those: byte r = 2^i * bit r.
template <int I>
__device__ __forceinline__ uint32_t spread4(uint32_t n) {
  return (n * (0x00204081u << I)) & (0x01010101u << I);
}

// 32 activation bits of one plane word -> 8 words of bytes (element 4q + r in byte r
// of word q), value 2^I * bit.  The 8 nibbles are isolated with two masks and a
// byte permute each (PRMT) instead of a shift + mask per nibble.
template <int I>
__device__ __forceinline__ void expand_word(uint32_t w, uint32_t (&o)[8]) {
  const uint32_t lo = w & 0x0F0F0F0Fu, hi = (w >> 4) & 0x0F0F0F0Fu;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    o[2 * b] = spread4<I>(__byte_perm(lo, 0u, 0x4440u + b));
    o[2 * b + 1] = spread4<I>(__byte_perm(hi, 0u, 0x4440u + b));
  }
}

// ------------------------------------------------------------------ weight expansion
// w_packed [W][N][kp] words -> wexp [W][n_pad][kpad*32] bytes (kpad = kp rounded up to
// 4 words; bytes past kp*32 are 0).  Plane j byte = 2^j b (unipolar) or 2^j (2b - 1)
// (bipolar); zero padding of the activations makes the value of pad bytes irrelevant.
__global__ void __launch_bounds__(256) expand_weights_kernel(const uint32_t* __restrict__ w_packed,
                                                             int8_t* __restrict__ wexp, int w_bits, int n,
                                                             int64_t kp, int64_t kpad, int bipolar) {
  const int64_t words = int64_t(w_bits) * n * kpad;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < words; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t kk = t % kpad, rest = t / kpad;
    const int64_t row = rest % n, j = rest / n;
    const uint32_t w = kk < kp ? w_packed[(j * n + row) * kp + kk] : 0u;
    const int32_t mag = 1 << j;
    uint32_t out[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t n4 = (w >> (4 * q)) & 0xFu;
      const uint32_t bits = (n4 * 0x00204081u) & 0x01010101u;  // 0/1 per byte
      uint32_t v = 0;
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int b = (bits >> (8 * r)) & 1;
        const int32_t val = bipolar ? (b ? mag : -mag) : (b ? mag : 0);
        v |= (uint32_t(val) & 0xFFu) << (8 * r);
      }
      out[q] = v;
    }
    uint4* dst = reinterpret_cast<uint4*>(wexp + (j * int64_t(n) + row) * kpad * 32 + kk * 32);
    dst[0] = make_uint4(out[0], out[1], out[2], out[3]);
    dst[1] = make_uint4(out[4], out[5], out[6], out[7]);
  }
}

// ----------------------------------------------------------------------- main kernel
template <int A_BITS, int W_BITS, int BN, int STAGES>
struct TcSmem {  // 1024 B of alignment slack + mbarriers / TMEM slot
  static constexpr int kABytes = A_BITS * BM * BKB;   // per stage
  static constexpr int kBBytes = W_BITS * BN * BKB;   // per stage
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kBytes = STAGES * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

template <int A_BITS, int W_BITS, int BN, int STAGES, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) tc_conv_kernel(const ConvProblem p, const int8_t* __restrict__ wexp,
                                                              const int64_t kpad) {
  using S = TcSmem<A_BITS, W_BITS, BN, STAGES>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  static_assert(MINB >= 1, "");
  // 1024-byte aligned tile region (SWIZZLE_128B atoms), barriers after the tiles
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + STAGES * S::kStageBytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + STAGES + 1);

  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t m0 = int64_t(blockIdx.x) * BM;
  const int n0 = blockIdx.y * BN;
  const int kp = int(p.kp);
  const int nchunks = int(kpad / kWordsPerStage);

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(smem_u32(mbar + s), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {  // TMEM: BN int32 columns x 128 lanes
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(BN < 32 ? 32 : BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // ---- this thread's A row (output pixel), its receptive-field origin, and which
  // half of the 128-byte K chunk it expands (packed words 2*half, 2*half+1)
  const int arow = tid & (BM - 1), half = tid >> 7;
  const int64_t m = m0 + arow;
  const bool row_ok = m < p.M;
  int iy0 = 0, ix0 = 0;
  int64_t img_base = 0;
  {
    const int64_t mm = row_ok ? m : 0;
    const int64_t hw = int64_t(p.oh) * p.ow;
    const int64_t b = mm / hw, rem = mm - b * hw;
    const int oy = int(rem / p.ow), ox = int(rem - int64_t(oy) * p.ow);
    iy0 = oy * p.sh - p.ph;
    ix0 = ox * p.sw - p.pw;
    img_base = b * int64_t(p.h) * p.w;
  }
  const uint32_t sw = uint32_t(arow & 7);  // 128B swizzle phase of this row

  // 8-byte piece (2 packed words per plane) this thread gathers for K chunk kc; the
  // piece lies inside one tap because Cw is even (implicit im2col, zero padding)
  auto gather = [&](int kc, uint2 (&v)[A_BITS]) {
    const int kk = kc * kWordsPerStage + 2 * half;
    const int tap = kk / p.kw_a;
    const int cw = kk - tap * p.kw_a;
    const int ky = tap / p.kwid, kx = tap - ky * p.kwid;
    const int iy = iy0 + ky, ix = ix0 + kx;
    const bool ok = row_ok && kk < kp && iy >= 0 && iy < p.h && ix >= 0 && ix < p.w;
    const uint32_t* src = p.act + (img_base + int64_t(iy) * p.w + ix) * p.kw_a + cw;
#pragma unroll
    for (int i = 0; i < A_BITS; ++i) {
      v[i] = make_uint2(0u, 0u);
      if (ok) v[i] = __ldg(reinterpret_cast<const uint2*>(src + i * p.act_plane));
    }
  };

  constexpr uint32_t kIdesc = idesc_i8<BN>();
  uint32_t phase_bits = 0;  // bit s = parity to wait for on stage s
  uint2 wa[A_BITS];
  gather(0, wa);

  for (int kc = 0; kc < nchunks; ++kc) {
    const int s = kc % STAGES;
    uint8_t* sA = smem + s * S::kStageBytes;
    uint8_t* sB = sA + S::kABytes;
    if (kc >= STAGES) {  // wait until the MMAs that read this stage have completed
      mbar_wait(smem_u32(mbar + s), (phase_bits >> s) & 1u);
      phase_bits ^= 1u << s;
    }
    // B: expanded weight rows n0..n0+BN, bytes [kc*128, kc*128+128) per plane
    {
      constexpr int kChunks = W_BITS * BN * (BKB / 16);
#pragma unroll 4
      for (int c = tid; c < kChunks; c += kThreads) {
        const int j = c / (BN * 8), rem = c - j * (BN * 8);
        const int r = rem >> 3, ch = rem & 7;
        const int n = n0 + r;
        const bool ok = n < p.oc;
        const int8_t* src = ok ? wexp + (int64_t(j) * p.oc + n) * (kpad * 32) + int64_t(kc) * BKB + ch * 16 : wexp;
        const uint32_t dst = smem_u32(sB + j * (BN * BKB) + r * BKB + ((ch ^ (r & 7)) << 4));
        cp_async16(dst, src, ok);
      }
      cp_async_commit();
    }
    // A: prefetch the next chunk's words, then expand this chunk's into swizzled smem
    uint2 wn[A_BITS];
    if (kc + 1 < nchunks) gather(kc + 1, wn);
#pragma unroll
    for (int i = 0; i < A_BITS; ++i) {
      uint8_t* rowp = sA + i * (BM * BKB) + (arow >> 3) * 1024 + (arow & 7) * 128;
#pragma unroll
      for (int wsel = 0; wsel < 2; ++wsel) {
        const uint32_t w = wsel ? wa[i].y : wa[i].x;
        uint32_t o[8];
        switch (i) {  // compile-time after unrolling
          case 0: expand_word<0>(w, o); break;
          case 1: expand_word<1>(w, o); break;
          case 2: expand_word<2>(w, o); break;
          default: expand_word<3>(w, o); break;
        }
        const uint32_t ch0 = uint32_t(4 * half + 2 * wsel);  // 16-byte chunks of this word
        *reinterpret_cast<uint4*>(rowp + ((ch0 ^ sw) << 4)) = make_uint4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<uint4*>(rowp + (((ch0 + 1) ^ sw) << 4)) = make_uint4(o[4], o[5], o[6], o[7]);
      }
    }
#pragma unroll
    for (int i = 0; i < A_BITS; ++i) wa[i] = wn[i];
    cp_async_wait<0>();
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
#pragma unroll
      for (int i = 0; i < A_BITS; ++i)
#pragma unroll
        for (int j = 0; j < W_BITS; ++j)
#pragma unroll
          for (int k = 0; k < BKB / 32; ++k) {
            const uint64_t ad = smem_desc_sw128(a_base + i * (BM * BKB) + k * 32);
            const uint64_t bd = smem_desc_sw128(b_base + j * (BN * BKB) + k * 32);
            mma_i8(tmem, ad, bd, kIdesc, (kc | i | j | k) != 0);
          }
      mma_commit(smem_u32(mbar + s));
    }
  }
  // wait for the last commit (covers all earlier MMAs)
  {
    const int s = (nchunks - 1) % STAGES;
    mbar_wait(smem_u32(mbar + s), (phase_bits >> s) & 1u);
  }
  tc_fence_after();

  // ---- epilogue, 64 columns at a time: warp w loads TMEM lanes 32*(w%4).. (rows) x 32
  // columns (half w/4 of the block) into a padded smem tile (ring buffers are free now),
  // then all threads write the 128 x 64 int32 block with coalesced 16-byte stores (each
  // output row segment is contiguous in NHWC / row-major memory).
  constexpr int kCB = 64, kLd = kCB + 4;  // +4 words: conflict-free 16-byte smem rows
  uint32_t* stile = reinterpret_cast<uint32_t*>(smem);
  const int quarter = warp & 3, colhalf = warp >> 2;
  const int trow = quarter * 32 + (tid & 31);
#pragma unroll 1
  for (int cb = 0; cb < BN; cb += kCB) {
    uint32_t r[32];
    const uint32_t taddr = tmem + (uint32_t(quarter * 32) << 16) + uint32_t(cb + colhalf * 32);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    uint32_t* srow = stile + trow * kLd + colhalf * 32;
#pragma unroll
    for (int v = 0; v < 8; ++v)
      *reinterpret_cast<uint4*>(srow + 4 * v) = make_uint4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
    __syncthreads();
    const int ncols = min(kCB, p.oc - (n0 + cb));  // valid columns of this block
    if ((p.oc & 3) == 0 && ncols == kCB) {
#pragma unroll
      for (int c = tid; c < BM * (kCB / 4); c += kThreads) {
        const int rr = c / (kCB / 4), c4 = c - rr * (kCB / 4);
        const int64_t grow = m0 + rr;
        if (grow < p.M)
          *reinterpret_cast<uint4*>(p.out + grow * p.oc + n0 + cb + 4 * c4) =
              *reinterpret_cast<const uint4*>(stile + rr * kLd + 4 * c4);
      }
    } else if (ncols > 0) {
      for (int c = tid; c < BM * kCB; c += kThreads) {
        const int rr = c / kCB, cc = c - rr * kCB;
        const int64_t grow = m0 + rr;
        if (grow < p.M && cc < ncols) p.out[grow * p.oc + n0 + cb + cc] = int32_t(stile[rr * kLd + cc]);
      }
    }
    __syncthreads();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN < 32 ? 32 : BN));
  }
}

// Stages: as many as fit while two CTAs (16 warps) still share an SM — a second CTA
// overlaps one tile's prologue / epilogue with another's main loop — else as many as fit
// one CTA (at least 2).
template <int A_BITS, int W_BITS, int BN>
cudaError_t launch_bn(const ConvProblem& p, const int8_t* wexp, int64_t kpad, cudaStream_t stream) {
  constexpr int kStageBytes = TcSmem<A_BITS, W_BITS, BN, 1>::kStageBytes;
  constexpr int kPerCta2 = (227 * 1024) / 2 - 2304;
  constexpr int kStages2 = kPerCta2 / kStageBytes;
  constexpr bool kTwo = kStages2 >= 2;
  constexpr int kStages1 = ((227 * 1024) - 2304) / kStageBytes;
  constexpr int STAGES = kTwo ? (kStages2 > 4 ? 4 : kStages2) : (kStages1 > 4 ? 4 : kStages1);
  static_assert(STAGES >= 2, "tensor-core tile does not fit two stages of shared memory");
  using S = TcSmem<A_BITS, W_BITS, BN, STAGES>;
  static_assert(S::kBytes <= 227 * 1024, "tensor-core tile does not fit shared memory");
  auto kern = tc_conv_kernel<A_BITS, W_BITS, BN, STAGES, kTwo ? 2 : 1>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kBytes);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid(unsigned((p.M + BM - 1) / BM), unsigned((p.oc + BN - 1) / BN));
  kern<<<grid, kThreads, S::kBytes, stream>>>(p, wexp, kpad);
  note_launch();
  return cudaPeekAtLastError();
}

template <int A_BITS, int W_BITS>
cudaError_t launch_aw(const ConvProblem& p, const int8_t* wexp, int64_t kpad, cudaStream_t stream) {
  if (p.oc <= 64) return launch_bn<A_BITS, W_BITS, 64>(p, wexp, kpad, stream);
  if constexpr (A_BITS * W_BITS <= 4) {
    if (p.oc > 128) return launch_bn<A_BITS, W_BITS, 256>(p, wexp, kpad, stream);
  }
  return launch_bn<A_BITS, W_BITS, 128>(p, wexp, kpad, stream);
}

}  // namespace tc

int64_t tc_weight_bytes(int64_t n, int64_t kp, int w_bits) {
  const int64_t kpad = (kp + tc::kWordsPerStage - 1) / tc::kWordsPerStage * tc::kWordsPerStage;
  return int64_t(w_bits) * n * kpad * 32;
}

bool tc_supported(int a_bits, int w_bits) {
  return a_bits >= 1 && a_bits <= 4 && w_bits >= 1 && w_bits <= 2;
}

cudaError_t launch_tc_conv(const ConvProblem& p, int8_t* wexp_ws, cudaStream_t stream) {
  if (!tc_supported(p.a_bits, p.w_bits)) return cudaErrorNotSupported;
  const int64_t kpad = (p.kp + tc::kWordsPerStage - 1) / tc::kWordsPerStage * tc::kWordsPerStage;
  {
    const int64_t words = int64_t(p.w_bits) * p.oc * kpad;
    int64_t blocks = (words + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    tc::expand_weights_kernel<<<unsigned(blocks), 256, 0, stream>>>(p.wt, wexp_ws, p.w_bits, p.oc, p.kp, kpad,
                                                                    p.bipolar);
    note_launch();
    cudaError_t e = cudaPeekAtLastError();
    if (e != cudaSuccess) return e;
  }
#define BS_TC(A, W) \
  if (p.a_bits == A && p.w_bits == W) return tc::launch_aw<A, W>(p, wexp_ws, kpad, stream);
  BS_TC(1, 1) BS_TC(2, 1) BS_TC(2, 2) BS_TC(1, 2) BS_TC(3, 1) BS_TC(3, 2) BS_TC(4, 1) BS_TC(4, 2)
#undef BS_TC
  return cudaErrorNotSupported;
}

}  // namespace bs
