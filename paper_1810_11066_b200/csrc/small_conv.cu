// small_conv.cu — one-launch bitserial conv2d / dense for small problems (batch 1), SURVEY
// §2.5 N6: the latency regime where "the computational needs of the convolutions ... can't
// amortize the bit-packing costs" and packing is part of the timed operator
// (PAPER.md:715).
//
// One launch covers several independent problems (e.g. the ten ResNet-18 layers of one
// image).  Per CTA: a TM x TN output tile of one problem and one K slice of it.
//  * Activation packing is fused: the CTA reads the uint8 NHWC codes of its implicit-im2col
//    slab (zero padding = code 0) and packs them into bit-plane words in shared memory
//    (the same LSB-first word layout as bs_bitpack), so no packed copy of
//    the activations ever reaches HBM.
//  * Weights are the caller's packed planes (bs_bitpack of OHWI; packed ahead of time,
//    PAPER.md:715), staged per K slice.
//  * Inner loop: AND + POPC per word pair on the integer pipes, shifted by 2^(i+j) (Eq. 1
//    inside Eq. 2); bipolar weights through the exact identity
//    2*U - (2^W - 1)*sum(a) with the activation sums taken from the packed words.
//  * The K slices of one tile are the CTAs of one thread-block cluster: their partial sums
//    are reduced through distributed shared memory (no atomics, no zeroed output, no second
//    launch) — the split-K that lets a handful of batch-1 tiles fill 148 SMs.
#include <cooperative_groups.h>

#include <algorithm>
#include <atomic>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace bs {
namespace small {

constexpr int kThreads = 256;
constexpr int TM = 32;   // output pixels (rows) per tile
constexpr int TN = 64;   // filters (columns) per tile
constexpr int KC = 32;   // k-words staged per round
constexpr int kPadA = TM + 1;  // a[plane][k][pixel] pitch: conflict-free transposed writes
constexpr int kPadW = KC + 2;  // w[plane][filter][k] pitch: 8-byte cp.async rows, 16 filters on distinct banks
constexpr int kItems = TM * KC / kThreads;  // activation words per thread per round (4)
constexpr int kMaxTaps = 64;

struct Prob {
  const uint8_t* act;  // [n][h][w][c] uint8 codes
  const uint32_t* wt;  // packed [w_bits][oc][kwords]
  int32_t* out;        // [n][oh][ow][oc]
  int n, h, w, c, oc, kh, kw, sh, sw, ph, pw, oh, ow;
  int cw;              // packed words per pixel per plane
  int kwords;          // kh * kw * cw
  int M;               // n * oh * ow
  int mt, nt;          // tiles along M and N
  int cta0;            // first CTA of this problem (a multiple of the cluster size)
  int ksp;             // K slices per tile (power of two <= the cluster size)
  int cw_shift;        // log2(cw), or -1
  int bipolar;
  int vec;             // c % 16 == 0 and 16-byte aligned rows: 16-byte code loads
};

struct Args {
  int nprob, ks;  // problems; cluster size (a tile's K slices are consecutive CTAs of one cluster)
  Prob prob[kSmallMax];
};

template <int A, int W>
struct Smem {
  uint32_t a[A][KC][kPadA];  // packed activation words [plane][k][pixel]
  uint32_t w[W][TN][kPadW];  // packed weight words [plane][filter][k]
  int part[TM][TN];          // this K slice's partial sums
  int asum[TM];              // this K slice's activation sums (bipolar)
  int pix_iy[TM], pix_ix[TM];  // receptive-field origin of each output pixel (M past the end: far out)
  int64_t pix_base[TM];        // its element offset in the activations (may point into the padding)
  int tap_ky[kMaxTaps], tap_kx[kMaxTaps], tap_off[kMaxTaps];  // filter taps (kh * kw <= kMaxTaps)
};

// 32 codes (element 4q + r in byte r of v[q]) of pixel row `src`, zero past `cnt`.
__device__ __forceinline__ void load_codes(const uint8_t* src, int cnt, bool vec, uint32_t (&v)[8]) {
  if (vec && cnt >= 32) {
    const uint4 lo = __ldg(reinterpret_cast<const uint4*>(src)), hi = __ldg(reinterpret_cast<const uint4*>(src) + 1);
    v[0] = lo.x; v[1] = lo.y; v[2] = lo.z; v[3] = lo.w; v[4] = hi.x; v[5] = hi.y; v[6] = hi.z; v[7] = hi.w;
    return;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    uint32_t x = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r)
      if (4 * q + r < cnt) x |= uint32_t(__ldg(src + 4 * q + r)) << (8 * r);
    v[q] = x;
  }
}

template <int A, int W>
__global__ void __launch_bounds__(kThreads) small_conv_kernel(const __grid_constant__ Args args) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  Smem<A, W>& sm = *reinterpret_cast<Smem<A, W>*>(smem_raw);
  const int tid = threadIdx.x;
  const int cl = args.ks;
  int pi = 0;
  while (pi + 1 < args.nprob && int(blockIdx.x) >= args.prob[pi + 1].cta0) ++pi;
  const Prob& P = args.prob[pi];
  // cluster rank r: tile (cluster * cl / ksp + r / ksp), K slice r % ksp
  const int local = int(blockIdx.x) - P.cta0, rank = local % cl, ksp = P.ksp;
  const int split = rank % ksp;
  const int tile = (local / cl) * (cl / ksp) + rank / ksp;
  const bool active = tile < P.mt * P.nt;
  const int mtile = tile % P.mt, ntile = tile / P.mt;
  const int m0 = mtile * TM, n0 = ntile * TN;
  // K slice [k0, k1): even word boundaries (packed rows have an even word count), so every
  // 8-byte weight copy is aligned and inside its row
  const int k0 = active ? int(int64_t(P.kwords) * split / ksp) & ~1 : 0;
  const int k1 = !active ? 0 : split == ksp - 1 ? P.kwords : int(int64_t(P.kwords) * (split + 1) / ksp) & ~1;

  // per-CTA geometry tables: each output pixel's receptive-field origin, each tap's offset
  for (int t = tid; t < TM; t += kThreads) {
    sm.asum[t] = 0;
    const int m = m0 + t;
    if (m < P.M) {
      const int ohw = P.oh * P.ow;
      const int b = m / ohw, rem = m - b * ohw, oy = rem / P.ow, ox = rem - oy * P.ow;
      const int iy = oy * P.sh - P.ph, ix = ox * P.sw - P.pw;
      sm.pix_iy[t] = iy;
      sm.pix_ix[t] = ix;
      sm.pix_base[t] = ((int64_t(b) * P.h + iy) * P.w + ix) * P.c;
    } else {
      sm.pix_iy[t] = -(1 << 28);  // every tap out of bounds
      sm.pix_ix[t] = 0;
      sm.pix_base[t] = 0;
    }
  }
  for (int t = tid; t < P.kh * P.kw && t < kMaxTaps; t += kThreads) {
    const int ky = t / P.kw, kx = t - ky * P.kw;
    sm.tap_ky[t] = ky;
    sm.tap_kx[t] = kx;
    sm.tap_off[t] = (ky * P.w + kx) * P.c;
  }
  const int tx = tid & 15, ty = tid >> 4;  // filters tx + 16 f, pixels ty + 16 p
  int acc[2][4];
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int f = 0; f < 4; ++f) acc[p][f] = 0;
  __syncthreads();

  for (int kc0 = k0; kc0 < k1; kc0 += KC) {
    const int kn = min(KC, k1 - kc0);
    // ---- weight slab: TN filters x kn words per plane, 8-byte cp.async (rows are contiguous
    // in K; k-word counts and offsets are even), issued first so its latency overlaps the
    // activation loads below
    const int kn2 = (kn + 1) >> 1;
    for (int it = tid; it < W * TN * kn2; it += kThreads) {
      const int k2 = it % kn2, rest = it / kn2, tn = rest % TN, j = rest / TN;
      const int n = n0 + tn;
      const bool ok = n < P.oc;
      const uint32_t* src = P.wt + (int64_t(j) * P.oc + (ok ? n : 0)) * P.kwords + kc0 + 2 * k2;
      cp_async8(smem_u32(&sm.w[j][tn][2 * k2]), src, ok);
    }
    cp_async_commit();
    // ---- activation slab: implicit im2col of TM output pixels x kn words from the uint8
    // codes, packed here.  All of a thread's loads are issued before any is used.
    uint32_t v[kItems][8];
    bool okv[kItems];
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
      const int it = tid + r * kThreads;
      const int tm = it / KC, kk = it - tm * KC;  // consecutive threads: consecutive words of one pixel
      const int k = kc0 + kk;
      bool ok = kk < kn;
      if (ok) {
        const int tap = P.cw_shift >= 0 ? k >> P.cw_shift : k / P.cw, wd = k - tap * P.cw;
        const int iy = sm.pix_iy[tm] + sm.tap_ky[tap], ix = sm.pix_ix[tm] + sm.tap_kx[tap];
        ok = unsigned(iy) < unsigned(P.h) && unsigned(ix) < unsigned(P.w);
        if (ok) load_codes(P.act + sm.pix_base[tm] + sm.tap_off[tap] + wd * 32, P.c - wd * 32, P.vec, v[r]);
      }
      okv[r] = ok;
    }
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
      const int it = tid + r * kThreads;
      const int tm = it / KC, kk = it - tm * KC;
      int s = 0;
#pragma unroll
      for (int i = 0; i < A; ++i) {
        const uint32_t word = okv[r] ? plane_word(v[r], i) : 0u;
        sm.a[i][kk][tm] = word;
        s += __popc(word) << i;
      }
      if (P.bipolar && s) atomicAdd(&sm.asum[tm], s);
    }
    cp_async_wait<0>();
    __syncthreads();
    // ---- AND + POPC (Eq. 1 per word pair, Eq. 2 weights)
    for (int kk = 0; kk < kn; ++kk) {
      uint32_t a[A][2], w[W][4];
#pragma unroll
      for (int i = 0; i < A; ++i)
#pragma unroll
        for (int p = 0; p < 2; ++p) a[i][p] = sm.a[i][kk][ty + 16 * p];
#pragma unroll
      for (int j = 0; j < W; ++j)
#pragma unroll
        for (int f = 0; f < 4; ++f) w[j][f] = sm.w[j][tx + 16 * f][kk];
#pragma unroll
      for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          int d = 0;
#pragma unroll
          for (int i = 0; i < A; ++i)
#pragma unroll
            for (int j = 0; j < W; ++j) d += __popc(a[i][p] & w[j][f]) << (i + j);
          acc[p][f] += d;
        }
    }
    __syncthreads();
  }

  // ---- reduce the K slices of the tile (ksp consecutive CTAs of the cluster) and store
  auto finish = [&](int tm, int tn, int u, int s) {
    const int m = m0 + tm, n = n0 + tn;
    if (m < P.M && n < P.oc) P.out[int64_t(m) * P.oc + n] = P.bipolar ? 2 * u - ((1 << W) - 1) * s : u;
  };
  if (cl == 1 || ksp == 1) {
    if (active) {
#pragma unroll
      for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int f = 0; f < 4; ++f) finish(ty + 16 * p, tx + 16 * f, acc[p][f], sm.asum[ty + 16 * p]);
    }
    return;  // (all CTAs of a cluster belong to one problem: none of them reads peers)
  }
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int f = 0; f < 4; ++f) sm.part[ty + 16 * p][tx + 16 * f] = acc[p][f];
  cg::cluster_group cluster = cg::this_cluster();
  cluster.sync();  // every slice's partials and sums are visible cluster-wide
  if (active) {  // this CTA reduces the pixels [split * TM / ksp, (split + 1) * TM / ksp) of its tile
    const int first = rank - split;  // cluster rank of the tile's slice 0
    const int r0 = split * TM / ksp, r1 = (split + 1) * TM / ksp;
    for (int o = tid; o < (r1 - r0) * TN; o += kThreads) {
      const int tm = r0 + o / TN, tn = o % TN;
      int u = 0, s = 0;
      for (int q = 0; q < ksp; ++q) {
        const Smem<A, W>* peer = cluster.map_shared_rank(&sm, first + q);
        u += peer->part[tm][tn];
        s += peer->asum[tm];
      }
      finish(tm, tn, u, s);
    }
  }
  cluster.sync();  // peers' shared memory stays alive until every reader is done
}

template <int A, int W>
cudaError_t launch_aw(const Args& a, int ctas, cudaStream_t stream) {
  auto kern = small_conv_kernel<A, W>;
  const int smem = int(sizeof(Smem<A, W>));
  static std::atomic<uint64_t> configured{0};  // per device: dynamic smem opt-in
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  const uint64_t bit = dev < 64 ? uint64_t(1) << dev : 0;
  if (!bit || !(configured.load(std::memory_order_acquire) & bit)) {
    if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) return e;
    if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) return e;
    configured.fetch_or(bit, std::memory_order_release);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(ctas), 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = size_t(smem);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(a.ks);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  note_launch();
  return e != cudaSuccess ? e : cudaPeekAtLastError();
}

}  // namespace small

bool small_supported(int a_bits, int w_bits) { return a_bits >= 1 && a_bits <= 4 && w_bits >= 1 && w_bits <= 2; }

// Per problem, K slices per tile: a power of two up to the cluster size 8, raised until a
// slice's AND+POPC work is at most twice the launch's average tile (so the long-K layers of a
// network do not form the tail), keeping >= 2 k-words per slice.  Splitting costs a cluster
// barrier and a distributed-shared-memory reduction (measured ~1.5 us per doubling at batch
// 1), so tiles of average work are never split.  The launch's cluster size is the largest
// slice count (1: no cluster).
void small_pick_ksp(const SmallConv* ps, int count, int* ksp) {
  const int forced = tuning(kTuneSmallKs);
  int64_t tiles = 0, total = 0;
  for (int q = 0; q < count; ++q) {
    const int64_t t = int64_t((ps[q].p.M + small::TM - 1) / small::TM) * ((ps[q].p.oc + small::TN - 1) / small::TN);
    tiles += t;
    total += t * ps[q].p.kp;
  }
  const int64_t avg = tiles ? total / tiles : 0;
  for (int q = 0; q < count; ++q) {
    int k = 1;
    if (forced) {
      k = forced;
    } else {
      while (k < 8 && ps[q].p.kp >= 4 * k && ps[q].p.kp / k > 2 * avg) k *= 2;
    }
    ksp[q] = k;
  }
}

cudaError_t launch_small_conv(const SmallConv* ps, int count, int a_bits, int w_bits, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  if (count > kSmallMax || !small_supported(a_bits, w_bits)) return cudaErrorNotSupported;
  small::Args a{};
  a.nprob = count;
  int ksp[kSmallMax];
  small_pick_ksp(ps, count, ksp);
  a.ks = 1;
  for (int q = 0; q < count; ++q) a.ks = std::max(a.ks, ksp[q]);
  int64_t ctas = 0;
  for (int q = 0; q < count; ++q) {
    const ConvProblem& p = ps[q].p;
    small::Prob& P = a.prob[q];
    P.act = ps[q].act;
    P.wt = p.wt;
    P.out = p.out;
    P.n = p.n; P.h = p.h; P.w = p.w; P.c = p.c_tap; P.oc = p.oc; P.kh = p.kh; P.kw = p.kwid;
    P.sh = p.sh; P.sw = p.sw; P.ph = p.ph; P.pw = p.pw; P.oh = p.oh; P.ow = p.ow;
    P.cw = p.kw_a;
    P.kwords = int(p.kp);
    P.M = int(p.M);
    P.mt = (P.M + small::TM - 1) / small::TM;
    P.nt = (p.oc + small::TN - 1) / small::TN;
    P.cta0 = int(ctas);
    P.ksp = ksp[q];
    P.cw_shift = -1;
    for (int sh = 0; sh < 31; ++sh)
      if ((1 << sh) == P.cw) P.cw_shift = sh;
    P.bipolar = p.bipolar == 1;
    P.vec = (p.c_tap % 16 == 0) && (reinterpret_cast<uintptr_t>(ps[q].act) % 16 == 0);
    if (p.kh * p.kwid > small::kMaxTaps) return cudaErrorNotSupported;
    const int64_t tiles = int64_t(P.mt) * P.nt, per = a.ks / P.ksp;  // tiles per cluster
    ctas += (tiles + per - 1) / per * a.ks;
    if (ctas > (int64_t(1) << 31) - 1) return cudaErrorInvalidValue;
  }
#define BS_SMALL(A, W) \
  if (a_bits == A && w_bits == W) return small::launch_aw<A, W>(a, int(ctas), stream);
  BS_SMALL(1, 1) BS_SMALL(2, 1) BS_SMALL(3, 1) BS_SMALL(4, 1) BS_SMALL(1, 2) BS_SMALL(2, 2) BS_SMALL(3, 2)
  BS_SMALL(4, 2)
#undef BS_SMALL
  return cudaErrorNotSupported;
}

}  // namespace bs
