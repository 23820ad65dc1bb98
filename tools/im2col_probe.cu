// im2col_probe.cu — what does a TMA im2col load (cp.async.bulk.tensor.4d ... .im2col) put in
// shared memory on this GPU?  Design probe for the TMA-fed digit conv kernel (not product
// code).  A uint8 NHWC tensor [N][H][W][CB bytes] with distinct bytes; for every filter tap
// (r, q) of a KHxKW / stride / pad convolution one load of `pixels` output pixels starting at
// output pixel m0, im2col offsets (q, r), coordinates (c0, ox0*s - p, oy0*s - p, n0), bounding
// box lower = -p, upper = (OW-1)*s - p - (W-1).  Expectation: row i = input pixel
// (n, oy*s - p + r, ox*s - p + q) of output pixel m0 + i (NHW-linear), zero when outside the
// image or n >= N.  Checks SWIZZLE_NONE (row i at i*CB) and SWIZZLE_32B/64B/128B (16-byte chunk
// j of row i at chunk j ^ ((i*CB/128) & (CB/16 - 1)) ... per the usual Hopper/Blackwell rule).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/im2col_probe tools/im2col_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                      \
    }                                                                                \
  } while (0)

__global__ void probe(const __grid_constant__ CUtensorMap map, int c0, int w0, int h0, int n0, int offw, int offh,
                      int bytes, uint8_t* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  const uint32_t sb = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
  const uint32_t sd = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) smem[i] = 0xEE;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(bytes) : "memory");
    const uint16_t ow16 = uint16_t(offw), oh16 = uint16_t(offh);
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6], {%7, %8};" ::"r"(sd),
        "l"(reinterpret_cast<uint64_t>(&map)), "r"(c0), "r"(w0), "r"(h0), "r"(n0), "r"(sb), "h"(ow16), "h"(oh16)
        : "memory");
    asm volatile(
        "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(sb)
        : "memory");
  }
  __syncthreads();
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) out[i] = smem[i];
}

static PFN_cuTensorMapEncodeIm2col_v12000 get_enc() {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(f);
}

static uint8_t val(int n, int h, int w, int c) { return uint8_t(1 + ((n * 131 + h * 31 + w * 7 + c * 3) % 251)); }

// one case; returns mismatches
static int run_case(int N, int H, int W, int Cb, int CB, int c0, int KH, int KW, int s, int p, int64_t m0, int pixels,
                    int swz) {
  auto enc = get_enc();
  if (!enc) {
    printf("no cuTensorMapEncodeIm2col\n");
    return -1;
  }
  const int OH = (H + 2 * p - KH) / s + 1, OW = (W + 2 * p - KW) / s + 1;
  std::vector<uint8_t> h_in(size_t(N) * H * W * Cb);
  for (int n = 0; n < N; ++n)
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x)
        for (int c = 0; c < Cb; ++c) h_in[((size_t(n) * H + y) * W + x) * Cb + c] = val(n, y, x, c);
  uint8_t *d_in, *d_out;
  const int bytes = pixels * CB;
  CK(cudaMalloc(&d_in, h_in.size()));
  CK(cudaMalloc(&d_out, bytes));
  CK(cudaMemcpy(d_in, h_in.data(), h_in.size(), cudaMemcpyHostToDevice));
  CUtensorMap map;
  const cuuint64_t dims[4] = {cuuint64_t(Cb), cuuint64_t(W), cuuint64_t(H), cuuint64_t(N)};
  const cuuint64_t strides[3] = {cuuint64_t(Cb), cuuint64_t(Cb) * W, cuuint64_t(Cb) * W * H};
  const int lower[2] = {-p, -p};  // W, H
  const int upper[2] = {(OW - 1) * s - p - (W - 1), (OH - 1) * s - p - (H - 1)};
  const cuuint32_t estr[4] = {1, cuuint32_t(s), cuuint32_t(s), 1};
  const CUtensorMapSwizzle sw[4] = {CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_SWIZZLE_64B,
                                    CU_TENSOR_MAP_SWIZZLE_128B};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, d_in, dims, strides, lower, upper, cuuint32_t(CB),
                   cuuint32_t(pixels), estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw[swz], CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d (N%d H%d W%d Cb%d CB%d s%d p%d swz%d)\n", int(r), N, H, W, Cb, CB, s, p, swz);
    return -1;
  }
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const int64_t hw = int64_t(OH) * OW;
  const int nn0 = int(m0 / hw), rem = int(m0 % hw), oy0 = rem / OW, ox0 = rem % OW;
  int bad_total = 0;
  std::vector<uint8_t> got(bytes);
  for (int ky = 0; ky < KH; ++ky)
    for (int kx = 0; kx < KW; ++kx) {
      probe<<<1, 256, bytes + 1024>>>(map, c0, ox0 * s - p, oy0 * s - p, nn0, kx, ky, bytes, d_out);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(got.data(), d_out, bytes, cudaMemcpyDeviceToHost));
      int bad = 0;
      for (int i = 0; i < pixels; ++i) {
        const int64_t m = m0 + i;
        const int n = int(m / hw), rr = int(m % hw), oy = rr / OW, ox = rr % OW;
        const int iy = oy * s - p + ky, ix = ox * s - p + kx;
        const bool inb = n < N && iy >= 0 && iy < H && ix >= 0 && ix < W;
        for (int c = 0; c < CB; ++c) {
          const uint8_t e = inb ? val(n, iy, ix, c0 + c) : 0;
          int pos = i * CB + c;
          if (swz) {  // 16-byte chunk XOR with the row-of-128B index bits within the swizzle span
            const int span = 16 << swz;             // 32, 64, 128
            const int lin = i * CB + c;
            const int chunk = (lin % span) / 16;
            const int rowsel = (lin / 128) % (span / 16);
            pos = lin - chunk * 16 + ((chunk ^ rowsel) * 16);
          }
          if (got[pos] != e) {
            if (bad < 4)
              printf("  tap(%d,%d) row %d c %d: got %d want %d (n %d iy %d ix %d)\n", ky, kx, i, c, got[pos], e, n, iy,
                     ix);
            ++bad;
          }
        }
      }
      bad_total += bad;
    }
  printf("case N%d H%d W%d Cb%d CB%d c0 %d K%dx%d s%d p%d m0 %lld px %d swz%d: %s (%d bad bytes)\n", N, H, W, Cb, CB,
         c0, KH, KW, s, p, (long long)m0, pixels, swz, bad_total ? "MISMATCH" : "ok", bad_total);
  cudaFree(d_in);
  cudaFree(d_out);
  return bad_total;
}

int main() {
  int fails = 0;
  fails += run_case(2, 5, 7, 32, 32, 0, 3, 3, 1, 1, 0, 128, 0) != 0;
  fails += run_case(2, 5, 7, 32, 32, 0, 3, 3, 1, 1, 3, 128, 0) != 0;
  fails += run_case(2, 6, 9, 32, 32, 0, 3, 3, 2, 1, 5, 128, 0) != 0;
  fails += run_case(3, 6, 10, 64, 32, 32, 1, 1, 2, 0, 7, 128, 0) != 0;
  fails += run_case(2, 7, 5, 32, 32, 0, 3, 3, 1, 1, 0, 128, 1) != 0;
  fails += run_case(2, 7, 5, 64, 64, 0, 3, 3, 1, 1, 9, 128, 2) != 0;
  fails += run_case(2, 7, 5, 256, 128, 128, 3, 3, 2, 1, 4, 128, 3) != 0;
  fails += run_case(4, 14, 14, 128, 128, 0, 3, 3, 1, 1, 600, 128, 3) != 0;
  fails += run_case(2, 5, 6, 32, 32, 0, 5, 3, 1, 2, 1, 128, 1) != 0;  // non-square filter
  printf("%s\n", fails ? "FAILURES" : "ALL OK");
  return fails ? 1 : 0;
}
