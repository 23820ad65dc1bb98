// tma_rate.cu — how fast can one SM pull activation pixels into shared memory?  (Design probe
// for the digit conv kernel's operand loads; not product code.)  Every CTA (one per SM) streams
// `iters` loads of 128 rows x cb bytes through a ring of Q shared-memory slots:
//   mode 0: TMA im2col (cp.async.bulk.tensor.4d.im2col), 3x3 taps, stride s, over a
//           [N][H][W][cb] uint8 tensor (one elected thread issues, mbarrier per slot)
//   mode 1: TMA tiled 2-D box (128 rows x cb bytes) over [rows][cb]
//   mode 2: cp.async 16-byte copies by 128 threads (one row each, cb/16 copies), per-slot
//           mbarrier via cp.async.mbarrier.arrive.noinc
// Prints GB/s of smem fill and ns per 128-row load per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_rate tools/tma_rate.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void wait_par(uint32_t bar, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(bar),
               "r"(par)
               : "memory");
}

struct Geo {
  int N, H, W, OH, OW, s, p, M;
};

__global__ void rate_kernel(const __grid_constant__ CUtensorMap map, const uint8_t* __restrict__ src, Geo g, int mode,
                            int cb, int Q, int iters, unsigned long long* out_clk, int px = 128) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bars[64];
  const int slot_bytes = px * cb;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int q = 0; q < Q; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bars[q])), "r"(mode == 2 ? 128 : 1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long t0 = clock64();
  const int ntile = (g.M + px - 1) / px;
  for (int it = 0; it < iters; ++it) {
    const int q = it % Q;
    const uint32_t bar = su32(&bars[q]);
    const uint32_t dst = su32(smem + q * slot_bytes);
    if (it >= Q) {  // wait for the slot's previous load to land before reusing it
      if (mode != 2 ? tid == 0 : tid < 128) wait_par(bar, ((it / Q) - 1) & 1);
    }
    const int tile = (blockIdx.x + (it / 9) * gridDim.x) % ntile, tap = it % 9;
    const int m0 = tile * px;
    if (mode == 0 && tid == 0) {
      const int hw = g.OH * g.OW, n = m0 / hw, rem = m0 % hw, oy = rem / g.OW, ox = rem % g.OW;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(slot_bytes) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
          "%5}], [%6], {%7, %8};" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(ox * g.s - g.p), "r"(oy * g.s - g.p), "r"(n), "r"(bar),
          "h"(uint16_t(tap % 3)), "h"(uint16_t(tap / 3))
          : "memory");
    } else if (mode == 1 && tid == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(slot_bytes) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              dst),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(m0), "r"(bar)
          : "memory");
    } else if (mode == 2 && tid < 128) {
      const int m = m0 + tid;
      const int hw = g.OH * g.OW, n = m / hw, rem = m % hw, oy = rem / g.OW, ox = rem % g.OW;
      const int iy = oy * g.s - g.p + tap / 3, ix = ox * g.s - g.p + tap % 3;
      const bool ok = n < g.N && iy >= 0 && iy < g.H && ix >= 0 && ix < g.W;
      const uint8_t* s = src + ((int64_t(n) * g.H + (ok ? iy : 0)) * g.W + (ok ? ix : 0)) * cb;
      for (int c = 0; c < cb; c += 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + tid * cb + c), "l"(s + c),
                     "r"(ok ? 16 : 0));
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
    }
  }
  // drain
  for (int it = iters; it < iters + Q; ++it) {
    const int q = it % Q;
    if (it >= Q && (mode != 2 ? tid == 0 : tid < 128)) wait_par(su32(&bars[q]), ((it / Q) - 1) & 1);
  }
  __syncthreads();
  if (tid == 0) out_clk[blockIdx.x] = clock64() - t0;
}

int main(int argc, char** argv) {
  int dev = 0, sms = 0, mhz = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, dev));
  void* f = nullptr;
  cudaDriverEntryPointQueryResult qr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f, cudaEnableDefault, &qr));
  auto enc_im2col = reinterpret_cast<PFN_cuTensorMapEncodeIm2col_v12000>(f);
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &qr));
  auto enc_tiled = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  const int N = 256, H = 56, W = 56;
  uint8_t* d;
  CK(cudaMalloc(&d, size_t(N) * H * W * 128));
  CK(cudaMemset(d, 1, size_t(N) * H * W * 128));
  unsigned long long* clk;
  CK(cudaMalloc(&clk, sms * sizeof(unsigned long long)));
  CK(cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const int iters = 2000;
  printf("{\"sms\": %d, \"clock_mhz\": %d, \"rows\": [\n", sms, mhz / 1000);
  bool first = true;
  for (int mode = 0; mode < 3; ++mode)
    for (int cb : {32, 64, 128})
      for (int s : {1, 2})
        for (int Q : {4, 8, 16, 32, 48}) {
          if (mode == 1 && s == 2) continue;
          if (Q * 128 * cb > 190 * 1024) continue;
          const int OH = (H + 2 - 3) / s + 1, OW = (W + 2 - 3) / s + 1;
          Geo g{N, H, W, OH, OW, s, 1, N * OH * OW};
          CUtensorMap map;
          CUresult r;
          if (mode == 0) {
            const cuuint64_t dims[4] = {cuuint64_t(cb), cuuint64_t(W), cuuint64_t(H), cuuint64_t(N)};
            const cuuint64_t str[3] = {cuuint64_t(cb), cuuint64_t(cb) * W, cuuint64_t(cb) * W * H};
            const int lo[2] = {-1, -1}, up[2] = {(OW - 1) * s - 1 - (W - 1), (OH - 1) * s - 1 - (H - 1)};
            const cuuint32_t es[4] = {1, cuuint32_t(s), cuuint32_t(s), 1};
            r = enc_im2col(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, d, dims, str, lo, up, cuuint32_t(cb), 128, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           cb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                     : (cb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B),
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          } else {
            const cuuint64_t dims[2] = {cuuint64_t(cb), cuuint64_t(N) * H * W};
            const cuuint64_t str[1] = {cuuint64_t(cb)};
            const cuuint32_t box[2] = {cuuint32_t(cb), 128}, es[2] = {1, 1};
            r = enc_tiled(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          cb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                    : (cb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B),
                          CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          }
          if (r != CUDA_SUCCESS) {
            printf("encode failed %d\n", int(r));
            return 1;
          }
          rate_kernel<<<sms, 256, Q * 128 * cb + 1024>>>(map, d, g, mode, cb, Q, iters, clk);  // warm
          CK(cudaDeviceSynchronize());
          cudaEvent_t e0, e1;
          cudaEventCreate(&e0);
          cudaEventCreate(&e1);
          cudaEventRecord(e0);
          rate_kernel<<<sms, 256, Q * 128 * cb + 1024>>>(map, d, g, mode, cb, Q, iters, clk);
          cudaEventRecord(e1);
          CK(cudaDeviceSynchronize());
          float ms = 0;
          cudaEventElapsedTime(&ms, e0, e1);
          const double bytes = double(sms) * iters * 128 * cb;
          printf("%s{\"mode\": \"%s\", \"cb\": %d, \"stride\": %d, \"Q\": %d, \"GBps\": %.1f, \"ns_per_load_per_sm\": %.1f}",
                 first ? "" : ",\n", mode == 0 ? "im2col" : (mode == 1 ? "tiled2d" : "cp.async"), cb, s, Q,
                 bytes / ms / 1e6, ms * 1e6 / iters);
          first = false;
        }
  printf("\n], \"im2col_pixels\": [\n");
  first = true;
  for (int cb : {32, 128})
    for (int px : {32, 64, 128, 256, 512})
      for (int Q : {4, 16}) {
        if (Q * px * cb > 190 * 1024) continue;
        const int s = 1, OH = H, OW = W;
        Geo g{N, H, W, OH, OW, s, 1, N * OH * OW};
        CUtensorMap map;
        const cuuint64_t dims[4] = {cuuint64_t(cb), cuuint64_t(W), cuuint64_t(H), cuuint64_t(N)};
        const cuuint64_t str[3] = {cuuint64_t(cb), cuuint64_t(cb) * W, cuuint64_t(cb) * W * H};
        const int lo[2] = {-1, -1}, up[2] = {-1, -1};
        const cuuint32_t es[4] = {1, 1, 1, 1};
        CUresult r = enc_im2col(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, d, dims, str, lo, up, cuuint32_t(cb), cuuint32_t(px),
                                es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                cb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_32B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d px %d\n", int(r), px); continue; }
        rate_kernel<<<sms, 256, Q * px * cb + 1024>>>(map, d, g, 0, cb, Q, iters, clk, px);
        CK(cudaDeviceSynchronize());
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        rate_kernel<<<sms, 256, Q * px * cb + 1024>>>(map, d, g, 0, cb, Q, iters, clk, px);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%s{\"cb\": %d, \"pixels\": %d, \"Q\": %d, \"ns_per_load_per_sm\": %.1f, \"ns_per_pixel\": %.2f}",
               first ? "" : ",\n", cb, px, Q, ms * 1e6 / iters, ms * 1e6 / iters / px);
        first = false;
      }
  printf("\n]}\n");
  return 0;
}
