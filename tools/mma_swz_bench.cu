// mma_swz_bench.cu — tcgen05.mma kind::mxf4 (SS) issue rate vs the shared-memory layout of the
// operands (B200, sm_100a): K-major no-swizzle (16-byte core matrices), 32-, 64- and 128-byte
// swizzle, with the A start address stepping by whole rows between MMAs (the window path's tap
// offsets) or fixed.  One CTA per SM, one thread issues R MMAs, commit, wait; clock64 around.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_swz tools/mma_swz_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// layout: 0 none (core matrices 8 x 16 B, SBO 128, LBO = lbo), 1 = SW128 (rows 128 B, SBO 1024),
// 2 = SW64 (rows 64 B, SBO 512), 3 = SW32 (rows 32 B, SBO 256)
__device__ __forceinline__ uint64_t desc(uint32_t saddr, int layout, uint32_t lbo) {
  const uint32_t sbo = layout == 0 ? 128 : (layout == 1 ? 1024 : (layout == 2 ? 512 : 256));
  const uint64_t code = layout == 0 ? 0 : (layout == 1 ? 2 : (layout == 2 ? 4 : 6));
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(((layout == 0 ? lbo : 16) >> 4) & 0x3FFF) << 16) |
         (uint64_t(sbo >> 4) << 32) | (uint64_t(1) << 46) | (code << 61);
}

template <int layout>
__global__ void __launch_bounds__(128, 1) bench(int n, int step_rows, int reps, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x11111111u * (i & 3);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (1u << 23) | (uint32_t(128 >> 4) << 24);
    const uint32_t rowb = layout == 0 ? 16 : (layout == 1 ? 128 : (layout == 2 ? 64 : 32));
    const uint32_t a0 = su32(smem), b0 = su32(smem + 65536);
    const uint32_t lbo = 128 * 16;  // no-swizzle: second 16-byte K half 2 KB later
    const uint64_t bd = desc(b0, layout, lbo);
    uint64_t ad[8];
    for (int i = 0; i < 8; ++i) ad[i] = desc(a0 + uint32_t((i * step_rows) & 63) * rowb, layout, lbo);
    long long t0 = clock64();
    for (int r = 0; r < reps; r += 8) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile(
            "{.reg .pred p; setp.ne.b32 p, %6, 0;\n"
            "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;}" ::"r"(tmem),
            "l"(ad[i]), "l"(bd), "r"(idesc), "r"(tmem + 256), "r"(tmem + 272), "r"(r + i));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
    asm volatile(
        "{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(su32(&bar))
        : "memory");
    long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(bench<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const char* names[4] = {"none", "sw128", "sw64", "sw32"};
  const int reps = 4096;
  for (int layout = 0; layout < 4; ++layout)
    for (int n : {64, 128, 256})
      for (int step : {0, 3}) {
        if (layout == 0) bench<0><<<148, 128, 100 * 1024>>>(n, step, reps, d);
        if (layout == 1) bench<1><<<148, 128, 100 * 1024>>>(n, step, reps, d);
        if (layout == 2) bench<2><<<148, 128, 100 * 1024>>>(n, step, reps, d);
        if (layout == 3) bench<3><<<148, 128, 100 * 1024>>>(n, step, reps, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long c = 0;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        printf("{\"layout\": \"%s\", \"n\": %d, \"a_step_rows\": %d, \"clk_per_mma\": %.1f, \"floor\": %d, \"err\": \"%s\"}\n",
               names[layout], n, step, double(c) / reps, 128 * n / 256, cudaGetErrorString(e));
      }
  return 0;
}
