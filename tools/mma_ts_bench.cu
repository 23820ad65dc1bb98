// mma_ts_bench.cu — tcgen05.mma kind::mxf4 block_scale (M = 128, K = 64) issue rate with the A
// operand in shared memory (SS) vs in tensor memory (TS, as the expansion kernel issues it), at
// N = 64 / 128 / 256 (B200, sm_100a).  One CTA per SM; one thread issues R MMAs, commit, wait;
// clock64 around it.  Prints cycles per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_ts tools/mma_ts_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// K-major, 128-byte swizzle (rows of 128 bytes, 8-row atoms of 1 KB)
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) | (uint64_t(1) << 46) |
         (uint64_t(2) << 61);
}

template <bool TS>
__global__ void __launch_bounds__(128, 1) bench(int n, int reps, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x22222222u * (i & 1);
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
  // tensor memory: accumulator columns [0, n), A (TS) at 256 + 8 i, scale factors at 384 / 400
  {
    const uint32_t lane_base = tmem + (uint32_t(warp * 32) << 16);
    const uint32_t v = 0x7F7F7F7Fu;  // UE8M0 scale 1.0; also a valid E2M1 pattern for A
#pragma unroll
    for (int c = 256; c < 448; c += 4)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %1, %1, %1};" ::"r"(lane_base + uint32_t(c)),
                   "r"(v)
                   : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (1u << 23) | (uint32_t(128 >> 4) << 24);
    const uint32_t a0 = su32(smem), b0 = su32(smem + 32768);
    const uint64_t bd = desc_sw128(b0);
    long long t0 = clock64();
    for (int r = 0; r < reps; r += 4) {
      if constexpr (TS) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          asm volatile(
              "{.reg .pred p; setp.ne.b32 p, %6, 0;\n"
              "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %3, [%4], [%5], p;}" ::"r"(
                  tmem),
              "r"(tmem + 256 + 8 * i), "l"(bd + uint64_t(2 * i)), "r"(idesc), "r"(tmem + 384), "r"(tmem + 400),
              "r"(r + i));
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          asm volatile(
              "{.reg .pred p; setp.ne.b32 p, %6, 0;\n"
              "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%4], [%5], p;}" ::"r"(
                  tmem),
              "l"(desc_sw128(a0) + uint64_t(2 * i)), "l"(bd + uint64_t(2 * i)), "r"(idesc), "r"(tmem + 384),
              "r"(tmem + 400), "r"(r + i));
      }
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
  cudaFuncSetAttribute(bench<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(bench<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int reps = 8192;
  for (int ts = 0; ts < 2; ++ts)
    for (int n : {64, 128, 256}) {
      if (ts)
        bench<true><<<148, 128, 100 * 1024>>>(n, reps, d);
      else
        bench<false><<<148, 128, 100 * 1024>>>(n, reps, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long c = 0;
      cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
      printf("{\"kind\": \"mxf4\", \"a\": \"%s\", \"n\": %d, \"clk_per_mma\": %.1f, \"err\": \"%s\"}\n", ts ? "tmem" : "smem",
             n, double(c) / reps, cudaGetErrorString(e));
    }
  return 0;
}
