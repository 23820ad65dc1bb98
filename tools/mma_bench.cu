// mma_bench.cu — tcgen05.mma issue-rate micro-benchmark (B200, sm_100a).
// One CTA per SM; one thread issues R back-to-back MMAs on fixed operands (SS: A and B
// in shared memory; TS: A in tensor memory), commits, waits; clock64 around it.
// Prints cycles per MMA and the implied per-SM MAC rate for each (kind, N, mode).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

template <int KIND, int N, bool TS>
__global__ void __launch_bounds__(128, 1) bench(int reps, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u * (i & 3);
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
    // i8: D s32 (2<<4), A u8, B s8 (1<<10); f16 kind: D f32 (1<<4), A/B bf16 (1<<7, 1<<10)
    const uint32_t idesc = (KIND == 0 ? ((2u << 4) | (1u << 10)) : ((1u << 4) | (1u << 7) | (1u << 10))) |
                           (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint64_t ad = desc_sw128(su32(smem)), bd = desc_sw128(su32(smem + 16384));
    const uint32_t ta = tmem + 256;  // A operand columns for TS
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (KIND == 0) {
        if (TS)
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;}"
                       ::"r"(tmem), "r"(ta), "l"(bd), "r"(idesc), "r"(r));
        else
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}"
                       ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(r));
      } else {
        if (TS)
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;}"
                       ::"r"(tmem), "r"(ta), "l"(bd), "r"(idesc), "r"(r));
        else
          asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}"
                       ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(r));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(su32(&bar))
                 : "memory");
    long long t1 = clock64();
    cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int KIND, int N, bool TS>
void run(int sms) {
  const int reps = 8192;
  unsigned long long* d;
  cudaMalloc(&d, sms * sizeof(unsigned long long));
  auto k = bench<KIND, N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<sms, 128, 100 * 1024>>>(16, d);
  cudaDeviceSynchronize();
  k<<<sms, 128, 100 * 1024>>>(reps, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double kk = KIND == 0 ? 32 : 16;  // K per instruction
  const double cpm = mx / reps;
  printf("{\"kind\": \"%s\", \"N\": %d, \"mode\": \"%s\", \"clk_per_mma\": %.2f, \"macs_per_clk_per_sm\": %.0f, \"err\": \"%s\"}\n",
         KIND == 0 ? "i8" : "bf16", N, TS ? "TS" : "SS", cpm, 128.0 * N * kk / cpm, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0, 64, false>(sms);
  run<0, 64, true>(sms);
  run<0, 128, false>(sms);
  run<0, 128, true>(sms);
  run<0, 256, false>(sms);
  run<0, 256, true>(sms);
  run<1, 64, false>(sms);
  run<1, 128, false>(sms);
  run<1, 256, false>(sms);
  run<1, 256, true>(sms);
  return 0;
}
