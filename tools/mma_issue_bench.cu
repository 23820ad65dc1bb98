// mma_issue_bench.cu — cost of issuing tcgen05.mma (i8, A from TMEM, M=128, N=128)
// from one warp, for several code shapes of the issue loop (stage ring of 4 stages x
// 2 planes x 4 K-steps, like the conv kernel).  Prints cycles per MMA; the hardware
// floor at N=128 is 64 (tools/mma_bench.cu).
//   V0: lane 0 only, descriptor rebuilt per MMA (the conv kernel before this test)
//   V1: lane 0 only, 64-bit descriptor precomputed per stage, + constant per MMA
//   V2: whole warp runs the loop, one elect.sync per MMA, precomputed descriptors
//   V3: whole warp, ONE asm block per stage: elect once, 8 MMAs with PTX adds inside
//   V4: kind::mxf4 block-scaled, A from TMEM, whole warp, elect per 2 MMAs (K = 64 each):
//       the FP4 conv kernel's issue shape (clk per 128x128x64 MMA)
//   V5: V4 with A from shared memory (SS)
//   V6: V4 with B in 64-byte rows, SWIZZLE_64B (the FP4 conv kernel's B layout)
//   V7: V6 + a tcgen05.commit to a stage mbarrier after every stage (4 MMAs), as the
//       conv kernel does to release each stage; V8: commit every 2 stages
//   V9: V7 + tcgen05.fence::after_thread_sync before each stage's MMAs (as after a wait)
//   V10: V9 + the wait itself: mbarrier.try_wait.parity on an already-completed phase
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_issue_bench tools/mma_issue_bench.cu
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
constexpr int N = 128;
constexpr uint32_t kIdesc = (2u << 4) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t acc) {
  asm volatile("{.reg .pred p; setp.ne.b32 p, %3, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %4, p;}" ::"r"(d),
               "r"(a), "l"(b), "r"(acc), "n"(kIdesc));
}
__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{.reg .pred p, e; .reg .b32 x; elect.sync x|e, 0xffffffff; setp.ne.b32 p, %3, 0;"
      " @e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %4, p;}" ::"r"(d),
      "r"(a), "l"(b), "r"(acc), "n"(kIdesc));
}
// 8 MMAs of one stage (planes i = 0,1 at +0/+32 columns, K steps k at +8 columns / +32
// bytes = +2 in the descriptor), one elect
__device__ __forceinline__ void mma_stage8(uint32_t d, uint32_t a, uint64_t b, uint32_t acc0) {
  asm volatile(
      "{.reg .pred p, e; .reg .b32 x, a1; .reg .b64 b1;\n"
      "elect.sync x|e, 0xffffffff;\n"
      "setp.ne.b32 p, %3, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %4, p;\n"
      "add.u32 a1, %1, 8; add.u64 b1, %2, 2;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], b1, %4, 1;\n"
      "add.u32 a1, %1, 16; add.u64 b1, %2, 4;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], b1, %4, 1;\n"
      "add.u32 a1, %1, 24; add.u64 b1, %2, 6;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], b1, %4, 1;\n"
      "add.u32 a1, %1, 32;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], %2, %4, 1;\n"
      "add.u32 a1, %1, 40; add.u64 b1, %2, 2;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], b1, %4, 1;\n"
      "add.u32 a1, %1, 48; add.u64 b1, %2, 4;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], b1, %4, 1;\n"
      "add.u32 a1, %1, 56; add.u64 b1, %2, 6;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], b1, %4, 1;\n"
      "}" ::"r"(d),
      "r"(a), "l"(b), "r"(acc0), "n"(kIdesc));
}

__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;
  d |= uint64_t(512 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(4) << 61;
  return d;
}
constexpr uint32_t kIdescF4 = (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (1u << 23) | (uint32_t(128 >> 4) << 24);
__device__ __forceinline__ void mma2_f4_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t sfa, uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{.reg .pred p, e; .reg .b32 x, a1; .reg .b64 b1;\n"
      "elect.sync x|e, 0xffffffff;\n"
      "setp.ne.b32 p, %3, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %4, [%5], [%6], p;\n"
      "add.u32 a1, %1, 8; add.u64 b1, %2, 2;\n"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [a1], b1, %4, [%5], [%6], 1;\n"
      "}" ::"r"(d), "r"(a), "l"(b), "r"(acc), "n"(kIdescF4), "r"(sfa), "r"(sfb));
}
__device__ __forceinline__ void mma2_f4_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t sfa, uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{.reg .pred p, e; .reg .b32 x; .reg .b64 a1, b1;\n"
      "elect.sync x|e, 0xffffffff;\n"
      "setp.ne.b32 p, %3, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %4, [%5], [%6], p;\n"
      "add.u64 a1, %1, 2; add.u64 b1, %2, 2;\n"
      "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], a1, b1, %4, [%5], [%6], 1;\n"
      "}" ::"r"(d), "l"(a), "l"(b), "r"(acc), "n"(kIdescF4), "r"(sfa), "r"(sfb));
}

template <int V>
__global__ void __launch_bounds__(128, 1) bench(int stages, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint64_t sbar[4];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u * (i & 3);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&sbar[i])));
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
  const uint32_t sbase = su32(smem);
  if (warp == 1 && (V >= 2 || lane == 0)) {
    long long t0 = clock64();
    for (int st = 0; st < stages; ++st) {
      const int s = st & 3;
      const uint32_t acc = tmem + ((st >> 4) & 1) * N;
      const uint32_t a0 = tmem + 256 + s * 64;
      const uint32_t b0 = sbase + s * (N * 128);
      if (V == 0) {
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int k = 0; k < 4; ++k) mma_ts(acc, a0 + i * 32 + k * 8, desc_sw128(b0 + k * 32), (st | i | k) & 15);
      } else if (V == 1 || V == 2) {
        const uint64_t bd = desc_sw128(b0);
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (V == 1)
              mma_ts(acc, a0 + i * 32 + k * 8, bd + 2 * k, (st | i | k) & 15);
            else
              mma_ts_elect(acc, a0 + i * 32 + k * 8, bd + 2 * k, (st | i | k) & 15);
          }
      } else if (V == 3) {
        mma_stage8(acc, a0, desc_sw128(b0), st & 15);
      } else if (V == 4) {  // per stage: 2 planes x 2 K64 steps, SF regions at 448 / 480
        mma2_f4_ts(acc, a0, desc_sw128(b0), tmem + 448, tmem + 480, st & 15);
        mma2_f4_ts(acc, a0 + 16, desc_sw128(b0), tmem + 452, tmem + 480, 1);
      } else if (V >= 6) {
        if (V == 10) {
          asm volatile("{.reg .pred p; W%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 1; @!p bra W%=;}" ::"r"(
                           su32(&bar))
                       : "memory");
        }
        if (V >= 9) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        mma2_f4_ts(acc, a0, desc_sw64(b0), tmem + 448, tmem + 480, st & 15);
        mma2_f4_ts(acc, a0 + 16, desc_sw64(b0), tmem + 452, tmem + 480, 1);
        if (V == 7 || V >= 9 || (V == 8 && (st & 1)))
          asm volatile(
              "{.reg .pred e; .reg .b32 x; elect.sync x|e, 0xffffffff;\n"
              "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}" ::"r"(su32(&sbar[s]))
              : "memory");
      } else {
        mma2_f4_ss(acc, desc_sw128(b0 + 32768), desc_sw128(b0), tmem + 448, tmem + 480, st & 15);
        mma2_f4_ss(acc, desc_sw128(b0 + 32768 + 64), desc_sw128(b0), tmem + 452, tmem + 480, 1);
      }
    }
    if (lane == 0)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                   : "memory");
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(su32(&bar))
                 : "memory");
    long long t1 = clock64();
    if (lane == 0) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int V>
void run(int sms) {
  const int stages = 1024;
  unsigned long long* d;
  cudaMalloc(&d, sms * sizeof(unsigned long long));
  auto k = bench<V>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<sms, 128, 100 * 1024>>>(8, d);
  cudaDeviceSynchronize();
  k<<<sms, 128, 100 * 1024>>>(stages, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("{\"variant\": %d, \"N\": %d, \"clk_per_mma\": %.2f, \"err\": \"%s\"}\n", V, N,
         mx / (stages * (V >= 4 ? 4.0 : 8.0)), cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>(sms);
  run<1>(sms);
  run<2>(sms);
  run<3>(sms);
  run<4>(sms);
  run<5>(sms);
  run<6>(sms);
  run<7>(sms);
  run<8>(sms);
  run<9>(sms);
  run<10>(sms);
  return 0;
}
