// Integer-pipe micro-benchmarks for the bitserial roofline (SURVEY §7 phase 1, §8d).
//
// Measures, per SM per SM-clock, the issue rate of the SASS instructions the
// bitserial inner loop is made of (Eq. 1/2: AND + popcount +
// weighted accumulate): POPC, LOP3, IADD3, IMAD, and mixes of them, so that the
// roofline the bench reports against is measured on this B200, not assumed.
//
// Each kernel runs NCH independent dependency chains per thread so the result is
// throughput-bound, one full wave of CTAs, and reads %clock64 + %globaltimer in
// every CTA to report the SM clock the run actually saw.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo tools/pipe_bench.cu -o tools/pipe_bench
// Output: one JSON object on stdout.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int NCH = 16;   // independent chains per thread
constexpr int UNR = 8;    // unrolled rounds per loop iteration

struct Stamp { unsigned long long c0, c1, t0, t1; };

// op ids
enum { OP_POPC = 0, OP_LOP3, OP_IADD3, OP_IMAD, OP_AND_POPC_ADD, OP_POPC_LOP3_1_1,
       OP_POPC_LOP3_1_3, OP_CSA_3_2, OP_FLO, OP_PRMT, OP_NUM };
static const char* kOpName[OP_NUM] = {
  "popc", "lop3", "iadd3", "imad", "and_popc_add", "popc+lop3(1:1)", "popc+lop3(1:3)",
  "popc+imad(1:1)", "flo", "prmt"};
// source instructions (per chain per round) we expect ptxas to emit, checked in SASS
static const int kInstPerRound[OP_NUM] = {1, 1, 1, 1, 3, 2, 4, 2, 1, 1};

template <int OP>
__global__ void __launch_bounds__(512) pipe_kernel(uint32_t* sink, Stamp* st, int iters, uint32_t seed) {
  uint32_t r[NCH], q[NCH];
#pragma unroll
  for (int i = 0; i < NCH; ++i) { r[i] = seed * (threadIdx.x + 3 * i + 1); q[i] = seed ^ (i * 0x9e3779b9u + threadIdx.x); }
  unsigned long long c0 = clock64(), t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
#pragma unroll
      for (int i = 0; i < NCH; ++i) {
        if constexpr (OP == OP_POPC) {
          asm volatile("popc.b32 %0, %0;" : "+r"(r[i]));
        } else if constexpr (OP == OP_LOP3) {
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[i]) : "r"(q[i]), "r"(q[(i + 1) % NCH]));
        } else if constexpr (OP == OP_IADD3) {
          asm volatile("{ .reg .u32 t; add.u32 t, %1, %2; add.u32 %0, %0, t; }" : "+r"(r[i]) : "r"(q[i]), "r"(q[(i + 1) % NCH]));
        } else if constexpr (OP == OP_IMAD) {
          asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[i]) : "r"(q[i]), "r"(q[(i + 1) % NCH]));
        } else if constexpr (OP == OP_AND_POPC_ADD) {
          // r += popc(q_i & q_{i+1}): the literal Eq. 1 step
          asm volatile("{ .reg .u32 t; and.b32 t, %1, %2; popc.b32 t, t; add.u32 %0, %0, t; }"
                       : "+r"(r[i]) : "r"(q[i]), "r"(q[(i + 1) % NCH] ^ r[i]));
        } else if constexpr (OP == OP_POPC_LOP3_1_1) {
          asm volatile("{ popc.b32 %0, %0; lop3.b32 %1, %1, %2, %0, 0x96; }" : "+r"(r[i]), "+r"(q[i]) : "r"(q[(i + 1) % NCH]));
        } else if constexpr (OP == OP_POPC_LOP3_1_3) {
          asm volatile("{ popc.b32 %0, %0; lop3.b32 %1, %1, %2, %0, 0x96; lop3.b32 %1, %1, %2, %0, 0xe8; lop3.b32 %1, %1, %2, %0, 0x1e;}"
                       : "+r"(r[i]), "+r"(q[i]) : "r"(q[(i + 1) % NCH]));
        } else if constexpr (OP == OP_CSA_3_2) {
          asm volatile("{ popc.b32 %0, %0; mad.lo.u32 %1, %1, %2, %0; }" : "+r"(r[i]), "+r"(q[i]) : "r"(q[(i + 1) % NCH]));
        } else if constexpr (OP == OP_FLO) {
          asm volatile("bfind.u32 %0, %0;" : "+r"(r[i]));
        } else if constexpr (OP == OP_PRMT) {
          asm volatile("prmt.b32 %0, %0, %1, 0x3210;" : "+r"(r[i]) : "r"(q[i]));
        }
      }
    }
  }
  unsigned long long c1 = clock64(), t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) acc += r[i] + q[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) st[blockIdx.x] = Stamp{c0, c1, t0, t1};
}

template <int OP>
static void run(int sms, int blocks_per_sm, int threads, int iters, bool last) {
  int grid = sms * blocks_per_sm;
  uint32_t* sink; Stamp* st;
  CK(cudaMalloc(&sink, sizeof(uint32_t) * grid * threads));
  CK(cudaMalloc(&st, sizeof(Stamp) * grid));
  pipe_kernel<OP><<<grid, threads>>>(sink, st, 2, 12345u);  // warm-up
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  pipe_kernel<OP><<<grid, threads>>>(sink, st, iters, 12345u);
  CK(cudaEventRecord(e1));
  CK(cudaDeviceSynchronize());
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  Stamp* h = (Stamp*)malloc(sizeof(Stamp) * grid);
  CK(cudaMemcpy(h, st, sizeof(Stamp) * grid, cudaMemcpyDeviceToHost));
  double cyc_sum = 0, ns_sum = 0, cyc_max = 0;
  for (int b = 0; b < grid; ++b) {
    double c = double(h[b].c1 - h[b].c0), t = double(h[b].t1 - h[b].t0);
    cyc_sum += c; ns_sum += t; if (c > cyc_max) cyc_max = c;
  }
  double mhz = cyc_sum / ns_sum * 1e3;
  // lane-ops per SM per clock, counted in source ops (one per chain per round)
  double lane_ops = double(grid) * threads * double(iters) * UNR * NCH;
  double per_sm_clk = lane_ops / (cyc_max * sms);
  printf("  {\"op\": \"%s\", \"src_ops_per_round\": %d, \"threads\": %d, \"blocks_per_sm\": %d, "
         "\"lane_ops_per_clk_per_sm\": %.2f, \"sm_mhz\": %.0f, \"kernel_ms\": %.3f}%s\n",
         kOpName[OP], kInstPerRound[OP], threads, blocks_per_sm, per_sm_clk, mhz, ms, last ? "" : ",");
  free(h); CK(cudaFree(sink)); CK(cudaFree(st));
}

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  int iters = argc > 1 ? atoi(argv[1]) : 4000;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\", \"l2_bytes\": %d, \"results\": [\n",
         p.name, sms, p.major, p.minor, p.l2CacheSize);
  run<OP_POPC>(sms, 2, 512, iters, false);
  run<OP_LOP3>(sms, 2, 512, iters, false);
  run<OP_IADD3>(sms, 2, 512, iters, false);
  run<OP_IMAD>(sms, 2, 512, iters, false);
  run<OP_AND_POPC_ADD>(sms, 2, 512, iters, false);
  run<OP_POPC_LOP3_1_1>(sms, 2, 512, iters, false);
  run<OP_POPC_LOP3_1_3>(sms, 2, 512, iters, false);
  run<OP_CSA_3_2>(sms, 2, 512, iters, false);
  run<OP_FLO>(sms, 2, 512, iters, false);
  run<OP_PRMT>(sms, 2, 512, iters, false);
  run<OP_POPC>(sms, 1, 256, iters, true);
  printf("]}\n");
  return 0;
}
