// store_bench.cu — output-drain micro-benchmark for the tensor-core conv epilogue (B200).
// A persistent grid (one CTA per SM) writes an int32 [M][OC] matrix tile by tile (128-row
// tiles, BN columns), the way tc_conv_kernel's epilogue warps do, with the per-box data
// optionally read from tensor memory (tcgen05.ld 32x32b.x32) first.  Variants:
//   mode 0  TMA store of 32x32 int32 boxes (128B swizzle), EW warps, NBUF staging buffers
//   mode 1  smem-staged, coalesced st.global.v4 (each warp instruction = 4 full 128B lines)
//   mode 2  direct st.global.v4 from registers, lane = row (8 partial-line stores per lane)
//   mode 3  TMA store of 32 rows x BN columns per warp (3-D box {32, BN/32, 32}, 128B swizzle)
//   plain   grid-stride st.global.v4 over the whole buffer (reference copy-free write rate)
// Prints one JSON line per variant (GB/s, best of trials, CUDA events).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/store_bench tools/store_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int MODE, int EW, int NBUF, int BN>
__global__ void __launch_bounds__(EW * 32 + 32, 1)
    store_kernel(const __grid_constant__ CUtensorMap map, int32_t* out, int M, int oc, int ntiles, int use_tmem) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == EW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (warp < EW) {
    const int q = warp & 3, cb0 = warp >> 2;
    constexpr int kStep = EW / 4;
    constexpr int kBox = MODE == 3 ? 32 * BN * 4 : 4096;
    uint8_t* ebuf = smem + warp * NBUF * kBox;
    const int ntn = oc / BN;
    int buf = 0, it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int m0 = (t / ntn) * 128, n0 = (t % ntn) * BN;
      const int row = m0 + q * 32 + lane;
      if (MODE == 3) {  // one 32 x BN box per warp (warps beyond 4 idle)
        if (cb0 != 0) continue;
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NBUF - 1) : "memory");
        __syncwarp();
        uint8_t* sb = ebuf + buf * kBox;
        for (int cb = 0; cb < BN / 32; ++cb) {
          uint32_t r[32];
          if (use_tmem)
            tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t((it & 1) * BN + cb * 32), r);
          else
#pragma unroll
            for (int c = 0; c < 32; ++c) r[c] = row * 7 + c + cb;
          const uint32_t line = uint32_t(lane * (BN / 32) + cb);  // 128-byte line index in the box
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<uint4*>(sb + line * 128 + ((uint32_t(c) ^ (line & 7)) << 4)) =
                make_uint4(r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          asm volatile(
              "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                  reinterpret_cast<uint64_t>(&map)),
              "r"(0), "r"(n0 / 32), "r"(m0 + q * 32), "r"(su32(sb))
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        buf = buf + 1 == NBUF ? 0 : buf + 1;
        continue;
      }
      for (int cb = cb0; cb < BN / 32; cb += kStep) {
        uint32_t r[32];
        if (use_tmem)
          tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t((it & 1) * BN + cb * 32), r);
        else
#pragma unroll
          for (int c = 0; c < 32; ++c) r[c] = row * 7 + c + cb;
        if (MODE == 2) {
          uint4* dst = reinterpret_cast<uint4*>(out + int64_t(row) * oc + n0 + cb * 32);
#pragma unroll
          for (int c = 0; c < 8; ++c) dst[c] = make_uint4(r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);
          continue;
        }
        if (MODE == 0 && lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NBUF - 1) : "memory");
        __syncwarp();
        uint8_t* sb = ebuf + buf * kBox + lane * 128;
        const uint32_t swz = uint32_t(lane & 7);
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint4*>(sb + ((uint32_t(c) ^ swz) << 4)) =
              make_uint4(r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);
        if (MODE == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                    reinterpret_cast<uint64_t>(&map)),
                "r"(n0 + cb * 32), "r"(m0 + q * 32), "r"(su32(ebuf + buf * kBox))
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        } else {  // MODE 1: coalesced re-read of the staged box, 4 rows x 128 B per instruction
          __syncwarp();
          const uint8_t* b0 = ebuf + buf * kBox;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = i * 4 + (lane >> 3), ch = lane & 7;
            const uint4 v = *reinterpret_cast<const uint4*>(b0 + rr * 128 + ((ch ^ (rr & 7)) << 4));
            *reinterpret_cast<uint4*>(out + int64_t(m0 + q * 32 + rr) * oc + n0 + cb * 32 + ch * 4) = v;
          }
          __syncwarp();
        }
        buf = buf + 1 == NBUF ? 0 : buf + 1;
      }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == EW) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

__global__ void plain_write(uint4* out, int64_t n16) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n16; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = make_uint4(uint32_t(i), 1u, 2u, 3u);
}

static bool encode(CUtensorMap* m, void* base, int M, int oc, int mode, int bn) {
  if (mode == 3) {
    const cuuint64_t dims[3] = {32, cuuint64_t(oc / 32), cuuint64_t(M)};
    const cuuint64_t strides[2] = {128, cuuint64_t(oc) * 4};
    const cuuint32_t box[3] = {32, cuuint32_t(bn / 32), 32};
    const cuuint32_t es[3] = {1, 1, 1};
    return cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_INT32, 3, base, dims, strides, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  const cuuint64_t dims[2] = {cuuint64_t(oc), cuuint64_t(M)};
  const cuuint64_t strides[1] = {cuuint64_t(oc) * 4};
  const cuuint32_t box[2] = {32, 32};
  const cuuint32_t es[2] = {1, 1};
  return cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, base, dims, strides, box, es,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int MODE, int EW, int NBUF, int BN>
void run(int32_t* out, int M, int oc, int sms, int use_tmem) {
  CUtensorMap map;
  if (!encode(&map, out, M, oc, MODE, BN)) {
    printf("{\"error\": \"encode\"}\n");
    return;
  }
  auto k = store_kernel<MODE, EW, NBUF, BN>;
  const int box = MODE == 3 ? 32 * BN * 4 : 4096;
  const int smem = 1024 + EW * NBUF * box;
  const int ntiles = (M / 128) * (oc / BN);
  const int grid = sms;
  int smem_launch = smem < 116 * 1024 ? 116 * 1024 : smem;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_launch);
  k<<<grid, EW * 32 + 32, smem_launch>>>(map, out, M, oc, ntiles, use_tmem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int tr = 0; tr < 5; ++tr) {
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k<<<grid, EW * 32 + 32, smem_launch>>>(map, out, M, oc, ntiles, use_tmem);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms / 5 < best ? ms / 5 : best;
  }
  const double bytes = double(M) * oc * 4;
  printf("{\"mode\": %d, \"ew\": %d, \"nbuf\": %d, \"bn\": %d, \"oc\": %d, \"tmem\": %d, \"us\": %.2f, \"gbs\": %.0f, \"err\": \"%s\"}\n",
         MODE, EW, NBUF, BN, oc, use_tmem, best * 1e3, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int M = 802816;
  int32_t* out;
  cudaMalloc(&out, size_t(M) * 256 * 4);
  {
    const int64_t n16 = int64_t(M) * 128 * 4 / 16;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    plain_write<<<sms * 8, 256>>>(reinterpret_cast<uint4*>(out), n16);
    float best = 1e30f;
    for (int tr = 0; tr < 5; ++tr) {
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) plain_write<<<sms * 8, 256>>>(reinterpret_cast<uint4*>(out), n16);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms / 5 < best ? ms / 5 : best;
    }
    printf("{\"mode\": \"plain\", \"us\": %.2f, \"gbs\": %.0f}\n", best * 1e3, n16 * 16.0 / best / 1e6);
  }
  for (int tm = 0; tm < 2; ++tm) {
    for (int oc : {128, 64, 256}) {
      if (oc == 64) {
        run<0, 8, 2, 64>(out, M, oc, sms, tm);
        run<0, 4, 4, 64>(out, M, oc, sms, tm);
        run<1, 8, 2, 64>(out, M, oc, sms, tm);
        run<2, 8, 2, 64>(out, M, oc, sms, tm);
        run<3, 4, 2, 64>(out, M, oc, sms, tm);
        run<3, 4, 4, 64>(out, M, oc, sms, tm);
      } else {
        run<0, 8, 2, 128>(out, M, oc, sms, tm);
        run<0, 8, 4, 128>(out, M, oc, sms, tm);
        run<0, 4, 4, 128>(out, M, oc, sms, tm);
        run<0, 16, 2, 128>(out, M, oc, sms, tm);
        run<1, 8, 2, 128>(out, M, oc, sms, tm);
        run<1, 16, 2, 128>(out, M, oc, sms, tm);
        run<2, 8, 2, 128>(out, M, oc, sms, tm);
        run<3, 4, 2, 128>(out, M, oc, sms, tm);
        run<3, 4, 3, 128>(out, M, oc, sms, tm);
      }
    }
  }
  return 0;
}
