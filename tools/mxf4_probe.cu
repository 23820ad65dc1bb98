// mxf4_probe.cu — does tcgen05.mma.kind::mxf4 (E2M1 x E2M1, UE8M0 block scales, f32
// accumulation) compute 0/1 binary dot products EXACTLY, and how fast?  (Design probe
// for an FP4 variant of the tensor-core bitserial kernel; not product code.)
// One CTA: A [128 x K] and B [N x K] packed E2M1 (2 per byte) in shared memory, K-major,
// 128B-swizzled; every scale factor in TMEM filled with one UE8M0 value.  Bits: A nibble
// 0b0001 (0.5) or 0, B nibble 0b0010 (+1.0) / 0b1010 (-1.0) (bipolar) ; scales 2^sa, 2^sb.
// Result D[m][n] = sum_k 0.5*a*2^sa * (+-1)*2^sb must equal the integer from the CPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mxf4_probe tools/mxf4_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 128;
constexpr int KC = 256;  // K elements per 128-byte swizzle row

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
// block-scaled idesc: a/b format E2M1 (=1 for kind::mxf4), scale UE8M0 (bit 23), K64
constexpr uint32_t kIdesc = (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (1u << 23) | (uint32_t(M >> 4) << 24);

// mode bits (probe2): 1 = A from TMEM (written with tcgen05.st, 8 elements per column,
// element 8c+e in nibble e of column c); 2 = scale factors only in ONE column per region
// (the next 15 columns hold a wrong scale); 4 = scales in byte lane `sfid` of the column
// (other byte lanes wrong) and idesc a_sf_id = b_sf_id = sfid.
template <int NN>
__global__ void probe2(const uint8_t* a_bits, const int8_t* b_val, int K, int sa, int sb, int mode, int sfid,
                       float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nkc = K / KC;
  uint8_t* sA = smem;
  uint8_t* sB = smem + nkc * M * 128;
  for (int idx = tid; idx < nkc * M * 128; idx += blockDim.x) {
    const int kc = idx / (M * 128), r = (idx / 128) % M, c = idx % 128;
    const int k0 = kc * KC + 2 * c;
    const uint8_t lo = a_bits[r * K + k0] ? 0x1 : 0x0, hi = a_bits[r * K + k0 + 1] ? 0x1 : 0x0;
    sA[kc * M * 128 + r * 128 + (((c >> 4) ^ (r & 7)) << 4) + (c & 15)] = uint8_t(lo | (hi << 4));
  }
  for (int idx = tid; idx < nkc * NN * 128; idx += blockDim.x) {
    const int kc = idx / (NN * 128), r = (idx / 128) % NN, c = idx % 128;
    const int k0 = kc * KC + 2 * c;
    auto enc = [](int8_t v) -> uint8_t { return v > 0 ? 0x2 : (v < 0 ? 0xA : 0x0); };
    sB[kc * NN * 128 + r * 128 + (((c >> 4) ^ (r & 7)) << 4) + (c & 15)] =
        uint8_t(enc(b_val[r * K + k0]) | (enc(b_val[r * K + k0 + 1]) << 4));
  }
  if (tid == 0) {
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
  const uint32_t lane_base = tmem + (uint32_t(warp * 32) << 16);
  // scale regions: A at column 256, B at 288; A operand (TS) at columns 320..
  {
    uint32_t good_a = 0x01010101u * uint32_t(127 + sa), good_b = 0x01010101u * uint32_t(127 + sb);
    const uint32_t bad = 0x01010101u * uint32_t(127 + 9);
    if (mode & 4) {  // only byte lane sfid correct
      const uint32_t m8 = 0xFFu << (8 * sfid);
      good_a = (good_a & m8) | (bad & ~m8);
      good_b = (good_b & m8) | (bad & ~m8);
    }
    for (int c = 0; c < 32; ++c) {
      const bool first = c < sfid;  // mode 2: the first `sfid` columns correct
      const uint32_t va = (mode & 2) && !first ? bad : good_a, vb = (mode & 2) && !first ? bad : good_b;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(lane_base + 256 + c), "r"(va) : "memory");
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(lane_base + 288 + c), "r"(vb) : "memory");
    }
    if (mode & 1) {  // A rows into TMEM: row = lane of this warp's quarter
      const int r = warp * 32 + lane;
      for (int c = 0; c < K / 8; ++c) {
        uint32_t w = 0;
        for (int e = 0; e < 8; ++e) w |= uint32_t(a_bits[r * K + 8 * c + e] ? 1 : 0) << (4 * e);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(lane_base + 320 + c), "r"(w) : "memory");
      }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t idesc = (1u << 7) | (1u << 10) | (uint32_t(NN >> 3) << 17) | (1u << 23) | (uint32_t(M >> 4) << 24) |
                         ((mode & 4) ? ((uint32_t(sfid) << 4) | (uint32_t(sfid) << 29)) : 0u);
  if (tid == 0) {
    for (int kc = 0; kc < nkc; ++kc)
      for (int k = 0; k < 4; ++k) {
        const uint64_t bd = desc_sw128(su32(sB + kc * NN * 128) + k * 32);
        const uint32_t acc = (kc | k) != 0;
        if (mode & 1) {
          const uint32_t ta = tmem + 320 + (kc * 4 + k) * 8;
          asm volatile(
              "{.reg .pred p; setp.ne.b32 p, %4, 0;"
              " tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %3, [%5], [%6], p;}" ::"r"(
                  tmem),
              "r"(ta), "l"(bd), "r"(idesc), "r"(acc), "r"(tmem + 256), "r"(tmem + 288));
        } else {
          const uint64_t ad = desc_sw128(su32(sA + kc * M * 128) + k * 32);
          asm volatile(
              "{.reg .pred p; setp.ne.b32 p, %4, 0;"
              " tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;}" ::"r"(
                  tmem),
              "l"(ad), "l"(bd), "r"(idesc), "r"(acc), "r"(tmem + 256), "r"(tmem + 288));
        }
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(su32(&bar))
                 : "memory");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    for (int c0 = 0; c0 < NN; c0 += 32) {
      uint32_t r[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(tmem + (uint32_t(warp * 32) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      const int row = warp * 32 + lane;
      for (int c = 0; c < 32; ++c) out[row * NN + c0 + c] = __uint_as_float(r[c]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int NN>
int run2(int mode, int sfid) {
  const int K = 512, sa = 2, sb = 1;
  std::vector<uint8_t> a(size_t(M) * K);
  std::vector<int8_t> b(size_t(NN) * K);
  srand(mode * 31 + sfid + NN);
  for (auto& x : a) x = rand() & 1;
  for (auto& x : b) x = (rand() & 1) ? 1 : -1;
  uint8_t* da; int8_t* db; float* dout;
  cudaMalloc(&da, a.size()); cudaMalloc(&db, b.size()); cudaMalloc(&dout, M * NN * 4);
  cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice);
  const int smem = (K / KC) * (M + NN) * 128 + 1024;
  cudaFuncSetAttribute(probe2<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe2<NN><<<1, 128, smem>>>(da, db, K, sa, sb, mode, sfid, dout);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> out(M * NN);
  cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
  long long bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < NN; ++n) {
      long long s = 0;
      for (int k = 0; k < K; ++k) s += (long long)a[size_t(m) * K + k] * b[size_t(n) * K + k];
      const long long want = s * (1ll << (sa + sb)) / 2;
      if ((double)out[m * NN + n] != (double)want) {
        if (bad < 2) printf("  mismatch m=%d n=%d got %.1f want %lld\n", m, n, out[m * NN + n], want);
        ++bad;
      }
    }
  printf("{\"probe2\": 1, \"N\": %d, \"mode\": %d, \"sfid\": %d, \"mismatches\": %lld, \"err\": \"%s\"}\n", NN, mode,
         sfid, bad, cudaGetErrorString(e));
  cudaFree(da); cudaFree(db); cudaFree(dout);
  return bad != 0 || e != cudaSuccess;
}

// a_bits: [M][K] 0/1 bytes; b_sign: [N][K] +1/-1/0 (0 = zero element)
__global__ void probe(const uint8_t* a_bits, const int8_t* b_val, int K, int sa, int sb, int reps, float* out,
                      unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int nkc = K / KC;
  uint8_t* sA = smem;                       // nkc x [128 rows x 128 B]
  uint8_t* sB = smem + nkc * M * 128;       // nkc x [N rows x 128 B]
  // pack + swizzle: row r, byte c (elements 2c, 2c+1) -> chunk (c/16) ^ (r&7)
  for (int idx = tid; idx < nkc * M * 128; idx += blockDim.x) {
    const int kc = idx / (M * 128), r = (idx / 128) % M, c = idx % 128;
    const int k0 = kc * KC + 2 * c;
    const uint8_t lo = a_bits[r * K + k0] ? 0x1 : 0x0, hi = a_bits[r * K + k0 + 1] ? 0x1 : 0x0;
    sA[kc * M * 128 + r * 128 + (((c >> 4) ^ (r & 7)) << 4) + (c & 15)] = uint8_t(lo | (hi << 4));
  }
  for (int idx = tid; idx < nkc * N * 128; idx += blockDim.x) {
    const int kc = idx / (N * 128), r = (idx / 128) % N, c = idx % 128;
    const int k0 = kc * KC + 2 * c;
    auto enc = [](int8_t v) -> uint8_t { return v > 0 ? 0x2 : (v < 0 ? 0xA : 0x0); };
    sB[kc * N * 128 + r * 128 + (((c >> 4) ^ (r & 7)) << 4) + (c & 15)] =
        uint8_t(enc(b_val[r * K + k0]) | (enc(b_val[r * K + k0 + 1]) << 4));
  }
  if (tid == 0) {
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
  // scale factors: columns 256..271 (A), 272..287 (B), every byte = UE8M0 (127 + s)
  {
    const uint32_t va = 0x01010101u * uint32_t(127 + sa), vb = 0x01010101u * uint32_t(127 + sb);
    const uint32_t lane_base = tmem + (uint32_t(warp * 32) << 16);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};"
                 ::"r"(lane_base + 256), "r"(va) : "memory");
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};"
                 ::"r"(lane_base + 272), "r"(vb) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
      for (int kc = 0; kc < nkc; ++kc)
        for (int k = 0; k < 4; ++k) {  // 4 x K64 per 128-byte row
          const uint64_t ad = desc_sw128(su32(sA + kc * M * 128) + k * 32);
          const uint64_t bd = desc_sw128(su32(sB + kc * N * 128) + k * 32);
          const uint32_t acc = (r | kc | k) != 0;
          asm volatile(
              "{.reg .pred p; setp.ne.b32 p, %4, 0;"
              " tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;}" ::"r"(
                  tmem),
              "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc), "r"(tmem + 256), "r"(tmem + 272));
        }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
    asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0; @!p bra W;}" ::"r"(su32(&bar))
                 : "memory");
    *cyc = (unsigned long long)(clock64() - t0);
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    for (int c0 = 0; c0 < N; c0 += 32) {
      uint32_t r[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(tmem + (uint32_t(warp * 32) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      const int row = warp * 32 + (tid & 31);
      for (int c = 0; c < 32; ++c) out[row * N + c0 + c] = __uint_as_float(r[c]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main(int argc, char** argv) {
  int fails = 0;
  struct Case { int K, sa, sb, ones, reps; };
  // ones: 0 random bits/signs; 1 all ones; 2 A ones, B +1 on the first half of K and random signs on
  // the rest (large running sum plus odd small increments: tests the accumulator's low bits)
  Case cases[] = {{256, 1, 0, 0, 1}, {1024, 1, 0, 0, 1}, {1024, 2, 1, 0, 1}, {1024, 4, 1, 0, 1}, {1024, 1, 0, 1, 1},
                  {1024, 4, 2, 1, 8}, {1024, 4, 2, 1, 24}, {1024, 1, 0, 2, 600}, {1024, 2, 0, 2, 700},
                  {1024, 1, 0, 0, 400}};
  for (const Case& cs : cases) {
    const int K = cs.K;
    std::vector<uint8_t> a(size_t(M) * K);
    std::vector<int8_t> b(size_t(N) * K);
    srand(K * 7 + cs.sa);
    for (auto& x : a) x = cs.ones ? 1 : (rand() & 1);
    for (size_t i = 0; i < b.size(); ++i)
      b[i] = cs.ones == 1 ? 1 : (cs.ones == 2 && int(i % K) < K / 2) ? 1 : ((rand() & 1) ? 1 : -1);
    uint8_t* da; int8_t* db; float* dout; unsigned long long* dc;
    cudaMalloc(&da, a.size()); cudaMalloc(&db, b.size()); cudaMalloc(&dout, M * N * 4); cudaMalloc(&dc, 8);
    cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice);
    const int smem = (K / KC) * (M + N) * 128 + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<<<1, 128, smem>>>(da, db, K, cs.sa, cs.sb, cs.reps, dout, dc);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> out(M * N);
    unsigned long long cyc = 0;
    cudaMemcpy(out.data(), dout, M * N * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    long long bad = 0, maxabs = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        long long s = 0;
        for (int k = 0; k < K; ++k) s += (long long)a[size_t(m) * K + k] * b[size_t(n) * K + k];
        // value = reps * s * 0.5 * 2^sa * 2^sb  (A element 0.5, B element +-1)
        const long long want = (long long)cs.reps * s * (1ll << (cs.sa + cs.sb)) / 2;
        maxabs = llabs(want) > maxabs ? llabs(want) : maxabs;
        if ((double)out[m * N + n] != (double)want) {
          if (bad < 3) printf("  mismatch m=%d n=%d got %.1f want %lld\n", m, n, out[m * N + n], want);
          ++bad;
        }
      }
    const double mmas = double(cs.reps) * (K / 64);
    printf("{\"K\": %d, \"sa\": %d, \"sb\": %d, \"ones\": %d, \"reps\": %d, \"max_abs\": %lld, \"mismatches\": %lld, "
           "\"clk_per_mma_k64\": %.1f, \"err\": \"%s\"}\n",
           K, cs.sa, cs.sb, cs.ones, cs.reps, maxabs, bad, cyc / mmas, cudaGetErrorString(e));
    fails += bad != 0 || e != cudaSuccess;
    cudaFree(da); cudaFree(db); cudaFree(dout); cudaFree(dc);
  }
  for (int mode : {0, 1}) {
    fails += run2<64>(mode, 0);
    fails += run2<128>(mode, 0);
    fails += run2<256>(mode, 0);
  }
  for (int ncols : {1, 2, 3, 4, 8, 16}) {  // mode 2: how many scale columns one MMA reads
    fails += run2<64>(2, ncols);
    fails += run2<128>(2, ncols);
    fails += run2<256>(2, ncols);
  }
  return fails ? 1 : 0;
}
