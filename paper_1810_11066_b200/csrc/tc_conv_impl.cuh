#pragma once
// tc_conv_impl.cuh — bitserial conv2d / dense on the 5th-generation tensor cores (tcgen05):
// the kernel template and its launch templates, shared by tc_conv.cu (prepared-weight single
// launches, weight expansion), tc_conv_group.cu (grouped launches) and tc_conv_raw.cu
// (packed-weight launches) so the three compile in parallel.
//
// Original header of tc_conv.cu:
//
// Eq. 2: out = sum_{i<A} sum_{j<W} 2^(i+j) * popcount(a_i AND w_j).
// For 0/1 vectors popcount(a_i AND w_j) = sum_k a_i[k] * w_j[k] (Eq. 1),
// a dense contraction, so every plane pair (i, j) is one binary dot product that the
// tensor core evaluates exactly in int8 x int8 -> int32:
//   * activation plane i is expanded from its packed uint32 words into bytes 2^i * a_i
//     (u8) inside shared memory — operands stay bit-packed in HBM (A/8 bytes per
//     element, the point of bit-packing);
//   * weight plane j is expanded once, ahead of time like the weight packing itself
//     (PAPER.md:715), into bytes 2^j * b_j (unipolar) or 2^j * (2 b_j - 1) (bipolar:
//     each weight bit-plane a +/-1 digit, reading R2);
//   * the A*W plane-pair products accumulate into one TMEM int32 accumulator with
//     tcgen05.mma.kind::i8 (bipolar needs no correction term in this form).
// The cost still grows with A*W (one MMA per plane pair): this is the
// bitserial method with its binary dot products on the tensor cores instead of the
// integer pipes.
//
// Kernel structure (persistent, warp-specialized, one CTA per SM, (4T + 6) warps):
//   warps 0..4T-1  expansion producers: T teams (T = 4) of 4 warps, one thread per output
//               row; team t expands the chunks g = t, t+T, ... of the CTA's (tile, K chunk)
//               sequence (T chunks in flight hide the per-chunk latency chain).  Implicit
//               im2col gather of the packed words with zero padding
//               through a thread-private cp.async ring; expansion to bytes in registers;
//               tcgen05.st straight into the stage's A operand in TENSOR memory (lane =
//               output row, 4 bytes per column); one arrive per warp on full_a.
//   warps 4T..4T+3 epilogue: TMEM (double-buffered accumulators, 2*BN columns) ->
//               tcgen05.ld 32x32b.x32 -> swizzled smem -> TMA store of 32x32 int32
//               boxes (clipped at ragged M / OC), overlapping the next tile's main loop.
//   warp 4T+4   TMA producer: expanded weight tile [W planes][BN rows][128 B] per stage
//               (cp.async.bulk.tensor, SWIZZLE_128B) onto full_b — or, when all of OC fits
//               one tile and all of K fits shared memory, the whole B once (resident).
//   warp 4T+5   MMA issuer: the whole warp walks the loop (warp-uniform operands), one
//               elected lane issues A*W*4 tcgen05.mma.kind::i8 (A from TMEM, B from smem,
//               K = 32 bytes each) per stage; tcgen05.commit frees the stage; the last
//               chunk of a tile commits to acc_full.
// Measured design points (profiles/r01d_*): the MMA warp's instruction count per MMA
// matters because it shares an SM sub-partition with ALU-bound producers; the producers
// are latency-bound (4 teams beat 2); the TMA-store epilogue beats direct stores.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace bs {
namespace tc {

constexpr int BM = 128;                   // UMMA M (cta_group::1): output rows per tile
constexpr int BKB = 128;                  // B bytes per row per plane per stage = one 128B swizzle row
// packed words per plane per row in one stage (K chunk): I8 4 (32 bytes per word),
// FP4 8 (16 bytes per word: a 256-element chunk, so each stage's fixed producer / MMA-issue
// cost is spread over four K=64 MMAs per digit pair)
constexpr int chunk_words(bool f4) { return f4 ? 8 : 4; }
#ifndef BS_TC_TEAMS
#define BS_TC_TEAMS 4
#endif
constexpr int kTeams = BS_TC_TEAMS;                    // producer teams (K chunks in flight)
constexpr int kProducerWarps = 4 * kTeams;             // a team = 4 warps = one thread per row
constexpr int kProducerThreads = kProducerWarps * 32;
constexpr int kBarBytes = 1024;  // mbarriers (2 per A stage, 2 per B slot, 4) and the TMEM address slot
#ifndef BS_TC_MAX_STAGES
#define BS_TC_MAX_STAGES 8
#endif
#ifndef BS_TC_EPI_WARPS
#define BS_TC_EPI_WARPS 8
#endif
constexpr int kEpiWarps = BS_TC_EPI_WARPS;              // 4 or 8 (warp % 4 = lane quarter)
constexpr int kEpiWarp0 = kProducerWarps;

constexpr int kTmaWarp = kProducerWarps + kEpiWarps;
constexpr int kMmaWarp = kProducerWarps + kEpiWarps + 1;
constexpr int kThreads = (kProducerWarps + kEpiWarps + 2) * 32;
constexpr int kEpiBufBytes = 32 * 128;  // one 32 x 32 int32 box
#ifndef BS_TC_EPI_BUFS
#define BS_TC_EPI_BUFS 2
#endif
constexpr int kEpiBufs = BS_TC_EPI_BUFS;  // staging buffers (TMA stores in flight) per epilogue warp
constexpr int kEpiBytes = kEpiWarps * kEpiBufs * kEpiBufBytes;
constexpr int kSmemLimit = 226 * 1024;  // dynamic shared memory (the kernel also has 1 KB static)
constexpr int kMinSmem = 116 * 1024;  // > half the SM: guarantees one CTA per SM (TMEM)
constexpr int kMaxTaps = 64;          // filter taps held in the shared-memory tap table
constexpr int kGroupMax = 16;         // problems in one grouped launch
constexpr int kMaxPeers = 8;          // extra destinations of a fused all-gather epilogue

// BS_TC_PROFILE builds (tools only) count cycles spent in each role's waits and print
// them per CTA 0 at exit; the product build compiles these to nothing.
#ifdef BS_TC_PROFILE
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#ifdef BS_TC_STAMP  // timeline printfs (they delay the warps that print: relative use only)
#define STAMP(name)                                                          \
  do {                                                                       \
    if (blockIdx.x == 0) printf("TCSTAMP %s warp %d t %llu\n", name, warp, gtime()); \
  } while (0);
#else
#define STAMP(name) \
  do {                \
  } while (0);
#endif
#define PROF_DECL long long _pt = 0, _pacc[7] = {0, 0, 0, 0, 0, 0, 0};
#define PROF_BEGIN _pt = clock64();
#define PROF_END(i) _pacc[i] += clock64() - _pt;
#else
#define STAMP(name) \
  do {                \
  } while (0);
#define PROF_DECL
#define PROF_BEGIN
#define PROF_END(i)
#endif

// ------------------------------------------------------------------ PTX wrappers
// Activation gathers allocate in L1: consecutive K chunks (filter taps) of a tile re-read
// mostly the same pixels (measured 4% faster over the ResNet layers than L1::no_allocate)
#ifndef BS_TC_LDG_HINT
#define BS_TC_LDG_HINT ""
#endif
__device__ __forceinline__ uint4 ldg_nc_v4(const uint32_t* p) {
  uint4 v;
  asm volatile("ld.global.nc" BS_TC_LDG_HINT ".v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ uint2 ldg_nc_v2(const uint32_t* p) {
  uint2 v;
  asm volatile("ld.global.nc" BS_TC_LDG_HINT ".v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void mbar_init(uint32_t addr, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count));
}
// try_wait with a suspend-time hint: a waiting warp sleeps until the phase completes
// (or the hint elapses) instead of re-issuing the probe — without it the producers'
// stage waits were ~20% of all issued instructions, taken from the MMA / epilogue warps
// that share their SM sub-partitions.
#ifndef BS_TC_SUSPEND_NS
#define BS_TC_SUSPEND_NS 20000
#endif
__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity), "n"(BS_TC_SUSPEND_NS)
      : "memory");
}
// Wait with a sleeping back-off (roles that are not on the MMA's critical path: producers
// waiting for a free stage, epilogue warps waiting for an accumulator): one probe, then
// probes separated by __nanosleep, so a waiting warp stops taking issue slots from the
// warps that share its scheduler (ncu: without it the probe loops were ~10% of all issued
// instructions of an output-bound layer).
#ifndef BS_TC_WAIT_NS
#define BS_TC_WAIT_NS 64
#endif
__device__ __forceinline__ bool mbar_try(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(uint32_t addr, uint32_t parity) {
  while (!mbar_try(addr, parity)) __nanosleep(BS_TC_WAIT_NS);
}
__device__ __forceinline__ void mbar_arrive(uint32_t addr) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t addr, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(addr), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, uint32_t src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(src)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// 128B-swizzled K-major UMMA shared-memory descriptor (SM100 layout, version 1):
// start address >> 4, LBO (unused for swizzled K-major) = 1, SBO = 1024 B (8 rows x
// 128 B) >> 4, layout type 2 = SWIZZLE_128B.  The tile base must be 1024-byte aligned;
// stepping K by 32 bytes inside the swizzle row is a +2 on the start field.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;  // version
  d |= uint64_t(2) << 61;  // SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::i8: D = S32, A = u8 (activation planes, 0 or 2^i),
// B = s8 (weight planes, +/-2^j or 0/2^j), both K-major, M = 128, N = BN.
constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | (0u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// A operand from tensor memory (lane = row, 4 int8 per 32-bit column), B from smem.
__device__ __forceinline__ void mma_i8_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// The 4 K-steps (32 bytes each) of one plane pair in one 128-byte K chunk, issued by one
// elected lane of the (converged) MMA warp: A columns +8 per step, B descriptor start
// +32 bytes (+2 encoded) per step.  Keeping the whole warp on the issue path makes every
// operand warp-uniform (uniform registers, no per-MMA R2UR / waterfall) — the MMA warp
// shares its SM sub-partition with ALU-bound producer warps, so its instruction count
// per MMA sets the tensor-core feed rate.
template <uint32_t IDESC = 0>  // IDESC != 0: compile-time instruction descriptor (single-problem launches)
__device__ __forceinline__ void mma4_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
  if constexpr (IDESC != 0) {
    asm volatile(
        "{.reg .pred p, e; .reg .b32 x, a1; .reg .b64 b1;\n"
        "elect.sync x|e, 0xffffffff;\n"
        "setp.ne.b32 p, %3, 0;\n"
        "@!e bra SKIP%=;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %4, p;\n"
        "add.u32 a1, %1, 8; add.u64 b1, %2, 2;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], b1, %4, 1;\n"
        "add.u32 a1, %1, 16; add.u64 b1, %2, 4;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], b1, %4, 1;\n"
        "add.u32 a1, %1, 24; add.u64 b1, %2, 6;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], b1, %4, 1;\n"
        "SKIP%=:\n"
        "}" ::"r"(d),
        "r"(a), "l"(b), "r"(accumulate), "n"(IDESC));
    return;
  }
  asm volatile(
      "{.reg .pred p, e; .reg .b32 x, a1; .reg .b64 b1;\n"
      "elect.sync x|e, 0xffffffff;\n"
      "setp.ne.b32 p, %3, 0;\n"
      "@!e bra SKIP%=;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %4, p;\n"
      "add.u32 a1, %1, 8; add.u64 b1, %2, 2;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], b1, %4, 1;\n"
      "add.u32 a1, %1, 16; add.u64 b1, %2, 4;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], b1, %4, 1;\n"
      "add.u32 a1, %1, 24; add.u64 b1, %2, 6;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [a1], b1, %4, 1;\n"
      "SKIP%=:\n"
      "}" ::"r"(d),
      "r"(a), "l"(b), "r"(accumulate), "r"(idesc));
}

// tcgen05.commit from the elected lane (the lane that issued the MMAs).
__device__ __forceinline__ void mma_commit_elect(uint32_t mbar) {
  asm volatile(
      "{.reg .pred e; .reg .b32 x; elect.sync x|e, 0xffffffff;\n"
      "@!e bra SKIP%=;\n"
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "SKIP%=:\n}" ::"r"(mbar)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar) : "memory");
}

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

// K order inside a packed word.  The tensor core only needs activations and weights
// in the SAME order along K, and each 32-byte MMA K-step covers exactly one packed
// word (32 elements), so within every word the elements are laid out transposed:
// byte position 4q + r (expanded word q, byte r) holds element 8r + q.  Expanded word
// q is then bit q of every byte of the packed word, so one shift and one AND make it.
// 32 activation bits of one plane word -> 8 words of bytes 2^I * bit; the shifts are
// multiplications (IMAD / IMAD.HI on the FMA pipe) so the ALU pipe only does the ANDs.
template <int I>
__device__ __forceinline__ void expand_word(uint32_t w, uint32_t (&o)[8]) {
  constexpr uint32_t M = 0x01010101u << I;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    uint32_t t;
    if (q == I)
      t = w;
    else if (q < I)
      t = w * (1u << (I - q));  // bit 8r+q -> 8r+I
    else
      t = __umulhi(w, 1u << (32 - (q - I)));  // w >> (q - I)
    o[q] = t & M;
  }
}

// 32 consecutive 32-bit TMEM columns of this thread's lane <- o[0..31].
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&o)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7]), "r"(o[8]), "r"(o[9]),
      "r"(o[10]), "r"(o[11]), "r"(o[12]), "r"(o[13]), "r"(o[14]), "r"(o[15]), "r"(o[16]), "r"(o[17]), "r"(o[18]),
      "r"(o[19]), "r"(o[20]), "r"(o[21]), "r"(o[22]), "r"(o[23]), "r"(o[24]), "r"(o[25]), "r"(o[26]), "r"(o[27]),
      "r"(o[28]), "r"(o[29]), "r"(o[30]), "r"(o[31])
      : "memory");
}

// One plane's four packed words of this thread (one 128-element K chunk) -> bytes
// 2^I * bit -> the 32 TMEM columns of the thread's lane for that plane.
template <int I>
__device__ __forceinline__ void expand_to_tmem(uint32_t taddr, uint4 v) {
  uint32_t o[32];
  uint32_t t[8];
  expand_word<I>(v.x, t);
#pragma unroll
  for (int q = 0; q < 8; ++q) o[q] = t[q];
  expand_word<I>(v.y, t);
#pragma unroll
  for (int q = 0; q < 8; ++q) o[8 + q] = t[q];
  expand_word<I>(v.z, t);
#pragma unroll
  for (int q = 0; q < 8; ++q) o[16 + q] = t[q];
  expand_word<I>(v.w, t);
#pragma unroll
  for (int q = 0; q < 8; ++q) o[24 + q] = t[q];
  tmem_st32(taddr, o);
}

// ---- FP4 (kind::mxf4) operand format.  Elements are packed E2M1 nibbles, 8 per 32-bit
// word; two bit planes (b_lo, b_hi) become one radix-4 digit nibble 0.5 * (b_lo + 2 b_hi)
// (digit_nibbles), and the digit weights 2^(2d+1), 2^(2e+1) are the UE8M0 block scale
// factors (constant per digit), so 0.5*2^(2d+1) * a_d * 0.5*2^(2e+1) * w_e =
// 4^(d+e) a_d w_e.  K order inside a packed word (shared with the weights): nibble r
// of expanded word q (q < 4) holds element 4r + q, so expanded word q = (w >> q) & 0x1..1.
// Products and partial sums are small integers times powers of two, exact in the FP32
// accumulator (tools/mxf4_probe.cu: bit-exact up to |sum| = 803,600 > the 737,280 bound).
__device__ __forceinline__ void expand_word_f4(uint32_t w, uint32_t (&o)[4]) {
  o[0] = w & 0x11111111u;
  o[1] = __umulhi(w, 1u << 31) & 0x11111111u;  // w >> 1 on the FMA pipe
  o[2] = __umulhi(w, 1u << 30) & 0x11111111u;
  o[3] = __umulhi(w, 1u << 29) & 0x11111111u;
}

// 16 consecutive 32-bit TMEM columns of this thread's lane <- o[0..15].
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&o)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7]), "r"(o[8]), "r"(o[9]),
      "r"(o[10]), "r"(o[11]), "r"(o[12]), "r"(o[13]), "r"(o[14]), "r"(o[15])
      : "memory");
}

// Radix-4 digits on the FP4 path.  An E2M1 nibble holds 0.5 x {0, 1, 2, 3} exactly
// (0b0000, 0b0001, 0b0010, 0b0011), so two bit planes (lo = plane 2d, hi = plane 2d+1)
// form ONE operand digit d of weight 4^d (scale factor 2^(2d+1)); each digit-pair MMA
// does the work of up to four plane-pair MMAs of Eq. 2 (the sum over planes is exact
// either way).  L, H: nibble bit-0 masks of the lo / hi plane (bit 4r of
// L = element bit).  mode 0 unsigned: L + 2H; 1 bipolar: (2L-1) + 2(2H-1) (single: 2L-1);
// 2 the digit holding the two's-complement top plane: L - 2H (single: -L).
template <bool HAS_HI>
__device__ __forceinline__ uint32_t digit_nibbles(uint32_t L, uint32_t H, int mode) {
  constexpr uint32_t M = 0x11111111u;
  if (mode == 0) return HAS_HI ? (L | (H << 1)) : L;
  if (mode == 1)  // +-0.5 (0b0001 / 0b1001), +-1.5 (0b0011 / 0b1011)
    return HAS_HI ? (M | ((~(L ^ H) & M) << 1) | ((~H & M) << 3)) : (M | ((L ^ M) << 3));
  return HAS_HI ? (L | ((H & ~L) << 1) | (H << 3)) : L * 9u;  // 0.5, -1, -0.5 / -0.5
}

// Expanded word q (q < 4) of one digit from packed plane words lo, hi, mode fixed at
// compile time.  Shifts are folded per q so the unsigned pair costs what two separate
// planes did (a shift and a mask per plane and word, merged by one LOP3):
// 0.5 * (b_lo + 2 b_hi) = nibble bit 0 from lo, bit 1 from hi.
template <int MODE, bool HAS_HI, int Q>
__device__ __forceinline__ uint32_t digit_word(uint32_t lo, uint32_t hi, uint32_t lox) {
  constexpr uint32_t M = 0x11111111u;
  const uint32_t L = (Q == 0 ? lo : lo >> Q) & M;
  if constexpr (MODE == 0) {
    if constexpr (!HAS_HI) return L;
    const uint32_t H2 = (Q == 0 ? hi << 1 : (Q == 1 ? hi : hi >> (Q - 1))) & (M << 1);
    return L | H2;
  } else if constexpr (MODE == 1) {  // bipolar: 1 | (lo == hi) << 1 | !hi << 3; single 1 | !lo << 3
    if constexpr (!HAS_HI) return M | (((Q == 3 ? ~lo : ~lo << (3 - Q))) & (M << 3));
    const uint32_t E = (Q == 0 ? ~lox << 1 : (Q == 1 ? ~lox : ~lox >> (Q - 1))) & (M << 1);  // lox = lo ^ hi
    const uint32_t S = (Q == 3 ? ~hi : ~hi << (3 - Q)) & (M << 3);
    return M | E | S;
  } else {  // the signed top digit: L - 2H (0.5, -1, -0.5); single: -L
    if constexpr (!HAS_HI) return L * 9u;
    const uint32_t H = (Q == 0 ? hi : hi >> Q) & M;
    return L | ((H & ~L) << 1) | (H << 3);
  }
}

// One digit's four packed words per plane (128 K elements) -> 16 TMEM columns of E2M1.
// `valid` (bipolar only): pieces of padding (bit clear) expand to 0, not to -1.5.
template <int MODE, bool HAS_HI>
__device__ __forceinline__ void expand_digit_f4(uint32_t taddr, uint4 lo, uint4 hi, uint32_t valid) {
  const uint32_t l4[4] = {lo.x, lo.y, lo.z, lo.w}, h4[4] = {hi.x, hi.y, hi.z, hi.w};
  uint32_t o[16];
#pragma unroll
  for (int wi = 0; wi < 4; ++wi) {
    const uint32_t l = l4[wi], h = HAS_HI ? h4[wi] : 0u, x = l ^ h;
    uint32_t t[4] = {digit_word<MODE, HAS_HI, 0>(l, h, x), digit_word<MODE, HAS_HI, 1>(l, h, x),
                     digit_word<MODE, HAS_HI, 2>(l, h, x), digit_word<MODE, HAS_HI, 3>(l, h, x)};
    if constexpr (MODE == 1) {
      const bool ok = (valid >> (wi >> 1)) & 1u;  // words 0-1: piece 0, words 2-3: piece 1
#pragma unroll
      for (int q = 0; q < 4; ++q) t[q] = ok ? t[q] : 0u;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) o[4 * wi + q] = t[q];
  }
  tmem_st16(taddr, o);
}

// Every digit of one chunk: digit D holds planes 2D, 2D+1; with MODE 2 (signed) only the
// digit holding plane A-1 uses the signed rule.
template <int A_BITS, int MODE, int KQ, int D = 0>
__device__ __forceinline__ void expand_digits_f4(uint32_t ta, const uint4 (&v)[A_BITS][KQ], uint32_t valid) {
  if constexpr (2 * D < A_BITS) {
    constexpr bool kHi = 2 * D + 1 < A_BITS;
    constexpr bool kTop = 2 * D + 2 >= A_BITS;
    constexpr int kMode = (MODE == 2 && !kTop) ? 0 : MODE;
#pragma unroll
    for (int q = 0; q < KQ; ++q)  // digit D's 32 columns per stage: 16 per 4-word group
      expand_digit_f4<kMode, kHi>(ta + uint32_t(D * 32 + q * 16), v[2 * D][q], v[kHi ? 2 * D + 1 : 2 * D][q],
                                  valid >> (2 * q));
    expand_digits_f4<A_BITS, MODE, KQ, D + 1>(ta, v, valid);
  }
}

// The 4 K-steps (64 elements = 8 TMEM columns / 32 bytes of a 128B-swizzled B row each)
// of one digit pair in one 256-element FP4 chunk.
template <uint32_t IDESC = 0>  // IDESC != 0: compile-time instruction descriptor (single-problem launches)
__device__ __forceinline__ void mma4_f4(uint32_t d, uint32_t a, uint64_t b, uint32_t sfa, uint32_t sfb, uint32_t idesc,
                                        uint32_t accumulate) {
  if constexpr (IDESC != 0) {
    asm volatile(
        "{.reg .pred p, e; .reg .b32 x, a1; .reg .b64 b1;\n"
        "elect.sync x|e, 0xffffffff;\n"
        "setp.ne.b32 p, %3, 0;\n"
        "@!e bra SKIP%=;\n"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %4, [%5], [%6], p;\n"
        "add.u32 a1, %1, 8; add.u64 b1, %2, 2;\n"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [a1], b1, %4, [%5], [%6], 1;\n"
        "add.u32 a1, %1, 16; add.u64 b1, %2, 4;\n"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [a1], b1, %4, [%5], [%6], 1;\n"
        "add.u32 a1, %1, 24; add.u64 b1, %2, 6;\n"
        "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [a1], b1, %4, [%5], [%6], 1;\n"
        "SKIP%=:\n"
        "}" ::"r"(d),
        "r"(a), "l"(b), "r"(accumulate), "n"(IDESC), "r"(sfa), "r"(sfb));
    return;
  }
  asm volatile(
      "{.reg .pred p, e; .reg .b32 x, a1; .reg .b64 b1;\n"
      "elect.sync x|e, 0xffffffff;\n"
      "setp.ne.b32 p, %3, 0;\n"
      "@!e bra SKIP%=;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [%1], %2, %4, [%5], [%6], p;\n"
      "add.u32 a1, %1, 8; add.u64 b1, %2, 2;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [a1], b1, %4, [%5], [%6], 1;\n"
      "add.u32 a1, %1, 16; add.u64 b1, %2, 4;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [a1], b1, %4, [%5], [%6], 1;\n"
      "add.u32 a1, %1, 24; add.u64 b1, %2, 6;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], [a1], b1, %4, [%5], [%6], 1;\n"
      "SKIP%=:\n"
      "}" ::"r"(d),
      "r"(a), "l"(b), "r"(accumulate), "r"(idesc), "r"(sfa), "r"(sfb));
}

// Block-scaled instruction descriptor, kind::mxf4: A, B = E2M1, scales UE8M0, K = 64,
// K-major, M = 128, N = BN (D is always F32).
constexpr uint32_t idesc_mxf4(int n) {
  return (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (1u << 23) | (uint32_t(BM >> 4) << 24);
}


// ------------------------------------------------------------------ weight expansion
// w_packed [W][N][kp] words -> wexp [W][N][kpad*32] bytes (kpad = kp rounded up to
// 4 words; bytes past kp*32 are 0), each 32-byte group in the transposed K order of
// expand_word.  Plane j byte = 2^j b (unipolar) or 2^j (2b - 1)
// (bipolar); zero padding of the activations makes the value of pad bytes irrelevant.
// Valid-element mask of packed weight word kk: a filter row is KH*KW taps of kw_tap
// words each holding c_tap elements (bits past c_tap in a tap's last word are padding);
// padding expands to 0 so it contributes nothing whatever the activation encoding.
__device__ __forceinline__ uint32_t tap_word_mask(int64_t kk, int64_t kp, int c_tap, int kw_tap) {
  if (kk >= kp) return 0u;
  const int wt = int(kk % kw_tap);
  const int lo = wt * 32;
  if (lo + 32 <= c_tap) return 0xFFFFFFFFu;
  if (lo >= c_tap) return 0u;
  return (1u << (c_tap - lo)) - 1u;
}

// Weight-plane value of a set / clear bit for encoding w_enc (0 unipolar, 1 bipolar,
// 2 signed two's complement: the top plane weighs -2^(W-1)).
__device__ __forceinline__ int plane_sign(int j, int w_bits, int w_enc) {
  return (w_enc == 2 && j == w_bits - 1) ? -1 : 1;
}
// ----------------------------------------------------------------------- main kernel
// F4 = false: kind::i8 (bytes; a chunk = 128 K elements = 4 packed words per plane and
// row); F4 = true: kind::mxf4 (packed E2M1 radix-4 digits, scale-factor regions in TMEM;
// a chunk = 256 K elements = 8 packed words).  Both: 128-byte B rows, SWIZZLE_128B, 32
// TMEM columns per plane / digit per stage, four K-steps per plane / digit pair.
template <int A_BITS, int W_BITS, int BN, bool F4, int NP = 1>
struct Cfg {
  // operand "planes": bit planes (I8), radix-4 digits of two bit planes (F4, digit_nibbles)
  static constexpr int kAP = F4 ? (A_BITS + 1) / 2 : A_BITS;
  static constexpr int kWP = F4 ? (W_BITS + 1) / 2 : W_BITS;
  static constexpr int kCW = chunk_words(F4);             // packed words per plane per row per stage
  static constexpr int kQ = kCW / 4;                      // 4-word groups per stage
  static constexpr int kBRow = BKB;                       // B bytes per row per plane per stage (128B swizzle)
  static constexpr int kAColsPlane = 32;                  // TMEM columns per plane / digit per stage
  static constexpr int kACols = kAP * kAColsPlane;        // TMEM columns of one stage's A planes
  static constexpr int kBBytes = kWP * BN * kBRow;        // shared memory per stage (B only)
  static constexpr int kSFCols = F4 ? 16 + 8 * kWP : 0;   // SFA: up to 4 x 4 cols; SFB: kWP x 8
  static constexpr int kFixed = 1024 /*align slack*/ + kBarBytes + NP * 512 /*tap tables*/ + kEpiBytes;
  static constexpr int kFitSmem = (kSmemLimit - kFixed) / kBBytes;   // B chunk slots that fit
  static constexpr int kFitTmem = (512 - 2 * BN - kSFCols) / kACols;  // accumulators: 2 x BN columns
  static constexpr int kFit = kFitSmem < kFitTmem ? kFitSmem : kFitTmem;
  // A operand ring (tensor memory): kStages stages, a multiple of the producer teams, so
  // every stage belongs to ONE team (chunk g -> team g % T, stage g % S): the team waits on
  // its stage's empty barrier with its own phase count (a hardware-suspended mbarrier wait,
  // no polling, and no two teams that could alias each other's phases).
  static constexpr int kFitA = kFitTmem > BS_TC_MAX_STAGES ? BS_TC_MAX_STAGES : kFitTmem;
  static constexpr int kTeamsUsed = kFitA < kTeams ? kFitA : kTeams;
  static constexpr int kStages = kFitA / kTeamsUsed * kTeamsUsed;
  // B operand (shared memory): kBSlots chunk slots, decoupled from the A ring.  A tile whose
  // K chunks all fit keeps its weights RESIDENT (chunk kc in slot kc) and the next tile of
  // the same (problem, N block) reuses them without a reload; longer K streams through the
  // slots as a ring (BPlan).
  static constexpr int kBSlots = kFitSmem > 32 ? 32 : kFitSmem;
  static constexpr int kUsed = kFixed + kBSlots * kBBytes;
  static constexpr int kBytes = kUsed < kMinSmem ? kMinSmem : kUsed;
  static constexpr int kTmemCols = 512;  // 2*BN accumulator columns + the A ring; one CTA per SM
  static constexpr int kSF0 = 2 * BN;               // first scale-factor column (F4)
  static constexpr int kAcol0 = 2 * BN + kSFCols;   // first A-ring column
};

// kEpiMcast: the fused all-gather's NVLS form — each staged box re-read row-contiguously and
// stored with multimem.st to the multicast address of the gathered C (one egress per box,
// the switch replicates it to every rank's copy, this rank's included).
enum EpiMode : int { kEpiDirect = 0, kEpiTma = 1, kEpiScalar = 2, kEpiMcast = 3 };


// 16 bytes to a multicast (NVLS) address: every device bound to the multicast object gets them.
__device__ __forceinline__ void multimem_st_v4(int32_t* p, uint4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

using bs::FastDiv;  // (common.cuh)
using bs::make_fastdiv;

// One problem of a launch (a single conv / dense, or one member of a group).
struct TcProb {
  ConvProblem p;
  int ntn;          // N blocks
  int nmb;          // M blocks (tiles are N-major: tile = nblk * nmb + mblk, so a CTA's consecutive
                    // tiles share an N block and its resident weights)
  int nchunks;      // K chunks (of 4 words) per tile
  int tile0;        // first tile of this problem in the launch's tile sequence
  int epi;          // EpiMode: direct 16-byte stores (OC % 4 == 0), TMA stores, or scalar
  uint32_t idesc;   // MMA instruction descriptor (N = 64 for OC <= 64 inside a BN = 128 group)
  FastDiv div_hw, div_ow, div_kwid, div_nm, div_kwa;  // n / (oh*ow), / ow, / kw, / nmb, / Cw
  int kwa_shift;    // log2(Cw) when Cw is a power of two, else -1
  int taps;         // kh * kw (the tap table is used when taps <= kMaxTaps)
};

// Launch arguments: NP problems whose tiles are concatenated (problem q owns tiles
// [tile0_q, tile0_{q+1})); CTAs walk the whole sequence with a grid stride, so every
// role sees its problem index only grow.  NP = 1 is the single-problem launch.
template <int NP>
struct TcArgs {
  int nprob, ntiles;  // problems, tiles of all problems
  int nset0, tiles0;  // grouped launches: problems [0, nset0) (tensor-heavy) own tiles [0, tiles0); the rest
                      // (output-heavy) [tiles0, ntiles); each CTA interleaves its tiles of the two sets
  int b_bytes;        // bytes of the B region (kBSlots chunk slots)
  int nbs;            // B chunk slots in use (<= kBSlots; BS_TUNE_TC_B_SLOTS caps it)
  int npeer;          // single-problem launches: every output box is also stored through peer[0..npeer)
  int32_t* mcast;     // single-problem kEpiMcast launches: multicast address of out[0][0]
  int blocked;        // raw-weight launches with several N blocks: each CTA walks a contiguous range of the
                      // N-major tiles, so the weights it expanded for an N block serve its next tiles
                      // (otherwise a grid stride: neighbouring CTAs on neighbouring tiles, which the
                      // output writes and the activation halos favour)
  int debug;          // BS_TC_PROFILE / BS_TC_KNOBS builds only: bit 0 skip output stores, 1 skip A tcgen05.st,
                      // 2 skip accumulator tcgen05.ld, 3 skip the producers' global loads,
                      // 4 MMA warp ignores full_a, 5 producers idle, 6 producers keep their first tile's
                    // row geometry, 7 no MMAs issued (timing experiments; results are wrong)
  TcProb prob[NP];
};
template <int NP>
struct TcMaps {
  CUtensorMap w[NP];    // prepared weights [W][oc][kpad bytes]
  CUtensorMap out[NP];  // int32 output [M][oc] (TMA-store epilogue)
  CUtensorMap peer[NP == 1 ? kMaxPeers : 1];  // fused all-gather: the same [M][oc] block in other ranks' buffers
};
#if defined(BS_TC_PROFILE) || defined(BS_TC_KNOBS)
#define DBG(bit) (args.debug & (1 << (bit)))
#else
#define DBG(bit) 0
#endif

// (M block, N block) of a problem's tile (N-major order).
__device__ __forceinline__ void tile_mn(const TcProb& P, int tile, uint32_t& mblk, uint32_t& nblk) {
  const uint32_t tl = uint32_t(tile - P.tile0);
  nblk = P.div_nm.div(tl);
  mblk = tl - nblk * P.div_nm.d;
}

// Where each K chunk's weights live in the B slots, decided identically by the TMA warp
// (which loads) and the MMA warp (which waits / releases) as both walk the tile sequence.
// Resident (nchunks <= slots): chunk kc in slot kc, loaded only when the (problem, N block)
// differs from the previous tile's; streaming: ring slots, always loaded.
struct BPlan {
  int key_pi = -1, key_nb = -1, ring = 0;
  __device__ __forceinline__ void next(int pi, int nb, int nchunks, int nslots, bool& res, bool& reload,
                                       int& slot0) {
    res = nchunks <= nslots;
    if (res) {
      reload = !(pi == key_pi && nb == key_nb);
      key_pi = pi;
      key_nb = nb;
      slot0 = 0;
    } else {
      reload = true;
      key_pi = -1;
      slot0 = ring;
      ring = (ring + nchunks) % nslots;
    }
  }
};

// RAW launches (weights given as packed planes, expanded in the kernel): the producer team
// that handles a K chunk also writes that chunk's weight slot when BPlan reloads it.  Every
// team walks every tile with its own BPlan copy to know each chunk's slot.  Several teams
// write the same slot in turn, so a parity wait on the slot's empty barrier could alias two
// phases; instead the (otherwise idle) TMA warp releases the slots in chunk order: it waits
// on each slot's empty barrier as the only waiter and publishes s_ready[slot] = the chunk
// that may now write it.
struct RawTrack {
  BPlan plan;
  bool res = false, reload = false;
  int slot0 = 0;
  __device__ __forceinline__ void enter(int pi, int nb, int nchunks, int nbs) {
    plan.next(pi, nb, nchunks, nbs, res, reload, slot0);
  }
};

// A CTA's tile sequence.  Single problem: blockIdx.x, +gridDim.x, ...  Grouped: the CTA's
// share of each set (same grid stride) merged in proportion, so tensor-heavy tiles (long
// K: producer / MMA work) alternate with output-heavy ones (1x1 layers: epilogue and HBM
// work) and the roles of one SM overlap the two kinds; the problem index is tracked per
// set (it only grows within a set).  Every role walks an identical copy.
template <int NP, bool BLOCKED = false>
struct TileSeq {
  int c, g, a, b, j0, j1, pi0, pi1;
  __device__ __forceinline__ explicit TileSeq(const TcArgs<NP>& args) {
    c = int(blockIdx.x);
    g = int(gridDim.x);
    const int t0 = NP > 1 ? args.tiles0 : args.ntiles, t1 = args.ntiles - t0;
    if (NP == 1 && BLOCKED && args.blocked) {  // a contiguous range of the N-major tiles: consecutive tiles share
      // an N block (its weights stay resident) even when the M blocks are fewer than the CTAs
      j0 = int(int64_t(c) * t0 / g);
      a = int(int64_t(c + 1) * t0 / g);
      b = 0;
      g = 1;
    } else if (NP == 1) {
      j0 = 0;
      a = t0 > c ? (t0 - 1 - c) / g + 1 : 0;
      b = 0;
    } else {  // grid stride: every CTA gets a share of each member (members are sorted by K)
      a = t0 > c ? (t0 - 1 - c) / g + 1 : 0;
      b = t1 > c ? (t1 - 1 - c) / g + 1 : 0;
      j0 = 0;
    }
    j1 = 0;
    pi0 = 0;
    pi1 = NP > 1 ? args.nset0 : 0;
  }
  // next tile and its problem; false when the CTA's sequence is done
  __device__ __forceinline__ bool next(const TcArgs<NP>& args, int& tile, int& pi) {
    if constexpr (NP == 1) {
      if (j0 >= a) return false;
      tile = (BLOCKED && args.blocked) ? j0 : c + j0 * g;  // blocked ranges start j0 at the range
      ++j0;
      pi = 0;
      return true;
    } else {
      const bool take0 = j0 < a && (j1 >= b || int64_t(2 * j0 + 1) * b <= int64_t(2 * j1 + 1) * a);
      if (take0) {
        tile = c + j0++ * g;
        while (pi0 + 1 < args.nset0 && tile >= args.prob[pi0 + 1].tile0) ++pi0;
        pi = pi0;
      } else if (j1 < b) {
        tile = args.tiles0 + c + j1++ * g;
        while (pi1 + 1 < args.nprob && tile >= args.prob[pi1 + 1].tile0) ++pi1;
        pi = pi1;
      } else {
        return false;
      }
      return true;
    }
  }
};

// Kernel variants (compile-time, so each path costs the others nothing): prepared weights
// loaded by TMA; RAW packed weight planes expanded by the producers; MCAST prepared weights with
// the NVLS multicast epilogue.
enum TcVariant : int { kVarPrep = 0, kVarRaw = 1, kVarMcast = 2 };

template <int A_BITS, int W_BITS, int BN, bool F4, int NP, int VAR = kVarPrep>
__global__ void __launch_bounds__(kThreads, 1)
    tc_conv_kernel(const __grid_constant__ TcArgs<NP> args, const __grid_constant__ TcMaps<NP> maps) {
  constexpr bool RAW = VAR == kVarRaw, MCAST = VAR == kVarMcast;
  static_assert(!RAW || (F4 && NP == 1), "raw-weight launches: FP4 format, single problem");
  static_assert(!RAW || BN == 64 || BN == 128, "raw-weight launches: the team's rows split a power-of-two BN");
  using C = Cfg<A_BITS, W_BITS, BN, F4, NP>;
  constexpr int S = C::kStages;   // A ring stages (tensor memory)
  constexpr int NB = C::kBSlots;  // B chunk slots (shared memory)
  static_assert(S >= 2 && NB >= 2, "tensor-core tile does not fit two stages");
  static_assert(C::kBytes <= kSmemLimit, "shared memory");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* s_stage = smem;                            // B: NB chunk slots
  uint8_t* s_epi = smem + args.b_bytes;               // epilogue staging: warps x bufs x 4 KB (1024-aligned)
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_epi + kEpiBytes);
  uint64_t* full_a = bars;
  uint64_t* empty = bars + S;           // A stage consumed (MMA commit)
  uint64_t* full_b = bars + 2 * S;      // B slot loaded (TMA transaction bytes)
  uint64_t* empty_b = bars + 2 * S + NB;  // B slot released before a reload (MMA commit)
  uint64_t* acc_full = bars + 2 * S + 2 * NB;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 4);
  int2* s_tap = reinterpret_cast<int2*>(reinterpret_cast<uint8_t*>(bars) + kBarBytes);  // [NP][kMaxTaps] {offset, ky<<16|kx}
  int* s_ready = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(bars) + kBarBytes - 256);  // RAW: [32] chunk allowed to write each B slot
  static_assert(8 * (2 * S + 2 * NB + 4) + 4 <= kBarBytes - 256, "barrier region");

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nbs = args.nbs;  // B slots in use (<= NB)
  if (lane == 0 && (warp == 0 || warp == kMmaWarp)) STAMP("start")
  PROF_DECL
#ifdef BS_TC_PROFILE
  const long long _t_start = clock64();
#endif

  // filter-tap tables (implicit im2col): word offset of tap (ky, kx) from the row's
  // receptive-field origin, and (ky, kx) for the bounds test
  for (int q = 0; q < args.nprob; ++q) {
    const TcProb& P = args.prob[q];
    if (P.taps <= kMaxTaps && tid < P.taps) {
      const int ky = tid / P.p.kwid, kx = tid - ky * P.p.kwid;
      s_tap[q * kMaxTaps + tid] = make_int2((ky * P.p.w + kx) * P.p.kw_a, (ky << 16) | kx);
    }
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(smem_u32(full_a + s), 4);  // the 4 warps of one team
      mbar_init(smem_u32(empty + s), 1);
    }
    for (int b = 0; b < 32; ++b) s_ready[b] = -1;
    for (int b = 0; b < NB; ++b) {
      mbar_init(smem_u32(full_b + b), RAW ? 4 : 1);  // RAW: the 4 warps of the team that expands it
      mbar_init(smem_u32(empty_b + b), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(smem_u32(acc_full + a), 1);
      mbar_init(smem_u32(acc_empty + a), kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (!RAW && warp == kTmaWarp && lane < args.nprob) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.w[lane])) : "memory");
    if (args.prob[lane].epi == kEpiTma)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.out[lane])) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // all 512 columns belong to this CTA (one CTA per SM): the allocation starts at lane 0,
  // column 0, so TMEM addresses are compile-time constants
  if (*tmem_slot != 0u) asm volatile("trap;");
  constexpr uint32_t tmem = 0;
  if (lane == 0 && warp == kMmaWarp) STAMP("prologue")
  if constexpr (F4) {
    // uniform UE8M0 scale factors: SFA digit d (4 columns) = 2^(2d+1), SFB digit e (8
    // columns) = 2^(2e+1); every byte of a region holds the digit's scale, so the MMA reads
    // the right value whatever its scale-factor layout (tools/mxf4_probe.cu: an M=128 /
    // N<=128 region spans 4 columns, N=256 8)
    if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 4) {
#pragma unroll
      for (int c0 = 0; c0 < C::kSFCols; c0 += 16) {  // 16 columns per store
        uint32_t v[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const int col = c0 + c;
          v[c] = 0x01010101u * uint32_t(col < 16 ? 128 + 2 * (col >> 2) : 128 + 2 * ((col - 16) >> 3));
        }
        tmem_st16(tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(C::kSF0 + c0), v);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }

  if (warp < 4 * C::kTeamsUsed && DBG(5)) {
    // knob 5: producers idle (MMA-only timing with knob 4)
  } else if (warp < 4 * C::kTeamsUsed) {
    // ================= expansion producers.  kTeams teams of 4 warps; team t expands the
    // chunks g = t, t+kTeams, ... of this CTA's (tile, K chunk) sequence, so kTeams chunks
    // are in flight.  Within a team, thread `arow` (warp % 4 == its TMEM lane quarter)
    // owns output row arow and all 4 packed words of each plane of the chunk.  The
    // packed words are loaded straight into registers one team step ahead (the kTeams
    // chunks in flight cover the load latency); all index arithmetic is shifts and
    // precomputed fast divisions (a team changes tile almost every step when K is short).
    constexpr int kTeams = C::kTeamsUsed;
    const int team = warp >> 2, arow = tid & (BM - 1);
    int pi = 0;  // problem of the chunk being loaded
    const uint32_t s_tap_u32 = smem_u32(s_tap);
#define LP args.prob[pi].p
    // the loaded problem's per-chunk fields in registers, refreshed when the problem
    // changes (grouped launches: a parameter indexed by a run-time problem number costs an
    // LDC per use; with NP = 1 these fold back into constant-bank operands)
    struct Hot {
      int64_t plane;
      int kp, kwa, kwa_shift, h, w, a_enc, nchunks;
      bool tap;
    };
    auto hot_of = [&](int q) {  // (next_tile0 is unused: the tile sequence tracks problems)
      const TcProb& P = args.prob[q];
      Hot r;
      r.plane = P.p.act_plane;
      r.kp = int(P.p.kp);
      r.kwa = P.p.kw_a;
      r.kwa_shift = P.kwa_shift;
      r.h = P.p.h;
      r.w = P.p.w;
      r.a_enc = P.p.a_enc;
      r.nchunks = P.nchunks;
      r.tap = P.taps <= kMaxTaps;
      return r;
    };
    Hot H = hot_of(0);
    // geometry of this thread's row in tile `t`
    bool rok = false;
    int iy0 = 0, ix0 = 0;
    const uint32_t* rbase = LP.act;  // image base (pixel 0 of the row's image), word units
    const uint32_t* rorg = LP.act;   // receptive-field origin (iy0, ix0) of the row (may lie in the padding)
    auto set_tile = [&](int t) {
      const TcProb& P = args.prob[pi];
      uint32_t mblk, nblk;
      tile_mn(P, t, mblk, nblk);
      const int64_t m = int64_t(mblk) * BM + arow;
      rok = m < P.p.M;
      const uint32_t mm = rok ? uint32_t(m) : 0u;
      const uint32_t b = P.div_hw.div(mm), rem = mm - b * P.div_hw.d;
      const uint32_t oy = P.div_ow.div(rem), ox = rem - oy * P.div_ow.d;
      iy0 = int(oy) * P.p.sh - P.p.ph;
      ix0 = int(ox) * P.p.sw - P.p.pw;
      // pixel index of the receptive-field origin in 32-bit arithmetic (N*H*W < 2^31,
      // ABI-checked; the origin may lie in the padding, i.e. slightly negative)
      const int img = int(b) * H.h;
      rbase = P.p.act + int64_t(img * H.w) * H.kwa;
      rorg = P.p.act + int64_t((img + iy0) * H.w + ix0) * H.kwa;
    };
    // source of the 2- or 4-word piece starting at filter word kk (kk even)
    auto piece = [&](int kk, bool& ok) -> const uint32_t* {
      const int kwa = H.kwa;
      int tap, cw;
      if (H.kwa_shift >= 0) {
        tap = kk >> H.kwa_shift;
        cw = kk & (kwa - 1);
      } else {
        tap = int(args.prob[pi].div_kwa.div(uint32_t(kk)));
        cw = kk - tap * kwa;
      }
      if (H.tap) {
        int2 e;  // explicit shared-space load (a generic load would take the long-scoreboard path)
        asm("ld.shared.v2.s32 {%0, %1}, [%2];"
                     : "=r"(e.x), "=r"(e.y)
                     : "r"(s_tap_u32 + uint32_t(8 * (pi * kMaxTaps + (tap < kMaxTaps ? tap : 0)))));
        const int iy = iy0 + (e.y >> 16), ix = ix0 + (e.y & 0xFFFF);
        ok = rok && kk < H.kp && unsigned(iy) < unsigned(H.h) && unsigned(ix) < unsigned(H.w);
        return rorg + e.x + cw;
      }
      const TcProb& P = args.prob[pi];
      const int ky = int(P.div_kwid.div(uint32_t(tap))), kx = tap - ky * P.p.kwid;
      const int iy = iy0 + ky, ix = ix0 + kx;
      ok = rok && kk < H.kp && unsigned(iy) < unsigned(H.h) && unsigned(ix) < unsigned(H.w);
      return rbase + (int64_t(iy) * H.w + ix) * kwa + cw;
    };
    // one chunk's kCW words per plane of this thread's row, as kQ uint4 groups; vm bit p =
    // 2-word piece p valid (padding / K tail pieces load as 0)
    constexpr int kQ = C::kQ;
    auto load = [&](int kc, uint4 (&v)[A_BITS][kQ], uint32_t& vm) {
      if (DBG(3)) {  // timing experiment: no global loads
#pragma unroll
        for (int i = 0; i < A_BITS; ++i)
#pragma unroll
          for (int q = 0; q < kQ; ++q) v[i][q] = make_uint4(kc, i, arow, q);
        vm = 0xFu;
        return;
      }
      const int64_t plane = H.plane;
      const int kk0 = kc * C::kCW;
      vm = 0u;
      if (kQ == 2 && (H.kwa & 7) == 0) {  // the 8 words lie in one tap
        bool ok;
        const uint32_t* s0 = piece(kk0, ok);
        vm = ok ? 0xFu : 0u;
#pragma unroll
        for (int i = 0; i < A_BITS; ++i)
#pragma unroll
          for (int q = 0; q < kQ; ++q)
            v[i][q] = ok ? ldg_nc_v4(s0 + i * plane + 4 * q) : make_uint4(0u, 0u, 0u, 0u);
      } else if ((H.kwa & 3) == 0) {  // 4-word groups, each in one tap
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
          bool ok;
          const uint32_t* s0 = piece(kk0 + 4 * q, ok);
          vm |= ok ? 3u << (2 * q) : 0u;
#pragma unroll
          for (int i = 0; i < A_BITS; ++i) v[i][q] = ok ? ldg_nc_v4(s0 + i * plane) : make_uint4(0u, 0u, 0u, 0u);
        }
      } else {  // Cw = 2 mod 4: 2-word pieces, a tap boundary inside every 4-word group
#pragma unroll
        for (int q = 0; q < kQ; ++q) {
          bool ok0, ok1;
          const uint32_t* s0 = piece(kk0 + 4 * q, ok0);
          const uint32_t* s1 = piece(kk0 + 4 * q + 2, ok1);
          vm |= ((ok0 ? 1u : 0u) | (ok1 ? 2u : 0u)) << (2 * q);
#pragma unroll
          for (int i = 0; i < A_BITS; ++i) {
            const uint2 lo = ok0 ? ldg_nc_v2(s0 + i * plane) : make_uint2(0u, 0u);
            const uint2 hi = ok1 ? ldg_nc_v2(s1 + i * plane) : make_uint2(0u, 0u);
            v[i][q] = make_uint4(lo.x, lo.y, hi.x, hi.y);
          }
        }
      }
    };
    // iterator of the next chunk to load: tile t (of problem pi), chunk kc
    TileSeq<NP, RAW> seq(args);
    int t = -1, kc = team, cur_tile = -1;
    RawTrack rt;  // RAW: weight-slot loads of every tile (all teams')
    auto next_tile = [&]() -> bool {
      const bool ok = seq.next(args, t, pi);
      if constexpr (RAW) {
        if (ok) {
          uint32_t mb_, nb_;
          tile_mn(args.prob[pi], t, mb_, nb_);
          rt.enter(pi, int(nb_), args.prob[pi].nchunks, nbs);
        }
      }
      return ok;
    };
    bool more = next_tile();
    if constexpr (NP > 1) H = hot_of(pi);
    auto carry = [&]() {  // move kc past the ends of tiles
      while (more && kc >= H.nchunks) {
        kc -= H.nchunks;
        const int prev = pi;
        more = next_tile();
        if constexpr (NP > 1) {
          if (more && pi != prev) H = hot_of(pi);
        }
      }
    };
    uint4 nxt[A_BITS][kQ];
    uint32_t nvm = 0;
    int nenc = 0;
    // RAW: the chunk's weight row (this thread's filter) prefetched with its activations
    constexpr int kRW = RAW ? W_BITS : 1;
    int wn = 0;  // the thread's filter row of the chunk's N block
    int wslot = 0, wreload = 0, wg = 0;  // the chunk's B slot, reload flag, its index in the CTA's chunk sequence
    int wkk0 = 0, lg = team;             // lg: sequence index of the chunk advance_load loads
    auto advance_load = [&]() -> bool {
      if (!more) return false;
      if (t != cur_tile && !(DBG(6) && cur_tile >= 0)) {  // knob 6: geometry of the first tile only
        set_tile(t);
        cur_tile = t;
      }
      load(kc, nxt, nvm);
      nenc = H.a_enc;
      if constexpr (RAW) {
        wslot = rt.res ? kc : (rt.slot0 + kc) % nbs;
        wreload = rt.reload;
        wg = lg;
        if (wreload) {  // (the weight words are loaded when the chunk is expanded: reloads are rare
          // when weights stay resident, and holding them from here would spill registers)
          uint32_t mb_, nb_;
          tile_mn(args.prob[pi], t, mb_, nb_);
          wn = int(nb_) * BN + (arow & (BN - 1));  // BN = 64: two threads per filter row (halves of it)
          wkk0 = kc * C::kCW;
        }
      }
      kc += kTeams;
      lg += kTeams;
      carry();
      return true;
    };
#undef LP
    carry();
    bool have = advance_load();
    const uint32_t lane_base = tmem + (uint32_t((warp & 3) * 32) << 16);
    for (int g = team; have; g += kTeams) {
      // one register buffer: this step expands nxt, then reloads it with the next step's
      // words, whose latency is covered by the tensor-memory store wait, the barrier
      // arrive and the next stage-free wait (two buffers would spill at 8 words per plane)
      uint4 (&v)[A_BITS][kQ] = nxt;
      const uint32_t vm = nvm;
      const int enc = nenc;
      const int stage = g % S;
      PROF_BEGIN
      mbar_wait_sleep(smem_u32(empty + stage), ((g / S) & 1) ^ 1);  // this team's stage: its previous chunk consumed
      PROF_END(1)
      tc_fence_after();
      PROF_BEGIN  // slot 2: digit formation + tcgen05.st issue
      const uint32_t ta = lane_base + uint32_t(C::kAcol0 + stage * C::kACols);
      if (DBG(1)) {
        uint32_t x = 0;
#pragma unroll
        for (int i = 0; i < A_BITS; ++i) x ^= v[i][0].x ^ v[i][0].y ^ v[i][kQ - 1].z ^ v[i][kQ - 1].w;
        if (x == 0x9e3779b9u) asm volatile("trap;");
      } else {
        if constexpr (F4) {
          if (enc == 0)
            expand_digits_f4<A_BITS, 0, kQ>(ta, v, vm);
          else if (enc == 1)
            expand_digits_f4<A_BITS, 1, kQ>(ta, v, vm);
          else
            expand_digits_f4<A_BITS, 2, kQ>(ta, v, vm);
        } else {
          expand_to_tmem<0>(ta, v[0][0]);
          if constexpr (A_BITS > 1) expand_to_tmem<1>(ta + 1 * (BKB / 4), v[1][0]);
          if constexpr (A_BITS > 2) expand_to_tmem<2>(ta + 2 * (BKB / 4), v[2][0]);
          if constexpr (A_BITS > 3) expand_to_tmem<3>(ta + 3 * (BKB / 4), v[3][0]);
        }
      }
      PROF_END(2)
      if constexpr (RAW) {
        if (wreload) {  // this chunk's weights: packed planes -> E2M1 digit rows of the B slot
          const TcProb& P = args.prob[0];
          // the team's 128 threads share the slot's BN rows: with BN = 64 each row's eight 16-byte
          // units are split between two threads (part 0: units 0-3, part 1: units 4-7)
          constexpr int kSplit = BM / BN, kQd = 4 / kSplit;
          const int wr = arow & (BN - 1), part = arow / BN;
          uint2 wnx[kRW][kQd];
          PROF_BEGIN  // slot 4 (RAW): weight-word loads
          {
            const int kp = int(P.p.kp);
            const bool rowok = wn < P.p.oc;
            const uint32_t* wrow = P.p.wt + (int64_t(wn) * kp + wkk0);
#pragma unroll
            for (int j = 0; j < kRW; ++j)
#pragma unroll
              for (int q = 0; q < kQd; ++q) {  // packed rows have an even word count: 2-word pieces are all-in or all-out
                const int qq = part * kQd + q;
                wnx[j][q] = (rowok && wkk0 + 2 * qq < kp) ? ldg_nc_v2(wrow + int64_t(j) * P.p.oc * kp + 2 * qq)
                                                          : make_uint2(0u, 0u);
              }
          }
          PROF_END(4)
          PROF_BEGIN  // slot 5 (RAW): wait for the slot's release
          for (;;) {  // the TMA warp released the slot to this chunk (its previous use consumed)
            int r;
            asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(r) : "r"(smem_u32(s_ready + wslot)) : "memory");
            if (r >= wg) break;
            __nanosleep(64);
          }
          PROF_END(5)
          PROF_BEGIN  // slot 6 (RAW): weight digit formation + shared-memory stores
          {
            uint8_t* brow = s_stage + wslot * C::kBBytes + wr * C::kBRow;
            const int wenc = P.p.bipolar;
#pragma unroll
            for (int e = 0; e < C::kWP; ++e) {
              constexpr int kDummy = 0;
              (void)kDummy;
#pragma unroll
              for (int wi = 0; wi < 2 * kQd; ++wi) {
                const int wd = part * 2 * kQd + wi;  // the 16-byte unit (packed word) of the row
                const uint32_t lo = wi & 1 ? wnx[2 * e][wi >> 1].y : wnx[2 * e][wi >> 1].x;
                const bool has_hi = 2 * e + 1 < W_BITS;
                const uint32_t hi = has_hi ? (wi & 1 ? wnx[(2 * e + 1) % kRW][wi >> 1].y
                                                     : wnx[(2 * e + 1) % kRW][wi >> 1].x) : 0u;
                uint32_t o[4];
                if (wenc == 1) {  // bipolar: +-0.5 / +-1.5 digits; padding elements must stay 0
                  const uint32_t valid = tap_word_mask(wkk0 + wd, P.p.kp, P.p.c_tap, P.p.kw_a);
                  const uint32_t x = lo ^ hi;
                  if (has_hi) {
                    o[0] = digit_word<1, true, 0>(lo, hi, x); o[1] = digit_word<1, true, 1>(lo, hi, x);
                    o[2] = digit_word<1, true, 2>(lo, hi, x); o[3] = digit_word<1, true, 3>(lo, hi, x);
                  } else {
                    o[0] = digit_word<1, false, 0>(lo, hi, x); o[1] = digit_word<1, false, 1>(lo, hi, x);
                    o[2] = digit_word<1, false, 2>(lo, hi, x); o[3] = digit_word<1, false, 3>(lo, hi, x);
                  }
#pragma unroll
                  for (int q = 0; q < 4; ++q) o[q] &= ((valid >> q) & 0x11111111u) * 0xFu;
                } else {  // unipolar: digit b_lo + 2 b_hi (padding bits are 0 in packed planes)
                  const uint32_t x = lo ^ hi;
                  if (has_hi) {
                    o[0] = digit_word<0, true, 0>(lo, hi, x); o[1] = digit_word<0, true, 1>(lo, hi, x);
                    o[2] = digit_word<0, true, 2>(lo, hi, x); o[3] = digit_word<0, true, 3>(lo, hi, x);
                  } else {
                    o[0] = digit_word<0, false, 0>(lo, hi, x); o[1] = digit_word<0, false, 1>(lo, hi, x);
                    o[2] = digit_word<0, false, 2>(lo, hi, x); o[3] = digit_word<0, false, 3>(lo, hi, x);
                  }
                }
                // 16-byte unit wd of this 128-byte row, 128B-swizzled as TMA would place it
                *reinterpret_cast<uint4*>(brow + e * BN * C::kBRow + ((uint32_t(wd) ^ uint32_t(wr & 7)) << 4)) =
                    make_uint4(o[0], o[1], o[2], o[3]);
              }
            }
          }
          fence_proxy_async();  // generic-proxy stores -> visible to the tensor core's smem reads
          __syncwarp();
          PROF_END(6)
          if (lane == 0) mbar_arrive(smem_u32(full_b + wslot));
        }
      }
      PROF_BEGIN  // slot 0: next step's address math and load issue
      have = advance_load();
      PROF_END(0)
      PROF_BEGIN  // slot 3: tensor-memory store completion
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      PROF_END(3)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(full_a + stage));
    }
  } else if (warp < kProducerWarps) {
    // producer warps of teams this configuration does not use: idle
  } else if (warp == kTmaWarp) {
    // ================= weight tiles by TMA: each K chunk's weights into its B slot unless
    // they are resident (BPlan); a slot is reloaded once the MMA released its previous use
    // (RAW launches: the producer teams write the slots; this warp releases each slot to
    // the chunk that writes it next, in chunk order — see RawTrack)
    if (RAW && lane == 0) {
      int pi = 0, tile = 0, g = 0;
      uint32_t ldpar = 0;  // bit b: parity of the writes released into B slot b
      BPlan plan;
      TileSeq<NP, RAW> seq(args);
      bool have = seq.next(args, tile, pi);
      while (have) {
        const TcProb& P = args.prob[pi];
        uint32_t mb, nb;
        tile_mn(P, tile, mb, nb);
        bool res, reload;
        int slot;
        plan.next(pi, int(nb), P.nchunks, nbs, res, reload, slot);
        for (int kc = 0; kc < P.nchunks; ++kc, ++g) {
          if (reload) {
            const uint32_t bit = 1u << slot;
            mbar_wait_sleep(smem_u32(empty_b + slot), (ldpar & bit) ? 0u : 1u);  // previous use consumed
            ldpar ^= bit;
            asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_ready + slot)), "r"(g) : "memory");
          }
          slot = (res || slot + 1 < nbs) ? slot + 1 : 0;
        }
        have = seq.next(args, tile, pi);
      }
    }
    if (!RAW && lane == 0) {
      int pi = 0, tile = 0;
      uint32_t ldpar = 0;  // bit b: parity of the loads issued into B slot b
      BPlan plan;
      for (TileSeq<NP, RAW> seq(args); seq.next(args, tile, pi);) {
        const TcProb& P = args.prob[pi];
        uint32_t mb, nb;
        tile_mn(P, tile, mb, nb);
        const int n0 = int(nb) * BN, nchunks = P.nchunks, oc = P.p.oc;
        const CUtensorMap* tw = &maps.w[pi];
        bool res, reload;
        int slot;
        plan.next(pi, int(nb), nchunks, nbs, res, reload, slot);
        for (int kc = 0; kc < nchunks && reload; ++kc) {
          {
            const uint32_t bit = 1u << slot;
            PROF_BEGIN
            mbar_wait_sleep(smem_u32(empty_b + slot), (ldpar & bit) ? 0u : 1u);  // the slot's previous use released
            PROF_END(0)
            ldpar ^= bit;
            const uint32_t fb = smem_u32(full_b + slot);
            mbar_expect_tx(fb, uint32_t(C::kBBytes));
            const uint32_t sB = smem_u32(s_stage + slot * C::kBBytes);
#pragma unroll
            for (int j = 0; j < C::kWP; ++j) tma_load_2d(sB + j * BN * C::kBRow, tw, kc * C::kBRow, j * oc + n0, fb);
          }
          slot = (res || slot + 1 < nbs) ? slot + 1 : 0;
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ================= MMA issuer: the whole warp walks the loop (uniform values); one
    // elected lane issues.  TMEM base is column 0 (all 512 columns are this CTA's).
    int stage = 0, acc = 0, pi = 0, tile = 0;
    uint32_t phase = 0, acc_phase = 0, fpar = 0;  // fpar bit b: parity of the loads consumed from B slot b
    bool first = true;
    const uint64_t bdesc0 = smem_desc_sw128(smem_u32(s_stage));
    BPlan plan;
    TileSeq<NP, RAW> seq(args);
    bool have = seq.next(args, tile, pi);
    while (have) {
      int ntile = 0, npi = 0;
      const bool nhave = seq.next(args, ntile, npi);
      // single-problem launches: N = BN is known at compile time (an immediate descriptor
      // saves a constant-bank reload per MMA); groups: the member's N (64 or BN)
      constexpr uint32_t kIdesc = NP == 1 ? (F4 ? idesc_mxf4(BN) : idesc_i8(BN)) : 0u;
      const TcProb& P = args.prob[pi];
      const uint32_t idesc = P.idesc;
      const int nchunks = P.nchunks;
      uint32_t mb, nb;
      tile_mn(P, tile, mb, nb);
      bool res, reload;
      int slot;
      plan.next(pi, int(nb), nchunks, nbs, res, reload, slot);
      bool keep = false;  // the next tile reuses this tile's resident weights: no release
      if (res && nhave && npi == pi) {
        uint32_t mb2, nb2;
        tile_mn(args.prob[npi], ntile, mb2, nb2);
        keep = nb2 == nb;
      }
      PROF_BEGIN
      mbar_wait(smem_u32(acc_empty + acc), acc_phase ^ 1u);
      PROF_END(0)
      tc_fence_after();
      const uint32_t tacc = uint32_t(acc * BN);
      for (int kc = 0; kc < nchunks; ++kc) {
        PROF_BEGIN
        if (!DBG(4)) mbar_wait(smem_u32(full_a + stage), phase);  // knob 4: MMA-only timing
        PROF_END(1)
        PROF_BEGIN
        if (reload) {
          mbar_wait(smem_u32(full_b + slot), (fpar >> slot) & 1u);
          fpar ^= 1u << slot;
        }
        PROF_END(2)
        PROF_BEGIN  // slot 4 (MMA warp): fence + MMA issue
        tc_fence_after();
        const uint32_t a_base = uint32_t(C::kAcol0 + stage * C::kACols);
        const uint64_t b_desc = bdesc0 + uint64_t((slot * C::kBBytes) >> 4);
#pragma unroll
        for (int i = 0; i < C::kAP; ++i)
#pragma unroll
          for (int j = 0; j < C::kWP; ++j) {
            if (DBG(7)) continue;  // knob 7: no MMAs (issue-path timing)
            if constexpr (F4)
              mma4_f4<kIdesc>(tacc, a_base + uint32_t(i * C::kAColsPlane), b_desc + uint64_t((j * BN * C::kBRow) >> 4),
                      uint32_t(C::kSF0 + 4 * i), uint32_t(C::kSF0 + 16 + 8 * j), idesc, (kc | i | j) != 0);
            else
              mma4_ts<kIdesc>(tacc, a_base + uint32_t(i * (BKB / 4)), b_desc + uint64_t((j * BN * BKB) >> 4), idesc,
                      (kc | i | j) != 0);
          }
        PROF_END(4)
        PROF_BEGIN  // slot 5 (MMA warp): stage / slot release commits
        mma_commit_elect(smem_u32(empty + stage));
        if (!keep) mma_commit_elect(smem_u32(empty_b + slot));
        PROF_END(5)
        if (++stage == S) {
          stage = 0;
          phase ^= 1u;
        }
        slot = (res || slot + 1 < nbs) ? slot + 1 : 0;
      }
      mma_commit_elect(smem_u32(acc_full + acc));
      if (lane == 0 && first) STAMP("first_tile_issued")
      first = false;
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
      tile = ntile;
      pi = npi;
      have = nhave;
    }
  } else {
    // ================= epilogue: warp q = warp % 4 owns TMEM lanes / tile rows 32q..32q+31
    const int q = warp & 3;
    const int ew = warp - kEpiWarp0, cb0 = ew >> 2;  // with 8 warps, two per lane quarter split the columns
    constexpr int kCbStep = kEpiWarps / 4;
    uint8_t* ebuf = s_epi + ew * (kEpiBufs * kEpiBufBytes);
    int acc = 0, buf = 0, pi = 0, tile = 0;
    uint32_t acc_phase = 0;
    bool first = true;
    for (TileSeq<NP, RAW> seq(args); seq.next(args, tile, pi);) {
      const TcProb& P = args.prob[pi];
      uint32_t mb, nb;
      tile_mn(P, tile, mb, nb);
      const int64_t m0 = int64_t(mb) * BM;
      const int n0 = int(nb) * BN;
      const int oc = P.p.oc, epi = P.epi;
      const int64_t M = P.p.M;
      int32_t* const out = P.p.out;
      const int ncb = min(BN, oc - n0 + 31) / 32;  // 32-column blocks holding valid columns
      PROF_BEGIN
      mbar_wait_sleep(smem_u32(acc_full + acc), acc_phase);
      PROF_END(0)
      if (lane == 0 && warp == kEpiWarp0 && first) STAMP("first_acc_full")
      first = false;
      tc_fence_after();
      bool released = false;
      for (int cb = cb0; cb < ncb; cb += kCbStep) {
        uint32_t r[32];
        if (DBG(2)) {
#pragma unroll
          for (int c = 0; c < 32; ++c) r[c] = c;
        } else {
          PROF_BEGIN
          tmem_ld32(tmem + (uint32_t(q * 32) << 16) + uint32_t(acc * BN + cb * 32), r);
          PROF_END(1)
          if constexpr (F4) {  // FP32 accumulator holding an exact integer (|v| < 2^22) -> int32:
            // one F2I per value (the conversion pipe; one issue slot per 32 values where the
            // v + 1.5*2^23 trick takes two — the epilogue's issue slots are the scarce resource)
#pragma unroll
            for (int c = 0; c < 32; ++c) r[c] = uint32_t(__float2int_rz(__uint_as_float(r[c])));
          }
        }
        if (cb + kCbStep >= ncb) {  // this warp's share of the accumulator drained: release it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(acc_empty + acc));
          released = true;
        }
        const int64_t row = m0 + q * 32 + lane;
        if (DBG(0)) {
          if (r[0] == 0x9e3779b9u) asm volatile("trap;");
        } else if (epi == kEpiDirect) {  // this lane's row segment: 128 contiguous bytes, 8 x 16-byte stores
          if (row < M && n0 + cb * 32 + 32 <= oc) {
            uint4* dst = reinterpret_cast<uint4*>(out + row * oc + n0 + cb * 32);
#pragma unroll
            for (int c = 0; c < 8; ++c) dst[c] = make_uint4(r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);
          } else if (row < M) {
            int32_t* dst = out + row * oc;
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              const int col = n0 + cb * 32 + c;
              if (col < oc) dst[col] = int32_t(r[c]);
            }
          }
        } else if (epi == kEpiTma) {
          PROF_BEGIN
          if (lane == 0) bulk_wait_read<kEpiBufs - 1>();  // the store that last used `buf` has read it
          __syncwarp();
          PROF_END(2)
          PROF_BEGIN
          uint8_t* sb = ebuf + buf * kEpiBufBytes + lane * 128;
          const uint32_t swz = uint32_t(lane & 7);
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<uint4*>(sb + ((uint32_t(c) ^ swz) << 4)) =
                make_uint4(r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            const uint32_t sbox = smem_u32(ebuf + buf * kEpiBufBytes);
            tma_store_2d(&maps.out[pi], n0 + cb * 32, int(m0) + q * 32, sbox);
            if constexpr (NP == 1)  // fused all-gather: the same staged box to every peer copy (NVLink)
              for (int d = 0; d < args.npeer; ++d) tma_store_2d(&maps.peer[d], n0 + cb * 32, int(m0) + q * 32, sbox);
            bulk_commit();
          }
          PROF_END(3)
          buf = buf + 1 == kEpiBufs ? 0 : buf + 1;
        } else if (MCAST) {  // swizzled staging, then row-contiguous multimem stores
          uint8_t* b0 = ebuf + buf * kEpiBufBytes;
          const uint32_t swz = uint32_t(lane & 7);
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<uint4*>(b0 + lane * 128 + ((uint32_t(c) ^ swz) << 4)) =
                make_uint4(r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 8; ++i) {  // 4 rows x 128 B per instruction (oc % 4 == 0)
            const int rr = i * 4 + (lane >> 3), ch = lane & 7;
            const uint4 v = *reinterpret_cast<const uint4*>(b0 + rr * 128 + ((uint32_t(ch) ^ uint32_t(rr & 7)) << 4));
            const int64_t grow = m0 + q * 32 + rr;
            const int col = n0 + cb * 32 + ch * 4;
            if (grow < M && col < oc) multimem_st_v4(args.mcast + grow * oc + col, v);
          }
          __syncwarp();
        } else {  // OC % 4 != 0: plain bounded stores
          if (row < M) {
            int32_t* dst = out + row * oc;
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              const int col = n0 + cb * 32 + c;
              if (col < oc) dst[col] = int32_t(r[c]);
            }
          }
        }
      }
      if (!released) {  // no column block for this warp (narrow tile): release at once
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(acc_empty + acc));
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
    }
    if (lane == 0) STAMP("epilogue_loop_done")
    if (lane == 0) bulk_wait_all();
    if (lane == 0) STAMP("stores_done")
  }

#ifdef BS_TC_PROFILE
  if (blockIdx.x == 0 && lane == 0)
    printf("TCPROF warp %d total %lld w0 %lld w1 %lld w2 %lld w3 %lld w4 %lld w5 %lld w6 %lld\n", warp,
           clock64() - _t_start, _pacc[0], _pacc[1], _pacc[2], _pacc[3], _pacc[4], _pacc[5], _pacc[6]);
#endif
  tc_fence_before();
  __syncthreads();
  if (lane == 0 && warp == kMmaWarp) STAMP("end")
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::kTmemCols));
  }
}

// ------------------------------------------------------------------------ host side
// cuTensorMapEncodeTiled through the runtime's driver entry point (the library does not
// link libcuda, so it still loads on hosts without a driver).
inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

inline bool encode_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* base, uint64_t inner, uint64_t outer,
               uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  return enc(map, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Fill one problem's launch record and tensor maps for tile width BN (the MMA uses N = 64
// when the problem's filters fit it).  Returns false when a tensor map cannot be encoded.
inline bool make_prob(TcProb& P, CUtensorMap& tw, CUtensorMap& to, const ConvProblem& p, const int8_t* wexp, int tile0,
               int bn, bool f4, int64_t& tiles) {
  P.p = p;
  P.ntn = (p.oc + bn - 1) / bn;
  P.nmb = int((p.M + BM - 1) / BM);
  tiles = int64_t(P.nmb) * P.ntn;
  const int64_t kpad = tc_kpad(p.kp, f4 ? kTcF4 : kTcI8);
  P.nchunks = int(kpad / chunk_words(f4));
  P.tile0 = tile0;
  // TMA-store epilogue by default (direct 16-byte stores of one row segment per lane
  // measured 1.4-1.8x slower on the output-bound layers); BS_TC_EPI=direct selects them.
  const bool want_direct = tuning(kTuneEpilogue) == 1;
  P.epi = (p.oc % 4) != 0 ? kEpiScalar : (want_direct ? kEpiDirect : kEpiTma);
  const int mma_n = p.oc <= 64 ? 64 : bn;
  P.idesc = f4 ? idesc_mxf4(mma_n) : idesc_i8(mma_n);
  P.div_hw = make_fastdiv(uint32_t(p.oh) * uint32_t(p.ow));
  P.div_ow = make_fastdiv(uint32_t(p.ow));
  P.div_kwid = make_fastdiv(uint32_t(p.kwid));
  P.div_nm = make_fastdiv(uint32_t(P.nmb));
  P.div_kwa = make_fastdiv(uint32_t(p.kw_a));
  P.taps = p.kh * p.kwid;
  // the table's int32 word offsets: (ky*W + kx)*Cw must fit
  if ((int64_t(p.kh) * p.w + p.kwid) * p.kw_a >= (int64_t(1) << 31)) P.taps = kMaxTaps + 1;
  P.kwa_shift = -1;
  for (int sh = 0; sh < 31; ++sh)
    if ((1 << sh) == p.kw_a) P.kwa_shift = sh;
  const int brow = BKB;
  const uint64_t wrow = uint64_t(kpad) * (f4 ? 16 : 32);  // prepared-weight row bytes
  const int wplanes = f4 ? (p.w_bits + 1) / 2 : p.w_bits;  // F4: radix-4 digits
  if (wexp && !encode_2d(&tw, CU_TENSOR_MAP_DATA_TYPE_UINT8, wexp, wrow, uint64_t(wplanes) * p.oc, wrow, brow, bn,
                         CU_TENSOR_MAP_SWIZZLE_128B))  // (raw-weight launches: no prepared weights)
    return false;
  if (P.epi == kEpiTma)
    return encode_2d(&to, CU_TENSOR_MAP_DATA_TYPE_INT32, p.out, uint64_t(p.oc), uint64_t(p.M), uint64_t(p.oc) * 4, 32,
                     32, CU_TENSOR_MAP_SWIZZLE_128B);
  to = tw;  // unused
  return true;
}

template <int A_BITS, int W_BITS, int BN, bool F4, int NP, int VAR = kVarPrep>
cudaError_t launch_bn(const ConvProblem* ps, const int8_t* const* wexps, int count, cudaStream_t stream,
                      int nset0 = -1, int32_t* const* peers = nullptr, int npeer = 0, int32_t* mcast = nullptr) {
  using C = Cfg<A_BITS, W_BITS, BN, F4, NP>;
  constexpr bool RAW = VAR == kVarRaw;
  auto kern = tc_conv_kernel<A_BITS, W_BITS, BN, F4, NP, VAR>;
  // the dynamic shared-memory opt-in is a per-device function attribute: set once per
  // device (a bit per device, set after the call succeeded; racing threads set it twice)
  static std::atomic<uint64_t> configured{0};
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  const uint64_t bit = dev < 64 ? uint64_t(1) << dev : 0;
  if (!bit || !(configured.load(std::memory_order_acquire) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
    if (e != cudaSuccess) return e;
    configured.fetch_or(bit, std::memory_order_release);
  }
  if (count < 1 || count > NP) return cudaErrorInvalidValue;
  TcArgs<NP> a;
  TcMaps<NP> maps;
  memset(&a, 0, sizeof(a));
  memset(&maps, 0, sizeof(maps));
  a.nprob = count;
  int64_t total = 0;
  for (int q = 0; q < count; ++q) {
    int64_t tiles = 0;
    if (!make_prob(a.prob[q], maps.w[q], maps.out[q], ps[q], RAW ? nullptr : wexps[q], int(total), BN, F4, tiles))
      return cudaErrorInvalidValue;
    total += tiles;
    if (total > (int64_t(1) << 31) - 1) return cudaErrorInvalidValue;
  }
  if (total == 0) return cudaSuccess;
  a.ntiles = int(total);
  a.nset0 = nset0 < 0 || nset0 > count ? count : nset0;
  a.blocked = RAW && a.prob[0].ntn > 1;
  if (npeer > 0) {  // fused all-gather (single problem, TMA-store epilogue)
    if (NP != 1 || npeer > kMaxPeers || a.prob[0].epi != kEpiTma) return cudaErrorNotSupported;
    const ConvProblem& p = ps[0];
    for (int d = 0; d < npeer; ++d)
      if (!encode_2d(&maps.peer[d], CU_TENSOR_MAP_DATA_TYPE_INT32, peers[d], uint64_t(p.oc), uint64_t(p.M),
                     uint64_t(p.oc) * 4, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B))
        return cudaErrorInvalidValue;
  }
  a.npeer = npeer;
  if ((mcast != nullptr) != (VAR == kVarMcast)) return cudaErrorInvalidValue;
  if (mcast) {  // NVLS fused all-gather (single problem, oc % 4 == 0)
    if (NP != 1 || a.prob[0].epi != kEpiTma || npeer > 0) return cudaErrorNotSupported;
    a.prob[0].epi = kEpiMcast;
    a.mcast = mcast;
  }
  a.tiles0 = a.nset0 < count ? a.prob[a.nset0].tile0 : a.ntiles;
  a.b_bytes = C::kBSlots * C::kBBytes;
#if defined(BS_TC_PROFILE) || defined(BS_TC_KNOBS)
  const char* dbg_env = getenv("BS_TC_DEBUG");  // experiment builds only
  a.debug = dbg_env ? atoi(dbg_env) : 0;
#endif
  const int cap = tuning(kTuneBSlots);
  a.nbs = cap >= 2 && cap < C::kBSlots ? cap : C::kBSlots;
  int smem_bytes = C::kFixed + a.b_bytes;
  if (smem_bytes < kMinSmem) smem_bytes = kMinSmem;
  const int grid = a.ntiles < device_sms() ? a.ntiles : device_sms();
  kern<<<grid, kThreads, smem_bytes, stream>>>(a, maps);
  note_launch();
  return cudaPeekAtLastError();
}

// Tile width: BN = 64 when the filters fit it, else 128 (the widest tile whose double-
// buffered accumulators leave TMEM room for the A ring).  BS_TC_BN overrides (tests).
inline int pick_bn(const ConvProblem& p) {
  if (const int v = tuning(kTuneTileN)) return v;
  return p.oc <= 64 ? 64 : 128;
}

template <int A_BITS, int W_BITS, bool F4>
cudaError_t launch_aw(const ConvProblem& p, const int8_t* wexp, cudaStream_t stream, int32_t* const* peers = nullptr,
                      int npeer = 0) {
  switch (pick_bn(p)) {
    case 128:
      if constexpr (Cfg<A_BITS, W_BITS, 128, F4>::kFit >= 2)
        return launch_bn<A_BITS, W_BITS, 128, F4, 1>(&p, &wexp, 1, stream, -1, peers, npeer);
      [[fallthrough]];
    default:
      return launch_bn<A_BITS, W_BITS, 64, F4, 1>(&p, &wexp, 1, stream, -1, peers, npeer);
  }
}

// The NVLS multicast epilogue variant (FP4, single problem; tc_conv_mcast.cu instantiates it).
template <int A_BITS, int W_BITS>
cudaError_t launch_mcast_aw(const ConvProblem& p, const int8_t* wexp, cudaStream_t stream, int32_t* mcast) {
  if (pick_bn(p) == 128) {
    if constexpr (Cfg<A_BITS, W_BITS, 128, true>::kFit >= 2)
      return launch_bn<A_BITS, W_BITS, 128, true, 1, kVarMcast>(&p, &wexp, 1, stream, -1, nullptr, 0, mcast);
  }
  return launch_bn<A_BITS, W_BITS, 64, true, 1, kVarMcast>(&p, &wexp, 1, stream, -1, nullptr, 0, mcast);
}

// Raw-weight launch (the three-call boundary: packed weight planes, no prepared copy): the
// producer teams expand each weight chunk into its B slot; BN = 64 when that keeps every
// K chunk of an N block resident and BN = 128 would stream (the expansion then runs once
// per N block and CTA instead of once per tile).
template <int A_BITS, int W_BITS>
cudaError_t launch_raw_aw(const ConvProblem& p, cudaStream_t stream) {
  using C128 = Cfg<A_BITS, W_BITS, 128, true, 1>;
  using C64 = Cfg<A_BITS, W_BITS, 64, true, 1>;
  const int nchunks = int(tc_kpad(p.kp, kTcF4) / chunk_words(true));
  int bn = pick_bn(p);
  if (bn == 128 && !tuning(kTuneTileN) && nchunks > C128::kBSlots && nchunks <= C64::kBSlots) bn = 64;
  if constexpr (C128::kFit >= 2) {
    if (bn == 128) return launch_bn<A_BITS, W_BITS, 128, true, 1, kVarRaw>(&p, nullptr, 1, stream);
  }
  return launch_bn<A_BITS, W_BITS, 64, true, 1, kVarRaw>(&p, nullptr, 1, stream);
}

// Group launch: up to kGroupMax problems of one (A, W) precision in one persistent
// kernel with BN-wide tiles (N = 64 MMAs for OC <= 64 members of a BN = 128 group).
// Problems are ordered by decreasing K so the cheapest tiles form the tail of every
// CTA's sequence.
template <int A_BITS, int W_BITS, int BN, bool F4>
cudaError_t launch_group_aw(const ConvProblem* ps, const int8_t* const* wexps, int count, cudaStream_t stream) {
  // a group of one is a single launch (instantiated once, in tc_conv.cu)
  if (count == 1) return launch_tc_conv_prepared(ps[0], wexps[0], F4 ? kTcF4 : kTcI8, stream);
  if constexpr (Cfg<A_BITS, W_BITS, BN, F4, kGroupMax>::kFit >= 2) {
    ConvProblem sp[kGroupMax];
    const int8_t* sw[kGroupMax];
    int order[kGroupMax];
    for (int q = 0; q < count; ++q) order[q] = q;
    std::stable_sort(order, order + count, [&](int x, int y) { return ps[x].kp > ps[y].kp; });
    for (int q = 0; q < count; ++q) {
      sp[q] = ps[order[q]];
      sw[q] = wexps[order[q]];
    }
    // set 0 (tensor-heavy): a tile's expansion + MMA work, ~256 clk per K chunk and plane
    // pair (measured producer rate), exceeds its epilogue's, ~BN*128*4 bytes at ~17 B/clk
    // (measured per-SM output rate); set 1: the rest.  Measured neutral on the ResNet-18
    // group (246 us either way), so one set is the default; BS_TC_SPLIT=1 interleaves.
    int nset0 = count;
    if (tuning(kTuneGroupSplit) == 1) {
        nset0 = 0;
        while (nset0 < count && int64_t(tc_kpad(sp[nset0].kp, F4 ? kTcF4 : kTcI8) / 4) * A_BITS * W_BITS * 256 >
                                    int64_t(BN) * BM * 4 / 17)
          ++nset0;
      }
    return launch_bn<A_BITS, W_BITS, BN, F4, kGroupMax>(sp, sw, count, stream, nset0);
  } else {
    for (int q = 0; q < count; ++q)
      if (cudaError_t e = launch_tc_conv_prepared(ps[q], wexps[q], F4 ? kTcF4 : kTcI8, stream)) return e;
    return cudaSuccess;
  }
}

}  // namespace tc

#define BS_TC_DISPATCH(CALL)                                                                          \
  BS_TC(1, 1, CALL) BS_TC(2, 1, CALL) BS_TC(2, 2, CALL) BS_TC(1, 2, CALL) BS_TC(3, 1, CALL)           \
  BS_TC(3, 2, CALL) BS_TC(4, 1, CALL) BS_TC(4, 2, CALL) BS_TC(1, 3, CALL) BS_TC(2, 3, CALL)           \
  BS_TC(3, 3, CALL) BS_TC(4, 3, CALL) BS_TC(1, 4, CALL) BS_TC(2, 4, CALL) BS_TC(3, 4, CALL)           \
  BS_TC(4, 4, CALL)

}  // namespace bs
