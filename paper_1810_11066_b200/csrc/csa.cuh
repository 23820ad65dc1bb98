// csa.cuh — carry-save (Harley-Seal style) compression of AND words before POPC.
//
// Eq. 2 needs, per output, sum_l 2^l * sum_{words at level l}
// popc(a_p & w_q) with l = p + q.  On B200 POPC issues at 16/clk/SM while LOP3 issues
// at 64/clk/SM (profiles/r01_int_pipe_rates.json), so a POPC-per-word loop leaves
// three quarters of the ALU idle.  A full adder on three words of the same level l,
//     s = x ^ y ^ z   (LOP3 0x96, stays at level l)
//     c = maj(x,y,z)  (LOP3 0xe8, moves to level l+1),
// satisfies popc(x)+popc(y)+popc(z) = popc(s) + 2 popc(c) exactly (bitwise), so each
// full adder trades one POPC for two LOP3.  Compressing every level down to <= 2
// words before counting moves the kernel from the POPC bound toward the ALU bound —
// the GPU analogue of the vectorized software popcount the paper uses on x86
// (Harley-Seal "vectorized software popcount", mula2017faster).
//
// Everything below is resolved at compile time: the plan (words per level, full
// adders per level) is a constexpr object, and all array indices are constants after
// unrolling, so the queues live in registers.
#pragma once
#include <cstdint>
#include <utility>

namespace bs {

template <int A, int W, int G>
struct CsaPlan {
  static constexpr int kLevels = A + W - 1 + 6;  // input levels + room for carries
  static constexpr int kWords = 2 * G;          // k-words per plane pair in a group
  int in[kLevels + 1];                          // input AND words at level l
  int n[kLevels + 1];                           // words at level l incl. carries
  int fa[kLevels + 1];                          // full adders applied at level l
  int cap;
  constexpr CsaPlan() : in(), n(), fa(), cap(0) {
    for (int l = 0; l <= kLevels; ++l) {
      int c = 0;
      for (int p = 0; p < A; ++p)
        for (int q = 0; q < W; ++q)
          if (p + q == l) ++c;
      in[l] = c * kWords;
    }
    int carry = 0;
    for (int l = 0; l <= kLevels; ++l) {
      n[l] = in[l] + carry;
      fa[l] = (l < kLevels && n[l] > 2) ? (n[l] - 1) / 2 : 0;  // reduce to <= 2 words
      carry = fa[l];
      if (n[l] + fa[l] > cap) cap = n[l] + fa[l];
    }
  }
  constexpr int popcounts() const {
    int s = 0;
    for (int l = 0; l <= kLevels; ++l) s += n[l] - 2 * fa[l];
    return s;
  }
};

// Cost model per word pair, in SMSP issue cycles of the binding pipe: POPC on the XU
// pipe (16/clk/SM -> 8 cycles per warp instruction per SMSP), LOP3 on the ALU pipe
// and the IMAD accumulations on the FMA pipe (64/clk/SM -> 2 cycles each).
template <int A, int W, int G>
constexpr double csa_cycles_per_word_pair() {
  constexpr CsaPlan<A, W, G> P{};
  int fa = 0;
  for (int l = 0; l <= CsaPlan<A, W, G>::kLevels; ++l) fa += P.fa[l];
  const int wp = A * W * 2 * G, lop = wp + 2 * fa, popc = P.popcounts();
  const double xu = 8.0 * popc, alu = 2.0 * lop, fma = 2.0 * popc;
  const double m = xu > alu ? xu : alu;
  return (m > fma ? m : fma) / wp;
}

// The same reduction flattened into a compile-time program over register slots:
// slots [0, A*W*2G) hold the AND words (p, q, v) -> (p*W + q)*2G + v; each full adder
// writes two new slots; the words left at each level are popcounted.  Executed with
// fold expressions over index sequences, so every register index is a template
// constant (no reliance on loop unrolling for the queues to stay in registers).
template <int A, int W, int G>
struct CsaProg {
  static constexpr int kIn = A * W * 2 * G;
  static constexpr int kMaxFa = kIn;   // each full adder removes >= 1 word
  static constexpr int kMaxPop = kIn;
  int nslots = 0, nfa = 0, npop = 0;
  int fx[kMaxFa] = {}, fy[kMaxFa] = {}, fz[kMaxFa] = {}, fs[kMaxFa] = {}, fc[kMaxFa] = {};
  int pslot[kMaxPop] = {}, plevel[kMaxPop] = {};
  constexpr CsaProg() {
    constexpr int LV = CsaPlan<A, W, G>::kLevels;
    int qd[LV + 2][kIn + kMaxFa] = {};
    int head[LV + 2] = {}, tail[LV + 2] = {};
    for (int p = 0; p < A; ++p)
      for (int q = 0; q < W; ++q)
        for (int v = 0; v < 2 * G; ++v) {
          const int l = p + q;
          qd[l][tail[l]++] = (p * W + q) * 2 * G + v;
        }
    nslots = kIn;
    for (int l = 0; l <= LV; ++l) {
      while (tail[l] - head[l] > 2) {
        const int x = qd[l][head[l]++], y = qd[l][head[l]++], z = qd[l][head[l]++];
        fx[nfa] = x; fy[nfa] = y; fz[nfa] = z;
        fs[nfa] = nslots++;
        fc[nfa] = nslots++;
        qd[l][tail[l]++] = fs[nfa];
        qd[l + 1][tail[l + 1]++] = fc[nfa];
        ++nfa;
      }
      while (head[l] < tail[l]) {
        pslot[npop] = qd[l][head[l]++];
        plevel[npop] = l;
        ++npop;
      }
    }
  }
};

// LOP3 through inline PTX so the front end cannot re-associate the AND / XOR3 / MAJ
// network (left to itself it folds the ANDs into 4-input functions that take more
// LOP3s than the tree); each call is exactly one LOP3.
template <int LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
  return d;
}

template <int A, int W, int G, int... I>
__device__ __forceinline__ void csa_run_fa(uint32_t* r, std::integer_sequence<int, I...>) {
  constexpr CsaProg<A, W, G> P{};
  ((r[P.fs[I]] = lop3<0x96>(r[P.fx[I]], r[P.fy[I]], r[P.fz[I]]),
    r[P.fc[I]] = lop3<0xe8>(r[P.fx[I]], r[P.fy[I]], r[P.fz[I]])), ...);
}

template <int A, int W, int G, int NW, int... I>
__device__ __forceinline__ int csa_run_pop(const uint32_t* r, int acc, const int (&wgt)[NW],
                                           std::integer_sequence<int, I...>) {
  constexpr CsaProg<A, W, G> P{};
  ((acc = __popc(r[P.pslot[I]]) * wgt[P.plevel[I]] + acc), ...);
  return acc;
}

// acc + sum_{p<A, q<W} 2^(p+q) * sum_{v<2G} popc(a[p][v] & w[q][v]), via the
// carry-save program above.  Exact for all inputs (a per-bit integer identity).
// `wgt[l]` must hold 2^l in registers the compiler cannot see through, so every
// accumulation is an IMAD on the FMA pipe, not a shift-add on the ALU (which already
// carries the AND and full-adder LOP3s).
template <int A, int W, int G>
__device__ __forceinline__ int csa_dot(int acc, const uint32_t (&a)[A][2 * G], const uint32_t (&w)[W][2 * G],
                                       const int (&wgt)[A + W + 6]) {
  constexpr CsaProg<A, W, G> P{};
  uint32_t r[P.nslots > 0 ? P.nslots : 1];
#pragma unroll
  for (int p = 0; p < A; ++p)
#pragma unroll
    for (int q = 0; q < W; ++q)
#pragma unroll
      for (int v = 0; v < 2 * G; ++v) r[(p * W + q) * 2 * G + v] = lop3<0xc0>(a[p][v], w[q][v], 0u);
  csa_run_fa<A, W, G>(r, std::make_integer_sequence<int, P.nfa>{});
  return csa_run_pop<A, W, G>(r, acc, wgt, std::make_integer_sequence<int, P.npop>{});
}

}  // namespace bs
