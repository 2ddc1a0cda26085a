// gk_bt2.cuh -- the block-transposed filtration (see gk_filter_bt2.cu for the
// method notes), templated on where the packed words live (GMem / SMem) so that
// the packed-input kernels and the fused ASCII kernels share one implementation.
#pragma once
#include "gk_common.cuh"
#include "gk_filter_core.cuh"

namespace gk {
namespace bt2 {

// load look-ahead (steps) of the sweep and of the per-e kernel
#ifndef GK_BT2_LA
#define GK_BT2_LA 2
#endif
#ifndef GK_BT2_LA_E
#define GK_BT2_LA_E 2
#endif

__device__ __forceinline__ uint32_t ones_if_neg(int x) { return __byte_perm((uint32_t)x, 0u, 0xBBBB); }
__device__ __forceinline__ uint32_t ones_if_nonneg(int x) { return ones_if_neg(~x); }

// Where the packed words of the lane's group live: GMem = the packed tile in
// global memory (position stride 32 uint2, read-only path), SMem = a group-major
// tile in shared memory (position stride 1; the fused ASCII kernels).
struct GMem {
  __device__ __forceinline__ static uint2 ld(const uint2* p, int pos) {
    return __ldg(p + (int64_t)pos * GK_WARP);
  }
  __device__ __forceinline__ static void prefetch(const uint2* p, int pos) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p + (int64_t)pos * GK_WARP));
  }
};
struct SMem {
  __device__ __forceinline__ static uint2 ld(const uint2* p, int pos) { return p[pos]; }
  __device__ __forceinline__ static void prefetch(const uint2*, int) {}
};
// word at position pos, clamped into [0, len) (checked paths only)
template <class M>
__device__ __forceinline__ uint2 ldc(const uint2* p, int pos, int len) {
  return M::ld(p, pos < 0 ? 0 : (pos >= len ? len - 1 : pos));
}

template <int B>
struct Win {
  static constexpr int W = B + 4;
  uint32_t h[W], l[W];
};

// F &= amend(mismatch(R, Qw)) over the block (unchecked)
template <int B>
__device__ __forceinline__ void mask_and(const Win<B>& R, const Win<B>& Qw, uint32_t (&F)[B]) {
  constexpr int W = B + 4;
  uint32_t x[W];
#pragma unroll
  for (int c = 0; c < W; ++c) x[c] = mismatch(R.h[c], R.l[c], Qw.h[c], Qw.l[c]);
#pragma unroll
  for (int u = 0; u < B; ++u) F[u] &= amend(x[u], x[u + 1], x[u + 2], x[u + 3], x[u + 4]);
}

// checked: raw = mismatch & sv (source valid) & tv (target valid); vac = forced 1
template <int B>
__device__ __forceinline__ void mask_and_checked(const Win<B>& R, const Win<B>& Qw,
                                                 const uint32_t (&sv)[B + 4],
                                                 const uint32_t (&tv)[B + 4],
                                                 const uint32_t (&vac)[B], uint32_t (&F)[B]) {
  constexpr int W = B + 4;
  uint32_t x[W];
#pragma unroll
  for (int c = 0; c < W; ++c) x[c] = mismatch(R.h[c], R.l[c], Qw.h[c], Qw.l[c]) & sv[c] & tv[c];
#pragma unroll
  for (int u = 0; u < B; ++u) F[u] &= amend(x[u], x[u + 1], x[u + 2], x[u + 3], x[u + 4]) | vac[u];
}

// Add N words of weight 2^P into bit-sliced planes pl[P..NP): a carry-save tree
// (full adders in pairs, a half adder for an odd word out), carries to P+1.
template <int P, int NP, int N>
__device__ __forceinline__ void csa_add(uint32_t (&pl)[NP], const uint32_t (&w)[N]) {
  if constexpr (N > 0 && P < NP) {
    constexpr int NN = N / 2 + (N & 1);
    uint32_t c[NN];
#pragma unroll
    for (int i = 0; i < N / 2; ++i) CsaCounter::fa(pl[P], w[2 * i], w[2 * i + 1], c[i]);
    if constexpr (N & 1) {
      c[NN - 1] = pl[P] & w[N - 1];
      pl[P] ^= w[N - 1];
    }
    csa_add<P + 1, NP, NN>(pl, c);
  }
}

// Per-k run-start counter of the sweep in shared memory: NP bit-sliced planes of
// 32 lanes (bank = lane).  Windows start at multiples of 4 and ib % B == 0, so a
// block's starts never depend on the previous block (readings R6, R7).
template <int B, int NP>
__device__ __forceinline__ void count_block_smem(uint32_t* p, const uint32_t (&F)[B]) {
  uint32_t st[B];
#pragma unroll
  for (int u = 0; u < B; ++u) st[u] = (u & 3) ? (F[u] & ~F[u - 1]) : F[u];
  uint32_t pl[NP];
#pragma unroll
  for (int b = 0; b < NP; ++b) pl[b] = p[b * 32];
  csa_add<0, NP, B>(pl, st);
#pragma unroll
  for (int b = 0; b < NP; ++b) p[b * 32] = pl[b];
}

template <int B>
__device__ __forceinline__ void count_block_reg(const uint32_t (&M)[B], CsaCounter& c) {
  uint32_t s[B];
#pragma unroll
  for (int u = 0; u < B; ++u) s[u] = (u & 3) ? (M[u] & ~M[u - 1]) : M[u];
#pragma unroll
  for (int h = 0; h + 8 <= B; h += 8) {
    uint32_t s8[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) s8[u] = s[h + u];
    c.add8(s8);
  }
  if constexpr (B % 8 == 4) {
    uint32_t s4[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) s4[u] = s[B - 4 + u];
    c.add4(s4);
  }
}

struct NoHook {
  static constexpr bool kSweep = false;
  template <int B>
  __device__ __forceinline__ void step(int, const uint32_t (&)[B]) const {}
};

template <int NP>
struct SweepHook {
  static constexpr bool kSweep = true;
  uint32_t* sm;  // this warp's counters, offset by lane: [k-1][NP][32]
  template <int B>
  __device__ __forceinline__ void step(int k, const uint32_t (&F)[B]) const {
    count_block_smem<B, NP>(sm + (k - 1) * NP * 32, F);
  }
};

// Steps k0..e of an edge block, rolled: windows and their source-validity words
// shift by register moves, one new (clamped) word and validity word per step.
template <int B, class M, class Hook>
__device__ __forceinline__ void checked_steps(const uint2* q, const Win<B>& R,
                                              const uint32_t (&tv)[B + 4], uint32_t (&F)[B],
                                              int ib, int len, int k0, int e, int edge_fix,
                                              const Hook& hook) {
  constexpr int W = B + 4;
  Win<B> D, I;
  uint32_t dv[W], iv[W], vd[B], vi[B];
  const int km = k0 - 1;
#pragma unroll
  for (int c = 0; c < W; ++c) {
    const int j = ib - 2 + c;
    const uint2 a = ldc<M>(q, j - km, len);
    const uint2 b = ldc<M>(q, j + km, len);
    D.h[c] = a.x;
    D.l[c] = a.y;
    I.h[c] = b.x;
    I.l[c] = b.y;
    dv[c] = ones_if_nonneg(j - km);
    iv[c] = ones_if_neg(j + km - len);
  }
  const uint32_t ef = edge_fix ? 0xFFFFFFFFu : 0u;
#pragma unroll
  for (int u = 0; u < B; ++u) {
    vd[u] = ef & ones_if_neg(ib + u - km);
    vi[u] = ef & ones_if_nonneg(ib + u - len + km);
  }
#pragma unroll 1
  for (int k = k0; k <= e; ++k) {
#pragma unroll
    for (int c = W - 1; c > 0; --c) {
      D.h[c] = D.h[c - 1];
      D.l[c] = D.l[c - 1];
      dv[c] = dv[c - 1];
    }
#pragma unroll
    for (int c = 0; c < W - 1; ++c) {
      I.h[c] = I.h[c + 1];
      I.l[c] = I.l[c + 1];
      iv[c] = iv[c + 1];
    }
    // vacated positions grow by one per step: [0, k) for D_k, [len-k, len) for I_k
#pragma unroll
    for (int u = B - 1; u > 0; --u) vd[u] = vd[u - 1];
#pragma unroll
    for (int u = 0; u < B - 1; ++u) vi[u] = vi[u + 1];
    const uint2 nd = ldc<M>(q, ib - 2 - k, len);
    const uint2 ni = ldc<M>(q, ib + B + 1 + k, len);
    D.h[0] = nd.x;
    D.l[0] = nd.y;
    dv[0] = ones_if_nonneg(ib - 2 - k);
    I.h[W - 1] = ni.x;
    I.l[W - 1] = ni.y;
    iv[W - 1] = ones_if_neg(ib + B + 1 + k - len);
    vd[0] = ef & ones_if_neg(ib - k);
    vi[B - 1] = ef & ones_if_nonneg(ib + B - 1 - len + k);
    mask_and_checked<B>(R, D, dv, tv, vd, F);
    mask_and_checked<B>(R, I, iv, tv, vi, F);
    hook.template step<B>(k, F);
  }
}

// One block [ib, ib+B).  R holds the reference window R[ib-2 .. ib+B+1] on entry
// (clamped loads at the edges, masked by tv) and the next block's window on exit.
template <int B, int LA, class M, class Hook>
__device__ __forceinline__ void block(const uint2* q, const uint2* r, Win<B>& R, int ib, int len,
                                      int e, int edge_fix, CsaCounter& cA, CsaCounter& cF,
                                      const Hook& hook) {
  constexpr int W = B + 4;
  uint2 rn[B];
#pragma unroll
  for (int d = 0; d < B; ++d) rn[d] = ldc<M>(r, ib + B + 2 + d, len);
  // the read words the next block's insertion masks touch for the first time
  // (positions ib+B+2+e .. ib+2B+1+e): start pulling them into L1 now
  {
    const int p0 = ib + B + 2 + e;
#pragma unroll
    for (int d = 0; d < B; ++d)
      if (p0 + d < len) M::prefetch(q, p0 + d);
  }
  const bool edge_t = (ib == 0) || (ib + B + 1 >= len);
  Win<B> Qh;
  uint32_t tv[W];
  if (edge_t) {
#pragma unroll
    for (int c = 0; c < W; ++c) {
      const int j = ib - 2 + c;
      const uint2 qv = ldc<M>(q, j, len);
      Qh.h[c] = qv.x;
      Qh.l[c] = qv.y;
      tv[c] = ones_if_nonneg(j) & ones_if_neg(j - len);
    }
  } else {
#pragma unroll
    for (int c = 0; c < W; ++c) {
      const uint2 qv = M::ld(q, ib - 2 + c);
      Qh.h[c] = qv.x;
      Qh.l[c] = qv.y;
      tv[c] = 0xFFFFFFFFu;
    }
  }
  // Hamming mask -> A0 = F at k = 0
  uint32_t F[B];
  {
    uint32_t x[W];
#pragma unroll
    for (int c = 0; c < W; ++c) x[c] = mismatch(R.h[c], R.l[c], Qh.h[c], Qh.l[c]) & tv[c];
#pragma unroll
    for (int u = 0; u < B; ++u) F[u] = amend(x[u], x[u + 1], x[u + 2], x[u + 3], x[u + 4]) & tv[u + 2];
  }
  count_block_reg<B>(F, cA);
  // steps 1..kend unchecked (all sources / targets in range, no vacated position);
  // the rest checked.  A look-ahead load is issued only while it stays in range
  // (k + LA <= ku): beyond that its step is a checked one and it is not needed.
  const int ku = edge_t ? 0 : min(ib - 2, len - ib - B - 2);
  const int kend = max(0, ku < e ? ku : e);
  if (kend > 0) {
    Win<B> D, I;
#pragma unroll
    for (int c = 0; c < W; ++c) {
      D.h[c] = I.h[c] = Qh.h[c];
      D.l[c] = I.l[c] = Qh.l[c];
    }
    uint2 qd[LA], qi[LA];
#pragma unroll
    for (int a = 0; a < LA; ++a) {
      if (a + 1 <= ku) {
        qd[a] = M::ld(q, ib - 3 - a);
        qi[a] = M::ld(q, ib + B + 2 + a);
      }
    }
#pragma unroll 1
    for (int k = 1; k <= kend; ++k) {
#pragma unroll
      for (int c = W - 1; c > 0; --c) {
        D.h[c] = D.h[c - 1];
        D.l[c] = D.l[c - 1];
      }
      D.h[0] = qd[0].x;
      D.l[0] = qd[0].y;
#pragma unroll
      for (int c = 0; c < W - 1; ++c) {
        I.h[c] = I.h[c + 1];
        I.l[c] = I.l[c + 1];
      }
      I.h[W - 1] = qi[0].x;
      I.l[W - 1] = qi[0].y;
#pragma unroll
      for (int a = 0; a < LA - 1; ++a) {
        qd[a] = qd[a + 1];
        qi[a] = qi[a + 1];
      }
      if (k + LA <= ku) {
        qd[LA - 1] = M::ld(q, ib - 2 - k - LA);
        qi[LA - 1] = M::ld(q, ib + B + 1 + k + LA);
      }
      mask_and<B>(R, D, F);
      mask_and<B>(R, I, F);
      hook.template step<B>(k, F);
    }
  }
  if (kend < e) checked_steps<B, M>(q, R, tv, F, ib, len, kend + 1, e, edge_fix, hook);
  if (!Hook::kSweep) count_block_reg<B>(F, cF);
  // slide the reference window by one block
#pragma unroll
  for (int c = 0; c < W - B; ++c) {
    R.h[c] = R.h[c + B];
    R.l[c] = R.l[c + B];
  }
#pragma unroll
  for (int d = 0; d < B; ++d) {
    R.h[W - B + d] = rn[d].x;
    R.l[W - B + d] = rn[d].y;
  }
}

template <int B, class M>
__device__ __forceinline__ void load_r0(const uint2* r, int len, Win<B>& R) {
#pragma unroll
  for (int c = 0; c < B + 4; ++c) {
    const uint2 v = ldc<M>(r, c - 2, len);
    R.h[c] = v.x;
    R.l[c] = v.y;
  }
}

}  // namespace bt2
}  // namespace gk
