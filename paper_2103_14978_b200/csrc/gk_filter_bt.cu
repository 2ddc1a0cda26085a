// gk_filter_bt.cu -- a2..a6 for any e: the block-transposed ("position block x
// mask") filtration, the kernel for e above the all-register single pass.
//
// The single pass (gk_filter_core.cuh) visits every base position once and
// evaluates all 2e+1 masks there, so it keeps 4 raw words per mask in registers:
// fine up to e = 11, impossible at e = 25 (51 masks).  Here the loop order is
// transposed inside a block of B = 8 positions [ib, ib+8):
//
//   for each block:
//     R[ib-2 .. ib+9], Q[ib-2 .. ib+9]                 (12-word windows, the
//                                                      block plus the 2-base
//                                                      amendment halo per side)
//     Hamming mask: x[c] = R[c] != Q[c]; A0 = amend(x); F = A0
//     for k = 1..e:
//       D_k: x[c] = R[c] != Q[c-k]   -> amend -> edge fix (:109) -> F &= ...
//       I_k: x[c] = R[c] != Q[c+k]   -> amend -> edge fix        -> F &= ...
//     count the window run starts of A0 and F       (:51, readings R6/R7)
//
// Only the block's F[8], the R window and two sliding read windows live in
// registers (~120 of them, independent of e).  The deletion window holds
// Q[ib-2-k .. ib+9-k]: going from k to k+1 drops one word and loads one
// (Q[ib-2-k-1]); the insertion window likewise (Q[ib+9+k+1]).  The windows are
// circular buffers whose rotation is resolved at compile time by unrolling the
// k loop in chunks of 12 steps (one full rotation), so no register moves.  The
// cost per (mask, position) cell is 5 LOP3 (2 mismatch + 3 amend/AND) plus the
// halo recomputation, 8 LOP3 per mask per block: 6 per cell at B = 8.
//
// Words come straight from global memory (coalesced: one base position of a
// tile's 32 groups is 256 contiguous bytes); every word is loaded by about
// (24 + 2e) / 8 block windows, so after the first touch they are L1 hits.
//
// Blocks whose windows reach outside [0, len) -- a vacated source of a shifted
// mask, or a position beyond the read -- run the CHECKED variant: raw words of
// vacated / outside positions are 0 (readings R2, R13), vacated positions are
// forced to 1 after amendment (edge fix, R4) unless edge_fix == 0 (original
// GateKeeper), and positions >= len take no part.
#include "gk_common.cuh"
#include "gk_filter_core.cuh"
#include "gk_kernels.cuh"

namespace gk {

namespace bt {

constexpr int B = 8;       // positions per block
constexpr int W = B + 4;   // window words (block + 2-base halo on each side)

struct Win {
  uint32_t h[W], l[W];
};

// One shifted mask of step k in an interior (unchecked) block.  The window
// word of logical index c (target position j = ib-2+c) sits at physical index
// (c -/+ ROT) mod W: the rotation is a compile-time constant.
template <int ROT, bool IS_D>
__device__ __forceinline__ void shifted_mask(const Win& R, const Win& Qw, uint32_t (&F)[B]) {
  uint32_t x[W];
#pragma unroll
  for (int c = 0; c < W; ++c) {
    const int p = IS_D ? (c - ROT + W) % W : (c + ROT) % W;
    x[c] = mismatch(R.h[c], R.l[c], Qw.h[p], Qw.l[p]);
  }
#pragma unroll
  for (int u = 0; u < B; ++u) F[u] &= amend(x[u], x[u + 1], x[u + 2], x[u + 3], x[u + 4]);
}

// One shifted mask of step k in an edge block (logical = physical window).
// Raw word of cell c = mismatch & sv[c] & tv[c]: sv = the source is not
// vacated (a plane that shifts with the window), tv = the target lies in
// [0, len) (fixed per cell) -- readings R2 / R13.  vac[u] = ~0 iff position
// ib+u is vacated by this shift: forced to 1 after amendment (edge fix,
// PAPER.md:109; 0 for the original GateKeeper).
__device__ __forceinline__ void shifted_mask_checked(const Win& R, const Win& Qw,
                                                     const uint32_t (&sv)[W],
                                                     const uint32_t (&tv)[W],
                                                     const uint32_t (&vac)[B], uint32_t (&F)[B]) {
  uint32_t x[W];
#pragma unroll
  for (int c = 0; c < W; ++c) x[c] = mismatch(R.h[c], R.l[c], Qw.h[c], Qw.l[c]) & sv[c] & tv[c];
#pragma unroll
  for (int u = 0; u < B; ++u) F[u] &= amend(x[u], x[u + 1], x[u + 2], x[u + 3], x[u + 4]) | vac[u];
}

// All-ones iff x >= 0 / x < 0, as data (a sign spread, not a predicate: the
// validity planes below are shifted as words and ANDed into LOP3s).
// (PRMT with sign replication: ptxas keeps these as words instead of turning the
// ANDs with them into predicated selects.)
__device__ __forceinline__ uint32_t ones_if_neg(int x) { return __byte_perm((uint32_t)x, 0u, 0xBBBB); }
__device__ __forceinline__ uint32_t ones_if_nonneg(int x) { return ones_if_neg(~x); }

__device__ __forceinline__ uint2 ldc(const uint2* p, int pos, int len) {
  return __ldg(p + (int64_t)(pos < 0 ? 0 : (pos >= len ? len - 1 : pos)) * GK_WARP);
}
__device__ __forceinline__ void prefetch_l1(const uint2* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
// The unchecked steps keep each read window in a ring of W+1 = 13 registers:
// the window of step k occupies 12 of them and the 13th is free, so the word of
// step k+1 is loaded into it one step ahead (no register moves, no load-use
// stall).  Logical cell c (target ib-2+c) of the deletion window sits in
// physical slot (c - tau) mod 13 after tau steps, of the insertion window in
// (c + tau) mod 13; 13 steps are one full rotation.
constexpr int W1 = W + 1;
struct Ring {
  uint32_t h[W1], l[W1];
};

template <int ROT, bool IS_D>
__device__ __forceinline__ void shifted_mask13(const Win& R, const Ring& Qw, uint32_t (&F)[B]) {
  uint32_t x[W];
#pragma unroll
  for (int c = 0; c < W; ++c) {
    const int p = IS_D ? (c - ROT + W1) % W1 : (c + ROT) % W1;
    x[c] = mismatch(R.h[c], R.l[c], Qw.h[p], Qw.l[p]);
  }
#pragma unroll
  for (int u = 0; u < B; ++u) F[u] &= amend(x[u], x[u + 1], x[u + 2], x[u + 3], x[u + 4]);
}

// Steps k = k0 .. min(k0+12, kend).  On entry the free slot 12 (rotation 0)
// holds the words of step k0; qd / qi point at Q[ib-2-k0] / Q[ib+9+k0] of this
// lane.  Step k loads the words of step k+1 (<= kend+1, in range: block()
// keeps kend below the first checked step).
template <class Hook>
__device__ __forceinline__ void chunk(const uint2* qd, const uint2* qi, const Win& R, Ring& D,
                                      Ring& I, uint32_t (&F)[B], int k0, int kend,
                                      const Hook& hook) {
#define GK_BT_STEP(T)                                                                  \
  if (k0 + (T) <= kend) {                                                              \
    const uint2 nd = __ldg(qd - 32 * ((T) + 1));                                       \
    const uint2 ni = __ldg(qi + 32 * ((T) + 1));                                       \
    D.h[(W1 + W - 1 - (T)) % W1] = nd.x;                                               \
    D.l[(W1 + W - 1 - (T)) % W1] = nd.y;                                               \
    I.h[(T) % W1] = ni.x;                                                              \
    I.l[(T) % W1] = ni.y;                                                              \
    shifted_mask13<((T) + 1) % W1, true>(R, D, F);                                     \
    shifted_mask13<((T) + 1) % W1, false>(R, I, F);                                    \
    hook(k0 + (T), F);                                                                 \
  } else {                                                                             \
    return;                                                                            \
  }
  GK_BT_STEP(0) GK_BT_STEP(1) GK_BT_STEP(2) GK_BT_STEP(3) GK_BT_STEP(4) GK_BT_STEP(5)
  GK_BT_STEP(6) GK_BT_STEP(7) GK_BT_STEP(8) GK_BT_STEP(9) GK_BT_STEP(10) GK_BT_STEP(11)
  GK_BT_STEP(12)
#undef GK_BT_STEP
}
static_assert(W1 == 13, "chunk() unrolls one full rotation of the 13-slot ring");

// Steps k = k0..e of an edge block, rolled (compact code): the windows and
// their source-validity planes shift by register moves (FMA-pipe IMAD.MOV),
// one new word and one validity word enter per step.
template <class Hook>
__device__ __forceinline__ void checked_steps(const uint2* q, const Win& R, const uint32_t (&tv)[W],
                                              uint32_t (&F)[B], int ib, int len, int k0, int e,
                                              int edge_fix, const Hook& hook) {
  // windows of step k0-1 in logical layout
  Win D, I;
  uint32_t dv[W], iv[W], vd[B], vi[B];
  const int km = k0 - 1;
#pragma unroll
  for (int c = 0; c < W; ++c) {
    const int j = ib - 2 + c;
    const uint2 a = ldc(q, j - km, len);
    const uint2 b = ldc(q, j + km, len);
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
    const uint2 nd = ldc(q, ib - 2 - k, len);
    const uint2 ni = ldc(q, ib + B + 1 + k, len);
    D.h[0] = nd.x;
    D.l[0] = nd.y;
    dv[0] = ones_if_nonneg(ib - 2 - k);
    I.h[W - 1] = ni.x;
    I.l[W - 1] = ni.y;
    iv[W - 1] = ones_if_neg(ib + B + 1 + k - len);
    vd[0] = ef & ones_if_neg(ib - k);  // the prefix [0, k-ib) grows at its top
    vi[B - 1] = ef & ones_if_nonneg(ib + B - 1 - len + k);
    shifted_mask_checked(R, D, dv, tv, vd, F);
    shifted_mask_checked(R, I, iv, tv, vi, F);
    hook(k, F);
  }
}

__device__ __forceinline__ void count_starts(const uint32_t (&M)[B], uint32_t& prev, CsaCounter& c) {
  // window run starts (R6, R7; ib % 8 == 0 so position ib+u starts a 4-base
  // window iff u % 4 == 0)
  uint32_t s[B];
#pragma unroll
  for (int u = 0; u < B; ++u) {
    s[u] = M[u] & ~(prev & notstart_of(u));
    prev = M[u];
  }
  c.add8(s);
}

// One block [ib, ib+B).  R holds the reference window R[ib-2 .. ib+9] on entry
// (edge blocks: clamped loads, masked by tv) and R[ib+6 .. ib+17] on exit; the
// 8 new words of the next window are loaded at entry, a whole block ahead of use.
template <class Hook>
__device__ __forceinline__ void block(const uint2* q, const uint2* r, Win& R, int ib, int len,
                                      int e, int edge_fix, CsaCounter& cA, CsaCounter& cF,
                                      uint32_t& aprev, uint32_t& fprev, const Hook& hook) {
  uint2 rn[B];
#pragma unroll
  for (int d = 0; d < B; ++d) rn[d] = ldc(r, ib + B + 2 + d, len);
  // the words the next block's insertion masks touch first: pull them into L1
  {
    const int p0 = ib + B + 2 + e;
    const uint2* pq = q + (int64_t)p0 * GK_WARP;
#pragma unroll
    for (int d = 0; d < B; ++d)
      if (p0 + d < len) prefetch_l1(pq + 32 * d);
  }
  // target positions outside [0, len) in the window: only the first and last blocks
  const bool edge_t = (ib == 0) || (ib + B + 1 >= len);
  Win Qh;
  uint32_t tv[W];
  if (edge_t) {
#pragma unroll
    for (int c = 0; c < W; ++c) {
      const int j = ib - 2 + c;
      const uint2 qv = ldc(q, j, len);
      Qh.h[c] = qv.x;
      Qh.l[c] = qv.y;
      tv[c] = ones_if_nonneg(j) & ones_if_neg(j - len);
    }
  } else {
    const uint2* qb = q + (int64_t)(ib - 2) * GK_WARP;
#pragma unroll
    for (int c = 0; c < W; ++c) {
      const uint2 qv = __ldg(qb + 32 * c);
      Qh.h[c] = qv.x;
      Qh.l[c] = qv.y;
      tv[c] = 0xFFFFFFFFu;
    }
  }
  // Hamming mask: raw words, amended -> A0; F starts as A0
  uint32_t F[B], A[B];
  {
    uint32_t x[W];
#pragma unroll
    for (int c = 0; c < W; ++c) x[c] = mismatch(R.h[c], R.l[c], Qh.h[c], Qh.l[c]) & tv[c];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      // positions >= len take no part (only the last block has any)
      A[u] = amend(x[u], x[u + 1], x[u + 2], x[u + 3], x[u + 4]) & tv[u + 2];
      F[u] = A[u];
    }
  }
  count_starts(A, aprev, cA);
  // shifted masks: steps k <= ku touch no vacated source, no vacated position
  // and no position outside [0, len): they run unchecked, both windows starting
  // as the Hamming window (k = 0); the rest run checked
  // (one step short of ku: the ring loads one step ahead and stays in range)
  const int ku = edge_t ? 0 : min(ib - 2, len - ib - B - 2) - 1;
  const int kend = max(0, ku < e ? ku : e);  // ku < 0 near the end: all steps checked
  if (kend > 0) {
    Ring D, I;
#pragma unroll
    for (int c = 0; c < W; ++c) {
      D.h[c] = I.h[c] = Qh.h[c];
      D.l[c] = I.l[c] = Qh.l[c];
    }
    const uint2* qd = q + (int64_t)(ib - 2) * GK_WARP;
    const uint2* qi = q + (int64_t)(ib + B + 1) * GK_WARP;
    {
      const uint2 a = __ldg(qd - 32), b = __ldg(qi + 32);
      D.h[W] = a.x;
      D.l[W] = a.y;
      I.h[W] = b.x;
      I.l[W] = b.y;
    }
#pragma unroll 1
    for (int k0 = 1; k0 <= kend; k0 += W1)
      chunk(qd - 32 * k0, qi + 32 * k0, R, D, I, F, k0, kend, hook);
  }
  if (kend < e) checked_steps(q, R, tv, F, ib, len, kend + 1, e, edge_fix, hook);
  if (!Hook::kSweep) count_starts(F, fprev, cF);
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

// Per-k hooks of block(): called with the block's F words once step k is ANDed
// in, i.e. with F_k = A0 & AND_{j<=k} (A*D_j & A*I_j).
struct NoHook {
  static constexpr bool kSweep = false;
  __device__ __forceinline__ void operator()(int, const uint32_t (&)[B]) const {}
};

// Threshold sweep: F_e of every e <= e_max is a prefix
// of the same AND chain, so one pass counts all of them.  The counter of F_k
// (NP bit-sliced planes, NP = the bits of the largest count 2*ceil(L/4): 6 at
// 100 bp, 7 at 150 / 250 bp) lives in shared memory, [k-1][NP][32 lanes]:
// bank = lane, conflict-free.
// Out of line: the 13-step unrolled chunk would otherwise carry 13 copies of
// the counting code (instruction-cache pressure, measured: stall_no_instruction).
template <int NP>
__device__ __noinline__ void sweep_count(uint32_t* p, uint32_t f0, uint32_t f1, uint32_t f2,
                                         uint32_t f3, uint32_t f4, uint32_t f5, uint32_t f6,
                                         uint32_t f7) {
  // windows start at positions ib and ib+4 (ib % 8 == 0): run starts never
  // depend on the previous block (R6, R7)
  uint32_t st[B];
  st[0] = f0;
  st[1] = f1 & ~f0;
  st[2] = f2 & ~f1;
  st[3] = f3 & ~f2;
  st[4] = f4;
  st[5] = f5 & ~f4;
  st[6] = f6 & ~f5;
  st[7] = f7 & ~f6;
  uint32_t ones = p[0], twos = p[32], fours = p[64], up[NP - 3];
#pragma unroll
  for (int b = 0; b < NP - 3; ++b) up[b] = p[(3 + b) * 32];
  // carry-save tree: 7 full adders, then the weight-8 carry ripples upwards
  uint32_t c0, c1, c2, c3, d0, d1, f;
  CsaCounter::fa(ones, st[0], st[1], c0);
  CsaCounter::fa(ones, st[2], st[3], c1);
  CsaCounter::fa(ones, st[4], st[5], c2);
  CsaCounter::fa(ones, st[6], st[7], c3);
  CsaCounter::fa(twos, c0, c1, d0);
  CsaCounter::fa(twos, c2, c3, d1);
  CsaCounter::fa(fours, d0, d1, f);
#pragma unroll
  for (int b = 0; b < NP - 3; ++b) {
    const uint32_t t = up[b] & f;
    up[b] ^= f;
    f = t;
  }
  p[0] = ones;
  p[32] = twos;
  p[64] = fours;
#pragma unroll
  for (int b = 0; b < NP - 3; ++b) p[(3 + b) * 32] = up[b];
}

template <int NP>
struct SweepHook {
  static constexpr bool kSweep = true;
  uint32_t* sm;  // this warp's counters, already offset by lane
  __device__ __forceinline__ void operator()(int k, const uint32_t (&F)[B]) const {
    sweep_count<NP>(sm + (k - 1) * NP * 32, F[0], F[1], F[2], F[3], F[4], F[5], F[6], F[7]);
  }
};

}  // namespace bt

__global__ void __launch_bounds__(128, 3) filter_bt_kernel(
    const uint2* __restrict__ reads, const uint2* __restrict__ refs,
    const uint32_t* __restrict__ rund, const uint32_t* __restrict__ fund, int64_t n, int len, int e,
    uint32_t* __restrict__ accept, uint8_t* __restrict__ errc, int edge_fix) {
  const int lane = threadIdx.x & 31;
  const int64_t tile = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t g = tile * 32 + lane;
  if (tile * 1024 >= n) return;
  const uint2* q = reads + tile * (int64_t)len * 32 + lane;
  const uint2* r = refs + tile * (int64_t)len * 32 + lane;
  CsaCounter cA, cF;
  cA.clear();
  cF.clear();
  uint32_t aprev = 0u, fprev = 0u;
  bt::Win R;
#pragma unroll
  for (int c = 0; c < bt::W; ++c) {
    const uint2 v = bt::ldc(r, c - 2, len);
    R.h[c] = v.x;
    R.l[c] = v.y;
  }
#pragma unroll 1
  for (int ib = 0; ib < len; ib += bt::B) {
    bt::block(q, r, R, ib, len, e, edge_fix, cA, cF, aprev, fprev, bt::NoHook{});
  }
  uint32_t a[8], f[8];
  cA.planes(a);
  cF.planes(f);
  if (g * 32 < n) finish_group(a, f, e, __ldg(rund + g) | __ldg(fund + g), g, n, accept, errc);
}

void launch_bt(const uint2* reads, const uint2* refs, const uint32_t* rund, const uint32_t* fund,
               int64_t n, int len, int e, uint32_t* accept, uint8_t* errc, int edge_fix,
               cudaStream_t stream) {
  const int64_t tiles = (n + 1023) / 1024;
  const int warps = 4;
  const int64_t blocks = (tiles + warps - 1) / warps;
  // no shared memory: give the whole unified L1 to the read windows' reuse
  cudaFuncSetAttribute(filter_bt_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
  count_launch();
  filter_bt_kernel<<<(unsigned)blocks, warps * 32, 0, stream>>>(reads, refs, rund, fund, n, len, e,
                                                                 accept, errc, edge_fix);
}

// a2-a6 for every e in [0, e_max] in one pass (gk_filter_sweep): the k loop of
// each block runs to e_max and the hook counts F_k after every step; the
// decision for e uses c0 (the Hamming-stage count, readings R5/R9) and count(F_e).
constexpr int SWEEP_WARPS = 2;
// minimum resident CTAs per SM requested from ptxas for the sweep (A/B knob)
#ifndef GK_SWEEP_MINB
#define GK_SWEEP_MINB 5
#endif

template <int NP>
__global__ void __launch_bounds__(SWEEP_WARPS * 32, GK_SWEEP_MINB) filter_bt_sweep_kernel(
    const uint2* __restrict__ reads, const uint2* __restrict__ refs,
    const uint32_t* __restrict__ rund, const uint32_t* __restrict__ fund, int64_t n, int len,
    int emax, uint32_t* __restrict__ accept, uint8_t* __restrict__ errc, int edge_fix) {
  extern __shared__ uint32_t sm_sweep[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t tile = (int64_t)blockIdx.x * SWEEP_WARPS + warp;
  const int64_t g = tile * 32 + lane;
  if (tile * 1024 >= n) return;
  uint32_t* mine = sm_sweep + (size_t)warp * emax * NP * 32 + lane;
  for (int j = 0; j < emax * NP; ++j) mine[j * 32] = 0u;
  const uint2* q = reads + tile * (int64_t)len * 32 + lane;
  const uint2* r = refs + tile * (int64_t)len * 32 + lane;
  CsaCounter cA, cF;
  cA.clear();
  cF.clear();
  uint32_t aprev = 0u, fprev = 0u;
  bt::Win R;
#pragma unroll
  for (int c = 0; c < bt::W; ++c) {
    const uint2 v = bt::ldc(r, c - 2, len);
    R.h[c] = v.x;
    R.l[c] = v.y;
  }
  const bt::SweepHook<NP> hook{mine};
#pragma unroll 1
  for (int ib = 0; ib < len; ib += bt::B) {
    bt::block(q, r, R, ib, len, emax, edge_fix, cA, cF, aprev, fprev, hook);
  }
  if (g * 32 >= n) return;
  uint32_t a[8], f[8];
  cA.planes(a);
  const uint32_t und = __ldg(rund + g) | __ldg(fund + g);
  const int64_t words = (n + 31) / 32;
#pragma unroll 1
  for (int e = 0; e <= emax; ++e) {
    if (e == 0) {
#pragma unroll
      for (int b = 0; b < 8; ++b) f[b] = a[b];
    } else {
      const uint32_t* p = mine + (e - 1) * NP * 32;
#pragma unroll
      for (int b = 0; b < 8; ++b) f[b] = b < NP ? p[b * 32] : 0u;
    }
    finish_group(a, f, e, und, g, n, accept + e * words, errc ? errc + e * n : nullptr);
  }
}

template <int NP>
static void launch_sweep_np(const uint2* reads, const uint2* refs, const uint32_t* rund,
                            const uint32_t* fund, int64_t n, int len, int emax, uint32_t* accept,
                            uint8_t* errc, int edge_fix, cudaStream_t stream) {
  const int64_t tiles = (n + 1023) / 1024;
  const int64_t blocks = (tiles + SWEEP_WARPS - 1) / SWEEP_WARPS;
  const size_t smem = (size_t)SWEEP_WARPS * emax * NP * 32 * 4;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(filter_bt_sweep_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  count_launch();
  filter_bt_sweep_kernel<NP><<<(unsigned)blocks, SWEEP_WARPS * 32, smem, stream>>>(
      reads, refs, rund, fund, n, len, emax, accept, errc, edge_fix);
}

void launch_bt_sweep(const uint2* reads, const uint2* refs, const uint32_t* rund,
                     const uint32_t* fund, int64_t n, int len, int emax, uint32_t* accept,
                     uint8_t* errc, int edge_fix, cudaStream_t stream) {
  // counter planes: enough bits for the largest count, 2 * ceil(len / 4) (R6, R7)
  const int maxc = 2 * ((len + 3) / 4);
  if (maxc < 64)
    launch_sweep_np<6>(reads, refs, rund, fund, n, len, emax, accept, errc, edge_fix, stream);
  else if (maxc < 128)
    launch_sweep_np<7>(reads, refs, rund, fund, n, len, emax, accept, errc, edge_fix, stream);
  else
    launch_sweep_np<8>(reads, refs, rund, fund, n, len, emax, accept, errc, edge_fix, stream);
}

}  // namespace gk
