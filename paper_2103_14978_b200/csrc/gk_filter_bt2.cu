// gk_filter_bt2.cu -- a2..a6 for any e, block-transposed, with a compact rolled
// k loop: the kernels behind gk_filter for e above the all-register single pass
// and behind gk_filter_sweep (every e <= e_max in one pass).
//
// Loop order (as gk_filter_bt.cu): per block of B positions [ib, ib+B) of a
// tile, the Hamming mask, then for k = 1..e the deletion and insertion masks of
// the block (W = B+4 cells: the block plus the 2-base amendment halo on each
// side), ANDed into the block's B words of F:
//
//   H   x[c] = R[j] != Q[j]          D_k  x[c] = R[j] != Q[j-k]
//   I_k x[c] = R[j] != Q[j+k]        (j = ib-2+c; Q = read, R = reference)
//
// What differs from gk_filter_bt.cu (round 1, 13-step unrolled register ring +
// an out-of-line per-k counter): the two read windows slide by plain register
// moves inside a ROLLED k loop -- the moves issue on the FMA pipe (IMAD.MOV)
// while the ALU pipe (LOP3) is the bottleneck, so they are nearly free, and the
// loop body (~200 instructions) fits the 6 KB L0 instruction cache; the per-k
// run counter of the sweep is inline.  The new word of each window is loaded LA
// steps ahead through a small register queue.  ncu of the round-1 kernel:
// stall_no_instruction 20% of samples, CALL/RET hot; LOP3 1.29x the model.
//
// Blocks whose steps would touch a vacated source, a vacated position or a
// target outside [0, len) run those steps CHECKED (rolled, validity words per
// cell, readings R2 / R4 / R13), exactly as gk_filter_bt.cu.
#include "gk_common.cuh"
#include "gk_filter_core.cuh"
#include "gk_kernels.cuh"

namespace gk {
namespace bt2 {

#ifndef GK_BT2_LA
#define GK_BT2_LA 2
#endif
constexpr int LA = GK_BT2_LA;  // load look-ahead (steps)

__device__ __forceinline__ uint32_t ones_if_neg(int x) { return __byte_perm((uint32_t)x, 0u, 0xBBBB); }
__device__ __forceinline__ uint32_t ones_if_nonneg(int x) { return ones_if_neg(~x); }

// word of (tile, lane) at position pos, clamped into [0, len) (checked paths only)
__device__ __forceinline__ uint2 ldc(const uint2* p, int pos, int len) {
  return __ldg(p + (int64_t)(pos < 0 ? 0 : (pos >= len ? len - 1 : pos)) * GK_WARP);
}
__device__ __forceinline__ uint2 ld(const uint2* p, int pos) {
  return __ldg(p + (int64_t)pos * GK_WARP);
}
__device__ __forceinline__ void prefetch_l1(const uint2* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
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
  // carry-save tree: B words into planes 0..; the carries ripple upwards
  uint32_t c1[B / 2];
#pragma unroll
  for (int i = 0; i < B / 2; ++i) CsaCounter::fa(pl[0], st[2 * i], st[2 * i + 1], c1[i]);
  uint32_t c2[B / 4];
#pragma unroll
  for (int i = 0; i < B / 4; ++i) CsaCounter::fa(pl[1], c1[2 * i], c1[2 * i + 1], c2[i]);
  uint32_t f;
  if constexpr (B == 8) {
    CsaCounter::fa(pl[2], c2[0], c2[1], f);
#pragma unroll
    for (int b = 3; b < NP; ++b) {
      const uint32_t t = pl[b] & f;
      pl[b] ^= f;
      f = t;
    }
  } else {  // B == 16
    uint32_t c3[2];
    CsaCounter::fa(pl[2], c2[0], c2[1], c3[0]);
    CsaCounter::fa(pl[2], c2[2], c2[3], c3[1]);
    CsaCounter::fa(pl[3], c3[0], c3[1], f);
#pragma unroll
    for (int b = 4; b < NP; ++b) {
      const uint32_t t = pl[b] & f;
      pl[b] ^= f;
      f = t;
    }
  }
#pragma unroll
  for (int b = 0; b < NP; ++b) p[b * 32] = pl[b];
}

template <int B>
__device__ __forceinline__ void count_block_reg(const uint32_t (&M)[B], CsaCounter& c) {
  uint32_t s[B];
#pragma unroll
  for (int u = 0; u < B; ++u) s[u] = (u & 3) ? (M[u] & ~M[u - 1]) : M[u];
#pragma unroll
  for (int h = 0; h < B; h += 8) {
    uint32_t s8[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) s8[u] = s[h + u];
    c.add8(s8);
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
template <int B, class Hook>
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
    vd[0] = ef & ones_if_neg(ib - k);
    vi[B - 1] = ef & ones_if_nonneg(ib + B - 1 - len + k);
    mask_and_checked<B>(R, D, dv, tv, vd, F);
    mask_and_checked<B>(R, I, iv, tv, vi, F);
    hook.template step<B>(k, F);
  }
}

// One block [ib, ib+B).  R holds the reference window R[ib-2 .. ib+B+1] on entry
// (clamped loads at the edges, masked by tv) and the next block's window on exit.
template <int B, class Hook>
__device__ __forceinline__ void block(const uint2* q, const uint2* r, Win<B>& R, int ib, int len,
                                      int e, int edge_fix, CsaCounter& cA, CsaCounter& cF,
                                      const Hook& hook) {
  constexpr int W = B + 4;
  uint2 rn[B];
#pragma unroll
  for (int d = 0; d < B; ++d) rn[d] = ldc(r, ib + B + 2 + d, len);
  // the read words the next block's insertion masks touch for the first time
  // (positions ib+B+2+e .. ib+2B+1+e): start pulling them into L1 now
  {
    const int p0 = ib + B + 2 + e;
#pragma unroll
    for (int d = 0; d < B; ++d)
      if (p0 + d < len) prefetch_l1(q + (int64_t)(p0 + d) * GK_WARP);
  }
  const bool edge_t = (ib == 0) || (ib + B + 1 >= len);
  Win<B> Qh;
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
#pragma unroll
    for (int c = 0; c < W; ++c) {
      const uint2 qv = ld(q, ib - 2 + c);
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
        qd[a] = ld(q, ib - 3 - a);
        qi[a] = ld(q, ib + B + 2 + a);
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
        qd[LA - 1] = ld(q, ib - 2 - k - LA);
        qi[LA - 1] = ld(q, ib + B + 1 + k + LA);
      }
      mask_and<B>(R, D, F);
      mask_and<B>(R, I, F);
      hook.template step<B>(k, F);
    }
  }
  if (kend < e) checked_steps<B>(q, R, tv, F, ib, len, kend + 1, e, edge_fix, hook);
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

template <int B>
__device__ __forceinline__ void load_r0(const uint2* r, int len, Win<B>& R) {
#pragma unroll
  for (int c = 0; c < B + 4; ++c) {
    const uint2 v = ldc(r, c - 2, len);
    R.h[c] = v.x;
    R.l[c] = v.y;
  }
}

}  // namespace bt2

#ifndef GK_BT2_B
#define GK_BT2_B 8
#endif
#ifndef GK_BT2_MINB
#define GK_BT2_MINB 3
#endif
#ifndef GK_BT2_SWEEP_MINB
#define GK_BT2_SWEEP_MINB 6
#endif

template <int B>
__global__ void __launch_bounds__(128, GK_BT2_MINB) filter_bt2_kernel(
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
  bt2::Win<B> R;
  bt2::load_r0<B>(r, len, R);
#pragma unroll 1
  for (int ib = 0; ib < len; ib += B)
    bt2::block<B>(q, r, R, ib, len, e, edge_fix, cA, cF, bt2::NoHook{});
  uint32_t a[8], f[8];
  cA.planes(a);
  cF.planes(f);
  if (g * 32 < n) finish_group(a, f, e, __ldg(rund + g) | __ldg(fund + g), g, n, accept, errc);
}

constexpr int BT2_SWEEP_WARPS = 2;

template <int B, int NP>
__global__ void __launch_bounds__(BT2_SWEEP_WARPS * 32, GK_BT2_SWEEP_MINB) filter_bt2_sweep_kernel(
    const uint2* __restrict__ reads, const uint2* __restrict__ refs,
    const uint32_t* __restrict__ rund, const uint32_t* __restrict__ fund, int64_t n, int len,
    int emax, uint32_t* __restrict__ accept, uint8_t* __restrict__ errc, int edge_fix) {
  extern __shared__ uint32_t sm_sweep2[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t tile = (int64_t)blockIdx.x * BT2_SWEEP_WARPS + warp;
  const int64_t g = tile * 32 + lane;
  if (tile * 1024 >= n) return;
  uint32_t* mine = sm_sweep2 + (size_t)warp * emax * NP * 32 + lane;
  for (int j = 0; j < emax * NP; ++j) mine[j * 32] = 0u;
  const uint2* q = reads + tile * (int64_t)len * 32 + lane;
  const uint2* r = refs + tile * (int64_t)len * 32 + lane;
  CsaCounter cA, cF;
  cA.clear();
  cF.clear();
  bt2::Win<B> R;
  bt2::load_r0<B>(r, len, R);
  const bt2::SweepHook<NP> hook{mine};
#pragma unroll 1
  for (int ib = 0; ib < len; ib += B)
    bt2::block<B>(q, r, R, ib, len, emax, edge_fix, cA, cF, hook);
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

void launch_bt2(const uint2* reads, const uint2* refs, const uint32_t* rund, const uint32_t* fund,
                int64_t n, int len, int e, uint32_t* accept, uint8_t* errc, int edge_fix,
                cudaStream_t stream) {
  constexpr int B = GK_BT2_B;
  const int64_t tiles = (n + 1023) / 1024;
  const int warps = 4;
  const int64_t blocks = (tiles + warps - 1) / warps;
  static thread_local bool attr_set = false;  // L1 carveout: once per thread
  if (!attr_set) {
    cudaFuncSetAttribute(filter_bt2_kernel<B>, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
    attr_set = true;
  }
  count_launch();
  filter_bt2_kernel<B><<<(unsigned)blocks, warps * 32, 0, stream>>>(reads, refs, rund, fund, n,
                                                                    len, e, accept, errc, edge_fix);
}

template <int NP>
static void launch_bt2_sweep_np(const uint2* reads, const uint2* refs, const uint32_t* rund,
                                const uint32_t* fund, int64_t n, int len, int emax,
                                uint32_t* accept, uint8_t* errc, int edge_fix,
                                cudaStream_t stream) {
  constexpr int B = GK_BT2_B;
  const int64_t tiles = (n + 1023) / 1024;
  const int64_t blocks = (tiles + BT2_SWEEP_WARPS - 1) / BT2_SWEEP_WARPS;
  const size_t smem = (size_t)BT2_SWEEP_WARPS * emax * NP * 32 * 4;
  static thread_local size_t attr_smem = 0;
  if (smem > 48 * 1024 && smem > attr_smem) {
    cudaFuncSetAttribute(filter_bt2_sweep_kernel<B, NP>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_smem = smem;
  }
  count_launch();
  filter_bt2_sweep_kernel<B, NP><<<(unsigned)blocks, BT2_SWEEP_WARPS * 32, smem, stream>>>(
      reads, refs, rund, fund, n, len, emax, accept, errc, edge_fix);
}

void launch_bt2_sweep(const uint2* reads, const uint2* refs, const uint32_t* rund,
                      const uint32_t* fund, int64_t n, int len, int emax, uint32_t* accept,
                      uint8_t* errc, int edge_fix, cudaStream_t stream) {
  // counter planes: enough bits for the largest count, 2 * ceil(len / 4) (R6, R7)
  const int maxc = 2 * ((len + 3) / 4);
  if (maxc < 64)
    launch_bt2_sweep_np<6>(reads, refs, rund, fund, n, len, emax, accept, errc, edge_fix, stream);
  else if (maxc < 128)
    launch_bt2_sweep_np<7>(reads, refs, rund, fund, n, len, emax, accept, errc, edge_fix, stream);
  else
    launch_bt2_sweep_np<8>(reads, refs, rund, fund, n, len, emax, accept, errc, edge_fix, stream);
}

}  // namespace gk
