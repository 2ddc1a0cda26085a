// gk_filter_core.cuh -- the per-group filtration of GateKeeper-GPU on bit-sliced words.
//
// One thread filters one GROUP of 32 pairs: every 32-bit word below carries one
// base position of those 32 pairs (bit j = pair j).  The thread streams the base
// positions i = 0..len-1 and, at each position, evaluates ALL 2e+1 masks of the
// method, so no mask is ever stored (the paper keeps 2e+1 full
// bit-vectors per thread in local memory, :85):
//
//   H   (Hamming)      x[i] = R[i] != Q[i]
//   D_k (deletion)     x[i] = R[i] != Q[i-k]   for i >= k,     0 at vacated i < k
//   I_k (insertion)    x[i] = R[i] != Q[i+k]   for i < len-k,  0 at vacated i >= len-k
//   (Q = read, R = reference segment; "read shifted by k bases", reading R1/R2)
//
// Each mask is amended at i from its raw values at i-2..i+2 (R3, gk::amend);
// GateKeeper-GPU's edge fix (:109) sets the vacated positions of D_k / I_k to 1
// AFTER amendment, which in an AND means: those positions simply do not take part
// (the vacated 0s still act as 0-neighbours during amendment).  The final word
// F[i] = A0[i] & AND_k AD_k[i] & AI_k[i]; errors are counted per 4-base window as
// run starts: start[i] = F[i] & ~F[i-1] (F[i] at a window's first base) (R6, R7).
//
// State kept in registers per thread (template E = e):
//   * a window of the read words Q[p-E .. p+E] (p = i+2 is the newest position);
//   * for each of the 2E+1 masks the raw words x[i-2], x[i-1], x[i], x[i+1];
//   * two bit-sliced carry-save counters (A0 starts -> c0, F starts -> c).
// Per position and mask: 2 LOP3 (mismatch) + 3 LOP3 (amend + AND).
#pragma once
#include "gk_common.cuh"
#include "gk_tma.cuh"

namespace gk {

// Carry-save bit-sliced counter: total = ones + 2*twos + 4*fours + 8*upper.
struct CsaCounter {
  uint32_t ones, twos, fours;
  uint32_t up[5];  // binary counter of weight-8 carries (planes 3..7)
  __host__ __device__ __forceinline__ void clear() {
    ones = twos = fours = 0u;
#pragma unroll
    for (int b = 0; b < 5; ++b) up[b] = 0u;
  }
  __host__ __device__ __forceinline__ void add_up(uint32_t s) {
#pragma unroll
    for (int b = 0; b < 5; ++b) {
      uint32_t t = up[b] & s;
      up[b] ^= s;
      s = t;
    }
  }
  __host__ __device__ __forceinline__ static void fa(uint32_t& acc, uint32_t a, uint32_t b,
                                                     uint32_t& carry) {
    carry = (acc & a) | (acc & b) | (a & b);
    acc = acc ^ a ^ b;
  }
  // one start word
  __host__ __device__ __forceinline__ void add1(uint32_t s) {
    uint32_t c = ones & s;
    ones ^= s;
    uint32_t c2 = twos & c;
    twos ^= c;
    uint32_t c3 = fours & c2;
    fours ^= c2;
    add_up(c3);
  }
  // eight start words (carry-save tree: 7 full adders + one ripple)
  __host__ __device__ __forceinline__ void add8(const uint32_t (&s)[8]) {
    uint32_t c0, c1, c2, c3, d0, d1, f0;
    fa(ones, s[0], s[1], c0);
    fa(ones, s[2], s[3], c1);
    fa(ones, s[4], s[5], c2);
    fa(ones, s[6], s[7], c3);
    fa(twos, c0, c1, d0);
    fa(twos, c2, c3, d1);
    fa(fours, d0, d1, f0);
    add_up(f0);
  }
  // four start words (3 full adders + one ripple)
  __host__ __device__ __forceinline__ void add4(const uint32_t (&s)[4]) {
    uint32_t c0, c1, d0;
    fa(ones, s[0], s[1], c0);
    fa(ones, s[2], s[3], c1);
    fa(twos, c0, c1, d0);
    const uint32_t f = fours & d0;
    fours ^= d0;
    add_up(f);
  }
  __host__ __device__ __forceinline__ void planes(uint32_t (&c)[8]) const {
    c[0] = ones;
    c[1] = twos;
    c[2] = fours;
#pragma unroll
    for (int b = 0; b < 5; ++b) c[3 + b] = up[b];
  }
};

// Read source: words of the thread's group at base position `pos`; (0,0) outside
// [0, len).  x = plane 0 (high bit), y = plane 1 (low bit).
struct GlobalGroupSrc {
  static constexpr bool kHoistLoads = true;
  const uint2* q;  // read  words of (tile, lane) at position 0; stride 32 uint2 per position
  const uint2* r;  // reference words
  int len;
  __device__ __forceinline__ uint2 ldq(int pos) const {
    return (pos >= 0 && pos < len) ? __ldg(q + (int64_t)pos * GK_WARP) : make_uint2(0u, 0u);
  }
  __device__ __forceinline__ uint2 ldr(int pos) const {
    return (pos >= 0 && pos < len) ? __ldg(r + (int64_t)pos * GK_WARP) : make_uint2(0u, 0u);
  }
  __device__ __forceinline__ uint2 ldq_nc(int pos) const { return __ldg(q + (int64_t)pos * GK_WARP); }
  __device__ __forceinline__ uint2 ldr_nc(int pos) const { return __ldg(r + (int64_t)pos * GK_WARP); }
};

template <int E>
struct SinglePass {
  static constexpr int NM = 2 * E + 1;  // mask 0 = H, 2k-1 = D_k, 2k = I_k
  static constexpr int QW = 2 * E + 1;  // Q[p-E .. p+E]
  uint32_t qh[QW], ql[QW];
  uint32_t x[NM][4];
  uint32_t fprev, aprev;
  CsaCounter cF, cA;

  __host__ __device__ __forceinline__ static constexpr int mask_k(int m) { return (m + 1) >> 1; }
  __host__ __device__ __forceinline__ static constexpr bool mask_is_d(int m) { return (m & 1) != 0; }
  __host__ __device__ __forceinline__ static constexpr int mask_q(int m) {
    return m == 0 ? E : (mask_is_d(m) ? E - mask_k(m) : E + mask_k(m));
  }

  // Window contents before the step that makes x at position p0 the newest:
  // Q[p0 - 1 - E + j] at j (j = 0 is dropped by that step).
  template <class Src>
  __host__ __device__ __forceinline__ void init(const Src& src, int p0) {
#pragma unroll
    for (int j = 0; j < QW; ++j) {
      uint2 v = src.ldq(p0 - 1 - E + j);
      qh[j] = v.x;
      ql[j] = v.y;
    }
#pragma unroll
    for (int m = 0; m < NM; ++m) x[m][0] = x[m][1] = x[m][2] = x[m][3] = 0u;
    fprev = aprev = 0u;
    cF.clear();
    cA.clear();
  }

  __host__ __device__ __forceinline__ void push_q(uint2 qn) {
#pragma unroll
    for (int j = 0; j < QW - 1; ++j) {
      qh[j] = qh[j + 1];
      ql[j] = ql[j + 1];
    }
    qh[QW - 1] = qn.x;
    ql[QW - 1] = qn.y;
  }

  // Raw mask words at position p (the newest).  CD: check the start side
  // (p >= 0, deletion vacancy p - k >= 0); CL: check the end side (p < len,
  // insertion vacancy p + k < len).  With a compile-time p (unrolled head) or
  // p = len - c (unrolled tail) these checks fold away.
  template <bool CD, bool CL>
  __host__ __device__ __forceinline__ void mismatch_all(int p, int len, uint2 rn,
                                                       uint32_t (&xn)[NM]) const {
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      const int j = mask_q(m);
      uint32_t v = mismatch(rn.x, rn.y, qh[j], ql[j]);
      bool ok = true;
      if (CD) ok = ok && (p >= 0) && (m == 0 || !mask_is_d(m) || p - mask_k(m) >= 0);
      if (CL) ok = ok && (p < len) && (m == 0 || mask_is_d(m) || p + mask_k(m) < len);
      xn[m] = ok ? v : 0u;
    }
  }

  // Priming step: only make x at p = i+2 the newest value (no finalize).
  template <bool CD, bool CL>
  __host__ __device__ __forceinline__ void prime(int i, int len, uint2 qn, uint2 rn) {
    push_q(qn);
    uint32_t xn[NM];
    mismatch_all<CD, CL>(i + 2, len, rn, xn);
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      x[m][0] = x[m][1];
      x[m][1] = x[m][2];
      x[m][2] = x[m][3];
      x[m][3] = xn[m];
    }
  }

  // Full step: x at p = i+2 becomes newest; position i is finalized.
  // notstart = ~0 unless i is the first base of a 4-base window (R7).
  // Returns the F and A0 run-start words of position i.
  template <bool CD, bool CL>
  __host__ __device__ __forceinline__ void step(int i, int len, uint2 qn, uint2 rn,
                                                uint32_t notstart, uint32_t& sF, uint32_t& sA) {
    push_q(qn);
    uint32_t xn[NM];
    mismatch_all<CD, CL>(i + 2, len, rn, xn);
    uint32_t F = 0xFFFFFFFFu, A0 = 0u;
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      const uint32_t a = amend(x[m][0], x[m][1], x[m][2], x[m][3], xn[m]);
      bool apply = true;  // edge fix: vacated positions are 1 after amendment (:109)
      if (CD && m != 0 && mask_is_d(m)) apply = i >= mask_k(m);
      if (CL && m != 0 && !mask_is_d(m)) apply = i < len - mask_k(m);
      if (m == 0) A0 = a;
      if (apply) F &= a;
      x[m][0] = x[m][1];
      x[m][1] = x[m][2];
      x[m][2] = x[m][3];
      x[m][3] = xn[m];
    }
    sF = F & ~(fprev & notstart);
    sA = A0 & ~(aprev & notstart);
    fprev = F;
    aprev = A0;
  }
};

__host__ __device__ __forceinline__ uint32_t notstart_of(int i) {
  return (i & 3) ? 0xFFFFFFFFu : 0u;
}

// Filter base positions [lo, hi) of the thread's group (lo % 4 == 0, so the
// counts of disjoint ranges add up: windows never straddle a range border).
//   * a range that starts at 0 runs a fully unrolled head [0, H) (H = E rounded
//     up to 8) in which every vacancy check of the deletion masks is a
//     compile-time constant;
//   * a range that ends at len runs a fully unrolled tail [len-E-2, len) whose
//     insertion-side checks are constants relative to len;
//   * the rest runs unchecked steps, 8 per iteration with a static carry-save
//     count tree, then up to 7 single steps.
// Short reads (or ranges that violate those assumptions) take checked steps.
template <int E, bool FULL = false, class Src>
__host__ __device__ __forceinline__ void run_range(SinglePass<E>& sp, const Src& src, int len,
                                                   int lo, int hi) {
  constexpr int H = ((E + 7) / 8) * 8;
  constexpr int T = E + 2;
  const bool head = FULL || lo == 0, tail = FULL || hi == len;
  const int mid_lo = head ? H : lo;
  const int mid_hi = tail ? len - T : hi;
  const bool fast = len >= H + T + E + 4 && mid_lo <= mid_hi && (head || lo >= E + 2) &&
                    (tail || hi <= len - T);
  if (!fast) {
    sp.init(src, lo - 2);
#pragma unroll 1
    for (int i = lo - 4; i < lo; ++i)
      sp.template prime<true, true>(i, len, src.ldq(i + 2 + E), src.ldr(i + 2));
#pragma unroll 1
    for (int i = lo; i < hi; ++i) {
      uint32_t sF, sA;
      sp.template step<true, true>(i, len, src.ldq(i + 2 + E), src.ldr(i + 2), notstart_of(i), sF,
                                   sA);
      sp.cF.add1(sF);
      sp.cA.add1(sA);
    }
    return;
  }
  sp.init(src, lo - 2);
  if (head) {
#pragma unroll
    for (int i = -4; i < 0; ++i)
      sp.template prime<true, false>(i, len, src.ldq(i + 2 + E), src.ldr(i + 2));
#pragma unroll
    for (int ib = 0; ib < H; ib += 8) {
      uint32_t sF[8], sA[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = ib + u;
        sp.template step<true, false>(i, len, src.ldq_nc(i + 2 + E), src.ldr_nc(i + 2),
                                      notstart_of(u), sF[u], sA[u]);
      }
      sp.cF.add8(sF);
      sp.cA.add8(sA);
    }
  } else {
#pragma unroll 1
    for (int i = lo - 4; i < lo; ++i)
      sp.template prime<false, false>(i, len, src.ldq_nc(i + 2 + E), src.ldr_nc(i + 2));
  }
  // unchecked middle
  const int m4 = mid_lo >> 2;
  const int n8 = (mid_hi - mid_lo) >> 3;
#pragma unroll 1
  for (int j = 0; j < n8; ++j) {
    const int ib = FULL ? H + (j << 3) : (m4 << 2) + (j << 3);
    uint32_t sF[8], sA[8];
    if constexpr (Src::kHoistLoads) {
      uint2 qn[8], rn[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        qn[u] = src.ldq_nc(ib + u + 2 + E);
        rn[u] = src.ldr_nc(ib + u + 2);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        sp.template step<false, false>(ib + u, len, qn[u], rn[u], notstart_of(u), sF[u], sA[u]);
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u)
        sp.template step<false, false>(ib + u, len, src.ldq_nc(ib + u + 2 + E),
                                       src.ldr_nc(ib + u + 2), notstart_of(u), sF[u], sA[u]);
    }
    sp.cF.add8(sF);
    sp.cA.add8(sA);
  }
#pragma unroll 1
  for (int i = mid_lo + 8 * n8; i < mid_hi; ++i) {
    uint32_t sF, sA;
    sp.template step<false, false>(i, len, src.ldq_nc(i + 2 + E), src.ldr_nc(i + 2),
                                   notstart_of(i), sF, sA);
    sp.cF.add1(sF);
    sp.cA.add1(sA);
  }
  if (tail) {
    const int i0 = len - T;
    uint32_t sF[T], sA[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int i = i0 + t;
      sp.template step<false, true>(i, len, src.ldq(i + 2 + E), t + 2 < T ? src.ldr_nc(i + 2)
                                                                          : make_uint2(0u, 0u),
                                    notstart_of(i), sF[t], sA[t]);
    }
#pragma unroll
    for (int t = 0; t < T; ++t) {
      sp.cF.add1(sF[t]);
      sp.cA.add1(sA[t]);
    }
  }
}

// Final decision of a group (Fig. S.1 :466-471, readings R5, R9):
//   early = c0 <= e  -> accept, errcount c0
//   e == 0 (no ASM)  -> reject otherwise, errcount c0
//   else             -> accept iff c <= e, errcount c
//   undefined pair   -> accept, errcount 255
__device__ __forceinline__ void finish_group(const uint32_t (&cA)[8], const uint32_t (&cF)[8],
                                             int e, uint32_t undef, int64_t g, int64_t n,
                                             uint32_t* __restrict__ accept,
                                             uint8_t* __restrict__ errc) {
  const uint32_t early = le_const(cA, e);
  uint32_t acc, err[8];
  if (e == 0) {
    acc = early;
#pragma unroll
    for (int b = 0; b < 8; ++b) err[b] = cA[b];
  } else {
    acc = early | le_const(cF, e);
#pragma unroll
    for (int b = 0; b < 8; ++b) err[b] = (early & cA[b]) | (~early & cF[b]);
  }
  acc |= undef;
#pragma unroll
  for (int b = 0; b < 8; ++b) err[b] |= undef;
  const int64_t first = g * 32;
  const int nval = (n - first) >= 32 ? 32 : (int)(n - first);
  const uint32_t vm = nval == 32 ? 0xFFFFFFFFu : ((1u << nval) - 1u);
  accept[g] = acc & vm;
  if (errc == nullptr) return;
  uint32_t bytes[8];
#pragma unroll
  for (int w = 0; w < 8; ++w) bytes[w] = count_bytes(err, w);
  if (nval == 32 && (reinterpret_cast<uintptr_t>(errc) & 15u) == 0) {
    uint4* o = reinterpret_cast<uint4*>(errc + first);
    o[0] = make_uint4(bytes[0], bytes[1], bytes[2], bytes[3]);
    o[1] = make_uint4(bytes[4], bytes[5], bytes[6], bytes[7]);
  } else {
    for (int j = 0; j < nval; ++j) errc[first + j] = (uint8_t)(bytes[j >> 2] >> (8 * (j & 3)));
  }
}

// Mask-major filtration of one group for any e (the fallback when e is above the
// register-resident instantiations): F[i] lives at F[i * fstride] (shared memory),
// the masks are visited one after the other (PAPER.md:49 loop order), each mask
// streamed over its valid positions with a 5-word window.
template <class Src>
__device__ __forceinline__ void generic_group(const Src& src, int len, int e, uint32_t undef,
                                              uint32_t* F, int fstride, uint32_t (&c0)[8],
                                              uint32_t (&cf)[8], bool edge_fix = true) {
  auto xmask = [&](int p, int shift, int lo, int hi) -> uint32_t {
    if (p < lo || p >= hi) return 0u;
    const uint2 q = src.ldq(p - shift);
    const uint2 r = src.ldr(p);
    return mismatch(r.x, r.y, q.x, q.y);
  };
  CsaCounter cA, cF;
  cA.clear();
  cF.clear();
  {  // Hamming mask -> A0 (the initial F) and its count c0
    uint32_t xm2 = 0u, xm1 = 0u, x0 = xmask(0, 0, 0, len), xp1 = xmask(1, 0, 0, len);
    uint32_t prev = 0u;
    for (int i = 0; i < len; ++i) {
      const uint32_t xp2 = xmask(i + 2, 0, 0, len);
      const uint32_t a = amend(xm2, xm1, x0, xp1, xp2);
      F[i * fstride] = a;
      cA.add1(a & ~(prev & ((i & 3) ? 0xFFFFFFFFu : 0u)));
      prev = a;
      xm2 = xm1; xm1 = x0; x0 = xp1; xp1 = xp2;
    }
  }
  cA.planes(c0);
  const uint32_t early = le_const(c0, e);
  if (e > 0 && (early | undef) != 0xFFFFFFFFu) {
    for (int k = 1; k <= e; ++k) {
      {  // deletion mask D_k: valid positions [k, len); positions < k forced to 1
         // (edge fix) -- or, original GateKeeper, left at their amended 0
        const int i0 = edge_fix ? k : 0;
        uint32_t xm2 = 0u, xm1 = 0u, x0 = xmask(i0, k, k, len), xp1 = xmask(i0 + 1, k, k, len);
        for (int i = i0; i < len; ++i) {
          const uint32_t xp2 = xmask(i + 2, k, k, len);
          F[i * fstride] &= amend(xm2, xm1, x0, xp1, xp2);
          xm2 = xm1; xm1 = x0; x0 = xp1; xp1 = xp2;
        }
      }
      {  // insertion mask I_k: valid positions [0, len-k); positions >= len-k forced to 1
        const int hi = len - k;
        const int i1 = edge_fix ? hi : len;
        uint32_t xm2 = 0u, xm1 = 0u, x0 = xmask(0, -k, 0, hi), xp1 = xmask(1, -k, 0, hi);
        for (int i = 0; i < i1; ++i) {
          const uint32_t xp2 = xmask(i + 2, -k, 0, hi);
          F[i * fstride] &= amend(xm2, xm1, x0, xp1, xp2);
          xm2 = xm1; xm1 = x0; x0 = xp1; xp1 = xp2;
        }
      }
    }
    uint32_t prev = 0u;
    for (int i = 0; i < len; ++i) {
      const uint32_t f = F[i * fstride];
      cF.add1(f & ~(prev & ((i & 3) ? 0xFFFFFFFFu : 0u)));
      prev = f;
    }
  }
  cF.planes(cf);
}

// Words of the thread's group streamed through a TMA ring in shared memory.
// Each stream (read words Q, reference words R) of the warp's tile is cut into
// blocks of 8 base positions (8 x 32 lanes x 8 B = 2 KB, contiguous in the packed
// layout); 4 ring slots per stream.  Blocks are loaded by cp.async.bulk with an
// mbarrier per slot; a lane reading the first position of a block waits for it,
// and finishing a block b releases block b-1 (long consumed) and refills its slot
// with block b+3.  Every position of a stream is read exactly once and in order
// (run_range guarantees this), so the block bookkeeping folds to constants in the
// unrolled code.
struct RingSrc {
  static constexpr bool kHoistLoads = false;
  const uint2* gq;  // tile base in global memory (uint2 units; position stride 32)
  const uint2* gr;
  uint2* sq;        // [4 slots][8 positions][32 lanes]
  uint2* sr;
  uint64_t* bq;     // 4 mbarriers per stream
  uint64_t* br;
  int len, nblk, lane;

  __device__ __forceinline__ void issue(const uint2* g, uint2* s, uint64_t* bar, int b) const {
    if (b >= nblk) return;
    const int np = (len - 8 * b) < 8 ? (len - 8 * b) : 8;
    const uint32_t bytes = (uint32_t)np * 256u;
    fence_proxy_async();
    mbar_arrive_expect_tx(&bar[b & 3], bytes);
    tma_load_1d(s + (b & 3) * 256, g + (int64_t)b * 256, bytes, &bar[b & 3]);
  }
  __device__ __forceinline__ void start() const {
    if (lane == 0) {
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        issue(gq, sq, bq, b);
        issue(gr, sr, br, b);
      }
    }
  }
  __device__ __forceinline__ uint2 rd(const uint2* g, uint2* s, uint64_t* bar, int pos) const {
    const int b = pos >> 3;
    if ((pos & 7) == 0) mbar_wait(&bar[b & 3], (uint32_t)(b >> 2) & 1u);
    const uint2 v = s[(b & 3) * 256 + (pos & 7) * 32 + lane];
    if ((pos & 7) == 7 && b >= 1) {
      __syncwarp();
      if (lane == 0) issue(g, s, bar, b + 3);
    }
    return v;
  }
  __device__ __forceinline__ uint2 ldq(int pos) const {
    return (pos >= 0 && pos < len) ? rd(gq, sq, bq, pos) : make_uint2(0u, 0u);
  }
  __device__ __forceinline__ uint2 ldr(int pos) const {
    return (pos >= 0 && pos < len) ? rd(gr, sr, br, pos) : make_uint2(0u, 0u);
  }
  __device__ __forceinline__ uint2 ldq_nc(int pos) const { return rd(gq, sq, bq, pos); }
  __device__ __forceinline__ uint2 ldr_nc(int pos) const { return rd(gr, sr, br, pos); }
};

// Words of the thread's group from a packed tile in shared memory:
// q[pos * pstride] / r[pos * pstride] (uint2 units), 0 outside [0, len).
struct SmemGroupSrc {
  static constexpr bool kHoistLoads = false;
  const uint2* q;
  const uint2* r;
  int len;
  int pstride;
  __device__ __forceinline__ uint2 ldq(int pos) const {
    return (pos >= 0 && pos < len) ? q[pos * pstride] : make_uint2(0u, 0u);
  }
  __device__ __forceinline__ uint2 ldr(int pos) const {
    return (pos >= 0 && pos < len) ? r[pos * pstride] : make_uint2(0u, 0u);
  }
  __device__ __forceinline__ uint2 ldq_nc(int pos) const { return q[pos * pstride]; }
  __device__ __forceinline__ uint2 ldr_nc(int pos) const { return r[pos * pstride]; }
};

}  // namespace gk
