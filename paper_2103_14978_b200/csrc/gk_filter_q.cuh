// gk_filter_q.cuh -- filtration for large e (GK_SP_EMAX < e <= GK_SPQ_EMAX).
//
// The 2e+1 masks of a tile are split across TWO warps (mask split): warp A owns
// the Hamming mask and the shifted masks k = 1..KA, warp B the masks
// k = KA+1..E.  Both warps stream the same base positions in lockstep, in blocks
// of 8 positions; each keeps the 4 raw-word windows of its own masks in
// registers (the per-position evaluation is the one of SinglePass<E>,
// gk_filter_core.cuh) and reads the read / reference words from one TMA ring
// in shared memory shared by the pair (16 slots x 8 positions for Q, 4 for R;
// the ring index of position pos is pos & 127).  Per block, warp B writes its
// partial AND of the 8 positions to shared memory, a named barrier pairs the
// two warps, warp A combines F = F_A & F_B, counts the window run starts and
// refills the ring slots that neither warp needs any more.
// Blocks whose positions touch a vacated or out-of-range base are evaluated
// with run-time checks; the others are unchecked (all masks valid).
#pragma once
#include "gk_filter_core.cuh"
#include "gk_tma.cuh"

namespace gk {

constexpr int QR_SLOTS = 16;  // Q ring: 16 x 8 positions
constexpr int RR_SLOTS = 4;   // R ring
constexpr int QR_BYTES = QR_SLOTS * 8 * 32 * 8;
constexpr int RR_BYTES = RR_SLOTS * 8 * 32 * 8;
constexpr int XB_BYTES = 2 * 8 * 32 * 4;  // double-buffered partial-AND exchange
constexpr int SPQ_PAIR_SMEM = QR_BYTES + RR_BYTES + XB_BYTES + (QR_SLOTS + RR_SLOTS) * 8;

struct QRing {
  const uint2* gq;  // tile base in global (uint2 units, position stride 32)
  const uint2* gr;
  uint32_t qsm;     // smem byte address of the Q ring + lane*8
  uint32_t rsm;     // smem byte address of the R ring + lane*8
  uint2* qptr;      // generic pointers of the rings (slot 0) for TMA destinations
  uint2* rptr;
  uint64_t* bq;
  uint64_t* br;
  int len, nblk, lane;
  int q_waited, q_released, r_waited, r_released;  // block bookkeeping (warp-uniform)

  __device__ __forceinline__ void issue(const uint2* g, uint2* ring, uint64_t* bars, int slots,
                                        int b) const {
    if (b >= nblk) return;
    const int np = (len - 8 * b) < 8 ? (len - 8 * b) : 8;
    const uint32_t bytes = (uint32_t)np * 256u;
    const int s = b & (slots - 1);
    fence_proxy_async();
    mbar_arrive_expect_tx(&bars[s], bytes);
    tma_load_1d(ring + s * 256, g + (int64_t)b * 256, bytes, &bars[s]);
  }
  __device__ __forceinline__ void reset() { q_waited = q_released = r_waited = r_released = 0; }
  __device__ __forceinline__ void start() const {  // one thread
    for (int b = 0; b < QR_SLOTS; ++b) issue(gq, qptr, bq, QR_SLOTS, b);
    for (int b = 0; b < RR_SLOTS; ++b) issue(gr, rptr, br, RR_SLOTS, b);
  }
  __device__ __forceinline__ void need_q(int bhi) {
    if (bhi >= nblk) bhi = nblk - 1;
    while (q_waited <= bhi) {
      mbar_wait(&bq[q_waited & (QR_SLOTS - 1)], (uint32_t)(q_waited / QR_SLOTS) & 1u);
      ++q_waited;
    }
  }
  __device__ __forceinline__ void need_r(int bhi) {
    if (bhi >= nblk) bhi = nblk - 1;
    while (r_waited <= bhi) {
      mbar_wait(&br[r_waited & (RR_SLOTS - 1)], (uint32_t)(r_waited / RR_SLOTS) & 1u);
      ++r_waited;
    }
  }
  // blocks < blo are not read again by either warp: refill their slots (one warp)
  __device__ __forceinline__ void done_q(int blo) {
    while (q_released < blo) {
      if (lane == 0) issue(gq, qptr, bq, QR_SLOTS, q_released + QR_SLOTS);
      ++q_released;
    }
  }
  __device__ __forceinline__ void done_r(int blo) {
    while (r_released < blo) {
      if (lane == 0) issue(gr, rptr, br, RR_SLOTS, r_released + RR_SLOTS);
      ++r_released;
    }
  }
  __device__ __forceinline__ static uint2 lds(uint32_t addr) {
    uint2 v;
    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr) : "memory");
    return v;
  }
  __device__ __forceinline__ uint2 q_at(int pos) const {
    return lds(qsm + (uint32_t)(pos & (QR_SLOTS * 8 - 1)) * 256u);
  }
  __device__ __forceinline__ uint2 r_at(int pos) const {
    return lds(rsm + (uint32_t)(pos & (RR_SLOTS * 8 - 1)) * 256u);
  }
};

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  __syncwarp();
  // non-.aligned form: the two warps of a pair reach it from different code
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Masks of one warp: optional Hamming mask, then D_k, I_k for k in [K0, K1].
// The read words the masks need are kept in two register windows, as in
// SinglePass<E>: the deletion window Q[p-K1 .. p-K0] and the insertion window
// Q[p+K0 .. p+K1] (p = i + 2 is the newest position); each step shifts both by
// one position and loads the new entries (Q[p-K0], Q[p+K1], and Q[p] for the
// Hamming mask) from the shared TMA ring.
template <bool WITH_H, int K0, int K1>
struct MaskSetQ {
  static constexpr int NK = K1 - K0 + 1;
  static constexpr int NM = (WITH_H ? 1 : 0) + 2 * NK;
  static constexpr int KMAX = K1;
  static constexpr int HB = WITH_H ? 1 : 0;
  uint32_t x[NM][4];
  uint32_t dh[NK], dl[NK];  // deletion window:  index j <-> Q[p - K1 + j]
  uint32_t ih[NK], il[NK];  // insertion window: index j <-> Q[p + K0 + j]

  __device__ __forceinline__ static constexpr bool is_h(int m) { return WITH_H && m == 0; }
  __device__ __forceinline__ static constexpr int kk(int m) {
    return is_h(m) ? 0 : K0 + ((m - HB) >> 1);
  }
  __device__ __forceinline__ static constexpr bool is_d(int m) {
    return !is_h(m) && (((m - HB) & 1) == 0);
  }

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int m = 0; m < NM; ++m) x[m][0] = x[m][1] = x[m][2] = x[m][3] = 0u;
#pragma unroll
    for (int j = 0; j < NK; ++j) dh[j] = dl[j] = ih[j] = il[j] = 0u;
  }

  __device__ __forceinline__ static uint2 qload(const QRing& ring, int pos, int len) {
    return (pos >= 0 && pos < len) ? ring.q_at(pos) : make_uint2(0u, 0u);
  }

  // Fill the windows for a first step whose newest position is p0 (checked loads).
  __device__ __forceinline__ void fill(const QRing& ring, int p0, int len) {
#pragma unroll
    for (int j = 0; j < NK; ++j) {
      const uint2 d = qload(ring, p0 - 1 - K1 + j, len);
      const uint2 v = qload(ring, p0 - 1 + K0 + j, len);
      dh[j] = d.x; dl[j] = d.y;
      ih[j] = v.x; il[j] = v.y;
    }
  }

  // One step (p = i + 2): shift the windows in (qd = Q[p-K0], qi = Q[p+K1],
  // q0 = Q[p]).  F: AND of this warp's amended masks at i; A0: amended Hamming
  // mask at i.  CHECKED: vacancy / range checks at run time (head, tail).
  template <bool CHECKED, bool FIN>
  __device__ __forceinline__ void step(int i, int len, uint2 rn, uint2 qd, uint2 qi, uint2 q0,
                                       uint32_t& F, uint32_t& A0) {
    const int p = i + 2;
#pragma unroll
    for (int j = 0; j < NK - 1; ++j) {
      dh[j] = dh[j + 1]; dl[j] = dl[j + 1];
      ih[j] = ih[j + 1]; il[j] = il[j + 1];
    }
    dh[NK - 1] = qd.x; dl[NK - 1] = qd.y;
    ih[NK - 1] = qi.x; il[NK - 1] = qi.y;
    F = 0xFFFFFFFFu;
    A0 = 0u;
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      uint32_t qh, ql;
      if (is_h(m)) {
        qh = q0.x; ql = q0.y;
      } else if (is_d(m)) {
        qh = dh[K1 - kk(m)]; ql = dl[K1 - kk(m)];
      } else {
        qh = ih[kk(m) - K0]; ql = il[kk(m) - K0];
      }
      uint32_t xn = mismatch(rn.x, rn.y, qh, ql);
      if constexpr (CHECKED) {
        const int qp = is_h(m) ? p : (is_d(m) ? p - kk(m) : p + kk(m));
        const bool ok = p >= 0 && p < len && qp >= 0 && qp < len;
        xn = ok ? xn : 0u;
      }
      if constexpr (FIN) {
        const uint32_t a = amend(x[m][0], x[m][1], x[m][2], x[m][3], xn);
        bool apply = true;
        if (CHECKED && !is_h(m)) apply = is_d(m) ? (i >= kk(m)) : (i < len - kk(m));
        if (is_h(m)) A0 = a;
        if (apply) F &= a;
      }
      x[m][0] = x[m][1];
      x[m][1] = x[m][2];
      x[m][2] = x[m][3];
      x[m][3] = xn;
    }
  }

  template <bool CHECKED, bool FIN>
  __device__ __forceinline__ void step_loading(const QRing& ring, int i, int len, uint32_t& F,
                                               uint32_t& A0) {
    const int p = i + 2;
    const uint2 rn = (p >= 0 && p < len) ? ring.r_at(p) : make_uint2(0u, 0u);
    const uint2 qd = qload(ring, p - K0, len);
    const uint2 qi = qload(ring, p + K1, len);
    const uint2 q0 = WITH_H ? qload(ring, p, len) : make_uint2(0u, 0u);
    step<CHECKED, FIN>(i, len, rn, qd, qi, q0, F, A0);
  }

  // 8 steps i = ib..ib+7 (ib % 8 == 0); `checked` selects the variant at run time.
  __device__ __forceinline__ void block(const QRing& ring, int ib, int len, bool checked,
                                        uint32_t (&F)[8], uint32_t (&A0)[8]) {
    if (!checked) {
      // all positions valid: ring addresses from per-block slot bases + immediates
      const int bi = ib >> 3;
      constexpr int CD0 = 2 - K0;       // c of Q[p - K0] at u = 0 (p = ib + 2 + u)
      constexpr int CI0 = 2 + K1;       // c of Q[p + K1]
      constexpr int LO = (CD0 < 2 ? CD0 : 2) >> 3;
      constexpr int HI = (CI0 + 7) >> 3;
      constexpr int NB = HI - LO + 1;
      uint32_t qb[NB];
#pragma unroll
      for (int d = 0; d < NB; ++d)
        qb[d] = ring.qsm + (uint32_t)((bi + LO + d) & (QR_SLOTS - 1)) * 2048u;
      const uint32_t rb0 = ring.rsm + (uint32_t)(bi & (RR_SLOTS - 1)) * 2048u;
      const uint32_t rb1 = ring.rsm + (uint32_t)((bi + 1) & (RR_SLOTS - 1)) * 2048u;
      auto qat = [&](int c) -> uint2 {  // Q[ib + c], c static
        const int cc = c - 8 * LO;
        return QRing::lds(qb[cc >> 3] + (uint32_t)(cc & 7) * 256u);
      };
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = u + 2;
        const uint2 rn = c < 8 ? QRing::lds(rb0 + c * 256u) : QRing::lds(rb1 + (c - 8) * 256u);
        const uint2 qd = qat(c - K0);
        const uint2 qi = qat(c + K1);
        const uint2 q0 = WITH_H ? qat(c) : make_uint2(0u, 0u);
        step<false, true>(ib + u, len, rn, qd, qi, q0, F[u], A0[u]);
      }
    } else {
#pragma unroll 1
      for (int u = 0; u < 8; ++u) step_loading<true, true>(ring, ib + u, len, F[u], A0[u]);
    }
  }

  // priming: windows for p0 = -2, then x at p = -2..1 (no finalize)
  __device__ __forceinline__ void prime(const QRing& ring, int len) {
    fill(ring, -2, len);
#pragma unroll 1
    for (int i = -4; i < 0; ++i) {
      uint32_t F, A0;
      step_loading<true, false>(ring, i, len, F, A0);
    }
  }
};

// Tile filtration by a warp pair.  Warp A (role 0) returns the counters.
template <int E, int KA>
__device__ __forceinline__ void run_pair(QRing& ring, int role, int len, uint32_t* xbuf,
                                         int bar_id, CsaCounter& cA, CsaCounter& cF) {
  const int lane = threadIdx.x & 31;
  const int nb = (len + 7) >> 3;
  if (role == 0) {
    MaskSetQ<true, 1, KA> ms;
    ms.init();
    ring.need_q((1 + KA) >> 3);
    ring.need_r(0);
    ms.prime(ring, len);
    uint32_t fprev = 0u, aprev = 0u;
    cA.clear();
    cF.clear();
#pragma unroll 1
    for (int jb = 0; jb < nb; ++jb) {
      const int ib = 8 * jb;
      ring.need_q((ib + 9 + KA) >> 3);
      ring.need_r((ib + 9) >> 3);
      const bool checked = !(ib >= KA && ib + 9 + KA < len);
      uint32_t F[8], A0[8];
      ms.block(ring, ib, len, checked, F, A0);
      named_bar(bar_id, 64);  // warp B's partial AND of this block is in xbuf[jb & 1]
      const uint32_t* xb = xbuf + (jb & 1) * 256 + lane;
      uint32_t sF[8], sA[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t f = F[u] & xb[u * 32];
        const uint32_t ns = notstart_of(u);
        sF[u] = f & ~(fprev & ns);
        sA[u] = A0[u] & ~(aprev & ns);
        fprev = f;
        aprev = A0[u];
      }
      cF.add8(sF);
      cA.add8(sA);
      // both warps are past block jb: release what block jb+1 does not need
      ring.done_q((ib + 10 - E) >> 3);
      ring.done_r((ib + 10) >> 3);
    }
  } else {
    MaskSetQ<false, KA + 1, E> ms;
    ms.init();
    ring.need_q((1 + E) >> 3);
    ring.need_r(0);
    ms.prime(ring, len);
#pragma unroll 1
    for (int jb = 0; jb < nb; ++jb) {
      const int ib = 8 * jb;
      ring.need_q((ib + 9 + E) >> 3);
      ring.need_r((ib + 9) >> 3);
      const bool checked = !(ib >= E && ib + 9 + E < len);
      uint32_t F[8], A0[8];
      ms.block(ring, ib, len, checked, F, A0);
      uint32_t* xb = xbuf + (jb & 1) * 256 + lane;
#pragma unroll
      for (int u = 0; u < 8; ++u) xb[u * 32] = F[u];
      named_bar(bar_id, 64);
    }
  }
}

}  // namespace gk
