// gk_filter_sp2.cu -- a2..a6 for one threshold e above the all-register single
// pass (e > GK_SP_EMAX): the single pass of gk_filter_core.cuh split over a PAIR
// of warps.
//
// The single pass (filter_sp_kernel<E>) streams the positions once and keeps,
// per mask, the 4 raw words the amendment window needs: no
// halo recomputation, LOP3 ~1.07x the model, but 2E+1 masks x 4 words + a
// 2E+1-word read window no longer fit one thread's registers beyond E = 11.
// The block-transposed kernel (gk_bt2.cuh) fits any e but recomputes a 4-word
// halo per block (B+4 mismatch words per B positions) and runs at 8 warps/SM.
// Here warp A of a pair holds the Hamming mask and the deletion masks D_1..D_E
// (read window Q[p-E..p]), warp B the insertion masks I_1..I_E (Q[p..p+E]), for
// the same 32 groups of a tile (lane = group of 32 pairs, bit-sliced words as
// everywhere): ~half the registers per thread, so 12 warps fit an SM.  Every 8
// positions warp A hands its partial AND (A0 & AND_k A*D_k) to warp B through a
// double-buffered shared-memory slot (one named barrier per pair and batch);
// warp B completes F = that & AND_k A*I_k and counts its runs, warp A counts A0's
// (the Hamming-stage count c0, readings R5 / R9).  Edge handling exactly as the
// single pass: vacated sources are 0 before amendment (R2), the edge fix sets
// the vacated positions of D_k / I_k to 1 after it (:109, R4), positions outside
// [0, len) are 0 and never counted (R13); windows start at multiples of 4 (R7).
#include <type_traits>

#include "gk_common.cuh"
#include "gk_filter_core.cuh"
#include "gk_kernels.cuh"
#include "gk_tma.cuh"

#ifndef GK_SP2_MINB
#define GK_SP2_MINB 3
#endif
#ifndef GK_SP2_RING
#define GK_SP2_RING 1  // 1: per-warp TMA rings; 0: read-only loads + L1 prefetch (A/B knob)
#endif
#ifndef GK_SP2_MINLEN
#define GK_SP2_MINLEN 128  // shorter reads: mostly checked batches, bt2 is faster there
#endif

namespace gk {
namespace sp2 {

// One side of the split single pass.  SIDE 0: mask 0 = H, mask k = D_k (k =
// 1..E), window Q[p-E .. p]; SIDE 1: mask m = I_{m+1}, window Q[p .. p+E]
// (p = i + 2, the newest position of the amendment window).
template <int E, int SIDE>
struct Half {
  static constexpr int NM = SIDE == 0 ? E + 1 : E;
  static constexpr int QW = E + 1;
  uint32_t qh[QW], ql[QW];
  uint32_t x[NM][4];

  __host__ __device__ __forceinline__ static constexpr int kk(int m) {
    return SIDE == 0 ? m : m + 1;
  }
  __host__ __device__ __forceinline__ static constexpr bool is_h(int m) {
    return SIDE == 0 && m == 0;
  }
  // window slot of mask m's read word at the newest position p
  __host__ __device__ __forceinline__ static constexpr int qidx(int m) {
    return SIDE == 0 ? E - kk(m) : kk(m);
  }
  // offset of the newest read word pushed per step, relative to p
  static constexpr int QNEW = SIDE == 0 ? 0 : E;

  // window before the step that makes p0 the newest position
  template <class Src>
  __device__ __forceinline__ void init(const Src& src, int p0) {
#pragma unroll
    for (int j = 0; j < QW; ++j) {
      const uint2 v = src.ldq(p0 - 1 + QNEW - E + j);
      qh[j] = v.x;
      ql[j] = v.y;
    }
#pragma unroll
    for (int m = 0; m < NM; ++m) x[m][0] = x[m][1] = x[m][2] = x[m][3] = 0u;
  }

  __device__ __forceinline__ void push_q(uint2 qn) {
#pragma unroll
    for (int j = 0; j < QW - 1; ++j) {
      qh[j] = qh[j + 1];
      ql[j] = ql[j + 1];
    }
    qh[QW - 1] = qn.x;
    ql[QW - 1] = qn.y;
  }

  // raw mask words at the newest position p (CD / CL: check the start / end side)
  template <bool CD, bool CL>
  __device__ __forceinline__ void mismatch_all(int p, int len, uint2 rn, uint32_t (&xn)[NM]) const {
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      const int j = qidx(m);
      const uint32_t v = mismatch(rn.x, rn.y, qh[j], ql[j]);
      bool ok = true;
      if (CD) ok = ok && (p >= 0) && (SIDE == 1 || is_h(m) || p - kk(m) >= 0);
      if (CL) ok = ok && (p < len) && (SIDE == 0 || p + kk(m) < len);
      xn[m] = ok ? v : 0u;
    }
  }

  template <bool CD, bool CL>
  __device__ __forceinline__ void prime(int i, int len, uint2 qn, uint2 rn) {
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

  // position i: returns this side's AND of the applied amended masks (SIDE 0:
  // including A0) and, for SIDE 0, A0 itself
  template <bool CD, bool CL>
  __device__ __forceinline__ void step(int i, int len, uint2 qn, uint2 rn, uint32_t& fpart,
                                       uint32_t& a0) {
    push_q(qn);
    uint32_t xn[NM];
    mismatch_all<CD, CL>(i + 2, len, rn, xn);
    uint32_t F = 0xFFFFFFFFu;
#pragma unroll
    for (int m = 0; m < NM; ++m) {
      const uint32_t a = amend(x[m][0], x[m][1], x[m][2], x[m][3], xn[m]);
      bool apply = true;  // edge fix: vacated positions are 1 after amendment (:109)
      if (SIDE == 0 && CD && !is_h(m)) apply = i >= kk(m);
      if (SIDE == 1 && CL) apply = i < len - kk(m);
      if (is_h(m)) a0 = a;
      if (apply) F &= a;
      x[m][0] = x[m][1];
      x[m][1] = x[m][2];
      x[m][2] = x[m][3];
      x[m][3] = xn[m];
    }
    fpart = F;
  }
};

__device__ __forceinline__ void bar_sync(int id) {
  asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id) {
  asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory");
}

constexpr size_t kRingBytes = 2 * 4 * 8 * 32 * 8 + 64;  // RingSrc of one warp (+ 8 mbarriers)
constexpr size_t kSmem = 4 * kRingBytes + 2 * 2 * 8 * 32 * 4;

}  // namespace sp2

// CTA = 2 pairs of warps; pair p filters tile 2*blockIdx.x + p.  Warp 2p = side
// A (H + deletion masks), warp 2p+1 = side B (insertion masks).  Each warp reads
// its words through its own TMA ring in shared memory (RingSrc; side B's read
// stream runs E positions ahead of side A's).  The hand-over slots are
// producer / consumer: A waits only for a slot B has released (named barrier
// "empty"), B only for a slot A has filled ("full"), so A can run up to two
// batches ahead.
template <int E>
__global__ void __launch_bounds__(128, GK_SP2_MINB) filter_sp2_kernel(
    const uint2* __restrict__ reads, const uint2* __restrict__ refs,
    const uint32_t* __restrict__ rund, const uint32_t* __restrict__ fund, int64_t n, int len,
    uint32_t* __restrict__ accept, uint8_t* __restrict__ errc) {
  extern __shared__ __align__(128) uint8_t sm_sp2[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pair = warp >> 1, side = warp & 1;
  const int64_t tile = (int64_t)blockIdx.x * 2 + pair;
  if (tile * 1024 >= n) return;  // both warps of the pair leave together
  uint32_t (*xbuf)[8][32] =
      reinterpret_cast<uint32_t (*)[8][32]>(sm_sp2 + 4 * sp2::kRingBytes) + 2 * pair;  // [slot]
  auto full_id = [&](int s) { return 1 + pair * 4 + s * 2; };
  auto empty_id = [&](int s) { return 2 + pair * 4 + s * 2; };
  const int fin_id = 9 + pair;
  uint8_t* mine = sm_sp2 + (size_t)warp * sp2::kRingBytes;
#if GK_SP2_RING
  RingSrc src;
  src.gq = reads + tile * (int64_t)len * 32;
  src.gr = refs + tile * (int64_t)len * 32;
  src.sq = reinterpret_cast<uint2*>(mine);
  src.sr = src.sq + 4 * 8 * 32;
  src.bq = reinterpret_cast<uint64_t*>(mine + 2 * 4 * 8 * 32 * 8);
  src.br = src.bq + 4;
  src.len = len;
  src.nblk = (len + 7) >> 3;
  src.lane = lane;
  if (lane == 0) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      mbar_init(&src.bq[b], 1);
      mbar_init(&src.br[b], 1);
    }
    fence_mbar_init();
  }
  __syncwarp();
  src.start();
#else
  (void)mine;
  GlobalGroupSrc src;
  src.q = reads + tile * (int64_t)len * 32 + lane;
  src.r = refs + tile * (int64_t)len * 32 + lane;
  src.len = len;
#endif
  CsaCounter cnt;  // side A: A0 run starts (c0); side B: F run starts
  cnt.clear();
  uint32_t prev = 0u;
  const int nb = (len + 7) >> 3;

  auto run = [&](auto& h, auto side_tag) {
    constexpr int SIDE = decltype(side_tag)::value;
    using H = std::remove_reference_t<decltype(h)>;
    h.init(src, -2);
#pragma unroll
    for (int i = -4; i < 0; ++i)
      h.template prime<true, true>(i, len, src.ldq(i + 2 + H::QNEW), src.ldr(i + 2));
#pragma unroll 1
    for (int b = 0; b < nb; ++b) {
      const int i0 = 8 * b;
      uint32_t fp[8], a0[8];
      // checked batches: SIDE A near the start (deletion vacancies, i < E) and at
      // the end (targets >= len); SIDE B near the end (insertion vacancies)
      const bool chk = SIDE == 0 ? (i0 < E || i0 + 8 + 2 > len) : (i0 + 8 + 2 + E > len);
#if !GK_SP2_RING
      {  // pull the next batch's words into L1 while this one computes
        const int pn = i0 + 8 + 2;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (pn + u + H::QNEW < len)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(src.q + (int64_t)(pn + u + H::QNEW) * GK_WARP));
          if (pn + u < len)
            asm volatile("prefetch.global.L1 [%0];" ::"l"(src.r + (int64_t)(pn + u) * GK_WARP));
        }
      }
#endif
      if (chk) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u;
          h.template step<true, true>(i, len, src.ldq(i + 2 + H::QNEW), src.ldr(i + 2), fp[u],
                                      a0[u]);
          if (i >= len) fp[u] = a0[u] = 0u;  // positions >= len: never counted (R13)
        }
      } else {
        uint2 qn[8], rn[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          qn[u] = src.ldq_nc(i0 + u + 2 + H::QNEW);
          rn[u] = src.ldr_nc(i0 + u + 2);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          h.template step<false, false>(i0 + u, len, qn[u], rn[u], fp[u], a0[u]);
      }
      const int slot = b & 1;
      uint32_t v[8];
      if (SIDE == 0) {
        if (b >= 2) sp2::bar_sync(empty_id(slot));
#pragma unroll
        for (int u = 0; u < 8; ++u) xbuf[slot][u][lane] = fp[u];
        sp2::bar_arrive(full_id(slot));
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = a0[u];
      } else {
        sp2::bar_sync(full_id(slot));
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = fp[u] & xbuf[slot][u][lane];
        sp2::bar_arrive(empty_id(slot));
      }
      uint32_t st[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        // (positions >= len occur only in checked batches, zeroed there: side B's
        // v = its part & side A's zeroed part)
        st[u] = v[u] & ~(prev & notstart_of(u));
        prev = v[u];
      }
      cnt.add8(st);
    }
  };
  if (side == 0) {
    sp2::Half<E, 0> h;
    run(h, std::integral_constant<int, 0>{});
    // drain: B's releases of the last (up to) two batches
    for (int b = nb - 2 < 0 ? 0 : nb - 2; b < nb; ++b) sp2::bar_sync(empty_id(b & 1));
  } else {
    sp2::Half<E, 1> h;
    run(h, std::integral_constant<int, 1>{});
  }
  // side A hands c0 to side B, which decides (finish_group)
  uint32_t planes[8];
  cnt.planes(planes);
  uint32_t* xc = &xbuf[0][0][0];  // every slot has been released by B
  if (side == 0) {
#pragma unroll
    for (int k = 0; k < 8; ++k) xc[k * 32 + lane] = planes[k];
    sp2::bar_arrive(fin_id);
  } else {
    sp2::bar_sync(fin_id);
    uint32_t cA[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) cA[k] = xc[k * 32 + lane];
    const int64_t g = tile * 32 + lane;
    if (g * 32 < n) finish_group(cA, planes, E, __ldg(rund + g) | __ldg(fund + g), g, n, accept, errc);
  }
}

template <int E>
static void launch_sp2_t(const uint2* reads, const uint2* refs, const uint32_t* rund,
                         const uint32_t* fund, int64_t n, int len, uint32_t* accept,
                         uint8_t* errc, cudaStream_t stream) {
  const int64_t tiles = (n + 1023) / 1024;
  const int64_t blocks = (tiles + 1) / 2;
  ensure_func_attr((const void*)filter_sp2_kernel<E>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                   (int)sp2::kSmem);
  count_launch();
  filter_sp2_kernel<E><<<(unsigned)blocks, 128, sp2::kSmem, stream>>>(reads, refs, rund, fund, n,
                                                                       len, accept, errc);
}

// e = 12 at len >= GK_SP2_MINLEN: the split single pass; false otherwise (the
// caller runs the block-transposed kernel).  e = 12 is the only threshold whose
// half passes fit 168 registers without spills (12 warps/SM); at e = 13-16 they
// spill 170-460 bytes and measured 7-39% slower than bt2, at 100 bp even e = 12
// is slower (mostly checked batches) -- profiles/r02_ab_sp2.jsonl.
bool launch_sp2(const uint2* reads, const uint2* refs, const uint32_t* rund, const uint32_t* fund,
                int64_t n, int len, int e, uint32_t* accept, uint8_t* errc, cudaStream_t stream) {
  if (len < GK_SP2_MINLEN) return false;
  switch (e) {
    case 12:
      launch_sp2_t<12>(reads, refs, rund, fund, n, len, accept, errc, stream);
      return true;
    default:
      return false;
  }
}

}  // namespace gk
