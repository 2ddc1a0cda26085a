// gk_fused.cu -- a1..a6 fused from ASCII: gk_filter_ascii (one threshold) and
// gk_filter_ascii_sweep (every threshold e <= e_max in one pass).
//
// The paper's "device-encoded" kernel encodes each pair inside the filtering
// thread; its trade-off is that encoding costs kernel time
// but saves the host-side preparation (Table S.17 :809-821).  On B200 the
// unfused path writes the 2-bit planes to HBM (L/4 bytes per sequence) and the
// filter reads them back; here they never leave shared memory.
//
// One CTA (4 warps) owns one tile of 1024 pairs (32 groups of 32):
//   phase E  warp w encodes the 16 spans (32 ASCII rows each, one contiguous
//            byte range, brought in by cp.async.bulk, double- or single-
//            buffered) of groups w, w+4, ... of both sets with the encoder of
//            gk_encode (gk_encode3.cuh), straight into a group-major tile in
//            shared memory: word (g, pos, plane) at (g*P + pos)*2 + plane, P =
//            len rounded up to odd (encode writes: 32 consecutive words; filter
//            reads: lane g at row g, conflict-free for an odd P);
//   phase F  the 4 warps split the tile's positions; lane g filters group g:
//            e <= GK_SP_EMAX: the single-pass core over a range of positions
//            (gk_filter_core.cuh, ranges start at multiples of 4 so the window
//            counts add up); larger e and the sweep: the block-transposed core
//            over a range of 8-position blocks (gk_bt2.cuh, SMem policy);
//   combine  per-warp bit-sliced counters are summed through shared memory and
//            warp 0 writes the tile's accept bits / error counts (finish_group).
// The last tile may be partial: spans that would read past the caller's
// (n-1)*stride+len bytes are staged with bounded loads instead of TMA, and
// pairs >= n are never written.
#include "gk_bt2.cuh"
#include "gk_common.cuh"
#include "gk_encode3.cuh"
#include "gk_encode_core.cuh"
#include "gk_filter_core.cuh"
#include "gk_kernels.cuh"
#include "gk_tma.cuh"

namespace gk {
namespace fz {

constexpr int NW = 4;  // warps per CTA

struct Layout {
  int P;           // uint2 per group row of the tile (len rounded up to odd)
  size_t set;      // bytes of one set's tile: 32 * P * 8
  uint32_t bufb;   // bytes of one span buffer
  int nbuf;        // span buffers per warp
  size_t xch;      // counter exchange bytes (may reuse the staging area)
  size_t stage;    // staging (+ exchange) area
  size_t total;
};

static Layout layout(int len, int stride, int sweep_rows, int np) {
  Layout L;
  L.P = len | 1;
  L.set = (size_t)32 * L.P * 8;
  L.bufb = ((uint32_t)(32 * stride + 32) + 127u) & ~127u;
  L.nbuf = 2;
  L.xch = sweep_rows > 0 ? (size_t)NW * ((size_t)sweep_rows * np + 8) * 32 * 4
                         : (size_t)NW * 16 * 32 * 4;
  for (;;) {
    const size_t st = (size_t)NW * L.nbuf * L.bufb;
    L.stage = st > L.xch ? st : L.xch;
    L.total = 2 * L.set + L.stage + 2 * 32 * 4 + NW * 2 * 8 + 64;
    // two CTAs per SM (8 warps) when shared memory allows: single-buffer the spans first
    if (L.total <= 113 * 1024 || L.nbuf == 1) break;
    L.nbuf = 1;
  }
  return L;
}

// One 16-position chunk of a staged span -> 32 words of the group's tile row.
template <bool ALN>
__device__ __forceinline__ void chunk(const uint8_t* buf, const uint32_t (&roff)[4],
                                      const uint32_t (&rsh)[4], int c, int len,
                                      const enc3::Lane& ln, uint32_t (&ag)[4], uint32_t (&ay)[4],
                                      uint32_t* row, bool tail) {
  uint32_t x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint8_t* a = buf + roff[i] + 16 * c;
    uint32_t w;
    if (ALN) {
      w = *reinterpret_cast<const uint32_t*>(a);
    } else {
      const uint32_t lo = *reinterpret_cast<const uint32_t*>(a);
      const uint32_t hi = *reinterpret_cast<const uint32_t*>(a + 4);
      w = __funnelshift_r(lo, hi, rsh[i]);
    }
    if (tail) {
      const int rem = len - 16 * c - 4 * ln.cw;
      const uint32_t bm =
          rem >= 4 ? 0xFFFFFFFFu : (rem <= 0 ? 0u : (0xFFFFFFFFu >> (32 - 8 * rem)));
      w = (w & bm) | (0x41414141u & ~bm);
    }
    x[i] = enc3::row_word(w, ln, ag[i], ay[i]);
  }
  uint32_t m = enc3::merge4(x[0], x[1], x[2], x[3], ln);
  m = enc3::transpose3(m, ln);
  const int lane = threadIdx.x & 31;
  const int pos = 16 * c + 4 * (lane & 3) + (lane >> 3);
  const int plane = ((lane >> 2) & 1) ? 0 : 1;  // b' = 1: ASCII bit 2 = high plane
  if (!tail || pos < len) row[pos * 2 + plane] = m;
}

template <int NCH, bool ALN>
__device__ __forceinline__ uint32_t encode_span(const uint8_t* sbuf, const uint32_t (&roff)[4],
                                                const uint32_t (&rsh)[4], int len,
                                                const enc3::Lane& ln, uint32_t* row) {
  const int nch = NCH > 0 ? NCH : (len + 15) >> 4;
  uint32_t ag[4] = {0u, 0u, 0u, 0u}, ay[4] = {0u, 0u, 0u, 0u};
  if (NCH > 0) {
#pragma unroll
    for (int c = 0; c < (NCH > 1 ? NCH - 1 : 0); ++c)
      chunk<ALN>(sbuf, roff, rsh, c, len, ln, ag, ay, row, false);
  } else {
#pragma unroll 1
    for (int c = 0; c < nch - 1; ++c) chunk<ALN>(sbuf, roff, rsh, c, len, ln, ag, ay, row, false);
  }
  chunk<ALN>(sbuf, roff, rsh, nch - 1, len, ln, ag, ay, row, true);
  return enc3::group_undef(ag, ay, ln);
}

// Phase E of one warp: spans k = 0..15 = (group w + 4*(k>>1), set k&1).
template <int NCH, bool ALN>
__device__ __forceinline__ void phase_encode(const uint8_t* __restrict__ reads,
                                             const uint8_t* __restrict__ refs, int stride,
                                             int len, int64_t n, int64_t tile, uint8_t* stg,
                                             const Layout& L, uint2* T, uint32_t* und,
                                             uint64_t* bars, uint32_t& phase_bits) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  enc3::Lane ln;
  ln.init(lane);
  uint32_t roff[4], rsh[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t a = (uint32_t)ln.rows[i] * (uint32_t)stride + 4u * (uint32_t)ln.cw;
    roff[i] = ALN ? a : (a & ~3u);
    rsh[i] = (a & 3u) * 8u;
  }
  const int64_t span = 32 * (int64_t)stride;
  const int64_t limit = (n - 1) * (int64_t)stride + len;  // bytes the caller owns per set
  auto src_of = [&](int k, int64_t& off) {
    const int g = warp + NW * (k >> 1);
    off = (tile * 32 + g) * span;
    return (k & 1) ? refs : reads;
  };
  // a span is brought in by TMA iff it lies inside the caller's bytes
  auto tma_ok = [&](int k) {
    int64_t off;
    src_of(k, off);
    return off + span <= limit;
  };
  auto issue = [&](int k) {
    if (!tma_ok(k)) return;
    int64_t off;
    const uint8_t* base = src_of(k, off);
    const int b = L.nbuf == 2 ? (k & 1) : 0;
    fence_proxy_async();
    mbar_arrive_expect_tx(&bars[b], (uint32_t)span);
    tma_load_1d(stg + (size_t)b * L.bufb, base + off, (uint32_t)span, &bars[b]);
  };
  constexpr int NSPAN = 16;
  if (lane == 0) {
    issue(0);
    if (L.nbuf == 2) issue(1);
  }
  uint32_t u = 0u;
#pragma unroll 1
  for (int k = 0; k < NSPAN; ++k) {
    const int b = L.nbuf == 2 ? (k & 1) : 0;
    const int g = warp + NW * (k >> 1);
    const int64_t first = (tile * 32 + g) * 32;  // first pair of the group
    const uint8_t* sbuf = stg + (size_t)b * L.bufb;
    if (first < n) {
      if (tma_ok(k)) {
        mbar_wait(&bars[b], (phase_bits >> b) & 1u);
        phase_bits ^= 1u << b;
      } else {  // bounded staging of the last rows of the batch
        int64_t off;
        const uint8_t* base = src_of(k, off);
        __syncwarp();
        stage_span(base + off, limit - off, const_cast<uint8_t*>(sbuf), lane, 32);
        __syncwarp();
      }
      uint32_t* row = reinterpret_cast<uint32_t*>(T + (size_t)(k & 1) * 32 * L.P + (size_t)g * L.P);
      u |= encode_span<NCH, ALN>(sbuf, roff, rsh, len, ln, row);
    }
    if (k & 1) {
      if (lane == 0) und[g] = u;
      u = 0u;
    }
    __syncwarp();
    if (lane == 0) {
      if (L.nbuf == 2) {
        if (k + 2 < NSPAN) issue(k + 2);
      } else if (k + 1 < NSPAN) {
        issue(k + 1);
      }
    }
  }
}

// Sum of bit-sliced 8-plane counters: a += b (ripple carry; b at stride 32 words).
__device__ __forceinline__ void add8(uint32_t (&a)[8], const uint32_t* b) {
  uint32_t carry = 0u;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t x = a[k], y = b[k * 32];
    a[k] = x ^ y ^ carry;
    carry = (x & y) | (carry & (x ^ y));
  }
}

template <int NP>
__device__ __forceinline__ void addnp(uint32_t (&a)[8], const uint32_t* b) {
  uint32_t carry = 0u;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t x = a[k], y = k < NP ? b[k * 32] : 0u;
    a[k] = x ^ y ^ carry;
    carry = (x & y) | (carry & (x ^ y));
  }
}

// Positions [lo, hi) of warp w (multiples of 4 apart, balanced in 4-base quads).
__device__ __forceinline__ void pos_range(int len, int w, int& lo, int& hi) {
  const int quads = (len + 3) >> 2;
  lo = 4 * ((quads * w) / NW);
  hi = 4 * ((quads * (w + 1)) / NW);
  if (hi > len) hi = len;
}

// 8-position blocks [b0, b1) of warp w: the first and last blocks (mostly checked
// steps) weigh about 1.5 interior blocks, so the split is by that weight.
__device__ __forceinline__ void block_range(int len, int w, int& b0, int& b1) {
  const int nb = (len + 7) >> 3;
  // weights: 3 for the two edge blocks, 2 for interior ones
  const int total = 2 * nb + (nb >= 2 ? 2 : 1);
  auto cut = [&](int part) {  // first block whose cumulative weight reaches part*total/NW
    const int target = (total * part + NW / 2) / NW;
    int acc = 0, b = 0;
    while (b < nb && acc < target) {
      acc += (b == 0 || b == nb - 1) ? 3 : 2;
      ++b;
    }
    return b;
  };
  b0 = cut(w);
  b1 = w == NW - 1 ? nb : cut(w + 1);
}

template <int B, class M>
__device__ __forceinline__ void load_r_at(const uint2* r, int len, int ib, bt2::Win<B>& R) {
#pragma unroll
  for (int c = 0; c < B + 4; ++c) {
    const uint2 v = bt2::ldc<M>(r, ib - 2 + c, len);
    R.h[c] = v.x;
    R.l[c] = v.y;
  }
}

struct Smem {
  uint2* T;        // [2][32][P]
  uint8_t* stg;    // staging / exchange
  uint32_t* und;   // [32]: undefined pairs of each group (read or reference)
  uint64_t* bars;  // [NW][2]
};

__device__ __forceinline__ Smem carve(uint8_t* sm, const Layout& L) {
  Smem s;
  s.T = reinterpret_cast<uint2*>(sm);
  s.stg = sm + 2 * L.set;
  s.und = reinterpret_cast<uint32_t*>(s.stg + L.stage);
  s.bars = reinterpret_cast<uint64_t*>(s.und + 64);
  return s;
}

__device__ __forceinline__ void init_bars(uint64_t* bars) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    mbar_init(&bars[2 * warp], 1);
    mbar_init(&bars[2 * warp + 1], 1);
    fence_mbar_init();
  }
  __syncwarp();
}

}  // namespace fz

// One threshold e.  EP >= 0: single-pass core sp<EP> (e == EP); EP < 0: bt2.
template <int EP, int NCH, bool ALN>
__global__ void __launch_bounds__(fz::NW * 32, 2) fused_kernel(
    const uint8_t* __restrict__ reads, const uint8_t* __restrict__ refs, int stride, int64_t n,
    int len, int e, fz::Layout L, uint32_t* __restrict__ accept, uint8_t* __restrict__ errc) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const fz::Smem s = fz::carve(sm, L);
  fz::init_bars(s.bars);
  const int64_t tile = blockIdx.x;
  uint32_t phase_bits = 0u;
  fz::phase_encode<NCH, ALN>(reads, refs, stride, len, n, tile, s.stg + (size_t)warp * L.nbuf * L.bufb,
                             L, s.T, s.und, s.bars + 2 * warp, phase_bits);
  __syncthreads();
  const uint2* q = s.T + (size_t)lane * L.P;
  const uint2* r = s.T + (size_t)32 * L.P + (size_t)lane * L.P;
  uint32_t cA[8], cF[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) cA[b] = cF[b] = 0u;
  if constexpr (EP >= 0) {
    int lo, hi;
    fz::pos_range(len, warp, lo, hi);
    if (lo < hi) {
      SmemGroupSrc src;
      src.q = q;
      src.r = r;
      src.len = len;
      src.pstride = 1;
      SinglePass<EP> sp;
      run_range<EP>(sp, src, len, lo, hi);
      sp.cA.planes(cA);
      sp.cF.planes(cF);
    }
  } else {
    int b0, b1;
    fz::block_range(len, warp, b0, b1);
    if (b0 < b1) {
      CsaCounter ca, cf;
      ca.clear();
      cf.clear();
      bt2::Win<8> R;
      fz::load_r_at<8, bt2::SMem>(r, len, 8 * b0, R);
#pragma unroll 1
      for (int b = b0; b < b1; ++b)
        bt2::block<8, GK_BT2_LA_E, bt2::SMem>(q, r, R, 8 * b, len, e, 1, ca, cf, bt2::NoHook{});
      ca.planes(cA);
      cf.planes(cF);
    }
  }
  uint32_t* xch = reinterpret_cast<uint32_t*>(s.stg);  // the staging area is free now
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    xch[(warp * 16 + b) * 32 + lane] = cA[b];
    xch[(warp * 16 + 8 + b) * 32 + lane] = cF[b];
  }
  __syncthreads();
  if (warp == 0) {
    for (int w = 1; w < fz::NW; ++w) {
      fz::add8(cA, xch + (w * 16) * 32 + lane);
      fz::add8(cF, xch + (w * 16 + 8) * 32 + lane);
    }
    const int64_t g = tile * 32 + lane;
    if (g * 32 < n) finish_group(cA, cF, e, s.und[lane], g, n, accept, errc);
  }
}

// Every threshold e = 0..emax in one pass (bt2 + per-k counters per warp).
template <int NP, int NCH, bool ALN>
__global__ void __launch_bounds__(fz::NW * 32, 2) fused_sweep_kernel(
    const uint8_t* __restrict__ reads, const uint8_t* __restrict__ refs, int stride, int64_t n,
    int len, int emax, fz::Layout L, uint32_t* __restrict__ accept, uint8_t* __restrict__ errc) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const fz::Smem s = fz::carve(sm, L);
  fz::init_bars(s.bars);
  const int64_t tile = blockIdx.x;
  uint32_t phase_bits = 0u;
  fz::phase_encode<NCH, ALN>(reads, refs, stride, len, n, tile, s.stg + (size_t)warp * L.nbuf * L.bufb,
                             L, s.T, s.und, s.bars + 2 * warp, phase_bits);
  __syncthreads();
  // per-warp exchange: [8 planes of cA][emax][NP] x 32 lanes (staging is free now)
  uint32_t* mine = reinterpret_cast<uint32_t*>(s.stg) + (size_t)warp * (emax * NP + 8) * 32;
  for (int j = 0; j < emax * NP; ++j) mine[(8 + j) * 32 + lane] = 0u;
  const uint2* q = s.T + (size_t)lane * L.P;
  const uint2* r = s.T + (size_t)32 * L.P + (size_t)lane * L.P;
  uint32_t cA[8];
  {
    CsaCounter ca, cf;
    ca.clear();
    cf.clear();
    int b0, b1;
    fz::block_range(len, warp, b0, b1);
    if (b0 < b1) {
      bt2::Win<8> R;
      fz::load_r_at<8, bt2::SMem>(r, len, 8 * b0, R);
      const bt2::SweepHook<NP> hook{mine + 8 * 32 + lane};
#pragma unroll 1
      for (int b = b0; b < b1; ++b)
        bt2::block<8, GK_BT2_LA, bt2::SMem>(q, r, R, 8 * b, len, emax, 1, ca, cf, hook);
    }
    ca.planes(cA);
  }
#pragma unroll
  for (int b = 0; b < 8; ++b) mine[b * 32 + lane] = cA[b];
  __syncthreads();
  // every warp finishes 1/NW of the thresholds for all 32 groups of the tile
  const uint32_t* x0 = reinterpret_cast<const uint32_t*>(s.stg);
  const size_t wstride = (size_t)(emax * NP + 8) * 32;
#pragma unroll
  for (int b = 0; b < 8; ++b) cA[b] = x0[b * 32 + lane];
  for (int w = 1; w < fz::NW; ++w) fz::add8(cA, x0 + w * wstride + lane);
  const int64_t g = tile * 32 + lane;
  if (g * 32 >= n) return;
  const uint32_t und = s.und[lane];
  const int64_t words = (n + 31) / 32;
  for (int e = warp; e <= emax; e += fz::NW) {
    uint32_t f[8];
    if (e == 0) {
#pragma unroll
      for (int b = 0; b < 8; ++b) f[b] = cA[b];
    } else {
#pragma unroll
      for (int b = 0; b < 8; ++b) f[b] = 0u;
      for (int w = 0; w < fz::NW; ++w)
        fz::addnp<NP>(f, x0 + w * wstride + (8 + (size_t)(e - 1) * NP) * 32 + lane);
    }
    finish_group(cA, f, e, und, g, n, accept + e * words, errc ? errc + e * n : nullptr);
  }
}

namespace fz {

template <class K>
static void launch(K kern, const Layout& L, int64_t n, const uint8_t* reads, const uint8_t* refs,
                   int stride, int len, int e, uint32_t* accept, uint8_t* errc,
                   cudaStream_t stream) {
  // dynamic shared memory opt-in (per device and kernel)
  if (L.total > 48 * 1024)
    ensure_func_attr((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                     (int)L.total);
  const int64_t tiles = (n + 1023) / 1024;
  count_launch();
  kern<<<(unsigned)tiles, NW * 32, L.total, stream>>>(reads, refs, stride, n, len, e, L, accept,
                                                      errc);
}

template <int NCH, bool ALN>
static bool fused_e(int e, const uint8_t* reads, const uint8_t* refs, int stride, int64_t n,
                    int len, uint32_t* accept, uint8_t* errc, cudaStream_t stream) {
  const Layout L = layout(len, stride, 0, 0);
  if (L.total > 227 * 1024) return false;
#define GK_FZ(E)                                                                            \
  case E:                                                                                   \
    launch(fused_kernel<E, NCH, ALN>, L, n, reads, refs, stride, len, e, accept, errc, stream); \
    return true;
  switch (e) {
    GK_FZ(0) GK_FZ(1) GK_FZ(2) GK_FZ(3) GK_FZ(4) GK_FZ(5) GK_FZ(6) GK_FZ(7) GK_FZ(8) GK_FZ(9)
    GK_FZ(10) GK_FZ(11)
    default:
      launch(fused_kernel<-1, NCH, ALN>, L, n, reads, refs, stride, len, e, accept, errc, stream);
      return true;
  }
#undef GK_FZ
}

template <int NCH, bool ALN>
static bool fused_sweep(int emax, const uint8_t* reads, const uint8_t* refs, int stride,
                        int64_t n, int len, uint32_t* accept, uint8_t* errc,
                        cudaStream_t stream) {
  const int maxc = 2 * ((len + 3) / 4);
  const int np = maxc < 64 ? 6 : (maxc < 128 ? 7 : 8);
  const Layout L = layout(len, stride, emax, np);
  if (L.total > 227 * 1024) return false;
  if (np == 6)
    launch(fused_sweep_kernel<6, NCH, ALN>, L, n, reads, refs, stride, len, emax, accept, errc,
           stream);
  else if (np == 7)
    launch(fused_sweep_kernel<7, NCH, ALN>, L, n, reads, refs, stride, len, emax, accept, errc,
           stream);
  else
    launch(fused_sweep_kernel<8, NCH, ALN>, L, n, reads, refs, stride, len, emax, accept, errc,
           stream);
  return true;
}

}  // namespace fz

// Returns false when the fused kernels cannot take the call (shared memory,
// alignment); the caller then runs the unfused path.
bool launch_fused(const uint8_t* reads, const uint8_t* refs, int64_t stride, int64_t n, int len,
                  int e, bool sweep, uint32_t* accept, uint8_t* errc, cudaStream_t stream) {
  if (((reinterpret_cast<uintptr_t>(reads) | reinterpret_cast<uintptr_t>(refs)) & 15u) != 0)
    return false;
  if (stride > 512) return false;
  const int nch = (len + 15) >> 4;
  const bool aln = (stride & 3) == 0;
  const int s = (int)stride;
#define GK_FZD(N)                                                                            \
  if (nch == N) {                                                                            \
    if (sweep)                                                                               \
      return aln ? fz::fused_sweep<N, true>(e, reads, refs, s, n, len, accept, errc, stream)  \
                 : fz::fused_sweep<N, false>(e, reads, refs, s, n, len, accept, errc, stream); \
    return aln ? fz::fused_e<N, true>(e, reads, refs, s, n, len, accept, errc, stream)        \
               : fz::fused_e<N, false>(e, reads, refs, s, n, len, accept, errc, stream);      \
  }
  GK_FZD(7)
  GK_FZD(10)
#undef GK_FZD
  if (sweep)
    return aln ? fz::fused_sweep<0, true>(e, reads, refs, s, n, len, accept, errc, stream)
               : fz::fused_sweep<0, false>(e, reads, refs, s, n, len, accept, errc, stream);
  return aln ? fz::fused_e<0, true>(e, reads, refs, s, n, len, accept, errc, stream)
             : fz::fused_e<0, false>(e, reads, refs, s, n, len, accept, errc, stream);
}

}  // namespace gk
