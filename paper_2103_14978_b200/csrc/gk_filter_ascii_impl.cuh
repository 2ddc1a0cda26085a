// gk_filter_ascii_impl.cuh -- a1..a6 fused: ASCII pairs -> accept bits / error counts.
//
// The paper's "device-encoded" kernel encodes each pair inside the filtering
// thread.  Here one CTA (4 warps) owns G groups (G*32 pairs, a
// whole tile when shared memory allows):
//   phase 1  every warp encodes groups w, w+4, ... : the 32 ASCII rows of a group
//            are staged in shared memory with 16-byte loads, then encoded by the
//            same code as gk_encode (gk_encode_core.cuh) straight into a packed
//            tile in shared memory -- the packed words never touch HBM;
//   phase 2  the 4 warps split the base positions of the tile (ranges start at
//            multiples of 4 so the window counts add up), lane g filtering group g
//            with the register-resident core (gk_filter_core.cuh); the per-warp
//            bit-sliced counters are summed through shared memory and warp 0
//            finishes the groups.
// For e above the register-resident instantiations warp 0 runs the mask-major
// fallback over the shared-memory tile instead.
#pragma once
#include "gk_common.cuh"
#include "gk_encode_core.cuh"
#include "gk_filter_core.cuh"
#include "gk_kernels.cuh"
#include "gk_tma.cuh"

#ifndef GK_ASCII_TMA
#define GK_ASCII_TMA 1
#endif

namespace gk {

struct AsciiLayout {
  int G;            // groups per CTA
  size_t packed;    // bytes of one packed set (len * G * 8)
  size_t staging;   // bytes of the per-warp ASCII staging (4 warps)
  size_t fbytes;    // bytes of F for the fallback
  size_t total;
};

static AsciiLayout ascii_layout(int len, int64_t stride, bool generic) {
  AsciiLayout L;
  for (int G = 32; G >= 8; G >>= 1) {
    L.G = G;
    L.packed = (size_t)len * (G + 1) * 8;  // [len][G+1] uint2 (odd pitch: fewer bank conflicts)
    L.staging = 4 * ((size_t)32 * (size_t)stride + 32);
    if (L.staging < 8192) L.staging = 8192;  // also holds the 4 x 16 x 32 counter exchange
    L.fbytes = generic ? (size_t)len * G * 4 : 0;
    L.total = 2 * L.packed + L.staging + L.fbytes + 256;
    if (L.total <= 224 * 1024) break;
  }
  return L;
}

// Sum of two bit-sliced 8-bit counters (ripple-carry adder per plane).
__device__ __forceinline__ void add_planes(uint32_t (&a)[8], const uint32_t* b, int bstride) {
  uint32_t carry = 0u;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t x = a[k], y = b[k * bstride];
    a[k] = x ^ y ^ carry;
    carry = (x & y) | (carry & (x ^ y));
  }
}

template <int E>  // E < 0: fallback for any e
__global__ void __launch_bounds__(128) filter_ascii_kernel(
    const uint8_t* __restrict__ reads, const uint8_t* __restrict__ refs, int64_t stride,
    int64_t n, int len, int e, int G, uint32_t packed_bytes, uint32_t staging_bytes,
    uint32_t* __restrict__ accept, uint8_t* __restrict__ errc) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint2* pq = reinterpret_cast<uint2*>(sm);                     // [len][G+1] read words
  uint2* pr = reinterpret_cast<uint2*>(sm + packed_bytes);      // [len][G+1] ref words
  const int P = G + 1;
  uint8_t* stg = sm + 2 * (size_t)packed_bytes;                 // 4 x (32*stride + 32)
  uint32_t* und = reinterpret_cast<uint32_t*>(stg + staging_bytes);  // [G]
  uint32_t* Fsm = und + 32;                                      // fallback F [len][G]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gbase = (int64_t)blockIdx.x * G;  // first group of this CTA
  const int64_t ngroups = (n + 31) / 32;
  const uint32_t wstage = (uint32_t)(32 * stride + 32);
  uint8_t* my_stage = stg + warp * wstage;
  const bool aligned = (stride % 4 == 0) && ((reinterpret_cast<uintptr_t>(reads) & 3u) == 0) &&
                       ((reinterpret_cast<uintptr_t>(refs) & 3u) == 0);

  // ---- phase 1: encode the CTA's groups into the shared-memory packed tile ----
  for (int gl = warp; gl < G; gl += 4) {
    const int64_t g = gbase + gl;
    uint32_t u = 0u;
    if (g < ngroups) {
      const int nvalid = (int)((n - g * 32) < 32 ? (n - g * 32) : 32);
      for (int set = 0; set < 2; ++set) {
        const uint8_t* base = (set == 0 ? reads : refs) + g * 32 * stride;
        const int64_t nbytes = (int64_t)(nvalid - 1) * stride + len;
        stage_span(base, nbytes, my_stage, lane, 32);
        __syncwarp();
        const uint32_t off = (uint32_t)(reinterpret_cast<uintptr_t>(base) & 15u);
        uint2* dst = (set == 0 ? pq : pr) + gl;
        auto emit = [&](int pos, uint32_t hi, uint32_t lo) { dst[pos * P] = make_uint2(hi, lo); };
        const uint32_t uu = aligned ? encode_group<true>(my_stage, off, (uint32_t)stride, nvalid, len, emit)
                                    : encode_group<false>(my_stage, off, (uint32_t)stride, nvalid, len, emit);
        u |= uu;
        __syncwarp();
      }
    } else {
      // groups past the end: all-'A' (never reported)
      for (int pos = lane; pos < len; pos += 32) {
        pq[pos * P + gl] = make_uint2(0u, 0u);
        pr[pos * P + gl] = make_uint2(0u, 0u);
      }
    }
    if (lane == 0) und[gl] = u;
  }
  __syncthreads();

  const int64_t g = gbase + lane;
  const bool active = lane < G && g < ngroups;
  SmemGroupSrc src;
  src.q = pq + lane;
  src.r = pr + lane;
  src.len = len;
  src.pstride = P;

  if constexpr (E >= 0) {
    // ---- phase 2: positions split across the 4 warps ----
    int chunk = (len + 3) / 4;
    chunk = (chunk + 3) & ~3;
    const int lo = warp * chunk;
    int hi = lo + chunk;
    if (hi > len) hi = len;
    uint32_t cA[8], cF[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) cA[b] = cF[b] = 0u;
    if (active && lo < hi) {
      SinglePass<E> sp;
      run_range<E>(sp, src, len, lo, hi);
      sp.cA.planes(cA);
      sp.cF.planes(cF);
    }
    // exchange counters through the (now free) staging area: [warp][16][32]
    uint32_t* xch = reinterpret_cast<uint32_t*>(stg);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      xch[(warp * 16 + b) * 32 + lane] = cA[b];
      xch[(warp * 16 + 8 + b) * 32 + lane] = cF[b];
    }
    __syncthreads();
    if (warp == 0 && active) {
      for (int w = 1; w < 4; ++w) {
        add_planes(cA, xch + (w * 16) * 32 + lane, 32);
        add_planes(cF, xch + (w * 16 + 8) * 32 + lane, 32);
      }
      finish_group(cA, cF, e, und[lane], g, n, accept, errc);
    }
  } else {
    if (warp == 0 && active) {
      uint32_t cA[8], cF[8];
      generic_group(src, len, e, und[lane], Fsm + lane, G, cA, cF);
      finish_group(cA, cF, e, und[lane], g, n, accept, errc);
    }
  }
}

// ---------------------------------------------------------------------------
// TMA version: CTA = 4 warps, G = 32 groups (one tile of 1024 pairs).  Phase 1:
// warp w encodes groups w, w+4, ...; the 32 read rows and the 32 reference rows
// of a group are each one contiguous span brought in by cp.async.bulk, two
// buffers per warp alternating between the read span and the reference span so
// that the next span lands while the current one is encoded.  The encoder is
// the one of gk_encode (encode_group_v2), emitting into the shared packed tile.
// Phase 2 as in the generic kernel.
template <int SM4, bool LPART, int NIT, uint32_t BUFB>
__device__ __forceinline__ void ascii_phase1(const uint8_t* __restrict__ reads,
                                             const uint8_t* __restrict__ refs, int stride,
                                             int len, int64_t gbase, uint2* pq, uint2* pr,
                                             uint32_t* und, uint8_t* stg, uint32_t buf_bytes,
                                             uint64_t* bars, int P) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t span = 32u * (uint32_t)stride;
  RowAddr<SM4> ra;
  ra.init(smem_u32(stg), (uint32_t)stride, lane);
  // span sequence: (g0 reads -> buf0), (g0 refs -> buf1), (g1 reads -> buf0), ...
  auto issue = [&](int k) {  // k-th span of this warp
    const int gl = warp + 4 * (k >> 1);
    const uint8_t* src = ((k & 1) ? refs : reads) + (gbase + gl) * (int64_t)span;
    uint64_t* bar = &bars[k & 1];
    fence_proxy_async();
    mbar_arrive_expect_tx(bar, span);
    tma_load_1d(stg + (k & 1) * buf_bytes, src, span, bar);
  };
  constexpr int NSPAN = 2 * 8;  // 8 groups per warp (G = 32), 2 spans each
  if (lane == 0) {
    issue(0);
    issue(1);
  }
  uint32_t u = 0u;
#pragma unroll 1
  for (int k = 0; k < NSPAN; ++k) {
    const int b = k & 1;
    mbar_wait(&bars[b], (uint32_t)(k >> 1) & 1u);
    const int gl = warp + 4 * (k >> 1);
    uint2* dst = (b ? pr : pq) + gl;
    auto emit = [&](int q, int m, uint32_t hi, uint32_t lo) { dst[(4 * q + m) * P] = make_uint2(hi, lo); };
    const uint32_t uu = b == 0 ? encode_group_v2<SM4, LPART, NIT, 0u>(ra, len, emit)
                               : encode_group_v2<SM4, LPART, NIT, BUFB>(ra, len, emit);
    u |= uu;
    if (b) {
      if (lane == 0) und[gl] = u;
      u = 0u;
    }
    __syncwarp();
    if (lane == 0 && k + 2 < NSPAN) issue(k + 2);
  }
}

template <int E, int PMAX>
__global__ void __launch_bounds__(128) filter_ascii_tma_kernel(
    const uint8_t* __restrict__ reads, const uint8_t* __restrict__ refs, int stride,
    int64_t ntiles_full, int64_t n, int len, int e, uint32_t* __restrict__ accept,
    uint8_t* __restrict__ errc) {
  constexpr int G = 32, P = G + 1;
  constexpr uint32_t BUF = 32u * PMAX;
  constexpr int NIT = PMAX / 128;
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* stg = sm;                                              // [4 warps][2][BUF]
  uint2* pq = reinterpret_cast<uint2*>(sm + 4 * 2 * BUF);        // [len][P]
  uint2* pr = pq + (size_t)len * P;
  uint32_t* und = reinterpret_cast<uint32_t*>(pr + (size_t)len * P);  // [32]
  uint64_t* bars = reinterpret_cast<uint64_t*>(und + 32) + 2 * warp;
  if (lane == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const int64_t tile = blockIdx.x;
  if (tile >= ntiles_full) return;
  const int64_t gbase = tile * G;
  uint8_t* mystg = stg + (size_t)warp * 2 * BUF;
  const bool lpart = (len & 3) != 0;
  switch ((stride & 3) * 2 + (lpart ? 1 : 0)) {
    case 0: ascii_phase1<0, false, NIT, BUF>(reads, refs, stride, len, gbase, pq, pr, und, mystg, BUF, bars, P); break;
    case 1: ascii_phase1<0, true, NIT, BUF>(reads, refs, stride, len, gbase, pq, pr, und, mystg, BUF, bars, P); break;
    case 2: ascii_phase1<1, false, NIT, BUF>(reads, refs, stride, len, gbase, pq, pr, und, mystg, BUF, bars, P); break;
    case 3: ascii_phase1<1, true, NIT, BUF>(reads, refs, stride, len, gbase, pq, pr, und, mystg, BUF, bars, P); break;
    case 4: ascii_phase1<2, false, NIT, BUF>(reads, refs, stride, len, gbase, pq, pr, und, mystg, BUF, bars, P); break;
    case 5: ascii_phase1<2, true, NIT, BUF>(reads, refs, stride, len, gbase, pq, pr, und, mystg, BUF, bars, P); break;
    case 6: ascii_phase1<3, false, NIT, BUF>(reads, refs, stride, len, gbase, pq, pr, und, mystg, BUF, bars, P); break;
    default: ascii_phase1<3, true, NIT, BUF>(reads, refs, stride, len, gbase, pq, pr, und, mystg, BUF, bars, P); break;
  }
  __syncthreads();

  const int64_t g = gbase + lane;
  SmemGroupSrc src;
  src.q = pq + lane;
  src.r = pr + lane;
  src.len = len;
  src.pstride = P;
  if constexpr (E >= 0) {
    int chunk = (len + 3) / 4;
    chunk = (chunk + 3) & ~3;
    const int lo = warp * chunk;
    int hi = lo + chunk;
    if (hi > len) hi = len;
    uint32_t cA[8], cF[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) cA[b] = cF[b] = 0u;
    if (lo < hi) {
      SinglePass<E> sp;
      run_range<E>(sp, src, len, lo, hi);
      sp.cA.planes(cA);
      sp.cF.planes(cF);
    }
    uint32_t* xch = reinterpret_cast<uint32_t*>(stg);  // staging is free now
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      xch[(warp * 16 + b) * 32 + lane] = cA[b];
      xch[(warp * 16 + 8 + b) * 32 + lane] = cF[b];
    }
    __syncthreads();
    if (warp == 0) {
      for (int w = 1; w < 4; ++w) {
        add_planes(cA, xch + (w * 16) * 32 + lane, 32);
        add_planes(cF, xch + (w * 16 + 8) * 32 + lane, 32);
      }
      finish_group(cA, cF, e, und[lane], g, n, accept, errc);
    }
  } else {
    if (warp == 0) {
      uint32_t cA[8], cF[8];
      uint32_t* Fsm = reinterpret_cast<uint32_t*>(stg);  // [len][32] fits in the staging area
      generic_group(src, len, e, und[lane], Fsm + lane, 32, cA, cF);
      finish_group(cA, cF, e, und[lane], g, n, accept, errc);
    }
  }
}

template <int E, int PMAX>
static void launch_ascii_tma(const uint8_t* reads, const uint8_t* refs, int stride,
                             int64_t ntiles, int64_t n, int len, int e, uint32_t* accept,
                             uint8_t* errc, cudaStream_t stream) {
  const size_t smem = (size_t)4 * 2 * 32 * PMAX + 2 * (size_t)len * 33 * 8 + 32 * 4 + 4 * 2 * 8 + 16;
  auto kern = filter_ascii_tma_kernel<E, PMAX>;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  count_launch();
  kern<<<(unsigned)ntiles, 128, smem, stream>>>(reads, refs, stride, ntiles, n, len, e, accept,
                                                errc);
}

// returns the number of tiles handled by the TMA kernel
template <int E>
static int64_t try_ascii_tma(const uint8_t* reads, const uint8_t* refs, int64_t stride, int64_t n,
                             int len, int e, uint32_t* accept, uint8_t* errc,
                             cudaStream_t stream) {
  if (!GK_ASCII_TMA) return 0;
  if (((reinterpret_cast<uintptr_t>(reads) | reinterpret_cast<uintptr_t>(refs)) & 15u) != 0)
    return 0;
  // a tile copies 1024*stride bytes per set: with stride > len the tile holding the
  // last row would over-read the caller's (n-1)*stride+len bytes -> generic path
  const int64_t ntiles = stride == len ? n / 1024 : (n - 1) / 1024;
  if (ntiles == 0) return 0;
  // the generic fallback (E < 0) keeps F[len][32] in the staging area
  if (E < 0 && (size_t)len * 32 * 4 > (size_t)4 * 2 * 32 * (stride <= 128 ? 128 : stride <= 256 ? 256 : 512))
    return 0;
  if (stride <= 128) launch_ascii_tma<E, 128>(reads, refs, (int)stride, ntiles, n, len, e, accept, errc, stream);
  else if (stride <= 256) launch_ascii_tma<E, 256>(reads, refs, (int)stride, ntiles, n, len, e, accept, errc, stream);
  else if (stride <= 384) launch_ascii_tma<E, 384>(reads, refs, (int)stride, ntiles, n, len, e, accept, errc, stream);
  else return 0;
  return ntiles;
}

template <int E>
static void launch_ascii_t(const uint8_t* reads, const uint8_t* refs, int64_t stride, int64_t n,
                           int len, int e, uint32_t* accept, uint8_t* errc, cudaStream_t stream) {
  const AsciiLayout L = ascii_layout(len, stride, E < 0);
  const int64_t ngroups = (n + 31) / 32;
  const int64_t blocks = (ngroups + L.G - 1) / L.G;
  if (L.total > 48 * 1024)
    cudaFuncSetAttribute(filter_ascii_kernel<E>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)L.total);
  count_launch();
  filter_ascii_kernel<E><<<(unsigned)blocks, 128, L.total, stream>>>(
      reads, refs, stride, n, len, e, L.G, (uint32_t)L.packed, (uint32_t)L.staging, accept, errc);
}

template <int E>
void launch_ascii_all(const uint8_t* reads, const uint8_t* refs, int64_t stride, int64_t n,
                             int len, int e, uint32_t* accept, uint8_t* errc,
                             cudaStream_t stream) {
  const int64_t done = try_ascii_tma<E>(reads, refs, stride, n, len, e, accept, errc, stream);
  const int64_t p0 = done * 1024;  // remaining pairs: generic kernel on shifted pointers
  if (p0 < n)
    launch_ascii_t<E>(reads + p0 * stride, refs + p0 * stride, stride, n - p0, len, e,
                      accept + p0 / 32, errc ? errc + p0 : nullptr, stream);
}

}  // namespace gk
