// gk_fused_l2.cu -- a1..a6 fused from ASCII with the packed tile staged in L2
// (gk_filter_ascii_ws): the encoder (HBM-bound) and the filtration (ALU-bound)
// of different tiles run at the same time on every SM.
//
// Why.  The unfused path (gk_encode x2 + gk_filter) runs the two phases one
// after the other over the whole batch: while the encoder streams ASCII at ~0.8
// of HBM the integer pipe is half idle, and while the filter saturates the ALU
// pipe HBM idles; in between the packed planes make a round trip through HBM
// (L/2 bytes per pair written, then read back).  The tile-per-CTA kernels of
// gk_fused.cu keep the tile in shared memory, which caps them at 1-2 CTAs per SM
// (51-128 KB per tile) and leaves their span loads latency-bound.
//
// Here a persistent CTA (4 warps) loops over tiles of 1024 pairs:
//   phase E  the tile's 64 spans (32 ASCII rows each, reads then references)
//            are encoded exactly as encode3_kernel does (gk_encode3.cuh: TMA
//            bulk span -> SWAR code/validity bits -> shuffle transpose ->
//            [plane][pos*5+group] in shared memory -> full 32-byte sectors) into
//            the CTA's slot of a global scratch buffer in the packed tile layout
//            (word (pos*32 + group)*2 + plane, include/gatekeeper.h).  One slot
//            per resident CTA (2*len*256 bytes: 51 KB at 100 bp, 128 KB at
//            250 bp), rewritten tile after tile, so the slots stay in the
//            126 MB L2 and the packed words never reach HBM;
//   phase F  the 4 warps split the tile's positions (lane = group of 32 pairs)
//            and run the same filtration cores as gk_filter (single pass
//            sp<E> for e <= GK_SP_EMAX, block-transposed bt2 above) on the
//            slot through ordinary (L1-coherent) global loads;
//   combine  per-warp bit-sliced counters are summed through shared memory and
//            warp 0 writes the tile's accept bits / error counts (finish_group).
// With 2-3 CTAs per SM the CTAs drift into different phases, so the encoder's
// HBM streaming overlaps the filtration's LOP3 stream.  The next tile's first
// spans are prefetched by TMA while the current tile is being filtered.
// Partial tiles: spans that would read past the caller's (n-1)*stride+len bytes
// are staged with bounded loads; groups past n are not encoded (their scratch
// words are stale, their pairs are never written).
#include "gk_bt2.cuh"
#include "gk_common.cuh"
#include "gk_encode3.cuh"
#include "gk_encode_core.cuh"
#include "gk_filter_core.cuh"
#include "gk_kernels.cuh"
#include "gk_tma.cuh"

#ifndef GK_L2_B
#define GK_L2_B 8  // positions per block of the bt2 phase
#endif
#ifndef GK_L2_MINB_SP
#define GK_L2_MINB_SP 3
#endif
#ifndef GK_L2_MINB_BT
#define GK_L2_MINB_BT 2
#endif
#ifndef GK_L2_L1PF
#define GK_L2_L1PF 1  // bt2 phase: prefetch upcoming read words into L1 (as bt2::GMem)
#endif
#ifndef GK_L2_EVF
#define GK_L2_EVF 1  // ASCII span loads with an L2 evict_first hint
#endif
#ifndef GK_L2_PF
#define GK_L2_PF 0  // spans prefetched into L2 beyond the TMA ring (per warp)
#endif
#ifndef GK_L2_NB
#define GK_L2_NB 2  // TMA span buffers per warp
#endif

namespace gk {
namespace l2f {

constexpr int NW = 4;  // warps per CTA

// Words of the lane's group in the CTA's scratch slot (position stride 32 uint2);
// plain loads: the slot was written by this CTA earlier in the kernel (the
// read-only path would not be coherent with those writes).
struct Src {
  static constexpr bool kHoistLoads = true;
  const uint2* q;
  const uint2* r;
  int len;
  __device__ __forceinline__ uint2 ldq(int pos) const {
    return (pos >= 0 && pos < len) ? q[(int64_t)pos * GK_WARP] : make_uint2(0u, 0u);
  }
  __device__ __forceinline__ uint2 ldr(int pos) const {
    return (pos >= 0 && pos < len) ? r[(int64_t)pos * GK_WARP] : make_uint2(0u, 0u);
  }
  __device__ __forceinline__ uint2 ldq_nc(int pos) const { return q[(int64_t)pos * GK_WARP]; }
  __device__ __forceinline__ uint2 ldr_nc(int pos) const { return r[(int64_t)pos * GK_WARP]; }
};

// bt2 memory policy for the slot (as bt2::GMem, without the read-only path)
struct Mem {
  __device__ __forceinline__ static uint2 ld(const uint2* p, int pos) {
    return p[(int64_t)pos * GK_WARP];
  }
  __device__ __forceinline__ static void prefetch(const uint2* p, int pos) {
#if GK_L2_L1PF
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p + (int64_t)pos * GK_WARP));
#endif
  }
};

// TMA bulk copy global -> shared with an L2 eviction-priority hint: the ASCII
// rows are read exactly once, so they should leave L2 before the tile slots do.
__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, uint32_t bytes,
                                                 uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Positions [lo, hi) of warp w (multiples of 4 apart, balanced in 4-base quads).
__device__ __forceinline__ void pos_range(int len, int w, int& lo, int& hi) {
  const int quads = (len + 3) >> 2;
  lo = 4 * ((quads * w) / NW);
  hi = 4 * ((quads * (w + 1)) / NW);
  if (hi > len) hi = len;
}

// B-position blocks [b0, b1) of warp w: the edge blocks (mostly checked steps)
// weigh 1.5 interior blocks.
template <int B>
__device__ __forceinline__ void block_range(int len, int w, int& b0, int& b1) {
  const int nb = (len + B - 1) / B;
  const int total = 2 * nb + (nb >= 2 ? 2 : 1);
  auto cut = [&](int part) {
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

// Sum of bit-sliced 8-plane counters: a += b (b at stride 32 words).
__device__ __forceinline__ void add8(uint32_t (&a)[8], const uint32_t* b) {
  uint32_t carry = 0u;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t x = a[k], y = b[k * 32];
    a[k] = x ^ y ^ carry;
    carry = (x & y) | (carry & (x ^ y));
  }
}

struct Cfg {
  uint32_t bufb;  // bytes of one span buffer
  uint32_t P;     // words per plane of the output staging ([2][P])
  int nb;         // span buffers per warp
  size_t smem;
  size_t slot;    // scratch bytes per CTA
};

static Cfg cfg_of(int len, int stride, int nb) {
  Cfg c;
  c.bufb = ((uint32_t)(32 * stride + 32) + 127u) & ~127u;
  uint32_t p = (uint32_t)(5 * len);
  p = (p + 31u) & ~31u;
  c.P = p + 16u;  // as encode3_kernel: the two planes' transposed writes hit disjoint banks
  c.nb = nb;
  c.smem = (size_t)NW * nb * c.bufb + (size_t)NW * 2 * c.P * 4 + (size_t)NW * 16 * 32 * 4 +
           64 * 4 + NW * nb * 8;
  c.slot = (size_t)2 * len * 32 * 8;
  return c;
}

}  // namespace l2f

// EP >= 0: single-pass sp<EP> (e == EP); EP < 0: bt2 with B-position blocks.
template <int EP, int NCH, int MODE, int NB, int B, int MINB>
__global__ void __launch_bounds__(l2f::NW * 32, MINB) fused_l2_kernel(
    const uint8_t* __restrict__ reads, const uint8_t* __restrict__ refs, int stride, int64_t n,
    int len, int e, uint32_t bufb, uint32_t P, uint2* ws, uint32_t* __restrict__ accept,
    uint8_t* __restrict__ errc) {
  using namespace l2f;
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* stage = sm + (size_t)warp * NB * bufb;
  // per-warp output staging [2][P] (4 groups x len positions, as encode3_kernel)
  uint32_t* outs = reinterpret_cast<uint32_t*>(sm + (size_t)NW * NB * bufb) + (size_t)warp * 2 * P;
  uint32_t* xch = reinterpret_cast<uint32_t*>(sm + (size_t)NW * NB * bufb) + (size_t)NW * 2 * P;
  uint32_t* und_s = xch + NW * 16 * 32;  // [2][32]
  uint64_t* mybar = reinterpret_cast<uint64_t*>(und_s + 64) + NB * warp;
  const int64_t tiles = (n + 1023) >> 10;
  if ((int64_t)blockIdx.x >= tiles) return;
  if (lane == 0) {
#pragma unroll
    for (int b = 0; b < NB; ++b) mbar_init(&mybar[b], 1);
    fence_mbar_init();
  }
  __syncwarp();
  enc3::Lane ln;
  ln.init(lane);
  uint32_t roff[4], rsh[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t a = (uint32_t)ln.rows[i] * (uint32_t)stride + 4u * (uint32_t)ln.cw;
    roff[i] = MODE == 0 ? a : (a & ~3u);
    rsh[i] = (a & 3u) * 8u;
  }
  const int s2 = (int)(rsh[0] >> 3);
  const uint32_t span = 32u * (uint32_t)stride;
  const int64_t limit = (n - 1) * (int64_t)stride + len;  // bytes the caller owns per set
  uint2* slot = ws + (size_t)blockIdx.x * 2 * len * 32;
  uint64_t policy = 0;
  if (GK_L2_EVF) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));

  // span j (0..15) of a tile for warp w: block bl = j >> 2 (set bl >> 1, 4-group
  // block w + 4*(bl & 1)), group 4*block + (j & 3)
  auto group_of = [&](int j) { return 4 * (warp + 4 * ((j >> 2) & 1)) + (j & 3); };
  auto span_at = [&](int64_t tile, int j, int64_t& off) -> const uint8_t* {
    const int64_t first = (tile * 32 + group_of(j)) * 32;
    off = first * (int64_t)stride;
    return (j >> 3) ? refs : reads;
  };
  auto valid_at = [&](int64_t tile, int j) { return (tile * 32 + group_of(j)) * 32 < n; };
  auto tma_at = [&](int64_t tile, int j) {
    int64_t off;
    span_at(tile, j, off);
    return valid_at(tile, j) && off + span <= limit;
  };
  // span c of this warp's sequence (c = 16 * tile_iteration + j)
  auto tile_of = [&](uint32_t c) { return (int64_t)blockIdx.x + (int64_t)(c >> 4) * gridDim.x; };
  auto issue = [&](uint32_t c) {
    const int64_t tile = tile_of(c);
    const int j = (int)(c & 15u);
    if (tile >= tiles || !tma_at(tile, j)) return;
    int64_t off;
    const uint8_t* base = span_at(tile, j, off);
    const int buf = (int)(c % NB);
    fence_proxy_async();
    mbar_arrive_expect_tx(&mybar[buf], span);
    if (GK_L2_EVF)
      tma_load_1d_hint(stage + (size_t)buf * bufb, base + off, span, &mybar[buf], policy);
    else
      tma_load_1d(stage + (size_t)buf * bufb, base + off, span, &mybar[buf]);
  };
  // L2 prefetch GK_L2_PF spans beyond the TMA ring: bytes in flight decoupled
  // from the shared memory of the ring
  auto prefetch = [&](uint32_t c) {
    const int64_t tile = tile_of(c);
    const int j = (int)(c & 15u);
    if (tile >= tiles || !tma_at(tile, j)) return;
    int64_t off;
    const uint8_t* base = span_at(tile, j, off);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + off), "r"(span)
                 : "memory");
  };
  if (lane == 0) {
#pragma unroll
    for (int b = 0; b < NB; ++b) issue((uint32_t)b);
#pragma unroll 1
    for (int d = 0; d < GK_L2_PF; ++d) prefetch((uint32_t)(NB + d));
  }
  uint32_t ph = 0u;  // parity bit per span buffer
  uint32_t cnt = 0u;
#pragma unroll 1
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    // ---- phase E: 16 spans per warp -> the slot (no CTA barrier inside)
#pragma unroll 1
    for (int j = 0; j < 16; ++j, ++cnt) {
      const int buf = (int)(cnt % NB);
      uint8_t* sbuf = stage + (size_t)buf * bufb;
      const bool valid = valid_at(tile, j);
      if (valid) {
        if (tma_at(tile, j)) {
          mbar_wait(&mybar[buf], (ph >> buf) & 1u);
          ph ^= 1u << buf;
        } else {  // bounded staging of the last rows of the batch
          int64_t off;
          const uint8_t* base = span_at(tile, j, off);
          __syncwarp();
          stage_span(base + off, limit - off, sbuf, lane, 32);
          __syncwarp();
        }
      }
      uint32_t und = 0u;
      if (valid) und = enc3_group<NCH, MODE>(sbuf, roff, rsh, s2, len, ln, outs, P, j & 3);
      if (lane == 0) und_s[(j >> 3) * 32 + group_of(j)] = und;
      __syncwarp();
      if (lane == 0) {  // refill this buffer with the span NB ahead (maybe the next tile's)
        issue(cnt + NB);
        prefetch(cnt + NB + GK_L2_PF);
      }
      if ((j & 3) == 3) {  // 4 groups done: copy out as full 32-byte sectors
        uint2* dst = slot + (size_t)(j >> 3) * len * 32 + 4 * (warp + 4 * ((j >> 2) & 1));
        for (int t = lane; t < 4 * len; t += 32) {
          const int pos = t >> 2, w = t & 3;
          dst[pos * 32 + w] = make_uint2(outs[pos * 5 + w], outs[P + pos * 5 + w]);
        }
        __syncwarp();
      }
    }
    __syncthreads();  // the slot and und_s are complete
    const uint32_t und = und_s[lane] | und_s[32 + lane];
    // ---- phase F: the warp's share of the positions, lane = group
    const uint2* q = slot + lane;
    const uint2* r = slot + (size_t)len * 32 + lane;
    uint32_t cA[8], cF[8];
    if constexpr (EP >= 0) {
#pragma unroll
      for (int b = 0; b < 8; ++b) cA[b] = cF[b] = 0u;
      int lo, hi;
      pos_range(len, warp, lo, hi);
      if (lo < hi) {
        Src src;
        src.q = q;
        src.r = r;
        src.len = len;
        SinglePass<EP> sp;
        run_range<EP>(sp, src, len, lo, hi);
        sp.cA.planes(cA);
        sp.cF.planes(cF);
      }
    } else {
      CsaCounter ca, cf;
      ca.clear();
      cf.clear();
      int b0, b1;
      block_range<B>(len, warp, b0, b1);
      if (b0 < b1) {
        bt2::Win<B> R;
#pragma unroll
        for (int c = 0; c < B + 4; ++c) {
          const uint2 v = bt2::ldc<Mem>(r, B * b0 - 2 + c, len);
          R.h[c] = v.x;
          R.l[c] = v.y;
        }
#pragma unroll 1
        for (int b = b0; b < b1; ++b)
          bt2::block<B, GK_BT2_LA_E, Mem>(q, r, R, B * b, len, e, 1, ca, cf, bt2::NoHook{});
      }
      ca.planes(cA);
      cf.planes(cF);
    }
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      xch[(warp * 16 + b) * 32 + lane] = cA[b];
      xch[(warp * 16 + 8 + b) * 32 + lane] = cF[b];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll 1
      for (int w = 1; w < NW; ++w) {
        add8(cA, xch + (w * 16) * 32 + lane);
        add8(cF, xch + (w * 16 + 8) * 32 + lane);
      }
      const int64_t g = tile * 32 + lane;
      if (g * 32 < n) finish_group(cA, cF, e, und, g, n, accept, errc);
    }
  }
}

namespace l2f {

// resident CTAs per SM asked of ptxas, per kernel kind (registers: sp ~150-170,
// bt2 with 16-position blocks ~250)
template <int EP>
struct Occ {
  static constexpr int MINB = EP >= 0 ? GK_L2_MINB_SP : GK_L2_MINB_BT;
};

template <int EP, int NCH, int MODE>
static void launch_t(const uint8_t* reads, const uint8_t* refs, int stride, int64_t n, int len,
                     int e, void* ws, size_t ws_bytes, uint32_t* accept, uint8_t* errc,
                     cudaStream_t stream) {
  constexpr int NB = GK_L2_NB;
  constexpr int B = GK_L2_B;
  const Cfg c = cfg_of(len, stride, NB);
  auto kern = fused_l2_kernel<EP, NCH, MODE, NB, B, Occ<EP>::MINB>;
  struct Seen {
    int dev;
    size_t smem;
    int grid;
  };
  static thread_local Seen seen{-1, 0, 0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (seen.dev != dev || seen.smem != c.smem) {
    if (c.smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
    int sms = 148, per_sm = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32, c.smem);
    seen = Seen{dev, c.smem, sms * (per_sm < 1 ? 1 : per_sm)};
  }
  const int64_t tiles = (n + 1023) / 1024;
  int64_t grid = seen.grid;
  const int64_t slots = (int64_t)(ws_bytes / c.slot);
  if (grid > slots) grid = slots;
  if (grid > tiles) grid = tiles;
  count_launch();
  kern<<<(unsigned)grid, NW * 32, c.smem, stream>>>(reads, refs, stride, n, len, e, c.bufb, c.P,
                                                     reinterpret_cast<uint2*>(ws), accept, errc);
}

template <int NCH, int MODE>
static bool dispatch_e(const uint8_t* reads, const uint8_t* refs, int stride, int64_t n, int len,
                       int e, void* ws, size_t ws_bytes, uint32_t* accept, uint8_t* errc,
                       cudaStream_t stream) {
#define GK_L2E(E)                                                                        \
  case E:                                                                                \
    launch_t<E, NCH, MODE>(reads, refs, stride, n, len, e, ws, ws_bytes, accept, errc,   \
                           stream);                                                      \
    return true;
  switch (e) {
    GK_L2E(5) GK_L2E(7)
    default:
      if (e <= GK_SP_EMAX) return false;
      launch_t<-1, NCH, MODE>(reads, refs, stride, n, len, e, ws, ws_bytes, accept, errc, stream);
      return true;
  }
#undef GK_L2E
}

}  // namespace l2f

// Scratch bytes for the L2-staged fused kernel: one slot per resident CTA.
size_t fused_l2_workspace_bytes(int len) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (size_t)sms * 3 * l2f::cfg_of(len, len, 1).slot;
}

// false: this (len, stride, e) has no L2-staged instantiation or the inputs are
// not 16-byte aligned / the workspace holds no slot; the caller falls back.
bool launch_fused_l2(const uint8_t* reads, const uint8_t* refs, int64_t stride, int64_t n,
                     int len, int e, void* ws, size_t ws_bytes, uint32_t* accept, uint8_t* errc,
                     cudaStream_t stream) {
  if (((reinterpret_cast<uintptr_t>(reads) | reinterpret_cast<uintptr_t>(refs) |
        reinterpret_cast<uintptr_t>(ws)) & 15u) != 0)
    return false;
  if (stride > 512 || ws == nullptr || ws_bytes < l2f::cfg_of(len, (int)stride, 1).slot) return false;
  const int nch = (len + 15) >> 4;
  const int mode = (stride & 3) == 0 ? 0 : ((stride & 3) == 2 ? 2 : 1);
  const int s = (int)stride;
  if (nch == 7 && mode == 0)
    return l2f::dispatch_e<7, 0>(reads, refs, s, n, len, e, ws, ws_bytes, accept, errc, stream);
  if (nch == 10 && mode == 2)
    return l2f::dispatch_e<10, 2>(reads, refs, s, n, len, e, ws, ws_bytes, accept, errc, stream);
  if (nch == 16 && mode == 2)
    return l2f::dispatch_e<16, 2>(reads, refs, s, n, len, e, ws, ws_bytes, accept, errc, stream);
  return false;
}

}  // namespace gk
