// gk_filter_ascii_impl.cuh -- a1..a6 fused, generic fallback: the kernel behind
// gk_filter_ascii when the tile-per-CTA kernels of gk_fused.cu do not fit in
// shared memory (long reads) or the inputs are not 16-byte aligned.
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
                      int len, int e, uint32_t* accept, uint8_t* errc, cudaStream_t stream) {
  launch_ascii_t<E>(reads, refs, stride, n, len, e, accept, errc, stream);
}

}  // namespace gk
