// gk_index.cu -- reference-index mode (PAPER.md section
// 3.5 :148-152): the reference genome is encoded ONCE on the device into bit
// planes (high code bit, low code bit, "undefined" bit per base; 2-bit code
// A=00 C=01 G=10 T=11, :49, :91-93; any byte outside ACGTacgt is undefined,
// :95 / reading R8), and each candidate (read, reference position) pair then
// takes its L-base reference window straight from the planes instead of
// shipping an ASCII copy of the segment per pair (:59, :87).  Reads are packed
// the same way (row r at bits [r*L, r*L+L)), so a read with many candidates is
// encoded once.
//
// gather: one CTA per tile, one warp per group of 32 pairs (lane j = pair j).  For each chunk of
// 32 positions lane j funnel-shifts its window bits out of two plane words
// (any bit offset), then a 5-stage shuffle transpose of the 32x32 bit matrix
// turns "32 positions of pair j" into "position i of 32 pairs" -- the
// bit-sliced packed layout of gk_encode (include/gatekeeper.h), which
// gk_filter / gk_filter_sweep consume unchanged.
#include "gk_common.cuh"
#include "gk_kernels.cuh"

namespace gk {

// ---- packing: ASCII rows -> bit planes ----------------------------------------
// One thread per 32 consecutive bases of the concatenation (row r, base i) ->
// bit r*len + i.  Code: high = ASCII bit 2, low = bit 1 ^ bit 2 (as gk_encode);
// undefined = not one of A C G T a c g t.
__global__ void pack_planes_kernel(const uint8_t* __restrict__ rows, int64_t n_rows, int len,
                                   int64_t stride, uint4* __restrict__ planes, int64_t nwords) {
  const int64_t total = n_rows * (int64_t)len;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = 0u, l = 0u, b = 0u;
    int64_t idx = w * 32;
    int64_t r = idx / len;
    int i = (int)(idx - r * len);
    for (int k = 0; k < 32 && idx + k < total; ++k) {
      const uint32_t c = __ldg(rows + r * stride + i);
      const uint32_t u = c & 0xDFu;  // upper case
      const bool valid = u == 'A' || u == 'C' || u == 'G' || u == 'T';
      const uint32_t b2 = (c >> 2) & 1u, b1 = (c >> 1) & 1u;
      h |= (valid ? b2 : 0u) << k;
      l |= (valid ? (b1 ^ b2) : 0u) << k;
      b |= (valid ? 0u : 1u) << k;
      if (++i == len) {
        i = 0;
        ++r;
      }
    }
    planes[w] = make_uint4(h, l, b, 0u);
  }
}

// ---- gather: windows -> bit-sliced packed words --------------------------------
// 32x32 bit transpose across a warp: on entry lane j holds x (bit i = element
// (j, i)); on exit lane i holds bit j = element (j, i).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
  const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int t = 0; t < 5; ++t) {
    const int s = 16 >> t;
    const uint32_t m = masks[t];
    const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, s);
    // lanes with bit s clear keep their low halves (bit blocks of size s) and take
    // the partner's low halves into their high halves; lanes with bit s set the
    // converse
    x = (lane & s) ? ((x & ~m) | ((y >> s) & m)) : ((x & m) | ((y << s) & ~m));
  }
  return x;
}

// Bits [bit, bit+32) of the three planes: two 16-byte loads (the planes of a
// 32-base block are interleaved, so a random window touches 2-3 sectors, not 6).
__device__ __forceinline__ void window_bits(const uint4* __restrict__ p, int64_t bit, uint32_t& h,
                                            uint32_t& l, uint32_t& b) {
  const int64_t w = bit >> 5;
  const uint32_t sh = (uint32_t)(bit & 31);
  const uint4 a = __ldg(p + w), c = __ldg(p + w + 1);
  h = __funnelshift_r(a.x, c.x, sh);
  l = __funnelshift_r(a.y, c.y, sh);
  b = __funnelshift_r(a.z, c.z, sh);
}

// One CTA of 32 warps per tile of 1024 pairs (warp = group of 32 pairs, lane =
// pair).  Per chunk of 32 positions each warp transposes its words into a
// shared [32 positions][32 groups] staging tile, so the tile's chunk -- 32 x
// 256 contiguous bytes of the packed layout -- leaves in full, coalesced lines
// (a warp alone would write 8-byte pieces at a 256-byte stride).
__global__ void __launch_bounds__(1024) gather_windows_kernel(
    const uint4* __restrict__ planes, int64_t nbases, const int64_t* __restrict__ offsets,
    int64_t n, int len, uint32_t* __restrict__ packed, uint32_t* __restrict__ undef) {
  __shared__ uint2 stage[32][32];  // [position in chunk][group in tile]
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t tile = blockIdx.x;
  const int64_t g = tile * 32 + warp;
  const int64_t p = g * 32 + lane;
  int64_t off = p < n ? offsets[p] : -1;
  // a window outside [0, nbases) makes the pair undefined (accepted, 255)
  const bool oob = p < n && (off < 0 || off + len > nbases);
  const bool live = p < n && !oob;
  if (!live) off = 0;
  uint32_t anybad = 0u;
  uint4* dst = reinterpret_cast<uint4*>(packed + tile * (int64_t)len * 64);
  for (int c0 = 0; c0 < len; c0 += 32) {
    const int nb = len - c0 < 32 ? len - c0 : 32;
    const uint32_t vm = nb == 32 ? 0xFFFFFFFFu : ((1u << nb) - 1u);
    uint32_t xh = 0u, xl = 0u;
    if (live) {
      uint32_t xb;
      window_bits(planes, off + c0, xh, xl, xb);
      xh &= vm;
      xl &= vm;
      anybad |= xb & vm;
    }
    const uint32_t yh = warp_transpose32(xh, lane);
    const uint32_t yl = warp_transpose32(xl, lane);
    stage[lane][warp] = make_uint2(yh, yl);
    __syncthreads();
    // nb positions x 256 bytes = nb * 16 uint4, contiguous from position c0
    const uint4* src = reinterpret_cast<const uint4*>(&stage[0][0]);
    for (int t = threadIdx.x; t < nb * 16; t += 1024) dst[(int64_t)c0 * 16 + t] = src[t];
    __syncthreads();
  }
  const uint32_t u = __ballot_sync(0xFFFFFFFFu, anybad != 0u || oob);
  if (lane == 0) undef[g] = u;
}

int launch_pack_planes(const uint8_t* rows, int64_t n_rows, int len, int64_t stride,
                       uint32_t* planes, cudaStream_t stream) {
  const int64_t total = n_rows * (int64_t)len;
  const int64_t nwords = (total + 31) / 32 + 1;  // + 1: the funnel shift's look-ahead word
  int64_t blocks = (nwords + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  count_launch();
  pack_planes_kernel<<<(unsigned)blocks, 256, 0, stream>>>(rows, n_rows, len, stride,
                                                           reinterpret_cast<uint4*>(planes), nwords);
  return 0;
}

int launch_gather_windows(const uint32_t* planes, int64_t nbases, const int64_t* offsets, int64_t n,
                          int len, uint32_t* packed, uint32_t* undef, cudaStream_t stream) {
  const int64_t tiles = (n + 1023) / 1024;  // whole tiles (zero-filled tail)
  count_launch();
  gather_windows_kernel<<<(unsigned)tiles, 1024, 0, stream>>>(
      reinterpret_cast<const uint4*>(planes), nbases, offsets, n, len, packed, undef);
  return 0;
}

}  // namespace gk
