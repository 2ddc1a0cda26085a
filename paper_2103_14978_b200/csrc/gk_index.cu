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
// gather: one warp per group of 32 pairs (lane j = pair j).  For each chunk of
// 32 positions lane j funnel-shifts its window bits out of two plane words
// (any bit offset), then a 5-stage shuffle transpose of the 32x32 bit matrix
// turns "32 positions of pair j" into "position i of 32 pairs" -- the
// bit-sliced packed layout of gk_encode (include/gatekeeper.h), which
// gk_filter / gk_filter_sweep consume unchanged.
#include "gk_common.cuh"

namespace gk {

// ---- packing: ASCII rows -> bit planes ----------------------------------------
// One thread per 32 consecutive bases of the concatenation (row r, base i) ->
// bit r*len + i.  Code: high = ASCII bit 2, low = bit 1 ^ bit 2 (as gk_encode);
// undefined = not one of A C G T a c g t.
__global__ void pack_planes_kernel(const uint8_t* __restrict__ rows, int64_t n_rows, int len,
                                   int64_t stride, uint32_t* __restrict__ hi,
                                   uint32_t* __restrict__ lo, uint32_t* __restrict__ bad,
                                   int64_t nwords) {
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
    hi[w] = h;
    lo[w] = l;
    bad[w] = b;
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

__device__ __forceinline__ uint32_t plane_bits(const uint32_t* __restrict__ p, int64_t bit) {
  const int64_t w = bit >> 5;
  const uint32_t sh = (uint32_t)(bit & 31);
  return __funnelshift_r(__ldg(p + w), __ldg(p + w + 1), sh);
}

__global__ void __launch_bounds__(128) gather_windows_kernel(
    const uint32_t* __restrict__ hi, const uint32_t* __restrict__ lo,
    const uint32_t* __restrict__ bad, int64_t nbases, const int64_t* __restrict__ offsets,
    int64_t n, int len, uint32_t* __restrict__ packed, uint32_t* __restrict__ undef,
    int64_t ngroups_total) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= ngroups_total) return;
  const int64_t p = g * 32 + lane;
  const int64_t tile = g >> 5;
  const int gl = (int)(g & 31);
  int64_t off = p < n ? offsets[p] : -1;
  // a window outside [0, nbases) makes the pair undefined (accepted, 255)
  bool oob = p < n && (off < 0 || off + len > nbases);
  const bool live = p < n && !oob;
  if (!live) off = 0;
  uint32_t anybad = 0u;
  uint2* out = reinterpret_cast<uint2*>(packed);
  for (int c0 = 0; c0 < len; c0 += 32) {
    const int nb = len - c0 < 32 ? len - c0 : 32;
    const uint32_t vm = nb == 32 ? 0xFFFFFFFFu : ((1u << nb) - 1u);
    uint32_t xh = 0u, xl = 0u;
    if (live) {
      xh = plane_bits(hi, off + c0) & vm;
      xl = plane_bits(lo, off + c0) & vm;
      anybad |= plane_bits(bad, off + c0) & vm;
    }
    const uint32_t yh = warp_transpose32(xh, lane);
    const uint32_t yl = warp_transpose32(xl, lane);
    if (lane < nb) out[(tile * len + c0 + lane) * 32 + gl] = make_uint2(yh, yl);
  }
  const uint32_t u = __ballot_sync(0xFFFFFFFFu, anybad != 0u || oob);
  if (lane == 0) undef[g] = u;
}

int launch_pack_planes(const uint8_t* rows, int64_t n_rows, int len, int64_t stride, uint32_t* hi,
                       uint32_t* lo, uint32_t* bad, cudaStream_t stream) {
  const int64_t total = n_rows * (int64_t)len;
  const int64_t nwords = (total + 31) / 32 + 1;  // + 1: the funnel shift's look-ahead word
  int64_t blocks = (nwords + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  pack_planes_kernel<<<(unsigned)blocks, 256, 0, stream>>>(rows, n_rows, len, stride, hi, lo, bad,
                                                           nwords);
  return 0;
}

int launch_gather_windows(const uint32_t* hi, const uint32_t* lo, const uint32_t* bad,
                          int64_t nbases, const int64_t* offsets, int64_t n, int len,
                          uint32_t* packed, uint32_t* undef, cudaStream_t stream) {
  const int64_t ngroups_total = (n + 1023) / 1024 * 32;  // whole tiles (zero-filled tail)
  const int64_t blocks = (ngroups_total + 3) / 4;
  gather_windows_kernel<<<(unsigned)blocks, 128, 0, stream>>>(hi, lo, bad, nbases, offsets, n, len,
                                                              packed, undef, ngroups_total);
  return 0;
}

}  // namespace gk
