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
// gather (gather2_kernel below): lane j = pair j funnel-shifts its window bits
// out of the plane blocks (any bit offset), then a 5-stage shuffle transpose of
// the 32x32 bit matrix turns "32 positions of pair j" into "position i of 32
// pairs" -- the bit-sliced packed layout of gk_encode (include/gatekeeper.h),
// which gk_filter / gk_filter_sweep consume unchanged.
#include "gk_common.cuh"
#include "gk_kernels.cuh"

namespace gk {

// ---- packing: ASCII rows -> bit planes ----------------------------------------
// Code: high = ASCII bit 2, low = bit 1 ^ bit 2 (as gk_encode); undefined = not
// one of A C G T a c g t (its code bits are 0).  Base r*len + i of the
// concatenation is bit (r*len+i) % 32 of plane word (r*len+i) / 32.
//
// Contiguous rows (one row -- a genome -- or stride == len): lane = plane word,
// its 32 bases are 32 contiguous bytes (two 16-byte loads; a warp reads 1 KB
// contiguous), decoded 4 bytes at a time with SWAR tests and a multiply-gather
// of the 4 byte bits into a nibble.  Other strides: one byte load per base.

// bits 0, 8, 16, 24 of y -> bits 0..3 (the partial products y_k * 2^(7m) land on
// distinct bits 8k+7m, so there are no carries; k+m = 3 gives bits 21..24)
__device__ __forceinline__ uint32_t gather4(uint32_t y) { return (y * 0x00204081u) >> 21 & 0xFu; }

// 4 ASCII bytes -> hi / lo / undefined nibbles (bit k = byte k)
__device__ __forceinline__ void decode4(uint32_t w, uint32_t& hn, uint32_t& ln, uint32_t& un) {
  const uint32_t x = (w ^ (w >> 1)) & 0x06060606u;  // lo at bit 1, hi at bit 2 of each byte
  // validity as gk_encode (gk_encode3.cuh row_word): bits 7,6,3 = 0,1,0 and
  // b4 == b2 & ~b1, b0 != b4
  const uint32_t y = w ^ 0x40404040u;
  const uint32_t g = (w ^ ((w << 2) & ~(w << 3))) | ~(w ^ (w << 4));
  const uint32_t bad = ((g >> 4) | (y >> 3) | (y >> 6) | (y >> 7)) & 0x01010101u;
  un = gather4(bad);
  hn = gather4((x >> 2) & 0x01010101u) & ~un;
  ln = gather4((x >> 1) & 0x01010101u) & ~un;
}

__global__ void pack_planes_contig_kernel(const uint8_t* __restrict__ seq, int64_t total,
                                          uint4* __restrict__ planes, int64_t nwords) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = 0u, l = 0u, u = 0u;
    const int64_t b0 = w * 32;
    if (b0 + 32 <= total) {
      const uint4* src = reinterpret_cast<const uint4*>(seq + b0);
      const uint4 v0 = __ldg(src), v1 = __ldg(src + 1);
      const uint32_t q[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        uint32_t hn, ln, un;
        decode4(q[k], hn, ln, un);
        h |= hn << (4 * k);
        l |= ln << (4 * k);
        u |= un << (4 * k);
      }
    } else {  // the last (partial) word and the look-ahead word: bytes < total only
      for (int k = 0; k < 32 && b0 + k < total; ++k) {
        uint32_t hn, ln, un;
        decode4(__ldg(seq + b0 + k), hn, ln, un);
        h |= (hn & 1u) << k;
        l |= (ln & 1u) << k;
        u |= (un & 1u) << k;
      }
    }
    planes[w] = make_uint4(h, l, u, 0u);
  }
}

__global__ void pack_planes_kernel(const uint8_t* __restrict__ rows, int64_t n_rows, int64_t len,
                                   int64_t stride, uint4* __restrict__ planes, int64_t nwords) {
  const int64_t total = n_rows * len;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwords;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = 0u, l = 0u, b = 0u;
    int64_t idx = w * 32;
    int64_t r = idx / len;
    int64_t i = idx - r * len;
    for (int k = 0; k < 32 && idx + k < total; ++k) {
      uint32_t hn, ln, un;
      decode4(__ldg(rows + r * stride + i), hn, ln, un);
      h |= (hn & 1u) << k;
      l |= (ln & 1u) << k;
      b |= (un & 1u) << k;
      if (++i == len) {
        i = 0;
        ++r;
      }
    }
    planes[w] = make_uint4(h, l, b, 0u);
  }
}

int launch_pack_planes(const uint8_t* rows, int64_t n_rows, int64_t len, int64_t stride,
                       uint32_t* planes, cudaStream_t stream) {
  const int64_t total = n_rows * len;
  const int64_t nwords = (total + 31) / 32 + 1;  // + 1: the funnel shift's look-ahead word
  int64_t blocks = (nwords + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  count_launch();
  if ((n_rows == 1 || stride == len) && (reinterpret_cast<uintptr_t>(rows) & 15u) == 0)
    pack_planes_contig_kernel<<<(unsigned)blocks, 256, 0, stream>>>(
        rows, total, reinterpret_cast<uint4*>(planes), nwords);
  else
    pack_planes_kernel<<<(unsigned)blocks, 256, 0, stream>>>(rows, n_rows, len, stride,
                                                             reinterpret_cast<uint4*>(planes),
                                                             nwords);
  return 0;
}

// ---- gather v2 --------------------------------------------------------------
// CTA = 4 warps = 4 consecutive groups (128 pairs), lane = pair.  Every lane
// issues the loads of its whole window up front (NCH+1 16-byte plane blocks:
// bits [off, off+32*NCH) are funnel shifts of consecutive blocks), then per
// 32-position chunk transposes its two plane words with a 5-stage shuffle
// transpose (rotate + select per stage: SHFL + SHF + LOP3) into a small
// [positions][4 groups] staging tile that leaves as full 32-byte sectors
// (4 groups x 8 bytes per position, as gk_encode's output).  One barrier per
// CTA; 3 KB of shared memory at 100 bp, so many CTAs per SM keep enough random
// window loads in flight (round 1: one 1024-thread CTA per tile, two barriers
// per chunk and two dependent loads per chunk: 25% of HBM).
struct T32 {
  uint32_t keep[5], rot[5];
  __device__ __forceinline__ void init(int lane) {
    const uint32_t Z[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      const int s = 16 >> t;
      const bool up = (lane & s) != 0;
      keep[t] = up ? ~Z[t] : Z[t];
      rot[t] = up ? (uint32_t)(32 - s) : (uint32_t)s;
    }
  }
  // lane j holds bit i = element (j, i) -> lane i holds bit j = element (j, i)
  __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, 16 >> t);
      const uint32_t r = __funnelshift_l(y, y, rot[t]);
      x = (x & keep[t]) | (r & ~keep[t]);
    }
    return x;
  }
};

template <int NCH>
__global__ void __launch_bounds__(128) gather2_kernel(
    const uint4* __restrict__ planes, int64_t nbases, const int64_t* __restrict__ offsets,
    int64_t n, int len, uint32_t* __restrict__ packed, uint32_t* __restrict__ undef) {
  extern __shared__ uint2 stage2[];  // [len][4]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t g = (int64_t)blockIdx.x * 4 + warp;
  const int64_t p = g * 32 + lane;
  int64_t off = p < n ? offsets[p] : -1;
  const bool oob = p < n && (off < 0 || off + len > nbases);
  const bool live = p < n && !oob;
  if (!live) off = 0;
  const int nch = (len + 31) >> 5;
  const int64_t w0 = off >> 5;
  const uint32_t sh = (uint32_t)(off & 31);
  uint4 blk[NCH + 1];
#pragma unroll
  for (int c = 0; c <= NCH; ++c)
    blk[c] = (live && c <= nch) ? __ldg(planes + w0 + c) : make_uint4(0u, 0u, 0u, 0u);
  T32 tr;
  tr.init(lane);
  uint32_t anybad = 0u;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    if (c < nch) {
      const int nb = len - 32 * c < 32 ? len - 32 * c : 32;
      const uint32_t vm = nb == 32 ? 0xFFFFFFFFu : ((1u << nb) - 1u);
      const uint32_t xh = __funnelshift_r(blk[c].x, blk[c + 1].x, sh) & vm;
      const uint32_t xl = __funnelshift_r(blk[c].y, blk[c + 1].y, sh) & vm;
      anybad |= __funnelshift_r(blk[c].z, blk[c + 1].z, sh) & vm;
      const uint32_t yh = tr(xh), yl = tr(xl);
      if (lane < nb) stage2[(32 * c + lane) * 4 + warp] = make_uint2(yh, yl);
    }
  }
  const uint32_t u = __ballot_sync(0xFFFFFFFFu, anybad != 0u || oob);
  if (lane == 0) undef[g] = u;
  __syncthreads();
  // 4 groups x 8 bytes per position: one 32-byte sector each
  const int64_t tile = (g - warp) >> 5;
  const int gl0 = (int)((g - warp) & 31);
  uint2* dst = reinterpret_cast<uint2*>(packed);
  for (int t = threadIdx.x; t < 4 * len; t += 128)
    dst[(tile * len + (t >> 2)) * 32 + gl0 + (t & 3)] = stage2[t];
}

int launch_gather_windows(const uint32_t* planes, int64_t nbases, const int64_t* offsets, int64_t n,
                          int len, uint32_t* packed, uint32_t* undef, cudaStream_t stream) {
  const int64_t tiles = (n + 1023) / 1024;  // whole tiles (zero-filled tail)
  const int64_t ctas = tiles * 8;
  const size_t smem = (size_t)len * 4 * 8;
  const uint4* pl = reinterpret_cast<const uint4*>(planes);
  count_launch();
  if (len <= 128)
    gather2_kernel<4><<<(unsigned)ctas, 128, smem, stream>>>(pl, nbases, offsets, n, len, packed, undef);
  else if (len <= 256)
    gather2_kernel<8><<<(unsigned)ctas, 128, smem, stream>>>(pl, nbases, offsets, n, len, packed, undef);
  else
    gather2_kernel<16><<<(unsigned)ctas, 128, smem, stream>>>(pl, nbases, offsets, n, len, packed, undef);
  return 0;
}

}  // namespace gk
