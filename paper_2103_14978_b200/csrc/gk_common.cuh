// gk_common.cuh -- shared device helpers of the B200 GateKeeper-GPU library.
//
// Bit-sliced representation: one 32-bit word
// holds ONE base position of 32 pairs (bit j = pair j of a group).  Every mask
// operation of the method is then a plain bitwise op on whole
// words: the XOR/OR mismatch of 32 pairs is 2 LOP3, the amendment of 32 pairs
// at one position is 3 LOP3 over the neighbouring positions' words, and a shift
// of the read by k bases is a change of word index (no funnel shifts, no carry
// bits -- the "carry-bit transfers" of PAPER.md:107 disappear).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define GK_WARP 32
#define GK_TILE_SEQS 1024
#define GK_MAXLEN 508

namespace gk {

// Word index of (tile, base position, lane, plane) in a packed set of length len.
__host__ __device__ __forceinline__ int64_t packed_index(int64_t tile, int len, int pos, int lane,
                                                         int plane) {
  return ((tile * len + pos) * GK_WARP + lane) * 2 + plane;
}

// Mismatch word of 32 pairs at one position: a base differs iff either bit of
// its 2-bit code differs (XOR, then OR of the two bits).
__host__ __device__ __forceinline__ uint32_t mismatch(uint32_t rh, uint32_t rl, uint32_t qh, uint32_t ql) {
  return (rh ^ qh) | (rl ^ ql);
}

// Amended value at position i from the raw mask words at i-2..i+2 (0 outside
// [0, len) and at vacated positions).  A 0 at i becomes 1 iff it lies in a
// maximal 0-run of length 1 or 2 bounded by 1s on both sides (reading R3):
//   run {i}      : x[i-1] & x[i+1]
//   run {i,i+1}  : x[i-1] & x[i+2]      (x[i+1] == 0 then)
//   run {i-1,i}  : x[i-2] & x[i+1]      (x[i-1] == 0 then)
__host__ __device__ __forceinline__ uint32_t amend(uint32_t xm2, uint32_t xm1, uint32_t x0, uint32_t xp1,
                                          uint32_t xp2) {
  return x0 | (xm1 & (xp1 | xp2)) | (xm2 & xp1);
}

// Bit-sliced 8-bit counter: c[b] bit j = bit b of pair j's count.
struct Counter8 {
  uint32_t c[8];
  __device__ __forceinline__ void clear() {
#pragma unroll
    for (int b = 0; b < 8; ++b) c[b] = 0u;
  }
  // add a 0/1 word (ripple through all planes)
  __device__ __forceinline__ void add1(uint32_t s) {
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      uint32_t t = c[b] & s;
      c[b] ^= s;
      s = t;
    }
  }
  // add a 2-bit word pair (w1:w0), values 0..3
  __device__ __forceinline__ void add2(uint32_t w0, uint32_t w1) {
    uint32_t carry = c[0] & w0;
    c[0] ^= w0;
    uint32_t s1 = c[1] ^ w1 ^ carry;
    carry = (c[1] & w1) | (c[1] & carry) | (w1 & carry);
    c[1] = s1;
#pragma unroll
    for (int b = 2; b < 8; ++b) {
      uint32_t t = c[b] & carry;
      c[b] ^= carry;
      carry = t;
    }
  }
};

// Bit mask of the pairs whose counter value is <= e (bit-sliced compare).
__host__ __device__ __forceinline__ uint32_t le_const(const uint32_t (&c)[8], int e) {
  if (e >= 255) return 0xFFFFFFFFu;
  uint32_t gt = 0u, eq = 0xFFFFFFFFu;
#pragma unroll
  for (int b = 7; b >= 0; --b) {
    if ((e >> b) & 1) {
      eq &= c[b];
    } else {
      gt |= eq & c[b];
      eq &= ~c[b];
    }
  }
  return ~gt;
}

// Spread a 4-bit nibble to bit 0 of four bytes (byte k <- bit k).  The four
// partial products nib_k * 2^(7m) land on bit k+7m; they are pairwise distinct,
// so no carries, and bit 8k is reached only by m = k.
__host__ __device__ __forceinline__ uint32_t nibble_to_bytes(uint32_t nib) {
  return (nib * 0x00204081u) & 0x01010101u;
}

// Bytes of pairs 4w..4w+3 from 8 count planes.
__host__ __device__ __forceinline__ uint32_t count_bytes(const uint32_t (&c)[8], int w) {
  uint32_t out = 0u;
#pragma unroll
  for (int b = 0; b < 8; ++b) out |= nibble_to_bytes((c[b] >> (4 * w)) & 0xFu) << b;
  return out;
}

}  // namespace gk
