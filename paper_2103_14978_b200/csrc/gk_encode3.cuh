// gk_encode3.cuh -- a1 (ASCII -> bit-sliced 2-bit planes) at a few instructions per
// byte: the group's 32 rows are staged in shared memory (one TMA bulk copy);
// every lane extracts the code bits of 4 rows x 4 bytes per 16-position chunk
// into one 32-bit word and a 3-stage shuffle transpose turns the 32 lanes' words
// into 32 "position x plane" words of the packed layout (bit j = row j).
//
// Per 4 bytes w of a row (SWAR, branch-free):
//  * code planes (A=00 C=01 G=10 T=11): for A C G T a c g t the
//    ASCII bit 2 is the high code bit and bit 1 ^ bit 2 the low one; bit 3 is 0,
//    so x = (w ^ (w >> 1)) & 0x06 per byte holds low at bit 1, high at bit 2.
//  * validity (reading R8): a byte is one of the 8 letters iff
//      bits 7,6,3 = 0,1,0        -> (w ^ 0x40) & 0xC8 == 0
//      b4 == b2 & ~b1, b0 != b4  -> bit 4 of  (w ^ (w<<2 & ~(w<<3))) | ~(w ^ w<<4)  == 0
//    (the 8 solutions are exactly 0x41 43 47 54 61 63 67 74).  Both tests are
//    ORed into per-row accumulators unmasked (OR commutes with the final mask).
//  The shifts left are IMADs (FMA pipe), the rest one LOP3 each (ALU pipe).
//
// Lane layout.  Lane l = cw + 4*rh (cw = 0..3: the lane's 4-byte column of the
// 16-byte chunk; rh = 0..7) holds rows r_i = rh0 + 2i + 8 rh1 + 16 rh2 (i = 0..3):
// rows spaced by 2, so that the transpose ends with bit r = row r (below).  The
// lane's merged word has bit t = b' + 2i + 8k for byte k (position 4cw+k) of row
// i, plane b' (0: low, 1: high).  A 32x32 transpose would take 5 shuffle stages;
// the load pattern already performed two of them (lane bits 0-1 = the column
// block), and 3 stages swap lane bits 2,3,4 with bit-index bits 0,3,4:
// afterwards lane l = cw + 4b' + 8k holds one position x plane word whose bit
// t = rh0 + 2i + 8rh1 + 16rh2 = r is row r.  Each stage is SHFL + SHF (rotate)
// + LOP3 (select).
#pragma once
#include "gk_common.cuh"
#include "gk_tma.cuh"

namespace gk {
namespace enc3 {

// FMA-pipe shifts (ptxas keeps mul.lo by a register as IMAD)
__device__ __forceinline__ uint32_t imul(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t imadhi(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t lop3_or(uint32_t a, uint32_t b, uint32_t c) {
  return a | b | c;
}

// Per-lane constants.
struct Lane {
  uint32_t m2, m4, m8, m16, m32, mh;  // multipliers in registers (keep them IMADs)
  uint32_t keep[3];                   // select masks of the 3 transpose stages
  uint32_t rot[3];                    // rotate amounts
  int rows[4];                        // r_i
  int cw;
  uint32_t lofix;                     // ~0 on the lanes that hold a low-plane word (b' = 0)
  __device__ __forceinline__ void init(int lane) {
    m2 = 2u; m4 = 4u; m8 = 8u; m16 = 16u; m32 = 32u; mh = 0x80000000u;
    cw = lane & 3;
    lofix = ((lane >> 2) & 1) ? 0u : 0xFFFFFFFFu;
    const int rh0 = (lane >> 2) & 1, rh1 = (lane >> 3) & 1, rh2 = (lane >> 4) & 1;
#pragma unroll
    for (int i = 0; i < 4; ++i) rows[i] = rh0 + 2 * i + 8 * rh1 + 16 * rh2;
    // stage s swaps lane bit LB[s] with bit-index bit TB[s]
    const int LB[3] = {2, 3, 4}, TB[3] = {0, 3, 4};
    const uint32_t Z[3] = {0x55555555u, 0x00FF00FFu, 0x0000FFFFu};  // bit-index bit TB = 0
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const bool up = (lane >> LB[s]) & 1;
      keep[s] = up ? ~Z[s] : Z[s];
      rot[s] = up ? 32u - (1u << TB[s]) : (1u << TB[s]);
    }
  }
};

// 32x32 transpose tail: 3 stages (lane bits 2,3,4 <-> bit-index bits 0,3,4).
__device__ __forceinline__ uint32_t transpose3(uint32_t m, const Lane& ln) {
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, m, 4 << s);
    const uint32_t r = __funnelshift_l(y, y, ln.rot[s]);
    m = (m & ln.keep[s]) | (r & ~ln.keep[s]);
  }
  return m;
}

// One row's 4 bytes: validity accumulators and the plane bits (low at bit 1,
// high at bit 2 of every byte).
__device__ __forceinline__ uint32_t row_word(uint32_t w, const Lane& ln, uint32_t& acc_g,
                                             uint32_t& acc_y) {
  const uint32_t s2 = imul(w, ln.m4), s3 = imul(w, ln.m8), s4 = imul(w, ln.m16);
  const uint32_t h = w ^ (s2 & ~s3);
  const uint32_t g = h | ~(w ^ s4);
  acc_g |= g;
  acc_y |= w ^ 0x40404040u;
  const uint32_t sh = imadhi(w, ln.mh, 0u);  // w >> 1 on the FMA pipe
  return (w ^ sh) & 0x06060606u;
}

// Merge the 4 rows' plane bits: bit t = b' + 2i + 8k.
__device__ __forceinline__ uint32_t merge4(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3,
                                           const Lane& ln) {
  uint32_t m = imadhi(x0, ln.mh, 0u);  // >> 1
  m = imad(x1, ln.m2, m);              // << 1
  m = imad(x2, ln.m8, m);              // << 3
  m = imad(x3, ln.m32, m);             // << 5
  return m;
}

// Row flags of the lane -> the group's undefined word (bit r = row r).
__device__ __forceinline__ uint32_t group_undef(const uint32_t (&ag)[4], const uint32_t (&ay)[4],
                                                const Lane& ln) {
  uint32_t u = 0u;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool bad = ((ag[i] & 0x10101010u) | (ay[i] & 0xC8C8C8C8u)) != 0u;
    u |= bad ? (1u << ln.rows[i]) : 0u;
  }
  return __reduce_or_sync(0xFFFFFFFFu, u);
}

// GK_ENC3_RAW = 1: merge the RAW ASCII bits 1 and 2 of the 4 rows (bit-field
// selects, no per-row code arithmetic) and form the low plane b1 ^ b2 AFTER the
// transpose: the transpose is a bit permutation, so XOR commutes with it, and
// lane l (b' = 0, raw b1) XORs the word of lane l ^ 4 (b' = 1, raw b2 = the high
// plane).  Per 16 positions: 4 fewer ALU shifts + 4 fewer LOP3 for 1 SHFL + 1 LOP3.
// Validity as row_word; `s3` = w << 3 is passed in (row 2 shares it with the merge).
__device__ __forceinline__ void row_valid(uint32_t w, uint32_t s3, const Lane& ln, uint32_t& acc_g,
                                          uint32_t& acc_y) {
  const uint32_t s2 = imul(w, ln.m4), s4 = imul(w, ln.m16);
  const uint32_t h = w ^ (s2 & ~s3);
  acc_g |= h | ~(w ^ s4);
  acc_y |= w ^ 0x40404040u;
}

// bit b' + 2i + 8k = ASCII bit (1 + b') of row i, byte k; also the validity of the rows
__device__ __forceinline__ uint32_t merge4_raw(const uint32_t (&w)[4], const Lane& ln,
                                               uint32_t (&ag)[4], uint32_t (&ay)[4]) {
  const uint32_t a = w[0] >> 1;
  const uint32_t b = imul(w[1], ln.m2);   // << 1
  const uint32_t c = imul(w[2], ln.m8);   // << 3
  const uint32_t d = imul(w[3], ln.m32);  // << 5
  row_valid(w[0], imul(w[0], ln.m8), ln, ag[0], ay[0]);
  row_valid(w[1], imul(w[1], ln.m8), ln, ag[1], ay[1]);
  row_valid(w[2], c, ln, ag[2], ay[2]);
  row_valid(w[3], imul(w[3], ln.m8), ln, ag[3], ay[3]);
  uint32_t m = (a & 0x03030303u) | (b & ~0x03030303u);
  m = (m & 0x0F0F0F0Fu) | (c & ~0x0F0F0F0Fu);
  return (m & 0x3F3F3F3Fu) | (d & ~0x3F3F3F3Fu);
}

// after transpose3 of a raw merged word: low plane = b1 ^ b2
__device__ __forceinline__ uint32_t low_fix(uint32_t m, const Lane& ln) {
  const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, m, 4);
  return m ^ (y & ln.lofix);
}

}  // namespace enc3

#ifndef GK_ENC3_RAW
#define GK_ENC3_RAW 1
#endif

// ---- group encoder of encode3_kernel (gk_encode.cu): outputs collected per
// block of 4 groups in shared memory, [plane][position * 5 + group]
template <bool ALN>
__device__ __forceinline__ void enc3_chunk(const uint8_t* buf, const uint32_t (&roff)[4],
                                           const uint32_t (&rsh)[4], int c, int len,
                                           const enc3::Lane& ln, uint32_t (&ag)[4],
                                           uint32_t (&ay)[4], uint32_t* outs, uint32_t P,
                                           int wg, bool tail) {
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
    if (tail) {  // bytes of positions >= len read as 'A' (valid, never stored)
      const int rem = len - 16 * c - 4 * ln.cw;
      const uint32_t bm =
          rem >= 4 ? 0xFFFFFFFFu : (rem <= 0 ? 0u : (0xFFFFFFFFu >> (32 - 8 * rem)));
      w = (w & bm) | (0x41414141u & ~bm);
    }
    if (GK_ENC3_RAW) x[i] = w;
    else x[i] = enc3::row_word(w, ln, ag[i], ay[i]);
  }
  uint32_t m = GK_ENC3_RAW ? enc3::merge4_raw(x, ln, ag, ay)
                           : enc3::merge4(x[0], x[1], x[2], x[3], ln);
  m = enc3::transpose3(m, ln);
  if (GK_ENC3_RAW) m = enc3::low_fix(m, ln);
  // lane = cw + 4b' + 8k: position 16c + 4cw + k, plane b' (0 = low -> paper plane 1)
  const int lane = threadIdx.x & 31;
  const int pos = 16 * c + 4 * (lane & 3) + (lane >> 3);
  const int plane = ((lane >> 2) & 1) ? 0 : 1;
  if (!tail || pos < len) outs[plane * P + pos * 5 + wg] = m;
}

// stride = 2 (mod 4): the rows of a lane all start at the same 2-byte offset
// (its rows have one parity), so every lane loads ONE aligned word per row (not
// two + a funnel shift: half the shared-memory loads) and a lane whose rows start
// 2 bytes into a word realigns its MERGED word instead: in the merged layout
// (bit = b' + 2i + 8k) a 2-position shift is a 16-bit funnel shift with the
// merged word of the next column (lane + 1, or for column 3 lane - 3 of the next
// chunk) -- one SHFL + one SHF per 16 positions.  Chunks are therefore emitted
// one step late, with one extra load chunk at the end.
__device__ __forceinline__ uint32_t enc3_merge_m2(const uint8_t* buf, const uint32_t (&roff)[4],
                                                  int s2, int c, int len, const enc3::Lane& ln,
                                                  uint32_t (&ag)[4], uint32_t (&ay)[4],
                                                  bool first, bool tail) {
  uint32_t x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t w = *reinterpret_cast<const uint32_t*>(buf + roff[i] + 16 * c);
    uint32_t bm = 0xFFFFFFFFu;
    if (first && s2 && ln.cw == 0) bm = 0xFFFF0000u;  // the 2 bytes before the row start
    if (tail) {
      const int rem = len - (16 * c + 4 * ln.cw - s2);  // bytes of positions < len
      bm &= rem >= 4 ? 0xFFFFFFFFu : (rem <= 0 ? 0u : (0xFFFFFFFFu >> (32 - 8 * rem)));
    }
    if (first || tail) w = (w & bm) | (0x41414141u & ~bm);
    if (GK_ENC3_RAW) x[i] = w;
    else x[i] = enc3::row_word(w, ln, ag[i], ay[i]);
  }
  if (GK_ENC3_RAW) return enc3::merge4_raw(x, ln, ag, ay);
  return enc3::merge4(x[0], x[1], x[2], x[3], ln);
}

__device__ __forceinline__ void enc3_emit(uint32_t m, int c, int len, const enc3::Lane& ln,
                                          uint32_t* outs, uint32_t P, int wg) {
  m = enc3::transpose3(m, ln);
  if (GK_ENC3_RAW) m = enc3::low_fix(m, ln);
  const int lane = threadIdx.x & 31;
  const int pos = 16 * c + 4 * (lane & 3) + (lane >> 3);
  const int plane = ((lane >> 2) & 1) ? 0 : 1;
  if (pos < len) outs[plane * P + pos * 5 + wg] = m;
}


// One group's staged span (32 rows at roff / rsh, MODE as encode3_kernel) ->
// outs[plane * P + pos * 5 + wg] for every position; returns the group's
// undefined word (bit r = row r).
template <int NCH, int MODE>
__device__ __forceinline__ uint32_t enc3_group(const uint8_t* sbuf, const uint32_t (&roff)[4],
                                               const uint32_t (&rsh)[4], int s2, int len,
                                               const enc3::Lane& ln, uint32_t* outs, uint32_t P,
                                               int wg) {
  const int lane = threadIdx.x & 31;
  const int nch = NCH > 0 ? NCH : (len + 15) >> 4;
  uint32_t ag[4] = {0u, 0u, 0u, 0u}, ay[4] = {0u, 0u, 0u, 0u};
  if constexpr (MODE == 2) {
    const int cw = ln.cw;
    const int src = cw == 3 ? lane - 3 : lane + 1;
    uint32_t prev = enc3_merge_m2(sbuf, roff, s2, 0, len, ln, ag, ay, true, nch <= 1);
#pragma unroll (NCH > 0 ? NCH : 1)
    for (int c = 1; c <= nch; ++c) {
      const uint32_t cur = enc3_merge_m2(sbuf, roff, s2, c, len, ln, ag, ay, false, c >= nch - 1);
      const uint32_t nxt = __shfl_sync(0xFFFFFFFFu, cw == 0 ? cur : prev, src);
      enc3_emit(__funnelshift_r(prev, nxt, (uint32_t)(8 * s2)), c - 1, len, ln, outs, P, wg);
      prev = cur;
    }
  } else {
    constexpr bool ALN = MODE == 0;
    if (NCH > 0) {
#pragma unroll
      for (int c = 0; c < (NCH > 1 ? NCH - 1 : 0); ++c)
        enc3_chunk<ALN>(sbuf, roff, rsh, c, len, ln, ag, ay, outs, P, wg, false);
    } else {
#pragma unroll 1
      for (int c = 0; c < nch - 1; ++c)
        enc3_chunk<ALN>(sbuf, roff, rsh, c, len, ln, ag, ay, outs, P, wg, false);
    }
    enc3_chunk<ALN>(sbuf, roff, rsh, nch - 1, len, ln, ag, ay, outs, P, wg, true);
  }
  return enc3::group_undef(ag, ay, ln);
}
}  // namespace gk
