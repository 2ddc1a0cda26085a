// gk_encode_core.cuh -- device functions of a1 (ASCII -> bit-sliced 2-bit planes),
// shared by gk_encode (encode_kernel) and the fused gk_filter_ascii kernel.
// See gk_encode.cu for the method notes.
#pragma once
#include "gk_common.cuh"

namespace gk {

// bit 2 of bytes 0..3 -> bits 28..31.  Partial products land on bit
// 28 + 8j - 7k (byte j, multiplier term k): == 28+k for j == k, >= 36 (dropped)
// for j > k, and on the distinct bits {7,14,15,21,22,23} for j < k: no carries.
__device__ __forceinline__ uint32_t gather_bit2(uint32_t r) { return (r & 0x04040404u) * 0x04081020u; }
// bit 1 of bytes 0..3 -> bits 28..31 (same argument, terms shifted by one).
__device__ __forceinline__ uint32_t gather_bit1(uint32_t r) { return (r & 0x02020202u) * 0x08102040u; }

// 0 iff all 4 bytes of w are in {A,C,G,T,a,c,g,t}.
__device__ __forceinline__ uint32_t invalid_bytes(uint32_t w) {
  uint32_t base = (w & 0x26262626u) | 0x41414141u;
  uint32_t tflag = (w >> 2) & ~(w >> 1) & 0x01010101u;
  return w ^ (base + 15u * tflag);
}

// 4 bytes of smem row starting at byte offset `off` (any alignment).
template <bool ALIGNED>
__device__ __forceinline__ uint32_t lds_u32(const uint8_t* sm, uint32_t off) {
  if (ALIGNED) return *reinterpret_cast<const uint32_t*>(sm + off);
  uint32_t a = off & ~3u;
  uint32_t lo = *reinterpret_cast<const uint32_t*>(sm + a);
  uint32_t hi = *reinterpret_cast<const uint32_t*>(sm + a + 4);
  return __funnelshift_r(lo, hi, (off & 3u) * 8u);
}

// Cooperative copy of bytes [src, src+nbytes) into smem so that global address
// a lands at sm[a - (src & ~15)]; 16-byte vector loads for the aligned middle.
__device__ __forceinline__ void stage_span(const uint8_t* src, int64_t nbytes, uint8_t* sm,
                                           int tid, int nthr) {
  uintptr_t a0 = reinterpret_cast<uintptr_t>(src);
  uintptr_t abase = a0 & ~uintptr_t(15);
  uintptr_t a1 = a0 + nbytes;
  uintptr_t m0 = (a0 + 15) & ~uintptr_t(15);
  uintptr_t m1 = a1 & ~uintptr_t(15);
  if (m0 > a1) m0 = a1;
  if (m1 < m0) m1 = m0;
  for (uintptr_t a = a0 + tid; a < m0; a += nthr)
    sm[a - abase] = *reinterpret_cast<const uint8_t*>(a);
  const int64_t nvec = (int64_t)((m1 - m0) >> 4);
  const uint4* gv = reinterpret_cast<const uint4*>(m0);
  uint4* sv = reinterpret_cast<uint4*>(sm + (m0 - abase));
  for (int64_t v = tid; v < nvec; v += nthr) sv[v] = __ldg(gv + v);
  for (uintptr_t a = m1 + tid; a < a1; a += nthr)
    sm[a - abase] = *reinterpret_cast<const uint8_t*>(a);
}

// Encode the 32 sequences of one group whose rows start in smem at
// sm + row0_off + s*stride (s = 0..31; rows >= nvalid are all-'A').
// Lane q handles base positions 4q..4q+3 (q = lane, lane+32, ...).
// emit(pos, hi_word, lo_word) is called for every position < len.
// Returns the group's undefined-sequence word (valid in all lanes).
template <bool ALIGNED, typename Emit>
__device__ __forceinline__ uint32_t encode_group(const uint8_t* sm, uint32_t row0_off,
                                                 uint32_t stride, int nvalid, int len,
                                                 Emit&& emit) {
  const int lane = threadIdx.x & 31;
  const int nquads = (len + 3) >> 2;
  uint32_t bad[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) bad[b] = 0u;

  for (int q = lane; q < nquads; q += 32) {
    uint32_t hb[4] = {0u, 0u, 0u, 0u}, lb[4] = {0u, 0u, 0u, 0u};
    const int rem = len - 4 * q;  // >= 1
    // byte mask of positions < len inside this quad
    const uint32_t posmask = rem >= 4 ? 0xFFFFFFFFu : (0xFFFFFFFFu >> (8 * (4 - rem)));
#pragma unroll
    for (int blk = 7; blk >= 0; --blk) {
      uint32_t w[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int s = 4 * blk + k;
        w[k] = s < nvalid ? lds_u32<ALIGNED>(sm, row0_off + (uint32_t)s * stride + 4u * q)
                          : 0x41414141u;
      }
      // validity of the 16 bytes (only positions < len)
      uint32_t e4[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) e4[k] = invalid_bytes(w[k]) & posmask;
      // byte transpose: r[m] byte k = w[k] byte m
      const uint32_t t0 = __byte_perm(w[0], w[1], 0x5140);
      const uint32_t t1 = __byte_perm(w[0], w[1], 0x7362);
      const uint32_t t2 = __byte_perm(w[2], w[3], 0x5140);
      const uint32_t t3 = __byte_perm(w[2], w[3], 0x7362);
      uint32_t r[4];
      r[0] = __byte_perm(t0, t2, 0x5410);
      r[1] = __byte_perm(t0, t2, 0x7632);
      r[2] = __byte_perm(t1, t3, 0x5410);
      r[3] = __byte_perm(t1, t3, 0x7632);
      // per-sequence error flags: fold the 4 positions of each row into byte k
      uint32_t ek = 0u;
#pragma unroll
      for (int k = 0; k < 4; ++k) ek |= (e4[k] != 0u ? 1u : 0u) << (8 * k);
      bad[blk] |= ek;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        hb[m] = __funnelshift_l(gather_bit2(r[m]), hb[m], 4);
        lb[m] = __funnelshift_l(gather_bit1(r[m]), lb[m], 4);
      }
    }
#pragma unroll
    for (int m = 0; m < 4; ++m)
      if (m < rem) emit(4 * q + m, hb[m], hb[m] ^ lb[m]);
  }
  uint32_t und = 0u;
#pragma unroll
  for (int blk = 0; blk < 8; ++blk) {
    const uint32_t b = __reduce_or_sync(0xFFFFFFFFu, bad[blk]);
#pragma unroll
    for (int k = 0; k < 4; ++k) und |= ((b >> (8 * k)) & 1u) << (4 * blk + k);
  }
  return und;
}


// ---------------------------------------------------------------------------
// Encoder v2 (TMA-staged): the 32 rows of a group sit in shared memory at
// buf + s*stride (buf 16-byte aligned); lane q encodes base positions
// 4q..4q+3 (q = lane + 32*it).  The smem address of every row at the lane's
// first column is computed once per kernel (32 registers), so each 4-byte
// word costs one LDS with an immediate offset (two LDS + one PRMT for rows
// whose start is not 4-byte aligned: their misalignment (s*stride) % 4 is a
// compile-time function of s and SM4 = stride % 4).
template <int SM4>
struct RowAddr {
  uint32_t a[32];
  __device__ __forceinline__ void init(uint32_t buf, uint32_t stride, int lane) {
#pragma unroll
    for (int s = 0; s < 32; ++s) a[s] = buf + (uint32_t)s * stride + 4u * lane - ((s * SM4) & 3);
  }
};

template <int SM4, int S, uint32_t OFF>
__device__ __forceinline__ uint32_t row_word(const RowAddr<SM4>& ra) {
  constexpr int d = (S * SM4) & 3;
  uint32_t lo;
  asm volatile("ld.shared.b32 %0, [%1+%2];" : "=r"(lo) : "r"(ra.a[S]), "n"(OFF));
  if constexpr (d == 0) {
    return lo;
  } else {
    uint32_t hi;
    asm volatile("ld.shared.b32 %0, [%1+%2];" : "=r"(hi) : "r"(ra.a[S]), "n"(OFF + 4));
    return __byte_perm(lo, hi, d == 1 ? 0x4321 : (d == 2 ? 0x5432 : 0x6543));
  }
}

// err | (w ^ canonical(w)): 0 in every byte of a valid base (see invalid_bytes).
__device__ __forceinline__ uint32_t acc_invalid(uint32_t bad, uint32_t w) {
  // m = canonical byte: 0x41 | (w & 0x26), +15 for T (b2 & ~b1); the two parts
  // have disjoint bits, so one IMAD (FMA pipe) and one LOP3 build it
  const uint32_t tflag = __umulhi(w, 1u << 30) & ~__umulhi(w, 1u << 31) & 0x01010101u;
  const uint32_t m = (tflag * 15u + 0x41414141u) | (w & 0x26262626u);
  return bad | (w ^ m);
}

template <int SM4, int BLK, bool LPART, uint32_t OFF>
__device__ __forceinline__ void encode_block(const RowAddr<SM4>& ra, const bool (&pm)[4],
                                             uint32_t& bad, uint32_t (&hb)[4],
                                             uint32_t (&lb)[4]) {
  const uint32_t w0 = row_word<SM4, 4 * BLK + 0, OFF>(ra);
  const uint32_t w1 = row_word<SM4, 4 * BLK + 1, OFF>(ra);
  const uint32_t w2 = row_word<SM4, 4 * BLK + 2, OFF>(ra);
  const uint32_t w3 = row_word<SM4, 4 * BLK + 3, OFF>(ra);
  const uint32_t t0 = __byte_perm(w0, w1, 0x5140);
  const uint32_t t1 = __byte_perm(w0, w1, 0x7362);
  const uint32_t t2 = __byte_perm(w2, w3, 0x5140);
  const uint32_t t3 = __byte_perm(w2, w3, 0x7362);
  uint32_t r[4];
  r[0] = __byte_perm(t0, t2, 0x5410);
  r[1] = __byte_perm(t0, t2, 0x7632);
  r[2] = __byte_perm(t1, t3, 0x5410);
  r[3] = __byte_perm(t1, t3, 0x7632);
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    uint32_t x = r[m];
    if (LPART) x = pm[m] ? x : 0x41414141u;  // positions >= len of the last quad
    bad = acc_invalid(bad, x);
    hb[m] = __funnelshift_l(gather_bit2(x), hb[m], 4);          // ALU pipe
    lb[m] = lb[m] * 16u + __umulhi(gather_bit1(x), 16u);        // FMA pipe
  }
}

template <int SM4, bool LPART, uint32_t OFF, typename Emit>
__device__ __forceinline__ void encode_quad(const RowAddr<SM4>& ra, int q, int rem,
                                            uint32_t (&bad)[8], Emit&& emit) {
  bool pm[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) pm[m] = m < rem;
  uint32_t hb[4] = {0u, 0u, 0u, 0u}, lb[4] = {0u, 0u, 0u, 0u};
  encode_block<SM4, 7, LPART, OFF>(ra, pm, bad[7], hb, lb);
  encode_block<SM4, 6, LPART, OFF>(ra, pm, bad[6], hb, lb);
  encode_block<SM4, 5, LPART, OFF>(ra, pm, bad[5], hb, lb);
  encode_block<SM4, 4, LPART, OFF>(ra, pm, bad[4], hb, lb);
  encode_block<SM4, 3, LPART, OFF>(ra, pm, bad[3], hb, lb);
  encode_block<SM4, 2, LPART, OFF>(ra, pm, bad[2], hb, lb);
  encode_block<SM4, 1, LPART, OFF>(ra, pm, bad[1], hb, lb);
  encode_block<SM4, 0, LPART, OFF>(ra, pm, bad[0], hb, lb);
#pragma unroll
  for (int m = 0; m < 4; ++m)
    if (m < rem) emit(q, m, hb[m], hb[m] ^ lb[m]);  // paper code: high = b2, low = b1^b2
}

// Sparse last quad iteration (NIT >= 2, R <= 16 quads left, e.g. 6 at 150 bp):
// instead of R lanes doing whole quads while 32-R idle, P lanes share a quad,
// each encoding 32/P of its rows (P = 2, 4, 8); the P partial words of a
// position are OR-combined with shuffles.  Rows are addressed at run time
// (row p*32/P + r of the lane's part), any alignment (two LDS + funnel shift).
// Returns the lane's undefined rows as a row bit mask (bit s = row s).
template <int SM4, int P, bool LPART, uint32_t OFF, typename Emit>
__device__ __forceinline__ uint32_t encode_tail(const RowAddr<SM4>& ra, int q0, int R, int len,
                                                uint32_t& anybad, Emit&& emit) {
  constexpr int RP = 32 / P;  // rows per part
  constexpr int NB = RP / 4;  // 4-row blocks per part
  const int lane = threadIdx.x & 31;
  const int qi = lane / P, part = lane % P;
  const int q = q0 + qi;
  const bool valid = qi < R;
  const uint32_t buf = ra.a[0] - 4u * (uint32_t)lane;
  const uint32_t stride = ra.a[1] - ra.a[0] + (uint32_t)(SM4 & 3);
  const int rem = len - 4 * q;
  bool pm[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) pm[m] = m < rem;
  uint32_t hb[4] = {0u, 0u, 0u, 0u}, lb[4] = {0u, 0u, 0u, 0u}, badj[NB];
#pragma unroll
  for (int j = NB - 1; j >= 0; --j) {
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t srow = (uint32_t)(part * RP + 4 * j + k);
      const uint32_t a = buf + OFF + srow * stride + 4u * (uint32_t)(valid ? q : q0);
      uint32_t lo, hi;
      asm volatile("ld.shared.b32 %0, [%1];" : "=r"(lo) : "r"(a & ~3u));
      asm volatile("ld.shared.b32 %0, [%1];" : "=r"(hi) : "r"((a & ~3u) + 4u));
      w[k] = __funnelshift_r(lo, hi, (a & 3u) * 8u);
    }
    const uint32_t t0 = __byte_perm(w[0], w[1], 0x5140);
    const uint32_t t1 = __byte_perm(w[0], w[1], 0x7362);
    const uint32_t t2 = __byte_perm(w[2], w[3], 0x5140);
    const uint32_t t3 = __byte_perm(w[2], w[3], 0x7362);
    uint32_t r[4];
    r[0] = __byte_perm(t0, t2, 0x5410);
    r[1] = __byte_perm(t0, t2, 0x7632);
    r[2] = __byte_perm(t1, t3, 0x5410);
    r[3] = __byte_perm(t1, t3, 0x7632);
    uint32_t bad = 0u;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      uint32_t x = r[m];
      if (LPART) x = pm[m] ? x : 0x41414141u;
      bad = acc_invalid(bad, x);
      hb[m] = __funnelshift_l(gather_bit2(x), hb[m], 4);
      lb[m] = lb[m] * 16u + __umulhi(gather_bit1(x), 16u);
    }
    badj[j] = valid ? bad : 0u;
  }
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    uint32_t h = hb[m] << (part * RP), l = lb[m] << (part * RP);
#pragma unroll
    for (int d = 1; d < P; d <<= 1) {
      h |= __shfl_xor_sync(0xFFFFFFFFu, h, d);
      l |= __shfl_xor_sync(0xFFFFFFFFu, l, d);
    }
    if (valid && part == 0 && m < rem) emit(q, m, h, h ^ l);
  }
  uint32_t rows = 0u;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    anybad |= badj[j];
    const uint32_t b = badj[j];
    const uint32_t nz = ((b & 0x7F7F7F7Fu) + 0x7F7F7F7Fu | b) & 0x80808080u;
    const uint32_t nib = (nz >> 7 & 1u) | (nz >> 14 & 2u) | (nz >> 21 & 4u) | (nz >> 28 & 8u);
    rows |= nib << (part * RP + 4 * j);
  }
  return rows;
}

// Encode all quads of the lane for the staged group at buffer offset BOFF
// (compile-time, like the quad offsets: the 32 row addresses stay in registers
// and every LDS uses an immediate offset).
// emit(q, m, hi_plane, lo_plane) for every position 4q+m < len.
template <int SM4, bool LPART, int NIT, uint32_t BOFF, typename Emit>
__device__ __forceinline__ uint32_t encode_group_v2(const RowAddr<SM4>& ra, int len,
                                                    Emit&& emit) {
  const int lane = threadIdx.x & 31;
  const int nquads = (len + 3) >> 2;
  uint32_t bad[8];
#pragma unroll
  for (int b = 0; b < 8; ++b) bad[b] = 0u;
  uint32_t tail_rows = 0u, tail_any = 0u;
#pragma unroll
  for (int it = 0; it < NIT; ++it) {
    const int q = lane + 32 * it;
    const int R = nquads - 32 * it;  // quads left for this iteration (warp-uniform)
    if (NIT >= 2 && it == NIT - 1 && R <= 16) {
      constexpr uint32_t TOFF = BOFF;
      if (R <= 0) {
      } else if (R <= 4) {
        tail_rows = encode_tail<SM4, 8, LPART, TOFF>(ra, 32 * it, R, len, tail_any, emit);
      } else if (R <= 8) {
        tail_rows = encode_tail<SM4, 4, LPART, TOFF>(ra, 32 * it, R, len, tail_any, emit);
      } else {
        tail_rows = encode_tail<SM4, 2, LPART, TOFF>(ra, 32 * it, R, len, tail_any, emit);
      }
      continue;
    }
    if (q < nquads) {
      const int rem = len - 4 * q;
      if (it == 0) encode_quad<SM4, LPART, BOFF>(ra, q, rem, bad, emit);
      else if (it == 1) encode_quad<SM4, LPART, BOFF + 128u>(ra, q, rem, bad, emit);
      else if (it == 2) encode_quad<SM4, LPART, BOFF + 256u>(ra, q, rem, bad, emit);
      else encode_quad<SM4, LPART, BOFF + 384u>(ra, q, rem, bad, emit);
    }
  }
  // undefined bases are rare (0.3% of pairs in the paper's Set_3, Table S.1
  // :509): one warp-wide OR decides whether the per-row flags are needed at all
  {
    uint32_t any = tail_any;
#pragma unroll
    for (int blk = 0; blk < 8; ++blk) any |= bad[blk];
    if (__reduce_or_sync(0xFFFFFFFFu, any) == 0u) return 0u;
  }
  uint32_t und = __reduce_or_sync(0xFFFFFFFFu, tail_rows);
#pragma unroll
  for (int blk = 0; blk < 8; ++blk) {
    const uint32_t b = __reduce_or_sync(0xFFFFFFFFu, bad[blk]);
    // byte k != 0 -> bit 4*blk+k
    const uint32_t nz = ((b & 0x7F7F7F7Fu) + 0x7F7F7F7Fu | b) & 0x80808080u;
    und |= ((nz >> 7) & 1u) << (4 * blk) | ((nz >> 15) & 1u) << (4 * blk + 1) |
           ((nz >> 23) & 1u) << (4 * blk + 2) | ((nz >> 31) & 1u) << (4 * blk + 3);
  }
  return und;
}

}  // namespace gk
