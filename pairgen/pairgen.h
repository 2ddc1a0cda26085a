/* pairgen.h -- seeded synthetic (read, candidate reference segment) pairs.
 *
 * TEST / BENCH INFRASTRUCTURE.  This module holds NO arithmetic of the
 * GateKeeper-GPU method (no encoding, no masks, no counting): it only draws
 * ASCII sequences.  It is the one piece of code that both the CPU oracle side
 * (host build, gcc) and the CUDA side (device build, nvcc) may use, so that both
 * see byte-identical inputs (task rule: "only the seeded input generators serve
 * both, from a module of their own").
 *
 * Recipe (calibrated from SURVEY.md 8(d) and the
 * paper's dataset description, PAPER.md:176 and Table S.1 :502-524):
 *   per pair idx: a counter-based stream s = seed ^ (idx * 0x9E3779B97F4A7C15),
 *   advanced with splitmix64; draws happen in the fixed order written below.
 *   1. src = SRC_LEN(L) uniform random bases; ref = src[0:L].
 *   2. class draw u in [0,1000):
 *        paper    profile: near (u<55): m ~ U{0..ceil(.1L)};
 *                          mid (u<655): m ~ U{ceil(.1L)+1..ceil(.4L)};
 *                          far (else) : read = fresh uniform bases sharing one
 *                                       16-base seed with ref at the same offset.
 *        balanced profile: far (u<50), else m ~ U{0..min(2*emax, ceil(.4L))}.
 *      read = src after m edits (sub 60% / ins 20% / del 20%, positions
 *      uniform in [0,L)), truncated to L: deletions pull in downstream bases.
 *   3. modifiers (draw v in [0,1000)):
 *        paper   : v<3  -> one 'N' at a random position of read or ref
 *                  (Set_3 has 92,414 undefined pairs of 30M = 0.31%, :509).
 *        balanced: v<10 -> one 'N'; v<20 -> one IUPAC code; v<70 -> random
 *                  per-base lower case on read and/or ref.
 *   Bytes stride[L..stride) of every row are set to '\n' (never read by the filter).
 */
#ifndef PAIRGEN_H
#define PAIRGEN_H

#include <stdint.h>

#if defined(__CUDACC__)
#define PG_HD __host__ __device__ __forceinline__
#else
#define PG_HD static inline
#endif

#define PG_SEED_DEFAULT 2103149780ULL
#define PG_PROFILE_PAPER 0
#define PG_PROFILE_BALANCED 1
#define PG_MAX_LEN 508
#define PG_BUF 1200

PG_HD uint64_t pg_next(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* uniform integer in [0, n), n < 2^32 */
PG_HD uint32_t pg_below(uint64_t* s, uint32_t n) {
  return (uint32_t)(((pg_next(s) >> 32) * (uint64_t)n) >> 32);
}

PG_HD int pg_src_len(int L) { return L + (2 * L + 4) / 5 + 16; }
PG_HD int pg_ceil_tenth(int L) { return (L + 9) / 10; }
PG_HD int pg_ceil_twofifth(int L) { return (2 * L + 4) / 5; }

PG_HD uint8_t pg_base(uint32_t c) {
  return (uint8_t)(c == 0 ? 'A' : c == 1 ? 'C' : c == 2 ? 'G' : 'T');
}

/* Writes read[0..L) and ref[0..L).  buf must hold PG_BUF bytes (scratch). */
PG_HD void pg_gen_pair(uint64_t seed, uint64_t idx, int L, int profile, int emax,
                       uint8_t* read, uint8_t* ref, uint8_t* buf) {
  uint64_t s = seed ^ (idx * 0x9E3779B97F4A7C15ULL);
  int srclen = pg_src_len(L);
  for (int i = 0; i < srclen; ++i) buf[i] = pg_base(pg_below(&s, 4));
  for (int i = 0; i < L; ++i) ref[i] = buf[i];

  uint32_t u = pg_below(&s, 1000);
  int far = 0, m = 0;
  int mmax = pg_ceil_twofifth(L);
  if (profile == PG_PROFILE_PAPER) {
    if (u < 55) {
      m = (int)pg_below(&s, (uint32_t)pg_ceil_tenth(L) + 1);
    } else if (u < 655) {
      int lo = pg_ceil_tenth(L) + 1;
      int hi = mmax;
      if (hi < lo) hi = lo;
      m = lo + (int)pg_below(&s, (uint32_t)(hi - lo + 1));
    } else {
      far = 1;
    }
  } else {
    if (u < 50) {
      far = 1;
    } else {
      int hi = 2 * emax;
      if (hi > mmax) hi = mmax;
      if (hi < 0) hi = 0;
      m = (int)pg_below(&s, (uint32_t)hi + 1);
    }
  }

  if (far) {
    for (int i = 0; i < L; ++i) read[i] = pg_base(pg_below(&s, 4));
    int seedlen = L < 16 ? L : 16;
    int off = (int)pg_below(&s, (uint32_t)(L - seedlen + 1));
    for (int i = 0; i < seedlen; ++i) read[off + i] = ref[off + i];
  } else {
    int len = srclen;
    for (int t = 0; t < m; ++t) {
      uint32_t kind = pg_below(&s, 10);   /* 0..5 sub, 6..7 ins, 8..9 del */
      int p = (int)pg_below(&s, (uint32_t)L);
      if (kind < 6) {
        uint8_t old = buf[p];
        uint32_t oc = old == 'A' ? 0 : old == 'C' ? 1 : old == 'G' ? 2 : 3;
        buf[p] = pg_base((oc + 1 + pg_below(&s, 3)) & 3);
      } else if (kind < 8) {
        uint8_t nb = pg_base(pg_below(&s, 4));
        if (len < PG_BUF) len++;
        for (int i = len - 1; i > p; --i) buf[i] = buf[i - 1];
        buf[p] = nb;
      } else {
        for (int i = p; i < len - 1; ++i) buf[i] = buf[i + 1];
        len--;
      }
    }
    for (int i = 0; i < L; ++i) read[i] = buf[i];
  }

  uint32_t v = pg_below(&s, 1000);
  if (profile == PG_PROFILE_PAPER) {
    if (v < 3) {
      uint8_t* t = pg_below(&s, 2) ? ref : read;
      t[pg_below(&s, (uint32_t)L)] = 'N';
    }
  } else {
    if (v < 10) {
      uint8_t* t = pg_below(&s, 2) ? ref : read;
      t[pg_below(&s, (uint32_t)L)] = 'N';
    } else if (v < 20) {
      const char iupac[10] = {'R', 'Y', 'K', 'M', 'S', 'W', 'B', 'D', 'H', 'V'};
      uint8_t* t = pg_below(&s, 2) ? ref : read;
      int p = (int)pg_below(&s, (uint32_t)L);
      t[p] = (uint8_t)iupac[pg_below(&s, 10)];
    } else if (v < 70) {
      uint32_t which = pg_below(&s, 3); /* 0 read, 1 ref, 2 both */
      for (int i = 0; i < L; ++i) {
        uint32_t r = pg_below(&s, 4);
        if ((which != 1) && (r & 1)) read[i] = (uint8_t)(read[i] | 0x20);
        if ((which != 0) && (r & 2)) ref[i] = (uint8_t)(ref[i] | 0x20);
      }
    }
  }
}

#endif /* PAIRGEN_H */
