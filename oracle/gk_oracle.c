/* gk_oracle.c -- plain, slow, obviously correct CPU oracle of GateKeeper-GPU's
 * per-pair pre-alignment filter (Bingol et al., arXiv 2103.14978).
 *
 * TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or constant with the CUDA product path
 * (paper_2103_14978_b200/csrc); the product never calls it.
 *
 * Every step follows the paper's description in the paper's order, one byte
 * per base / mask position, no bit packing, no blocking or fusion:
 *   PAPER.md:49   2-bit encoding A=00 C=01 G=10 T=11; Hamming mask by XOR;
 *                 shifted read by k for deletion / insertion; XOR with the
 *                 reference; OR of every 2-bit pair -> one bit per base.
 *   PAPER.md:51   amend short 0-streaks; AND of the 2e+1 masks; windowed count
 *                 with a look-up table; reject iff count > e.
 *   PAPER.md:95   pairs containing 'N' pass without filtration.
 *   PAPER.md:107  shifts are per base with carry (here: plain array indexing).
 *   PAPER.md:109  GateKeeper-GPU's edge fix: after amendment, the vacated
 *                 leading/trailing bits of the shifted masks are ORed to 1.
 *   Fig. S.1 worked flow: Hamming-stage count decides
 *                 whether approximate string matching (ASM) begins.
 * Readings R1-R13 of the garbled / silent passages are listed in DESIGN.md
 * ("Readings of the paper").  Functions whose results no paper value or
 * closed form pins are marked "parity unpinned" there; here the Hamming
 * stage, amendment boundary rule, shifts, AND, count and decision are pinned
 * by tests/golden (Fig. S.1, Fig. 2) and tests/test_oracle_*.py invariants.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GKO_MAX_LEN 508

/* 2-bit code of a base, PAPER.md:49 (A=00, C=01, G=10, T=11).  Lower case is
 * the same base (reading R8).  Any other byte -> -1 ("undefined", :95). */
int gko_code(uint8_t b) {
  switch (b) {
    case 'A': case 'a': return 0;
    case 'C': case 'c': return 1;
    case 'G': case 'g': return 2;
    case 'T': case 't': return 3;
    default: return -1;
  }
}

/* One base of the XOR row between the reference and the read shifted by k
 * bases (R1).  shift > 0: read moved toward higher positions (deletion mask,
 * Fig. 2 ">>"), shift < 0: toward lower positions (insertion mask, "<<"),
 * shift == 0: Hamming mask.  A vacated position XORs to 00 (R2: the vacated
 * bits are 0 in the shifted masks; Fig. 2 I1 row prints 00). */
static int xor_code(const int* q, const int* r, int L, int i, int shift) {
  int j = i - shift;
  if (j < 0 || j >= L) return 0;
  return r[i] ^ q[j];
}

/* Public: the 2-bit XOR row (values 0..3), for the Fig. 2 pin. */
int gko_xor_row(const uint8_t* read, const uint8_t* ref, int L, int shift, uint8_t* out) {
  int q[GKO_MAX_LEN], r[GKO_MAX_LEN];
  if (L < 1 || L > GKO_MAX_LEN) return -1;
  for (int i = 0; i < L; ++i) {
    q[i] = gko_code(read[i]);
    r[i] = gko_code(ref[i]);
    if (q[i] < 0 || r[i] < 0) return -2;
  }
  for (int i = 0; i < L; ++i) out[i] = (uint8_t)xor_code(q, r, L, i, shift);
  return 0;
}

/* Mask from an XOR row: every 2-bit pair combined with OR. */
static void mask_from_xor(const int* q, const int* r, int L, int shift, uint8_t* M) {
  for (int i = 0; i < L; ++i) {
    int x = xor_code(q, r, L, i, shift);
    M[i] = (uint8_t)(((x >> 1) & 1) | (x & 1));
  }
}

/* Amendment (R3): every maximal run of 0s [a,b) that is bounded
 * by 1s on both sides (a > 0 and b < L) and is at most 2 long becomes 1s.
 * Runs touching position 0 or L-1 are never amended (Fig. S.1 :455, :458). */
void gko_amend(const uint8_t* M, int L, uint8_t* A) {
  for (int i = 0; i < L; ++i) A[i] = M[i];
  int i = 0;
  while (i < L) {
    if (M[i] != 0) { ++i; continue; }
    int a = i;
    while (i < L && M[i] == 0) ++i;
    int b = i;
    if (a > 0 && b < L && (b - a) <= 2)
      for (int t = a; t < b; ++t) A[t] = 1;
  }
}

/* Windowed error count (R6/R7): windows of 4 bases starting at
 * base 0; each window contributes the number of maximal runs of 1s inside it
 * (the look-up table entry of its 4-bit pattern); the last window may be
 * partial.  Fig. S.1 counts 17 ones in 5 windows as 5 errors (:468). */
int gko_count(const uint8_t* M, int L) {
  int c = 0;
  for (int w = 0; w < L; w += 4) {
    int end = w + 4 < L ? w + 4 : L;
    int prev = 0;
    for (int i = w; i < end; ++i) {
      if (M[i] && !prev) ++c;
      prev = M[i];
    }
  }
  return c;
}

/* The filtration of one pair ("filtration").
 * masks (optional): (4e+3)*L bytes: H0, A0, then per k=1..e: D_k, A*D_k,
 * I_k, A*I_k, then F (only filled when the ASM loop runs; zeros otherwise).
 * edge_fix = 1: GateKeeper-GPU (:109); 0: original GateKeeper (Fig. S.1).
 * Outputs accept (0/1) and err: 255 for an undefined pair (:95, R8), else the
 * count of the stage that decided (R5, R9). */
int gko_filter_pair(const uint8_t* read, const uint8_t* ref, int L, int e, int edge_fix,
                    int* accept, int* err, uint8_t* masks) {
  int q[GKO_MAX_LEN], r[GKO_MAX_LEN];
  uint8_t H0[GKO_MAX_LEN], A0[GKO_MAX_LEN], F[GKO_MAX_LEN];
  uint8_t D[GKO_MAX_LEN], AD[GKO_MAX_LEN], I[GKO_MAX_LEN], AI[GKO_MAX_LEN];
  if (L < 1 || L > GKO_MAX_LEN || e < 0 || e >= L) return -1;
  if (masks) memset(masks, 0, (size_t)(4 * e + 3) * (size_t)L);

  /* Preprocessing: 2-bit encoding; 'N' (any non-ACGT byte) passes (:95). */
  int undefined = 0;
  for (int i = 0; i < L; ++i) {
    q[i] = gko_code(read[i]);
    r[i] = gko_code(ref[i]);
    if (q[i] < 0 || r[i] < 0) undefined = 1;
  }
  if (undefined) { *accept = 1; *err = 255; return 0; }

  /* Hamming mask (exact match detection, :49) and its amended form. */
  mask_from_xor(q, r, L, 0, H0);
  gko_amend(H0, L, A0);
  if (masks) { memcpy(masks, H0, (size_t)L); memcpy(masks + L, A0, (size_t)L); }

  /* Error counting on the Hamming stage; "e > E, therefore ASM begins"
   * (Fig. S.1 :466-467, R5).  With e = 0 there is no ASM (:49). */
  int c0 = gko_count(A0, L);
  if (c0 <= e) { *accept = 1; *err = c0; return 0; }
  if (e == 0) { *accept = 0; *err = c0; return 0; }

  /* Approximate string matching: k = 1..e, one deletion and one insertion
   * mask per k (:49), amended (:51), edge-fixed after amendment (:109),
   * ANDed with all others (:51). */
  for (int i = 0; i < L; ++i) F[i] = A0[i];
  for (int k = 1; k <= e; ++k) {
    mask_from_xor(q, r, L, +k, D);   /* deletion: read shifted right (">>") */
    mask_from_xor(q, r, L, -k, I);   /* insertion: read shifted left ("<<") */
    gko_amend(D, L, AD);
    gko_amend(I, L, AI);
    if (edge_fix) {
      for (int i = 0; i < k && i < L; ++i) AD[i] = 1;            /* leading */
      for (int i = L - k; i < L; ++i) if (i >= 0) AI[i] = 1;     /* trailing */
    }
    for (int i = 0; i < L; ++i) F[i] = (uint8_t)(F[i] & AD[i] & AI[i]);
    if (masks) {
      uint8_t* m = masks + (size_t)(2 + 4 * (k - 1)) * (size_t)L;
      memcpy(m, D, (size_t)L);
      memcpy(m + L, AD, (size_t)L);
      memcpy(m + 2 * L, I, (size_t)L);
      memcpy(m + 3 * L, AI, (size_t)L);
    }
  }
  if (masks) memcpy(masks + (size_t)(2 + 4 * e) * (size_t)L, F, (size_t)L);

  /* Decision: rejected iff the number of errors exceeds e (:51). */
  int c = gko_count(F, L);
  *accept = c <= e ? 1 : 0;
  *err = c;
  return 0;
}

/* Threshold sweep of one pair in a single pass (the prefix property of the AND
 * chain): the final bit-vector for threshold e is
 *     F_e = A0 AND (A*D_1 AND A*I_1) AND ... AND (A*D_e AND A*I_e)
 * (PAPER.md:49 "2e+1 masks", :51 "AND"), so F_e = F_{e-1} AND A*D_e AND A*I_e
 * and one pass over k = 1..emax yields F_e for every e <= emax.  Each k builds
 * its masks exactly as gko_filter_pair does (same functions, same order).  The
 * decision for each e is gko_filter_pair's: c0 <= e accepts with c0 (R5), e = 0
 * rejects with c0 (:49), else count(F_e) decides (:51).  Pairs with c0 <= k
 * need no F_k (every e >= c0 is decided by the Hamming stage), so the k loop
 * stops there.  accept[e], err[e] for e = 0..emax (stride 1 per e). */
int gko_sweep_pair(const uint8_t* read, const uint8_t* ref, int L, int emax, int edge_fix,
                   uint8_t* accept, uint8_t* err, int64_t estride) {
  int q[GKO_MAX_LEN], r[GKO_MAX_LEN];
  uint8_t H0[GKO_MAX_LEN], A0[GKO_MAX_LEN], F[GKO_MAX_LEN];
  uint8_t D[GKO_MAX_LEN], AD[GKO_MAX_LEN], I[GKO_MAX_LEN], AI[GKO_MAX_LEN];
  if (L < 1 || L > GKO_MAX_LEN || emax < 0 || emax >= L) return -1;

  int undefined = 0;
  for (int i = 0; i < L; ++i) {
    q[i] = gko_code(read[i]);
    r[i] = gko_code(ref[i]);
    if (q[i] < 0 || r[i] < 0) undefined = 1;
  }
  if (undefined) {                                     /* :95 */
    for (int e = 0; e <= emax; ++e) { accept[e * estride] = 1; err[e * estride] = 255; }
    return 0;
  }
  mask_from_xor(q, r, L, 0, H0);                       /* :49 */
  gko_amend(H0, L, A0);                                /* :51 */
  int c0 = gko_count(A0, L);
  /* e = 0: no ASM (:49); every e >= c0: Hamming-stage accept (R5) */
  accept[0] = c0 <= 0 ? 1 : 0;
  err[0] = (uint8_t)c0;
  for (int e = 1; e <= emax; ++e)
    if (c0 <= e) { accept[e * estride] = 1; err[e * estride] = (uint8_t)c0; }

  for (int i = 0; i < L; ++i) F[i] = A0[i];
  for (int k = 1; k <= emax && k < c0; ++k) {          /* F_k = F_{k-1} & A*D_k & A*I_k */
    mask_from_xor(q, r, L, +k, D);
    mask_from_xor(q, r, L, -k, I);
    gko_amend(D, L, AD);
    gko_amend(I, L, AI);
    if (edge_fix) {                                    /* :109 */
      for (int i = 0; i < k && i < L; ++i) AD[i] = 1;
      for (int i = L - k; i < L; ++i) if (i >= 0) AI[i] = 1;
    }
    for (int i = 0; i < L; ++i) F[i] = (uint8_t)(F[i] & AD[i] & AI[i]);
    int c = gko_count(F, L);                           /* :51 decision for e = k */
    accept[k * estride] = c <= k ? 1 : 0;
    err[k * estride] = (uint8_t)c;
  }
  return 0;
}

/* ---- batch driver (pthreads; a pure scheduling wrapper) ------------------ */
typedef struct {
  const uint8_t *reads, *refs;
  int64_t lo, hi, stride;
  int L, e, emax, edge_fix, sweep;
  uint8_t *accept, *err;
  int64_t n;
  int rc;
} gko_job;

static void* gko_worker(void* arg) {
  gko_job* j = (gko_job*)arg;
  for (int64_t p = j->lo; p < j->hi; ++p) {
    const uint8_t* rd = j->reads + p * j->stride;
    const uint8_t* rf = j->refs + p * j->stride;
    if (!j->sweep) {
      int a, c;
      if (gko_filter_pair(rd, rf, j->L, j->e, j->edge_fix, &a, &c, 0)) { j->rc = -1; return 0; }
      j->accept[p] = (uint8_t)a;
      if (j->err) j->err[p] = (uint8_t)c;
    } else if (j->sweep == 2) {
      if (gko_sweep_pair(rd, rf, j->L, j->emax, j->edge_fix, j->accept + p, j->err + p, j->n)) {
        j->rc = -1;
        return 0;
      }
    } else {
      for (int e = 0; e <= j->emax; ++e) {
        int a, c;
        if (gko_filter_pair(rd, rf, j->L, e, j->edge_fix, &a, &c, 0)) { j->rc = -1; return 0; }
        j->accept[(int64_t)e * j->n + p] = (uint8_t)a;
        if (j->err) j->err[(int64_t)e * j->n + p] = (uint8_t)c;
      }
    }
  }
  return 0;
}

static int gko_run(gko_job* base, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (base->n < 256) nthreads = 1;
  pthread_t th[256];
  gko_job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = *base;
    jobs[t].lo = base->n * t / nthreads;
    jobs[t].hi = base->n * (t + 1) / nthreads;
    jobs[t].rc = 0;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], 0, gko_worker, &jobs[t]);
  gko_worker(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], 0);
  for (int t = 0; t < nthreads; ++t) if (jobs[t].rc) return jobs[t].rc;
  return 0;
}

/* accept[n] (0/1), err[n] (may be NULL) for one threshold e. */
int gko_filter(const uint8_t* reads, const uint8_t* refs, int64_t n, int L, int64_t stride,
               int e, int edge_fix, uint8_t* accept, uint8_t* err, int nthreads) {
  if (n < 0 || L < 1 || L > GKO_MAX_LEN || stride < L || e < 0 || e >= L) return -1;
  gko_job j;
  memset(&j, 0, sizeof j);
  j.reads = reads; j.refs = refs; j.n = n; j.L = L; j.stride = stride; j.e = e;
  j.edge_fix = edge_fix; j.accept = accept; j.err = err;
  return gko_run(&j, nthreads);
}

/* Threshold sweep: accept[(emax+1)][n], err[(emax+1)][n]; each e is an
 * independent call of the filtration above (no shortcut). */
int gko_sweep(const uint8_t* reads, const uint8_t* refs, int64_t n, int L, int64_t stride,
              int emax, int edge_fix, uint8_t* accept, uint8_t* err, int nthreads) {
  if (n < 0 || L < 1 || L > GKO_MAX_LEN || stride < L || emax < 0 || emax >= L) return -1;
  gko_job j;
  memset(&j, 0, sizeof j);
  j.reads = reads; j.refs = refs; j.n = n; j.L = L; j.stride = stride; j.emax = emax;
  j.edge_fix = edge_fix; j.accept = accept; j.err = err; j.sweep = 1;
  return gko_run(&j, nthreads);
}

/* Threshold sweep in one pass per pair (gko_sweep_pair): the same outputs as
 * gko_sweep, pinned row for row against it (tests/test_oracle_sweep.py).
 * Used for full-size parity, where e_max+1 independent filtrations per pair
 * would cost hours of CPU. */
int gko_sweep_prefix(const uint8_t* reads, const uint8_t* refs, int64_t n, int L, int64_t stride,
                     int emax, int edge_fix, uint8_t* accept, uint8_t* err, int nthreads) {
  if (n < 0 || L < 1 || L > GKO_MAX_LEN || stride < L || emax < 0 || emax >= L) return -1;
  gko_job j;
  memset(&j, 0, sizeof j);
  j.reads = reads; j.refs = refs; j.n = n; j.L = L; j.stride = stride; j.emax = emax;
  j.edge_fix = edge_fix; j.accept = accept; j.err = err; j.sweep = 2;
  return gko_run(&j, nthreads);
}

/* ---- ground truth: global edit distance (textbook Levenshtein DP) -------- */
/* Edlib's global edit distance is the accuracy ground
 * truth; this is the plain O(La*Lb) dynamic program of Levenshtein [17]. */
int gko_levenshtein(const uint8_t* a, int La, const uint8_t* b, int Lb) {
  if (La < 0 || Lb < 0 || La > 4096 || Lb > 4096) return -1;
  int* prev = (int*)malloc(sizeof(int) * (size_t)(Lb + 1));
  int* cur = (int*)malloc(sizeof(int) * (size_t)(Lb + 1));
  for (int j = 0; j <= Lb; ++j) prev[j] = j;
  for (int i = 1; i <= La; ++i) {
    cur[0] = i;
    for (int j = 1; j <= Lb; ++j) {
      int sub = prev[j - 1] + (a[i - 1] != b[j - 1]);
      int del = prev[j] + 1;
      int ins = cur[j - 1] + 1;
      int m = sub < del ? sub : del;
      cur[j] = m < ins ? m : ins;
    }
    int* t = prev; prev = cur; cur = t;
  }
  int d = prev[Lb];
  free(prev);
  free(cur);
  return d;
}

/* ---- reference packer for the library's bit-sliced layout ---------------- */
/* Layout (include/gatekeeper.h, "packed sequence layout"): sequence s lives in
 * tile t = s / 1024, lane g = (s / 32) % 32, bit j = s % 32; the 32-bit word
 * ((t * L + i) * 32 + g) * 2 + p holds, at bit j, plane p of base i of s:
 * p = 0 the high bit, p = 1 the low bit of the 2-bit code.
 * undef[t * 32 + g] bit j = 1 iff s has a byte outside {A,C,G,T,a,c,g,t}.
 * Sequences s >= n (tail of the last tile) are all 'A' and defined.  Plane
 * bits of an undefined sequence are not specified by the layout and are
 * reported here as 0 (tests compare them only for defined sequences). */
int gko_pack(const uint8_t* seqs, int64_t n, int L, int64_t stride, uint32_t* words,
             uint32_t* undef) {
  if (n < 0 || L < 1 || L > GKO_MAX_LEN || stride < L) return -1;
  int64_t tiles = (n + 1023) / 1024;
  memset(words, 0, (size_t)(tiles * L * 64) * sizeof(uint32_t));
  memset(undef, 0, (size_t)(tiles * 32) * sizeof(uint32_t));
  for (int64_t s = 0; s < n; ++s) {
    int64_t t = s / 1024;
    int g = (int)((s / 32) % 32);
    int j = (int)(s % 32);
    int bad = 0;
    for (int i = 0; i < L; ++i)
      if (gko_code(seqs[s * stride + i]) < 0) bad = 1;
    if (bad) { undef[t * 32 + g] |= 1u << j; continue; }
    for (int i = 0; i < L; ++i) {
      int c = gko_code(seqs[s * stride + i]);
      int64_t w = ((t * L + i) * 32 + g) * 2;
      if ((c >> 1) & 1) words[w + 0] |= 1u << j;
      if (c & 1) words[w + 1] |= 1u << j;
    }
  }
  return 0;
}

/* Batch ground truth for false-accept / false-reject accounting (A23):
 * dist[p] = gko_levenshtein(read_p, ref_p) over the first L bytes of each row. */
typedef struct {
  const uint8_t *reads, *refs;
  int64_t lo, hi, stride;
  int L;
  int32_t* dist;
} gko_edjob;

static void* gko_edworker(void* arg) {
  gko_edjob* j = (gko_edjob*)arg;
  for (int64_t p = j->lo; p < j->hi; ++p)
    j->dist[p] = gko_levenshtein(j->reads + p * j->stride, j->L, j->refs + p * j->stride, j->L);
  return 0;
}

int gko_edit_batch(const uint8_t* reads, const uint8_t* refs, int64_t n, int L, int64_t stride,
                   int32_t* dist, int nthreads) {
  if (n < 0 || L < 0 || stride < L) return -1;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (n < 256) nthreads = 1;
  pthread_t th[256];
  gko_edjob jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].reads = reads; jobs[t].refs = refs; jobs[t].stride = stride; jobs[t].L = L;
    jobs[t].dist = dist; jobs[t].lo = n * t / nthreads; jobs[t].hi = n * (t + 1) / nthreads;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], 0, gko_edworker, &jobs[t]);
  gko_edworker(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], 0);
  return 0;
}
