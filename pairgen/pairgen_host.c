/* pairgen_host.c -- host build of pairgen.h (TEST / BENCH INFRASTRUCTURE). */
#include <pthread.h>
#include <stdint.h>
#include <string.h>

#include "pairgen.h"

typedef struct {
  uint64_t seed, idx0;
  int64_t lo, hi;
  int L, profile, emax;
  uint8_t *reads, *refs;
  int64_t stride;
} pg_job;

static void* pg_worker(void* arg) {
  pg_job* j = (pg_job*)arg;
  uint8_t buf[PG_BUF];
  for (int64_t i = j->lo; i < j->hi; ++i) {
    uint8_t* r = j->reads + i * j->stride;
    uint8_t* f = j->refs + i * j->stride;
    pg_gen_pair(j->seed, j->idx0 + (uint64_t)i, j->L, j->profile, j->emax, r, f, buf);
    if (j->stride > j->L) {
      memset(r + j->L, '\n', (size_t)(j->stride - j->L));
      memset(f + j->L, '\n', (size_t)(j->stride - j->L));
    }
  }
  return 0;
}

int pg_gen_pairs(uint64_t seed, uint64_t idx0, int64_t n, int L, int profile, int emax,
                 uint8_t* reads, uint8_t* refs, int64_t stride, int nthreads) {
  if (L < 1 || L > PG_MAX_LEN || stride < L || n < 0) return -1;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (n < 4096) nthreads = 1;
  pthread_t th[256];
  pg_job jobs[256];
  for (int t = 0; t < nthreads; ++t) {
    jobs[t].seed = seed;
    jobs[t].idx0 = idx0;
    jobs[t].lo = n * t / nthreads;
    jobs[t].hi = n * (t + 1) / nthreads;
    jobs[t].L = L;
    jobs[t].profile = profile;
    jobs[t].emax = emax;
    jobs[t].reads = reads;
    jobs[t].refs = refs;
    jobs[t].stride = stride;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], 0, pg_worker, &jobs[t]);
  pg_worker(&jobs[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(th[t], 0);
  return 0;
}
