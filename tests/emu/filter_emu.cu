// Host emulation of the product filter core (gk_filter_core.cuh) for CPU debugging.
// TEST INFRASTRUCTURE: runs the very same SinglePass/run_range code on the host,
// one "lane" after the other, so the algorithm can be checked against the oracle
// without a GPU.  The GPU parity tests (tests/test_parity_gpu.py) are the real gate.
#include <stdint.h>
#include <string.h>
#include "../../paper_2103_14978_b200/csrc/gk_filter_core.cuh"

using namespace gk;

struct HostSrc {
  static constexpr bool kHoistLoads = true;
  const uint32_t* q;  // packed words of (tile) base; index ((pos*32)+lane)*2
  const uint32_t* r;
  int lane, len;
  __host__ __device__ uint2 ld(const uint32_t* p, int pos) const {
    if (pos < 0 || pos >= len) return make_uint2(0u, 0u);
    const uint32_t* w = p + ((int64_t)pos * 32 + lane) * 2;
    return make_uint2(w[0], w[1]);
  }
  __host__ __device__ uint2 ldq(int pos) const { return ld(q, pos); }
  __host__ __device__ uint2 ldr(int pos) const { return ld(r, pos); }
  __host__ __device__ uint2 ldq_nc(int pos) const { return ld(q, pos); }
  __host__ __device__ uint2 ldr_nc(int pos) const { return ld(r, pos); }
};

static int value(const uint32_t (&c)[8], int j) {
  int v = 0;
  for (int b = 0; b < 8; ++b) v |= ((c[b] >> j) & 1) << b;
  return v;
}

template <int E>
static void run(const uint32_t* q, const uint32_t* r, const uint32_t* uq, const uint32_t* ur,
                int64_t n, int len, uint8_t* acc, uint8_t* err, int split) {
  const int64_t tiles = (n + 1023) / 1024;
  for (int64_t t = 0; t < tiles; ++t) {
    for (int lane = 0; lane < 32; ++lane) {
      const int64_t g = t * 32 + lane;
      if (g * 32 >= n) continue;
      HostSrc src{q + t * (int64_t)len * 64, r + t * (int64_t)len * 64, lane, len};
      int cA[32] = {0}, cF[32] = {0};
      int chunk = split > 1 ? (((len + split - 1) / split + 3) & ~3) : len;
      for (int lo = 0; lo < len; lo += chunk) {
        int hi = lo + chunk < len ? lo + chunk : len;
        SinglePass<E> sp;
        run_range<E>(sp, src, len, lo, hi);
        uint32_t a[8], f[8];
        sp.cA.planes(a);
        sp.cF.planes(f);
        for (int j = 0; j < 32; ++j) { cA[j] += value(a, j); cF[j] += value(f, j); }
      }
      const uint32_t und = uq[g] | ur[g];
      for (int j = 0; j < 32; ++j) {
        const int64_t p = g * 32 + j;
        if (p >= n) break;
        int a, c;
        if ((und >> j) & 1) { a = 1; c = 255; }
        else if (cA[j] <= E) { a = 1; c = cA[j]; }
        else if (E == 0) { a = 0; c = cA[j]; }
        else { a = cF[j] <= E; c = cF[j]; }
        acc[p] = (uint8_t)a;
        err[p] = (uint8_t)c;
      }
    }
  }
}

template <int E>
static int dispatch(int e, const uint32_t* q, const uint32_t* r, const uint32_t* uq,
                    const uint32_t* ur, int64_t n, int len, uint8_t* acc, uint8_t* err, int split) {
  if (e == E) { run<E>(q, r, uq, ur, n, len, acc, err, split); return 0; }
  if constexpr (E > 0) return dispatch<E - 1>(e, q, r, uq, ur, n, len, acc, err, split);
  return -1;
}

extern "C" int emu_filter(const uint32_t* q, const uint32_t* r, const uint32_t* uq,
                          const uint32_t* ur, int64_t n, int len, int e, uint8_t* acc,
                          uint8_t* err, int split) {
  return dispatch<11>(e, q, r, uq, ur, n, len, acc, err, split);
}
