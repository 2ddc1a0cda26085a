// pairgen_dev.cu -- device build of pairgen.h (TEST / BENCH INFRASTRUCTURE).
// Generates the same pairs as pairgen_host.c directly in HBM, so the bench's
// 30M-pair / 1B-pair shards never cross PCIe.  Not part of the product library.
#include <cuda_runtime.h>
#include <stdint.h>

#include "pairgen.h"

__global__ void pg_gen_kernel(uint64_t seed, uint64_t idx0, int64_t n, int L, int profile,
                              int emax, uint8_t* __restrict__ reads, uint8_t* __restrict__ refs,
                              int64_t stride) {
  uint8_t buf[PG_BUF];
  uint8_t rd[PG_MAX_LEN];
  uint8_t rf[PG_MAX_LEN];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    pg_gen_pair(seed, idx0 + (uint64_t)i, L, profile, emax, rd, rf, buf);
    uint8_t* r = reads + i * stride;
    uint8_t* f = refs + i * stride;
    for (int j = 0; j < L; ++j) {
      r[j] = rd[j];
      f[j] = rf[j];
    }
    for (int64_t j = L; j < stride; ++j) {
      r[j] = '\n';
      f[j] = '\n';
    }
  }
}

extern "C" int pg_gen_pairs_cuda(uint64_t seed, uint64_t idx0, int64_t n, int L, int profile,
                                 int emax, uint8_t* d_reads, uint8_t* d_refs, int64_t stride,
                                 void* stream) {
  if (L < 1 || L > PG_MAX_LEN || stride < L || n < 0) return -1;
  if (n == 0) return 0;
  int threads = 128;
  int64_t blocks = (n + threads - 1) / threads;
  if (blocks > 148 * 64) blocks = 148 * 64;
  pg_gen_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(
      seed, idx0, n, L, profile, emax, d_reads, d_refs, stride);
  return cudaGetLastError() == cudaSuccess ? 0 : -6;
}
