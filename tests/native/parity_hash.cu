// parity_hash.cu -- TEST INFRASTRUCTURE: device side of tests/parity_hash.py.
//
// Per-chunk order-independent 64-bit hashes of the CUDA path's (accept, errcount)
// rows, with the same definition as parity_hash.hash_rows_np (written
// independently; no product code, no oracle code):
//   key  = p << 16 | e << 9 | c << 1 | a     (p = global pair index)
//   hash = sum splitmix64_finalize(key + 0x9E3779B97F4A7C15)  mod 2^64
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint64_t mix(uint64_t key) {
  uint64_t z = key + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void hash_kernel(const uint32_t* __restrict__ acc, int64_t acc_stride,
                            const uint8_t* __restrict__ err, int64_t err_stride, int64_t n,
                            const int* __restrict__ es, int64_t p_first, int64_t idx0,
                            int64_t chunk, unsigned long long* __restrict__ out,
                            int64_t nchunks) {
  const int row = blockIdx.y;
  const uint64_t e = (uint64_t)es[row];
  const uint32_t* a = acc + row * acc_stride;
  const uint8_t* c = err + row * err_stride;
  unsigned long long* o = out + row * nchunks;
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    uint64_t h = 0;
    int64_t ch = -1;
    if (i < n) {
      const uint64_t p = (uint64_t)(p_first + i);
      const uint64_t bit = (a[i >> 5] >> (i & 31)) & 1u;
      h = mix((p << 16) | (e << 9) | ((uint64_t)c[i] << 1) | bit);
      ch = (p_first + i - idx0) / chunk;
    }
    // warp reduction when the whole warp is in one chunk (the common case)
    const int64_t ch0 = __shfl_sync(0xFFFFFFFFu, ch, 0);
    const bool same = __all_sync(0xFFFFFFFFu, ch == ch0 || ch < 0);
    if (same) {
      for (int off = 16; off > 0; off >>= 1) h += __shfl_xor_sync(0xFFFFFFFFu, h, off);
      if (lane == 0 && ch0 >= 0) atomicAdd(&o[ch0], (unsigned long long)h);
    } else if (ch >= 0) {
      atomicAdd(&o[ch], (unsigned long long)h);
    }
  }
}

extern "C" int ph_hash_rows(const void* acc, int64_t acc_stride_words, const void* err,
                            int64_t err_stride, int64_t n, int rows, const void* es,
                            int64_t p_first, int64_t idx0, int64_t chunk, void* out,
                            int64_t nchunks, void* stream) {
  if (n <= 0) return 0;
  if (rows < 1 || chunk < 1 || rows > 65535) return -1;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 4096) blocks = 4096;
  hash_kernel<<<dim3((unsigned)blocks, (unsigned)rows), 256, 0, (cudaStream_t)stream>>>(
      (const uint32_t*)acc, acc_stride_words, (const uint8_t*)err, err_stride, n, (const int*)es,
      p_first, idx0, chunk, (unsigned long long*)out, nchunks);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
