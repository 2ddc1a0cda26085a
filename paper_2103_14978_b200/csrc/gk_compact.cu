// gk_compact.cu -- a7: ordered indices of the accepted pairs.
//
// The paper's host scans the result buffer for '1's before verification
// (PAPER.md:166-168).  Here the accept bits (one u32 per 32 pairs, as written by
// gk_filter) are compacted on the device: pass 1 counts the set bits of each
// CTA's chunk (popc), pass 2 re-reads the chunk, turns the per-CTA totals into
// its global offset and writes every accepted pair index in ascending order
// (a per-thread exclusive scan of popc, then one index per set bit).
#include "gk_common.cuh"
#include "gk_kernels.cuh"

namespace gk {

// GK_COMPACT_STAGED=1 (default): shared-memory-staged index writes; 0: the
// earlier shuffle loop with direct global stores (A/B knob)
#ifndef GK_COMPACT_STAGED
#define GK_COMPACT_STAGED 1
#endif

constexpr int CP_THREADS = 256;
constexpr int CP_WORDS_PER_THREAD = 8;
constexpr int CP_WORDS_PER_CTA = CP_THREADS * CP_WORDS_PER_THREAD;  // 65536 pairs

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* sm_warp,
                                                         uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) sm_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < (CP_THREADS / 32) ? sm_warp[lane] : 0u;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, w, d);
      if (lane >= d) w += y;
    }
    if (lane < (CP_THREADS / 32)) sm_warp[lane] = w;
  }
  __syncthreads();
  total = sm_warp[CP_THREADS / 32 - 1];
  const uint32_t before = warp > 0 ? sm_warp[warp - 1] : 0u;
  return before + x - v;
}

__device__ __forceinline__ uint32_t load_word(const uint32_t* bits, int64_t w, int64_t nwords,
                                              int64_t n) {
  if (w >= nwords) return 0u;
  uint32_t v = __ldg(bits + w);
  const int64_t first = w * 32;
  if (first + 32 > n) v &= (1u << (int)(n - first)) - 1u;  // bits >= n are ignored
  return v;
}

// blockIdx.y = row of a batch (gk_compact_rows): rows of accept bits at
// bits + y * bstride, counts at cta_counts + y * gridDim.x.
__global__ void __launch_bounds__(CP_THREADS) compact_count_kernel(const uint32_t* __restrict__ bits,
                                                                   int64_t n,
                                                                   uint32_t* __restrict__ cta_counts,
                                                                   int64_t bstride) {
  __shared__ uint32_t sm[CP_THREADS / 32];
  bits += blockIdx.y * bstride;
  cta_counts += (size_t)blockIdx.y * gridDim.x;
  const int64_t nwords = (n + 31) / 32;
  const int64_t w0 = (int64_t)blockIdx.x * CP_WORDS_PER_CTA + threadIdx.x;
  uint32_t c = 0u;
#pragma unroll
  for (int t = 0; t < CP_WORDS_PER_THREAD; ++t)
    c += __popc(load_word(bits, w0 + (int64_t)t * CP_THREADS, nwords, n));
  uint32_t total;
  block_exclusive_scan(c, sm, total);
  if (threadIdx.x == 0) cta_counts[blockIdx.x] = total;
}

__global__ void __launch_bounds__(CP_THREADS) compact_write_kernel(
    const uint32_t* __restrict__ bits, int64_t n, const uint32_t* __restrict__ cta_counts,
    uint32_t* __restrict__ idx, unsigned long long* __restrict__ n_acc, int64_t bstride,
    int64_t istride, uint32_t ibase) {
  bits += blockIdx.y * bstride;
  cta_counts += (size_t)blockIdx.y * gridDim.x;
  if (idx != nullptr) idx += blockIdx.y * istride;
  n_acc += blockIdx.y;
  // CTA: 8 warps x 256 consecutive words.  Warp offsets come from a block scan of
  // the warps' popcounts; inside a warp the words are visited in order and lane j
  // writes the index of bit j, so each word's accepted pairs are one contiguous,
  // coalesced run of indices.
  __shared__ uint32_t sm[CP_THREADS / 32];
  __shared__ unsigned long long sm_part[CP_THREADS / 32];
  __shared__ unsigned long long sm_base;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nwords = (n + 31) / 32;
  unsigned long long part = 0ull;
  for (unsigned b = threadIdx.x; b < blockIdx.x; b += CP_THREADS) part += cta_counts[b];
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) part += __shfl_down_sync(0xFFFFFFFFu, part, d);
  if (lane == 0) sm_part[warp] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0ull;
    for (int w = 0; w < CP_THREADS / 32; ++w) s += sm_part[w];
    sm_base = s;
  }
  const int64_t wbase = (int64_t)blockIdx.x * CP_WORDS_PER_CTA + (int64_t)warp * 256;
  uint32_t words[CP_WORDS_PER_THREAD];
  uint32_t c = 0u;
#pragma unroll
  for (int t = 0; t < CP_WORDS_PER_THREAD; ++t) {
    words[t] = load_word(bits, wbase + 32 * t + lane, nwords, n);
    c += __popc(words[t]);
  }
  uint32_t total;
  const uint32_t before = block_exclusive_scan(c, sm, total);  // lanes of warp w before lane
  // warp start offset = exclusive prefix of lane 0 of this warp
  const uint32_t warp_off = __shfl_sync(0xFFFFFFFFu, before, 0);
  unsigned long long o = sm_base + warp_off;
#if GK_COMPACT_STAGED
  // staged variant: per 32-word chunk each lane expands its own word's set bits
  // (ffs loop) into the warp's shared-memory slice at its scanned offset, then
  // the warp copies the chunk's run out with coalesced stores
  __shared__ uint32_t stage[CP_THREADS / 32][1024];
  if (idx != nullptr) {
    uint32_t* st = stage[warp];
#pragma unroll 1
    for (int t = 0; t < CP_WORDS_PER_THREAD; ++t) {
      uint32_t w = words[t];
      const uint32_t c = __popc(w);
      uint32_t x = c;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, d);
        if (lane >= d) x += y;
      }
      const uint32_t tot = __shfl_sync(0xFFFFFFFFu, x, 31);
      uint32_t pos = x - c;
      const uint32_t base = (uint32_t)((wbase + 32 * t + lane) * 32) + ibase;
      while (w) {
        st[pos++] = base + (uint32_t)(__ffs(w) - 1);
        w &= w - 1u;
      }
      __syncwarp();
      for (uint32_t j = lane; j < tot; j += 32) idx[o + j] = st[j];
      __syncwarp();
      o += tot;
    }
  }
#else
  if (idx != nullptr) {
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int t = 0; t < CP_WORDS_PER_THREAD; ++t) {
#pragma unroll 4
      for (int src = 0; src < 32; ++src) {
        const uint32_t v = __shfl_sync(0xFFFFFFFFu, words[t], src);
        if (v == 0u) continue;
        if ((v >> lane) & 1u)
          idx[o + __popc(v & lt)] = (uint32_t)((wbase + 32 * t + src) * 32 + lane) + ibase;
        o += __popc(v);
      }
    }
  }
#endif
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *n_acc = sm_base + total;
}

size_t compact_workspace_bytes(int64_t n, int rows) {
  const int64_t nwords = (n + 31) / 32;
  const int64_t ctas = (nwords + CP_WORDS_PER_CTA - 1) / CP_WORDS_PER_CTA;
  return (size_t)(ctas > 0 ? ctas : 1) * (size_t)(rows > 0 ? rows : 1) * sizeof(uint32_t);
}

// rows x ceil(n/65536) CTAs per kernel: one launch pair for a whole batch of rows
int launch_compact(const uint32_t* bits, int64_t n, uint32_t* idx, uint64_t* n_acc, void* ws,
                   cudaStream_t stream, int rows, int64_t bstride, int64_t istride,
                   uint32_t ibase) {
  const int64_t nwords = (n + 31) / 32;
  const int64_t ctas = (nwords + CP_WORDS_PER_CTA - 1) / CP_WORDS_PER_CTA;
  uint32_t* counts = reinterpret_cast<uint32_t*>(ws);
  const dim3 grid((unsigned)ctas, (unsigned)rows);
  count_launch(2);
  compact_count_kernel<<<grid, CP_THREADS, 0, stream>>>(bits, n, counts, bstride);
  compact_write_kernel<<<grid, CP_THREADS, 0, stream>>>(
      bits, n, counts, idx, reinterpret_cast<unsigned long long*>(n_acc), bstride, istride, ibase);
  return 0;
}

}  // namespace gk
