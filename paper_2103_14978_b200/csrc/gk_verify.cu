// gk_verify.cu -- the ground truth of the paper's accuracy study on the device:
// exact global edit distance of every pair ("Edlib [...] in global
// mode" decides whether a filtered pair is a false accept or a false reject),
// and the false-accept / false-reject tallies of a set of filter decisions
// (Tables S.2-S.12).
//
// Distance: the bit-vector algorithm of Myers (1999) in Hyyroe's formulation
// for global (Levenshtein) distance, one thread per pair, the read as the
// pattern (W = ceil(L/64) 64-bit words) and the reference segment as the text.
// Per text byte c:  Eq = Peq[c]; Xv = Eq | Mv; Xh = (((Eq & Pv) + Pv) ^ Pv) | Eq;
// Ph = Mv | ~(Xh | Pv); Mh = Pv & Xh; score += Ph[m-1] - Mh[m-1];
// Ph = (Ph << 1) | 1 (global: D[0][j] = j); Mh <<= 1; Pv = Mh | ~(Xv | Ph);
// Mv = Ph & Xv -- the addition and the shifts carry across words.  Bytes are
// compared exactly (as the oracle's textbook DP does): Peq is kept for the 8
// letters A C G T a c g t; a text byte outside them gets its Eq by scanning the
// read (rare: 'N' and IUPAC codes).
#include "gk_common.cuh"
#include "gk_kernels.cuh"

namespace gk {

__device__ __forceinline__ int letter_class(uint32_t c) {
  switch (c) {
    case 'A': return 0;
    case 'C': return 1;
    case 'G': return 2;
    case 'T': return 3;
    case 'a': return 4;
    case 'c': return 5;
    case 'g': return 6;
    case 't': return 7;
    default: return -1;
  }
}

constexpr int ED_THREADS = 128;

template <int W>
__global__ void __launch_bounds__(ED_THREADS) edit_distance_kernel(
    const uint8_t* __restrict__ reads, const uint8_t* __restrict__ refs, int64_t stride,
    int64_t n, int len, int32_t* __restrict__ dist) {
  // Peq[class][word] of every thread: [8][W][ED_THREADS] u64 in shared memory
  extern __shared__ uint64_t peq_sm[];
  const int64_t p = (int64_t)blockIdx.x * ED_THREADS + threadIdx.x;
  if (p >= n) return;
  uint64_t* peq = peq_sm + threadIdx.x;
#pragma unroll
  for (int j = 0; j < 8 * W; ++j) peq[j * ED_THREADS] = 0ull;
  const uint8_t* q = reads + p * stride;
  const uint8_t* r = refs + p * stride;
  for (int i = 0; i < len; ++i) {
    const int c = letter_class(__ldg(q + i));
    if (c >= 0) peq[(c * W + (i >> 6)) * ED_THREADS] |= 1ull << (i & 63);
  }
  uint64_t Pv[W], Mv[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    Pv[w] = ~0ull;
    Mv[w] = 0ull;
  }
  const int lw = (len - 1) >> 6;
  const uint64_t top = 1ull << ((len - 1) & 63);
  int score = len;
  for (int j = 0; j < len; ++j) {
    const uint32_t ch = __ldg(r + j);
    const int c = letter_class(ch);
    uint64_t eq[W];
    if (c >= 0) {
#pragma unroll
      for (int w = 0; w < W; ++w) eq[w] = peq[(c * W + w) * ED_THREADS];
    } else {
#pragma unroll
      for (int w = 0; w < W; ++w) eq[w] = 0ull;
      for (int i = 0; i < len; ++i)
        if (__ldg(q + i) == ch) {
#pragma unroll
          for (int w = 0; w < W; ++w)
            if (w == (i >> 6)) eq[w] |= 1ull << (i & 63);
        }
    }
    uint64_t cin = 0ull, ph_in = 1ull, mh_in = 0ull;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint64_t e = eq[w], pv = Pv[w], mv = Mv[w];
      const uint64_t xv = e | mv;
      const uint64_t t = e & pv;
      const uint64_t s1 = t + pv;
      const uint64_t s = s1 + cin;
      cin = (uint64_t)((s1 < t) | (s < s1));
      const uint64_t xh = (s ^ pv) | e;
      const uint64_t ph = mv | ~(xh | pv);
      const uint64_t mh = pv & xh;
      if (w == lw) score += (int)((ph & top) != 0) - (int)((mh & top) != 0);
      const uint64_t phs = (ph << 1) | ph_in;
      const uint64_t mhs = (mh << 1) | mh_in;
      ph_in = ph >> 63;
      mh_in = mh >> 63;
      Pv[w] = mhs | ~(xv | phs);
      Mv[w] = phs & xv;
    }
  }
  dist[p] = score;
}

template <int W>
static void launch_ed(const uint8_t* reads, const uint8_t* refs, int64_t stride, int64_t n,
                      int len, int32_t* dist, cudaStream_t stream) {
  const size_t smem = (size_t)8 * W * ED_THREADS * 8;
  if (smem > 48 * 1024)
    ensure_func_attr((const void*)edit_distance_kernel<W>,
                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t blocks = (n + ED_THREADS - 1) / ED_THREADS;
  count_launch();
  edit_distance_kernel<W><<<(unsigned)blocks, ED_THREADS, smem, stream>>>(reads, refs, stride, n,
                                                                           len, dist);
}

int launch_edit_distance(const uint8_t* reads, const uint8_t* refs, int64_t stride, int64_t n,
                         int len, int32_t* dist, cudaStream_t stream) {
  switch ((len + 63) >> 6) {
    case 1: launch_ed<1>(reads, refs, stride, n, len, dist, stream); break;
    case 2: launch_ed<2>(reads, refs, stride, n, len, dist, stream); break;
    case 3: launch_ed<3>(reads, refs, stride, n, len, dist, stream); break;
    case 4: launch_ed<4>(reads, refs, stride, n, len, dist, stream); break;
    case 5: launch_ed<5>(reads, refs, stride, n, len, dist, stream); break;
    case 6: launch_ed<6>(reads, refs, stride, n, len, dist, stream); break;
    case 7: launch_ed<7>(reads, refs, stride, n, len, dist, stream); break;
    default: launch_ed<8>(reads, refs, stride, n, len, dist, stream); break;
  }
  return 0;
}

// Tallies of a set of decisions against the distances: per row r (threshold
// e_list[r]) counts[r][0..3] += defined pairs, accepted, false accepts
// (accepted, dist > e), false rejects (rejected, dist <= e).  Undefined pairs
// (errcount 255) are left out, as the paper's sets exclude them
// from the accuracy study.
__global__ void accuracy_kernel(const uint32_t* __restrict__ accept, int64_t astride,
                                const uint8_t* __restrict__ errc, int64_t estride,
                                const int32_t* __restrict__ dist, int64_t n,
                                const int32_t* __restrict__ e_list,
                                unsigned long long* __restrict__ counts) {
  const int row = blockIdx.y;
  const int e = e_list[row];
  unsigned long long c[4] = {0ull, 0ull, 0ull, 0ull};
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    if (errc[row * estride + p] == 255) continue;
    const bool acc = (accept[row * astride + (p >> 5)] >> (p & 31)) & 1u;
    const int d = dist[p];
    c[0] += 1;
    c[1] += acc;
    c[2] += acc && d > e;
    c[3] += !acc && d <= e;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    unsigned long long v = c[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&counts[row * 4 + k], v);
  }
}

int launch_accuracy(const uint32_t* accept, int64_t astride, const uint8_t* errc, int64_t estride,
                    const int32_t* dist, int64_t n, const int32_t* e_list, int rows,
                    unsigned long long* counts, cudaStream_t stream) {
  cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * 4 * (size_t)rows, stream);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (n + 255) / 256;
  if (blocks > 4 * sms) blocks = 4 * sms;
  count_launch();
  accuracy_kernel<<<dim3((unsigned)blocks, (unsigned)rows), 256, 0, stream>>>(
      accept, astride, errc, estride, dist, n, e_list, counts);
  return 0;
}

}  // namespace gk
