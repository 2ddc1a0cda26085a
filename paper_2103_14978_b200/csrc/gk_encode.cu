// gk_encode.cu -- a1: ASCII -> bit-sliced 2-bit planes (+ undefined flags).
//
// every base becomes a 2-bit code (A=00 C=01 G=10 T=11, :49);
// pairs with a base outside the alphabet pass unfiltered (:95), so the encoder
// also flags "undefined" sequences.  The paper encodes one sequence per thread
// into 7 words (:93, :105); here one warp encodes one group of 32 sequences and
// writes the bit-sliced layout of include/gatekeeper.h, in which a 32-bit word
// holds one base position of 32 sequences.
//
// Per 4 bytes the work is branch-free SWAR integer code:
//   * validity: m = ((w & 0x26) | 0x41) + 15*[bit2 & ~bit1] per byte reproduces
//     the byte iff it is one of A C G T a c g t (the 8 values m can take are
//     exactly that set), so bad |= w ^ m is 0 iff all 4 bytes are valid;
//   * code planes: plane0 (high) = ASCII bit 2, plane1 (low) = bit 1 ^ bit 2
//     (A 0x41 -> 00, C 0x43 -> 01, G 0x47 -> 10, T 0x54 -> 11, case-free);
//   * transposition: a 4x4 byte transpose (8 PRMT) turns 4 rows x 4 positions
//     into 4 positions x 4 rows, then one IMAD per plane gathers bit b of the 4
//     bytes into a nibble (no carries: see gather_bit2/gather_bit1) and one funnel
//     shift appends the nibble to the 32-sequence word.
#include "gk_common.cuh"
#include "gk_encode_core.cuh"
#include "gk_kernels.cuh"

namespace gk {

template <bool ALIGNED>
__global__ void __launch_bounds__(128) encode_kernel(const uint8_t* __restrict__ seqs,
                                                     int64_t n, int len, int64_t stride,
                                                     uint32_t* __restrict__ packed,
                                                     uint32_t* __restrict__ undef,
                                                     int groups_per_cta) {
  extern __shared__ __align__(16) uint8_t sm_enc[];
  const int64_t ngroups = (n + 31) / 32;
  const int64_t g0 = (int64_t)blockIdx.x * groups_per_cta;
  const int64_t s0 = g0 * 32;
  int64_t s1 = s0 + (int64_t)groups_per_cta * 32;
  if (s1 > n) s1 = n;
  // stage rows s0..s1-1 (first len bytes of the last row)
  const uint8_t* src = seqs + s0 * stride;
  const int64_t nbytes = (s1 - 1 - s0) * stride + len;
  stage_span(src, nbytes, sm_enc, threadIdx.x, blockDim.x);
  __syncthreads();
  const uint32_t base_off = (uint32_t)(reinterpret_cast<uintptr_t>(src) & 15u);

  const int warp = threadIdx.x >> 5;
  const int64_t g = g0 + warp;
  if (warp >= groups_per_cta || g >= ngroups) return;
  const int64_t tile = g >> 5;
  const int lane_in_tile = (int)(g & 31);
  const int nvalid = (int)((n - g * 32) < 32 ? (n - g * 32) : 32);
  const uint32_t row0 = base_off + (uint32_t)(warp * 32) * (uint32_t)stride;
  uint2* out = reinterpret_cast<uint2*>(packed);
  const uint32_t und = encode_group<ALIGNED>(
      sm_enc, row0, (uint32_t)stride, nvalid, len, [&](int pos, uint32_t hi, uint32_t lo) {
        out[packed_index(tile, len, pos, lane_in_tile, 0) >> 1] = make_uint2(hi, lo);
      });
  if ((threadIdx.x & 31) == 0) undef[g] = und;
}

// Tail groups of the last tile (g >= ngroups up to the tile boundary): all 'A'.
__global__ void encode_tail_kernel(int64_t first_group, int64_t end_group, int len,
                                   uint32_t* __restrict__ packed, uint32_t* __restrict__ undef) {
  const int64_t total = (end_group - first_group) * len;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = first_group + i / len;
    const int pos = (int)(i % len);
    reinterpret_cast<uint2*>(packed)[packed_index(g >> 5, len, pos, (int)(g & 31), 0) >> 1] =
        make_uint2(0u, 0u);
    if (pos == 0) undef[g] = 0u;
  }
}

int launch_encode(const uint8_t* seqs, int64_t n, int len, int64_t stride, uint32_t* packed,
                  uint32_t* undef, cudaStream_t stream) {
  const int64_t ngroups = (n + 31) / 32;
  int gpc = (int)(49152 / (32 * stride));
  if (gpc > 4) gpc = 4;
  if (gpc < 1) gpc = 1;
  const size_t smem = (size_t)gpc * 32 * (size_t)stride + 32;
  const int64_t blocks = (ngroups + gpc - 1) / gpc;
  const bool aligned = (stride % 4 == 0) && ((reinterpret_cast<uintptr_t>(seqs) & 3u) == 0);
  if (smem > 48 * 1024) {
    cudaFuncSetAttribute(encode_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaFuncSetAttribute(encode_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  }
  if (aligned)
    encode_kernel<true><<<(unsigned)blocks, gpc * 32, smem, stream>>>(seqs, n, len, stride,
                                                                      packed, undef, gpc);
  else
    encode_kernel<false><<<(unsigned)blocks, gpc * 32, smem, stream>>>(seqs, n, len, stride,
                                                                       packed, undef, gpc);
  const int64_t tile_end = ((ngroups + 31) / 32) * 32;
  if (tile_end > ngroups) {
    const int64_t total = (tile_end - ngroups) * len;
    const int threads = 256;
    const int64_t tb = (total + threads - 1) / threads;
    encode_tail_kernel<<<(unsigned)(tb < 1024 ? tb : 1024), threads, 0, stream>>>(
        ngroups, tile_end, len, packed, undef);
  }
  return 0;
}

}  // namespace gk
