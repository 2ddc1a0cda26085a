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
#include "gk_tma.cuh"

#ifndef GK_ENCODE_TMA
#define GK_ENCODE_TMA 1
#endif
// minimum resident CTAs per SM requested from ptxas for the TMA encoder (A/B knob)
#ifndef GK_ENC_MINB
#define GK_ENC_MINB 1
#endif
// The 256-byte staging variant runs at 3 CTAs per SM (168 registers) when its last
// lane-iteration is the sparse shared-quad tail (len <= 192, e.g. 150 bp: 1.63 ->
// 1.54 ms per 30M) and at the register-unbounded 2 CTAs per SM otherwise (250 bp:
// 3 CTAs measured 2.11 -> 2.19 ms); profiles/r01l_encoder_wide_minb_ab.jsonl.
#ifndef GK_ENC_MINB_SPARSE
#define GK_ENC_MINB_SPARSE 3
#endif

namespace gk {

// Generic encoder: any alignment / stride / tail; also the tail of the TMA path.
template <bool ALIGNED>
__global__ void __launch_bounds__(128) encode_kernel(const uint8_t* __restrict__ seqs,
                                                     int64_t n, int len, int64_t stride,
                                                     uint32_t* __restrict__ packed,
                                                     uint32_t* __restrict__ undef,
                                                     int groups_per_cta, int64_t first_group) {
  extern __shared__ __align__(16) uint8_t sm_enc[];
  const int64_t ngroups = (n + 31) / 32;
  const int64_t g0 = first_group + (int64_t)blockIdx.x * groups_per_cta;
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

// TMA encoder: full blocks of 4 groups (128 sequences).  Persistent CTAs of 4
// warps; warp w encodes group 4b+w of block b.  Its 32 rows (one contiguous span
// of 32*stride bytes) arrive by one cp.async.bulk into a double buffer, the next
// block's span being prefetched while the current one is encoded.  The 4 groups'
// words are collected in shared memory and written out as full 32-byte sectors.
template <int PMAX, int SM4, bool LPART, int MB>
__global__ void __launch_bounds__(128, MB) encode_tma_kernel(const uint8_t* __restrict__ seqs,
                                                         int64_t nblocks, int len, int stride,
                                                         uint32_t* __restrict__ packed,
                                                         uint32_t* __restrict__ undef) {
  constexpr int NIT = PMAX / 128;          // quad iterations per lane (4 bytes x 32 lanes)
  constexpr uint32_t BUF = 32u * PMAX;     // bytes of one staging buffer
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* stage = sm + (size_t)warp * 2 * BUF;                    // [2][32*PMAX]
  const int nq = (len + 3) >> 2;
  uint2* outt0 = reinterpret_cast<uint2*>(sm + 4 * 2 * BUF);       // 2 x [4 warps][4 m][nq]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 4 * 2 * BUF + (size_t)2 * 16 * 8 * nq);
  uint64_t* mybar = bars + 2 * warp;
  if (lane == 0) {
    mbar_init(&mybar[0], 1);
    mbar_init(&mybar[1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  RowAddr<SM4> ra;
  ra.init(smem_u32(stage), (uint32_t)stride, lane);
  const uint32_t span = 32u * (uint32_t)stride;

  int64_t b = blockIdx.x;
  if (b >= nblocks) return;
  if (lane == 0) {
    mbar_arrive_expect_tx(&mybar[0], span);
    tma_load_1d(stage, seqs + (4 * b + warp) * (int64_t)span, span, &mybar[0]);
  }
  for (int i = 0; b < nblocks; ++i, b += gridDim.x) {
    const int buf = i & 1;
    const int64_t bn = b + gridDim.x;
    if (lane == 0 && bn < nblocks) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&mybar[buf ^ 1], span);
      tma_load_1d(stage + (buf ^ 1) * BUF, seqs + (4 * bn + warp) * (int64_t)span, span,
                  &mybar[buf ^ 1]);
    }
    mbar_wait(&mybar[buf], (uint32_t)(i >> 1) & 1u);  // buffer buf's (i>>1)-th use
    const int64_t g = 4 * b + warp;
    uint2* outt = outt0 + (size_t)(i & 1) * 16 * nq;  // double-buffered: one barrier per block
    uint2* myout = outt + (size_t)warp * 4 * nq;
    auto emit = [&](int q, int m, uint32_t hi, uint32_t lo) { myout[m * nq + q] = make_uint2(hi, lo); };
    const uint32_t und = buf == 0 ? encode_group_v2<SM4, LPART, NIT, 0u>(ra, len, emit)
                                  : encode_group_v2<SM4, LPART, NIT, BUF>(ra, len, emit);
    if (lane == 0) undef[g] = und;
    __syncwarp();
    __syncthreads();
    // write the 4 groups' words: per position 32 contiguous bytes
    const int64_t tile = (4 * b) >> 5;
    const int gl0 = (int)((4 * b) & 31);
    uint2* dst = reinterpret_cast<uint2*>(packed);
    for (int t = threadIdx.x; t < 4 * len; t += 128) {
      const int pos = t >> 2, w = t & 3;
      dst[((tile * len + pos) * 32 + gl0 + w)] = outt[((size_t)w * 4 + (pos & 3)) * nq + (pos >> 2)];
    }
  }
}

template <int PMAX, int SM4, bool LPART>
static void launch_tma(const uint8_t* seqs, int64_t nblocks, int len, int stride,
                       uint32_t* packed, uint32_t* undef, cudaStream_t stream) {
  const int nq = (len + 3) >> 2;
  const size_t smem = (size_t)4 * 2 * 32 * PMAX + (size_t)2 * 16 * 8 * nq + 64;
  constexpr int MB = PMAX == 128 ? GK_ENC_MINB : 1;
  constexpr int MB_SPARSE = PMAX == 256 ? GK_ENC_MINB_SPARSE : MB;
  const bool sparse_tail = PMAX == 256 && nq - 32 <= 16;  // NIT = 2, R <= 16 quads
  auto kern = sparse_tail ? encode_tma_kernel<PMAX, SM4, LPART, MB_SPARSE>
                          : encode_tma_kernel<PMAX, SM4, LPART, MB>;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > nblocks) grid = nblocks;
  count_launch();
  kern<<<(unsigned)grid, 128, smem, stream>>>(seqs, nblocks, len, stride, packed, undef);
}

template <int PMAX>
static void dispatch_tma(const uint8_t* seqs, int64_t nblocks, int len, int stride,
                         uint32_t* packed, uint32_t* undef, cudaStream_t stream) {
  const bool lpart = (len & 3) != 0;
  switch (stride & 3) {
    case 0: lpart ? launch_tma<PMAX, 0, true>(seqs, nblocks, len, stride, packed, undef, stream)
                  : launch_tma<PMAX, 0, false>(seqs, nblocks, len, stride, packed, undef, stream); break;
    case 1: lpart ? launch_tma<PMAX, 1, true>(seqs, nblocks, len, stride, packed, undef, stream)
                  : launch_tma<PMAX, 1, false>(seqs, nblocks, len, stride, packed, undef, stream); break;
    case 2: lpart ? launch_tma<PMAX, 2, true>(seqs, nblocks, len, stride, packed, undef, stream)
                  : launch_tma<PMAX, 2, false>(seqs, nblocks, len, stride, packed, undef, stream); break;
    default: lpart ? launch_tma<PMAX, 3, true>(seqs, nblocks, len, stride, packed, undef, stream)
                   : launch_tma<PMAX, 3, false>(seqs, nblocks, len, stride, packed, undef, stream); break;
  }
}

static void launch_generic(const uint8_t* seqs, int64_t n, int len, int64_t stride,
                           uint32_t* packed, uint32_t* undef, int64_t first_group,
                           cudaStream_t stream) {
  const int64_t ngroups = (n + 31) / 32 - first_group;
  if (ngroups <= 0) return;
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
  count_launch();
  if (aligned)
    encode_kernel<true><<<(unsigned)blocks, gpc * 32, smem, stream>>>(seqs, n, len, stride,
                                                                      packed, undef, gpc, first_group);
  else
    encode_kernel<false><<<(unsigned)blocks, gpc * 32, smem, stream>>>(seqs, n, len, stride,
                                                                       packed, undef, gpc, first_group);
}

int launch_encode(const uint8_t* seqs, int64_t n, int len, int64_t stride, uint32_t* packed,
                  uint32_t* undef, cudaStream_t stream) {
  const int64_t ngroups = (n + 31) / 32;
  int64_t first_generic = 0;
  const bool tma_ok = ((reinterpret_cast<uintptr_t>(seqs) & 15u) == 0) && stride <= 512 &&
                      GK_ENCODE_TMA;
  if (tma_ok) {
    // full blocks of 4 groups; a block copies 128*stride bytes, so when stride > len
    // the block holding the last row would read stride-len bytes past the caller's
    // (n-1)*stride+len: that block goes to the generic path, which stops at len
    const int64_t nblocks = stride == len ? n / 128 : (n - 1) / 128;
    if (nblocks > 0) {
      if (stride <= 128) dispatch_tma<128>(seqs, nblocks, len, (int)stride, packed, undef, stream);
      else if (stride <= 256) dispatch_tma<256>(seqs, nblocks, len, (int)stride, packed, undef, stream);
      else dispatch_tma<512>(seqs, nblocks, len, (int)stride, packed, undef, stream);
    }
    first_generic = nblocks * 4;
  }
  launch_generic(seqs, n, len, stride, packed, undef, first_generic, stream);
  const int64_t tile_end = ((ngroups + 31) / 32) * 32;
  if (tile_end > ngroups) {
    const int64_t total = (tile_end - ngroups) * len;
    const int threads = 256;
    const int64_t tb = (total + threads - 1) / threads;
    count_launch();
    encode_tail_kernel<<<(unsigned)(tb < 1024 ? tb : 1024), threads, 0, stream>>>(
        ngroups, tile_end, len, packed, undef);
  }
  return 0;
}

}  // namespace gk
