// gk_encode.cu -- a1: ASCII -> bit-sliced 2-bit planes (+ undefined flags).
//
// every base becomes a 2-bit code (A=00 C=01 G=10 T=11, :49);
// pairs with a base outside the alphabet pass unfiltered (:95), so the encoder
// also flags "undefined" sequences.  The paper encodes one sequence per thread
// into 7 words (:93, :105); here one warp encodes one group of 32 sequences and
// writes the bit-sliced layout of include/gatekeeper.h, in which a 32-bit word
// holds one base position of 32 sequences.
//
// The full blocks of 128 sequences run encode3_kernel (gk_encode3.cuh: per 4
// bytes a SWAR validity test + code-bit extraction, then a 3-stage shuffle
// transpose per 16 positions; about 1.6 ALU + 1.25 FMA instructions per input
// byte); the rest (a partial last block, misaligned input) runs the generic
// encode_kernel (gk_encode_core.cuh, 4x4 byte transposes + bit gathers).
#include "gk_common.cuh"
#include "gk_encode3.cuh"
#include "gk_encode_core.cuh"
#include "gk_kernels.cuh"
#include "gk_tma.cuh"

// minimum resident CTAs per SM asked of ptxas for encode3_kernel (A/B knob)
// span buffers per warp (A/B knob): 2 = double-buffered, 1 = more CTAs per SM
#ifndef GK_ENC3_NBUF
#define GK_ENC3_NBUF 0  // 0: per length class (launch_enc3_t)
#endif
#ifndef GK_ENC3_MINB
#define GK_ENC3_MINB 0  // 0: per length class (launch_enc3_t)
#endif
#ifndef GK_ENC3_PF
#define GK_ENC3_PF 0  // L2 prefetch distance in blocks (A/B knob; 1-2 measured 1.1-1.5x slower)
#endif
#ifndef GK_ENC3_OB
#define GK_ENC3_OB 0  // output staging buffers (0: per length class)
#endif
#ifndef GK_ENC3_VEC
#define GK_ENC3_VEC 1  // copy-out with 16-byte stores (below 241 bp)
#endif
#ifndef GK_ENCODE_TMA
#define GK_ENCODE_TMA 1
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

// TMA encoder (gk_encode3.cuh): full blocks of 4 groups (128 sequences).
// Persistent CTAs of 4 warps; warp w encodes group 4b+w of block b.  Its 32
// rows (one contiguous span of 32*stride bytes) arrive by one cp.async.bulk into
// a per-warp double buffer, the next block's span being prefetched while the
// current one is encoded.  The 4 groups' words are collected in shared memory
// ([plane][position*5 + group]: conflict-free transposed writes; one buffer, so
// that 3 CTAs fit an SM at 250 bp) and leave as full 32-byte sectors (4 groups x
// 8 bytes per position).
// NCH > 0: compile-time number of 16-position chunks (immediate LDS offsets);
// NCH == 0: runtime.  ALN: every row start is 4-byte aligned (stride % 4 == 0).
template <int NCH, int MODE, int MB, int NB, int OB>
__global__ void __launch_bounds__(128, MB) encode3_kernel(const uint8_t* __restrict__ seqs,
                                                         int64_t nblocks, int len, int stride,
                                                         uint32_t bufb, uint32_t P,
                                                         uint32_t* __restrict__ packed,
                                                         uint32_t* __restrict__ undef) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* stage = sm + (size_t)warp * NB * bufb;                              // [NB][bufb]
  uint32_t* outs0 = reinterpret_cast<uint32_t*>(sm + (size_t)4 * NB * bufb);   // [OB][2][P]
  uint64_t* bars = reinterpret_cast<uint64_t*>(outs0 + OB * 2 * P);
  uint64_t* mybar = bars + 2 * warp;
  if (lane == 0) {
    mbar_init(&mybar[0], 1);
    mbar_init(&mybar[1], 1);
    fence_mbar_init();
  }
  __syncwarp();
  enc3::Lane ln;
  ln.init(lane);
  uint32_t roff[4], rsh[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t a = (uint32_t)ln.rows[i] * (uint32_t)stride + 4u * (uint32_t)ln.cw;
    roff[i] = MODE == 0 ? a : (a & ~3u);
    rsh[i] = (a & 3u) * 8u;
  }
  const int s2 = (int)(rsh[0] >> 3);  // MODE 2: the lane's rows start 0 or 2 bytes into a word
  const uint32_t span = 32u * (uint32_t)stride;

  int64_t b = blockIdx.x;
  if (b >= nblocks) return;
  if (lane == 0) {
    mbar_arrive_expect_tx(&mybar[0], span);
    tma_load_1d(stage, seqs + (4 * b + warp) * (int64_t)span, span, &mybar[0]);
  }
  for (int it = 0; b < nblocks; ++it, b += gridDim.x) {
    const int buf = NB == 2 ? (it & 1) : 0;
    const int64_t bn = b + gridDim.x;
    if (GK_ENC3_PF > 0 && lane == 0) {  // L2 prefetch of the span GK_ENC3_PF blocks past bn
      const int64_t bp = bn + (int64_t)GK_ENC3_PF * gridDim.x;
      if (bp < nblocks)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                         seqs + (4 * bp + warp) * (int64_t)span),
                     "r"(span)
                     : "memory");
    }
    if (NB == 2 && lane == 0 && bn < nblocks) {
      fence_proxy_async();
      mbar_arrive_expect_tx(&mybar[buf ^ 1], span);
      tma_load_1d(stage + (buf ^ 1) * bufb, seqs + (4 * bn + warp) * (int64_t)span, span,
                  &mybar[buf ^ 1]);
    }
    mbar_wait(&mybar[buf], NB == 2 ? ((uint32_t)(it >> 1) & 1u) : ((uint32_t)it & 1u));
    const uint8_t* sbuf = stage + buf * bufb;
    // OB = 1 output staging buffer (smem for more CTAs per SM): the previous block's
    // copy-out must be complete before it is overwritten; OB = 2: the barrier before
    // the copy-out of block it+1 already orders the copy-out of block it before the
    // encode of block it+2 into the same buffer
    uint32_t* outs = outs0 + (OB == 2 ? (size_t)(it & 1) * 2 * P : 0);
    if (OB == 1 && it > 0) __syncthreads();
    const uint32_t und = enc3_group<NCH, MODE>(sbuf, roff, rsh, s2, len, ln, outs, P, warp);
    if (lane == 0) undef[4 * b + warp] = und;
    if (NB == 1) {  // single buffer: the next span lands during the copy-out below
      __syncwarp();
      if (lane == 0 && bn < nblocks) {
        fence_proxy_async();
        mbar_arrive_expect_tx(&mybar[0], span);
        tma_load_1d(stage, seqs + (4 * bn + warp) * (int64_t)span, span, &mybar[0]);
      }
    }
    __syncthreads();
    // write the 4 groups' words: per position 32 contiguous bytes
    const int64_t tile = (4 * b) >> 5;
    const int gl0 = (int)((4 * b) & 31);
    // 16-byte stores (two groups, both planes, per thread and step): +2-3% at 100 / 150
    // bp, -1.4% at 250 bp (profiles/r02_ab_encoder_vec.jsonl), so not at 250 bp
    if (GK_ENC3_VEC && NCH != 16) {
      uint4* dst4 = reinterpret_cast<uint4*>(packed) + ((tile * len) * 32 + gl0) / 2;
      for (int t = threadIdx.x; t < 2 * len; t += 128) {
        const int pos = t >> 1, w = (t & 1) * 2;
        const uint32_t* o = outs + pos * 5 + w;
        dst4[pos * 16 + (w >> 1)] = make_uint4(o[0], o[P], o[1], o[P + 1]);
      }
    } else {
      uint2* dst = reinterpret_cast<uint2*>(packed);
      for (int t = threadIdx.x; t < 4 * len; t += 128) {
        const int pos = t >> 2, w = t & 3;
        dst[((tile * len + pos) * 32 + gl0 + w)] =
            make_uint2(outs[pos * 5 + w], outs[P + pos * 5 + w]);
      }
    }
  }
}

struct Enc3Cfg {
  uint32_t bufb, P;
  size_t smem;
};

static Enc3Cfg enc3_cfg(int len, int stride, int nbuf, int nob) {
  Enc3Cfg c;
  c.bufb = ((uint32_t)(32 * stride + 32) + 127u) & ~127u;
  uint32_t p = (uint32_t)(5 * len);
  p = (p + 31u) & ~31u;
  c.P = p + 16u;  // P = 16 (mod 32): the two planes' transposed writes hit disjoint banks
  c.smem = (size_t)4 * nbuf * c.bufb + (size_t)nob * 2 * c.P * 4 + 8 * 8;
  return c;
}

template <int NCH, int MODE>
static void launch_enc3_t(const uint8_t* seqs, int64_t nblocks, int len, int stride,
                          uint32_t* packed, uint32_t* undef, cudaStream_t stream) {
  // registers vs resident CTAs and span buffers per warp, measured per length class
  // (profiles/r02_ab_encoder_minb.jsonl, r02_ab_encoder_nbuf.jsonl): 100 bp double-
  // buffered at 8 CTAs/SM (64 regs; 1.51 -> 1.39 ms per 2 x 30M); 150 bp single-
  // buffered at 7 (2.40 -> 2.25 ms); 250 bp single-buffered at 5 (3.95 -> 3.51 ms)
  constexpr int MB = GK_ENC3_MINB > 0 ? GK_ENC3_MINB : (NCH == 7 ? 8 : (NCH == 10 ? 7 : (NCH == 16 ? 5 : 1)));
  constexpr int NB = GK_ENC3_NBUF > 0 ? GK_ENC3_NBUF : (NCH == 7 || NCH == 0 ? 2 : 1);
  // 150 bp: a second output staging buffer still fits 7 CTAs/SM and saves one CTA
  // barrier per block (profiles/r02_ab_encoder_ob.jsonl)
  constexpr int OB = GK_ENC3_OB > 0 ? GK_ENC3_OB : (NCH == 10 ? 2 : 1);
  const Enc3Cfg c = enc3_cfg(len, stride, NB, OB);
  auto kern = encode3_kernel<NCH, MODE, MB, NB, OB>;
  // launch configuration cached per (device, smem): the attribute and occupancy
  // queries are host round trips, kept off the per-call path
  static thread_local int cached_dev = -1, cached_grid = 0;
  static thread_local size_t cached_smem = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cached_dev || c.smem != cached_smem) {
    if (c.smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem);
    int sms = 148, per_sm = 1;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, c.smem);
    cached_grid = sms * (per_sm < 1 ? 1 : per_sm);
    cached_dev = dev;
    cached_smem = c.smem;
  }
  int64_t grid = cached_grid;
  if (grid > nblocks) grid = nblocks;
  count_launch();
  kern<<<(unsigned)grid, 128, c.smem, stream>>>(seqs, nblocks, len, stride, c.bufb, c.P, packed,
                                                undef);
}

static void launch_enc3(const uint8_t* seqs, int64_t nblocks, int len, int stride,
                        uint32_t* packed, uint32_t* undef, cudaStream_t stream) {
  const int nch = (len + 15) >> 4;
  // MODE 0: rows 4-byte aligned; 2: stride = 2 (mod 4) (one load per word + merged-word
  // realignment); 1: any other stride (two loads + funnel shift per word)
  const int mode = (stride & 3) == 0 ? 0 : ((stride & 3) == 2 ? 2 : 1);
#define GK_ENC3(N)                                                                        \
  if (nch == N) {                                                                         \
    if (mode == 0) launch_enc3_t<N, 0>(seqs, nblocks, len, stride, packed, undef, stream); \
    else if (mode == 2) launch_enc3_t<N, 2>(seqs, nblocks, len, stride, packed, undef, stream); \
    else launch_enc3_t<N, 1>(seqs, nblocks, len, stride, packed, undef, stream);          \
    return;                                                                               \
  }
  GK_ENC3(7)   // 97..112 bp (100 bp)
  GK_ENC3(10)  // 145..160 bp (150 bp)
  GK_ENC3(16)  // 241..256 bp (250 bp)
#undef GK_ENC3
  if (mode == 0) launch_enc3_t<0, 0>(seqs, nblocks, len, stride, packed, undef, stream);
  else if (mode == 2) launch_enc3_t<0, 2>(seqs, nblocks, len, stride, packed, undef, stream);
  else launch_enc3_t<0, 1>(seqs, nblocks, len, stride, packed, undef, stream);
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
    ensure_func_attr((const void*)encode_kernel<true>,
                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ensure_func_attr((const void*)encode_kernel<false>,
                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
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
    if (nblocks > 0) launch_enc3(seqs, nblocks, len, (int)stride, packed, undef, stream);
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
