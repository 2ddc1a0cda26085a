// gk_filter.cu -- a2..a6: the filtration of packed pairs (gk_filter).
//
// Launch geometry: one warp per tile of 1024 pairs, one lane per group of 32
// pairs (lane g reads the words of group g: 32 lanes x 8 bytes = 256 contiguous
// bytes per base position, so every load instruction of the warp is one fully
// used 256-byte segment).  The paper runs one filtration per thread (:79); here
// one thread runs 32 filtrations at once, one per bit of every word.
//
// Two kernels:
//   * filter_sp<E>  (e == E <= GK_SP_EMAX): single pass, everything in registers
//     (gk_filter_core.cuh).  Positions are split into checked head/tail steps and
//     an unchecked middle that is unrolled by 8 (static carry-save count tree).
//   * filter_generic (any e): mask-major, F kept in shared memory, one mask at a
//     time; the fallback for e > GK_SP_EMAX.
#include "gk_common.cuh"
#include "gk_filter_core.cuh"
#include "gk_kernels.cuh"

// resident CTAs per SM asked of ptxas for sp<6>, sp<7> (3: 168 registers instead of
// 172-186, 12 warps instead of 8; 150 bp e=7 0.82 -> 0.78 ms, 100 bp e=6 0.51 -> 0.47 ms
// per 30M pairs, profiles/r02_ab_sp_minb.jsonl) and sp<4>, sp<5> (A/B knob)
#ifndef GK_SP_MINB67
#define GK_SP_MINB67 3
#endif
#ifndef GK_SP_MINB45
#define GK_SP_MINB45 1
#endif
#ifndef GK_FILTER_RING
#define GK_FILTER_RING 1
#endif

namespace gk {

template <int E>
__global__ void __launch_bounds__(128, (E >= 6 && E <= 7) ? GK_SP_MINB67 : ((E >= 4 && E <= 5) ? GK_SP_MINB45 : 1)) filter_sp_kernel(
    const uint2* __restrict__ reads, const uint2* __restrict__ refs,
    const uint32_t* __restrict__ rund, const uint32_t* __restrict__ fund, int64_t n, int len,
    uint32_t* __restrict__ accept, uint8_t* __restrict__ errc) {
  const int lane = threadIdx.x & 31;
  const int64_t tile = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t g = tile * 32 + lane;
  if (tile * 1024 >= n) return;  // whole warp leaves together (warp-level TMA ring)
#if GK_FILTER_RING
  extern __shared__ __align__(128) uint8_t sm_ring[];
  const int warp = threadIdx.x >> 5;
  uint8_t* mine = sm_ring + (size_t)warp * (2 * 4 * 8 * 32 * 8 + 64);
  RingSrc src;
  src.gq = reads + tile * (int64_t)len * 32;
  src.gr = refs + tile * (int64_t)len * 32;
  src.sq = reinterpret_cast<uint2*>(mine);
  src.sr = src.sq + 4 * 8 * 32;
  src.bq = reinterpret_cast<uint64_t*>(mine + 2 * 4 * 8 * 32 * 8);
  src.br = src.bq + 4;
  src.len = len;
  src.nblk = (len + 7) >> 3;
  src.lane = lane;
  if (lane == 0) {
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      mbar_init(&src.bq[b], 1);
      mbar_init(&src.br[b], 1);
    }
    fence_mbar_init();
  }
  __syncwarp();
  src.start();
#else
  GlobalGroupSrc src;
  src.q = reads + tile * (int64_t)len * 32 + lane;
  src.r = refs + tile * (int64_t)len * 32 + lane;
  src.len = len;
#endif

  SinglePass<E> sp;
  run_range<E, true>(sp, src, len, 0, len);
  uint32_t cA[8], cF[8];
  sp.cA.planes(cA);
  sp.cF.planes(cF);
  if (g * 32 < n) finish_group(cA, cF, E, __ldg(rund + g) | __ldg(fund + g), g, n, accept, errc);
}

// ---------------------------------------------------------------------------
// Generic fallback: mask-major, F[pos][lane] in shared memory.
__global__ void __launch_bounds__(128) filter_generic_kernel(
    const uint2* __restrict__ reads, const uint2* __restrict__ refs,
    const uint32_t* __restrict__ rund, const uint32_t* __restrict__ fund, int64_t n, int len,
    int e, uint32_t* __restrict__ accept, uint8_t* __restrict__ errc, int edge_fix) {
  extern __shared__ uint32_t sm_f[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t tile = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  const int64_t g = tile * 32 + lane;
  if (g * 32 >= n) return;
  GlobalGroupSrc src;
  src.q = reads + tile * (int64_t)len * 32 + lane;
  src.r = refs + tile * (int64_t)len * 32 + lane;
  src.len = len;
  const uint32_t undef = __ldg(rund + g) | __ldg(fund + g);
  uint32_t cA[8], cF[8];
  generic_group(src, len, e, undef, sm_f + (size_t)warp * len * 32 + lane, 32, cA, cF,
                edge_fix != 0);
  finish_group(cA, cF, e, undef, g, n, accept, errc);
}

template <int E>
static void launch_sp(const uint2* reads, const uint2* refs, const uint32_t* rund,
                      const uint32_t* fund, int64_t n, int len, uint32_t* accept, uint8_t* errc,
                      cudaStream_t stream) {
  const int64_t tiles = (n + 1023) / 1024;
  const int warps = 4;
  const int64_t blocks = (tiles + warps - 1) / warps;
  const size_t smem = GK_FILTER_RING ? (size_t)warps * (2 * 4 * 8 * 32 * 8 + 64) : 0;
  if (smem > 48 * 1024)
    ensure_func_attr((const void*)filter_sp_kernel<E>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                     (int)smem);
  count_launch();
  filter_sp_kernel<E><<<(unsigned)blocks, warps * 32, smem, stream>>>(reads, refs, rund, fund, n,
                                                                       len, accept, errc);
}

template <int E>
static bool dispatch_sp(int e, const uint2* reads, const uint2* refs, const uint32_t* rund,
                        const uint32_t* fund, int64_t n, int len, uint32_t* accept,
                        uint8_t* errc, cudaStream_t stream) {
  if (e == E) {
    launch_sp<E>(reads, refs, rund, fund, n, len, accept, errc, stream);
    return true;
  }
  if constexpr (E > 0) return dispatch_sp<E - 1>(e, reads, refs, rund, fund, n, len, accept, errc, stream);
  return false;
}

#ifndef GK_SP2
#define GK_SP2 1
#endif
bool launch_sp2(const uint2* reads, const uint2* refs, const uint32_t* rund, const uint32_t* fund,
                int64_t n, int len, int e, uint32_t* accept, uint8_t* errc, cudaStream_t stream);
void launch_bt2(const uint2* reads, const uint2* refs, const uint32_t* rund, const uint32_t* fund,
                int64_t n, int len, int e, uint32_t* accept, uint8_t* errc, int edge_fix,
                cudaStream_t stream);
int launch_filter(const uint32_t* reads, const uint32_t* refs, const uint32_t* rund,
                  const uint32_t* fund, int64_t n, int len, int e, uint32_t* accept,
                  uint8_t* errc, int flags, cudaStream_t stream) {
  const int force_generic = flags & 1;  // GK_FLAG_GENERIC
  const int edge_fix = (flags & 2) ? 0 : 1;  // GK_FLAG_NO_EDGE_FIX
  const uint2* r2 = reinterpret_cast<const uint2*>(reads);
  const uint2* f2 = reinterpret_cast<const uint2*>(refs);
  // e <= GK_SP_EMAX: the all-register single pass; above it (and for the
  // original GateKeeper, or on request) the block-transposed kernel, which
  // measured 1.3-1.7x faster than the earlier warp-pair split at e = 12..25
  // (profiles/r01_cmp_bt.jsonl)
  if (!force_generic && ((flags & 4) || !edge_fix || e > GK_SP_EMAX)) {
    // e just above the all-register single pass: the warp-pair split single pass
    // (gk_filter_sp2.cu), else the block-transposed kernel (any e, any flags)
    if (GK_SP2 && !(flags & 4) && edge_fix &&
        launch_sp2(r2, f2, rund, fund, n, len, e, accept, errc, stream))
      return 0;
    launch_bt2(r2, f2, rund, fund, n, len, e, accept, errc, edge_fix, stream);
    return 0;
  }
  if (!force_generic &&
      dispatch_sp<GK_SP_EMAX>(e, r2, f2, rund, fund, n, len, accept, errc, stream))
    return 0;
  const int64_t tiles = (n + 1023) / 1024;
  int warps = (int)(48 * 1024 / (len * 32 * 4));
  if (warps > 4) warps = 4;
  if (warps < 1) warps = 1;
  const size_t smem = (size_t)warps * len * 32 * 4;
  if (smem > 48 * 1024)
    ensure_func_attr((const void*)filter_generic_kernel,
                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t blocks = (tiles + warps - 1) / warps;
  count_launch();
  filter_generic_kernel<<<(unsigned)blocks, warps * 32, smem, stream>>>(r2, f2, rund, fund, n,
                                                                        len, e, accept, errc,
                                                                        edge_fix);
  return 0;
}

void launch_bt2_sweep(const uint2* reads, const uint2* refs, const uint32_t* rund,
                      const uint32_t* fund, int64_t n, int len, int emax, uint32_t* accept,
                      uint8_t* errc, int edge_fix, cudaStream_t stream);

int launch_filter_sweep(const uint32_t* reads, const uint32_t* refs, const uint32_t* rund,
                        const uint32_t* fund, int64_t n, int len, int emax, uint32_t* accept,
                        uint8_t* errc, int flags, cudaStream_t stream) {
  // the one-pass kernel keeps emax counters of up to 8 planes per warp in shared
  // memory (2 warps per CTA): beyond ~100 thresholds they no longer fit, and the
  // rows are produced by one gk_filter launch per e instead (same results).  The
  // cut-off is by capacity, not occupancy, on purpose: near it only 1-2 CTAs (2-4
  // warps) fit an SM, but the per-e fallback evaluates sum_e (2e+1) = (e_max+1)^2
  // mask passes instead of 2 e_max + 1 (26x more at e_max = 50), which no
  // occupancy gain can make up
  const int maxc = 2 * ((len + 3) / 4);
  const int np = maxc < 64 ? 6 : (maxc < 128 ? 7 : 8);
  const size_t smem = (size_t)2 * emax * np * 32 * 4;
  if (smem <= 200 * 1024) {
    launch_bt2_sweep(
        reinterpret_cast<const uint2*>(reads), reinterpret_cast<const uint2*>(refs), rund, fund, n,
        len, emax, accept, errc, (flags & 2) ? 0 : 1, stream);
    return 0;
  }
  const int64_t words = (n + 31) / 32;
  for (int e = 0; e <= emax; ++e)
    launch_filter(reads, refs, rund, fund, n, len, e, accept + e * words,
                  errc ? errc + e * n : nullptr, flags & 2, stream);
  return 0;
}

}  // namespace gk
