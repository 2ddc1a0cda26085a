// gk_filter_bt2.cu -- a2..a6 for any e, block-transposed, with a compact rolled
// k loop: the kernels behind gk_filter for e above the all-register single pass
// and behind gk_filter_sweep (every e <= e_max in one pass).
//
// Loop order: per block of B positions [ib, ib+B) of a
// tile, the Hamming mask, then for k = 1..e the deletion and insertion masks of
// the block (W = B+4 cells: the block plus the 2-base amendment halo on each
// side), ANDed into the block's B words of F:
//
//   H   x[c] = R[j] != Q[j]          D_k  x[c] = R[j] != Q[j-k]
//   I_k x[c] = R[j] != Q[j+k]        (j = ib-2+c; Q = read, R = reference)
//
// What differs from round 1's gk_filter_bt.cu (removed in round 2; 13-step unrolled register ring +
// an out-of-line per-k counter): the two read windows slide by plain register
// moves inside a ROLLED k loop -- the moves issue on the FMA pipe (IMAD.MOV)
// while the ALU pipe (LOP3) is the bottleneck, so they are nearly free, and the
// loop body (~200 instructions) fits the 6 KB L0 instruction cache; the per-k
// run counter of the sweep is inline.  The new word of each window is loaded LA
// steps ahead through a small register queue.  ncu of the round-1 kernel:
// stall_no_instruction 20% of samples, CALL/RET hot; LOP3 1.29x the model.
//
// Blocks whose steps would touch a vacated source, a vacated position or a
// target outside [0, len) run those steps CHECKED (rolled, validity words per
// cell, readings R2 / R4 / R13).
#include "gk_bt2.cuh"
#include "gk_common.cuh"
#include "gk_filter_core.cuh"
#include "gk_kernels.cuh"

namespace gk {


#ifndef GK_BT2_B
#define GK_BT2_B 8      // positions per block of the sweep kernel
#endif
#ifndef GK_BT2_B_E
#define GK_BT2_B_E 16   // positions per block of the per-e kernel (2 CTAs/SM, 252 regs)
#endif
#ifndef GK_BT2_MINB
#define GK_BT2_MINB 2   // resident CTAs per SM asked of ptxas (per-e kernel)
#endif
#ifndef GK_BT2_E_WARPS
#define GK_BT2_E_WARPS 4  // warps (tiles) per CTA of the per-e kernel
#endif
#ifndef GK_BT2_SWEEP_MINB
#define GK_BT2_SWEEP_MINB 6
#endif
#ifndef GK_BT2_SWEEP_B16_LEN
#define GK_BT2_SWEEP_B16_LEN 200  // reads at least this long take 16-position sweep blocks
#endif

template <int B>
__global__ void __launch_bounds__(GK_BT2_E_WARPS * 32, GK_BT2_MINB) filter_bt2_kernel(
    const uint2* __restrict__ reads, const uint2* __restrict__ refs,
    const uint32_t* __restrict__ rund, const uint32_t* __restrict__ fund, int64_t n, int len, int e,
    uint32_t* __restrict__ accept, uint8_t* __restrict__ errc, int edge_fix) {
  const int lane = threadIdx.x & 31;
  const int64_t tile = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t g = tile * 32 + lane;
  if (tile * 1024 >= n) return;
  const uint2* q = reads + tile * (int64_t)len * 32 + lane;
  const uint2* r = refs + tile * (int64_t)len * 32 + lane;
  CsaCounter cA, cF;
  cA.clear();
  cF.clear();
  bt2::Win<B> R;
  bt2::load_r0<B, bt2::GMem>(r, len, R);
#pragma unroll 1
  for (int ib = 0; ib < len; ib += B)
    bt2::block<B, GK_BT2_LA_E, bt2::GMem>(q, r, R, ib, len, e, edge_fix, cA, cF, bt2::NoHook{});
  uint32_t a[8], f[8];
  cA.planes(a);
  cF.planes(f);
  if (g * 32 < n) finish_group(a, f, e, __ldg(rund + g) | __ldg(fund + g), g, n, accept, errc);
}

#ifndef GK_BT2_SWEEP_WARPS
#define GK_BT2_SWEEP_WARPS 2
#endif
constexpr int BT2_SWEEP_WARPS = GK_BT2_SWEEP_WARPS;

template <int B, int NP, int MINB>
__global__ void __launch_bounds__(BT2_SWEEP_WARPS * 32, MINB) filter_bt2_sweep_kernel(
    const uint2* __restrict__ reads, const uint2* __restrict__ refs,
    const uint32_t* __restrict__ rund, const uint32_t* __restrict__ fund, int64_t n, int len,
    int emax, uint32_t* __restrict__ accept, uint8_t* __restrict__ errc, int edge_fix) {
  extern __shared__ uint32_t sm_sweep2[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t tile = (int64_t)blockIdx.x * BT2_SWEEP_WARPS + warp;
  const int64_t g = tile * 32 + lane;
  if (tile * 1024 >= n) return;
  uint32_t* mine = sm_sweep2 + (size_t)warp * emax * NP * 32 + lane;
  for (int j = 0; j < emax * NP; ++j) mine[j * 32] = 0u;
  const uint2* q = reads + tile * (int64_t)len * 32 + lane;
  const uint2* r = refs + tile * (int64_t)len * 32 + lane;
  CsaCounter cA, cF;
  cA.clear();
  cF.clear();
  bt2::Win<B> R;
  bt2::load_r0<B, bt2::GMem>(r, len, R);
  const bt2::SweepHook<NP> hook{mine};
#pragma unroll 1
  for (int ib = 0; ib < len; ib += B)
    bt2::block<B, GK_BT2_LA, bt2::GMem>(q, r, R, ib, len, emax, edge_fix, cA, cF, hook);
  if (g * 32 >= n) return;
  uint32_t a[8], f[8];
  cA.planes(a);
  const uint32_t und = __ldg(rund + g) | __ldg(fund + g);
  const int64_t words = (n + 31) / 32;
#pragma unroll 1
  for (int e = 0; e <= emax; ++e) {
    if (e == 0) {
#pragma unroll
      for (int b = 0; b < 8; ++b) f[b] = a[b];
    } else {
      const uint32_t* p = mine + (e - 1) * NP * 32;
#pragma unroll
      for (int b = 0; b < 8; ++b) f[b] = b < NP ? p[b * 32] : 0u;
    }
    finish_group(a, f, e, und, g, n, accept + e * words, errc ? errc + e * n : nullptr);
  }
}

void launch_bt2(const uint2* reads, const uint2* refs, const uint32_t* rund, const uint32_t* fund,
                int64_t n, int len, int e, uint32_t* accept, uint8_t* errc, int edge_fix,
                cudaStream_t stream) {
  constexpr int B = GK_BT2_B_E;
  const int64_t tiles = (n + 1023) / 1024;
  const int warps = GK_BT2_E_WARPS;
  const int64_t blocks = (tiles + warps - 1) / warps;
  ensure_func_attr((const void*)filter_bt2_kernel<B>,
                   cudaFuncAttributePreferredSharedMemoryCarveout, 0);  // all L1
  count_launch();
  filter_bt2_kernel<B><<<(unsigned)blocks, warps * 32, 0, stream>>>(reads, refs, rund, fund, n,
                                                                    len, e, accept, errc, edge_fix);
}

template <int B, int NP, int MINB>
static void launch_bt2_sweep_np(const uint2* reads, const uint2* refs, const uint32_t* rund,
                                const uint32_t* fund, int64_t n, int len, int emax,
                                uint32_t* accept, uint8_t* errc, int edge_fix,
                                cudaStream_t stream) {
  const int64_t tiles = (n + 1023) / 1024;
  const int64_t blocks = (tiles + BT2_SWEEP_WARPS - 1) / BT2_SWEEP_WARPS;
  const size_t smem = (size_t)BT2_SWEEP_WARPS * emax * NP * 32 * 4;
  if (smem > 48 * 1024)
    ensure_func_attr((const void*)filter_bt2_sweep_kernel<B, NP, MINB>,
                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  count_launch();
  filter_bt2_sweep_kernel<B, NP, MINB><<<(unsigned)blocks, BT2_SWEEP_WARPS * 32, smem, stream>>>(
      reads, refs, rund, fund, n, len, emax, accept, errc, edge_fix);
}

void launch_bt2_sweep(const uint2* reads, const uint2* refs, const uint32_t* rund,
                      const uint32_t* fund, int64_t n, int len, int emax, uint32_t* accept,
                      uint8_t* errc, int edge_fix, cudaStream_t stream) {
  // counter planes: enough bits for the largest count, 2 * ceil(len / 4) (R6, R7).
  // Block size by read length (profiles/r02_ab_sweep_block.jsonl, 30M pairs): 8-position
  // blocks at 6 CTAs/SM (157 regs, 12 warps) are fastest at 100 / 150 bp; 16-position
  // blocks (1.1x instead of 1.2x the model's mismatch work; 255 regs, 8 warps) at
  // 250 bp (7.17 -> 6.65 ms at e_max = 25).
  const int maxc = 2 * ((len + 3) / 4);
  if (len >= GK_BT2_SWEEP_B16_LEN) {
    if (maxc < 128)
      launch_bt2_sweep_np<16, 7, 4>(reads, refs, rund, fund, n, len, emax, accept, errc, edge_fix,
                                    stream);
    else
      launch_bt2_sweep_np<16, 8, 4>(reads, refs, rund, fund, n, len, emax, accept, errc, edge_fix,
                                    stream);
  } else if (maxc < 64) {
    launch_bt2_sweep_np<GK_BT2_B, 6, GK_BT2_SWEEP_MINB>(reads, refs, rund, fund, n, len, emax,
                                                        accept, errc, edge_fix, stream);
  } else if (maxc < 128) {
    launch_bt2_sweep_np<GK_BT2_B, 7, GK_BT2_SWEEP_MINB>(reads, refs, rund, fund, n, len, emax,
                                                        accept, errc, edge_fix, stream);
  } else {
    launch_bt2_sweep_np<GK_BT2_B, 8, GK_BT2_SWEEP_MINB>(reads, refs, rund, fund, n, len, emax,
                                                        accept, errc, edge_fix, stream);
  }
}

}  // namespace gk
