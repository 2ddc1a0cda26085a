// gk_filter_q_impl.cuh -- the large-e kernel (filter_spq_kernel<E>, a warp pair per
// tile, see gk_filter_q.cuh) and its launcher; instantiated in gk_filter_q*.cu.
#pragma once
#include "gk_filter_q.cuh"
#include "gk_kernels.cuh"

namespace gk {

constexpr int SPQ_PAIRS = 2;  // tiles per CTA (2 warps each)

template <int E>
__global__ void __launch_bounds__(SPQ_PAIRS * 64) filter_spq_kernel(
    const uint2* __restrict__ reads, const uint2* __restrict__ refs,
    const uint32_t* __restrict__ rund, const uint32_t* __restrict__ fund, int64_t n, int len,
    uint32_t* __restrict__ accept, uint8_t* __restrict__ errc) {
  constexpr int KA = E / 2;
  extern __shared__ __align__(128) uint8_t sm_q[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pair = warp >> 1, role = warp & 1;
  const int64_t tile = (int64_t)blockIdx.x * SPQ_PAIRS + pair;
  uint8_t* mine = sm_q + (size_t)pair * SPQ_PAIR_SMEM;
  QRing ring;
  ring.gq = reads + tile * (int64_t)len * 32;
  ring.gr = refs + tile * (int64_t)len * 32;
  ring.qptr = reinterpret_cast<uint2*>(mine);
  ring.rptr = reinterpret_cast<uint2*>(mine + QR_BYTES);
  uint32_t* xbuf = reinterpret_cast<uint32_t*>(mine + QR_BYTES + RR_BYTES);
  ring.qsm = smem_u32(mine) + 8u * lane;
  ring.rsm = smem_u32(mine + QR_BYTES) + 8u * lane;
  ring.bq = reinterpret_cast<uint64_t*>(mine + QR_BYTES + RR_BYTES + XB_BYTES);
  ring.br = ring.bq + QR_SLOTS;
  ring.len = len;
  ring.nblk = (len + 7) >> 3;
  ring.lane = lane;
  ring.reset();
  if (role == 0 && lane == 0) {
    for (int b = 0; b < QR_SLOTS; ++b) mbar_init(&ring.bq[b], 1);
    for (int b = 0; b < RR_SLOTS; ++b) mbar_init(&ring.br[b], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tile * 1024 >= n) return;  // both warps of the pair leave together
  if (role == 0 && lane == 0) ring.start();
  CsaCounter cA, cF;
  run_pair<E, KA>(ring, role, len, xbuf, 1 + pair, cA, cF);
  if (role == 0) {
    const int64_t g = tile * 32 + lane;
    uint32_t a[8], f[8];
    cA.planes(a);
    cF.planes(f);
    if (g * 32 < n) finish_group(a, f, E, __ldg(rund + g) | __ldg(fund + g), g, n, accept, errc);
  }
}

template <int E>
void launch_spq(const uint2* reads, const uint2* refs, const uint32_t* rund, const uint32_t* fund,
                int64_t n, int len, uint32_t* accept, uint8_t* errc, cudaStream_t stream) {
  const int64_t tiles = (n + 1023) / 1024;
  const int64_t blocks = (tiles + SPQ_PAIRS - 1) / SPQ_PAIRS;
  const size_t smem = (size_t)SPQ_PAIRS * SPQ_PAIR_SMEM;
  cudaFuncSetAttribute(filter_spq_kernel<E>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  filter_spq_kernel<E><<<(unsigned)blocks, SPQ_PAIRS * 64, smem, stream>>>(
      reads, refs, rund, fund, n, len, accept, errc);
}

}  // namespace gk
