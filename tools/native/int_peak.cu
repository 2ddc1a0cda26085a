// int_peak.cu -- measured integer-pipe peaks of this B200 (the denominator of the
// filter's ALU roofline; SURVEY.md 8(d) "must be microbenchmarked on the box").
//
// Each kernel runs at full occupancy (148 SMs x 2048 threads); every thread
// keeps NCH independent dependency chains of one instruction type (so the
// 4-cycle pipe latency is hidden) in a fully unrolled loop, and stores the
// chains at the end so nothing is dead.  The instruction is forced with inline
// PTX and checked in the SASS (tools/int_peak_sass.txt):
//   lop3   LOP3.LUT     (alu pipe)       the filter's mask / counter logic
//   iadd3  IADD3        (alu pipe)
//   shf    SHF.L.W      (alu pipe)
//   prmt   PRMT         (alu pipe)
//   imad   IMAD         (fma pipe)
//   mix    LOP3 + IMAD interleaved 1:1 (both pipes issuing)
// Result: thread-instructions per second (lane-ops/s) for each.
#include <cuda_runtime.h>
#include <stdint.h>

#define NCH 8
#define ITERS 4096

template <int OP>
__device__ __forceinline__ uint32_t op(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  if (OP == 0) asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  if (OP == 1) asm volatile("{.reg .u32 t; add.u32 t, %1, %2; add.u32 %0, t, %3;}"
                            : "=r"(d) : "r"(a), "r"(b), "r"(c));
  if (OP == 2) asm volatile("shf.l.wrap.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  if (OP == 3) asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  if (OP == 4) asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

template <int OP>
__global__ void __launch_bounds__(256) peak_kernel(uint32_t* out, uint32_t seed) {
  uint32_t x[NCH];
  const uint32_t t = threadIdx.x + blockIdx.x * blockDim.x;
#pragma unroll
  for (int i = 0; i < NCH; ++i) x[i] = t * 0x9E3779B9u + i * 0x7F4A7C15u + seed;
  const uint32_t b = seed | 1u, c = seed * 3u + 0x1234u;
#pragma unroll 1
  for (int it = 0; it < ITERS; it += 16) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int i = 0; i < NCH; ++i) {
        if (OP == 5) {
          x[i] = (i & 1) ? op<4>(x[i], b, c) : op<0>(x[i], b, c);
        } else {
          x[i] = op<OP>(x[i], b, c);
        }
      }
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) s ^= x[i];
  out[t] = s;
}

template <int OP>
static double run(uint32_t* out, int sms, int reps) {
  const int threads = 256, blocks = sms * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  peak_kernel<OP><<<blocks, threads>>>(out, 1u);  // warm-up
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) peak_kernel<OP><<<blocks, threads>>>(out, (uint32_t)r);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double ops = (double)blocks * threads * ITERS * NCH * reps;
  return ops / (ms * 1e-3);
}

// out_ops[6]: thread-instructions/s for lop3, iadd3, shf, prmt, imad, mix (lop3+imad).
// Returns 0, or -1 on a CUDA error.
extern "C" int ip_measure(double* out_ops, int reps) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint32_t* out = nullptr;
  if (cudaMalloc(&out, (size_t)sms * 8 * 256 * 4) != cudaSuccess) return -1;
  out_ops[0] = run<0>(out, sms, reps);
  out_ops[1] = run<1>(out, sms, reps);
  out_ops[2] = run<2>(out, sms, reps);
  out_ops[3] = run<3>(out, sms, reps);
  out_ops[4] = run<4>(out, sms, reps);
  out_ops[5] = run<5>(out, sms, reps);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
