// gk_kernels.cuh -- internal launch entry points (C++; the C ABI is in gk_api.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef GK_SP_EMAX
#define GK_SP_EMAX 11  // largest e with an all-register single-pass filter instantiation
#endif

namespace gk {

// Process-wide count of kernels launched by the library (gk_launch_count in the
// C ABI): the bench's "gpu_launches" is read from it, not estimated.
void count_launch(int k = 1);

// cudaFuncSetAttribute(f, attr, value) on the current device unless this host
// thread already set that value there (attributes are per device: a thread that
// drives several GPUs sets them on each; repeated calls stay off the host path).
void ensure_func_attr(const void* f, cudaFuncAttribute attr, int value);

int launch_encode(const uint8_t* seqs, int64_t n, int len, int64_t stride, uint32_t* packed,
                  uint32_t* undef, cudaStream_t stream);

int launch_filter(const uint32_t* reads, const uint32_t* refs, const uint32_t* rund,
                  const uint32_t* fund, int64_t n, int len, int e, uint32_t* accept,
                  uint8_t* errc, int flags, cudaStream_t stream);

int launch_filter_sweep(const uint32_t* reads, const uint32_t* refs, const uint32_t* rund,
                        const uint32_t* fund, int64_t n, int len, int emax, uint32_t* accept,
                        uint8_t* errc, int flags, cudaStream_t stream);

int launch_filter_ascii(const uint8_t* reads, const uint8_t* refs, int64_t stride, int64_t n,
                        int len, int e, uint32_t* accept, uint8_t* errc, cudaStream_t stream);

// tile-per-CTA fused ASCII kernels (gk_fused.cu); false = cannot take the call
bool launch_fused(const uint8_t* reads, const uint8_t* refs, int64_t stride, int64_t n, int len,
                  int e, bool sweep, uint32_t* accept, uint8_t* errc, cudaStream_t stream);

size_t compact_workspace_bytes(int64_t n, int rows = 1);
// ibase is added to every written index (chunked host pipelines: absolute indices)
int launch_compact(const uint32_t* bits, int64_t n, uint32_t* idx, uint64_t* n_acc, void* ws,
                   cudaStream_t stream, int rows = 1, int64_t bstride = 0, int64_t istride = 0,
                   uint32_t ibase = 0);

}  // namespace gk
