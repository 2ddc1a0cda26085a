// gk_filter_ascii.cu -- dispatch of the fused ASCII filter (a1..a6): the
// tile-per-CTA kernels of gk_fused.cu, else the generic fallback of
// gk_filter_ascii_impl.cuh (instantiated in gk_filter_ascii_p*.cu).
#include "gk_kernels.cuh"
#include <cuda_runtime.h>
#include <stdint.h>

namespace gk {

template <int E>
void launch_ascii_all(const uint8_t* reads, const uint8_t* refs, int64_t stride, int64_t n,
                      int len, int e, uint32_t* accept, uint8_t* errc, cudaStream_t stream);

template <int E>
static bool dispatch_ascii(int e, const uint8_t* reads, const uint8_t* refs, int64_t stride,
                           int64_t n, int len, uint32_t* accept, uint8_t* errc,
                           cudaStream_t stream) {
  if (e == E) {
    launch_ascii_all<E>(reads, refs, stride, n, len, e, accept, errc, stream);
    return true;
  }
  if constexpr (E > 0) return dispatch_ascii<E - 1>(e, reads, refs, stride, n, len, accept, errc, stream);
  return false;
}

bool launch_fused(const uint8_t* reads, const uint8_t* refs, int64_t stride, int64_t n, int len,
                  int e, bool sweep, uint32_t* accept, uint8_t* errc, cudaStream_t stream);

int launch_filter_ascii(const uint8_t* reads, const uint8_t* refs, int64_t stride, int64_t n,
                        int len, int e, uint32_t* accept, uint8_t* errc, cudaStream_t stream) {
  // the tile-per-CTA fused kernels (gk_fused.cu); else the generic fallback
  if (launch_fused(reads, refs, stride, n, len, e, false, accept, errc, stream)) return 0;
  if (!dispatch_ascii<GK_SP_EMAX>(e, reads, refs, stride, n, len, accept, errc, stream))
    launch_ascii_all<-1>(reads, refs, stride, n, len, e, accept, errc, stream);
  return 0;
}

}  // namespace gk
