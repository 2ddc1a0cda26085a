// gk_filter_q1.cu -- instantiations of the large-e filter (parallel build unit).
#include "gk_filter_q_impl.cuh"

namespace gk {
template void launch_spq<13>(const uint2*, const uint2*, const uint32_t*, const uint32_t*, int64_t, int,
                              uint32_t*, uint8_t*, cudaStream_t);
template void launch_spq<15>(const uint2*, const uint2*, const uint32_t*, const uint32_t*, int64_t, int,
                              uint32_t*, uint8_t*, cudaStream_t);
template void launch_spq<17>(const uint2*, const uint2*, const uint32_t*, const uint32_t*, int64_t, int,
                              uint32_t*, uint8_t*, cudaStream_t);
template void launch_spq<19>(const uint2*, const uint2*, const uint32_t*, const uint32_t*, int64_t, int,
                              uint32_t*, uint8_t*, cudaStream_t);
template void launch_spq<21>(const uint2*, const uint2*, const uint32_t*, const uint32_t*, int64_t, int,
                              uint32_t*, uint8_t*, cudaStream_t);
template void launch_spq<23>(const uint2*, const uint2*, const uint32_t*, const uint32_t*, int64_t, int,
                              uint32_t*, uint8_t*, cudaStream_t);
template void launch_spq<25>(const uint2*, const uint2*, const uint32_t*, const uint32_t*, int64_t, int,
                              uint32_t*, uint8_t*, cudaStream_t);
}  // namespace gk
