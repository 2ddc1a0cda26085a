// gk_filter_q0.cu -- instantiations of the large-e filter (parallel build unit).
#include "gk_filter_q_impl.cuh"

namespace gk {
template void launch_spq<12>(const uint2*, const uint2*, const uint32_t*, const uint32_t*, int64_t, int,
                              uint32_t*, uint8_t*, cudaStream_t);
template void launch_spq<14>(const uint2*, const uint2*, const uint32_t*, const uint32_t*, int64_t, int,
                              uint32_t*, uint8_t*, cudaStream_t);
template void launch_spq<16>(const uint2*, const uint2*, const uint32_t*, const uint32_t*, int64_t, int,
                              uint32_t*, uint8_t*, cudaStream_t);
template void launch_spq<18>(const uint2*, const uint2*, const uint32_t*, const uint32_t*, int64_t, int,
                              uint32_t*, uint8_t*, cudaStream_t);
template void launch_spq<20>(const uint2*, const uint2*, const uint32_t*, const uint32_t*, int64_t, int,
                              uint32_t*, uint8_t*, cudaStream_t);
template void launch_spq<22>(const uint2*, const uint2*, const uint32_t*, const uint32_t*, int64_t, int,
                              uint32_t*, uint8_t*, cudaStream_t);
template void launch_spq<24>(const uint2*, const uint2*, const uint32_t*, const uint32_t*, int64_t, int,
                              uint32_t*, uint8_t*, cudaStream_t);
}  // namespace gk
