// gk_filter_ascii_p2.cu -- instantiations of the fused filter (parallel build unit).
#include "gk_filter_ascii_impl.cuh"

namespace gk {
template void launch_ascii_all<2>(const uint8_t*, const uint8_t*, int64_t, int64_t, int, int,
                                     uint32_t*, uint8_t*, cudaStream_t);
template void launch_ascii_all<6>(const uint8_t*, const uint8_t*, int64_t, int64_t, int, int,
                                     uint32_t*, uint8_t*, cudaStream_t);
template void launch_ascii_all<10>(const uint8_t*, const uint8_t*, int64_t, int64_t, int, int,
                                     uint32_t*, uint8_t*, cudaStream_t);
}  // namespace gk
