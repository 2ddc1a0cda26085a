// gk_filter_ascii_p1.cu -- instantiations of the fused filter (parallel build unit).
#include "gk_filter_ascii_impl.cuh"

namespace gk {
template void launch_ascii_all<1>(const uint8_t*, const uint8_t*, int64_t, int64_t, int, int,
                                     uint32_t*, uint8_t*, cudaStream_t);
template void launch_ascii_all<5>(const uint8_t*, const uint8_t*, int64_t, int64_t, int, int,
                                     uint32_t*, uint8_t*, cudaStream_t);
template void launch_ascii_all<9>(const uint8_t*, const uint8_t*, int64_t, int64_t, int, int,
                                     uint32_t*, uint8_t*, cudaStream_t);
}  // namespace gk
