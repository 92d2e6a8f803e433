// March kernels of variant 4 (see fused_cfg.cuh), one translation unit per variant so
// the variants compile in parallel.
#include "fused_march.cuh"

namespace ngf {
template int march_prepare<double, V4>(size_t);
template void march_launch<double, V4>(const FusedArgs<double>&, cudaStream_t);
// f32 with one slot per thread: the latency-bound small levels (few CTAs per SM)
template int march_prepare<float, V4>(size_t);
template void march_launch<float, V4>(const FusedArgs<float>&, cudaStream_t);
}  // namespace ngf
