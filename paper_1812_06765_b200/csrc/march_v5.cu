// March kernels of variant 5 (see fused_cfg.cuh), one translation unit per variant so
// the variants compile in parallel.
#include "fused_march.cuh"

namespace ngf {
template int march_prepare<double, V5>(size_t);
template void march_launch<double, V5>(const FusedArgs<double>&, cudaStream_t);
// f32 with one slot per thread: the latency-bound small levels (few CTAs per SM)
template int march_prepare<float, V5>(size_t);
template void march_launch<float, V5>(const FusedArgs<float>&, cudaStream_t);
}  // namespace ngf
