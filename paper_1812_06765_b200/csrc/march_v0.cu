// March kernels of variant 0 (see fused_cfg.cuh), one translation unit per variant so
// the variants compile in parallel.
#include "fused_march.cuh"

namespace ngf {
template int march_prepare<float, V0>(size_t);
template void march_launch<float, V0>(const FusedArgs<float>&, cudaStream_t);
template int march_prepare<double, V0>(size_t);
template void march_launch<double, V0>(const FusedArgs<double>&, cudaStream_t);
}  // namespace ngf
