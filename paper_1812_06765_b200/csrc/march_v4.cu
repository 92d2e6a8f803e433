// March kernels of variant 4 (see fused_cfg.cuh), one translation unit per variant so
// the variants compile in parallel.
#include "fused_march.cuh"

namespace ngf {
template int march_prepare<double, V4>(size_t);
template void march_launch<double, V4>(const FusedArgs<double>&, cudaStream_t);
}  // namespace ngf
