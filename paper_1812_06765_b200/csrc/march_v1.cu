// March kernels of variant 1 (see fused_cfg.cuh), one translation unit per variant so
// the variants compile in parallel.
#include "fused_march.cuh"

namespace ngf {
template int march_prepare<float, V1>(size_t);
template void march_launch<float, V1>(const FusedArgs<float>&, cudaStream_t);
}  // namespace ngf
