// March kernels of variant 2 (see fused_cfg.cuh), one translation unit per variant so
// the variants compile in parallel.
#include "fused_march.cuh"

namespace ngf {
template int march_prepare<float, V2>(size_t);
template void march_launch<float, V2>(const FusedArgs<float>&, cudaStream_t);
}  // namespace ngf
