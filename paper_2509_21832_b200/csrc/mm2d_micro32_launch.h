// Host-side entry points of the 32 x 32 fused micro kernel, compiled in its
// own translation unit (mm2d_micro32.cu) so the library builds in parallel.
#pragma once
#include <cuda_runtime.h>
#include "mm2d_micro.cuh"

namespace mm2d {
namespace m32 {
// raise the dynamic shared-memory limit on the current device; resident CTAs per SM
cudaError_t setup(int* ctas_per_sm);
void launch_micro32(const MicroArgs& a, dim3 grid, cudaStream_t s);
void launch_wall_ghat(const MicroArgs& a, double* out, int nblocks, cudaStream_t s);
}  // namespace m32
}  // namespace mm2d
