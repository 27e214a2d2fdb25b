// Translation unit of the 32 x 32 fused micro kernel (mm2d_micro32.cuh).
#include "mm2d_micro32.cuh"
#include "mm2d_micro32_launch.h"

namespace mm2d {
namespace m32 {

cudaError_t setup(int* ctas_per_sm) {
    const void* fns[2] = {reinterpret_cast<const void*>(&k_micro32<4, false>),
                          reinterpret_cast<const void*>(&k_micro32<4, true>)};
    const size_t sm = smem_bytes_v3<4>();
    for (const void* fn : fns) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sm);
        if (e != cudaSuccess) return e;
    }
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, fns[0], 128, sm);
}

void launch_micro32(const MicroArgs& a, dim3 grid, cudaStream_t s) {
    const Geometry& g = a.g;
    const bool mir = g.xlo == GM_MIRROR || g.xhi == GM_MIRROR || g.ylo == GM_MIRROR ||
                     g.yhi == GM_MIRROR;
    if (mir) k_micro32<4, true><<<grid, 128, smem_bytes_v3<4>(), s>>>(a);
    else k_micro32<4, false><<<grid, 128, smem_bytes_v3<4>(), s>>>(a);
}

void launch_wall_ghat(const MicroArgs& a, double* out, int nblocks, cudaStream_t s) {
    k_wall_ghat<<<nblocks, 128, 0, s>>>(a, out);
}

}  // namespace m32
}  // namespace mm2d
