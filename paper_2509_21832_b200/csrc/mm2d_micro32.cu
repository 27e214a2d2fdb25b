// Translation unit of the 32 x 32 fused micro kernel (mm2d_micro32.cuh).
#include <algorithm>
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
        // all of the unified L1 as shared memory: 4 CTAs x 55 KB per SM (the
        // occupancy query below reports 1 CTA/SM under the default carveout)
        e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 (int)cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
    }
    // resident CTAs per SM from the kernel's registers and shared memory (the
    // runtime's occupancy query reports 1 for this kernel, while 4 run)
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, fns[0]);
    if (e != cudaSuccess) return e;
    int dev = 0, regs_sm = 0, smem_sm = 0, rsv = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
    const int by_regs = regs_sm / std::max(1, fa.numRegs * 128);
    const int by_smem = smem_sm / (int)(sm + fa.sharedSizeBytes + rsv);
    *ctas_per_sm = std::max(1, std::min(by_regs, by_smem));
    return cudaSuccess;
}

void launch_micro32(const MicroArgs& a, dim3 grid, cudaStream_t s) {
    const Geometry& g = a.g;
    const bool mir = g.xlo == GM_MIRROR || g.xhi == GM_MIRROR || g.ylo == GM_MIRROR ||
                     g.yhi == GM_MIRROR;
    if (mir) launch_pdl(k_micro32<4, true>, grid, dim3(128), smem_bytes_v3<4>(), s, a);
    else launch_pdl(k_micro32<4, false>, grid, dim3(128), smem_bytes_v3<4>(), s, a);
}

void launch_wall_ghat(const MicroArgs& a, double* out, int nblocks, cudaStream_t s) {
    launch_pdl(k_wall_ghat, dim3(nblocks), dim3(128), 0, s, a, out);
}

}  // namespace m32
}  // namespace mm2d
