// Does SHFL compete with LDS for the shared-memory pipe on B200?  Cycles per
// loop iteration with 16 warps per SM for: LDS.128 only, SHFL only, both.
// (Decides whether k_micro32's row reduction should move from shared
// memory to warp shuffles.)
#include <cstdio>
#include <cuda_runtime.h>

template <int NL, int NS>
__global__ void k(double* out, int iters) {
    __shared__ __align__(16) double s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned addr = (unsigned)__cvta_generic_to_shared(s + 2 * lane);
    unsigned a0 = lane, a1 = lane * 3, a2 = lane * 5, a3 = lane * 7;
    unsigned long long x0 = 0, x1 = 0;
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (NL) {
#pragma unroll
                for (int q = 0; q < NL; ++q) {
                    double vx, vy;
                    asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(vx), "=d"(vy) : "r"(addr));
                    x0 ^= __double_as_longlong(vx);
                    x1 ^= __double_as_longlong(vy);
                }
            }
#pragma unroll
            for (int q = 0; q < NS; ++q) {
                a0 = __shfl_xor_sync(0xffffffffu, a0, 1) + 1;
                a1 = __shfl_xor_sync(0xffffffffu, a1, 2) + 1;
                a2 = __shfl_xor_sync(0xffffffffu, a2, 4) + 1;
                a3 = __shfl_xor_sync(0xffffffffu, a3, 8) + 1;
            }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (double)(t1 - t0);
    if ((x0 ^ x1 ^ a0 ^ a1 ^ a2 ^ a3) == 12345ull) out[1000 + threadIdx.x] = 1.0;
}

template <int NL, int NS>
void run(const char* name) {
    double* d;
    cudaMalloc(&d, sizeof(double) * 4096);
    const int iters = 1000, warps = 16;
    k<NL, NS><<<148, 32 * warps>>>(d, 10);
    k<NL, NS><<<148, 32 * warps>>>(d, iters);
    cudaDeviceSynchronize();
    double h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int i = 0; i < 148; ++i) cyc += h[i];
    cyc /= 148;
    printf("%-36s %.2f SM-cyc per (warp x unit)\n", name, cyc / (iters * 8.0 * warps));
}

int main() {
    run<1, 0>("1 LDS.128 (32 distinct)");
    run<0, 1>("4 SHFL.32");
    run<1, 1>("1 LDS.128 + 4 SHFL.32");
    run<2, 1>("2 LDS.128 + 4 SHFL.32");
    run<1, 2>("1 LDS.128 + 8 SHFL.32");
    return 0;
}
