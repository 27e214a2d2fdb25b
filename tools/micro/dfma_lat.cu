// fp64 latency / throughput on B200: dependent DFMA chain (1 warp per SM)
// and independent chains at 16 warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, int iters, double a, double b) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (threadIdx.x == 0) out[blockIdx.x] = (double)(t1 - t0);
    if (s == 1.2345) out[1000] = s;
}
template <int CH>
void run(int warps, const char* name) {
    double* d; cudaMalloc(&d, 8192);
    k<CH><<<148, 32 * warps>>>(d, 10, 0.999, 1e-3);
    k<CH><<<148, 32 * warps>>>(d, 2000, 0.999, 1e-3);
    cudaDeviceSynchronize();
    double h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
    const double per_warp_op = c / (2000.0 * 16 * CH);
    printf("%-34s warps/SM %2d: %.2f cyc per op per warp, %.3f SM-cyc per warp-op\n", name, warps,
           per_warp_op, per_warp_op / warps);
}
int main() {
    run<1>(1, "dependent chain (latency)");
    run<2>(1, "2 chains");
    run<4>(1, "4 chains");
    run<8>(1, "8 chains");
    run<8>(4, "8 chains");
    run<8>(16, "8 chains (throughput)");
    run<1>(16, "1 chain");
    run<2>(16, "2 chains");
    return 0;
}
