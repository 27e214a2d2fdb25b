// Shared-memory LDS.128 / LDS.64 throughput by lane->address pattern on B200:
// cycles per warp-instruction with 16 warps per SM issuing back to back.
// Used to choose the thread -> velocity-node mapping of k_micro32 (which of
// its table loads cost 1, 2 or 4 shared-memory wavefronts).
#include <cstdio>
#include <cuda_runtime.h>

template <int PAT, int W>
__global__ void k(double* out, int iters) {
    __shared__ __align__(16) double s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31, q = lane >> 3, r = lane & 7;
    int idx;   // index in units of W doubles
    switch (PAT) {
        case 0: idx = r; break;                       // quarter: 8 distinct, same across quarters (L)
        case 1: idx = 5 * q; break;                   // quarter-uniform, distinct across quarters (K)
        case 2: idx = 0; break;                       // warp-uniform
        case 3: idx = lane; break;                    // 32 distinct consecutive
        case 4: idx = r & 1; break;                   // quarter: 2 distinct, same across quarters
        case 5: idx = (r & 1) + 2 * q; break;         // quarter: 2 distinct, 8 distinct overall
        case 6: idx = (r & 3); break;                 // quarter: 4 distinct, same across quarters
        case 7: idx = (r & 3) + 4 * q; break;         // quarter: 4 distinct, 16 overall
        case 8: idx = (lane >> 4) * 5; break;         // half-warp uniform
        case 9: idx = (r & 1) * 4 + 8 * (q & 1); break;  // quarter 2 distinct, halves differ
        case 10: idx = (lane & 1) + 2 * (lane >> 3); break; // quarter: 2 distinct, consecutive, quarters differ
        case 11: idx = ((lane >> 1) & 3) + 4 * (lane >> 3); break; // quarter: 4 distinct consecutive, quarters differ (16 overall)
        case 12: idx = ((lane >> 1) & 3); break;       // quarter: 4 distinct consecutive, same across quarters
        case 13: idx = ((lane >> 1) & 3) + 8 * (lane >> 4); break; // quarter 4 consecutive, halves differ by 8
        case 14: idx = ((lane >> 1) & 3) + 32 * (lane >> 3); break; // quarter 4 consecutive, quarters 256 B apart
        case 15: idx = (lane & 1) + 2 * ((lane >> 3) & 3); break;   // mapping B, L-table pair word
        case 16: idx = ((lane >> 1) & 3) * 5; break;               // mapping B, K pair-word, stride 5 words
        case 17: idx = ((lane >> 1) & 3) * 4; break;               // stride 4 words (64 B)
        case 18: idx = ((lane >> 1) & 3) * 6; break;               // stride 6 words
        case 19: idx = ((lane >> 1) & 3); break;                   // = 12 (consecutive)
        default: idx = 0;
    }
    const double* p = s + W * idx + 64 * (threadIdx.x >> 5) * 0;
    unsigned long long acc0 = 0, acc1 = 0;
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            if (W == 2) {
                double2 v;
                asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"((unsigned)__cvta_generic_to_shared(p + 2 * ((u * 7) & 15) * 0)));
                acc0 ^= __double_as_longlong(v.x); acc1 ^= __double_as_longlong(v.y);
            } else {
                double v;
                asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
                acc0 ^= __double_as_longlong(v);
            }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (double)(t1 - t0);
    if ((acc0 ^ acc1) == 12345ull) out[1000 + threadIdx.x] = 1.0;
}

template <int PAT, int W>
void run(const char* name) {
    double* d;
    cudaMalloc(&d, sizeof(double) * 4096);
    const int iters = 2000, warps = 16;
    k<PAT, W><<<148, 32 * warps>>>(d, 10);
    k<PAT, W><<<148, 32 * warps>>>(d, iters);
    cudaDeviceSynchronize();
    double h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = 0;
    for (int i = 0; i < 148; ++i) cyc += h[i];
    cyc /= 148;
    const double per = cyc / (iters * 16.0 * warps);   // SM cycles per warp-instruction
    printf("%-44s W=%d  %.2f cyc/warp-LDS\n", name, W, per);
    cudaFree(d);
}

int main() {
    run<12, 2>("LDS.128 quarter 4 consec (pairs), same across q");
    run<13, 2>("LDS.128 quarter 4 consec (pairs), halves differ");
    run<15, 2>("LDS.128 mapping B L-word");
    run<16, 2>("LDS.128 mapping B K-word stride 5");
    run<17, 2>("LDS.128 K-word stride 4");
    run<18, 2>("LDS.128 K-word stride 6");
    run<16, 1>("LDS.64 K stride 5 (x2 doubles)");
    run<15, 1>("LDS.64 mapping B L");
    return 0;
}
