// The ten kernel-contract functions of the reference's plugin module
// `micromacro._kernels` (_fallback.py:27-173, _core.pyx:20-322), as plain
// sm_100a kernels on device pointers.  They exist for unit parity and for
// callers that use the reference's kernel-level API; the timestep itself
// runs the fused kernels (mm2d_micro.cuh).
#pragma once
#include "mm2d_common.cuh"

namespace mm2d {

__device__ __forceinline__ double block_sum(double v, double* sh) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    for (int q = 0; q < nw; ++q) t += sh[q];
    return t;
}

__global__ void kc_maxwellian(int S, int nv1, int nv2, const double* rho, const double* u1,
                              const double* u2, const double* T, const double* v1,
                              const double* v2, double* M) {
    const size_t V = (size_t)nv1 * nv2, n = (size_t)S * V;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n;
         t += (size_t)gridDim.x * blockDim.x) {
        const size_t c = t / V;
        const int k = (int)((t % V) / nv2), l = (int)(t % nv2);
        const double pref = rho[c] / (2.0 * kPi * T[c]);
        const double inv2T = 1.0 / (2.0 * T[c]);
        const double w1 = v1[k] - u1[c], w2 = v2[l] - u2[c];
        M[t] = pref * exp(-(w1 * w1 + w2 * w2) * inv2T);
    }
}

// per-cell projection coefficients of F: one CTA per cell
__device__ __forceinline__ void proj_coeffs_block(const double* F, int nv1, int nv2,
                                                  const double* v1, const double* v2,
                                                  double rho, double u1, double u2, double T,
                                                  double dv, double* sh, double a[4]) {
    const int V = nv1 * nv2;
    const double st = sqrt(T);
    double s1 = 0, s2 = 0, s3 = 0, s4 = 0;
    for (int n = threadIdx.x; n < V; n += blockDim.x) {
        const int k = n / nv2, l = n % nv2;
        const double w1 = (v1[k] - u1) / st, w2 = (v2[l] - u2) / st;
        const double b4 = 0.5 * (w1 * w1 + w2 * w2) - 1.0;
        const double f = F[n];
        s1 += f; s2 += f * w1; s3 += f * w2; s4 += f * b4;
    }
    const double scale = dv / rho;
    a[0] = block_sum(s1, sh) * scale;
    a[1] = block_sum(s2, sh) * scale;
    a[2] = block_sum(s3, sh) * scale;
    a[3] = block_sum(s4, sh) * scale;
}

__global__ void kc_project(int nv1, int nv2, const double* F, const double* M, const double* rho,
                           const double* u1, const double* u2, const double* T, const double* v1,
                           const double* v2, double dv, double* out) {
    __shared__ double sh[32];
    const size_t c = blockIdx.x, V = (size_t)nv1 * nv2;
    double a[4];
    proj_coeffs_block(F + c * V, nv1, nv2, v1, v2, rho[c], u1[c], u2[c], T[c], dv, sh, a);
    const double st = sqrt(T[c]);
    for (int n = threadIdx.x; n < (int)V; n += blockDim.x) {
        const int k = n / nv2, l = n % nv2;
        const double w1 = (v1[k] - u1[c]) / st, w2 = (v2[l] - u2[c]) / st;
        const double b4 = 0.5 * (w1 * w1 + w2 * w2) - 1.0;
        out[c * V + n] = (a[0] + w1 * a[1] + w2 * a[2] + b4 * a[3]) * M[c * V + n];
    }
}

// transport_stage_2d: Z into out first, then the projection, then the update
__global__ void kc_transport(int nx, int ny, int nv1, int nv2, const double* Gext,
                             const double* M, const double* rho, const double* u1,
                             const double* u2, const double* T, const double* v1,
                             const double* v2, double d, double dt, int axis, double* out) {
    __shared__ double sh[32];
    const int c = blockIdx.x;
    const int i = c / ny, j = c % ny;
    const size_t V = (size_t)nv1 * nv2;
    const int eny = axis == 1 ? ny + 2 : ny;
    const int io = axis == 0 ? i + 1 : i, jo = axis == 1 ? j + 1 : j;
    const double* g0 = Gext + ((size_t)io * eny + jo) * V;
    const double* gm = axis == 0 ? Gext + ((size_t)(io - 1) * eny + jo) * V : g0 - V;
    const double* gp = axis == 0 ? Gext + ((size_t)(io + 1) * eny + jo) * V : g0 + V;
    double* z = out + (size_t)c * V;
    for (int n = threadIdx.x; n < (int)V; n += blockDim.x) {
        const int k = n / nv2, l = n % nv2;
        const double vk = axis == 0 ? v1[k] : v2[l];
        z[n] = vk >= 0.0 ? vk * (g0[n] - gm[n]) / d : vk * (gp[n] - g0[n]) / d;
    }
    __syncthreads();
    const double dv = (v1[1] - v1[0]) * (v2[1] - v2[0]);
    double a[4];
    proj_coeffs_block(z, nv1, nv2, v1, v2, rho[c], u1[c], u2[c], T[c], dv, sh, a);
    const double st = sqrt(T[c]);
    for (int n = threadIdx.x; n < (int)V; n += blockDim.x) {
        const int k = n / nv2, l = n % nv2;
        const double w1 = (v1[k] - u1[c]) / st, w2 = (v2[l] - u2[c]) / st;
        const double b4 = 0.5 * (w1 * w1 + w2 * w2) - 1.0;
        const double zh = (a[0] + w1 * a[1] + w2 * a[2] + b4 * a[3]) * M[(size_t)c * V + n];
        z[n] = g0[n] - dt * (z[n] - zh);
    }
}

__global__ void kc_ghat(int S, int nv1, int nv2, const double* M, const double* u1,
                        const double* u2, const double* T, const double* s11, const double* s12,
                        const double* gT1, const double* gT2, const double* tau, const double* v1,
                        const double* v2, double* out) {
    const size_t V = (size_t)nv1 * nv2, n = (size_t)S * V;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n;
         t += (size_t)gridDim.x * blockDim.x) {
        const size_t c = t / V;
        const int k = (int)((t % V) / nv2), l = (int)(t % nv2);
        const double inv2T = 1.0 / (2.0 * T[c]), invT = 1.0 / T[c], invtau = 1.0 / tau[c];
        const double w1 = v1[k] - u1[c], w2 = v2[l] - u2[c];
        const double bs = (-w2 * w2 * s11[c] + 2.0 * w1 * w2 * s12[c] + w1 * w1 * s11[c]) * inv2T;
        const double cg = ((w1 * w1 + w2 * w2) * inv2T - 2.0) * (w1 * gT1[c] + w2 * gT2[c]) * invT;
        out[t] = -(bs + cg) * M[t] * invtau;
    }
}

__global__ void kc_gauss(int S, int nv1, int nv2, double* Ghat, const double* M, const double* rho,
                         const double* u1, const double* u2, const double* m11,
                         const double* m12, const double* m22, double eps, const double* v1,
                         const double* v2) {
    const size_t V = (size_t)nv1 * nv2, n = (size_t)S * V;
    const double inveps = 1.0 / eps;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n;
         t += (size_t)gridDim.x * blockDim.x) {
        const size_t c = t / V;
        const int k = (int)((t % V) / nv2), l = (int)(t % nv2);
        const double c11 = m11[c], c12 = m12[c], c22 = m22[c];
        const double det = c11 * c22 - c12 * c12;
        const double pref = rho[c] / (2.0 * kPi * sqrt(det));
        const double w1 = v1[k] - u1[c], w2 = v2[l] - u2[c];
        const double quad = (c22 * w1 * w1 - 2.0 * c12 * w1 * w2 + c11 * w2 * w2) / det;
        Ghat[t] += (pref * exp(-0.5 * quad) - M[t]) * inveps;
    }
}

__global__ void kc_lowrank(int S, int V, double* out, int nterms, const double* coeffs,
                           const double* shapes) {
    const size_t n = (size_t)S * V;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n;
         t += (size_t)gridDim.x * blockDim.x) {
        const size_t c = t / V, q = t % V;
        double acc = out[t];
        for (int m = 0; m < nterms; ++m) acc += coeffs[(size_t)m * S + c] * shapes[(size_t)m * V + q];
        out[t] = acc;
    }
}

__global__ void kc_relax(int S, int V, const double* G, const double* Ghat, const double* tau,
                         double dt, double eps, double* out) {
    const size_t n = (size_t)S * V;
    for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < n;
         t += (size_t)gridDim.x * blockDim.x) {
        const size_t c = t / V;
        const double denom = eps + dt * tau[c];
        out[t] = (eps / denom) * G[t] + (dt * tau[c] / denom) * Ghat[t];
    }
}

__global__ void kc_heat(int S, int nv1, int nv2, const double* G, const double* u1,
                        const double* u2, const double* v1, const double* v2, double f,
                        double* H) {
    __shared__ double sh[32];
    const size_t c = blockIdx.x, V = (size_t)nv1 * nv2;
    double s[4] = {0, 0, 0, 0};
    for (int n = threadIdx.x; n < (int)V; n += blockDim.x) {
        const int k = n / nv2, l = n % nv2;
        const double w1 = v1[k] - u1[c], w2 = v2[l] - u2[c], g = G[c * V + n];
        s[0] += w1 * w1 * w1 * g; s[1] += w1 * w1 * w2 * g;
        s[2] += w1 * w2 * w2 * g; s[3] += w2 * w2 * w2 * g;
    }
    for (int q = 0; q < 4; ++q) {
        const double t = block_sum(s[q], sh);
        if (threadIdx.x == 0) H[(size_t)q * S + c] = f * t;
    }
}

__global__ void kc_upwind1d(int nx, int nv, const double* Gext, const double* v, double dx,
                            double* Z) {
    const int n = nx * nv;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const int i = t / nv, k = t % nv;
        const double vk = v[k];
        Z[t] = vk >= 0.0 ? vk * (Gext[(i + 1) * nv + k] - Gext[i * nv + k]) / dx
                         : vk * (Gext[(i + 2) * nv + k] - Gext[(i + 1) * nv + k]) / dx;
    }
}

__global__ void kc_project1d(int nv, const double* F, const double* M, const double* rho,
                             const double* u, const double* T, const double* v, double dv,
                             double* out) {
    __shared__ double sh[32];
    const int i = blockIdx.x;
    const double st = sqrt(T[i]);
    double s1 = 0, s2 = 0, s3 = 0;
    for (int k = threadIdx.x; k < nv; k += blockDim.x) {
        const double w = (v[k] - u[i]) / st;
        const double b3 = 1.4142135623730950488 * (0.5 * w * w - 0.5);
        const double f = F[(size_t)i * nv + k];
        s1 += f; s2 += f * w; s3 += f * b3;
    }
    const double scale = dv / rho[i];
    const double a1 = block_sum(s1, sh) * scale, a2 = block_sum(s2, sh) * scale;
    const double a3 = block_sum(s3, sh) * scale;
    for (int k = threadIdx.x; k < nv; k += blockDim.x) {
        const double w = (v[k] - u[i]) / st;
        const double b3 = 1.4142135623730950488 * (0.5 * w * w - 0.5);
        out[(size_t)i * nv + k] = (a1 + w * a2 + b3 * a3) * M[(size_t)i * nv + k];
    }
}

}  // namespace mm2d
