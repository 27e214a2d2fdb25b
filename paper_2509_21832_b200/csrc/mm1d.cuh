// 1D1V BGK micro-macro step (BASELINE config 1), restating the reference's
// step_1d (runner/loop.py:31-51): micro_step_1d (micro1d.py:40-64) with
// upwind_z_1d / project_field_1d (_core.pyx:20-63), interface temperatures
// and wall closures (boundary.py:94-170), heat_flux_1d (macro1d.py:16-19,
// raw v^3 and a 1/2 factor) and the Maxwellian KFVS macro step
// (macro1d.py:22-92).
//
// Generic path: two kernels per step.  k1_micro (one CTA per cell)
// recomputes the primitives of its cell and both neighbours straight from Q,
// so no per-cell parameter pass is needed; k1_macro (one thread per cell)
// does the same for the flux differences.
#pragma once
#include "mm2d_common.cuh"

namespace mm2d {
namespace d1 {

struct Geo1 {
    int nx, nv;
    double dx, dv;
    int face[2];        // 0 periodic, 1 extrapolate, 2 wall
    double wallT[2];
    int tau_kind;
    double tau_value;
    double eps;
};

// error stages of the 1D check (primitives_1d, gas_state.py:44-54)
enum { E1_DENSITY = 0, E1_TEMPERATURE = 1 };

__device__ __forceinline__ double tau1(const Geo1& g, double rho, double T) {
    switch (g.tau_kind) {
        case 0: return 3.2 * sqrt(T / (2.0 * kPi));
        case 1: return rho * T;
        case 2: return (0.4625 * kPi) * rho;
        case 3: return (3.0 * kPi * 0.436 / sqrt(2.0)) * rho;
        default: return g.tau_value;
    }
}

struct Prim1 {
    double rho, u, T;
};

// primitives_1d (gas_state.py:44-54), without the checks
__device__ __forceinline__ Prim1 prim1(const double* q) {
    Prim1 p;
    p.rho = q[0];
    p.u = q[1] / p.rho;
    p.T = (2.0 * q[2] - p.rho * p.u * p.u) / p.rho;
    return p;
}

__device__ __forceinline__ void alpha_beta(double u, double T, double& al, double& bp, double& bm) {
    al = sqrt(T / (2.0 * kPi)) * exp(-u * u / (2.0 * T));
    const double s = erf(u / sqrt(2.0 * T));
    bp = 0.5 * (1.0 + s);
    bm = 0.5 * (1.0 - s);
}

// wall_density_1d (boundary.py:94-105)
__device__ __forceinline__ double wall_rho(const Prim1& p, double Tw, bool right) {
    double al, bp, bm;
    alpha_beta(p.u, p.T, al, bp, bm);
    return right ? sqrt(2.0 * kPi / Tw) * (p.rho * al + p.rho * p.u * bp)
                 : sqrt(2.0 * kPi / Tw) * (p.rho * al - p.rho * p.u * bm);
}

// wall_interface_temperature_1d (boundary.py:108-122)
__device__ __forceinline__ double wall_T(const Prim1& p, double Tw, bool right) {
    double al, bp, bm;
    alpha_beta(p.u, p.T, al, bp, bm);
    const double rw = wall_rho(p, Tw, right);
    const double rho = p.rho, u = p.u, T = p.T;
    if (!right)
        return (0.5 * rw * Tw + rho * ((T + u * u) * bm - u * al)) / (0.5 * rw + rho * bm);
    return (rho * ((T + u * u) * bp + u * al) + 0.5 * rw * Tw) / (rho * bp + 0.5 * rw);
}

// interface temperature m in [0, nx] (interface_temperatures_1d, boundary.py:125-138);
// Pl / Pr are the primitives of cells m-1 and m (wrapped for periodic faces,
// the edge cell otherwise)
__device__ __forceinline__ double iface_T(const Geo1& g, int m, const Prim1& Pl, const Prim1& Pr) {
    if ((m > 0 && m < g.nx) || g.face[0] == 0) return 0.5 * (Pr.T + Pl.T);
    const bool right = m == g.nx;
    const Prim1& e = right ? Pl : Pr;
    const int f = right ? 1 : 0;
    return g.face[f] == 1 ? e.T : wall_T(e, g.wallT[f], right);
}

// KFVS flux between primitive states (kfvs_flux_1d, macro1d.py:34-51)
__device__ __forceinline__ void kfvs1(const Prim1& L, const Prim1& R, double F[3]) {
    double out[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int side = 0; side < 2; ++side) {
        const Prim1& p = side ? R : L;
        const double sign = side ? -1.0 : 1.0;
        double al, bp, bm;
        alpha_beta(p.u, p.T, al, bp, bm);
        const double rho = p.rho, u = p.u, T = p.T;
        const double half[3] = {rho, rho * u, 0.5 * rho * (2.0 * T + u * u)};
        const double beta = side ? bm : bp;
        const double f[3] = {rho * u, rho * (T + u * u), 0.5 * rho * u * (3.0 * T + u * u)};
#pragma unroll
        for (int m = 0; m < 3; ++m) out[m] = out[m] + sign * al * half[m] + beta * f[m];
    }
    F[0] = out[0]; F[1] = out[1]; F[2] = out[2];
}

// interface flux m in [0, nx] (interface_fluxes_1d, macro1d.py:54-75)
__device__ __forceinline__ void iface_flux(const Geo1& g, int m, const Prim1& Pl, const Prim1& Pr,
                                           double F[3]) {
    if ((m > 0 && m < g.nx) || g.face[0] == 0) { kfvs1(Pl, Pr, F); return; }
    const bool right = m == g.nx;
    const Prim1& e = right ? Pl : Pr;
    const int f = right ? 1 : 0;
    if (g.face[f] == 1) { kfvs1(e, e, F); return; }
    Prim1 w;
    w.rho = wall_rho(e, g.wallT[f], right);
    w.u = 0.0;
    w.T = g.wallT[f];
    if (right) kfvs1(e, w, F);
    else kfvs1(w, e, F);
}

// interface heat flux m in [0, nx] (interface_heat_flux_1d, boundary.py:160-170)
__device__ __forceinline__ double iface_heat(const Geo1& g, int m, double hl, double hr) {
    if ((m > 0 && m < g.nx) || g.face[0] == 0) return 0.5 * (hr + hl);
    const bool right = m == g.nx;
    const double h = right ? hl : hr;
    return g.face[right ? 1 : 0] == 1 ? h : 0.5 * h;
}

// neighbour cell index with the face rule: wrap if periodic, else the edge cell
__device__ __forceinline__ int nb1(const Geo1& g, int c) {
    if (c < 0) return g.face[0] == 0 ? g.nx - 1 : 0;
    if (c >= g.nx) return g.face[0] == 0 ? 0 : g.nx - 1;
    return c;
}

struct Args1 {
    Geo1 g;
    const double* Q;      // (nx, 3)
    const double* G;      // (nx, nv)
    double* Qout;
    double* Gout;
    double* H;            // (nx)
    const double* v;      // (nv) cell-centred velocities
    const double* v3;     // (nv) v^3 (host pow, as numpy's v**3)
    const double* src;    // (nx, nv) projected micro source or null
    const double* qsrc;   // (nx, 3) macro source or null
    unsigned long long* err;   // [0] merged key, [1] failing Q pointer, [2] steps done,
                               // [3] key raised by k1_micro (merged into [0] by k1_macro)
    double dt;
};

__device__ __forceinline__ void flag1(const Args1& a, int stage, int cell) {
    atomicMin(a.err + 3, err_key(0, stage, (unsigned long long)cell));   // k1_micro's own word
    a.err[1] = (unsigned long long)(size_t)a.Q;
}

// micro_step_1d for one cell per CTA: upwind Z, the three projection sums,
// BGK target, blend with the relax weights, then the heat-flux moment.
__global__ void k1_micro(Args1 a) {
    __shared__ double sh[4][32];
    const Geo1& g = a.g;
    if (*(volatile const unsigned long long*)a.err != kNoError) return;   // earlier launches only
    const int i = blockIdx.x;
    const int nv = g.nv;
    const Prim1 P = prim1(a.Q + 3 * i);
    if (threadIdx.x == 0) {
        if (!(P.rho > 0.0)) flag1(a, E1_DENSITY, i);
        else if (!(P.T > 0.0)) flag1(a, E1_TEMPERATURE, i);
    }
    const Prim1 Pl = prim1(a.Q + 3 * nb1(g, i - 1));
    const Prim1 Pr = prim1(a.Q + 3 * nb1(g, i + 1));
    const double tau = tau1(g, P.rho, P.T);
    const double* Gi = a.G + (size_t)i * nv;
    // G ghosts: wrap / copy / zero at a wall (extend_micro_1d, boundary.py:141-157)
    const double* Gl = i > 0 ? Gi - nv
                             : (g.face[0] == 0 ? a.G + (size_t)(g.nx - 1) * nv
                                               : g.face[0] == 1 ? Gi : nullptr);
    const double* Gr = i < g.nx - 1 ? Gi + nv
                                    : (g.face[1] == 0 ? a.G : g.face[1] == 1 ? Gi : nullptr);
    const double st = sqrt(P.T);
    double s1 = 0, s2 = 0, s3 = 0;
    for (int k = threadIdx.x; k < nv; k += blockDim.x) {
        const double vk = a.v[k];
        const double z = vk >= 0.0 ? vk * (Gi[k] - (Gl ? Gl[k] : 0.0)) / g.dx
                                   : vk * ((Gr ? Gr[k] : 0.0) - Gi[k]) / g.dx;
        const double w = (vk - P.u) / st;
        const double b3 = 1.4142135623730950488 * (0.5 * w * w - 0.5);
        s1 += z; s2 += z * w; s3 += z * b3;
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    s1 = warp_sum(s1); s2 = warp_sum(s2); s3 = warp_sum(s3);
    if (lane == 0) { sh[0][wid] = s1; sh[1][wid] = s2; sh[2][wid] = s3; }
    if (threadIdx.x == 0) sh[3][0] = iface_T(g, i, Pl, P);
    if (threadIdx.x == 1 % blockDim.x) sh[3][1] = iface_T(g, i + 1, P, Pr);
    __syncthreads();
    double a1 = 0, a2 = 0, a3 = 0;
    for (int q = 0; q < nw; ++q) { a1 += sh[0][q]; a2 += sh[1][q]; a3 += sh[2][q]; }
    const double scale = g.dv / P.rho;
    a1 *= scale; a2 *= scale; a3 *= scale;
    const double dT = (sh[3][1] - sh[3][0]) / (g.dx * P.T);
    const double denom = g.eps + a.dt * tau;
    const double wg = g.eps / denom, wh = a.dt * tau / denom;
    const double pref = P.rho / sqrt(2.0 * kPi * P.T);
    double hsum = 0.0;
    for (int k = threadIdx.x; k < nv; k += blockDim.x) {
        const double vk = a.v[k];
        const double z = vk >= 0.0 ? vk * (Gi[k] - (Gl ? Gl[k] : 0.0)) / g.dx
                                   : vk * ((Gr ? Gr[k] : 0.0) - Gi[k]) / g.dx;
        const double w = (vk - P.u) / st;
        const double b3 = 1.4142135623730950488 * (0.5 * w * w - 0.5);
        const double wv = vk - P.u;
        const double M = pref * exp(-(wv * wv) / (2.0 * P.T));
        const double zh = (a1 + w * a2 + b3 * a3) * M;
        double gh = -((wv * wv * wv) / (2.0 * P.T) - 1.5 * wv) * (dT / tau) * M;
        if (a.src) gh = gh + a.src[(size_t)i * nv + k] / tau;
        const double gp = wg * (Gi[k] - a.dt * (z - zh)) + wh * gh;
        a.Gout[(size_t)i * nv + k] = gp;
        hsum += gp * a.v3[k];
    }
    hsum = warp_sum(hsum);
    __syncthreads();
    if (lane == 0) sh[0][wid] = hsum;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < nw; ++q) t += sh[0][q];
        a.H[i] = 0.5 * g.eps * g.dv * t;
    }
}

// macro_step_1d (macro1d.py:78-92): flux differences, heat flux, source
__global__ void k1_macro(Args1 a) {
    const Geo1& g = a.g;
    if (err_gate(a.err, 3)) return;   // k1_micro of this step or an earlier failure
    const double r = a.dt / g.dx;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.nx; i += gridDim.x * blockDim.x) {
        const int il = nb1(g, i - 1), ir = nb1(g, i + 1);
        const Prim1 P = prim1(a.Q + 3 * i);
        const Prim1 Pl = prim1(a.Q + 3 * il);
        const Prim1 Pr = prim1(a.Q + 3 * ir);
        double Fm[3], Fp[3];
        iface_flux(g, i, Pl, P, Fm);
        iface_flux(g, i + 1, P, Pr, Fp);
        const double h = a.H[i];
        double q[3];
#pragma unroll
        for (int m = 0; m < 3; ++m) q[m] = a.Q[3 * i + m] - r * (Fp[m] - Fm[m]);
        q[2] -= r * (iface_heat(g, i + 1, h, a.H[ir]) - iface_heat(g, i, a.H[il], h));
        if (a.qsrc) {
#pragma unroll
            for (int m = 0; m < 3; ++m) q[m] += a.dt * a.qsrc[3 * i + m];
        }
#pragma unroll
        for (int m = 0; m < 3; ++m) a.Qout[3 * i + m] = q[m];
    }
}

// value of the failing check, from the preserved input of the failing step
__global__ void k1_err_value(const double* Q, int stage, int cell, double* out) {
    const Prim1 p = prim1(Q + 3 * cell);
    *out = stage == E1_DENSITY ? p.rho : p.T;
}

}  // namespace d1
}  // namespace mm2d
