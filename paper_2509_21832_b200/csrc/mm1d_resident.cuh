// Cluster-resident 1D run: the whole (Q, G) state of run_1d's loop
// (runner/loop.py:54-72) lives in the distributed shared memory of ONE
// thread-block cluster for all n steps, so a 512-step config-1 run is a
// single launch.  CTA r of the cluster owns cells [r*cpc, (r+1)*cpc), one
// warp per cell.  Neighbour data (G rows, primitives, split fluxes, H of
// cells c0-1 and c0+cpc) is read from the neighbouring CTA's shared memory
// through the cluster mapping; two cluster barriers per step:
//   A  micro update of the cell into the other G buffer, its heat flux and
//      its KFVS half-range split fluxes A+ = a h + b+ f, A- = -a h + b- f
//      (kfvs_flux_1d, macro1d.py:34-51: F_{m} = A+(m-1) + A-(m))
//   -- barrier --
//   B  Q+ = Q - dt/dx (F_{i+1/2} - F_{i-1/2}) - heat-flux difference, then the
//      primitives of Q+ (and their check) for the next step
//   -- barrier --
// The arithmetic is the reference's; reciprocals are hoisted out of the
// node loops and the KFVS sum is re-associated as A+ + A-, which moves
// results by O(1 ulp) against the generic step (k1_micro / k1_macro).
// Errors: the failing thread sets the error flag in EVERY CTA's shared
// memory before the barrier, so the whole cluster leaves the loop at the
// same step with the failing step's input intact (primitives_1d,
// gas_state.py:44-54).
#pragma once
#include <cooperative_groups.h>

#include "mm1d.cuh"

namespace mm2d {
namespace d1 {

namespace cg = cooperative_groups;

struct Res1 {
    Geo1 g;
    int cpc;                 // cells per CTA (a power of two)
    int lg;                  // log2(cpc)
    double* Q;               // (nx,3) in/out
    double* G;               // (nx,nv) in/out
    double* H;               // (nx) out: heat flux of the last completed step
    const double* v;
    const double* v3;
    unsigned long long* err;
    double dt;
    int nsteps;
    int* done;               // completed steps (written by CTA 0)
};

// shared layout (doubles): Gs[2][cpc*nv] | Qs[cpc*3] | Ps[cpc*4] | Fl[cpc*8] | Fe[8] | flag
__host__ __device__ inline size_t res1_smem(int cpc, int nv) {
    return sizeof(double) * ((size_t)2 * cpc * nv + 3 * (size_t)cpc + 4 * (size_t)cpc +
                             8 * (size_t)cpc + 8 + 2);
}

// half-range split fluxes of one state (kfvs_flux_1d's two halves)
__device__ __forceinline__ void split_flux(double rho, double u, double T, double Ap[3],
                                           double Am[3]) {
    double al, bp, bm;
    alpha_beta(u, T, al, bp, bm);
    const double half[3] = {rho, rho * u, 0.5 * rho * (2.0 * T + u * u)};
    const double f[3] = {rho * u, rho * (T + u * u), 0.5 * rho * u * (3.0 * T + u * u)};
#pragma unroll
    for (int m = 0; m < 3; ++m) {
        Ap[m] = al * half[m] + bp * f[m];
        Am[m] = -al * half[m] + bm * f[m];
    }
}

template <int NJ>
__global__ void __launch_bounds__(512) k1_resident(Res1 a) {
    extern __shared__ __align__(16) double smem[];
    cg::cluster_group cl = cg::this_cluster();
    const Geo1& g = a.g;
    const int nv = g.nv, cpc = a.cpc;
    const int rank = (int)cl.block_rank();
    const int C = (int)cl.num_blocks();
    const int c0 = rank * cpc;
    const int cnt = max(0, min(cpc, g.nx - c0));
    double* Gs0 = smem;
    double* Gs1 = smem + (size_t)cpc * nv;
    double* Qs = Gs1 + (size_t)cpc * nv;
    double* Ps = Qs + 3 * cpc;
    double* Fl = Ps + 4 * cpc;
    double* Fe = Fl + 8 * cpc;
    int* flag = reinterpret_cast<int*>(Fe + 8);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
    const double idx = 1.0 / g.dx;
    const double r = a.dt / g.dx;

    // cell c's record (stride doubles per cell) in the shared memory of its owner
    auto remote = [&](double* base, int c, int stride) -> double* {
        const int rr = c >> a.lg;
        return cl.map_shared_rank(base, rr) + (size_t)stride * (c - rr * cpc);
    };
    auto raise = [&](int stage, int cell) {
        atomicMin(a.err, err_key(0, stage, (unsigned long long)cell));
        for (int q = 0; q < C; ++q) *cl.map_shared_rank(flag, q) = 1;
    };

    // ---- prologue: load the state, primitives (and their check) of Q^0 ----
    for (int n = tid; n < cnt * nv; n += blockDim.x) Gs0[n] = a.G[(size_t)c0 * nv + n];
    for (int n = tid; n < cnt * 3; n += blockDim.x) Qs[n] = a.Q[(size_t)c0 * 3 + n];
    if (tid == 0)
        *flag = (*(volatile unsigned long long*)a.err != kNoError ||
                 *(volatile unsigned long long*)(a.err + 3) != kNoError) ? 1 : 0;
    double vk[NJ], v3k[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const int k = lane + 32 * j;
        vk[j] = k < nv ? a.v[k] : 0.0;
        v3k[j] = k < nv ? a.v3[k] : 0.0;
    }
    cl.sync();     // every flag initialised before anyone may raise
    for (int lc = tid; lc < cnt; lc += blockDim.x) {
        const Prim1 P = prim1(Qs + 3 * lc);
        Ps[4 * lc] = P.rho; Ps[4 * lc + 1] = P.u; Ps[4 * lc + 2] = P.T;
        if (!(P.rho > 0.0)) raise(E1_DENSITY, c0 + lc);
        else if (!(P.T > 0.0)) raise(E1_TEMPERATURE, c0 + lc);
    }
    const double* Fe0 = remote(Fe, 0, 0);                 // left-edge wall flux (owner of cell 0)
    const double* Fe1 = remote(Fe, g.nx - 1, 0) + 4;      // right-edge wall flux
    cl.sync();

    int cur = 0, completed = 0;
    for (int step = 0; step < a.nsteps; ++step) {
        if (*(volatile int*)flag) break;     // uniform: every CTA holds the same flag
        double* Gcur = cur ? Gs1 : Gs0;
        double* Gnxt = cur ? Gs0 : Gs1;
        // ---- phase A: micro update, one warp per owned cell ----
        for (int lc = wid; lc < cnt; lc += nw) {
            const int i = c0 + lc;
            const int il = nb1(g, i - 1), ir = nb1(g, i + 1);
            const double rho = Ps[4 * lc], u = Ps[4 * lc + 1], T = Ps[4 * lc + 2];
            const Prim1 P = {rho, u, T};
            const Prim1 Pl = {0.0, 0.0, remote(Ps, il, 4)[2]};
            const Prim1 Pr = {0.0, 0.0, remote(Ps, ir, 4)[2]};
            const double* Gi = Gcur + (size_t)nv * lc;
            // G ghosts: neighbour row (wrapped), own row (extrapolate), zero (wall)
            const double* Gl = (i == 0 && g.face[0] == 2) ? nullptr : remote(Gcur, il, nv);
            const double* Gr = (i == g.nx - 1 && g.face[1] == 2) ? nullptr : remote(Gcur, ir, nv);
            const double tau = tau1(g, rho, T);
            const double ist = 1.0 / sqrt(T);
            double z[NJ], gi[NJ];
            double s1 = 0, s2 = 0, s3 = 0;
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int k = lane + 32 * j;
                z[j] = 0.0;
                gi[j] = 0.0;
                if (k < nv) {
                    gi[j] = Gi[k];
                    z[j] = vk[j] >= 0.0 ? vk[j] * (gi[j] - (Gl ? Gl[k] : 0.0)) * idx
                                        : vk[j] * ((Gr ? Gr[k] : 0.0) - gi[j]) * idx;
                    const double w = (vk[j] - u) * ist;
                    const double b3 = 1.4142135623730950488 * (0.5 * w * w - 0.5);
                    s1 += z[j]; s2 += z[j] * w; s3 += z[j] * b3;
                }
            }
            // split fluxes of the cell (independent of the sums: overlaps them)
            double Ap[3], Am[3];
            split_flux(rho, u, T, Ap, Am);
            s1 = warp_sum(s1); s2 = warp_sum(s2); s3 = warp_sum(s3);
            const double scale = g.dv / rho;
            const double a1 = s1 * scale, a2 = s2 * scale, a3 = s3 * scale;
            // at a non-periodic edge iface_T uses the cell's own state (P)
            const double thl = iface_T(g, i, Pl, P);
            const double thr = iface_T(g, i + 1, P, Pr);
            const double dT = (thr - thl) / (g.dx * T);
            const double denom = g.eps + a.dt * tau;
            const double wg = g.eps / denom, wh = a.dt * tau / denom;
            const double pref = rho / sqrt(2.0 * kPi * T);
            const double i2T = 1.0 / (2.0 * T);
            const double gq = dT / tau;
            double* Go = Gnxt + (size_t)nv * lc;
            double hsum = 0.0;
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const int k = lane + 32 * j;
                if (k < nv) {
                    const double wv = vk[j] - u;
                    const double w = wv * ist;
                    const double b3 = 1.4142135623730950488 * (0.5 * w * w - 0.5);
                    const double M = pref * exp(-(wv * wv) * i2T);
                    const double zh = (a1 + w * a2 + b3 * a3) * M;
                    const double gh = -((wv * wv * wv) * i2T - 1.5 * wv) * gq * M;
                    const double gp = wg * (gi[j] - a.dt * (z[j] - zh)) + wh * gh;
                    Go[k] = gp;
                    hsum += gp * v3k[j];
                }
            }
            hsum = warp_sum(hsum);
            if (lane < 3) {
                Fl[8 * lc + lane] = Ap[lane];
                Fl[8 * lc + 3 + lane] = Am[lane];
            }
            if (lane == 3) Fl[8 * lc + 6] = 0.5 * g.eps * g.dv * hsum;
            // diffuse-wall ghost-state fluxes (interface_fluxes_1d, macro1d.py:66-75)
            if (i == 0 && g.face[0] == 2) {
                double Wp[3], Wm[3];
                split_flux(wall_rho(P, g.wallT[0], false), 0.0, g.wallT[0], Wp, Wm);
                if (lane < 3) Fe[lane] = Wp[lane];
            }
            if (i == g.nx - 1 && g.face[1] == 2) {
                double Wp[3], Wm[3];
                split_flux(wall_rho(P, g.wallT[1], true), 0.0, g.wallT[1], Wp, Wm);
                if (lane < 3) Fe[4 + lane] = Wm[lane];
            }
        }
        cl.sync();
        // ---- phase B: macro update of the cell, primitives for the next step ----
        for (int lc = tid; lc < cnt; lc += blockDim.x) {
            const int i = c0 + lc;
            const double* FlL = remote(Fl, nb1(g, i - 1), 8);
            const double* FlR = remote(Fl, nb1(g, i + 1), 8);
            const double* me = Fl + 8 * lc;
            const double* ApL = (i == 0 && g.face[0] == 2) ? Fe0 : FlL;       // A+ of the left state
            const double* AmR = (i == g.nx - 1 && g.face[1] == 2) ? Fe1 : FlR + 3;
            const double h = me[6];
            const double Hm = iface_heat(g, i, FlL[6], h);
            const double Hp = iface_heat(g, i + 1, h, FlR[6]);
            double q[3];
#pragma unroll
            for (int m = 0; m < 3; ++m) {
                const double Fm = ApL[m] + me[3 + m];
                const double Fp = me[m] + AmR[m];
                q[m] = Qs[3 * lc + m] - r * (Fp - Fm);
            }
            q[2] -= r * (Hp - Hm);
#pragma unroll
            for (int m = 0; m < 3; ++m) Qs[3 * lc + m] = q[m];
            const Prim1 P = prim1(q);
            Ps[4 * lc] = P.rho; Ps[4 * lc + 1] = P.u; Ps[4 * lc + 2] = P.T;
            if (!(P.rho > 0.0)) raise(E1_DENSITY, i);
            else if (!(P.T > 0.0)) raise(E1_TEMPERATURE, i);
        }
        cl.sync();
        cur ^= 1;
        ++completed;
    }
    const double* Gf = cur ? Gs1 : Gs0;
    for (int n = tid; n < cnt * nv; n += blockDim.x) a.G[(size_t)c0 * nv + n] = Gf[n];
    for (int n = tid; n < cnt * 3; n += blockDim.x) a.Q[(size_t)c0 * 3 + n] = Qs[n];
    for (int n = tid; n < cnt; n += blockDim.x) a.H[c0 + n] = Fl[8 * n + 6];
    if (rank == 0 && tid == 0) {
        *a.done = completed;
        if (*flag) a.err[1] = (unsigned long long)(size_t)a.Q;
    }
    cl.sync();   // keep every CTA's shared memory alive until remote readers are done
}

}  // namespace d1
}  // namespace mm2d
