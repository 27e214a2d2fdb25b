// Macro update: Strang-split TR-BDF2 pressure relaxation around KFVS x and y
// sweeps of the 6-moment system, with the micro-supplied heat tensor as
// interface-averaged sources (macro2d.py:224-240).
//
// Two kernels, one thread per cell:
//   k_macro_x: Q* = relax(Q^n) on the 3-cell x stencil, KFVS x-fluxes,
//              heat divergence -> Q** (written to the Qx ring; also on the
//              ghost rows when the y face is a received halo, like the
//              worker-grid's extended-range x-sweep, parallel.py:305-313)
//   k_macro_y: KFVS y-fluxes on Q**, heat divergence, [+dt*source],
//              final relax -> Q^{n+1}
// The macro state is ~1% of the bytes of G, so these are latency-bound
// tiny kernels; the arithmetic mirrors the reference's NumPy expression
// order so results agree to a few ulps.
#pragma once
#include "mm2d_common.cuh"
#include "mm2d_prep.cuh"

namespace mm2d {

struct MacroArgs {
    Geometry g;
    const double* Qr;       // ring Q^n
    const double* Hr;       // ring heat tensor (AoS)
    double* Qx;             // ring Q** (x-swept)
    double* Hout;           // (4, bx, by) heat tensor output (SoA) or null
    double* Qout;           // (bx, by, 6)
    const double* qsrc;     // (bx, by, 6) or null
    unsigned long long* err;
    double dt, eps, nu, rx, ry;   // rx = dt/dx, ry = dt/dy
    int tau_kind;
    double tau_value;
    unsigned step;
};

// relax_pressure_2d (macro2d.py:55-70) on one cell
__device__ __forceinline__ void relax_cell(const MacroArgs& a, const double* q, double* o) {
    double rho, u1, u2, t11, t12, t22;
    prims_fast(q, rho, u1, u2, t11, t12, t22);
    const double T = 0.5 * (t11 + t22);
    const double tau = tau_model(a.tau_kind, a.tau_value, rho, T);
    const double z = tau * (1.0 - a.nu) * a.dt;
    const double e2 = 48.0 * a.eps * a.eps;
    const double W = (e2 - 10.0 * z * a.eps) / (e2 + 14.0 * z * a.eps + z * z);
    const double p11 = rho * t11, p12 = rho * t12, p22 = rho * t22;
    o[0] = q[0]; o[1] = q[1]; o[2] = q[2];
    o[3] = rho * u1 * u1 + 0.5 * ((1.0 + W) * p11 + (1.0 - W) * p22);
    o[4] = rho * u1 * u2 + W * p12;
    o[5] = rho * u2 * u2 + 0.5 * ((1.0 - W) * p11 + (1.0 + W) * p22);
}

// pressure-primitive state (rho, u1, u2, P11, P12, P22) of a conserved
// vector (_pressure_fields, macro2d.py:201-203)
__device__ __forceinline__ void pstate(const double* q, double* s) {
    double rho, u1, u2, t11, t12, t22;
    prims_fast(q, rho, u1, u2, t11, t12, t22);
    s[0] = rho; s[1] = u1; s[2] = u2;
    s[3] = rho * t11; s[4] = rho * t12; s[5] = rho * t22;
}

// validity of a conserved vector (primitives_2d checks)
__device__ __forceinline__ int bad_state(const double* q) {
    if (!(q[0] > 0.0)) return 1;
    double rho, u1, u2, t11, t12, t22;
    prims_of(q, rho, u1, u2, t11, t12, t22);
    const double tol = 1e-14 * (t11 + t22);
    const double det = t11 * t22 - t12 * t12;
    return ((t11 <= tol) || (det <= tol * tol)) ? 2 : 0;
}

// diffuse-wall ghost pressure state from the current-stage edge state
// (_extended_states, macro2d.py:153-181 with wall_ghost_state_2d)
__device__ __forceinline__ void wall_pstate(const Geometry& g, int face, const double* edge,
                                            double* s) {
    const double rho = edge[0];
    const double t11 = edge[3] / rho, t22 = edge[5] / rho;
    const double Tw = g.wallT[face], U = g.wallU[face];
    const double sign = (face == 0 || face == 2) ? -1.0 : 1.0;
    double rw;
    if (face < 2) { rw = wall_density(rho, edge[1], t11, Tw, sign); s[1] = 0.0; s[2] = U; }
    else { rw = wall_density(rho, edge[2], t22, Tw, sign); s[1] = U; s[2] = 0.0; }
    s[0] = rw; s[3] = rw * Tw; s[4] = rw * 0.0; s[5] = rw * Tw;
}

// one side's share of the KFVS flux: _split_parts_x/_y + _kfvs
// (macro2d.py:102-138), sgn = +1 for the left/lower state, -1 for right/upper
template <int AXIS>
__device__ __forceinline__ void kfvs_half(const double* s, double sgn, double* out) {
    const double rho = s[0], u1 = s[1], u2 = s[2], p11 = s[3], p12 = s[4], p22 = s[5];
    double a, b, J[6], K[6];
    // two divisions per half (1/rho, 1/P_aa) instead of four
    const double irho = 1.0 / rho;
    if (AXIS == 0) {
        const double rp = 1.0 / p11;
        const double h = 0.5 * rho * rp;         // rho / (2 P11)
        a = sqrt((2.0 / kPi) * p11 * irho) * exp(-u1 * u1 * h);
        b = erf(u1 * sqrt(h));
        J[0] = rho; J[1] = rho * u1; J[2] = rho * u2;
        J[3] = rho * u1 * u1 + 2.0 * p11;
        J[4] = rho * u1 * u2 + 2.0 * p12;
        J[5] = rho * u2 * u2 + p22 + p12 * p12 * rp;
        K[0] = rho * u1; K[1] = rho * u1 * u1 + p11; K[2] = rho * u1 * u2 + p12;
        K[3] = rho * (u1 * u1 * u1) + 3.0 * u1 * p11;
        K[4] = rho * u1 * u1 * u2 + u2 * p11 + 2.0 * u1 * p12;
        K[5] = rho * u1 * u2 * u2 + u1 * p22 + 2.0 * u2 * p12;
    } else {
        const double rp = 1.0 / p22;
        const double h = 0.5 * rho * rp;         // rho / (2 P22)
        a = sqrt((2.0 / kPi) * p22 * irho) * exp(-u2 * u2 * h);
        b = erf(u2 * sqrt(h));
        J[0] = rho; J[1] = rho * u1; J[2] = rho * u2;
        J[3] = rho * u1 * u1 + p11 + p12 * p12 * rp;
        J[4] = rho * u1 * u2 + 2.0 * p12;
        J[5] = rho * u2 * u2 + 2.0 * p22;
        K[0] = rho * u2; K[1] = rho * u1 * u2 + p12; K[2] = rho * u2 * u2 + p22;
        K[3] = rho * u1 * u1 * u2 + u2 * p11 + 2.0 * u1 * p12;
        K[4] = rho * u1 * u2 * u2 + u1 * p22 + 2.0 * u2 * p12;
        K[5] = rho * (u2 * u2 * u2) + 3.0 * u2 * p22;
    }
    const double sa = sgn * a, sb = 1.0 + sgn * b;
#pragma unroll
    for (int m = 0; m < 6; ++m) out[m] = 0.5 * (sa * J[m] + sb * K[m]);
}

// Tiled sweeps: every cell's relaxed state, pressure state and both KFVS
// half fluxes are computed ONCE and shared with the neighbours (shared
// memory along x, warp shuffles along y), instead of each cell recomputing
// its neighbours' (3 relaxations and 4 half fluxes per cell before).  The
// interface flux keeps the expression (0 + L_left) + R_right, so results are
// bitwise those of the untiled kernels.
#ifndef MM2D_MX_TI
#define MM2D_MX_TI 10   // tile rows along x: 6 / 8 / 10 / 12 / 14 -> 0.263 / 0.295 / 0.255 / 0.314 / 0.285 ms at C5
#endif
#ifndef MM2D_MX_MINB
#define MM2D_MX_MINB 0   // 0: no minimum (58 registers, the fastest: 0.294 ms at C5; 6 -> 0.318, tiles of 12 -> 0.320)
#endif
#if MM2D_MX_MINB > 0
#define MM2D_MX_BOUNDS __launch_bounds__(MX_TJ * (MX_TI + 2), MM2D_MX_MINB)
#else
#define MM2D_MX_BOUNDS __launch_bounds__(MX_TJ * (MX_TI + 2))
#endif
constexpr int MX_TI = MM2D_MX_TI;        // output cells per CTA along x
constexpr int MX_TJ = 32;                // cells per CTA along y (one warp row)

// x-sweep: block (32, MX_TI + 2); thread (lane, r) owns cell (i0 - 1 + r, j)
__global__ void MM2D_MX_BOUNDS k_macro_x(MacroArgs a) {
    pdl_enter();
    __shared__ double sL[MX_TI + 2][6][MX_TJ], sR[MX_TI + 2][6][MX_TJ];
    const Geometry& g = a.g;
    if (err_gate(a.err, EW_PREP)) return;
    const int jlo = g.qylo == GM_HALO ? -1 : 0;
    const int jhi = g.qyhi == GM_HALO ? g.by : g.by - 1;
    const int lane = threadIdx.x, r = threadIdx.y;
    const int i = blockIdx.x * MX_TI - 1 + r;
    const int j = jlo + blockIdx.y * MX_TJ + lane;
    const bool jok = j <= jhi;
    const bool out = jok && r >= 1 && r <= MX_TI && i < g.bx;
    double qc[6];
    if (jok && i >= -1 && i <= g.bx) {
        double s[6], L[6], R[6];
        if (i == -1 && g.wall[0]) {              // diffuse wall: from the edge cell
            double qe[6], se[6];
            relax_cell(a, a.Qr + 6 * ring_index(g, 0, j), qe);
            pstate(qe, se);
            wall_pstate(g, 0, se, s);
        } else if (i == g.bx && g.wall[1]) {
            double qe[6], se[6];
            relax_cell(a, a.Qr + 6 * ring_index(g, g.bx - 1, j), qe);
            pstate(qe, se);
            wall_pstate(g, 1, se, s);
        } else {
            relax_cell(a, a.Qr + 6 * ring_index(g, i, j), qc);
            pstate(qc, s);
        }
        kfvs_half<0>(s, 1.0, L);
        kfvs_half<0>(s, -1.0, R);
#pragma unroll
        for (int m = 0; m < 6; ++m) { sL[r][m][lane] = L[m]; sR[r][m][lane] = R[m]; }
    }
    __syncthreads();
    if (!out) return;
    if (j >= 0 && j < g.by) {
        const int bs = bad_state(qc);
        if (bs) {
            const unsigned long long gcell =
                (unsigned long long)(g.i0 + i) * g.ny + (unsigned long long)(g.j0 + j);
            atomicMin(a.err + EW_MX, err_key(a.step, bs == 1 ? ES_XS_RHO : ES_XS_SPD, gcell));
        }
    }
    MM2D_CHECK(i >= -1 && i <= g.bx && j >= -1 && j <= g.by);
    double* o = a.Qx + 6 * ring_index(g, i, j);
#pragma unroll
    for (int m = 0; m < 6; ++m) {
        const double Fm = (0.0 + sL[r - 1][m][lane]) + sR[r][m][lane];
        const double Fp = (0.0 + sL[r][m][lane]) + sR[r + 1][m][lane];
        o[m] = qc[m] - a.rx * (Fp - Fm);
    }
    // heat: interface means of H111, H112, H122 (x-sweep sources); ghost
    // cells resolved on the fly (interface_heat_2d rules)
    double hc[4], hl[4], hr[4];
    load_ring_h(g, a.Hr, i, j, hc);
    load_ring_h(g, a.Hr, i - 1, j, hl);
    load_ring_h(g, a.Hr, i + 1, j, hr);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double hp = 0.5 * (hr[c] + hc[c]);
        const double hm = 0.5 * (hc[c] + hl[c]);
        o[3 + c] -= a.rx * (hp - hm);
    }
}

// y-sweep: one warp per 30 output cells along y; lane l owns cell
// j0 - 1 + l and takes its neighbours' half fluxes by shuffles
constexpr int MY_OUT = 30;
#ifndef MM2D_MY_MINB
#define MM2D_MY_MINB 8   // 64 registers (a few spills): 0.273 -> 0.230 ms at C5; 6: 0.247
#endif
__global__ void __launch_bounds__(128, MM2D_MY_MINB) k_macro_y(MacroArgs a) {
    pdl_enter();
    const Geometry& g = a.g;
    if (err_gate(a.err, EW_MX)) return;
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.y * 4 + (threadIdx.x >> 5);
    if (i >= g.bx) return;                       // warp-uniform
    const int j = blockIdx.x * MY_OUT - 1 + lane;
    const int n = g.bx * g.by;
    double qc[6], s[6], L[6], R[6];
    const bool own = j >= 0 && j < g.by;
    if (own) {
#pragma unroll
        for (int m = 0; m < 6; ++m) qc[m] = a.Qx[6 * ring_index(g, i, j) + m];
        pstate(qc, s);
    } else if (j == -1 || j == g.by) {
        const bool lo = j < 0;
        const int mode = lo ? g.qylo : g.qyhi;
        if (mode == GM_HALO || mode == GM_WRAP) {
            const int jj = mode == GM_HALO ? j : (lo ? g.by - 1 : 0);
            pstate(a.Qx + 6 * ring_index(g, i, jj), s);
        } else {
            double se[6];
            pstate(a.Qx + 6 * ring_index(g, i, lo ? 0 : g.by - 1), se);
            if (g.wall[lo ? 2 : 3]) wall_pstate(g, lo ? 2 : 3, se, s);
            else for (int m = 0; m < 6; ++m) s[m] = se[m];
            if (mode == GM_MIRROR) { s[2] = -s[2]; s[4] = -s[4]; }   // specular image
        }
    } else {
        for (int m = 0; m < 6; ++m) s[m] = 1.0;   // beyond the ring: unused
        s[1] = s[2] = s[4] = 0.0;
    }
    kfvs_half<1>(s, 1.0, L);
    kfvs_half<1>(s, -1.0, R);
    double Ld[6], Ru[6];
#pragma unroll
    for (int m = 0; m < 6; ++m) {
        Ld[m] = __shfl_up_sync(0xffffffffu, L[m], 1);
        Ru[m] = __shfl_down_sync(0xffffffffu, R[m], 1);
    }
    if (!own || lane == 0 || lane == 31) return;
    const int t = i * g.by + j;
    const unsigned long long gcell =
        (unsigned long long)(g.i0 + i) * g.ny + (unsigned long long)(g.j0 + j);
    {
        const int bs = bad_state(qc);
        if (bs) atomicMin(a.err + EW_MY, err_key(a.step, bs == 1 ? ES_YS_RHO : ES_YS_SPD, gcell));
    }
    double q3[6];
#pragma unroll
    for (int m = 0; m < 6; ++m) {
        const double Fm = (0.0 + Ld[m]) + R[m];
        const double Fp = (0.0 + L[m]) + Ru[m];
        q3[m] = qc[m] - a.ry * (Fp - Fm);
    }
    MM2D_CHECK(i >= 0 && i < g.bx && j >= -1 && j <= g.by);
    const double* hc = a.Hr + 4 * ring_index(g, i, j);
    double hd[4], hu[4];
    load_ring_h(g, a.Hr, i, j - 1, hd);
    load_ring_h(g, a.Hr, i, j + 1, hu);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const double hp = 0.5 * (hu[c + 1] + hc[c + 1]);
        const double hm = 0.5 * (hc[c + 1] + hd[c + 1]);
        q3[3 + c] -= a.ry * (hp - hm);
    }
    if (a.qsrc) {
        const double* sq = a.qsrc + 6 * ((size_t)i * g.by + j);
#pragma unroll
        for (int m = 0; m < 6; ++m) q3[m] = q3[m] + a.dt * sq[m];
    }
    // the step's heat tensor, SoA (4, bx, by) (macro2d.py:23-29)
    if (a.Hout) {
#pragma unroll
        for (int c = 0; c < 4; ++c) a.Hout[(size_t)c * n + t] = hc[c];
    }
    double* qo = a.Qout + 6 * ((size_t)i * g.by + j);
    const int bs3 = bad_state(q3);
    if (bs3) {
        // keep Q*** so the host can report the offending value
        atomicMin(a.err + EW_MY, err_key(a.step, bs3 == 1 ? ES_RL_RHO : ES_RL_SPD, gcell));
        for (int m = 0; m < 6; ++m) qo[m] = q3[m];
    } else {
        relax_cell(a, q3, qo);
    }
}

}  // namespace mm2d
