// Ring fill and per-cell preparation kernels (macro state at t^n).
#pragma once
#include "mm2d_common.cuh"

namespace mm2d {

// Resolve ring cell (i, j) of a field whose ghost rules are (mxlo, mxhi,
// mylo, myhi) -- the rules of extract_ring (parallel.py:109-150), which for
// a single rank reduce to the serial ghost rules (boundary.py:181-241):
// y is resolved first, then x within the resolved row.
//   returns 0: interior cell (si, sj) of the source block
//           1: ring cell (si, sj) that holds received halo data
//           2: zero
// flip: bit 0 the source is mirrored in v1 (specular x face), bit 1 in v2.
enum { RS_INTERIOR = 0, RS_RING = 1, RS_ZERO = 2 };

__device__ __forceinline__ int resolve_ring(int bx, int by, int mxlo, int mxhi, int mylo,
                                            int myhi, int i, int j, int& si, int& sj,
                                            int& flip) {
    bool yhalo = false;
    int jj = j;
    flip = 0;
    if (j < 0 || j >= by) {
        const int m = j < 0 ? mylo : myhi;
        if (m == GM_ZERO) return RS_ZERO;
        if (m == GM_HALO) yhalo = true;
        else if (m == GM_WRAP) jj = (j + by) % by;
        else jj = j < 0 ? 0 : by - 1;
        if (m == GM_MIRROR) flip |= 2;
    }
    int ii = i;
    if (i < 0 || i >= bx) {
        const int m = i < 0 ? mxlo : mxhi;
        if (m == GM_ZERO) return RS_ZERO;
        if (m == GM_HALO) { si = i; sj = jj; return RS_RING; }
        if (m == GM_WRAP) ii = (i + bx) % bx;
        else ii = i < 0 ? 0 : bx - 1;
        if (m == GM_MIRROR) flip |= 1;
    }
    si = ii; sj = jj;
    return yhalo ? RS_RING : RS_INTERIOR;
}

// sign of conserved component c of a mirrored ghost: rho u1 flips with v1,
// rho u2 with v2, E12 with either
__device__ __forceinline__ double q_mirror_sign(int c, int flip) {
    const int odd = (c == 1 ? (flip & 1) : 0) ^ (c == 2 ? (flip >> 1) : 0) ^
                    (c == 4 ? ((flip & 1) ^ (flip >> 1)) : 0);
    return odd ? -1.0 : 1.0;
}
// heat component c (H111, H112, H122, H222): odd in v1 for c = 0, 2, odd in
// v2 for c = 1, 3
__device__ __forceinline__ double h_mirror_sign(int c, int flip) {
    const int odd = ((c == 0 || c == 2) ? (flip & 1) : (flip >> 1));
    return odd ? -1.0 : 1.0;
}

// Conserved state of ring cell (i, j) resolved from the owned block Q or a
// received halo cell of the ring (never a cell this step writes), with the
// specular signs applied.  Returns false if (i, j) is itself a received cell.
__device__ __forceinline__ bool load_ring_q(const Geometry& g, const double* __restrict__ Q,
                                            const double* Qr, int i, int j, double* q) {
    int si, sj, flip;
    const int rs = resolve_ring(g.bx, g.by, g.qxlo, g.qxhi, g.qylo, g.qyhi, i, j, si, sj, flip);
    const double* src;
    bool own_copy = true;
    if (rs == RS_INTERIOR) {
        src = Q + 6 * ((size_t)si * g.by + sj);
    } else if (rs == RS_RING) {
        src = Qr + 6 * ring_index(g, si, sj);
        own_copy = !(si == i && sj == j);
    } else {
#pragma unroll
        for (int c = 0; c < 6; ++c) q[c] = 0.0;
        return true;
    }
#pragma unroll
    for (int c = 0; c < 6; ++c) q[c] = flip ? q_mirror_sign(c, flip) * src[c] : src[c];
    return own_copy;
}

// Fill the ghost ring of Hr (owned part written by the micro kernel).
// Heat ghosts: periodic wrap, extrapolate copy, wall zero, i.e. the rules of
// interface_heat_2d (boundary.py:224-241): the interface value is the mean
// of the two neighbours, which at a wall is half the edge value.
__global__ void k_fill_hring(Geometry g, double* __restrict__ Hr) {
    const int n = (g.bx + 2) * (g.by + 2);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const int i = t / (g.by + 2) - 1, j = t % (g.by + 2) - 1;
        if (i >= 0 && i < g.bx && j >= 0 && j < g.by) continue;
        int si, sj, flip;
        const int rs = resolve_ring(g.bx, g.by, g.hxlo, g.hxhi, g.hylo, g.hyhi, i, j, si, sj, flip);
        double* dst = Hr + 4 * t;
        if (rs == RS_ZERO) {
#pragma unroll
            for (int c = 0; c < 4; ++c) dst[c] = 0.0;
        } else {
            if (rs == RS_RING && si == i && sj == j) continue;
            const double* src = Hr + 4 * ring_index(g, si, sj);
#pragma unroll
            for (int c = 0; c < 4; ++c) dst[c] = flip ? h_mirror_sign(c, flip) * src[c] : src[c];
        }
    }
}

// Heat tensor of ring cell (i, j): owned and received cells from the ring,
// ghosts resolved on the fly (wrap / copy / zero / specular image), which is
// what the ring fill k_fill_hring stores.
__device__ __forceinline__ void load_ring_h(const Geometry& g, const double* Hr, int i, int j,
                                            double* h) {
    int si, sj, flip;
    const int rs = resolve_ring(g.bx, g.by, g.hxlo, g.hxhi, g.hylo, g.hyhi, i, j, si, sj, flip);
    if (rs == RS_ZERO) {
#pragma unroll
        for (int c = 0; c < 4; ++c) h[c] = 0.0;
        return;
    }
    const double* src = Hr + 4 * ring_index(g, si, sj);
#pragma unroll
    for (int c = 0; c < 4; ++c) h[c] = flip ? h_mirror_sign(c, flip) * src[c] : src[c];
}

struct PrepArgs {
    Geometry g;
    const double* Q;              // owned block (bx, by, 6)
    double* Qr;                   // ring, written here (received halo cells kept)
    CellPar* P;
    unsigned long long* err;      // the context's error words (ErrWord)
    unsigned long long* iso;      // [4]: max|m11-T|, max|m12|, max|m22-T|, max T (bit patterns)
    double dt, eps, nu, dv;
    int tau_kind;
    double tau_value;
    unsigned step;
    int gauss;                    // nu != 0
    double h2x, h2y;              // 1 / (2 dx), 1 / (2 dy)
};

__device__ __forceinline__ double tau_model(int kind, double value, double rho, double T) {
    switch (kind) {
        case 0: return 3.2 * sqrt(T / (2.0 * kPi));            // hard_sphere_1d
        case 1: return rho * T;                                // pressure_1d
        case 2: return (0.4625 * kPi) * rho;                   // esbgk_2d
        case 3: return (3.0 * kPi * 0.436 / sqrt(2.0)) * rho;  // bgk_2d
        default: return value;                                 // constant
    }
}

// wall_density_ratio_2d (boundary.py:248-260) times rho
__device__ __forceinline__ double wall_density(double rho, double ua, double taa, double Tw,
                                               double sign) {
    double R = sqrt(taa / Tw) * exp(-ua * ua / (2.0 * taa)) +
               ua * sqrt(kPi / (2.0 * Tw)) * (erf(ua / sqrt(2.0 * taa)) + sign);
    return rho * R;
}

__device__ __forceinline__ void prims_of(const double* q, double& rho, double& u1, double& u2,
                                         double& t11, double& t12, double& t22) {
    rho = q[0];
    u1 = q[1] / rho;
    u2 = q[2] / rho;
    t11 = q[3] / rho - u1 * u1;
    t12 = q[4] / rho - u1 * u2;
    t22 = q[5] / rho - u2 * u2;
}

// Primitives with one reciprocal of rho instead of five divisions (~1 ulp
// from prims_of).  Used where the result only feeds the evolution (neighbour
// gradients, relaxation, KFVS states); every validity check and every
// reported InvalidStateError value goes through the exact prims_of.
__device__ __forceinline__ void prims_fast(const double* q, double& rho, double& u1, double& u2,
                                           double& t11, double& t12, double& t22) {
    rho = q[0];
    const double ir = 1.0 / rho;
    u1 = q[1] * ir;
    u2 = q[2] * ir;
    t11 = q[3] * ir - u1 * u1;
    t12 = q[4] * ir - u1 * u2;
    t22 = q[5] * ir - u2 * u2;
}

// Per ring cell: primitives, tau, Maxwellian and Gaussian prefactors, relax
// weights; per owned cell also the centred gradients (micro2d.py:37-60),
// the modified tensor with its SPD check (gas_state.py:138-146), the
// isotropy maxima (micro2d.py:63-67) and the diffuse-wall ghost densities
// of edge cells (boundary.py:248-290).
//
// NB holds the neighbour primitives of an owned cell: nb(s, d, k) is
// component k (u1, u2, T) of the neighbour at offset s ? +1 : -1 along axis d
// (0 x, 1 y), as prims_fast gives them.
template <class NB, class ST>
__device__ __forceinline__ void prep_cell(const PrepArgs& a, int t, int i, int j, const NB& nb,
                                          const ST& store) {
    const Geometry& g = a.g;
    {
        const bool own = i >= 0 && i < g.bx && j >= 0 && j < g.by;
        // the ring fill (extract_ring rules) fused in: this cell's state from
        // Q / a received halo cell, written to the ring for the macro sweeps
        double q[6];
        if (load_ring_q(g, a.Q, a.Qr, i, j, q)) {
#pragma unroll
            for (int c = 0; c < 6; ++c) a.Qr[6 * t + c] = q[c];
        }
        CellPar P;
        double rho, u1, u2, t11, t12, t22;
        rho = q[0];
        const unsigned long long gcell =
            (unsigned long long)(g.i0 + i) * g.ny + (unsigned long long)(g.j0 + j);
        if (own && !(rho > 0.0)) atomicMin(a.err + EW_PREP, err_key(a.step, ES_PRIM_RHO, gcell));
        prims_of(q, rho, u1, u2, t11, t12, t22);
        const double T = 0.5 * (t11 + t22);
        if (own) {
            const double tol = 1e-14 * (t11 + t22);
            const double det = t11 * t22 - t12 * t12;
            if ((t11 <= tol) || (det <= tol * tol)) atomicMin(a.err + EW_PREP, err_key(a.step, ES_PRIM_SPD, gcell));
        }
        P.u1 = u1; P.u2 = u2;
        // reciprocals shared between the derived constants (each division
        // costs ~40 instructions with its slow-path guard)
        const double invT = 1.0 / T;
        P.isT = rsqrt(T);
        P.invT = invT;
        P.inv2T = 0.5 * invT;                   // == 1 / (2T) exactly
        P.pref = rho * invT * (0.5 / kPi);
        const double tau = tau_model(a.tau_kind, a.tau_value, rho, T);
        P.tau = tau;
        P.invtau = 1.0 / tau;
        P.scale = a.dv / rho;
        const double rden = 1.0 / (a.eps + a.dt * tau);
        P.wg = a.eps * rden;
        P.wh = a.dt * tau * rden;
        P.s11 = P.s12 = P.gT1 = P.gT2 = 0.0;
        P.gpref = P.gq11 = P.gq22 = P.gq12 = 0.0;
        P.rw[0] = P.rw[1] = P.rw[2] = P.rw[3] = 0.0;
        P.pad = 0.0;
        if (a.gauss) {
            const double m11 = (1.0 - a.nu) * T + a.nu * t11;
            const double m12 = a.nu * t12;
            const double m22 = (1.0 - a.nu) * T + a.nu * t22;
            const double det = m11 * m22 - m12 * m12;
            const double rdet = 1.0 / det;
            P.gpref = rho * (0.5 / kPi) * rsqrt(det);
            P.gq11 = -0.5 * m22 * rdet;  // coefficient of W1^2 in the exponent
            P.gq22 = -0.5 * m11 * rdet;  // coefficient of W2^2
            P.gq12 = m12 * rdet;         // coefficient of W1 W2
            if (own) {
                const double tol = 1e-14 * (m11 + m22);
                if ((m11 <= tol) || (det <= tol * tol))
                    atomicMin(a.err + EW_PREP, err_key(a.step, ES_MOD_SPD, gcell));
                if (a.eps < 1e-10) {
                    atomic_max_pos(&a.iso[0], fabs(m11 - T));
                    atomic_max_pos(&a.iso[1], fabs(m12));
                    atomic_max_pos(&a.iso[2], fabs(m22 - T));
                    atomic_max_pos(&a.iso[3], T > 0.0 ? T : 0.0);
                }
            }
        }
        if (own) {
            // centred differences over the ring (extend_macro_scalar_2d:
            // wrap for periodic, copy otherwise)
            double xu1[2], xu2[2], xT[2], yu1[2], yu2[2], yT[2];
            for (int s = 0; s < 2; ++s) {
                xu1[s] = nb(s, 0, 0); xu2[s] = nb(s, 0, 1); xT[s] = nb(s, 0, 2);
                yu1[s] = nb(s, 1, 0); yu2[s] = nb(s, 1, 1); yT[s] = nb(s, 1, 2);
            }
            const double du1x = (xu1[1] - xu1[0]) * a.h2x;
            const double du2x = (xu2[1] - xu2[0]) * a.h2x;
            const double du1y = (yu1[1] - yu1[0]) * a.h2y;
            const double du2y = (yu2[1] - yu2[0]) * a.h2y;
            P.s11 = du1x - du2y;
            P.s12 = du1y + du2x;
            P.gT1 = (xT[1] - xT[0]) * a.h2x;
            P.gT2 = (yT[1] - yT[0]) * a.h2y;
            // wall ghost densities of edge cells (zero-mass-flux closure)
            if (g.wall[0] && i == 0) P.rw[0] = wall_density(rho, u1, t11, g.wallT[0], -1.0);
            if (g.wall[1] && i == g.bx - 1) P.rw[1] = wall_density(rho, u1, t11, g.wallT[1], 1.0);
            if (g.wall[2] && j == 0) P.rw[2] = wall_density(rho, u2, t22, g.wallT[2], -1.0);
            if (g.wall[3] && j == g.by - 1) P.rw[3] = wall_density(rho, u2, t22, g.wallT[3], 1.0);
        }
        store(P);
    }
}

// (u1, u2, T) of ring cell (i, j) as the centred gradients use them
__device__ __forceinline__ void nb_prims(const PrepArgs& a, int i, int j, double* w) {
    double qn[6], r_, a11, a12, a22;
    load_ring_q(a.g, a.Q, a.Qr, i, j, qn);
    prims_fast(qn, r_, w[0], w[1], a11, a12, a22);
    w[2] = 0.5 * (a11 + a22);
}

// One thread per ring cell; each owned cell re-derives its four neighbours'
// primitives from Q (the reference's extend + centred difference).
__global__ void k_prep(PrepArgs a) {
    pdl_enter();
    const Geometry& g = a.g;
    if (err_gate(a.err, EW_MY)) return;   // failed in an earlier launch
    const int n = (g.bx + 2) * (g.by + 2);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const int i = t / (g.by + 2) - 1, j = t % (g.by + 2) - 1;
        double w[2][2][3];
        if (i >= 0 && i < g.bx && j >= 0 && j < g.by) {
            for (int s = 0; s < 2; ++s) {
                nb_prims(a, i + (s ? 1 : -1), j, w[s][0]);
                nb_prims(a, i, j + (s ? 1 : -1), w[s][1]);
            }
        }
        prep_cell(a, t, i, j, [&](int s, int d, int k) { return w[s][d][k]; },
                  [&](const CellPar& P) {
                      MM2D_CHECK(t >= 0 && t < n);
                      reinterpret_cast<CellPar*>(a.P)[t] = P;
                  });
    }
}

// Tiled variant: a CTA owns a PT_I x PT_J tile of ring cells.  It first
// derives (u1, u2, T) once per cell of the tile plus its one-cell halo into
// shared memory, then every cell of the tile reads its neighbours from
// there: one Q load and one primitive evaluation per cell instead of five,
// and the same prims_fast arithmetic, so the CellPar bits are unchanged.
#ifndef MM2D_PREP_TI
#define MM2D_PREP_TI 4   // tile rows (warps per CTA); 4 measured faster than 8
#endif
constexpr int PT_I = MM2D_PREP_TI, PT_J = 32, PT_THREADS = PT_I * PT_J;
constexpr size_t kPrepStageBytes = sizeof(double) * 32 * PT_THREADS;   // 32-double rows (swizzled)

__device__ __forceinline__ int prep_tiles(const Geometry& g) {
    return ((g.bx + 2 + PT_I - 1) / PT_I) * ((g.by + 2 + PT_J - 1) / PT_J);
}

// (resident-CTA minimums measured slower: 6 -> +5 %, 8 -> +15 %; an explicit 1 lets
// ptxas take more registers and is slower too)
__global__ void __launch_bounds__(PT_THREADS) k_prep_tiled(PrepArgs a) {
    pdl_enter();
    const Geometry& g = a.g;
    if (err_gate(a.err, EW_MY)) return;   // failed in an earlier launch
    __shared__ double sw[3][PT_I + 2][PT_J + 2];
    extern __shared__ double stage[];   // [PT_THREADS][32] CellPar staging (swizzled)
    const int ntj = (g.by + 2 + PT_J - 1) / PT_J;
    const int ntiles = prep_tiles(g);
    const int li = threadIdx.x / PT_J, lj = threadIdx.x % PT_J;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int ri0 = (tile / ntj) * PT_I, rj0 = (tile % ntj) * PT_J;
        __syncthreads();   // the previous tile's readers are done
        // halo cell (hi, hj) is cell (ri0 + hi - 2, rj0 + hj - 2); only the
        // neighbours of owned cells, i in [-1, bx] and j in [-1, by], are used
        for (int h = threadIdx.x; h < (PT_I + 2) * (PT_J + 2); h += PT_THREADS) {
            const int hi = h / (PT_J + 2), hj = h % (PT_J + 2);
            const int i = ri0 + hi - 2, j = rj0 + hj - 2;
            if (i < -1 || i > g.bx || j < -1 || j > g.by) continue;
            double w[3];
            nb_prims(a, i, j, w);
            sw[0][hi][hj] = w[0]; sw[1][hi][hj] = w[1]; sw[2][hi][hj] = w[2];
        }
        __syncthreads();
        const int ri = ri0 + li, rj = rj0 + lj;
        const int nrow = min(PT_J, g.by + 2 - rj0);   // cells of this tile row
        double* st = stage + threadIdx.x * 32;
        if (ri < g.bx + 2 && rj < g.by + 2) {
            prep_cell(a, ri * (g.by + 2) + rj, ri - 1, rj - 1, [&](int s, int d, int k) {
                const int di = d == 0 ? (s ? 2 : 0) : 1, dj = d == 1 ? (s ? 2 : 0) : 1;
                return sw[k][li + di][lj + dj];
            }, [&](const CellPar& P) {
                // stage with an XOR swizzle (bank = e ^ lane: conflict-free)
                const double* pv = reinterpret_cast<const double*>(&P);
#pragma unroll
                for (int e = 0; e < kParD; ++e) st[e ^ lj] = pv[e];
            });
        }
        __syncwarp();
        // the warp's tile row is nrow contiguous CellPars: write them as
        // 512-byte coalesced runs of double2
        if (ri < g.bx + 2) {
            MM2D_CHECK(rj0 + nrow <= g.by + 2 && nrow > 0);
            double* dst = reinterpret_cast<double*>(a.P) + ((size_t)ri * (g.by + 2) + rj0) * kParD;
            const double* wst = stage + (threadIdx.x - lj) * 32;
            for (int f = 2 * lj; f < nrow * kParD; f += 64) {
                const int c = f / kParD, e = f - c * kParD;
                const double x0 = wst[c * 32 + (e ^ c)], x1 = wst[c * 32 + ((e + 1) ^ c)];
                *reinterpret_cast<double2*>(dst + f) = make_double2(x0, x1);
            }
        }
    }
}

}  // namespace mm2d
