// Fused single-pass micro kernel: x-transport (+ projection), y-transport
// (+ projection), ES-BGK target g^, diffuse-wall override, implicit
// relaxation and the heat-tensor moment, for every (cell, velocity node).
//
// Restates, fused, the reference's micro_step_2d (micro2d.py:102-127) with
// transport_stage_2d (_core.pyx:128-198), ghat_2d (_core.pyx:201-225),
// add_gaussian_term_2d (_core.pyx:228-250), add_lowrank_4d (253-267),
// ghat_override_2d (boundary.py:343-378), relax_2d (_core.pyx:270-286) and
// heat_tensor_2d (_core.pyx:289-322).
//
// Work decomposition.  A CTA owns a strip of BX cells in x and a segment of
// LY rows in y and marches up the segment.  Thread t owns a fixed set of
// velocity nodes for every cell it touches, so every spatial stencil (upwind
// differences in x and y) is thread-local; only the per-cell velocity
// reductions (projection sums, heat moments) cross threads, through a
// one-barrier block all-reduce.  The x-stage result G* of the last three
// rows lives in a thread-private shared-memory ring, so HBM sees G^n read
// once (plus the one-cell x halo, which is only half a cell per row since
// the upwind direction picks one side per node) and G^{n+1} written once.
//
// Row pipeline (per row j of the segment):
//   x-stage(j+1): G*(j+1) = G^n - dt (Z_x - Zhat_x)     [reduction 1]
//   y-stage(j):   G**(j)  = G*(j) - dt (Z_y - Zhat_y)   [reduction 2, also
//                                                        carries H(j-1)]
//   target g^(j), wall override (strip rows only), relax, store G^{n+1}(j)
#pragma once
#include "mm2d_common.cuh"

namespace mm2d {

struct MicroArgs {
    Geometry g;
    const double* G;          // (bx, by, V) G^n
    double* Gout;             // (bx, by, V) G^{n+1}
    const double* hxlo;       // G halos (HALO faces only).  Packed (received) form:
    const double* hxhi;       //   x: by cells, y: bx + 2 cells (corners at 0, bx+1), hys = V.
    const double* hylo;       // Peer form (mm2d_halo_peer): the pointers address the
    const double* hyhi;       //   neighbour blocks' own G arrays, read in place over
    size_t hys;               //   NVLink / peer memory: x faces are the neighbour's edge
    const double* hc[4];      //   column (contiguous), y-face cell i sits at hy + (i + 1) hys
    int hpeer;                //   with hys = by V, and the four corner cells come from the
                              //   diagonal neighbours (hc: bottom-left, bottom-right,
                              //   top-left, top-right)
    const double* hnb[8];     // peer form: the neighbours' G bases (debug bounds checks)
    const CellPar* P;         // ring
    double* Hr;               // ring, AoS [ring][4]
    const double* v1;         // velocity centres
    const double* v2;
    const unsigned long long* err;
    const unsigned long long* iso;   // isotropy maxima (eps < 1e-10 guard)
    const double* src_coeffs; // (nsrc, bx, by) or null
    const double* src_shapes; // (nsrc, V)
    int nsrc;
    const double* wall_ghat;  // precomputed wall-strip targets (k_wall_ghat)
    const double* zero;       // V zeros (zero ghosts of the specialised kernel)
    int ly;                   // rows per segment
    int nband;                // k_micro32: 0 = uniform bands of ly rows, else band
    int band_j0[9];           //   b covers rows [band_j0[b], band_j0[b+1]) (all columns)
    int gauss;                // nu != 0
    int part;                 // 0 all CTAs; 1 only CTAs that read no received G halo
                              // (run while the halo exchange is in flight); 2 only the others
    double dt, eps, inveps, idx, idy, dv, hfac;  // hfac = eps * dv
    // k_micro32's raw-moment projection sums: dx/dt, dy/dt, (dx/dt)^2, (dy/dx)^2
    // (the scales between its node coordinates dt |v| / dx and the velocities)
    double ikx, iky, ikx2, ryx;
};

// Does the CTA owning columns [i0, i1) and rows [j0, j1) read a received G
// halo (an x halo column or a y halo row, corners included)?  Selects the
// CTAs of each part of a split launch (MicroArgs::part).
__device__ __forceinline__ bool reads_halo(const Geometry& g, int i0, int i1, int j0, int j1) {
    return (i0 == 0 && g.xlo == GM_HALO) || (i1 >= g.bx && g.xhi == GM_HALO) ||
           (j0 == 0 && g.ylo == GM_HALO) || (j1 >= g.by && g.yhi == GM_HALO);
}
__device__ __forceinline__ bool skip_part(const MicroArgs& a, int i0, int i1, int j0, int j1) {
    return a.part != 0 && (reads_halo(a.g, i0, i1, j0, j1) == (a.part == 1));
}

// Pointer to G^n of ring cell (i, r) or nullptr for a zero ghost.  *mir is
// set when the cell is the specular image (k reversed) of the returned one;
// rows of a specular y face are never read here (row_kind 3).
__device__ __forceinline__ const double* gn_cell(const MicroArgs& a, int i, int r,
                                                 bool* mir = nullptr) {
    const Geometry& g = a.g;
    const size_t V = (size_t)g.V;
    if (mir) *mir = false;
    bool yhalo = false;
    int rr = r;
    if (r < 0 || r >= g.by) {
        const int m = r < 0 ? g.ylo : g.yhi;
        if (m == GM_ZERO) return nullptr;
        if (m == GM_HALO) yhalo = true;
        else if (m == GM_WRAP) rr = (r + g.by) % g.by;
        else rr = r < 0 ? 0 : g.by - 1;
    }
    int ii = i;
    if (i < 0 || i >= g.bx) {
        const int m = i < 0 ? g.xlo : g.xhi;
        if (m == GM_ZERO) return nullptr;
        if (m == GM_HALO) {
            if (yhalo)
                return a.hpeer ? a.hc[(r < 0 ? 0 : 2) + (i < 0 ? 0 : 1)]
                               : (r < 0 ? a.hylo : a.hyhi) + (size_t)(i < 0 ? 0 : g.bx + 1) * V;
            return (i < 0 ? a.hxlo : a.hxhi) + (size_t)rr * V;
        }
        if (m == GM_WRAP) ii = (i + g.bx) % g.bx;
        else ii = i < 0 ? 0 : g.bx - 1;
        if (m == GM_MIRROR && mir) *mir = true;
    }
    if (yhalo) return (r < 0 ? a.hylo : a.hyhi) + (size_t)(ii + 1) * a.hys;
    return a.G + ((size_t)ii * g.by + rr) * V;
}

// How a ring row r is obtained for the y-stage ghosts of G*:
//   0 compute the x-stage on it, 1 copy of the adjacent owned row, 2 zero,
//   3 specular image of the adjacent owned row (l reversed).
__device__ __forceinline__ int row_kind(const Geometry& g, int r) {
    if (r >= 0 && r < g.by) return 0;
    const int m = r < 0 ? g.ylo : g.yhi;
    if (m == GM_WRAP || m == GM_HALO) return 0;
    return m == GM_COPY ? 1 : m == GM_MIRROR ? 3 : 2;
}

// Per-cell tables in shared memory for one row slot:
//   par[BX] CellPar, E1[BX][nv1], E2[BX][nv2], GA[BX][nv1], GB[BX][nv2]
template <int BX>
struct RowTables {
    CellPar* par;
    double* E1;
    double* E2;
    double* GA;
    double* GB;
};

template <int BX>
__device__ __forceinline__ RowTables<BX> row_tables(double* base, int slot, int nv1, int nv2) {
    const int per = BX * (32 + 2 * nv1 + 2 * nv2);
    double* p = base + (size_t)slot * per;
    RowTables<BX> t;
    t.par = reinterpret_cast<CellPar*>(p);
    t.E1 = p + BX * 32;
    t.E2 = t.E1 + BX * nv1;
    t.GA = t.E2 + BX * nv2;
    t.GB = t.GA + BX * nv1;
    return t;
}

// NE velocity nodes per thread.  FAST: nodes come in 16-byte pairs sharing
// the same v1 row (nv2 even); generic: scalar nodes (any nv1, nv2).
template <int NE, bool FAST>
struct NodeMap {
    int node[NE];
    int k[NE];
    int l[NE];
    bool ok[NE];
    __device__ __forceinline__ void init(int tid, int NT, int nv2, int V) {
#pragma unroll
        for (int e = 0; e < NE; ++e) {
            const int n = FAST ? 2 * (tid + (e >> 1) * NT) + (e & 1) : tid + e * NT;
            node[e] = n;
            ok[e] = n < V;
            const int nn = ok[e] ? n : 0;
            k[e] = nn / nv2;
            l[e] = nn - k[e] * nv2;
        }
    }
    __device__ __forceinline__ void load(const double* __restrict__ p, double (&v)[NE]) const {
        if (p == nullptr) {
#pragma unroll
            for (int e = 0; e < NE; ++e) v[e] = 0.0;
            return;
        }
        if (FAST) {
#pragma unroll
            for (int e = 0; e < NE; e += 2) {
                if (ok[e]) {
                    const double2 x = __ldg(reinterpret_cast<const double2*>(p + node[e]));
                    v[e] = x.x; v[e + 1] = x.y;
                } else { v[e] = 0.0; v[e + 1] = 0.0; }
            }
        } else {
#pragma unroll
            for (int e = 0; e < NE; ++e) v[e] = ok[e] ? __ldg(p + node[e]) : 0.0;
        }
    }
    __device__ __forceinline__ void store(double* __restrict__ p, const double (&v)[NE]) const {
        if (FAST) {
#pragma unroll
            for (int e = 0; e < NE; e += 2)
                if (ok[e]) *reinterpret_cast<double2*>(p + node[e]) = make_double2(v[e], v[e + 1]);
        } else {
#pragma unroll
            for (int e = 0; e < NE; ++e) if (ok[e]) p[node[e]] = v[e];
        }
    }
    // thread-private shared-memory slots (same node indexing as global)
    __device__ __forceinline__ void sload(const double* p, double (&v)[NE]) const {
        if (FAST) {
#pragma unroll
            for (int e = 0; e < NE; e += 2) {
                if (ok[e]) {
                    const double2 x = *reinterpret_cast<const double2*>(p + node[e]);
                    v[e] = x.x; v[e + 1] = x.y;
                } else { v[e] = 0.0; v[e + 1] = 0.0; }
            }
        } else {
#pragma unroll
            for (int e = 0; e < NE; ++e) v[e] = ok[e] ? p[node[e]] : 0.0;
        }
    }
    __device__ __forceinline__ void sstore(double* p, const double (&v)[NE]) const {
        if (FAST) {
#pragma unroll
            for (int e = 0; e < NE; e += 2)
                if (ok[e]) *reinterpret_cast<double2*>(p + node[e]) = make_double2(v[e], v[e + 1]);
        } else {
#pragma unroll
            for (int e = 0; e < NE; ++e) if (ok[e]) p[node[e]] = v[e];
        }
    }
};

// Build the per-cell tables of ring row r into a slot: CellPar copy, the
// separable Maxwellian factors E1[k] = exp(-(v1_k-u1)^2/(2T)),
// E2[l] = exp(-(v2_l-u2)^2/(2T)) (M = pref E1 E2, _core.pyx:66-84), and the
// separable Gaussian factors GA[k] = exp(-c22 W1^2 / (2 det)),
// GB[l] = exp(-c11 W2^2 / (2 det)) (_core.pyx:228-250).
template <int BX>
__device__ __forceinline__ void build_row(const MicroArgs& a, const RowTables<BX>& t, int ic0,
                                          int r, const double* v1s, const double* v2s) {
    const Geometry& g = a.g;
    const int nv1 = g.nv1, nv2 = g.nv2;
    for (int q = threadIdx.x; q < BX * kParD; q += blockDim.x) {
        const int b = q / kParD, c = q - b * kParD;
        const int i = min(ic0 + b, g.bx - 1);
        reinterpret_cast<double*>(t.par)[q] =
            reinterpret_cast<const double*>(a.P + ring_index(g, i, r))[c];
    }
    const int per = nv1 + nv2;
    for (int q = threadIdx.x; q < BX * per; q += blockDim.x) {
        const int b = q / per, m = q - b * per;
        const int i = min(ic0 + b, g.bx - 1);
        const CellPar& P = a.P[ring_index(g, i, r)];
        if (m < nv1) {
            const double w = v1s[m] - P.u1;
            t.E1[b * nv1 + m] = exp(-(w * w) * P.inv2T);
            if (a.gauss) t.GA[b * nv1 + m] = exp(P.gq11 * (w * w));
        } else {
            const int l = m - nv1;
            const double w = v2s[l] - P.u2;
            t.E2[b * nv2 + l] = exp(-(w * w) * P.inv2T);
            if (a.gauss) t.GB[b * nv2 + l] = exp(P.gq22 * (w * w));
        }
    }
}

template <int NE, int BX, bool FAST>
__global__ void __launch_bounds__(256) k_micro(MicroArgs a) {
    extern __shared__ __align__(16) double smem[];
    const Geometry& g = a.g;
    if (err_pending(a.err, EW_PREP)) return;
    const int NT = blockDim.x;
    const int nwarps = NT >> 5;
    const int tid = threadIdx.x;
    const int V = g.V, nv1 = g.nv1, nv2 = g.nv2;
    const int ic0 = blockIdx.x * BX;                 // first owned cell of the strip
    const int nb = min(BX, g.bx - ic0);              // owned cells in this strip
    const int j0s = blockIdx.y * a.ly;
    const int j1s = min(j0s + a.ly, g.by);
    if (skip_part(a, ic0, ic0 + nb, j0s, j1s)) return;

    // ---- shared memory carve-up ----
    double* gstar = smem;                                         // [3][BX][V]
    double* tabs = gstar + 3 * BX * (size_t)V;                    // [4][BX*(32+2nv1+2nv2)]
    double* red = tabs + 4 * BX * (size_t)(32 + 2 * nv1 + 2 * nv2);  // [2][32][8*BX]
    double* v1s = red + 2 * 32 * 8 * BX;
    double* v2s = v1s + nv1;
    for (int q = tid; q < nv1; q += NT) v1s[q] = a.v1[q];
    for (int q = tid; q < nv2; q += NT) v2s[q] = a.v2[q];

    NodeMap<NE, FAST> nm;
    nm.init(tid, NT, nv2, V);

    const bool skip_gauss = a.gauss && a.eps < 1e-10 &&
        __longlong_as_double(a.iso[0]) <= 1e-13 * __longlong_as_double(a.iso[3]) &&
        __longlong_as_double(a.iso[1]) <= 1e-13 * __longlong_as_double(a.iso[3]) &&
        __longlong_as_double(a.iso[2]) <= 1e-13 * __longlong_as_double(a.iso[3]);
    const bool gauss = a.gauss && !skip_gauss;

    int parity = 0;
    auto slot_of = [&](int r) { return (r + 4) & 3; };          // r >= -1
    auto gs_ptr = [&](int r, int b) { return gstar + ((size_t)(((r + 3) % 3) * BX + b)) * V; };

    __syncthreads();   // v1s / v2s visible
    // prologue tables: rows j0s-1, j0s, j0s+1
    for (int r = j0s - 1; r <= j0s + 1; ++r)
        if (r <= j1s && row_kind(g, r) == 0)
            build_row<BX>(a, row_tables<BX>(tabs, slot_of(r), nv1, nv2), ic0, r, v1s, v2s);
    __syncthreads();

    // prefetch registers for the next x-stage row
    double pf[BX][NE];
    double ph[NE];

    auto prefetch = [&](int r) {
#pragma unroll
        for (int b = 0; b < BX; ++b) nm.load(b < nb ? gn_cell(a, ic0 + b, r) : nullptr, pf[b]);
        bool ml, mr;
        const double* hl = gn_cell(a, ic0 - 1, r, &ml);
        const double* hr = gn_cell(a, ic0 + nb, r, &mr);
        if (ml || mr) {
            // specular x face: the halo node (k, l) is the edge cell's (nv1-1-k, l)
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                const bool left = v1s[nm.k[e]] >= 0.0;
                const double* hp = left ? hl : hr;
                const bool m = left ? ml : mr;
                const int node = m ? (nv1 - 1 - nm.k[e]) * nv2 + nm.l[e] : nm.node[e];
                ph[e] = (hp != nullptr && nm.ok[e]) ? __ldg(hp + node) : 0.0;
            }
        } else if (FAST) {
#pragma unroll
            for (int e = 0; e < NE; e += 2) {
                const double* hp = v1s[nm.k[e]] >= 0.0 ? hl : hr;
                if (hp != nullptr && nm.ok[e]) {
                    const double2 x = __ldg(reinterpret_cast<const double2*>(hp + nm.node[e]));
                    ph[e] = x.x; ph[e + 1] = x.y;
                } else { ph[e] = 0.0; ph[e + 1] = 0.0; }
            }
        } else {
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                const double* hp = v1s[nm.k[e]] >= 0.0 ? hl : hr;
                ph[e] = (hp != nullptr && nm.ok[e]) ? __ldg(hp + nm.node[e]) : 0.0;
            }
        }
    };

    // x-stage on ring row r from the prefetched registers -> G*(r) in smem
    auto xstage = [&](int r) {
        const RowTables<BX> t = row_tables<BX>(tabs, slot_of(r), nv1, nv2);
        double s[4 * BX];
        double tv[BX][NE];
#pragma unroll
        for (int q = 0; q < 4 * BX; ++q) s[q] = 0.0;
#pragma unroll
        for (int b = 0; b < BX; ++b) {
            const CellPar& P = t.par[b];
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                const int k = nm.k[e], l = nm.l[e];
                const double v1 = v1s[k];
                const double gc = pf[b][e];
                const double gl = (b == 0) ? ph[e] : pf[b > 0 ? b - 1 : 0][e];
                const double gr = (b == BX - 1 || b == nb - 1) ? ph[e] : pf[b < BX - 1 ? b + 1 : b][e];
                const double d = v1 >= 0.0 ? gc - gl : gr - gc;
                double Z = v1 * d * a.idx;
                if (!nm.ok[e] || b >= nb) Z = 0.0;
                const double w1 = (v1 - P.u1) * P.isT;
                const double w2 = (v2s[l] - P.u2) * P.isT;
                const double b4 = 0.5 * (w1 * w1 + w2 * w2) - 1.0;
                s[4 * b + 0] += Z;
                s[4 * b + 1] = fma(Z, w1, s[4 * b + 1]);
                s[4 * b + 2] = fma(Z, w2, s[4 * b + 2]);
                s[4 * b + 3] = fma(Z, b4, s[4 * b + 3]);
                tv[b][e] = gc - a.dt * Z;
            }
        }
        block_allreduce<4 * BX>(s, red, parity, nwarps);
#pragma unroll
        for (int b = 0; b < BX; ++b) {
            const CellPar& P = t.par[b];
            const double a1 = s[4 * b] * P.scale, a2 = s[4 * b + 1] * P.scale;
            const double a3 = s[4 * b + 2] * P.scale, a4 = s[4 * b + 3] * P.scale;
            double o[NE];
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                const int k = nm.k[e], l = nm.l[e];
                const double w1 = (v1s[k] - P.u1) * P.isT;
                const double w2 = (v2s[l] - P.u2) * P.isT;
                const double b4 = 0.5 * (w1 * w1 + w2 * w2) - 1.0;
                const double M = P.pref * t.E1[b * nv1 + k] * t.E2[b * nv2 + l];
                const double zh = (a1 + w1 * a2 + w2 * a3 + b4 * a4) * M;
                o[e] = fma(a.dt, zh, tv[b][e]);
            }
            nm.sstore(gs_ptr(r, b), o);
        }
    };

    auto fill_row = [&](int r, int kind, int src) {   // copy (1), zero (2) or mirror (3)
        if (kind == 3) __syncthreads();   // the source row was stored by other threads
#pragma unroll
        for (int b = 0; b < BX; ++b) {
            double o[NE];
            if (kind == 1) nm.sload(gs_ptr(src, b), o);
            else if (kind == 3) {
                const double* sr = gs_ptr(src, b);
#pragma unroll
                for (int e = 0; e < NE; ++e)
                    o[e] = nm.ok[e] ? sr[nm.k[e] * nv2 + (nv2 - 1 - nm.l[e])] : 0.0;
            } else {
#pragma unroll
                for (int e = 0; e < NE; ++e) o[e] = 0.0;
            }
            nm.sstore(gs_ptr(r, b), o);
        }
    };

    // ---- prologue: G*(j0s-1), G*(j0s) ----
    const int k_lo = row_kind(g, j0s - 1);
    if (k_lo == 0) { prefetch(j0s - 1); xstage(j0s - 1); }
    prefetch(j0s);
    xstage(j0s);
    if (k_lo != 0) fill_row(j0s - 1, k_lo, j0s);
    int knext = row_kind(g, j0s + 1);
    if (j0s + 1 <= j1s && knext == 0) prefetch(j0s + 1);

    double hs[4 * BX];          // pending heat partial sums of row j-1
    bool hpend = false;
    int hrow = -1;
#pragma unroll
    for (int q = 0; q < 4 * BX; ++q) hs[q] = 0.0;

    for (int j = j0s; j < j1s; ++j) {
        // tables for row j+2 (used by the next iteration's x-stage)
        if (j + 2 <= j1s && row_kind(g, j + 2) == 0)
            build_row<BX>(a, row_tables<BX>(tabs, slot_of(j + 2), nv1, nv2), ic0, j + 2, v1s, v2s);
        // ---- x-stage for row j+1 ----
        const int kj1 = row_kind(g, j + 1);
        if (kj1 == 0) {
            xstage(j + 1);
            if (j + 2 <= j1s && row_kind(g, j + 2) == 0) prefetch(j + 2);
        } else {
            fill_row(j + 1, kj1, j);
        }
        // ---- y-stage for row j (+ pending H of row j-1) ----
        const RowTables<BX> t = row_tables<BX>(tabs, slot_of(j), nv1, nv2);
        double s[8 * BX];
        double ty[BX][NE];
#pragma unroll
        for (int q = 0; q < 4 * BX; ++q) { s[q] = 0.0; s[4 * BX + q] = hs[q]; }
#pragma unroll
        for (int b = 0; b < BX; ++b) {
            const CellPar& P = t.par[b];
            double gm[NE], gc[NE], gp[NE];
            nm.sload(gs_ptr(j - 1, b), gm);
            nm.sload(gs_ptr(j, b), gc);
            nm.sload(gs_ptr(j + 1, b), gp);
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                const int k = nm.k[e], l = nm.l[e];
                const double v2 = v2s[l];
                const double d = v2 >= 0.0 ? gc[e] - gm[e] : gp[e] - gc[e];
                double Z = v2 * d * a.idy;
                if (!nm.ok[e] || b >= nb) Z = 0.0;
                const double w1 = (v1s[k] - P.u1) * P.isT;
                const double w2 = (v2 - P.u2) * P.isT;
                const double b4 = 0.5 * (w1 * w1 + w2 * w2) - 1.0;
                s[4 * b + 0] += Z;
                s[4 * b + 1] = fma(Z, w1, s[4 * b + 1]);
                s[4 * b + 2] = fma(Z, w2, s[4 * b + 2]);
                s[4 * b + 3] = fma(Z, b4, s[4 * b + 3]);
                ty[b][e] = gc[e] - a.dt * Z;
            }
        }
        block_allreduce<8 * BX>(s, red, parity, nwarps);
        if (hpend) {
            // write H(j-1): thread q < 4*nb writes cell q/4, component q%4
#pragma unroll
            for (int q = 0; q < 4 * BX; ++q)
                if (tid == q && (q >> 2) < nb)
                    a.Hr[4 * ring_index(g, ic0 + (q >> 2), hrow) + (q & 3)] = a.hfac * s[4 * BX + q];
        }
        // ---- G**, target g^, relax ----
        double gss[BX][NE], gh[BX][NE];
        bool strip = false;
        const int gj = g.j0 + j;
#pragma unroll
        for (int b = 0; b < BX; ++b) {
            const CellPar& P = t.par[b];
            const double a1 = s[4 * b] * P.scale, a2 = s[4 * b + 1] * P.scale;
            const double a3 = s[4 * b + 2] * P.scale, a4 = s[4 * b + 3] * P.scale;
            const int i = ic0 + b;
            const bool on = b < nb &&
                ((g.wall[0] && i == 0) || (g.wall[1] && i == g.bx - 1) ||
                 (g.wall[2] && j == 0) || (g.wall[3] && j == g.by - 1));
            strip = strip || on;
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                const int k = nm.k[e], l = nm.l[e];
                const double W1 = v1s[k] - P.u1;
                const double W2 = v2s[l] - P.u2;
                const double w1 = W1 * P.isT, w2 = W2 * P.isT;
                const double b4 = 0.5 * (w1 * w1 + w2 * w2) - 1.0;
                const double M = P.pref * t.E1[b * nv1 + k] * t.E2[b * nv2 + l];
                const double zh = (a1 + w1 * a2 + w2 * a3 + b4 * a4) * M;
                gss[b][e] = fma(a.dt, zh, ty[b][e]);
                // ghat_2d (_core.pyx:220-224)
                const double bs = (W1 * W1 - W2 * W2) * P.s11 + 2.0 * W1 * W2 * P.s12;
                const double cg = ((W1 * W1 + W2 * W2) * P.inv2T - 2.0) * (W1 * P.gT1 + W2 * P.gT2) * P.invT;
                double h = -(bs * P.inv2T + cg) * M * P.invtau;
                if (gauss) {
                    // add_gaussian_term_2d (_core.pyx:244-249), separable form
                    const double Gs = P.gpref * t.GA[b * nv1 + k] * t.GB[b * nv2 + l] *
                                      exp(P.gq12 * W1 * W2);
                    h += (Gs - M) * a.inveps;
                }
                if (a.nsrc > 0 && b < nb && nm.ok[e]) {
                    // add_lowrank_4d with coeffs / tau (micro2d.py:120-123)
                    const size_t cell = (size_t)i * g.by + j;
                    const size_t S = (size_t)g.bx * g.by;
                    for (int m = 0; m < a.nsrc; ++m)
                        h += (a.src_coeffs[m * S + cell] / P.tau) * a.src_shapes[(size_t)m * V + nm.node[e]];
                }
                gh[b][e] = h;
            }
        }
        if (strip) {
            // ghat_override_2d (boundary.py:343-378) for wall-strip cells:
            // g^ = -(Mterm - Pi[Mterm]) / tau with Mterm the upwind transport
            // of the Maxwellian built with ghost wall Maxwellians.
            double so[4 * BX];
            double mt[BX][NE];
#pragma unroll
            for (int q = 0; q < 4 * BX; ++q) so[q] = 0.0;
#pragma unroll
            for (int b = 0; b < BX; ++b) {
                const CellPar& P = t.par[b];
                const int i = min(ic0 + b, g.bx - 1);
#pragma unroll
                for (int e = 0; e < NE; ++e) {
                    const int k = nm.k[e], l = nm.l[e];
                    const double v1 = v1s[k], v2 = v2s[l];
                    const double M = P.pref * t.E1[b * nv1 + k] * t.E2[b * nv2 + l];
                    double Mn[4];
#pragma unroll
                    for (int f = 0; f < 4; ++f) {
                        const int ii = i + (f == 0 ? -1 : f == 1 ? 1 : 0);
                        const int jj = j + (f == 2 ? -1 : f == 3 ? 1 : 0);
                        const bool outside = ii < 0 || ii >= g.bx || jj < 0 || jj >= g.by;
                        if (outside && g.wall[f]) {
                            const double Tw = g.wallT[f], U = g.wallU[f];
                            const double g1 = f < 2 ? 0.0 : U, g2 = f < 2 ? U : 0.0;
                            const double x1 = v1 - g1, x2 = v2 - g2;
                            Mn[f] = P.rw[f] / (2.0 * kPi * Tw) * exp(-(x1 * x1 + x2 * x2) / (2.0 * Tw));
                        } else {
                            const CellPar& Q = a.P[ring_index(g, ii, jj)];
                            const double x1 = v1 - Q.u1, x2 = v2 - Q.u2;
                            Mn[f] = Q.pref * exp(-(x1 * x1 + x2 * x2) * Q.inv2T);
                        }
                    }
                    const double vm1 = v1 < 0.0 ? v1 : 0.0, vp1 = v1 > 0.0 ? v1 : 0.0;
                    const double vm2 = v2 < 0.0 ? v2 : 0.0, vp2 = v2 > 0.0 ? v2 : 0.0;
                    double Mt = (vm1 * (Mn[1] - M) + vp1 * (M - Mn[0])) * a.idx +
                                (vm2 * (Mn[3] - M) + vp2 * (M - Mn[2])) * a.idy;
                    if (!nm.ok[e] || b >= nb) Mt = 0.0;
                    const double w1 = (v1 - P.u1) * P.isT, w2 = (v2 - P.u2) * P.isT;
                    const double b4 = 0.5 * (w1 * w1 + w2 * w2) - 1.0;
                    so[4 * b + 0] += Mt;
                    so[4 * b + 1] = fma(Mt, w1, so[4 * b + 1]);
                    so[4 * b + 2] = fma(Mt, w2, so[4 * b + 2]);
                    so[4 * b + 3] = fma(Mt, b4, so[4 * b + 3]);
                    mt[b][e] = Mt;
                }
            }
            block_allreduce<4 * BX>(so, red, parity, nwarps);
#pragma unroll
            for (int b = 0; b < BX; ++b) {
                const CellPar& P = t.par[b];
                const int i = ic0 + b;
                const bool on = b < nb &&
                    ((g.wall[0] && i == 0) || (g.wall[1] && i == g.bx - 1) ||
                     (g.wall[2] && j == 0) || (g.wall[3] && j == g.by - 1));
                if (!on) continue;
                const double a1 = so[4 * b] * P.scale, a2 = so[4 * b + 1] * P.scale;
                const double a3 = so[4 * b + 2] * P.scale, a4 = so[4 * b + 3] * P.scale;
#pragma unroll
                for (int e = 0; e < NE; ++e) {
                    const int k = nm.k[e], l = nm.l[e];
                    const double w1 = (v1s[k] - P.u1) * P.isT, w2 = (v2s[l] - P.u2) * P.isT;
                    const double b4 = 0.5 * (w1 * w1 + w2 * w2) - 1.0;
                    const double M = P.pref * t.E1[b * nv1 + k] * t.E2[b * nv2 + l];
                    const double pi = (a1 + w1 * a2 + w2 * a3 + b4 * a4) * M;
                    gh[b][e] = -(mt[b][e] - pi) / P.tau;
                }
            }
        }
        // relax (_core.pyx:280-285), store, heat partial sums (u^n)
#pragma unroll
        for (int q = 0; q < 4 * BX; ++q) hs[q] = 0.0;
#pragma unroll
        for (int b = 0; b < BX; ++b) {
            const CellPar& P = t.par[b];
            double o[NE];
#pragma unroll
            for (int e = 0; e < NE; ++e) {
                const int k = nm.k[e], l = nm.l[e];
                double gp = P.wg * gss[b][e] + P.wh * gh[b][e];
                if (!nm.ok[e] || b >= nb) gp = 0.0;
                o[e] = gp;
                const double W1 = v1s[k] - P.u1, W2 = v2s[l] - P.u2;
                const double t1 = W1 * W1 * gp, t2 = W2 * W2 * gp;
                hs[4 * b + 0] = fma(t1, W1, hs[4 * b + 0]);
                hs[4 * b + 1] = fma(t1, W2, hs[4 * b + 1]);
                hs[4 * b + 2] = fma(t2, W1, hs[4 * b + 2]);
                hs[4 * b + 3] = fma(t2, W2, hs[4 * b + 3]);
            }
            if (b < nb) nm.store(a.Gout + ((size_t)(ic0 + b) * g.by + j) * V, o);
        }
        hpend = true;
        hrow = j;
    }
    // last pending heat row
    if (hpend) {
        block_allreduce<4 * BX>(hs, red, parity, nwarps);
#pragma unroll
        for (int q = 0; q < 4 * BX; ++q)
            if (tid == q && (q >> 2) < nb)
                a.Hr[4 * ring_index(g, ic0 + (q >> 2), hrow) + (q & 3)] = a.hfac * hs[q];
    }
}

// dynamic shared memory bytes for k_micro
inline size_t micro_smem_bytes(int BX, int V, int nv1, int nv2) {
    return sizeof(double) * ((size_t)3 * BX * V + (size_t)4 * BX * (32 + 2 * nv1 + 2 * nv2) +
                             (size_t)2 * 32 * 8 * BX + nv1 + nv2);
}

}  // namespace mm2d
