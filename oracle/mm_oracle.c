/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle for the micro-macro ES-BGK timestep.
 *
 * A plain-C restatement of the reference solver's per-timestep algorithm
 * (arxiv/paper_2509_21832, package `micromacro`).  It is the parity checker
 * for the CUDA product path and the CPU baseline leg of bench.py; nothing in
 * the product (paper_2509_21832_b200/) links, imports or calls it.
 *
 * Parity pinned: the fixtures in tests/golden/ were produced by running the reference
 * itself (compiled Cython backend) with tests/golden/make_golden.py; the
 * oracle is checked against them in tests/test_oracle_golden.py.
 *
 * Every function cites the reference file:line it restates (paths relative
 * to pkg/src/micromacro/).  Loop order and operation order follow the
 * reference's compiled kernels (_kernels/_core.pyx: sequential left-to-right
 * velocity sums) and its NumPy expressions (elementwise, same association),
 * so results agree with the reference to a few ulps; the only differences
 * come from libm exp/erf/pow vs NumPy/SciPy's implementations.
 *
 * Layouts (C-contiguous fp64, identical to the reference):
 *   2D: Q[i][j][6], G[i][j][k][l] (l fastest), H[4][i][j]
 *   1D: Q[i][3],    G[i][k]
 * Face kinds: 0 periodic, 1 extrapolate, 2 diffuse wall, 3 specular wall.
 * Specular walls are an EXTENSION (BASELINE config 4 wording; the reference
 * has only diffuse walls): every ghost is the mirror image of the edge cell
 * in the wall-normal velocity, v_n -> -v_n (micro ghosts: node index
 * reversed along the normal axis; macro ghosts: normal momentum and E12
 * negated; heat ghosts: components odd in v_n negated).  Parity of this
 * rule is unpinned (no reference implementation exists).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <stdint.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define PI_D 3.141592653589793238462643383279502884
#define SQRT2_D 1.4142135623730950488016887242096980786

enum { FACE_PERIODIC = 0, FACE_EXTRAPOLATE = 1, FACE_WALL = 2, FACE_SPECULAR = 3 };
enum { TAU_HARD_SPHERE_1D = 0, TAU_PRESSURE_1D = 1, TAU_ESBGK_2D = 2,
       TAU_BGK_2D = 3, TAU_CONSTANT = 4 };

/* error codes mirror the reference's exception categories (errors.py) */
enum { MMO_OK = 0, MMO_CONFIG = 2, MMO_INVALID_STATE = 3 };
enum { ERR_NONE = 0, ERR_DENSITY = 1, ERR_PRESSURE_SPD = 2, ERR_MODIFIED_SPD = 3,
       ERR_TEMPERATURE = 4 };

typedef struct {
    int code;      /* ERR_* */
    int i, j;      /* offending cell (j = -1 in 1D) */
    double value;
} mmo_err;

typedef struct {
    int nx, ny, nv1, nv2;
    double dx, dy;
    const double *v1, *v2;  /* velocity cell centres */
    int face[4];            /* left, right, bottom, top */
    double wall_T[4], wall_U[4];
    int tau_kind;
    double tau_value;
    double nu;
    double eps;
} mmo_cfg2d;

typedef struct {
    int nx, nv;
    double dx;
    const double *v;
    int face[2];
    double wall_T[2];
    int tau_kind;
    double tau_value;
    double eps;
} mmo_cfg1d;

/* ------------------------------------------------------------------------ */
/* collision model: gas_state.py:166-199 (constants at gas_state.py:21-27)   */
/* ------------------------------------------------------------------------ */
static double tau_of(int kind, double value, double rho, double T)
{
    switch (kind) {
    case TAU_HARD_SPHERE_1D: return 3.2 * sqrt(T / (2.0 * PI_D));
    case TAU_PRESSURE_1D: return rho * T;
    case TAU_ESBGK_2D: return (0.4625 * PI_D) * rho;
    case TAU_BGK_2D: return (3.0 * PI_D * 0.436 / sqrt(2.0)) * rho;
    default: return value;
    }
}

/* ------------------------------------------------------------------------ */
/* 2D primitives with validation: gas_state.py:81-108                        */
/* ------------------------------------------------------------------------ */
typedef struct { double rho, u1, u2, t11, t12, t22, T; } prim2;

static void prim_of(const double *q, prim2 *p)
{
    p->rho = q[0];
    p->u1 = q[1] / p->rho;
    p->u2 = q[2] / p->rho;
    p->t11 = q[3] / p->rho - p->u1 * p->u1;
    p->t12 = q[4] / p->rho - p->u1 * p->u2;
    p->t22 = q[5] / p->rho - p->u2 * p->u2;
    p->T = 0.5 * (p->t11 + p->t22);
}

/* check_spd_2x2 (gas_state.py:81-90): bad if a11 <= tol or det <= tol^2 */
static int spd_bad(double a11, double a12, double a22, double *det_out)
{
    double tol = 1e-14 * (a11 + a22);
    double det = a11 * a22 - a12 * a12;
    *det_out = det;
    return (a11 <= tol) || (det <= tol * tol);
}

/* primitives_2d over a field: density check first (whole field), then the
 * SPD check; the first offending cell in C order is reported, as
 * np.argmax(bad) does (gas_state.py:31-37). */
static int prims_field(int n, int ny, const double *Q, prim2 *P, mmo_err *err)
{
    for (int c = 0; c < n; ++c) {
        if (!(Q[6 * c] > 0.0)) {
            err->code = ERR_DENSITY; err->i = c / ny; err->j = c % ny;
            err->value = Q[6 * c];
            return MMO_INVALID_STATE;
        }
    }
    for (int c = 0; c < n; ++c) prim_of(Q + 6 * c, P + c);
    for (int c = 0; c < n; ++c) {
        double det;
        if (spd_bad(P[c].t11, P[c].t12, P[c].t22, &det)) {
            err->code = ERR_PRESSURE_SPD; err->i = c / ny; err->j = c % ny;
            err->value = det;
            return MMO_INVALID_STATE;
        }
    }
    return MMO_OK;
}

/* ------------------------------------------------------------------------ */
/* kernels, restating _kernels/_core.pyx                                     */
/* ------------------------------------------------------------------------ */

/* _core.pyx:66-84 */
void mmo_maxwellian_field_2d(int nx, int ny, const double *rho, const double *u1,
                             const double *u2, const double *T, int nv1,
                             const double *v1, int nv2, const double *v2,
                             double *M)
{
    #pragma omp parallel for schedule(static)
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j) {
            int c = i * ny + j;
            double pref = rho[c] / (2.0 * PI_D * T[c]);
            double inv2T = 1.0 / (2.0 * T[c]);
            double *m = M + (size_t)c * nv1 * nv2;
            for (int k = 0; k < nv1; ++k) {
                double w1 = v1[k] - u1[c];
                for (int l = 0; l < nv2; ++l) {
                    double w2 = v2[l] - u2[c];
                    m[k * nv2 + l] = pref * exp(-(w1 * w1 + w2 * w2) * inv2T);
                }
            }
        }
}

/* per-cell projection coefficients, _core.pyx:99-118 */
static void proj_coeffs(const double *F, int nv1, const double *v1, int nv2,
                        const double *v2, double rho, double u1, double u2,
                        double T, double dv, double a[4])
{
    double st = sqrt(T), scale = dv / rho;
    double a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0;
    for (int k = 0; k < nv1; ++k) {
        double w1 = (v1[k] - u1) / st;
        for (int l = 0; l < nv2; ++l) {
            double w2 = (v2[l] - u2) / st;
            double b4 = 0.5 * (w1 * w1 + w2 * w2) - 1.0;
            double f = F[k * nv2 + l];
            a1 += f; a2 += f * w1; a3 += f * w2; a4 += f * b4;
        }
    }
    a[0] = a1 * scale; a[1] = a2 * scale; a[2] = a3 * scale; a[3] = a4 * scale;
}

/* _core.pyx:87-125 */
void mmo_project_field_2d(int nx, int ny, int nv1, int nv2, const double *F,
                          const double *M, const double *rho, const double *u1,
                          const double *u2, const double *T, const double *v1,
                          const double *v2, double dv, double *out)
{
    size_t V = (size_t)nv1 * nv2;
    #pragma omp parallel for schedule(static)
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j) {
            int c = i * ny + j;
            double a[4];
            proj_coeffs(F + c * V, nv1, v1, nv2, v2, rho[c], u1[c], u2[c], T[c], dv, a);
            double st = sqrt(T[c]);
            for (int k = 0; k < nv1; ++k) {
                double w1 = (v1[k] - u1[c]) / st;
                for (int l = 0; l < nv2; ++l) {
                    double w2 = (v2[l] - u2[c]) / st;
                    double b4 = 0.5 * (w1 * w1 + w2 * w2) - 1.0;
                    out[c * V + k * nv2 + l] =
                        (a[0] + w1 * a[1] + w2 * a[2] + b4 * a[3]) * M[c * V + k * nv2 + l];
                }
            }
        }
}

/* _core.pyx:128-198.  G_ext carries one ghost layer on `axis`. */
void mmo_transport_stage_2d(int nx, int ny, int nv1, int nv2, const double *G_ext,
                            const double *M, const double *rho, const double *u1,
                            const double *u2, const double *T, const double *v1,
                            const double *v2, double d, double dt, int axis,
                            double *out)
{
    size_t V = (size_t)nv1 * nv2;
    double dv = (v1[1] - v1[0]) * (v2[1] - v2[0]);
    int eny = axis == 1 ? ny + 2 : ny;   /* extended y extent of G_ext */
    #pragma omp parallel
    {
        double *zbuf = (double *)malloc(V * sizeof(double));
        #pragma omp for schedule(static)
        for (int i = 0; i < nx; ++i)
            for (int j = 0; j < ny; ++j) {
                int io = axis == 0 ? i + 1 : i;
                int jo = axis == 1 ? j + 1 : j;
#define GE(ii, jj, kk, ll) G_ext[((size_t)(ii) * eny + (jj)) * V + (kk) * nv2 + (ll)]
                if (axis == 0) {
                    for (int k = 0; k < nv1; ++k) {
                        double vk = v1[k];
                        if (vk >= 0.0)
                            for (int l = 0; l < nv2; ++l)
                                zbuf[k * nv2 + l] = vk * (GE(io, jo, k, l) - GE(io - 1, jo, k, l)) / d;
                        else
                            for (int l = 0; l < nv2; ++l)
                                zbuf[k * nv2 + l] = vk * (GE(io + 1, jo, k, l) - GE(io, jo, k, l)) / d;
                    }
                } else {
                    for (int k = 0; k < nv1; ++k)
                        for (int l = 0; l < nv2; ++l) {
                            double vk = v2[l];
                            if (vk >= 0.0)
                                zbuf[k * nv2 + l] = vk * (GE(io, jo, k, l) - GE(io, jo - 1, k, l)) / d;
                            else
                                zbuf[k * nv2 + l] = vk * (GE(io, jo + 1, k, l) - GE(io, jo, k, l)) / d;
                        }
                }
                int c = i * ny + j;
                double a[4];
                proj_coeffs(zbuf, nv1, v1, nv2, v2, rho[c], u1[c], u2[c], T[c], dv, a);
                double st = sqrt(T[c]);
                for (int k = 0; k < nv1; ++k) {
                    double w1 = (v1[k] - u1[c]) / st;
                    for (int l = 0; l < nv2; ++l) {
                        double w2 = (v2[l] - u2[c]) / st;
                        double b4 = 0.5 * (w1 * w1 + w2 * w2) - 1.0;
                        double zh = (a[0] + w1 * a[1] + w2 * a[2] + b4 * a[3]) * M[c * V + k * nv2 + l];
                        out[c * V + k * nv2 + l] = GE(io, jo, k, l) - dt * (zbuf[k * nv2 + l] - zh);
                    }
                }
#undef GE
            }
        free(zbuf);
    }
}

/* _core.pyx:201-225 */
void mmo_ghat_2d(int nx, int ny, int nv1, int nv2, const double *M,
                 const double *u1, const double *u2, const double *T,
                 const double *s11, const double *s12, const double *gT1,
                 const double *gT2, const double *tau, const double *v1,
                 const double *v2, double *out)
{
    size_t V = (size_t)nv1 * nv2;
    #pragma omp parallel for schedule(static)
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j) {
            int c = i * ny + j;
            double inv2T = 1.0 / (2.0 * T[c]);
            double invT = 1.0 / T[c];
            double invtau = 1.0 / tau[c];
            for (int k = 0; k < nv1; ++k) {
                double w1 = v1[k] - u1[c];
                for (int l = 0; l < nv2; ++l) {
                    double w2 = v2[l] - u2[c];
                    double bs = (-w2 * w2 * s11[c] + 2.0 * w1 * w2 * s12[c] + w1 * w1 * s11[c]) * inv2T;
                    double cg = ((w1 * w1 + w2 * w2) * inv2T - 2.0) * (w1 * gT1[c] + w2 * gT2[c]) * invT;
                    out[c * V + k * nv2 + l] = -(bs + cg) * M[c * V + k * nv2 + l] * invtau;
                }
            }
        }
}

/* _core.pyx:228-250 (in place on Ghat) */
void mmo_add_gaussian_term_2d(int nx, int ny, int nv1, int nv2, double *Ghat,
                              const double *M, const double *rho, const double *u1,
                              const double *u2, const double *m11, const double *m12,
                              const double *m22, double eps, const double *v1,
                              const double *v2)
{
    size_t V = (size_t)nv1 * nv2;
    double inveps = 1.0 / eps;
    #pragma omp parallel for schedule(static)
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j) {
            int c = i * ny + j;
            double c11 = m11[c], c12 = m12[c], c22 = m22[c];
            double det = c11 * c22 - c12 * c12;
            double pref = rho[c] / (2.0 * PI_D * sqrt(det));
            for (int k = 0; k < nv1; ++k) {
                double w1 = v1[k] - u1[c];
                for (int l = 0; l < nv2; ++l) {
                    double w2 = v2[l] - u2[c];
                    double quad = (c22 * w1 * w1 - 2.0 * c12 * w1 * w2 + c11 * w2 * w2) / det;
                    Ghat[c * V + k * nv2 + l] += (pref * exp(-0.5 * quad) - M[c * V + k * nv2 + l]) * inveps;
                }
            }
        }
}

/* _core.pyx:253-267 (in place) */
void mmo_add_lowrank_4d(int nx, int ny, int nv1, int nv2, double *out, int nterms,
                        const double *coeffs, const double *shapes)
{
    size_t V = (size_t)nv1 * nv2, S = (size_t)nx * ny;
    #pragma omp parallel for schedule(static)
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j) {
            size_t c = (size_t)i * ny + j;
            for (int m = 0; m < nterms; ++m) {
                double cm = coeffs[m * S + c];
                for (size_t n = 0; n < V; ++n) out[c * V + n] += cm * shapes[m * V + n];
            }
        }
}

/* _core.pyx:270-286 */
void mmo_relax_2d(int nx, int ny, int nv1, int nv2, const double *G,
                  const double *Ghat, const double *tau, double dt, double eps,
                  double *out)
{
    size_t V = (size_t)nv1 * nv2;
    #pragma omp parallel for schedule(static)
    for (int c = 0; c < nx * ny; ++c) {
        double denom = eps + dt * tau[c];
        double wg = eps / denom, wh = dt * tau[c] / denom;
        for (size_t n = 0; n < V; ++n)
            out[c * V + n] = wg * G[c * V + n] + wh * Ghat[c * V + n];
    }
}

/* _core.pyx:289-322; H is (4, nx, ny) */
void mmo_heat_tensor_2d(int nx, int ny, int nv1, int nv2, const double *G,
                        const double *u1, const double *u2, const double *v1,
                        const double *v2, double dv, double eps, double *H)
{
    size_t V = (size_t)nv1 * nv2, S = (size_t)nx * ny;
    double f = eps * dv;
    #pragma omp parallel for schedule(static)
    for (int c = 0; c < nx * ny; ++c) {
        double s111 = 0.0, s112 = 0.0, s122 = 0.0, s222 = 0.0;
        for (int k = 0; k < nv1; ++k) {
            double w1 = v1[k] - u1[c];
            for (int l = 0; l < nv2; ++l) {
                double w2 = v2[l] - u2[c];
                double g = G[c * V + k * nv2 + l];
                s111 += w1 * w1 * w1 * g;
                s112 += w1 * w1 * w2 * g;
                s122 += w1 * w2 * w2 * g;
                s222 += w2 * w2 * w2 * g;
            }
        }
        H[0 * S + c] = f * s111; H[1 * S + c] = f * s112;
        H[2 * S + c] = f * s122; H[3 * S + c] = f * s222;
    }
}

/* _core.pyx:20-33 */
void mmo_upwind_z_1d(int nx, int nv, const double *G_ext, const double *v, double dx,
                     double *Z)
{
    for (int i = 0; i < nx; ++i)
        for (int k = 0; k < nv; ++k) {
            double vk = v[k];
            if (vk >= 0.0) Z[i * nv + k] = vk * (G_ext[(i + 1) * nv + k] - G_ext[i * nv + k]) / dx;
            else Z[i * nv + k] = vk * (G_ext[(i + 2) * nv + k] - G_ext[(i + 1) * nv + k]) / dx;
        }
}

/* _core.pyx:36-63 */
void mmo_project_field_1d(int nx, int nv, const double *F, const double *M,
                          const double *rho, const double *u, const double *T,
                          const double *v, double dv, double *out)
{
    for (int i = 0; i < nx; ++i) {
        double st = sqrt(T[i]), scale = dv / rho[i];
        double a1 = 0.0, a2 = 0.0, a3 = 0.0;
        for (int k = 0; k < nv; ++k) {
            double w = (v[k] - u[i]) / st;
            double b3 = SQRT2_D * (0.5 * w * w - 0.5);
            double f = F[i * nv + k];
            a1 += f; a2 += f * w; a3 += f * b3;
        }
        a1 *= scale; a2 *= scale; a3 *= scale;
        for (int k = 0; k < nv; ++k) {
            double w = (v[k] - u[i]) / st;
            double b3 = SQRT2_D * (0.5 * w * w - 0.5);
            out[i * nv + k] = (a1 + w * a2 + b3 * a3) * M[i * nv + k];
        }
    }
}

/* ------------------------------------------------------------------------ */
/* 2D boundary machinery: boundary.py:181-378                                */
/* ------------------------------------------------------------------------ */

/* specular ghost of one cell: the edge cell mirrored in v_n (axis 0: k
 * reversed, axis 1: l reversed) */
static void mirror_cell(const mmo_cfg2d *cf, const double *edge, int axis, double *dst)
{
    int nv1 = cf->nv1, nv2 = cf->nv2;
    for (int k = 0; k < nv1; ++k)
        for (int l = 0; l < nv2; ++l)
            dst[k * nv2 + l] = axis == 0 ? edge[(nv1 - 1 - k) * nv2 + l]
                                         : edge[k * nv2 + (nv2 - 1 - l)];
}

/* extend_micro_2d (boundary.py:181-210): wrap / copy edge / zero (wall) /
 * mirror (specular extension) */
static void extend_micro(const mmo_cfg2d *cf, const double *G, int axis, double *G_ext)
{
    int nx = cf->nx, ny = cf->ny;
    size_t V = (size_t)cf->nv1 * cf->nv2;
    int lo = cf->face[axis == 0 ? 0 : 2], hi = cf->face[axis == 0 ? 1 : 3];
    if (axis == 0) {
        size_t row = (size_t)ny * V;
        memcpy(G_ext + row, G, (size_t)nx * row * sizeof(double));
        if (lo == FACE_PERIODIC) {
            memcpy(G_ext, G + (size_t)(nx - 1) * row, row * sizeof(double));
            memcpy(G_ext + (size_t)(nx + 1) * row, G, row * sizeof(double));
            return;
        }
        if (lo == FACE_EXTRAPOLATE) memcpy(G_ext, G, row * sizeof(double));
        else if (lo == FACE_SPECULAR)
            for (int j = 0; j < ny; ++j) mirror_cell(cf, G + (size_t)j * V, 0, G_ext + (size_t)j * V);
        else memset(G_ext, 0, row * sizeof(double));
        if (hi == FACE_EXTRAPOLATE)
            memcpy(G_ext + (size_t)(nx + 1) * row, G + (size_t)(nx - 1) * row, row * sizeof(double));
        else if (hi == FACE_SPECULAR)
            for (int j = 0; j < ny; ++j)
                mirror_cell(cf, G + (size_t)((nx - 1) * ny + j) * V, 0,
                            G_ext + (size_t)((nx + 1) * ny + j) * V);
        else memset(G_ext + (size_t)(nx + 1) * row, 0, row * sizeof(double));
    } else {
        int eny = ny + 2;
        #pragma omp parallel for schedule(static)
        for (int i = 0; i < nx; ++i) {
            double *dst = G_ext + (size_t)i * eny * V;
            const double *src = G + (size_t)i * ny * V;
            memcpy(dst + V, src, (size_t)ny * V * sizeof(double));
            if (lo == FACE_PERIODIC) {
                memcpy(dst, src + (size_t)(ny - 1) * V, V * sizeof(double));
                memcpy(dst + (size_t)(ny + 1) * V, src, V * sizeof(double));
            } else {
                if (lo == FACE_EXTRAPOLATE) memcpy(dst, src, V * sizeof(double));
                else if (lo == FACE_SPECULAR) mirror_cell(cf, src, 1, dst);
                else memset(dst, 0, V * sizeof(double));
                if (hi == FACE_EXTRAPOLATE)
                    memcpy(dst + (size_t)(ny + 1) * V, src + (size_t)(ny - 1) * V, V * sizeof(double));
                else if (hi == FACE_SPECULAR)
                    mirror_cell(cf, src + (size_t)(ny - 1) * V, 1, dst + (size_t)(ny + 1) * V);
                else memset(dst + (size_t)(ny + 1) * V, 0, V * sizeof(double));
            }
        }
    }
}

/* extend_macro_scalar_2d (boundary.py:213-221): wrap for periodic else copy;
 * at a specular face the ghost of a field odd in that axis' velocity (u1 in
 * x, u2 in y) is the negated edge value (odd_x / odd_y) */
static double ext_scalar(const mmo_cfg2d *cf, const double *f, int i, int j, int odd_x, int odd_y)
{
    int nx = cf->nx, ny = cf->ny;
    double sg = 1.0;
    if ((i < 0 && cf->face[0] == FACE_SPECULAR) || (i >= nx && cf->face[1] == FACE_SPECULAR))
        if (odd_x) sg = -sg;
    if ((j < 0 && cf->face[2] == FACE_SPECULAR) || (j >= ny && cf->face[3] == FACE_SPECULAR))
        if (odd_y) sg = -sg;
    if (i < 0) i = cf->face[0] == FACE_PERIODIC ? nx - 1 : 0;
    if (i >= nx) i = cf->face[0] == FACE_PERIODIC ? 0 : nx - 1;
    if (j < 0) j = cf->face[2] == FACE_PERIODIC ? ny - 1 : 0;
    if (j >= ny) j = cf->face[2] == FACE_PERIODIC ? 0 : ny - 1;
    return sg < 0.0 ? -f[i * ny + j] : f[i * ny + j];
}

static const int SIGN_2D[4] = { -1, +1, -1, +1 };   /* boundary.py:263 */

/* wall_density_ratio_2d (boundary.py:248-260) times rho (266-270) */
static double wall_density(double rho, double ua, double taa, double Tw, int sign)
{
    double R = sqrt(taa / Tw) * exp(-ua * ua / (2.0 * taa))
             + ua * sqrt(PI_D / (2.0 * Tw)) * (erf(ua / sqrt(2.0 * taa)) + (double)sign);
    return rho * R;
}

/* wall_ghost_state_2d (boundary.py:273-290): (rho_w, g1, g2, T11, T12, T22) */
static void wall_ghost_state(const mmo_cfg2d *cf, int face, double rho, double u1,
                             double u2, double t11, double t22, double out[6])
{
    double Tw = cf->wall_T[face], U = cf->wall_U[face];
    if (face < 2) {
        out[0] = wall_density(rho, u1, t11, Tw, SIGN_2D[face]);
        out[1] = 0.0; out[2] = U;
    } else {
        out[0] = wall_density(rho, u2, t22, Tw, SIGN_2D[face]);
        out[1] = U; out[2] = 0.0;
    }
    out[3] = Tw; out[4] = 0.0; out[5] = Tw;
}

/* _wall_maxwellian_layer (boundary.py:293-301) at one (k, l) */
static double wall_maxwellian(double rw, double g1, double g2, double Tw, double v1, double v2)
{
    double w1 = v1 - g1, w2 = v2 - g2;
    return rw / (2.0 * PI_D * Tw) * exp(-(w1 * w1 + w2 * w2) / (2.0 * Tw));
}

/* ghat_override_2d (boundary.py:343-378).  Builds the upwind Maxwellian
 * transport term with ghost Maxwellians (extend_maxwellian_2d, 304-340),
 * projects it with project_field_2d and overwrites the wall strips. */
static void ghat_override(const mmo_cfg2d *cf, double *Ghat, const double *M,
                          const prim2 *P, const double *rho, const double *u1,
                          const double *u2, const double *T, const double *tau)
{
    int nx = cf->nx, ny = cf->ny, nv1 = cf->nv1, nv2 = cf->nv2;
    size_t V = (size_t)nv1 * nv2;
    const double *v1 = cf->v1, *v2 = cf->v2;
    double dv = (v1[1] - v1[0]) * (v2[1] - v2[0]);
    int any = 0;
    for (int f = 0; f < 4; ++f) any |= cf->face[f] == FACE_WALL;
    if (!any) return;
    #pragma omp parallel
    {
        double *Mt = (double *)malloc(V * sizeof(double));
        double *Mn[4];
        for (int f = 0; f < 4; ++f) Mn[f] = (double *)malloc(V * sizeof(double));
        #pragma omp for schedule(dynamic)
        for (int i = 0; i < nx; ++i)
            for (int j = 0; j < ny; ++j) {
                int on = (cf->face[0] == FACE_WALL && i == 0) || (cf->face[1] == FACE_WALL && i == nx - 1)
                      || (cf->face[2] == FACE_WALL && j == 0) || (cf->face[3] == FACE_WALL && j == ny - 1);
                if (!on) continue;
                int c = i * ny + j;
                /* neighbour Maxwellians: 0 = x-1, 1 = x+1, 2 = y-1, 3 = y+1 */
                for (int f = 0; f < 4; ++f) {
                    int ii = i + (f == 0 ? -1 : f == 1 ? 1 : 0);
                    int jj = j + (f == 2 ? -1 : f == 3 ? 1 : 0);
                    int outside = ii < 0 || ii >= nx || jj < 0 || jj >= ny;
                    int face = f;   /* face index coincides with the neighbour slot */
                    if (outside && cf->face[face] == FACE_WALL) {
                        /* wall-emitted Maxwellian from the edge cell (i, j) */
                        const prim2 *e = &P[c];
                        double g[6];
                        wall_ghost_state(cf, face, e->rho, e->u1, e->u2, e->t11, e->t22, g);
                        for (int k = 0; k < nv1; ++k)
                            for (int l = 0; l < nv2; ++l)
                                Mn[f][k * nv2 + l] = wall_maxwellian(g[0], g[1], g[2], cf->wall_T[face], v1[k], v2[l]);
                        continue;
                    }
                    if (outside && cf->face[face] == FACE_SPECULAR) {
                        mirror_cell(cf, M + (size_t)c * V, face < 2 ? 0 : 1, Mn[f]);
                        continue;
                    }
                    if (outside) {
                        if (cf->face[face] == FACE_PERIODIC) {
                            ii = (ii + nx) % nx; jj = (jj + ny) % ny;
                        } else {
                            ii = ii < 0 ? 0 : ii >= nx ? nx - 1 : ii;
                            jj = jj < 0 ? 0 : jj >= ny ? ny - 1 : jj;
                        }
                    }
                    memcpy(Mn[f], M + (size_t)(ii * ny + jj) * V, V * sizeof(double));
                }
                const double *m = M + (size_t)c * V;
                for (int k = 0; k < nv1; ++k) {
                    double vm1 = v1[k] < 0.0 ? v1[k] : 0.0, vp1 = v1[k] > 0.0 ? v1[k] : 0.0;
                    for (int l = 0; l < nv2; ++l) {
                        double vm2 = v2[l] < 0.0 ? v2[l] : 0.0, vp2 = v2[l] > 0.0 ? v2[l] : 0.0;
                        int n = k * nv2 + l;
                        Mt[n] = (vm1 * (Mn[1][n] - m[n]) + vp1 * (m[n] - Mn[0][n])) / cf->dx
                              + (vm2 * (Mn[3][n] - m[n]) + vp2 * (m[n] - Mn[2][n])) / cf->dy;
                    }
                }
                double a[4];
                proj_coeffs(Mt, nv1, v1, nv2, v2, rho[c], u1[c], u2[c], T[c], dv, a);
                double st = sqrt(T[c]);
                for (int k = 0; k < nv1; ++k) {
                    double w1 = (v1[k] - u1[c]) / st;
                    for (int l = 0; l < nv2; ++l) {
                        double w2 = (v2[l] - u2[c]) / st;
                        double b4 = 0.5 * (w1 * w1 + w2 * w2) - 1.0;
                        int n = k * nv2 + l;
                        double pi_n = (a[0] + w1 * a[1] + w2 * a[2] + b4 * a[3]) * m[n];
                        Ghat[(size_t)c * V + n] = -(Mt[n] - pi_n) / tau[c];
                    }
                }
            }
        free(Mt);
        for (int f = 0; f < 4; ++f) free(Mn[f]);
    }
}

/* ------------------------------------------------------------------------ */
/* macro 2D: macro2d.py                                                      */
/* ------------------------------------------------------------------------ */

/* relax_pressure_2d (macro2d.py:55-70), trbdf2_w (41-52) */
static int relax_pressure(const mmo_cfg2d *cf, double dt, const double *Q, double *Qn,
                          prim2 *P, mmo_err *err)
{
    int n = cf->nx * cf->ny;
    int rc = prims_field(n, cf->ny, Q, P, err);
    if (rc) return rc;
    double e2 = 48.0 * cf->eps * cf->eps;
    for (int c = 0; c < n; ++c) {
        const prim2 *p = &P[c];
        double tau = tau_of(cf->tau_kind, cf->tau_value, p->rho, p->T);
        double z = tau * (1.0 - cf->nu) * dt;
        double W = (e2 - 10.0 * z * cf->eps) / (e2 + 14.0 * z * cf->eps + z * z);
        double p11 = p->rho * p->t11, p12 = p->rho * p->t12, p22 = p->rho * p->t22;
        double *q = Qn + 6 * c;
        q[0] = Q[6 * c]; q[1] = Q[6 * c + 1]; q[2] = Q[6 * c + 2];
        q[3] = p->rho * p->u1 * p->u1 + 0.5 * ((1.0 + W) * p11 + (1.0 - W) * p22);
        q[4] = p->rho * p->u1 * p->u2 + W * p12;
        q[5] = p->rho * p->u2 * p->u2 + 0.5 * ((1.0 - W) * p11 + (1.0 + W) * p22);
    }
    return MMO_OK;
}

/* _split_parts_x/_y (macro2d.py:102-127) and the half of _kfvs (130-138)
 * contributed by one side: sgn = +1 left/down, -1 right/up. */
static void kfvs_half(int axis, const double s[6], double sgn, double out[6])
{
    double rho = s[0], u1 = s[1], u2 = s[2], p11 = s[3], p12 = s[4], p22 = s[5];
    double a, b, J[6], K[6];
    if (axis == 0) {
        a = sqrt(2.0 * p11 / (PI_D * rho)) * exp(-rho * u1 * u1 / (2.0 * p11));
        b = erf(u1 * sqrt(rho / (2.0 * p11)));
        J[0] = rho; J[1] = rho * u1; J[2] = rho * u2;
        J[3] = rho * u1 * u1 + 2.0 * p11;
        J[4] = rho * u1 * u2 + 2.0 * p12;
        J[5] = rho * u2 * u2 + p22 + p12 * p12 / p11;
        /* physical_flux_x_2d (77-87) */
        K[0] = rho * u1; K[1] = rho * u1 * u1 + p11; K[2] = rho * u1 * u2 + p12;
        K[3] = rho * pow(u1, 3.0) + 3.0 * u1 * p11;
        K[4] = rho * u1 * u1 * u2 + u2 * p11 + 2.0 * u1 * p12;
        K[5] = rho * u1 * u2 * u2 + u1 * p22 + 2.0 * u2 * p12;
    } else {
        a = sqrt(2.0 * p22 / (PI_D * rho)) * exp(-rho * u2 * u2 / (2.0 * p22));
        b = erf(u2 * sqrt(rho / (2.0 * p22)));
        J[0] = rho; J[1] = rho * u1; J[2] = rho * u2;
        J[3] = rho * u1 * u1 + p11 + p12 * p12 / p22;
        J[4] = rho * u1 * u2 + 2.0 * p12;
        J[5] = rho * u2 * u2 + 2.0 * p22;
        /* physical_flux_y_2d (90-99) */
        K[0] = rho * u2; K[1] = rho * u1 * u2 + p12; K[2] = rho * u2 * u2 + p22;
        K[3] = rho * u1 * u1 * u2 + u2 * p11 + 2.0 * u1 * p12;
        K[4] = rho * u1 * u2 * u2 + u1 * p22 + 2.0 * u2 * p12;
        K[5] = rho * pow(u2, 3.0) + 3.0 * u2 * p22;
    }
    double sa = sgn * a, sb = 1.0 + sgn * b;
    for (int m = 0; m < 6; ++m) out[m] = 0.5 * (sa * J[m] + sb * K[m]);
}

/* pressure-primitive state of one cell (_pressure_fields, 201-203) */
static void pstate(const prim2 *p, double s[6])
{
    s[0] = p->rho; s[1] = p->u1; s[2] = p->u2;
    s[3] = p->rho * p->t11; s[4] = p->rho * p->t12; s[5] = p->rho * p->t22;
}

/* extended state beyond a physical face (_extended_states, 153-181) */
static void ghost_pstate(const mmo_cfg2d *cf, int face, const double edge[6], double s[6])
{
    if (cf->face[face] == FACE_EXTRAPOLATE) { memcpy(s, edge, 6 * sizeof(double)); return; }
    if (cf->face[face] == FACE_SPECULAR) {
        /* mirror image: normal velocity and P12 change sign */
        memcpy(s, edge, 6 * sizeof(double));
        s[face < 2 ? 1 : 2] = -edge[face < 2 ? 1 : 2];
        s[4] = -edge[4];
        return;
    }
    double rho = edge[0];
    double t11 = edge[3] / rho, t22 = edge[5] / rho;
    double g[6];
    wall_ghost_state(cf, face, rho, edge[1], edge[2], t11, t22, g);
    s[0] = g[0]; s[1] = g[1]; s[2] = g[2];
    s[3] = g[0] * g[3]; s[4] = g[0] * g[4]; s[5] = g[0] * g[5];
}

/* interface_heat_2d (boundary.py:224-241) at interface index m in [0, n].
 * Specular faces: mean of the edge value and its mirror image, which is
 * -edge for the components odd in v_n (odd != 0). */
static double iface_heat(const mmo_cfg2d *cf, int axis, const double *h, int n,
                         int stride, int m, int odd)
{
    int lo = cf->face[axis == 0 ? 0 : 2], hi = cf->face[axis == 0 ? 1 : 3];
    if (m > 0 && m < n) return 0.5 * (h[m * stride] + h[(m - 1) * stride]);
    if (lo == FACE_PERIODIC) return 0.5 * (h[0] + h[(n - 1) * stride]);
    if (m == 0) {
        if (lo == FACE_SPECULAR) return 0.5 * (h[0] + (odd ? -h[0] : h[0]));
        return lo == FACE_EXTRAPOLATE ? h[0] : 0.5 * h[0];
    }
    double e = h[(n - 1) * stride];
    if (hi == FACE_SPECULAR) return 0.5 * ((odd ? -e : e) + e);
    return hi == FACE_EXTRAPOLATE ? e : 0.5 * e;
}

/* _sweep (macro2d.py:206-221) along `axis`; hc = the three H components */
static int sweep(const mmo_cfg2d *cf, const double *Q, const double *const hc[3],
                 double dt, int axis, double *Qn, prim2 *P, mmo_err *err)
{
    int nx = cf->nx, ny = cf->ny, n = nx * ny;
    int rc = prims_field(n, ny, Q, P, err);
    if (rc) return rc;
    double d = axis == 0 ? cf->dx : cf->dy;
    double r = dt / d;
    int len = axis == 0 ? nx : ny;                 /* cells along the axis */
    int lines = axis == 0 ? ny : nx;
    #pragma omp parallel for schedule(static)
    for (int line = 0; line < lines; ++line) {
        double *F = (double *)malloc((size_t)(len + 1) * 6 * sizeof(double));
        int face_lo = axis == 0 ? 0 : 2, face_hi = face_lo + 1;
        for (int m = 0; m <= len; ++m) {
            double L[6], R[6], sl[6], sr[6];
            int il = m - 1, ir = m;
            /* left state */
            if (il < 0) {
                if (cf->face[face_lo] == FACE_PERIODIC) il = len - 1;
            }
            if (ir >= len) {
                if (cf->face[face_hi] == FACE_PERIODIC) ir = 0;
            }
#define CELL(p) (axis == 0 ? ((p) * ny + line) : (line * ny + (p)))
            if (il >= 0) pstate(&P[CELL(il)], sl);
            if (ir < len) pstate(&P[CELL(ir)], sr);
            if (il < 0) ghost_pstate(cf, face_lo, sr, sl);
            if (ir >= len) ghost_pstate(cf, face_hi, sl, sr);
            kfvs_half(axis, sl, 1.0, L);
            kfvs_half(axis, sr, -1.0, R);
            for (int q = 0; q < 6; ++q) F[m * 6 + q] = (0.0 + L[q]) + R[q];
        }
        for (int p = 0; p < len; ++p) {
            int c = CELL(p);
            for (int q = 0; q < 6; ++q)
                Qn[6 * c + q] = Q[6 * c + q] - r * (F[(p + 1) * 6 + q] - F[p * 6 + q]);
        }
        for (int t = 0; t < 3; ++t) {
            const double *h = hc[t];
            int stride = axis == 0 ? ny : 1;
            const double *hl = axis == 0 ? h + line : h + (size_t)line * ny;
            for (int p = 0; p < len; ++p) {
                int c = CELL(p);
                /* H111, H122 odd in v1; H112, H222 odd in v2: in both sweeps
                 * the components t = 0 and 2 are the odd ones */
                double hp = iface_heat(cf, axis, hl, len, stride, p + 1, t != 1);
                double hm = iface_heat(cf, axis, hl, len, stride, p, t != 1);
                Qn[6 * c + 3 + t] -= r * (hp - hm);
            }
        }
#undef CELL
        free(F);
    }
    return MMO_OK;
}

/* ------------------------------------------------------------------------ */
/* full 2D step: runner/loop.py:82-111 with micro2d.py:102-127 and         */
/* macro2d.py:224-240                                                       */
/* ------------------------------------------------------------------------ */
int mmo_step_2d(const mmo_cfg2d *cf, const double *Q, const double *G, double dt,
                int nsrc, const double *src_coeffs, const double *src_shapes,
                const double *qsrc, double *Q_out, double *G_out, double *H_out,
                mmo_err *err)
{
    int nx = cf->nx, ny = cf->ny, nv1 = cf->nv1, nv2 = cf->nv2;
    int n = nx * ny;
    size_t V = (size_t)nv1 * nv2, SV = (size_t)n * V;
    const double *v1 = cf->v1, *v2 = cf->v2;
    int rc = MMO_OK;
    err->code = ERR_NONE; err->i = err->j = -1; err->value = 0.0;

    prim2 *P = (prim2 *)malloc((size_t)n * sizeof(prim2));
    double *rho = (double *)malloc((size_t)n * sizeof(double) * 14);
    double *u1 = rho + n, *u2 = rho + 2 * n, *T = rho + 3 * n, *tau = rho + 4 * n;
    double *s11 = rho + 5 * n, *s12 = rho + 6 * n, *gT1 = rho + 7 * n, *gT2 = rho + 8 * n;
    double *m11 = rho + 9 * n, *m12 = rho + 10 * n, *m22 = rho + 11 * n;
    double *M = (double *)malloc(SV * sizeof(double));
    size_t ext_n = (size_t)(nx + 2) * (ny + 2) * V;
    double *Gext = (double *)malloc(ext_n * sizeof(double));
    double *Gs = (double *)malloc(SV * sizeof(double));
    double *Gss = (double *)malloc(SV * sizeof(double));
    double *Ghat = (double *)malloc(SV * sizeof(double));
    double *Qa = (double *)malloc((size_t)n * 6 * sizeof(double) * 3);
    double *Qb = Qa + 6 * n, *Qc = Qa + 12 * n;

    /* prims at t^n (loop.py:98) and tau (loop.py:99) */
    rc = prims_field(n, ny, Q, P, err);
    if (rc) goto done;
    for (int c = 0; c < n; ++c) {
        rho[c] = P[c].rho; u1[c] = P[c].u1; u2[c] = P[c].u2; T[c] = P[c].T;
        tau[c] = tau_of(cf->tau_kind, cf->tau_value, P[c].rho, P[c].T);
    }
    /* M^n (loop.py:100-103) */
    mmo_maxwellian_field_2d(nx, ny, rho, u1, u2, T, nv1, v1, nv2, v2, M);

    /* x-transport (micro2d.py:23-27) then y-transport on G* (30-34) */
    extend_micro(cf, G, 0, Gext);
    mmo_transport_stage_2d(nx, ny, nv1, nv2, Gext, M, rho, u1, u2, T, v1, v2, cf->dx, dt, 0, Gs);
    extend_micro(cf, Gs, 1, Gext);
    mmo_transport_stage_2d(nx, ny, nv1, nv2, Gext, M, rho, u1, u2, T, v1, v2, cf->dy, dt, 1, Gss);

    /* ghat (micro2d.py:70-99) with sigma_grad_t_2d (37-60) */
    for (int i = 0; i < nx; ++i)
        for (int j = 0; j < ny; ++j) {
            int c = i * ny + j;
            double du1x = (ext_scalar(cf, u1, i + 1, j, 1, 0) - ext_scalar(cf, u1, i - 1, j, 1, 0)) / (2.0 * cf->dx);
            double du2x = (ext_scalar(cf, u2, i + 1, j, 0, 1) - ext_scalar(cf, u2, i - 1, j, 0, 1)) / (2.0 * cf->dx);
            double du1y = (ext_scalar(cf, u1, i, j + 1, 1, 0) - ext_scalar(cf, u1, i, j - 1, 1, 0)) / (2.0 * cf->dy);
            double du2y = (ext_scalar(cf, u2, i, j + 1, 0, 1) - ext_scalar(cf, u2, i, j - 1, 0, 1)) / (2.0 * cf->dy);
            s11[c] = du1x - du2y;
            s12[c] = du1y + du2x;
            gT1[c] = (ext_scalar(cf, T, i + 1, j, 0, 0) - ext_scalar(cf, T, i - 1, j, 0, 0)) / (2.0 * cf->dx);
            gT2[c] = (ext_scalar(cf, T, i, j + 1, 0, 0) - ext_scalar(cf, T, i, j - 1, 0, 0)) / (2.0 * cf->dy);
        }
    mmo_ghat_2d(nx, ny, nv1, nv2, M, u1, u2, T, s11, s12, gT1, gT2, tau, v1, v2, Ghat);
    if (cf->nu != 0.0) {
        /* modify_tensor (gas_state.py:138-146) with its SPD check */
        for (int c = 0; c < n; ++c) {
            m11[c] = (1.0 - cf->nu) * T[c] + cf->nu * P[c].t11;
            m12[c] = cf->nu * P[c].t12;
            m22[c] = (1.0 - cf->nu) * T[c] + cf->nu * P[c].t22;
        }
        for (int c = 0; c < n; ++c) {
            double det;
            if (spd_bad(m11[c], m12[c], m22[c], &det)) {
                err->code = ERR_MODIFIED_SPD; err->i = c / ny; err->j = c % ny; err->value = det;
                rc = MMO_INVALID_STATE;
                goto done;
            }
        }
        /* _is_isotropic (micro2d.py:63-67) guard for eps < 1e-10 (96) */
        int iso = 0;
        if (cf->eps < 1e-10) {
            double tmax = T[0], d11 = 0, d12 = 0, d22 = 0;
            for (int c = 0; c < n; ++c) {
                if (T[c] > tmax) tmax = T[c];
                if (fabs(m11[c] - T[c]) > d11) d11 = fabs(m11[c] - T[c]);
                if (fabs(m12[c]) > d12) d12 = fabs(m12[c]);
                if (fabs(m22[c] - T[c]) > d22) d22 = fabs(m22[c] - T[c]);
            }
            double tol = 1e-13 * tmax;
            iso = d11 <= tol && d12 <= tol && d22 <= tol;
        }
        if (!iso)
            mmo_add_gaussian_term_2d(nx, ny, nv1, nv2, Ghat, M, rho, u1, u2, m11, m12, m22,
                                     cf->eps, v1, v2);
    }
    /* optional manufactured-solution source (micro2d.py:120-123) */
    if (nsrc > 0) {
        double *cs = (double *)malloc((size_t)nsrc * n * sizeof(double));
        for (int m = 0; m < nsrc; ++m)
            for (int c = 0; c < n; ++c) cs[m * n + c] = src_coeffs[m * n + c] / tau[c];
        mmo_add_lowrank_4d(nx, ny, nv1, nv2, Ghat, nsrc, cs, src_shapes);
        free(cs);
    }
    /* diffuse-wall override (micro2d.py:124-126) */
    ghat_override(cf, Ghat, M, P, rho, u1, u2, T, tau);
    /* implicit collision (micro2d.py:127) */
    mmo_relax_2d(nx, ny, nv1, nv2, Gss, Ghat, tau, dt, cf->eps, G_out);

    /* heat tensor with u^n (loop.py:108) */
    double dv = (v1[1] - v1[0]) * (v2[1] - v2[0]);
    mmo_heat_tensor_2d(nx, ny, nv1, nv2, G_out, u1, u2, v1, v2, dv, cf->eps, H_out);

    /* macro step (macro2d.py:224-240) */
    {
        const double *H111 = H_out, *H112 = H_out + n, *H122 = H_out + 2 * n, *H222 = H_out + 3 * n;
        const double *hx[3] = { H111, H112, H122 };
        const double *hy[3] = { H112, H122, H222 };
        rc = relax_pressure(cf, dt, Q, Qa, P, err); if (rc) goto done;
        rc = sweep(cf, Qa, hx, dt, 0, Qb, P, err); if (rc) goto done;
        rc = sweep(cf, Qb, hy, dt, 1, Qc, P, err); if (rc) goto done;
        if (qsrc)
            for (int c = 0; c < 6 * n; ++c) Qc[c] = Qc[c] + dt * qsrc[c];
        rc = relax_pressure(cf, dt, Qc, Q_out, P, err); if (rc) goto done;
    }
done:
    free(P); free(rho); free(M); free(Gext); free(Gs); free(Gss); free(Ghat); free(Qa);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* 1D path (config 1): runner/loop.py:31-51, micro1d.py, macro1d.py,         */
/* boundary.py:84-170                                                        */
/* ------------------------------------------------------------------------ */
static void alpha_beta(double u, double T, double *alpha, double *bp, double *bm)
{
    *alpha = sqrt(T / (2.0 * PI_D)) * exp(-u * u / (2.0 * T));
    double s = erf(u / sqrt(2.0 * T));
    *bp = 0.5 * (1.0 + s); *bm = 0.5 * (1.0 - s);
}

/* wall_density_1d (boundary.py:94-105) */
static double wall_density_1d(double rho, double u, double T, double Tw, int right)
{
    double alpha, bp, bm;
    alpha_beta(u, T, &alpha, &bp, &bm);
    if (!right) return sqrt(2.0 * PI_D / Tw) * (rho * alpha - rho * u * bm);
    return sqrt(2.0 * PI_D / Tw) * (rho * alpha + rho * u * bp);
}

/* wall_interface_temperature_1d (boundary.py:108-122) */
static double wall_iface_T_1d(double rho, double u, double T, double Tw, int right)
{
    double alpha, bp, bm;
    alpha_beta(u, T, &alpha, &bp, &bm);
    double rho_w = wall_density_1d(rho, u, T, Tw, right);
    double num, den;
    if (!right) {
        num = 0.5 * rho_w * Tw + rho * ((T + u * u) * bm - u * alpha);
        den = 0.5 * rho_w + rho * bm;
    } else {
        num = rho * ((T + u * u) * bp + u * alpha) + 0.5 * rho_w * Tw;
        den = rho * bp + 0.5 * rho_w;
    }
    return num / den;
}

/* kfvs_flux_1d (macro1d.py:34-51) */
static void kfvs_1d(const double l[3], const double r[3], double F[3])
{
    double out[3] = { 0.0, 0.0, 0.0 };
    for (int side = 0; side < 2; ++side) {
        const double *s = side == 0 ? l : r;
        double sign = side == 0 ? 1.0 : -1.0;
        double rho = s[0], u = s[1], T = s[2];
        double alpha, bp, bm;
        alpha_beta(u, T, &alpha, &bp, &bm);
        double half[3] = { rho, rho * u, 0.5 * rho * (2.0 * T + u * u) };
        double beta = sign > 0 ? bp : bm;
        /* physical_flux_1d (macro1d.py:28-31) */
        double f[3] = { rho * u, rho * (T + u * u), 0.5 * rho * u * (3.0 * T + u * u) };
        for (int m = 0; m < 3; ++m) out[m] = out[m] + sign * alpha * half[m] + beta * f[m];
    }
    memcpy(F, out, sizeof(out));
}

int mmo_step_1d(const mmo_cfg1d *cf, const double *Q, const double *G, double dt,
                const double *src /*(nx,nv) or NULL*/, const double *qsrc /*(nx,3) or NULL*/,
                double *Q_out, double *G_out, double *H_out, mmo_err *err)
{
    int nx = cf->nx, nv = cf->nv;
    const double *v = cf->v;
    double dx = cf->dx, dv = v[1] - v[0];
    err->code = ERR_NONE; err->i = err->j = -1; err->value = 0.0;
    double *rho = (double *)malloc((size_t)nx * 5 * sizeof(double));
    double *u = rho + nx, *T = rho + 2 * nx, *tau = rho + 3 * nx;
    double *M = (double *)malloc((size_t)nx * nv * sizeof(double));
    double *Gext = (double *)malloc((size_t)(nx + 2) * nv * sizeof(double));
    double *Z = (double *)malloc((size_t)nx * nv * sizeof(double));
    double *Zh = (double *)malloc((size_t)nx * nv * sizeof(double));
    double *Th = (double *)malloc((size_t)(nx + 1) * sizeof(double));
    double *F = (double *)malloc((size_t)(nx + 1) * 3 * sizeof(double));
    double *Hh = (double *)malloc((size_t)(nx + 1) * sizeof(double));
    int rc = MMO_OK;
    /* primitives_1d (gas_state.py:43-53) */
    for (int i = 0; i < nx; ++i)
        if (!(Q[3 * i] > 0.0)) { err->code = ERR_DENSITY; err->i = i; err->value = Q[3 * i]; rc = MMO_INVALID_STATE; goto done; }
    for (int i = 0; i < nx; ++i) {
        rho[i] = Q[3 * i]; u[i] = Q[3 * i + 1] / rho[i];
        T[i] = (2.0 * Q[3 * i + 2] - rho[i] * u[i] * u[i]) / rho[i];
    }
    for (int i = 0; i < nx; ++i)
        if (!(T[i] > 0.0)) { err->code = ERR_TEMPERATURE; err->i = i; err->value = T[i]; rc = MMO_INVALID_STATE; goto done; }
    for (int i = 0; i < nx; ++i) tau[i] = tau_of(cf->tau_kind, cf->tau_value, rho[i], T[i]);
    /* maxwellian_1d (gas_state.py:128-129) */
    for (int i = 0; i < nx; ++i)
        for (int k = 0; k < nv; ++k)
            M[i * nv + k] = rho[i] / sqrt(2.0 * PI_D * T[i]) * exp(-pow(v[k] - u[i], 2.0) / (2.0 * T[i]));
    /* extend_micro_1d (boundary.py:141-157) */
    memcpy(Gext + nv, G, (size_t)nx * nv * sizeof(double));
    if (cf->face[0] == FACE_PERIODIC) {
        memcpy(Gext, G + (size_t)(nx - 1) * nv, nv * sizeof(double));
        memcpy(Gext + (size_t)(nx + 1) * nv, G, nv * sizeof(double));
    } else {
        if (cf->face[0] == FACE_EXTRAPOLATE) memcpy(Gext, G, nv * sizeof(double));
        else memset(Gext, 0, nv * sizeof(double));
        if (cf->face[1] == FACE_EXTRAPOLATE) memcpy(Gext + (size_t)(nx + 1) * nv, G + (size_t)(nx - 1) * nv, nv * sizeof(double));
        else memset(Gext + (size_t)(nx + 1) * nv, 0, nv * sizeof(double));
    }
    mmo_upwind_z_1d(nx, nv, Gext, v, dx, Z);
    mmo_project_field_1d(nx, nv, Z, M, rho, u, T, v, dv, Zh);
    /* interface_temperatures_1d (boundary.py:125-138) */
    for (int m = 1; m < nx; ++m) Th[m] = 0.5 * (T[m] + T[m - 1]);
    if (cf->face[0] == FACE_PERIODIC) Th[0] = Th[nx] = 0.5 * (T[0] + T[nx - 1]);
    else {
        Th[0] = cf->face[0] == FACE_EXTRAPOLATE ? T[0] : wall_iface_T_1d(rho[0], u[0], T[0], cf->wall_T[0], 0);
        Th[nx] = cf->face[1] == FACE_EXTRAPOLATE ? T[nx - 1]
               : wall_iface_T_1d(rho[nx - 1], u[nx - 1], T[nx - 1], cf->wall_T[1], 1);
    }
    /* ghat_1d (micro1d.py:22-31) and the blend (micro1d.py:56-64) */
    for (int i = 0; i < nx; ++i) {
        double dT = (Th[i + 1] - Th[i]) / (dx * T[i]);
        double wg = cf->eps / (cf->eps + dt * tau[i]);
        double wh = dt * tau[i] / (cf->eps + dt * tau[i]);
        for (int k = 0; k < nv; ++k) {
            double w = v[k] - u[i];
            double gh = -(pow(w, 3.0) / (2.0 * T[i]) - 1.5 * w) * (dT / tau[i]) * M[i * nv + k];
            if (src) gh = gh + src[i * nv + k] / tau[i];
            G_out[i * nv + k] = wg * (G[i * nv + k] - dt * (Z[i * nv + k] - Zh[i * nv + k])) + wh * gh;
        }
    }
    /* heat_flux_1d (macro1d.py:16-19): 0.5 eps dv (G @ v^3) */
    for (int i = 0; i < nx; ++i) {
        double s = 0.0;
        for (int k = 0; k < nv; ++k) s += G_out[i * nv + k] * pow(v[k], 3.0);
        H_out[i] = 0.5 * cf->eps * dv * s;
    }
    /* macro_step_1d (macro1d.py:78-92) with interface_fluxes_1d (54-75) */
    for (int m = 1; m < nx; ++m) {
        double l[3] = { rho[m - 1], u[m - 1], T[m - 1] }, r[3] = { rho[m], u[m], T[m] };
        kfvs_1d(l, r, F + 3 * m);
    }
    {
        double s0[3] = { rho[0], u[0], T[0] }, sn[3] = { rho[nx - 1], u[nx - 1], T[nx - 1] };
        if (cf->face[0] == FACE_PERIODIC) {
            kfvs_1d(sn, s0, F);
            memcpy(F + 3 * nx, F, 3 * sizeof(double));
        } else {
            if (cf->face[0] == FACE_EXTRAPOLATE) kfvs_1d(s0, s0, F);
            else {
                double w[3] = { wall_density_1d(rho[0], u[0], T[0], cf->wall_T[0], 0), 0.0, cf->wall_T[0] };
                kfvs_1d(w, s0, F);
            }
            if (cf->face[1] == FACE_EXTRAPOLATE) kfvs_1d(sn, sn, F + 3 * nx);
            else {
                double w[3] = { wall_density_1d(rho[nx - 1], u[nx - 1], T[nx - 1], cf->wall_T[1], 1), 0.0, cf->wall_T[1] };
                kfvs_1d(sn, w, F + 3 * nx);
            }
        }
    }
    /* interface_heat_flux_1d (boundary.py:160-170) */
    for (int m = 1; m < nx; ++m) Hh[m] = 0.5 * (H_out[m] + H_out[m - 1]);
    if (cf->face[0] == FACE_PERIODIC) Hh[0] = Hh[nx] = 0.5 * (H_out[0] + H_out[nx - 1]);
    else {
        Hh[0] = cf->face[0] == FACE_EXTRAPOLATE ? H_out[0] : 0.5 * H_out[0];
        Hh[nx] = cf->face[1] == FACE_EXTRAPOLATE ? H_out[nx - 1] : 0.5 * H_out[nx - 1];
    }
    {
        double r = dt / dx;
        for (int i = 0; i < nx; ++i) {
            for (int q = 0; q < 3; ++q) Q_out[3 * i + q] = Q[3 * i + q] - r * (F[3 * (i + 1) + q] - F[3 * i + q]);
            Q_out[3 * i + 2] -= r * (Hh[i + 1] - Hh[i]);
            if (qsrc) for (int q = 0; q < 3; ++q) Q_out[3 * i + q] += dt * qsrc[3 * i + q];
        }
    }
done:
    free(rho); free(M); free(Gext); free(Z); free(Zh); free(Th); free(F); free(Hh);
    return rc;
}

int mmo_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void mmo_set_num_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
