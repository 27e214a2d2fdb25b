/*
 * mm1d.h -- C ABI of the 1D1V micro-macro BGK timestep (BASELINE config 1),
 * exported by the same libmm2d.so as mm2d.h.
 *
 * Drop-in boundary for the reference's 1D time-stepper
 * `micromacro.runner.loop.step_1d` / `run_1d`
 * (reference pkg/src/micromacro/runner/loop.py:24-72).  Entry points replace
 *   mm1d_create / mm1d_destroy   the (mesh, bc, eps, model) problem objects
 *                                consumed by step_1d (loop.py:31-43)
 *   mm1d_step                    one step_1d call on device-resident state
 *                                (loop.py:31-51), with the optional MMS source
 *                                hooks (loop.py:44-50)
 *   mm1d_upload / mm1d_run /
 *   mm1d_download                run_1d's loop (loop.py:54-72), state in HBM
 *   mm1d_check                   the InvalidStateError raised by
 *                                primitives_1d (gas_state.py:44-54)
 *
 * Layouts: Q[i][3] = (rho, rho u, E) (gas_state.py:57-59), G[i][k]
 * (micro1d.py:40), H[i] (macro1d.py:16-19).  Conventions as in mm2d.h:
 * d_* device pointers, h_* host pointers, `stream` a cudaStream_t as void*
 * (NULL = default stream), return codes 0 ok / 2 config / 3 state / 5 internal.
 */
#ifndef MM1D_H
#define MM1D_H

#ifdef __cplusplus
extern "C" {
#endif

/* 1D state errors reported by mm1d_check (gas_state.py:48-53) */
#define MM1D_STATE_DENSITY 1
#define MM1D_STATE_TEMPERATURE 4

typedef struct mm1d_config {
    int nx;                   /* mesh.space[0] = Axis(x_min, x_max, nx)   (mesh.py) */
    double x_min, x_max;
    int nv;                   /* mesh.velocity[0] = Axis(v_min, v_max, nv)          */
    double v_min, v_max;
    int face[2];              /* left, right: MM2D_FACE_* (boundary.py:84-91)      */
    double wall_T[2];         /* diffuse-wall temperatures                          */
    int tau_kind;             /* MM2D_TAU_* (gas_state.py:166-199)                  */
    double tau_value;
    double eps;
    int device;
} mm1d_config;

typedef struct mm1d_ctx mm1d_ctx;

int mm1d_create(const mm1d_config* cfg, mm1d_ctx** out);
int mm1d_destroy(mm1d_ctx* ctx);
const char* mm1d_last_error(mm1d_ctx* ctx);

/* one step_1d (loop.py:31-51) on device arrays: Q (nx,3), G (nx,nv) -> Q_out,
 * G_out and H (nx) = heat_flux_1d of G_out; d_src (nx,nv) is the projected
 * micro source and d_qsrc (nx,3) the moment source at t^n (both nullable). */
int mm1d_step(mm1d_ctx* ctx, const double* d_Q, const double* d_G, double dt, double* d_Qout,
              double* d_Gout, double* d_H, const double* d_src, const double* d_qsrc,
              void* stream);

/* run_1d's loop (loop.py:54-72) on context-owned state: upload, nsteps steps
 * of a cluster-resident kernel (one launch) or a CUDA-graph replay, download. */
int mm1d_upload(mm1d_ctx* ctx, const double* h_Q, const double* h_G);
int mm1d_run(mm1d_ctx* ctx, double dt, int nsteps);
int mm1d_download(mm1d_ctx* ctx, double* h_Q, double* h_G, double* h_H);
/* 1 if mm1d_run uses the single-launch cluster-resident kernel, else 0 */
int mm1d_resident(mm1d_ctx* ctx);

/* pending InvalidStateError: returns 3 and fills kind (MM1D_STATE_*), the
 * first offending cell and its value; 0 if none.  Synchronises and clears. */
int mm1d_check(mm1d_ctx* ctx, int* kind, int* i, double* value);

#ifdef __cplusplus
}
#endif

#endif /* MM1D_H */
