/*
 * mm2d.h -- C ABI of the B200-native micro-macro ES-BGK 2D2V timestep
 * (libmm2d.so, built from paper_2509_21832_b200/csrc/).
 *
 * This is the drop-in boundary for the reference's hot path, the serial
 * time-stepper `micromacro.runner.loop.step_2d` / `run_2d`
 * (reference pkg/src/micromacro/runner/loop.py:82-129) and the worker-grid
 * runner `run_parallel_2d` (pkg/src/micromacro/runner/parallel.py:404-473).
 * The reference has no C/C++ FFI of its own: its only native boundary is the
 * Python-level kernel plugin module `micromacro._kernels`
 * (pkg/src/micromacro/_kernels/__init__.py:20-61).  The entry points below
 * replace
 *   mm2d_create / mm2d_destroy   the (mesh, bc, eps, model) problem objects
 *                                consumed by step_2d (loop.py:82-99)
 *   mm2d_step                    one step_2d call on device-resident state
 *                                (loop.py:82-111)
 *   mm2d_upload / mm2d_run /
 *   mm2d_download                run_2d's time loop (loop.py:114-129) with the
 *                                state kept in HBM between steps
 *   mm2d_heat_tensor             heat_flux_tensor_2d (macro2d.py:23-29)
 *   mm2d_check                   the InvalidStateError raised by
 *                                primitives_2d / modify_tensor
 *                                (gas_state.py:31-37, 81-108, 138-146)
 * and the mm2d_k_* functions mirror the ten `_kernels` plugin functions
 * (pkg/src/micromacro/_kernels/_fallback.py:27-173) on device pointers.
 *
 * Conventions
 *   - all arrays are C-contiguous fp64 in the reference's layouts:
 *       Q[i][j][6] = (rho, rho u1, rho u2, E11, E12, E22)   (loop.py:78)
 *       G[i][j][k][l]  (l = v2 index fastest)               (_fallback.py:8-11)
 *       H[4][i][j] = (H111, H112, H122, H222)               (macro2d.py:23-29)
 *   - pointers named d_* are device pointers, h_* host pointers;
 *   - `stream` is a cudaStream_t passed as void* (NULL = the default stream);
 *   - return codes follow the reference CLI's error categories
 *     (runner/cli.py:149-164): 0 ok, 2 configuration, 3 invalid state,
 *     5 internal (CUDA/NCCL failure).
 */
#ifndef MM2D_H
#define MM2D_H

#ifdef __cplusplus
extern "C" {
#endif

#define MM2D_OK 0
#define MM2D_ERR_CONFIG 2
#define MM2D_ERR_STATE 3
#define MM2D_ERR_INTERNAL 5

/* face kinds (boundary.py:21-36) */
#define MM2D_FACE_PERIODIC 0
#define MM2D_FACE_EXTRAPOLATE 1
#define MM2D_FACE_WALL 2
/* specularly reflecting wall: extension, the reference has diffuse walls only
   (mirror ghosts in the wall-normal velocity; needs a symmetric velocity axis) */
#define MM2D_FACE_SPECULAR 3

/* collision models (gas_state.py:166-199) */
#define MM2D_TAU_HARD_SPHERE_1D 0
#define MM2D_TAU_PRESSURE_1D 1
#define MM2D_TAU_ESBGK_2D 2
#define MM2D_TAU_BGK_2D 3
#define MM2D_TAU_CONSTANT 4

/* InvalidStateError kinds reported by mm2d_check */
#define MM2D_STATE_DENSITY 1      /* "non-positive density" */
#define MM2D_STATE_PRESSURE 2     /* "pressure tensor is not positive definite" */
#define MM2D_STATE_MODIFIED 3     /* "modified temperature tensor is not positive definite" */

typedef struct mm2d_config {
    /* global spatial grid: Axis(x_min, x_max, nx) x Axis(y_min, y_max, ny) */
    int nx, ny;
    double x_min, x_max, y_min, y_max;
    /* velocity grid: Axis(v1_min, v1_max, nv1) x Axis(v2_min, v2_max, nv2) */
    int nv1, nv2;
    double v1_min, v1_max, v2_min, v2_max;
    /* faces: left, right, bottom, top (BoundarySpec2D, boundary.py:57-77) */
    int face[4];
    double wall_T[4];          /* WallSpec.temperature */
    double wall_U[4];          /* WallSpec.velocity (tangential) */
    /* CollisionModel(kind, nu, value), knudsen number eps */
    int tau_kind;
    double tau_value;
    double nu;
    double eps;
    /* block domain decomposition: px x py ranks, this rank at (rx, ry)
     * (make_plans, parallel.py:69-93); 1 x 1 for a single GPU */
    int px, py, rx, ry;
    int device;                /* CUDA device ordinal */
} mm2d_config;

typedef struct mm2d_ctx mm2d_ctx;

/* lifecycle */
int mm2d_create(const mm2d_config *cfg, mm2d_ctx **out);
int mm2d_destroy(mm2d_ctx *ctx);
const char *mm2d_last_error(mm2d_ctx *ctx);
int mm2d_version(void);
/* version of the fused micro kernel (k_micro32); ties committed ncu
 * captures (profiles/micro_traffic.json) to the code that produced them */
int mm2d_kernel_version(void);

/* local block geometry of this rank: (bx, by) cells starting at (i0, j0) */
int mm2d_block(mm2d_ctx *ctx, int *bx, int *by, int *i0, int *j0);

/* one step_2d on caller-owned device buffers (local block layouts).  The
 * inputs are not modified.  d_H may be NULL.  d_src_coeffs (nsrc, bx, by)
 * and d_src_shapes (nsrc, nv1, nv2) add the manufactured-solution low-rank
 * source (micro2d.py:120-123); d_qsrc (bx, by, 6) the macro source
 * (macro2d.py:238-239); all three may be NULL / nsrc = 0. */
int mm2d_step(mm2d_ctx *ctx, const double *d_Q, const double *d_G, double dt,
              double *d_Qout, double *d_Gout, double *d_H,
              int nsrc, const double *d_src_coeffs, const double *d_src_shapes,
              const double *d_qsrc, void *stream);

/* the same step split at the heat-tensor exchange point of the block
 * decomposition (parallel.py:384-394): phase 0 = macro ring + per-cell prep
 * + fused micro kernel (writes G^{n+1} and the owned heat tensor), phase 1 =
 * heat ring + KFVS/TR-BDF2 macro update.  Between them a multi-rank run
 * exchanges the heat-tensor halo (mm2d_halo_*, field 2).  Phase 0 may itself
 * be split around the G halo exchange so the exchange overlaps interior-cell
 * compute: phase 2 = prep + the micro CTAs that read no received G halo
 * (needs only the Q halo), phase 3 = the remaining micro CTAs (after the G
 * halo has landed); 2 then 3 is bitwise identical to 0.  Finer still,
 * phase 4 = prep only and phase 5 = the interior micro CTAs only, so 3 can
 * run on a second stream concurrently with 5 (4, 5 | 3 is bitwise 0). */
int mm2d_step_phase(mm2d_ctx *ctx, int phase, const double *d_Q, const double *d_G, double dt,
                    double *d_Qout, double *d_Gout, double *d_H,
                    int nsrc, const double *d_src_coeffs, const double *d_src_shapes,
                    const double *d_qsrc, void *stream);

/* context-owned state (ping-pong buffers in HBM) */
int mm2d_alloc_state(mm2d_ctx *ctx);
int mm2d_upload(mm2d_ctx *ctx, const double *h_Q, const double *h_G);
int mm2d_upload_device(mm2d_ctx *ctx, const double *d_Q, const double *d_G);
/* attach caller-owned ping-pong state (device pointers, not freed by the
 * context): A = (d_Qa, d_Ga) holds the current state, B receives the next;
 * d_H (4, bx, by) receives the heat tensor of the last step (may be NULL) */
int mm2d_attach_state(mm2d_ctx *ctx, double *d_Qa, double *d_Ga, double *d_Qb,
                      double *d_Gb, double *d_H);
/* which of the two state slots (0 = A, 1 = B) holds the current state */
int mm2d_current_index(mm2d_ctx *ctx);
/* stream the context orders itself after / before (e.g. the framework's
 * current stream); mm2d_run waits on it and makes it wait on the result */
int mm2d_set_stream(mm2d_ctx *ctx, void *stream);
/* nsteps steps of size dt; captured once into a CUDA graph per dt */
int mm2d_run(mm2d_ctx *ctx, double dt, int nsteps);
int mm2d_download(mm2d_ctx *ctx, double *h_Q, double *h_G, double *h_H);
/* device pointers of the current context-owned state */
int mm2d_state_ptrs(mm2d_ctx *ctx, double **d_Q, double **d_G, double **d_H);

/* heat tensor (4, bx, by) of G with the velocity of Q (frame_2d moments,
 * runner/cases.py:167-176; macro2d.py:23-29) */
int mm2d_heat_tensor(mm2d_ctx *ctx, const double *d_G, const double *d_Q,
                     double *d_H, void *stream);

/* steady-state tracking of the run driver (runner/cases.py:217-222,
 * max |Q^{n+1} - Q^n| over the last 10% of steps): *d_max = max(*d_max,
 * max_k |a_k - b_k|) over n doubles, on the device (no host sync).  *d_max
 * must start non-negative (e.g. 0). */
int mm2d_max_abs_diff(mm2d_ctx *ctx, const double *d_a, const double *d_b, long long n,
                      double *d_max, void *stream);

/* synchronise and report the sticky device error word.  Returns MM2D_OK or
 * MM2D_ERR_STATE with *kind = MM2D_STATE_*, (*i, *j) the global cell and
 * *value the offending value (density or determinant). */
int mm2d_check(mm2d_ctx *ctx, int *kind, int *i, int *j, double *value);
int mm2d_sync(mm2d_ctx *ctx);

/* multi-GPU halo exchange hooks (extract_ring semantics, parallel.py:109-150).
 * The transfer itself is driven by the host (NCCL send/recv through
 * torch.distributed, or device copies between contexts of one process);
 * these expose the context's staging buffers.  `which`: 0 = micro field G
 * (V doubles per cell, received in place into the kernel's halo buffers),
 * 1 = macro state Q (6), 2 = heat tensor H (4).  Slots: 0 left, 1 right,
 * 2 bottom, 3 top, 4 bottom-left, 5 bottom-right, 6 top-left, 7 top-right;
 * send slot s goes to the neighbour in direction s and lands in its receive
 * slot opposite(s).  count = doubles in the slot (0 when the face is a
 * physical boundary).  pack: G and Q from d_src (block layout), H from the
 * heat ring; unpack scatters received Q / H ghosts into their rings. */
int mm2d_halo_info(mm2d_ctx *ctx, int which, int slot, double **d_send,
                   double **d_recv, long long *count);
int mm2d_halo_pack(mm2d_ctx *ctx, int which, const double *d_src, void *stream);
int mm2d_halo_unpack(mm2d_ctx *ctx, int which, void *stream);

/* Peer form of the G halo (no reference counterpart: the reference's workers
 * copy their strips through shared memory, parallel.py:153-182).  d_nbG[s] is
 * the base of the CURRENT G^n array (bx, by, nv1, nv2) of the neighbour block
 * in slot s (NULL for an inactive slot), dereferenceable from this context's
 * device: a block on the same GPU, a peer GPU with access enabled
 * (mm2d_enable_peer_access, NVLink / NVSwitch), or a CUDA-IPC mapping of
 * another process's array.  The micro kernels of the following steps then read
 * every ghost cell in place from those arrays -- the perimeter CTAs' bulk
 * copies fetch the halo rows straight from the neighbour's HBM -- so field 0
 * needs no pack, transfer or receive buffer.  Every block of a decomposition
 * has this block's shape (make_plans).  The caller orders the steps: a
 * neighbour's G^n must be complete, and this block's G^{n+1} buffer must no
 * longer be read by a neighbour, when the step is enqueued (the Q ring
 * exchange that precedes every step gives both).  Pass NULL to return to the
 * packed form.  Call again whenever the neighbours' arrays change (ping-pong). */
int mm2d_halo_peer(mm2d_ctx *ctx, const double *const *d_nbG);
int mm2d_enable_peer_access(int device, int peer_device);

/* One process per GPU: state arrays a neighbour process can map.
 * mm2d_ipc_alloc: a cudaMalloc allocation on the current device plus its
 * 64-byte CUDA-IPC handle; mm2d_ipc_open maps another process's allocation
 * (peer access enabled lazily) and returns the pointer to pass to
 * mm2d_halo_peer; close / free release them. */
int mm2d_ipc_alloc(long long bytes, void **d_ptr, unsigned char *handle64);
int mm2d_ipc_open(const unsigned char *handle64, void **d_ptr);
int mm2d_ipc_close(void *d_ptr);
int mm2d_ipc_free(void *d_ptr);

/* ---- the ten kernel-contract functions (_kernels plugin API) ----
 * device pointers, reference layouts; `ext` arrays carry one ghost layer on
 * the differenced axis. */
int mm2d_k_maxwellian_field_2d(int nx, int ny, int nv1, int nv2, const double *rho,
                               const double *u1, const double *u2, const double *T,
                               const double *v1, const double *v2, double *M, void *stream);
int mm2d_k_project_field_2d(int nx, int ny, int nv1, int nv2, const double *F,
                            const double *M, const double *rho, const double *u1,
                            const double *u2, const double *T, const double *v1,
                            const double *v2, double dv, double *out, void *stream);
int mm2d_k_transport_stage_2d(int nx, int ny, int nv1, int nv2, const double *G_ext,
                              const double *M, const double *rho, const double *u1,
                              const double *u2, const double *T, const double *v1,
                              const double *v2, double d, double dt, int axis,
                              double *out, void *stream);
int mm2d_k_ghat_2d(int nx, int ny, int nv1, int nv2, const double *M, const double *rho,
                   const double *u1, const double *u2, const double *T,
                   const double *s11, const double *s12, const double *gT1,
                   const double *gT2, const double *tau, const double *v1,
                   const double *v2, double *out, void *stream);
int mm2d_k_add_gaussian_term_2d(int nx, int ny, int nv1, int nv2, double *Ghat,
                                const double *M, const double *rho, const double *u1,
                                const double *u2, const double *m11, const double *m12,
                                const double *m22, double eps, const double *v1,
                                const double *v2, void *stream);
int mm2d_k_add_lowrank_4d(int nx, int ny, int nv1, int nv2, double *out, int nterms,
                          const double *coeffs, const double *shapes, void *stream);
int mm2d_k_relax_2d(int nx, int ny, int nv1, int nv2, const double *G, const double *Ghat,
                    const double *tau, double dt, double eps, double *out, void *stream);
int mm2d_k_heat_tensor_2d(int nx, int ny, int nv1, int nv2, const double *G,
                          const double *u1, const double *u2, const double *v1,
                          const double *v2, double dv, double eps, double *H, void *stream);
int mm2d_k_upwind_z_1d(int nx, int nv, const double *G_ext, const double *v, double dx,
                       double *Z, void *stream);
int mm2d_k_project_field_1d(int nx, int nv, const double *F, const double *M,
                            const double *rho, const double *u, const double *T,
                            const double *v, double dv, double *out, void *stream);

/* per-kernel device time on the attached/owned state: captures nrep steps
 * as ONE CUDA graph (the path mm2d_run replays) with external event-record
 * nodes around every kernel, launches it once and returns the mean
 * milliseconds per launch in ms[0..6] = (none), prep, micro, (none),
 * macro_x, macro_y, (none) */
int mm2d_time_kernels(mm2d_ctx *ctx, double dt, int nrep, double *ms);

/* device launches counted since the last reset (bench.py's gpu_launches) */
long long mm2d_launch_count(void);
void mm2d_reset_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* MM2D_H */
