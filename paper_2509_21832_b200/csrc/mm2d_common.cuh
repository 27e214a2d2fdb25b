// Shared device-side definitions for the B200 micro-macro ES-BGK 2D2V step.
//
// Data layout in HBM (local block of bx x by cells owned by this rank):
//   G      [bx][by][V]        fp64, V = nv1*nv2, v2 index fastest (the
//                             reference's layout, _fallback.py:8-11)
//   P      [(bx+2)][(by+2)]   CellPar per ring cell (owned block plus a
//                             one-cell ring, corners included), rebuilt each
//                             step from Q^n by the prep kernel
//   Qr     [(bx+2)][(by+2)][6] Q^n with ghosts (wrap / copy / received halo)
//   Hr     [(bx+2)][(by+2)][4] heat tensor with ghosts (AoS)
//   Qx     [(bx+2)][(by+2)][6] x-swept macro state (Strang stage 2)
// Ring coordinates run from -1 to bx (x) and -1 to by (y); ring index
// ri(i, j) = (i + 1) * (by + 2) + (j + 1).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <utility>

namespace mm2d {

constexpr double kPi = 3.141592653589793238462643383279502884;

// face kinds as in mm2d.h
enum FaceKind { FACE_PERIODIC = 0, FACE_EXTRAPOLATE = 1, FACE_WALL = 2 };

// How a ghost layer of the LOCAL block is filled.
//   WRAP: periodic face owned entirely by this rank (index wraps locally)
//   COPY: zero-gradient copy of the edge layer (extrapolate; walls for macro)
//   ZERO: zero ghost (micro / heat fields at diffuse walls)
//   HALO: received from a neighbour rank (interior or periodic-across-ranks)
// GM_MIRROR: specular wall (extension) -- the ghost is the edge cell mirrored
// in the wall-normal velocity (G: node index reversed along the normal axis;
// Q: normal momentum and E12 negated; H: components odd in v_n negated)
enum GhostMode { GM_WRAP = 0, GM_COPY = 1, GM_ZERO = 2, GM_HALO = 3, GM_MIRROR = 4 };

// stage/check codes of the sticky error word; the key orders failures the
// way the reference raises them within one step (loop.py:98, micro2d.py:92,
// macro2d.py:63 and 202 via primitives_2d, in call order).
enum ErrStage {
    ES_PRIM_RHO = 0,   // primitives_2d(Q^n): density          (S0)
    ES_PRIM_SPD = 1,   // primitives_2d(Q^n): pressure tensor
    ES_MOD_SPD = 2,    // modify_tensor SPD check               (S1)
    ES_XS_RHO = 3,     // _sweep x: primitives_2d(Q*)          (S3)
    ES_XS_SPD = 4,
    ES_YS_RHO = 5,     // _sweep y: primitives_2d(Q**)         (S4)
    ES_YS_SPD = 6,
    ES_RL_RHO = 7,     // final relax: primitives_2d(Q***)     (S5)
    ES_RL_SPD = 8,
};

// error key: step (24 bits) | stage (4 bits) | global cell (36 bits)
__host__ __device__ inline unsigned long long err_key(unsigned step, unsigned stage,
                                                      unsigned long long cell) {
    return ((unsigned long long)step << 40) | ((unsigned long long)stage << 36) | cell;
}
constexpr unsigned long long kNoError = ~0ull;

// Debug build (make EXTRA=-DMM2D_DEBUG_CHECKS=1 OUT=../libmm2d_dbg.so):
// device-side bounds checks on the shared-memory, tensor-memory and global
// indices the kernels compute; a failed check prints the site and traps.
// This stands in for compute-sanitizer, which is closed on the GPU pool
// (profiles/r02_compute_sanitizer_closed.log).  Release builds compile the
// checks away.
#ifndef MM2D_DEBUG_CHECKS
#define MM2D_DEBUG_CHECKS 0
#endif
#if MM2D_DEBUG_CHECKS
#include <cstdio>
#define MM2D_CHECK(cond)                                                                   \
    do {                                                                                   \
        if (!(cond)) {                                                                     \
            printf("MM2D_CHECK failed: %s at %s:%d (block %d,%d thread %d)\n", #cond,      \
                   __FILE__, __LINE__, (int)blockIdx.x, (int)blockIdx.y, (int)threadIdx.x); \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#else
#define MM2D_CHECK(cond) \
    do {                 \
    } while (0)
#endif

// Error words of a context (8 x u64): [0] E, the merged key of every
// completed kernel; [1..4] isotropy maxima; [5] R_prep, [6] R_mx, [7] R_my,
// the keys raised by k_prep, k_macro_x and k_macro_y.  A kernel raises into
// its OWN word and skips its work only on keys raised by earlier launches:
// its gate is min(E, R of the kernel before it), both of which are stable
// while it runs, so every CTA of one launch takes the same decision and a
// launch never stops itself part-way (the minimum over all its offending
// cells is what the reference's first-failure order asks for).  The kernel
// also folds that predecessor word into E (atomicMin is idempotent), so E
// accumulates every failure one launch later; mm2d_check reads min(E, R_*).
enum ErrWord { EW_E = 0, EW_ISO = 1, EW_PREP = 5, EW_MX = 6, EW_MY = 7, EW_N = 8 };

__device__ __forceinline__ bool err_gate(unsigned long long* w, int prev) {
    const unsigned long long rp = *(volatile const unsigned long long*)(w + prev);
    if (rp != kNoError && threadIdx.x == 0 && threadIdx.y == 0 && blockIdx.x == 0 &&
        blockIdx.y == 0)
        atomicMin(w + EW_E, rp);
    const unsigned long long e = *(volatile const unsigned long long*)(w + EW_E);
    return (e < rp ? e : rp) != kNoError;
}
// read-only form for kernels that raise nothing (the micro kernels)
__device__ __forceinline__ bool err_pending(const unsigned long long* w, int prev) {
    const unsigned long long rp = w[prev], e = w[EW_E];
    return (e < rp ? e : rp) != kNoError;
}

// Per-ring-cell parameters produced by the prep kernel (all from Q^n).
struct __align__(16) CellPar {
    double u1, u2, isT, tau;            // 0-3   velocity (gas_state.py:93-108), 1/sqrt(T), tau
    double pref, inv2T, invT, scale;    // 4-7   rho/(2 pi T), 1/(2T), 1/T, dv/rho
    double s11, s12, gT1, gT2;          // 8-11  sigma and grad T (micro2d.py:37-60)
    double wg, wh, invtau, gpref;       // 12-15 relax weights, 1/tau, Gaussian rho/(2 pi sqrt det)
    double gq11, gq22, gq12, pad;       // 16-19 Gaussian exponents c22/det, c11/det, c12/det
    double rw[4];                       // 20-23 diffuse-wall ghost densities (left,right,bottom,top)
};
// (round 1's 32-double layout also carried rho, T, the temperature tensor and
// the modified tensor, which no kernel reads: a quarter of the prep's writes)
constexpr int kParD = 24;               // doubles per CellPar
static_assert(sizeof(CellPar) == kParD * sizeof(double), "CellPar layout");

struct Geometry {
    int bx, by;          // local block
    int i0, j0;          // global offset of the block
    int nx, ny;          // global grid
    int nv1, nv2, V;
    int xlo, xhi, ylo, yhi;     // GhostMode of the four local faces (micro G)
    int qxlo, qxhi, qylo, qyhi; // GhostMode for macro fields (walls copy)
    int hxlo, hxhi, hylo, hyhi; // GhostMode for the heat tensor (walls zero)
    int wall[4];                // physical diffuse wall on face f
    int phys[4];                // face f is a physical boundary of the global domain
    double wallT[4], wallU[4];
    double dx, dy;
};

__host__ __device__ inline int ring_index(const Geometry& g, int i, int j) {
    return (i + 1) * (g.by + 2) + (j + 1);
}

// Programmatic dependent launch: the step's kernels are launched with
// programmatic stream serialization (launch_pdl), so a kernel's CTAs can be
// resident before its predecessor has finished.  Every such kernel waits for
// the predecessor's completion and memory flush first, then lets its own
// successor be scheduled.  (Both are no-ops under a normal launch.)
template <bool kTrigger = true>
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (kTrigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

#ifndef MM2D_PDL
#define MM2D_PDL 0   // measured slower at C2: off
#endif
// launch with programmatic stream serialization (MM2D_PDL=0: a plain launch)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = block;
    lc.dynamicSmemBytes = smem;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = MM2D_PDL;
    lc.attrs = at;
    lc.numAttrs = 1;
    return cudaLaunchKernelEx(&lc, kernel, std::forward<Args>(args)...);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    return v;
}

// Block-wide all-reduce of N doubles per thread (N a power of two <= 32).
// Warp stage: transposed butterfly (each level halves the number of values a
// lane carries), so a warp spends log2(N) + (5 - log2 N) ... = N - 1 + ...
// shuffles instead of 5N.  Cross-warp stage: one shared-memory slot per
// (warp, value), then every warp re-sums the NW partials redundantly and
// broadcasts with shuffles, so only ONE __syncthreads is needed.
// scratch must hold 2 * NW * N doubles; `parity` alternates the halves so a
// fast warp entering the next reduction cannot overwrite partials a slow warp
// is still reading.
template <int N>
__device__ __forceinline__ void block_allreduce(double (&v)[N], double* scratch,
                                                int& parity, int nwarps) {
    static_assert(N >= 1 && N <= 32 && (N & (N - 1)) == 0, "N must be a power of two <= 32");
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    // transposed butterfly
    int cnt = N;
    int idx = 0;
    int mask = 16;
#pragma unroll
    for (int lvl = 0; (1 << lvl) < N; ++lvl) {
        const int half = cnt >> 1;
        const bool up = (lane & mask) != 0;
#pragma unroll
        for (int q = 0; q < N / 2; ++q) {
            if (q < half) {
                double send = up ? v[q] : v[q + half];
                double keep = up ? v[q + half] : v[q];
                v[q] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
            }
        }
        if (up) idx += half;
        cnt = half;
        mask >>= 1;
    }
    double s = v[0];
    for (; mask > 0; mask >>= 1) s += __shfl_xor_sync(0xffffffffu, s, mask);
    // lanes sharing idx hold the same warp total; the lowest one writes
    double* buf = scratch + parity * (32 * N);
    const int low_bits = 32 / N;   // lanes per value
    if ((lane & (low_bits - 1)) == 0) buf[warp * N + idx] = s;
    parity ^= 1;
    __syncthreads();
    // redundant cross-warp sum: lane L handles value (L % N) over a strided
    // subset of warps, then lanes combine and broadcast.
    const int vid = lane % N;
    const int grp = lane / N;           // 0 .. 32/N - 1
    const int ngrp = 32 / N;
    double t = 0.0;
    for (int w = grp; w < nwarps; w += ngrp) t += buf[w * N + vid];
#pragma unroll
    for (int m = N; m < 32; m <<= 1) t += __shfl_xor_sync(0xffffffffu, t, m);
#pragma unroll
    for (int q = 0; q < N; ++q) v[q] = __shfl_sync(0xffffffffu, t, q);
}

// pack/unpack of positive doubles for atomicMax
__device__ __forceinline__ void atomic_max_pos(unsigned long long* addr, double v) {
    atomicMax(addr, (unsigned long long)__double_as_longlong(v));
}

}  // namespace mm2d
