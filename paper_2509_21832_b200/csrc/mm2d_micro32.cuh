// Fused micro kernel specialised for the 32 x 32 velocity grid of every
// benchmark configuration (V = 1024 nodes per cell).  Same mathematics as the
// generic k_micro (mm2d_micro.cuh), reorganised for the fp64 issue budget:
//
//  * 128 threads per CTA, 8 nodes per thread: thread t owns the 16-byte node
//    pairs (k, l..l+1) with k = t/16 + 8p (p = 0..3) and l = 2 (t % 16), so a
//    warp touches 512 contiguous bytes per pair and all upwind stencils are
//    thread-local.
//  * Everything that depends on (cell, k) or (cell, l) only -- the separable
//    Maxwellian factors, the projection basis w1, w2, b4, the closed-form
//    target's polynomial pieces, the separable ES-BGK Gaussian factors -- is
//    built once per cell into shared-memory tables (K-table [32][8],
//    L-table [8][32], Gaussian tables), so a node costs a handful of FMAs.
//  * One block reduction per row: the y-projection sums of row j, the
//    x-projection sums of row j+2 and the heat moments of row j-1 share it.
//  * G* lives in a 3-row thread-private shared-memory ring; the x-stage of
//    row j+2 first stores G - dt Z there and adds the projection one
//    iteration later, once its sums are reduced.
//  * Diffuse-wall strip targets (boundary.py:343-378) do not depend on G and
//    are precomputed by k_wall_ghat into a small buffer.
//
// Row loop (iteration j, rows j0-3 .. j1; steps are predicated on validity):
//   1. recon G*(j+1)   2. y-sums(j)   3. x-stage(j+2), prefetch G^n(j+3)
//   4. reduction [y(j) | x(j+2) | H(j-1)], write H(j-1)
//   5. G**(j), target, relax, store G^{n+1}(j), heat partials H(j)
#pragma once
#include <type_traits>
#include "mm2d_common.cuh"
#include "mm2d_micro.cuh"

// version of this kernel: bump on every change that alters its code, so
// committed ncu captures (profiles/micro_traffic.json) stay tied to it
#ifndef M32_KERNEL_VERSION
#define M32_KERNEL_VERSION 33
#endif

// Projection sums in raw velocity moments (v28).  1: each thread weights its
// upwind differences with its own, cell-independent node coordinates (the
// sign-folded upwind coefficients it already holds in registers), the row
// reduction adds raw moments (1, v1, v2, |v|^2), and the reducer warp of each
// stage converts the four totals once per cell into the coefficients of the
// projection polynomial c0 + c1 v1 + c2 v2 + c3 |v|^2 (raw_to_coef), which
// every thread evaluates at its nodes again from registers.  The K-table
// loses (w1, h1), (cx w1, cx h1) and the L-table w2, h2: 24 of a thread's 52
// shared-memory table loads per row.  0: the v27 form (normalised basis
// w1, w2, b4 from the tables).
#ifndef M32_RAW
#define M32_RAW 1
#endif

// Projection polynomial tabulated per cell (v31, needs M32_RAW).  Its value at a
// node is (X(k) + Z(l)) M: the k part times the Maxwellian's k factor, AL[k] =
// X(k) pE1[k], and the l part times its l factor, BE[l] = Z(l) E2[l], depend on
// k or l alone.  1: the reducer warp that converts a stage's totals also writes
// the 32 + 32 values into the row's K- and L-table (one lane per entry), and
// every thread loads its four AL and two BE instead of evaluating them (19 fp64
// operations per thread and stage, 16 of every 17 of them redundant across the
// threads that share a k or an l).  0: v30, every thread evaluates its own.
#ifndef M32_TABPROJ
#define M32_TABPROJ M32_RAW
#endif

#ifndef MICRO32_MINB
#define MICRO32_MINB 4   // resident CTAs per SM the register budget is sized for: 4 x 128
                         // threads at 128 registers and 55 KB of shared memory (the K-table
                         // drops its W1^2 / W1^3 pair to fit).  Measured against 3 CTAs at
                         // 166 registers: C4 5.47 vs 5.84 ms, C2 (band 64) 0.390 vs 0.405 ms.
#endif

#ifndef M32_NS
#define M32_NS 8   // reducer threads per reduced value (the shuffle levels are log2 of it)
#endif
#ifndef M32_PDL_TRIGGER
#define M32_PDL_TRIGGER 0
#endif
#ifndef M32_SHORT_FILL
#define M32_SHORT_FILL 1
#endif

namespace mm2d {
namespace m32 {

constexpr int NV = 32;
constexpr int V = NV * NV;
constexpr int NT = 128;              // threads of the default 8-node (NP = 4) variant
constexpr int NP = 4;                // node pairs per thread (default variant)
constexpr int TSLOTS = 4;            // table slots (rows j..j+3; the slot rebuilt
                                     // at iteration j last held row j-1)
#ifndef M32_W1POW_TABLE
#if MICRO32_MINB >= 4
#define M32_W1POW_TABLE 0            // 4 CTAs/SM: recompute W1^2, W1^3 to fit 56 KB
#else
#define M32_W1POW_TABLE 1
#endif
#endif
#if M32_RAW
#if M32_TABPROJ
constexpr int KW = M32_W1POW_TABLE ? 12 : 10;   // K-table entries per k
constexpr int LR = 8;                           // L-table rows
#else
constexpr int KW = M32_W1POW_TABLE ? 8 : 6;     // K-table entries per k
constexpr int LR = 6;                           // L-table rows
#endif
#else
constexpr int KW = M32_W1POW_TABLE ? 12 : 10;   // K-table entries per k
constexpr int LR = 8;
#endif
constexpr int KT = 0;                // K-table [32][KW]
constexpr int LT = KT + KW * NV;     // L-table [LR][32]
constexpr int GK = LT + LR * NV;     // Gaussian k-table [32][2] (GA, GD)
constexpr int GL = GK + 2 * NV;      // Gaussian l-table [32] (GB)
constexpr int XT = GL + NV;          // Gaussian cross-term tables per even l = 2 lp:
                                     //   (X0, R)[16], (R^2, R^4)[16] as double2, R^8[16]
constexpr int TAB = XT + 5 * 16;     // 816 doubles per cell
// K-table pairs (16-byte loads): (w1, h1) (pE1, W1) (cx w1, cx h1) (W1^2, W1^3)
// (pE1 f0, pE1 f1) (pE1 f2, pE1) -- the target polynomial's W2-power
// coefficients pre-multiplied by the Maxwellian's k factor, the x-sum weights
// by the upwind coefficient
#if M32_RAW
#if M32_W1POW_TABLE
enum { K_PE1, K_W1, K_W12, K_W13, K_F0, K_F1, K_F2, K_PE1B, K_PEX, K_ALX, K_ALY, K_PADK };
#else
// (K_PEX, K_ALX): pE1 again next to the x-stage's AL, one 16-byte load in the recon
enum { K_PE1, K_W1, K_F0, K_F1, K_F2, K_PE1B, K_PEX, K_ALX, K_ALY, K_PADK };
#endif
// L-table rows: E2, W2, E2 W2, E2 W2^2, f3 E2 W2^3
enum { L_E2, L_W2, L_EW1, L_EW2, L_EW3, L_PAD, L_BEX, L_BEY };
#else
#if M32_W1POW_TABLE
enum { K_W1N, K_H1, K_PE1, K_W1, K_XW, K_XH, K_W12, K_W13, K_F0, K_F1, K_F2, K_PE1B };
#else
enum { K_W1N, K_H1, K_PE1, K_W1, K_XW, K_XH, K_F0, K_F1, K_F2, K_PE1B };
#endif
// L-table rows: E2, w2, h2, W2, E2 W2, E2 W2^2, f3 E2 W2^3
enum { L_E2, L_W2N, L_H2, L_W2, L_EW1, L_EW2, L_EW3, L_PAD };
#endif
// cross-term tables per even l = 2 lp: X0 = exp(q12 W1_0 W2), R = exp(q12 dv1 W2),
// R^2, R^4, R^8 (the thread's base node k = kb gets X0 R^kb, its next pairs
// R^8); lp-major with a 16-byte stride, so a quarter-warp's eight lp read
// 128 contiguous bytes (the previous 32-byte stride took 8 wavefronts)
enum { X_X0R = 0, X_R24 = 2 * 16, X_R8 = 4 * 16 };

inline size_t smem_bytes() {
    return sizeof(double) * (3 * V + TSLOTS * TAB + 4 * 16 + 16 + 2 * NV);
}

__device__ __forceinline__ double2 lds2(const double* p) {
    return *reinterpret_cast<const double2*>(p);
}
__device__ __forceinline__ void sts2(double* p, double a, double b) {
    *reinterpret_cast<double2*>(p) = make_double2(a, b);
}

// one-row block all-reduce of 16 doubles with 4 warps: transposed butterfly
// in the warp, per-warp partials through shared memory, 16 threads finish.
__device__ __forceinline__ void reduce16(double (&v)[16], double* sred) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int idx = 0;
#pragma unroll
    for (int lvl = 0; lvl < 4; ++lvl) {
        const int mask = 16 >> lvl;
        const int half = 8 >> lvl;
        const bool up = (lane & mask) != 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (q < half) {
                const double send = up ? v[q] : v[q + half];
                const double keep = up ? v[q + half] : v[q];
                v[q] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
            }
        }
        if (up) idx += half;
    }
    const double s = v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
    if ((lane & 1) == 0) sred[warp * 16 + idx] = s;
    __syncthreads();
    if (threadIdx.x < 16)
        sred[64 + threadIdx.x] = (sred[threadIdx.x] + sred[16 + threadIdx.x]) +
                                 (sred[32 + threadIdx.x] + sred[48 + threadIdx.x]);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; q += 2) {
        const double2 x = lds2(sred + 64 + q);
        v[q] = x.x;
        v[q + 1] = x.y;
    }
}

// Row header stored in each table slot (doubles): per-cell scalars the node
// loops need, so they come from shared memory instead of global loads.
enum { H_SCALE, H_WG, H_MTW, H_MEW, H_GQ12, H_WH, H_U1, H_U2, H_IST, H_INVT, H_N = 12 };
constexpr int HD = TAB;              // header offset inside a slot
constexpr int SLOT = TAB + H_N;      // doubles per table slot

// exp(x) to ~1 ulp for x <= 709, table-driven: x = (64 m + i) ln2/64 + r
// with |r| <= ln2/128 (Cody-Waite, two-part ln2/64), e^x = 2^m 2^(i/64) e^r,
// e^r - 1 = r P(r) by a degree-5 Horner polynomial (truncation < 3e-20, each
// step one DFMA with a constant-bank operand), 2^(i/64) from a 64-entry
// shared-memory table (correctly rounded, generated at 60 digits).  Results
// below ~1e-307 flush to zero (they only ever enter here as negligible
// factors).  ~20 instructions against ~40 for the previous polynomial-only
// version and ~50 for libdevice exp.
__constant__ double kExp2Tab[64] = {
    1.0, 1.0108892860517005, 1.0218971486541166, 1.0330248790212284,
    1.0442737824274138, 1.0556451783605572, 1.0671404006768237, 1.0787607977571199,
    1.0905077326652577, 1.102382583307841, 1.1143867425958924, 1.1265216186082418,
    1.1387886347566916, 1.1511892299529827, 1.1637248587775775, 1.1763969916502812,
    1.189207115002721, 1.202156731452703, 1.215247359980469, 1.22848053610687,
    1.241857812073484, 1.255380757024691, 1.2690509571917332, 1.2828700160787783,
    1.2968395546510096, 1.3109612115247644, 1.3252366431597413, 1.339667524053303,
    1.3542555469368927, 1.3690024229745905, 1.383909881963832, 1.3989796725383112,
    1.4142135623730951, 1.42961333839197, 1.4451808069770467, 1.460917794180647,
    1.4768261459394993, 1.4929077282912648, 1.5091644275934228, 1.5255981507445384,
    1.5422108254079407, 1.559004400237837, 1.5759808451078865, 1.593142151342267,
    1.6104903319492543, 1.6280274218573478, 1.645755478153965, 1.6636765803267364,
    1.681792830507429, 1.7001063537185235, 1.718619298122478, 1.7373338352737062,
    1.7562521603732995, 1.7753764925265212, 1.7947090750031072, 1.8142521755003989,
    1.8340080864093424, 1.8539791250833855, 1.8741676341103, 1.8945759815869656,
    1.9152065613971474, 1.9360617934922943, 1.9571441241754002, 1.978456026387951};

// the reduction and polynomial constants sit in the constant bank so every
// step is one DFMA with a c[][] operand (64-bit literals would each cost a
// pair of uniform-register moves)
__constant__ double kExpC[7] = {92.33248261689366,          // 64 / ln 2
                                -0.010830424696249145,      // ln2/64, high part
                                -3.623510646634843e-19,     // ln2/64, low part
                                1.3888888888888889e-03, 8.3333333333333333e-03,
                                4.1666666666666667e-02, 1.6666666666666667e-01};

__device__ __forceinline__ double fexp(double x, const double* etab) {
    const double SH = 6755399441055744.0;   // 1.5 * 2^52: round-to-int shifter
    double t = fma(x, kExpC[0], SH);
    const int n = __double2loint(t);
    t -= SH;
    double r = fma(t, kExpC[1], x);
    r = fma(t, kExpC[2], r);
    double p = fma(r, kExpC[3], kExpC[4]);
    p = fma(p, r, kExpC[5]);
    p = fma(p, r, kExpC[6]);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    const double q = p * r;                               // e^r - 1
    const double T = etab[n & 63];
    const double e = fma(T, q, T);
    const int hi = __double2hiint(e) + ((n >> 6) << 20);
    return n < -1020 * 64 ? 0.0 : __hiloint2double(hi, __double2loint(e));
}

// Block all-reduce of the row's 12 sums (y | x | heat) through shared
// memory: every thread stores its partials value-major (conflict-free 8-byte
// stores), 96 threads each add 16 partials of one value (rotated start so a
// warp's 16-byte loads hit 8 distinct bank groups), 8-lane shuffles finish,
// and all threads read the 12 totals back.  Two barriers, ~50 instructions.
// tree sum of a per-pair contribution array
template <int N>
__device__ __forceinline__ double tsum(const double (&c)[N]) {
    if constexpr (N == 8) return ((c[0] + c[1]) + (c[2] + c[3])) + ((c[4] + c[5]) + (c[6] + c[7]));
    else if constexpr (N == 4) return (c[0] + c[1]) + (c[2] + c[3]);
    else if constexpr (N == 2) return c[0] + c[1];
    else return c[0];
}

#ifndef M32_TMEM_RED
#define M32_TMEM_RED 0   // 1: warp-level row reduction through tensor memory (measured); 0: shared memory
#endif
#if M32_TMEM_RED
// per-warp totals [4][12] + the 8 projection totals, sharing the space with
// the specular exchange (NP doubles per thread, two rounds)
template <int NT_> constexpr int red_size() { return NT_ * 4; }   // doubles
#else
template <int NT_> constexpr int red_size() { return 12 * NT_ + 16; }   // doubles
#endif

// The totals' hand-over (v28): 1: the reducer threads arrive on an mbarrier once
// their totals are written and every thread waits for that phase, so warp 0
// (which builds the heaviest table in the same window) is not part of the
// hand-over and the row has ONE CTA-wide barrier; 0: a second __syncthreads.
#ifndef M32_EPOW
#define M32_EPOW 1
#endif
// v32: three trades of l-indexed table loads (4 shared-memory wavefronts each, the
// L1TEX pipe being the loaded unit again after v31) against a few fp64 operations
// or registers.  M32_EPOW: E2 W2^n (n = 1..3) formed in the thread from E2 and W2
// (8 fp64) instead of three loads; M32_RPOW: R^2, R^4, R^8 of the Gaussian cross
// term squared up in the thread (3 fp64) instead of two loads; M32_KEEPL: row j's
// E2 and W2 kept in registers from the target evaluation to step 5 instead of two
// reloads after the hand-over.  C5 micro 20.89 -> 20.70 -> 20.52 -> 20.36 ms.
#ifndef M32_KEEPL
#define M32_KEEPL 1
#endif
#ifndef M32_RPOW
#define M32_RPOW 1
#endif
#ifndef M32_MBAR_B
#define M32_MBAR_B 0
#endif
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity);
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar);

// phase A: store partials, barrier.  phase B + totals: reduce12_end.  Work
// that touches neither the partials nor the totals may sit in between.
template <int NT_>
__device__ __forceinline__ void reduce12_begin(const double (&v)[12], double* sred) {
#pragma unroll
    for (int q = 0; q < 12; ++q) sred[q * NT_ + threadIdx.x] = v[q];
    __syncthreads();
}

// (phase B: the heat totals go straight to the heat ring from their
// reducer threads; every thread reads back the 8 projection totals)
#if M32_RAW
// Totals of a stage's raw moments N0 = sum Y, N1 = sum (s xi) Y, N2 = sum (s' eta) Y,
// N3 = sum (xi^2 + ryx eta^2) Y, in the threads' node coordinates xi = dt |v1| / dx,
// eta = dt |v2| / dy  ->  the coefficients of the projection polynomial
// q = C0 + C1 (s xi) + C2 (s' eta) + C3 (xi^2 + ryx eta^2), scaled by sc, with
// Pi[Y] = q M (_core.pyx:171-199: the normalised sums A1..A4 of the basis
// 1, w1, w2, b4 = (w1^2 + w2^2)/2 - 1, expanded about the cell's u and T).
__device__ __forceinline__ void raw_to_coef(const MicroArgs& a, const double* hdr, double sc,
                                            double N0, double N1, double N2, double N3,
                                            double (&C)[4]) {
    const double2 u = lds2(hdr + H_U1);
    const double2 tt = lds2(hdr + H_IST);          // 1/sqrt(T), 1/T
    const double isT = tt.x, invT = tt.y;
    const double m1 = N1 * a.ikx, m2 = N2 * a.iky, m3 = N3 * a.ikx2;
    const double uu = fma(u.x, u.x, u.y * u.y);
    const double A2 = isT * fma(-u.x, N0, m1);
    const double A3 = isT * fma(-u.y, N0, m2);
    const double A4 = fma(0.5 * invT, fma(uu, N0, fma(-2.0, fma(u.x, m1, u.y * m2), m3)), -N0);
    const double a1 = N0 * sc, a2 = A2 * sc, a3 = A3 * sc, a4 = A4 * sc;
    const double c3 = 0.5 * a4 * invT;
    const double c1 = fma(a2, isT, -2.0 * c3 * u.x);
    const double c2 = fma(a3, isT, -2.0 * c3 * u.y);
    const double c0 = fma(c3, uu, fma(-isT, fma(a2, u.x, a3 * u.y), a1 - a4));
    C[0] = c0;
    C[1] = c1 * a.ikx;
    C[2] = c2 * a.iky;
    C[3] = c3 * a.ikx2;
}
#endif

template <int NT_>
__device__ __forceinline__ void reduce12_end(double (&v)[12], double* sred, double* hdst,
                                             double hfac, const MicroArgs& a, const double* Ty,
                                             const double* Tx, unsigned long long* mbarB,
                                             unsigned parityB, double* Tyw, double* Txw,
                                             const double* v1s, const double* v2s) {
    constexpr int NS = NT_ >= 128 ? M32_NS : 4;  // segments per value (threads per value)
    constexpr int SEG = NT_ / NS;           // partials per (value, segment)
    constexpr int L2N = SEG / 2;            // double2 loads per segment
    // the reducers are the LAST 12 * NS threads (warps 1-3 at NT = 128), so
    // warp 0, which builds the heaviest table (K) in the same window, is not
    // on the reduction's critical path
    constexpr int R0 = NT_ - 12 * NS > 0 ? ((NT_ - 12 * NS) & ~31) : 0;
    const int tid = threadIdx.x - R0;
    // whole warps take part so the shuffles below are well defined
    if (tid >= 0 && (tid & ~31) < 12 * NS) {
        const bool act = tid < 12 * NS;
        const int vid = act ? tid / NS : 0, seg = tid % NS;
        const double* src = sred + vid * NT_ + SEG * seg;
        double u[L2N];
#pragma unroll
        for (int q = 0; q < L2N; ++q) {
            const double2 x = lds2(src + 2 * ((q + seg) & (L2N - 1)));
            u[q] = x.x + x.y;
        }
#pragma unroll
        for (int w = 1; w < L2N; w <<= 1)
#pragma unroll
            for (int q = 0; q < L2N; q += 2 * w) u[q] += u[q + w];
        double acc = u[0];
        if (NS >= 8) acc += __shfl_xor_sync(0xffffffffu, acc, 4);
        if (NS >= 4) acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        if (NS >= 2) acc += __shfl_xor_sync(0xffffffffu, acc, 1);
#if M32_RAW
        // warp 0 of the reducers holds the y totals (vid 0-3, eight lanes each),
        // warp 1 the x totals: gather the four, convert once per cell
        static_assert(NT_ < 128 || M32_NS == 8, "raw-moment conversion assumes 8 lanes per value");
        if (tid < 64) {
            const double N0 = __shfl_sync(0xffffffffu, acc, 0), N1 = __shfl_sync(0xffffffffu, acc, 8);
            const double N2 = __shfl_sync(0xffffffffu, acc, 16), N3 = __shfl_sync(0xffffffffu, acc, 24);
            const bool isy = tid < 32;
            const double* hdr = (isy ? Ty : Tx) + HD;
            const double2 sw = lds2(hdr + H_SCALE);        // scale, wg
            double Cf[4];
            raw_to_coef(a, hdr, isy ? sw.x * sw.y : sw.x, N0, N1, N2, N3, Cf);
#if M32_TABPROJ
            // lane m tabulates the polynomial's k part at k = m and its l part at
            // l = m, in the node coordinates the threads use (same expressions as
            // their cx / cy, so the same doubles)
            {
                const int m = tid & 31;
                double* Tw = isy ? Tyw : Txw;
                const double v1m = v1s[m], v2m = v2s[m];
                const double xi = (m < NV / 2 ? -a.dt : a.dt) * v1m * a.idx;
                const double eta = (v2m < 0.0 ? -a.dt : a.dt) * v2m * a.idy;
                const double X = fma(xi, fma(Cf[3], xi, m < NV / 2 ? -Cf[1] : Cf[1]), Cf[0]);
                const double Z = eta * fma(Cf[3] * a.ryx, eta, v2m < 0.0 ? -Cf[2] : Cf[2]);
                double* K = Tw + KT + KW * m;
                K[isy ? K_ALY : K_ALX] = X * K[K_PE1];
                Tw[LT + (isy ? L_BEY : L_BEX) * NV + m] = Z * Tw[LT + L_E2 * NV + m];
            }
#else
            if ((tid & 31) == 0) {
                sts2(sred + 12 * NT_ + (isy ? 0 : 4), Cf[0], Cf[1]);
                sts2(sred + 12 * NT_ + (isy ? 2 : 6), Cf[2], Cf[3]);
            }
#endif
        } else if (act && seg == 0 && hdst) hdst[vid - 8] = hfac * acc;
#else
        if (act && seg == 0) {
            if (vid < 8) sred[12 * NT_ + vid] = acc;
            else if (hdst) hdst[vid - 8] = hfac * acc;
        }
#endif
#if M32_MBAR_B
        mbar_arrive(mbarB);
#endif
    }
#if M32_MBAR_B
    // (also orders the next row's partial stores after the reducers' loads)
    mbar_wait(mbarB, parityB);
#else
    __syncthreads();
#endif
#if !(M32_RAW && M32_TABPROJ)
#pragma unroll
    for (int q = 0; q < 8; q += 2) {
        const double2 x = lds2(sred + 12 * NT_ + q);
        v[q] = x.x;
        v[q + 1] = x.y;
    }
#endif
}

// build the per-cell tables from the shared copy P of the cell's CellPar.
// Warp 0 (which does not reduce) the K-table's Maxwellian factor and the
// target coefficients it scales, warp 1 the L-table, warp 2 the Gaussian
// cross-term table, warp 3 the exp-free K-table pairs and the Gaussian GA, GB
// and GD: the six exps per cell spread 1 / 1 / 1 / 3 (warps 1 and 2 also carry
// the longest reductions, with the totals' conversion).  The closed-form target polynomial is
// stored pre-scaled by mtw = -wh/tau with the Gaussian's -M wh/eps folded
// into U.  As a polynomial in W2 the bracket is f0(k) + f1(k) W2 + f2(k) W2^2
// + f3 W2^3 (f3 cell-constant), so with the Maxwellian's factors folded in the
// node evaluates acc = (pE1 f0) E2 + (pE1 f1) (E2 W2) + (pE1 f2) (E2 W2^2)
// + pE1 (f3 E2 W2^3) (+ the Gaussian) with one product and three FMAs.
template <int KS>
__device__ __forceinline__ void build_tables(const MicroArgs& a, double* T, const CellPar& P,
                                             const double* v1s, const double* v2s, bool gauss,
                                             const double* etab) {
    const double mtw = -P.invtau * P.wh;
    const int t = threadIdx.x;
    const int m = t & 31;
    if (t < 32) {
        const double W1 = v1s[m] - P.u1;
        const double W1s = W1 * W1;
        const double q1 = W1s * P.inv2T - 2.0;
        const double p1 = W1 * P.gT1 * P.invT;
        const double U = W1s * P.s11 * P.inv2T + q1 * p1;
        const double pe = P.pref * fexp(-W1s * P.inv2T, etab);
        double* K = T + KT + KW * m;
        sts2(K + K_PE1, pe, W1);
        // bracket U + V + c W2 + q1 p2 + p1 q2 (_core.pyx:220-224) by powers of W2:
        // f0 = U, f1 = (W1 s12 + q1 gT2) / T, f2 = (p1 - s11) / (2T), f3 = gT2 / (2T^2)
        sts2(K + K_F0, pe * fma(mtw, U, gauss ? -a.inveps * P.wh : 0.0),
             pe * (mtw * ((W1 * P.s12 + q1 * P.gT2) * P.invT)));
#if M32_EPOW
        // (pE1 f2, pE1 f3): the thread forms E2 W2^3 itself, so f3 rides with pE1 here
        sts2(K + K_F2, pe * (mtw * ((p1 - P.s11) * P.inv2T)),
             pe * (mtw * (P.gT2 * P.invT * P.inv2T)));
#else
        sts2(K + K_F2, pe * (mtw * ((p1 - P.s11) * P.inv2T)), pe);   // pE1 again: one 16-byte load in the target
#endif
#if M32_TABPROJ
        K[K_PEX] = pe;
#endif
        if (m == 0) {
            sts2(T + HD + H_SCALE, P.scale, P.wg);
            sts2(T + HD + H_MTW, mtw, a.inveps * P.wh);
            sts2(T + HD + H_GQ12, P.gq12, P.wh);
            sts2(T + HD + H_U1, P.u1, P.u2);
            sts2(T + HD + H_IST, P.isT, P.invT);
        }
    } else if (t < 64) {
        const double W2 = v2s[m] - P.u2;
        const double W2s = W2 * W2;
        const double E2 = fexp(-W2s * P.inv2T, etab);
        double* L = T + LT + m;
        L[L_E2 * NV] = E2;
#if !M32_RAW
        const double w2 = W2 * P.isT;
        L[L_W2N * NV] = w2;
        L[L_H2 * NV] = 0.5 * w2 * w2;
#endif
        L[L_W2 * NV] = W2;
#if !M32_EPOW
        L[L_EW1 * NV] = E2 * W2;
        L[L_EW2 * NV] = E2 * W2s;
        L[L_EW3 * NV] = (mtw * (P.gT2 * P.invT * P.inv2T)) * (E2 * (W2s * W2));
#endif
    } else if (gauss && t < 96) {
        // (GA, the Gaussian's k factor, is built by warp 3: this warp also reduces and
        // converts the x sums, and the row time follows the busiest warp -- moving
        // that one exp evened the roles out: C5 -1.0 %, C2 -1.6 %)
        // lanes 0-15: X0 at l = 2m; lanes 16-31: R and its powers at l = 2(m-16)
        const int lp = m & 15;
        const double W2e = v2s[2 * lp] - P.u2;
        const double x = fexp(P.gq12 * (m < 16 ? v1s[0] - P.u1 : v1s[1] - v1s[0]) * W2e, etab);
        double* X = T + XT;
        if (m < 16) {
            X[X_X0R + 2 * lp] = x;
        } else {
            X[X_X0R + 2 * lp + 1] = x;
#if !M32_RPOW
            const double r2 = x * x, r4 = r2 * r2;
            sts2(X + X_R24 + 2 * lp, r2, r4);
            X[X_R8 + lp] = r4 * r4;
#endif
        }
    } else {
        // the exp-free K-table pairs (off warp 0's critical path)
        const double W1 = v1s[m] - P.u1;
        const double W1s = W1 * W1;
        double* K = T + KT + KW * m;
#if !M32_RAW
        const double w1 = W1 * P.isT;
        const double h1 = 0.5 * w1 * w1 - 1.0;
        // the x-stage upwind coefficient (sign folded: v1 < 0 exactly for k < 16)
        const double cxm = (m < NV / 2 ? -a.dt : a.dt) * v1s[m] * a.idx;
        sts2(K + K_W1N, w1, h1);
        sts2(K + K_XW, cxm * w1, cxm * h1);
#endif
#if M32_W1POW_TABLE
        sts2(K + K_W12, W1s, W1s * W1);
#endif
        if (gauss) {
            const double W2 = v2s[m] - P.u2;
            T[GK + 2 * m] = P.gpref * a.inveps * P.wh * fexp(P.gq11 * W1s, etab);    // GA'
            T[GL + m] = fexp(P.gq22 * (W2 * W2), etab);                              // GB
            T[GK + 2 * m + 1] = fexp(P.gq12 * W1 * (v2s[1] - v2s[0]), etab);         // GD
        }
    }
}

// 16-byte asynchronous global -> shared copy (LDGSTS) and its fences
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gsrc));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }
__device__ __forceinline__ void cp_async_wait_prev() { asm volatile("cp.async.wait_group 1;\n" ::); }

// Bulk (TMA) copies global -> shared completing on an mbarrier.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "MBW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra MBW_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Thread-private rows in tensor memory.  A warp may only touch its own
// 32-lane quadrant, and every thread its own lane, which is exactly the
// access pattern of the thread-private G* ring: 8 doubles of a thread's row
// are 16 consecutive 32-bit columns of its lane, moved by ONE
// tcgen05.ld/st .32x32b.x16 (against four 16-byte LDS/STS in shared memory).
#ifndef TM_SPLIT
#define TM_SPLIT 1   // tcgen05 ld/st instructions per 8-double row (1: .x16, 2: .x8, 4: .x4)
#endif
template <int N>   // N doubles = 2N columns
__device__ __forceinline__ void tm_st_n(unsigned addr, const double* v);
template <int N>
__device__ __forceinline__ void tm_ld_n(unsigned addr, double* v);
template <>
__device__ __forceinline__ void tm_st_n<8>(unsigned addr, const double* v) {
    // the doubles are split inside PTX so ptxas can place them straight into
    // the 16 consecutive registers STTM reads
    asm volatile(
        "{\n .reg .b32 a<16>;\n"
        " mov.b64 {a0, a1}, %1;\n mov.b64 {a2, a3}, %2;\n mov.b64 {a4, a5}, %3;\n"
        " mov.b64 {a6, a7}, %4;\n mov.b64 {a8, a9}, %5;\n mov.b64 {a10, a11}, %6;\n"
        " mov.b64 {a12, a13}, %7;\n mov.b64 {a14, a15}, %8;\n"
        " tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {a0, a1, a2, a3, a4, a5, a6, a7, a8, a9, "
        "a10, a11, a12, a13, a14, a15};\n}\n" ::"r"(addr),
        "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3]), "d"(v[4]), "d"(v[5]), "d"(v[6]), "d"(v[7])
        : "memory");
}
template <>
__device__ __forceinline__ void tm_st_n<4>(unsigned addr, const double* v) {
    asm volatile(
        "{\n .reg .b32 a<8>;\n"
        " mov.b64 {a0, a1}, %1;\n mov.b64 {a2, a3}, %2;\n mov.b64 {a4, a5}, %3;\n"
        " mov.b64 {a6, a7}, %4;\n"
        " tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {a0, a1, a2, a3, a4, a5, a6, a7};\n}\n" ::"r"(addr),
        "d"(v[0]), "d"(v[1]), "d"(v[2]), "d"(v[3])
        : "memory");
}
template <>
__device__ __forceinline__ void tm_st_n<2>(unsigned addr, const double* v) {
    asm volatile(
        "{\n .reg .b32 a<4>;\n"
        " mov.b64 {a0, a1}, %1;\n mov.b64 {a2, a3}, %2;\n"
        " tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {a0, a1, a2, a3};\n}\n" ::"r"(addr),
        "d"(v[0]), "d"(v[1])
        : "memory");
}
template <>
__device__ __forceinline__ void tm_ld_n<8>(unsigned addr, double* v) {
    asm volatile(
        "{\n .reg .b32 a<16>;\n"
        " tcgen05.ld.sync.aligned.32x32b.x16.b32 {a0, a1, a2, a3, a4, a5, a6, a7, a8, a9, a10, "
        "a11, a12, a13, a14, a15}, [%8];\n"
        " tcgen05.wait::ld.sync.aligned;\n"
        " mov.b64 %0, {a0, a1};\n mov.b64 %1, {a2, a3};\n mov.b64 %2, {a4, a5};\n"
        " mov.b64 %3, {a6, a7};\n mov.b64 %4, {a8, a9};\n mov.b64 %5, {a10, a11};\n"
        " mov.b64 %6, {a12, a13};\n mov.b64 %7, {a14, a15};\n}\n"
        : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]), "=d"(v[4]), "=d"(v[5]), "=d"(v[6]),
          "=d"(v[7])
        : "r"(addr)
        : "memory");
}
template <>
__device__ __forceinline__ void tm_ld_n<4>(unsigned addr, double* v) {
    asm volatile(
        "{\n .reg .b32 a<8>;\n"
        " tcgen05.ld.sync.aligned.32x32b.x8.b32 {a0, a1, a2, a3, a4, a5, a6, a7}, [%4];\n"
        " mov.b64 %0, {a0, a1};\n mov.b64 %1, {a2, a3};\n mov.b64 %2, {a4, a5};\n"
        " mov.b64 %3, {a6, a7};\n}\n"
        : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
        : "r"(addr)
        : "memory");
}
template <>
__device__ __forceinline__ void tm_ld_n<2>(unsigned addr, double* v) {
    asm volatile(
        "{\n .reg .b32 a<4>;\n"
        " tcgen05.ld.sync.aligned.32x32b.x4.b32 {a0, a1, a2, a3}, [%2];\n"
        " mov.b64 %0, {a0, a1};\n mov.b64 %1, {a2, a3};\n}\n"
        : "=d"(v[0]), "=d"(v[1])
        : "r"(addr)
        : "memory");
}
__device__ __forceinline__ void tm_st8(unsigned addr, const double (&v)[8]) {
    constexpr int N = 8 / TM_SPLIT;
#pragma unroll
    for (int q = 0; q < TM_SPLIT; ++q) tm_st_n<N>(addr + 2 * N * q, v + N * q);
}
__device__ __forceinline__ void tm_ld8(unsigned addr, double (&v)[8]) {
    constexpr int N = 8 / TM_SPLIT;
    if constexpr (TM_SPLIT == 1) {
        tm_ld_n<8>(addr, v);
    } else {
#pragma unroll
        for (int q = 0; q < TM_SPLIT; ++q) tm_ld_n<N>(addr + 2 * N * q, v + N * q);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    }
}
__device__ __forceinline__ void tm_wait_st() {
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}
#if M32_TMEM_RED
// Row reduction of the 12 per-thread sums (y | x | heat) without shared-
// memory partials: the L1TEX pipe that shared memory and shuffles share is
// the kernel's binding resource, the tensor-memory port is not.
// Phase A, per warp: each thread stores its 12 sums in its own TMEM lane
// (columns tred .. tred + 23); 16x256b loads hand thread t the sums
// (t % 4) + 4 r (r = 0..2) of lanes t / 4, t / 4 + 8, t / 4 + 16 and
// t / 4 + 24, which it adds; three shuffle levels over the lane bits 2-4
// finish the warp total, and lanes 0-3 store the warp's 12 totals; barrier.
// Phase B (reduce12_end_tm): 12 threads add the four warps' totals, the
// heat totals go straight to the heat ring; barrier; every thread reads the
// 8 projection totals.  Fixed order throughout, so results stay bitwise
// reproducible.
__device__ __forceinline__ void tm_ld16x256_x2(unsigned addr, double (&v)[4]) {
    asm volatile(
        "{\n .reg .b32 a<8>;\n"
        " tcgen05.ld.sync.aligned.16x256b.x2.b32 {a0, a1, a2, a3, a4, a5, a6, a7}, [%4];\n"
        " mov.b64 %0, {a0, a1};\n mov.b64 %1, {a2, a3};\n mov.b64 %2, {a4, a5};\n"
        " mov.b64 %3, {a6, a7};\n}\n"
        : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
        : "r"(addr)
        : "memory");
}
__device__ __forceinline__ void tm_ld16x256_x1(unsigned addr, double (&v)[2]) {
    asm volatile(
        "{\n .reg .b32 a<4>;\n"
        " tcgen05.ld.sync.aligned.16x256b.x1.b32 {a0, a1, a2, a3}, [%2];\n"
        " mov.b64 %0, {a0, a1};\n mov.b64 %1, {a2, a3};\n}\n"
        : "=d"(v[0]), "=d"(v[1])
        : "r"(addr)
        : "memory");
}

__device__ __forceinline__ void reduce12_begin_tm(const double (&v)[12], double* sred,
                                                  unsigned tred) {
    tm_st_n<8>(tred, v);
    tm_st_n<4>(tred + 16, v + 8);
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    // lanes 0-15 then 16-31 of the warp's quadrant; per load: [lane t/4, r]
    // [lane t/4 + 8, r] for r = 0, 1 (x2) and r = 2 (x1)
    double a01[4], a2[2], b01[4], b2[2];
    tm_ld16x256_x2(tred, a01);
    tm_ld16x256_x1(tred + 16, a2);
    tm_ld16x256_x2(tred + (16u << 16), b01);
    tm_ld16x256_x1(tred + (16u << 16) + 16, b2);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    double q[3] = {(a01[0] + a01[1]) + (b01[0] + b01[1]), (a01[2] + a01[3]) + (b01[2] + b01[3]),
                   (a2[0] + a2[1]) + (b2[0] + b2[1])};
#pragma unroll
    for (int m = 4; m <= 16; m <<= 1)
#pragma unroll
        for (int r = 0; r < 3; ++r) q[r] += __shfl_xor_sync(0xffffffffu, q[r], m);
    const int lane = threadIdx.x & 31;
    if (lane < 4) {
        double* w = sred + 12 * (threadIdx.x >> 5) + lane;
        w[0] = q[0];
        w[4] = q[1];
        w[8] = q[2];
    }
    __syncthreads();
}

__device__ __forceinline__ void reduce12_end_tm(double (&v)[12], double* sred, double* hdst,
                                                double hfac) {
    // warp 1 (a reducer-free warp's table work is on warp 0) adds the warp totals
    const int r = (int)threadIdx.x - 32;
    if (r >= 0 && r < 12) {
        const double t = (sred[r] + sred[12 + r]) + (sred[24 + r] + sred[36 + r]);
        if (r < 8) sred[48 + r] = t;
        else if (hdst) hdst[r - 8] = hfac * t;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 8; q += 2) {
        const double2 x = lds2(sred + 48 + q);
        v[q] = x.x;
        v[q + 1] = x.y;
    }
}
#endif

#if M32_TMEM_RED && M32_RAW
#error "M32_TMEM_RED is only implemented for the v27 (M32_RAW=0) reduction"
#endif
#if M32_TMEM_RED
constexpr int TM_COLS = 128;         // G* ring (3 rows x 16 columns) + the row reduction (24)
constexpr int TM_RED = 64;           // first reduction column
#else
constexpr int TM_COLS = 64;          // 3 rows x 16 columns, rounded to a power of two
#endif

template <int NP_>
inline size_t smem_bytes_v3() {
    constexpr int NT_ = 512 / NP_;
    return sizeof(double) * (2 * V + TSLOTS * SLOT + red_size<NT_>() + 4 * 32 + 2 * NV + 2 + 64 + 2);
}

// The host selects this kernel only when the velocity axes make the upwind
// direction a compile-time property of the node pair: v1 < 0 exactly for
// k < 16 (pairs p = 0, 1 difference towards the right neighbour), and both
// nodes of every (l, l+1) pair share the sign of v2.
//
// Per-thread sums use running accumulators: for a transport stage the four
// projection sums of the thread's nodes are
//   s0 = Y0 + Y1,  s1 = sum_p w1_p (y0 + y1)_p,  s2 = w2_l Y0 + w2_r Y1,
//   s3 = sum_p h1_p (y0 + y1)_p + h2_l Y0 + h2_r Y1
// with Y0 / Y1 the sums over the thread's left / right nodes of the pair
// (b4 = h1 + h2, w2 and h2 are per-thread constants), and the heat moments
// are accumulated as A_a = sum W1^a o per node column, then weighted by the
// thread's W2 powers.  The row loop runs a predicate-free body for the rows
// away from the piece ends.
// MIR: the instantiation for problems with a specular face (the others are
// compiled without any mirror code, so the benchmark path's code is untouched)
template <int NP_, bool MIR>
__global__ void __launch_bounds__(512 / NP_, MICRO32_MINB) k_micro32(MicroArgs a) {
    // (no early trigger: the macro sweep's CTAs would sit on the SMs while
    // the bands finish; M32_PDL_TRIGGER=1 measures that variant)
    pdl_enter<M32_PDL_TRIGGER != 0>();
    static_assert(NP_ == 4, "the TMEM ring is laid out for 4 node pairs per thread");
    constexpr int NT_ = 512 / NP_;       // threads per CTA
    constexpr int KS = 32 / NP_;         // k step between a thread's node pairs
    extern __shared__ __align__(16) double smem[];
    const Geometry& g = a.g;
    if (a.part != 0) {
        const int b0 = a.nband ? a.band_j0[blockIdx.y] : blockIdx.y * a.ly;
        const int b1 = a.nband ? a.band_j0[blockIdx.y + 1] : min(g.by, b0 + a.ly);
        if (skip_part(a, blockIdx.x, blockIdx.x + 1, b0, b1)) return;
    }
    const int tid = threadIdx.x;
    // thread -> nodes: l pair lp, k base kb.  Warps 0/2 take the v2 < 0 half
    // (l < 16), warps 1/3 the v2 >= 0 half, so the y-upwind direction is
    // warp-uniform (the TMEM ring's loads are warp-collective).
    const int lp = (tid & 7) + 8 * ((tid >> 5) & 1);
    const int kb = ((tid >> 3) & 3) + 4 * (tid >> 6);
    const int lb = lp << 1;

    double* stg = smem;                             // [2][V] x-stage row: own | halo
    double* tabs = stg + 2 * V;                     // [TSLOTS][SLOT]
    double* sred = tabs + TSLOTS * SLOT;            // [12][NT] partials + [12] totals
    double* pring = sred + red_size<NT_>();         // [4][32] staged CellPar rows
    double* v1s = pring + 4 * 32;
    double* v2s = v1s + NV;
    double* etab = v2s + NV + 2;                    // [64] 2^(i/64)
    const size_t V_ = V;
#if MM2D_DEBUG_CHECKS
    {
        unsigned dyn;
        asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
        MM2D_CHECK((size_t)(etab + 64 + 2 - smem) * sizeof(double) <= dyn);
    }
#endif

    const int i = blockIdx.x;
    const int j0s = a.nband ? a.band_j0[blockIdx.y] : blockIdx.y * a.ly;
    const int j1s = a.nband ? a.band_j0[blockIdx.y + 1] : min(g.by, j0s + a.ly);
    const int k_lo = row_kind(g, j0s - 1);          // ghost-row kinds at the piece ends
    const int k_hi = row_kind(g, j1s);

    // G^n column pointers for interior rows (stride V per row); ghost rows
    // go through gn_cell.  Zero ghosts point at a zero row with stride 0.
    const double* own_b = a.G + (size_t)i * g.by * V_;
    const double* lft_b;
    const double* rgt_b;
    size_t lft_s = V_, rgt_s = V_;
    if (i > 0) lft_b = own_b - (size_t)g.by * V_;
    else if (g.xlo == GM_HALO) lft_b = a.hxlo;
    else if (g.xlo == GM_WRAP) lft_b = a.G + (size_t)(g.bx - 1) * g.by * V_;
    else if (g.xlo == GM_COPY || (MIR && g.xlo == GM_MIRROR)) lft_b = own_b;
    else { lft_b = a.zero; lft_s = 0; }
    if (i < g.bx - 1) rgt_b = own_b + (size_t)g.by * V_;
    else if (g.xhi == GM_HALO) rgt_b = a.hxhi;
    else if (g.xhi == GM_WRAP) rgt_b = a.G;
    else if (g.xhi == GM_COPY || (MIR && g.xhi == GM_MIRROR)) rgt_b = own_b;
    else { rgt_b = a.zero; rgt_s = 0; }
    // specular x faces: the upwind neighbour of node (k, l) is the edge cell's
    // own node (31 - k, l), already staged with the own row, so the x-stage
    // reads it from there (the halo copy of these CTAs is unused).  These
    // columns run every row through the general body, so the steady body
    // carries no mirror test.
    // (recomputed at the use sites from blockIdx / the constant bank so they
    // hold no registers across the steady loop)
    auto mir_l = [&]() { return MIR && blockIdx.x == 0 && g.xlo == GM_MIRROR; };
    auto mir_r = [&]() { return MIR && (int)blockIdx.x == g.bx - 1 && g.xhi == GM_MIRROR; };

    const bool on_x = (g.wall[0] && i == 0) || (g.wall[1] && i == g.bx - 1);
    const double* wx = on_x ? a.wall_ghat + ((size_t)(i == 0 ? 0 : 1) * g.by) * V_ : nullptr;
    double* out_b = a.Gout + (size_t)i * g.by * V_;
    const double* wb = g.wall[2] ? a.wall_ghat + ((size_t)2 * g.by + i) * V_ : nullptr;
    const double* wt = g.wall[3] ? a.wall_ghat + ((size_t)2 * g.by + g.bx + i) * V_ : nullptr;

    // rows computed by the x-stage: the contiguous range [rlo, rhi] (ghost
    // rows that are copies or zeros excluded)
    const int rlo = k_lo == 0 ? j0s - 1 : j0s;
    const int rhi = k_hi == 0 ? j1s : j1s - 1;
    auto computes = [&](int r) { return (unsigned)(r - rlo) <= (unsigned)(rhi - rlo); };

    // CellPar of ring row r -> pring[r & 3], 12 threads x 16 bytes; one
    // commit group per call so wait_group 1 leaves exactly the newest in flight
    auto stage_par = [&](int r, bool on) {
        if (on && tid < kParD / 2)
            cp_async16(pring + 32 * (r & 3) + 2 * tid,
                       reinterpret_cast<const double*>(a.P + ring_index(g, i, r)) + 2 * tid);
        cp_async_commit();
    };
    // Every CTA start waits on memory several times (its first CellPar rows,
    // its first bulk G row, the error word, the velocity axes): issue the
    // asynchronous copies first so those latencies overlap.
    stage_par(j0s - 1, computes(j0s - 1));
    stage_par(j0s, computes(j0s));
    // x-stage rows arrive by TMA: own row -> stg[0:V], the right neighbour's
    // k < 16 half -> stg[V:V+V/2], the left neighbour's k >= 16 half ->
    // stg[V+V/2:2V], so every node's upwind neighbour sits at the node's own
    // offset.  Thread 0 arms the mbarrier and issues three bulk copies once
    // the previous row's readers have passed a CTA barrier.
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(v2s + NV);
    if (tid == 0) {
        mbar_init(mbar, 1);
        mbar_init(mbar + 1, (12 * M32_NS + 31) & ~31);   // the totals: one arrival per thread of the reducer warps
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    unsigned nload = 0;            // bulk loads issued (mbarrier phase = parity)
    const int jfirst = j0s - (M32_SHORT_FILL ? 3 : 4);   // first row-loop iteration (phase 0 of the totals' mbarrier)
    auto prefetch = [&](int r, auto steady) {
        if (tid != 0) { ++nload; return; }
        const double *own, *hl, *hr;
        if (decltype(steady)::value || (r >= 0 && r < g.by)) {
            own = own_b + (size_t)r * V_;
            hl = lft_b + (size_t)r * lft_s;
            hr = rgt_b + (size_t)r * rgt_s;
        } else {
            own = gn_cell(a, i, r);
            hl = gn_cell(a, i - 1, r);
            hr = gn_cell(a, i + 1, r);
            if (!own) own = a.zero;
            if (!hl) hl = a.zero;
            if (!hr) hr = a.zero;
        }
#if MM2D_DEBUG_CHECKS
        {
            auto inbuf = [&](const double* p, int half) {
                const double* e = p + (half ? V / 2 : V);
                const size_t nG = (size_t)g.bx * g.by * V_;
                if (a.hpeer) {
                    for (int s8 = 0; s8 < 8; ++s8)
                        if (a.hnb[s8] && p >= a.hnb[s8] && e <= a.hnb[s8] + nG) return true;
                    return (p >= a.G && e <= a.G + nG) || (p >= a.zero && e <= a.zero + V_);
                }
                return (p >= a.G && e <= a.G + nG) || (p >= a.zero && e <= a.zero + V_) ||
                       (a.hxlo && p >= a.hxlo && e <= a.hxlo + (size_t)g.by * V_) ||
                       (a.hxhi && p >= a.hxhi && e <= a.hxhi + (size_t)g.by * V_) ||
                       (a.hylo && p >= a.hylo && e <= a.hylo + (size_t)(g.bx + 2) * V_) ||
                       (a.hyhi && p >= a.hyhi && e <= a.hyhi + (size_t)(g.bx + 2) * V_);
            };
            MM2D_CHECK(inbuf(own, 0));
            MM2D_CHECK(inbuf(hr, 1));
            MM2D_CHECK(inbuf(hl + V / 2, 1));
        }
#endif
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_expect_tx(mbar, 2 * V * sizeof(double));
        bulk_g2s(stg, own, V * sizeof(double), mbar);
        bulk_g2s(stg + V, hr, V / 2 * sizeof(double), mbar);
        bulk_g2s(stg + V + V / 2, hl + V / 2, V / 2 * sizeof(double), mbar);
        ++nload;
    };

    if (computes(j0s - 1)) prefetch(j0s - 1, std::false_type());
    if (err_pending(a.err, EW_PREP)) {
        // an earlier stage failed: leave the step's inputs untouched, after
        // the copies in flight have landed
        cp_async_wait_all();
        if (tid == 0 && nload) mbar_wait(mbar, 0);
        __syncthreads();
        return;
    }
    if (tid < NV) v1s[tid] = a.v1[tid];
    else if (tid < 2 * NV) v2s[tid - NV] = a.v2[tid - NV];
    if (tid < 64) etab[tid] = kExp2Tab[tid];

    const bool gauss = a.gauss && !(a.eps < 1e-10 &&
        __longlong_as_double(a.iso[0]) <= 1e-13 * __longlong_as_double(a.iso[3]) &&
        __longlong_as_double(a.iso[1]) <= 1e-13 * __longlong_as_double(a.iso[3]) &&
        __longlong_as_double(a.iso[2]) <= 1e-13 * __longlong_as_double(a.iso[3]));
    __syncthreads();

    // per-thread constants: node offsets and sign-folded upwind coefficients
    // Y = c (G_self - G_upwind): the reference's v (G_i - G_{i-1}) / d for
    // v >= 0 and v (G_{i+1} - G_i) / d for v < 0 (_core.pyx:152-168)
    // node-pair offsets: off(p) = off0 + 256 p into a cell's block,
    // koff(p) = koff0 + 64 p into the K-table (immediate offsets in SASS)
    const int off0 = 32 * kb + lb;
    const int koff0 = KT + KW * kb;
#define off_(p) (off0 + 32 * KS * (p))
#define koff_(p) (koff0 + KW * KS * (p))
    double cx[NP_];
#pragma unroll
    for (int p = 0; p < NP_; ++p)
        cx[p] = (p < NP_ / 2 ? -a.dt : a.dt) * v1s[kb + KS * p] * a.idx;
    const bool negy = v2s[lb] < 0.0;
    const double sy = negy ? -a.dt : a.dt;
    const double cy0 = sy * v2s[lb] * a.idy, cy1 = sy * v2s[lb + 1] * a.idy;
    // x with the sign of the thread's v2 (one XOR on the high word)
    const int sbit = negy ? (int)0x80000000 : 0;
    auto sflip = [&](double x) { return __hiloint2double(__double2hiint(x) ^ sbit, __double2loint(x)); };
    const int xsel = lp * 2;       // this thread's cross-term table entries
    cp_async_wait_all();
    __syncthreads();

    // the G* ring: 64 TMEM columns, allocated by warp 0
    unsigned* tslot = reinterpret_cast<unsigned*>(etab + 64);
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         smem_u32(tslot)),
                     "n"(TM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const unsigned tbase = *reinterpret_cast<volatile unsigned*>(tslot);
    const unsigned tq = tbase + ((unsigned)(tid & ~31) << 16);   // this warp's lane quadrant
    // rotating slot pointers: ring rows (j-1, j, j+1); table rows
    // (j, j+1, j+2, j+3, j-1)
    unsigned R0 = tq, R1 = tq + 16, R2 = tq + 32;   // TMEM ring rows (j-1, j, j+1)
    MM2D_CHECK(off_(NP_ - 1) + 2 <= V && koff_(NP_ - 1) + KW <= LT && xsel + 2 <= 2 * 16);
    double* T0 = tabs;
    double* T1 = tabs + SLOT;
    double* T2 = tabs + 2 * SLOT;
    double* T3 = tabs + 3 * SLOT;

#if !M32_TABPROJ
    double ax[4] = {0, 0, 0, 0};   // x-projection sums of the pending row
#endif
    double hs[4] = {0, 0, 0, 0};   // heat partial sums of the previous row
    double ty[2 * NP_];            // G* - dt Z_y of the current row
#pragma unroll
    for (int q = 0; q < 2 * NP_; ++q) ty[q] = 0.0;

    // Transport stages work on the upwind differences d = G_self - G_upwind:
    // the stage output is G - c d (one FMA) and the four projection sums of
    // Y = c d are formed from d with the coefficient folded into the weights.
    // x-stage: c depends on k only, so the K-table carries (c w1, c h1).
    // y-stage: c depends on l only (cy0, cy1), applied once per thread.

    // G* row mirrored in v2 (l -> 31 - l) for specular y faces: the image of
    // this thread's pair (lb, lb+1) is pair 30 - lb of the thread with the
    // same k base in the partner warp (tid ^ 0x27), swapped.  Exchanged
    // through the (idle) reduction partials; CTA-uniform call sites only.
#if M32_TMEM_RED
    // (half a row per round: the reduction area holds NP doubles per thread)
    static_assert(red_size<NT_>() >= NP_ * NT_, "mirror exchange needs NP doubles per thread");
    auto mirror_l = [&](double (&v)[2 * NP_]) {
        double* xch = sred;
        const int pt = tid ^ 0x27;
#pragma unroll
        for (int h = 0; h < 2 * NP_; h += NP_) {
#pragma unroll
            for (int q = 0; q < NP_; q += 2) sts2(xch + NP_ * tid + q, v[h + q], v[h + q + 1]);
            __syncthreads();
#pragma unroll
            for (int q = 0; q < NP_; q += 2) {
                const double2 x = lds2(xch + NP_ * pt + q);
                v[h + q] = x.y;
                v[h + q + 1] = x.x;
            }
            __syncthreads();
        }
    };
#else
    auto mirror_l = [&](double (&v)[2 * NP_]) {
        double* xch = sred;
#pragma unroll
        for (int q = 0; q < 2 * NP_; q += 2) sts2(xch + 2 * NP_ * tid + q, v[q], v[q + 1]);
        __syncthreads();
        const int pt = tid ^ 0x27;
#pragma unroll
        for (int q = 0; q < 2 * NP_; q += 2) {
            const double2 x = lds2(xch + 2 * NP_ * pt + q);
            v[q] = x.y;
            v[q + 1] = x.x;
        }
        __syncthreads();
    };
#endif

    auto body = [&](int j, auto steady) {
        constexpr bool ST = decltype(steady)::value;
        const int rx = j + 2;       // x-stage row
        const int rc = j + 1;       // recon row
        const bool row_j = ST || (j >= j0s && j < j1s);
        // 0. stage the CellPar of row j+5 (its tables are built two
        //    iterations from now)
        stage_par(j + 5, ST || computes(j + 5));
        // 1. recon G*(j+1) = (G - dt Z) + dt Zhat_x (kept in gst for the
        //    v2 < 0 warps' y-stage, stored to the ring for the others)
        double gst[2 * NP_];
        tm_wait_st();
        if (ST || computes(rc)) {
            const double* T = T1;
            const double2 E2 = lds2(T + LT + L_E2 * NV + lb);
#if M32_TABPROJ
            // the x-stage's projection polynomial, tabulated by the reducer warp
            // one row ago: BE[l] here, (pE1, AL)[k] per pair below
            const double2 bEx = lds2(T + LT + L_BEX * NV + lb);
            const double bE0 = bEx.x, bE1 = bEx.y;
#elif M32_RAW
            // projection polynomial of the x-stage totals at the thread's nodes,
            // split as (C0 + C1 s xi + C3 xi^2) + eta (C2 s' + C3 ryx eta)
            const double c2s = sflip(ax[2]), c3y = ax[3] * a.ryx;
            const double bE0 = cy0 * fma(c3y, cy0, c2s) * E2.x;
            const double bE1 = cy1 * fma(c3y, cy1, c2s) * E2.y;
#else
            const double sc = T[HD + H_SCALE];
            const double a1 = ax[0] * sc, a2 = ax[1] * sc, a3 = ax[2] * sc, a4 = ax[3] * sc;
            const double2 w2 = lds2(T + LT + L_W2N * NV + lb);
            const double2 h2 = lds2(T + LT + L_H2 * NV + lb);
            const double bE0 = fma(w2.x, a3, h2.x * a4) * E2.x;
            const double bE1 = fma(w2.y, a3, h2.y * a4) * E2.y;
#endif
            MM2D_CHECK(R2 >= tq && R2 + 16 <= tq + TM_COLS && R1 >= tq && R0 >= tq);
            tm_ld8(R2, gst);
#pragma unroll
            for (int p = 0; p < NP_; ++p) {
#if M32_TABPROJ
                const double2 pa = lds2(T + koff_(p) + K_PEX);   // pE1, AL
                const double pe = pa.x, alp = pa.y;
#else
                const double pe = T[koff_(p) + K_PE1];
#endif
#if M32_TABPROJ
#elif M32_RAW
                const double alp =
                    fma(cx[p], fma(ax[3], cx[p], p < NP_ / 2 ? -ax[1] : ax[1]), ax[0]) * pe;
#else
                const double2 wh = lds2(T + koff_(p) + K_W1N);   // w1, h1
                const double alp = fma(wh.x, a2, fma(wh.y, a4, a1)) * pe;
#endif
                gst[2 * p] = fma(alp, E2.x, fma(bE0, pe, gst[2 * p]));
                gst[2 * p + 1] = fma(alp, E2.y, fma(bE1, pe, gst[2 * p + 1]));
            }
            tm_st8(R2, gst);
        } else if ((rc == j1s && k_hi != 0) || (rc == j0s - 1 && k_lo == 2)) {
            // ghost rows: zero (wall), copy or specular image of the adjacent owned row
            if (rc == j1s && k_hi == 1) tm_ld8(R1, gst);
            else if (MIR && rc == j1s && k_hi == 3) {
                tm_ld8(R1, gst);
                mirror_l(gst);
            } else {
#pragma unroll
                for (int q = 0; q < 2 * NP_; ++q) gst[q] = 0.0;
            }
            tm_st8(R2, gst);
        } else {
#pragma unroll
            for (int q = 0; q < 2 * NP_; ++q) gst[q] = 0.0;
        }
        if (!ST && rc == j0s && (k_lo == 1 || (MIR && k_lo == 3))) {
            // bottom ghost by copy / specular image, once G*(j0s) is complete
            double gb[2 * NP_];
#pragma unroll
            for (int q = 0; q < 2 * NP_; ++q) gb[q] = gst[q];
            if (MIR && k_lo == 3) mirror_l(gb);
            tm_wait_st();
            tm_st8(R1, gb);
        }
        double s[12];
#pragma unroll
        for (int q = 0; q < 8; ++q) s[q] = 0.0;
        // 2. y-stage of row j: d = G*_j - G*_upwind, G** - dt Zhat = G*_j - cy d.
        //    Both rows come back from the ring (the upwind row is j+1 for the
        //    v2 < 0 warps, j-1 for the others; warp-uniform), so the recon
        //    registers die at their store and no register copies are needed.
        if (row_j) {
            tm_wait_st();                  // G*(j+1) and any ghost copy are in the ring
            double c[2 * NP_];
            tm_ld8(R1, c);
            tm_ld8(negy ? R2 : R0, gst);
#if !M32_RAW
            const double2 w2 = lds2(T0 + LT + L_W2N * NV + lb);
            const double2 h2 = lds2(T0 + LT + L_H2 * NV + lb);
#endif
            double D0, D1, S1, S3;
#pragma unroll
            for (int p = 0; p < NP_; ++p) {
                const double d0 = c[2 * p] - gst[2 * p], d1 = c[2 * p + 1] - gst[2 * p + 1];
                ty[2 * p] = fma(-cy0, d0, c[2 * p]);
                ty[2 * p + 1] = fma(-cy1, d1, c[2 * p + 1]);
                const double e = fma(cy0, d0, cy1 * d1);
#if M32_RAW
                // raw moments of Y in the thread's coordinates: s xi, xi^2
                const double t = cx[p] * e;
                if (p == 0) {
                    D0 = d0; D1 = d1; S1 = -t; S3 = cx[p] * t;
                } else {
                    D0 += d0; D1 += d1; S1 = p < NP_ / 2 ? S1 - t : S1 + t; S3 = fma(cx[p], t, S3);
                }
#else
                const double2 wh = lds2(T0 + koff_(p) + K_W1N);   // w1, h1
                if (p == 0) {
                    D0 = d0; D1 = d1; S1 = wh.x * e; S3 = wh.y * e;
                } else {
                    D0 += d0; D1 += d1; S1 = fma(wh.x, e, S1); S3 = fma(wh.y, e, S3);
                }
#endif
            }
            const double Y0 = cy0 * D0, Y1 = cy1 * D1;
            s[0] = Y0 + Y1;
            s[1] = S1;
#if M32_RAW
            const double z0 = cy0 * Y0, z1 = cy1 * Y1;
            s[2] = sflip(z0 + z1);
            s[3] = fma(a.ryx, fma(cy0, z0, cy1 * z1), S3);
#else
            s[2] = fma(w2.x, Y0, w2.y * Y1);
            s[3] = S3 + fma(h2.x, Y0, h2.y * Y1);
#endif
        }
        // 3. x-stage of row j+2 into the slot of row j-1: G - dt Z_x = G - cx d
        const bool do_x = ST || computes(rx);
        if (do_x) {
            mbar_wait(mbar, (nload - 1) & 1);   // this row's bulk loads (issued one iteration ago)
#if !M32_RAW
            const double* T = T2;
            const double2 w2 = lds2(T + LT + L_W2N * NV + lb);
            const double2 h2 = lds2(T + LT + L_H2 * NV + lb);
#endif
            double xs[2 * NP_];
            double Y0, Y1, S1, S3;
#pragma unroll
            for (int p = 0; p < NP_; ++p) {
                const bool mir = MIR && !ST && (p < NP_ / 2 ? mir_r() : mir_l());
                const double2 c = lds2(stg + off_(p));
                const double2 h = lds2(stg + (mir ? NV * (NV - 1 - kb - KS * p) + lb : V + off_(p)));
                const double d0 = c.x - h.x, d1 = c.y - h.y;
                xs[2 * p] = fma(-cx[p], d0, c.x);
                xs[2 * p + 1] = fma(-cx[p], d1, c.y);
                const double e = d0 + d1;
#if M32_RAW
                const double t = cx[p] * (cx[p] * e);              // xi (y0 + y1)
                if (p == 0) {
                    Y0 = cx[p] * d0; Y1 = cx[p] * d1; S1 = -t; S3 = cx[p] * t;
                } else {
                    Y0 = fma(cx[p], d0, Y0); Y1 = fma(cx[p], d1, Y1);
                    S1 = p < NP_ / 2 ? S1 - t : S1 + t; S3 = fma(cx[p], t, S3);
                }
#else
                const double2 xw = lds2(T + koff_(p) + K_XW);      // cx w1, cx h1
                if (p == 0) {
                    Y0 = cx[p] * d0; Y1 = cx[p] * d1; S1 = xw.x * e; S3 = xw.y * e;
                } else {
                    Y0 = fma(cx[p], d0, Y0); Y1 = fma(cx[p], d1, Y1);
                    S1 = fma(xw.x, e, S1); S3 = fma(xw.y, e, S3);
                }
#endif
            }
            tm_st8(R0, xs);
            s[4] = Y0 + Y1;
            s[5] = S1;
#if M32_RAW
            const double z0 = cy0 * Y0, z1 = cy1 * Y1;
            s[6] = sflip(z0 + z1);
            s[7] = fma(a.ryx, fma(cy0, z0, cy1 * z1), S3);
#else
            s[6] = fma(w2.x, Y0, w2.y * Y1);
            s[7] = S3 + fma(h2.x, Y0, h2.y * Y1);
#endif
        }
        s[8] = hs[0]; s[9] = hs[1]; s[10] = hs[2]; s[11] = hs[3];
        // 4. the row's block reduction; the CellPar staged one iteration
        //    ago (row j+4) lands before it
        cp_async_wait_prev();
#if M32_TMEM_RED
        reduce12_begin_tm(s, sred, tq + TM_RED);
#else
        reduce12_begin<NT_>(s, sred);
#endif
        // every thread is past this row's x-stage reads: refill the staging
        if (ST || computes(rx + 1)) prefetch(rx + 1, steady);
        // tables for row j+3, built while the reduction's second phase runs:
        // slot T3 is read from iteration j+1 on, after this reduction's
        // closing barrier, and every reader of its previous row has passed
        // the opening barrier above
        if (ST || computes(j + 3))
            build_tables<KS>(a, T3, *reinterpret_cast<const CellPar*>(pring + 32 * ((j + 3) & 3)),
                             v1s, v2s, gauss, etab);
        // target + Gaussian of row j: independent of the projection sums, so
        // it is evaluated inside the reduction window
        double acc[2 * NP_];
        const double* wsrc = wx ? wx + (size_t)j * V_
                                : (ST ? nullptr : (j == 0 ? wb : (j == g.by - 1 ? wt : nullptr)));
        // acc = wh g^ + wg (G* - dt Z_y): everything of G^{n+1}(j) but the
        // y-projection, which waits for this reduction
#if M32_KEEPL
        double2 E2j = make_double2(0.0, 0.0), W2j = make_double2(0.0, 0.0);   // row j's l factors, kept for step 5
#endif
        if (row_j) {
            const double* T = T0;
            const double wg = T[HD + H_WG];
#if M32_KEEPL
            E2j = lds2(T + LT + L_E2 * NV + lb);
            W2j = lds2(T + LT + L_W2 * NV + lb);
#endif
            if (wsrc == nullptr) {
#if M32_KEEPL
                const double2 E2 = E2j;
#else
                const double2 E2 = lds2(T + LT + L_E2 * NV + lb);
#endif
#if M32_EPOW
                // E2 W2^n from E2 and W2 in the thread (8 fp64) instead of three
                // more 16-byte table loads (the l-indexed loads cost 4 wavefronts each)
#if M32_KEEPL
                const double2 W2t = W2j;
#else
                const double2 W2t = lds2(T + LT + L_W2 * NV + lb);
#endif
                const double2 e1 = make_double2(E2.x * W2t.x, E2.y * W2t.y);
                const double2 e2 = make_double2(e1.x * W2t.x, e1.y * W2t.y);
                const double2 e3 = make_double2(e2.x * W2t.x, e2.y * W2t.y);   // (f3 is in the K-table entry)
#else
                const double2 e1 = lds2(T + LT + L_EW1 * NV + lb);
                const double2 e2 = lds2(T + LT + L_EW2 * NV + lb);
                const double2 e3 = lds2(T + LT + L_EW3 * NV + lb);
#endif
                // ES-BGK Gaussian GA GB X with X(k, l) = exp(q12 W1 W2): the
                // thread's base X0 R^kb from the cross-term table, then R^8 per pair
                double2 GB = make_double2(0.0, 0.0);
                double Xq[NP_];            // X(k, lb) of the thread's pairs, as a product tree
#pragma unroll
                for (int p = 0; p < NP_; ++p) Xq[p] = 0.0;
                if (gauss) {
                    GB = lds2(T + GL + lb);
                    const double2 x0 = lds2(T + XT + X_X0R + xsel);   // X0, R
#if M32_RPOW
                    // R^2, R^4, R^8 squared up in the thread (3 fp64) instead of
                    // two more table loads
                    double2 r24;
                    r24.x = x0.y * x0.y;
                    r24.y = r24.x * r24.x;
                    const double r8 = r24.y * r24.y;
#else
                    const double2 r24 = lds2(T + XT + X_R24 + xsel);  // R^2, R^4
                    const double r8 = T[XT + X_R8 + lp];
#endif
                    const double xb = (x0.x * ((kb & 1) ? x0.y : 1.0)) *
                                      (((kb & 2) ? r24.x : 1.0) * ((kb & 4) ? r24.y : 1.0));
                    const double r16 = r8 * r8;
                    Xq[0] = xb;
                    Xq[1] = xb * r8;
                    Xq[2] = xb * r16;
                    Xq[3] = xb * (r16 * r8);
                }
#pragma unroll
                for (int p = 0; p < NP_; ++p) {
                    const double* K = T + koff_(p);
                    // closed-form target (_core.pyx:220-224), factored and
                    // pre-scaled by -wh/tau (minus wh/eps when Gaussian)
                    const double2 f01 = lds2(K + K_F0);   // pe f0', pe f1'
                    const double2 f2p = lds2(K + K_F2);   // pe f2', pe f3' (pe itself without M32_EPOW)
                    const double f2 = f2p.x, pe = f2p.y;
                    double P0 = fma(wg, ty[2 * p], f01.x * E2.x);
                    double P1 = fma(wg, ty[2 * p + 1], f01.x * E2.y);
                    P0 = fma(f01.y, e1.x, P0); P1 = fma(f01.y, e1.y, P1);
                    P0 = fma(f2, e2.x, P0); P1 = fma(f2, e2.y, P1);
                    P0 = fma(pe, e3.x, P0); P1 = fma(pe, e3.y, P1);
                    if (gauss) {
                        // + Gaussian wh/eps, Gaussian = GA GB X
                        const double2 gad = lds2(T + GK + 2 * (kb + KS * p));   // GA', GD
                        const double Y0 = gad.x * Xq[p];
                        P0 = fma(GB.x, Y0, P0);
                        P1 = fma(GB.y, Y0 * gad.y, P1);
                    }
                    acc[2 * p] = P0;
                    acc[2 * p + 1] = P1;
                }
            } else {
                // wall-strip target (boundary.py:343-378), precomputed
                const double wh_ = T[HD + H_WH];
#pragma unroll
                for (int p = 0; p < NP_; ++p) {
                    const double2 w = __ldg(reinterpret_cast<const double2*>(wsrc + off_(p)));
                    acc[2 * p] = fma(wg, ty[2 * p], wh_ * w.x);
                    acc[2 * p + 1] = fma(wg, ty[2 * p + 1], wh_ * w.y);
                }
            }
        }
#if M32_TMEM_RED
        reduce12_end_tm(s, sred,
#else
        reduce12_end<NT_>(s, sred,
#endif
                          (ST || (j - 1 >= j0s && j - 1 < j1s)) ? a.Hr + 4 * ring_index(g, i, j - 1)
                                                                : nullptr,
                          a.hfac
#if !M32_TMEM_RED
                          , a, T0, T2, mbar + 1, (unsigned)(j - jfirst) & 1, T0, T2, v1s, v2s
#endif
                          );
#if !M32_TABPROJ
        if (do_x) {
            ax[0] = s[4]; ax[1] = s[5]; ax[2] = s[6]; ax[3] = s[7];
        }
#endif
        // 5. G**(j), relax, store, heat partials
        hs[0] = hs[1] = hs[2] = hs[3] = 0.0;
        if (row_j) {
            // G^{n+1} = acc + wg Zhat_y, Zhat_y = (a1 + w1 a2 + h1 a4 + w2 a3 + h2 a4) M
            // split as (al pE1) E2 + pE1 (b E2) with wg folded into the a's
            const double* T = T0;
#if M32_KEEPL
            const double2 E2 = E2j, W2 = W2j;
#else
            const double2 E2 = lds2(T + LT + L_E2 * NV + lb);
            const double2 W2 = lds2(T + LT + L_W2 * NV + lb);
#endif
#if M32_TABPROJ
            const double2 bEy = lds2(T + LT + L_BEY * NV + lb);
            const double bE0 = bEy.x, bE1 = bEy.y;
#elif M32_RAW
            // (the y totals arrive as polynomial coefficients, scale and wg folded in)
            const double c2s = sflip(s[2]), c3y = s[3] * a.ryx;
            const double bE0 = cy0 * fma(c3y, cy0, c2s) * E2.x;
            const double bE1 = cy1 * fma(c3y, cy1, c2s) * E2.y;
#else
            const double sc = T[HD + H_SCALE] * T[HD + H_WG];
            const double a1 = s[0] * sc, a2 = s[1] * sc, a3 = s[2] * sc, a4 = s[3] * sc;
            const double2 w2 = lds2(T + LT + L_W2N * NV + lb);
            const double2 h2 = lds2(T + LT + L_H2 * NV + lb);
            const double bE0 = fma(w2.x, a3, h2.x * a4) * E2.x;
            const double bE1 = fma(w2.y, a3, h2.y * a4) * E2.y;
#endif
            MM2D_CHECK(j >= 0 && j < g.by && j >= j0s && j < j1s);
            MM2D_CHECK(T0 >= tabs && T0 + SLOT <= tabs + TSLOTS * SLOT);
            double* out = out_b + (size_t)j * V_;
            double A0x, A0y, A1x, A1y, A2x, A2y, A3x, A3y;
#pragma unroll
            for (int p = 0; p < NP_; ++p) {
                const double* K = T + koff_(p);
                const double2 pw = lds2(K + K_PE1);     // pE1, W1
#if M32_W1POW_TABLE
                const double2 w3 = lds2(K + K_W12);     // W1^2, W1^3
#else
                double2 w3;
                w3.x = pw.y * pw.y;
                w3.y = w3.x * pw.y;
#endif
#if M32_TABPROJ
                const double alp = K[K_ALY];
#elif M32_RAW
                const double alp =
                    fma(cx[p], fma(s[3], cx[p], p < NP_ / 2 ? -s[1] : s[1]), s[0]) * pw.x;
#else
                const double2 wh = lds2(K + K_W1N);     // w1, h1
                const double alp = fma(wh.x, a2, fma(wh.y, a4, a1)) * pw.x;
#endif
                const double o0 = fma(alp, E2.x, fma(bE0, pw.x, acc[2 * p]));
                const double o1 = fma(alp, E2.y, fma(bE1, pw.x, acc[2 * p + 1]));
                *reinterpret_cast<double2*>(out + off_(p)) = make_double2(o0, o1);
                // heat moments about u^n (_core.pyx:303-321): A_a = sum W1^a o
                if (p == 0) {
                    A0x = o0; A0y = o1;
                    A1x = pw.y * o0; A1y = pw.y * o1;
                    A2x = w3.x * o0; A2y = w3.x * o1;
                    A3x = w3.y * o0; A3y = w3.y * o1;
                } else {
                    A0x += o0; A0y += o1;
                    A1x = fma(pw.y, o0, A1x); A1y = fma(pw.y, o1, A1y);
                    A2x = fma(w3.x, o0, A2x); A2y = fma(w3.x, o1, A2y);
                    A3x = fma(w3.y, o0, A3x); A3y = fma(w3.y, o1, A3y);
                }
            }
            const double W2xx = W2.x * W2.x, W2yy = W2.y * W2.y;
            hs[0] = A3x + A3y;
            hs[1] = fma(W2.x, A2x, W2.y * A2y);
            hs[2] = fma(W2xx, A1x, W2yy * A1y);
            hs[3] = fma(W2xx * W2.x, A0x, (W2yy * W2.y) * A0y);
        }
        // rotate slots for the next row
        {
            const unsigned r0 = R0; R0 = R1; R1 = R2; R2 = r0;
            double* t0 = T0; T0 = T1; T1 = T2; T2 = T3; T3 = t0;
        }
    };

    // steady rows: every stage active, no ghost rows, no wall rows
    const int js_lo = j0s + 1, js_hi = (MIR && (mir_l() || mir_r())) ? js_lo - 1 : min(rhi - 5, j1s - 1);
#if M32_SHORT_FILL
    // The first pipeline iteration (j0s - 4) would only stage CellPar row
    // j0s + 1, issue the bulk load of x-stage row j0s - 1 (issued at entry)
    // and build its tables; done here, without that iteration's reduction and its two
    // barriers, so a band pays one pipeline-fill iteration less.
    int j = j0s - 3;
    stage_par(j0s + 1, computes(j0s + 1));
    if (computes(j0s - 1)) {   // (its bulk load was issued at entry)
        build_tables<KS>(a, T3, *reinterpret_cast<const CellPar*>(pring + 32 * ((j0s - 1) & 3)),
                         v1s, v2s, gauss, etab);
    }
    __syncthreads();
    {
        const unsigned r0 = R0; R0 = R1; R1 = R2; R2 = r0;
        double* t0 = T0; T0 = T1; T1 = T2; T2 = T3; T3 = t0;
    }
#else
    int j = j0s - 4;
#endif
    for (; j < js_lo && j <= j1s; ++j) body(j, std::false_type());
    for (; j <= js_hi; ++j) body(j, std::true_type());
    for (; j <= j1s; ++j) body(j, std::false_type());
    // release the ring (every warp's TMEM traffic has completed)
    tm_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (tid < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tbase),
                     "n"(TM_COLS)
                     : "memory");
#undef off_
#undef koff_
}

// Diffuse-wall strip targets: g^ = -(Mterm - Pi[Mterm]) / tau for every
// wall-adjacent cell (boundary.py:343-378; _wall_maxwellian_layer 293-301,
// extend_maxwellian_2d 304-340).  One CTA per strip cell; faces laid out
// left (by), right (by), bottom (bx), top (bx).
__global__ void __launch_bounds__(128) k_wall_ghat(MicroArgs a, double* out) {
    pdl_enter();
    __shared__ double sh[32];
    const Geometry& g = a.g;
    if (err_pending(a.err, EW_PREP)) return;
    const int e = blockIdx.x;
    int f, i, j;
    if (e < g.by) { f = 0; i = 0; j = e; }
    else if (e < 2 * g.by) { f = 1; i = g.bx - 1; j = e - g.by; }
    else if (e < 2 * g.by + g.bx) { f = 2; i = e - 2 * g.by; j = 0; }
    else { f = 3; i = e - 2 * g.by - g.bx; j = g.by - 1; }
    if (!g.wall[f]) return;
    const CellPar& P = a.P[ring_index(g, i, j)];
    const int nv2 = g.nv2, V = g.V;
    double s[4] = {0, 0, 0, 0};
    double mt[16];
    int cnt = 0;
    for (int n = threadIdx.x; n < V; n += blockDim.x, ++cnt) {
        const int k = n / nv2, l = n % nv2;
        const double v1 = a.v1[k], v2 = a.v2[l];
        const double x1 = v1 - P.u1, x2 = v2 - P.u2;
        const double M = P.pref * exp(-(x1 * x1 + x2 * x2) * P.inv2T);
        double Mn[4];
        for (int q = 0; q < 4; ++q) {
            const int ii = i + (q == 0 ? -1 : q == 1 ? 1 : 0);
            const int jj = j + (q == 2 ? -1 : q == 3 ? 1 : 0);
            const bool outside = ii < 0 || ii >= g.bx || jj < 0 || jj >= g.by;
            if (outside && g.wall[q]) {
                const double Tw = g.wallT[q], U = g.wallU[q];
                const double g1 = q < 2 ? 0.0 : U, g2 = q < 2 ? U : 0.0;
                const double y1 = v1 - g1, y2 = v2 - g2;
                Mn[q] = P.rw[q] / (2.0 * kPi * Tw) * exp(-(y1 * y1 + y2 * y2) / (2.0 * Tw));
            } else {
                const CellPar& Q = a.P[ring_index(g, ii, jj)];
                const double y1 = v1 - Q.u1, y2 = v2 - Q.u2;
                Mn[q] = Q.pref * exp(-(y1 * y1 + y2 * y2) * Q.inv2T);
            }
        }
        const double vm1 = v1 < 0.0 ? v1 : 0.0, vp1 = v1 > 0.0 ? v1 : 0.0;
        const double vm2 = v2 < 0.0 ? v2 : 0.0, vp2 = v2 > 0.0 ? v2 : 0.0;
        const double Mt = (vm1 * (Mn[1] - M) + vp1 * (M - Mn[0])) * a.idx +
                          (vm2 * (Mn[3] - M) + vp2 * (M - Mn[2])) * a.idy;
        const double w1 = x1 * P.isT, w2 = x2 * P.isT;
        const double b4 = 0.5 * (w1 * w1 + w2 * w2) - 1.0;
        s[0] += Mt; s[1] += Mt * w1; s[2] += Mt * w2; s[3] += Mt * b4;
        mt[cnt] = Mt;
    }
    double c[4];
    for (int q = 0; q < 4; ++q) {
        double v = warp_sum(s[q]);
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        __syncthreads();
        if (lane == 0) sh[w] = v;
        __syncthreads();
        double t = 0.0;
        for (int u = 0; u < (int)(blockDim.x >> 5); ++u) t += sh[u];
        c[q] = t * P.scale;
    }
    double* o = out + (size_t)e * V;
    cnt = 0;
    for (int n = threadIdx.x; n < V; n += blockDim.x, ++cnt) {
        const int k = n / nv2, l = n % nv2;
        const double x1 = a.v1[k] - P.u1, x2 = a.v2[l] - P.u2;
        const double M = P.pref * exp(-(x1 * x1 + x2 * x2) * P.inv2T);
        const double w1 = x1 * P.isT, w2 = x2 * P.isT;
        const double b4 = 0.5 * (w1 * w1 + w2 * w2) - 1.0;
        const double pi = (c[0] + w1 * c[1] + w2 * c[2] + b4 * c[3]) * M;
        o[n] = -(mt[cnt] - pi) * P.invtau;
    }
}

}  // namespace m32
}  // namespace mm2d
