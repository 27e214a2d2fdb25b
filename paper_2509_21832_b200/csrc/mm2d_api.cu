// C ABI of libmm2d.so (declared in include/mm2d.h).  Owns the per-problem
// context: device buffers, launch configuration, CUDA graphs and the sticky
// error word.  See mm2d.h for the reference interfaces each entry replaces.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "mm2d.h"

// k_prep_tiled (shared-memory neighbour primitives) or the one-thread-per-
// cell k_prep; both produce the same CellPar bits
#ifndef MM2D_PREP_TILED
#define MM2D_PREP_TILED 1
#endif
#include "mm2d_common.cuh"
#include "mm2d_contract.cuh"
#include "mm2d_macro.cuh"
#include "mm2d_micro.cuh"
// The 32 x 32 micro kernel is compiled inside this translation unit: NVVM
// emits measurably better code for it here than in a standalone TU
// (0.419 vs 0.429 ms at C2, same source; tools/ab.sh).
#include "mm2d_micro32.cu"
#include "mm2d_prep.cuh"

using namespace mm2d;

// launches issued by this library (both the 2D and the 1D entry points)
std::atomic<long long> g_launches{0};

struct mm2d_ctx {
    mm2d_config cfg;
    Geometry g;
    int dev = 0;
    cudaStream_t stream = nullptr;
    double* d_v1 = nullptr;
    double* d_v2 = nullptr;
    CellPar* d_P = nullptr;
    double* d_Qr = nullptr;
    double* d_Hr = nullptr;
    double* d_Qx = nullptr;
    unsigned long long* d_err = nullptr;   // ErrWord layout (mm2d_common.cuh) + [8] error value
    unsigned long long* h_err = nullptr;   // pinned read-back of the 9 words
    cudaStream_t last_s = nullptr;         // stream of the last enqueued step (mm2d_check syncs it)
    // halo buffers for the micro field (multi-rank only)
    double* d_gh[4] = {nullptr, nullptr, nullptr, nullptr};
    double* d_wallg = nullptr;     // wall-strip targets (fast kernel)
    double* d_zero = nullptr;      // V zeros
    bool use32 = false;            // specialised 32 x 32 micro kernel
    std::vector<int> bands32;      // non-uniform band boundaries (empty: uniform ly32)
    int ly32 = 32;
    // context-owned state
    double* d_Qs[2] = {nullptr, nullptr};
    double* d_Gs[2] = {nullptr, nullptr};
    double* d_Hsoa = nullptr;
    int cur = 0;
    // micro launch configuration
    int BX = 2, NE = 4, NT = 256, ly = 32;
    bool fast = true;
    size_t smem = 0;
    const void* micro_fn = nullptr;
    // graphs for context-owned stepping (parity 0: A->B, 1: B->A)
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    double graph_dt = 0.0;
    double last_dt = 0.0;
    double* last_Qout = nullptr;
    bool counting = true;
    long long launches_per_step = 7;
    bool state_owned = false;
    cudaStream_t user_stream = nullptr;
    bool have_user_stream = false;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    // halo staging (multi-rank): [field G/Q/H][slot]
    bool halo_ready = false;
    int halo_cells[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // peer form of the G halos (mm2d_halo_peer): the neighbours' current G arrays
    const double* peerG[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    bool peer = false;
    double* hsend[3][8] = {};
    double* hrecv[3][8] = {};
    int sms = 148;                 // multiprocessors of the context's device
    std::string err;
};

#define CK(call)                                                                       \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess) {                                                       \
            if (ctx) ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);    \
            return MM2D_ERR_INTERNAL;                                                  \
        }                                                                              \
    } while (0)

static int fail_cfg(mm2d_ctx* ctx, const std::string& m) {
    if (ctx) ctx->err = m;
    return MM2D_ERR_CONFIG;
}

// ---- micro kernel instantiations ----
template <int NE, int BX, bool FAST>
static const void* micro_ptr() {
    return reinterpret_cast<const void*>(&k_micro<NE, BX, FAST>);
}

static const void* pick_micro(int NE, int BX, bool fast) {
#define PICK(ne, bx)                                              \
    if (NE == ne && BX == bx) return fast ? micro_ptr<ne, bx, true>() : micro_ptr<ne, bx, false>();
    PICK(2, 1) PICK(2, 2) PICK(4, 1) PICK(4, 2) PICK(8, 1) PICK(8, 2)
#undef PICK
    return nullptr;
}

static int ghost_mode(const mm2d_config& c, int face, bool at_edge, int nranks_axis, int field) {
    // field 0: micro G (walls zero), 1: macro Q (walls copy), 2: heat (walls zero);
    // specular walls mirror every field
    if (!at_edge) return GM_HALO;
    const int kind = c.face[face];
    if (kind == MM2D_FACE_PERIODIC) return nranks_axis > 1 ? GM_HALO : GM_WRAP;
    if (kind == MM2D_FACE_EXTRAPOLATE) return GM_COPY;
    if (kind == MM2D_FACE_SPECULAR) return GM_MIRROR;
    return field == 1 ? GM_COPY : GM_ZERO;
}

// Band layout for k_micro32 when the block is too small for uniform bands
// to fill the resident CTA slots in whole waves (C2: 256 columns, 592
// slots).  Every column gets L long bands of H rows plus one short band of
// R = by - L H rows; the L bx long CTAs take one slot each for H + 4 row
// times (4 = the row pipeline's fill) while the spare slots run the bx short
// CTAs back to back, so H is the smallest height at which
//     spare (H + 4) >= bx (R + 4),   spare = slots - L bx.
// All columns share the band boundaries, so neighbouring columns still run
// the same rows together (the x-halo halves stay in L2).  Chosen over
// uniform bands of `ly` rows (makespan ~ waves (ly + 4)) when it is at
// least 3% shorter.  Measured at C2: uniform 64 -> 0.391 ms, [112,112,32]
// -> 0.377 ms; [114,114,28] 0.377, [116,116,24] 0.383, [108,108,40] 0.392.
static std::vector<int> pick_bands(int bx, int by, long long slots, int ly) {
    // pipeline fill in row-iterations: a long band pays ov once; a short band,
    // run back to back with others in a spare slot, also pays its CTA start
    // (measured optimum at C2: 114/114/28, step 0.3879 ms vs 0.3904 for
    // 112/112/32 and 0.394 for 116/116/24, which ov_s = 8 reproduces)
    const long long ov = 4, ov_s = 8;
    const long long nb = (by + ly - 1) / ly;
    const long long waves = ((long long)bx * nb + slots - 1) / slots;
    double best = (double)waves * (ly + ov);
    std::vector<int> out;
    for (int L = 1; L <= 8 && (long long)L * bx < slots; ++L) {
        const long long spare = slots - (long long)L * bx;
        const long long num = (long long)bx * (by + ov_s) - ov * spare;
        const long long den = spare + (long long)L * bx;
        const long long H = (num + den - 1) / den;
        const long long R = by - L * H;
        if (H < 16 || R < 1 || R >= H) continue;
        if ((double)(H + ov) < 0.97 * best) {
            best = (double)(H + ov);
            out.assign(1, 0);
            for (int b = 1; b <= L; ++b) out.push_back((int)(b * H));
            out.push_back(by);
        }
    }
    return out;
}

extern "C" int mm2d_version(void) { return 1; }

extern "C" int mm2d_kernel_version(void) { return M32_KERNEL_VERSION; }

extern "C" const char* mm2d_last_error(mm2d_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

extern "C" long long mm2d_launch_count(void) { return g_launches.load(); }
extern "C" void mm2d_reset_launch_count(void) { g_launches.store(0); }

extern "C" int mm2d_create(const mm2d_config* cfg, mm2d_ctx** out) {
    if (!cfg || !out) return MM2D_ERR_CONFIG;
    *out = nullptr;
    mm2d_ctx* ctx = new mm2d_ctx();
    ctx->cfg = *cfg;
    const mm2d_config& c = ctx->cfg;
    if (c.nx < 1 || c.ny < 1 || c.nv1 < 2 || c.nv2 < 2) {
        int r = fail_cfg(ctx, "grid sizes must be nx, ny >= 1 and nv1, nv2 >= 2");
        delete ctx;
        return r;
    }
    if (c.px < 1 || c.py < 1 || c.nx % c.px || c.ny % c.py || c.rx < 0 || c.rx >= c.px ||
        c.ry < 0 || c.ry >= c.py) {
        int r = fail_cfg(ctx, "rank grid must divide the spatial grid (make_plans)");
        delete ctx;
        return r;
    }
    for (int f = 0; f < 4; ++f)
        if (c.face[f] < 0 || c.face[f] > 3) {
            int r = fail_cfg(ctx, "unknown face kind");
            delete ctx;
            return r;
        }
    if ((c.face[0] == MM2D_FACE_PERIODIC) != (c.face[1] == MM2D_FACE_PERIODIC) ||
        (c.face[2] == MM2D_FACE_PERIODIC) != (c.face[3] == MM2D_FACE_PERIODIC)) {
        int r = fail_cfg(ctx, "periodic boundaries must come in pairs");
        delete ctx;
        return r;
    }
    {
        // specular faces mirror the node index along the wall normal, which is
        // the reflection v_n -> -v_n only on an axis symmetric about zero
        const double lo[2] = {c.v1_min, c.v2_min}, hi[2] = {c.v1_max, c.v2_max};
        for (int f = 0; f < 4; ++f) {
            if (c.face[f] != MM2D_FACE_SPECULAR) continue;
            const int ax = f < 2 ? 0 : 1;
            if (!(std::fabs(lo[ax] + hi[ax]) <= 1e-14 * (hi[ax] - lo[ax]))) {
                int r = fail_cfg(ctx, "specular walls need a velocity axis symmetric about zero "
                                      "along the wall normal");
                delete ctx;
                return r;
            }
        }
    }
    if (!(c.nu >= -1.0 && c.nu < 1.0)) {
        int r = fail_cfg(ctx, "nu must lie in [-1, 1)");
        delete ctx;
        return r;
    }
    ctx->dev = c.device;
    if (cudaSetDevice(ctx->dev) != cudaSuccess) {
        int r = fail_cfg(ctx, "cudaSetDevice failed");
        delete ctx;
        return r;
    }
    Geometry& g = ctx->g;
    memset(&g, 0, sizeof(g));
    g.nx = c.nx; g.ny = c.ny;
    g.bx = c.nx / c.px; g.by = c.ny / c.py;
    g.i0 = c.rx * g.bx; g.j0 = c.ry * g.by;
    g.nv1 = c.nv1; g.nv2 = c.nv2; g.V = c.nv1 * c.nv2;
    g.dx = (c.x_max - c.x_min) / c.nx;
    g.dy = (c.y_max - c.y_min) / c.ny;
    const bool e[4] = {c.rx == 0, c.rx == c.px - 1, c.ry == 0, c.ry == c.py - 1};
    const int nr[4] = {c.px, c.px, c.py, c.py};
    int* gm[3][4] = {{&g.xlo, &g.xhi, &g.ylo, &g.yhi},
                     {&g.qxlo, &g.qxhi, &g.qylo, &g.qyhi},
                     {&g.hxlo, &g.hxhi, &g.hylo, &g.hyhi}};
    for (int fld = 0; fld < 3; ++fld)
        for (int f = 0; f < 4; ++f) *gm[fld][f] = ghost_mode(c, f, e[f], nr[f], fld);
    for (int f = 0; f < 4; ++f) {
        g.phys[f] = e[f] && c.face[f] != MM2D_FACE_PERIODIC;
        g.wall[f] = e[f] && c.face[f] == MM2D_FACE_WALL;
        g.wallT[f] = c.wall_T[f];
        g.wallU[f] = c.wall_U[f];
        if (c.face[f] == MM2D_FACE_WALL && !(c.wall_T[f] > 0.0)) {
            int r = fail_cfg(ctx, "wall temperature must be positive");
            delete ctx;
            return r;
        }
    }
    // launch configuration of the fused micro kernel
    const int V = g.V;
    ctx->fast = (c.nv2 % 2) == 0;
    int NE = 2;
    if (ctx->fast) {
        NE = V <= 512 ? 2 : V <= 1024 ? 4 : 8;
    } else {
        NE = V <= 1024 ? 4 : 8;
    }
    const int per = (V + NE - 1) / NE;
    int NT = ((per + 31) / 32) * 32;
    if (NT > 256) {
        int r = fail_cfg(ctx, "velocity grid too large (nv1*nv2 <= 2048 supported)");
        delete ctx;
        return r;
    }
    ctx->NE = NE;
    ctx->NT = NT;
    ctx->BX = (g.bx >= 2 && V <= 1024) ? 2 : 1;
    ctx->ly = std::min(g.by, 32);
    ctx->micro_fn = pick_micro(NE, ctx->BX, ctx->fast);
    ctx->smem = micro_smem_bytes(ctx->BX, V, c.nv1, c.nv2);
    if (!ctx->micro_fn) {
        int r = fail_cfg(ctx, "no micro kernel instantiation for this velocity grid");
        delete ctx;
        return r;
    }
    ctx->use32 = c.nv1 == 32 && c.nv2 == 32 && getenv("MM2D_GENERIC") == nullptr;
    if (ctx->use32) {
        // the specialised kernel folds the upwind sign per node pair: both
        // nodes of every (l, l+1) pair must share the sign of v2
        const double h2 = (c.v2_max - c.v2_min) / c.nv2;
        for (int l = 0; l < c.nv2; l += 2) {
            const double a0 = c.v2_min + (l + 0.5) * h2, a1 = c.v2_min + (l + 1.5) * h2;
            if ((a0 < 0.0) != (a1 < 0.0)) ctx->use32 = false;
        }
        // and the x upwind direction must flip exactly between k = 15 and 16
        const double h1 = (c.v1_max - c.v1_min) / c.nv1;
        for (int k = 0; k < c.nv1; ++k) {
            const double vk = c.v1_min + (k + 0.5) * h1;
            if ((vk < 0.0) != (k < 16)) ctx->use32 = false;
        }
    }
    if (ctx->use32) {
        int occ = 0, nsm = 0;
        if (m32::setup(&occ) != cudaSuccess) {
            int r = fail_cfg(ctx, "shared memory request too large for k_micro32");
            delete ctx;
            return r;
        }
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->dev);
        // Band height: a CTA walks one column through ly rows, paying ~4
        // pipeline-fill iterations per band.  Measured on C2 (256 x 256,
        // 148 SMs x 4 CTAs, kernel v18): ly 32 / 40 / 43 / 48 / 56 / 64 / 86 / 128
        // give 0.412 / 0.398 / 0.409 / 0.410 / 0.409 / 0.390 / 0.438 / 0.419 ms
        // (partial-wave effects dominate at 256 columns); at C4 (1024^2) 64
        // and 56 give 5.47 and 5.51 ms.
        // Taller blocks take taller bands (fewer pipeline fills per row; the
        // many waves hide the tail).  Step times measured with
        // tools/band_bench.py (two alternating rounds, ms/step):
        //   C3 512^2:  bands 446/66 1.448, uniform 128 1.425, 192 1.504, 256 1.437
        //   C4 1024^2: uniform 64 5.72, 160 5.60-5.65, 192 5.64-5.68, 256 5.72
        //   C5 2048^2: uniform 64 23.41, 192 23.10-23.15, 320 22.90-23.04, 384 22.93-23.15
        const char* ly = getenv("MM2D_LY");
        const int ly_def = g.by >= 2048 ? 320 : g.by >= 1024 ? 160 : g.by >= 512 ? 128 : 64;
        ctx->ly32 = ly ? std::max(1, atoi(ly)) : ly_def;
        // explicit band heights (same for every column), e.g. MM2D_BANDS=114,114,22,6
        if (const char* bs = getenv("MM2D_BANDS")) {
            std::vector<int> h;
            for (const char* q = bs; *q;) {
                h.push_back(atoi(q));
                while (*q && *q != ',') ++q;
                if (*q == ',') ++q;
            }
            int acc = 0;
            ctx->bands32.push_back(0);
            for (int x : h) {
                if (x <= 0 || (int)ctx->bands32.size() > 8) break;
                acc = std::min(g.by, acc + x);
                ctx->bands32.push_back(acc);
                if (acc == g.by) break;
            }
            if (ctx->bands32.back() != g.by) ctx->bands32.clear();   // must cover the block
        } else if (!ly && g.by < 512) {
            ctx->bands32 = pick_bands(g.bx, g.by, (long long)std::max(occ, 1) * std::max(nsm, 1),
                                      ctx->ly32);
        }
        ctx->ly32 = std::min(ctx->ly32, g.by);
        if (getenv("MM2D_VERBOSE")) {
            fprintf(stderr, "mm2d: k_micro32 %d CTAs/SM x %d SMs, block %d x %d, bands", occ, nsm,
                    g.bx, g.by);
            if (ctx->bands32.empty()) fprintf(stderr, " uniform %d\n", ctx->ly32);
            else {
                for (size_t b = 1; b < ctx->bands32.size(); ++b)
                    fprintf(stderr, " %d", ctx->bands32[b] - ctx->bands32[b - 1]);
                fprintf(stderr, "\n");
            }
        }
    }
    if (cudaFuncSetAttribute(ctx->micro_fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)ctx->smem) != cudaSuccess) {
        int r = fail_cfg(ctx, "shared memory request too large for the micro kernel");
        delete ctx;
        return r;
    }
    // buffers
    const size_t ring = (size_t)(g.bx + 2) * (g.by + 2);
    std::vector<double> v1(c.nv1), v2(c.nv2);
    const double h1 = (c.v1_max - c.v1_min) / c.nv1, h2 = (c.v2_max - c.v2_min) / c.nv2;
    for (int k = 0; k < c.nv1; ++k) v1[k] = c.v1_min + ((k + 1) - 0.5) * h1;
    for (int l = 0; l < c.nv2; ++l) v2[l] = c.v2_min + ((l + 1) - 0.5) * h2;
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    CK(cudaMalloc(&ctx->d_v1, sizeof(double) * c.nv1));
    CK(cudaMalloc(&ctx->d_v2, sizeof(double) * c.nv2));
    CK(cudaMemcpy(ctx->d_v1, v1.data(), sizeof(double) * c.nv1, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->d_v2, v2.data(), sizeof(double) * c.nv2, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&ctx->d_P, sizeof(CellPar) * ring));
    CK(cudaMalloc(&ctx->d_Qr, sizeof(double) * 6 * ring));
    CK(cudaMalloc(&ctx->d_Hr, sizeof(double) * 4 * ring));
    CK(cudaMalloc(&ctx->d_Qx, sizeof(double) * 6 * ring));
    CK(cudaMemset(ctx->d_Qr, 0, sizeof(double) * 6 * ring));
    CK(cudaMemset(ctx->d_Hr, 0, sizeof(double) * 4 * ring));
    CK(cudaMemset(ctx->d_Qx, 0, sizeof(double) * 6 * ring));
    CK(cudaMalloc(&ctx->d_err, sizeof(unsigned long long) * (EW_N + 1)));
    CK(cudaMallocHost(&ctx->h_err, sizeof(unsigned long long) * (EW_N + 1)));
    {
        unsigned long long init[EW_N + 1] = {kNoError, 0, 0, 0, 0, kNoError, kNoError, kNoError, 0};
        CK(cudaMemcpy(ctx->d_err, init, sizeof(init), cudaMemcpyHostToDevice));
    }
    // the launch attribute the tiled prep needs, set once here (outside any
    // stream capture) instead of on the launch path
    CK(cudaFuncSetAttribute(k_prep_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)kPrepStageBytes));
    {
        int sms = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->dev));
        ctx->sms = sms > 0 ? sms : 148;
    }
    const size_t Vs = (size_t)V;
    for (int f = 0; f < 4; ++f) {
        const bool halo = *gm[0][f] == GM_HALO;
        if (!halo) continue;
        const size_t cells = f < 2 ? (size_t)g.by : (size_t)g.bx + 2;
        CK(cudaMalloc(&ctx->d_gh[f], sizeof(double) * cells * Vs));
        CK(cudaMemset(ctx->d_gh[f], 0, sizeof(double) * cells * Vs));
    }
    CK(cudaMalloc(&ctx->d_zero, sizeof(double) * Vs));
    CK(cudaMemset(ctx->d_zero, 0, sizeof(double) * Vs));
    if (ctx->use32 && (g.wall[0] || g.wall[1] || g.wall[2] || g.wall[3])) {
        const size_t n = (size_t)(2 * g.by + 2 * g.bx) * Vs;
        CK(cudaMalloc(&ctx->d_wallg, sizeof(double) * n));
        CK(cudaMemset(ctx->d_wallg, 0, sizeof(double) * n));
    }
    *out = ctx;
    return MM2D_OK;
}

extern "C" int mm2d_destroy(mm2d_ctx* ctx) {
    if (!ctx) return MM2D_OK;
    cudaSetDevice(ctx->dev);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (int p = 0; p < 2; ++p) {
        if (ctx->gexec[p]) cudaGraphExecDestroy(ctx->gexec[p]);
        if (ctx->state_owned) {
            cudaFree(ctx->d_Qs[p]);
            cudaFree(ctx->d_Gs[p]);
        }
    }
    if (ctx->state_owned) cudaFree(ctx->d_Hsoa);
    if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
    if (ctx->ev_out) cudaEventDestroy(ctx->ev_out);
    for (int f = 0; f < 3; ++f)
        for (int q = 0; q < 8; ++q) {
            cudaFree(ctx->hsend[f][q]);
            if (f > 0) cudaFree(ctx->hrecv[f][q]);
        }
    for (int f = 0; f < 4; ++f) cudaFree(ctx->d_gh[f]);
    cudaFree(ctx->d_wallg);
    cudaFree(ctx->d_zero);
    cudaFree(ctx->d_v1); cudaFree(ctx->d_v2); cudaFree(ctx->d_P); cudaFree(ctx->d_Qr);
    cudaFree(ctx->d_Hr); cudaFree(ctx->d_Qx); cudaFree(ctx->d_err);
    if (ctx->h_err) cudaFreeHost(ctx->h_err);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return MM2D_OK;
}

extern "C" int mm2d_block(mm2d_ctx* ctx, int* bx, int* by, int* i0, int* j0) {
    if (!ctx) return MM2D_ERR_CONFIG;
    if (bx) *bx = ctx->g.bx;
    if (by) *by = ctx->g.by;
    if (i0) *i0 = ctx->g.i0;
    if (j0) *j0 = ctx->g.j0;
    return MM2D_OK;
}

// (4, bx, by) SoA heat tensor from the ring
__global__ void k_h_soa(Geometry g, const double* Hr, double* H) {
    const int n = g.bx * g.by;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const int i = t / g.by, j = t % g.by;
        const double* h = Hr + 4 * ring_index(g, i, j);
        for (int c = 0; c < 4; ++c) H[(size_t)c * n + t] = h[c];
    }
}

static int grid_for(long long n, int threads) {
    long long b = (n + threads - 1) / threads;
    return (int)std::max(1LL, std::min(b, 148LL * 32));
}

// enqueue one full step on `s` (graph-capturable: no host syncs)
static int enqueue_step(mm2d_ctx* ctx, const double* Q, const double* G, double dt, double* Qout,
                        double* Gout, double* H, int nsrc, const double* sc, const double* ss,
                        const double* qsrc, cudaStream_t s, cudaEvent_t* ev = nullptr,
                        int phases = 3, int part = 0, int mode = 0) {
    // part: micro CTAs launched (0 all, 1 those that read no received G halo,
    // 2 the others); mode: 0 prep + micro, 1 prep only, 2 micro only
    // event marks: plain records, or external record nodes when capturing
    // (mm2d_time_kernels times the captured graph itself)
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (ev) CK(cudaStreamIsCapturing(s, &cap));
#define MARK(q) \
    if (ev) CK(cudaEventRecordWithFlags(ev[q], s, cap == cudaStreamCaptureStatusActive ? \
                                                       cudaEventRecordExternal : cudaEventRecordDefault))
    const Geometry& g = ctx->g;
    const mm2d_config& c = ctx->cfg;
    const long long ring = (long long)(g.bx + 2) * (g.by + 2);
    const bool gauss = c.nu != 0.0;
    // isotropy maxima for the eps < 1e-10 guard (micro2d.py:96)
    long long nl = 0;
    if (gauss && c.eps < 1e-10 && (phases & 1) && mode != 2) {
        // (reset by the call that runs k_prep, which rebuilds the maxima; a
        // micro-only call of a split step reads them)
        CK(cudaMemsetAsync(ctx->d_err + 1, 0, sizeof(unsigned long long) * 4, s));
    }
    ctx->last_dt = dt;
    ctx->last_Qout = Qout;
    ctx->last_s = s;
    if (phases & 1) {
    MARK(0);
    MARK(1);   // (the Q ring is filled by k_prep)
    PrepArgs pa;
    pa.g = g; pa.Q = Q; pa.Qr = ctx->d_Qr; pa.P = ctx->d_P; pa.err = ctx->d_err; pa.iso = ctx->d_err + 1;
    pa.dt = dt; pa.eps = c.eps; pa.nu = c.nu;
    {
        const double h1 = (c.v1_max - c.v1_min) / c.nv1, h2 = (c.v2_max - c.v2_min) / c.nv2;
        const double v10 = c.v1_min + 0.5 * h1, v11 = c.v1_min + 1.5 * h1;
        const double v20 = c.v2_min + 0.5 * h2, v21 = c.v2_min + 1.5 * h2;
        pa.dv = (v11 - v10) * (v21 - v20);
    }
    pa.tau_kind = c.tau_kind; pa.tau_value = c.tau_value;
    pa.step = 0;
    pa.gauss = gauss;
    pa.h2x = 0.5 / g.dx; pa.h2y = 0.5 / g.dy;
    if (mode != 2) {
#if MM2D_PREP_TILED
        {
            const int nt = ((g.bx + 2 + PT_I - 1) / PT_I) * ((g.by + 2 + PT_J - 1) / PT_J);
            CK(launch_pdl(k_prep_tiled, dim3(std::max(1, std::min(nt, ctx->sms * 8))),
                          dim3(PT_THREADS), kPrepStageBytes, s, pa));
        }
#else
        CK(launch_pdl(k_prep, dim3(grid_for(ring, 128)), dim3(128), 0, s, pa));
#endif
        ++nl;
    }
    MARK(2);
    MicroArgs ma;
    memset(&ma, 0, sizeof(ma));
    ma.g = g; ma.G = G; ma.Gout = Gout;
    ma.hxlo = ctx->d_gh[0]; ma.hxhi = ctx->d_gh[1]; ma.hylo = ctx->d_gh[2]; ma.hyhi = ctx->d_gh[3];
    ma.hys = (size_t)g.V;
    if (ctx->peer) {
        // the neighbours' G arrays in place (every block of a decomposition
        // has this block's shape): slot s of mm2d_halo_* order
        const size_t Vz = (size_t)g.V, col = (size_t)g.by * Vz;
        const double* const* nb = ctx->peerG;
        ma.hpeer = 1;
        ma.hys = col;
        ma.hxlo = nb[0] ? nb[0] + (size_t)(g.bx - 1) * col : nullptr;       // its last column
        ma.hxhi = nb[1];                                                     // its first column
        ma.hylo = nb[2] ? nb[2] + (size_t)(g.by - 1) * Vz - col : nullptr;   // its top row
        ma.hyhi = nb[3] ? nb[3] - col : nullptr;                             // its bottom row
        ma.hc[0] = nb[4] ? nb[4] + (size_t)(g.bx - 1) * col + (size_t)(g.by - 1) * Vz : nullptr;
        ma.hc[1] = nb[5] ? nb[5] + (size_t)(g.by - 1) * Vz : nullptr;
        ma.hc[2] = nb[6] ? nb[6] + (size_t)(g.bx - 1) * col : nullptr;
        ma.hc[3] = nb[7];
        for (int s8 = 0; s8 < 8; ++s8) ma.hnb[s8] = nb[s8];
    }
    ma.P = ctx->d_P; ma.Hr = ctx->d_Hr; ma.v1 = ctx->d_v1; ma.v2 = ctx->d_v2;
    ma.err = ctx->d_err; ma.iso = ctx->d_err + 1;
    ma.src_coeffs = sc; ma.src_shapes = ss; ma.nsrc = nsrc;
    ma.ly = ctx->ly; ma.gauss = gauss;
    ma.dt = dt; ma.eps = c.eps; ma.inveps = 1.0 / c.eps;
    ma.idx = 1.0 / g.dx; ma.idy = 1.0 / g.dy;
    ma.dv = pa.dv; ma.hfac = c.eps * pa.dv;
    ma.ikx = dt != 0.0 ? g.dx / dt : 0.0; ma.iky = dt != 0.0 ? g.dy / dt : 0.0;
    ma.ikx2 = ma.ikx * ma.ikx; ma.ryx = (g.dy / g.dx) * (g.dy / g.dx);
    ma.wall_ghat = ctx->d_wallg;
    ma.zero = ctx->d_zero;
    ma.part = part;
    if (mode == 1) {
        if (ctx->use32 && nsrc == 0 && ctx->d_wallg) {
            m32::launch_wall_ghat(ma, ctx->d_wallg, 2 * g.by + 2 * g.bx, s);
            ++nl;
        }
    } else if (ctx->use32 && nsrc == 0) {
        if (ctx->d_wallg && mode != 2) {
            m32::launch_wall_ghat(ma, ctx->d_wallg, 2 * g.by + 2 * g.bx, s);
            ++nl;
        }
        ma.ly = ctx->ly32;
        dim3 grid(g.bx, (g.by + ctx->ly32 - 1) / ctx->ly32);
        if (!ctx->bands32.empty()) {
            ma.nband = (int)ctx->bands32.size() - 1;
            for (int b = 0; b <= ma.nband; ++b) ma.band_j0[b] = ctx->bands32[b];
            grid.y = ma.nband;
        }
        m32::launch_micro32(ma, grid, s);
    } else {
        dim3 grid((g.bx + ctx->BX - 1) / ctx->BX, (g.by + ctx->ly - 1) / ctx->ly);
        void* args[] = {&ma};
        CK(cudaLaunchKernel(ctx->micro_fn, grid, dim3(ctx->NT), args, ctx->smem, s));
    }
    MARK(3);
    if (mode != 1) nl += 1;
    }   // phase 0: prep (with the Q ring), micro
    if (phases & 2) {
    MARK(4);   // (heat ghosts are resolved inside the sweeps)
    MacroArgs mc;
    mc.g = g; mc.Qr = ctx->d_Qr; mc.Hr = ctx->d_Hr; mc.Qx = ctx->d_Qx; mc.Qout = Qout;
    mc.qsrc = qsrc; mc.err = ctx->d_err; mc.dt = dt; mc.eps = c.eps; mc.nu = c.nu;
    mc.rx = dt / g.dx; mc.ry = dt / g.dy; mc.tau_kind = c.tau_kind; mc.tau_value = c.tau_value;
    mc.step = 0;
    mc.Hout = H;
    {
        const int jlo = g.qylo == GM_HALO ? -1 : 0, jhi = g.qyhi == GM_HALO ? g.by : g.by - 1;
        dim3 gx((g.bx + MX_TI - 1) / MX_TI, (jhi - jlo + 1 + MX_TJ - 1) / MX_TJ);
        CK(launch_pdl(k_macro_x, gx, dim3(MX_TJ, MX_TI + 2), 0, s, mc));
    }
    MARK(5);
    CK(launch_pdl(k_macro_y, dim3((g.by + MY_OUT - 1) / MY_OUT, (g.bx + 3) / 4), dim3(128), 0, s,
                  mc));
    MARK(6);
    nl += 2;
    MARK(7);   // (the SoA heat output is written by k_macro_y)
    }   // phase 1: macro sweeps
#undef MARK
    CK(cudaGetLastError());
    if (phases == 3) ctx->launches_per_step = nl;
    if (ctx->counting) g_launches += nl;
    return MM2D_OK;
}

extern "C" int mm2d_step_phase(mm2d_ctx* ctx, int phase, const double* d_Q, const double* d_G,
                               double dt, double* d_Qout, double* d_Gout, double* d_H, int nsrc,
                               const double* d_src_coeffs, const double* d_src_shapes,
                               const double* d_qsrc, void* stream) {
    if (!ctx || phase < 0 || phase > 5) return fail_cfg(ctx, "phase must be 0 to 5");
    CK(cudaSetDevice(ctx->dev));
    // phase 0 split around the G halo exchange: 2 = prep + the micro CTAs
    // that read no received halo, 3 = the CTAs that do; or finer, so the two
    // micro parts can run concurrently on two streams: 4 = prep only, 5 = the
    // interior micro CTAs only
    static const int part_of[6] = {0, 0, 1, 2, 0, 1};
    static const int mode_of[6] = {0, 0, 0, 2, 1, 2};
    return enqueue_step(ctx, d_Q, d_G, dt, d_Qout, d_Gout, d_H, nsrc, d_src_coeffs,
                        d_src_shapes, d_qsrc, (cudaStream_t)stream, nullptr,
                        phase == 1 ? 2 : 1, part_of[phase], mode_of[phase]);
}

extern "C" int mm2d_step(mm2d_ctx* ctx, const double* d_Q, const double* d_G, double dt,
                         double* d_Qout, double* d_Gout, double* d_H, int nsrc,
                         const double* d_src_coeffs, const double* d_src_shapes,
                         const double* d_qsrc, void* stream) {
    if (!ctx) return MM2D_ERR_CONFIG;
    CK(cudaSetDevice(ctx->dev));
    cudaStream_t s = (cudaStream_t)stream;   // 0 = the legacy default stream
    return enqueue_step(ctx, d_Q, d_G, dt, d_Qout, d_Gout, d_H, nsrc, d_src_coeffs,
                        d_src_shapes, d_qsrc, s);
}

static void drop_graphs(mm2d_ctx* ctx) {
    for (int p = 0; p < 2; ++p)
        if (ctx->gexec[p]) { cudaGraphExecDestroy(ctx->gexec[p]); ctx->gexec[p] = nullptr; }
}

extern "C" int mm2d_alloc_state(mm2d_ctx* ctx) {
    if (!ctx) return MM2D_ERR_CONFIG;
    CK(cudaSetDevice(ctx->dev));
    if (!ctx->state_owned) {
        drop_graphs(ctx);
        for (int p = 0; p < 2; ++p) ctx->d_Qs[p] = ctx->d_Gs[p] = nullptr;
        ctx->d_Hsoa = nullptr;
        ctx->state_owned = true;
    }
    const size_t cells = (size_t)ctx->g.bx * ctx->g.by;
    for (int p = 0; p < 2; ++p) {
        if (!ctx->d_Qs[p]) CK(cudaMalloc(&ctx->d_Qs[p], sizeof(double) * 6 * cells));
        if (!ctx->d_Gs[p]) CK(cudaMalloc(&ctx->d_Gs[p], sizeof(double) * cells * ctx->g.V));
    }
    if (!ctx->d_Hsoa) CK(cudaMalloc(&ctx->d_Hsoa, sizeof(double) * 4 * cells));
    ctx->cur = 0;
    return MM2D_OK;
}

extern "C" int mm2d_attach_state(mm2d_ctx* ctx, double* d_Qa, double* d_Ga, double* d_Qb,
                                 double* d_Gb, double* d_H) {
    if (!ctx || !d_Qa || !d_Ga || !d_Qb || !d_Gb) return fail_cfg(ctx, "attach needs 4 buffers");
    CK(cudaSetDevice(ctx->dev));
    if (ctx->state_owned) {
        for (int p = 0; p < 2; ++p) { cudaFree(ctx->d_Qs[p]); cudaFree(ctx->d_Gs[p]); }
        cudaFree(ctx->d_Hsoa);
        ctx->state_owned = false;
    }
    const bool same = ctx->d_Qs[0] == d_Qa && ctx->d_Gs[0] == d_Ga && ctx->d_Qs[1] == d_Qb &&
                      ctx->d_Gs[1] == d_Gb && ctx->d_Hsoa == d_H;
    if (!same) drop_graphs(ctx);
    ctx->d_Qs[0] = d_Qa; ctx->d_Gs[0] = d_Ga; ctx->d_Qs[1] = d_Qb; ctx->d_Gs[1] = d_Gb;
    ctx->d_Hsoa = d_H;
    ctx->cur = 0;
    return MM2D_OK;
}

extern "C" int mm2d_current_index(mm2d_ctx* ctx) { return ctx ? ctx->cur : -1; }

extern "C" int mm2d_set_stream(mm2d_ctx* ctx, void* stream) {
    if (!ctx) return MM2D_ERR_CONFIG;
    CK(cudaSetDevice(ctx->dev));
    ctx->user_stream = (cudaStream_t)stream;
    ctx->have_user_stream = true;
    if (!ctx->ev_in) CK(cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming));
    if (!ctx->ev_out) CK(cudaEventCreateWithFlags(&ctx->ev_out, cudaEventDisableTiming));
    return MM2D_OK;
}

extern "C" int mm2d_upload(mm2d_ctx* ctx, const double* h_Q, const double* h_G) {
    if (!ctx) return MM2D_ERR_CONFIG;
    int r = mm2d_alloc_state(ctx);
    if (r) return r;
    const size_t cells = (size_t)ctx->g.bx * ctx->g.by;
    CK(cudaMemcpyAsync(ctx->d_Qs[ctx->cur], h_Q, sizeof(double) * 6 * cells,
                       cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->d_Gs[ctx->cur], h_G, sizeof(double) * cells * ctx->g.V,
                       cudaMemcpyHostToDevice, ctx->stream));
    return MM2D_OK;
}

extern "C" int mm2d_upload_device(mm2d_ctx* ctx, const double* d_Q, const double* d_G) {
    if (!ctx) return MM2D_ERR_CONFIG;
    int r = mm2d_alloc_state(ctx);
    if (r) return r;
    const size_t cells = (size_t)ctx->g.bx * ctx->g.by;
    CK(cudaMemcpyAsync(ctx->d_Qs[ctx->cur], d_Q, sizeof(double) * 6 * cells,
                       cudaMemcpyDeviceToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->d_Gs[ctx->cur], d_G, sizeof(double) * cells * ctx->g.V,
                       cudaMemcpyDeviceToDevice, ctx->stream));
    return MM2D_OK;
}

extern "C" int mm2d_run(mm2d_ctx* ctx, double dt, int nsteps) {
    if (!ctx || !ctx->d_Qs[0]) return fail_cfg(ctx, "mm2d_run needs context-owned state");
    CK(cudaSetDevice(ctx->dev));
    if (ctx->graph_dt != dt || !ctx->gexec[0]) {
        drop_graphs(ctx);
        for (int p = 0; p < 2; ++p) {
            cudaGraph_t graph;
            CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
            ctx->counting = false;
            int r = enqueue_step(ctx, ctx->d_Qs[p], ctx->d_Gs[p], dt, ctx->d_Qs[1 - p],
                                 ctx->d_Gs[1 - p], ctx->d_Hsoa, 0, nullptr, nullptr, nullptr,
                                 ctx->stream);
            ctx->counting = true;
            cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
            if (r) return r;
            CK(e);
            CK(cudaGraphInstantiate(&ctx->gexec[p], graph, 0));
            cudaGraphDestroy(graph);
        }
        ctx->graph_dt = dt;
    }
    if (ctx->have_user_stream) {
        CK(cudaEventRecord(ctx->ev_in, ctx->user_stream));
        CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_in, 0));
    }
    for (int n = 0; n < nsteps; ++n) {
        CK(cudaGraphLaunch(ctx->gexec[ctx->cur], ctx->stream));
        ctx->last_s = ctx->stream;
        ctx->cur ^= 1;
        g_launches += ctx->launches_per_step;
    }
    if (ctx->have_user_stream) {
        CK(cudaEventRecord(ctx->ev_out, ctx->stream));
        CK(cudaStreamWaitEvent(ctx->user_stream, ctx->ev_out, 0));
    }
    return MM2D_OK;
}

extern "C" int mm2d_time_kernels(mm2d_ctx* ctx, double dt, int nrep, double* ms) {
    if (!ctx || !ctx->d_Qs[0] || !ms || nrep < 1) return fail_cfg(ctx, "time_kernels needs state");
    CK(cudaSetDevice(ctx->dev));
    std::vector<cudaEvent_t> ev((size_t)8 * nrep, nullptr);
    for (auto& e : ev) CK(cudaEventCreate(&e));
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    ctx->counting = false;
    int cur = ctx->cur, rc = MM2D_OK;
    for (int r = 0; r < nrep && rc == MM2D_OK; ++r, cur ^= 1)
        rc = enqueue_step(ctx, ctx->d_Qs[cur], ctx->d_Gs[cur], dt, ctx->d_Qs[1 - cur],
                          ctx->d_Gs[1 - cur], ctx->d_Hsoa, 0, nullptr, nullptr, nullptr,
                          ctx->stream, &ev[(size_t)8 * r]);
    ctx->counting = true;
    cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
    if (rc) return rc;
    CK(e);
    CK(cudaGraphInstantiate(&exec, graph, 0));
    cudaGraphDestroy(graph);
    if (ctx->have_user_stream) {
        CK(cudaEventRecord(ctx->ev_in, ctx->user_stream));
        CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_in, 0));
    }
    CK(cudaGraphLaunch(exec, ctx->stream));
    ctx->last_s = ctx->stream;
    ctx->cur = cur;
    CK(cudaStreamSynchronize(ctx->stream));
    cudaGraphExecDestroy(exec);
    for (int r = 0; r < nrep; ++r)
        for (int q = 0; q < 7; ++q) {
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, ev[(size_t)8 * r + q], ev[(size_t)8 * r + q + 1]));
            acc[q] += t;
        }
    for (int q = 0; q < 7; ++q) ms[q] = acc[q] / nrep;
    for (auto& x : ev) cudaEventDestroy(x);
    return MM2D_OK;
}

extern "C" int mm2d_download(mm2d_ctx* ctx, double* h_Q, double* h_G, double* h_H) {
    if (!ctx || !ctx->d_Qs[0]) return fail_cfg(ctx, "no context-owned state");
    CK(cudaSetDevice(ctx->dev));
    const size_t cells = (size_t)ctx->g.bx * ctx->g.by;
    if (h_Q)
        CK(cudaMemcpyAsync(h_Q, ctx->d_Qs[ctx->cur], sizeof(double) * 6 * cells,
                           cudaMemcpyDeviceToHost, ctx->stream));
    if (h_G)
        CK(cudaMemcpyAsync(h_G, ctx->d_Gs[ctx->cur], sizeof(double) * cells * ctx->g.V,
                           cudaMemcpyDeviceToHost, ctx->stream));
    if (h_H)
        CK(cudaMemcpyAsync(h_H, ctx->d_Hsoa, sizeof(double) * 4 * cells, cudaMemcpyDeviceToHost,
                           ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return MM2D_OK;
}

extern "C" int mm2d_state_ptrs(mm2d_ctx* ctx, double** d_Q, double** d_G, double** d_H) {
    if (!ctx || !ctx->d_Qs[0]) return fail_cfg(ctx, "no context-owned state");
    if (d_Q) *d_Q = ctx->d_Qs[ctx->cur];
    if (d_G) *d_G = ctx->d_Gs[ctx->cur];
    if (d_H) *d_H = ctx->d_Hsoa;
    return MM2D_OK;
}

// frame-style heat tensor: u from the given Q (cases.py:167-176)
__global__ void k_heat_frame(Geometry g, const double* G, const double* Q, const double* v1,
                             const double* v2, double f, double* H) {
    __shared__ double sh[32];
    const size_t c = blockIdx.x, V = (size_t)g.V;
    const double rho = Q[6 * c], u1 = Q[6 * c + 1] / rho, u2 = Q[6 * c + 2] / rho;
    double s[4] = {0, 0, 0, 0};
    for (int n = threadIdx.x; n < (int)V; n += blockDim.x) {
        const int k = n / g.nv2, l = n % g.nv2;
        const double w1 = v1[k] - u1, w2 = v2[l] - u2, gg = G[c * V + n];
        s[0] += w1 * w1 * w1 * gg; s[1] += w1 * w1 * w2 * gg;
        s[2] += w1 * w2 * w2 * gg; s[3] += w2 * w2 * w2 * gg;
    }
    const size_t S = (size_t)g.bx * g.by;
    for (int q = 0; q < 4; ++q) {
        const double t = block_sum(s[q], sh);
        if (threadIdx.x == 0) H[q * S + c] = f * t;
    }
}

extern "C" int mm2d_heat_tensor(mm2d_ctx* ctx, const double* d_G, const double* d_Q,
                                double* d_H, void* stream) {
    if (!ctx) return MM2D_ERR_CONFIG;
    CK(cudaSetDevice(ctx->dev));
    cudaStream_t s = (cudaStream_t)stream;   // 0 = the legacy default stream
    const mm2d_config& c = ctx->cfg;
    const double h1 = (c.v1_max - c.v1_min) / c.nv1, h2 = (c.v2_max - c.v2_min) / c.nv2;
    const double dv = ((c.v1_min + 1.5 * h1) - (c.v1_min + 0.5 * h1)) *
                      ((c.v2_min + 1.5 * h2) - (c.v2_min + 0.5 * h2));
    k_heat_frame<<<ctx->g.bx * ctx->g.by, 256, 0, s>>>(ctx->g, d_G, d_Q, ctx->d_v1, ctx->d_v2,
                                                       c.eps * dv, d_H);
    CK(cudaGetLastError());
    g_launches += 1;
    return MM2D_OK;
}

// max |a - b| accumulated into *out (non-negative doubles order like their
// bit patterns, so an unsigned atomicMax is an exact max)
__global__ void k_max_abs_diff(const double* a, const double* b, long long n, double* out) {
    double m = 0.0;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x)
        m = fmax(m, fabs(a[t] - b[t]));
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0)
        atomic_max_pos(reinterpret_cast<unsigned long long*>(out), m);
}

extern "C" int mm2d_max_abs_diff(mm2d_ctx* ctx, const double* d_a, const double* d_b, long long n,
                                 double* d_max, void* stream) {
    if (!ctx || !d_a || !d_b || !d_max || n < 0) return fail_cfg(ctx, "max_abs_diff arguments");
    CK(cudaSetDevice(ctx->dev));
    if (n == 0) return MM2D_OK;
    k_max_abs_diff<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(d_a, d_b, n, d_max);
    CK(cudaGetLastError());
    g_launches += 1;
    return MM2D_OK;
}

extern "C" int mm2d_sync(mm2d_ctx* ctx) {
    if (!ctx) return MM2D_ERR_CONFIG;
    CK(cudaSetDevice(ctx->dev));
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaDeviceSynchronize());
    return MM2D_OK;
}

// value of the failing check, recomputed from the preserved stage input
__global__ void k_err_value(Geometry g, int stage, int i, int j, const double* Qr,
                            const double* Qx, const double* Qout, double nu, int tau_kind, double tau_value,
                            double dt, double eps, double* out) {
    double q[6];
    const double* src = (stage <= ES_MOD_SPD) ? Qr + 6 * ring_index(g, i, j)
                        : (stage >= ES_RL_RHO) ? Qout + 6 * ((size_t)i * g.by + j)
                                               : Qx + 6 * ring_index(g, i, j);
    for (int m = 0; m < 6; ++m) q[m] = src[m];
    if (stage == ES_XS_RHO || stage == ES_XS_SPD) {
        MacroArgs a;
        a.dt = dt; a.eps = eps; a.nu = nu; a.tau_kind = tau_kind; a.tau_value = tau_value;
        double o[6];
        relax_cell(a, q, o);
        for (int m = 0; m < 6; ++m) q[m] = o[m];
    }
    double rho, u1, u2, t11, t12, t22;
    rho = q[0];
    if (stage == ES_PRIM_RHO || stage == ES_XS_RHO || stage == ES_YS_RHO || stage == ES_RL_RHO) {
        *out = rho;
        return;
    }
    prims_of(q, rho, u1, u2, t11, t12, t22);
    if (stage == ES_MOD_SPD) {
        const double T = 0.5 * (t11 + t22);
        const double m11 = (1.0 - nu) * T + nu * t11, m12 = nu * t12, m22 = (1.0 - nu) * T + nu * t22;
        *out = m11 * m22 - m12 * m12;
        return;
    }
    *out = t11 * t22 - t12 * t12;
}

extern "C" int mm2d_check(mm2d_ctx* ctx, int* kind, int* i, int* j, double* value) {
    if (!ctx) return MM2D_ERR_CONFIG;
    CK(cudaSetDevice(ctx->dev));
    // stream-scoped: wait for the context's last step only, not the device
    cudaStream_t s = ctx->last_s;
    unsigned long long* h = ctx->h_err;
    CK(cudaMemcpyAsync(h, ctx->d_err, sizeof(unsigned long long) * EW_N, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    unsigned long long key = h[EW_E];
    for (int w : {EW_PREP, EW_MX, EW_MY}) key = h[w] < key ? h[w] : key;
    if (key == kNoError) return MM2D_OK;
    const int stage = (int)((key >> 36) & 0xf);
    const unsigned long long cell = key & ((1ull << 36) - 1);
    const int gi = (int)(cell / ctx->g.ny), gj = (int)(cell % ctx->g.ny);
    const int li = gi - ctx->g.i0, lj = gj - ctx->g.j0;
    int k = MM2D_STATE_PRESSURE;
    if (stage == ES_PRIM_RHO || stage == ES_XS_RHO || stage == ES_YS_RHO || stage == ES_RL_RHO)
        k = MM2D_STATE_DENSITY;
    else if (stage == ES_MOD_SPD)
        k = MM2D_STATE_MODIFIED;
    double* d_v = reinterpret_cast<double*>(ctx->d_err + EW_N);
    const mm2d_config& c = ctx->cfg;
    k_err_value<<<1, 1, 0, s>>>(ctx->g, stage, li, lj, ctx->d_Qr, ctx->d_Qx, ctx->last_Qout, c.nu,
                                c.tau_kind, c.tau_value, ctx->last_dt, c.eps, d_v);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h + EW_N, d_v, sizeof(double), cudaMemcpyDeviceToHost, s));
    // report once: the next step starts from clean error words (the
    // reference raises per call); kNoError is all-ones bytes
    CK(cudaMemsetAsync(ctx->d_err + EW_E, 0xff, sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(ctx->d_err + EW_PREP, 0xff, sizeof(unsigned long long) * 3, s));
    CK(cudaStreamSynchronize(s));
    double v;
    memcpy(&v, h + EW_N, sizeof(double));
    if (kind) *kind = k;
    if (i) *i = gi;
    if (j) *j = gj;
    if (value) *value = v;
    char buf[160];
    snprintf(buf, sizeof buf, "invalid state (stage %d) at cell (%d, %d)", stage, gi, gj);
    ctx->err = buf;
    return MM2D_ERR_STATE;
}

// ---------------------------------------------------------------------------
// halo exchange staging (block decomposition, parallel.py:109-150)
// slots: 0 L, 1 R, 2 B, 3 T, 4 BL, 5 BR, 6 TL, 7 TR.  Send slot s carries
// this block's edge cells towards neighbour s, which receives them as its
// ghost cells of slot opposite(s).
// ---------------------------------------------------------------------------
static const int kOpp[8] = {1, 0, 3, 2, 7, 6, 5, 4};

static bool slot_active(const Geometry& g, int s) {
    const bool L = g.xlo == GM_HALO, R = g.xhi == GM_HALO, B = g.ylo == GM_HALO, T = g.yhi == GM_HALO;
    switch (s) {
        case 0: return L; case 1: return R; case 2: return B; case 3: return T;
        case 4: return L && B; case 5: return R && B; case 6: return L && T; default: return R && T;
    }
}
static int slot_cells(const Geometry& g, int s) { return s < 2 ? g.by : s < 4 ? g.bx : 1; }
static int field_width(const Geometry& g, int f) { return f == 0 ? g.V : f == 1 ? 6 : 4; }

// edge cell (send) and ghost cell (receive) of slot s, element e
__host__ __device__ inline void slot_cell(const Geometry& g, int s, int e, bool ghost, int& i, int& j) {
    switch (s) {
        case 0: i = ghost ? -1 : 0; j = e; break;
        case 1: i = ghost ? g.bx : g.bx - 1; j = e; break;
        case 2: i = e; j = ghost ? -1 : 0; break;
        case 3: i = e; j = ghost ? g.by : g.by - 1; break;
        case 4: i = ghost ? -1 : 0; j = ghost ? -1 : 0; break;
        case 5: i = ghost ? g.bx : g.bx - 1; j = ghost ? -1 : 0; break;
        case 6: i = ghost ? -1 : 0; j = ghost ? g.by : g.by - 1; break;
        default: i = ghost ? g.bx : g.bx - 1; j = ghost ? g.by : g.by - 1; break;
    }
}

struct HaloDesc {
    double* buf[8];      // staging (send) or receive buffers per slot
    int cells[8];        // 0 when inactive
    int width;           // doubles per cell
};

// pack edge cells of a block-layout field (G: V doubles per cell, Q: 6) or
// of the heat ring (H: from Hr) into the send buffers
__global__ void k_halo_pack(Geometry g, int field, const double* __restrict__ src,
                            const double* __restrict__ Hr, HaloDesc d) {
    const int w = d.width;
    for (int s = 0; s < 8; ++s) {
        if (!d.cells[s]) continue;
        const long long n = (long long)d.cells[s] * w;
        for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
             t += (long long)gridDim.x * blockDim.x) {
            const int e = (int)(t / w), c = (int)(t % w);
            int i, j;
            slot_cell(g, s, e, false, i, j);
            d.buf[s][t] = field == 2 ? Hr[4 * ring_index(g, i, j) + c]
                                     : src[((size_t)i * g.by + j) * w + c];
        }
    }
}

// scatter received Q / H ghosts into their ring
__global__ void k_halo_unpack(Geometry g, double* __restrict__ ringbuf, HaloDesc d) {
    const int w = d.width;
    for (int s = 0; s < 8; ++s) {
        if (!d.cells[s]) continue;
        const long long n = (long long)d.cells[s] * w;
        for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
             t += (long long)gridDim.x * blockDim.x) {
            const int e = (int)(t / w), c = (int)(t % w);
            int i, j;
            slot_cell(g, s, e, true, i, j);
            ringbuf[w * ring_index(g, i, j) + c] = d.buf[s][t];
        }
    }
}

static int ensure_halo(mm2d_ctx* ctx) {
    if (ctx->halo_ready) return MM2D_OK;
    const Geometry& g = ctx->g;
    const size_t V = (size_t)g.V;
    for (int f = 0; f < 3; ++f)
        for (int s = 0; s < 8; ++s) {
            const int n = slot_active(g, s) ? slot_cells(g, s) : 0;
            ctx->halo_cells[s] = n;
            const size_t cnt = (size_t)n * field_width(g, f);
            ctx->hsend[f][s] = nullptr;
            ctx->hrecv[f][s] = nullptr;
            if (!n) continue;
            CK(cudaMalloc(&ctx->hsend[f][s], sizeof(double) * cnt));
            if (f == 0) {
                // G arrives directly in the micro kernel's halo buffers
                double* base = nullptr;
                switch (s) {
                    case 0: base = ctx->d_gh[0]; break;
                    case 1: base = ctx->d_gh[1]; break;
                    case 2: base = ctx->d_gh[2] + V; break;
                    case 3: base = ctx->d_gh[3] + V; break;
                    case 4: base = ctx->d_gh[2]; break;
                    case 5: base = ctx->d_gh[2] + (size_t)(g.bx + 1) * V; break;
                    case 6: base = ctx->d_gh[3]; break;
                    default: base = ctx->d_gh[3] + (size_t)(g.bx + 1) * V; break;
                }
                ctx->hrecv[f][s] = base;
            } else {
                CK(cudaMalloc(&ctx->hrecv[f][s], sizeof(double) * cnt));
            }
        }
    ctx->halo_ready = true;
    return MM2D_OK;
}

extern "C" int mm2d_halo_info(mm2d_ctx* ctx, int which, int slot, double** d_send,
                              double** d_recv, long long* count) {
    if (!ctx || which < 0 || which > 2 || slot < 0 || slot > 7) return fail_cfg(ctx, "bad halo slot");
    CK(cudaSetDevice(ctx->dev));
    int r = ensure_halo(ctx);
    if (r) return r;
    const int n = ctx->halo_cells[slot];
    if (d_send) *d_send = ctx->hsend[which][slot];
    if (d_recv) *d_recv = ctx->hrecv[which][slot];
    if (count) *count = (long long)n * field_width(ctx->g, which);
    return MM2D_OK;
}

static HaloDesc halo_desc(mm2d_ctx* ctx, int which, bool send) {
    HaloDesc d;
    for (int s = 0; s < 8; ++s) {
        d.buf[s] = send ? ctx->hsend[which][s] : ctx->hrecv[which][s];
        d.cells[s] = ctx->halo_cells[s];
    }
    d.width = field_width(ctx->g, which);
    return d;
}

extern "C" int mm2d_halo_peer(mm2d_ctx* ctx, const double* const* d_nbG) {
    if (!ctx) return MM2D_ERR_CONFIG;
    if (!d_nbG) {
        ctx->peer = false;
        return MM2D_OK;
    }
    const Geometry& g = ctx->g;
    for (int s = 0; s < 8; ++s) {
        ctx->peerG[s] = d_nbG[s];
        if (slot_active(g, s) && !d_nbG[s]) return fail_cfg(ctx, "mm2d_halo_peer: active slot without a neighbour array");
    }
    ctx->peer = true;
    return MM2D_OK;
}

extern "C" int mm2d_enable_peer_access(int device, int peer_device) {
    if (device == peer_device) return MM2D_OK;
    int can = 0;
    if (cudaDeviceCanAccessPeer(&can, device, peer_device) != cudaSuccess || !can)
        return MM2D_ERR_CONFIG;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
    cudaSetDevice(cur);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return MM2D_OK;
    }
    return e == cudaSuccess ? MM2D_OK : MM2D_ERR_INTERNAL;
}

// Device arrays another process can map (one process per GPU): plain
// cudaMalloc allocations with their CUDA-IPC handle (64 bytes).
extern "C" int mm2d_ipc_alloc(long long bytes, void** d_ptr, unsigned char* handle64) {
    if (!d_ptr || !handle64 || bytes <= 0) return MM2D_ERR_CONFIG;
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    void* p = nullptr;
    if (cudaMalloc(&p, (size_t)bytes) != cudaSuccess) return MM2D_ERR_INTERNAL;
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, p) != cudaSuccess) {
        cudaFree(p);
        return MM2D_ERR_INTERNAL;
    }
    memcpy(handle64, &h, 64);
    *d_ptr = p;
    return MM2D_OK;
}

extern "C" int mm2d_ipc_open(const unsigned char* handle64, void** d_ptr) {
    if (!d_ptr || !handle64) return MM2D_ERR_CONFIG;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        return MM2D_ERR_INTERNAL;
    }
    *d_ptr = p;
    return MM2D_OK;
}

extern "C" int mm2d_ipc_close(void* d_ptr) {
    return cudaIpcCloseMemHandle(d_ptr) == cudaSuccess ? MM2D_OK : MM2D_ERR_INTERNAL;
}

extern "C" int mm2d_ipc_free(void* d_ptr) {
    return cudaFree(d_ptr) == cudaSuccess ? MM2D_OK : MM2D_ERR_INTERNAL;
}

extern "C" int mm2d_halo_pack(mm2d_ctx* ctx, int which, const double* d_src, void* stream) {
    if (!ctx || which < 0 || which > 2) return fail_cfg(ctx, "bad halo field");
    CK(cudaSetDevice(ctx->dev));
    int r = ensure_halo(ctx);
    if (r) return r;
    const HaloDesc d = halo_desc(ctx, which, true);
    long long tot = 0;
    for (int s = 0; s < 8; ++s) tot += (long long)d.cells[s] * d.width;
    if (!tot) return MM2D_OK;
    k_halo_pack<<<grid_for(tot / 4 + 1, 256), 256, 0, (cudaStream_t)stream>>>(
        ctx->g, which, d_src, ctx->d_Hr, d);
    CK(cudaGetLastError());
    g_launches += 1;
    return MM2D_OK;
}

extern "C" int mm2d_halo_unpack(mm2d_ctx* ctx, int which, void* stream) {
    if (!ctx || which < 0 || which > 2) return fail_cfg(ctx, "bad halo field");
    CK(cudaSetDevice(ctx->dev));
    int r = ensure_halo(ctx);
    if (r) return r;
    if (which == 0) return MM2D_OK;   // G is received in place
    const HaloDesc d = halo_desc(ctx, which, false);
    long long tot = 0;
    for (int s = 0; s < 8; ++s) tot += (long long)d.cells[s] * d.width;
    if (!tot) return MM2D_OK;
    k_halo_unpack<<<grid_for(tot, 256), 256, 0, (cudaStream_t)stream>>>(
        ctx->g, which == 1 ? ctx->d_Qr : ctx->d_Hr, d);
    CK(cudaGetLastError());
    g_launches += 1;
    return MM2D_OK;
}

// ---------------------------------------------------------------------------
// the ten kernel-contract entry points
// ---------------------------------------------------------------------------
#define KCK()                                                         \
    do {                                                              \
        cudaError_t e_ = cudaGetLastError();                          \
        if (e_ != cudaSuccess) return MM2D_ERR_INTERNAL;              \
        g_launches += 1;                                              \
        return MM2D_OK;                                               \
    } while (0)

static int nblk(size_t n) { return (int)std::min<size_t>((n + 255) / 256, 148 * 64); }

extern "C" int mm2d_k_maxwellian_field_2d(int nx, int ny, int nv1, int nv2, const double* rho,
                                          const double* u1, const double* u2, const double* T,
                                          const double* v1, const double* v2, double* M,
                                          void* stream) {
    kc_maxwellian<<<nblk((size_t)nx * ny * nv1 * nv2), 256, 0, (cudaStream_t)stream>>>(
        nx * ny, nv1, nv2, rho, u1, u2, T, v1, v2, M);
    KCK();
}

extern "C" int mm2d_k_project_field_2d(int nx, int ny, int nv1, int nv2, const double* F,
                                       const double* M, const double* rho, const double* u1,
                                       const double* u2, const double* T, const double* v1,
                                       const double* v2, double dv, double* out, void* stream) {
    kc_project<<<nx * ny, 128, 0, (cudaStream_t)stream>>>(nv1, nv2, F, M, rho, u1, u2, T, v1, v2,
                                                          dv, out);
    KCK();
}

extern "C" int mm2d_k_transport_stage_2d(int nx, int ny, int nv1, int nv2, const double* G_ext,
                                         const double* M, const double* rho, const double* u1,
                                         const double* u2, const double* T, const double* v1,
                                         const double* v2, double d, double dt, int axis,
                                         double* out, void* stream) {
    kc_transport<<<nx * ny, 128, 0, (cudaStream_t)stream>>>(nx, ny, nv1, nv2, G_ext, M, rho, u1,
                                                            u2, T, v1, v2, d, dt, axis, out);
    KCK();
}

extern "C" int mm2d_k_ghat_2d(int nx, int ny, int nv1, int nv2, const double* M, const double* rho,
                              const double* u1, const double* u2, const double* T,
                              const double* s11, const double* s12, const double* gT1,
                              const double* gT2, const double* tau, const double* v1,
                              const double* v2, double* out, void* stream) {
    (void)rho;
    kc_ghat<<<nblk((size_t)nx * ny * nv1 * nv2), 256, 0, (cudaStream_t)stream>>>(
        nx * ny, nv1, nv2, M, u1, u2, T, s11, s12, gT1, gT2, tau, v1, v2, out);
    KCK();
}

extern "C" int mm2d_k_add_gaussian_term_2d(int nx, int ny, int nv1, int nv2, double* Ghat,
                                           const double* M, const double* rho, const double* u1,
                                           const double* u2, const double* m11, const double* m12,
                                           const double* m22, double eps, const double* v1,
                                           const double* v2, void* stream) {
    kc_gauss<<<nblk((size_t)nx * ny * nv1 * nv2), 256, 0, (cudaStream_t)stream>>>(
        nx * ny, nv1, nv2, Ghat, M, rho, u1, u2, m11, m12, m22, eps, v1, v2);
    KCK();
}

extern "C" int mm2d_k_add_lowrank_4d(int nx, int ny, int nv1, int nv2, double* out, int nterms,
                                     const double* coeffs, const double* shapes, void* stream) {
    kc_lowrank<<<nblk((size_t)nx * ny * nv1 * nv2), 256, 0, (cudaStream_t)stream>>>(
        nx * ny, nv1 * nv2, out, nterms, coeffs, shapes);
    KCK();
}

extern "C" int mm2d_k_relax_2d(int nx, int ny, int nv1, int nv2, const double* G,
                               const double* Ghat, const double* tau, double dt, double eps,
                               double* out, void* stream) {
    kc_relax<<<nblk((size_t)nx * ny * nv1 * nv2), 256, 0, (cudaStream_t)stream>>>(
        nx * ny, nv1 * nv2, G, Ghat, tau, dt, eps, out);
    KCK();
}

extern "C" int mm2d_k_heat_tensor_2d(int nx, int ny, int nv1, int nv2, const double* G,
                                     const double* u1, const double* u2, const double* v1,
                                     const double* v2, double dv, double eps, double* H,
                                     void* stream) {
    kc_heat<<<nx * ny, 128, 0, (cudaStream_t)stream>>>(nx * ny, nv1, nv2, G, u1, u2, v1, v2,
                                                       eps * dv, H);
    KCK();
}

extern "C" int mm2d_k_upwind_z_1d(int nx, int nv, const double* G_ext, const double* v, double dx,
                                  double* Z, void* stream) {
    kc_upwind1d<<<nblk((size_t)nx * nv), 256, 0, (cudaStream_t)stream>>>(nx, nv, G_ext, v, dx, Z);
    KCK();
}

extern "C" int mm2d_k_project_field_1d(int nx, int nv, const double* F, const double* M,
                                       const double* rho, const double* u, const double* T,
                                       const double* v, double dv, double* out, void* stream) {
    kc_project1d<<<nx, 64, 0, (cudaStream_t)stream>>>(nv, F, M, rho, u, T, v, dv, out);
    KCK();
}
