// C ABI of the 1D1V step (declared in include/mm1d.h), part of libmm2d.so.
// Owns the per-problem context: velocity tables, the sticky error word,
// context-owned state, the graph of the generic two-kernel step and the
// launch configuration of the cluster-resident run kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <string>

#include "mm1d.h"
#include "mm2d.h"
#include "mm1d.cuh"
#include "mm1d_resident.cuh"

using namespace mm2d;
using namespace mm2d::d1;

extern std::atomic<long long> g_launches;

struct mm1d_ctx {
    mm1d_config cfg;
    Geo1 g;
    int dev = 0;
    cudaStream_t stream = nullptr;
    double* d_v = nullptr;
    double* d_v3 = nullptr;
    unsigned long long* d_err = nullptr;   // [0] key, [1] failing Q pointer, [2] steps done
    double* d_Q[2] = {nullptr, nullptr};
    double* d_G[2] = {nullptr, nullptr};
    double* d_H = nullptr;
    int cur = 0;
    int threads = 64;
    // cluster-resident run
    bool resident = false;
    int cluster = 0, cpc = 0, rthreads = 32;
    const void* rfn = nullptr;
    size_t rsmem = 0;
    // graph of the generic step (parity 0: A->B, 1: B->A)
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    double graph_dt = 0.0;
    std::string err;
};

#define CK1(call)                                                                      \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess) {                                                       \
            if (ctx) ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);    \
            return MM2D_ERR_INTERNAL;                                                  \
        }                                                                              \
    } while (0)

static int fail1(mm1d_ctx* ctx, const std::string& m) {
    if (ctx) ctx->err = m;
    return MM2D_ERR_CONFIG;
}

template <int NJ>
static const void* resident_fn() {
    return reinterpret_cast<const void*>(&k1_resident<NJ>);
}

// choose the largest cluster (16, 8, ... CTAs) that can hold the state in
// shared memory and can be co-scheduled on this device
static void plan_resident(mm1d_ctx* ctx) {
    ctx->resident = false;
    if (std::getenv("MM1D_NO_RESIDENT")) return;
    const int nx = ctx->g.nx, nv = ctx->g.nv;
    const int nj = (nv + 31) / 32;
    const void* fn = nj <= 1 ? resident_fn<1>() : nj <= 2 ? resident_fn<2>()
                   : nj <= 4 ? resident_fn<4>() : nj <= 8 ? resident_fn<8>() : nullptr;
    if (!fn) return;
    cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int C = 16; C >= 1; C >>= 1) {
        if (C > nx && C > 1) continue;
        int cpc = 1;
        while (cpc * C < nx) cpc <<= 1;     // power of two: owner = cell >> log2(cpc)
        const size_t sm = res1_smem(cpc, nv);
        if (sm > 200 * 1024) return;   // larger clusters were tried first
        if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) !=
            cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        const int threads = 32 * std::min(cpc, 16);
        cudaLaunchConfig_t lc = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.gridDim = dim3(C);
        lc.blockDim = dim3(threads);
        lc.dynamicSmemBytes = sm;
        lc.attrs = at;
        lc.numAttrs = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, fn, &lc) != cudaSuccess || ncl < 1) {
            cudaGetLastError();
            continue;
        }
        ctx->resident = true;
        ctx->cluster = C;
        ctx->cpc = cpc;
        ctx->rsmem = sm;
        ctx->rthreads = threads;
        ctx->rfn = fn;
        return;
    }
}

extern "C" int mm1d_create(const mm1d_config* cfg, mm1d_ctx** out) {
    if (!cfg || !out) return MM2D_ERR_CONFIG;
    *out = nullptr;
    mm1d_ctx* ctx = new mm1d_ctx();
    ctx->cfg = *cfg;
    const mm1d_config& c = ctx->cfg;
    auto bad = [&](const char* m) {
        int r = fail1(ctx, m);
        delete ctx;
        return r;
    };
    if (c.nx < 1 || c.nv < 2) return bad("grid sizes must be nx >= 1 and nv >= 2");
    if (!(c.x_max > c.x_min) || !(c.v_max > c.v_min)) return bad("axes need max > min");
    for (int f = 0; f < 2; ++f) {
        if (c.face[f] < MM2D_FACE_PERIODIC || c.face[f] > MM2D_FACE_WALL)
            return bad("unknown face kind");
        if (c.face[f] == MM2D_FACE_WALL && !(c.wall_T[f] > 0.0))
            return bad("wall temperature must be positive");
    }
    if ((c.face[0] == MM2D_FACE_PERIODIC) != (c.face[1] == MM2D_FACE_PERIODIC))
        return bad("periodic faces must be paired");
    if (c.tau_kind < MM2D_TAU_HARD_SPHERE_1D || c.tau_kind > MM2D_TAU_CONSTANT)
        return bad("unknown collision model");
    ctx->dev = c.device;
    if (cudaSetDevice(ctx->dev) != cudaSuccess) return bad("cannot select the CUDA device");
    // the reference's cell_centers (mesh.py) and spacings, on the host in fp64
    const double hx = (c.x_max - c.x_min) / c.nx, hv = (c.v_max - c.v_min) / c.nv;
    double* v = new double[c.nv];
    double* v3 = new double[c.nv];
    for (int k = 0; k < c.nv; ++k) {
        v[k] = c.v_min + ((double)(k + 1) - 0.5) * hv;
        v3[k] = std::pow(v[k], 3.0);   // numpy's v ** 3 (macro1d.py:19)
    }
    Geo1& g = ctx->g;
    g.nx = c.nx; g.nv = c.nv;
    g.dx = hx;
    g.dv = v[1] - v[0];            // micro1d.py:49, macro1d.py:18
    g.face[0] = c.face[0]; g.face[1] = c.face[1];
    g.wallT[0] = c.wall_T[0]; g.wallT[1] = c.wall_T[1];
    g.tau_kind = c.tau_kind; g.tau_value = c.tau_value; g.eps = c.eps;
    int rc = MM2D_OK;
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&ctx->d_v, sizeof(double) * c.nv) != cudaSuccess ||
        cudaMalloc(&ctx->d_v3, sizeof(double) * c.nv) != cudaSuccess ||
        cudaMalloc(&ctx->d_err, sizeof(unsigned long long) * 4) != cudaSuccess ||
        cudaMemcpy(ctx->d_v, v, sizeof(double) * c.nv, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(ctx->d_v3, v3, sizeof(double) * c.nv, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemset(ctx->d_err, 0xff, sizeof(unsigned long long) * 4) != cudaSuccess)
        rc = MM2D_ERR_INTERNAL;
    delete[] v;
    delete[] v3;
    if (rc) {
        ctx->err = "CUDA allocation failed";
        cudaGetLastError();
        *out = ctx;
        return rc;
    }
    ctx->threads = std::min(256, ((c.nv + 31) / 32) * 32);
    plan_resident(ctx);
    *out = ctx;
    return MM2D_OK;
}

static void drop_graphs1(mm1d_ctx* ctx) {
    for (int p = 0; p < 2; ++p)
        if (ctx->gexec[p]) { cudaGraphExecDestroy(ctx->gexec[p]); ctx->gexec[p] = nullptr; }
}

extern "C" int mm1d_destroy(mm1d_ctx* ctx) {
    if (!ctx) return MM2D_OK;
    cudaSetDevice(ctx->dev);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    drop_graphs1(ctx);
    for (int p = 0; p < 2; ++p) { cudaFree(ctx->d_Q[p]); cudaFree(ctx->d_G[p]); }
    cudaFree(ctx->d_H);
    cudaFree(ctx->d_v);
    cudaFree(ctx->d_v3);
    cudaFree(ctx->d_err);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return MM2D_OK;
}

extern "C" const char* mm1d_last_error(mm1d_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

extern "C" int mm1d_resident(mm1d_ctx* ctx) { return ctx && ctx->resident ? 1 : 0; }

static int enqueue1(mm1d_ctx* ctx, const double* Q, const double* G, double dt, double* Qo,
                    double* Go, double* H, const double* src, const double* qsrc,
                    cudaStream_t s, bool count) {
    if (!Q || !G || !Qo || !Go || !H) return fail1(ctx, "mm1d_step needs Q, G, Q_out, G_out, H");
    Args1 a;
    a.g = ctx->g;
    a.Q = Q; a.G = G; a.Qout = Qo; a.Gout = Go; a.H = H;
    a.v = ctx->d_v; a.v3 = ctx->d_v3;
    a.src = src; a.qsrc = qsrc;
    a.err = ctx->d_err;
    a.dt = dt;
    k1_micro<<<ctx->g.nx, ctx->threads, 0, s>>>(a);
    const int nb = (ctx->g.nx + 127) / 128;
    k1_macro<<<nb, 128, 0, s>>>(a);
    CK1(cudaGetLastError());
    if (count) g_launches += 2;
    return MM2D_OK;
}

extern "C" int mm1d_step(mm1d_ctx* ctx, const double* d_Q, const double* d_G, double dt,
                         double* d_Qout, double* d_Gout, double* d_H, const double* d_src,
                         const double* d_qsrc, void* stream) {
    if (!ctx) return MM2D_ERR_CONFIG;
    CK1(cudaSetDevice(ctx->dev));
    return enqueue1(ctx, d_Q, d_G, dt, d_Qout, d_Gout, d_H, d_src, d_qsrc, (cudaStream_t)stream,
                    true);
}

static int alloc_state1(mm1d_ctx* ctx) {
    const size_t nx = ctx->g.nx, nv = ctx->g.nv;
    for (int p = 0; p < 2; ++p) {
        if (!ctx->d_Q[p]) CK1(cudaMalloc(&ctx->d_Q[p], sizeof(double) * 3 * nx));
        if (!ctx->d_G[p]) CK1(cudaMalloc(&ctx->d_G[p], sizeof(double) * nx * nv));
    }
    if (!ctx->d_H) {
        CK1(cudaMalloc(&ctx->d_H, sizeof(double) * nx));
        CK1(cudaMemsetAsync(ctx->d_H, 0, sizeof(double) * nx, ctx->stream));
    }
    return MM2D_OK;
}

extern "C" int mm1d_upload(mm1d_ctx* ctx, const double* h_Q, const double* h_G) {
    if (!ctx || !h_Q || !h_G) return fail1(ctx, "mm1d_upload needs Q and G");
    CK1(cudaSetDevice(ctx->dev));
    int r = alloc_state1(ctx);
    if (r) return r;
    ctx->cur = 0;
    const size_t nx = ctx->g.nx, nv = ctx->g.nv;
    CK1(cudaMemcpyAsync(ctx->d_Q[0], h_Q, sizeof(double) * 3 * nx, cudaMemcpyHostToDevice,
                        ctx->stream));
    CK1(cudaMemcpyAsync(ctx->d_G[0], h_G, sizeof(double) * nx * nv, cudaMemcpyHostToDevice,
                        ctx->stream));
    CK1(cudaStreamSynchronize(ctx->stream));
    return MM2D_OK;
}

extern "C" int mm1d_run(mm1d_ctx* ctx, double dt, int nsteps) {
    if (!ctx || !ctx->d_Q[0]) return fail1(ctx, "mm1d_run needs uploaded state");
    if (nsteps < 0) return fail1(ctx, "nsteps must be >= 0");
    if (nsteps == 0) return MM2D_OK;
    CK1(cudaSetDevice(ctx->dev));
    if (ctx->resident) {
        Res1 a;
        a.g = ctx->g;
        a.cpc = ctx->cpc;
        a.lg = 0;
        while ((1 << a.lg) < ctx->cpc) ++a.lg;
        a.Q = ctx->d_Q[ctx->cur];
        a.G = ctx->d_G[ctx->cur];
        a.H = ctx->d_H;
        a.v = ctx->d_v; a.v3 = ctx->d_v3;
        a.err = ctx->d_err;
        a.dt = dt;
        a.nsteps = nsteps;
        a.done = reinterpret_cast<int*>(ctx->d_err + 2);
        cudaLaunchConfig_t lc = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = ctx->cluster;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.gridDim = dim3(ctx->cluster);
        lc.blockDim = dim3(ctx->rthreads);
        lc.dynamicSmemBytes = ctx->rsmem;
        lc.stream = ctx->stream;
        lc.attrs = at;
        lc.numAttrs = 1;
        void* args[] = {&a};
        CK1(cudaLaunchKernelExC(&lc, ctx->rfn, args));
        g_launches += 1;
        return MM2D_OK;
    }
    if (ctx->graph_dt != dt || !ctx->gexec[0]) {
        drop_graphs1(ctx);
        for (int p = 0; p < 2; ++p) {
            cudaGraph_t graph;
            CK1(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
            int r = enqueue1(ctx, ctx->d_Q[p], ctx->d_G[p], dt, ctx->d_Q[1 - p], ctx->d_G[1 - p],
                             ctx->d_H, nullptr, nullptr, ctx->stream, false);
            cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
            if (r) return r;
            CK1(e);
            CK1(cudaGraphInstantiate(&ctx->gexec[p], graph, 0));
            cudaGraphDestroy(graph);
        }
        ctx->graph_dt = dt;
    }
    for (int n = 0; n < nsteps; ++n) {
        CK1(cudaGraphLaunch(ctx->gexec[ctx->cur], ctx->stream));
        ctx->cur ^= 1;
    }
    g_launches += 2LL * nsteps;
    return MM2D_OK;
}

extern "C" int mm1d_download(mm1d_ctx* ctx, double* h_Q, double* h_G, double* h_H) {
    if (!ctx || !ctx->d_Q[0]) return fail1(ctx, "no context-owned state");
    CK1(cudaSetDevice(ctx->dev));
    const size_t nx = ctx->g.nx, nv = ctx->g.nv;
    if (h_Q)
        CK1(cudaMemcpyAsync(h_Q, ctx->d_Q[ctx->cur], sizeof(double) * 3 * nx,
                            cudaMemcpyDeviceToHost, ctx->stream));
    if (h_G)
        CK1(cudaMemcpyAsync(h_G, ctx->d_G[ctx->cur], sizeof(double) * nx * nv,
                            cudaMemcpyDeviceToHost, ctx->stream));
    if (h_H)
        CK1(cudaMemcpyAsync(h_H, ctx->d_H, sizeof(double) * nx, cudaMemcpyDeviceToHost,
                            ctx->stream));
    CK1(cudaStreamSynchronize(ctx->stream));
    return MM2D_OK;
}

extern "C" int mm1d_check(mm1d_ctx* ctx, int* kind, int* i, double* value) {
    if (!ctx) return MM2D_ERR_CONFIG;
    CK1(cudaSetDevice(ctx->dev));
    CK1(cudaDeviceSynchronize());
    unsigned long long w[4];
    CK1(cudaMemcpy(w, ctx->d_err, sizeof(w), cudaMemcpyDeviceToHost));
    if (w[3] < w[0]) w[0] = w[3];
    if (w[0] == kNoError) return MM2D_OK;
    const int stage = (int)((w[0] >> 36) & 0xf);
    const int cell = (int)(w[0] & ((1ull << 36) - 1));
    double* d_v;
    double v = 0.0;
    CK1(cudaMalloc(&d_v, sizeof(double)));
    k1_err_value<<<1, 1>>>(reinterpret_cast<const double*>((size_t)w[1]), stage, cell, d_v);
    CK1(cudaMemcpy(&v, d_v, sizeof(double), cudaMemcpyDeviceToHost));
    cudaFree(d_v);
    CK1(cudaMemset(ctx->d_err, 0xff, sizeof(unsigned long long)));
    CK1(cudaMemset(ctx->d_err + 3, 0xff, sizeof(unsigned long long)));
    if (kind) *kind = stage == E1_DENSITY ? MM1D_STATE_DENSITY : MM1D_STATE_TEMPERATURE;
    if (i) *i = cell;
    if (value) *value = v;
    return MM2D_ERR_STATE;
}
