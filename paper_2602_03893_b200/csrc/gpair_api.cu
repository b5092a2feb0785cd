// gpair_api.cu -- the C ABI of include/gpair.h.
//
// Host logic only: argument validation, operator constants, kernel sequencing
// on the caller's stream, the NCCL all-reduce call site (kernel sharding,
// SURVEY 8e) and optional CUDA-event profiling.  All arithmetic of the
// method runs in the kernels of gpair_kernels.cu / gpair_setup.cu.
#include <dlfcn.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "gpair_ctx.h"

using gpair::EpiParams;

namespace {

thread_local std::string g_static_err;

// Table of the factorised-Gaussian fast path (gpair_internal.cuh TabConst):
// c_i = exp2(K m^2) and d_i = -m c_i, m = i - W/2, in fp64 with
// K = -log2(e) h^2 / (2 sigma^2), each rounded once to fp32.  A table error is
// SYSTEMATIC (the same at window position m for every pair) and dense
// amplitudes cancel strongly in y, so the entries are kept at full fp32
// precision (a 20-bit table measured 1e-3 elementwise at cfg4).  Enabled for
// full windows of W = cnt_int samples with W % 4 == 0 and TAB_MIN <= W <=
// TAB_MAX (the per-pair chain then spans |m| <= 16);
// GPAIR_NO_TAB=1 in the environment keeps the per-sample MUFU path, GPAIR_ADJ_NO_LCF=1 /
// GPAIR_ADJ_NO_T=1 skip the LCF / sensor-lane adjoints (A/B runs and the fallback tests).
void build_tab(gpair_ctx* c) {
    gpair::TabConst t{};
    const gpair::OpConst& k = c->k;
    const int W = k.cnt_int;
    auto env1 = [](const char* n) {
        const char* v = std::getenv(n);
        return v && v[0] == '1';
    };
    c->dbg = (env1("GPAIR_NO_TAB") ? gpair::DBG_NO_TAB : 0) | (env1("GPAIR_ADJ_NO_LCF") ? gpair::DBG_ADJ_NO_LCF : 0) |
             (env1("GPAIR_ADJ_NO_T") ? gpair::DBG_ADJ_NO_T : 0) | (env1("GPAIR_ADJ_NO_MP") ? gpair::DBG_ADJ_NO_MP : 0);
    t.on = (W >= gpair::TAB_MIN && W % 4 == 0 && W <= gpair::TAB_MAX && !k.gen && !(c->dbg & gpair::DBG_NO_TAB)) ? 1 : 0;
    t.K = k.K1u;
    t.m2K = -2.0f * k.K1u;
    t.kappa = (float)(-2.0 * (double)k.K1u * 0.6931471805599453);
    t.inv_h = (float)k.inv_h;
    if (t.on) {
        const int C = W / 2;
        const double Kd = -1.4426950408889634 * k.h * k.h / (2.0 * k.sigma * k.sigma);
        float cf[gpair::TAB_MAX], df[gpair::TAB_MAX];
        for (int i = 0; i < W; ++i) {
            const int m = i - C;
            const double cv = std::exp2(Kd * (double)m * (double)m);
            cf[i] = (float)cv;                 // each entry rounded once from fp64:
            df[i] = (float)(-(double)m * cv);  // the table's error is common to every pair
        }
        for (int i = 0; i < 11; ++i) {  // union-window Gaussian G_p = 2^{K (p - 11)^2}, p = 2i, 2i + 1
            const float g0 = (float)std::exp2(Kd * (2.0 * i - 11) * (2.0 * i - 11));
            const float g1 = (float)std::exp2(Kd * (2.0 * i - 10) * (2.0 * i - 10));
            t.g2[i] = ((gpair::f2_t)__builtin_bit_cast(uint32_t, g1) << 32) | __builtin_bit_cast(uint32_t, g0);
        }
        for (int i = 0; i < W; i += 2) {
            t.c2[i / 2] = ((gpair::f2_t)__builtin_bit_cast(uint32_t, cf[i + 1]) << 32) | __builtin_bit_cast(uint32_t, cf[i]);
            t.d2[i / 2] = ((gpair::f2_t)__builtin_bit_cast(uint32_t, df[i + 1]) << 32) | __builtin_bit_cast(uint32_t, df[i]);
        }
    }
    c->tab = t;
}

// ---------------------------------------------------------------- NCCL (dlopen)
typedef int nccl_res_t;
struct nccl_uid_t {
    char internal[128];
};
struct NcclApi {
    bool tried = false, ok = false;
    nccl_res_t (*GetUniqueId)(nccl_uid_t*) = nullptr;
    nccl_res_t (*CommInitRank)(void**, int, nccl_uid_t, int) = nullptr;
    nccl_res_t (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    nccl_res_t (*CommDestroy)(void*) = nullptr;
    const char* (*GetErrorString)(nccl_res_t) = nullptr;
    // point-to-point (VCR z-slab halo exchange, row f2)
    nccl_res_t (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    nccl_res_t (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    nccl_res_t (*GroupStart)() = nullptr;
    nccl_res_t (*GroupEnd)() = nullptr;
    nccl_res_t (*CommCount)(void*, int*) = nullptr;
    nccl_res_t (*CommUserRank)(void*, int*) = nullptr;
};
NcclApi g_nccl;
constexpr int NCCL_INT32 = 2, NCCL_FLOAT32 = 7, NCCL_FLOAT64 = 8, NCCL_SUM = 0;

bool nccl_load() {
    if (g_nccl.tried) return g_nccl.ok;
    g_nccl.tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return false;
    g_nccl.GetUniqueId = (nccl_res_t(*)(nccl_uid_t*))dlsym(h, "ncclGetUniqueId");
    g_nccl.CommInitRank = (nccl_res_t(*)(void**, int, nccl_uid_t, int))dlsym(h, "ncclCommInitRank");
    g_nccl.AllReduce = (nccl_res_t(*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(h, "ncclAllReduce");
    g_nccl.CommDestroy = (nccl_res_t(*)(void*))dlsym(h, "ncclCommDestroy");
    g_nccl.GetErrorString = (const char* (*)(nccl_res_t))dlsym(h, "ncclGetErrorString");
    g_nccl.Send = (nccl_res_t(*)(const void*, size_t, int, int, void*, cudaStream_t))dlsym(h, "ncclSend");
    g_nccl.Recv = (nccl_res_t(*)(void*, size_t, int, int, void*, cudaStream_t))dlsym(h, "ncclRecv");
    g_nccl.GroupStart = (nccl_res_t(*)())dlsym(h, "ncclGroupStart");
    g_nccl.GroupEnd = (nccl_res_t(*)())dlsym(h, "ncclGroupEnd");
    g_nccl.CommCount = (nccl_res_t(*)(void*, int*))dlsym(h, "ncclCommCount");
    g_nccl.CommUserRank = (nccl_res_t(*)(void*, int*))dlsym(h, "ncclCommUserRank");
    g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllReduce && g_nccl.CommDestroy && g_nccl.Send &&
                g_nccl.Recv && g_nccl.GroupStart && g_nccl.GroupEnd && g_nccl.CommCount && g_nccl.CommUserRank;
    return g_nccl.ok;
}

// ---------------------------------------------------------------- helpers
gpair_status fail(gpair_ctx* c, gpair_status s, const std::string& msg) {
    if (c)
        c->err = msg;
    else
        g_static_err = msg;
    return s;
}

gpair_status cuda_fail(gpair_ctx* c, cudaError_t e, const char* where) {
    std::string m = std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    return fail(c, GPAIR_ERR_CUDA, m);
}

#define API_CUDA(c, x, where)                              \
    do {                                                   \
        cudaError_t e_ = (x);                              \
        if (e_ != cudaSuccess) return cuda_fail(c, e_, where); \
    } while (0)

bool finite_pos(double x) { return std::isfinite(x) && x > 0.0; }

// Event-timed launch wrapper.
// NVTX ranges (domain "gpair", one per stage; header-only nvtx3, no-ops unless a
// tool such as nsys or ncu --nvtx is attached): they bracket the enqueue of each
// stage's kernels, so a timeline attributes every launch to its stage.
nvtxDomainHandle_t nvtx_domain() {
    static nvtxDomainHandle_t d = nvtxDomainCreateA("gpair");
    return d;
}
const char* const kStageName[GPAIR_PROF_N] = {"gather", "forward", "reduce", "allreduce",
                                              "residual", "adjoint", "loss", "vcr"};
struct NvtxRange {
    explicit NvtxRange(const char* name) {
        nvtxEventAttributes_t a{};
        a.version = NVTX_VERSION;
        a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
        a.messageType = NVTX_MESSAGE_TYPE_ASCII;
        a.message.ascii = name;
        nvtxDomainRangePushEx(nvtx_domain(), &a);
    }
    ~NvtxRange() { nvtxDomainRangePop(nvtx_domain()); }
};

struct ProfScope {
    gpair_ctx* c;
    int id;
    cudaStream_t st;
    cudaEvent_t a = nullptr, b = nullptr;
    NvtxRange nv;
    ProfScope(gpair_ctx* c_, int id_, cudaStream_t st_) : c(c_), id(id_), st(st_), nv(kStageName[id_]) {
        if (!c->prof_on) return;
        a = take();
        b = take();
        if (a) cudaEventRecord(a, st);
    }
    cudaEvent_t take() {
        cudaEvent_t e = nullptr;
        if (!c->prof_free.empty()) {
            e = c->prof_free.back();
            c->prof_free.pop_back();
        } else if (cudaEventCreate(&e) != cudaSuccess) {
            e = nullptr;
        }
        return e;
    }
    ~ProfScope() {
        if (!c->prof_on || !a || !b) return;
        cudaEventRecord(b, st);
        c->prof_pending.push_back({id, a, b});
    }
};

void prof_drain(gpair_ctx* c) {
    for (auto& p : c->prof_pending) {
        float ms = 0.f;
        if (cudaEventSynchronize(p.stop) == cudaSuccess && cudaEventElapsedTime(&ms, p.start, p.stop) == cudaSuccess) {
            c->prof_ms[p.id] += ms;
            c->prof_n[p.id] += 1;
        }
        c->prof_free.push_back(p.start);
        c->prof_free.push_back(p.stop);
    }
    c->prof_pending.clear();
}

void free_ctx(gpair_ctx* c) {
    if (!c) return;
    cudaFree(c->d_sens);
    cudaFree(c->d_kd);
    cudaFree(c->d_cell);
    cudaFree(c->d_grp);
    cudaFree(c->d_orig);
    cudaFree(c->d_perm);
    cudaFree(c->d_wlo_f);
    cudaFree(c->d_rent);
    cudaFree(c->d_partial);
    cudaFree(c->d_wlo_a);
    cudaFree(c->d_gpart);
    cudaFree(c->d_gtab);
    cudaFree(c->d_wlo_m);
    cudaFree(c->d_mp);
    cudaFree(c->d_mp_coef);
    cudaFree(c->d_amp);
    cudaFree(c->d_y);
    cudaFree(c->d_delta);
    cudaFree(c->d_loss_part);
    cudaFree(c->d_count);
    cudaFree(c->d_flags);
    cudaFree(c->d_taps);
    cudaFree(c->d_dconv);
    cudaFree(c->d_ksig);
    cudaFree(c->d_near_f);
    cudaFree(c->d_near_a);
    cudaFree(c->d_near_rseg);
    cudaFree(c->d_near_cseg);
    cudaFree(c->d_near_row);
    cudaFree(c->d_ynear);
    cudaFree(c->d_gnear);
    cudaFree(c->d_vcr_u);
    cudaFree(c->d_vcr_part);
    cudaFree(c->d_vcr_g);
    cudaFree(c->d_vcr_x);
    prof_drain(c);
    for (auto e : c->prof_free) cudaEventDestroy(e);
    for (auto e : c->ev_f)
        if (e) cudaEventDestroy(e);
    for (auto e : c->ev_r)
        if (e) cudaEventDestroy(e);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    if (c->st2) cudaStreamDestroy(c->st2);
    delete c;
}

// The sensor-group pipeline of gpair_iterate (opt-in): the forward and the
// sensor-lane adjoint run group by group (256 sensors) on the caller's stream while the
// reducer (and, at world > 1, the all-reduce of that group's y rows and its residual) of
// group g runs on an internal high-priority stream as soon as forward group g is done; the
// adjoint of group g waits only for its own residual rows.  Memory-bound reduction and the
// collective overlap the shared-memory / FMA-bound kernels.
gpair_status pipeline_init(gpair_ctx* c) {
    if (c->st2) return GPAIR_OK;
    int lo = 0, hi = 0;
    cudaError_t e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&c->st2, cudaStreamNonBlocking, hi);
    for (int g = 0; g < 64 && e == cudaSuccess; ++g) {
        e = cudaEventCreateWithFlags(&c->ev_f[g], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_r[g], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
    return e == cudaSuccess ? GPAIR_OK : cuda_fail(c, e, "pipeline streams/events");
}

bool pipeline_eligible(const gpair_ctx* c) {
    const int ak = gpair::adjoint_kernel(c);
    return c->pipeline && !c->assa && !c->n_near && c->f_warps == 8 &&
           (ak == gpair::ADJ_MP || ak == gpair::ADJ_LCF || ak == gpair::ADJ_TAB_T || ak == gpair::ADJ_SL) && gpair::adjoint_groups(c) <= 64 &&
           256 % (32 * (c->f_warps / c->f_split)) == 0;
}

struct WindowReset {
    gpair_ctx* c;
    ~WindowReset() {
        c->lg0 = c->lng = c->lj0 = c->lnj = 0;
        c->lskip_gather = false;
    }
};

gpair_status sticky_check(gpair_ctx* c) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(c, e, "pending asynchronous CUDA error");
    return GPAIR_OK;
}

gpair_status allreduce(gpair_ctx* c, float* y, cudaStream_t st) {
    if (!c->coll) return GPAIR_OK;
    ProfScope ps(c, GPAIR_PROF_ALLREDUCE, st);
    nccl_res_t r = g_nccl.AllReduce(y, y, (size_t)c->Nd * c->Nt, NCCL_FLOAT32, NCCL_SUM, c->nccl, st);
    if (r != 0)
        return fail(c, GPAIR_ERR_NCCL,
                    std::string("ncclAllReduce failed: ") + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
    return GPAIR_OK;
}

gpair_status nccl_check(gpair_ctx* c, nccl_res_t r, const char* what) {
    if (r == 0) return GPAIR_OK;
    return fail(c, GPAIR_ERR_NCCL, std::string(what) + " failed: " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
}

// R_VCR under kernel sharding (row f2): rank r owns the
// z planes [z0, z0 + nzo) of the global grid, ranks in z order.  Its state's
// own planes are copied into c->d_vcr_x between HALO planes received from each
// neighbour (ncclSend/ncclRecv in one group: the 2 planes next to the slab
// boundary go to and come from ranks r - 1 and r + 1), then the slab kernels
// give the own planes' gradient and the slab's value, which one 8-byte
// all-reduce sums into the global R_VCR (d_vcr_part[vcr_nb]).
constexpr int VCR_HALO = 2;  // the stencils' reach (gpair_vcr.cu)

// The halo buffer [lower halo | own planes | upper halo] of this rank's slab.
int64_t vcr_halo_elems(const gpair_ctx* c, const int32_t* grid) {
    const int64_t P = (int64_t)grid[0] * grid[1];
    const int lo = c->rank > 0 ? VCR_HALO : 0, hi = c->rank < c->world - 1 ? VCR_HALO : 0;
    return P * (lo + c->M / P + hi);
}

// Buffers and layout come from gpair_vcr_prepare (validated on every rank, allocated
// before the first iteration: no allocation or early return between collectives).
gpair_status vcr_sharded(gpair_ctx* c, const float* z, int npc, const gpair_step* s, cudaStream_t st) {
    constexpr int HALO = VCR_HALO;
    const int32_t* grid = c->vcr_grid;
    const int64_t P = (int64_t)grid[0] * grid[1];
    const int nzo = (int)(c->M / P), z0 = c->vcr_z0;
    const int lo = c->rank > 0 ? HALO : 0, hi = c->rank < c->world - 1 ? HALO : 0;
    float* xb = c->d_vcr_x;
    API_CUDA(c, cudaMemcpyAsync(xb + P * lo, z, sizeof(float) * (size_t)c->M, cudaMemcpyDeviceToDevice, st),
             "vcr own planes");
    gpair_status gs = nccl_check(c, g_nccl.GroupStart(), "ncclGroupStart");
    if (gs) return gs;
    if (lo) {
        gs = nccl_check(c, g_nccl.Send(z, (size_t)(P * HALO), NCCL_FLOAT32, c->rank - 1, c->nccl, st), "ncclSend");
        if (!gs) gs = nccl_check(c, g_nccl.Recv(xb, (size_t)(P * HALO), NCCL_FLOAT32, c->rank - 1, c->nccl, st), "ncclRecv");
    }
    if (hi && !gs) {
        gs = nccl_check(c, g_nccl.Send(z + P * (nzo - HALO), (size_t)(P * HALO), NCCL_FLOAT32, c->rank + 1, c->nccl, st),
                        "ncclSend");
        if (!gs)
            gs = nccl_check(c, g_nccl.Recv(xb + P * (lo + nzo), (size_t)(P * HALO), NCCL_FLOAT32, c->rank + 1, c->nccl, st),
                            "ncclRecv");
    }
    gpair_status ge = nccl_check(c, g_nccl.GroupEnd(), "ncclGroupEnd");
    if (gs) return gs;
    if (ge) return ge;
    API_CUDA(c, gpair::launch_vcr_slab(c, grid, z0, nzo, xb, z0 - lo, npc, s->eps_npc, s->beta, s->eps_reg,
                                       c->d_vcr_g, nullptr, st),
             "vcr (slab)");
    API_CUDA(c, gpair::launch_vcr_total(c, st), "vcr total");
    return nccl_check(c, g_nccl.AllReduce(c->d_vcr_part + c->vcr_nb, c->d_vcr_part + c->vcr_nb, 1, NCCL_FLOAT64, NCCL_SUM,
                                          c->nccl, st),
                      "ncclAllReduce (R_VCR)");
}

}  // namespace

extern "C" {

const char* gpair_version(void) { return "gpair-b200 0.1 (sm_100a)"; }

const char* gpair_strerror(gpair_status s) {
    switch (s) {
        case GPAIR_OK: return "ok";
        case GPAIR_ERR_INVALID_ARGUMENT: return "invalid argument";
        case GPAIR_ERR_GEOMETRY: return "geometry conflict";
        case GPAIR_ERR_RESOURCE: return "resource limit";
        case GPAIR_ERR_NUMERICAL: return "numerical failure";
        case GPAIR_ERR_CUDA: return "CUDA error";
        case GPAIR_ERR_NCCL: return "NCCL error";
    }
    return "unknown status";
}

const char* gpair_last_error(const gpair_ctx* ctx) { return ctx ? ctx->err.c_str() : g_static_err.c_str(); }

double gpair_cawr_lr(int64_t t, double eta_min, double eta_max, int64_t T0, int64_t Tmult, int printed_formula) {
    if (T0 < 1 || Tmult < 1 || t < 0) return NAN;
    double T_cur, T_i;
    if (printed_formula || Tmult == 1) {
        // Eq. 24 as printed: T_cur = t mod T0, T_i = T0 Tmult^floor(t/T0)
        T_cur = (double)(t % T0);
        T_i = (double)T0 * std::pow((double)Tmult, (double)(t / T0));
    } else {
        // SGDR restarts: periods T0, T0 Tmult, T0 Tmult^2, ...
        int64_t start = 0, period = T0;
        while (t >= start + period) {
            start += period;
            period *= Tmult;
        }
        T_cur = (double)(t - start);
        T_i = (double)period;
    }
    return eta_min + 0.5 * (eta_max - eta_min) * (1.0 + std::cos(M_PI * T_cur / T_i));
}

gpair_status gpair_create(gpair_ctx** out, const gpair_desc* d, void* stream) {
    NvtxRange nvtx_call("create");
    if (!out) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (!d) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "desc is NULL");
    if (!finite_pos(d->sound_speed)) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "sound_speed must be finite > 0");
    if (!finite_pos(d->sampling_rate)) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "sampling_rate must be finite > 0");
    if (!finite_pos(d->sigma)) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "sigma must be finite > 0");
    if (!finite_pos(d->window_k)) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "window_k must be finite > 0");
    if (!std::isfinite(d->t0)) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "t0 must be finite");
    if (d->n_samples < 1) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "n_samples must be >= 1");
    if (d->n_sensors < 1) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "n_sensors must be >= 1");
    if (d->n_kernels < 1) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "n_kernels must be >= 1");
    if (!d->centers || !d->sensors) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "centers/sensors NULL");
    const bool nf = (d->flags & GPAIR_NEAR_FIELD) != 0;
    const bool gen = nf || d->sigmas;
    if (gen && (d->flags & GPAIR_TOF_ASSA))
        return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "per-kernel sigmas / near field need the exact operator");
    double s_max = d->sigma;
    if (d->sigmas) {  // validate sigma_i > 0 finite; the largest sizes the windows (row f4)
        std::vector<float> hs((size_t)d->n_kernels);
        cudaError_t e0 = cudaMemcpyAsync(hs.data(), d->sigmas, sizeof(float) * hs.size(), cudaMemcpyDeviceToHost,
                                         (cudaStream_t)stream);
        if (e0 == cudaSuccess) e0 = cudaStreamSynchronize((cudaStream_t)stream);
        if (e0 != cudaSuccess) return cuda_fail(nullptr, e0, "reading sigmas");
        s_max = 0.0;
        for (float x : hs) {
            if (!(x > 0.f) || !std::isfinite(x))
                return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "sigmas must be finite > 0");
            s_max = std::max(s_max, (double)x);
        }
    }
    if (d->world < 1 || d->rank < 0 || d->rank >= d->world)
        return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "rank/world invalid");
    const bool coll = d->world > 1 || (d->flags & GPAIR_COLLECTIVE);
    if (coll && !d->nccl_comm)
        return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "world > 1 (or GPAIR_COLLECTIVE) needs nccl_comm");
    if ((int64_t)d->n_sensors * d->n_samples >= (1LL << 31))
        return fail(nullptr, GPAIR_ERR_RESOURCE, "N_d * N_t must be < 2^31");
    if (d->n_kernels >= (1LL << 31) - 64) return fail(nullptr, GPAIR_ERR_RESOURCE, "n_kernels must be < 2^31 - 64");
    if (coll) {
        if (!nccl_load()) return fail(nullptr, GPAIR_ERR_NCCL, "cannot dlopen libnccl.so.2");
        int cn = 0, cr = -1;
        if (g_nccl.CommCount(d->nccl_comm, &cn) != 0 || g_nccl.CommUserRank(d->nccl_comm, &cr) != 0)
            return fail(nullptr, GPAIR_ERR_NCCL, "ncclCommCount / ncclCommUserRank failed on nccl_comm");
        if (cn != d->world || cr != d->rank)
            return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "nccl_comm size / rank differ from world / rank");
    }

    // operator constants (fp64 on the host)
    const double v = d->sound_speed, fs = d->sampling_rate, s = d->sigma, kk = d->window_k;
    const double h = v / fs;
    const double log2e = 1.4426950408889634;
    gpair::OpConst k{};
    k.v = v;
    k.fs = fs;
    k.t0 = d->t0;
    k.ks = kk * (d->sigmas ? s_max : s);  // same expression as the oracle's k * sigma
    k.Nt = d->n_samples;
    k.Nd = d->n_sensors;
    double Lw = 2.0 * k.ks / h;
    double Lr = std::nearbyint(Lw);
    int wmax = (std::fabs(Lw - Lr) < 1e-6 * std::max(1.0, Lw)) ? (int)Lr : (int)std::ceil(Lw);
    k.wmax = std::max(wmax, 1);
    k.h = h;
    k.inv_h = 1.0 / h;
    k.t0fs = d->t0 * fs;
    k.ku = (float)(k.ks / h);
    {
        // window length 2 k sigma / h an exact integer (the fp32 ku doubled is
        // that integer): the fp32 fast path derives the upper edge from the
        // lower one (gpair_internal.cuh pair_setup)
        const double two = 2.0 * (double)k.ku;
        k.cnt_int = (two == std::nearbyint(two) && std::fabs(Lw - two) < 1e-9 * std::max(1.0, Lw) && two >= 1.0)
                        ? (int)two
                        : 0;
        k.c_lo = -k.ku - 0.5f;
        k.c_u = k.ku - 0.5f;
    }
    k.K1u = (float)(-log2e * h * h / (2.0 * s * s));
    k.win_half = k.ks;
    k.kwin = kk;
    k.sigma = s;
    k.per_sigma = d->sigmas ? 1 : 0;
    k.gen = gen ? 1 : 0;
    k.nf = nf ? 1 : 0;
    k.nf_add = std::max(0.0, -v * d->t0);
    k.nf_thr_max = nf ? (k.ks + k.nf_add) * (1.0 + 1e-6) + 1e-12 : -1.0;
    if (gen) k.cnt_int = 0;
    k.two_over_h = (float)(2.0 / h);
    const bool assa = (d->flags & GPAIR_TOF_ASSA) != 0;
    std::vector<float> taps;
    if (assa) {
        // Eq. 8, integer arithmetic as in oracle.assa_params (reading A2)
        const int nmin = d->assa_nmin > 0 ? d->assa_nmin : 25;
        if (nmin < 3) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "assa_nmin must be >= 3");
        char buf[64];
        snprintf(buf, sizeof(buf), "%.12g", kk * s * fs / v);
        const double ratio = std::strtod(buf, nullptr);
        const int n_half = std::max(1, (int)std::ceil(ratio));
        const int num = nmin - 1, den = 2 * n_half;
        const int alpha = std::max(1, (num + den - 1) / den);
        k.alpha = alpha;
        k.n_half = n_half;
        k.K = alpha * n_half;
        k.fs_up = (double)alpha * fs;
        if (2 * k.K + 1 > 1024) return fail(nullptr, GPAIR_ERR_RESOURCE, "ASSA taps table > 1024 entries");
        if ((int64_t)alpha * d->n_samples >= (1LL << 30)) return fail(nullptr, GPAIR_ERR_RESOURCE, "alpha N_t too large");
        // Eq. 11 taps in fp64, C = 1/2 (reading A1)
        const double dt_up = 1.0 / k.fs_up;
        taps.resize(2 * k.K + 1);
        for (int q = -k.K; q <= k.K; ++q) {
            const double dq = -v * (double)q * dt_up;
            taps[q + k.K] = (float)(0.5 * dq * std::exp(-(dq * dq) / (2.0 * s * s)));
        }
        k.win_half = std::max(k.ks, (n_half + 1) * h);
    }

    gpair_ctx* c = new (std::nothrow) gpair_ctx();
    if (!c) return fail(nullptr, GPAIR_ERR_RESOURCE, "host allocation failed");
    cudaError_t e = cudaGetDevice(&c->device);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(nullptr, e, "cudaGetDevice");
    }
    c->k = k;
    build_tab(c);
    c->M = d->n_kernels;
    c->Nd = d->n_sensors;
    c->Nt = d->n_samples;
    c->rank = d->rank;
    c->world = d->world;
    c->coll = (d->world > 1 || (d->flags & GPAIR_COLLECTIVE)) ? 1 : 0;
    c->nccl = d->nccl_comm;
    c->flags = d->flags;
    c->assa = assa ? 1 : 0;
    c->gen = gen ? 1 : 0;
    c->nf = nf ? 1 : 0;
    c->create_sigmas = d->sigmas;
    cudaStream_t st = (cudaStream_t)stream;
    std::string why;
    int geom_err = 0;
    e = gpair::build_geometry(c, d->centers, d->sensors, st, why, geom_err);
    if (e != cudaSuccess) {
        std::string m = std::string("gpair_create: ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")" +
                        (why.empty() ? "" : " at " + why);
        free_ctx(c);
        return fail(nullptr, e == cudaErrorMemoryAllocation ? GPAIR_ERR_RESOURCE : GPAIR_ERR_CUDA, m);
    }
    if (geom_err) {
        free_ctx(c);
        return fail(nullptr, (gpair_status)geom_err, why);
    }
    {
        // opt-in (GPAIR_PIPELINE=1): measured 74.6 vs 74.1 ms at cfg4 on one GPU -- the forward fills
        // every SM, so the reducer finds no room to overlap and four group launches add tails
        const char* pp = std::getenv("GPAIR_PIPELINE");
        c->pipeline = (pp && pp[0] == '1') ? 1 : 0;
        if (c->pipeline && pipeline_eligible(c) && pipeline_init(c) != GPAIR_OK) {
            std::string m = c->err;
            free_ctx(c);
            return fail(nullptr, GPAIR_ERR_CUDA, m);
        }
    }
    if (assa) {
        e = cudaMalloc(&c->d_taps, sizeof(float) * taps.size());
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(c->d_taps, taps.data(), sizeof(float) * taps.size(), cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMalloc(&c->d_dconv, sizeof(float) * (size_t)c->Nd * k.alpha * c->Nt);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            std::string m = std::string("gpair_create (ASSA buffers): ") + cudaGetErrorString(e);
            free_ctx(c);
            return fail(nullptr, GPAIR_ERR_RESOURCE, m);
        }
        c->workspace_bytes += (int64_t)(sizeof(float) * (taps.size() + (size_t)c->Nd * k.alpha * c->Nt));
    }
    c->create_sigmas = nullptr;
    *out = c;
    return GPAIR_OK;
}

gpair_status gpair_destroy(gpair_ctx* ctx) {
    if (!ctx) return GPAIR_OK;
    cudaDeviceSynchronize();
    free_ctx(ctx);
    return GPAIR_OK;
}

gpair_status gpair_get_info(const gpair_ctx* c, gpair_info* o) {
    if (!c || !o) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "NULL argument");
    o->n_kernels = c->M;
    o->n_kernels_padded = c->Mpad;
    o->n_cells = c->ncells;
    o->fwd_region_cells = c->f_cpr;
    o->fwd_regions = c->f_regions;
    o->fwd_window = c->Lf;
    o->fwd_warps = c->f_warps;
    o->adj_region_cells = c->a_cpr;
    o->adj_regions = c->a_regions;
    o->adj_window = c->La;
    o->wmax = c->k.wmax;
    o->grid_detected = c->grid_detected;
    o->max_eps = c->max_eps;
    o->workspace_bytes = c->workspace_bytes;
    o->assa = c->assa;
    o->assa_alpha = c->k.alpha;
    o->assa_n_half = c->k.n_half;
    o->assa_K = c->k.K;
    o->general = c->gen;
    o->near_rows = c->n_near_rows;
    o->near_pairs = c->n_near;
    o->tab = ((c->ser == 0 || c->ser == gpair::SER_FAST5) && c->tab.on) ? 1 : 0;
    o->adj_kernel = c->assa ? (c->mp_on ? gpair::ADJ_MP : 0) : gpair::adjoint_kernel(c);
    o->collective = c->coll;
    o->fwd_union = c->f_union;
    o->adj_fit_err = c->mp_fit_err;
    o->adj_row_bytes = c->mp_on ? (c->assa ? 4 : c->mp_row) : 0;
    return GPAIR_OK;
}

static gpair_status do_forward_core(gpair_ctx* c, const float* src, int npc, float eps, float* y,
                                    const float* b, cudaStream_t st) {
    {
        ProfScope ps(c, GPAIR_PROF_GATHER, st);
        API_CUDA(c, gpair::launch_gather(c, src, npc, eps, st), "gather");
    }
    {
        ProfScope ps(c, GPAIR_PROF_FORWARD, st);
        API_CUDA(c, c->assa ? gpair::launch_assa_forward(c, st) : gpair::launch_forward(c, st), "forward");
        if (c->n_near) API_CUDA(c, gpair::launch_near_forward(c, st), "near-field forward");
    }
    if (!c->coll) {
        ProfScope ps(c, GPAIR_PROF_REDUCE, st);
        API_CUDA(c, gpair::launch_reduce(c, y, b, b ? c->d_delta : nullptr, st), "reduce");
    } else {
        {
            ProfScope ps(c, GPAIR_PROF_REDUCE, st);
            API_CUDA(c, gpair::launch_reduce(c, y, nullptr, nullptr, st), "reduce");
        }
        gpair_status s = allreduce(c, y, st);
        if (s != GPAIR_OK) return s;
        if (b) {
            ProfScope ps(c, GPAIR_PROF_RESIDUAL, st);
            API_CUDA(c, gpair::launch_residual(c, y, b, c->d_delta, st), "residual");
        }
    }
    return GPAIR_OK;
}

gpair_status gpair_forward(gpair_ctx* c, const float* amplitudes, float* signals, void* stream) {
    if (!c) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!amplitudes || !signals) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "amplitudes/signals NULL");
    gpair_status s = sticky_check(c);
    if (s) return s;
    return do_forward_core(c, amplitudes, 0, 0.f, signals, nullptr, (cudaStream_t)stream);
}

gpair_status gpair_adjoint(gpair_ctx* c, const float* residual, float* grad, void* stream) {
    if (!c) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!residual || !grad) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "residual/grad NULL");
    gpair_status s = sticky_check(c);
    if (s) return s;
    cudaStream_t st = (cudaStream_t)stream;
    EpiParams ep{};
    ep.scale = 1.f;
    ep.g_out = grad;
    ProfScope ps(c, GPAIR_PROF_ADJOINT, st);
    if (c->n_near) {
        API_CUDA(c, gpair::launch_near_adjoint(c, residual, st), "near-field adjoint");
        ep.g_add = c->d_gnear;
    }
    API_CUDA(c,
             c->assa ? gpair::launch_assa_adjoint(c, residual, gpair::EPI_GRAD, ep, st)
                     : gpair::launch_adjoint(c, residual, gpair::EPI_GRAD, ep, st),
             "adjoint");
    return GPAIR_OK;
}

static gpair_status check_vcr_args(gpair_ctx* c, const int32_t* grid, float beta, float eps) {
    if (!grid) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "grid is NULL");
    for (int d = 0; d < 3; ++d)
        if (grid[d] < 1) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "grid dimensions must be >= 1");
    if ((int64_t)grid[0] * grid[1] * grid[2] > ((int64_t)1 << 31) / 9)
        return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "grid too large");
    if (!std::isfinite(beta)) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "beta not finite");
    if (!(eps > 0.f) || !std::isfinite(eps)) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "eps_reg must be > 0");
    return GPAIR_OK;
}

gpair_status gpair_vcr(gpair_ctx* c, const int32_t* grid, const float* x, float beta, float eps, float* grad,
                       float* value, void* stream) {
    if (!c) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!x) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "x is NULL");
    gpair_status gs = check_vcr_args(c, grid, beta, eps);
    if (gs) return gs;
    gs = sticky_check(c);
    if (gs) return gs;
    cudaStream_t st = (cudaStream_t)stream;
    ProfScope ps(c, GPAIR_PROF_VCR, st);
    API_CUDA(c, gpair::launch_vcr(c, grid, x, 0, 0.f, beta, eps, grad, value, st), "vcr");
    return GPAIR_OK;
}

gpair_status gpair_vcr_slab(gpair_ctx* c, const int32_t* grid, int32_t z0, int32_t nz_own, const float* x_ext,
                            int32_t ext_z0, int32_t ext_nz, float beta, float eps, float* grad, float* value,
                            void* stream) {
    if (!c) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!x_ext) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "x_ext is NULL");
    gpair_status gs = check_vcr_args(c, grid, beta, eps);
    if (gs) return gs;
    int zu0, zu1, zx0, zx1;
    if (gpair::vcr_slab_ranges(grid, z0, nz_own, &zu0, &zu1, &zx0, &zx1) != cudaSuccess)
        return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "own planes [z0, z0 + nz_own) not inside the grid");
    if (ext_z0 > zx0 || (int64_t)ext_z0 + ext_nz < zx1 || ext_z0 < 0 || (int64_t)ext_z0 + ext_nz > grid[2])
        return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "x_ext must cover planes [max(0, z0-2), min(n_z, z0+nz_own+2))");
    gs = sticky_check(c);
    if (gs) return gs;
    cudaStream_t st = (cudaStream_t)stream;
    ProfScope ps(c, GPAIR_PROF_VCR, st);
    API_CUDA(c, gpair::launch_vcr_slab(c, grid, z0, nz_own, x_ext, ext_z0, 0, 0.f, beta, eps, grad, value, st),
             "vcr (slab)");
    return GPAIR_OK;
}

gpair_status gpair_vcr_prepare(gpair_ctx* c, const int32_t* grid, int32_t z0, void* stream) {
    if (!c) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "ctx is NULL");
    gpair_status gs = check_vcr_args(c, grid, 0.f, 1.f);
    if (gs) return gs;
    gs = sticky_check(c);
    if (gs) return gs;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t P = (int64_t)grid[0] * grid[1];
    const int64_t nzo = c->M % P ? 0 : c->M / P;
    std::string why;
    if (!nzo) why = "n_kernels is not whole z planes of grid";
    else if (!c->coll && (nzo != grid[2] || z0 != 0)) why = "world 1: grid must be the kernels' own grid, z0 = 0";
    else if (c->world > 1 && nzo < 2) why = "world > 1 needs >= 2 z planes per rank";
    else if (z0 < 0 || z0 + nzo > grid[2]) why = "slab [z0, z0 + M / (nx ny)) outside the grid";
    if (c->coll) {
        // every rank contributes (z0, nz, error) in its own slot; one summing all-reduce
        // gives every rank the whole table, so every rank takes the same decision
        const int W = c->world;
        std::vector<int32_t> h((size_t)3 * W, 0);
        h[3 * c->rank] = z0;
        h[3 * c->rank + 1] = (int32_t)nzo;
        h[3 * c->rank + 2] = why.empty() ? 0 : 1;
        int32_t* d = nullptr;
        API_CUDA(c, cudaMalloc(&d, sizeof(int32_t) * h.size()), "vcr prepare table");
        cudaError_t e = cudaMemcpyAsync(d, h.data(), sizeof(int32_t) * h.size(), cudaMemcpyHostToDevice, st);
        nccl_res_t r = e == cudaSuccess ? g_nccl.AllReduce(d, d, h.size(), NCCL_INT32, NCCL_SUM, c->nccl, st) : 0;
        if (e == cudaSuccess && r == 0) e = cudaMemcpyAsync(h.data(), d, sizeof(int32_t) * h.size(), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess && r == 0) e = cudaStreamSynchronize(st);
        cudaFree(d);
        if (e != cudaSuccess) return cuda_fail(c, e, "vcr prepare exchange");
        if (r != 0) return nccl_check(c, r, "ncclAllReduce (vcr prepare)");
        int32_t expect = 0;
        for (int q = 0; q < W && why.empty(); ++q) {
            if (h[3 * q + 2]) why = "rank " + std::to_string(q) + " rejected its slab";
            else if (h[3 * q] != expect) why = "slabs are not contiguous whole z planes in rank order";
            expect = h[3 * q] + h[3 * q + 1];
        }
        if (why.empty() && expect != grid[2]) why = "slabs do not cover the grid's n_z planes";
    }
    if (!why.empty()) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "gpair_vcr_prepare: " + why);
    const int64_t n = c->coll ? vcr_halo_elems(c, grid) : 0;
    if (c->coll && c->vcr_x_n != n) {
        cudaFree(c->d_vcr_x);
        c->d_vcr_x = nullptr;
        c->vcr_x_n = 0;
        API_CUDA(c, cudaMalloc(&c->d_vcr_x, sizeof(float) * (size_t)n), "vcr halo buffer");
        c->vcr_x_n = n;
        c->workspace_bytes += (int64_t)sizeof(float) * n;
    }
    API_CUDA(c, gpair::vcr_slab_ensure(c, grid, z0, (int)nzo), "vcr workspace");
    for (int d = 0; d < 3; ++d) c->vcr_grid[d] = grid[d];
    c->vcr_z0 = z0;
    c->vcr_prepared = 1;
    return GPAIR_OK;
}

gpair_status gpair_iterate(gpair_ctx* c, float* z, float* m, float* v, const float* b, const gpair_step* s,
                           float* signals_out, float* x_out, float* loss_out, void* stream) {
    NvtxRange nvtx_call("iterate");
    if (!c) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!z || !b || !s) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "z/b/step NULL");
    if (s->mode != 0 && s->mode != 1) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "mode must be 0 (NPC) or 1 (clamp)");
    if (s->mode == 0 && (!m || !v)) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "Adam state m/v NULL");
    if (s->mode == 0 && s->step < 1) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "step must be >= 1");
    if (!std::isfinite(s->lr)) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "lr not finite");
    gpair_status st0 = sticky_check(c);
    if (st0) return st0;
    const bool reg = s->lam != 0.f;
    if (reg) {
        if (!(s->lam > 0.f) || !std::isfinite(s->lam)) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "lam must be >= 0");
        gpair_status gs = check_vcr_args(c, s->grid, s->beta, s->eps_reg);
        if (gs) return gs;
        const int64_t P = (int64_t)s->grid[0] * s->grid[1];
        if (!c->coll) {
            if (P * s->grid[2] != c->M) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "grid[0] grid[1] grid[2] != n_kernels");
        } else if (!c->vcr_prepared || s->z0 != c->vcr_z0 || s->grid[0] != c->vcr_grid[0] ||
                   s->grid[1] != c->vcr_grid[1] || s->grid[2] != c->vcr_grid[2]) {
            // the slab layout was agreed by every rank in gpair_vcr_prepare, so this is
            // the same decision on every rank that prepared the same layout
            return fail(c, GPAIR_ERR_INVALID_ARGUMENT,
                        "lam > 0 on the collective path needs gpair_vcr_prepare(grid, z0) with the same grid / z0");
        }
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int npc = s->mode == 0;
    float* y = signals_out ? signals_out : c->d_y;
    if (reg) {  // R_VCR and its gradient at the pre-update x (Alg. 2)
        ProfScope ps(c, GPAIR_PROF_VCR, st);
        if (!c->coll) {
            API_CUDA(c, gpair::vcr_slab_ensure(c, s->grid, 0, s->grid[2]), "vcr workspace");  // d_vcr_g exists
            API_CUDA(c, gpair::launch_vcr(c, s->grid, z, npc, s->eps_npc, s->beta, s->eps_reg, c->d_vcr_g, nullptr, st),
                     "vcr");
        } else {
            gpair_status gs = vcr_sharded(c, z, npc, s, st);
            if (gs) return gs;
        }
    }
    // fp64 R_VCR for the loss: the per-block partials (world 1) or the all-reduced total
    const double* reg_part = reg ? (!c->coll ? c->d_vcr_part : c->d_vcr_part + c->vcr_nb) : nullptr;
    const int32_t reg_n = reg ? (!c->coll ? c->vcr_nb : 1) : 0;
    EpiParams ep{};
    const double N = (double)c->Nd * (double)c->Nt;
    ep.scale = s->grad_scale > 0.f ? s->grad_scale : (float)(2.0 / N);
    ep.lr = s->lr;
    ep.beta1 = s->beta1;
    ep.beta2 = s->beta2;
    ep.adam_eps = s->adam_eps;
    ep.eps_npc = s->eps_npc;
    if (npc) {
        ep.bc1 = (float)(1.0 / (1.0 - std::pow((double)s->beta1, (double)s->step)));
        ep.bc2 = (float)(1.0 / (1.0 - std::pow((double)s->beta2, (double)s->step)));
    }
    ep.z = z;
    ep.m = m;
    ep.v = v;
    ep.x_out = x_out;
    ep.g_reg = reg ? c->d_vcr_g : nullptr;
    ep.lam = s->lam;
    const int emode = npc ? gpair::EPI_NPC_ADAM : gpair::EPI_CLAMP;
    if (c->st2 && pipeline_eligible(c)) {
        WindowReset wr{c};
        cudaStream_t s2 = c->st2;
        float* yy = (!c->coll && !signals_out) ? nullptr : y;
        {
            ProfScope ps(c, GPAIR_PROF_GATHER, st);
            API_CUDA(c, gpair::launch_gather(c, z, npc, s->eps_npc, st), "gather");
        }
        const int G = (c->Nd + 255) / 256;  // 256-sensor pipeline groups
        for (int g = 0; g < G; ++g) {
            {
                ProfScope ps(c, GPAIR_PROF_FORWARD, st);
                c->lg0 = g;
                c->lng = 1;
                API_CUDA(c, gpair::launch_forward(c, st), "forward (group)");
            }
            API_CUDA(c, cudaEventRecord(c->ev_f[g], st), "event");
            API_CUDA(c, cudaStreamWaitEvent(s2, c->ev_f[g], 0), "event wait");
            c->lj0 = g * 256;
            c->lnj = std::min(256, c->Nd - g * 256);
            if (!c->coll) {
                ProfScope ps(c, GPAIR_PROF_REDUCE, s2);
                API_CUDA(c, gpair::launch_reduce(c, yy, b, c->d_delta, s2), "reduce (group)");
            } else {
                {
                    ProfScope ps(c, GPAIR_PROF_REDUCE, s2);
                    API_CUDA(c, gpair::launch_reduce(c, y, nullptr, nullptr, s2), "reduce (group)");
                }
                {
                    ProfScope ps(c, GPAIR_PROF_ALLREDUCE, s2);
                    nccl_res_t rr = g_nccl.AllReduce(y + (size_t)c->lj0 * c->Nt, y + (size_t)c->lj0 * c->Nt,
                                                     (size_t)c->lnj * c->Nt, NCCL_FLOAT32, NCCL_SUM, c->nccl, s2);
                    if (rr != 0)
                        return fail(c, GPAIR_ERR_NCCL, std::string("ncclAllReduce failed: ") +
                                                           (g_nccl.GetErrorString ? g_nccl.GetErrorString(rr) : "?"));
                }
                ProfScope ps(c, GPAIR_PROF_RESIDUAL, s2);
                API_CUDA(c, gpair::launch_residual(c, y, b, c->d_delta, s2), "residual (group)");
            }
            API_CUDA(c, cudaEventRecord(c->ev_r[g], s2), "event");
        }
        c->n_loss_part = c->Nd;  // per-sensor loss partials, all groups written on s2
        c->lj0 = c->lnj = 0;
        if (loss_out || (c->flags & GPAIR_CHECK_FINITE)) {
            ProfScope ps(c, GPAIR_PROF_LOSS, s2);
            float* lo = loss_out ? loss_out : (float*)(c->d_count);
            API_CUDA(c,
                     reg ? gpair::launch_loss(c, lo, s2, reg_part, reg_n, (double)s->lam)
                         : gpair::launch_loss(c, lo, s2),
                     "loss");
        }
        API_CUDA(c, cudaEventRecord(c->ev_join, s2), "event");
        c->lskip_gather = true;
        for (int g = 0; g < G; ++g) {
            API_CUDA(c, cudaStreamWaitEvent(st, c->ev_r[g], 0), "event wait");
            ProfScope ps(c, GPAIR_PROF_ADJOINT, st);
            c->lg0 = g;
            c->lng = 1;
            API_CUDA(c, gpair::launch_adjoint(c, c->d_delta, emode, ep, st), "adjoint (group)");
        }
        API_CUDA(c, cudaStreamWaitEvent(st, c->ev_join, 0), "event wait");
        {
            ProfScope ps(c, GPAIR_PROF_ADJOINT, st);
            API_CUDA(c, gpair::launch_adjoint_gather(c, emode, ep, st), "adjoint gather + update");
        }
        if (c->flags & GPAIR_CHECK_FINITE) {
            float h = 0.f;
            float* lo = loss_out ? loss_out : (float*)(c->d_count);
            API_CUDA(c, cudaMemcpyAsync(&h, lo, sizeof(float), cudaMemcpyDeviceToHost, st), "loss readback");
            API_CUDA(c, cudaStreamSynchronize(st), "loss sync");
            if (!std::isfinite(h)) return fail(c, GPAIR_ERR_NUMERICAL, "loss is not finite");
        }
        return GPAIR_OK;
    }
    gpair_status r = do_forward_core(c, z, npc, s->eps_npc, (!c->coll && !signals_out) ? nullptr : y, b, st);
    if (r) return r;
    if (loss_out || (c->flags & GPAIR_CHECK_FINITE)) {
        ProfScope ps(c, GPAIR_PROF_LOSS, st);
        float* lo = loss_out ? loss_out : (float*)(c->d_count);  // scratch word when only checking
        API_CUDA(c,
                 reg ? gpair::launch_loss(c, lo, st, reg_part, reg_n, (double)s->lam)
                     : gpair::launch_loss(c, lo, st),
                 "loss");
        if (c->flags & GPAIR_CHECK_FINITE) {
            float h = 0.f;
            API_CUDA(c, cudaMemcpyAsync(&h, lo, sizeof(float), cudaMemcpyDeviceToHost, st), "loss readback");
            API_CUDA(c, cudaStreamSynchronize(st), "loss sync");
            if (!std::isfinite(h)) return fail(c, GPAIR_ERR_NUMERICAL, "loss is not finite");
        }
    }
    ProfScope ps(c, GPAIR_PROF_ADJOINT, st);
    if (c->n_near) {
        API_CUDA(c, gpair::launch_near_adjoint(c, c->d_delta, st), "near-field adjoint");
        ep.g_add = c->d_gnear;
    }
    API_CUDA(c,
             c->assa ? gpair::launch_assa_adjoint(c, c->d_delta, emode, ep, st)
                     : gpair::launch_adjoint(c, c->d_delta, emode, ep, st),
             "adjoint+update");
    return GPAIR_OK;
}

gpair_status gpair_count_pair_samples(gpair_ctx* c, int64_t* out, void* stream) {
    if (!c || !out) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "NULL argument");
    if (c->gen) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "count is not defined for per-kernel sigma / near field");
    cudaStream_t st = (cudaStream_t)stream;
    API_CUDA(c, c->assa ? gpair::launch_assa_count(c, st) : gpair::launch_count(c, st), "count");
    unsigned long long h = 0;
    API_CUDA(c, cudaMemcpyAsync(&h, c->d_count, sizeof(h), cudaMemcpyDeviceToHost, st), "count readback");
    API_CUDA(c, cudaStreamSynchronize(st), "count sync");
    *out = (int64_t)h;
    return GPAIR_OK;
}

gpair_status gpair_profile_enable(gpair_ctx* c, int enable) {
    if (!c) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "ctx is NULL");
    prof_drain(c);
    for (int i = 0; i < GPAIR_PROF_N; ++i) {
        c->prof_ms[i] = 0.0;
        c->prof_n[i] = 0;
    }
    c->n_launch = 0;
    c->prof_on = enable != 0;
    return GPAIR_OK;
}

gpair_status gpair_profile_read(gpair_ctx* c, gpair_profile* out) {
    if (!c || !out) return fail(c, GPAIR_ERR_INVALID_ARGUMENT, "NULL argument");
    prof_drain(c);
    for (int i = 0; i < GPAIR_PROF_N; ++i) {
        out->ms[i] = c->prof_ms[i];
        out->launches[i] = c->prof_n[i];
    }
    out->kernels = c->n_launch;
    return GPAIR_OK;
}

gpair_status gpair_nccl_unique_id(void* uid) {
    if (!uid) return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "NULL buffer");
    if (!nccl_load()) return fail(nullptr, GPAIR_ERR_NCCL, "cannot dlopen libnccl.so.2");
    nccl_uid_t id;
    nccl_res_t r = g_nccl.GetUniqueId(&id);
    if (r != 0) return fail(nullptr, GPAIR_ERR_NCCL, "ncclGetUniqueId failed");
    memcpy(uid, id.internal, 128);
    return GPAIR_OK;
}

gpair_status gpair_nccl_comm_init(void** comm, int32_t world, const void* uid, int32_t rank) {
    if (!comm || !uid || world < 1 || rank < 0 || rank >= world)
        return fail(nullptr, GPAIR_ERR_INVALID_ARGUMENT, "bad argument");
    if (!nccl_load()) return fail(nullptr, GPAIR_ERR_NCCL, "cannot dlopen libnccl.so.2");
    nccl_uid_t id;
    memcpy(id.internal, uid, 128);
    nccl_res_t r = g_nccl.CommInitRank(comm, world, id, rank);
    if (r != 0)
        return fail(nullptr, GPAIR_ERR_NCCL,
                    std::string("ncclCommInitRank failed: ") + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
    return GPAIR_OK;
}

gpair_status gpair_nccl_comm_destroy(void* comm) {
    if (!comm) return GPAIR_OK;
    if (!nccl_load()) return fail(nullptr, GPAIR_ERR_NCCL, "cannot dlopen libnccl.so.2");
    g_nccl.CommDestroy(comm);
    return GPAIR_OK;
}

}  // extern "C"
