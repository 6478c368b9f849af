// chem_api.cu — the C ABI of include/chem.h: validation, structure matching, workspace, and the
// host side of the bulk-sparse schedule (Alg. 3).
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: phase ranges for nsys / ncu --nvtx (no cost unattached)

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/chem.h"
#include "chem_launch.cuh"


using namespace chem;

namespace {

constexpr double kLockEff = 0.9;   // chem_opts.lockstep = 2: lockstep while the last bulk SIMT efficiency < 0.9
constexpr double kHintAcc = 0.9;   // chem_opts.schedule_lpt = 2: heavy-first only while the layout's hints
                                   // predicted the last call's per-cell substeps this well (sum min/max)
constexpr int kStreamBS = 256;     // gate / compaction / box cost
constexpr int kPointBS = 128;      // point kernels

// ------------------------------------------------------------------ per-structure operations
struct Ops {
    const char* name;
    int ns, nr, nsa;
    size_t params_size;
    bool (*match)(const chem_mech_desc*);
    void (*fill)(const chem_mech_desc*, void*);
    cudaError_t (*rates)(const void*, int64_t, int64_t, const double*, const double*, const double*, double*,
                         cudaStream_t);
    cudaError_t (*rhs)(const void*, int64_t, int64_t, const double*, const double*, const double*, double*,
                       cudaStream_t);
    cudaError_t (*jacobian)(const void*, int64_t, int64_t, const double*, const double*, const double*, double*,
                            cudaStream_t);
    cudaError_t (*temperature)(const void*, int64_t, int64_t, const double*, const double*, double*,
                               unsigned long long*, cudaStream_t);
    cudaError_t (*energy)(const void*, int64_t, int64_t, const double*, const double*, double*, cudaStream_t);
    cudaError_t (*integrate)(const void*, int method, const LaunchCtx&, const uint32_t*, int64_t, int kmax,
                             int refill, int fin, int grid, cudaStream_t);
    cudaError_t (*integrate_lock)(const void*, int method, const LaunchCtx&, const uint32_t*, int64_t, int kmax,
                                  int refill, int fin, int nsm, cudaStream_t);
    int (*blocks_per_sm)(int method);
    size_t integrate_smem;
};

inline int grid_for(int64_t n, int bs, int cap = 148 * 32)
{
    const int64_t g = (n + bs - 1) / bs;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, cap));
}

template <class M>
struct MechOps {
    using P = Params<M>;

    static bool match(const chem_mech_desc* d)
    {
        if (d->ns != M::NS || d->nr != M::NR) return false;
        for (int r = 0; r < M::NR; ++r) {
            if (d->type[r] != M::kind(r) || (d->reversible[r] != 0) != (M::rev(r) != 0)) return false;
            for (int k = 0; k < M::NS; ++k) {
                if (d->nu_f[r * M::NS + k] != (double)M::nuf(r, k)) return false;
                if (d->nu_r[r * M::NS + k] != (double)M::nur(r, k)) return false;
            }
            if (M::kind(r) != 0) {
                int cnt = 0;
                for (int k = 0; k < M::NS; ++k) {
                    if (d->eff[r * M::NS + k] != 1.0) {
                        if (cnt >= M::neff(r) || M::eff_sp(r, cnt) != k) return false;
                        ++cnt;
                    }
                }
                if (cnt != M::neff(r)) return false;
            }
            if (M::kind(r) == 3 && ((d->troe[4 * r + 3] > 0.0) != (M::troe_t2(r) != 0))) return false;
        }
        return true;
    }

    static void fill(const chem_mech_desc* d, void* out)
    {
        P& p = *static_cast<P*>(out);
        std::memset(&p, 0, sizeof(P));
        const int ns = M::NS, nr = M::NR;
        double tmid0 = d->T_range[1];
        bool common = true;
        p.T_valid_lo = -1e300;
        p.T_valid_hi = 1e300;
        for (int k = 0; k < ns; ++k) {
            p.W[k] = d->W[k];
            p.invW[k] = 1.0 / d->W[k];
            p.Tmid[k] = d->T_range[3 * k + 1];
            common = common && (p.Tmid[k] == tmid0);
            p.T_valid_lo = std::max(p.T_valid_lo, d->T_range[3 * k + 0]);
            p.T_valid_hi = std::min(p.T_valid_hi, d->T_range[3 * k + 2]);
            for (int rg = 0; rg < 2; ++rg) {
                const double* a = (rg == 0 ? d->nasa_lo : d->nasa_hi) + 7 * k;
                p.cpc[rg][k][0] = a[0]; p.cpc[rg][k][1] = a[1]; p.cpc[rg][k][2] = a[2];
                p.cpc[rg][k][3] = a[3]; p.cpc[rg][k][4] = a[4];
                p.hc[rg][k][0] = a[0]; p.hc[rg][k][1] = a[1] / 2; p.hc[rg][k][2] = a[2] / 3;
                p.hc[rg][k][3] = a[3] / 4; p.hc[rg][k][4] = a[4] / 5; p.hc[rg][k][5] = a[5];
                p.sc[rg][k][0] = a[0]; p.sc[rg][k][1] = a[1]; p.sc[rg][k][2] = a[2] / 2;
                p.sc[rg][k][3] = a[3] / 3; p.sc[rg][k][4] = a[4] / 4; p.sc[rg][k][5] = a[6];
                p.dcp[rg][k][0] = a[1]; p.dcp[rg][k][1] = 2 * a[2]; p.dcp[rg][k][2] = 3 * a[3];
                p.dcp[rg][k][3] = 4 * a[4];
            }
        }
        p.Tmid_common = common ? tmid0 : -1.0;
        for (int r = 0; r < nr; ++r) {
            p.lnA[r] = std::log(d->A[r]);
            p.b[r] = d->b[r];
            p.EaR[r] = d->Ea[r] / d->R;
            if (M::kind(r) >= 2) {
                p.lnA0[r] = std::log(d->A0[r]);
                p.b0[r] = d->b0[r];
                p.Ea0R[r] = d->Ea0[r] / d->R;
            }
            if (M::kind(r) == 3) {
                const double* t = d->troe + 4 * r;
                p.troe_a[r] = t[0];
                p.troe_iT3[r] = t[1] != 0.0 ? std::min(1.0 / t[1], 1e300) : 1e300;
                p.troe_iT1[r] = t[2] != 0.0 ? std::min(1.0 / t[2], 1e300) : 1e300;
                p.troe_T2[r] = t[3];
                // Fc is exactly alpha in double for 1 K < T < 1e6 K when T*** <= 1e-20 and T* >= 1e20
                p.troe_const[r] = (t[1] > 0.0 && t[1] <= 1e-20 && t[2] >= 1e20 && !(t[3] > 0.0)) ? 1 : 0;
                p.troe_L[r] = std::log10(t[0]);
            }
            for (int i = 0; i < M::neff(r); ++i) p.effm1[M::eff_off(r) + i] = d->eff[r * ns + M::eff_sp(r, i)] - 1.0;
        }
        p.R = d->R;
        p.lnp0R = std::log(d->p_ref / d->R);
    }

    static cudaError_t rates(const void* pp, int64_t n, int64_t ld, const double* rho, const double* T,
                             const double* Y, double* w, cudaStream_t s)
    {
        if (n == 0) return cudaSuccess;
        k_rates<M><<<grid_for(n, kPointBS), kPointBS, 0, s>>>(*static_cast<const P*>(pp), n, ld, rho, T, Y, w);
        return cudaGetLastError();
    }
    static cudaError_t rhs(const void* pp, int64_t n, int64_t ld, const double* rho, const double* T,
                           const double* Y, double* f, cudaStream_t s)
    {
        if (n == 0) return cudaSuccess;
        k_rhs<M><<<grid_for(n, kPointBS), kPointBS, 0, s>>>(*static_cast<const P*>(pp), n, ld, rho, T, Y, f);
        return cudaGetLastError();
    }
    static cudaError_t jacobian(const void* pp, int64_t n, int64_t ld, const double* rho, const double* T,
                                const double* Y, double* J, cudaStream_t s)
    {
        if (n == 0) return cudaSuccess;
        constexpr int BS = 32;
        const size_t sm = (size_t)(M::NS + 1) * (M::NS + 1) * 8 * BS;
        cudaError_t e = cudaFuncSetAttribute(k_jacobian<M, BS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (e != cudaSuccess) return e;
        k_jacobian<M, BS><<<(unsigned)((n + BS - 1) / BS), BS, sm, s>>>(*static_cast<const P*>(pp), n, ld, rho, T, Y, J);
        return cudaGetLastError();
    }
    static cudaError_t temperature(const void* pp, int64_t n, int64_t ld, const double* e, const double* Y,
                                   double* T, unsigned long long* nfail, cudaStream_t s)
    {
        if (n == 0) return cudaSuccess;
        k_temperature<M><<<grid_for(n, kPointBS), kPointBS, 0, s>>>(*static_cast<const P*>(pp), n, ld, e, Y, T, nfail);
        return cudaGetLastError();
    }
    static cudaError_t energy(const void* pp, int64_t n, int64_t ld, const double* T, const double* Y, double* e,
                              cudaStream_t s)
    {
        if (n == 0) return cudaSuccess;
        k_energy<M><<<grid_for(n, kPointBS), kPointBS, 0, s>>>(*static_cast<const P*>(pp), n, ld, T, Y, e);
        return cudaGetLastError();
    }

    // ---- integration launchers (defined in chem_launch_impl.cuh, instantiated in launch_*.cu)
    // lockstep launch (chem_opts.lockstep, heavy-first schedule); Rosenbrock methods only
    static cudaError_t integrate_lock(const void* pp, int method, const LaunchCtx& L, const uint32_t* ids,
                                      int64_t n, int kmax, int refill, int fin, int nsm, cudaStream_t s)
    {
        const P& p = *static_cast<const P*>(pp);
        if (method == CHEM_METHOD_RODAS3) return Launch<M, Rodas3>::lock(p, L, ids, n, kmax, refill, fin, nsm, s);
        return Launch<M, Rodas4>::lock(p, L, ids, n, kmax, refill, fin, nsm, s);
    }
    static cudaError_t integrate(const void* pp, int method, const LaunchCtx& L, const uint32_t* ids,
                                 int64_t n, int kmax, int refill, int fin, int grid, cudaStream_t s)
    {
        const P& p = *static_cast<const P*>(pp);
        if (method == CHEM_METHOD_RODAS3) return Launch<M, Rodas3>::run(p, L, ids, n, kmax, refill, fin, grid, s);
        if (method == CHEM_METHOD_EXPLICIT) return Launch<M, Explicit>::run(p, L, ids, n, kmax, refill, fin, grid, s);
        return Launch<M, Rodas4>::run(p, L, ids, n, kmax, refill, fin, grid, s);
    }
    static int blocks_per_sm(int method)
    {
        if (method == CHEM_METHOD_EXPLICIT) return Launch<M, Explicit>::blocks_per_sm();
        if (method == CHEM_METHOD_RODAS3) return Launch<M, Rodas3>::blocks_per_sm();
        return Launch<M, Rodas4>::blocks_per_sm();
    }

    static Ops ops()
    {
        Ops o;
        o.name = M::kName;
        o.ns = M::NS;
        o.nr = M::NR;
        o.nsa = M::NSA;
        o.params_size = sizeof(P);
        o.match = &match;
        o.fill = &fill;
        o.rates = &rates;
        o.rhs = &rhs;
        o.jacobian = &jacobian;
        o.temperature = &temperature;
        o.energy = &energy;
        o.integrate = &integrate;
        o.integrate_lock = &integrate_lock;
        o.blocks_per_sm = &blocks_per_sm;
        o.integrate_smem = Launch<M, Rodas4>::smem();
        return o;
    }
};

const std::vector<Ops>& registry()
{
    static std::vector<Ops> r = [] {
        std::vector<Ops> v;
#define CHEM_REG(M) v.push_back(MechOps<M>::ops());
        CHEM_FOR_EACH_MECH(CHEM_REG)
#undef CHEM_REG
        return v;
    }();
    return r;
}

// ------------------------------------------------------------------ validation
int validate(const chem_mech_desc* d)
{
    if (!d || d->ns < 1 || d->ns > 32 || d->nr < 0 || d->ne < 1) return CHEM_EINVAL;
    if (!d->W || !d->nasa_lo || !d->nasa_hi || !d->T_range || !d->elem || (d->nr > 0 && (!d->nu_f || !d->nu_r ||
        !d->A || !d->b || !d->Ea || !d->type || !d->reversible || !d->eff || !d->A0 || !d->b0 || !d->Ea0 || !d->troe)))
        return CHEM_EINVAL;
    if (!(d->R > 0.0) || !(d->p_ref > 0.0)) return CHEM_EMECH;
    const int ns = d->ns;
    for (int k = 0; k < ns; ++k) {
        if (!(d->W[k] > 0.0) || !std::isfinite(d->W[k])) return CHEM_EMECH;
        const double* t = d->T_range + 3 * k;
        if (!(t[0] < t[1] && t[1] < t[2])) return CHEM_EMECH;
        for (int i = 0; i < 7; ++i)
            if (!std::isfinite(d->nasa_lo[7 * k + i]) || !std::isfinite(d->nasa_hi[7 * k + i])) return CHEM_EMECH;
    }
    for (int r = 0; r < d->nr; ++r) {
        if (d->type[r] < 0 || d->type[r] > 3) return CHEM_EMECH;
        if (!(d->A[r] > 0.0) || !std::isfinite(d->b[r]) || !std::isfinite(d->Ea[r])) return CHEM_EMECH;
        if (d->type[r] >= 2 && !(d->A0[r] > 0.0)) return CHEM_EMECH;
        double dm = 0.0, gm = 0.0;
        for (int k = 0; k < ns; ++k) {
            const double f = d->nu_f[r * ns + k], b = d->nu_r[r * ns + k];
            if (f < 0 || b < 0 || f != std::floor(f) || b != std::floor(b)) return CHEM_EMECH;
            if (d->eff[r * ns + k] < 0.0) return CHEM_EMECH;
            dm += (b - f) * d->W[k];
            gm += (b + f) * d->W[k];
        }
        if (std::fabs(dm) > 1e-10 * gm) return CHEM_EMECH;
        for (int e = 0; e < d->ne; ++e) {
            double s = 0.0;
            for (int k = 0; k < ns; ++k) s += (d->nu_r[r * ns + k] - d->nu_f[r * ns + k]) * d->elem[k * d->ne + e];
            if (s != 0.0) return CHEM_EMECH;
        }
    }
    return CHEM_OK;
}

// ------------------------------------------------------------------ workspace layout
struct WsLayout {
    size_t stats, boxes, start, cell_t, cell_h, steps, box, hint, state, ids0, idsA, idsB, key0, key1, total;
};

inline size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

WsLayout ws_layout(int64_t N, int32_t B)
{
    WsLayout w;
    size_t o = 0;
    w.stats = o; o = al256(o + S_NSTATS * 8);
    w.boxes = o; o = al256(o + (size_t)B * sizeof(DevBox));
    w.start = o; o = al256(o + (size_t)(B + 1) * 8);
    w.cell_t = o; o = al256(o + (size_t)N * 8);
    w.cell_h = o; o = al256(o + (size_t)N * 8);
    w.steps = o; o = al256(o + (size_t)N * 4);
    w.box = o; o = al256(o + (size_t)N * 4);
    w.hint = o; o = al256(o + (size_t)N * 4);
    w.state = o; o = al256(o + (size_t)N);
    w.ids0 = o; o = al256(o + (size_t)N * 4);
    w.idsA = o; o = al256(o + (size_t)N * 4);
    w.idsB = o; o = al256(o + (size_t)N * 4);
    w.key0 = o; o = al256(o + (size_t)N * 4);     // heavy-first schedule: cost hints and their sort buffer
    w.key1 = o; o = al256(o + (size_t)N * 4);
    w.total = o;
    return w;
}

}  // namespace

// ------------------------------------------------------------------ the context
struct chem_ctx {
    int device = 0;
    const Ops* ops = nullptr;
    std::vector<unsigned char> params;
    chem_opts opts;
    int num_sms = 148;
    int sticky = 0;
    int32_t h_cap = 0;
    DevBox* h_boxes = nullptr;        // pinned, mapped (d_boxes: its device alias)
    int64_t* h_start = nullptr;       // pinned, mapped
    unsigned long long* h_stats = nullptr;  // pinned, mapped [S_NSTATS]
    DevBox* d_boxes = nullptr;
    int64_t* d_start = nullptr;
    unsigned long long* d_stats = nullptr;
    unsigned long long* d_sig = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int32_t* trace = nullptr;        // device [trace_rows][nboxes] activity trace (App. B), or null
    int32_t trace_rows = 0;
    double simt_eff = 1.0;           // bulk SIMT efficiency of the last call (lockstep = 2 input)
    unsigned long long* h_sig = nullptr;   // pinned [6]: staging of the signature + hint-accuracy slots
    struct WsRecord { const void* ws; int64_t total; int32_t nboxes; };
    std::vector<WsRecord> ws_last;   // layout of the last call on each workspace (chem_cell_status)
};

namespace {

int cuda_fail(chem_ctx* c, cudaError_t e)
{
    if (e == cudaSuccess) return CHEM_OK;
    if (c) c->sticky = CHEM_ECUDA;
    std::fprintf(stderr, "libchem: CUDA error %s\n", cudaGetErrorString(e));
    return CHEM_ECUDA;
}

// Pinned host buffer mapped into the device address space (h: host pointer, d: its device alias).
template <class T>
bool alloc_mapped(T*& h, T*& d, size_t count)
{
    h = nullptr;
    d = nullptr;
    if (cudaHostAlloc((void**)&h, sizeof(T) * count, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
        return false;
    if (cudaHostGetDevicePointer((void**)&d, (void*)h, 0) != cudaSuccess) return false;
    return true;
}

int ensure_host_boxes(chem_ctx* c, int32_t nb)
{
    if (nb <= c->h_cap) return CHEM_OK;
    if (c->h_boxes) cudaFreeHost(c->h_boxes);
    if (c->h_start) cudaFreeHost(c->h_start);
    c->h_boxes = nullptr;
    c->h_start = nullptr;
    int cap = std::max(nb, 64);
    if (!alloc_mapped(c->h_boxes, c->d_boxes, cap)) return CHEM_ECUDA;
    if (!alloc_mapped(c->h_start, c->d_start, cap + 1)) return CHEM_ECUDA;
    c->h_cap = cap;
    return CHEM_OK;
}

// lane-refill batch of the sparse launch (k_integrate's `refill`): cost-sorted list / gate-ordered list
constexpr int kRefillSorted = 1, kRefillUnsorted = 8;

// NVTX range for one scope (the call and its Alg. 3 phases show up by name on a profiler timeline)
struct NvtxScope {
    explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
    ~NvtxScope() { nvtxRangePop(); }
};

thread_local int64_t t_launches = 0;   // kernels enqueued by the current call (chem_stats.kernel_launches)

// The call's bookkeeping transfers (box table in, counters out; a few hundred bytes to ~100 KB) and its
// small memsets run as kernels on the caller's stream, through the mapped buffers above, never as
// copy-engine operations: a stream whose previous command was a cudaMemcpyAsync / cudaMemsetAsync lets
// its next command start only when the copy engine is through with every larger copy queued on it by
// then, so a host-buffer caller that overlaps the D2H of one box group with the next call (HostRunner)
// saw each call wait for the previous group's whole D2H (tools/e2e_timeline.py, profiles/r02_e2e_timeline_*).
__global__ void k_copy_words(const unsigned long long* __restrict__ src, unsigned long long* __restrict__ dst,
                             int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

__global__ void k_zero_bytes(unsigned char* __restrict__ dst, int64_t n)
{
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = 0;
}

cudaError_t copy_words(void* dst, const void* src, size_t bytes, cudaStream_t s)   // bytes % 8 == 0
{
    const int64_t n = (int64_t)(bytes / 8);
    if (n == 0) return cudaSuccess;
    const int grid = (int)std::min<int64_t>(64, (n + 255) / 256);
    k_copy_words<<<grid, 256, 0, s>>>(static_cast<const unsigned long long*>(src),
                                       static_cast<unsigned long long*>(dst), n);
    ++t_launches;
    return cudaGetLastError();
}

cudaError_t zero_bytes(void* dst, size_t bytes, cudaStream_t s)
{
    if (bytes == 0) return cudaSuccess;
    const int grid = (int)std::min<int64_t>(256, ((int64_t)bytes + 255) / 256);
    k_zero_bytes<<<grid, 256, 0, s>>>(static_cast<unsigned char*>(dst), (int64_t)bytes);
    ++t_launches;
    return cudaGetLastError();
}

float elapsed(chem_ctx* c)
{
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
    return ms;
}

}  // namespace

extern "C" {

void chem_default_opts(chem_opts* o)
{
    if (!o) return;
    o->T_min = 500.0;
    o->kmax_bulk = 5;
    o->n_active_star = -1;      // auto: one resident wave of the integration kernel (37 888 on B200)
    o->kmax_sparse = 100000;
    o->atol_T = 1e-6;
    o->method = CHEM_METHOD_RODAS4;
    o->compact_bulk = 1;
    o->eps_change = 0.01;
    o->h0_factor = 0.01;
    o->lockstep = 2;
    o->kmax_first = 1;
    o->schedule_lpt = 2;
}

const char* chem_strerror(int code)
{
    switch (code) {
    case CHEM_OK: return "ok";
    case CHEM_EINVAL: return "invalid argument";
    case CHEM_EMECH: return "mechanism tables fail validation";
    case CHEM_ENOSTRUCT: return "mechanism reaction structure is not compiled into libchem (run gen_structure, rebuild)";
    case CHEM_ECUDA: return "CUDA error";
    case CHEM_ENOWS: return "workspace too small";
    default: return "unknown error";
    }
}

static int check_opts(const chem_opts* o)
{
    if (o->kmax_bulk < 1 || o->kmax_sparse < 1 || !(o->atol_T > 0.0) ||
        (o->method < CHEM_METHOD_RODAS4 || o->method > CHEM_METHOD_EXPLICIT) ||
        !std::isfinite(o->T_min) || !(o->eps_change > 0.0 && o->eps_change <= 1.0) ||
        o->lockstep < 0 || o->lockstep > 2 || o->kmax_first < 0 || o->schedule_lpt < 0 || o->schedule_lpt > 3 ||
        !(o->h0_factor > 0.0 && o->h0_factor <= 1.0) || (o->compact_bulk != 0 && o->compact_bulk != 1))
        return CHEM_EINVAL;
    return CHEM_OK;
}

int chem_init(const chem_mech_desc* mech, const chem_opts* opts, int device, chem_ctx** out)
{
    if (!out) return CHEM_EINVAL;
    *out = nullptr;
    int rc = validate(mech);
    if (rc != CHEM_OK) return rc;
    chem_opts o;
    chem_default_opts(&o);
    if (opts) o = *opts;
    if (check_opts(&o) != CHEM_OK) return CHEM_EINVAL;
    const Ops* ops = nullptr;
    for (const Ops& x : registry())
        if (x.match(mech)) { ops = &x; break; }
    if (!ops) return CHEM_ENOSTRUCT;
    if (cudaSetDevice(device) != cudaSuccess) return CHEM_ECUDA;
    chem_ctx* c = new (std::nothrow) chem_ctx();
    if (!c) return CHEM_ECUDA;
    c->device = device;
    c->ops = ops;
    c->opts = o;
    c->params.resize(ops->params_size);
    ops->fill(mech, c->params.data());
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (!alloc_mapped(c->h_stats, c->d_stats, S_NSTATS) || !alloc_mapped(c->h_sig, c->d_sig, 6) ||
        cudaEventCreate(&c->ev[0]) != cudaSuccess || cudaEventCreate(&c->ev[1]) != cudaSuccess ||
        ensure_host_boxes(c, 64) != CHEM_OK) {
        chem_finalize(c);
        return CHEM_ECUDA;
    }
    *out = c;
    return CHEM_OK;
}

void chem_finalize(chem_ctx* c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->h_boxes) cudaFreeHost(c->h_boxes);
    if (c->h_start) cudaFreeHost(c->h_start);
    if (c->h_stats) cudaFreeHost(c->h_stats);
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    if (c->h_sig) cudaFreeHost(c->h_sig);
    delete c;
}

const char* chem_structure_name(const chem_ctx* c) { return (c && c->ops) ? c->ops->name : ""; }

int chem_set_trace(chem_ctx* c, int32_t* trace, int32_t rows)
{
    if (!c || rows < 0 || (rows > 0 && !trace)) return CHEM_EINVAL;
    c->trace = rows > 0 ? trace : nullptr;
    c->trace_rows = rows;
    return CHEM_OK;
}

int chem_set_opts(chem_ctx* c, const chem_opts* o)
{
    if (!c || !o || check_opts(o) != CHEM_OK) return CHEM_EINVAL;
    c->opts = *o;
    return CHEM_OK;
}

size_t chem_workspace_bytes(const chem_ctx* c, int64_t max_cells, int32_t max_boxes)
{
    if (!c || max_cells < 0 || max_boxes < 1) return 0;
    return ws_layout(max_cells, max_boxes).total;
}

#define CHEM_PRE(c)                                        \
    do {                                                   \
        if (!(c)) return CHEM_EINVAL;                      \
        if ((c)->sticky) return (c)->sticky;               \
        if (cudaSetDevice((c)->device) != cudaSuccess) return CHEM_ECUDA; \
    } while (0)

int chem_rates(chem_ctx* c, int64_t n, int64_t ld, const double* rho, const double* T, const double* Y,
               double* wdot, void* stream)
{
    CHEM_PRE(c);
    if (n < 0 || ld < n || (n > 0 && (!rho || !T || !Y || !wdot))) return CHEM_EINVAL;
    return cuda_fail(c, c->ops->rates(c->params.data(), n, ld, rho, T, Y, wdot, (cudaStream_t)stream));
}

int chem_rhs(chem_ctx* c, int64_t n, int64_t ld, const double* rho, const double* T, const double* Y, double* f,
             void* stream)
{
    CHEM_PRE(c);
    if (n < 0 || ld < n || (n > 0 && (!rho || !T || !Y || !f))) return CHEM_EINVAL;
    return cuda_fail(c, c->ops->rhs(c->params.data(), n, ld, rho, T, Y, f, (cudaStream_t)stream));
}

int chem_jacobian(chem_ctx* c, int64_t n, int64_t ld, const double* rho, const double* T, const double* Y,
                  double* J, void* stream)
{
    CHEM_PRE(c);
    if (n < 0 || ld < n || (n > 0 && (!rho || !T || !Y || !J))) return CHEM_EINVAL;
    return cuda_fail(c, c->ops->jacobian(c->params.data(), n, ld, rho, T, Y, J, (cudaStream_t)stream));
}

int chem_temperature(chem_ctx* c, int64_t n, int64_t ld, const double* e, const double* Y, double* T, void* stream)
{
    CHEM_PRE(c);
    if (n < 0 || ld < n || (n > 0 && (!e || !Y || !T))) return CHEM_EINVAL;
    return cuda_fail(c, c->ops->temperature(c->params.data(), n, ld, e, Y, T, nullptr, (cudaStream_t)stream));
}

int chem_internal_energy(chem_ctx* c, int64_t n, int64_t ld, const double* U, double* e, void* stream)
{
    CHEM_PRE(c);
    if (n < 0 || ld < n || (n > 0 && (!U || !e))) return CHEM_EINVAL;
    if (n == 0) return CHEM_OK;
    k_internal_energy<<<grid_for(n, kPointBS), kPointBS, 0, (cudaStream_t)stream>>>(n, ld, U, e);
    return cuda_fail(c, cudaGetLastError());
}

int chem_energy(chem_ctx* c, int64_t n, int64_t ld, const double* T, const double* Y, double* e, void* stream)
{
    CHEM_PRE(c);
    if (n < 0 || ld < n || (n > 0 && (!e || !Y || !T))) return CHEM_EINVAL;
    return cuda_fail(c, c->ops->energy(c->params.data(), n, ld, T, Y, e, (cudaStream_t)stream));
}

int chem_cell_status(chem_ctx* c, const void* ws, size_t ws_bytes, int64_t first, int64_t n, int8_t* status,
                     int32_t* substeps, void* stream)
{
    CHEM_PRE(c);
    if (!ws || first < 0 || n < 0) return CHEM_EINVAL;
    const chem_ctx::WsRecord* rec = nullptr;
    for (const auto& r : c->ws_last)
        if (r.ws == ws) rec = &r;
    if (!rec || first + n > rec->total) return CHEM_EINVAL;
    const WsLayout W = ws_layout(rec->total, rec->nboxes);
    if (ws_bytes < W.total) return CHEM_ENOWS;
    if (n == 0) return CHEM_OK;
    if (!status && !substeps) return CHEM_OK;
    const char* base = static_cast<const char*>(ws);
    const uint8_t* state = reinterpret_cast<const uint8_t*>(base + W.state) + first;
    const int32_t* steps = reinterpret_cast<const int32_t*>(base + W.steps) + first;
    k_cell_status<<<grid_for(n, kStreamBS), kStreamBS, 0, (cudaStream_t)stream>>>(state, steps, n, status, substeps);
    return cuda_fail(c, cudaGetLastError());
}

int chem_box_active(chem_ctx* c, int32_t nboxes, const chem_box* boxes, int32_t* active, void* ws, size_t ws_bytes,
                    void* stream)
{
    CHEM_PRE(c);
    if (nboxes < 1 || !boxes || !active || !ws) return CHEM_EINVAL;
    for (int b = 0; b < nboxes; ++b)
        if (boxes[b].ncells < 0 || (boxes[b].ncells > 0 && !boxes[b].T)) return CHEM_EINVAL;
    if (ws_bytes < ws_layout(0, nboxes).total) return CHEM_ENOWS;
    if (ensure_host_boxes(c, nboxes) != CHEM_OK) return CHEM_ECUDA;
    cudaStream_t s = (cudaStream_t)stream;
    int64_t maxn = 0;
    for (int b = 0; b < nboxes; ++b) {
        const chem_box& x = boxes[b];
        c->h_boxes[b] = DevBox{x.rho, x.e, x.T, x.Y, x.solid, x.ncells, x.ld, x.dt};
        maxn = std::max(maxn, (int64_t)x.ncells);
    }
    char* base = static_cast<char*>(ws);
    const WsLayout W = ws_layout(0, nboxes);
    cudaError_t e;
    if ((e = copy_words(base + W.boxes, c->d_boxes, sizeof(DevBox) * nboxes, s)) != cudaSuccess ||
        (e = zero_bytes(active, sizeof(int32_t) * nboxes, s)) != cudaSuccess)
        return cuda_fail(c, e);
    const int slices = (int)std::max<int64_t>(1, std::min<int64_t>(64, (maxn + 4095) / 4096));
    k_box_active<kStreamBS><<<dim3(nboxes, slices), kStreamBS, 0, s>>>(reinterpret_cast<const DevBox*>(base + W.boxes),
                                                                      c->opts.T_min, active);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(c, e);
    return cuda_fail(c, cudaStreamSynchronize(s));   // the pinned box table is reused by the next call
}

int chem_integrate(chem_ctx* c, int64_t n, int64_t ld, const double* rho, const double* e, double* T, double* Y,
                   const uint8_t* solid, double dt, double rtol, double atol, void* ws, size_t ws_bytes,
                   chem_stats* stats, void* stream)
{
    chem_box b;
    b.rho = rho;
    b.e = e;
    b.T = T;
    b.Y = Y;
    b.solid = solid;
    b.ncells = n;
    b.ld = ld;
    b.dt = dt;
    return chem_integrate_boxes(c, 1, &b, rtol, atol, ws, ws_bytes, nullptr, stats, stream);
}

int chem_integrate_boxes(chem_ctx* c, int32_t nboxes, const chem_box* boxes, double rtol, double atol, void* ws,
                         size_t ws_bytes, double* box_cost, chem_stats* stats, void* stream)
{
    CHEM_PRE(c);
    NvtxScope nvtx_call("chem_integrate_boxes");
    if (nboxes < 1 || !boxes || !(rtol > 0.0) || !(atol > 0.0) || !ws) return CHEM_EINVAL;
    int64_t total = 0;
    for (int b = 0; b < nboxes; ++b) {
        const chem_box& x = boxes[b];
        if (x.ncells < 0 || x.ld < x.ncells || !(x.dt > 0.0) || !std::isfinite(x.dt)) return CHEM_EINVAL;
        if (x.ncells > 0 && (!x.rho || !x.e || !x.T || !x.Y)) return CHEM_EINVAL;
        total += x.ncells;
    }
    if (total >= (int64_t)0xffffffffLL) return CHEM_EINVAL;  // 32-bit cell index map
    const WsLayout W = ws_layout(total, nboxes);
    if (ws_bytes < W.total) return CHEM_ENOWS;
    {
        bool found = false;
        for (auto& r : c->ws_last)
            if (r.ws == ws) { r.total = total; r.nboxes = nboxes; found = true; }
        if (!found) {
            if (c->ws_last.size() >= 64) c->ws_last.erase(c->ws_last.begin());
            c->ws_last.push_back({ws, total, nboxes});
        }
    }
    if (ensure_host_boxes(c, nboxes) != CHEM_OK) return CHEM_ECUDA;
    cudaStream_t s = (cudaStream_t)stream;
    const chem_opts& o = c->opts;
    const Ops& ops = *c->ops;
    char* base = static_cast<char*>(ws);

    int64_t acc = 0;
    for (int b = 0; b < nboxes; ++b) {
        const chem_box& x = boxes[b];
        c->h_boxes[b] = DevBox{x.rho, x.e, x.T, x.Y, x.solid, x.ncells, x.ld, x.dt};
        c->h_start[b] = acc;
        acc += x.ncells;
    }
    c->h_start[nboxes] = acc;

    LaunchCtx L;
    L.boxes = reinterpret_cast<const DevBox*>(base + W.boxes);
    L.box_start = reinterpret_cast<const int64_t*>(base + W.start);
    L.nboxes = nboxes;
    L.total = total;
    L.cell_t = reinterpret_cast<double*>(base + W.cell_t);
    L.cell_h = reinterpret_cast<double*>(base + W.cell_h);
    L.state = reinterpret_cast<uint8_t*>(base + W.state);
    L.cell_steps = reinterpret_cast<int32_t*>(base + W.steps);
    L.cell_box = reinterpret_cast<int32_t*>(base + W.box);
    L.cell_hint = reinterpret_cast<int32_t*>(base + W.hint);
    L.stats = reinterpret_cast<unsigned long long*>(base + W.stats);
    L.rtol = rtol;
    L.atol = atol;
    L.atolT = o.atol_T;
    L.T_min = o.T_min;
    L.eps_change = o.eps_change;
    L.h0_factor = o.h0_factor;
    L.kmax_call = o.kmax_sparse;
    uint32_t* ids0 = reinterpret_cast<uint32_t*>(base + W.ids0);
    uint32_t* idsA = reinterpret_cast<uint32_t*>(base + W.idsA);
    uint32_t* idsB = reinterpret_cast<uint32_t*>(base + W.idsB);

    chem_stats st;
    std::memset(&st, 0, sizeof(st));
    st.cells = total;
    t_launches = 0;
    cudaError_t e;
#define CK(x)                                        \
    do {                                             \
        if ((e = (x)) != cudaSuccess) return cuda_fail(c, e); \
    } while (0)

    CK(copy_words(base + W.boxes, c->d_boxes, sizeof(DevBox) * nboxes, s));
    CK(copy_words(base + W.start, c->d_start, sizeof(int64_t) * (nboxes + 1), s));
    CK(zero_bytes(L.stats, S_SIG0 * 8, s));   // the layout signature slots persist across calls
    if (box_cost) CK(zero_bytes(box_cost, sizeof(double) * nboxes, s));
    if (total == 0) {
        CK(cudaStreamSynchronize(s));
        st.kernel_launches = t_launches;
        if (stats) *stats = st;
        return CHEM_OK;
    }

    auto read_count = [&](int64_t& v) -> cudaError_t {
        cudaError_t r = copy_words(c->d_stats, L.stats, S_NSTATS * 8, s);
        if (r != cudaSuccess) return r;
        r = cudaStreamSynchronize(s);
        v = (int64_t)c->h_stats[S_COUNT_ACTIVE];
        return r;
    };

    // ---- Alg. 3 §1: gate + count + index map
    nvtxMarkA("chem: gate");
    CK(cudaEventRecord(c->ev[0], s));
    uint32_t* key0 = reinterpret_cast<uint32_t*>(base + W.key0);
    uint32_t* key1 = reinterpret_cast<uint32_t*>(base + W.key1);
    k_gate<kStreamBS><<<grid_for(total, kStreamBS), kStreamBS, 0, s>>>(L, ids0, key0);
    ++t_launches;
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->ev[1], s));
    int64_t n_active = 0;
    CK(read_count(n_active));
    st.t_gate_ms = elapsed(c);
    st.active0 = n_active;
    const bool tracing = c->trace && c->trace_rows > 0;
    if (tracing) {
        CK(zero_bytes(c->trace, sizeof(int32_t) * (size_t)c->trace_rows * nboxes, s));
        if (n_active > 0) {
            k_box_count<kStreamBS><<<grid_for(n_active, kStreamBS), kStreamBS, 0, s>>>(L, ids0, n_active, c->trace);
            ++t_launches;
            CK(cudaGetLastError());
        }
    }

    // ---- Heavy-first schedule (chem_opts.schedule_lpt).  When the cost hints are
    // skewed (heavy cells, > kHeavySteps substeps last call, carry half the work, or the costs vary),
    // the round-robin bulk bursts would start the long chains late and leave them as the tail, and
    // mix short and long cells in one warp.  Instead the
    // index map is sorted by hint, heaviest first (stable LSD radix sort: ties keep gate order), and
    // the whole list runs as one persistent lockstep launch with warp-batched refill: the longest
    // chains start at once and light cells fill the slots that free up (longest-processing-time
    // first).  Per-cell arithmetic is unchanged, so results are bitwise those of the default.
    // The workspace's per-cell substep counts (left by the last call that used this workspace) are
    // this call's cost hints only if that call integrated the same cell layout: same total, box count
    // and first box, recorded in the workspace's signature slots (read with the count above).
    const unsigned long long sig[3] = {(unsigned long long)total, (unsigned long long)nboxes,
                                       (unsigned long long)(uintptr_t)boxes[0].rho};
    const bool history = c->h_stats[S_SIG0] == sig[0] && c->h_stats[S_SIG1] == sig[1] && c->h_stats[S_SIG2] == sig[2];
    // hint accuracy of this layout's previous call (sum min / sum max of hint vs actual substeps over
    // its cells), valid if that call had hints of its own; then reset the slots for this call
    const bool acc_known = history && c->h_stats[S_HINT_VALID] == 1 && c->h_stats[S_HINT_MAX] > 0;
    const double acc_prev = acc_known ? (double)c->h_stats[S_HINT_MIN] / (double)c->h_stats[S_HINT_MAX] : -1.0;
    std::memcpy(c->h_sig, sig, sizeof(sig));
    c->h_sig[3] = 0;
    c->h_sig[4] = 0;
    c->h_sig[5] = history ? 1 : 0;
    static_assert(S_HINT_MIN == S_SIG2 + 1 && S_HINT_VALID == S_SIG2 + 3, "signature + hint slots are contiguous");
    CK(copy_words(L.stats + S_SIG0, c->d_sig, 6 * sizeof(unsigned long long), s));
    const uint64_t pred_total = c->h_stats[S_PRED_TOTAL], pred_heavy = c->h_stats[S_PRED_HEAVY];
    const uint64_t pred_max = c->h_stats[S_PRED_MAX];
    const bool eligible = n_active > 0 && o.method != CHEM_METHOD_EXPLICIT;
    // hints that vary (max above 1.5x the mean) or put half the work in heavy cells
    const bool skewed = history && pred_total > 0 &&
                        (2 * pred_heavy >= pred_total ||
                         (double)pred_max * (double)n_active > 1.5 * (double)pred_total);
    // auto: skewed hints that have been predictive (or whose predictiveness is not known yet)
    bool lpt = eligible && (o.schedule_lpt == 1 ||
                            (o.schedule_lpt == 2 && skewed && (!acc_known || acc_prev >= kHintAcc)));
    // otherwise (auto, or schedule_lpt = 3) the cells predict their own cost after the first burst
    const bool predict = eligible && !lpt && (o.schedule_lpt == 2 || o.schedule_lpt == 3);
    st.lpt = lpt ? 1 : 0;
    const uint32_t* cur = ids0;
    int64_t n_cur = n_active;
    uint32_t* nxt = idsA;
    // heavy-first order: stable counting sort of the list into cost buckets, heaviest first
    // (k_bucket_*); the per-tile histogram lives in the workspace's key1 section (n/4 entries)
    auto sort_desc = [&](const uint32_t* keys, const uint32_t* ids_in, int64_t n, uint32_t* ids_out) -> cudaError_t {
        unsigned* hist = reinterpret_cast<unsigned*>(key1);
        const int ntiles = (int)((n + kSortTile - 1) / kSortTile);
        k_bucket_hist<<<ntiles, kSortBS, 0, s>>>(keys, n, hist, ntiles);
        ++t_launches;
        k_scan_excl<<<1, 1024, 0, s>>>(hist, (int64_t)ntiles * kCostBuckets);
        ++t_launches;
        k_bucket_scatter<<<ntiles, kSortBS, 0, s>>>(keys, ids_in, n, hist, ntiles, ids_out);
        ++t_launches;
        return cudaGetLastError();
    };
    if (lpt) {
        // ids0 (the gate's list) stays intact for the box cost: the sorted list goes to idsA
        CK(sort_desc(key0, ids0, n_active, idsA));
        cur = idsA;
        nxt = idsB;
    }

    // ---- Alg. 3 §2: bulk bursts while N_active > N*
    nvtxMarkA("chem: bulk");
    // lockstep bursts (chem_opts.lockstep; auto: the previous call's bulk SIMT efficiency was low)
    const bool lock = o.method != CHEM_METHOD_EXPLICIT &&
                      (o.lockstep == 1 || (o.lockstep == 2 && c->simt_eff < kLockEff));
    st.lockstep = lock;
    unsigned long long att_skip = 0, ws_skip = 0;   // the one-substep first burst is not a SIMT sample
    // N* (P:181): negative = one resident wave of the integration kernel (SMs x resident cells per SM):
    // below it a bulk burst can no longer fill the GPU, so the persistent sparse launch takes over
    // (B200 sweep, profiles/r01_nstar_sweep.txt; the paper's 1e4 was tuned on H100).
    const int64_t wave = (int64_t)c->num_sms * ops.blocks_per_sm(o.method) * kIntegrateBS;   // resident cells
    const int64_t nstar = o.n_active_star >= 0 ? o.n_active_star : wave;
    while (!lpt && n_cur > nstar && n_cur > 0) {
        const bool first_burst = lock && st.bulk_iters == 0 && o.kmax_first > 0;
        const int kmax_b = first_burst ? o.kmax_first : o.kmax_bulk;
        const bool all_cells = !o.compact_bulk;
        const uint32_t* lst = all_cells ? nullptr : cur;
        const int64_t nl = all_cells ? total : n_cur;
        CK(cudaEventRecord(c->ev[0], s));
        ++t_launches;
        if (lock)
            CK(ops.integrate_lock(c->params.data(), o.method, L, lst, nl, kmax_b, 0, 0, c->num_sms, s));
        else
            CK(ops.integrate(c->params.data(), o.method, L, lst, nl, kmax_b, 0, 0,
                             (int)((nl + kIntegrateBS - 1) / kIntegrateBS), s));
        CK(cudaEventRecord(c->ev[1], s));
        CK(cudaEventSynchronize(c->ev[1]));
        st.t_bulk_ms += elapsed(c);
        CK(cudaEventRecord(c->ev[0], s));
        CK(zero_bytes(L.stats + S_COUNT_ACTIVE, 8, s));
        k_compact<kStreamBS><<<grid_for(nl, kStreamBS), kStreamBS, 0, s>>>(L, lst, nl, nxt);
        ++t_launches;
        CK(cudaGetLastError());
        CK(cudaEventRecord(c->ev[1], s));
        CK(read_count(n_cur));
        st.t_compact_ms += elapsed(c);
        if (first_burst) {
            att_skip = c->h_stats[S_ATTEMPTED];
            ws_skip = c->h_stats[S_WARP_SUBSTEPS];
        }
        if (st.bulk_iters < 16) st.active_per_iter[st.bulk_iters] = n_cur;
        st.bulk_iters++;
        if (tracing && st.bulk_iters < c->trace_rows && n_cur > 0) {
            k_box_count<kStreamBS><<<grid_for(n_cur, kStreamBS), kStreamBS, 0, s>>>(
                L, nxt, n_cur, c->trace + (size_t)st.bulk_iters * nboxes);
            ++t_launches;
            CK(cudaGetLastError());
        }
        cur = nxt;
        nxt = (nxt == idsA) ? idsB : idsA;
        // (the order matters only while more cells remain than one resident wave holds)
        if (predict && st.bulk_iters == 1 && n_cur > 0 && (o.schedule_lpt == 3 || n_cur > wave)) {
            // heavy-first on in-call predictions: the remaining substeps (dt - t)/h of every cell still
            // active after the first burst; skewed (max > 1.5 mean) or forced -> sort, one persistent launch
            CK(zero_bytes(L.stats + S_PRED2_TOTAL, 16, s));
            k_predict<kStreamBS><<<grid_for(n_cur, kStreamBS), kStreamBS, 0, s>>>(L, cur, n_cur, key0);
            ++t_launches;
            CK(cudaGetLastError());
            int64_t dummy;
            CK(read_count(dummy));
            const uint64_t p_tot = c->h_stats[S_PRED2_TOTAL], p_max = c->h_stats[S_PRED2_MAX];
            if (o.schedule_lpt == 3 || (double)p_max * (double)n_cur > 1.5 * (double)p_tot) {
                CK(sort_desc(key0, cur, n_cur, nxt));             // cur is idsA or idsB, never ids0
                cur = nxt;
                nxt = (cur == idsA) ? idsB : idsA;
                lpt = true;
                st.lpt = 2;
                break;
            }
        }
    }

    if (st.bulk_iters > 0) {
        st.bulk_substeps = (int64_t)c->h_stats[S_ATTEMPTED];
        st.warp_substeps = (int64_t)c->h_stats[S_WARP_SUBSTEPS];
        const unsigned long long ws = c->h_stats[S_WARP_SUBSTEPS] - ws_skip;
        if (ws > 0) c->simt_eff = (double)(c->h_stats[S_ATTEMPTED] - att_skip) / (32.0 * (double)ws);
    }

    // ---- Alg. 3 §3: sparse integration over the index map (persistent, lane refill)
    nvtxMarkA("chem: sparse");
    st.sparse_cells = n_cur;
    if (n_cur > 0) {
        CK(zero_bytes(L.stats + S_CURSOR, 8, s));
        CK(cudaEventRecord(c->ev[0], s));
        if (st.lpt == 1) {
            // heavy-first on the previous call's hints: the whole active list, light cells included, as
            // persistent lockstep blocks (one per SM) with lane refill - a free-running refill grid costs
            // 1-substep cells their coalesced loads (cfg5 at the production tolerance 507 vs 345, r02)
            ++t_launches;
            CK(ops.integrate_lock(c->params.data(), o.method, L, cur, n_cur, o.kmax_sparse, kRefillSorted, 1,
                                  c->num_sms, s));
        } else {
            // the sparse list (after the bursts; sorted heaviest first under the in-call prediction) on
            // the free-running persistent grid with lane refill (lockstep costs 2-7 % here, r02t)
            const int grid = std::max(1, std::min<int>(c->num_sms * ops.blocks_per_sm(o.method),
                                                       (int)((n_cur + kIntegrateBS - 1) / kIntegrateBS)));
            ++t_launches;
            CK(ops.integrate(c->params.data(), o.method, L, cur, n_cur, o.kmax_sparse,
                             lpt ? kRefillSorted : kRefillUnsorted, 1, grid, s));
        }
        CK(cudaEventRecord(c->ev[1], s));
    }
    if (box_cost && n_active > 0) {
        k_box_cost<kStreamBS><<<grid_for(n_active, kStreamBS), kStreamBS, 0, s>>>(L, ids0, n_active, box_cost);
        ++t_launches;
        CK(cudaGetLastError());
    }
    CK(copy_words(c->d_stats, L.stats, S_NSTATS * 8, s));
    CK(cudaStreamSynchronize(s));
    if (n_cur > 0) st.t_sparse_ms = elapsed(c);
    const unsigned long long* hs = c->h_stats;
    st.steps_attempted = (int64_t)hs[S_ATTEMPTED];
    st.steps_accepted = (int64_t)hs[S_ACCEPTED];
    st.steps_frozen = (int64_t)hs[S_FROZEN];
    st.rhs_evals = (int64_t)hs[S_RHS];
    st.jac_evals = (int64_t)hs[S_JAC];
    st.lu_count = (int64_t)hs[S_LU];
    st.n_newton_fail = (int64_t)hs[S_NEWTON_FAIL];
    st.n_nonfinite = (int64_t)hs[S_NONFINITE];
    st.n_T_range = (int64_t)hs[S_TRANGE];
    st.n_unfinished = (int64_t)hs[S_UNFINISHED];
    st.hint_accuracy = (history && hs[S_HINT_MAX] > 0) ? (double)hs[S_HINT_MIN] / (double)hs[S_HINT_MAX] : -1.0;
    unsigned long long db = hs[S_DRIFT_BITS];
    std::memcpy(&st.max_energy_drift, &db, 8);
    st.kernel_launches = t_launches;
    if (stats) *stats = st;
#undef CK
    return CHEM_OK;
}

}  // extern "C"
