// runtime.cu -- libpdd host runtime: the C ABI of include/pdd.h.
//
// Owns the device state carved from a caller-provided workspace, enqueues the kernels of
// canonical.cu / sweep.cu on the caller's stream, and drives the two loops of the method:
//   * the coarse Jacobi solve: batches of self-stopping sweeps, residual history
//     on the device, one 4-byte readback per batch;
//   * the fine solve: rounds of {activation / compaction -> tile sweep kernel}
//     with one 24-byte counter readback per round, patchy bucket threshold (P:744-749,
//     P:831), and a full-grid Jacobi verification pass when no tile is active.
#include "../../include/pdd.h"
#include "pdd_internal.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

using namespace pdd;

namespace {

thread_local std::string g_err;

// A/B switches of the development builds only: the product library (built without PDD_DEV) reads
// no environment variable, so a stray variable cannot change its schedule or tile geometry.
#ifndef PDD_DEV
#define PDD_DEV 0
#endif
const char *dev_env(const char *name)
{
#if PDD_DEV
    return std::getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

// Every entry point runs on the device that owns the context's workspace, whatever device the
// calling thread has current (a second GPU in the same process), and restores the caller's.
struct DevGuard {
    int prev = -1, dev = -1;
    explicit DevGuard(int d) : dev(d)
    {
        if (d < 0) return;
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != d) cudaSetDevice(d);
    }
    ~DevGuard()
    {
        if (dev >= 0 && prev >= 0 && prev != dev) cudaSetDevice(prev);
    }
};

constexpr size_t kAlign = 256;
constexpr int kMaxPatches = 32768;
constexpr int64_t kMaxCoarseSweeps = 1 << 20;

size_t coef_count(const pdd_coef &c, int n)
{
    switch (c.kind) {
    case PDD_COEF_ROW:
    case PDD_COEF_COL: return (size_t)n;
    case PDD_COEF_FIELD: return (size_t)n * n;
    default: return 0;
    }
}

struct Carver {
    char *base;
    size_t off = 0;
    explicit Carver(void *b) : base((char *)b) {}
    template <class T>
    T *take(size_t count)
    {
        off = (off + kAlign - 1) / kAlign * kAlign;
        T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
        off += count * sizeof(T);
        return p;
    }
};

// device copies of one problem
struct ProbBufs {
    DProblem d;
    double *ctrl = nullptr;
    double *coef[8] = {nullptr};   // speed, drift0, drift1, s00, s01, s10, s11, cost
    uint8_t *kind = nullptr;
    int16_t *sector = nullptr;
    double *cost_ctrl = nullptr;   // N_A (or null)
};

const pdd_coef *coef_ptr(const pdd_problem *p, int k)
{
    switch (k) {
    case 0: return &p->speed;
    case 1: return &p->drift[0];
    case 2: return &p->drift[1];
    case 3: return &p->sigma[0][0];
    case 4: return &p->sigma[0][1];
    case 5: return &p->sigma[1][0];
    case 6: return &p->sigma[1][1];
    default: return &p->cost;
    }
}

void carve_problem(Carver &cv, const pdd_problem *p, ProbBufs &b, bool with_sector)
{
    const int n = p->n;
    b.ctrl = cv.take<double>(2 * (size_t)p->n_controls);
    for (int k = 0; k < 8; ++k) {
        const size_t c = coef_count(*coef_ptr(p, k), n);
        b.coef[k] = c ? cv.take<double>(c) : nullptr;
    }
    b.kind = cv.take<uint8_t>((size_t)n * n);
    b.sector = with_sector ? cv.take<int16_t>((size_t)n * n) : nullptr;
    b.cost_ctrl = p->cost_ctrl ? cv.take<double>((size_t)p->n_controls) : nullptr;
}

int na_pad_of(int na) { return na <= 32 ? 32 : (na <= 64 ? 64 : 0); }

}  // namespace

struct pdd_ctx {
    std::string err;
    cudaStream_t stream = nullptr;
    int precision = 32;
    bool owns_nothing = true;
    pdd_problem fine{}, coarse{};
    bool has_coarse = false;
    ProbBufs F, Cc;
    // fine fields
    double *V = nullptr, *uhat = nullptr, *uc[2] = {nullptr, nullptr};
    double *uc_final = nullptr;
    uint8_t *astar = nullptr;
    int16_t *labels = nullptr;
    int32_t *succ0 = nullptr, *succA = nullptr, *succB = nullptr;
    float *f32buf = nullptr;
    unsigned long long *res_hist = nullptr;
    uint8_t *cflag = nullptr;   // coarse active-tile change flags, 2 x tiles
    CoarseRowEntry *crowtab = nullptr;   // coarse row-invariant table (n_c x N_A)
    CoarseRowEntry *frowtab = nullptr;   // the same for the fine-grid synthesis (n x N_A)
    bool coarse_rowuniform = false, fine_rowuniform = false;
    bool coarse_stage = false;   // coarse reach + 1 <= staged halo
    bool synth_stage = false;    // fine sigma = 0 reach + 1 <= staged halo (synthesis)
    bool coarse_tiled = false;  // coarse reach < tile: active-tile sweeps
    // fine-problem quantities that need the caller's host arrays: computed once in pdd_create
    // (those arrays are only valid during that call; ctx->fine / ctx->coarse keep no pointers)
    double fine_reach = 0.0;
    int fine_halo = 0;
    bool fine_row_uniform_all = false;   // row_uniform(): speed, drift, sigma and cost
    int *dev_int = nullptr;     // [0] sweeps_done, [1] jump changed flag
    void *rowtab = nullptr;
    size_t rowtab_bytes = 0;
    TileState T{};
    int max_tiles = 0;
    // work-queue schedule (schedule 2)
    bool prepared_queue_ok = false;
    QueueCtl *qctl = nullptr;
    int32_t *qring = nullptr;
    unsigned qcap = 0;
    int *qstate = nullptr;
    int32_t *qrank = nullptr;
    int32_t *qscratch = nullptr;
    double *outbuf = nullptr;
    // host pinned
    ActCounters *h_cnt = nullptr;
    int *h_int = nullptr;
    RoundCtl *rctl = nullptr;      // device round state (workspace)
    RoundCtl *h_ctl = nullptr;     // pinned host mirror
    // state
    bool coarse_done = false, synth_done = false;
    int labels_mode = 0;        // 0 none, 1 patchy, 2 static
    int n_patches = 0;
    int n_patch_slots = 0;
    int static_px = 1, static_py = 1;
    // sweep configuration
    int path = 0, WY = 0, WX = 0, Hx = 0;
    TileGeom g{};
    int n_tiles = 0;
    int prepared_kernel = -1;
    int prepared_geo = -1;           // path-3 tile of the prepared geometry (p3_geometry_choice)
    int force_tile_rows = 0;         // pdd_set_tile_shape: 0 auto, 16 or 32
    int force_tile_cols = 0;         // pdd_set_tile_cols: 0 auto, 64 or 128
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t evp[2][64] = {};  // per-round sweep-kernel timing inside a batch (lazy)
    long long launches = 0;     // kernels enqueued by this context (all calls)
    int device = -1;            // device ordinal of the workspace (DevGuard)
    bool mode_patchy = false;   // the current pdd_solve runs the patchy decomposition
};

static pdd_status fail(pdd_ctx *c, pdd_status s, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    else g_err = buf;
    return s;
}

#define CK(call)                                                                             \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail(ctx, PDD_E_CUDA, "%s failed: %s (%s:%d)", #call,                     \
                        cudaGetErrorString(e_), __FILE__, __LINE__);                         \
    } while (0)

#define CK0(call)                                                                            \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail(nullptr, PDD_E_CUDA, "%s failed: %s (%s:%d)", #call,                 \
                        cudaGetErrorString(e_), __FILE__, __LINE__);                         \
    } while (0)

static pdd_status validate(const pdd_problem *p, const char *what)
{
    if (!p) return fail(nullptr, PDD_E_INVALID, "%s problem is NULL", what);
    if (p->n < 3) return fail(nullptr, PDD_E_INVALID, "%s: n = %d < 3", what, p->n);
    if (!(p->hi > p->lo)) return fail(nullptr, PDD_E_INVALID, "%s: hi <= lo", what);
    if (!(p->dx > 0.0) || !(p->h > 0.0))
        return fail(nullptr, PDD_E_INVALID, "%s: dx and h must be > 0", what);
    if (!(p->lambda >= 0.0)) return fail(nullptr, PDD_E_INVALID, "%s: lambda must be >= 0", what);
    if (p->sigma_mode != 0 && p->sigma_mode != 1)
        return fail(nullptr, PDD_E_INVALID, "%s: sigma_mode must be 0 or 1", what);
    if (p->sigma_mode == 1 && p->p != 1)
        return fail(nullptr, PDD_E_INVALID, "%s: sigma_mode 1 (sigma(x,a) = s(x) a) needs p = 1", what);
    if (p->n_controls < 1 || p->n_controls > 128)
        return fail(nullptr, PDD_E_INVALID, "%s: N_A = %d outside 1..128", what, p->n_controls);
    if (!p->controls) return fail(nullptr, PDD_E_INVALID, "%s: controls is NULL", what);
    if (p->p < 0 || p->p > 2) return fail(nullptr, PDD_E_INVALID, "%s: p = %d outside 0..2", what, p->p);
    if (!p->kind) return fail(nullptr, PDD_E_INVALID, "%s: kind is NULL", what);
    for (int k = 0; k < 8; ++k) {
        const pdd_coef *c = coef_ptr(p, k);
        if (c->kind < 0 || c->kind > 3) return fail(nullptr, PDD_E_INVALID, "%s: bad coef kind", what);
        if (c->kind != PDD_COEF_CONST && !c->data)
            return fail(nullptr, PDD_E_INVALID, "%s: coefficient %d has NULL data", what, k);
    }
    // l(x, a) = l(x) + m(a) > 0 (R33)
    double mmin = 0.0;
    if (p->cost_ctrl) {
        mmin = INFINITY;
        for (int k = 0; k < p->n_controls; ++k) {
            if (!std::isfinite(p->cost_ctrl[k]))
                return fail(nullptr, PDD_E_INVALID, "%s: cost_ctrl must be finite", what);
            mmin = std::min(mmin, p->cost_ctrl[k]);
        }
    }
    const pdd_coef &l = p->cost;
    const size_t cnt = coef_count(l, p->n);
    if (cnt == 0) {
        if (!(l.value + mmin > 0.0)) return fail(nullptr, PDD_E_INVALID, "%s: running cost must be > 0", what);
    } else {
        for (size_t i = 0; i < cnt; ++i)
            if (!(l.data[i] + mmin > 0.0)) return fail(nullptr, PDD_E_INVALID, "%s: running cost must be > 0", what);
    }
    // exit problems (lambda = 0): the obstacle value 1/lambda does not exist (R8)
    if (p->lambda == 0.0)
        for (size_t k = 0; k < (size_t)p->n * p->n; ++k)
            if (p->kind[k] == 2)
                return fail(nullptr, PDD_E_INVALID, "%s: obstacles need lambda > 0", what);
    return PDD_OK;
}

static bool row_uniform(const pdd_problem *p);

static double coef_max_abs(const pdd_coef &c, int n)
{
    const size_t cnt = coef_count(c, n);
    if (!cnt) return std::fabs(c.value);
    double m = 0.0;
    for (size_t i = 0; i < cnt; ++i) m = std::max(m, std::fabs(c.data[i]));
    return m;
}

// reach of the foot points in cells (R4): (h max|f| + sc max|sigma_j|)/dx
static double reach_cells(const pdd_problem *p)
{
    double amax = 0.0;
    for (int k = 0; k < p->n_controls; ++k)
        amax = std::max(amax, std::hypot(p->controls[2 * k], p->controls[2 * k + 1]));
    const double fmax = coef_max_abs(p->speed, p->n) * amax +
                        std::hypot(coef_max_abs(p->drift[0], p->n), coef_max_abs(p->drift[1], p->n));
    double smax = 0.0;
    if (p->p > 0) {
        const double sc = p->diffusion_scale == 0 ? std::sqrt(p->h * p->p) : std::sqrt(p->h);
        if (p->sigma_mode == 1)
            smax = sc * coef_max_abs(p->sigma[0][0], p->n) * amax;
        else
            for (int k = 0; k < p->p; ++k)
                smax = std::max(smax, sc * std::hypot(coef_max_abs(p->sigma[k][0], p->n),
                                                      coef_max_abs(p->sigma[k][1], p->n)));
    }
    return (p->h * fmax + smax) / p->dx;
}

static int halo_of(const pdd_problem *p)
{
    const double r = reach_cells(p);
    return (int)std::floor(r * (1.0 + 1e-9) + 1e-9) + 2;
}

static void make_dproblem(const pdd_problem *p, ProbBufs &b)
{
    DProblem &d = b.d;
    d.n = p->n;
    d.lo = p->lo;
    d.dx = p->dx;
    d.h = p->h;
    d.lambda = p->lambda;
    d.beta = 1.0 / (1.0 + p->lambda * p->h);
    d.q = p->h / p->dx;
    d.sc = p->p > 0 ? (p->diffusion_scale == 0 ? std::sqrt(p->h * (double)p->p) : std::sqrt(p->h)) / p->dx
                    : 0.0;
    double lmax = 0.0;
    const size_t cl = coef_count(p->cost, p->n);
    if (!cl) lmax = p->cost.value;
    else for (size_t i = 0; i < cl; ++i) lmax = std::max(lmax, p->cost.data[i]);
    d.lmax_x = lmax;
    if (p->cost_ctrl) {
        double mmax = -INFINITY;
        for (int k = 0; k < p->n_controls; ++k) mmax = std::max(mmax, p->cost_ctrl[k]);
        lmax = lmax + mmax;
    }
    d.lmax = lmax;
    // canonical: same expressions as the oracle; exit problems (lambda = 0) start at the "very
    // big value" of P:818-819 (R11)
    d.v0 = p->lambda > 0.0 ? (p->h * lmax) / (1.0 - d.beta) : 1e6;
    d.sigma_mode = p->sigma_mode;
    d.cost_ctrl = b.cost_ctrl;
    d.na = p->n_controls;
    d.ctrl = b.ctrl;
    DCoef *dc[8] = {&d.speed, &d.drift[0], &d.drift[1], &d.sigma[0][0], &d.sigma[0][1],
                    &d.sigma[1][0], &d.sigma[1][1], &d.cost};
    for (int k = 0; k < 8; ++k) {
        const pdd_coef *c = coef_ptr(p, k);
        dc[k]->kind = c->kind;
        dc[k]->value = c->value;
        dc[k]->data = b.coef[k];
    }
    d.p = p->p;
    d.kind = b.kind;
}

static size_t layout(pdd_ctx *c, void *ws, const pdd_problem *f, const pdd_problem *cp)
{
    Carver cv(ws);
    const int n = f->n;
    const size_t N = (size_t)n * n;
    ProbBufs F, Cc;
    carve_problem(cv, f, F, f->sector != nullptr);
    if (cp) carve_problem(cv, cp, Cc, false);
    double *V = cv.take<double>(N);
    double *uhat = cp ? cv.take<double>(N) : nullptr;
    double *uc0 = cp ? cv.take<double>((size_t)cp->n * cp->n) : nullptr;
    double *uc1 = cp ? cv.take<double>((size_t)cp->n * cp->n) : nullptr;
    unsigned long long *rh = cp ? cv.take<unsigned long long>(kMaxCoarseSweeps) : nullptr;
    const int ctn = cp ? (cp->n + coarse_tile() - 1) / coarse_tile() : 0;
    uint8_t *cflag = cp ? cv.take<uint8_t>(2 * (size_t)ctn * ctn) : nullptr;
    CoarseRowEntry *crt = cp ? cv.take<CoarseRowEntry>((size_t)cp->n * cp->n_controls) : nullptr;
    CoarseRowEntry *frt = cp ? cv.take<CoarseRowEntry>((size_t)n * f->n_controls) : nullptr;
    uint8_t *astar = cv.take<uint8_t>(N);
    int16_t *labels = cv.take<int16_t>(N);
    int32_t *s0 = cp ? cv.take<int32_t>(N) : nullptr;
    int32_t *sA = cp ? cv.take<int32_t>(N) : nullptr;
    int32_t *sB = cp ? cv.take<int32_t>(N) : nullptr;
    float *f32 = cv.take<float>(N);                     // fp32 staging for pdd_get_values
    int *di = cv.take<int>(8);
    const int napad = na_pad_of(f->n_controls);
    const size_t rtb = napad ? (size_t)n * napad * 160 : 0;   // >= sizeof(RowEntry<double,4,4>)
    void *rt = rtb ? cv.take<unsigned char>(rtb) : nullptr;
    const int tmax = ((n + 15) / 16) * ((n + 31) / 32);   // tiles >= 16 rows x 32 columns
    TileState T{};
    T.tile_free = cv.take<int32_t>(tmax);
    T.tile_minu = cv.take<double>(tmax);
    T.tile_res = cv.take<double>(tmax);
    T.tile_chg = cv.take<double>(tmax);
    T.tile_edge = cv.take<float>(4 * (size_t)tmax);
    T.tile_lab_cnt = cv.take<int32_t>(tmax);
    T.tile_lab_off = cv.take<int32_t>((size_t)tmax + 1);
    T.tile_lab_ids = cv.take<int16_t>(N);   // a tile has at most as many labels as nodes
    T.tile_lab_cap = (int64_t)32 * tmax;    // per-entry residuals of the partial verifications
    T.tile_lab_res = cv.take<unsigned long long>((size_t)T.tile_lab_cap);
    T.tile_round = cv.take<int32_t>(tmax);
    T.tile_orient = cv.take<uint8_t>(tmax);
    T.tile_stamp = cv.take<int32_t>(tmax);
    T.tile_sweeps = cv.take<int32_t>(tmax);
    T.list[0] = cv.take<int32_t>(tmax);
    T.list[1] = cv.take<int32_t>(tmax);
    T.all_list = cv.take<int32_t>(tmax);
    T.patch_round = cv.take<int32_t>(kMaxPatches + 1);
    T.patch_res = cv.take<unsigned long long>(kMaxPatches + 1);
    T.counters = cv.take<ActCounters>(1);
    T.tile_key = cv.take<double>(tmax);
    T.tile_group = cv.take<int32_t>(tmax);
    T.order = cv.take<int32_t>(tmax);
    T.done = cv.take<int>(tmax);
    T.stamp = cv.take<long long>(tmax);
    T.ocounters = cv.take<OrdCounters>(1);
    RoundCtl *rctl = cv.take<RoundCtl>(1);
    unsigned qcap = 1;   // > tiles + resident sweep CTAs (ticket ring, sweep.cu)
    while (qcap < 2u * (unsigned)tmax + 8192u) qcap <<= 1;
    QueueCtl *qctl = cv.take<QueueCtl>(1);
    int32_t *qring = cv.take<int32_t>(qcap);
    int *qstate = cv.take<int>(tmax);
    int32_t *qrank = cv.take<int32_t>(tmax);
    int32_t *qscr = cv.take<int32_t>(queue_order_scratch_ints());
    if (c) {
        c->rctl = rctl;
        c->qctl = qctl;
        c->qring = qring;
        c->qcap = qcap;
        c->qstate = qstate;
        c->qrank = qrank;
        c->qscratch = qscr;
        c->F = F;
        c->Cc = Cc;
        c->V = V;
        c->uhat = uhat;
        c->uc[0] = uc0;
        c->uc[1] = uc1;
        c->res_hist = rh;
        c->cflag = cflag;
        c->crowtab = crt;
        c->frowtab = frt;
        c->astar = astar;
        c->labels = labels;
        c->succ0 = s0;
        c->succA = sA;
        c->succB = sB;
        c->f32buf = f32;
        c->dev_int = di;
        c->rowtab = rt;
        c->rowtab_bytes = rtb;
        c->T = T;
        c->max_tiles = tmax;
    }
    return cv.off + kAlign;
}

extern "C" {

const char *pdd_version(void) { return "pdd-b200 0.1 (sm_100a)"; }

const char *pdd_last_error(const pdd_ctx *ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

long long pdd_kernel_launches(const pdd_ctx *ctx) { return ctx ? ctx->launches : 0; }

pdd_status pdd_workspace_bytes(const pdd_problem *fine, const pdd_problem *coarse,
                               int32_t precision, size_t *bytes)
{
    pdd_status s = validate(fine, "fine");
    if (s != PDD_OK) return s;
    if (coarse && (s = validate(coarse, "coarse")) != PDD_OK) return s;
    if (precision != 32 && precision != 64)
        return fail(nullptr, PDD_E_INVALID, "precision must be 32 or 64");
    if (!bytes) return fail(nullptr, PDD_E_INVALID, "bytes is NULL");
    *bytes = layout(nullptr, nullptr, fine, coarse);
    return PDD_OK;
}

static pdd_status copy_problem(pdd_ctx *ctx, const pdd_problem *p, ProbBufs &b, bool sector)
{
    const int n = p->n;
    CK(cudaMemcpyAsync(b.ctrl, p->controls, sizeof(double) * 2 * p->n_controls,
                       cudaMemcpyHostToDevice, ctx->stream));
    for (int k = 0; k < 8; ++k) {
        const pdd_coef *c = coef_ptr(p, k);
        const size_t cnt = coef_count(*c, n);
        if (cnt) CK(cudaMemcpyAsync(b.coef[k], c->data, sizeof(double) * cnt,
                                    cudaMemcpyHostToDevice, ctx->stream));
    }
    CK(cudaMemcpyAsync(b.kind, p->kind, (size_t)n * n, cudaMemcpyHostToDevice, ctx->stream));
    if (p->cost_ctrl)
        CK(cudaMemcpyAsync(b.cost_ctrl, p->cost_ctrl, sizeof(double) * p->n_controls,
                           cudaMemcpyHostToDevice, ctx->stream));
    if (sector && b.sector)
        CK(cudaMemcpyAsync(b.sector, p->sector, sizeof(int16_t) * n * n, cudaMemcpyHostToDevice,
                           ctx->stream));
    make_dproblem(p, b);
    return PDD_OK;
}

pdd_status pdd_create(const pdd_problem *fine, const pdd_problem *coarse, int32_t precision,
                      void *stream, void *workspace, size_t workspace_bytes, pdd_ctx **out)
{
    if (!out) return fail(nullptr, PDD_E_INVALID, "out is NULL");
    *out = nullptr;
    size_t need = 0;
    pdd_status s = pdd_workspace_bytes(fine, coarse, precision, &need);
    if (s != PDD_OK) return s;
    if (!workspace) return fail(nullptr, PDD_E_INVALID, "workspace is NULL");
    if (workspace_bytes < need)
        return fail(nullptr, PDD_E_NOMEM, "workspace of %zu bytes < %zu needed", workspace_bytes, need);
    if (coarse) {
        if (coarse->lo != fine->lo || coarse->hi != fine->hi)
            return fail(nullptr, PDD_E_INVALID, "coarse and fine boxes differ");
        if ((fine->n - 1) % (coarse->n - 1) != 0)
            return fail(nullptr, PDD_E_INVALID, "coarse grid (n=%d) does not nest in fine grid (n=%d)",
                        coarse->n, fine->n);
        if (coarse->p != 0)
            return fail(nullptr, PDD_E_INVALID, "the coarse problem must have sigma = 0 (p = 0), P:825");
    }
    pdd_ctx *ctx = new pdd_ctx();
    ctx->stream = (cudaStream_t)stream;
    {
        // the device that owns the workspace becomes the context's device
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, workspace) == cudaSuccess && pa.type == cudaMemoryTypeDevice)
            ctx->device = pa.device;
        else
            cudaGetLastError();   // not a device pointer known to the runtime: keep the current device
    }
    DevGuard dev_guard(ctx->device);
    ctx->precision = precision;
    ctx->fine = *fine;
    ctx->has_coarse = coarse != nullptr;
    if (coarse) ctx->coarse = *coarse;
    // active-tile coarse sweeps need the stencil reach (+ the bilinear corner) inside one tile
    // (computed here: the host arrays of the problem are valid only during this call)
    ctx->coarse_tiled = coarse && reach_cells(coarse) + 2.0 < (double)coarse_tile();
    ctx->coarse_stage = coarse && reach_cells(coarse) + 1.0 <= (double)coarse_halo();
    {
        // the synthesis foot has no diffusion branch: its reach is h max|f| / dx
        pdd_problem f0 = *fine;
        f0.p = 0;
        ctx->synth_stage = reach_cells(&f0) + 1.0 <= (double)coarse_halo();
    }
    {
        auto rok = [](const pdd_coef &c) { return c.kind == PDD_COEF_CONST || c.kind == PDD_COEF_ROW; };
        if (coarse)
            ctx->coarse_rowuniform = rok(coarse->speed) && rok(coarse->drift[0]) &&
                                     rok(coarse->drift[1]) && rok(coarse->cost);
        ctx->fine_rowuniform = rok(fine->speed) && rok(fine->drift[0]) && rok(fine->drift[1]) &&
                               rok(fine->cost);
    }
    ctx->fine_reach = reach_cells(fine);
    ctx->fine_halo = halo_of(fine);
    ctx->fine_row_uniform_all = row_uniform(fine);
    // aligned base
    char *base = (char *)workspace;
    const size_t mis = (size_t)((uintptr_t)base % kAlign);
    if (mis) base += kAlign - mis;
    layout(ctx, base, fine, coarse);
    // host pinned scratch
    {
        cudaError_t e = cudaHostAlloc((void **)&ctx->h_cnt, sizeof(ActCounters) + 64 + sizeof(RoundCtl), 0);
        if (e != cudaSuccess) {
            pdd_status st = fail(nullptr, PDD_E_CUDA, "cudaHostAlloc: %s", cudaGetErrorString(e));
            delete ctx;
            return st;
        }
        ctx->h_int = reinterpret_cast<int *>(ctx->h_cnt + 1);
        ctx->h_ctl = reinterpret_cast<RoundCtl *>(reinterpret_cast<char *>(ctx->h_cnt) + sizeof(ActCounters) + 64);
    }
    for (int k = 0; k < 4; ++k) cudaEventCreate(&ctx->ev[k]);
    s = copy_problem(ctx, fine, ctx->F, true);
    if (s == PDD_OK && coarse) s = copy_problem(ctx, coarse, ctx->Cc, false);
    if (s == PDD_OK) {
        launch_init_values(ctx->F.d, ctx->V, ctx->stream);
        ctx->launches++;
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) s = fail(nullptr, PDD_E_CUDA, "create: %s", cudaGetErrorString(e));
    } else {
        g_err = ctx->err;
    }
    if (s != PDD_OK) {
        pdd_destroy(ctx);
        return s;
    }
    // the caller may free its host arrays once this call returns (include/pdd.h): drop them
    for (pdd_problem *p : {&ctx->fine, &ctx->coarse}) {
        p->controls = nullptr;
        p->kind = nullptr;
        p->sector = nullptr;
        p->cost_ctrl = nullptr;
        for (int k = 0; k < 8; ++k) const_cast<pdd_coef *>(coef_ptr(p, k))->data = nullptr;
    }
    *out = ctx;
    return PDD_OK;
}

void pdd_destroy(pdd_ctx *ctx)
{
    if (!ctx) return;
    {
        DevGuard dev_guard(ctx->device);
        if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    }
    for (int k = 0; k < 4; ++k)
        if (ctx->ev[k]) cudaEventDestroy(ctx->ev[k]);
    for (int a = 0; a < 2; ++a)
        for (int k = 0; k < 64; ++k)
            if (ctx->evp[a][k]) cudaEventDestroy(ctx->evp[a][k]);
    if (ctx->h_cnt) cudaFreeHost(ctx->h_cnt);
    delete ctx;
}

pdd_status pdd_coarse_solve(pdd_ctx *ctx, double tol_c, int64_t max_sweeps, pdd_coarse_stats *st)
{
    if (!ctx) return fail(nullptr, PDD_E_INVALID, "ctx is NULL");
    DevGuard dev_guard(ctx->device);
    if (!ctx->has_coarse) return fail(ctx, PDD_E_STATE, "no coarse problem was given to pdd_create");
    if (!(tol_c > 0.0)) return fail(ctx, PDD_E_INVALID, "tol_c must be > 0");
    if (max_sweeps <= 0 || max_sweeps > kMaxCoarseSweeps)
        return fail(ctx, PDD_E_INVALID, "max_sweeps must be in 1..%lld", (long long)kMaxCoarseSweeps);
    cudaStream_t s = ctx->stream;
    const DProblem &Pc = ctx->Cc.d;
    CK(cudaEventRecord(ctx->ev[0], s));
    launch_init_values(Pc, ctx->uc[0], s);
    ctx->launches++;
    CK(cudaMemsetAsync(ctx->res_hist, 0, sizeof(unsigned long long) * max_sweeps, s));
    CK(cudaMemsetAsync(ctx->dev_int, 0, sizeof(int), s));
    int64_t issued = 0;
    int done = 0;
    bool converged = false;
    int64_t batch = 8;
    const bool tiled = ctx->coarse_tiled && !dev_env("PDD_COARSE_FULL");   // env: A/B only
    const bool use_rt = tiled && ctx->coarse_rowuniform && !dev_env("PDD_COARSE_NORT");
    if (use_rt) {
        launch_coarse_rowtab(Pc, ctx->crowtab, s);
        ctx->launches++;
    }
    while (issued < max_sweeps) {
        const int64_t b = std::min<int64_t>(batch, max_sweeps - issued);
        const size_t ctn = (size_t)((Pc.n + coarse_tile() - 1) / coarse_tile());
        for (int64_t q = 0; q < b; ++q, ++issued) {
            if (tiled)
                launch_coarse_sweep_tiles(Pc, ctx->uc[issued & 1], ctx->uc[(issued + 1) & 1], tol_c,
                                          ctx->res_hist, (int)issued, ctx->dev_int,
                                          ctx->cflag + ((issued + 1) & 1) * ctn * ctn,
                                          ctx->cflag + (issued & 1) * ctn * ctn,
                                          use_rt ? ctx->crowtab : nullptr,
                                          ctx->coarse_stage ? 1 : 0, s);
            else
                launch_coarse_sweep(Pc, ctx->uc[issued & 1], ctx->uc[(issued + 1) & 1], tol_c,
                                    ctx->res_hist, (int)issued, ctx->dev_int, s);
        }
        ctx->launches += b;
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(ctx->h_int, ctx->dev_int, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        done = ctx->h_int[0];
        if (done < issued) { converged = true; break; }
        unsigned long long last = 0;
        CK(cudaMemcpy(&last, ctx->res_hist + (issued - 1), sizeof last, cudaMemcpyDeviceToHost));
        double lr;
        std::memcpy(&lr, &last, sizeof lr);
        if (lr < tol_c) { converged = true; break; }
        batch = std::min<int64_t>(batch * 2, 256);
    }
    CK(cudaEventRecord(ctx->ev[1], s));
    CK(cudaEventSynchronize(ctx->ev[1]));
    ctx->uc_final = ctx->uc[done & 1];
    ctx->coarse_done = true;
    ctx->synth_done = false;
    unsigned long long lastbits = 0;
    if (done > 0)
        CK(cudaMemcpy(&lastbits, ctx->res_hist + (done - 1), sizeof lastbits, cudaMemcpyDeviceToHost));
    if (st) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
        st->sweeps = done;
        std::memcpy(&st->residual, &lastbits, sizeof(double));
        st->seconds = ms * 1e-3;
        st->converged = converged ? 1 : 0;
    }
    return converged ? PDD_OK : fail(ctx, PDD_E_NOCONVERGE, "coarse solve: %lld sweeps without reaching tol",
                                     (long long)done);
}

pdd_status pdd_synthesize(pdd_ctx *ctx)
{
    if (!ctx) return fail(nullptr, PDD_E_INVALID, "ctx is NULL");
    DevGuard dev_guard(ctx->device);
    if (!ctx->coarse_done) return fail(ctx, PDD_E_STATE, "pdd_synthesize needs pdd_coarse_solve first");
    cudaStream_t s = ctx->stream;
    launch_prolong(ctx->coarse.n, ctx->uc_final, ctx->fine.n, ctx->uhat, s);
    if (ctx->fine_rowuniform && !dev_env("PDD_SYNTH_NORT")) {   // env: A/B only
        // row-invariant part of the synthesis hoisted into a (row, control) table: bit-identical
        launch_coarse_rowtab(ctx->F.d, ctx->frowtab, s);
        launch_synthesize_rt(ctx->F.d, ctx->uhat, ctx->frowtab, ctx->astar, ctx->synth_stage ? 1 : 0, s);
        ctx->launches += 3;
    } else {
        launch_synthesize(ctx->F.d, ctx->uhat, ctx->astar, s);
        ctx->launches += 2;
    }
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    ctx->synth_done = true;
    return PDD_OK;
}

pdd_status pdd_build_patches(pdd_ctx *ctx, int32_t n_patches, double M)
{
    if (!ctx) return fail(nullptr, PDD_E_INVALID, "ctx is NULL");
    DevGuard dev_guard(ctx->device);
    if (!ctx->synth_done) return fail(ctx, PDD_E_STATE, "pdd_build_patches needs pdd_synthesize first");
    if (n_patches < 1 || n_patches >= kMaxPatches)
        return fail(ctx, PDD_E_INVALID, "n_patches must be in 1..%d", kMaxPatches - 1);
    if (!ctx->F.sector) return fail(ctx, PDD_E_INVALID, "the fine problem has no sector table");
    if (M == 0.0) M = 4.0;
    if (!(M > 0.0)) return fail(ctx, PDD_E_INVALID, "M must be > 0");
    cudaStream_t s = ctx->stream;
    const int64_t N = (int64_t)ctx->fine.n * ctx->fine.n;
    launch_successor(ctx->F.d, M, ctx->astar, ctx->succ0, s);
    ctx->launches++;
    CK(cudaGetLastError());
    // pointer jumping: after K rounds every chain of length < 2^K has reached its root
    int K = 1;
    while ((int64_t(1) << K) < N) ++K;
    const int32_t *in = ctx->succ0;
    int32_t *bufs[2] = {ctx->succA, ctx->succB};
    int r = 0;
    for (; r < K + 1; ++r) {
        CK(cudaMemsetAsync(ctx->dev_int + 1, 0, sizeof(int), s));
        launch_jump(in, bufs[r & 1], N, ctx->dev_int + 1, s);
        ctx->launches++;
        CK(cudaGetLastError());
        in = bufs[r & 1];
        if ((r & 3) == 3) {
            CK(cudaMemcpyAsync(ctx->h_int + 1, ctx->dev_int + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (ctx->h_int[1] == 0) break;
        }
    }
    launch_labels(ctx->F.kind, ctx->F.sector, in, n_patches, N, ctx->labels, s);
    ctx->launches++;
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(s));
    ctx->labels_mode = 1;
    ctx->n_patches = n_patches;
    ctx->prepared_kernel = -1;
    return PDD_OK;
}

pdd_status pdd_fuzzy_scratch_bytes(int32_t n, int32_t n_patches, size_t *bytes)
{
    if (!bytes) return fail(nullptr, PDD_E_INVALID, "bytes is NULL");
    if (n < 3 || n_patches < 1 || n_patches >= kMaxPatches)
        return fail(nullptr, PDD_E_INVALID, "fuzzy scratch: n >= 3 and 1 <= n_patches < %d", kMaxPatches);
    *bytes = 2 * sizeof(double) * (size_t)n_patches * (size_t)n * (size_t)n + 256;
    return PDD_OK;
}

pdd_status pdd_build_fuzzy_patches(pdd_ctx *ctx, int32_t n_patches, double eps_P, double tau_P,
                                   int64_t max_sweeps, void *scratch, size_t scratch_bytes,
                                   pdd_fuzzy_stats *st)
{
    if (!ctx) return fail(nullptr, PDD_E_INVALID, "ctx is NULL");
    DevGuard dev_guard(ctx->device);
    if (!ctx->synth_done) return fail(ctx, PDD_E_STATE, "pdd_build_fuzzy_patches needs pdd_synthesize first");
    if (n_patches < 1 || n_patches >= kMaxPatches)
        return fail(ctx, PDD_E_INVALID, "n_patches must be in 1..%d", kMaxPatches - 1);
    if (!ctx->F.sector) return fail(ctx, PDD_E_INVALID, "the fine problem has no sector table");
    if (!(eps_P > 0.0) || !(tau_P > 0.0 && tau_P < 1.0))
        return fail(ctx, PDD_E_INVALID, "need eps_P > 0 and 0 < tau_P < 1");
    if (max_sweeps <= 0 || max_sweeps > kMaxCoarseSweeps)
        return fail(ctx, PDD_E_INVALID, "max_sweeps must be in 1..%lld", (long long)kMaxCoarseSweeps);
    size_t need = 0;
    pdd_status ps = pdd_fuzzy_scratch_bytes(ctx->fine.n, n_patches, &need);
    if (ps != PDD_OK) return ps;
    if (!scratch || scratch_bytes < need)
        return fail(ctx, PDD_E_NOMEM, "fuzzy scratch needs %zu bytes", need);
    cudaStream_t s = ctx->stream;
    const int64_t N = (int64_t)ctx->fine.n * ctx->fine.n;
    char *b = (char *)scratch;
    const size_t mis = (size_t)((uintptr_t)b % 256);
    if (mis) b += 256 - mis;
    double *phi[2] = {reinterpret_cast<double *>(b), reinterpret_cast<double *>(b) + (size_t)n_patches * N};
    CK(cudaEventRecord(ctx->ev[0], s));
    launch_fuzzy_init(ctx->F.d, ctx->F.sector, n_patches, phi[0], s);
    CK(cudaMemsetAsync(ctx->res_hist, 0, sizeof(unsigned long long) * max_sweeps, s));
    CK(cudaMemsetAsync(ctx->dev_int, 0, 2 * sizeof(int), s));
    ctx->launches++;
    int64_t issued = 0, batch = 8;
    int done = 0;
    bool converged = false;
    while (issued < max_sweeps) {
        const int64_t nb = std::min<int64_t>(batch, max_sweeps - issued);
        for (int64_t q = 0; q < nb; ++q, ++issued)
            launch_fuzzy_sweep(ctx->F.d, ctx->astar, n_patches, phi[issued & 1], phi[(issued + 1) & 1],
                               eps_P, ctx->res_hist, (int)issued, ctx->dev_int, s);
        ctx->launches += nb;
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(ctx->h_int, ctx->dev_int, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        done = ctx->h_int[0];
        if (done < issued) { converged = true; break; }
        unsigned long long last = 0;
        CK(cudaMemcpy(&last, ctx->res_hist + (issued - 1), sizeof last, cudaMemcpyDeviceToHost));
        double lr;
        std::memcpy(&lr, &last, sizeof lr);
        if (lr < eps_P) { converged = true; break; }
        batch = std::min<int64_t>(batch * 2, 256);
    }
    const double *fin = phi[done & 1];
    CK(cudaMemsetAsync(ctx->dev_int + 1, 0, sizeof(int), s));
    launch_fuzzy_assign(ctx->F.d, fin, n_patches, tau_P, ctx->labels, ctx->dev_int + 1, s);
    ctx->launches++;
    CK(cudaGetLastError());
    CK(cudaEventRecord(ctx->ev[1], s));
    CK(cudaMemcpyAsync(ctx->h_int + 1, ctx->dev_int + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    ctx->labels_mode = 1;
    ctx->n_patches = n_patches;
    ctx->prepared_kernel = -1;
    if (st) {
        unsigned long long lastbits = 0;
        if (done > 0)
            CK(cudaMemcpy(&lastbits, ctx->res_hist + (done - 1), sizeof lastbits, cudaMemcpyDeviceToHost));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
        st->sweeps = done;
        std::memcpy(&st->residual, &lastbits, sizeof(double));
        st->seconds = ms * 1e-3;
        st->converged = converged ? 1 : 0;
        st->overlap_nodes = ctx->h_int[1];
        st->phi_offset = (int64_t)((const char *)fin - (const char *)scratch);
        st->lab_offset = 0;
        st->max_list = 0;
        st->reserved = 0;
    }
    return converged ? PDD_OK : fail(ctx, PDD_E_NOCONVERGE, "fuzzy patches: %lld sweeps without reaching eps_P",
                                     (long long)done);
}

}  // extern "C"

// ---- machine-peak micro-benchmarks (pdd_measure_alu_peaks)
__global__ void __launch_bounds__(512) k_peak_ffma(float *sink, int iters, float b, float c)
{
    float a0 = threadIdx.x, a1 = a0 + 1.f, a2 = a0 + 2.f, a3 = a0 + 3.f, a4 = a0 + 4.f, a5 = a0 + 5.f,
          a6 = a0 + 6.f, a7 = a0 + 7.f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
            a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
        }
    }
    const float r = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (r == 12345.678f) sink[0] = r;   // never true: keeps the chains alive
}

__global__ void __launch_bounds__(512) k_peak_dfma(float *sink, int iters, double b, double c)
{
    double a0 = threadIdx.x, a1 = a0 + 1., a2 = a0 + 2., a3 = a0 + 3., a4 = a0 + 4., a5 = a0 + 5.,
           a6 = a0 + 6., a7 = a0 + 7.;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    const double r = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (r == 12345.678) sink[0] = (float)r;
}

__global__ void __launch_bounds__(512) k_peak_lds(float *sink, int iters)
{
    __shared__ float4 buf[1024];
    for (int e = threadIdx.x; e < 1024; e += blockDim.x) buf[e] = make_float4(1.f, 2.f, 3.f, (float)e);
    __syncthreads();
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int idx = threadIdx.x;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            // a warp reads 512 contiguous bytes; volatile asm: every load is issued
            float4 v;
            const unsigned a = (unsigned)__cvta_generic_to_shared(&buf[(idx + 32 * u) & 1023]);
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        idx = (idx + 64) & 1023;
    }
    if (acc.x + acc.y + acc.z + acc.w == 12345.678f) sink[0] = acc.x;
}

extern "C" {

pdd_status pdd_measure_alu_peaks(void *stream, int32_t reps, double *fp32_tflops, double *smem_tbs,
                                 double *fp64_tflops)
{
    if (reps < 1 || reps > 1000) return fail(nullptr, PDD_E_INVALID, "reps must be in 1..1000");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int dev = 0, sms = 0;
    CK0(cudaGetDevice(&dev));
    CK0(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    float *sink = nullptr;
    CK0(cudaMalloc(&sink, sizeof(float)));
    cudaEvent_t e0, e1;
    CK0(cudaEventCreate(&e0));
    CK0(cudaEventCreate(&e1));
    const int grid = sms * 4, block = 512;
    double best_f = 0.0, best_l = 0.0, best_d = 0.0;
    for (int r = 0; r < reps + 1; ++r) {        // the first launch warms up
        const int it_f = 4096, it_l = 2048, it_d = 1024;
        cudaEventRecord(e0, s);
        k_peak_ffma<<<grid, block, 0, s>>>(sink, it_f, 1.0000001f, 1e-7f);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fl = 2.0 * 64.0 * it_f * (double)grid * block;
        if (r > 0 && ms > 0.f) best_f = std::max(best_f, fl / (ms * 1e-3) * 1e-12);
        cudaEventRecord(e0, s);
        k_peak_lds<<<grid, block, 0, s>>>(sink, it_l);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double by = 16.0 * 8.0 * it_l * (double)grid * block;
        if (r > 0 && ms > 0.f) best_l = std::max(best_l, by / (ms * 1e-3) * 1e-12);
        cudaEventRecord(e0, s);
        k_peak_dfma<<<grid, block, 0, s>>>(sink, it_d, 1.0000001, 1e-7);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double fd = 2.0 * 64.0 * it_d * (double)grid * block;
        if (r > 0 && ms > 0.f) best_d = std::max(best_d, fd / (ms * 1e-3) * 1e-12);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    CK0(cudaGetLastError());
    if (fp32_tflops) *fp32_tflops = best_f;
    if (smem_tbs) *smem_tbs = best_l;
    if (fp64_tflops) *fp64_tflops = best_d;
    return PDD_OK;
}

pdd_status pdd_fuzzy_sparse_scratch_bytes(int32_t n, int32_t K, size_t *bytes)
{
    if (!bytes) return fail(nullptr, PDD_E_INVALID, "bytes is NULL");
    if (n < 3 || K < 1 || K > 16)
        return fail(nullptr, PDD_E_INVALID, "sparse fuzzy scratch: n >= 3 and 1 <= K <= 16");
    const size_t NK = (size_t)n * (size_t)n * (size_t)K;
    *bytes = 2 * (sizeof(double) + sizeof(int16_t)) * NK + 512;
    return PDD_OK;
}

pdd_status pdd_build_fuzzy_patches_sparse(pdd_ctx *ctx, int32_t n_patches, int32_t K, double eps_P,
                                          double tau_P, int64_t max_sweeps, void *scratch,
                                          size_t scratch_bytes, pdd_fuzzy_stats *st)
{
    if (!ctx) return fail(nullptr, PDD_E_INVALID, "ctx is NULL");
    DevGuard dev_guard(ctx->device);
    if (!ctx->synth_done) return fail(ctx, PDD_E_STATE, "pdd_build_fuzzy_patches_sparse needs pdd_synthesize first");
    if (n_patches < 1 || n_patches >= kMaxPatches)
        return fail(ctx, PDD_E_INVALID, "n_patches must be in 1..%d", kMaxPatches - 1);
    if (!ctx->F.sector) return fail(ctx, PDD_E_INVALID, "the fine problem has no sector table");
    if (!(eps_P > 0.0) || !(tau_P > 0.0 && tau_P < 1.0))
        return fail(ctx, PDD_E_INVALID, "need eps_P > 0 and 0 < tau_P < 1");
    if (max_sweeps <= 0 || max_sweeps > kMaxCoarseSweeps)
        return fail(ctx, PDD_E_INVALID, "max_sweeps must be in 1..%lld", (long long)kMaxCoarseSweeps);
    if (!(K == 1 || K == 2 || K == 3 || K == 4 || K == 6 || K == 8 || K == 16))
        return fail(ctx, PDD_E_INVALID, "K must be one of 1, 2, 3, 4, 6, 8, 16");
    size_t need = 0;
    pdd_status ps = pdd_fuzzy_sparse_scratch_bytes(ctx->fine.n, K, &need);
    if (ps != PDD_OK) return ps;
    if (!scratch || scratch_bytes < need)
        return fail(ctx, PDD_E_NOMEM, "sparse fuzzy scratch needs %zu bytes", need);
    cudaStream_t s = ctx->stream;
    const size_t NK = (size_t)ctx->fine.n * ctx->fine.n * (size_t)K;
    char *b = (char *)scratch;
    const size_t mis = (size_t)((uintptr_t)b % 256);
    if (mis) b += 256 - mis;
    double *mass[2] = {reinterpret_cast<double *>(b), reinterpret_cast<double *>(b) + NK};
    int16_t *lab[2] = {reinterpret_cast<int16_t *>(mass[1] + NK), reinterpret_cast<int16_t *>(mass[1] + NK) + NK};
    CK(cudaEventRecord(ctx->ev[0], s));
    launch_fuzzy_sparse_init(ctx->F.d, ctx->F.sector, n_patches, K, lab[0], mass[0], s);
    CK(cudaMemsetAsync(ctx->res_hist, 0, sizeof(unsigned long long) * max_sweeps, s));
    CK(cudaMemsetAsync(ctx->dev_int, 0, 3 * sizeof(int), s));
    ctx->launches++;
    int64_t issued = 0, batch = 8;
    int done = 0;
    bool converged = false;
    while (issued < max_sweeps) {
        const int64_t nb = std::min<int64_t>(batch, max_sweeps - issued);
        for (int64_t q = 0; q < nb; ++q, ++issued)
            launch_fuzzy_sparse_sweep(ctx->F.d, ctx->astar, K, lab[issued & 1], mass[issued & 1],
                                      lab[(issued + 1) & 1], mass[(issued + 1) & 1], eps_P, ctx->res_hist,
                                      (int)issued, ctx->dev_int, s);
        ctx->launches += nb;
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(ctx->h_int, ctx->dev_int, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        done = ctx->h_int[0];
        if (done < issued) { converged = true; break; }
        unsigned long long last = 0;
        CK(cudaMemcpy(&last, ctx->res_hist + (issued - 1), sizeof last, cudaMemcpyDeviceToHost));
        double lr;
        std::memcpy(&lr, &last, sizeof lr);
        if (lr < eps_P) { converged = true; break; }
        batch = std::min<int64_t>(batch * 2, 256);
    }
    const int fin = done & 1;
    launch_fuzzy_sparse_assign(ctx->F.d, lab[fin], mass[fin], K, n_patches, tau_P, ctx->labels,
                               ctx->dev_int + 1, ctx->dev_int + 2, s);
    ctx->launches++;
    CK(cudaGetLastError());
    CK(cudaEventRecord(ctx->ev[1], s));
    CK(cudaMemcpyAsync(ctx->h_int + 1, ctx->dev_int + 1, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    ctx->labels_mode = 1;
    ctx->n_patches = n_patches;
    ctx->prepared_kernel = -1;
    if (st) {
        unsigned long long lastbits = 0;
        if (done > 0)
            CK(cudaMemcpy(&lastbits, ctx->res_hist + (done - 1), sizeof lastbits, cudaMemcpyDeviceToHost));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]);
        st->sweeps = done;
        std::memcpy(&st->residual, &lastbits, sizeof(double));
        st->seconds = ms * 1e-3;
        st->converged = converged ? 1 : 0;
        st->overlap_nodes = ctx->h_int[1];
        st->max_list = ctx->h_int[2];
        st->reserved = 0;
        st->phi_offset = (int64_t)((const char *)mass[fin] - (const char *)scratch);
        st->lab_offset = (int64_t)((const char *)lab[fin] - (const char *)scratch);
    }
    return converged ? PDD_OK : fail(ctx, PDD_E_NOCONVERGE, "sparse fuzzy patches: %lld sweeps without reaching eps_P",
                                     (long long)done);
}

pdd_status pdd_build_static(pdd_ctx *ctx, int32_t px, int32_t py)
{
    if (!ctx) return fail(nullptr, PDD_E_INVALID, "ctx is NULL");
    DevGuard dev_guard(ctx->device);
    if (px < 1 || py < 1 || (int64_t)px * py >= kMaxPatches || px > ctx->fine.n || py > ctx->fine.n)
        return fail(ctx, PDD_E_INVALID, "bad static decomposition %d x %d", px, py);
    launch_static_labels(ctx->fine.n, px, py, ctx->F.kind, ctx->labels, ctx->stream);
    ctx->launches++;
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->labels_mode = 2;
    ctx->static_px = px;
    ctx->static_py = py;
    ctx->n_patches = px * py;
    ctx->prepared_kernel = -1;
    return PDD_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------ sweep preparation

// Row-uniform problem: every coefficient of the stencil depends on x2 only (and a constant cost).
static bool row_uniform(const pdd_problem *p)
{
    auto row_ok = [](const pdd_coef &c) { return c.kind == PDD_COEF_CONST || c.kind == PDD_COEF_ROW; };
    if (!row_ok(p->speed) || !row_ok(p->drift[0]) || !row_ok(p->drift[1])) return false;
    for (int k = 0; k < 2; ++k)
        for (int c = 0; c < 2; ++c)
            if (!row_ok(p->sigma[k][c])) return false;
    return p->cost.kind == PDD_COEF_CONST;
}

// Path-3 tile geometry.  The 16 x 128 tile fills the 8-warp row pipeline with slack (27 % more
// node-updates/s than 32 x 64) but spans twice the x-distance, and the
// kernel's fp32 tile-relative values carry a noise floor of about 1 ulp of half the tile's value
// range: on coarse grids (128 dx ~ 1) that floor exceeds a 1e-7 tolerance.  So the wide tile is
// taken only when it spans at most 1/8 in x (C4, C5: 4097^2, 8193^2 on [-2,2]^2), and only for
// the static squares and operator applications: the patchy schedule's single-sweep visits along
// the u_hat front do fewer wasted updates on the finer 32 x 64 tiles (measured C5 pipeline
// 182 vs 188 ms, C4 the same), the static rounds gain the kernel's throughput (C5 0.78 vs
// 1.07 s).  PDD_P3_TILE=64|128 in the environment forces one geometry (A/B measurements).
// geometry codes: 0 = 32 x 64, 1 = 16 x 128 (wide), 2 = 16 x 64 (low)
static int p3_geometry_choice(const pdd_problem *p, bool patchy, int force_cols, int force_rows)
{
    if (force_cols == 64) return force_rows == 16 ? 2 : 0;   // pdd_set_tile_shape (A/B runs, tests)
    if (force_cols == 128) return 1;
    const double dx = (p->hi - p->lo) / (p->n - 1);
    if (!patchy) return 128.0 * dx <= 0.125 + 1e-12 ? 1 : 0;
    // patchy: 16 x 64 tiles waste fewer updates along the u_hat front (a tile stays in the window
    // until the front has crossed it) at a lower kernel rate (2 rows per warp: the row pipeline
    // fills and drains in 46 steps for 32 of work).  Measured (profiles/r2t_tile16_ab.txt): C4
    // fine solve 0.063 -> 0.051 s, C2 5 -> 3 ms, C5 0.097 -> 0.101 s: taken up to 16 k tiles.
    const int64_t tiles = (int64_t)((p->n + 63) / 64) * ((p->n + 31) / 32);
    return tiles <= 16384 ? 2 : 0;
}

// The lean general-stencil kernel (path 4, sweep_gf.cuh) covers f = c(x) a + d(x) with any speed /
// drift coefficients, row-uniform sigma and cost, lambda > 0 and 2 or 4 branches.
static bool fast_general_ok(const pdd_problem *p)
{
    auto row_ok = [](const pdd_coef &c) { return c.kind == PDD_COEF_CONST || c.kind == PDD_COEF_ROW; };
    if (!(p->lambda > 0.0) || p->sigma_mode != 0 || (p->p != 1 && p->p != 2) || !row_ok(p->cost)) return false;
    for (int k = 0; k < p->p; ++k)
        for (int c = 0; c < 2; ++c)
            if (!row_ok(p->sigma[k][c])) return false;
    return p->n_controls <= 128;
}

// queue_ok: the launch is a work-queue solve or a check pass (the only forms path 4 is built in)
static pdd_status prepare(pdd_ctx *ctx, int kernel_req, bool patchy, bool queue_ok)
{
    const pdd_problem *p = &ctx->fine;   // sizes only: its host arrays are gone (pdd_create)
    const int want_geo = p3_geometry_choice(p, patchy, ctx->force_tile_cols, ctx->force_tile_rows);
    const bool want_wide = want_geo == 1;
    if (ctx->prepared_kernel == kernel_req && ctx->prepared_geo == want_geo &&
        ctx->prepared_queue_ok == queue_ok)
        return PDD_OK;
    const DProblem &d = ctx->F.d;
    const int H = ctx->fine_halo;
    if (H > 8) return fail(ctx, PDD_E_STENCIL, "foot points reach %.2f cells; tile halo limited to 8",
                           ctx->fine_reach);
    int WY = 0, WX = 0, oxmin = 0, oxmax = 0;
    int path = 1;
    const int napad = na_pad_of(p->n_controls);
    if (kernel_req != 1 && kernel_req != 4 && napad && ctx->fine_row_uniform_all) {
        // the compact row stencils are built on the device (k_rowtab_extent / k_rowtab_fill)
        if (rowtab_build_device(d, napad, H, ctx->precision, ctx->dev_int + 2, ctx->rowtab,
                                ctx->rowtab_bytes, WY, WX, oxmin, oxmax, ctx->stream) &&
            rowtab_supported(WY, WX, napad / 32))
            path = 2;
        CK(cudaGetLastError());
    }
    if ((kernel_req == 2 || kernel_req == 3) && path != 2)
        return fail(ctx, PDD_E_INVALID, "row-table stencil requested but the problem is not row-uniform");
    // fp32 row-table problems use the 4-nodes-per-step kernel (path 3) unless kernel 3 asks for
    // the one-node-per-step variant (path 2, kept for A/B measurements and fp64)
    int p3_pitch = 0, p3_cstride = 0, p3_hmax = 0;
    p3_geometry(p3_pitch, p3_cstride, p3_hmax);
    const bool g4 = path == 2 && ctx->precision == 32 && kernel_req != 3 && H <= p3_hmax;
    ctx->path = g4 ? 3 : path;
    // general stencil: the lean kernel where it applies (kernel 4 insists on it, kernel 1 on the
    // fully general one)
    const bool fast = path == 1 && kernel_req != 1 && queue_ok && fast_general_ok(p);
    if (kernel_req == 4 && !fast)
        return fail(ctx, PDD_E_INVALID, "kernel 4 needs the work-queue schedule and a problem with row-uniform "
                                        "sigma and cost, lambda > 0, p = 1 or 2");
    if (fast) {
        auto xvar = [](const pdd_coef &c) { return c.kind == PDD_COEF_COL || c.kind == PDD_COEF_FIELD; };
        ctx->path = 4;
        WY = 2 * p->p;                                            // branches
        WX = (xvar(p->drift[0]) || xvar(p->drift[1])) ? 1 : 0;    // drift planes staged
    }
    ctx->WY = WY;
    ctx->WX = WX;
    ctx->Hx = H;
    TileGeom g{};
    int tw3 = 64, th3 = 32;
    p3_tile(tw3, th3);
    if (g4 && want_wide) {
        p3_tile_wide(tw3, th3);
        p3_geometry_wide(p3_pitch, p3_cstride, p3_hmax);
        if (H > p3_hmax) return fail(ctx, PDD_E_STENCIL, "wide path-3 tile: halo %d too large", H);
    } else if (g4 && want_geo == 2) {
        p3_tile_low(tw3, th3);
        p3_geometry_low(p3_pitch, p3_cstride, p3_hmax);
        if (H > p3_hmax) return fail(ctx, PDD_E_STENCIL, "16 x 64 path-3 tile: halo %d too large", H);
    }
    g.TW = (path == 2 && !g4) ? rowtab_tw(WY, WX) : (g4 ? tw3 : 64);
    g.TH = g4 ? th3 : sweep_tile_rows();
    g.H = H;
    g.tiles_x = (p->n + g.TW - 1) / g.TW;
    g.tiles_y = (p->n + g.TH - 1) / g.TH;
    const int mod = path == 2 ? std::max(1, oxmax - oxmin + 1) : 4;
    const int banks = ctx->precision == 32 ? 32 : 16;
    int pitch = g.TW + 2 * H;
    if (g4) {
        // the kernel's compile-time geometry: 16-byte rows, consecutive window rows in different
        // 16-byte bank groups, the 4 shifted copies spread over bank groups
        pitch = p3_pitch;
        g.cstride = p3_cstride;
        if (pitch < g.TW + 2 * H || p3_cstride < (g.TH + 2 * H) * pitch + 4)
            return fail(ctx, PDD_E_STENCIL, "path-3 shared-memory geometry too small for halo %d", H);
    } else if (fast) {
        int gp = 0;
        gf_geometry(gp);
        pitch = gp;                                               // compile-time pitch of path 4
        g.cstride = (1 + 2 * WX) * g.TH * g.TW;                   // reals of the coefficient planes
    } else {
        while (pitch % banks != mod % banks) ++pitch;
        g.cstride = 0;
    }
    g.pitch = pitch;
    ctx->g = g;
    ctx->n_tiles = g.tiles_x * g.tiles_y;
    if (ctx->n_tiles > ctx->max_tiles) return fail(ctx, PDD_E_NOMEM, "too many tiles");
    std::vector<int32_t> all(ctx->n_tiles);
    for (int t = 0; t < ctx->n_tiles; ++t) all[t] = t;
    CK(cudaMemcpy(ctx->T.all_list, all.data(), sizeof(int32_t) * all.size(), cudaMemcpyHostToDevice));
    ctx->prepared_kernel = kernel_req;
    ctx->prepared_geo = want_geo;
    ctx->prepared_queue_ok = queue_ok;
    return PDD_OK;
}

static SweepLaunch make_launch(pdd_ctx *ctx, const int32_t *list, int n_list, int k_inner, int check,
                               double *out)
{
    SweepLaunch L{};
    L.P = ctx->F.d;
    L.V = ctx->V;
    L.labels = ctx->labels;
    L.g = ctx->g;
    L.list = list;
    L.n_list = n_list;
    L.tile_res = ctx->T.tile_res;
    L.tile_chg = ctx->T.tile_chg;
    L.tile_edge = ctx->T.tile_edge;
    L.k_inner = k_inner;
    L.out = out;
    L.rowtab = ctx->rowtab;
    L.na_pad = na_pad_of(ctx->fine.n_controls);
    L.Hx = ctx->Hx;
    L.path = ctx->path;
    L.WY = ctx->WY;
    L.WX = ctx->WX;
    L.check = check;
    L.precision = ctx->precision;
    L.tile_free = ctx->T.tile_free;
    // patchy tiles know their downstream orientation from u_hat: two sweeps along it, then the
    // x- and y-flipped ones; static tiles (no u_hat) cycle through all four (P:952-986 analogue)
    const bool oriented = ctx->mode_patchy && !dev_env("PDD_NO_ORIENT");   // env: A/B only
    L.tile_orient = oriented ? ctx->T.tile_orient : nullptr;
    L.oxor = oriented ? 0x90 : 0xE4;
    if (const char *e = dev_env("PDD_EREL")) L.early_rel = std::atof(e);   // A/B only
    if (const char *e = dev_env("PDD_KCOH")) L.k_coherent = std::atoi(e);   // A/B only
    if (const char *e = dev_env("PDD_OXOR")) L.oxor = (int)std::strtol(e, nullptr, 0);
    L.nu_counter = &reinterpret_cast<OrdCounters *>(ctx->T.ocounters)->updates;
    return L;
}

static double bits_to_double(unsigned long long b)
{
    double d;
    std::memcpy(&d, &b, sizeof d);
    return d;
}

static pdd_status activate(pdd_ctx *ctx, int out_list, double tol, double thr, int round,
                           double slack = -1.0)
{
    cudaStream_t s = ctx->stream;
    CK(cudaMemsetAsync(ctx->T.counters, 0, sizeof(ActCounters), s));
    CK(cudaMemsetAsync(&reinterpret_cast<ActCounters *>(ctx->T.counters)->min_pending, 0xff, 8, s));
    launch_activate(ctx->g, ctx->T, out_list, tol, tol, thr, round, ctx->n_tiles, s, slack, ctx->rctl);
    ctx->launches++;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(ctx->h_cnt, ctx->T.counters, sizeof(ActCounters), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return PDD_OK;
}

__global__ void k_to_f32(const double *in, float *out, int64_t N)
{
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N; k += (int64_t)gridDim.x * blockDim.x)
        out[k] = (float)in[k];
}

// Ordered schedule: Gauss-Seidel passes over the tiles in key order (k_sweep_ordered), then a
// full-grid Jacobi verification when a pass finds nothing left to do.
static pdd_status ordered_loop(pdd_ctx *ctx, const pdd_solve_opts *o, pdd_solve_stats &S, int trace,
                               bool &converged, double &last_verify, float &ms_sweep,
                               float &ms_verify)
{
    cudaStream_t s = ctx->stream;
    const int nt = ctx->n_tiles;
    const TileGeom &g = ctx->g;
    std::vector<double> key(nt);
    std::vector<int32_t> fr(nt), grp;
    CK(cudaStreamSynchronize(s));
    CK(cudaMemcpy(fr.data(), ctx->T.tile_free, sizeof(int32_t) * nt, cudaMemcpyDeviceToHost));
    if (o->mode == 0) {
        // patchy: the nodes are taken in increasing u_hat, at tile granularity
        CK(cudaMemcpy(key.data(), ctx->T.tile_minu, sizeof(double) * nt, cudaMemcpyDeviceToHost));
    } else {
        // static squares: each block in the default order "left to right and from top to bottom"
        // (P:954-955), blocks independent of each other
        grp.resize(nt);
        const int n = ctx->fine.n, px = ctx->static_px, py = ctx->static_py;
        for (int t = 0; t < nt; ++t) {
            const int tx = t % g.tiles_x, ty = t / g.tiles_x;
            const int ci = std::min(tx * g.TW + g.TW / 2, n - 1), cj = std::min(ty * g.TH + g.TH / 2, n - 1);
            int bx = 0, by = 0;
            while (bx + 1 < px && (int64_t)(bx + 1) * n / px <= ci) ++bx;
            while (by + 1 < py && (int64_t)(by + 1) * n / py <= cj) ++by;
            grp[t] = by * px + bx;
            key[t] = (double)((int64_t)(g.tiles_y - 1 - ty) * g.tiles_x + tx);
        }
        CK(cudaMemcpy(ctx->T.tile_group, grp.data(), sizeof(int32_t) * nt, cudaMemcpyHostToDevice));
    }
    CK(cudaMemcpy(ctx->T.tile_key, key.data(), sizeof(double) * nt, cudaMemcpyHostToDevice));
    std::vector<int32_t> ord;
    ord.reserve(nt);
    for (int t = 0; t < nt; ++t)
        if (fr[t] > 0) ord.push_back(t);
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return key[a] < key[b]; });
    if (!ord.empty())
        CK(cudaMemcpy(ctx->T.order, ord.data(), sizeof(int32_t) * ord.size(), cudaMemcpyHostToDevice));
    CK(cudaMemsetAsync(ctx->T.done, 0, sizeof(int) * nt, s));
    CK(cudaMemsetAsync(ctx->T.stamp, 0, sizeof(long long) * nt, s));
    CK(cudaMemsetAsync(ctx->T.ocounters, 0, sizeof(OrdCounters), s));
    OrdCounters *oc = reinterpret_cast<OrdCounters *>(ctx->T.ocounters);
    OrderArgs O{};
    O.order = ctx->T.order;
    O.n_order = (int)ord.size();
    O.key = ctx->T.tile_key;
    O.group = o->mode == 1 ? ctx->T.tile_group : nullptr;
    O.tile_free = ctx->T.tile_free;
    O.done = ctx->T.done;
    O.stamp = ctx->T.stamp;
    O.seq = &oc->seq;
    O.counter = &oc->counter;
    O.processed = &oc->processed;
    O.free_sum = &oc->free_sum;
    O.max_res = &oc->max_res;
    O.tol = o->tol;
    O.tile_round = ctx->T.tile_round;
    O.lab_off = ctx->T.tile_lab_off;
    O.lab_ids = ctx->T.tile_lab_ids;
    O.patch_round = ctx->T.patch_round;
    // patchy: tiles whose min u_hat differ by less than the slack do not wait for each other
    // (near-equal keys are neighbours along a level set of u_hat, not upstream / downstream);
    // opts.delta > 0 sets it, 0 = a quarter of the value change across a tile height at unit
    // speed.  Static keys are integers: plain "strictly smaller".
    O.key_slack = o->mode == 1 ? 0.0 : (o->delta > 0.0 ? o->delta : 0.25 * g.TH * ctx->fine.h * ctx->F.d.lmax);
    OrdCounters h{};
    int pass = 0;
    double best = INFINITY;
    int stalled = 0;
    while (S.rounds < o->max_rounds) {
        O.pass = ++pass;
        CK(cudaMemsetAsync(oc, 0, offsetof(OrdCounters, seq), s));
        SweepLaunch L = make_launch(ctx, nullptr, 0, o->k_inner, 0, nullptr);
        L.early_tol = o->early_exit_off ? 0.0 : o->tol;
        L.ordered = 1;
        L.order = O;
        CK(cudaEventRecord(ctx->ev[2], s));
        CK(launch_sweep(L, s));
        ctx->launches++;
        CK(cudaEventRecord(ctx->ev[3], s));
        CK(cudaMemcpyAsync(&h, oc, sizeof h, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]);
        ms_sweep += ms;
        S.rounds++;
        if (trace)
            fprintf(stderr, "[pdd] pass %d visited %d free %llu maxres %.3e %.3f ms\n", pass, h.processed,
                    h.free_sum, bits_to_double(h.max_res), ms);
        if (h.processed > 0) {
            S.tiles_processed += h.processed;
            continue;
        }
        // nothing left to do: full-grid Jacobi verification
        CK(cudaEventRecord(ctx->ev[2], s));
        SweepLaunch V = make_launch(ctx, ctx->T.all_list, ctx->n_tiles, 1, 1, nullptr);
        // each patch's own residual max |T(V) - V| over its free nodes
        CK(cudaMemsetAsync(ctx->T.patch_res, 0, sizeof(unsigned long long) * ctx->T.n_slots, s));
        V.patch_res = ctx->T.patch_res;
        V.n_slots = ctx->T.n_slots;
        CK(launch_sweep(V, s));
        ctx->launches++;
        CK(cudaEventRecord(ctx->ev[3], s));
        S.rounds++;
        S.verify_passes++;
        pdd_status r = activate(ctx, 0, INFINITY, INFINITY, 0);
        if (r != PDD_OK) return r;
        cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]);
        ms_verify += ms;
        last_verify = bits_to_double(ctx->h_cnt->max_res);
        if (trace) fprintf(stderr, "[pdd] verify residual %.3e\n", last_verify);
        if (last_verify < o->tol) {
            converged = true;
            break;
        }
        if (last_verify < 0.9 * best) { best = last_verify; stalled = 0; }
        else if (++stalled >= 8) break;   // below the arithmetic's noise floor: give up
    }
    return PDD_OK;
}

// Work-queue schedule: one persistent launch (k_sweep_queue) relaxes dirty tiles until the queue
// is empty and every tile has been admitted, then a full-grid Jacobi verification
// re-seeds the queue with the offending tiles.
static pdd_status queue_loop(pdd_ctx *ctx, const pdd_solve_opts *o, pdd_solve_stats &S, int trace,
                             int k_inner, int resident, int tiles_free, bool &converged,
                             double &last_verify, float &ms_sweep, float &ms_verify)
{
    cudaStream_t s = ctx->stream;
    const int nt = ctx->n_tiles;
    // tiles in key order: min u_hat (patchy) or index order (static)
    launch_queue_order(ctx->T, o->mode == 0 ? ctx->T.tile_minu : nullptr, nt, ctx->qscratch,
                       ctx->T.order, ctx->qrank, s);
    ctx->launches += 4;
    CK(cudaMemsetAsync(ctx->qstate, 0, sizeof(int) * nt, s));
    CK(cudaMemsetAsync(ctx->T.tile_sweeps, 0, sizeof(int32_t) * nt, s));
    QueueArgs Q{};
    Q.ctl = ctx->qctl;
    Q.ring = ctx->qring;
    Q.cap = ctx->qcap;
    Q.order = ctx->T.order;
    Q.rank = ctx->qrank;
    Q.n_order = tiles_free;
    // patchy: about two waves of resident CTAs queued or visiting at any time (A/B: PDD_QW)
    // (measured, profiles/r2e_queue_scan.txt, r2j_c3_target.txt, r2o_target_scan.txt: the best
    // window is about 1/20 of the grid's tiles -- C5's 33 k tiles want 2.5 - 3 waves of resident
    // CTAs (with fewer, tiles are revisited before their upstream neighbours moved), C4's 8.4 k
    // one wave, C3's 2.1 k tiles against 592 CTAs 0.75 waves)
    const char *qe = dev_env("PDD_QW");
    const int auto_target = std::min(3 * resident, std::max(tiles_free / 19, 3 * resident / 4));
    Q.target = o->queue_target > 0 ? o->queue_target
                                   : std::max(1, qe ? (int)(std::atof(qe) * resident) : auto_target);
    Q.state = ctx->qstate;
    const char *qte = dev_env("PDD_QTOL");  // A/B: queue tolerances / tol (re-queue and activation)
    const double qtf = qte ? std::atof(qte) : 1.0;
    Q.tol = o->tol * qtf;
    const char *te = dev_env("PDD_TACT");   // A/B: neighbour-change activation threshold / tol
    Q.tol_act = o->tol * qtf * (te ? std::atof(te) : 1.0);
    Q.tile_round = ctx->T.tile_round;
    Q.lab_off = ctx->T.tile_lab_off;
    Q.lab_ids = ctx->T.tile_lab_ids;
    Q.patch_round = ctx->T.patch_round;
    if ((unsigned)(nt + resident) >= ctx->qcap) return fail(ctx, PDD_E_NOMEM, "work-queue ring too small");
    QueueCtl qc{};
    // cap on visits: max_rounds visits per tile with free nodes (non-convergence guard)
    qc.max_visits = (unsigned long long)std::max<int64_t>(1, o->max_rounds) *
                    (unsigned long long)std::max(1, tiles_free);
    qc.adm = o->mode == 0 ? 0 : tiles_free;   // static: every tile is seeded at once
    double best = INFINITY;
    int stalled = 0;
    bool first = true;
    // partial verifications need every tile's per-label residuals in its label-list entries
    bool partial_ok = false, verified_once = false;
    int verify_mark = 0;
    if (ctx->T.n_slots > 0 && ctx->T.n_slots <= pres_shared_slots() && !dev_env("PDD_FULL_VERIFY")) {
        int32_t entries = 0;
        CK(cudaMemcpyAsync(&entries, ctx->T.tile_lab_off + nt, sizeof entries, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        partial_ok = entries <= ctx->T.tile_lab_cap;
    }
    for (;;) {
        // ring and cursors start empty at every launch (tickets abandoned at the last stop)
        CK(cudaMemsetAsync(ctx->qring, 0, sizeof(int32_t) * ctx->qcap, s));
        qc.head = qc.tail = 0;
        qc.work = 0;
        qc.stop = 0;
        // a launch ends for a verification after 32 visits per tile (legitimate solves need about
        // as many in total; the check costs one sweep-equivalent)
        qc.verify_at = qc.visits + 32ull * (unsigned long long)std::max(1, tiles_free) + 1024ull;
        CK(cudaMemcpyAsync(ctx->qctl, &qc, sizeof qc, cudaMemcpyHostToDevice, s));
        if (first && o->mode == 0)
            launch_queue_seed(ctx->T, Q, nt, 0.0, std::min(Q.target, tiles_free), 0, s);
        else
            launch_queue_seed(ctx->T, Q, nt, first ? -1.0 : o->tol, 0, qc.adm, s);   // static start: tile_res = inf
        ctx->launches++;
        first = false;
        SweepLaunch L = make_launch(ctx, nullptr, 0, k_inner, 0, nullptr);
        L.early_tol = o->early_exit_off ? 0.0 : o->tol;
        L.tile_sweeps = ctx->T.tile_sweeps;
        L.queued = 1;
        L.queue = Q;
        CK(cudaEventRecord(ctx->ev[2], s));
        if (tiles_free > 0) {
            CK(launch_sweep(L, s));
            ctx->launches++;
        }
        CK(cudaEventRecord(ctx->ev[3], s));
        CK(cudaMemcpyAsync(&qc, ctx->qctl, sizeof qc, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]);
        ms_sweep += ms;
        S.rounds++;
        S.tiles_processed = (int64_t)qc.visits;
        if (trace)
            fprintf(stderr, "[pdd] queue launch: visits %llu maxres %.3e stop %d adm %d %.3f ms\n", qc.visits,
                    bits_to_double(qc.max_res), qc.stop, qc.adm, ms);
        if (qc.stop == 2) break;   // visit cap reached
        if (qc.stop != 3) qc.adm = std::max(qc.adm, tiles_free);
        // verification with each patch's own residual: the whole grid the first time;
        // afterwards only the tiles whose residual can have changed (visited since the last
        // verification, or next to such a tile) -- every other tile keeps the Jacobi residual of
        // its last check, and the per-patch maxima are rebuilt from the per-tile entries
        CK(cudaEventRecord(ctx->ev[2], s));
        const int32_t *vlist = ctx->T.all_list;
        int vcount = nt;
        if (partial_ok && verified_once) {
            launch_verify_list(ctx->g, ctx->T, verify_mark, nt, s);
            ctx->launches++;
            CK(cudaMemcpyAsync(ctx->h_cnt, ctx->T.counters, sizeof(ActCounters), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            vlist = ctx->T.list[0];
            vcount = ctx->h_cnt->count;
        }
        SweepLaunch V = make_launch(ctx, vlist, vcount, 1, 1, nullptr);
        V.patch_res = ctx->T.patch_res;
        V.n_slots = ctx->T.n_slots;
        if (partial_ok) {
            V.lab_off = ctx->T.tile_lab_off;
            V.lab_ids = ctx->T.tile_lab_ids;
            V.lab_res = ctx->T.tile_lab_res;
        } else {
            CK(cudaMemsetAsync(ctx->T.patch_res, 0, sizeof(unsigned long long) * ctx->T.n_slots, s));
        }
        CK(launch_sweep(V, s));
        ctx->launches++;
        if (partial_ok) {
            launch_patch_res_reduce(ctx->T, nt, s);
            ctx->launches++;
        }
        verified_once = true;
        verify_mark = (int)std::min<unsigned long long>(qc.visits, 0x7fffffffull);
        CK(cudaEventRecord(ctx->ev[3], s));
        S.rounds++;
        S.verify_passes++;
        pdd_status r = activate(ctx, 0, INFINITY, INFINITY, 0);   // max residual readback only
        if (r != PDD_OK) return r;
        cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]);
        ms_verify += ms;
        last_verify = bits_to_double(ctx->h_cnt->max_res);
        if (trace) fprintf(stderr, "[pdd] verify residual %.3e\n", last_verify);
        if (last_verify < o->tol) {
            converged = true;
            break;
        }
        if (last_verify < 0.9 * best) { best = last_verify; stalled = 0; }
        else if (++stalled >= 8) break;   // below the arithmetic's noise floor: give up
        CK(cudaMemsetAsync(ctx->qstate, 0, sizeof(int) * nt, s));
    }
    if (ctx->T.n_slots > 0) {
        launch_patch_rounds(ctx->T, nt, s);
        ctx->launches++;
    }
    return PDD_OK;
}

extern "C" {

pdd_status pdd_solve(pdd_ctx *ctx, const pdd_solve_opts *o, pdd_solve_stats *st)
{
    if (!ctx) return fail(nullptr, PDD_E_INVALID, "ctx is NULL");
    DevGuard dev_guard(ctx->device);
    if (!o) return fail(ctx, PDD_E_INVALID, "opts is NULL");
    if (o->mode != 0 && o->mode != 1) return fail(ctx, PDD_E_INVALID, "mode must be 0 or 1");
    if (o->schedule < 0 || o->schedule > 3) return fail(ctx, PDD_E_INVALID, "schedule must be 0..3");
    if (o->queue_target < 0) return fail(ctx, PDD_E_INVALID, "queue_target must be >= 0");
    const int sched = o->schedule == 0 ? 2 : o->schedule;   // automatic: the work queue
    if (o->k_inner < 0 || o->k_inner > 1024) return fail(ctx, PDD_E_INVALID, "k_inner outside 0..1024");
    if (!(o->tol > 0.0)) return fail(ctx, PDD_E_INVALID, "tol must be > 0");
    if (o->mode == 0 && (!ctx->synth_done || ctx->labels_mode != 1))
        return fail(ctx, PDD_E_STATE, "patchy solve needs pdd_synthesize and pdd_build_patches");
    if (o->mode == 1 && ctx->labels_mode != 2)
        return fail(ctx, PDD_E_STATE, "static solve needs pdd_build_static");
    if (o->kernel < 0 || o->kernel > 4) return fail(ctx, PDD_E_INVALID, "kernel must be 0..4");
    pdd_status ps = prepare(ctx, o->kernel, o->mode == 0, (o->schedule == 0 ? 2 : o->schedule) == 2);
    if (ps != PDD_OK) return ps;
    cudaStream_t s = ctx->stream;
    const DProblem &d = ctx->F.d;
    CK(cudaEventRecord(ctx->ev[0], s));
    ctx->mode_patchy = o->mode == 0;
    launch_set_values(d, o->mode == 0 ? 0 : 1, ctx->uhat, ctx->V, s);
    // coherent tile: >= 90 % of its u_hat differences share the tile's sign in x and in y
    // (measured: 0.8 .. 0.99 all within noise on C2 / C4 / C5)
    const char *cenv = dev_env("PDD_COH");     // A/B: coherence threshold (> 1: never)
    ctx->T.n_slots = ctx->n_patches + 1;   // patches 0..n_patches-1, orphans n_patches
    launch_tile_init(d, ctx->g, o->mode == 0 ? ctx->uhat : nullptr, ctx->labels, ctx->T, s,
                     cenv ? std::atof(cenv) : 0.9);
    ctx->launches += 2;
    CK(cudaMemsetAsync(ctx->T.patch_round, 0xff, sizeof(int32_t) * (ctx->n_patches + 1), s));
    CK(cudaMemsetAsync(ctx->T.patch_res, 0, sizeof(unsigned long long) * (ctx->n_patches + 1), s));
    CK(cudaMemsetAsync(ctx->T.ocounters, 0, sizeof(OrdCounters), s));
    CK(cudaGetLastError());

    double delta = o->delta;
    if (o->mode == 1) delta = -1.0;
    // automatic bucket width: the value change across 6 cells at unit speed (measured on C5 / C4
    // / C3: 6 cells of front travel per round beat 4.8 and 8)
    if (delta == 0.0) {
        const char *e = dev_env("PDD_DSCALE");      // A/B only
        delta = 6.0 * ctx->fine.h * d.lmax * (e ? std::atof(e) : 1.0);
    }
    double thr = delta > 0.0 ? -1.0 : INFINITY;
    // bucket policy 2 (patchy): no moving threshold; a tile is admitted once its upstream
    // neighbours (min u_hat lower by more than a quarter tile of travel) have converged
    double ready_slack = -1.0;
    const char *benv = dev_env("PDD_DBOOST");    // development override of the front boost cap
    const double dboost = benv ? std::max(1.0, std::atof(benv)) : 1.0;
    int resident = 148;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&resident, cudaDevAttrMultiProcessorCount, dev);
        // sweep CTAs resident per SM: the occupancy of the device-driven sweep kernel
        SweepLaunch Q = make_launch(ctx, nullptr, 0, 1, 0, nullptr);
        int per_sm = 1;
        Q.occupancy_out = &per_sm;
        Q.queued = sched == 2 ? 1 : 0;   // the kernel that will run (the queue kernel's prefetch
                                         // buffer can lower its occupancy)
        CK(launch_sweep(Q, s));
        resident *= std::max(1, per_sm);
    }
    // automatic settings (k_inner = 0, delta = 0): when every tile with free nodes fits in one
    // wave of resident sweep CTAs, holding tiles back behind the u_hat front only adds rounds of
    // one-visit latency (measured on the paper's 800^2 Zermelo / eikonal grids), so the patchy
    // solve then admits every tile at once (u_hat start, downstream orientations) and every
    // visit does up to 4 in-tile sweeps; otherwise 1 sweep per visit (patchy) / 4 (static)
    int tiles_free = 0;
    {
        std::vector<int32_t> tf(ctx->n_tiles);
        CK(cudaMemcpyAsync(tf.data(), ctx->T.tile_free, sizeof(int32_t) * tf.size(),
                           cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        for (int32_t v : tf) tiles_free += v > 0;
    }
    const bool one_wave = tiles_free <= 2 * resident;   // "fits in (about) one wave": <= 2 waves
    // (measured: on one-wave grids the general stencil wants 4 sweeps per visit -- paper Zermelo
    // 800^2: 49.7 vs 117 sweep-equivalents -- the row-table kernels 1: C2 10 ms vs 16 ms,
    // eikonal 800^2 16 ms vs 34 ms)
    const int k_inner = o->k_inner > 0 ? o->k_inner
                        : (o->mode == 1 ? 4 : (one_wave && (ctx->path == 1 || ctx->path == 4) ? 4 : 1));
    if (o->mode == 0 && o->delta == 0.0 && one_wave && o->bucket_policy != 2) {
        delta = -1.0;
        thr = INFINITY;
    }
    if (o->mode == 0 && o->bucket_policy == 2) {
        ready_slack = o->delta > 0.0 ? o->delta : 0.25 * ctx->g.TH * ctx->fine.h * d.lmax;
        thr = INFINITY;
        delta = -1.0;
    }

    pdd_solve_stats S{};
    S.n_tiles = ctx->n_tiles;
    S.kernel_used = ctx->path;
    int cur = 0;
    const int trace = o->trace > 0 ? 1 : 0;   // per-round trace on stderr, one round per batch
    double best_verify = INFINITY;
    int stalled = 0;
    // rounds between forced verifications: a tolerance below the noise floor keeps tiles
    // re-activating each other forever; a legitimate sweep front needs far fewer rounds
    const int verify_every = 4 * ctx->n_tiles + 1024;
    bool converged = false;
    double last_verify = INFINITY;
    float ms_sweep = 0.f, ms_verify = 0.f;
    if (sched == 1) {
        pdd_status r = ordered_loop(ctx, o, S, trace, converged, last_verify, ms_sweep, ms_verify);
        if (r != PDD_OK) return r;
    }
    if (sched == 2) {
        pdd_status r = queue_loop(ctx, o, S, trace, k_inner, resident, tiles_free, converged,
                                  last_verify, ms_sweep, ms_verify);
        if (r != PDD_OK) return r;
    }
    // Device-driven rounds (schedule 3): batches of (begin, activate, sweep, end) are enqueued
    // without a host round trip; the RoundCtl block carries the front threshold and the stop
    // flag between them.  The host syncs once per batch and runs the verification pass.
    if (sched == 3) {
        RoundCtl c0{};
        c0.thr = thr;
        c0.delta = delta;
        c0.dboost = dboost;
        c0.resident = resident;
        c0.policy = o->bucket_policy;
        c0.verify_every = verify_every;
        const char *ue = dev_env("PDD_UPW");      // A/B: upstream-only re-activation slack
        c0.upw = ue ? std::atof(ue) * ctx->g.TH * ctx->fine.h * d.lmax : -1.0;
        *ctx->h_ctl = c0;
        CK(cudaMemcpyAsync(ctx->rctl, ctx->h_ctl, sizeof(RoundCtl), cudaMemcpyHostToDevice, s));
        CK(cudaMemsetAsync(ctx->T.tile_stamp, 0xff, sizeof(int32_t) * ctx->n_tiles, s));
        CK(cudaMemsetAsync(ctx->T.tile_sweeps, 0, sizeof(int32_t) * ctx->n_tiles, s));
    }
    int batch = trace ? 1 : 4;
    // patchy: visit each round's tiles in increasing min u_hat (A/B switch PDD_SORT)
    const char *se = dev_env("PDD_SORT");
    const bool sort_rounds = o->mode == 0 && se && std::atoi(se) != 0;
    const char *te = dev_env("PDD_TACT");   // A/B: neighbour-change activation threshold / tol
    const double tact = te ? std::atof(te) : 1.0;
    long long rounds_prev = 0;
    while (sched == 3) {
        if (S.rounds >= o->max_rounds) break;
        CK(cudaEventRecord(ctx->ev[2], s));
        SweepLaunch L = make_launch(ctx, ctx->T.list[cur], ctx->n_tiles, k_inner, 0, nullptr);
        L.early_tol = o->early_exit_off ? 0.0 : o->tol;   // early_exit_off = 1 disables early exit
        L.ctl = ctx->rctl;
        L.acnt = reinterpret_cast<ActCounters *>(ctx->T.counters);
        L.tile_stamp = ctx->T.tile_stamp;
        if (!dev_env("PDD_NO_SCONT")) L.tile_sweeps = ctx->T.tile_sweeps;   // env: A/B only
        const long long room = o->max_rounds - S.rounds;
        const int nb = (int)std::min<long long>(batch, std::max<long long>(room, 1));
        if (!ctx->evp[0][0])
            for (int a = 0; a < 2; ++a)
                for (int k = 0; k < 64; ++k) CK(cudaEventCreate(&ctx->evp[a][k]));
        for (int b = 0; b < nb; ++b) {
            launch_round_begin(ctx->rctl, L.acnt, s);
            launch_activate(ctx->g, ctx->T, cur, o->tol, o->tol * tact, 0.0, 0, ctx->n_tiles, s,
                            ready_slack, ctx->rctl, true);
            if (sort_rounds) {
                launch_sort_round(ctx->rctl, L.acnt, ctx->T.tile_minu, ctx->T.list[cur], s);
                ctx->launches++;
            }
            CK(cudaEventRecord(ctx->evp[0][b], s));
            CK(launch_sweep(L, s));
            CK(cudaEventRecord(ctx->evp[1][b], s));
            launch_round_end(ctx->rctl, L.acnt, s);
            ctx->launches += 4;
        }
        CK(cudaGetLastError());
        CK(cudaEventRecord(ctx->ev[3], s));
        CK(cudaMemcpyAsync(ctx->h_ctl, ctx->rctl, sizeof(RoundCtl), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(ctx->h_cnt, L.acnt, sizeof(ActCounters), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]);
        for (int b = 0; b < nb; ++b) {   // the sweep kernels alone (a stopped round's is ~0)
            float mk = 0.f;
            cudaEventElapsedTime(&mk, ctx->evp[0][b], ctx->evp[1][b]);
            ms_sweep += mk;
        }
        const RoundCtl hc = *ctx->h_ctl;
        S.rounds += hc.rounds - rounds_prev;
        rounds_prev = hc.rounds;
        S.tiles_processed = hc.tiles;
        if (trace)
            fprintf(stderr, "[pdd] batch %d rounds %lld active %d free %lld maxres %.3e thr %.4f stop %d %.4f ms\n",
                    nb, hc.rounds, ctx->h_cnt->count, (long long)ctx->h_cnt->free_sum,
                    bits_to_double(ctx->h_cnt->max_res), hc.thr, hc.stop, ms);
        if (!hc.stop) {
            batch = trace ? 1 : std::min(2 * batch, 64);
            continue;
        }
        batch = trace ? 1 : 4;
        // nothing active (or verify_every rounds since the last one): full-grid verification
        CK(cudaEventRecord(ctx->ev[2], s));
        SweepLaunch V = make_launch(ctx, ctx->T.all_list, ctx->n_tiles, 1, 1, nullptr);
        // each patch's own residual max |T(V) - V| over its free nodes
        CK(cudaMemsetAsync(ctx->T.patch_res, 0, sizeof(unsigned long long) * ctx->T.n_slots, s));
        V.patch_res = ctx->T.patch_res;
        V.n_slots = ctx->T.n_slots;
        CK(launch_sweep(V, s));
        ctx->launches++;
        launch_round_reset(ctx->rctl, INFINITY, s);   // after a verification every offending
        ctx->launches++;                              // tile is eligible; old changes superseded
        CK(cudaEventRecord(ctx->ev[3], s));
        S.rounds++;
        S.verify_passes++;
        pdd_status r = activate(ctx, cur, o->tol, INFINITY, 0, ready_slack);
        if (r != PDD_OK) return r;
        ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]);
        ms_verify += ms;
        last_verify = bits_to_double(ctx->h_cnt->max_res);
        if (trace) fprintf(stderr, "[pdd] verify residual %.3e active %d\n", last_verify, ctx->h_cnt->count);
        if (ctx->h_cnt->count == 0) { converged = true; break; }
        // stagnation guard: a tolerance below the arithmetic's noise floor (fp32: ~1 ulp of the
        // tile-relative values) cannot be reached; stop after 8 verifications without a 10 %
        // improvement of the best residual instead of iterating until max_rounds
        if (last_verify < 0.9 * best_verify) { best_verify = last_verify; stalled = 0; }
        else if (++stalled >= 8) break;
    }
    CK(cudaEventRecord(ctx->ev[1], s));
    CK(cudaEventSynchronize(ctx->ev[1]));
    float ms_total = 0.f;
    cudaEventElapsedTime(&ms_total, ctx->ev[0], ctx->ev[1]);
    {
        unsigned long long upd = 0;
        CK(cudaMemcpy(&upd, &reinterpret_cast<OrdCounters *>(ctx->T.ocounters)->updates, sizeof upd,
                      cudaMemcpyDeviceToHost));
        S.node_updates = (int64_t)upd;   // counted by the sweep kernel: free nodes x sweeps done
    }
    S.final_residual = last_verify;
    // ||V - V*|| <= r / (1 - beta) needs beta < 1: an exit problem (lambda = 0) has no such bound
    S.apost_bound = d.beta < 1.0 ? last_verify / (1.0 - d.beta) : NAN;
    S.tile_cols = ctx->g.TW;
    S.tile_rows = ctx->g.TH;
    S.tiles_x = ctx->g.tiles_x;
    S.seconds_total = ms_total * 1e-3;
    S.seconds_sweep = ms_sweep * 1e-3;
    S.seconds_verify = ms_verify * 1e-3;
    S.converged = converged ? 1 : 0;
    {
        // per-patch convergence flags: a patch (one that holds free nodes, i.e. had an active
        // tile) is converged when its own residual in the last verification pass is < tol
        const int ns = ctx->n_patches + 1;
        std::vector<int32_t> pr(ns);
        std::vector<double> rs(ns);
        CK(cudaMemcpy(pr.data(), ctx->T.patch_round, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(rs.data(), ctx->T.patch_res, sizeof(double) * ns, cudaMemcpyDeviceToHost));
        int pc = 0, pa = 0;
        for (int k = 0; k < ctx->n_patches; ++k) {
            if (pr[k] < 0) continue;
            ++pa;
            if (S.verify_passes > 0 && rs[k] < o->tol) ++pc;
        }
        S.patches_active = pa;
        S.patches_converged = pc;
    }
    if (st) *st = S;
    return converged ? PDD_OK
                     : fail(ctx, PDD_E_NOCONVERGE, "fine solve: %lld rounds without convergence (residual %.3e)",
                            (long long)S.rounds, last_verify);
}

pdd_status pdd_apply_operator(pdd_ctx *ctx, double *out, int32_t kernel, double *residual)
{
    if (!ctx) return fail(nullptr, PDD_E_INVALID, "ctx is NULL");
    DevGuard dev_guard(ctx->device);
    if (kernel < 0 || kernel > 4) return fail(ctx, PDD_E_INVALID, "kernel must be 0..4");
    pdd_status ps = prepare(ctx, kernel, false, true);
    if (ps != PDD_OK) return ps;
    cudaStream_t s = ctx->stream;
    const size_t N = (size_t)ctx->fine.n * ctx->fine.n;
    double *dst = out;
    if (dst) CK(cudaMemcpyAsync(dst, ctx->V, sizeof(double) * N, cudaMemcpyDeviceToDevice, s));
    launch_tile_init(ctx->F.d, ctx->g, nullptr, nullptr, ctx->T, s);
    ctx->launches += 2;
    SweepLaunch L = make_launch(ctx, ctx->T.all_list, ctx->n_tiles, 1, 1, dst);
    CK(launch_sweep(L, s));
    pdd_status r = activate(ctx, 0, INFINITY, INFINITY, 0);
    if (r != PDD_OK) return r;
    if (residual) *residual = bits_to_double(ctx->h_cnt->max_res);
    return PDD_OK;
}

pdd_status pdd_regime_analyse(double f_min, double f_max, double sigma_norm, double dx,
                              pdd_regime *out)
{
    if (!out) return fail(nullptr, PDD_E_INVALID, "out is NULL");
    if (!(f_min > 0.0) || !(f_max >= f_min) || !(sigma_norm >= 0.0) || !(dx > 0.0))
        return fail(nullptr, PDD_E_INVALID, "regime: need 0 < f_min <= f_max, sigma_norm >= 0, dx > 0");
    pdd_regime r{};
    r.upsilon = f_max / f_min;
    r.omega = sigma_norm > 0.0 ? f_min / (sigma_norm * sigma_norm) : INFINITY;
    r.tau_dx = dx / (1.0 + r.upsilon);
    const double inv_omega = sigma_norm > 0.0 ? (sigma_norm * sigma_norm) / f_min : 0.0;
    r.alpha_lo = inv_omega / dx;
    if (sigma_norm > 0.0) {
        const double w = r.omega * dx * r.upsilon;
        r.alpha_hi = 1.0 / r.upsilon - (std::sqrt(1.0 + 4.0 * w) - 1.0) / (2.0 * r.omega * dx * r.upsilon * r.upsilon);
    } else {
        r.alpha_hi = 1.0 / r.upsilon;
    }
    r.hyperbolic = inv_omega < r.tau_dx * (1.0 - 1e-12) ? 1 : 0;
    r.alpha = r.hyperbolic ? 1.0 / (1.0 + r.upsilon) : 0.99 * r.alpha_hi;
    r.h = r.alpha * dx / f_min;
    r.eps_threshold = f_min * dx / (2.0 * (1.0 + r.upsilon));
    *out = r;
    return PDD_OK;
}

pdd_status pdd_get_patch_rounds(pdd_ctx *ctx, int32_t *dst, int32_t count)
{
    if (!ctx || !dst) return fail(ctx, PDD_E_INVALID, "NULL argument");
    if (count > ctx->n_patches + 1) count = ctx->n_patches + 1;
    CK(cudaMemcpy(dst, ctx->T.patch_round, sizeof(int32_t) * count, cudaMemcpyDeviceToHost));
    return PDD_OK;
}

pdd_status pdd_get_patch_residuals(pdd_ctx *ctx, double *dst, int32_t count)
{
    if (!ctx || !dst) return fail(ctx, PDD_E_INVALID, "NULL argument");
    if (count > ctx->n_patches + 1) count = ctx->n_patches + 1;
    CK(cudaMemcpy(dst, ctx->T.patch_res, sizeof(double) * count, cudaMemcpyDeviceToHost));
    return PDD_OK;
}

pdd_status pdd_get_tile_rounds(pdd_ctx *ctx, int32_t *dst, int32_t count)
{
    if (!ctx || !dst) return fail(ctx, PDD_E_INVALID, "NULL argument");
    if (ctx->prepared_kernel < 0) return fail(ctx, PDD_E_STATE, "no solve has run");
    if (count > ctx->n_tiles) count = ctx->n_tiles;
    CK(cudaMemcpy(dst, ctx->T.tile_round, sizeof(int32_t) * count, cudaMemcpyDeviceToHost));
    return PDD_OK;
}

pdd_status pdd_set_tile_shape(pdd_ctx *ctx, int32_t rows, int32_t cols)
{
    if (!ctx) return fail(nullptr, PDD_E_INVALID, "ctx is NULL");
    DevGuard dev_guard(ctx->device);
    const bool ok = (rows == 0 && cols == 0) || (rows == 32 && cols == 64) || (rows == 16 && cols == 128) ||
                    (rows == 16 && cols == 64);
    if (!ok) return fail(ctx, PDD_E_INVALID, "tile shape must be 0 x 0 (automatic), 32 x 64, 16 x 128 or 16 x 64");
    ctx->force_tile_cols = cols;
    ctx->force_tile_rows = rows;
    return PDD_OK;
}

pdd_status pdd_choose_tile_shape(int32_t n, double lo, double hi, int32_t patchy, int32_t *rows,
                                 int32_t *cols)
{
    if (n < 3 || !(hi > lo) || !rows || !cols)
        return fail(nullptr, PDD_E_INVALID, "pdd_choose_tile_shape: need n >= 3, hi > lo and output pointers");
    pdd_problem p{};
    p.n = n;
    p.lo = lo;
    p.hi = hi;
    const int geo = p3_geometry_choice(&p, patchy != 0, 0, 0);
    *rows = geo == 0 ? 32 : 16;
    *cols = geo == 1 ? 128 : 64;
    return PDD_OK;
}

pdd_status pdd_set_tile_cols(pdd_ctx *ctx, int32_t cols)
{
    if (!ctx) return fail(nullptr, PDD_E_INVALID, "ctx is NULL");
    DevGuard dev_guard(ctx->device);
    if (cols != 0 && cols != 64 && cols != 128) return fail(ctx, PDD_E_INVALID, "tile cols must be 0, 64 or 128");
    return pdd_set_tile_shape(ctx, cols == 64 ? 32 : cols == 128 ? 16 : 0, cols);
}

static pdd_status fetch(pdd_ctx *ctx, void *dst, const void *src, size_t bytes, int on_device)
{
    if (!dst) return fail(ctx, PDD_E_INVALID, "dst is NULL");
    if (!src) return fail(ctx, PDD_E_STATE, "array not computed yet");
    CK(cudaMemcpyAsync(dst, src, bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return PDD_OK;
}


pdd_status pdd_get_values(pdd_ctx *ctx, void *dst, int32_t dst_on_device, int32_t as_fp64)
{
    if (!ctx) return fail(nullptr, PDD_E_INVALID, "ctx is NULL");
    DevGuard dev_guard(ctx->device);
    const size_t N = (size_t)ctx->fine.n * ctx->fine.n;
    if (as_fp64) return fetch(ctx, dst, ctx->V, sizeof(double) * N, dst_on_device);
    if (!dst) return fail(ctx, PDD_E_INVALID, "dst is NULL");
    // convert on the device; host destinations get one D2H copy of the fp32 staging buffer
    float *f = dst_on_device ? (float *)dst : ctx->f32buf;
    k_to_f32<<<4 * 148, 256, 0, ctx->stream>>>(ctx->V, f, (int64_t)N);
    ctx->launches++;
    CK(cudaGetLastError());
    if (!dst_on_device)
        CK(cudaMemcpyAsync(dst, f, sizeof(float) * N, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return PDD_OK;
}

pdd_status pdd_set_values(pdd_ctx *ctx, const double *src, int32_t src_on_device)
{
    if (!ctx || !src) return fail(ctx, PDD_E_INVALID, "NULL argument");
    const size_t N = (size_t)ctx->fine.n * ctx->fine.n;
    CK(cudaMemcpyAsync(ctx->V, src, sizeof(double) * N,
                       src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return PDD_OK;
}

pdd_status pdd_get_uhat(pdd_ctx *ctx, double *dst, int32_t on_device)
{
    if (!ctx) return fail(nullptr, PDD_E_INVALID, "ctx is NULL");
    DevGuard dev_guard(ctx->device);
    if (!ctx->synth_done) return fail(ctx, PDD_E_STATE, "u_hat not computed (pdd_synthesize)");
    return fetch(ctx, dst, ctx->uhat, sizeof(double) * ctx->fine.n * ctx->fine.n, on_device);
}

pdd_status pdd_get_coarse_values(pdd_ctx *ctx, double *dst, int32_t on_device)
{
    if (!ctx) return fail(nullptr, PDD_E_INVALID, "ctx is NULL");
    DevGuard dev_guard(ctx->device);
    if (!ctx->coarse_done) return fail(ctx, PDD_E_STATE, "u_c not computed (pdd_coarse_solve)");
    return fetch(ctx, dst, ctx->uc_final, sizeof(double) * ctx->coarse.n * ctx->coarse.n, on_device);
}

pdd_status pdd_get_controls(pdd_ctx *ctx, uint8_t *dst, int32_t on_device)
{
    if (!ctx) return fail(nullptr, PDD_E_INVALID, "ctx is NULL");
    DevGuard dev_guard(ctx->device);
    if (!ctx->synth_done) return fail(ctx, PDD_E_STATE, "a* not computed (pdd_synthesize)");
    return fetch(ctx, dst, ctx->astar, (size_t)ctx->fine.n * ctx->fine.n, on_device);
}

pdd_status pdd_get_labels(pdd_ctx *ctx, int16_t *dst, int32_t on_device)
{
    if (!ctx) return fail(nullptr, PDD_E_INVALID, "ctx is NULL");
    DevGuard dev_guard(ctx->device);
    if (!ctx->labels_mode) return fail(ctx, PDD_E_STATE, "labels not built");
    return fetch(ctx, dst, ctx->labels, sizeof(int16_t) * ctx->fine.n * ctx->fine.n, on_device);
}

pdd_status pdd_get_successors(pdd_ctx *ctx, int32_t *dst, int32_t on_device)
{
    if (!ctx) return fail(nullptr, PDD_E_INVALID, "ctx is NULL");
    DevGuard dev_guard(ctx->device);
    if (ctx->labels_mode != 1) return fail(ctx, PDD_E_STATE, "successors not built (pdd_build_patches)");
    return fetch(ctx, dst, ctx->succ0, sizeof(int32_t) * ctx->fine.n * ctx->fine.n, on_device);
}

}  // extern "C"
