// sweep.cu -- the hot path: the semi-Lagrangian value-iteration sweep of the self-dependency-free
// scheme (SLscheme3; discount R1-R3) on the fine grid, run over an active-tile list.
//
// One CTA (8 warps) per active tile of TH x TW nodes.  The CTA stages the tile plus a halo of H
// cells (H = ceil(reach) + 1, R4) of V in shared memory, relative to a per-tile reference value
// V_ref (u = V - V_ref; fp32 or fp64 arithmetic, fp64 storage in HBM, R27), relaxes it k_inner
// times in place (chaotic relaxation: a valid schedule of the same monotone contraction, so it
// converges to the same fixed point, P:452-472 + R29), then writes changed nodes back.
//
// Thread mapping ("lane = control"): a warp walks the nodes of one row left to right; lane L
// holds controls k = L + 32 c (c < CPL) and computes their candidate values, then a 5-step
// __shfl_xor_sync butterfly takes the min over controls (the discrete min of P:376-377).
//
// Two stencil paths:
//  * general (path 1): every lane evaluates its controls' 2p foot points
//        x_i + h f(x_i, a_k) +- sqrt(h p) sigma_j(x_i),   f = c(x) a + d(x)
//    in cell units relative to the node (no absolute coordinates: fp32-safe at 8193^2),
//    clamps them to the box (R5), gathers the 4 bilinear corners from shared memory, removes
//    the node's own corner (its weight goes to Lambda0) and combines
//        v_k - V_ref = (D + beta w R'_k) / (1 - beta w Lambda0_k),  D = h l - (1 - beta) V_ref
//    (the same operator written relative to V_ref; exact algebra, R27).
//  * row-table (path 2): when c, d and sigma depend on x2 only (C1, C2, C4, C5), every interior
//    node of a row has the same stencil per control.  A host-built table holds, per (row,
//    control), the branch-merged compact stencil: window origin (oy, ox), WY x WX weights
//    W = beta w lambda / (1 - beta Lambda0) and E = 1/(1 - beta Lambda0).  Each lane keeps its
//    controls' weights and a WY x WX window of u in registers and slides the window along the
//    row: per node and control it loads WY new values (conflict-free: the pitch is chosen so
//    the distinct window origins of a warp fall in distinct banks) and issues WY*WX FFMAs.
//    Nodes within H of the x-boundary (x clamping) and Dirichlet nodes fall back to the general
//    stencil / are skipped (warp-uniform branches on per-row ballot masks).
// Check mode (K10 of SURVEY.md): one pure Jacobi pass, no update; residual per tile, optional
// output T(V) (pdd_apply_operator).
#include "pdd_internal.cuh"

#include <math.h>
#include <stdio.h>

#include <algorithm>

// PDD_WIDE_UNIT: this file compiled a second time with PDD_P3_WIDE=1 (build.py) gives the
// 16 x 128 path-3 tile in namespace pdd::wide; the host picks the geometry per problem
// (runtime.cu: p3_use_wide) and launch_sweep forwards path-3 launches of 128-column tiles here
#ifndef PDD_WIDE_UNIT
#define PDD_WIDE_UNIT 0
#endif
// PDD_LOW_UNIT: a third build with PDD_P3_TH=16 gives the 16 x 64 path-3 tile in namespace pdd::low
// (patchy solves on grids of up to ~16 k tiles: fewer wasted updates along the u_hat front)
#ifndef PDD_LOW_UNIT
#define PDD_LOW_UNIT 0
#endif
#define PDD_ALT_UNIT (PDD_WIDE_UNIT || PDD_LOW_UNIT)

namespace pdd {
#if PDD_WIDE_UNIT
namespace wide {
#elif PDD_LOW_UNIT
namespace low {
#endif

#ifndef PDD_MIN_BLOCKS
#define PDD_MIN_BLOCKS 0    // override of the __launch_bounds__ min CTAs per SM (0 = per path)
#endif

// register cap per path: the GS row-table kernel (path 3) at 80 registers keeps 3 CTAs (24
// warps) per SM without spills -- measured 1.6x faster than its unconstrained 137-register build
#ifndef PDD_MIN_BLOCKS1
#define PDD_MIN_BLOCKS1 2   // path 1 (general stencil) CTAs per SM bound (measured: C3 patchy
                            // 0.124 -> 0.106 s, static 0.29 -> 0.22 s against 1 CTA/SM)
#endif
#ifndef PDD_MIN_BLOCKS4
#define PDD_MIN_BLOCKS4 4   // path 4 (lean general stencil): 64 registers at 8 warps, 32 warps / SM
#endif
#ifndef PDD_MIN_BLOCKS3
#define PDD_MIN_BLOCKS3 3   // path 3 (row-table GS) CTAs per SM bound: 80 registers at 8 warps
#endif
template <int PATH>
constexpr int min_blocks() { return PDD_MIN_BLOCKS > 0 ? PDD_MIN_BLOCKS : (PATH == 3 ? PDD_MIN_BLOCKS3 : PATH == 1 ? PDD_MIN_BLOCKS1 : PATH == 4 ? PDD_MIN_BLOCKS4 : 1); }
#ifndef PDD_TH
#define PDD_TH 16           // tile rows of the general / fp64 kernels (paths 1, 2, 4; multiple of NW).
                            // 16 since round 2: under the work queue smaller tiles waste fewer
                            // updates along the front and fill the GPU on mid-size grids (measured,
                            // profiles/r2w_general_tile16_ab.txt: C3 patchy fine solve 49 -> 35 ms,
                            // static 141 -> 118 ms; C5@2049 fp64 patchy 0.249 -> 0.165 s; the
                            // paper's 800^2 workloads within 2 %)
#endif
constexpr int TH = PDD_TH;      // tile rows
constexpr int PROG_N = 32;      // row-pipeline progress counters per CTA: the tallest tile (32 x 64)
#ifndef PDD_NW
#define PDD_NW 8
#endif
constexpr int NW = PDD_NW;      // warps per CTA
constexpr int RPW = TH / NW;    // rows per warp
constexpr int TW_GENERAL = 64;
constexpr unsigned FULL = 0xffffffffu;

// path 4 in fp64 needs twice the registers: 2 CTAs / SM
template <typename real, int PATH>
constexpr int min_blocks_r() { return (PATH == 4 && sizeof(real) == 8) ? 2 : min_blocks<PATH>(); }
// PDD_CHECKED (development builds; compute-sanitizer is not available on the GPU pool): bounds
// checks of the kernels' own making on every shared-memory address the sweeps form (window loads,
// corner gathers, commits, staging stores) and on tile indices; violations are counted in g_fault
// (read by pdd_dev_faults) instead of trapping.  scripts/run_checked.sh runs the GPU tests on it.
#ifndef PDD_CHECKED
#define PDD_CHECKED 0
#endif
#if PDD_CHECKED
__device__ unsigned long long g_fault[2];   // [0] violations, [1] code of the first one
__device__ __forceinline__ void chk_fail(int code)
{
    atomicAdd(&g_fault[0], 1ull);
    atomicCAS(&g_fault[1], 0ull, (unsigned long long)code);
}
struct ChkBounds { const char *lo, *hi; };
__device__ __forceinline__ ChkBounds &chk_bounds()
{
    __shared__ ChkBounds b;
    return b;
}
#define PDD_CHK(cond, code) do { if (!(cond)) chk_fail(code); } while (0)
// the bytes [p, p + n reals) lie inside the staged V tile (+ halo, all shifted copies)
#define PDD_CHK_TILE(p, n, code)                                                              \
    PDD_CHK((const char *)(p) >= chk_bounds().lo && (const char *)((p) + (n)) <= chk_bounds().hi, code)
#else
#define PDD_CHK(cond, code) ((void)0)
#define PDD_CHK_TILE(p, n, code) ((void)0)
#endif

template <int WY, int WX>
struct TWOf { static constexpr int value = WX > 0 ? WX * (64 / (WX > 0 ? WX : 1)) : 64; };   // multiple of WX, <= 64

int rowtab_tw(int WY, int WX) { (void)WY; return WX * (64 / WX); }
void p3_geometry(int &pitch, int &cstride, int &hmax);
int sweep_tile_rows() { return TH; }

bool rowtab_supported(int WY, int WX, int cpl)
{
    return cpl >= 1 && cpl <= 2 &&
           ((WY == 3 && WX == 3) || (WY == 2 && WX == 5) || (WY == 4 && WX == 4));
}

size_t rowtab_entry_bytes(int precision, int WY, int WX)
{
    if (precision == 32) {
        if (WY == 3 && WX == 3) return sizeof(RowEntry<float, 3, 3>);
        if (WY == 2 && WX == 5) return sizeof(RowEntry<float, 2, 5>);
        return sizeof(RowEntry<float, 4, 4>);
    }
    if (WY == 3 && WX == 3) return sizeof(RowEntry<double, 3, 3>);
    if (WY == 2 && WX == 5) return sizeof(RowEntry<double, 2, 5>);
    return sizeof(RowEntry<double, 4, 4>);
}

template <typename real>
struct KP {
    DProblem P;
    double *V;
    TileGeom g;
    const int32_t *list;
    double *tile_res, *tile_chg;
    float *tile_edge;
    int k_inner;
    double *out;
    const void *rowtab;
    int na_pad;
    int Hx;
    double early_tol;     // path 3: stop the in-tile sweeps once a sweep changes less than this
    const int32_t *tile_free;
    unsigned long long *nu_counter;
    const uint8_t *tile_orient;
    int oxor;             // packed 2-bit orientation xor per sweep mod 4
    double early_rel;     // also stop once a sweep changes less than this x the first sweep
    int k_coherent;       // in-tile sweeps of a coherent tile (tile_orient bit 2)
    const RoundCtl *ctl;  // device-driven round (k_sweep_dyn), else NULL
    ActCounters *acnt;
    int32_t *tile_stamp;
    int32_t *tile_sweeps;
    const int16_t *labels;            // check mode: patch labels for the per-patch residuals
    unsigned long long *patch_res;    //   per-patch max |T(V) - V| (fp64 bits) or NULL
    const int32_t *lab_off;           //   with lab_res: per-tile, per-label residuals into the
    const int16_t *lab_ids;           //   tile's CSR entries instead of atomics on patch_res
    unsigned long long *lab_res;
    int n_slots;
};

__device__ __forceinline__ float rmin(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ double rmin(double a, double b) { return fmin(a, b); }
__device__ __forceinline__ float rmax(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double rmax(double a, double b) { return fmax(a, b); }
__device__ __forceinline__ float rfloor(float a) { return floorf(a); }
__device__ __forceinline__ double rfloor(double a) { return floor(a); }
__device__ __forceinline__ float rabs(float a) { return fabsf(a); }
__device__ __forceinline__ double rabs(double a) { return fabs(a); }
template <typename real> __device__ __forceinline__ real rinf();
template <> __device__ __forceinline__ float rinf<float>() { return __int_as_float(0x7f800000); }
template <> __device__ __forceinline__ double rinf<double>() { return __longlong_as_double(0x7ff0000000000000LL); }

template <typename real>
__device__ __forceinline__ real warp_min(real v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = rmin(v, __shfl_xor_sync(FULL, v, o));
    return v;
}

#ifndef PDD_REDUX
#define PDD_REDUX 1
#endif
#if PDD_REDUX
// fp32 min over the warp in ONE integer REDUX instead of a 5-step shuffle butterfly: the float is
// mapped to a signed int of the same order (negative values: magnitude bits flipped), reduced by
// redux.sync.min.s32 and mapped back -- exact, the result is one of the inputs (measured on C5:
// sweep kernel +20 % node-updates/s; the f32 form of redux.sync is lowered to shuffles on sm_100a)
template <>
__device__ __forceinline__ float warp_min<float>(float v)
{
    const int i = __float_as_int(v);
    int k = i ^ ((i >> 31) & 0x7fffffff);
    k = __reduce_min_sync(FULL, k);
    return __int_as_float(k ^ ((k >> 31) & 0x7fffffff));
}
#endif

// Per-node coefficients of the general stencil (values at node (gi, gj)); loaded from global
// memory by node_coef.  The row-pipelined kernel prefetches them for a whole row at its start so
// that no global load sits on the node-by-node dependency chain.
template <typename real>
struct NodeCoef {
    real c, d1, d2, o[2][2], sa, D;
};

template <typename real>
__device__ __forceinline__ NodeCoef<real> node_coef(const DProblem &P, int gi, int gj, real D,
                                                    double Vref)
{
    const int n = P.n;
    NodeCoef<real> r;
    r.c = (real)coef_at(P.speed, gi, gj, n);
    r.d1 = (real)coef_at(P.drift[0], gi, gj, n);
    r.d2 = (real)coef_at(P.drift[1], gi, gj, n);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        r.o[k][0] = k < P.p ? (real)(P.sc * coef_at(P.sigma[k][0], gi, gj, n)) : (real)0;
        r.o[k][1] = k < P.p ? (real)(P.sc * coef_at(P.sigma[k][1], gi, gj, n)) : (real)0;
    }
    // sigma(x, a) = s(x) a (sigma_mode 1, R32): the single noise column follows the control
    r.sa = P.sigma_mode == 1 ? (real)(P.sc * coef_at(P.sigma[0][0], gi, gj, n)) : (real)0;
    // a running-cost field needs D = h l(x_i) - (1 - beta) V_ref per node (fp64 then rounded)
    r.D = P.cost.kind != 0 ? (real)(P.h * coef_at(P.cost, gi, gj, n) - (1.0 - P.beta) * Vref) : D;
    return r;
}

template <typename real>
__device__ __forceinline__ real general_node_c(const DProblem &P, const real *__restrict__ s_ctrl,
                                               const real *base, int pitch, int gi, int gj,
                                               const NodeCoef<real> &nc);

// General stencil at one node (lane = control).  base points at the node in shared memory.
template <typename real>
__device__ __forceinline__ real general_node(const DProblem &P, const real *__restrict__ s_ctrl,
                                          const real *base, int pitch, int gi, int gj, real D,
                                          double Vref)
{
    return general_node_c<real>(P, s_ctrl, base, pitch, gi, gj, node_coef<real>(P, gi, gj, D, Vref));
}

// Out-of-line form for the nodes with x-clamped feet of the row-table kernel (boundary tiles
// only): keeps the general stencil's registers out of the 80-register row loop.
template <typename real>
__device__ __noinline__ real general_node_edge(const DProblem &P, const real *__restrict__ s_ctrl,
                                               const real *base, int pitch, int gi, int gj, real D,
                                               double Vref)
{
    return general_node<real>(P, s_ctrl, base, pitch, gi, gj, D, Vref);
}

template <typename real>
__device__ __forceinline__ real general_node_c(const DProblem &P, const real *__restrict__ s_ctrl,
                                               const real *base, int pitch, int gi, int gj,
                                               const NodeCoef<real> &nc)
{
    const int lane = threadIdx.x & 31;
    const int n = P.n;
    const real c = nc.c, d1 = nc.d1, d2 = nc.d2;
    const int p = P.p;
    const int nb = p > 0 ? 2 * p : 1;
    real off[2][2] = {{nc.o[0][0], nc.o[0][1]}, {nc.o[1][0], nc.o[1][1]}};
    const real q = (real)P.q;
    const real bw = (real)(P.beta / (double)nb);
    const real xlo = (real)(-gi), xhi = (real)(n - 1 - gi);
    const real ylo = (real)(-gj), yhi = (real)(n - 1 - gj);
    const real cxm = (real)(n - 2 - gi), cym = (real)(n - 2 - gj);
    const real D = nc.D;
    const real sa = nc.sa;
    const real uself = *base;
    const bool big_self = rabs(uself) > (real)1e3;   // |u_self| >> any value difference of a tile
    real best = rinf<real>();
    for (int k = lane; k < P.na; k += 32) {
        const real bx = q * (c * s_ctrl[2 * k] + d1);
        const real by = q * (c * s_ctrl[2 * k + 1] + d2);
        if (P.sigma_mode == 1) {
            off[0][0] = sa * s_ctrl[2 * k];
            off[0][1] = sa * s_ctrl[2 * k + 1];
        }
        // l(x, a_k) = l(x) + m(a_k) (R33)
        const real Dk = P.cost_ctrl ? D + (real)(P.h * __ldg(P.cost_ctrl + k)) : D;
        real R = 0, L0 = 0;
        for (int b = 0; b < nb; ++b) {
            real xr = bx, yr = by;
            if (p > 0) {
                const int kk = b >> 1;
                if (b & 1) { xr -= off[kk][0]; yr -= off[kk][1]; }
                else       { xr += off[kk][0]; yr += off[kk][1]; }
            }
            xr = rmin(rmax(xr, xlo), xhi);
            yr = rmin(rmax(yr, ylo), yhi);
            const real fx = rmin(rfloor(xr), cxm);
            const real fy = rmin(rfloor(yr), cym);
            const real tx = xr - fx, ty = yr - fy;
            const real *pc = base + (int)fy * pitch + (int)fx;
            PDD_CHK_TILE(pc, 2, 3);
            PDD_CHK_TILE(pc + pitch, 2, 3);
            const real ws = rmax((real)0, (real)1 - rabs(xr)) * rmax((real)0, (real)1 - rabs(yr));
            if (big_self) {
                // the node's own corner enters with value 0 (its weight goes to Lambda0,
                // P:433-436): excluding it, rather than subtracting ws u_self afterwards, keeps R
                // exact when u_self is large (an exit problem's 1e6 start value next to the
                // front, fp32); warp-uniform branch, taken only for such nodes
                const int ix = (int)fx, iy = (int)fy;
                const real u00 = (ix == 0 && iy == 0) ? (real)0 : pc[0];
                const real u10 = (ix == -1 && iy == 0) ? (real)0 : pc[1];
                const real u01 = (ix == 0 && iy == -1) ? (real)0 : pc[pitch];
                const real u11 = (ix == -1 && iy == -1) ? (real)0 : pc[pitch + 1];
                const real a0 = u00 + tx * (u10 - u00);
                const real a1 = u01 + tx * (u11 - u01);
                R += a0 + ty * (a1 - a0);
            } else {
                const real u00 = pc[0], u10 = pc[1], u01 = pc[pitch], u11 = pc[pitch + 1];
                const real a0 = u00 + tx * (u10 - u00);
                const real a1 = u01 + tx * (u11 - u01);
                R += (a0 + ty * (a1 - a0)) - ws * uself;
            }
            L0 += ws;
        }
        const real v = (Dk + bw * R) / ((real)1 - bw * L0);
        best = rmin(best, v);
    }
    return warp_min(best);
}

// per-row ballot masks: bit lx set = Dirichlet or outside the grid (dmask) / needs the general
// stencil because its feet may be clamped in x (emask)
__device__ __forceinline__ void row_masks(const DProblem &P, int TW, int i0, int gj, int Hx,
                                          unsigned long long &dmask, unsigned long long &emask)
{
    const int lane = threadIdx.x & 31;
    const int n = P.n;
    dmask = 0ull;
    emask = 0ull;
    for (int part = 0; part < (TW + 31) / 32; ++part) {
        const int lx = part * 32 + lane;
        const int gi = i0 + lx;
        const bool oob = lx >= TW || gi >= n;
        const bool dir = oob || P.kind[(int64_t)gj * n + gi] != 0;
        const bool edge = !dir && (gi < Hx || gi > n - 1 - Hx);
        dmask |= (unsigned long long)__ballot_sync(FULL, dir) << (32 * part);
        emask |= (unsigned long long)__ballot_sync(FULL, edge) << (32 * part);
    }
}

// Per-patch residual of a verification pass (check mode: each patch's own
// sup-norm residual): the CTA accumulates max |T(V) - V| per label in shared memory (labels <
// PRES_SH; larger ones go straight to global atomics) and flushes it once per tile visit.
constexpr int PRES_SH = 512;
__device__ __forceinline__ unsigned long long *pres_table()
{
    __shared__ unsigned long long t[PRES_SH];
    return t;
}
template <typename real>
__device__ __forceinline__ void patch_acc(const KP<real> &A, int64_t gidx, double r)
{
    const int lab = A.labels[gidx];
    if (lab < 0 || lab >= A.n_slots) return;
    const unsigned long long b = (unsigned long long)__double_as_longlong(r);
    if (lab < PRES_SH) atomicMax(pres_table() + lab, b);
    else atomicMax(A.patch_res + lab, b);
}

// NCOPY: the G4 path keeps 4 copies of the tile shifted by q floats (copy q of element e at
// q*cstride + q + e) so that every lane's 4-column window load is a 16-byte aligned LDS.128.
template <typename real, bool CHECK, int NCOPY = 1>
__device__ __forceinline__ void commit_node(real *p, real best, bool last, real &res,
                                            double *out, int64_t gidx, double Vref,
                                            int cstride = 0, const KP<real> *A = nullptr)
{
    if ((threadIdx.x & 31) == 0) {
        const real old = *p;
        if (last) res = rmax(res, rabs(best - old));
        if constexpr (!CHECK) {
#pragma unroll
            for (int q = 0; q < NCOPY; ++q) {
                PDD_CHK_TILE(p + q * cstride + q, 1, 4);
                p[q * cstride + q] = best;
            }
        } else {
            if (out) out[gidx] = Vref + (double)best;
            if (A && A->patch_res) patch_acc(*A, gidx, (double)rabs(best - old));
        }
    }
}

// ------------------------------------------------------------------ row processors
template <typename real, bool CHECK>
__device__ __forceinline__ void row_general(const KP<real> &A, real *s_u, const real *s_ctrl,
                                            int pitch, int H, int TW, int i0, int ly, int gj,
                                            real D, bool last, real &res, double Vref)
{
    unsigned long long dmask, emask;
    row_masks(A.P, TW, i0, gj, 0, dmask, emask);
    const int n = A.P.n;
    real *rowp = s_u + (ly + H) * pitch + H;
    for (int lx = 0; lx < TW; ++lx) {
        if ((dmask >> lx) & 1ull) continue;
        const int gi = i0 + lx;
        const real best = general_node<real>(A.P, s_ctrl, rowp + lx, pitch, gi, gj, D, Vref);
        commit_node<real, CHECK>(rowp + lx, best, last, res, A.out, (int64_t)gj * n + gi, Vref, 0, &A);
    }
}

template <typename real, int CPL, int WY, int WX, bool CHECK>
__device__ __forceinline__ void row_table(const KP<real> &A, real *s_u, const real *s_ctrl,
                                          int pitch, int H, int i0, int ly, int gj, real D,
                                          bool last, real &res, double Vref)
{
    constexpr int TW = TWOf<WY, WX>::value;
    const int lane = threadIdx.x & 31;
    const int n = A.P.n;
    unsigned long long dmask, emask;
    row_masks(A.P, TW, i0, gj, A.Hx, dmask, emask);

    const RowEntry<real, WY, WX> *tab =
        reinterpret_cast<const RowEntry<real, WY, WX> *>(A.rowtab) + (int64_t)gj * A.na_pad;
    real Wt[CPL][WY * WX];
    real c0[CPL];
    int base[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const int k = lane + 32 * c;
        const RowEntry<real, WY, WX> &e = tab[k];
        const real Dk = (k < A.P.na && A.P.cost_ctrl) ? D + (real)(A.P.h * A.P.cost_ctrl[k]) : D;   // R33
        c0[c] = k < A.P.na ? Dk * e.E : rinf<real>();
#pragma unroll
        for (int m = 0; m < WY * WX; ++m) Wt[c][m] = e.W[m];
        base[c] = (ly + H + e.oy) * pitch + H + e.ox;
    }
    real win[CPL][WY][WX];
#pragma unroll
    for (int c = 0; c < CPL; ++c)
#pragma unroll
        for (int r = 0; r < WY; ++r)
#pragma unroll
            for (int x = 0; x < WX - 1; ++x) win[c][r][x] = s_u[base[c] + r * pitch + x];

    real *rowp = s_u + (ly + H) * pitch + H;
    for (int g = 0; g < TW; g += WX) {
#pragma unroll
        for (int s = 0; s < WX; ++s) {
            const int lx = g + s;
#pragma unroll
            for (int c = 0; c < CPL; ++c)
#pragma unroll
                for (int r = 0; r < WY; ++r)
                    win[c][r][(s + WX - 1) % WX] = s_u[base[c] + r * pitch + lx + WX - 1];
            if (((dmask | emask) >> lx) & 1ull) continue;
            real best = rinf<real>();
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                real acc = c0[c];
#pragma unroll
                for (int r = 0; r < WY; ++r)
#pragma unroll
                    for (int x = 0; x < WX; ++x)
                        acc = fma(Wt[c][r * WX + x], win[c][r][(s + x) % WX], acc);
                best = rmin(best, acc);
            }
            best = warp_min(best);
            commit_node<real, CHECK>(rowp + lx, best, last, res, A.out,
                                     (int64_t)gj * n + i0 + lx, Vref, 0, &A);
        }
    }
    // nodes whose feet may be clamped in x: general stencil (same Jacobi-in-row semantics)
    unsigned long long em = emask & ~dmask;
    while (em) {
        const int lx = __ffsll((long long)em) - 1;
        em &= em - 1;
        const real best = general_node<real>(A.P, s_ctrl, rowp + lx, pitch, i0 + lx, gj, D, Vref);
        commit_node<real, CHECK>(rowp + lx, best, last, res, A.out, (int64_t)gj * n + i0 + lx,
                                 Vref, 0, &A);
    }
}

#ifndef PDD_BIGREF
#define PDD_BIGREF 1     // V_ref = staged min on a tile whose values span > 1 + |min| (R39)
#endif
#ifndef PDD_PREFETCH
#define PDD_PREFETCH 0   // 1: L2 prefetch of the next tile while sweeping (measured slower: spills)
#endif
#ifndef PDD_TILE_KEY
#define PDD_TILE_KEY 0
#endif
#ifndef PDD_FASTWB
#define PDD_FASTWB 1     // single-sweep visits: write-back without reading the old V
#endif
#ifndef PDD_EDGE_ACT
#define PDD_EDGE_ACT 0   // 1: re-activate a tile only for changes in the neighbour's facing strip
#endif
#ifndef PDD_GSG
#define PDD_GSG 1    // path 1 (general stencil) uses the Gauss-Seidel tile sweeps of sweep_gs.cuh
#endif
#include "sweep_gs.cuh"
#include "sweep_gf.cuh"

constexpr bool kRawMinRef = PDD_RAWMIN != 0;   // fp32 path 3: V_ref = staged min (sweep_gs.cuh)

// PDD_TIMING (development builds): thread 0 of every CTA adds the cycles of each phase of a tile
// visit to g_phase (0 fetch / queue, 1 stage loads, 2 convert + smem stores, 3 sweeps, 4 residual
// reduction, 5 write-back, 6 bookkeeping); read and reset by pdd_dev_phases()
#ifndef PDD_TIMING
#define PDD_TIMING 0
#endif
#if PDD_TIMING
__device__ unsigned long long g_phase[8];
__device__ __forceinline__ void phase_mark(int i, long long &t_prev)
{
    if (threadIdx.x == 0) {
        const long long now = clock64();
        atomicAdd(&g_phase[i], (unsigned long long)(now - t_prev));
        t_prev = now;
    }
}
#define PDD_PHASE(i) phase_mark(i, t_phase)
#else
#define PDD_PHASE(i) ((void)0)
#endif

// ------------------------------------------------------------------ work-queue schedule
// Tile states: 0 clean, 1 queued, 2 visiting, 3 visiting and dirtied meanwhile.  A queued or
// visiting tile holds one unit of ctl->work (an admission in flight reserves one too); the queue
// is drained for good when work reaches 0 with every tile admitted.
// The ring is a ticket queue: a consumer takes ticket h = head++ and waits for slot h & (cap - 1)
// to be filled; a producer takes position p = tail++ and fills slot p & (cap - 1).  No CTA ever
// polls the cursors, each waits on its own slot (cap > tiles + resident CTAs: two outstanding
// tickets never share a slot).
__device__ __forceinline__ int q_ld(const int *p) { return *(volatile const int *)p; }

__device__ __forceinline__ void q_push(const QueueArgs &Q, int t)
{
    const unsigned long long pos = atomicAdd(&Q.ctl->tail, 1ull);
    volatile int32_t *slot = Q.ring + (pos & (unsigned long long)(Q.cap - 1));
    while (*slot != 0) __nanosleep(32);   // the consumer of the previous lap still reads it
    *slot = t + 1;
}

// one unit of work is gone; the last one (with every tile admitted) ends the launch
__device__ __forceinline__ void q_release(const QueueArgs &Q)
{
    if (atomicSub(&Q.ctl->work, 1) == 1 && q_ld(&Q.ctl->adm) >= Q.n_order) atomicExch(&Q.ctl->stop, 1);
}

// admit the next tile of the key order (lock-free: the reservation of a unit of work comes first,
// so work cannot reach 0 while an admission is in flight)
__device__ __forceinline__ void q_admit_one(const QueueArgs &Q)
{
    atomicAdd(&Q.ctl->work, 1);
    const int a = atomicAdd(&Q.ctl->adm, 1);
    if (a < Q.n_order) {
        const int t = Q.order[a];
        if (atomicCAS(Q.state + t, 0, 1) == 0) {   // else a neighbour queued it already
            q_push(Q, t);
            return;
        }
    }
    q_release(Q);
}

// a neighbour dirtied tile t
__device__ __forceinline__ void q_mark_dirty(const QueueArgs &Q, int t)
{
    int st = q_ld(Q.state + t);
    for (;;) {
        if (st == 0) {
            const int o = atomicCAS(Q.state + t, 0, 1);
            if (o == 0) {
                atomicAdd(&Q.ctl->work, 1);
                q_push(Q, t);
                return;
            }
            st = o;
        } else if (st == 2) {
            const int o = atomicCAS(Q.state + t, 2, 3);
            if (o == 2) return;
            st = o;
        } else {
            return;   // already queued, or visiting and already dirty
        }
    }
}

// thread 0: a consumer ticket, and the tile that arrives on it: >= 0, -1 once the queue has
// stopped, or (block = false) -3 while the slot is still empty -- the ticket stays valid
__device__ __forceinline__ unsigned long long q_ticket(const QueueArgs &Q)
{
    return atomicAdd(&Q.ctl->head, 1ull);
}

__device__ __forceinline__ int q_take(const QueueArgs &Q, unsigned long long ticket, bool block)
{
    volatile int32_t *slot = Q.ring + (ticket & (unsigned long long)(Q.cap - 1));
    int v;
    // watchdog: no visit finished anywhere for ~1 s of waiting (a visit takes ~0.1 ms) can only be
    // a lost unit of work: stop with the non-convergence code instead of hanging the GPU
    unsigned long long seen = *(volatile unsigned long long *)&Q.ctl->visits;
    long long t0 = clock64();
    for (;;) {
        if (q_ld(&Q.ctl->stop) >= 2) return -1;   // visit cap / verification due: leave the rest queued
        if ((v = *slot) != 0) break;
        if (q_ld(&Q.ctl->stop)) return -1;
        if (!block) return -3;
        __nanosleep(200);
        if (clock64() - t0 > (1ll << 31)) {
            const unsigned long long now = *(volatile unsigned long long *)&Q.ctl->visits;
            if (now == seen) atomicExch(&Q.ctl->stop, 2);
            seen = now;
            t0 = clock64();
        }
    }
    *slot = 0;
    const int t = v - 1;
    PDD_CHK(t >= 0 && Q.rank[t] < Q.n_order, 6);
    atomicExch(Q.state + t, 2);   // queued -> visiting (only the consumer changes state 1)
    __threadfence();              // acquire: the visit's loads of V come after the state change
    return t;
}

// after the visit (one thread): back to the queue when dirtied meanwhile or not converged, else
// clean -- and, patchy, the next tiles of the key order take its place
__device__ __forceinline__ void q_finish(const QueueArgs &Q, int t, bool self_dirty)
{
    if (!self_dirty && atomicCAS(Q.state + t, 2, 0) == 2) {
#pragma unroll 1
        for (int k = 0; k < 4; ++k) {
            if (q_ld(&Q.ctl->adm) >= Q.n_order || q_ld(&Q.ctl->work) > Q.target) break;
            q_admit_one(Q);
        }
        q_release(Q);
        return;
    }
    atomicExch(Q.state + t, 1);   // not converged, or 3: a neighbour changed during the visit
    q_push(Q, t);
}

// ------------------------------------------------------------------ tile prefetch (work queue)
// The work-queue kernel overlaps the staging of its NEXT tile with the end of the current visit:
// once the sweeps are done, thread 0 takes the next tile off the queue and every thread issues
// asynchronous 8-byte global -> shared copies (cp.async, LDGSTS in SASS) of that tile + halo of V
// (fp64) into a staging buffer; the residual reduction, the write-back and the queue bookkeeping
// of the current tile run meanwhile, and the next visit starts with its values already on chip.
// Element e of the (TH + 2H) x (TW + 2H) block belongs to thread e % 256 for the copy and for the
// read, so a thread's cp.async.wait_group is all the synchronisation the buffer needs.
// (V rows are only 8-byte aligned -- n is odd -- so neither 16-byte cp.async nor a TMA tensor map
// applies; ordering against other CTAs' writes of V: the consumer's acquire in q_take.)
struct Pref {
    double *stage;                // staging buffer, (TH + 2H)(TW + 2H) doubles
    const QueueArgs *Q;
    unsigned long long *ticket;   // shared: the consumer ticket taken for the next tile
    int *next;                    // shared: next tile (>= 0), -1 queue stopped, -3 not there yet
};

template <int PATH, int WY, int WX>
struct TileDims {
    static constexpr int TW = PATH == 2 ? TWOf<WY, WX>::value : PATH == 3 ? TW3 : TW_GENERAL;
    static constexpr int THt = PATH == 3 ? TH3 : TH;
    static constexpr int MAXE = ((THt + 16) * (TW + 16) + NW * 32 - 1) / (NW * 32);   // H <= 8
};

__device__ __forceinline__ void cp_async8(double *dst_shared, const double *src_global)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst_shared);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src_global) : "memory");
}

template <typename real, int PATH, int WY, int WX>
__device__ __forceinline__ void stage_issue(const KP<real> &A, int t, double *stage)
{
    constexpr int TW = TileDims<PATH, WY, WX>::TW, THt = TileDims<PATH, WY, WX>::THt;
    constexpr int MAXE = TileDims<PATH, WY, WX>::MAXE;
    const int H = A.g.H, n = A.P.n;
    const int i0 = (t % A.g.tiles_x) * TW, j0 = (t / A.g.tiles_x) * THt;
    const int W2 = TW + 2 * H, H2 = THt + 2 * H;
#pragma unroll
    for (int m = 0; m < MAXE; ++m) {
        const int e = threadIdx.x + m * NW * 32;
        if (e < H2 * W2) {
            const int r = e / W2, c = e - r * W2;
            const int gj = j0 - H + r, gi = i0 - H + c;
            if (gj >= 0 && gj < n && gi >= 0 && gi < n) cp_async8(stage + e, A.V + (int64_t)gj * n + gi);
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// ------------------------------------------------------------------ one tile visit
// Stage tile + halo, relax k_inner times, write back.  Global V is read with ld.global.cg (L2):
// in the persistent schedules other CTAs update V during the launch.  PREF: the values were
// prefetched into pf->stage (stage_issue), and the next tile is prefetched before the write-back.
template <typename real, int PATH, int CPL, int WY, int WX, bool CHECK, bool PREF = false>
__device__ __forceinline__ void sweep_tile(const KP<real> &A, int t, unsigned char *smem_raw,
                                           double *res_out, double *chg_out,
#if PDD_TIMING
                                           long long &t_phase,
#endif
                                           const Pref *pf = nullptr)
{
    PDD_PHASE(0);
    constexpr int TW = PATH == 2 ? TWOf<WY, WX>::value : PATH == 3 ? TW3 : TW_GENERAL;
    constexpr int THt = PATH == 3 ? TH3 : TH;      // tile rows of this path
    constexpr int NCOPY = PATH == 3 ? 4 : 1;
    double *s_red = reinterpret_cast<double *>(smem_raw);            // NW
    volatile int *s_prog = reinterpret_cast<volatile int *>(s_red + NW);   // PROG_N progress counters
    real *s_ctrl = reinterpret_cast<real *>(s_red + NW + PROG_N / 2);   // 2 * 128
    real *s_u = s_ctrl + 256;
    const int H = A.g.H, pitch = A.g.pitch;
    const int n = A.P.n;
    const int i0 = (t % A.g.tiles_x) * TW;
    const int j0 = (t / A.g.tiles_x) * THt;
#if PDD_CHECKED
    PDD_CHK(t >= 0 && t < A.g.tiles_x * A.g.tiles_y, 1);
    if (threadIdx.x == 0) {
        chk_bounds().lo = (const char *)s_u;
        chk_bounds().hi = (const char *)(s_u + (PATH == 3 ? 4 * A.g.cstride : (THt + 2 * H) * pitch));
    }
    __syncthreads();
#endif
    // stage tile + halo (coalesced fp64 row reads, held in registers: one consistent snapshot
    // even while neighbouring CTAs of the same round write their tiles), converted relative to
    // V_ref = the tile-centre value (|u| at most half the tile's value range), or with PDD_RAWMIN
    // min(V0, minimum of the staged values): every u >= 0 and D >= 0, so every candidate
    // c0 + sum W u is >= 0 and the fp32 min over controls can compare raw float bits
    const int W2 = TW + 2 * H, H2 = THt + 2 * H;
    constexpr int MAXE = ((THt + 16) * (TW + 16) + NW * 32 - 1) / (NW * 32);   // (TH + 2H)(TW + 2H), H <= 8
    double vs[MAXE];
    double vmin = INFINITY;
    __shared__ double s_cref;                       // PREF: the staged tile-centre value
    const int ci = min(i0 + TW / 2, n - 1), cj = min(j0 + THt / 2, n - 1);
    const int e_c = (cj - j0 + H) * W2 + (ci - i0 + H);
    if constexpr (PREF) asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int m = 0; m < MAXE; ++m) {
        const int e = threadIdx.x + m * (int)blockDim.x;
        vs[m] = INFINITY;
        if (e < H2 * W2) {
            const int r = e / W2, c = e - r * W2;
            const int gj = j0 - H + r, gi = i0 - H + c;
            if (gj >= 0 && gj < n && gi >= 0 && gi < n) {
                if constexpr (PREF) {
                    vs[m] = pf->stage[e];           // this thread's own cp.async landed it
                    if (e == e_c) s_cref = vs[m];
                } else {
                    vs[m] = __ldcg(A.V + (int64_t)gj * n + gi);
                }
                vmin = fmin(vmin, vs[m]);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) vmin = fmin(vmin, __shfl_xor_sync(FULL, vmin, o));
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = vmin;
    __syncthreads();
    PDD_PHASE(1);
    // V_ref <= V0 keeps D = h l - (1 - beta) V_ref >= 0 also for inputs above the supersolution
    // V0 (pdd_apply_operator on arbitrary V, u_hat above V0 in enclosed regions)
    double Vref;
    if constexpr (PATH == 3 && sizeof(real) == 4 && kRawMinRef) {
        Vref = A.P.v0;
#pragma unroll
        for (int w = 0; w < NW; ++w) Vref = fmin(Vref, s_red[w]);
    } else {
        // the tile-centre value keeps |u| smallest (fp64 runs to r <= 1e-12 (1 - beta) sit at a
        // few ulp of u) -- except on a tile whose staged values span more than 1 + |min| (an exit
        // problem's 1e6 start values, or values interpolated from them, next to the front, R39):
        // then the smallest staged value, so that the nodes the front has reached keep full
        // precision next to the placeholders
        if constexpr (PREF) Vref = s_cref;          // same snapshot as the staged values
        else Vref = __ldcg(A.V + (int64_t)cj * n + ci);
        if (PDD_BIGREF) {
            double vminb = s_red[0];
#pragma unroll
            for (int w = 1; w < NW; ++w) vminb = fmin(vminb, s_red[w]);
            double vmax = -INFINITY;
#pragma unroll
            for (int m = 0; m < MAXE; ++m) vmax = fmax(vmax, vs[m] < INFINITY ? vs[m] : -INFINITY);
            const int wide = __syncthreads_or(vmax - vminb > 1.0 + fabs(vminb));
            if (wide) Vref = vminb;
        }
    }
#pragma unroll
    for (int m = 0; m < MAXE; ++m) {
        const int e = threadIdx.x + m * (int)blockDim.x;
        if (e < H2 * W2) {
            const int r = e / W2, c = e - r * W2;
            const real v = vs[m] < INFINITY ? (real)(vs[m] - Vref) : (real)0;
#pragma unroll
            for (int q = 0; q < NCOPY; ++q) {
                PDD_CHK_TILE(s_u + q * A.g.cstride + q + r * pitch + c, 1, 2);
                s_u[q * A.g.cstride + q + r * pitch + c] = v;
            }
        }
    }
    if constexpr (PATH == 4) {
        // q a_k, h m(a_k) and the tile's x-varying coefficient planes: c, then q d1, q d2 (WX)
        real *s_cf = s_u + (TH + 2 * H) * GF_PITCH;
        real *s_hm = s_cf + A.g.cstride;
        for (int e = threadIdx.x; e < 2 * A.P.na; e += blockDim.x) s_ctrl[e] = (real)(A.P.q * A.P.ctrl[e]);
        for (int e = threadIdx.x; e < A.P.na; e += blockDim.x)
            s_hm[e] = A.P.cost_ctrl ? (real)(A.P.h * A.P.cost_ctrl[e]) : (real)0;
        for (int e = threadIdx.x; e < TH * TW; e += blockDim.x) {
            const int ly = e / TW, lx = e - ly * TW;
            const int gi = min(i0 + lx, n - 1), gj = min(j0 + ly, n - 1);
            s_cf[e] = (real)coef_at(A.P.speed, gi, gj, n);
            if constexpr (WX != 0) {
                s_cf[TH * TW + e] = (real)(A.P.q * coef_at(A.P.drift[0], gi, gj, n));
                s_cf[2 * TH * TW + e] = (real)(A.P.q * coef_at(A.P.drift[1], gi, gj, n));
            }
        }
    } else {
        for (int e = threadIdx.x; e < 2 * A.P.na; e += blockDim.x) s_ctrl[e] = (real)A.P.ctrl[e];
    }
    if (threadIdx.x < THt) s_prog[threadIdx.x] = 0;
    if constexpr (CHECK) {
        if (A.patch_res)
            for (int e = threadIdx.x; e < PRES_SH; e += blockDim.x) pres_table()[e] = 0ull;
    }
    __syncthreads();
    PDD_PHASE(2);

    // D = h l - (1 - beta) V_ref >= 0 (V_ref <= V0 = h l / (1 - beta); the clamp removes fp64
    // rounding noise at V_ref = V0) for a constant cost; a cost field uses D per node in the
    // general path
    const double Dd = A.P.h * A.P.lmax_x - (1.0 - A.P.beta) * Vref;
    const real D = (real)((PATH == 3 && sizeof(real) == 4 && kRawMinRef) ? fmax(Dd, 0.0) : Dd);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    real res = 0;
    int done_sweeps = CHECK ? 1 : A.k_inner;
    float edge4[4] = {-1.f, -1.f, -1.f, -1.f};   // path 3: per-side change bounds (else: chg)
    if constexpr (PATH == 3 && sizeof(real) == 4) {
        const int ot = A.tile_orient ? A.tile_orient[t] : 0;
        const int kin = (ot & 4) ? min(A.k_inner, A.k_coherent) : A.k_inner;
        // a coherent tile restarts from its downstream orientation on every visit; any other
        // tile continues the orientation cycle where its last visit stopped
        const int sbase = (A.tile_sweeps && !(ot & 4)) ? A.tile_sweeps[t] : 0;
        done_sweeps = tile_gs4<CPL, WY, WX, CHECK>(A, s_u, s_ctrl, s_prog, s_red, pitch,
                                                   A.g.cstride, H, i0, j0, D, kin, res, Vref, ot & 3,
                                                   sbase, edge4);
    } else if constexpr (PATH == 4) {
        // lean general stencil (sweep_gf.cuh): CPL unused, WY = branches NB, WX = 1 when the drift
        // varies along x; coefficient planes behind the V tile, h m(a) behind them
        const real *s_cf = s_u + (TH + 2 * H) * GF_PITCH;
        const real *s_hm = s_cf + A.g.cstride;
        const int ot = A.tile_orient ? A.tile_orient[t] : 0;
        const int kin = (ot & 4) ? min(A.k_inner, A.k_coherent) : A.k_inner;
        const int sbase = (A.tile_sweeps && !(ot & 4)) ? A.tile_sweeps[t] : 0;
        done_sweeps = tile_gsf<real, WY, WX != 0, CHECK>(A, s_u, s_ctrl, s_hm, s_cf, s_prog, s_red, H, i0,
                                                        j0, kin, res, Vref, ot & 3, sbase);
    } else if constexpr (PATH == 1 && PDD_GSG) {
        const int ot = A.tile_orient ? A.tile_orient[t] : 0;
        const int kin = (ot & 4) ? min(A.k_inner, A.k_coherent) : A.k_inner;
        const int sbase = (A.tile_sweeps && !(ot & 4)) ? A.tile_sweeps[t] : 0;
        done_sweeps = tile_gsg<real, CHECK>(A, s_u, s_ctrl, s_prog, s_red, pitch, H, i0, j0, D,
                                            kin, res, Vref, ot & 3, sbase);
    } else {
        const int sweeps = CHECK ? 1 : A.k_inner;
        for (int sw = 0; sw < sweeps; ++sw) {
            const bool last = sw == sweeps - 1;
            for (int rr = 0; rr < RPW; ++rr) {
                const int ly = warp * RPW + ((sw & 1) ? RPW - 1 - rr : rr);
                const int gj = j0 + ly;
                if (gj >= n) continue;
                if constexpr (PATH == 2)
                    row_table<real, CPL, WY, WX, CHECK>(A, s_u, s_ctrl, pitch, H, i0, ly, gj, D,
                                                        last, res, Vref);
                else
                    row_general<real, CHECK>(A, s_u, s_ctrl, pitch, H, TW, i0, ly, gj, D, last,
                                             res, Vref);
            }
            if (!CHECK) __syncthreads();
        }
    }

    PDD_PHASE(3);
    // tile residual of the last sweep (path 3 commits from lanes 0, 8, 16, 24)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) res = rmax(res, __shfl_xor_sync(FULL, res, o));
    if (lane == 0) s_red[warp] = (double)res;
    if constexpr (PREF) {
        // the sweeps are done: take the next tile off the queue (if one is there already) ...
        if (threadIdx.x == 0) {
            *pf->ticket = q_ticket(*pf->Q);
            *pf->next = q_take(*pf->Q, *pf->ticket, false);
        }
    }
    __syncthreads();
    if constexpr (PREF) {
        // ... and start its copies: they overlap the reduction, the write-back and the queue
        // bookkeeping of this visit (every thread has read its staged values long ago)
        const int tn = *pf->next;
        if (tn >= 0) stage_issue<real, PATH, WY, WX>(A, tn, pf->stage);
    }
    double rmaxv = 0.0;
    for (int w = 0; w < NW; ++w) rmaxv = fmax(rmaxv, s_red[w]);
    if (threadIdx.x == 0) A.tile_res[t] = rmaxv;
    if (res_out) *res_out = rmaxv;
    if constexpr (CHECK) {
        if (A.patch_res && A.lab_res) {
            // per-label residuals of THIS tile into its CSR entries (labels < PRES_SH: the caller
            // checks n_slots): a later partial verification replaces only the visited tiles' entries
            for (int k = A.lab_off[t] + threadIdx.x; k < A.lab_off[t + 1]; k += blockDim.x)
                A.lab_res[k] = pres_table()[A.lab_ids[k]];
        } else if (A.patch_res) {
            const int m = min(A.n_slots, PRES_SH);
            for (int e = threadIdx.x; e < m; e += blockDim.x) {
                const unsigned long long v = pres_table()[e];
                if (v) atomicMax(A.patch_res + e, v);
            }
        }
        __syncthreads();
        return;
    }
    __syncthreads();
    PDD_PHASE(4);

    // write back changed interior nodes, net change of the visit
    double chg = 0.0;
    if (PDD_FASTWB && done_sweeps == 1) {
        // one sweep: the visit's net change of a node IS that sweep's change, so the tile's net
        // change is the sweep residual (rmaxv) and the write-back needs no read of the old V
        // (a dependent global load per node on the visit's critical path); every free node is
        // written (an unchanged node is rewritten within the arithmetic's rounding of V - V_ref)
        constexpr int PER = (THt * TW + NW * 32 - 1) / (NW * 32);
        uint8_t kd[PER];
#pragma unroll
        for (int m = 0; m < PER; ++m) {
            const int e = threadIdx.x + m * NW * 32;
            const int ly = e / TW, lx = e - ly * TW;
            const int gi = i0 + lx, gj = j0 + ly;
            kd[m] = (e < THt * TW && gi < n && gj < n) ? A.P.kind[(int64_t)gj * n + gi] : (uint8_t)1;
        }
#pragma unroll
        for (int m = 0; m < PER; ++m) {
            const int e = threadIdx.x + m * NW * 32;
            if (kd[m] != 0) continue;
            const int ly = e / TW, lx = e - ly * TW;
            PDD_CHK(j0 + ly < n && i0 + lx < n, 5);
            A.V[(int64_t)(j0 + ly) * n + i0 + lx] = Vref + (double)s_u[(ly + H) * pitch + lx + H];
        }
        chg = rmaxv;
    } else
    for (int e = threadIdx.x; e < THt * TW; e += blockDim.x) {
        const int ly = e / TW, lx = e - ly * TW;
        const int gi = i0 + lx, gj = j0 + ly;
        if (gi >= n || gj >= n) continue;
        const int64_t gidx = (int64_t)gj * n + gi;
        if (A.P.kind[gidx] != 0) continue;
        // the visit's net change is measured on the stored values: an update below the
        // rounding of V = V_ref + u (fp64 runs: |u| << |V|) changes nothing and wakes nobody
        const double vnew = Vref + (double)s_u[(ly + H) * pitch + lx + H];
        const double vold = __ldcg(A.V + gidx);
        if (vnew != vold) {
            A.V[gidx] = vnew;
            chg = fmax(chg, fabs(vnew - vold));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) chg = fmax(chg, __shfl_xor_sync(FULL, chg, o));
    if (lane == 0) s_red[warp] = chg;
    __syncthreads();
    double cm = 0.0;
    for (int w = 0; w < NW; ++w) cm = fmax(cm, s_red[w]);
    if (threadIdx.x == 0) {
        A.tile_chg[t] = cm;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            A.tile_edge[4 * t + q] = edge4[q] >= 0.f ? fminf(edge4[q], (float)cm) : (float)cm;
        if (A.tile_stamp) A.tile_stamp[t] = A.ctl->sweep_id + 1;
        if (A.tile_sweeps) A.tile_sweeps[t] += done_sweeps;
        if (A.nu_counter)   // node-updates actually performed (early exit aware)
            atomicAdd(A.nu_counter, (unsigned long long)A.tile_free[t] * (unsigned long long)done_sweeps);
    }
    if (chg_out) *chg_out = cm;
    __syncthreads();
    PDD_PHASE(5);
}

// Round schedule: one CTA per listed tile (chaotic relaxation across the tiles of a launch).
template <typename real, int PATH, int CPL, int WY, int WX, bool CHECK>
__global__ void __launch_bounds__(NW * 32, min_blocks_r<real, PATH>()) k_sweep(KP<real> A)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    #if PDD_TIMING
    long long t_phase = clock64();
    sweep_tile<real, PATH, CPL, WY, WX, CHECK>(A, A.list[blockIdx.x], smem_raw, nullptr, nullptr, t_phase);
#else
    sweep_tile<real, PATH, CPL, WY, WX, CHECK>(A, A.list[blockIdx.x], smem_raw, nullptr, nullptr);
#endif
}

// Device-driven round: persistent CTAs take the activated tiles one at a time (dynamic fetch),
// the count is the activation's -- no host round trip between activation and sweep.
template <typename real, int PATH, int CPL, int WY, int WX>
__global__ void __launch_bounds__(NW * 32, min_blocks_r<real, PATH>()) k_sweep_dyn(KP<real> A)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int s_t;
    if (A.ctl->stop) return;
    const int count = A.acnt->count;
#if PDD_TIMING
    long long t_phase = clock64();
#endif
#if PDD_PREFETCH
    // fetch one tile ahead and pull its tile + halo rows of V into L2 while the current tile is
    // swept, so that the next visit's staging loads hit L2 instead of HBM
    __shared__ int s_next;
    if (threadIdx.x == 0) {
        const int i = atomicAdd(&A.acnt->fetch, 1);
        s_next = i < count ? A.list[i] : -1;
    }
    for (;;) {
        __syncthreads();
        const int t = s_next;
        __syncthreads();
        if (t < 0) return;
        if (threadIdx.x == 0) {
            const int i = atomicAdd(&A.acnt->fetch, 1);
            s_next = i < count ? A.list[i] : -1;
        }
        __syncthreads();
        const int tn = s_next;
        if (tn >= 0) {
            const int TWt = PATH == 2 ? TWOf<WY, WX>::value : PATH == 3 ? TW3 : TW_GENERAL;
            const int THq = PATH == 3 ? TH3 : TH;
            const int n = A.P.n, H = A.g.H;
            const int i0 = (tn % A.g.tiles_x) * TWt - H, j0 = (tn / A.g.tiles_x) * THq - H;
            const int rows = THq + 2 * H, cols = TWt + 2 * H;
            // one 128-byte line per thread-step: 16 doubles
            const int lines_per_row = (cols + 15) / 16 + 1;
            for (int e = threadIdx.x; e < rows * lines_per_row; e += blockDim.x) {
                const int r = e / lines_per_row, c = (e - r * lines_per_row) * 16;
                const int gj = j0 + r, gi = min(max(i0 + c, 0), n - 1);
                if (gj >= 0 && gj < n)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(A.V + (int64_t)gj * n + gi));
            }
        }
        #if PDD_TIMING
        sweep_tile<real, PATH, CPL, WY, WX, false>(A, t, smem_raw, nullptr, nullptr, t_phase);
#else
        sweep_tile<real, PATH, CPL, WY, WX, false>(A, t, smem_raw, nullptr, nullptr);
#endif
    }
#else
    for (;;) {
        if (threadIdx.x == 0) {
            const int i = atomicAdd(&A.acnt->fetch, 1);
            s_t = i < count ? A.list[i] : -1;
        }
        __syncthreads();
        const int t = s_t;
        __syncthreads();
        if (t < 0) return;
        #if PDD_TIMING
        sweep_tile<real, PATH, CPL, WY, WX, false>(A, t, smem_raw, nullptr, nullptr, t_phase);
#else
        sweep_tile<real, PATH, CPL, WY, WX, false>(A, t, smem_raw, nullptr, nullptr);
#endif
    }
#endif
}

// Ordered schedule (one pass): persistent CTAs take tiles in ascending key order (P:744-749,
// u_hat for the patchy method; block-lexicographic for the static squares)
// and visit a tile only after every neighbour with a smaller key (and the same group, when
// groups are given) has finished its visit of this pass: a Gauss-Seidel pass over tiles in the
// key order.  Deadlock-free: a tile waits only on tiles taken earlier from the same counter.
// A tile is skipped (but still marked done) when its last residual is < tol and no neighbour
// changed by >= tol after its last visit (visit stamps).
template <typename real, int PATH, int CPL, int WY, int WX>
__global__ void __launch_bounds__(NW * 32, min_blocks_r<real, PATH>()) k_sweep_ordered(KP<real> A, OrderArgs O)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int s_idx;
    const int tid = threadIdx.x;
#if PDD_TIMING
    long long t_phase = clock64();
#endif
    for (;;) {
        if (tid == 0) s_idx = atomicAdd(O.counter, 1);
        __syncthreads();
        const int idx = s_idx;
        if (idx >= O.n_order) break;
        const int t = O.order[idx];
        const int tx = t % A.g.tiles_x, ty = t / A.g.tiles_x;
        const double kt = O.key[t];
        const int gt = O.group ? O.group[t] : -1;
        const long long st = ((volatile long long *)O.stamp)[t];
        bool pred = false;
        if (tid < 9) {
            if (tid == 8) {
                pred = ((volatile double *)A.tile_res)[t] >= O.tol;
            } else {
                const int k = tid < 4 ? tid : tid + 1;            // skip the centre
                const int ax = tx + (k % 3) - 1, ay = ty + (k / 3) - 1;
                if (ax >= 0 && ay >= 0 && ax < A.g.tiles_x && ay < A.g.tiles_y) {
                    const int nb = ay * A.g.tiles_x + ax;
                    // a tile without free nodes is not in the order (the host lists only tiles
                    // with tile_free > 0) and never finishes a pass: nothing to wait for
                    if (O.tile_free[nb] > 0 && O.key[nb] < kt - O.key_slack &&
                        (!O.group || O.group[nb] == gt)) {
                        while (((volatile int *)O.done)[nb] < O.pass) __nanosleep(64);
                        __threadfence();
                    }
                    pred = ((volatile double *)A.tile_chg)[nb] >= O.tol &&
                           ((volatile long long *)O.stamp)[nb] > st;
                }
            }
        }
        const bool need = __syncthreads_or(pred) && O.tile_free[t] > 0;
        if (need) {
            double r = 0.0, c = 0.0;
#if PDD_TIMING
            sweep_tile<real, PATH, CPL, WY, WX, false>(A, t, smem_raw, &r, &c, t_phase);
#else
            sweep_tile<real, PATH, CPL, WY, WX, false>(A, t, smem_raw, &r, &c);
#endif
            if (tid == 0 && O.tile_round) {
                O.tile_round[t] = max(O.tile_round[t], O.pass);
                for (int k = O.lab_off[t]; k < O.lab_off[t + 1]; ++k) atomicMax(&O.patch_round[O.lab_ids[k]], O.pass);
            }
            if (tid == 0) {
                O.stamp[t] = (long long)atomicAdd(O.seq, 1ull) + 1;
                atomicAdd(O.processed, 1);
                atomicAdd(O.free_sum, (unsigned long long)O.tile_free[t]);
                atomicMax(O.max_res, (unsigned long long)__double_as_longlong(r));
            }
        }
        if (tid == 0) {
            __threadfence();
            ((volatile int *)O.done)[t] = O.pass;
        }
        __syncthreads();
    }
}

// bytes of dynamic shared memory of a sweep CTA before the prefetch staging buffer
template <typename real, int PATH>
__host__ __device__ constexpr size_t sweep_smem_base(int H, int pitch, int cstride)
{
    // path 4: cstride carries the size of the coefficient planes, 128 reals of h m(a) follow
    return NW * sizeof(double) + PROG_N * sizeof(int) + 256 * sizeof(real) +
           (PATH == 3 ? (size_t)4 * cstride
                      : (size_t)(TH + 2 * H) * pitch + (PATH == 4 ? (size_t)cstride + 128 : 0)) * sizeof(real);
}
// Measured (profiles/r2g_prefetch_ab.txt): the prefetch pays on the general-stencil kernel (C3:
// fine solve -5 %), whose CTAs use little shared memory; on the fp32 row-table kernel (path 3) the
// staging buffer takes the three resident CTAs to 220 KB of the SM's 228 KB (the L1 that serves
// the row-table and node-kind reads shrinks to the minimum) and the other two CTAs already cover
// a CTA's staging latency: C5 +6 %, C4 +3 % slower.  So path 3 stages with plain loads
// (PDD_PREFETCH3=1 builds the prefetch there too, for A/B runs; never on the 16 x 128 tile, where
// three CTAs would not fit).
#ifndef PDD_PREFETCH3
#define PDD_PREFETCH3 0
#endif
template <int PATH>
__host__ __device__ constexpr bool queue_prefetch()
{
    return PATH != 3 || (PDD_PREFETCH3 != 0 && TW3 != 128);
}

template <typename real, int PATH, int CPL, int WY, int WX>
__global__ void __launch_bounds__(NW * 32, min_blocks_r<real, PATH>()) k_sweep_queue(KP<real> A, QueueArgs Q)
{
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr bool PREF = queue_prefetch<PATH>();
    __shared__ int s_t, s_next;
    __shared__ unsigned long long s_ticket;
    const int tid = threadIdx.x;
    Pref pf;
    pf.stage = reinterpret_cast<double *>(
        smem_raw + ((sweep_smem_base<real, PATH>(A.g.H, A.g.pitch, A.g.cstride) + 15) & ~(size_t)15));
    pf.Q = &Q;
    pf.ticket = &s_ticket;
    pf.next = &s_next;
#if PDD_TIMING
    long long t_phase = clock64();
#endif
    // nothing seeded and nothing left to admit: no producer would ever end the wait
    if (tid == 0 && q_ld(&Q.ctl->work) == 0 && q_ld(&Q.ctl->adm) >= Q.n_order) atomicExch(&Q.ctl->stop, 1);
    if (tid == 0) s_t = q_take(Q, q_ticket(Q), true);
    __syncthreads();
    int t = s_t;
    if (t < 0) return;
    if constexpr (PREF) stage_issue<real, PATH, WY, WX>(A, t, pf.stage);
    for (;;) {
        double r = 0.0, c = 0.0;
        if (tid == 0) s_next = -3;
#if PDD_TIMING
        sweep_tile<real, PATH, CPL, WY, WX, false, PREF>(A, t, smem_raw, &r, &c, t_phase, &pf);
#else
        sweep_tile<real, PATH, CPL, WY, WX, false, PREF>(A, t, smem_raw, &r, &c, &pf);   // ends with a barrier
#endif
        if (tid < 32) {
            if (tid < 9 && tid != 4 && c >= Q.tol_act) {
                __threadfence();   // this visit's V writes before anyone sees the dirty marks
                const int tx = t % A.g.tiles_x, ty = t / A.g.tiles_x;
                const int ax = tx + (tid % 3) - 1, ay = ty + (tid / 3) - 1;
                if (ax >= 0 && ay >= 0 && ax < A.g.tiles_x && ay < A.g.tiles_y) {
                    const int nb = ay * A.g.tiles_x + ax;
                    // only admitted tiles: the others are dirty anyway and enter on admission
                    if (Q.rank[nb] < q_ld(&Q.ctl->adm)) q_mark_dirty(Q, nb);
                }
            }
            __syncwarp();          // the neighbours hold their units of work before t gives up its own
            if (tid == 4) {
                const unsigned long long seq = atomicAdd(&Q.ctl->visits, 1ull) + 1;
                if (r >= Q.tol) atomicMax(&Q.ctl->max_res, (unsigned long long)__double_as_longlong(r));
                if (Q.tile_round) Q.tile_round[t] = (int32_t)seq;   // per-patch rounds: k_patch_rounds
                if (seq >= Q.ctl->max_visits) atomicExch(&Q.ctl->stop, 2);
                else if (seq >= Q.ctl->verify_at) atomicCAS(&Q.ctl->stop, 0, 3);
                q_finish(Q, t, r >= Q.tol);
            }
        }
        PDD_PHASE(6);
        // the next tile: prefetched during the visit, or wait for it now
        if (tid == 0) {
            int tn = s_next;
            const bool waited = tn == -3;
            if (waited) tn = q_take(Q, PREF ? s_ticket : q_ticket(Q), true);
            s_t = tn;
            s_next = waited ? -3 : tn;
        }
        __syncthreads();
        t = s_t;
        if (t < 0) {
            PDD_PHASE(0);
            return;
        }
        if constexpr (PREF) {
            if (s_next == -3) stage_issue<real, PATH, WY, WX>(A, t, pf.stage);
        }
        __syncthreads();           // s_next is reset at the top of the loop
    }
}

template <typename real, int PATH, int CPL, int WY, int WX, bool CHECK>
static cudaError_t launch_one(const SweepLaunch &L, cudaStream_t s)
{
    KP<real> A;
    A.P = L.P;
    A.V = L.V;
    A.g = L.g;
    A.list = L.list;
    A.tile_res = L.tile_res;
    A.tile_chg = L.tile_chg;
    A.tile_edge = L.tile_edge;
    A.k_inner = L.k_inner;
    A.out = L.out;
    A.rowtab = L.rowtab;
    A.na_pad = L.na_pad;
    A.Hx = L.Hx;
    A.early_tol = L.early_tol;
    A.tile_free = L.tile_free;
    A.tile_orient = L.tile_orient;
    A.oxor = L.oxor;
    A.early_rel = L.early_rel;
    A.k_coherent = L.k_coherent;
    A.ctl = L.ctl;
    A.acnt = L.acnt;
    A.tile_stamp = L.tile_stamp;
    A.tile_sweeps = L.tile_sweeps;
    A.nu_counter = L.nu_counter;
    A.labels = L.labels;
    A.patch_res = CHECK ? L.patch_res : nullptr;
    A.lab_off = L.lab_off;
    A.lab_ids = L.lab_ids;
    A.lab_res = CHECK ? L.lab_res : nullptr;
    A.n_slots = L.n_slots;
    const size_t smem_base = sweep_smem_base<real, PATH>(L.g.H, L.g.pitch, L.g.cstride);
    const int tw_ = PATH == 2 ? TWOf<WY, WX>::value : PATH == 3 ? TW3 : TW_GENERAL;
    const int th_ = PATH == 3 ? TH3 : TH;
    // the work-queue kernel adds the staging buffer of its tile prefetch
    const size_t smem = (L.queued && !CHECK && queue_prefetch<PATH>())
                            ? ((smem_base + 15) & ~(size_t)15) +
                                  sizeof(double) * (size_t)(th_ + 2 * L.g.H) * (tw_ + 2 * L.g.H)
                            : smem_base;
    // (the opt-in for large dynamic shared memory is taken from 40 KB on: the kernels' static shared
    // memory -- up to 4 KB for the per-patch residual table of check launches -- counts against
    // the 48 KB default limit too)
    // path 4 is built for the work queue and for check launches only
    if constexpr (PATH == 4 && !CHECK) {
        if (!L.queued) return cudaErrorInvalidValue;
    }
    if constexpr (PATH != 4) if (L.ordered && !CHECK) {
        auto kern = k_sweep_ordered<real, PATH, CPL, WY, WX>;
        if (smem > 40 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem);
            if (e != cudaSuccess) return e;
        }
        int per_sm = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32, smem);
        if (e != cudaSuccess) return e;
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        int grid = std::max(1, per_sm) * sms;
        if (grid > L.order.n_order) grid = L.order.n_order;
        if (grid <= 0) return cudaSuccess;
        kern<<<grid, NW * 32, smem, s>>>(A, L.order);
        return cudaGetLastError();
    }
    if (L.queued && !CHECK) {
        auto kern = k_sweep_queue<real, PATH, CPL, WY, WX>;
        if (smem > 40 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem);
            if (e != cudaSuccess) return e;
        }
        int per_sm = 0, dev = 0, sms = 148;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32, smem);
        if (e != cudaSuccess) return e;
        if (L.occupancy_out) {
            *L.occupancy_out = std::max(1, per_sm);
            return cudaSuccess;
        }
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        // every CTA must be resident at once: idle CTAs spin on the queue
        kern<<<std::max(1, per_sm) * sms, NW * 32, smem, s>>>(A, L.queue);
        return cudaGetLastError();
    }
    if constexpr (PATH != 4) if ((L.ctl || L.occupancy_out) && !CHECK) {
        auto kern = k_sweep_dyn<real, PATH, CPL, WY, WX>;
        // occupancy and the shared-memory attribute are per device: cached per device ordinal
        constexpr int kMaxDev = 64;
        static int per_sm_dev[kMaxDev] = {}, sms_dev[kMaxDev] = {};
        int dev = 0;
        cudaGetDevice(&dev);
        int per_sm = 0, sms = 0;
        if (dev >= kMaxDev || per_sm_dev[dev] == 0) {
            if (smem > 40 * 1024) {
                cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)smem);
                if (e != cudaSuccess) return e;
            }
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NW * 32, smem);
            if (e != cudaSuccess) return e;
            per_sm = std::max(1, per_sm);
            if (dev < kMaxDev) { per_sm_dev[dev] = per_sm; sms_dev[dev] = sms; }
        } else {
            per_sm = per_sm_dev[dev];
            sms = sms_dev[dev];
        }
        if (L.occupancy_out) {
            *L.occupancy_out = per_sm;
            return cudaSuccess;
        }
        int grid = per_sm * sms;
        if (grid > L.n_list) grid = L.n_list;     // n_list: upper bound of the count
        if (grid <= 0) return cudaSuccess;
        kern<<<grid, NW * 32, smem, s>>>(A);
        return cudaGetLastError();
    }
    if constexpr (PATH != 4 || CHECK) {
        auto kern = k_sweep<real, PATH, CPL, WY, WX, CHECK>;
        if (smem > 40 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem);
            if (e != cudaSuccess) return e;
        }
        if (L.n_list <= 0) return cudaSuccess;
        kern<<<L.n_list, NW * 32, smem, s>>>(A);
        return cudaGetLastError();
    }
    return cudaErrorInvalidValue;
}

template <typename real, bool CHECK>
static cudaError_t dispatch(const SweepLaunch &L, cudaStream_t s)
{
    if (L.path == 1) return launch_one<real, 1, 1, 1, 1, CHECK>(L, s);
    if (L.path == 4) {
        // lean general stencil: WY = branches (2 or 4), WX = drift varies along x; only the
        // work queue and check launches are built for it (runtime.cu prepare())
        if (L.ordered || (L.ctl && !CHECK)) return cudaErrorInvalidValue;
        if (L.WY == 2) return L.WX ? launch_one<real, 4, 1, 2, 1, CHECK>(L, s) : launch_one<real, 4, 1, 2, 0, CHECK>(L, s);
        if (L.WY == 4) return L.WX ? launch_one<real, 4, 1, 4, 1, CHECK>(L, s) : launch_one<real, 4, 1, 4, 0, CHECK>(L, s);
        return cudaErrorInvalidValue;
    }
    const int cpl = L.na_pad / 32;
    if constexpr (sizeof(real) == 4) {
        if (L.path == 3) {
#define PDD_RT4(WY_, WX_)                                                                    \
            if (L.WY == WY_ && L.WX == WX_) {                                               \
                if (cpl == 1) return launch_one<float, 3, 1, WY_, WX_, CHECK>(L, s);        \
                return launch_one<float, 3, 2, WY_, WX_, CHECK>(L, s);                      \
            }
            PDD_RT4(3, 3)
            PDD_RT4(2, 5)
            PDD_RT4(4, 4)
#undef PDD_RT4
            return cudaErrorInvalidValue;
        }
    }
#define PDD_RT(WY_, WX_)                                                                     \
    if (L.WY == WY_ && L.WX == WX_) {                                                        \
        if (cpl == 1) return launch_one<real, 2, 1, WY_, WX_, CHECK>(L, s);                  \
        return launch_one<real, 2, 2, WY_, WX_, CHECK>(L, s);                                \
    }
    PDD_RT(3, 3)
    PDD_RT(2, 5)
    PDD_RT(4, 4)
#undef PDD_RT
    return cudaErrorInvalidValue;
}

void p3_geometry(int &pitch, int &cstride, int &hmax)
{
    pitch = P3_PITCH;
    cstride = P3_CSTRIDE;
    hmax = P3_HMAX;
}

#if !PDD_ALT_UNIT
void gf_geometry(int &pitch) { pitch = GF_PITCH; }
int pres_shared_slots() { return PRES_SH; }
#endif

void p3_tile(int &tw, int &th)
{
    tw = TW3;
    th = TH3;
}

cudaError_t launch_sweep(const SweepLaunch &L, cudaStream_t s)
{
#if !PDD_ALT_UNIT
    if (L.path == 3 && L.g.TW == 128) return launch_sweep_wide(L, s);
    if (L.path == 3 && L.g.TH == 16) return launch_sweep_low(L, s);
#endif
    if (L.precision == 32) return L.check ? dispatch<float, true>(L, s) : dispatch<float, false>(L, s);
    return L.check ? dispatch<double, true>(L, s) : dispatch<double, false>(L, s);
}

#if PDD_CHECKED
void dev_faults(unsigned long long *out2, bool add)
{
    unsigned long long h[2], z[2] = {};
    cudaMemcpyFromSymbol(h, g_fault, sizeof h);
    cudaMemcpyToSymbol(g_fault, z, sizeof z);
    out2[0] = (add ? out2[0] : 0ull) + h[0];
    if (!add || out2[1] == 0ull) out2[1] = h[1];
}
#endif

#if PDD_TIMING
void dev_phases(unsigned long long *out8, bool add)
{
    unsigned long long h[8], z[8] = {};
    cudaMemcpyFromSymbol(h, g_phase, sizeof h);
    cudaMemcpyToSymbol(g_phase, z, sizeof z);
    for (int i = 0; i < 8; ++i) out8[i] = (add ? out8[i] : 0ull) + h[i];
}
#endif

#if PDD_WIDE_UNIT
static_assert(TW3 == 128, "the wide unit is built with PDD_P3_WIDE=1");
}  // namespace wide

cudaError_t launch_sweep_wide(const SweepLaunch &L, cudaStream_t s) { return wide::launch_sweep(L, s); }
void p3_geometry_wide(int &pitch, int &cstride, int &hmax) { wide::p3_geometry(pitch, cstride, hmax); }
void p3_tile_wide(int &tw, int &th) { wide::p3_tile(tw, th); }
#elif PDD_LOW_UNIT
static_assert(TW3 == 64 && TH3 == 16, "the low unit is built with PDD_P3_TH=16");
}  // namespace low

cudaError_t launch_sweep_low(const SweepLaunch &L, cudaStream_t s) { return low::launch_sweep(L, s); }
void p3_geometry_low(int &pitch, int &cstride, int &hmax) { low::p3_geometry(pitch, cstride, hmax); }
void p3_tile_low(int &tw, int &th) { low::p3_tile(tw, th); }
#else
// ------------------------------------------------------------------ tile bookkeeping
__global__ void k_tile_init(DProblem P, TileGeom g, const double *uhat, const int16_t *labels,
                            TileState T, double coh_thr)
{
    __shared__ int s_free;
    __shared__ unsigned long long s_min, s_max;
    __shared__ double s_sum;
    __shared__ int s_nlab;
    __shared__ double s_dx, s_dy;
    extern __shared__ unsigned s_bm[];   // bitmap of the tile's patch labels (T.n_slots bits)
    __shared__ int s_sx[2], s_sy[2];     // u_hat differences by sign (x pairs, y pairs)
    const int t = blockIdx.x;
    const int i0 = (t % g.tiles_x) * g.TW, j0 = (t / g.tiles_x) * g.TH;
    const int n = P.n;
    if (threadIdx.x == 0) {
        s_free = 0;
        s_min = 0xffffffffffffffffull;
        s_max = 0ull;
        s_sum = 0.0;
        s_nlab = 0;
        s_dx = 0.0;
        s_dy = 0.0;
        s_sx[0] = s_sx[1] = s_sy[0] = s_sy[1] = 0;
    }
    const int nwords = labels ? (T.n_slots + 31) / 32 : 0;
    for (int w = threadIdx.x; w < nwords; w += blockDim.x) s_bm[w] = 0u;
    __syncthreads();
    int cnt = 0, nlab = 0;
    double mn = INFINITY, mx = 0.0, sm = 0.0, dx = 0.0, dy = 0.0;
    int sx[2] = {0, 0}, sy[2] = {0, 0};
    for (int e = threadIdx.x; e < g.TW * g.TH; e += blockDim.x) {
        const int ly = e / g.TW, lx = e - ly * g.TW;
        const int gi = i0 + lx, gj = j0 + ly;
        if (gi >= n || gj >= n) continue;
        const int64_t k = (int64_t)gj * n + gi;
        if (P.kind[k] != 0) continue;
        ++cnt;
        if (uhat) {
            mn = fmin(mn, uhat[k]);
            mx = fmax(mx, uhat[k]);
            sm += uhat[k];
            // direction in which u_hat grows = direction information travels (values depend on
            // smaller neighbouring values): the first in-tile sweep follows it
            if (lx + 1 < g.TW && gi + 1 < n && P.kind[k + 1] == 0) {
                const double d = uhat[k + 1] - uhat[k];
                dx += d;
                sx[d < 0.0] += 1;
            }
            if (ly + 1 < g.TH && gj + 1 < n && P.kind[k + n] == 0) {
                const double d = uhat[k + n] - uhat[k];
                dy += d;
                sy[d < 0.0] += 1;
            }
        }
        if (labels) {
            // distinct labels of the tile's free nodes (patches and the orphan slot): most nodes
            // share a label already set, so look before the atomic
            const int lab = labels[k];
            if (lab >= 0 && lab < T.n_slots) {
                const unsigned bit = 1u << (lab & 31);
                if (!(((volatile unsigned *)s_bm)[lab >> 5] & bit) &&
                    !(atomicOr(&s_bm[lab >> 5], bit) & bit))
                    ++nlab;
            }
        }
    }
    // warp-level reductions first: one shared atomic per warp and quantity
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        cnt += __shfl_xor_sync(FULL, cnt, o);
        nlab += __shfl_xor_sync(FULL, nlab, o);
        mn = fmin(mn, __shfl_xor_sync(FULL, mn, o));
        mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
        sm += __shfl_xor_sync(FULL, sm, o);
        dx += __shfl_xor_sync(FULL, dx, o);
        dy += __shfl_xor_sync(FULL, dy, o);
        sx[0] += __shfl_xor_sync(FULL, sx[0], o);
        sx[1] += __shfl_xor_sync(FULL, sx[1], o);
        sy[0] += __shfl_xor_sync(FULL, sy[0], o);
        sy[1] += __shfl_xor_sync(FULL, sy[1], o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&s_free, cnt);
        if (nlab) atomicAdd(&s_nlab, nlab);
        if (uhat) {
            atomicAdd(&s_dx, dx);
            atomicAdd(&s_dy, dy);
            atomicAdd(&s_sx[0], sx[0]);
            atomicAdd(&s_sx[1], sx[1]);
            atomicAdd(&s_sy[0], sy[0]);
            atomicAdd(&s_sy[1], sy[1]);
        }
        if (mn < INFINITY) atomicMin(&s_min, (unsigned long long)__double_as_longlong(fmax(mn, 0.0)));
        if (mx > 0.0) atomicMax(&s_max, (unsigned long long)__double_as_longlong(mx));
        if (sm != 0.0) atomicAdd(&s_sum, sm);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        T.tile_free[t] = s_free;
        // admission key of the patchy front: the tile's smallest u_hat (PDD_TILE_KEY 0), or a
        // point between its smallest and its mean (1: mean, 2: midpoint of min and mean)
        double key = __longlong_as_double((long long)s_min);
        if (PDD_TILE_KEY == 1 && s_free > 0) key = s_sum / s_free;
        if (PDD_TILE_KEY == 2 && s_free > 0) key = 0.5 * (key + s_sum / s_free);
        T.tile_minu[t] = uhat ? (s_free > 0 ? key : INFINITY) : 0.0;
        T.tile_res[t] = s_free > 0 ? INFINITY : 0.0;
        T.tile_chg[t] = 0.0;
        for (int q = 0; q < 4; ++q) T.tile_edge[4 * t + q] = 0.f;
        if (labels) T.tile_lab_cnt[t] = s_nlab;
        T.tile_round[t] = -1;
        // coherent tile: (nearly) every u_hat difference has the tile's sign in x and in y, so
        // one sweep in that orientation carries information across the whole tile
        const int ox = s_dx < 0.0, oy = s_dy < 0.0;
        const int nx = s_sx[0] + s_sx[1], ny = s_sy[0] + s_sy[1];
        const bool coh = nx > 0 && ny > 0 && s_sx[ox] >= coh_thr * nx && s_sy[oy] >= coh_thr * ny;
        T.tile_orient[t] = (uint8_t)(ox | (oy << 1) | (coh ? 4 : 0));
    }
}

// exclusive scan of the per-tile label counts into the CSR offsets (one CTA; a one-off per solve)
__global__ void __launch_bounds__(1024) k_scan_offsets(const int32_t *cnt, int32_t *off, int n)
{
    __shared__ int s_part[1024];
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int b = threadIdx.x * per, e = min(n, b + per);
    int sum = 0;
    for (int i = b; i < e; ++i) sum += cnt[i];
    s_part[threadIdx.x] = sum;
    __syncthreads();
    for (int d = 1; d < (int)blockDim.x; d <<= 1) {   // Hillis-Steele inclusive scan
        const int v = threadIdx.x >= d ? s_part[threadIdx.x - d] : 0;
        __syncthreads();
        s_part[threadIdx.x] += v;
        __syncthreads();
    }
    int run = s_part[threadIdx.x] - sum;
    for (int i = b; i < e; ++i) {
        off[i] = run;
        run += cnt[i];
    }
    if (threadIdx.x == blockDim.x - 1) off[n] = s_part[threadIdx.x];
}

// fill the tile's label list from the same bitmap (labels in ascending order)
__global__ void k_tile_labels(DProblem P, TileGeom g, const int16_t *labels, TileState T)
{
    extern __shared__ unsigned s_bm[];
    const int t = blockIdx.x;
    const int i0 = (t % g.tiles_x) * g.TW, j0 = (t / g.tiles_x) * g.TH;
    const int n = P.n;
    const int nwords = (T.n_slots + 31) / 32;
    for (int w = threadIdx.x; w < nwords; w += blockDim.x) s_bm[w] = 0u;
    __syncthreads();
    for (int e = threadIdx.x; e < g.TW * g.TH; e += blockDim.x) {
        const int ly = e / g.TW, lx = e - ly * g.TW;
        const int gi = i0 + lx, gj = j0 + ly;
        if (gi >= n || gj >= n) continue;
        const int64_t k = (int64_t)gj * n + gi;
        if (P.kind[k] != 0) continue;
        const int lab = labels[k];
        if (lab >= 0 && lab < T.n_slots) {
            const unsigned bit = 1u << (lab & 31);
            if (!(((volatile unsigned *)s_bm)[lab >> 5] & bit)) atomicOr(&s_bm[lab >> 5], bit);
        }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        // lane L compacts words [L per, (L + 1) per) after the lanes before it
        const int lane = threadIdx.x, per = (nwords + 31) / 32;
        const int b = lane * per, e = min(nwords, b + per);
        int c = 0;
        for (int w = b; w < e; ++w) c += __popc(s_bm[w]);
        int incl = c;
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += v;
        }
        int pos = T.tile_lab_off[t] + incl - c;
        for (int w = b; w < e; ++w) {
            unsigned m = s_bm[w];
            while (m) {
                const int bit = __ffs(m) - 1;
                m &= m - 1;
                T.tile_lab_ids[pos++] = (int16_t)(32 * w + bit);
            }
        }
    }
}

void launch_tile_init(const DProblem &P, const TileGeom &g, const double *uhat,
                      const int16_t *labels, TileState &T, cudaStream_t s, double coh_thr)
{
    const int nt = g.tiles_x * g.tiles_y;
    const size_t bm = labels ? sizeof(unsigned) * (size_t)((T.n_slots + 31) / 32) : 0;
    k_tile_init<<<nt, 256, bm, s>>>(P, g, uhat, labels, T, coh_thr);
    if (labels) {
        k_scan_offsets<<<1, 1024, 0, s>>>(T.tile_lab_cnt, T.tile_lab_off, nt);
        k_tile_labels<<<nt, 256, bm, s>>>(P, g, labels, T);
    }
}

__global__ void k_set_values(DProblem P, int mode, const double *uhat, double *V)
{
    const int64_t N = (int64_t)P.n * P.n;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t kd = P.kind[k];
        V[k] = kd == 1 ? 0.0 : kd == 2 ? 1.0 / P.lambda : (mode == 0 ? uhat[k] : P.v0);
    }
}

void launch_set_values(const DProblem &P, int mode, const double *uhat, double *V,
                       cudaStream_t s)
{
    const int64_t N = (int64_t)P.n * P.n;
    int64_t grid = (N + 255) / 256;
    if (grid > 148 * 32) grid = 148 * 32;
    k_set_values<<<(int)grid, 256, 0, s>>>(P, mode, uhat, V);
}

__global__ void k_activate(TileGeom g, TileState T, int out_list, double tol, double tol_act,
                           double thr, int round, int n_tiles, double slack, const RoundCtl *ctl,
                           bool from_ctl)
{
    if (from_ctl) {
        if (ctl->stop) return;
        thr = ctl->thr;
        round = ctl->round;
    }
    const int sid = ctl ? ctl->sweep_id : 0;
    const double upw = ctl ? ctl->upw : -1.0;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    ActCounters *C = reinterpret_cast<ActCounters *>(T.counters);
    bool take = false;
    int fr = 0;
    // warp-aggregated max residual / min pending key (one global atomic per warp, not per tile)
    unsigned long long wres = 0ull, wpend = 0xffffffffffffffffull;
    if (t < n_tiles) {
        fr = T.tile_free[t];
        if (fr > 0) {
            const double r = T.tile_res[t];
            wres = (unsigned long long)__double_as_longlong(fmax(r, 0.0));
            bool need = r >= tol;
            if (!need) {
                const int tx = t % g.tiles_x, ty = t / g.tiles_x;
                for (int dy = -1; dy <= 1 && !need; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        const int ax = tx + dx, ay = ty + dy;
                        if ((dx | dy) == 0 || ax < 0 || ay < 0 || ax >= g.tiles_x || ay >= g.tiles_y)
                            continue;
                        const int nb = ay * g.tiles_x + ax;
                        // the change of the neighbour's side strip facing this tile (a diagonal
                        // neighbour's corner: the smaller of its two strips bounds it)
                        double cf = T.tile_chg[nb];
                        if (PDD_EDGE_ACT) {
                            const float *ed = T.tile_edge + 4 * (size_t)nb;   // W, E, S, N
                            const float ex = dx < 0 ? ed[1] : dx > 0 ? ed[0] : INFINITY;
                            const float ey = dy < 0 ? ed[3] : dy > 0 ? ed[2] : INFINITY;
                            cf = fmin(cf, (double)fminf(ex, ey));
                        }
                        if (cf >= tol_act && (!ctl || T.tile_stamp[nb] == sid) &&
                            (upw < 0.0 || T.tile_minu[nb] <= T.tile_minu[t] + upw)) {
                            need = true;
                            break;
                        }
                    }
            }
            if (need && slack >= 0.0) {
                // upstream-ready rule (patchy): wait while a neighbour whose min u_hat is lower by
                // more than `slack` (an upstream tile in the causal order) has not
                // converged yet -- the GPU form of processing the nodes in increasing u_hat
                const double mu = T.tile_minu[t];
                const int tx = t % g.tiles_x, ty = t / g.tiles_x;
                for (int dy = -1; dy <= 1 && need; ++dy)
                    for (int dx = -1; dx <= 1; ++dx) {
                        const int ax = tx + dx, ay = ty + dy;
                        if ((dx | dy) == 0 || ax < 0 || ay < 0 || ax >= g.tiles_x || ay >= g.tiles_y)
                            continue;
                        const int nb = ay * g.tiles_x + ax;
                        if (T.tile_free[nb] > 0 && T.tile_minu[nb] < mu - slack && T.tile_res[nb] >= tol) {
                            need = false;
                            break;
                        }
                    }
            }
            if (need) {
                const double mu = T.tile_minu[t];
                if (mu <= thr) {
                    take = true;
                    // activation trace: the round in which each patch last had an active tile
                    T.tile_round[t] = max(T.tile_round[t], round);
                    if (T.n_slots > 0)
                        for (int k = T.tile_lab_off[t]; k < T.tile_lab_off[t + 1]; ++k)
                            atomicMax(&T.patch_round[T.tile_lab_ids[k]], round);
                } else {
                    wpend = (unsigned long long)__double_as_longlong(fmax(mu, 0.0));
                }
            }
        }
    }
    {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            wres = max(wres, __shfl_xor_sync(FULL, wres, o));
            wpend = min(wpend, __shfl_xor_sync(FULL, wpend, o));
        }
        if ((threadIdx.x & 31) == 0) {
            if (wres) atomicMax(&C->max_res, wres);
            if (wpend != 0xffffffffffffffffull) atomicMin(&C->min_pending, wpend);
        }
    }
    // warp-aggregated append
    const unsigned m = __ballot_sync(FULL, take);
    if (m) {
        const int lane = threadIdx.x & 31;
        const int leader = __ffs(m) - 1;
        int basei = 0;
        long long fsum = 0;
        if (take) fsum = fr;
        for (int o = 16; o > 0; o >>= 1) fsum += __shfl_xor_sync(FULL, fsum, o);
        if (lane == leader) {
            basei = atomicAdd(&C->count, __popc(m));
            atomicAdd(reinterpret_cast<unsigned long long *>(&C->free_sum), (unsigned long long)fsum);
        }
        basei = __shfl_sync(FULL, basei, leader);
        if (take) T.list[out_list][basei + __popc(m & ((1u << lane) - 1u))] = t;
    }
}

void launch_activate(const TileGeom &g, TileState &T, int out_list, double tol, double tol_act,
                     double thr, int round, int n_tiles, cudaStream_t s, double slack,
                     const RoundCtl *ctl, bool from_ctl)
{
    k_activate<<<(n_tiles + 255) / 256, 256, 0, s>>>(g, T, out_list, tol, tol_act, thr, round,
                                                     n_tiles, slack, ctl, from_ctl);
}

// Order a round's active list by the tiles' min u_hat (the paper's processing order)
// so that the dynamic fetch of k_sweep_dyn visits upstream tiles first: one CTA, bitonic sort of
// (key, tile) pairs in shared memory; lists longer than SORT_MAX keep their activation order.
constexpr int SORT_MAX = 4096;
__global__ void __launch_bounds__(1024) k_sort_round(const RoundCtl *ctl, const ActCounters *c,
                                                      const double *key, int32_t *list)
{
    __shared__ float sk[SORT_MAX];
    __shared__ int32_t sv[SORT_MAX];
    if (ctl->stop) return;
    const int cnt = c->count;
    if (cnt <= 1 || cnt > SORT_MAX) return;
    int m = 1;
    while (m < cnt) m <<= 1;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        if (i < cnt) {
            const int t = list[i];
            sk[i] = (float)key[t];
            sv[i] = t;
        } else {
            sk[i] = __int_as_float(0x7f800000);
            sv[i] = -1;
        }
    }
    __syncthreads();
    for (int k = 2; k <= m; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < m; i += blockDim.x) {
                const int l = i ^ j;
                if (l > i) {
                    const bool up = (i & k) == 0;
                    const float a = sk[i], b = sk[l];
                    if ((a > b) == up) {
                        sk[i] = b; sk[l] = a;
                        const int32_t tv = sv[i]; sv[i] = sv[l]; sv[l] = tv;
                    }
                }
            }
            __syncthreads();
        }
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) list[i] = sv[i];
}

void launch_sort_round(const RoundCtl *ctl, const ActCounters *c, const double *key, int32_t *list,
                       cudaStream_t s)
{
    k_sort_round<<<1, 1024, 0, s>>>(ctl, c, key, list);
}

// ------------------------------------------------------------------ device-driven rounds
__global__ void k_round_begin(RoundCtl *ctl, ActCounters *c)
{
    if (ctl->stop) return;
    if (ctl->since_verify >= ctl->verify_every) {   // overdue verification
        ctl->stop = 1;
        return;
    }
    c->count = 0;
    c->fetch = 0;
    c->free_sum = 0;
    c->min_pending = 0xffffffffffffffffull;
    c->max_res = 0;
}

__global__ void k_round_end(RoundCtl *ctl, const ActCounters *c)
{
    if (ctl->stop) return;
    const int count = c->count;
    if (count > 0) {
        ctl->rounds += 1;
        ctl->tiles += count;
        ctl->sweep_id += 1;
        ctl->since_verify += 1;
        ctl->round += 1;
        // bucket policy 0: the front advances every round, faster while the round under-fills
        // the GPU (same latency as a full wave); policy 1: the bucket opens when it has settled
        if (ctl->delta > 0.0 && ctl->policy == 0) {
            const double fill = (double)ctl->resident / (double)count;
            ctl->thr += ctl->delta * fmin(ctl->dboost, fmax(1.0, fill));
        }
        return;
    }
    const unsigned long long pb = c->min_pending;
    const double pend = __longlong_as_double((long long)pb);
    if (pb != 0xffffffffffffffffull && isfinite(pend)) {
        ctl->thr = fmax(ctl->thr, pend) + (ctl->delta > 0.0 ? ctl->delta : 0.0);
        return;
    }
    ctl->stop = 1;        // nothing active: the host runs the full-grid verification
}

__global__ void k_round_reset(RoundCtl *ctl, double thr)
{
    ctl->stop = 0;
    ctl->thr = thr;
    ctl->since_verify = 0;
    ctl->sweep_id += 1;   // the verification supersedes every recorded tile change
    ctl->round += 1;
}

// Key order of the tiles with free nodes for the work queue (a counting sort on NB buckets of the
// min-u_hat key: admission needs the order of the front, not a total order of near-equal keys;
// key == NULL: tile index order).  rank[t] = position, INT_MAX for tiles without free nodes.
constexpr int QNB = 32768;
__global__ void k_qo_max(const TileState T, const double *key, int n_tiles, unsigned long long *kmax)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long b = 0ull;
    if (t < n_tiles && T.tile_free[t] > 0 && key && isfinite(key[t]))
        b = (unsigned long long)__double_as_longlong(fmax(key[t], 0.0));
    for (int o = 16; o > 0; o >>= 1) b = max(b, __shfl_xor_sync(FULL, b, o));
    if ((threadIdx.x & 31) == 0 && b) atomicMax(kmax, b);
}
__device__ __forceinline__ int qo_bucket(const double *key, int t, const unsigned long long *kmax)
{
    if (!key) return 0;
    const double km = __longlong_as_double((long long)*kmax);
    const double k = key[t];
    if (!(km > 0.0) || !isfinite(k)) return isfinite(k) ? 0 : QNB - 1;
    return min(QNB - 1, max(0, (int)(fmax(k, 0.0) / km * (QNB - 1))));
}
__global__ void k_qo_hist(const TileState T, const double *key, int n_tiles,
                          const unsigned long long *kmax, int32_t *hist, int32_t *rank)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tiles) return;
    rank[t] = 0x7fffffff;
    if (T.tile_free[t] > 0) atomicAdd(hist + qo_bucket(key, t, kmax), 1);
}
__global__ void k_qo_scatter(const TileState T, const double *key, int n_tiles,
                             const unsigned long long *kmax, const int32_t *off, int32_t *cursor,
                             int32_t *order, int32_t *rank)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tiles || T.tile_free[t] <= 0) return;
    const int b = qo_bucket(key, t, kmax);
    const int pos = off[b] + atomicAdd(cursor + b, 1);
    order[pos] = t;
    rank[t] = pos;
}

void launch_queue_order(const TileState &T, const double *key, int n_tiles, int32_t *scratch,
                        int32_t *order, int32_t *rank, cudaStream_t s)
{
    // scratch: QNB hist + (QNB + 1) offsets + QNB cursors + 2 (kmax)
    int32_t *hist = scratch, *off = scratch + QNB, *cur = off + QNB + 1;
    unsigned long long *kmax = reinterpret_cast<unsigned long long *>(cur + QNB + 1);
    cudaMemsetAsync(hist, 0, sizeof(int32_t) * QNB, s);
    cudaMemsetAsync(cur, 0, sizeof(int32_t) * QNB, s);
    cudaMemsetAsync(kmax, 0, sizeof(unsigned long long), s);
    const int g = (n_tiles + 255) / 256;
    k_qo_max<<<g, 256, 0, s>>>(T, key, n_tiles, kmax);
    k_qo_hist<<<g, 256, 0, s>>>(T, key, n_tiles, kmax, hist, rank);
    k_scan_offsets<<<1, 1024, 0, s>>>(hist, off, QNB);
    k_qo_scatter<<<g, 256, 0, s>>>(T, key, n_tiles, kmax, off, cur, order, rank);
}
size_t queue_order_scratch_ints() { return 3 * (size_t)QNB + 1 + 4; }

// (re-)seed the work queue (ring zeroed, cursors at 0): first > 0 takes the first `first` tiles of
// the key order (start of a patchy solve), else every tile among the first `adm` of the order
// whose residual is >= tol (static start, or the offending tiles of a verification pass);
// warp-aggregated reservations
__global__ void k_queue_seed(TileState T, QueueArgs Q, int n_tiles, double tol, int first, int adm)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    int t = -1;
    if (first > 0) {
        if (i < first && i < Q.n_order) t = Q.order[i];
    } else if (i < n_tiles && T.tile_free[i] > 0 && T.tile_res[i] >= tol && Q.rank[i] < adm) {
        t = i;   // admitted tiles only: the others enter in key order
    }
    const bool take = t >= 0;
    const unsigned m = __ballot_sync(FULL, take);
    if (!m) return;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    unsigned long long pos = 0;
    if (lane == leader) {
        atomicAdd(&Q.ctl->work, __popc(m));
        if (first > 0) atomicAdd(&Q.ctl->adm, __popc(m));
        pos = atomicAdd(&Q.ctl->tail, (unsigned long long)__popc(m));
    }
    pos = __shfl_sync(FULL, pos, leader);
    if (take) {
        Q.state[t] = 1;
        Q.ring[(pos + __popc(m & ((1u << lane) - 1u))) & (unsigned long long)(Q.cap - 1)] = t + 1;
    }
}

void launch_queue_seed(const TileState &T, const QueueArgs &Q, int n_tiles, double tol, int first,
                       int adm, cudaStream_t s)
{
    const int m = first > 0 ? first : n_tiles;
    k_queue_seed<<<(m + 255) / 256, 256, 0, s>>>(T, Q, n_tiles, tol, first, adm);
}

// per-patch activation trace of the work-queue schedule: the last visit of any tile holding nodes
// of the patch (the tile label CSR of k_tile_labels)
__global__ void k_patch_rounds(const int32_t *tile_round, const int32_t *lab_off, const int16_t *lab_ids,
                               int32_t *patch_round, int n_tiles)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tiles || tile_round[t] < 0) return;
    for (int k = lab_off[t]; k < lab_off[t + 1]; ++k) atomicMax(&patch_round[lab_ids[k]], tile_round[t]);
}

__global__ void k_verify_list(TileGeom g, TileState T, int mark, int n_tiles)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    ActCounters *C = reinterpret_cast<ActCounters *>(T.counters);
    bool take = false;
    if (t < n_tiles && T.tile_free[t] > 0) {
        const int tx = t % g.tiles_x, ty = t / g.tiles_x;
        for (int dy = -1; dy <= 1 && !take; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const int ax = tx + dx, ay = ty + dy;
                if (ax < 0 || ay < 0 || ax >= g.tiles_x || ay >= g.tiles_y) continue;
                if (T.tile_round[ay * g.tiles_x + ax] > mark) { take = true; break; }
            }
    }
    const unsigned m = __ballot_sync(FULL, take);
    if (!m) return;
    const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
    int basei = 0;
    if (lane == leader) basei = atomicAdd(&C->count, __popc(m));
    basei = __shfl_sync(FULL, basei, leader);
    if (take) T.list[0][basei + __popc(m & ((1u << lane) - 1u))] = t;
}

void launch_verify_list(const TileGeom &g, const TileState &T, int mark, int n_tiles, cudaStream_t s)
{
    cudaMemsetAsync(T.counters, 0, sizeof(ActCounters), s);
    k_verify_list<<<(n_tiles + 255) / 256, 256, 0, s>>>(g, T, mark, n_tiles);
}

__global__ void k_patch_res_reduce(TileState T, int n_tiles)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tiles) return;
    for (int k = T.tile_lab_off[t]; k < T.tile_lab_off[t + 1]; ++k) {
        const unsigned long long v = T.tile_lab_res[k];
        if (v) atomicMax(T.patch_res + T.tile_lab_ids[k], v);
    }
}

void launch_patch_res_reduce(const TileState &T, int n_tiles, cudaStream_t s)
{
    cudaMemsetAsync(T.patch_res, 0, sizeof(unsigned long long) * T.n_slots, s);
    k_patch_res_reduce<<<(n_tiles + 255) / 256, 256, 0, s>>>(T, n_tiles);
}

void launch_patch_rounds(const TileState &T, int n_tiles, cudaStream_t s)
{
    k_patch_rounds<<<(n_tiles + 255) / 256, 256, 0, s>>>(T.tile_round, T.tile_lab_off, T.tile_lab_ids,
                                                         T.patch_round, n_tiles);
}

void launch_round_begin(RoundCtl *ctl, ActCounters *c, cudaStream_t s) { k_round_begin<<<1, 1, 0, s>>>(ctl, c); }
void launch_round_end(RoundCtl *ctl, const ActCounters *c, cudaStream_t s) { k_round_end<<<1, 1, 0, s>>>(ctl, c); }
void launch_round_reset(RoundCtl *ctl, double thr, cudaStream_t s) { k_round_reset<<<1, 1, 0, s>>>(ctl, thr); }

}  // namespace pdd

namespace pdd {

// ------------------------------------------------------------------ row-table construction
// One thread per (row j, control a): the 2p foot points of an interior node of row j, relative to
// the node (x not clamped: nodes within H of the x-boundary use the general stencil; y clamped
// to the box as the row dictates, R5), in fp64.  k_rowtab_extent finds the smallest window
// (WY x WX) holding every control's non-self corners; k_rowtab_fill writes the branch-merged
// compact stencil W = beta w lambda / (1 - beta Lambda0), E = 1/(1 - beta Lambda0).
__device__ __forceinline__ void rt_feet(const DProblem &P, int j, int a, int b, double &xr,
                                        double &yr)
{
    const int n = P.n;
    const double c = coef_at(P.speed, 0, j, n);
    const double d1 = coef_at(P.drift[0], 0, j, n);
    const double d2 = coef_at(P.drift[1], 0, j, n);
    xr = P.q * (c * P.ctrl[2 * a] + d1);
    yr = P.q * (c * P.ctrl[2 * a + 1] + d2);
    if (P.p > 0) {
        const int kk = b >> 1;
        double ox = P.sc * coef_at(P.sigma[kk][0], 0, j, n);
        double oy = P.sc * coef_at(P.sigma[kk][1], 0, j, n);
        if (P.sigma_mode == 1) {            // sigma(x, a) = s(x) a (R32)
            const double sa = P.sc * coef_at(P.sigma[0][0], 0, j, n);
            ox = sa * P.ctrl[2 * a];
            oy = sa * P.ctrl[2 * a + 1];
        }
        if (b & 1) { xr -= ox; yr -= oy; } else { xr += ox; yr += oy; }
    }
    yr = fmin(fmax(yr, (double)-j), (double)(n - 1 - j));
}

__global__ void k_rowtab_extent(DProblem P, int *ext)
{
    const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (id >= (int64_t)P.n * P.na) return;
    const int j = (int)(id / P.na), a = (int)(id % P.na);
    const int nb = P.p > 0 ? 2 * P.p : 1;
    int ymin = 1 << 30, ymax = -(1 << 30), xmin = 1 << 30, xmax = -(1 << 30);
    for (int b = 0; b < nb; ++b) {
        double xr, yr;
        rt_feet(P, j, a, b, xr, yr);
        const int fx = (int)floor(xr);
        const int fy = (int)fmin(floor(yr), (double)(P.n - 2 - j));
        xmin = min(xmin, fx); xmax = max(xmax, fx + 1);
        ymin = min(ymin, fy); ymax = max(ymax, fy + 1);
    }
    atomicMax(&ext[0], ymax - ymin + 1);
    atomicMax(&ext[1], xmax - xmin + 1);
}

template <typename real, int WY, int WX>
__global__ void k_rowtab_fill(DProblem P, int napad, int H, RowEntry<real, WY, WX> *tab, int *oxr)
{
    const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (id >= (int64_t)P.n * napad) return;
    const int j = (int)(id / napad), a = (int)(id % napad);
    RowEntry<real, WY, WX> e;
    e.oy = 0; e.ox = 0; e.E = 0;
#pragma unroll
    for (int m = 0; m < WY * WX; ++m) e.W[m] = 0;
    if (a < P.na) {
        const int nb = P.p > 0 ? 2 * P.p : 1;
        const double w = 1.0 / nb;
        int cdy[8 * 4], cdx[8 * 4];
        double cw[8 * 4];
        int ncn = 0, ymin = 1 << 30, xmin = 1 << 30;
        double lam0 = 0.0;
        for (int b = 0; b < nb; ++b) {
            double xr, yr;
            rt_feet(P, j, a, b, xr, yr);
            const double fx = floor(xr);
            const double fy = fmin(floor(yr), (double)(P.n - 2 - j));
            const double tx = xr - fx, ty = yr - fy;
            const double ww[4] = {(1 - tx) * (1 - ty), tx * (1 - ty), (1 - tx) * ty, tx * ty};
            for (int t = 0; t < 4; ++t) {
                const int dx = (int)fx + (t & 1), dy = (int)fy + (t >> 1);
                if (dx == 0 && dy == 0) { lam0 += w * ww[t]; continue; }
                cdy[ncn] = dy; cdx[ncn] = dx; cw[ncn] = w * ww[t]; ++ncn;
                ymin = min(ymin, dy); xmin = min(xmin, dx);
            }
        }
        int oy = max(min(ymin, H - (WY - 1)), -H);
        int ox = max(min(xmin, H - (WX - 1)), -H);
        const double Ek = 1.0 / (1.0 - P.beta * lam0);
        double acc[WY * WX];
#pragma unroll
        for (int m = 0; m < WY * WX; ++m) acc[m] = 0.0;
        for (int t = 0; t < ncn; ++t) {
            const int r = cdy[t] - oy, x = cdx[t] - ox;
            if (r >= 0 && r < WY && x >= 0 && x < WX) acc[r * WX + x] += cw[t];
        }
        e.oy = oy; e.ox = ox; e.E = (real)Ek;
#pragma unroll
        for (int m = 0; m < WY * WX; ++m) e.W[m] = (real)(P.beta * acc[m] * Ek);
        atomicMin(&oxr[0], ox);
        atomicMax(&oxr[1], ox);
    }
    tab[id] = e;
}

bool rowtab_build_device(const DProblem &P, int napad, int H, int precision, int *scratch,
                         void *tab, size_t tab_bytes, int &WY, int &WX, int &oxmin, int &oxmax,
                         cudaStream_t s)
{
    int h[4] = {0, 0, 1 << 30, -(1 << 30)};
    if (cudaMemcpyAsync(scratch, h, sizeof h, cudaMemcpyHostToDevice, s) != cudaSuccess) return false;
    const int64_t m = (int64_t)P.n * P.na;
    k_rowtab_extent<<<(unsigned)((m + 255) / 256), 256, 0, s>>>(P, scratch);
    if (cudaMemcpyAsync(h, scratch, 2 * sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess) return false;
    if (cudaStreamSynchronize(s) != cudaSuccess) return false;
    const int cand[3][2] = {{3, 3}, {2, 5}, {4, 4}};
    WY = WX = 0;
    for (auto &cw : cand)
        if (h[0] <= cw[0] && h[1] <= cw[1]) { WY = cw[0]; WX = cw[1]; break; }
    if (!WY) return false;
    const int64_t mt = (int64_t)P.n * napad;
    if ((size_t)mt * rowtab_entry_bytes(precision, WY, WX) > tab_bytes) return false;
    const unsigned grid = (unsigned)((mt + 127) / 128);
#define PDD_RTF(WY_, WX_)                                                                        \
    if (WY == WY_ && WX == WX_) {                                                                \
        if (precision == 32)                                                                     \
            k_rowtab_fill<float, WY_, WX_><<<grid, 128, 0, s>>>(                                 \
                P, napad, H, reinterpret_cast<RowEntry<float, WY_, WX_> *>(tab), scratch + 2);   \
        else                                                                                     \
            k_rowtab_fill<double, WY_, WX_><<<grid, 128, 0, s>>>(                                \
                P, napad, H, reinterpret_cast<RowEntry<double, WY_, WX_> *>(tab), scratch + 2);  \
    }
    PDD_RTF(3, 3)
    PDD_RTF(2, 5)
    PDD_RTF(4, 4)
#undef PDD_RTF
    if (cudaMemcpyAsync(h + 2, scratch + 2, 2 * sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess)
        return false;
    if (cudaStreamSynchronize(s) != cudaSuccess) return false;
    oxmin = h[2];
    oxmax = h[3];
    return true;
}

#endif  // !PDD_ALT_UNIT

}  // namespace pdd

#if PDD_CHECKED && !PDD_ALT_UNIT
// negative control of the checked build: one deliberately failing check (code 99) must be counted
namespace pdd {
__global__ void k_fault_selftest(const float *p)
{
    __shared__ float buf[32];
    if (threadIdx.x == 0) {
        chk_bounds().lo = (const char *)buf;
        chk_bounds().hi = (const char *)(buf + 32);
    }
    __syncthreads();
    PDD_CHK_TILE(buf + threadIdx.x, 1, 98);          // inside: must not count
    if (threadIdx.x == 0) PDD_CHK_TILE(buf + 32, 1, 99);   // one past the end: must count
    (void)p;
}
}  // namespace pdd
extern "C" void pdd_dev_fault_selftest()
{
    pdd::k_fault_selftest<<<1, 32>>>(nullptr);
    cudaDeviceSynchronize();
}
namespace pdd { namespace wide { void dev_faults(unsigned long long *out2, bool add); } }
namespace pdd { namespace low { void dev_faults(unsigned long long *out2, bool add); } }
// checked builds only: bounds violations counted by the sweep kernels since the last call
extern "C" void pdd_dev_faults(unsigned long long *out2)
{
    cudaDeviceSynchronize();
    pdd::dev_faults(out2, false);
    pdd::wide::dev_faults(out2, true);
    pdd::low::dev_faults(out2, true);
}
#endif

#if PDD_TIMING && !PDD_ALT_UNIT
namespace pdd { namespace wide { void dev_phases(unsigned long long *out8, bool add); } }
namespace pdd { namespace low { void dev_phases(unsigned long long *out8, bool add); } }
// development builds only: cycles per visit phase summed over all CTAs since the last call
extern "C" void pdd_dev_phases(unsigned long long *out8)
{
    cudaDeviceSynchronize();
    pdd::dev_phases(out8, false);
    pdd::wide::dev_phases(out8, true);
    pdd::low::dev_phases(out8, true);
}
#endif
