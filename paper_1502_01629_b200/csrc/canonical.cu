// canonical.cu -- the decision stages of the pre-computation on sm_100a.
//
// Their integer outputs (a*, labels) must be bit-exact with any IEEE-754 evaluation of the same
// expressions, so this translation unit is compiled with --fmad=false and every fp64 operation
// is written with an explicit round-to-nearest intrinsic in the order fixed by DESIGN.md
// reading R30 ("canonical arithmetic"):
//   f = c a + d;  b = q f;  g = i + b;  clamp g to [0, n-1];  cell = min(floor g, n-2);
//   t = g - cell;  w00 = (1-tx)(1-ty), w10 = tx(1-ty), w01 = (1-tx)ty, w11 = tx ty;
//   sums in corner order 00, 10, 01, 11.
//
// Kernels (one thread per node unless noted):
//   k_init_values   V0 on free nodes, Dirichlet values (R8, R11)
//   k_coarse_sweep  one Jacobi sweep of the sigma = 0 scheme on G_c (SLscheme3
//                   P:473-491 with discount R3) + sup-norm residual; stops itself once the
//                   previous sweep's residual is < tol (so the result does not depend on how
//                   many sweeps the host enqueues)
//                   (k_coarse_sweep_tiles: the same sweep on the 16 x 16 tiles whose neighbourhood
//                   changed, tile + halo and the row-invariant table staged in shared memory; interior
//                   tiles take canon_node_update_fast -- all bit-identical rewrites, see there)
//   k_prolong       u_hat = bilinear(u_c) (R15)
//   k_synthesize    a* = argmin_k [h l + beta u_hat(x + h f)] (R16)
//                   (k_synthesize_rt_s: strips of 16 x 16 tiles with u_hat and the table staged)
//   k_successor     nearest node to x + M f*/|f*| (R18)
//   k_jump          pointer jumping s <- s[s]
//   k_labels        label = sector[root] for target roots, orphan otherwise (R17)
//   k_static_labels equal squares (R19)
#include "pdd_internal.cuh"

#include <math.h>

namespace pdd {

#define DADD(a, b) __dadd_rn((a), (b))
#define DSUB(a, b) __dsub_rn((a), (b))
#define DMUL(a, b) __dmul_rn((a), (b))
#define DDIV(a, b) __ddiv_rn((a), (b))

// bilinear stencil at (gx, gy) in node units (clamped), corners 00, 10, 01, 11
__device__ __forceinline__ void canon_stencil(int n, double gx, double gy, int64_t cr[4],
                                              double wg[4])
{
    const double top = (double)(n - 1);
    if (gx < 0.0) gx = 0.0;
    if (gx > top) gx = top;
    if (gy < 0.0) gy = 0.0;
    if (gy > top) gy = top;
    int cx = (int)floor(gx), cy = (int)floor(gy);
    if (cx > n - 2) cx = n - 2;
    if (cy > n - 2) cy = n - 2;
    const double tx = DSUB(gx, (double)cx);
    const double ty = DSUB(gy, (double)cy);
    const double ux = DSUB(1.0, tx), uy = DSUB(1.0, ty);
    wg[0] = DMUL(ux, uy);
    wg[1] = DMUL(tx, uy);
    wg[2] = DMUL(ux, ty);
    wg[3] = DMUL(tx, ty);
    cr[0] = (int64_t)cy * n + cx;
    cr[1] = cr[0] + 1;
    cr[2] = cr[0] + n;
    cr[3] = cr[0] + n + 1;
}

__global__ void k_init_values(DProblem P, double *V)
{
    const int64_t N = (int64_t)P.n * P.n;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t kd = P.kind[k];
        V[k] = kd == 0 ? P.v0 : (kd == 1 ? 0.0 : DDIV(1.0, P.lambda));
    }
}

// Exact minimum over controls of the IEEE quotients num_a / den_a (num > 0, den > 0) with few
// fp64 divisions: an fp32 estimate (relative error < 1e-6) of each quotient selects the controls
// whose quotient can still be the minimum (within a 1e-5 window of the running estimate); only
// those get the IEEE division.  Rounding is monotone, so min_a rn(num_a / den_a) = rn(q*) for the
// exact minimiser a*, which is always among the candidates: the result is bit-identical to
// dividing for every control.  Up to EXK candidates are kept; beyond that they are divided at once.
#ifndef PDD_COARSE_SMEM
#define PDD_COARSE_SMEM 1   // tiled coarse sweep: V tile + halo staged in shared memory
#endif
#ifndef PDD_COARSE_RTSMEM
#define PDD_COARSE_RTSMEM 1   // ... and the tile's rows of the row-invariant table
#endif
#ifndef PDD_CANON_UNROLL
#define PDD_CANON_UNROLL 2   // controls per loop trip in the staged coarse / synthesis kernels (A/B: profiles/r4_canon_ab.txt)
#endif
#ifndef PDD_CANON_MINB
#define PDD_CANON_MINB 4     // __launch_bounds__ min blocks per SM of those kernels (A/B)
#endif
#define PDD_PRAGMA_(x) _Pragma(#x)
#define PDD_UNROLL_(n) PDD_PRAGMA_(unroll n)
#ifndef PDD_EXACT_MIN
#define PDD_EXACT_MIN 0   // measured slower on sm_100a (C5 coarse 31 vs 24 ms): kept as an option
#endif
// tile geometry of the staged coarse sweep and synthesis: CT x CT nodes per CTA, halo of CH cells
constexpr int CT = 16;
constexpr int CH = 4;
constexpr int CSW = CT + 2 * CH;   // staged row width
constexpr int EXK = 4;
struct ExactMin {
    float mt = INFINITY;                     // running estimate of the minimum
    double cn[EXK], cd[EXK];
    int cnt = 0;
    double vex = INFINITY;                   // exact min of the candidates beyond EXK
    __device__ __forceinline__ void add(double num, double den)
    {
        const float q = __fdividef((float)num, (float)den);
        if (q < mt * (1.0f - 1e-5f)) {            // clearly below every candidate so far
            cnt = 0;
            vex = INFINITY;
        } else if (q > mt * (1.0f + 1e-5f)) {
            return;                               // cannot be the minimum
        }
        mt = fminf(mt, q);
        if (cnt < EXK) {
            cn[cnt] = num;
            cd[cnt] = den;
            ++cnt;
        } else {
            vex = fmin(vex, DDIV(num, den));
        }
    }
    __device__ __forceinline__ double result() const
    {
        double b = vex;
#pragma unroll
        for (int k = 0; k < EXK; ++k)
            if (k < cnt) b = fmin(b, DDIV(cn[k], cd[k]));
        return b;
    }
};

// sigma = 0 node update of the modified scheme (one foot point, w = 1)
__device__ double canon_node_update(const DProblem &P, const double *V, int i, int j)
{
    const int n = P.n;
    const int64_t self = (int64_t)j * n + i;
    const double c = coef_at(P.speed, i, j, n);
    const double d1 = coef_at(P.drift[0], i, j, n);
    const double d2 = coef_at(P.drift[1], i, j, n);
    const double l = coef_at(P.cost, i, j, n);
    double best = INFINITY;
    for (int a = 0; a < P.na; ++a) {
        const double hl = DMUL(P.h, P.cost_ctrl ? DADD(l, P.cost_ctrl[a]) : l);   // R33
        const double f1 = DADD(DMUL(c, P.ctrl[2 * a]), d1);
        const double f2 = DADD(DMUL(c, P.ctrl[2 * a + 1]), d2);
        const double gx = DADD((double)i, DMUL(P.q, f1));
        const double gy = DADD((double)j, DMUL(P.q, f2));
        int64_t cr[4];
        double wg[4];
        canon_stencil(n, gx, gy, cr, wg);
        double lam0 = 0.0, rp = 0.0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            if (cr[t] == self) lam0 = DADD(lam0, wg[t]);
            else rp = DADD(rp, DMUL(wg[t], V[cr[t]]));
        }
        const double v = DDIV(DADD(hl, DMUL(P.beta, rp)), DSUB(1.0, DMUL(P.beta, lam0)));
        if (v < best) best = v;
    }
    return best;
}

// Row-invariant part of the coarse update when every coefficient depends on x2 only (C2, C4, C5):
// per (row j, control a) the x offset q f1, the clamped y cell / fraction and h l(x, a), computed
// with exactly the operations (and order) of canon_node_update -- the table only hoists them out
// of the node loop, so the sweep stays bit-identical.
__global__ void k_coarse_rowtab(DProblem P, CoarseRowEntry *tab)
{
    const int64_t id = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (id >= (int64_t)P.n * P.na) return;
    const int n = P.n;
    const int j = (int)(id / P.na), a = (int)(id % P.na);
    const double c = coef_at(P.speed, 0, j, n);
    const double f1 = DADD(DMUL(c, P.ctrl[2 * a]), coef_at(P.drift[0], 0, j, n));
    const double f2 = DADD(DMUL(c, P.ctrl[2 * a + 1]), coef_at(P.drift[1], 0, j, n));
    CoarseRowEntry e;
    e.bxq = DMUL(P.q, f1);
    double gy = DADD((double)j, DMUL(P.q, f2));
    const double top = (double)(n - 1);
    if (gy < 0.0) gy = 0.0;
    if (gy > top) gy = top;
    int cy = (int)floor(gy);
    if (cy > n - 2) cy = n - 2;
    e.ty = DSUB(gy, (double)cy);
    e.uy = DSUB(1.0, e.ty);
    const double l = coef_at(P.cost, 0, j, n);
    e.hl = DMUL(P.h, P.cost_ctrl ? DADD(l, P.cost_ctrl[a]) : l);
    e.cy = cy;
    // interior fast path (canon_ctrl_fast): x cell relative to the node, corner that is the node
    const double fb = floor(e.bxq);
    e.fbd = fb;
    const int fbi = fb < -1000.0 ? -1000 : (fb > 1000.0 ? 1000 : (int)fb);
    const int sx = fbi == 0 ? 0 : (fbi == -1 ? 1 : -1);         // corner column that holds x = i
    const int sy = cy == j ? 0 : (cy + 1 == j ? 1 : -1);        // corner row that holds y = j
    const int sc = (sx >= 0 && sy >= 0) ? 2 * sy + sx : -1;
    e.pk = (((cy - j) * CSW + fbi + 32768) & 0xffff) | (sc >= 0 ? (0x10000 << sc) : 0);
    tab[id] = e;
}

// canon_node_update with the row-invariant table (same operations on every node)
__device__ double canon_node_update_rt(const DProblem &P, const double *V, int i, int j,
                                       const CoarseRowEntry *__restrict__ row)
{
    const int n = P.n;
    const int64_t self = (int64_t)j * n + i;
    const double top = (double)(n - 1);
    double best = INFINITY;
    ExactMin em;
    for (int a = 0; a < P.na; ++a) {
        const CoarseRowEntry e = row[a];
        double gx = DADD((double)i, e.bxq);
        if (gx < 0.0) gx = 0.0;
        if (gx > top) gx = top;
        int cx = (int)floor(gx);
        if (cx > n - 2) cx = n - 2;
        const double tx = DSUB(gx, (double)cx);
        const double ux = DSUB(1.0, tx);
        const double wg[4] = {DMUL(ux, e.uy), DMUL(tx, e.uy), DMUL(ux, e.ty), DMUL(tx, e.ty)};
        const int64_t c0 = (int64_t)e.cy * n + cx;
        const int64_t cr[4] = {c0, c0 + 1, c0 + n, c0 + n + 1};
        double lam0 = 0.0, rp = 0.0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            if (cr[t] == self) lam0 = DADD(lam0, wg[t]);
            else rp = DADD(rp, DMUL(wg[t], V[cr[t]]));
        }
        if (PDD_EXACT_MIN) {
            em.add(DADD(e.hl, DMUL(P.beta, rp)), DSUB(1.0, DMUL(P.beta, lam0)));
        } else {
            const double v = DDIV(DADD(e.hl, DMUL(P.beta, rp)), DSUB(1.0, DMUL(P.beta, lam0)));
            if (v < best) best = v;
        }
    }
    return PDD_EXACT_MIN ? em.result() : best;
}

// The same update reading V from a shared-memory copy of the tile + halo (CH cells): the 4 x N_A
// corner gathers per node hit shared memory instead of L1/L2 (the coarse sweep stalled on them:
// long scoreboard 3.4 per issue).  Same values, same operations: bit-identical.
__device__ double canon_node_update_rt_s(const DProblem &P, const double *__restrict__ sV, int i,
                                         int j, int ib, int jb, const CoarseRowEntry *__restrict__ row)
{
    const int n = P.n;
    const double top = (double)(n - 1);
    double best = INFINITY;
    PDD_UNROLL_(PDD_CANON_UNROLL)
    for (int a = 0; a < P.na; ++a) {
        const CoarseRowEntry e = row[a];
        double gx = DADD((double)i, e.bxq);
        if (gx < 0.0) gx = 0.0;
        if (gx > top) gx = top;
        int cx = (int)floor(gx);
        if (cx > n - 2) cx = n - 2;
        const double tx = DSUB(gx, (double)cx);
        const double ux = DSUB(1.0, tx);
        const double wg[4] = {DMUL(ux, e.uy), DMUL(tx, e.uy), DMUL(ux, e.ty), DMUL(tx, e.ty)};
        const int s0 = (e.cy - jb) * CSW + (cx - ib);
        const int sr[4] = {s0, s0 + 1, s0 + CSW, s0 + CSW + 1};
        const bool self[4] = {cx == i && e.cy == j, cx + 1 == i && e.cy == j,
                              cx == i && e.cy + 1 == j, cx + 1 == i && e.cy + 1 == j};
        double lam0 = 0.0, rp = 0.0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            if (self[t]) lam0 = DADD(lam0, wg[t]);
            else rp = DADD(rp, DMUL(wg[t], sV[sr[t]]));
        }
        const double v = DDIV(DADD(e.hl, DMUL(P.beta, rp)), DSUB(1.0, DMUL(P.beta, lam0)));
        if (v < best) best = v;
    }
    return best;
}

// ---- interior fast path of the staged coarse sweep and synthesis (bit-identical) ----------------
// In a tile none of whose feet is clamped in x (columns in [CH, n-1-CH]; the y clamps are already
// in the table) the per-control work of canon_node_update_rt_s shrinks without changing a bit:
//  * cell: g = rn(i + q f1) lies in [i + fb, i + fb + 1] for fb = floor(q f1) (both ends are
//    representable and rounding is monotone), so floor(g) = i + fb unless g == i + fb + 1; then
//    t = g - (i + fb) == 1 and that control is evaluated by the generic code (canon_ctrl_generic).
//    i + fb is formed by an exact fp64 addition: no float <-> int conversion, no clamps.
//  * the offset of corner 00 in the staged tile and the corner that is the node itself depend on
//    (row, control) only and come from the table (CoarseRowEntry::pk).
//  * the sum over the non-self corners keeps the corner order 00, 10, 01, 11; its first term is not
//    added to 0.0 (0.0 + x == x for every x but -0.0, and the products w V are >= +0.0), lam0 is the
//    self corner's weight (0.0 + w == w).
//  * the minimum of the IEEE quotients num_a / den_a (den_a = 1 - beta lam0 > 0 for beta < 1) is the
//    quotient of the exact minimiser, because rounding is monotone; the minimiser is found without
//    dividing: num_a / den_a < num_b / den_b  <=>  num_a den_b < num_b den_a, decided by the rounded
//    products when they differ (monotone rounding again) and by the exact FMA residuals when they are
//    equal.  One IEEE division of the minimiser at the end: the bits of min_a rn(num_a / den_a).
#ifndef PDD_CANON_FAST
#define PDD_CANON_FAST 1
#endif

// one control in the generic form: numerator and denominator of its quotient (same operations as
// canon_node_update_rt_s)
__device__ __noinline__ double2 canon_ctrl_generic(int n, double beta, const double *sV, int i, int j,
                                                   int ib, int jb, double bxq, double ty, double uy,
                                                   double hl, int cy)
{
    const double top = (double)(n - 1);
    double gx = DADD((double)i, bxq);
    if (gx < 0.0) gx = 0.0;
    if (gx > top) gx = top;
    int cx = (int)floor(gx);
    if (cx > n - 2) cx = n - 2;
    const double tx = DSUB(gx, (double)cx);
    const double ux = DSUB(1.0, tx);
    const double wg[4] = {DMUL(ux, uy), DMUL(tx, uy), DMUL(ux, ty), DMUL(tx, ty)};
    const int s0 = (cy - jb) * CSW + (cx - ib);
    const int sr[4] = {s0, s0 + 1, s0 + CSW, s0 + CSW + 1};
    const bool self[4] = {cx == i && cy == j, cx + 1 == i && cy == j, cx == i && cy + 1 == j,
                          cx + 1 == i && cy + 1 == j};
    double lam0 = 0.0, rp = 0.0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        if (self[t]) lam0 = DADD(lam0, wg[t]);
        else rp = DADD(rp, DMUL(wg[t], sV[sr[t]]));
    }
    return make_double2(DADD(hl, DMUL(beta, rp)), DSUB(1.0, DMUL(beta, lam0)));
}

__device__ __forceinline__ double canon_node_update_fast(const DProblem &P, const double *__restrict__ sV,
                                                         int i, int j, int ib, int jb,
                                                         const CoarseRowEntry *__restrict__ row)
{
    const double id = (double)i;
    const double beta = P.beta;
    const int sself = (j - jb) * CSW + (i - ib) - 32768;
    double nb = INFINITY, db = 1.0;          // the best quotient so far as numerator / denominator
    PDD_UNROLL_(PDD_CANON_UNROLL)
    for (int a = 0; a < P.na; ++a) {
        const double bxq = row[a].bxq, fbd = row[a].fbd;
        const double gx = DADD(id, bxq);
        const double tx = DSUB(gx, DADD(id, fbd));
        double num, den;
        if (__double2hiint(tx) >= 0x3ff00000) {          // t == 1: the rounded foot is the next integer
            const double2 nd = canon_ctrl_generic(P.n, beta, sV, i, j, ib, jb, bxq, row[a].ty, row[a].uy,
                                                  row[a].hl, row[a].cy);
            num = nd.x;
            den = nd.y;
        } else {
            const double ty = row[a].ty, uy = row[a].uy;
            const int pk = row[a].pk;
            const int s0 = sself + (pk & 0xffff);
            const double ux = DSUB(1.0, tx);
            const double w0 = DMUL(ux, uy), w1 = DMUL(tx, uy), w2 = DMUL(ux, ty), w3 = DMUL(tx, ty);
            // the corner that is the node itself (one-hot in bits 16..19 of pk, none: 0) contributes
            // +0.0 in its place of the corner-order sum: x + 0.0 == x
            const double p0 = (pk & 0x10000) ? 0.0 : DMUL(w0, sV[s0]);
            const double p1 = (pk & 0x20000) ? 0.0 : DMUL(w1, sV[s0 + 1]);
            const double p2 = (pk & 0x40000) ? 0.0 : DMUL(w2, sV[s0 + CSW]);
            const double p3 = (pk & 0x80000) ? 0.0 : DMUL(w3, sV[s0 + CSW + 1]);
            const bool has = pk & 0xf0000, bx = pk & 0xa0000, by = pk & 0xc0000;
            const double rp = DADD(DADD(DADD(p0, p1), p2), p3);
            const double lam0 = DMUL(bx ? tx : ux, by ? ty : uy);     // the self corner's weight
            num = DADD(row[a].hl, DMUL(beta, rp));
            den = has ? DSUB(1.0, DMUL(beta, lam0)) : 1.0;            // 1 - beta 0 == 1
        }
        const double c1 = DMUL(num, db), c2 = DMUL(nb, den);
        bool take = c1 < c2;
        if (c1 == c2) take = __fma_rn(num, db, -c1) < __fma_rn(nb, den, -c2);
        if (take) {
            nb = num;
            db = den;
        }
    }
    return DDIV(nb, db);
}

__global__ void k_coarse_sweep(DProblem P, const double *__restrict__ Vin, double *__restrict__ Vout,
                               double tol, unsigned long long *res_hist, int sweep,
                               int *sweeps_done)
{
    // stop once the previous sweep has converged: Vout keeps nothing new, the converged
    // iterate stays in the buffer written by sweep (sweeps_done - 1)
    if (sweep > 0 && __longlong_as_double((long long)res_hist[sweep - 1]) < tol) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(sweeps_done, 1);
    const int n = P.n;
    const int64_t N = (int64_t)n * n;
    double res = 0.0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        if (P.kind[k] != 0) { Vout[k] = Vin[k]; continue; }
        const double v = canon_node_update(P, Vin, (int)(k % n), (int)(k / n));
        Vout[k] = v;
        const double d = fabs(DSUB(v, Vin[k]));
        if (d > res) res = d;
    }
    // non-negative doubles order like their bit patterns
    for (int o = 16; o > 0; o >>= 1) res = fmax(res, __shfl_xor_sync(0xffffffffu, res, o));
    if ((threadIdx.x & 31) == 0 && res > 0.0)
        atomicMax(&res_hist[sweep], (unsigned long long)__double_as_longlong(res));
}

// The same Jacobi sweep restricted to the tiles (CT x CT nodes, one CTA each) whose 3 x 3 tile
// neighbourhood changed in the previous sweep; every other tile copies Vin -> Vout.  Exact (bit
// for bit the result of k_coarse_sweep): a node's update reads only nodes within its stencil
// reach (< CT cells, checked by the host), so if none of them changed since the last sweep its
// new value is the value the last sweep wrote, i.e. Vin.  Ahead of the front (V0, stationary) and
// behind it (converged) most tiles are skipped.  fprev / fout: per-tile "changed" flags of the
// previous / this sweep (fprev unused at sweep 0).
__global__ void __launch_bounds__(CT * CT, PDD_CANON_MINB) k_coarse_sweep_tiles(
    DProblem P, const double *__restrict__ Vin, double *__restrict__ Vout, double tol,
    unsigned long long *res_hist, int sweep, int *sweeps_done, const uint8_t *fprev,
    uint8_t *fout, int tiles_x, const CoarseRowEntry *rowtab, int stage_ok)
{
    if (sweep > 0 && __longlong_as_double((long long)res_hist[sweep - 1]) < tol) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(sweeps_done, 1);
    __shared__ int s_act;
    const int n = P.n;
    const int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
    const int tiles_y = (n + CT - 1) / CT;
    if (threadIdx.x == 0) {
        int act = sweep == 0;
        for (int dy = -1; dy <= 1 && !act; ++dy)
            for (int dx = -1; dx <= 1; ++dx) {
                const int ax = tx + dx, ay = ty + dy;
                if (ax >= 0 && ay >= 0 && ax < tiles_x && ay < tiles_y && fprev[ay * tiles_x + ax]) {
                    act = 1;
                    break;
                }
            }
        s_act = act;
    }
    __syncthreads();
    const int i = tx * CT + (int)(threadIdx.x % CT), j = ty * CT + (int)(threadIdx.x / CT);
    const int ib = tx * CT - CH, jb = ty * CT - CH;
    __shared__ double sV[CSW * CSW];
    extern __shared__ CoarseRowEntry sRT[];      // the tile's CT rows of the row table (if sized)
    const bool staged = rowtab && PDD_COARSE_SMEM && s_act && stage_ok;
    // interior tile (no foot clamped in x), table rows staged, den > 0: the fast path above
    const bool fast = PDD_CANON_FAST && staged && stage_ok > 1 && P.beta < 1.0 && tx * CT >= CH &&
                      tx * CT + CT - 1 + CH <= n - 1;
    if (staged) {
        for (int e = threadIdx.x; e < CSW * CSW; e += CT * CT) {
            const int gi = ib + e % CSW, gj = jb + e / CSW;
            sV[e] = (gi >= 0 && gj >= 0 && gi < n && gj < n) ? Vin[(int64_t)gj * n + gi] : 0.0;
        }
        if (stage_ok > 1) {
            const int rows = min(CT, n - ty * CT);
            for (int e = threadIdx.x; e < rows * P.na; e += CT * CT)
                sRT[e] = rowtab[(int64_t)ty * CT * P.na + e];
        }
        __syncthreads();
    }
    double res = 0.0;
    int changed = 0;
    if (i < n && j < n) {
        const int64_t k = (int64_t)j * n + i;
        const double vin = Vin[k];
        if (!s_act || P.kind[k] != 0) {
            Vout[k] = vin;
        } else {
            const double v = fast ? canon_node_update_fast(P, sV, i, j, ib, jb, sRT + (j - ty * CT) * P.na)
                           : staged ? canon_node_update_rt_s(P, sV, i, j, ib, jb,
                                                             stage_ok > 1 ? sRT + (j - ty * CT) * P.na
                                                                          : rowtab + (int64_t)j * P.na)
                           : rowtab ? canon_node_update_rt(P, Vin, i, j, rowtab + (int64_t)j * P.na)
                                    : canon_node_update(P, Vin, i, j);
            Vout[k] = v;
            res = fabs(DSUB(v, vin));
            changed = __double_as_longlong(v) != __double_as_longlong(vin);
        }
    }
    changed = __syncthreads_or(changed);
    if (threadIdx.x == 0) fout[blockIdx.x] = (uint8_t)(changed != 0);
    for (int o = 16; o > 0; o >>= 1) res = fmax(res, __shfl_xor_sync(0xffffffffu, res, o));
    if ((threadIdx.x & 31) == 0 && res > 0.0)
        atomicMax(&res_hist[sweep], (unsigned long long)__double_as_longlong(res));
}

__global__ void k_prolong(int nc, const double *__restrict__ uc, int n, int r, double *__restrict__ out)
{
    const int64_t N = (int64_t)n * n;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(k % n), j = (int)(k / n);
        int I = i / r, J = j / r;
        if (I > nc - 2) I = nc - 2;
        if (J > nc - 2) J = nc - 2;
        const double tx = DDIV((double)(i - I * r), (double)r);
        const double ty = DDIV((double)(j - J * r), (double)r);
        const double w00 = DMUL(DSUB(1.0, tx), DSUB(1.0, ty)), w10 = DMUL(tx, DSUB(1.0, ty));
        const double w01 = DMUL(DSUB(1.0, tx), ty), w11 = DMUL(tx, ty);
        const int64_t b = (int64_t)J * nc + I;
        double s = DMUL(w00, uc[b]);
        s = DADD(s, DMUL(w10, uc[b + 1]));
        s = DADD(s, DMUL(w01, uc[b + nc]));
        s = DADD(s, DMUL(w11, uc[b + nc + 1]));
        out[k] = s;
    }
}

__global__ void k_synthesize(DProblem P, const double *__restrict__ uhat, uint8_t *__restrict__ astar)
{
    const int n = P.n;
    const int64_t N = (int64_t)n * n;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        if (P.kind[k] != 0) { astar[k] = 255; continue; }
        const int i = (int)(k % n), j = (int)(k / n);
        const double c = coef_at(P.speed, i, j, n);
        const double d1 = coef_at(P.drift[0], i, j, n);
        const double d2 = coef_at(P.drift[1], i, j, n);
        const double lx = coef_at(P.cost, i, j, n);
        double best = INFINITY;
        int arg = -1;
        for (int a = 0; a < P.na; ++a) {
            const double hl = DMUL(P.h, P.cost_ctrl ? DADD(lx, P.cost_ctrl[a]) : lx);   // R33
            const double f1 = DADD(DMUL(c, P.ctrl[2 * a]), d1);
            const double f2 = DADD(DMUL(c, P.ctrl[2 * a + 1]), d2);
            const double gx = DADD((double)i, DMUL(P.q, f1));
            const double gy = DADD((double)j, DMUL(P.q, f2));
            int64_t cr[4];
            double wg[4];
            canon_stencil(n, gx, gy, cr, wg);
            double s = DMUL(wg[0], uhat[cr[0]]);
            s = DADD(s, DMUL(wg[1], uhat[cr[1]]));
            s = DADD(s, DMUL(wg[2], uhat[cr[2]]));
            s = DADD(s, DMUL(wg[3], uhat[cr[3]]));
            const double v = DADD(hl, DMUL(P.beta, s));
            if (v < best) { best = v; arg = a; }
        }
        astar[k] = (uint8_t)arg;
    }
}

// ------------------------------------------------------------------ fuzzy patches (NEXT #2)
// phi_p = chi_{Gamma_p} on the Dirichlet set, 0 on free nodes; patch-major layout.
__global__ void k_fuzzy_init(DProblem P, const int16_t *__restrict__ sector, int np, double *phi)
{
    const int64_t N = (int64_t)P.n * P.n;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int sp = P.kind[k] == 1 ? sector[k] : -1;
        for (int p = 0; p < np; ++p) phi[(int64_t)p * N + k] = sp == p ? 1.0 : 0.0;
    }
}

// One Jacobi sweep of the SL advection scheme phi_p(x_i) = phi_p(x_i + h f(x_i, a*(x_i)))
// (Eq. discrete-advection) for every patch, canonical fp64 (the synthesis foot,
// corner sums in the order 00, 10, 01, 11); self-stopping once the previous sweep's change was
// < eps (same protocol as k_coarse_sweep).
__global__ void k_fuzzy_sweep(DProblem P, const uint8_t *__restrict__ astar, int np,
                              const double *__restrict__ cur, double *__restrict__ nxt, double eps,
                              unsigned long long *res_hist, int sweep, int *sweeps_done)
{
    if (sweep > 0 && __longlong_as_double((long long)res_hist[sweep - 1]) < eps) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(sweeps_done, 1);
    const int n = P.n;
    const int64_t N = (int64_t)n * n;
    double res = 0.0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        if (P.kind[k] != 0) {
            for (int p = 0; p < np; ++p) nxt[(int64_t)p * N + k] = cur[(int64_t)p * N + k];
            continue;
        }
        const int i = (int)(k % n), j = (int)(k / n);
        const int a = astar[k];
        const double c = coef_at(P.speed, i, j, n);
        const double f1 = DADD(DMUL(c, P.ctrl[2 * a]), coef_at(P.drift[0], i, j, n));
        const double f2 = DADD(DMUL(c, P.ctrl[2 * a + 1]), coef_at(P.drift[1], i, j, n));
        int64_t cr[4];
        double wg[4];
        canon_stencil(n, DADD((double)i, DMUL(P.q, f1)), DADD((double)j, DMUL(P.q, f2)), cr, wg);
        for (int p = 0; p < np; ++p) {
            const double *F = cur + (int64_t)p * N;
            double v = DMUL(wg[0], F[cr[0]]);
            v = DADD(v, DMUL(wg[1], F[cr[1]]));
            v = DADD(v, DMUL(wg[2], F[cr[2]]));
            v = DADD(v, DMUL(wg[3], F[cr[3]]));
            nxt[(int64_t)p * N + k] = v;
            res = fmax(res, fabs(DSUB(v, F[k])));
        }
    }
    for (int o = 16; o > 0; o >>= 1) res = fmax(res, __shfl_xor_sync(0xffffffffu, res, o));
    if ((threadIdx.x & 31) == 0 && res > 0.0)
        atomicMax(&res_hist[sweep], (unsigned long long)__double_as_longlong(res));
}

// Thresholding / ownership (R38): owner = the patch of largest phi_p (lowest p on
// ties; it belongs to Omega_p = {phi_p >= tau} whenever any patch does), orphan n_patches when no
// phi_p is positive; members = number of patches with phi_p >= tau (overlap degree).
__global__ void k_fuzzy_assign(DProblem P, const double *__restrict__ phi, int np, double tau,
                               int16_t *__restrict__ labels, int *overlap)
{
    const int64_t N = (int64_t)P.n * P.n;
    int ov = 0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t kd = P.kind[k];
        if (kd != 0) { labels[k] = kd == 1 ? -1 : -2; continue; }
        int best = -1, cnt = 0;
        double bv = 0.0;
        for (int p = 0; p < np; ++p) {
            const double v = phi[(int64_t)p * N + k];
            if (v >= tau) ++cnt;
            if (v > bv) { bv = v; best = p; }
        }
        labels[k] = (int16_t)(best < 0 ? np : best);
        ov += cnt >= 2;
    }
    for (int o = 16; o > 0; o >>= 1) ov += __shfl_xor_sync(0xffffffffu, ov, o);
    if ((threadIdx.x & 31) == 0 && ov) atomicAdd(overlap, ov);
}

// ------------------------------------------------------------------ sparse fuzzy patches
// Per node the K largest (patch, phi_p) pairs, sorted by (phi_p descending, patch ascending),
// empty slots (-1, 0) last (reading R40; the dense fields above need 16 N_P n^2 bytes, this form
// 20 K n^2).  One Jacobi sweep merges the four corner lists in the order 00, 10, 01, 11 -- a
// label's partial sums are added in corner order: the dense expression with its zero terms left
// out, so with K >= the number of patches reaching a node the result has the dense bits.
template <int K>
__device__ __forceinline__ void sparse_topk_insert(int16_t *ol, double *om, int &cnt, int16_t l, double m)
{
    int pos = cnt;
    while (pos > 0 && (om[pos - 1] < m || (om[pos - 1] == m && ol[pos - 1] > l))) --pos;
    if (pos >= K) return;
    const int last = cnt < K ? cnt : K - 1;
    for (int s = last; s > pos; --s) { ol[s] = ol[s - 1]; om[s] = om[s - 1]; }
    ol[pos] = l;
    om[pos] = m;
    if (cnt < K) ++cnt;
}

__global__ void k_fuzzy_sparse_init(DProblem P, const int16_t *__restrict__ sector, int np, int K,
                                    int16_t *lab, double *mass)
{
    const int64_t N = (int64_t)P.n * P.n;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int sp = P.kind[k] == 1 ? sector[k] : -1;
        const bool on = sp >= 0 && sp < np;
        for (int s = 0; s < K; ++s) {
            lab[k * K + s] = (s == 0 && on) ? (int16_t)sp : (int16_t)-1;
            mass[k * K + s] = (s == 0 && on) ? 1.0 : 0.0;
        }
    }
}

template <int K>
__global__ void k_fuzzy_sparse_sweep(DProblem P, const uint8_t *__restrict__ astar,
                                     const int16_t *__restrict__ clab, const double *__restrict__ cm,
                                     int16_t *__restrict__ nlab, double *__restrict__ nm, double eps,
                                     unsigned long long *res_hist, int sweep, int *sweeps_done)
{
    if (sweep > 0 && __longlong_as_double((long long)res_hist[sweep - 1]) < eps) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(sweeps_done, 1);
    const int n = P.n;
    const int64_t N = (int64_t)n * n;
    double res = 0.0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        if (P.kind[k] != 0) {
#pragma unroll
            for (int s = 0; s < K; ++s) { nlab[k * K + s] = clab[k * K + s]; nm[k * K + s] = cm[k * K + s]; }
            continue;
        }
        const int i = (int)(k % n), j = (int)(k / n);
        const int a = astar[k];
        const double c = coef_at(P.speed, i, j, n);
        const double f1 = DADD(DMUL(c, P.ctrl[2 * a]), coef_at(P.drift[0], i, j, n));
        const double f2 = DADD(DMUL(c, P.ctrl[2 * a + 1]), coef_at(P.drift[1], i, j, n));
        int64_t cr[4];
        double wg[4];
        canon_stencil(n, DADD((double)i, DMUL(P.q, f1)), DADD((double)j, DMUL(P.q, f2)), cr, wg);
        int16_t al[4 * K];
        double am[4 * K];
        int na = 0;
        for (int t = 0; t < 4; ++t)
            for (int s = 0; s < K; ++s) {
                const int16_t l = clab[cr[t] * K + s];
                if (l < 0) continue;
                const double term = DMUL(wg[t], cm[cr[t] * K + s]);
                int idx = 0;
                while (idx < na && al[idx] != l) ++idx;
                if (idx < na) am[idx] = DADD(am[idx], term);
                else { al[na] = l; am[na] = term; ++na; }
            }
        int16_t ol[K], oldl[K];
        double om[K], oldm[K];
        int cnt = 0;
        for (int idx = 0; idx < na; ++idx)
            if (am[idx] > 0.0) sparse_topk_insert<K>(ol, om, cnt, al[idx], am[idx]);
#pragma unroll
        for (int u = 0; u < K; ++u) { oldl[u] = clab[k * K + u]; oldm[u] = cm[k * K + u]; }
        for (int s = 0; s < cnt; ++s) {
            double old = 0.0;
            for (int u = 0; u < K; ++u)
                if (oldl[u] == ol[s]) old = oldm[u];
            res = fmax(res, fabs(DSUB(om[s], old)));
        }
        for (int u = 0; u < K; ++u) {
            if (oldl[u] < 0) continue;
            bool found = false;
            for (int s = 0; s < cnt; ++s) found |= ol[s] == oldl[u];
            if (!found) res = fmax(res, oldm[u]);
        }
        for (int s = 0; s < K; ++s) {
            nlab[k * K + s] = s < cnt ? ol[s] : (int16_t)-1;
            nm[k * K + s] = s < cnt ? om[s] : 0.0;
        }
    }
    for (int o = 16; o > 0; o >>= 1) res = fmax(res, __shfl_xor_sync(0xffffffffu, res, o));
    if ((threadIdx.x & 31) == 0 && res > 0.0)
        atomicMax(&res_hist[sweep], (unsigned long long)__double_as_longlong(res));
}

// owner = first listed patch (largest phi_p, lowest p on ties), orphan np when the list is empty;
// overlap: free nodes with >= 2 listed patches of phi_p >= tau; maxlist: the longest list found
// (== K means some node may have lost memberships to the truncation)
__global__ void k_fuzzy_sparse_assign(DProblem P, const int16_t *__restrict__ lab,
                                      const double *__restrict__ mass, int K, int np, double tau,
                                      int16_t *__restrict__ labels, int *overlap, int *maxlist)
{
    const int64_t N = (int64_t)P.n * P.n;
    int ov = 0, ml = 0;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t kd = P.kind[k];
        if (kd != 0) { labels[k] = kd == 1 ? -1 : -2; continue; }
        int cnt = 0, len = 0;
        for (int s = 0; s < K; ++s) {
            if (lab[k * K + s] < 0) continue;
            ++len;
            if (mass[k * K + s] >= tau) ++cnt;
        }
        labels[k] = lab[k * K] >= 0 ? lab[k * K] : (int16_t)np;
        ov += cnt >= 2;
        ml = max(ml, len);
    }
    for (int o = 16; o > 0; o >>= 1) {
        ov += __shfl_xor_sync(0xffffffffu, ov, o);
        ml = max(ml, __shfl_xor_sync(0xffffffffu, ml, o));
    }
    if ((threadIdx.x & 31) == 0) {
        if (ov) atomicAdd(overlap, ov);
        atomicMax(maxlist, ml);
    }
}

// k_synthesize with the row-invariant table of k_coarse_rowtab built on the fine grid (row-uniform
// coefficients): the same operations per (node, control), the row-dependent ones hoisted
__global__ void k_synthesize_rt(DProblem P, const double *__restrict__ uhat,
                                const CoarseRowEntry *__restrict__ tab, uint8_t *__restrict__ astar)
{
    const int n = P.n;
    const int64_t N = (int64_t)n * n;
    const double top = (double)(n - 1);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        if (P.kind[k] != 0) { astar[k] = 255; continue; }
        const int i = (int)(k % n), j = (int)(k / n);
        const CoarseRowEntry *row = tab + (int64_t)j * P.na;
        double best = INFINITY;
        int arg = -1;
        for (int a = 0; a < P.na; ++a) {
            const CoarseRowEntry e = row[a];
            double gx = DADD((double)i, e.bxq);
            if (gx < 0.0) gx = 0.0;
            if (gx > top) gx = top;
            int cx = (int)floor(gx);
            if (cx > n - 2) cx = n - 2;
            const double tx = DSUB(gx, (double)cx);
            const double ux = DSUB(1.0, tx);
            const int64_t c0 = (int64_t)e.cy * n + cx;
            double s = DMUL(DMUL(ux, e.uy), uhat[c0]);
            s = DADD(s, DMUL(DMUL(tx, e.uy), uhat[c0 + 1]));
            s = DADD(s, DMUL(DMUL(ux, e.ty), uhat[c0 + n]));
            s = DADD(s, DMUL(DMUL(tx, e.ty), uhat[c0 + n + 1]));
            const double v = DADD(e.hl, DMUL(P.beta, s));
            if (v < best) { best = v; arg = a; }
        }
        astar[k] = (uint8_t)arg;
    }
}

// k_synthesize_rt on 16 x 16 node tiles with u_hat's tile + halo (CH cells) staged in shared
// memory: the 4 N_A gathers per node hit shared memory.  Same operations: bit-identical.
#ifndef PDD_SYNTH_UNROLL
#define PDD_SYNTH_UNROLL 4 // controls per loop trip of the strip kernel (A/B)
#endif
#ifndef PDD_SYNTH_STRIP
#define PDD_SYNTH_STRIP 8  // tiles per CTA (one strip of a tile row)
#endif
// A CTA walks `strip` consecutive tiles of one tile row; when `rt_staged` the 16 rows of the table
// it needs are copied to shared memory once per CTA (the per-control table reads from global memory
// were the kernel's main stall: long scoreboard 6.6 per issue, profiles/r4b_*).
template <bool rt_staged>
__global__ void __launch_bounds__(256, PDD_CANON_MINB) k_synthesize_rt_s(DProblem P, const double *__restrict__ uhat,
                                                         const CoarseRowEntry *__restrict__ tab,
                                                         uint8_t *__restrict__ astar, int tiles_x,
                                                         int strip)
{
    __shared__ double sU[CSW * CSW];
    extern __shared__ CoarseRowEntry sRTs[];
    const int n = P.n;
    const int strips_x = (tiles_x + strip - 1) / strip;
    const int ty = blockIdx.x / strips_x, tx0 = (blockIdx.x % strips_x) * strip;
    const int jb = ty * 16 - CH;
    const int j = ty * 16 + (int)(threadIdx.x >> 4);
    if (rt_staged) {
        const int rows = min(16, n - ty * 16);
        for (int e = threadIdx.x; e < rows * P.na; e += 256) sRTs[e] = tab[(int64_t)ty * 16 * P.na + e];
    }
    const CoarseRowEntry *row = rt_staged ? sRTs + (j - ty * 16) * P.na : tab + (int64_t)min(j, n - 1) * P.na;
    const double top = (double)(n - 1);
    for (int tx = tx0; tx < min(tx0 + strip, tiles_x); ++tx) {
        const int ib = tx * 16 - CH;
        __syncthreads();                       // the previous tile's readers are done (and sRTs is filled)
        for (int e = threadIdx.x; e < CSW * CSW; e += 256) {
            const int gi = ib + e % CSW, gj = jb + e / CSW;
            sU[e] = (gi >= 0 && gj >= 0 && gi < n && gj < n) ? uhat[(int64_t)gj * n + gi] : 0.0;
        }
        __syncthreads();
        const int i = tx * 16 + (int)(threadIdx.x & 15);
        if (i >= n || j >= n) continue;
        const int64_t k = (int64_t)j * n + i;
        if (P.kind[k] != 0) { astar[k] = 255; continue; }
        double best = INFINITY;
        int arg = -1;
        if (tx * 16 >= CH && tx * 16 + 15 + CH <= n - 1) {
            // interior tile: with reach <= CH - 1 no foot of its nodes is clamped in x (0 <= i + q f1 <=
            // n - 1 and floor <= n - 2), so the three clamps below are dropped -- same bits, 2 FP64
            // compares fewer per control on a kernel bound by the FP64 pipe (profiles/r4n_synth_*)
            PDD_UNROLL_(PDD_SYNTH_UNROLL)
            for (int a = 0; a < P.na; ++a) {
                const CoarseRowEntry e = row[a];
                const double gx = DADD((double)i, e.bxq);
                const int cx = (int)floor(gx);
                const double tx2 = DSUB(gx, (double)cx);
                const double ux = DSUB(1.0, tx2);
                const int s0 = (e.cy - jb) * CSW + (cx - ib);
                double sm = DMUL(DMUL(ux, e.uy), sU[s0]);
                sm = DADD(sm, DMUL(DMUL(tx2, e.uy), sU[s0 + 1]));
                sm = DADD(sm, DMUL(DMUL(ux, e.ty), sU[s0 + CSW]));
                sm = DADD(sm, DMUL(DMUL(tx2, e.ty), sU[s0 + CSW + 1]));
                const double v = DADD(e.hl, DMUL(P.beta, sm));
                if (v < best) { best = v; arg = a; }
            }
            astar[k] = (uint8_t)arg;
            continue;
        }
        PDD_UNROLL_(PDD_SYNTH_UNROLL)
        for (int a = 0; a < P.na; ++a) {
            const CoarseRowEntry e = row[a];
            double gx = DADD((double)i, e.bxq);
            if (gx < 0.0) gx = 0.0;
            if (gx > top) gx = top;
            int cx = (int)floor(gx);
            if (cx > n - 2) cx = n - 2;
            const double tx2 = DSUB(gx, (double)cx);
            const double ux = DSUB(1.0, tx2);
            const int s0 = (e.cy - jb) * CSW + (cx - ib);
            double sm = DMUL(DMUL(ux, e.uy), sU[s0]);
            sm = DADD(sm, DMUL(DMUL(tx2, e.uy), sU[s0 + 1]));
            sm = DADD(sm, DMUL(DMUL(ux, e.ty), sU[s0 + CSW]));
            sm = DADD(sm, DMUL(DMUL(tx2, e.ty), sU[s0 + CSW + 1]));
            const double v = DADD(e.hl, DMUL(P.beta, sm));
            if (v < best) { best = v; arg = a; }
        }
        astar[k] = (uint8_t)arg;
    }
}

__global__ void k_successor(DProblem P, double M, const uint8_t *__restrict__ astar,
                            int32_t *__restrict__ succ)
{
    const int n = P.n;
    const int64_t N = (int64_t)n * n;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        if (P.kind[k] != 0) { succ[k] = (int32_t)k; continue; }
        const int i = (int)(k % n), j = (int)(k / n);
        const int a = astar[k];
        const double c = coef_at(P.speed, i, j, n);
        const double f1 = DADD(DMUL(c, P.ctrl[2 * a]), coef_at(P.drift[0], i, j, n));
        const double f2 = DADD(DMUL(c, P.ctrl[2 * a + 1]), coef_at(P.drift[1], i, j, n));
        const double nrm = __dsqrt_rn(DADD(DMUL(f1, f1), DMUL(f2, f2)));
        if (nrm == 0.0) { succ[k] = (int32_t)k; continue; }
        const double u1 = DDIV(f1, nrm), u2 = DDIV(f2, nrm);
        const double gx = DADD((double)i, DMUL(M, u1));
        const double gy = DADD((double)j, DMUL(M, u2));
        int si = (int)floor(DADD(gx, 0.5)), sj = (int)floor(DADD(gy, 0.5));
        si = si < 0 ? 0 : (si > n - 1 ? n - 1 : si);
        sj = sj < 0 ? 0 : (sj > n - 1 ? n - 1 : sj);
        succ[k] = (int32_t)((int64_t)sj * n + si);
    }
}

__global__ void k_jump(const int32_t *__restrict__ in, int32_t *__restrict__ out, int64_t N,
                       int *changed)
{
    bool ch = false;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t s = in[k];
        const int32_t ss = in[s];
        out[k] = ss;
        ch |= (ss != s);
    }
    if (__any_sync(0xffffffffu, ch) && (threadIdx.x & 31) == 0) atomicOr(changed, 1);
}

__global__ void k_labels(const uint8_t *__restrict__ kind, const int16_t *__restrict__ sector,
                         const int32_t *__restrict__ root, int n_patches, int64_t N,
                         int16_t *__restrict__ labels)
{
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t kd = kind[k];
        if (kd == 1) { labels[k] = -1; continue; }
        if (kd == 2) { labels[k] = -2; continue; }
        const int32_t r = root[k];
        labels[k] = kind[r] == 1 ? sector[r] : (int16_t)n_patches;
    }
}

__global__ void k_static_labels(int n, int px, int py, const uint8_t *__restrict__ kind,
                                int16_t *__restrict__ labels)
{
    const int64_t N = (int64_t)n * n;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(k % n), j = (int)(k / n);
        int bx = (int)(((int64_t)i * px) / n), by = (int)(((int64_t)j * py) / n);
        // boundaries floor(k n / P): the largest b with floor(b n / P) <= i
        while (bx + 1 < px && ((int64_t)(bx + 1) * n) / px <= i) ++bx;
        while (bx > 0 && ((int64_t)bx * n) / px > i) --bx;
        while (by + 1 < py && ((int64_t)(by + 1) * n) / py <= j) ++by;
        while (by > 0 && ((int64_t)by * n) / py > j) --by;
        const uint8_t kd = kind[k];
        labels[k] = kd == 1 ? -1 : kd == 2 ? -2 : (int16_t)(by * px + bx);
    }
}

static int grid_for(int64_t N, int block)
{
    int64_t g = (N + block - 1) / block;
    if (g > 148 * 32) g = 148 * 32;
    return (int)(g < 1 ? 1 : g);
}

void launch_init_values(const DProblem &P, double *V, cudaStream_t s)
{
    const int64_t N = (int64_t)P.n * P.n;
    k_init_values<<<grid_for(N, 256), 256, 0, s>>>(P, V);
}

void launch_coarse_sweep(const DProblem &P, const double *Vin, double *Vout, double tol,
                         unsigned long long *res_hist, int sweep, int *sweeps_done,
                         cudaStream_t s)
{
    const int64_t N = (int64_t)P.n * P.n;
    k_coarse_sweep<<<grid_for(N, 128), 128, 0, s>>>(P, Vin, Vout, tol, res_hist, sweep,
                                                     sweeps_done);
}

void launch_coarse_sweep_tiles(const DProblem &P, const double *Vin, double *Vout, double tol,
                               unsigned long long *res_hist, int sweep, int *sweeps_done,
                               const uint8_t *fprev, uint8_t *fout, const CoarseRowEntry *rowtab,
                               int stage_ok, cudaStream_t s)
{
    const int tx = (P.n + CT - 1) / CT;
    // stage the tile's rows of the row table too when they fit (stage_ok = 2)
    size_t dyn = 0;
    if (stage_ok && rowtab && PDD_COARSE_RTSMEM) {
        dyn = sizeof(CoarseRowEntry) * CT * (size_t)P.na;
        if (dyn > 64 * 1024) dyn = 0;
        else {
            // the attribute is per device: set it once on each device the library runs on
            static bool attr[64] = {};
            int dev = 0;
            cudaGetDevice(&dev);
            if (dev < 0 || dev >= 64 || !attr[dev]) {
                cudaFuncSetAttribute(k_coarse_sweep_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
                if (dev >= 0 && dev < 64) attr[dev] = true;
            }
            stage_ok = 2;
        }
    }
    k_coarse_sweep_tiles<<<tx * tx, CT * CT, dyn, s>>>(P, Vin, Vout, tol, res_hist, sweep,
                                                       sweeps_done, fprev, fout, tx, rowtab, stage_ok);
}

int coarse_halo() { return CH; }

void launch_coarse_rowtab(const DProblem &P, CoarseRowEntry *tab, cudaStream_t s)
{
    const int64_t m = (int64_t)P.n * P.na;
    k_coarse_rowtab<<<grid_for(m, 128), 128, 0, s>>>(P, tab);
}

int coarse_tile() { return CT; }

void launch_fuzzy_init(const DProblem &P, const int16_t *sector, int np, double *phi, cudaStream_t s)
{
    const int64_t N = (int64_t)P.n * P.n;
    k_fuzzy_init<<<grid_for(N, 256), 256, 0, s>>>(P, sector, np, phi);
}

void launch_fuzzy_sweep(const DProblem &P, const uint8_t *astar, int np, const double *cur,
                        double *nxt, double eps, unsigned long long *res_hist, int sweep,
                        int *sweeps_done, cudaStream_t s)
{
    const int64_t N = (int64_t)P.n * P.n;
    k_fuzzy_sweep<<<grid_for(N, 128), 128, 0, s>>>(P, astar, np, cur, nxt, eps, res_hist, sweep,
                                                    sweeps_done);
}

void launch_fuzzy_sparse_init(const DProblem &P, const int16_t *sector, int np, int K, int16_t *lab,
                              double *mass, cudaStream_t s)
{
    const int64_t N = (int64_t)P.n * P.n;
    k_fuzzy_sparse_init<<<grid_for(N, 256), 256, 0, s>>>(P, sector, np, K, lab, mass);
}

bool launch_fuzzy_sparse_sweep(const DProblem &P, const uint8_t *astar, int K, const int16_t *clab,
                               const double *cm, int16_t *nlab, double *nm, double eps,
                               unsigned long long *res_hist, int sweep, int *sweeps_done, cudaStream_t s)
{
    const int64_t N = (int64_t)P.n * P.n;
    const int g = grid_for(N, 128);
#define PDD_FS(K_)                                                                                     \
    case K_:                                                                                           \
        k_fuzzy_sparse_sweep<K_><<<g, 128, 0, s>>>(P, astar, clab, cm, nlab, nm, eps, res_hist, sweep, \
                                                   sweeps_done);                                       \
        return true;
    switch (K) {
        PDD_FS(1) PDD_FS(2) PDD_FS(3) PDD_FS(4) PDD_FS(6) PDD_FS(8) PDD_FS(16)
    default: return false;
    }
#undef PDD_FS
}

void launch_fuzzy_sparse_assign(const DProblem &P, const int16_t *lab, const double *mass, int K, int np,
                                double tau, int16_t *labels, int *overlap, int *maxlist, cudaStream_t s)
{
    const int64_t N = (int64_t)P.n * P.n;
    k_fuzzy_sparse_assign<<<grid_for(N, 256), 256, 0, s>>>(P, lab, mass, K, np, tau, labels, overlap, maxlist);
}

void launch_fuzzy_assign(const DProblem &P, const double *phi, int np, double tau, int16_t *labels,
                         int *overlap, cudaStream_t s)
{
    const int64_t N = (int64_t)P.n * P.n;
    k_fuzzy_assign<<<grid_for(N, 256), 256, 0, s>>>(P, phi, np, tau, labels, overlap);
}

void launch_prolong(int nc, const double *uc, int n, double *out, cudaStream_t s)
{
    const int64_t N = (int64_t)n * n;
    k_prolong<<<grid_for(N, 256), 256, 0, s>>>(nc, uc, n, (n - 1) / (nc - 1), out);
}

void launch_synthesize_rt(const DProblem &P, const double *uhat, const CoarseRowEntry *tab,
                          uint8_t *astar, int stage_ok, cudaStream_t s)
{
    if (stage_ok && PDD_COARSE_SMEM) {
        const int tx = (P.n + 15) / 16;
        // strips of PDD_SYNTH_STRIP tiles; the CTA's 16 table rows staged in shared memory when they fit
        // (shorter strips on small grids: keep >= 8 CTAs per SM in the grid)
        int strip = PDD_SYNTH_STRIP;
        while (strip > 1 && ((tx + strip - 1) / strip) * tx < 148 * 8) strip /= 2;
        const int strips_x = (tx + strip - 1) / strip;
        size_t dyn = sizeof(CoarseRowEntry) * 16 * (size_t)P.na;
        if (dyn > 64 * 1024) dyn = 0;
        else {
            static bool attr[64] = {};
            int dev = 0;
            cudaGetDevice(&dev);
            if (dev < 0 || dev >= 64 || !attr[dev]) {
                cudaFuncSetAttribute(k_synthesize_rt_s<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
                if (dev >= 0 && dev < 64) attr[dev] = true;
            }
        }
        if (dyn) k_synthesize_rt_s<true><<<strips_x * tx, 256, dyn, s>>>(P, uhat, tab, astar, tx, strip);
        else k_synthesize_rt_s<false><<<strips_x * tx, 256, 0, s>>>(P, uhat, tab, astar, tx, strip);
        return;
    }
    const int64_t N = (int64_t)P.n * P.n;
    k_synthesize_rt<<<grid_for(N, 128), 128, 0, s>>>(P, uhat, tab, astar);
}

void launch_synthesize(const DProblem &P, const double *uhat, uint8_t *astar, cudaStream_t s)
{
    const int64_t N = (int64_t)P.n * P.n;
    k_synthesize<<<grid_for(N, 128), 128, 0, s>>>(P, uhat, astar);
}

void launch_successor(const DProblem &P, double M, const uint8_t *astar, int32_t *succ,
                      cudaStream_t s)
{
    const int64_t N = (int64_t)P.n * P.n;
    k_successor<<<grid_for(N, 256), 256, 0, s>>>(P, M, astar, succ);
}

void launch_jump(const int32_t *in, int32_t *out, int64_t N, int *changed, cudaStream_t s)
{
    k_jump<<<grid_for(N, 256), 256, 0, s>>>(in, out, N, changed);
}

void launch_labels(const uint8_t *kind, const int16_t *sector, const int32_t *root,
                   int n_patches, int64_t N, int16_t *labels, cudaStream_t s)
{
    k_labels<<<grid_for(N, 256), 256, 0, s>>>(kind, sector, root, n_patches, N, labels);
}

void launch_static_labels(int n, int px, int py, const uint8_t *kind, int16_t *labels,
                          cudaStream_t s)
{
    const int64_t N = (int64_t)n * n;
    k_static_labels<<<grid_for(N, 256), 256, 0, s>>>(n, px, py, kind, labels);
}

}  // namespace pdd
