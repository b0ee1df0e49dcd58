/*
 * pdd_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity oracle).
 *
 * A plain, slow, fp64 CPU implementation of what the hot path of arXiv 1502.01629 computes.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library.  It shares no code, header, table or constant generator with the CUDA
 * path (paper_1502_01629_b200/); both read the same input arrays built by pdd_inputs/.
 *
 * Citations: P:<line> = PAPER.md, S:<line> = SPEC.md, R<k> = reading k listed in DESIGN.md.
 *
 * Every floating-point expression below is written in the order of DESIGN.md reading R30
 * ("canonical arithmetic"): compile with -O2 -ffp-contract=off, no -ffast-math, so that the
 * decision stages (coarse solve, prolongation, synthesis, successor) give the same bits as any
 * other IEEE-754 implementation that evaluates the same expressions in the same order.
 *
 * Functions (each cites the passage it follows):
 *   orc_node_update  : SL scheme at one node.  scheme 0 = modified scheme (SLscheme3) P:473-491
 *                      with the discount of BASELINE.json (R1, R3); scheme 1 = original scheme
 *                      (SLscheme2) P:366-375 (test-only).  Markov-chain foot points P:369 with
 *                      the sqrt(h p) scaling of the north star (R2).
 *   orc_jacobi       : fixed-point iteration u <- T(u) on all free nodes at once (plain
 *                      definition of the fixed point; S:279-296 stats semantics).
 *   orc_gauss_seidel : same operator in place, in a given node order (test-only).
 *   orc_prolong      : bilinear reconstruction of u_c on G.
 *   orc_synthesize   : discrete synthesis, Eq. (discrete-synthesis) P:768-773 with discount (R16).
 *   orc_successor / orc_labels : patch labelling by following the synthesised optimal field to
 *                      the target (north star; R17, R18), sequential chase with memo.
 *   orc_static_labels: static equal-square decomposition P:1110-1111 (R19).
 *   orc_*_at         : the same definitions evaluated at sampled nodes (full-size parity).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int32_t kind;        /* 0 const, 1 row (x2), 2 col (x1), 3 field n*n */
    double value;
    const double *data;
} orc_coef;

typedef struct {
    int32_t n;
    double lo, dx, h, lambda;
    int32_t na;
    const double *ctrl;  /* 2*na: (a1, a2) per control */
    orc_coef speed;      /* c(x): f(x,a) = c(x) a + d(x) */
    orc_coef drift[2];   /* d(x) */
    int32_t p;           /* noise columns sigma_k, k < p */
    orc_coef sigma[2][2];/* sigma[k][component] */
    orc_coef cost;       /* l(x) */
    int32_t diffusion_scale; /* 0: sqrt(h p), 1: sqrt(h) */
    const uint8_t *kind; /* 0 free, 1 target (V = 0), 2 obstacle (V = 1/lambda) */
    /* general nonlinear terms (readings R32/R33):
     * sigma_mode 1: one noise column along the control, sigma(x,a) = s(x) a with s = sigma[0][0]
     *               (the paper's sigma_3(x,a) = d_eps(x) a; p must be 1);
     * cost_ctrl:    per-control additive cost m(a_k), l(x,a) = l(x) + m(a) (the paper's l_3),
     *               NULL = 0. */
    int32_t sigma_mode;
    const double *cost_ctrl;
} orc_problem;

/* running cost l(x_i, a_k) (R33) */
static double cost_of(const orc_problem *P, double lx, int a)
{
    return P->cost_ctrl ? lx + P->cost_ctrl[a] : lx;
}

static double coef_at(const orc_coef *c, int i, int j, int n)
{
    switch (c->kind) {
    case 0: return c->value;
    case 1: return c->data[j];
    case 2: return c->data[i];
    default: return c->data[(int64_t)j * n + i];
    }
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_threads(int t)
{
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

/* Dirichlet value of a non-free node: target -> g = 0, obstacle -> 1/lambda (R8). */
static double dirichlet_value(const orc_problem *P, int64_t idx)
{
    return P->kind[idx] == 1 ? 0.0 : 1.0 / P->lambda;
}

/* beta = 1/(1 + lambda h) (BASELINE.json configs). */
double orc_beta(const orc_problem *P) { return 1.0 / (1.0 + P->lambda * P->h); }

/* Initial guess V0 (R11): free nodes h*l_max/(1 - beta), the smallest constant supersolution;
 * lambda = 0 (exit problems) uses the "very big value" 1e6 of P:818-819.  Dirichlet nodes keep g. */
void orc_init_v0(const orc_problem *P, double *V)
{
    const int n = P->n;
    double lmax = 0.0;
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            double l = coef_at(&P->cost, i, j, n);
            if (l > lmax) lmax = l;
        }
    if (P->cost_ctrl) {
        double mmax = -INFINITY;
        for (int a = 0; a < P->na; ++a)
            if (P->cost_ctrl[a] > mmax) mmax = P->cost_ctrl[a];
        lmax = lmax + mmax;
    }
    double beta = orc_beta(P);
    double v0 = P->lambda > 0.0 ? (P->h * lmax) / (1.0 - beta) : 1e6;
    for (int64_t k = 0; k < (int64_t)n * n; ++k)
        V[k] = P->kind[k] == 0 ? v0 : dirichlet_value(P, k);
}

/* Bilinear reconstruction of V at the point (gx, gy) given in node units (Fig. 2,
 * P:403-412).  The point is clamped to the grid box (R5); the cell is the one whose lower-left
 * corner is floor(g) (the last cell at the upper edge).  Corner order 00, 10, 01, 11.
 * Returns the weights and corner indices. */
static void bilinear_stencil(int n, double gx, double gy, int64_t corner[4], double wgt[4])
{
    if (gx < 0.0) gx = 0.0;
    if (gx > (double)(n - 1)) gx = (double)(n - 1);
    if (gy < 0.0) gy = 0.0;
    if (gy > (double)(n - 1)) gy = (double)(n - 1);
    int cx = (int)floor(gx);
    int cy = (int)floor(gy);
    if (cx > n - 2) cx = n - 2;
    if (cy > n - 2) cy = n - 2;
    double tx = gx - (double)cx;
    double ty = gy - (double)cy;
    wgt[0] = (1.0 - tx) * (1.0 - ty);
    wgt[1] = tx * (1.0 - ty);
    wgt[2] = (1.0 - tx) * ty;
    wgt[3] = tx * ty;
    corner[0] = (int64_t)cy * n + cx;
    corner[1] = (int64_t)cy * n + cx + 1;
    corner[2] = (int64_t)(cy + 1) * n + cx;
    corner[3] = (int64_t)(cy + 1) * n + cx + 1;
}

/* Exposed for pin P1: weights of the bilinear stencil at (gx, gy) on an n-grid. */
void orc_bilinear_weights(int n, double gx, double gy, int64_t *corner, double *wgt)
{
    bilinear_stencil(n, gx, gy, corner, wgt);
}

/* One node of the SL scheme (P:366-375 / P:473-491), discounted per BASELINE.json:
 *   foot points x_{i,k}^{a,s} = x_i + h f(x_i,a) + s * sc * sigma_k(x_i), s = +-1, k < p
 *       (one foot point x_i + h f when p = 0);  sc = sqrt(h p) (R2) or sqrt(h);
 *   Lambda0(a) = (1/2p) sum lambda_{i0}      (weight of x_i itself)
 *   R'(a)      = (1/2p) sum_{corners != x_i} lambda u(corner)
 *   scheme 0 (SLscheme3 + discount, R3):  v(a) = (h l + beta R'(a)) / (1 - beta Lambda0(a))
 *   scheme 1 (SLscheme2 + discount):      v(a) = h l + beta (R'(a) + Lambda0(a) u(x_i))
 *   u(x_i) = min_a v(a); argmin = lowest index on ties (strict <, R10).
 * All positions in node units: g = i + q f (+ offset), q = h/dx. */
double orc_node_update(const orc_problem *P, const double *V, int i, int j, int scheme,
                       int32_t *argmin_out)
{
    const int n = P->n;
    const int64_t self = (int64_t)j * n + i;
    const double beta = orc_beta(P);
    const double q = P->h / P->dx;
    const int nb = P->p > 0 ? 2 * P->p : 1;
    const double w = 1.0 / (double)nb;
    double sc = 0.0;
    if (P->p > 0)
        sc = (P->diffusion_scale == 0 ? sqrt(P->h * (double)P->p) : sqrt(P->h)) / P->dx;
    const double c = coef_at(&P->speed, i, j, n);
    const double d1 = coef_at(&P->drift[0], i, j, n);
    const double d2 = coef_at(&P->drift[1], i, j, n);
    const double l = coef_at(&P->cost, i, j, n);
    double off[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    for (int k = 0; k < P->p; ++k) {
        off[k][0] = sc * coef_at(&P->sigma[k][0], i, j, n);
        off[k][1] = sc * coef_at(&P->sigma[k][1], i, j, n);
    }
    const double sa = P->sigma_mode == 1 ? sc * coef_at(&P->sigma[0][0], i, j, n) : 0.0;
    double best = INFINITY;
    int32_t arg = -1;
    for (int a = 0; a < P->na; ++a) {
        if (P->sigma_mode == 1) {   /* sigma(x,a) = s(x) a: the column follows the control */
            off[0][0] = sa * P->ctrl[2 * a];
            off[0][1] = sa * P->ctrl[2 * a + 1];
        }
        const double la = cost_of(P, l, a);
        const double f1 = c * P->ctrl[2 * a] + d1;
        const double f2 = c * P->ctrl[2 * a + 1] + d2;
        const double bx = q * f1;
        const double by = q * f2;
        double lam0 = 0.0, rp = 0.0;
        for (int b = 0; b < nb; ++b) {
            double gx = (double)i + bx;
            double gy = (double)j + by;
            if (P->p > 0) {
                const int k = b >> 1;
                if ((b & 1) == 0) { gx = gx + off[k][0]; gy = gy + off[k][1]; }
                else              { gx = gx - off[k][0]; gy = gy - off[k][1]; }
            }
            int64_t cr[4];
            double wg[4];
            bilinear_stencil(n, gx, gy, cr, wg);
            double self_w = 0.0, sum = 0.0;
            for (int t = 0; t < 4; ++t) {
                if (cr[t] == self) self_w = self_w + wg[t];
                else sum = sum + wg[t] * V[cr[t]];
            }
            lam0 = lam0 + w * self_w;
            rp = rp + w * sum;
        }
        double v;
        if (scheme == 0) v = (P->h * la + beta * rp) / (1.0 - beta * lam0);
        else v = P->h * la + beta * (rp + lam0 * V[self]);
        if (v < best) { best = v; arg = a; }
    }
    if (argmin_out) *argmin_out = arg;
    return best;
}

/* Exposed for pin P2: Lambda0(a), R'(a) per control at one node (no discount applied). */
void orc_node_lambdas(const orc_problem *P, const double *V, int i, int j, double *lam0_out,
                      double *rp_out)
{
    const int n = P->n;
    const int64_t self = (int64_t)j * n + i;
    const double q = P->h / P->dx;
    const int nb = P->p > 0 ? 2 * P->p : 1;
    const double w = 1.0 / (double)nb;
    double sc = 0.0;
    if (P->p > 0)
        sc = (P->diffusion_scale == 0 ? sqrt(P->h * (double)P->p) : sqrt(P->h)) / P->dx;
    const double c = coef_at(&P->speed, i, j, n);
    const double d1 = coef_at(&P->drift[0], i, j, n);
    const double d2 = coef_at(&P->drift[1], i, j, n);
    for (int a = 0; a < P->na; ++a) {
        const double bx = q * (c * P->ctrl[2 * a] + d1);
        const double by = q * (c * P->ctrl[2 * a + 1] + d2);
        double lam0 = 0.0, rp = 0.0;
        for (int b = 0; b < nb; ++b) {
            double gx = (double)i + bx, gy = (double)j + by;
            if (P->p > 0) {
                const int k = b >> 1;
                double ox = sc * coef_at(&P->sigma[k][0], i, j, n);
                double oy = sc * coef_at(&P->sigma[k][1], i, j, n);
                if (P->sigma_mode == 1) {
                    const double sa = sc * coef_at(&P->sigma[0][0], i, j, n);
                    ox = sa * P->ctrl[2 * a];
                    oy = sa * P->ctrl[2 * a + 1];
                }
                if ((b & 1) == 0) { gx = gx + ox; gy = gy + oy; }
                else              { gx = gx - ox; gy = gy - oy; }
            }
            int64_t cr[4];
            double wg[4];
            bilinear_stencil(n, gx, gy, cr, wg);
            double self_w = 0.0, sum = 0.0;
            for (int t = 0; t < 4; ++t) {
                if (cr[t] == self) self_w = self_w + wg[t];
                else sum = sum + wg[t] * V[cr[t]];
            }
            lam0 = lam0 + w * self_w;
            rp = rp + w * sum;
        }
        lam0_out[a] = lam0;
        rp_out[a] = rp;
    }
}

/* T(V) on every node (Dirichlet nodes copy V); returns max |T(V) - V| over free nodes. */
double orc_apply(const orc_problem *P, const double *V, double *out, int scheme, int32_t *argmin)
{
    const int n = P->n;
    double res = 0.0;
#pragma omp parallel for schedule(static) reduction(max : res)
    for (int j = 0; j < n; ++j) {
        for (int i = 0; i < n; ++i) {
            const int64_t k = (int64_t)j * n + i;
            if (P->kind[k] != 0) {
                out[k] = V[k];
                if (argmin) argmin[k] = -1;
                continue;
            }
            int32_t a;
            const double v = orc_node_update(P, V, i, j, scheme, &a);
            out[k] = v;
            if (argmin) argmin[k] = a;
            const double d = fabs(v - V[k]);
            if (d > res) res = d;
        }
    }
    return res;
}

/* T(V) at sampled node indices (full-size parity by property). */
void orc_apply_at(const orc_problem *P, const double *V, const int64_t *idx, int64_t m,
                  double *out, int32_t *argmin)
{
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t t = 0; t < m; ++t) {
        const int64_t k = idx[t];
        const int i = (int)(k % P->n), j = (int)(k / P->n);
        int32_t a = -1;
        out[t] = P->kind[k] != 0 ? V[k] : orc_node_update(P, V, i, j, 0, &a);
        if (argmin) argmin[t] = a;
    }
}

/* Jacobi fixed-point iteration u^{m+1} = T(u^m) from the given V (in/out), until the sup-norm
 * change of a sweep is < tol or max_sweeps.  Counts the final (check) sweep.
 * hist (optional, length max_sweeps) receives the per-sweep residuals.  Returns sweeps. */
int64_t orc_jacobi(const orc_problem *P, double *V, double tol, int64_t max_sweeps, int scheme,
                   double *res_out, double *hist)
{
    const int64_t N = (int64_t)P->n * P->n;
    double *W = (double *)malloc(sizeof(double) * (size_t)N);
    if (!W) return -1;
    double *cur = V, *nxt = W;
    int64_t s = 0;
    double res = INFINITY;
    while (s < max_sweeps) {
        res = orc_apply(P, cur, nxt, scheme, NULL);
        if (hist) hist[s] = res;
        ++s;
        double *t = cur; cur = nxt; nxt = t;
        if (res < tol) break;
    }
    if (cur != V) memcpy(V, cur, sizeof(double) * (size_t)N);
    free(W);
    if (res_out) *res_out = res;
    return s;
}

/* Gauss-Seidel sweeps in place following order[0..m) (test-only mode). */
int64_t orc_gauss_seidel(const orc_problem *P, double *V, const int64_t *order, int64_t m,
                         double tol, int64_t max_sweeps, int scheme, double *res_out)
{
    int64_t s = 0;
    double res = INFINITY;
    while (s < max_sweeps) {
        res = 0.0;
        for (int64_t t = 0; t < m; ++t) {
            const int64_t k = order[t];
            if (P->kind[k] != 0) continue;
            const double v = orc_node_update(P, V, (int)(k % P->n), (int)(k / P->n), scheme, NULL);
            const double d = fabs(v - V[k]);
            if (d > res) res = d;
            V[k] = v;
        }
        ++s;
        if (res < tol) break;
    }
    if (res_out) *res_out = res;
    return s;
}

/* Prolongation u_hat = bilinear(u_c) on G.  Fine node (i, j) sits at
 * coarse position (i/r, j/r), r = (n-1)/(n_c-1); coarse cell I = min(i div r, n_c-2), fraction
 * t = (i - I r)/r (exact dyadic for r a power of two); sum in corner order 00, 10, 01, 11. */
static double prolong_one(int nc, const double *uc, int r, int i, int j)
{
    int I = i / r, J = j / r;
    if (I > nc - 2) I = nc - 2;
    if (J > nc - 2) J = nc - 2;
    const double tx = (double)(i - I * r) / (double)r;
    const double ty = (double)(j - J * r) / (double)r;
    const double w00 = (1.0 - tx) * (1.0 - ty), w10 = tx * (1.0 - ty);
    const double w01 = (1.0 - tx) * ty, w11 = tx * ty;
    const int64_t b = (int64_t)J * nc + I;
    double s = w00 * uc[b];
    s = s + w10 * uc[b + 1];
    s = s + w01 * uc[b + nc];
    s = s + w11 * uc[b + nc + 1];
    return s;
}

int orc_prolong(int nc, const double *uc, int n, double *out)
{
    if (nc < 2 || (n - 1) % (nc - 1) != 0) return 1;
    const int r = (n - 1) / (nc - 1);
#pragma omp parallel for schedule(static)
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) out[(int64_t)j * n + i] = prolong_one(nc, uc, r, i, j);
    return 0;
}

/* Discrete synthesis (R16): a*(x_i) = argmin_a [ h l + beta u_hat(x_i + h f(x_i, a)) ]
 * with the plain bilinear value (no self exclusion: it is an evaluation).  sigma = 0 foot.
 * ``uhat_fn`` gives u_hat at a fine node; either a stored array or the coarse field on the fly. */
typedef struct {
    const double *uhat; /* if non-NULL: stored u_hat */
    int nc; const double *uc; int r;
} uhat_src;

static double uhat_at(const uhat_src *U, int n, int64_t k)
{
    if (U->uhat) return U->uhat[k];
    return prolong_one(U->nc, U->uc, U->r, (int)(k % n), (int)(k / n));
}

static int32_t synth_one(const orc_problem *P, const uhat_src *U, int i, int j)
{
    const int n = P->n;
    const double beta = orc_beta(P);
    const double q = P->h / P->dx;
    const double c = coef_at(&P->speed, i, j, n);
    const double d1 = coef_at(&P->drift[0], i, j, n);
    const double d2 = coef_at(&P->drift[1], i, j, n);
    const double l = coef_at(&P->cost, i, j, n);
    double best = INFINITY;
    int32_t arg = -1;
    for (int a = 0; a < P->na; ++a) {
        const double f1 = c * P->ctrl[2 * a] + d1;
        const double f2 = c * P->ctrl[2 * a + 1] + d2;
        const double gx = (double)i + q * f1;
        const double gy = (double)j + q * f2;
        int64_t cr[4];
        double wg[4];
        bilinear_stencil(n, gx, gy, cr, wg);
        double s = wg[0] * uhat_at(U, n, cr[0]);
        s = s + wg[1] * uhat_at(U, n, cr[1]);
        s = s + wg[2] * uhat_at(U, n, cr[2]);
        s = s + wg[3] * uhat_at(U, n, cr[3]);
        const double v = P->h * cost_of(P, l, a) + beta * s;
        if (v < best) { best = v; arg = a; }
    }
    return arg;
}

void orc_synthesize(const orc_problem *P, const double *uhat, uint8_t *astar)
{
    const int n = P->n;
    uhat_src U = {uhat, 0, NULL, 0};
#pragma omp parallel for schedule(static)
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            const int64_t k = (int64_t)j * n + i;
            astar[k] = P->kind[k] != 0 ? 255 : (uint8_t)synth_one(P, &U, i, j);
        }
}

/* Successor of a free node (R18): nearest node to x_i + M f*(x_i)/|f*(x_i)|, in node units,
 * f* = f(x_i, a*(x_i)); round half up (floor(g + 1/2)), clamp to the grid.  |f*| = 0 -> itself
 * (an orphan).  Dirichlet nodes are their own successors. */
static int64_t successor_one(const orc_problem *P, int a, int i, int j, double M)
{
    const int n = P->n;
    const double c = coef_at(&P->speed, i, j, n);
    const double f1 = c * P->ctrl[2 * a] + coef_at(&P->drift[0], i, j, n);
    const double f2 = c * P->ctrl[2 * a + 1] + coef_at(&P->drift[1], i, j, n);
    const double nrm = sqrt(f1 * f1 + f2 * f2);
    if (nrm == 0.0) return (int64_t)j * n + i;
    const double u1 = f1 / nrm, u2 = f2 / nrm;
    const double gx = (double)i + M * u1;
    const double gy = (double)j + M * u2;
    int si = (int)floor(gx + 0.5), sj = (int)floor(gy + 0.5);
    if (si < 0) si = 0;
    if (si > n - 1) si = n - 1;
    if (sj < 0) sj = 0;
    if (sj > n - 1) sj = n - 1;
    return (int64_t)sj * n + si;
}

void orc_successor(const orc_problem *P, const uint8_t *astar, double M, int64_t *succ)
{
    const int n = P->n;
#pragma omp parallel for schedule(static)
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < n; ++i) {
            const int64_t k = (int64_t)j * n + i;
            succ[k] = P->kind[k] != 0 ? k : successor_one(P, astar[k], i, j, M);
        }
}

/* Labels (R17, R18): a free node's patch is the sector Gamma_p of the target node its
 * successor chain reaches; a chain ending on an obstacle, on a free fixed point or in a cycle
 * is an orphan (label n_patches).  Dirichlet nodes: -1 target, -2 obstacle.  Sequential chase
 * with a 3-state memo (unvisited / on the current walk / done). */
int orc_labels(const orc_problem *P, const int64_t *succ, const int32_t *sector, int n_patches,
               int16_t *labels)
{
    const int64_t N = (int64_t)P->n * P->n;
    uint8_t *state = (uint8_t *)calloc((size_t)N, 1);
    int32_t *root = (int32_t *)malloc(sizeof(int32_t) * (size_t)N);
    int64_t *path = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
    if (!state || !root || !path) { free(state); free(root); free(path); return 1; }
    for (int64_t k = 0; k < N; ++k) {
        if (P->kind[k] == 1) { state[k] = 2; root[k] = sector[k]; labels[k] = -1; }
        else if (P->kind[k] == 2) { state[k] = 2; root[k] = n_patches; labels[k] = -2; }
    }
    for (int64_t k = 0; k < N; ++k) {
        if (state[k] == 2) continue;
        int64_t len = 0, x = k;
        int32_t result;
        for (;;) {
            if (state[x] == 2) { result = root[x]; break; }
            if (state[x] == 1) { result = n_patches; break; }   /* cycle */
            state[x] = 1;
            path[len++] = x;
            const int64_t nx = succ[x];
            if (nx == x) { result = n_patches; break; }           /* free fixed point */
            x = nx;
        }
        for (int64_t t = 0; t < len; ++t) {
            state[path[t]] = 2;
            root[path[t]] = result;
            labels[path[t]] = (int16_t)result;
        }
    }
    free(state); free(root); free(path);
    return 0;
}

/* Label of one sampled node with u_hat evaluated from u_c on the fly (full-size parity):
 * chase successors, synthesising a* at every visited node. */
int32_t orc_label_at(const orc_problem *P, int nc, const double *uc, const int32_t *sector,
                     int n_patches, double M, int64_t k, int64_t max_steps)
{
    const int n = P->n;
    uhat_src U = {NULL, nc, uc, (n - 1) / (nc - 1)};
    if (P->kind[k] == 1) return -1;
    if (P->kind[k] == 2) return -2;
    int64_t x = k;
    for (int64_t s = 0; s < max_steps; ++s) {
        if (P->kind[x] == 1) return sector[x];
        if (P->kind[x] == 2) return n_patches;
        const int i = (int)(x % n), j = (int)(x / n);
        const int32_t a = synth_one(P, &U, i, j);
        const int64_t nx = successor_one(P, a, i, j, M);
        if (nx == x) return n_patches;
        x = nx;
    }
    return n_patches; /* longer than max_steps: only a cycle can do that when max_steps >= #nodes */
}

void orc_astar_at(const orc_problem *P, int nc, const double *uc, const int64_t *idx, int64_t m,
                  int32_t *out)
{
    const int n = P->n;
    uhat_src U = {NULL, nc, uc, (n - 1) / (nc - 1)};
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t t = 0; t < m; ++t) {
        const int64_t k = idx[t];
        out[t] = P->kind[k] != 0 ? 255 : synth_one(P, &U, (int)(k % n), (int)(k / n));
    }
}

void orc_uhat_at(int n, int nc, const double *uc, const int64_t *idx, int64_t m, double *out)
{
    const int r = (n - 1) / (nc - 1);
    for (int64_t t = 0; t < m; ++t)
        out[t] = prolong_one(nc, uc, r, (int)(idx[t] % n), (int)(idx[t] / n));
}

/* Static equal squares (R19): block boundaries floor(k n / P); label = by*px + bx;
 * Dirichlet nodes -1 (target) / -2 (obstacle). */
void orc_static_labels(int n, int px, int py, const uint8_t *kind, int16_t *labels)
{
    for (int j = 0; j < n; ++j) {
        int by = 0;
        while (by + 1 < py && (int64_t)(by + 1) * n / py <= j) ++by;
        for (int i = 0; i < n; ++i) {
            int bx = 0;
            while (bx + 1 < px && (int64_t)(bx + 1) * n / px <= i) ++bx;
            const int64_t k = (int64_t)j * n + i;
            labels[k] = kind[k] == 1 ? -1 : kind[k] == 2 ? -2 : (int16_t)(by * px + bx);
        }
    }
}

/* Fuzzy patches of the paper (reading R38).
 * phi_p = chi_{Gamma_p} on the Dirichlet set (target node of sector p: 1, any other Dirichlet
 * node: 0), 0 on free nodes; then the semi-Lagrangian advection scheme Eq. (discrete-advection)
 *     phi_p(x_i) = phi_p(x_i + h f(x_i, a*(x_i)))        (bilinear, sigma = 0 foot, clamped)
 * iterated for all p at once by Jacobi (every node from the previous iterate) until the sup-norm
 * change of a sweep is < eps_P (the paper's "poor tolerance"); the count includes that sweep.
 * Canonical arithmetic (R30): the foot is the synthesis foot f = c a + d, g = i + q f, and the
 * value w00 v00 + w10 v10 + w01 v01 + w11 v11 summed in that order.  phi: n_patches * N
 * (patch-major).  Returns the number of sweeps (max_sweeps if not converged). */
int64_t orc_fuzzy_phi(const orc_problem *P, const uint8_t *astar, const int32_t *sector,
                      int n_patches, double eps_P, int64_t max_sweeps, double *phi,
                      double *residual_out)
{
    const int n = P->n;
    const int64_t N = (int64_t)n * n;
    const double q = P->h / P->dx;
    double *cur = phi;
    double *nxt = (double *)malloc(sizeof(double) * (size_t)N * (size_t)n_patches);
    for (int p = 0; p < n_patches; ++p)
        for (int64_t k = 0; k < N; ++k)
            cur[(int64_t)p * N + k] = (P->kind[k] == 1 && sector[k] == p) ? 1.0 : 0.0;
    int64_t s = 0;
    double res = INFINITY;
    while (s < max_sweeps) {
        res = 0.0;
#pragma omp parallel for schedule(static) reduction(max : res)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                const int64_t k = (int64_t)j * n + i;
                if (P->kind[k] != 0) {
                    for (int p = 0; p < n_patches; ++p) nxt[(int64_t)p * N + k] = cur[(int64_t)p * N + k];
                    continue;
                }
                const int a = astar[k];
                const double c = coef_at(&P->speed, i, j, n);
                const double f1 = c * P->ctrl[2 * a] + coef_at(&P->drift[0], i, j, n);
                const double f2 = c * P->ctrl[2 * a + 1] + coef_at(&P->drift[1], i, j, n);
                int64_t cr[4];
                double wg[4];
                bilinear_stencil(n, (double)i + q * f1, (double)j + q * f2, cr, wg);
                for (int p = 0; p < n_patches; ++p) {
                    const double *F = cur + (int64_t)p * N;
                    double v = wg[0] * F[cr[0]];
                    v = v + wg[1] * F[cr[1]];
                    v = v + wg[2] * F[cr[2]];
                    v = v + wg[3] * F[cr[3]];
                    nxt[(int64_t)p * N + k] = v;
                    const double d = fabs(v - F[k]);
                    if (d > res) res = d;
                }
            }
        double *t = cur; cur = nxt; nxt = t;
        ++s;
        if (res < eps_P) break;
    }
    if (cur != phi) {
        memcpy(phi, cur, sizeof(double) * (size_t)N * (size_t)n_patches);
        nxt = cur;
    }
    free(nxt);
    if (residual_out) *residual_out = res;
    return s;
}

/* Thresholding and ownership (reading R38): Omega_p = {phi_p >= tau_P}; the owner of
 * a free node is the patch of largest phi_p (lowest p on ties) -- it is a member of Omega_p
 * whenever any patch is; no positive phi_p at all -> orphan label n_patches.  Target -1,
 * obstacle -2.  members (optional): number of patches with phi_p >= tau_P (overlap degree). */
void orc_fuzzy_assign(const orc_problem *P, const double *phi, int n_patches, double tau_P,
                      int16_t *labels, uint8_t *members)
{
    const int64_t N = (int64_t)P->n * P->n;
    for (int64_t k = 0; k < N; ++k) {
        if (P->kind[k] != 0) {
            labels[k] = P->kind[k] == 1 ? -1 : -2;
            if (members) members[k] = 0;
            continue;
        }
        int best = -1, cnt = 0;
        double bv = 0.0;
        for (int p = 0; p < n_patches; ++p) {
            const double v = phi[(int64_t)p * N + k];
            if (v >= tau_P) ++cnt;
            if (v > bv) { bv = v; best = p; }
        }
        labels[k] = (int16_t)(best < 0 ? n_patches : best);
        if (members) members[k] = (uint8_t)(cnt > 255 ? 255 : cnt);
    }
}

/* Sparse form of the fuzzy patches ("per-node top-K (label, mass)"; the
 * paper's construction P:777-803 with hundreds of patches, reading R40).  Every node keeps at most
 * K pairs (p, phi_p): the K largest phi_p of the node (ties: lower p first), stored in that order;
 * a patch that is not listed has phi_p = 0 there.  One Jacobi sweep of the same advection scheme
 *     phi_p(x_i) = w00 phi_p(c00) + w10 phi_p(c10) + w01 phi_p(c01) + w11 phi_p(c11)
 * merges the lists of the four corners IN THE ORDER 00, 10, 01, 11 (a label's partial sums are
 * added in corner order, exactly the dense expression with its zero terms left out), drops the
 * labels whose sum is 0 and keeps the K largest.  With K >= the number of patches that reach a
 * node this IS the dense iteration (same bits); a smaller K truncates the smallest memberships
 * (the dropped mass is reported by orc_fuzzy_sparse_assign).  The sweep change is the largest
 * |new phi_p - old phi_p| over the labels listed before or after; iteration stops at the first
 * sweep with change < eps_P.  lab / mass: N * K (node-major; empty slot: label -1, mass 0). */
static void sparse_insert_topk(int K, int16_t *ol, double *om, int *cnt, int16_t l, double m)
{
    /* insertion into a list sorted by (mass descending, label ascending), capacity K */
    int pos = *cnt;
    while (pos > 0 && (om[pos - 1] < m || (om[pos - 1] == m && ol[pos - 1] > l))) --pos;
    if (pos >= K) return;
    const int last = *cnt < K ? *cnt : K - 1;
    for (int s = last; s > pos; --s) { ol[s] = ol[s - 1]; om[s] = om[s - 1]; }
    ol[pos] = l;
    om[pos] = m;
    if (*cnt < K) ++*cnt;
}

int64_t orc_fuzzy_sparse(const orc_problem *P, const uint8_t *astar, const int32_t *sector,
                         int n_patches, int K, double eps_P, int64_t max_sweeps, int16_t *lab,
                         double *mass, double *residual_out)
{
    const int n = P->n;
    const int64_t N = (int64_t)n * n;
    const double q = P->h / P->dx;
    if (K < 1 || K > 16) return -1;
    int16_t *clab = lab, *nlab = (int16_t *)malloc(sizeof(int16_t) * (size_t)N * K);
    double *cm = mass, *nm = (double *)malloc(sizeof(double) * (size_t)N * K);
    for (int64_t k = 0; k < N; ++k)
        for (int s = 0; s < K; ++s) {
            const int on = s == 0 && P->kind[k] == 1 && sector[k] >= 0 && sector[k] < n_patches;
            clab[k * K + s] = on ? (int16_t)sector[k] : (int16_t)-1;
            cm[k * K + s] = on ? 1.0 : 0.0;
        }
    int64_t sw = 0;
    double res = INFINITY;
    while (sw < max_sweeps) {
        res = 0.0;
#pragma omp parallel for schedule(static) reduction(max : res)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                const int64_t k = (int64_t)j * n + i;
                if (P->kind[k] != 0) {
                    for (int s = 0; s < K; ++s) { nlab[k * K + s] = clab[k * K + s]; nm[k * K + s] = cm[k * K + s]; }
                    continue;
                }
                const int a = astar[k];
                const double c = coef_at(&P->speed, i, j, n);
                const double f1 = c * P->ctrl[2 * a] + coef_at(&P->drift[0], i, j, n);
                const double f2 = c * P->ctrl[2 * a + 1] + coef_at(&P->drift[1], i, j, n);
                int64_t cr[4];
                double wg[4];
                bilinear_stencil(n, (double)i + q * f1, (double)j + q * f2, cr, wg);
                int16_t al[64];
                double am[64];
                int na = 0;
                for (int t = 0; t < 4; ++t)            /* corner order 00, 10, 01, 11 */
                    for (int s = 0; s < K; ++s) {
                        const int16_t l = clab[cr[t] * K + s];
                        if (l < 0) continue;
                        const double term = wg[t] * cm[cr[t] * K + s];
                        int idx = 0;
                        while (idx < na && al[idx] != l) ++idx;
                        if (idx < na) am[idx] = am[idx] + term;
                        else { al[na] = l; am[na] = term; ++na; }
                    }
                int16_t ol[16];
                double om[16];
                int cnt = 0;
                for (int idx = 0; idx < na; ++idx)
                    if (am[idx] > 0.0) sparse_insert_topk(K, ol, om, &cnt, al[idx], am[idx]);
                /* change of the sweep over the labels listed before or after */
                for (int s = 0; s < cnt; ++s) {
                    double old = 0.0;
                    for (int u = 0; u < K; ++u)
                        if (clab[k * K + u] == ol[s]) old = cm[k * K + u];
                    const double d = fabs(om[s] - old);
                    if (d > res) res = d;
                }
                for (int u = 0; u < K; ++u) {
                    const int16_t l = clab[k * K + u];
                    if (l < 0) continue;
                    int found = 0;
                    for (int s = 0; s < cnt; ++s) found |= ol[s] == l;
                    if (!found && cm[k * K + u] > res) res = cm[k * K + u];
                }
                for (int s = 0; s < K; ++s) {
                    nlab[k * K + s] = s < cnt ? ol[s] : (int16_t)-1;
                    nm[k * K + s] = s < cnt ? om[s] : 0.0;
                }
            }
        { int16_t *t = clab; clab = nlab; nlab = t; }
        { double *t = cm; cm = nm; nm = t; }
        ++sw;
        if (res < eps_P) break;
    }
    if (clab != lab) {
        memcpy(lab, clab, sizeof(int16_t) * (size_t)N * K);
        memcpy(mass, cm, sizeof(double) * (size_t)N * K);
        nlab = clab;
        nm = cm;
    }
    free(nlab);
    free(nm);
    if (residual_out) *residual_out = res;
    return sw;
}

/* Ownership from the sparse lists (same rule as orc_fuzzy_assign): owner = the first listed patch
 * (largest phi_p, lowest p on ties), orphan n_patches when the list is empty; members = listed
 * patches with phi_p >= tau_P. */
void orc_fuzzy_sparse_assign(const orc_problem *P, const int16_t *lab, const double *mass, int K,
                             int n_patches, double tau_P, int16_t *labels, uint8_t *members)
{
    const int64_t N = (int64_t)P->n * P->n;
    for (int64_t k = 0; k < N; ++k) {
        if (P->kind[k] != 0) {
            labels[k] = P->kind[k] == 1 ? -1 : -2;
            if (members) members[k] = 0;
            continue;
        }
        int cnt = 0;
        for (int s = 0; s < K; ++s)
            if (lab[k * K + s] >= 0 && mass[k * K + s] >= tau_P) ++cnt;
        labels[k] = (int16_t)(lab[k * K] >= 0 ? lab[k * K] : n_patches);
        if (members) members[k] = (uint8_t)cnt;
    }
}
