/*
 * pdd.h -- C ABI of libpdd: the B200 (sm_100a) hot path of the patchy domain decomposition
 * method for stationary second-order HJB equations, arXiv 1502.01629.
 *
 * Citations: P:<line> = the paper's LaTeX source, R<k> = a reading of the paper
 * listed in DESIGN.md section "Readings".
 *
 * The calls follow the paper's algorithm:
 *   Initialization   pdd_create          grid G, coarse grid G_c, controls, data
 *   Pre-computation  pdd_coarse_solve    u_c on G_c, sigma = 0, until eps_c
 *                    pdd_synthesize      u_hat = interp(u_c) on G, feedback a*        P:826-827
 *                    pdd_build_patches   split of the Dirichlet set + patches
 *                    pdd_build_fuzzy_patches[_sparse]  the paper's fuzzy patches
 *                    pdd_build_static    static equal-square decomposition (DD)
 *   Computation      pdd_solve           patch-parallel fine solve until eps
 *                    pdd_get_*           fetch V, a*, labels, u_hat, u_c
 *
 * The scheme (P:366-375 with the self-dependency removal P:433-491, discounted as in
 * BASELINE.json, R1-R3): for a free node x_i,
 *   V(x_i) = min_k ( h l(x_i, a_k) + beta R'_k ) / ( 1 - beta Lambda0_k ),  beta = 1/(1 + lambda h),
 * foot points x_i + h f(x_i, a_k) +- sqrt(h p) sigma_j(x_i, a_k) (j < p; one foot point when
 * p = 0; sigma_j depends on a_k only with sigma_mode 1),
 * f(x, a) = c(x) a + d(x); R'_k / Lambda0_k = branch-averaged bilinear weight of the corners
 * other than x_i / of x_i itself; feet are clamped to the box (R5).  Target nodes hold V = 0,
 * obstacle nodes V = 1/lambda (R8).
 *
 * Conventions
 *   - Grid: n nodes per axis on [lo, hi]^2, dx = (hi - lo)/(n - 1), node (i, j) at
 *     (lo + i dx, lo + j dx), linear index j*n + i (x fastest), row-major.
 *   - All host arrays passed to pdd_create are COPIED to the device inside the call; the caller
 *     keeps ownership and may free them when the call returns.
 *   - The device workspace is owned by the caller (e.g. a PyTorch uint8 tensor) and must stay
 *     alive until pdd_destroy.  libpdd never calls cudaMalloc.
 *   - Every call runs on the device that owns the workspace given to pdd_create, whatever device
 *     the calling thread has current, and restores the caller's current device on return.
 *   - Every call enqueues its work on the stream given to pdd_create and synchronises that
 *     stream before returning, so returned statistics and fetched arrays are final.
 *   - Errors: every call returns a pdd_status; the message is in pdd_last_error(ctx)
 *     (pdd_last_error(NULL) for pdd_create / pdd_workspace_bytes failures).  No C++ exception
 *     crosses the ABI.  On PDD_E_CUDA the context must be destroyed.
 */
#ifndef PDD_H
#define PDD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    PDD_OK = 0,
    PDD_E_INVALID = 1,    /* bad argument: n < 3, hi <= lo, N_A outside 1..128, p outside 0..2,
                             lambda < 0, obstacles with lambda = 0, l <= 0, sigma_mode 1 with
                             p != 1, sizes that do not nest, NULL pointers */
    PDD_E_NOCONVERGE = 2, /* max rounds / sweeps reached; values stay fetchable */
    PDD_E_IO = 3,         /* reserved */
    PDD_E_CUDA = 4,       /* a CUDA call failed; see pdd_last_error */
    PDD_E_STATE = 5,      /* call out of order (e.g. synthesize before coarse_solve) */
    PDD_E_NOMEM = 6,      /* workspace smaller than pdd_workspace_bytes */
    PDD_E_STENCIL = 7     /* foot points reach farther than the tile halo supports (R4) */
} pdd_status;

typedef enum {
    PDD_COEF_CONST = 0,   /* value                                   */
    PDD_COEF_ROW = 1,     /* data[j], depends on x2 only (n values)   */
    PDD_COEF_COL = 2,     /* data[i], depends on x1 only (n values)   */
    PDD_COEF_FIELD = 3    /* data[j*n + i] (n*n values)                */
} pdd_coef_kind;

/* A coefficient of the problem (Eq. HJB2). data: host pointer, fp64. */
typedef struct {
    int32_t kind;
    double value;
    const double *data;
} pdd_coef;

/* One discretised problem on one grid (fine G or coarse G_c).  All pointers are HOST pointers. */
typedef struct {
    int32_t n;              /* nodes per axis, >= 3                                         */
    double lo, hi;          /* square box [lo, hi]^2                                        */
    double dx;              /* (hi - lo)/(n - 1), given explicitly (both sides use this value) */
    double h;               /* time step of the SL scheme (R13: h = dx in BASELINE configs) */
    double lambda;          /* discount >= 0; beta = 1/(1 + lambda h).  lambda = 0: the paper's
                               exit-time problems (g = 0 on target nodes, e.g. the
                               boundary ring); V starts at 1e6 (R11), no obstacles */
    int32_t n_controls;     /* N_A, 1..128                                      */
    const double *controls; /* 2*N_A values (a1, a2) per control                            */
    pdd_coef speed;         /* c(x)                                                         */
    pdd_coef drift[2];      /* d(x) = (d1, d2)                                              */
    int32_t p;              /* noise columns 0..2; 2p Markov branches (1 foot when p = 0)  */
    pdd_coef sigma[2][2];   /* sigma_j(x) component c = sigma[j][c]                          */
    pdd_coef cost;          /* l(x) > 0                                                     */
    int32_t diffusion_scale;/* 0: sqrt(h p) (north star), 1: sqrt(h)                */
    const uint8_t *kind;    /* n*n: 0 free, 1 target (V = 0), 2 obstacle (V = 1/lambda)     */
    const int16_t *sector;  /* n*n: Gamma_p id of target nodes (R17), ignored elsewhere; may be
                               NULL on the coarse grid or when no patches are built           */
    /* General nonlinear terms (readings R32, R33):                     */
    int32_t sigma_mode;     /* 0: noise columns sigma_j(x) as above; 1: ONE column along the
                               control, sigma(x, a) = s(x) a with s = sigma[0][0] (p must be 1;
                               the paper's sigma_3(x,a) = d_eps(x) a)                         */
    const double *cost_ctrl;/* N_A values m(a_k) or NULL: running cost l(x, a_k) = l(x) + m(a_k)
                               (the paper's l_3); l(x) + min m must stay > 0                  */
} pdd_problem;

typedef struct pdd_ctx pdd_ctx;

/* Fine solve options (pdd_solve). */
typedef struct {
    int32_t mode;        /* 0 patchy: V starts at u_hat, tiles activated in ascending u_hat
                            order; 1 static: V starts at V0 (R11)         */
    int32_t k_inner;     /* in-tile Gauss-Seidel sweeps per tile visit (>= 1; 0 = automatic:
                            1 patchy, 4 static, and 4 for a patchy general-stencil grid whose
                            tiles fit in about one wave of sweep CTAs -- on such grids the
                            u_hat front is off when delta = 0).  Patchy tiles sweep first in their downstream orientation
                            (the signs of u_hat's differences over the tile); incoherent tiles
                            continue an orientation cycle across visits                     */
    double tol;          /* sup-norm residual tolerance eps                                  */
    int64_t max_rounds;  /* cap on tile rounds (schedule 2: on the average number of visits
                            per tile with free nodes)                                      */
    double delta;        /* patchy bucket width in value units; 0 = automatic; < 0 = off      */
    int32_t kernel;      /* 0 auto, 1 general stencil, 2 row-table stencil, 3 row-table one
                            node per warp step (A/B only), 4 lean general stencil.  The
                            fp32 row-table kernel's tile is 32 x 64 nodes, 16 x 64 for patchy
                            solves on grids of up to 16 k tiles, 16 x 128 for static solves
                            where 128 dx <= 1/8 (pdd_set_tile_shape
                            forces one geometry)                                             */
    int32_t schedule;    /* 0 automatic (= 2);
                            1 ordered: Gauss-Seidel passes over the tiles in key order (u_hat
                            for patchy, block-lexicographic for static), each tile waiting for
                            its lower-key neighbours (delta = key slack);
                            2 queue: one persistent launch whose CTAs take dirty tiles from a
                            work queue, visit them (an in-tile Gauss-Seidel solve) and mark the
                            neighbours of changed tiles dirty -- asynchronous relaxation, no
                            rounds; patchy admits tiles in min-u_hat order:
                            a tile that converges admits the next one, so that about
                            queue_target tiles are queued or being visited; a full-grid
                            verification pass re-seeds the queue if needed;
                            3 rounds: rounds over the list of active tiles (one launch per
                            round); patchy admits tiles in buckets of min u_hat of width
                            delta                                                            */
    int32_t early_exit_off; /* 1: every tile visit does all k_inner sweeps (A/B; default 0: a
                            visit stops after the first sweep changing no node by >= tol)   */
    int32_t bucket_policy;  /* patchy, schedule 3: 0 moving front (the threshold advances every
                            round, faster while a round under-fills the GPU); 1 classic
                            Delta-stepping (a bucket opens once the previous one settled); 2
                            upstream-ready (no front: a tile waits for unconverged neighbours
                            with min u_hat lower by more than delta)                        */
    int32_t trace;       /* > 0: one line per round on stderr (one round per batch)          */
    int32_t queue_target; /* schedule 2, patchy: tiles kept queued or visiting; 0 = automatic
                            (two waves of resident sweep CTAs)                             */
} pdd_solve_opts;

typedef struct {
    int64_t rounds;            /* tile rounds, including verification passes   */
    int64_t node_updates;      /* free-node updates performed by the sweep kernel           */
    int64_t tiles_processed;
    int64_t verify_passes;
    double final_residual;     /* last full-grid Jacobi residual ||T(V) - V||_inf            */
    double apost_bound;        /* final_residual / (1 - beta): bound on ||V - V*||_inf; NaN
                                  for exit problems (lambda = 0, beta = 1: no such bound)   */
    double seconds_total;      /* wall time of pdd_solve on the stream (CUDA events)        */
    double seconds_sweep;      /* summed duration of the sweep-kernel launches (events)      */
    double seconds_verify;
    int32_t converged;
    int32_t n_tiles;
    int32_t kernel_used;       /* 1 general, 2 row-table (fp64 / one node per step), 3 fp32
                                  row-table four nodes per step                           */
    int32_t patches_active;    /* patches holding free nodes (each had an active tile)      */
    int32_t patches_converged; /* patches whose own residual max_{x_i in patch} |T(V) - V|
                                  in the last verification pass is < tol (
                                  pdd_get_patch_residuals)                                */
    int32_t tile_cols, tile_rows, tiles_x;   /* tile geometry of the solve (tile t covers
                                  columns (t % tiles_x) tile_cols.., rows (t / tiles_x) tile_rows..) */
} pdd_solve_stats;

typedef struct {
    int64_t sweeps;       /* Jacobi sweeps including the final check sweep                 */
    double residual;      /* residual of the last sweep                                    */
    double seconds;
    int32_t converged;
    int32_t reserved;
} pdd_coarse_stats;

const char *pdd_version(void);

/* Bytes of device workspace pdd_create needs for this (fine, coarse) pair at this precision
 * (32 or 64: the arithmetic of the fine sweep; V is stored in fp64 in both).  coarse may be NULL. */
pdd_status pdd_workspace_bytes(const pdd_problem *fine, const pdd_problem *coarse,
                               int32_t precision, size_t *bytes);

/* Validate the problem, carve the workspace, copy every input array to the device.
 * stream: a cudaStream_t (NULL = legacy default stream).  device_workspace: >= the size
 * reported by pdd_workspace_bytes, 256-byte aligned. */
pdd_status pdd_create(const pdd_problem *fine, const pdd_problem *coarse, int32_t precision,
                      void *stream, void *device_workspace, size_t workspace_bytes,
                      pdd_ctx **out);

/* u_c: Jacobi fixed point of the scheme with sigma = 0 on G_c from V0, stopped at the first
 * sweep whose residual is < tol_c (R14).  Canonical fp64 arithmetic (R30), so u_c
 * is bit-identical to any IEEE implementation of the same expressions.  Needs a coarse problem. */
pdd_status pdd_coarse_solve(pdd_ctx *ctx, double tol_c, int64_t max_sweeps, pdd_coarse_stats *st);

/* u_hat = bilinear(u_c) on G (R15) and a*(x_i) = argmin_k [h l + beta u_hat(x_i +
 * h f(x_i, a_k))], lowest k on ties (R16).  Canonical fp64. */
pdd_status pdd_synthesize(pdd_ctx *ctx);

/* Patch labels (R17, R18): successor s(i) = nearest node to x_i + M f* / |f*| (cells), pointer
 * jumping to the root of every successor chain; label = sector[root] when the root is a target
 * node, n_patches (orphan) otherwise; -1 on target nodes, -2 on obstacles.  M = 0 => 4. */
pdd_status pdd_build_patches(pdd_ctx *ctx, int32_t n_patches, double M);

/* The paper's own patch construction (reading R38): phi_p = chi_{Gamma_p} advected
 * along the synthesised feedback by the semi-Lagrangian scheme phi_p(x_i) = phi_p(x_i + h f(x_i,
 * a*(x_i))) (Eq. discrete-advection; sigma = 0 foot, bilinear, canonical fp64, Jacobi for all
 * patches at once) until the sweep change is < eps_P (the paper's "poor tolerance"); then
 * Omega_p = {phi_p >= tau_P} and the owner of a node is the patch of largest phi_p (lowest p on
 * ties), orphan n_patches when every phi_p is 0; -1 target, -2 obstacle.  Replaces the labels of
 * pdd_build_patches (a patchy pdd_solve then reports per-patch rounds for these patches).
 * scratch: caller-owned DEVICE memory of >= pdd_fuzzy_scratch_bytes(n, n_patches) bytes (two
 * patch-major fields n_patches x n*n fp64, i.e. 16 n_patches n^2 bytes: the paper's few-patch
 * decompositions; the successor labels of pdd_build_patches scale to hundreds of patches); on
 * return the final phi starts at scratch + st->phi_offset.  Needs pdd_synthesize. */
typedef struct {
    int64_t sweeps;        /* Jacobi sweeps including the last (converged) one                 */
    double residual;       /* change of the last sweep                                         */
    double seconds;
    int32_t converged;
    int32_t overlap_nodes; /* free nodes in >= 2 patches Omega_p (phi_p >= tau_P)              */
    int64_t phi_offset;    /* byte offset of the final phi fields (sparse: the masses, n*n*K
                              doubles) inside scratch                                          */
    int64_t lab_offset;    /* sparse form: byte offset of the final patch lists (n*n*K int16)  */
    int32_t max_list;      /* sparse form: longest per-node list (== K: memberships may have
                              been truncated)                                                  */
    int32_t reserved;
} pdd_fuzzy_stats;
pdd_status pdd_fuzzy_scratch_bytes(int32_t n, int32_t n_patches, size_t *bytes);
pdd_status pdd_build_fuzzy_patches(pdd_ctx *ctx, int32_t n_patches, double eps_P, double tau_P,
                                   int64_t max_sweeps, void *scratch, size_t scratch_bytes,
                                   pdd_fuzzy_stats *st);

/* The same construction in sparse form for decompositions with hundreds of patches (SURVEY.md
 * 8(f) NEXT #2, reading R40): every node keeps its K largest (patch, phi_p) pairs, sorted by
 * (phi_p descending, patch ascending), node-major, empty slots (-1, 0) last; a Jacobi sweep merges
 * the lists of the foot's four corners in the order 00, 10, 01, 11 and keeps the K largest sums.
 * With K >= the number of patches that reach a node the lists hold the dense phi bit for bit; a
 * smaller K drops the smallest memberships (st->max_list == K flags that this may have happened).
 * Owner = first listed patch, orphan n_patches for an empty list; overlap_nodes counts free nodes
 * with >= 2 listed patches of phi_p >= tau_P.  K in {1, 2, 3, 4, 6, 8, 16}.  scratch: DEVICE
 * memory of >= pdd_fuzzy_sparse_scratch_bytes(n, K) bytes (20 K n^2 + 512). */
pdd_status pdd_fuzzy_sparse_scratch_bytes(int32_t n, int32_t K, size_t *bytes);
pdd_status pdd_build_fuzzy_patches_sparse(pdd_ctx *ctx, int32_t n_patches, int32_t K, double eps_P,
                                          double tau_P, int64_t max_sweeps, void *scratch,
                                          size_t scratch_bytes, pdd_fuzzy_stats *st);

/* Static equal squares: px columns x py rows, boundaries floor(k n / P) (R19). */
pdd_status pdd_build_static(pdd_ctx *ctx, int32_t px, int32_t py);

/* The fine solve: tile visits (in-tile Gauss-Seidel sweeps of the scheme) scheduled by
 * opts->schedule -- by default one persistent launch whose CTAs take dirty tiles from a work
 * queue -- until no tile is dirty, then a full-grid Jacobi verification that also
 * records every patch's own residual; offending tiles are re-queued and the solve continues
 * while the verification residual is >= tol.  Returns PDD_E_NOCONVERGE (statistics still
 * written) when max_rounds is exhausted or the residual stagnates above tol (a tolerance below
 * the arithmetic's noise floor).  mode 0 needs pdd_synthesize and pdd_build_patches (or one of
 * the fuzzy-patch builders), mode 1 needs pdd_build_static. */
pdd_status pdd_solve(pdd_ctx *ctx, const pdd_solve_opts *opts, pdd_solve_stats *st);

/* One application of the operator: out = T(V) on every node (Dirichlet nodes copy V), fp64
 * output, arithmetic of the context's precision; *residual = max |T(V) - V| over free nodes.
 * out: DEVICE memory (n*n doubles) or NULL (residual only).  kernel: as pdd_solve_opts.kernel. */
pdd_status pdd_apply_operator(pdd_ctx *ctx, double *out, int32_t kernel, double *residual);

/* Fetch / set arrays (n*n unless noted).  *_on_device selects device (1) or host (0) memory. */
pdd_status pdd_get_values(pdd_ctx *ctx, void *dst, int32_t dst_on_device, int32_t as_fp64);
pdd_status pdd_set_values(pdd_ctx *ctx, const double *src, int32_t src_on_device);
pdd_status pdd_get_uhat(pdd_ctx *ctx, double *dst, int32_t dst_on_device);
pdd_status pdd_get_coarse_values(pdd_ctx *ctx, double *dst, int32_t dst_on_device); /* n_c^2 */
pdd_status pdd_get_controls(pdd_ctx *ctx, uint8_t *dst, int32_t dst_on_device);  /* 255: Dirichlet */
pdd_status pdd_get_labels(pdd_ctx *ctx, int16_t *dst, int32_t dst_on_device);
pdd_status pdd_get_successors(pdd_ctx *ctx, int32_t *dst, int32_t dst_on_device);

/* Per-patch convergence report of the last pdd_solve (each patch iterates until its
 * own sup-norm residual is below tol).  n_patches + 1 entries (the last one = orphans); dst is
 * HOST memory; count is clipped to n_patches + 1.
 *   pdd_get_patch_rounds:    activation trace: the last round in which a tile holding free nodes
 *                            of the patch was active (-1: never) = max over those tiles of
 *                            pdd_get_tile_rounds
 *   pdd_get_patch_residuals: max over the patch's free nodes of |T(V) - V| in the last full-grid
 *                            verification pass (the kernel's arithmetic), 0 for an empty patch
 *   pdd_get_tile_rounds:     per tile (pdd_solve_stats.n_tiles, geometry tile_cols x tile_rows)
 *                            the last round that activated it (-1: never); PDD_E_STATE before
 *                            the first pdd_solve. */
pdd_status pdd_get_patch_rounds(pdd_ctx *ctx, int32_t *dst, int32_t count);
pdd_status pdd_get_patch_residuals(pdd_ctx *ctx, double *dst, int32_t count);
pdd_status pdd_get_tile_rounds(pdd_ctx *ctx, int32_t *dst, int32_t count);

/* Force the fp32 row-table kernel's tile geometry for the following solves / operator
 * applications: rows x cols = 0 x 0 automatic (16 x 64 for patchy solves on
 * grids of up to 16 k tiles, 16 x 128 for static solves where 128 dx <= 1/8, else 32 x 64), or
 * 32 x 64, 16 x 128, 16 x 64.  For A/B measurements and the forced-geometry parity tests;
 * PDD_E_INVALID for any other value.  pdd_set_tile_cols(cols): 0, 64 (32 x 64) or 128 (16 x 128). */
pdd_status pdd_set_tile_shape(pdd_ctx *ctx, int32_t rows, int32_t cols);
/* The automatic choice above for a fine grid of n nodes per side on [lo, hi]^2 (host arithmetic,
 * no context, no GPU): rows x cols of the fp32 row-table kernel's tile for a patchy (1) or static
 * (0) solve. */
pdd_status pdd_choose_tile_shape(int32_t n, double lo, double hi, int32_t patchy, int32_t *rows,
                                 int32_t *cols);
pdd_status pdd_set_tile_cols(pdd_ctx *ctx, int32_t cols);

/* The upwind diffusion ball analysis of P:528-697 (host arithmetic, no context, no GPU).
 * Inputs: f_min, f_max = min / max of |f(x,a)| over Omega x A (> 0), sigma_norm = ||sigma||_inf
 * (the longest diffusion row; sqrt(2 eps) for sigma = sqrt(2 eps) I), dx.
 *   omega     = f_min / sigma_norm^2                      (+inf when sigma = 0)
 *   upsilon   = f_max / f_min
 *   alpha_lo  = 1 / (omega dx)                            Eq. (lower-alpha)
 *   alpha_hi  = 1/upsilon - (sqrt(1 + 4 omega dx upsilon) - 1) / (2 omega dx upsilon^2)
 *                                                         Eq. (upper-alpha)
 *   tau_dx    = dx / (1 + upsilon);  hyperbolic = 1/omega < tau_dx   Eq. (hyperbolicity)
 *               (equality, up to 1e-12 relative, counts as not hyperbolic: reading R37)
 *   alpha     = 1/(1 + upsilon) when hyperbolic, else 0.99 alpha_hi (the paper keeps
 *               the upper bound and gives up the lower one; reading R36)
 *   h         = alpha dx / f_min
 *   eps_threshold = f_min dx / (2 (1 + upsilon)): the eps below which sigma = sqrt(2 eps) I is
 *               hyperbolic (dx/4 for the eikonal equation, dx/120 for Zermelo
 *               P:1240-1244). */
typedef struct {
    double omega, upsilon, alpha_lo, alpha_hi, alpha, h, tau_dx, eps_threshold;
    int32_t hyperbolic;
    int32_t reserved;
} pdd_regime;
pdd_status pdd_regime_analyse(double f_min, double f_max, double sigma_norm, double dx,
                              pdd_regime *out);

/* Measurement aid (the roofline denominators are measured on the box, not taken
 * from a data sheet).  Runs two micro-benchmarks on the current device and `stream`:
 *   fp32_tflops: dependent-free FFMA chains (8 per thread, every SM full): 2 flop per FFMA lane;
 *   smem_tbs:    conflict-free 16-byte shared-memory loads (LDS.128) from every warp of every SM;
 *   fp64_tflops: the same chains with DFMA.
 * Each is the best of `reps` launches timed with CUDA events (any output may be NULL).  Not part
 * of the hot path. */
pdd_status pdd_measure_alu_peaks(void *stream, int32_t reps, double *fp32_tflops, double *smem_tbs,
                                 double *fp64_tflops);

/* Number of kernels this context has enqueued since pdd_create (all calls). */
long long pdd_kernel_launches(const pdd_ctx *ctx);

const char *pdd_last_error(const pdd_ctx *ctx);
void pdd_destroy(pdd_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* PDD_H */
