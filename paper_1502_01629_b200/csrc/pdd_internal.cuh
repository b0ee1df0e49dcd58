// pdd_internal.cuh -- device-side problem description and launch wrappers shared by the
// libpdd translation units (runtime.cu, canonical.cu, sweep.cu).  Product code only; nothing
// here is shared with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pdd {

// A coefficient on the device: CONST value, ROW (x2) / COL (x1) table, or n*n FIELD.
struct DCoef {
    int kind;
    double value;
    const double *data;
};

__host__ __device__ __forceinline__ double coef_at(const DCoef &c, int i, int j, int n)
{
    switch (c.kind) {
    case 0: return c.value;
    case 1: return c.data[j];
    case 2: return c.data[i];
    default: return c.data[(int64_t)j * n + i];
    }
}

// One discretised problem (fine G or coarse G_c), device pointers.
struct DProblem {
    int n;
    double lo, dx, h, lambda;
    double beta;      // 1/(1 + lambda h)
    double q;         // h/dx: drift displacement in cells per unit speed
    double sc;        // diffusion displacement in cells per unit sigma: sqrt(h p)/dx or sqrt(h)/dx
    double lmax;      // max_x l(x)
    double v0;        // h lmax/(1 - beta): initial supersolution (R11)
    int na;
    const double *ctrl;  // 2*na
    DCoef speed, drift[2], sigma[2][2], cost;
    int p;
    const uint8_t *kind;
    int sigma_mode;          // 1: sigma(x, a) = s(x) a, s = sigma[0][0], p = 1 (R32)
    const double *cost_ctrl; // N_A additive costs m(a_k) or NULL (R33)
    double lmax_x;           // max_x l(x) (lmax above includes max m, for V0 and the front step)
};

// running cost l(x_i, a_k) = l(x_i) + m(a_k) (R33), canonical order of the oracle's cost_of
__host__ __device__ __forceinline__ double cost_at(const DProblem &P, double lx, int a)
{
    return P.cost_ctrl ? lx + P.cost_ctrl[a] : lx;
}

// Row-table stencil entry (row-uniform coefficients): for one grid row j and one control k,
// the branch-merged compact stencil of an interior node relative to the node:
//   v_k - V_ref = c_k + sum_{r<WY, x<WX} W[r][x] u(j + oy + r, i + ox + x),
//   c_k = D E,  D = h l - (1 - beta) V_ref,  E = 1/(1 - beta Lambda0_k),
//   W = beta w (sum of non-self bilinear weights of all branches at that node) E.
template <typename real, int WY, int WX>
struct RowEntry {
    int oy, ox;
    real E;
    real W[WY * WX];
};

// ---------------------------------------------------------------- canonical.cu launchers
void launch_init_values(const DProblem &P, double *V, cudaStream_t s);
void launch_coarse_sweep(const DProblem &P, const double *Vin, double *Vout, double tol,
                         unsigned long long *res_hist, int sweep, int *sweeps_done,
                         cudaStream_t s);
// row-invariant part of the coarse node update (row-uniform coefficients), per (row, control)
struct CoarseRowEntry {
    double bxq;      // q f1
    double ty, uy;   // clamped y fraction and 1 - ty
    double hl;       // h l(x, a)
    double fbd;      // floor(q f1) (an integer): an unclamped foot's x cell is i + fbd or i + fbd + 1
    int cy;          // y cell
    int pk;          // interior fast path: low 16 bits = (cy - j) * CSW + floor(q f1) + 32768 (offset of
                     // the stencil's corner 00 from the node in the staged tile); bits 16..19: one-hot,
                     // the corner (00, 10, 01, 11) that is the node itself when the x cell is i + fbd
};
void launch_coarse_rowtab(const DProblem &P, CoarseRowEntry *tab, cudaStream_t s);
// synthesis with the same row-invariant table built on the fine grid (bit-identical)
void launch_synthesize_rt(const DProblem &P, const double *uhat, const CoarseRowEntry *tab,
                          uint8_t *astar, int stage_ok, cudaStream_t s);
// active-tile form of the same sweep (bit-identical; fprev/fout: per-tile change flags; rowtab:
// the row-invariant table or NULL)
void launch_coarse_sweep_tiles(const DProblem &P, const double *Vin, double *Vout, double tol,
                               unsigned long long *res_hist, int sweep, int *sweeps_done,
                               const uint8_t *fprev, uint8_t *fout, const CoarseRowEntry *rowtab,
                               int stage_ok, cudaStream_t s);
int coarse_halo();   // halo of the shared-memory staged coarse sweep (needs reach + 1 <= halo)
int coarse_tile();
// fuzzy patches: phi_p init, one Jacobi advection sweep, thresholding
void launch_fuzzy_init(const DProblem &P, const int16_t *sector, int np, double *phi, cudaStream_t s);
void launch_fuzzy_sweep(const DProblem &P, const uint8_t *astar, int np, const double *cur,
                        double *nxt, double eps, unsigned long long *res_hist, int sweep,
                        int *sweeps_done, cudaStream_t s);
void launch_fuzzy_assign(const DProblem &P, const double *phi, int np, double tau, int16_t *labels,
                         int *overlap, cudaStream_t s);
// sparse top-K form (per node K (patch, phi_p) pairs, node-major); K in {1,2,3,4,6,8,16}
void launch_fuzzy_sparse_init(const DProblem &P, const int16_t *sector, int np, int K, int16_t *lab,
                              double *mass, cudaStream_t s);
bool launch_fuzzy_sparse_sweep(const DProblem &P, const uint8_t *astar, int K, const int16_t *clab,
                               const double *cm, int16_t *nlab, double *nm, double eps,
                               unsigned long long *res_hist, int sweep, int *sweeps_done, cudaStream_t s);
void launch_fuzzy_sparse_assign(const DProblem &P, const int16_t *lab, const double *mass, int K, int np,
                                double tau, int16_t *labels, int *overlap, int *maxlist, cudaStream_t s);
void launch_prolong(int nc, const double *uc, int n, double *out, cudaStream_t s);
void launch_synthesize(const DProblem &P, const double *uhat, uint8_t *astar, cudaStream_t s);
void launch_successor(const DProblem &P, double M, const uint8_t *astar, int32_t *succ,
                      cudaStream_t s);
void launch_jump(const int32_t *in, int32_t *out, int64_t N, int *changed, cudaStream_t s);
void launch_labels(const uint8_t *kind, const int16_t *sector, const int32_t *root,
                   int n_patches, int64_t N, int16_t *labels, cudaStream_t s);
void launch_static_labels(int n, int px, int py, const uint8_t *kind, int16_t *labels,
                          cudaStream_t s);

// ---------------------------------------------------------------- sweep.cu
struct TileGeom {
    int TW, TH, H, tiles_x, tiles_y, pitch;
    int cstride;   // floats between the 4 shifted smem copies (path 3)
};

struct TileState {
    int32_t *tile_free;      // free nodes per tile
    double *tile_minu;       // min u_hat over free nodes (patchy bucket key)
    double *tile_res;        // last in-tile residual (or verification residual)
    double *tile_chg;        // net change of the last visit (0 if not visited this round)
    float *tile_edge;        // 4 per tile: bound on the last visit's change within H of the tile's
                             // west / east / south / north side (what a neighbour's stencil reads)
    // the distinct patch labels of each tile (free nodes only; orphans = n_patches), CSR:
    // tile t holds tile_lab_ids[tile_lab_off[t] .. tile_lab_off[t + 1])
    int32_t *tile_lab_cnt;   // per tile: number of distinct labels (k_tile_init)
    int32_t *tile_lab_off;   // n_tiles + 1 offsets (k_scan_offsets)
    int16_t *tile_lab_ids;   // capacity n*n: a tile has at most as many labels as nodes
    unsigned long long *tile_lab_res;   // per CSR entry: max |T(V) - V| over the tile's free nodes of
                                        // that label in the tile's last check visit (fp64 bits);
                                        // capacity tile_lab_cap entries (partial verifications)
    int64_t tile_lab_cap;
    int32_t *tile_round;     // per tile: last activation round that took it (-1: never)
    int n_slots;             // patch slots: n_patches + 1 (the last one = orphans); 0 = none
    uint8_t *tile_orient;    // first in-tile sweep orientation (bit 0: -x, bit 1: -y)
    int32_t *tile_stamp;     // sweep id that wrote tile_chg (valid iff == RoundCtl::sweep_id)
    int32_t *tile_sweeps;    // in-tile sweeps done so far this solve (orientation schedule)
    int32_t *list[2];        // active tile lists
    int32_t *all_list;       // tiles with free nodes
    int32_t *patch_round;    // per patch: last round with an active tile (activation trace)
    unsigned long long *patch_res;   // per patch: max |T(V) - V| over its free nodes in the
                                     // last verification pass (fp64 bits, >= 0 orders as u64)
    void *counters;          // ActCounters (device)
    // ordered schedule
    double *tile_key;        // sort key per tile
    int32_t *tile_group;     // static block of the tile (dependency groups), or unused
    int32_t *order;          // tile ids sorted by key
    int *done;               // last pass that finished the tile
    long long *stamp;        // visit sequence number of the tile's last visit
    void *ocounters;         // OrdCounters (device)
};

struct OrdCounters {
    int counter;
    int processed;
    unsigned long long free_sum;
    unsigned long long max_res;
    unsigned long long seq;
    unsigned long long updates;   // node-updates performed in the current pdd_solve
};

struct ActCounters {
    int32_t count;
    int32_t fetch;                    // device-driven rounds: next list entry to take
    long long free_sum;
    unsigned long long min_pending;   // ordered bits of the min u_hat of needy ineligible tiles
    unsigned long long max_res;       // ordered bits of the max tile residual
};

// Device-driven rounds: the host enqueues batches of (begin, activate, sweep, end) without
// synchronising; this block carries the round state between the kernels of a batch.
struct RoundCtl {
    double thr;              // bucket threshold of the moving front (patchy), +inf: none
    double delta;            // threshold step per round (<= 0: no front)
    double dboost;           // cap of the under-fill boost of the step
    int resident;            // sweep CTAs the GPU holds at once
    int policy;              // opts.reserved[1]
    int stop;                // 0 run, 1 nothing active / verification due (host verifies)
    int round;               // activation round counter (patch bookkeeping)
    int sweep_id;            // sweeps launched so far; tile_chg valid iff tile_stamp == sweep_id
    int since_verify;        // sweep rounds since the last verification
    int verify_every;        // force a verification after this many
    int pad;
    double upw;              // >= 0: only neighbours with min u_hat <= own + upw re-activate
    long long rounds;        // sweep rounds (pdd_solve_stats.rounds share)
    long long tiles;         // tiles processed
};

// Ordered schedule (k_sweep_ordered): one Gauss-Seidel pass over the tiles in key order.
struct OrderArgs {
    const int32_t *order;         // tile ids sorted by key
    int n_order;
    const double *key;            // per tile: min u_hat (patchy) or block-lexicographic rank
    const int32_t *group;         // per tile group (static block) or NULL: dependencies only
                                  // between tiles of the same group
    const int32_t *tile_free;
    int *done;                    // per tile: last pass whose visit (or skip) finished
    long long *stamp;             // per tile: visit sequence number of its last visit
    unsigned long long *seq;      // global visit sequence counter
    int *counter;                 // work counter of this pass
    int *processed;               // tiles visited this pass
    unsigned long long *free_sum; // free nodes of the visited tiles
    unsigned long long *max_res;  // ordered bits of the max visit residual
    int pass;                     // pass id (>= 1)
    double tol;
    double key_slack;             // wait only for neighbours with key < own key - key_slack
    int32_t *tile_round;          // activation trace (pass id of the tile's last visit) and
    const int32_t *lab_off;       //   the per-patch rounds through the tile label CSR
    const int16_t *lab_ids;
    int32_t *patch_round;
};

// Work-queue schedule (k_sweep_queue): persistent CTAs take dirty tiles from a ticket ring, visit
// them and mark the neighbours of changed tiles dirty -- asynchronous (chaotic) relaxation of the
// same monotone contraction (R29) without rounds.  Patchy: tiles enter in key order (min u_hat,
// P:744-749) so that about `target` tiles are queued or being visited at any time: a tile that
// converges admits the next one of the order (a sliding window of the lowest unconverged keys).
// Static: every tile is queued at the start.
struct QueueCtl {
    unsigned long long head;         // consumer tickets handed out (monotone)
    unsigned long long tail;         // ring positions handed to producers (monotone)
    unsigned long long visits;       // tile visits so far (the visit sequence number)
    unsigned long long max_visits;   // stop = 2 once reached (non-convergence guard)
    unsigned long long verify_at;    // stop = 3 once reached: the host runs a verification pass (a
                                     // tolerance below the arithmetic's noise floor keeps tiles
                                     // re-queuing each other; the Jacobi check is authoritative)
    int work;                        // tiles queued or being visited (+ admissions in flight)
    int adm;                         // next position of the key order to admit (>= n_order: all in)
    int stop;                        // 1: queue drained for good, 2: visit cap, 3: verification due
    int pad;
    unsigned long long max_res;      // ordered bits of the max visit residual (report)
};
struct QueueArgs {
    QueueCtl *ctl;
    int32_t *ring;                   // cap slots, 0 = empty, else tile + 1
    unsigned cap;                    // power of two > tiles + resident CTAs
    const int32_t *order;            // tiles with free nodes in key order
    const int32_t *rank;             // position of each tile in order (INT_MAX: not listed)
    int n_order;
    int target;                      // admission keeps about this many tiles queued or visiting
    int *state;                      // per tile: 0 clean, 1 queued, 2 visiting, 3 visiting + dirty
    double tol;                      // re-queue a tile whose last sweep changed >= tol
    double tol_act;                  // mark the 8 neighbours dirty when the visit changed >= tol_act
    int32_t *tile_round;             // per tile: sequence number of its last visit
    const int32_t *lab_off;          // tile label CSR -> per-patch last visit sequence
    const int16_t *lab_ids;
    int32_t *patch_round;
};

struct SweepLaunch {
    DProblem P;
    double *V;
    const int16_t *labels;
    unsigned long long *patch_res;       // check mode: per-patch residual max (or NULL)
    int n_slots;                         // patch slots of labels / patch_res
    const int32_t *lab_off = nullptr;    // check mode with lab_res: the tile label CSR; every tile
    const int16_t *lab_ids = nullptr;    //   writes its per-label residuals into its CSR entries
    unsigned long long *lab_res = nullptr;   // (then launch_patch_res_reduce gives patch_res)
    TileGeom g;
    const int32_t *list;
    int n_list;
    double *tile_res, *tile_chg;
    float *tile_edge;
    int k_inner;
    double *out;             // check mode with output (apply operator)
    const void *rowtab;      // RowEntry array [n][na_pad]
    int na_pad;
    int Hx;                  // nodes with i < Hx or i > n-1-Hx use the general stencil
    int path;                // 1 general, 2 row-table, 3 row-table fp32 G=4, 4 lean general
                             // (WY = branches, WX = 1: drift planes staged)
    int WY, WX;              // row-table window
    int check;               // 1: pure Jacobi residual, no update
    int precision;           // 32 | 64
    int ordered;             // 1: k_sweep_ordered with `order` (one pass)
    OrderArgs order;
    int queued = 0;          // 1: k_sweep_queue with `queue`
    QueueArgs queue{};
    double early_tol;        // > 0: a tile visit stops after the first sweep changing < early_tol
    const int32_t *tile_free;            // free nodes per tile (node-update accounting)
    const uint8_t *tile_orient;          // per-tile first sweep orientation (or null: +x+y)
    int oxor = 0xE4;                     // sweep s mod 4 uses orientation o0 ^ ((oxor >> 2s) & 3)
    double early_rel = 0.0;              // relative early exit (0: off)
    int k_coherent = 1 << 30;            // sweeps per visit of a coherent tile
    unsigned long long *nu_counter;      // += free nodes x sweeps done, per visit (or NULL)
    RoundCtl *ctl = nullptr;             // device-driven round: persistent grid, list/count from
    ActCounters *acnt = nullptr;         //   the activation counters, stamps tile_chg
    int32_t *tile_stamp = nullptr;
    int32_t *tile_sweeps = nullptr;      // orientation schedule continues across visits
    int *occupancy_out = nullptr;        // != NULL: report the device-driven kernel's resident
                                         //   CTAs per SM and launch nothing
};

// work-queue schedule: (re-)seed the zeroed ring -- first > 0: with the first `first` tiles of the
// key order (start of a patchy solve); else with every tile among the first `adm` of the order
// whose residual is >= tol (static start: tol < 0 takes all; after a verification pass: the
// offending tiles)
void launch_queue_seed(const TileState &T, const QueueArgs &Q, int n_tiles, double tol, int first,
                       int adm, cudaStream_t s);
// partial verification of the work-queue schedule: list (T.list[0], count in T.counters) of the
// tiles with free nodes whose 3 x 3 tile neighbourhood holds a tile visited after `mark`
void launch_verify_list(const TileGeom &g, const TileState &T, int mark, int n_tiles, cudaStream_t s);
// patch_res[p] = max over the CSR entries of label p of tile_lab_res (n_slots entries zeroed first)
void launch_patch_res_reduce(const TileState &T, int n_tiles, cudaStream_t s);
// per-patch activation trace from the per-tile one (work queue: patch_round[p] = max tile_round
// over the tiles holding nodes of p)
void launch_patch_rounds(const TileState &T, int n_tiles, cudaStream_t s);
// order / rank of the tiles with free nodes by key (NULL: tile index order); scratch of
// queue_order_scratch_ints() ints
void launch_queue_order(const TileState &T, const double *key, int n_tiles, int32_t *scratch,
                        int32_t *order, int32_t *rank, cudaStream_t s);
size_t queue_order_scratch_ints();

// device-driven round kernels (one thread each) around the activation and the sweep
void launch_round_begin(RoundCtl *ctl, ActCounters *c, cudaStream_t s);
void launch_round_end(RoundCtl *ctl, const ActCounters *c, cudaStream_t s);
void launch_round_reset(RoundCtl *ctl, double thr, cudaStream_t s);
// order the round's active list by key (patchy: min u_hat) before the sweep
void launch_sort_round(const RoundCtl *ctl, const ActCounters *c, const double *key, int32_t *list,
                       cudaStream_t s);

// tile bookkeeping of a solve: free counts, min u_hat keys, orientations and (labels != NULL)
// the CSR of the distinct patch labels of every tile (three kernels)
void launch_tile_init(const DProblem &P, const TileGeom &g, const double *uhat,
                      const int16_t *labels, TileState &T, cudaStream_t s, double coh_thr = 2.0);
void launch_set_values(const DProblem &P, int mode, const double *uhat, double *V,
                       cudaStream_t s);
// slack >= 0: patchy upstream-ready rule (a tile waits for unconverged neighbours whose min u_hat
// is lower by more than slack); < 0: off
// ctl != NULL: tile_chg counts only where tile_stamp == ctl->sweep_id; with from_ctl, thr and
// round come from ctl and nothing happens once ctl->stop is set (device-driven rounds)
void launch_activate(const TileGeom &g, TileState &T, int out_list, double tol, double tol_act,
                     double thr, int round, int n_tiles, cudaStream_t s, double slack = -1.0,
                     const RoundCtl *ctl = nullptr, bool from_ctl = false);
cudaError_t launch_sweep(const SweepLaunch &L, cudaStream_t s);
bool rowtab_supported(int WY, int WX, int cpl);
int rowtab_tw(int WY, int WX);
int sweep_tile_rows();
// compile-time shared-memory geometry of the path-3 kernel (rows pitch, copy stride, max halo)
void p3_geometry(int &pitch, int &cstride, int &hmax);
void p3_tile(int &tw, int &th);   // path-3 tile columns / rows
void gf_geometry(int &pitch);      // compile-time shared-memory pitch of path 4 (sweep_gf.cuh)
int pres_shared_slots();           // patch labels a check CTA accumulates in shared memory
// the 16 x 128 path-3 tile (sweep.cu built with PDD_WIDE_UNIT=1)
cudaError_t launch_sweep_wide(const SweepLaunch &L, cudaStream_t s);
void p3_geometry_wide(int &pitch, int &cstride, int &hmax);
void p3_tile_wide(int &tw, int &th);
// the 16 x 64 path-3 tile (sweep.cu built with PDD_LOW_UNIT=1, PDD_P3_TH=16)
cudaError_t launch_sweep_low(const SweepLaunch &L, cudaStream_t s);
void p3_geometry_low(int &pitch, int &cstride, int &hmax);
void p3_tile_low(int &tw, int &th);
// Build the row-stencil table on the device; false if no supported window fits.
bool rowtab_build_device(const DProblem &P, int napad, int H, int precision, int *scratch,
                         void *tab, size_t tab_bytes, int &WY, int &WX, int &oxmin, int &oxmax,
                         cudaStream_t s);
size_t rowtab_entry_bytes(int precision, int WY, int WX);

}  // namespace pdd
