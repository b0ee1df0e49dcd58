// sweep_gf.cuh -- path 4 of k_sweep: the general stencil (coefficient FIELDS: C3's speed c(x), the
// paper's Zermelo drift) on an instruction diet (included by sweep.cu; uses its helpers).
//
// Same scheme and same tile schedule as path 1 (sweep_gs.cuh: row_gsg / tile_gsg): SLscheme3 node
// update (R1-R3), lane = control, one node per warp step, exact Gauss-Seidel tile
// sweeps in four orientations with the rows pipelined over the 8 warps.  What differs is the cost
// of a node.  Path 1 evaluates the fully general operator (runtime branch count, sigma(x, a),
// cost fields, exit-problem placeholders, clamping) behind nine warp shuffles of per-node
// coefficients: ~220 warp-instructions per node at 32 controls, 128 registers, 2 CTAs / SM --
// 3.5 % of the FP32 peak on C3.  Path 4 takes the common sub-class
//     f(x, a) = c(x) a + d(x),  sigma and l row-uniform (CONST / ROW),  lambda > 0,  NB = 2 or 4
// and
//   * stages the x-varying coefficient planes of the tile in shared memory next to V (c, and
//     q d1, q d2 when DRIFTX): a node's coefficients are broadcast LDS, no shuffles, no registers
//     held across the row;
//   * unrolls the NB branches at compile time (4 independent bilinear chains per lane), floors by
//     conversion (F2I.FLOOR / I2F), uses a compile-time shared-memory pitch (corner loads with
//     immediate offsets), and clamps feet only in tiles within H of the domain boundary (EDGE);
//   * accumulates the full bilinear sum S and the self weight L0 = sum hat(x) hat(y) per control and
//     removes the node's own corner once, R' = S - L0 u_self, instead of per branch.
// Everything else (exit problems, sigma(x, a), cost fields, NB = 1) stays on path 1.

constexpr int GF_PITCH = 100;   // >= 64 + 2 * 8, = 4 mod 32 (corner loads of one lane: rows 4 banks apart)

template <typename real> __device__ __forceinline__ int gf_floor(real x);
template <> __device__ __forceinline__ int gf_floor<float>(float x) { return __float2int_rd(x); }
template <> __device__ __forceinline__ int gf_floor<double>(double x) { return __double2int_rd(x); }

// row-uniform quantities of the fast general stencil (one set per row, in registers)
template <typename real>
struct GfRow {
    real o[2][2];     // diffusion offsets in cells: sc sigma[k][0], sc sigma[k][1]
    real qd1, qd2;    // q d1, q d2 (used when the drift is row-uniform)
    real D;           // h l(row) - (1 - beta) V_ref
    real bw;          // beta / NB
};

template <typename real, int NB, bool DRIFTX, bool EDGE>
__device__ __forceinline__ real gf_node(const DProblem &P, const real *__restrict__ s_qa,
                                        const real *__restrict__ s_hm, const real *base,
                                        const real *cf, const GfRow<real> &R, int gi, int gj)
{
    constexpr int pitch = GF_PITCH;
    const int lane = threadIdx.x & 31;
    const int n = P.n;
    const real c = cf[0];
    const real qd1 = DRIFTX ? cf[TH * TW_GENERAL] : R.qd1;
    const real qd2 = DRIFTX ? cf[2 * TH * TW_GENERAL] : R.qd2;
    const real uself = *base;
    real best = rinf<real>();
    for (int k = lane; k < P.na; k += 32) {
        const real bx = fma(c, s_qa[2 * k], qd1);
        const real by = fma(c, s_qa[2 * k + 1], qd2);
        real S = 0, L0 = 0;
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            real x = (b & 1) ? bx - R.o[b >> 1][0] : bx + R.o[b >> 1][0];
            real y = (b & 1) ? by - R.o[b >> 1][1] : by + R.o[b >> 1][1];
            int ix, iy;
            if constexpr (EDGE) {   // feet clamped to the box (R5); cell = min(floor, n - 2)
                x = rmin(rmax(x, (real)(-gi)), (real)(n - 1 - gi));
                y = rmin(rmax(y, (real)(-gj)), (real)(n - 1 - gj));
                ix = min(gf_floor<real>(x), n - 2 - gi);
                iy = min(gf_floor<real>(y), n - 2 - gj);
            } else {
                ix = gf_floor<real>(x);
                iy = gf_floor<real>(y);
            }
            const real tx = x - (real)ix, ty = y - (real)iy;
            const real *pc = base + iy * pitch + ix;
            PDD_CHK_TILE(pc, 2, 20);
            PDD_CHK_TILE(pc + pitch, 2, 20);
            const real u00 = pc[0], u10 = pc[1], u01 = pc[pitch], u11 = pc[pitch + 1];
            const real a0 = fma(tx, u10 - u00, u00);
            const real a1 = fma(tx, u11 - u01, u01);
            S += fma(ty, a1 - a0, a0);
            // bilinear weight of the node's own corner: hat(x) hat(y)
            const real hx = rmax((real)0, (real)1 - rabs(x)), hy = rmax((real)0, (real)1 - rabs(y));
            L0 = fma(hx, hy, L0);
        }
        const real Rp = fma(-L0, uself, S);                       // R' = S - Lambda0 u_self
        const real v = (R.D + s_hm[k] + R.bw * Rp) / ((real)1 - R.bw * L0);
        best = rmin(best, v);
    }
    return warp_min(best);
}

template <typename real, int NB, bool DRIFTX, bool EDGE, bool CHECK, bool XNEG>
__device__ __forceinline__ void row_gsf(const KP<real> &A, real *s_u, const real *s_qa,
                                        const real *s_hm, const real *s_cf, volatile int *s_prog,
                                        int H, int i0, int ly, int gj, int jj, int base, int lead,
                                        real &res, double Vref)
{
    constexpr int TW = TW_GENERAL;
    constexpr int NG = TW / 4;
    const int n = A.P.n;
    const DProblem &P = A.P;
    unsigned long long dmask, emask;
    row_masks(P, TW, i0, gj, 0, dmask, emask);
    real *rowp = s_u + (ly + H) * GF_PITCH + H;
    const real *cfrow = s_cf + ly * TW;
    const unsigned prog_prev =
        (unsigned)__cvta_generic_to_shared((const void *)(s_prog + (jj > 0 ? jj - 1 : 0)));
    GfRow<real> R;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        R.o[k][0] = 2 * k < NB ? (real)(P.sc * coef_at(P.sigma[k][0], 0, gj, n)) : (real)0;
        R.o[k][1] = 2 * k < NB ? (real)(P.sc * coef_at(P.sigma[k][1], 0, gj, n)) : (real)0;
    }
    R.qd1 = DRIFTX ? (real)0 : (real)(P.q * coef_at(P.drift[0], 0, gj, n));
    R.qd2 = DRIFTX ? (real)0 : (real)(P.q * coef_at(P.drift[1], 0, gj, n));
    R.D = (real)(P.h * coef_at(P.cost, 0, gj, n) - (1.0 - P.beta) * Vref);
    R.bw = (real)(P.beta / (double)NB);
    for (int gs = 0; gs < NG; ++gs) {
        if (!CHECK && jj > 0) {
            const int need = base + min(gs + lead, NG);
            while (prog_acquire_addr(prog_prev) < need) PDD_SPIN_PAUSE();
        }
#pragma unroll 1
        for (int t = 0; t < 4; ++t) {
            const int lx = XNEG ? TW - 1 - (4 * gs + t) : 4 * gs + t;
            if ((dmask >> lx) & 1ull) continue;
            const real best = gf_node<real, NB, DRIFTX, EDGE>(P, s_qa, s_hm, rowp + lx, cfrow + lx, R,
                                                              i0 + lx, gj);
            commit_node<real, CHECK>(rowp + lx, best, true, res, A.out, (int64_t)gj * n + i0 + lx, Vref, 0, &A);
            __syncwarp();      // lane 0's commit is seen by every lane's next gathers
        }
        if (!CHECK && (threadIdx.x & 31) == 0) prog_release(s_prog + jj, base + gs + 1);
    }
}

template <typename real, int NB, bool DRIFTX, bool CHECK>
__device__ __forceinline__ int tile_gsf(const KP<real> &A, real *s_u, const real *s_qa,
                                        const real *s_hm, const real *s_cf, volatile int *s_prog,
                                        double *s_red, int H, int i0, int j0, int k_inner,
                                        real &res, double Vref, int o0, int sbase)
{
    constexpr int NG = 16;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int n = A.P.n;
    const int lead = 1 + (3 + H) / 4;
    const int sweeps = CHECK ? 1 : k_inner;
    // a tile within H of the domain boundary holds feet that leave the box: clamped variant
    const bool edge_tile = i0 < H || j0 < H || i0 + TW_GENERAL > n - 1 - H || j0 + TH > n - 1 - H;
    double first = 0.0;
    for (int sw = 0; sw < sweeps; ++sw) {
        res = (real)0;
        const int orient = ((A.oxor >> (2 * ((sbase + sw) & 3))) & 3) ^ o0;
        const bool xneg = orient & 1, yneg = orient & 2;
        const int base = sw * NG;
        for (int k = 0; k < TH / NW; ++k) {
            const int jj = warp + NW * k;
            const int ly = yneg ? TH - 1 - jj : jj;
            const int gj = j0 + ly;
            if (gj >= n) {
                if (lane == 0) s_prog[jj] = base + NG;
                continue;
            }
#define PDD_GF_ROW(E_, X_)                                                                         \
            row_gsf<real, NB, DRIFTX, E_, CHECK, X_>(A, s_u, s_qa, s_hm, s_cf, s_prog, H, i0, ly, gj, jj, \
                                                     base, lead, res, Vref)
            if (edge_tile) {
                if (xneg) PDD_GF_ROW(true, true); else PDD_GF_ROW(true, false);
            } else {
                if (xneg) PDD_GF_ROW(false, true); else PDD_GF_ROW(false, false);
            }
#undef PDD_GF_ROW
        }
        if (CHECK) break;
        real r = res;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r = rmax(r, __shfl_xor_sync(FULL, r, o));
        if (lane == 0) s_red[warp] = (double)r;
        __syncthreads();
        if (A.early_tol > 0.0 && sw + 1 < sweeps) {
            double m = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) m = fmax(m, s_red[w]);
            __syncthreads();
            if (sw == 0) first = m;
            if (m < A.early_tol || m < A.early_rel * first) return sw + 1;
        }
    }
    return sweeps;
}
