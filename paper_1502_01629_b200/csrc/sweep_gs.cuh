// sweep_gs.cuh -- path 3 of k_sweep: fp32 row-table stencil, in-tile Gauss-Seidel sweeps in four
// alternating orientations (included by sweep.cu; uses its helpers).
//
// Why: the paper's speed-up comes from processing nodes in a causal order, each node seeing the
// freshest values of the nodes it depends on (2 / 26 sweeps instead of
// 176 / 145).  Inside a tile we use fast-sweeping orientations (+x+y, -x+y, +x-y, -x-y for sweeps
// 0, 1, 2, 3 mod 4): every sweep is an exact Gauss-Seidel pass in its orientation.  Fixed points
// are unchanged (any order of a monotone contraction, R29).
//
// One sweep over the TH x 64 tile:
//   * a warp processes a row 4 nodes ("group") at a time, lane = control (CPL controls per lane).
//     Its controls' WY x (WX+3) window is loaded FRESH from shared memory for every group (so the
//     previous group's nodes are seen updated) and the 4 x CPL candidate sums are accumulated at
//     once (72 FFMA per group at C5: the bulk of the work, full ILP);
//   * the 4 nodes are then finished IN SWEEP ORDER: node k's candidates are corrected for the new
//     values of the nodes of the same group finished before it (their weights in node k's stencil
//     are the row-table weights at relative column -1, -2, -3 (+x) or +1, +2, +3 (-x)), then a
//     5-step __shfl_xor butterfly takes the min over controls -- exact Gauss-Seidel along x;
//   * rows follow the sweep order through a software pipeline over the 8 warps (position jj of
//     the sweep order belongs to warp jj % 8): position jj starts group gs only after position
//     jj-1 has committed groups up to gs + lead - 1 (the window reaches < 4 + H columns ahead),
//     signalled through per-position progress counters in shared memory -- Gauss-Seidel along y.
// Window loads: copy q is chosen so that window column t = 0 is 16-byte aligned; columns 0..3
// come from one LDS.128, columns 4.. from a second LDS.64 / LDS.128.

#ifndef PDD_SPIN_NS
#define PDD_SPIN_NS 32    // pause (ns) between polls of the previous row's progress counter; 0 = plain
                          // spin.  A waiting warp's polls compete for issue slots with the working
                          // warps of the SM: measured under the work queue (profiles/r3j_spin_ab.txt)
                          // 32 or 100 ns give +2 % kernel throughput on C5 / C4 (patchy and static)
#endif
#if PDD_SPIN_NS > 0
#define PDD_SPIN_PAUSE() __nanosleep(PDD_SPIN_NS)
#else
#define PDD_SPIN_PAUSE() ((void)0)
#endif

// Row-pipeline progress counters: release store by the producing warp (after __syncwarp, so the
// whole warp's node commits are ordered before it), acquire load by the consumer -- lighter than
// two CTA-wide sequentially consistent fences per group.
#ifndef PDD_ACQREL
#define PDD_ACQREL 1
#endif
__device__ __forceinline__ void prog_release(volatile int *p, int v)
{
#if PDD_ACQREL == 2
    // relaxed: volatile store behind a compiler barrier, no hardware fence (development A/B; the
    // node commits of this warp precede it in program order on the SM's in-order LSU; a late
    // commit would only make the next row read an older iterate, which chaotic relaxation allows)
    const unsigned a = (unsigned)__cvta_generic_to_shared((const void *)p);
    asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
#elif PDD_ACQREL
    const unsigned a = (unsigned)__cvta_generic_to_shared((const void *)p);
    asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
#else
    __threadfence_block();
    *p = v;
#endif
}

__device__ __forceinline__ int prog_acquire_addr(unsigned a)
{
    int v;
#if PDD_ACQREL == 2
    asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
#else
    asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
#endif
    return v;
}

__device__ __forceinline__ int prog_acquire(volatile int *p)
{
#if PDD_ACQREL
    const unsigned a = (unsigned)__cvta_generic_to_shared((const void *)p);
    int v;
    asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
#else
    const int v = *p;
    __threadfence_block();
    return v;
#endif
}

// path-3 shared-memory geometry for H <= 4 (runtime.cu prepare() uses the same numbers): rows of
// 76 floats (16-byte aligned, odd number of 16-byte groups), 4 shifted copies 3048 floats apart
// ((TH + 8) x 76 + 4 rounded so the copies start in different bank groups)
// PDD_P3_WIDE: tiles of 16 rows x 128 columns instead of 32 x 64 (same 2048 nodes): 32 groups per
// row against the 8-warp row pipeline's 2 x 8 = 16 groups of lead, so the ring of warps has slack
// and a single-sweep visit fills / drains the pipeline in 62 instead of 78 group steps.
#ifndef PDD_P3_WIDE
#define PDD_P3_WIDE 0
#endif
#ifndef PDD_P3_TW
#define PDD_P3_TW (PDD_P3_WIDE ? 128 : 64)
#endif
#ifndef PDD_P3_TH
#define PDD_P3_TH (PDD_P3_WIDE ? 16 : 32)
#endif
constexpr int P3_HMAX = 4;
constexpr int TW3 = PDD_P3_TW;   // path-3 tile columns (64 or 128)
constexpr int TH3 = PDD_P3_TH;   // path-3 tile rows (multiple of 8)
// rows of TW3 + 2 H_max floats rounded up to 16 bytes with an odd number of float4 (consecutive
// window rows in different 16-byte bank groups); the 4 shifted copies (TH3 + 8) rows + 4 apart,
// rounded so that they start in different bank groups
constexpr int p3_pitch_of(int tw)
{
    int p = tw + 2 * P3_HMAX;
    while (p % 4 != 0 || ((p / 4) & 1) == 0) ++p;
    return p;
}
constexpr int p3_cstride_of(int th, int pitch)
{
    int c = (th + 2 * P3_HMAX) * pitch + 4;
    while (c % 4 != 0 || ((c / 4) % 8) != 2) ++c;
    return c;
}
constexpr int P3_PITCH = p3_pitch_of(TW3);
constexpr int P3_CSTRIDE = p3_cstride_of(TH3, P3_PITCH);
static_assert(TW3 == 64 || TW3 == 128, "path-3 tile width");
static_assert(TH3 <= 32 && PDD_TH <= 32, "PROG_N progress counters per CTA");

// per-row masks for up to 128 columns: bit lx of word lx >> 6
__device__ __forceinline__ void row_masks128(const DProblem &P, int TW, int i0, int gj, int Hx,
                                             unsigned long long dm[2], unsigned long long em[2])
{
    const int lane = threadIdx.x & 31;
    const int n = P.n;
    dm[0] = dm[1] = em[0] = em[1] = 0ull;
#pragma unroll
    for (int part = 0; part < 4; ++part) {
        if (part * 32 >= TW) break;
        const int lx = part * 32 + lane;
        const int gi = i0 + lx;
        const bool oob = lx >= TW || gi >= n;
        const bool dir = oob || P.kind[(int64_t)gj * n + gi] != 0;
        const bool edge = !dir && (gi < Hx || gi > n - 1 - Hx);
        dm[part >> 1] |= (unsigned long long)__ballot_sync(FULL, dir) << (32 * (part & 1));
        em[part >> 1] |= (unsigned long long)__ballot_sync(FULL, edge) << (32 * (part & 1));
    }
}

// PDD_RAWMIN 1: V_ref = min of the staged tile, all candidates >= 0, REDUX on the raw float bits
// (saves 4 ALU ops per node, ~3 % on C5) -- off by default: |u| then spans the whole tile range
// instead of half of it, and on coarse grids (tile value range ~1) the fp32 noise floor
// (1 ulp of u = 1.2e-7) rises above a 1e-7 tolerance
#ifndef PDD_EDGE_CALL
#define PDD_EDGE_CALL 0   // 1: the general stencil as an out-of-line call (measured slower)
#endif

#ifndef PDD_RAWMIN
#define PDD_RAWMIN 0
#endif

template <int CPL, int WY, int WX, bool CHECK, bool XNEG, bool EDGE>
__device__ __forceinline__ void row_gs4(const KP<float> &A, float *s_u, const float *s_ctrl,
                                        volatile int *s_prog, int pitch_rt, int cstride_rt, int H,
                                        int i0, int ly, int gj, int jj, int base, int lead,
                                        float D, bool last, float &res, double Vref, float &eW,
                                        float &eE, float &rowmax)
{
    // compile-time smem geometry (P3_PITCH / P3_CSTRIDE, checked against the host's TileGeom):
    // every window row / shifted-copy offset becomes an immediate of the LDS / STS
    (void)pitch_rt;
    (void)cstride_rt;
    constexpr int pitch = P3_PITCH, cstride = P3_CSTRIDE;
    constexpr int TW = TW3;
    constexpr int NG = TW / 4;                 // groups per row (<= 32)
    constexpr int NWC = WX + 3;                // window columns used per group
    constexpr bool xneg = XNEG;
    const int lane = threadIdx.x & 31;
    const int n = A.P.n;
    // ---- row setup (independent of other rows: overlaps the wait for jj - 1)
    unsigned long long dm[2], em2[2];
    row_masks128(A.P, TW, i0, gj, A.Hx, dm, em2);
    const unsigned long long skip[2] = {dm[0] | em2[0], dm[1] | em2[1]};
    const RowEntry<float, WY, WX> *tab =
        reinterpret_cast<const RowEntry<float, WY, WX> *>(A.rowtab) + (int64_t)gj * A.na_pad;
    float Wt[CPL][WY * WX];
    float c0[CPL];
    float wc[CPL][3];          // weights of the 1st, 2nd, 3rd previous node of the row
    const float *src[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        const int kk = lane + 32 * c;
        const RowEntry<float, WY, WX> &e = tab[kk];
        const float Dk = (kk < A.P.na && A.P.cost_ctrl) ? D + (float)(A.P.h * A.P.cost_ctrl[kk]) : D;   // R33
        c0[c] = kk < A.P.na ? Dk * e.E : rinf<float>();
#pragma unroll
        for (int m = 0; m < WY * WX; ++m) Wt[c][m] = e.W[m];
        const int oy = e.oy, ox = e.ox;
        const int e0 = (ly + H + oy) * pitch + H + ox;       // window (0,0) at lx = 0
        const int q = (4 - (e0 & 3)) & 3;                    // column 0 aligned
        src[c] = s_u + q * cstride + q + e0;
        const int r0 = -oy;
#pragma unroll
        for (int d = 1; d <= 3; ++d) {
            const int xw = (xneg ? d : -d) - ox;
            wc[c][d - 1] = (r0 >= 0 && r0 < WY && xw >= 0 && xw < WX) ? e.W[r0 * WX + xw] : 0.f;
        }
    }
    float *rowp = s_u + (ly + H) * pitch + H;
    const int eo = (ly + H) * pitch + H;                      // node row, lx = 0
    const int qo = (4 - (eo & 3)) & 3;
    const float *oldp = s_u + qo * cstride + qo + eo;         // aligned old-value loads
    // commit: lane L < 16 writes node nd = L & 3 of each group into shifted copy L >> 2
    const int nd = lane & 3;
    float *cptr = rowp + (lane >> 2) * (cstride + 1) + nd;
    // per-lane skip bits of its node in every group (bit G = node 4G + nd is special)
    unsigned skip16 = 0u;
#pragma unroll
    for (int G = 0; G < NG; ++G) {
        const int b = 4 * G + nd;
        skip16 |= (unsigned)((skip[b >> 6] >> (b & 63)) & 1ull) << G;
    }
    const unsigned prog_prev = (unsigned)__cvta_generic_to_shared((const void *)(s_prog + (jj > 0 ? jj - 1 : 0)));
    const unsigned long long edge[2] = {EDGE ? (em2[0] & ~dm[0]) : 0ull, EDGE ? (em2[1] & ~dm[1]) : 0ull};
    for (int gs = 0; gs < NG; ++gs) {
        const int G = xneg ? NG - 1 - gs : gs;
        const int g = 4 * G;
        if (!CHECK && jj > 0) {
            const int need = base + min(gs + lead, NG);
            while (prog_acquire_addr(prog_prev) < need) PDD_SPIN_PAUSE();
        }
        // candidate sums, one control at a time (the window of a control is dead once its four
        // sums are formed: keeps the live set small enough for 3 CTAs / SM without remat)
        float acc[CPL][4];
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            float win[WY][8];
#pragma unroll
            for (int r = 0; r < WY; ++r) {
                const float *p = src[c] + r * pitch + g;
                PDD_CHK_TILE(p, NWC > 6 ? 8 : NWC > 4 ? 6 : 4, 10);
                PDD_CHK(((size_t)p & 15) == 0, 11);
                const float4 v = *reinterpret_cast<const float4 *>(p);
                win[r][0] = v.x; win[r][1] = v.y; win[r][2] = v.z; win[r][3] = v.w;
                if constexpr (NWC > 6) {
                    const float4 w = *reinterpret_cast<const float4 *>(p + 4);
                    win[r][4] = w.x; win[r][5] = w.y; win[r][6] = w.z; win[r][7] = w.w;
                } else if constexpr (NWC > 4) {
                    const float2 w = *reinterpret_cast<const float2 *>(p + 4);
                    win[r][4] = w.x; win[r][5] = w.y;
                }
            }
#pragma unroll
            for (int gg = 0; gg < 4; ++gg) {
                float a = c0[c];
#pragma unroll
                for (int r = 0; r < WY; ++r)
#pragma unroll
                    for (int x = 0; x < WX; ++x)
                        a = fmaf(Wt[c][r * WX + x], win[r][gg + x], a);
                acc[c][gg] = a;
            }
        }
        const unsigned sk4 = (unsigned)(skip[g >> 6] >> (g & 63)) & 0xfu;   // special nodes of this group
        PDD_CHK_TILE(oldp + g, 4, 12);
        const float4 o4 = *reinterpret_cast<const float4 *>(oldp + g);
        const float old[4] = {o4.x, o4.y, o4.z, o4.w};
        float nv[4], dlt[4], rd[4];
        // finish the 4 nodes in sweep order with in-group Gauss-Seidel corrections
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const int gg = xneg ? 3 - s : s;
            float m = rinf<float>();
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                float a = acc[c][gg];
#pragma unroll
                for (int d = 1; d <= s; ++d) a = fmaf(wc[c][d - 1], dlt[xneg ? gg + d : gg - d], a);
                m = fminf(m, a);
            }
#if PDD_RAWMIN
            // all candidates are >= 0 (V_ref = min of the staged tile, sweep_tile): non-negative
            // floats order like their bit patterns, so one REDUX on the raw bits is the min
            m = __int_as_float(__reduce_min_sync(FULL, __float_as_int(m)));
#else
            m = warp_min(m);     // fp32: one integer REDUX on order-mapped bits
#endif
            const bool sk = (sk4 >> gg) & 1u;
            nv[gg] = m;
            rd[gg] = sk ? 0.f : m - old[gg];
            dlt[gg] = CHECK ? 0.f : rd[gg];
        }
        if constexpr (CHECK) {
            // per-patch residuals of a verification pass: lane nd < 4 owns node g + nd
            if (A.patch_res && lane < 4 && !((sk4 >> nd) & 1u)) {
                float r = rd[0];
                r = nd == 1 ? rd[1] : r;
                r = nd == 2 ? rd[2] : r;
                r = nd == 3 ? rd[3] : r;
                patch_acc(A, (int64_t)gj * n + i0 + g + nd, (double)fabsf(r));
            }
        }
        {
            const float gm = fmaxf(fmaxf(fabsf(rd[0]), fabsf(rd[1])), fmaxf(fabsf(rd[2]), fabsf(rd[3])));
            if (last) res = fmaxf(res, gm);
            if constexpr (PDD_EDGE_ACT != 0) {
                rowmax = fmaxf(rowmax, gm);
                if (G == 0) eW = fmaxf(eW, gm);        // columns 0..3 cover the west strip (H <= 4)
                if (G == NG - 1) eE = fmaxf(eE, gm);   // and TW-4..TW-1 the east strip
            }
        }
        {
            // lane L < 16 writes node L & 3 of the group into shifted copy L >> 2 (one STS)
            float x = nv[0];
            x = nd == 1 ? nv[1] : x;
            x = nd == 2 ? nv[2] : x;
            x = nd == 3 ? nv[3] : x;
            if (!((skip16 >> G) & 1u)) {
                if (!CHECK) {
                    if (lane < 16) {
                        PDD_CHK_TILE(cptr + g, 1, 13);
                        cptr[g] = x;
                    }
                } else if (A.out && lane < 4) {
                    A.out[(int64_t)gj * n + i0 + g + nd] = Vref + (double)x;
                }
            }
        }
        // nodes of this group whose feet may be clamped in x (within H of the domain's x-boundary):
        // general stencil, in the row pipeline so the next row sees them.  Only the tiles at the
        // domain's x-boundary instantiate this (EDGE): the interior tiles' loop carries none of
        // the general stencil's live ranges (0 spills at 80 registers)
        if constexpr (EDGE) {
            unsigned em = (unsigned)(edge[g >> 6] >> (g & 63)) & 0xfu;
            if (em) {
                __syncwarp();
                while (em) {
                    const int lx = g + __ffs(em) - 1;
                    em &= em - 1;
                    const float best = PDD_EDGE_CALL
                        ? general_node_edge<float>(A.P, s_ctrl, rowp + lx, pitch, i0 + lx, gj, D, Vref)
                        : general_node<float>(A.P, s_ctrl, rowp + lx, pitch, i0 + lx, gj, D, Vref);
                    commit_node<float, CHECK, 4>(rowp + lx, best, last, res, A.out,
                                                 (int64_t)gj * n + i0 + lx, Vref, cstride, &A);
                }
            }
        }
        if (!CHECK) {
            __syncwarp();
            if (lane == 0) prog_release(s_prog + jj, base + gs + 1);
        } else {
            __syncwarp();
        }
    }
}

// CTA-wide maxima of the per-warp side bounds (all threads get them)
__device__ __forceinline__ void tile_edges_out(float eW, float eE, float eS, float eN,
                                               float (*s_edge)[NW], float edge4[4])
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float v[4] = {eW, eE, eS, eN};
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[q] = fmaxf(v[q], __shfl_xor_sync(FULL, v[q], o));
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < 4; ++q) s_edge[q][warp] = v[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        float m = 0.f;
#pragma unroll
        for (int w = 0; w < NW; ++w) m = fmaxf(m, s_edge[q][w]);
        edge4[q] = m;
    }
}

template <int CPL, int WY, int WX, bool CHECK>
__device__ __forceinline__ int tile_gs4(const KP<float> &A, float *s_u, const float *s_ctrl,
                                         volatile int *s_prog, double *s_red, int pitch,
                                         int cstride, int H, int i0, int j0, float D, int k_inner,
                                         float &res, double Vref, int o0, int sbase,
                                         float edge4[4])
{
    constexpr int NG = TW3 / 4;
    __shared__ float s_edge[4][NW];
    float eW = 0.f, eE = 0.f, eS = 0.f, eN = 0.f;   // per-side change bounds, summed over sweeps
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int n = A.P.n;
    const int lead = 1 + (3 + H) / 4;          // groups the previous row must be ahead
    const int sweeps = CHECK ? 1 : k_inner;
    double first = 0.0;                        // change of the visit's first sweep
    const bool edge_tile = i0 < A.Hx || i0 + TW3 > n - 1 - A.Hx;   // holds nodes with x-clamped feet

    for (int sw = 0; sw < sweeps; ++sw) {
        // every sweep tracks its residual: a tile that is converged w.r.t. its halo stops early
        // (early_tol > 0) instead of spending the remaining in-tile sweeps
        const bool last = true;
        res = 0.f;
        const int orient = ((A.oxor >> (2 * ((sbase + sw) & 3))) & 3) ^ o0;   // o0: downstream first
        const bool xneg = orient & 1, yneg = orient & 2;
        const int base = sw * NG;              // progress counters are monotone across sweeps
        float sW = 0.f, sE = 0.f, sS = 0.f, sN = 0.f;   // this sweep's side maxima (this warp)
        for (int k = 0; k < TH3 / NW; ++k) {
            const int jj = warp + NW * k;      // position in this sweep's row order
            const int ly = yneg ? TH3 - 1 - jj : jj;
            const int gj = j0 + ly;
            if (gj >= n) {
                if (lane == 0) s_prog[jj] = base + NG;
                continue;
            }
            float rowmax = 0.f;
            if (edge_tile) {
                if (xneg)
                    row_gs4<CPL, WY, WX, CHECK, true, true>(A, s_u, s_ctrl, s_prog, pitch, cstride, H, i0,
                                                            ly, gj, jj, base, lead, D, last, res, Vref, sW, sE, rowmax);
                else
                    row_gs4<CPL, WY, WX, CHECK, false, true>(A, s_u, s_ctrl, s_prog, pitch, cstride, H, i0,
                                                             ly, gj, jj, base, lead, D, last, res, Vref, sW, sE, rowmax);
            } else {
                if (xneg)
                    row_gs4<CPL, WY, WX, CHECK, true, false>(A, s_u, s_ctrl, s_prog, pitch, cstride, H, i0,
                                                             ly, gj, jj, base, lead, D, last, res, Vref, sW, sE, rowmax);
                else
                    row_gs4<CPL, WY, WX, CHECK, false, false>(A, s_u, s_ctrl, s_prog, pitch, cstride, H, i0,
                                                              ly, gj, jj, base, lead, D, last, res, Vref, sW, sE, rowmax);
            }
            if constexpr (PDD_EDGE_ACT != 0) {
                if (ly < P3_HMAX) sS = fmaxf(sS, rowmax);            // rows of the south strip
                if (ly >= TH3 - P3_HMAX) sN = fmaxf(sN, rowmax);     // and of the north strip
            }
        }
        if constexpr (PDD_EDGE_ACT != 0) {
            if (edge_tile) sW = sE = sS = sN = fmaxf(fmaxf(sW, sE), fmaxf(fmaxf(sS, sN), res));
            eW += sW; eE += sE; eS += sS; eN += sN;
        }
        if (CHECK) break;
        float r = res;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r = fmaxf(r, __shfl_xor_sync(FULL, r, o));
        if (lane == 0) s_red[warp] = (double)r;
        __syncthreads();
        if (A.early_tol > 0.0 && sw + 1 < sweeps) {
            double m = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) m = fmax(m, s_red[w]);
            __syncthreads();                   // s_red is reused by the next sweep
            if (sw == 0) first = m;
            if (m < A.early_tol || m < A.early_rel * first) {
                if constexpr (PDD_EDGE_ACT != 0) tile_edges_out(eW, eE, eS, eN, s_edge, edge4);
                return sw + 1;   // sweeps done
            }
        }
    }
    if constexpr (!CHECK && PDD_EDGE_ACT != 0) tile_edges_out(eW, eE, eS, eN, s_edge, edge4);
    return sweeps;
}


// ------------------------------------------------------------------------------------------
// General-stencil Gauss-Seidel sweeps (path 1: any coefficients, incl. fields such as C3's c(x)
// and the general nonlinear terms; fp32 or fp64).  Same schedule as the row-table kernel: the
// TH x 64 tile is swept k_inner times in the four fast-sweeping orientations (downstream first
// for patchy tiles), a warp finishes its row one node at a time in the sweep's x order (each
// node's gathers see the nodes finished before it: Gauss-Seidel along x), and rows follow the
// sweep's y order through the same progress-counter pipeline over the 8 warps (a row starts a
// 4-node group once the previous row is `lead` groups ahead): Gauss-Seidel along y.
template <typename real, bool CHECK, bool XNEG>
__device__ __forceinline__ void row_gsg(const KP<real> &A, real *s_u, const real *s_ctrl,
                                        volatile int *s_prog, int pitch, int H, int i0, int ly,
                                        int gj, int jj, int base, int lead, real D, real &res,
                                        double Vref)
{
    constexpr int TW = 64;
    constexpr int NG = TW / 4;
    const int lane = threadIdx.x & 31;
    const int n = A.P.n;
    unsigned long long dmask, emask;
    row_masks(A.P, TW, i0, gj, 0, dmask, emask);
    real *rowp = s_u + (ly + H) * pitch + H;
    const unsigned prog_prev =
        (unsigned)__cvta_generic_to_shared((const void *)(s_prog + (jj > 0 ? jj - 1 : 0)));
    // the row's coefficients, prefetched: lane L holds nodes L and L + 32 (global loads overlap
    // the wait for the previous row instead of sitting on every node's dependency chain)
    const NodeCoef<real> nc0 = node_coef<real>(A.P, min(i0 + lane, n - 1), gj, D, Vref);
    const NodeCoef<real> nc1 = node_coef<real>(A.P, min(i0 + lane + 32, n - 1), gj, D, Vref);
    for (int gs = 0; gs < NG; ++gs) {
        if (!CHECK && jj > 0) {
            const int need = base + min(gs + lead, NG);
            while (prog_acquire_addr(prog_prev) < need) PDD_SPIN_PAUSE();
        }
#pragma unroll 1
        for (int t = 0; t < 4; ++t) {
            const int lx = XNEG ? TW - 1 - (4 * gs + t) : 4 * gs + t;
            if ((dmask >> lx) & 1ull) continue;
            const NodeCoef<real> &src = lx < 32 ? nc0 : nc1;
            NodeCoef<real> nc;
            const int sl = lx & 31;
            nc.c = __shfl_sync(FULL, src.c, sl);
            nc.d1 = __shfl_sync(FULL, src.d1, sl);
            nc.d2 = __shfl_sync(FULL, src.d2, sl);
            nc.o[0][0] = __shfl_sync(FULL, src.o[0][0], sl);
            nc.o[0][1] = __shfl_sync(FULL, src.o[0][1], sl);
            nc.o[1][0] = __shfl_sync(FULL, src.o[1][0], sl);
            nc.o[1][1] = __shfl_sync(FULL, src.o[1][1], sl);
            nc.sa = __shfl_sync(FULL, src.sa, sl);
            nc.D = __shfl_sync(FULL, src.D, sl);
            const real best = general_node_c<real>(A.P, s_ctrl, rowp + lx, pitch, i0 + lx, gj, nc);
            commit_node<real, CHECK>(rowp + lx, best, true, res, A.out, (int64_t)gj * n + i0 + lx, Vref, 0, &A);
            __syncwarp();      // lane 0's commit is seen by every lane's next gathers
        }
        if (!CHECK && lane == 0) prog_release(s_prog + jj, base + gs + 1);
    }
}

template <typename real, bool CHECK>
__device__ __forceinline__ int tile_gsg(const KP<real> &A, real *s_u, const real *s_ctrl,
                                        volatile int *s_prog, double *s_red, int pitch, int H,
                                        int i0, int j0, real D, int k_inner, real &res,
                                        double Vref, int o0, int sbase)
{
    constexpr int NG = 16;
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int n = A.P.n;
    const int lead = 1 + (3 + H) / 4;
    const int sweeps = CHECK ? 1 : k_inner;
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
            if (xneg)
                row_gsg<real, CHECK, true>(A, s_u, s_ctrl, s_prog, pitch, H, i0, ly, gj, jj, base,
                                           lead, D, res, Vref);
            else
                row_gsg<real, CHECK, false>(A, s_u, s_ctrl, s_prog, pitch, H, i0, ly, gj, jj, base,
                                            lead, D, res, Vref);
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
