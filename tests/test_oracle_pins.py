"""Pins of the fp64 oracle against what the paper and the mathematics fix (DESIGN.md "Oracle
pins").  None of these compares the oracle with itself: each checks a printed value, a closed
form, an invariant, a special case or an independent exact method.

P1  bilinear weights (S:63 worked example), partition of unity, affine exactness
P2  explicit form (SLexplicit) P:445-472: S:258 worked value, S:259 toy, implicit fixed-point
    substitution with discount
P3  sigma = 0: V -> (1 - exp(-lambda T_A))/lambda with T_A the N_A-gon gauge time, O(dx)
P4  half-plane target: exact geometric series V_n = ((1+lambda h)/lambda)(1 - beta^n)
P5  half-plane with sigma = s I: rows equal the 1-D Bellman solution (1-D policy iteration)
P6  whole operator: Howard policy iteration (exact linear solves) on the implicit scheme
P8  Gauss-Seidel (several orders) = Jacobi fixed point
P9  monotonicity V <= W  =>  T(V) <= T(W) (exact in fp)
P10 bounds 0 <= V <= h l_max/(1-beta), Dirichlet values kept
P11 D4 symmetry on C1
P13 paper Table 0 (golden fixture): SLscheme3 2 / 26 sweeps, SLscheme2 within +-15%
P14 exit problem: |V - (1 - max(|x1|,|x2|))| <= 2 dx, decreasing in N
P16 prolongation: coarse-coincident nodes exact, affine fields exact
P17 synthesis on the exact half-plane field picks the axial control
"""
import math
import os

import numpy as np
import pytest

import oracle as O
import pdd_inputs as I

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


# ---------------------------------------------------------------------------------- P1
def test_p1_bilinear_worked_example():
    row = [r for r in _golden("spec_examples.txt") if r[0] == "bilinear"][0]
    px, py = float(row[1]), float(row[2])
    expect = [float(v) for v in row[3:7]]
    cr, w = O.bilinear_weights(5, 1.0 + px, 2.0 + py)
    assert list(cr) == [2 * 5 + 1, 2 * 5 + 2, 3 * 5 + 1, 3 * 5 + 2]
    assert np.allclose(w, expect, atol=1e-15)


def test_p1_partition_and_affine():
    rng = np.random.default_rng(0)
    n = 9
    for _ in range(200):
        gx, gy = rng.uniform(-1, n), rng.uniform(-1, n)   # includes clamped points
        cr, w = O.bilinear_weights(n, gx, gy)
        assert np.all(w >= 0) and abs(w.sum() - 1.0) < 1e-15
        cx, cy = min(max(gx, 0), n - 1), min(max(gy, 0), n - 1)
        ii, jj = cr % n, cr // n
        assert abs(np.dot(w, 2.0 * ii - 3.0 * jj + 0.5) - (2.0 * cx - 3.0 * cy + 0.5)) < 1e-12


# ---------------------------------------------------------------------------------- P2
def _toy_p2():
    """f = (1,0), sigma = 0, h = 0.05, dx = 0.1, lambda = 0, right neighbour = 0."""
    n = 5
    kind = np.zeros((n, n), np.uint8)
    kind[:, 3:] = I.KIND_TARGET
    z = I.Coef.const(0.0)
    return I.make_instance("p2", n, 0.0, 0.4, n_a=1, lam=0.0, speed=z,
                           drift=(I.Coef.const(1.0), z), kind=kind, h=0.05)


def test_p2_worked_value():
    row = [r for r in _golden("spec_examples.txt") if r[0] == "explicit_value"][0]
    inst = _toy_p2()
    V = np.full(inst.n * inst.n, 1e6)
    V[inst.kind == I.KIND_TARGET] = 0.0
    v, a = O.node_update(inst, V, 2, 2)
    assert abs(v - float(row[1])) < 1e-15 and a == 0
    # the original scheme depends on u(x_i) itself (Eq. self-dependency)
    v2, _ = O.node_update(inst, V, 2, 2, scheme=1)
    assert v2 > 1e5


def test_p2_two_control_toy():
    row = [r for r in _golden("spec_examples.txt") if r[0] == "two_control"][0]
    l0a, l1a, l0b, l1b, expect = map(float, row[1:])
    # explicit value min(L1/(1-L0)) solves the implicit equation u = min(L0 u + L1)
    v = min(l1a / (1 - l0a), l1b / (1 - l0b))
    assert v == expect and abs(min(l0a * v + l1a, l0b * v + l1b) - v) < 1e-15


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_p2_explicit_solves_implicit(seed):
    """For random V and every free node, v = T(V)_i satisfies the implicit Eq. (SLimplicit)
    with discount: v = min_a [h l + beta (R'(a) + Lambda0(a) v)]."""
    inst = I.random_instance(11, seed, n_a=12)
    rng = np.random.default_rng(seed)
    V = rng.uniform(0, 2, inst.n * inst.n)
    beta = inst.beta
    for k in np.nonzero(inst.kind == I.KIND_FREE)[0][:40]:
        i, j = k % inst.n, k // inst.n
        v, _ = O.node_update(inst, V, i, j)
        l0, rp = O.node_lambdas(inst, V, i, j)
        assert np.all(l0 <= 1.0)   # = 1 only where clamping folds every foot onto x_i; beta < 1
        impl = np.min(inst.h * 1.0 + beta * (rp + l0 * v))
        assert abs(impl - v) < 1e-13


# ---------------------------------------------------------------------------------- P3
def _gauge_time(x, y, n_a, r):
    """T_A(x) = min{t : dist(x, P_t) <= r}, P_t = t * conv{a_k}: minimum time to the ball B_r
    with the convexified control set (relaxed controls)."""
    ang = 2 * np.pi * np.arange(n_a) / n_a
    vx, vy = np.cos(ang), np.sin(ang)
    pts = np.stack([x, y], -1)

    def dist_poly(t):
        ax, ay = t[:, None] * vx[None], t[:, None] * vy[None]
        bx, by = np.roll(ax, -1, 1), np.roll(ay, -1, 1)
        ex, ey = bx - ax, by - ay
        px, py = pts[:, 0:1] - ax, pts[:, 1:2] - ay
        L = ex * ex + ey * ey
        s = np.clip((px * ex + py * ey) / np.where(L > 0, L, 1), 0, 1)
        d = np.hypot(px - s * ex, py - s * ey).min(1)
        inside = np.all(ex * py - ey * px >= 0, axis=1)   # CCW polygon
        return np.where(inside, 0.0, d)

    lo = np.zeros(len(x))
    hi = np.full(len(x), 4.0)
    for _ in range(60):
        mid = 0.5 * (lo + hi)
        ok = dist_poly(mid) <= r
        hi = np.where(ok, mid, hi)
        lo = np.where(ok, lo, mid)
    return hi


def test_p3_sigma0_gauge_closed_form_converges():
    errs = []
    for n in (51, 101, 201):
        inst = I.make_instance("p3", n, -1.0, 1.0, n_a=16, lam=1.0,
                               kind=I.ball_target(n, -1.0, 2.0 / (n - 1), (0, 0), 0.1)[0]
                               .astype(np.uint8))
        V = O.jacobi(inst, tol=1e-12)["V"]
        xs = inst.x(np.arange(n))
        X, Y = np.meshgrid(xs, xs, indexing="xy")
        free = inst.kind == 0
        T = _gauge_time(X.reshape(-1)[free], Y.reshape(-1)[free], 16, 0.1)
        exact = (1 - np.exp(-inst.lam * T)) / inst.lam
        errs.append(np.abs(V[free] - exact).max())
    assert errs[0] > errs[1] > errs[2]
    assert errs[2] < 0.015
    assert errs[1] / errs[2] > 1.5        # first order in dx


# ---------------------------------------------------------------------------------- P4 / P17
@pytest.mark.parametrize("lam,n_a", [(1.0, 16), (0.5, 32), (2.0, 8)])
def test_p4_halfplane_exact(lam, n_a):
    inst = I.halfplane_instance(n=21, n_a=n_a, lam=lam, edge_cells=2)
    V = O.jacobi(inst, tol=1e-15, max_sweeps=5000)["V"].reshape(inst.n, inst.n)
    h, beta = inst.h, inst.beta
    ncell = np.arange(inst.n) - 1                     # cells from the target edge (column 1)
    exact = np.where(ncell > 0, (1 + lam * h) / lam * (1 - beta ** np.maximum(ncell, 0)), 0.0)
    assert np.abs(V - exact[None, :]).max() < 1e-13
    _, _, am = O.apply(inst, V.reshape(-1), with_argmin=True)
    free = inst.kind == 0
    assert np.all(am[free] == n_a // 2)


def test_p17_synthesis_on_exact_field():
    inst = I.halfplane_instance(n=33, n_a=16, lam=1.0, edge_cells=3)
    h, beta = inst.h, inst.beta
    ncell = np.maximum(np.arange(inst.n) - 2, 0)
    uhat = np.tile((1 + h) * (1 - beta ** ncell), inst.n)
    a = O.synthesize(inst, uhat)
    assert np.all(a[inst.kind == 0] == 8) and np.all(a[inst.kind != 0] == 255)


# ---------------------------------------------------------------------------------- P5
def _bilin1d(n, g):
    g = min(max(g, 0.0), n - 1.0)
    c = min(int(math.floor(g)), n - 2)
    t = g - c
    return c, t


def test_p5_diffusion_reduces_to_1d():
    s = 0.3 * math.sqrt(1.0 / 20)
    inst = I.halfplane_instance(n=21, n_a=16, lam=1.0, sigma=s, edge_cells=2)
    V = O.jacobi(inst, tol=1e-15, max_sweeps=20000)["V"].reshape(inst.n, inst.n)
    n, h, beta, dx = inst.n, inst.h, inst.beta, inst.dx
    sc = math.sqrt(h * 2) / dx
    # 1-D MDP: state = column; branches: x +- sc*s (x-column), and x twice (the y-column)
    free = np.arange(n) >= 2
    ctrl = inst.controls
    pol = np.zeros(n, int)
    for _ in range(100):
        P = np.zeros((n, n))
        for i in np.nonzero(free)[0]:
            b = i + ctrl[pol[i], 0]
            for g in (b + sc * s, b - sc * s, b, b):
                c, t = _bilin1d(n, g)
                P[i, c] += 0.25 * (1 - t)
                P[i, c + 1] += 0.25 * t
        A = np.eye(n) - beta * P
        A[~free] = 0
        A[~free, ~free] = 1
        rhs = np.where(free, h, 0.0)
        v = np.linalg.solve(A, rhs)
        newpol = pol.copy()
        for i in np.nonzero(free)[0]:
            vals = []
            for a in range(len(ctrl)):
                b = i + ctrl[a, 0]
                acc = 0.0
                for g in (b + sc * s, b - sc * s, b, b):
                    c, t = _bilin1d(n, g)
                    acc += 0.25 * ((1 - t) * v[c] + t * v[c + 1])
                vals.append(h + beta * acc)
            best = int(np.argmin(vals))
            if vals[best] < vals[newpol[i]] - 1e-15:
                newpol[i] = best
        if np.array_equal(newpol, pol):
            break
        pol = newpol
    assert np.abs(V - v[None, :]).max() < 1e-12


# ---------------------------------------------------------------------------------- P6
def _stencil(n, gx, gy):
    gx = min(max(gx, 0.0), n - 1.0)
    gy = min(max(gy, 0.0), n - 1.0)
    cx, cy = min(int(math.floor(gx)), n - 2), min(int(math.floor(gy)), n - 2)
    tx, ty = gx - cx, gy - cy
    return [(cy * n + cx, (1 - tx) * (1 - ty)), (cy * n + cx + 1, tx * (1 - ty)),
            ((cy + 1) * n + cx, (1 - tx) * ty), ((cy + 1) * n + cx + 1, tx * ty)]


def _transitions(inst, k, a):
    """Implicit scheme (SLscheme2): transition row of node k under control a."""
    n = inst.n
    i, j = k % n, k // n
    q = inst.h / inst.dx
    c = inst.speed.at(i, j, n)
    f = c * inst.controls[a] + np.array([inst.drift[0].at(i, j, n), inst.drift[1].at(i, j, n)])
    sc = 0.0
    if inst.p:
        sc = (math.sqrt(inst.h * inst.p) if inst.diffusion_scale == 0 else math.sqrt(inst.h)) / inst.dx
    pts = []
    if inst.p == 0:
        pts.append(q * f)
    for kk in range(inst.p):
        if inst.sigma_mode == 1:      # sigma(x,a) = s(x) a (R32)
            o = sc * inst.sigma[0][0].at(i, j, n) * np.asarray(inst.controls[a], dtype=float)
        else:
            o = sc * np.array([inst.sigma[kk][0].at(i, j, n), inst.sigma[kk][1].at(i, j, n)])
        pts += [q * f + o, q * f - o]
    row = {}
    for g in pts:
        for idx, w in _stencil(n, i + g[0], j + g[1]):
            row[idx] = row.get(idx, 0.0) + w / len(pts)
    return row


@pytest.mark.parametrize("n,seed,p", [(7, 11, 2), (9, 12, 2), (12, 13, 1), (10, 14, 0)])
def test_p6_policy_iteration_matches_jacobi(n, seed, p):
    inst = I.random_instance(n, seed, n_a=8, p=p)
    N = n * n
    beta, h = inst.beta, inst.h
    free = inst.kind == I.KIND_FREE
    dval = np.where(inst.kind == I.KIND_OBSTACLE, 1.0 / inst.lam, 0.0)
    rows = {(k, a): _transitions(inst, k, a) for k in np.nonzero(free)[0] for a in range(8)}
    pol = {k: 0 for k in np.nonzero(free)[0]}
    for _ in range(200):
        A = np.eye(N)
        rhs = dval.copy()
        for k, a in pol.items():
            rhs[k] = h * 1.0
            for idx, w in rows[(k, a)].items():
                A[k, idx] -= beta * w
        v = np.linalg.solve(A, rhs)
        changed = False
        for k in pol:
            vals = [h + beta * sum(w * v[idx] for idx, w in rows[(k, a)].items()) for a in range(8)]
            b = int(np.argmin(vals))
            if vals[b] < vals[pol[k]] - 1e-14:
                pol[k] = b
                changed = True
        if not changed:
            break
    J = O.jacobi(inst, tol=1e-15, max_sweeps=100000)
    assert np.abs(J["V"] - v).max() < 1e-12
    # the Jacobi fixed point satisfies the implicit scheme node by node (P7 brute force)
    for k in list(pol)[:30]:
        vals = [h + beta * sum(w * J["V"][idx] for idx, w in rows[(k, a)].items()) for a in range(8)]
        assert abs(min(vals) - J["V"][k]) < 1e-12


def _howard(inst):
    """Howard policy iteration with dense solves on the implicit scheme (P:366-375 with the
    discount; exit problems: lambda = 0, g = 0 on the boundary ring).  Cost per control
    h l(x_i, a) = h (l(x_i) + m(a)) (R33).  Independent of the oracle's code."""
    n, N = inst.n, inst.n * inst.n
    na = inst.n_controls
    beta, h = inst.beta, inst.h
    free = np.nonzero(inst.kind == I.KIND_FREE)[0]
    dval = np.where(inst.kind == I.KIND_OBSTACLE, 1.0 / inst.lam if inst.lam > 0 else 0.0, 0.0)
    mm = inst.cost_ctrl if inst.cost_ctrl is not None else np.zeros(na)
    rows = {(k, a): _transitions(inst, k, a) for k in free for a in range(na)}
    cost = {(k, a): h * (inst.cost.at(k % n, k // n, n) + mm[a]) for k in free for a in range(na)}
    # start from the policy that moves straight to the nearest boundary side (proper for exit
    # problems: every policy iterate stays proper, the value only decreases)
    pol = {}
    for k in free:
        i, j = k % n, k // n
        side = int(np.argmin([n - 1 - i, j, i, n - 1 - j]))      # +x, -y, -x, +y
        target = [0.0, -0.5 * math.pi, math.pi, 0.5 * math.pi][side]
        ang = np.arctan2(inst.controls[:, 1], inst.controls[:, 0])
        pol[k] = int(np.argmin(np.abs(np.angle(np.exp(1j * (ang - target))))))
    for _ in range(300):
        A = np.eye(N)
        rhs = dval.copy()
        for k, a in pol.items():
            rhs[k] = cost[(k, a)]
            for idx, w in rows[(k, a)].items():
                A[k, idx] -= beta * w
        v = np.linalg.solve(A, rhs)
        changed = False
        for k in pol:
            vals = [cost[(k, a)] + beta * sum(w * v[idx] for idx, w in rows[(k, a)].items())
                    for a in range(na)]
            b = int(np.argmin(vals))
            if vals[b] < vals[pol[k]] - 1e-14:
                pol[k] = b
                changed = True
        if not changed:
            return v
    raise AssertionError("policy iteration did not stop")


@pytest.mark.parametrize("cost,sigma,lam", [(3, 3, 0.0), (2, 2, 0.0), (3, 1, 0.0), (1, 3, 0.0),
                                            (3, 3, 1.0)])
def test_p6b_general_nonlinear_terms_policy_iteration(cost, sigma, lam):
    """P6 for the general nonlinear terms of P:1047-1064: control-dependent diffusion
    sigma_3(x,a) = d_eps(x) a and cost l_3(x,a) = 1 + |x1 x2| + |a1/(2+a2)| (exit problem,
    lambda = 0, and a discounted variant): the oracle's Jacobi fixed point equals the exact
    solution of the finite MDP found by policy iteration."""
    inst = I.general_instance(11, cost=cost, sigma=sigma, eps=0.1, lam=lam, n_a=8)
    v = _howard(inst)
    J = O.jacobi(inst, tol=1e-15, max_sweeps=200000)
    assert np.abs(J["V"] - v).max() < 1e-11


def test_p6c_control_aligned_diffusion_differs_and_reduces():
    """sigma_3 = d a must move the feet along the control (not the axes): with d = 0 it reduces
    to sigma_1 bit for bit, and with d > 0 it differs from sigma_2 = d I."""
    i1 = I.general_instance(17, cost=1, sigma=1)
    i3 = I.general_instance(17, cost=1, sigma=3, eps=0.0)
    assert np.array_equal(O.jacobi(i1, tol=1e-13)["V"], O.jacobi(i3, tol=1e-13)["V"])
    i2 = I.general_instance(17, cost=1, sigma=2)
    i3 = I.general_instance(17, cost=1, sigma=3)
    assert np.abs(O.jacobi(i2, tol=1e-13)["V"] - O.jacobi(i3, tol=1e-13)["V"]).max() > 1e-3


# ---------------------------------------------------------------------------------- P8 / P9
def test_p8_gauss_seidel_orders_match_jacobi():
    inst = I.random_instance(17, 5, n_a=8)
    N = inst.n * inst.n
    Vj = O.jacobi(inst, tol=1e-15, max_sweeps=100000)["V"]
    rng = np.random.default_rng(5)
    for order in (np.arange(N), np.arange(N)[::-1], rng.permutation(N)):
        Vg = O.gauss_seidel(inst, order, tol=1e-15, max_sweeps=100000)["V"]
        assert np.abs(Vg - Vj).max() < 1e-13


def test_p9_monotone():
    inst = I.random_instance(13, 7, n_a=8)
    rng = np.random.default_rng(7)
    for _ in range(10):
        V = rng.uniform(0, 2, inst.n * inst.n)
        W = V + rng.uniform(0, 0.5, V.size) * (rng.uniform(size=V.size) < 0.5)
        TV, _ = O.apply(inst, V)
        TW, _ = O.apply(inst, W)
        assert np.all(TV <= TW)


# ---------------------------------------------------------------------------------- P10 / P11
@pytest.fixture(scope="module")
def c1_solution():
    inst = I.make_config("C1")
    return inst, O.jacobi(inst, tol=1e-14, max_sweeps=100000)


def test_p10_bounds(c1_solution):
    inst, r = c1_solution
    V = r["V"]
    vmax = inst.h * 1.0 / (1 - inst.beta)
    assert np.all(V >= 0) and np.all(V <= vmax)
    assert np.all(V[inst.kind == I.KIND_TARGET] == 0.0)
    assert np.all(V[inst.kind == I.KIND_FREE] > 0)


def test_p11_d4_symmetry(c1_solution):
    inst, r = c1_solution
    V = r["V"].reshape(inst.n, inst.n)
    tol = 1e-12 * V.max()
    for W in (V[:, ::-1], V[::-1, :], V.T, V.T[::-1, ::-1]):
        assert np.abs(W - V).max() < tol


def test_c1_matches_survey_scratch(c1_solution):
    inst = I.make_config("C1")
    r = O.jacobi(inst, tol=1e-9)
    assert r["sweeps"] == 44                       # SURVEY.md Appendix A (C1 exactly)
    assert abs(r["V"].max() - 0.762571) < 1e-6


# ---------------------------------------------------------------------------------- P13
def _paper_order(n):
    # "left to right and from top to bottom": top row first
    return np.array([j * n + i for j in range(n - 1, -1, -1) for i in range(n)])


@pytest.mark.parametrize("eq,problem", [("A", "advection"), ("B", "eikonal")])
def test_p13_table0_sigma0_rows(eq, problem):
    row = [r for r in _golden("table0_iterations.txt") if r[0] == eq and r[2] == "0"][0]
    sl2, sl3 = int(row[3]), int(row[4])
    n = 52    # reading R26b: "50x50" = 50 x 50 interior nodes inside the boundary ring
    inst = I.exit_instance(n, problem=problem)
    for tol in (1e-6, 1e-9, 1e-12):
        r3 = O.gauss_seidel(inst, _paper_order(n), tol=tol, scheme=0)
        assert r3["sweeps"] == sl3
    r2 = O.gauss_seidel(inst, _paper_order(n), tol=1e-12, scheme=1)
    assert abs(r2["sweeps"] - sl2) <= 0.15 * sl2


# ---------------------------------------------------------------------------------- P14
def test_p14_exit_eikonal_accuracy():
    errs = []
    for n in (101, 201):
        inst = I.exit_instance(n, problem="eikonal", h_ratio=0.5)
        order = _paper_order(n)
        V = O.gauss_seidel(inst, order, tol=1e-12)["V"]
        xs = inst.x(np.arange(n))
        X, Y = np.meshgrid(xs, xs, indexing="xy")
        exact = 1 - np.maximum(np.abs(X), np.abs(Y)).reshape(-1)
        err = np.abs(V - exact).max()
        assert err <= 2 * inst.dx
        errs.append(err)
    assert errs[1] <= errs[0]


# ---------------------------------------------------------------------------------- P16
def test_p16_prolongation():
    rng = np.random.default_rng(3)
    nc, r = 9, 8
    n = (nc - 1) * r + 1
    uc = rng.uniform(size=nc * nc)
    u = O.prolong(nc, uc, n).reshape(n, n)
    assert np.array_equal(u[::r, ::r], uc.reshape(nc, nc))
    xc = np.arange(nc)
    Xc, Yc = np.meshgrid(xc, xc, indexing="xy")
    aff = (0.25 + 0.5 * Xc - 0.75 * Yc).reshape(-1)
    ua = O.prolong(nc, aff, n).reshape(n, n)
    xf = np.arange(n) / r
    Xf, Yf = np.meshgrid(xf, xf, indexing="xy")
    assert np.abs(ua - (0.25 + 0.5 * Xf - 0.75 * Yf)).max() < 1e-14
