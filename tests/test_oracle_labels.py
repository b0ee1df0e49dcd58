"""Pins of the oracle's labelling stage (successor rule, pointer chase, static squares, sampled
forms, synthesis tie rule) against hand-computed graphs, SPEC's geometric checks and closed
forms.  None of these compares the oracle with itself.

The label rule is a convention of this build (readings R17/R18: successor = the node
nearest to x_i + M f*/|f*| in cells, rounding half up, clamped to the grid; label = sector of the
target node the successor chain reaches; an obstacle root, a free fixed point or a cycle gives the
orphan label N_P; -1 target, -2 obstacle).  Its pins:
  L1  hand-built 9x9 graph: chain into a target, a 2-cycle, a chain ending on an obstacle, a node
      with |f*| = 0, edge-clamped self loops, a diagonal jump; expected successors and labels are
      written out by hand below
  L2  rounding: half-up (not half-even, not truncation) at exact half-way points; edge clamping
  L3  SPEC.md:392-393 (build_decomposition, eikonal N_P = 4): the owner of (0, -0.5) is the
      bottom side; SPEC.md:571 (criterion 11): >= 95 % agreement with the nearest-side partition
      and patch sizes within 2 % of the interior count
  L4  C2 at full size: no orphans, 16 non-empty patches; >= 85 % of free nodes in
      their ideal 22.5 degree wedge on the exact distance field (SURVEY Q18 measured 85.0 %), and
      the pipeline's (coarse u_hat) agreement reported with a 55 % floor (measured 60.2 %)
  L5  invariants on C3/C5 shapes: the label is constant along successor chains and a labelled
      chain reaches a target node of its own sector
  L6  static squares = the closed form floor(k n / P) (n = 401, P = 4: blocks 100/100/100/101)
  L7  the sampled oracle forms (orc_uhat_at / orc_astar_at / orc_label_at / orc_apply_at) equal the
      full-array functions
  L8  synthesis: exact ties resolve to the lowest index; the running cost enters as h (l + m(a))
      and beta multiplies only the interpolated value (hand-computed example)
  L9  instance pins (tests/golden/instances.txt): R7 target counts equal the lattice-point count
      of the disc (Gauss circle numbers 21 / 1257 / 2061 / 8245 / 5249), instance fingerprints
"""
import math
import os

import numpy as np
import pytest

import oracle as O
import pdd_inputs as I

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _grid9(n_a=8, speed=None):
    """9 x 9 nodes on [0, 8]^2 (dx = h = 1, lambda = 1), no Dirichlet nodes yet."""
    kind = np.zeros(81, dtype=np.uint8)
    return I.make_instance("hand9", 9, 0.0, 8.0, n_a=n_a, lam=1.0, kind=kind,
                           speed=speed if speed is not None else I.Coef.const(1.0))


def _k(i, j, n=9):
    return j * n + i


E, NE, N, NW, W, SW, S, SE = range(8)   # unit_circle_controls(8): k * 45 degrees from (1, 0)


def _hand_instance():
    """L1 instance: targets (0,3) (0,4) (0,5) with sectors 0, 1, 2 (N_P = 3), an obstacle at
    (4,1), speed 0 at (6,4) (|f*| = 0), a* = W everywhere except the hand-set nodes."""
    speed = np.ones(81)
    speed[_k(6, 4)] = 0.0
    inst = _grid9(speed=I.Coef.field(speed))
    kind = inst.kind
    sector = np.full(81, -1, dtype=np.int32)
    for s, j in enumerate((3, 4, 5)):
        kind[_k(0, j)] = I.KIND_TARGET
        sector[_k(0, j)] = s
    kind[_k(4, 1)] = I.KIND_OBSTACLE
    inst.sector = sector
    inst.n_patches = 3
    astar = np.full(81, W, dtype=np.uint8)
    for i in range(0, 6):
        astar[_k(i, 7)] = E          # row 7: (0..5,7) east, (6..8,7) west: 2-cycle (5,7)<->(6,7)
    astar[_k(2, 2)] = NW             # diagonal jump (2,2) -> (1,3)
    astar[_k(3, 5)] = S              # (3,5) -> (3,4): row 5 east of it joins row 4's chain
    astar[kind != 0] = 255
    return inst, astar


# expected labels of the L1 graph, row j = 0 (bottom) .. 8 (top), columns i = 0..8 (orphan = 3)
_HAND_LABELS = [
    [3, 3, 3, 3, 3, 3, 3, 3, 3],       # j=0: chains end at the self loop (0,0)
    [3, 3, 3, 3, -2, 3, 3, 3, 3],      # j=1: (5..8,1) end on the obstacle (4,1)
    [3, 3, 0, 0, 0, 0, 0, 0, 0],       # j=2: (2,2) jumps NW to (1,3) -> target sector 0
    [-1, 0, 0, 0, 0, 0, 0, 0, 0],      # j=3: into target (0,3), sector 0
    [-1, 1, 1, 1, 1, 1, 3, 3, 3],      # j=4: (6,4) has |f*| = 0, (7,4) (8,4) chain into it
    [-1, 2, 2, 1, 1, 1, 1, 1, 1],      # j=5: (3,5) steps S into row 4's chain
    [3, 3, 3, 3, 3, 3, 3, 3, 3],       # j=6
    [3, 3, 3, 3, 3, 3, 3, 3, 3],       # j=7: everything runs into the 2-cycle
    [3, 3, 3, 3, 3, 3, 3, 3, 3],       # j=8
]


def test_l1_hand_graph_successors():
    inst, astar = _hand_instance()
    succ = O.successor(inst, astar, M=1.0)
    exp = np.empty(81, dtype=np.int64)
    for j in range(9):
        for i in range(9):
            exp[_k(i, j)] = _k(max(i - 1, 0), j)           # W, clamped at column 0
    for i in range(0, 6):
        exp[_k(i, 7)] = _k(i + 1, 7)                        # E
    exp[_k(2, 2)] = _k(1, 3)          # (2 - 0.707, 2 + 0.707) = (1.29, 2.71) -> nearest (1, 3)
    exp[_k(3, 5)] = _k(3, 4)
    exp[_k(6, 4)] = _k(6, 4)          # |f*| = 0: its own successor
    for k in np.nonzero(inst.kind != 0)[0]:
        exp[k] = k                    # Dirichlet nodes are their own successors
    assert np.array_equal(succ, exp)


def test_l1_hand_graph_labels():
    inst, astar = _hand_instance()
    succ = O.successor(inst, astar, M=1.0)
    lab = O.labels(inst, succ, n_patches=3).reshape(9, 9)
    assert np.array_equal(lab, np.array(_HAND_LABELS, dtype=np.int16))


def test_l1_single_patch_and_label_range():
    inst, astar = _hand_instance()
    succ = O.successor(inst, astar, M=1.0)
    inst.sector[inst.kind == I.KIND_TARGET] = 0
    lab = O.labels(inst, succ, n_patches=1)
    # one patch: every chain into the target gets 0, the rest stay orphans (label 1)
    ref = np.array(_HAND_LABELS, dtype=np.int16).reshape(-1)
    exp = np.where(ref >= 0, np.where(ref == 3, 1, 0), ref)
    assert np.array_equal(lab, exp)


# ---------------------------------------------------------------------------------- L2
def test_l2_rounding_half_up_and_clamping():
    inst = _grid9()
    astar = np.full(81, E, dtype=np.uint8)
    astar[_k(5, 4)] = W
    astar[_k(4, 6)] = N
    astar[_k(1, 1)] = SW
    # M = 2.5: exact half-way points (dyadic)
    s = O.successor(inst, astar, M=2.5)
    assert s[_k(2, 4)] == _k(5, 4)    # 4.5 -> 5 (half-even would give 4)
    assert s[_k(3, 4)] == _k(6, 4)    # 5.5 -> 6
    assert s[_k(5, 4)] == _k(3, 4)    # 5 - 2.5 = 2.5 -> 3 (half-even / truncation give 2)
    # M = 1.6: nearest, not truncated
    s = O.successor(inst, astar, M=1.6)
    assert s[_k(1, 4)] == _k(3, 4)    # 2.6 -> 3
    assert s[_k(5, 4)] == _k(3, 4)    # 3.4 -> 3
    # M = 4: jumps past the box are clamped to it
    s = O.successor(inst, astar, M=4.0)
    assert s[_k(6, 4)] == _k(8, 4)    # 10 -> 8
    assert s[_k(8, 4)] == _k(8, 4)    # clamped onto itself
    assert s[_k(4, 6)] == _k(4, 8)    # N: 10 -> 8
    assert s[_k(1, 1)] == _k(0, 0)    # SW: (1 - 2.83, 1 - 2.83) -> (-2, -2) -> (0, 0)


# ---------------------------------------------------------------------------------- L3
@pytest.fixture(scope="module")
def eikonal_np4():
    inst = I.paper_instance("eikonal", 100, 0.0)
    ref = O.solve_pipeline(inst, fine=False)
    return inst, ref


def _nearest_side(n):
    """Exact nearest-side partition of the square's nodes (sector ids of boundary_side_sectors:
    0 right, 1 top, 2 left, 3 bottom); -1 where two sides are equally near (the diagonals)."""
    i = np.arange(n)[None, :].repeat(n, 0)
    j = np.arange(n)[:, None].repeat(n, 1)
    d = np.stack([n - 1 - i, n - 1 - j, i, j])          # right, top, left, bottom
    m = d.min(axis=0)
    side = d.argmin(axis=0)
    tie = (d == m[None]).sum(axis=0) > 1
    return np.where(tie, -1, side).reshape(-1)


def test_l3_spec_eikonal_four_triangles(eikonal_np4):
    inst, ref = eikonal_np4
    n = inst.n
    lab = ref["labels"]
    # the boundary split itself: sector 3 is the bottom side (j = 0) without its corners' share
    assert inst.sector[n // 2] == 3 and inst.sector[(n - 1) * n + n // 2] == 1
    # the owner of (0, -0.5) is the bottom-side patch
    i0 = int(round((0.0 - inst.lo) / inst.dx))
    j0 = int(round((-0.5 - inst.lo) / inst.dx))
    assert lab[j0 * n + i0] == 3
    # SPEC.md:571 (criterion 11): >= 95 % agreement with the exact nearest-side partition
    free = inst.kind == I.KIND_FREE
    near = _nearest_side(n)
    cmp = free & (near >= 0)
    agree = float(np.mean(lab[cmp] == near[cmp]))
    assert agree >= 0.95, agree
    sizes = np.array([np.count_nonzero(lab[free] == p) for p in range(4)])
    assert np.count_nonzero(lab[free] == 4) == 0             # no orphans
    assert (sizes.max() - sizes.min()) <= 0.02 * free.sum(), sizes


# ---------------------------------------------------------------------------------- L4
def _wedge_agreement(inst, lab):
    n = inst.n
    free = inst.kind == I.KIND_FREE
    assert np.count_nonzero(lab[free] == inst.n_patches) == 0          # 0 orphans
    used = np.unique(lab[free])
    assert used.size == 16 and used.min() == 0 and used.max() == 15
    # ideal wedge: floor(16 theta / 2 pi) of the node's angle about the target centre node
    c = n // 2
    idx = np.nonzero(free)[0]
    th = np.mod(np.arctan2(idx // n - c, idx % n - c), 2.0 * math.pi)
    wedge = np.minimum(np.floor(16 * th / (2.0 * math.pi)).astype(np.int64), 15)
    return float(np.mean(lab[idx] == wedge))


def test_l4_c2_wedges_exact_distance():
    """The label rule on the exact (continuous) value's distance field u = max(|x| - r, 0): chains
    run radially, so the labels are the 22.5 degree wedges up to the 32-direction quantisation of
    the synthesised controls (SURVEY Q18 measured 85.0 % on such a field)."""
    inst = I.make_config("C2")
    n = inst.n
    x = (np.arange(n) - n // 2) * inst.dx
    u = np.maximum(np.hypot(x[None, :], x[:, None]).reshape(-1) - 0.1, 0.0)
    a = O.synthesize(inst, u)
    lab = O.labels(inst, O.successor(inst, a))
    agree = _wedge_agreement(inst, lab)
    print(f"C2 wedge agreement (exact-distance u_hat): {agree:.4f}")
    assert agree >= 0.85, agree


def test_l4_c2_wedges_pipeline():
    """The same on the pipeline's u_hat (sigma = 0 coarse solve on 51^2, where the r = 0.1 target
    spans 2.5 coarse cells): chains funnel into the faces of the coarse target polygon, so the
    patches are coarser wedges (measured 60.2 %).  Reported, with a floor."""
    inst = I.make_config("C2")
    ref = O.solve_pipeline(inst, fine=False)
    agree = _wedge_agreement(inst, ref["labels"])
    print(f"C2 wedge agreement (pipeline u_hat): {agree:.4f}")
    assert agree >= 0.55, agree
    free = inst.kind == I.KIND_FREE
    sizes = np.bincount(ref["labels"][free], minlength=16)
    assert sizes.min() > 0


# ---------------------------------------------------------------------------------- L5
@pytest.mark.parametrize("cfg,n", [("C3", 513), ("C5", 513)])
def test_l5_label_invariants(cfg, n):
    inst = I.make_config(cfg, n=n)
    ref = O.solve_pipeline(inst, fine=False)
    succ, lab = ref["succ"], ref["labels"]
    free = np.nonzero(inst.kind == I.KIND_FREE)[0]
    nxt = succ[free]
    nf = inst.kind[nxt] == I.KIND_FREE
    # constant along chains (between free nodes)
    assert np.array_equal(lab[free[nf]], lab[nxt[nf]])
    # a labelled chain reaches a target node of its own sector: follow every chain to its end
    cur = succ.copy()
    for _ in range(64):
        cur = cur[cur]
    ok = lab[free] < inst.n_patches
    ends = cur[free[ok]]
    assert np.all(inst.kind[ends] == I.KIND_TARGET)
    assert np.array_equal(inst.sector[ends], lab[free[ok]].astype(np.int32))
    # and every orphan's chain does not end on a target node
    orph = free[~ok]
    assert np.all(inst.kind[cur[orph]] != I.KIND_TARGET)


# ---------------------------------------------------------------------------------- L6
def test_l6_static_closed_form():
    n, P = 401, 4
    kind = np.zeros(n * n, dtype=np.uint8)
    kind[(n // 2) * n + n // 2] = I.KIND_TARGET
    kind[7] = I.KIND_OBSTACLE
    inst = I.make_instance("static401", n, -1.0, 1.0, n_a=4, lam=1.0, kind=kind)
    lab = O.static_labels(inst, P, P).reshape(n, n)
    widths = [(k + 1) * n // P - k * n // P for k in range(P)]
    assert widths == [100, 100, 100, 101]
    blk = np.repeat(np.arange(P), widths)
    exp = blk[:, None] * P + blk[None, :]                 # by * px + bx, rows j
    exp = exp.astype(np.int16).reshape(-1)
    exp[kind == I.KIND_TARGET] = -1
    exp[kind == I.KIND_OBSTACLE] = -2
    assert np.array_equal(lab.reshape(-1), exp)
    # non-square split (C4's 16 x 8): columns in x1, rows in x2
    lab2 = O.static_labels(inst, 16, 8).reshape(n, n)
    assert lab2[0, n - 1] == 15 and lab2[n - 1, 0] == 7 * 16


# ---------------------------------------------------------------------------------- L7
@pytest.mark.parametrize("cfg,n", [("C3", 129), ("C4", 257), ("C5", 257)])
def test_l7_sampled_forms_equal_full_arrays(cfg, n):
    inst = I.make_config(cfg, n=n)
    ref = O.solve_pipeline(inst, fine=False)
    rng = np.random.default_rng(7)
    idx = np.sort(rng.choice(inst.n * inst.n, size=400, replace=False)).astype(np.int64)
    assert np.array_equal(O.uhat_at(inst, ref["uc"], idx).view(np.uint64),
                          ref["uhat"][idx].view(np.uint64))
    a = O.astar_at(inst, ref["uc"], idx)
    full = ref["astar"][idx].astype(np.int32)
    assert np.array_equal(a, full)
    for k in idx[:120]:
        assert O.label_at(inst, ref["uc"], int(k)) == ref["labels"][k], k
    V = ref["uhat"].copy()
    T, res = O.apply(inst, V)
    Ts, _ = O.apply_at(inst, V, idx)
    assert np.array_equal(Ts.view(np.uint64), T[idx].view(np.uint64))


# ---------------------------------------------------------------------------------- L8
def test_l8_synthesis_tie_lowest_index():
    inst = _grid9(n_a=4)                      # axis controls: every foot is a node (exact values)
    uhat = np.full(81, 0.25)                  # constant u_hat, l = 1: every control ties
    a = O.synthesize(inst, uhat)
    assert np.all(a == 0)                     # SPEC: "constant u_hat ... for l = 1, index 0"


def test_l8_synthesis_cost_placement():
    """lambda = 10, h = dx = 1 (beta = 1/11); 4 axis controls E, N, W, S; u_hat = x1 (exact under
    bilinear interpolation); m(a) = (0, 0, 0.5, 0).  The candidates h (l + m_k) + beta u_hat(x + a_k)
    differ by m_k + beta a1_k: E 1/11, N 0, W 0.5 - 1/11, S 0 -> N (index 1; S ties, higher index).
    beta (h (l + m) + u_hat) would pick W (m_k + a1_k: 1, 0, -0.5, 0)."""
    kind = np.zeros(81, dtype=np.uint8)
    inst = I.make_instance("hand9c", 9, 0.0, 8.0, n_a=4, lam=10.0, kind=kind,
                           cost_ctrl=np.array([0.0, 0.0, 0.5, 0.0]))
    x = np.tile(np.arange(9, dtype=np.float64), 9)
    a = O.synthesize(inst, x)
    inner = np.array([_k(i, j) for j in range(1, 8) for i in range(1, 8)])
    assert np.all(a[inner] == 1), a.reshape(9, 9)
    # without the per-control cost, W is the only control moving down u_hat: it wins
    inst.cost_ctrl = None
    a = O.synthesize(inst, x)
    assert np.all(a[inner] == 2)


# ---------------------------------------------------------------------------------- L9
def _golden(name):
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                k, *v = line.split()
                out[k] = v
    return out


def _lattice_disc_count(r2):
    """#{(a, b) in Z^2 : a^2 + b^2 <= r2} by brute force."""
    m = int(math.isqrt(int(math.floor(r2)))) + 1
    a = np.arange(-m, m + 1)
    return int(np.count_nonzero(a[:, None] ** 2 + a[None, :] ** 2 <= r2))


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4", "C5"])
def test_l9_target_counts(cfg):
    g = _golden("instances.txt")
    n = I.FULL_N[cfg]
    lo, hi = (-1.0, 1.0) if cfg in ("C1", "C2") else (-2.0, 2.0)
    dx = (hi - lo) / (n - 1)
    centre, r = {"C1": ((0, 0), 0.1), "C2": ((0, 0), 0.1), "C3": ((0, 0), 0.05),
                 "C4": (I.C4_TARGET, I.C4_TARGET_R), "C5": ((0, 0), 0.02)}[cfg]
    mask, _ = I.ball_target(n, lo, dx, centre, r)
    count = int(np.count_nonzero(mask))
    assert count == int(g["targets_" + cfg][0])
    # the lattice-point count of the disc of radius r/dx (Gauss circle problem)
    assert count == _lattice_disc_count((r / dx) ** 2 + 1e-9)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4"])
def test_l9_fingerprints(cfg):
    g = _golden("instances.txt")
    assert I.make_config(cfg).fingerprint() == g["fingerprint_" + cfg][0]
