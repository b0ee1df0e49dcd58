"""Pins of the oracle's fuzzy patches (Eq. (discrete-advection); reading R38) against
what the mathematics fixes, independently of the oracle's code:
* phi_p is the absorption probability of the Markov chain whose transitions are the bilinear
  weights of the foot x_i + h f(x_i, a*(x_i)): an exact dense linear solve on tiny grids;
* the SPEC examples: advection b = (1,0) with Gamma_p = right side -> phi ~ 1, left side -> 0;
  one patch covering the whole boundary -> phi = 1;
* the thresholding / ownership rule on hand-made phi values."""
import math

import numpy as np
import pytest

import oracle as O
import pdd_inputs as I


def _stencil(n, gx, gy):
    gx = min(max(gx, 0.0), n - 1.0)
    gy = min(max(gy, 0.0), n - 1.0)
    cx, cy = min(int(math.floor(gx)), n - 2), min(int(math.floor(gy)), n - 2)
    tx, ty = gx - cx, gy - cy
    return [(cy * n + cx, (1 - tx) * (1 - ty)), (cy * n + cx + 1, tx * (1 - ty)),
            ((cy + 1) * n + cx, (1 - tx) * ty), ((cy + 1) * n + cx + 1, tx * ty)]


@pytest.mark.parametrize("problem,eps", [("eikonal", 0.0), ("zermelo", 0.0)])
def test_phi_is_the_absorption_probability(problem, eps):
    inst = I.paper_instance(problem, 10, eps, coarse_cells=5)
    ref = O.solve_pipeline(inst, fine=False)
    n, N = inst.n, inst.n * inst.n
    q = inst.h / inst.dx
    A = np.eye(N)
    rhs = np.zeros((N, 4))
    for k in range(N):
        if inst.kind[k] != 0:
            if inst.sector[k] >= 0:
                rhs[k, inst.sector[k]] = 1.0
            continue
        i, j = k % n, k // n
        a = int(ref["astar"][k])
        c = inst.speed.at(i, j, n)
        f = c * inst.controls[a] + np.array([inst.drift[0].at(i, j, n), inst.drift[1].at(i, j, n)])
        for idx, w in _stencil(n, i + q * f[0], j + q * f[1]):
            A[k, idx] -= w
    exact = np.linalg.solve(A, rhs).T          # (4, N)
    fz = O.fuzzy_phi(inst, ref["astar"], 4, 1e-15)
    assert np.abs(fz["phi"] - exact).max() < 1e-10
    # every chain is absorbed on the boundary: the probabilities sum to one
    assert np.abs(exact.sum(0) - 1.0).max() < 1e-12


def _advection(n, side):
    inst = I.exit_instance(n, problem="advection", eps=0.0)
    inst.drift = (I.Coef.const(1.0), I.Coef.const(0.0))       # foot to the right: b = (1, 0)
    mask = inst.kind == I.KIND_TARGET
    inst.sector = I.boundary_side_sectors(n, mask, 4)
    inst.n_patches = 4
    return inst


def test_spec_advection_examples():
    n = 33
    inst = _advection(n, 0)
    astar = np.where(inst.kind == 0, 0, 255).astype(np.uint8)
    fz = O.fuzzy_phi(inst, astar, 4, 1e-13)
    free = inst.kind == 0
    assert np.all(fz["phi"][0][free] > 1.0 - 1e-10)            # right side: phi ~ 1
    assert np.all(fz["phi"][2][free] == 0.0)                   # left side: phi = 0
    one = _advection(n, 0)
    one.sector = np.where(one.kind == I.KIND_TARGET, 0, -1).astype(np.int32)
    f1 = O.fuzzy_phi(one, astar, 1, 1e-13)
    assert np.all(np.abs(f1["phi"][0][free] - 1.0) < 1e-10)   # whole boundary: phi = 1


def test_threshold_and_ownership_rule():
    inst = I.paper_instance("eikonal", 4, 0.0, coarse_cells=None)
    N = inst.n * inst.n
    free = np.nonzero(inst.kind == 0)[0]
    phi = np.zeros((2, N))
    k0, k1, k2, k3 = free[:4]
    phi[:, k0] = (0.6, 0.3)        # owner 0, one member
    phi[:, k1] = (0.6, 0.55)       # owner 0, overlap {0, 1}
    phi[:, k2] = (0.2, 0.4)        # no candidate at tau 0.5: argmax -> owner 1
    phi[:, k3] = (0.45, 0.45)      # tie -> lowest patch
    lab, mem = O.fuzzy_assign(inst, phi, 0.5)
    assert (lab[k0], mem[k0]) == (0, 1)
    assert (lab[k1], mem[k1]) == (0, 2)
    assert (lab[k2], mem[k2]) == (1, 0)
    assert (lab[k3], mem[k3]) == (0, 0)
    rest = free[4:]
    assert np.all(lab[rest] == 2)                               # all zero: orphan label N_P
    assert np.all(lab[inst.kind == I.KIND_TARGET] == -1)


# ---- sparse top-K form (reading R40): pinned to the dense iteration (itself
# pinned to the absorption probabilities above) and to what truncation can and cannot do

def _dense_from_sparse(lab, mass, n_patches):
    N, K = lab.shape
    phi = np.zeros((n_patches, N))
    for s in range(K):
        ok = lab[:, s] >= 0
        phi[lab[ok, s].astype(np.int64), np.nonzero(ok)[0]] = mass[ok, s]
    return phi


@pytest.mark.parametrize("maker,npatch", [
    (lambda: I.paper_instance("eikonal", 20, 0.0, coarse_cells=10), 4),
    (lambda: I.paper_instance("zermelo", 20, 0.0, coarse_cells=10), 4),
    (lambda: I.make_config("C2", n=65, n_coarse=17), 16)])
def test_sparse_equals_dense_when_nothing_is_truncated(maker, npatch):
    """K >= number of patches: the sparse sweep is the dense expression with its zero terms left
    out -- same bits, same sweep count, same owners and overlap degrees."""
    inst = maker()
    ref = O.solve_pipeline(inst, fine=False)
    dn = O.fuzzy_phi(inst, ref["astar"], npatch, 1e-9)
    sp = O.fuzzy_sparse(inst, ref["astar"], npatch, min(npatch, 16), 1e-9, tau_P=0.3)
    assert sp["sweeps"] == dn["sweeps"]
    assert sp["residual"] == dn["residual"]
    phi = _dense_from_sparse(sp["lab"], sp["mass"], npatch)
    assert np.array_equal(phi.view(np.uint64), dn["phi"].view(np.uint64))
    lab, mem = O.fuzzy_assign(inst, dn["phi"], 0.3)
    assert np.array_equal(sp["labels"], lab) and np.array_equal(sp["members"], mem)
    # the lists are sorted by (mass descending, label ascending), empty slots last
    m, l = sp["mass"], sp["lab"].astype(np.int64)
    assert np.all(m[:, :-1] >= m[:, 1:])
    tie = (m[:, :-1] == m[:, 1:]) & (l[:, 1:] >= 0)
    assert np.all(l[:, :-1][tie] < l[:, 1:][tie])
    assert np.all((l < 0) == (m == 0.0))


def test_sparse_truncation_only_drops_mass():
    """K < overlap: every kept phi_p is <= its dense value (weights are >= 0, so dropping terms
    can only lower later sums), the listed masses sum to <= 1, and the owner is the dense owner
    wherever the dense runner-up is clearly smaller."""
    inst = I.make_config("C2", n=65, n_coarse=17)
    ref = O.solve_pipeline(inst, fine=False)
    dn = O.fuzzy_phi(inst, ref["astar"], 16, 1e-9)
    sp = O.fuzzy_sparse(inst, ref["astar"], 16, 2, 1e-9, tau_P=0.3)
    phi = _dense_from_sparse(sp["lab"], sp["mass"], 16)
    assert np.all(phi <= dn["phi"] + 1e-15)
    assert sp["mass"].sum(1).max() <= 1.0 + 1e-12
    free = inst.kind == 0
    srt = np.sort(dn["phi"], axis=0)
    clear = free & (srt[-1] - srt[-2] > 0.2)
    lab, _ = O.fuzzy_assign(inst, dn["phi"], 0.3)
    assert clear.sum() > 0.5 * free.sum()
    assert np.array_equal(sp["labels"][clear], lab[clear])
    # K = 4 of 16 patches (at most 5 reach a node here): 99 % of all owners are the dense ones
    s4 = O.fuzzy_sparse(inst, ref["astar"], 16, 4, 1e-9, tau_P=0.3)
    assert (s4["labels"][free] != lab[free]).mean() < 0.01
    # K = 1 keeps the single strongest patch per node: still a valid ownership map
    s1 = O.fuzzy_sparse(inst, ref["astar"], 16, 1, 1e-9)
    assert np.all((s1["labels"][free] >= 0) & (s1["labels"][free] <= 16))


def test_sparse_hand_example():
    """One free node between two target nodes of different sectors on a 3-node line: the foot
    lands 1/4 of the way to the right neighbour: phi = (3/4 of itself + 1/4 of sector 1) ... the
    fixed point of phi_1 = 0.75 phi_1 + 0.25 is 1, approached as 1 - 0.75^k."""
    n = 3
    kind = np.full((n, n), I.KIND_TARGET, np.uint8)
    kind[1, 1] = I.KIND_FREE
    sector = np.zeros((n, n), np.int32)
    sector[:, 2] = 1
    sector[1, 1] = -1
    inst = I.make_instance("line", n, 0.0, 2.0, n_a=4, lam=1.0, kind=kind.reshape(-1),
                           sector=sector.reshape(-1), h=0.25)
    astar = np.full(n * n, 255, np.uint8)
    astar[4] = 0                                   # control (1, 0): foot at x + 0.25 cells
    sp = O.fuzzy_sparse(inst, astar, 2, 2, 1e-30, max_sweeps=5)
    assert sp["sweeps"] == 5
    assert sp["lab"][4, 0] == 1 and sp["lab"][4, 1] == -1
    assert abs(sp["mass"][4, 0] - (1.0 - 0.75 ** 5)) < 1e-15
