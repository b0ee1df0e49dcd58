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
