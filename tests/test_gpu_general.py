"""GPU parity for the general nonlinear terms of the paper
and the exit-time problems they are posed on (lambda = 0, g = 0 on the boundary ring):

    f(x,a) = c(x) a,  c = 1 + max{x2, max{x1, 0}};  d_eps = sqrt(2 eps) chi_{x2 >= 0}
    sigma_1 = 0, sigma_2 = d_eps I, sigma_3(x,a) = d_eps a   (control-aligned 1-D Wiener process)
    l_1 = 1, l_2 = 1 + |x1 x2|, l_3(x,a) = l_2 + |a1/(2+a2)|

The oracle (pinned by the Howard policy-iteration tests P6b/P6c) is the reference; the CUDA path
runs through the C ABI.  Exit problems have beta = 1, so the a-posteriori bound r/(1 - beta) does
not apply: both sides are driven to residuals far below the comparison tolerance instead."""
import numpy as np
import pytest

import oracle as O
import pdd_inputs as I

pytestmark = pytest.mark.gpu


def _solve(inst, precision, mode="static", tol=None, kernel=0, k_inner=4):
    from paper_1502_01629_b200 import Solver
    s = Solver(inst, precision=precision)
    if mode == "static":
        s.build_static(*inst.static_blocks)
    else:
        s.coarse_solve(inst.tol_coarse)
        s.synthesize()
        s.build_patches(inst.n_patches)
    st = s.solve(mode, tol=tol if tol else (1e-13 if precision == 64 else 1e-6), k_inner=k_inner,
                 kernel=kernel, raise_on_noconverge=(precision == 64))
    V = s.get_values()
    s.close()
    return V, st


def _check(V, ref, precision):
    err = float(np.abs(V - ref).max())
    if precision == 64:
        assert err <= 1e-10, err
    else:
        assert err <= 5e-5 * float(np.abs(ref).max()), err


@pytest.mark.parametrize("cost", [1, 2, 3])
@pytest.mark.parametrize("sigma", [1, 2, 3])
def test_nine_cost_diffusion_pairs_fp64(cost, sigma):
    """All nine (l_i, sigma_j) pairs of Fig. (generalsigmacost) at n = 65 (general stencil path:
    c(x) is a field), fp64 against the oracle's Jacobi fixed point."""
    inst = I.general_instance(65, cost=cost, sigma=sigma)
    ref = O.jacobi(inst, tol=1e-14, max_sweeps=10 ** 6)["V"]
    V, st = _solve(inst, 64)
    assert st["kernel_used"] == 1
    _check(V, ref, 64)


@pytest.mark.parametrize("cost,sigma", [(3, 3), (2, 2)])
def test_general_pairs_fp32(cost, sigma):
    inst = I.general_instance(97, cost=cost, sigma=sigma)
    ref = O.jacobi(inst, tol=1e-14, max_sweeps=10 ** 6)["V"]
    V, _ = _solve(inst, 32)
    _check(V, ref, 32)


def _row_uniform_variant(n, lam=0.0):
    """sigma_3 and the per-control cost m(a) on a row-uniform problem (constant speed and
    x-cost, d_eps per row): exercises the row-table kernels (path 2 fp64, path 3 fp32)."""
    inst = I.general_instance(n, cost=3, sigma=3, lam=lam, eps=0.002)   # window fits 4 x 4
    inst.speed = I.Coef.const(1.5)
    inst.cost = I.Coef.const(1.0)
    return inst


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("lam", [0.0, 1.0])
def test_control_aligned_diffusion_row_table(precision, lam):
    inst = _row_uniform_variant(129, lam)
    ref = O.jacobi(inst, tol=1e-14, max_sweeps=10 ** 6)["V"]
    V, st = _solve(inst, precision)
    assert st["kernel_used"] == (2 if precision == 64 else 3)
    _check(V, ref, precision)


@pytest.mark.parametrize("cost,sigma", [(3, 3), (3, 2), (2, 3)])
def test_operator_parity_random_values(cost, sigma):
    """T(V) on the same random V (values in [0, 1]): fp64 node by node to 1e-12."""
    from paper_1502_01629_b200 import Solver
    inst = I.general_instance(77, cost=cost, sigma=sigma)
    rng = np.random.default_rng(7)
    W = rng.uniform(0.0, 1.0, inst.n * inst.n)
    W[inst.kind != 0] = 0.0
    s = Solver(inst, precision=64)
    out, _ = s.apply_operator(W)
    s.close()
    ref, _ = O.apply(inst, W)
    assert np.abs(out - ref).max() < 1e-12


@pytest.mark.parametrize("cost,sigma", [(3, 3), (1, 2)])
def test_patchy_pipeline_exit_problem(cost, sigma):
    """The whole patchy pipeline on an exit problem with the general terms: coarse solve
    (sigma = 0, per-control cost) bit-exact, synthesis with l(x, a) bit-exact, the four
    boundary-side patches bit-exact, fine V within the bar."""
    from paper_1502_01629_b200 import Solver
    inst = I.general_instance(129, cost=cost, sigma=sigma, n_coarse=17)
    ref = O.solve_pipeline(inst, tol=1e-14)
    s = Solver(inst, precision=64)
    cs = s.coarse_solve(inst.tol_coarse)
    assert cs["sweeps"] == ref["coarse_sweeps"]
    assert np.array_equal(s.get_coarse_values().view(np.uint64), ref["uc"].view(np.uint64))
    s.synthesize()
    assert np.array_equal(s.get_controls(), ref["astar"])
    s.build_patches(inst.n_patches)
    assert np.array_equal(s.get_labels(), ref["labels"])
    st = s.solve("patchy", tol=1e-13)
    assert st["converged"] == 1
    _check(s.get_values(), ref["V"], 64)
    s.close()


@pytest.mark.parametrize("problem,eps_P", [("eikonal", 1e-3), ("zermelo", 1e-4)])
def test_fuzzy_patches_bit_exact(problem, eps_P):
    """The paper's fuzzy patches on the GPU: canonical fp64 advection of phi_p along
    the synthesised feedback -- sweep count, phi and the thresholded labels bit-exact with the
    oracle; the patchy solve then runs on these patches."""
    from paper_1502_01629_b200 import Solver
    inst = I.paper_instance(problem, 200, 1e-9)
    ref = O.solve_pipeline(inst, tol=1e-14)
    fz = O.fuzzy_phi(inst, ref["astar"], 4, eps_P)
    lab, mem = O.fuzzy_assign(inst, fz["phi"], 0.5)
    s = Solver(inst, precision=64)
    s.coarse_solve(inst.tol_coarse)
    s.synthesize()
    st = s.build_fuzzy_patches(4, eps_P=eps_P, tau_P=0.5, return_phi=True)
    assert st["converged"] == 1 and st["sweeps"] == fz["sweeps"]
    assert np.array_equal(st["phi"].view(np.uint64), fz["phi"].view(np.uint64))
    assert np.array_equal(s.get_labels(), lab)
    assert st["overlap_nodes"] == int(np.count_nonzero(mem >= 2))
    sol = s.solve("patchy", tol=1e-13)
    assert sol["converged"] == 1
    assert float(np.abs(s.get_values() - ref["V"]).max()) <= 1e-10
    s.close()
