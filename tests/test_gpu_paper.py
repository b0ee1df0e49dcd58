"""GPU parity on the paper's own performance workloads (Tables 1-2; SURVEY.md 8(f)
NEXT #3): eikonal-diffusion and Zermelo exit problems on [-1,1]^2 (lambda = 0, g = 0 on the
boundary), sigma = sqrt(2 eps) I with the sqrt(h) scaling, the paper's time step
h = alpha dx / f_min, four boundary-side patches, coarse grid of 50^2 cells.  Below and above the
upwind diffusion ball threshold (eps = dx/4 resp. dx/120)."""
import numpy as np
import pytest

import oracle as O
import pdd_inputs as I

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("problem,eps", [("eikonal", 1e-9), ("eikonal", 2.5e-3), ("eikonal", 1e-2),
                                         ("zermelo", 1e-9), ("zermelo", 1e-3)])
def test_paper_workload_pipeline_fp64(problem, eps):
    from paper_1502_01629_b200 import Solver
    inst = I.paper_instance(problem, 100, eps)
    ref = O.solve_pipeline(inst, tol=1e-14)
    s = Solver(inst, precision=64)
    cs = s.coarse_solve(inst.tol_coarse)
    assert cs["sweeps"] == ref["coarse_sweeps"]
    assert np.array_equal(s.get_coarse_values().view(np.uint64), ref["uc"].view(np.uint64))
    s.synthesize()
    assert np.array_equal(s.get_controls(), ref["astar"])
    s.build_patches(inst.n_patches)
    assert np.array_equal(s.get_labels(), ref["labels"])
    for mode in ("patchy", "static"):
        if mode == "static":
            s.build_static(*inst.static_blocks)
        st = s.solve(mode, tol=1e-13)
        assert st["converged"] == 1
        err = float(np.abs(s.get_values() - ref["V"]).max())
        assert err <= 1e-10, (mode, err)
    s.close()


@pytest.mark.parametrize("problem", ["eikonal", "zermelo"])
def test_paper_workload_fp32_larger_grid(problem):
    from paper_1502_01629_b200 import Solver
    inst = I.paper_instance(problem, 400, 1e-6)
    ref = O.jacobi(inst, tol=1e-13, max_sweeps=10 ** 6)["V"]
    s = Solver(inst, precision=32)
    s.coarse_solve(inst.tol_coarse)
    s.synthesize()
    s.build_patches(inst.n_patches)
    # exit problems have no discount contraction: the fp32 noise floor of the general stencil
    # (feet from fp32 coefficient fields) sits near 1e-7, so the fp32 runs stop at 1e-6
    st = s.solve("patchy", tol=1e-6)
    assert st["converged"] == 1
    err = float(np.abs(s.get_values() - ref).max())
    assert err <= 5e-5 * float(np.abs(ref).max()), err
    s.close()
