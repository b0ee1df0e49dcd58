"""Full-size parity at BASELINE.json's own grids (C3 2049^2, C4 4097^2, C5 8193^2), in the launch
configuration bench.py times (patchy pipeline, fp32, rounds schedule, k_inner = 4).

The oracle cannot run the fine solve at these sizes (C5: ~5.8k Jacobi sweeps, hours), so:
  * everything the oracle CAN compute one by one is compared exactly: u_c (full coarse grid,
    bit-exact), u_hat and a* at sampled nodes (bit-exact), patch labels at sampled nodes (the
    oracle chases the successor chain, synthesising a* on the fly: bit-exact), static labels;
  * V is checked through properties that hold at any size: the oracle's fp64 operator T applied
    to the GPU's V at sampled nodes gives a residual <= 2 tol (the GPU verified < tol in fp32),
    0 <= V <= h l_max / (1 - beta), V = 0 on the target;
  * C5 in fp64: the oracle evaluates T(V) on ALL 67 M nodes; the residual r certifies
    ||V - V*|| <= r / (1 - beta) (contraction, R29) <= 1e-10.
"""
import numpy as np
import pytest

import oracle as O
import pdd_inputs as I

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

_CACHE = {}


def _instance(cfg):
    if cfg not in _CACHE:
        _CACHE[cfg] = I.make_config(cfg)
    return _CACHE[cfg]


def _free_sample(inst, m, seed):
    rng = np.random.default_rng(seed)
    free = np.nonzero(inst.kind == I.KIND_FREE)[0]
    return np.sort(rng.choice(free, size=min(m, free.size), replace=False)).astype(np.int64)


@pytest.mark.parametrize("cfg", ["C3", "C4", "C5"])
def test_fullsize_pipeline_parity(cfg):
    from paper_1502_01629_b200 import Solver
    inst = _instance(cfg)
    ref_c = O.coarse_solve(inst)
    s = Solver(inst, precision=32)
    cs = s.coarse_solve(inst.tol_coarse)
    assert cs["sweeps"] == ref_c["sweeps"]
    assert np.array_equal(s.get_coarse_values().view(np.uint64), ref_c["V"].view(np.uint64))
    s.synthesize()
    idx = _free_sample(inst, 20000, 1)
    uhat = s.get_uhat()
    assert np.array_equal(uhat[idx].view(np.uint64), O.uhat_at(inst, ref_c["V"], idx).view(np.uint64))
    a = s.get_controls()
    assert np.array_equal(a[idx].astype(np.int32), O.astar_at(inst, ref_c["V"], idx))
    s.build_patches(inst.n_patches)
    lab = s.get_labels()
    for k in _free_sample(inst, 150, 2):
        assert lab[k] == O.label_at(inst, ref_c["V"], int(k)), k
    # the fine solve in the bench's configuration
    st = s.solve("patchy", tol=inst.tol, k_inner=4)
    assert st["converged"] == 1 and st["final_residual"] < inst.tol
    V = s.get_values()
    vmax = inst.h * 1.0 / (1.0 - inst.beta)
    assert np.all(V[inst.kind == I.KIND_TARGET] == 0.0)
    free = inst.kind == I.KIND_FREE
    assert V[free].min() > 0.0 and V[free].max() <= vmax
    if cfg == "C4":
        assert np.all(V[inst.kind == I.KIND_OBSTACLE] == 1.0 / inst.lam)
    idx = _free_sample(inst, 200000, 3)
    T, _ = O.apply_at(inst, V, idx)
    assert np.abs(T - V[idx]).max() <= 2 * inst.tol
    # static decomposition: labels closed form, same fixed point within the fp32 bar
    s.build_static(*inst.static_blocks)
    sl = s.get_labels()
    ref_sl = O.static_labels(inst)
    assert np.array_equal(sl, ref_sl)
    st2 = s.solve("static", tol=inst.tol, k_inner=4)
    assert st2["converged"] == 1
    V2 = s.get_values()
    assert np.abs(V2 - V).max() <= 5e-5 * V.max()
    s.close()


def test_fullsize_c5_fp64_certified():
    from paper_1502_01629_b200 import Solver
    inst = _instance("C5")
    s = Solver(inst, precision=64)
    s.coarse_solve(inst.tol_coarse)
    s.synthesize()
    s.build_patches(inst.n_patches)
    bound = 1e-10
    st = s.solve("patchy", tol=0.2 * bound * (1.0 - inst.beta), k_inner=4)
    assert st["converged"] == 1
    V = s.get_values()
    s.close()
    _, r = O.apply(inst, V)                       # oracle fp64 T on all 67 M nodes
    assert r / (1.0 - inst.beta) <= bound, r
