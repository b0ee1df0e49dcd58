"""Sparse fuzzy patches on the GPU (include/pdd.h: pdd_build_fuzzy_patches_sparse; SURVEY 8(f)
NEXT #2, reading R40) against the oracle's sparse iteration: sweep count, the per-node (patch,
phi_p) lists bit for bit, owners, overlap degree -- on C2 (16 patches, full size), C5 at 1025^2
(256 patches) and a paper workload (4 side patches, K = 4: nothing truncated, dense bits) -- and
the patchy solve on those patches."""
import numpy as np
import pytest

import oracle as O
import pdd_inputs as I

pytestmark = pytest.mark.gpu


def _pre(inst, precision=32):
    from paper_1502_01629_b200 import Solver
    s = Solver(inst, precision=precision)
    s.coarse_solve(inst.tol_coarse)
    s.synthesize()
    return s


@pytest.mark.parametrize("cfg,n,K,eps_P", [("C2", None, 4, 1e-3), ("C2", None, 2, 1e-3),
                                           ("C5", 1025, 4, 1e-2), ("C4", 513, 3, 1e-2)])
def test_sparse_lists_bit_exact(cfg, n, K, eps_P):
    inst = I.make_config(cfg, n=n)
    s = _pre(inst)
    astar = s.get_controls()
    ref = O.fuzzy_sparse(inst, astar, inst.n_patches, K, eps_P, tau_P=0.3)
    st = s.build_fuzzy_patches_sparse(inst.n_patches, K=K, eps_P=eps_P, tau_P=0.3, return_lists=True)
    assert st["converged"] == 1 and st["sweeps"] == ref["sweeps"]
    assert np.array_equal(st["lab"], ref["lab"])
    assert np.array_equal(st["mass"].view(np.uint64), ref["mass"].view(np.uint64))
    assert np.array_equal(s.get_labels(), ref["labels"])
    free = inst.kind == I.KIND_FREE
    assert st["overlap_nodes"] == int(np.count_nonzero(ref["members"][free] >= 2))
    assert st["max_list"] == int((ref["lab"][free] >= 0).sum(1).max())
    # decomposition quality: every free node has an owner among the patches that reach it
    own = ref["labels"][free]
    print(f"{cfg}@{inst.n} K={K}: sweeps {st['sweeps']}, overlap nodes {st['overlap_nodes']}, "
          f"longest list {st['max_list']}, orphans {(own == inst.n_patches).mean():.4f}, "
          f"patches used {np.unique(own[own < inst.n_patches]).size}/{inst.n_patches}")
    # the patchy solve runs on these patches (per-patch report included)
    sol = s.solve("patchy", tol=1e-7)
    assert sol["converged"] == 1 and sol["patches_converged"] == sol["patches_active"]
    s.close()


def test_sparse_equals_dense_on_the_paper_workload():
    """Four side patches, K = 4: no truncation, so the sparse lists hold the dense phi bits."""
    inst = I.paper_instance("eikonal", 200, 1e-9)
    s = _pre(inst, precision=64)
    dense = s.build_fuzzy_patches(4, eps_P=1e-3, tau_P=0.5, return_phi=True)
    lab_dense = s.get_labels().copy()
    sp = s.build_fuzzy_patches_sparse(4, K=4, eps_P=1e-3, tau_P=0.5, return_lists=True)
    assert sp["sweeps"] == dense["sweeps"] and sp["overlap_nodes"] == dense["overlap_nodes"]
    N = inst.n * inst.n
    phi = np.zeros((4, N))
    for slot in range(4):
        ok = sp["lab"][:, slot] >= 0
        phi[sp["lab"][ok, slot].astype(np.int64), np.nonzero(ok)[0]] = sp["mass"][ok, slot]
    assert np.array_equal(phi.view(np.uint64), dense["phi"].view(np.uint64))
    assert np.array_equal(s.get_labels(), lab_dense)
    s.close()


def test_sparse_argument_checks():
    from paper_1502_01629_b200 import PddError
    from paper_1502_01629_b200 import _native as N
    inst = I.make_config("C2", n=101)
    s = _pre(inst)
    with pytest.raises(PddError) as e:
        s.build_fuzzy_patches_sparse(16, K=5)
    assert e.value.status == N.PDD_E_INVALID
    with pytest.raises(PddError) as e:
        s.build_fuzzy_patches_sparse(16, K=4, tau_P=1.5)
    assert e.value.status == N.PDD_E_INVALID
    s.close()
