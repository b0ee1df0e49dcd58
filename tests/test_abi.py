"""CPU-side checks of the boundary: libpdd.so loads and exports every symbol include/pdd.h
declares; the ctypes structs match the header's layout; argument validation errors are
reported without touching a GPU.  (No compute calls: there is no GPU here.)"""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pdd.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1502_01629_b200 import build as B
    B.build()
    from paper_1502_01629_b200 import _native as N
    return N.lib()


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(pdd_[a-z_]+)\s*\(", txt)))


def test_header_symbols_exported(lib):
    from paper_1502_01629_b200 import _native as N
    declared = _declared()
    out = subprocess.run(["nm", "-D", "--defined-only", N.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (pdd_\w+)", out))
    missing = [d for d in declared if d not in exported]
    assert not missing, missing
    assert sorted(N.EXPORTS) == declared


def test_library_is_sm100a(lib):
    from paper_1502_01629_b200 import _native as N
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_struct_sizes_match_c(tmp_path):
    """Compile a tiny C program against include/pdd.h and compare sizeof/offsetof with ctypes."""
    from paper_1502_01629_b200 import _native as N
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "pdd.h"\nint main(){'
                   'printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(pdd_problem), sizeof(pdd_coef),'
                   'sizeof(pdd_solve_opts), sizeof(pdd_solve_stats), sizeof(pdd_coarse_stats),'
                   'offsetof(pdd_problem, kind), offsetof(pdd_problem, sigma),'
                   'offsetof(pdd_problem, cost_ctrl), sizeof(pdd_regime), sizeof(pdd_fuzzy_stats));return 0;}')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    vals = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()))
    py = [C.sizeof(N.pdd_problem), C.sizeof(N.pdd_coef), C.sizeof(N.pdd_solve_opts),
          C.sizeof(N.pdd_solve_stats), C.sizeof(N.pdd_coarse_stats),
          N.pdd_problem.kind.offset, N.pdd_problem.sigma.offset, N.pdd_problem.cost_ctrl.offset,
          C.sizeof(N.pdd_regime), C.sizeof(N.pdd_fuzzy_stats)]
    assert vals == py


def test_validation_errors_without_gpu(lib):
    """pdd_workspace_bytes validates the problem on the host."""
    import pdd_inputs as I
    from paper_1502_01629_b200 import _ProblemView, _native as N
    inst = I.make_config("C1")
    v = _ProblemView(inst)
    nb = C.c_size_t(0)
    assert lib.pdd_workspace_bytes(C.byref(v.s), None, 32, C.byref(nb)) == N.PDD_OK
    assert nb.value > 8 * inst.n * inst.n
    bad = _ProblemView(inst)
    bad.s.n = 2
    assert lib.pdd_workspace_bytes(C.byref(bad.s), None, 32, C.byref(nb)) == N.PDD_E_INVALID
    assert b"n = 2" in lib.pdd_last_error(None)
    bad = _ProblemView(inst)
    bad.s.n_controls = 0
    assert lib.pdd_workspace_bytes(C.byref(bad.s), None, 32, C.byref(nb)) == N.PDD_E_INVALID
    bad = _ProblemView(inst)
    bad.s.lam = -1.0
    assert lib.pdd_workspace_bytes(C.byref(bad.s), None, 32, C.byref(nb)) == N.PDD_E_INVALID
    ok = _ProblemView(inst)
    ok.s.lam = 0.0                      # exit problem without obstacles: valid
    assert lib.pdd_workspace_bytes(C.byref(ok.s), None, 32, C.byref(nb)) == N.PDD_OK
    obst = _ProblemView(I.make_config("C4", n=65))
    obst.s.lam = 0.0                    # obstacle value 1/lambda undefined
    assert lib.pdd_workspace_bytes(C.byref(obst.s), None, 32, C.byref(nb)) == N.PDD_E_INVALID
    assert b"obstacles" in lib.pdd_last_error(None)
    bad = _ProblemView(inst)
    bad.s.sigma_mode = 1                # sigma(x,a) = s(x) a needs p = 1 (C1 has p = 2)
    assert lib.pdd_workspace_bytes(C.byref(bad.s), None, 32, C.byref(nb)) == N.PDD_E_INVALID
    g = I.general_instance(17, cost=3, sigma=3)
    assert lib.pdd_workspace_bytes(C.byref(_ProblemView(g).s), None, 32, C.byref(nb)) == N.PDD_OK
    g.cost_ctrl = g.cost_ctrl - 10.0    # l(x) + m(a) <= 0
    assert lib.pdd_workspace_bytes(C.byref(_ProblemView(g).s), None, 32, C.byref(nb)) == N.PDD_E_INVALID
    assert lib.pdd_workspace_bytes(C.byref(v.s), None, 16, C.byref(nb)) == N.PDD_E_INVALID
    bad = _ProblemView(inst)
    bad.s.cost.value = 0.0
    assert lib.pdd_workspace_bytes(C.byref(bad.s), None, 32, C.byref(nb)) == N.PDD_E_INVALID


def test_workspace_scales_with_grid(lib):
    import pdd_inputs as I
    from paper_1502_01629_b200 import _ProblemView
    sizes = []
    for n in (201, 401, 801):
        inst = I.make_config("C2", n=n)
        f, c = _ProblemView(inst), _ProblemView(inst.coarse, False)
        nb = C.c_size_t(0)
        assert lib.pdd_workspace_bytes(C.byref(f.s), C.byref(c.s), 32, C.byref(nb)) == 0
        sizes.append(nb.value)
    # the per-node arrays dominate the growth: doubling n quadruples the increment
    r = (sizes[2] - sizes[1]) / (sizes[1] - sizes[0])
    assert 3.5 < r < 4.5


def test_fuzzy_scratch_bytes_and_validation(lib):
    from paper_1502_01629_b200 import _native as N
    nb = C.c_size_t(0)
    assert lib.pdd_fuzzy_scratch_bytes(101, 4, C.byref(nb)) == N.PDD_OK
    assert nb.value == 2 * 8 * 4 * 101 * 101 + 256            # two patch-major fp64 fields
    assert lib.pdd_fuzzy_scratch_bytes(2, 4, C.byref(nb)) == N.PDD_E_INVALID
    assert lib.pdd_fuzzy_scratch_bytes(101, 0, C.byref(nb)) == N.PDD_E_INVALID


def test_boundary_side_sectors_split_the_ring_evenly():
    """SPEC's example for the paper's four sides: N = 101, N_P = 4 -> four subsets
    of 100 boundary nodes, corners assigned counter-clockwise; N_P = 1 -> the whole boundary."""
    import pdd_inputs as I
    n = 101
    inst = I.paper_instance("eikonal", n - 1, 0.0, coarse_cells=None)
    sec = inst.sector
    ring = inst.kind == I.KIND_TARGET
    assert ring.sum() == 4 * (n - 1)
    assert sorted(np.bincount(sec[ring], minlength=4).tolist()) == [100, 100, 100, 100]
    grid = sec.reshape(n, n)
    assert set(grid[0, 1:-1]) == {3} and set(grid[-1, 1:-1]) == {1}      # bottom / top sides
    assert set(grid[1:-1, 0]) == {2} and set(grid[1:-1, -1]) == {0}      # left / right sides
    one = I.boundary_side_sectors(n, ring, 1)
    assert set(one[ring]) == {0} and np.all(one[~ring] == -1)


def test_automatic_tile_shape_rule(lib):
    """Host logic of the fp32 row-table tile choice: 16 x 64 for patchy solves
    on grids of up to 16 k tiles (C2, C4), 32 x 64 above (C5); static solves take 16 x 128 where
    128 dx <= 1/8 (C4, C5 at full size), else 32 x 64."""
    import ctypes as C
    import pdd_inputs as I
    from paper_1502_01629_b200 import _native as N

    def shape(cfg, patchy, n=None):
        inst = I.make_config(cfg, n=n) if cfg != "C5" or n else None
        nn, lo, hi = (inst.n, inst.lo, inst.hi) if inst is not None else (8193, -2.0, 2.0)
        r, c = C.c_int32(0), C.c_int32(0)
        assert lib.pdd_choose_tile_shape(nn, lo, hi, patchy, C.byref(r), C.byref(c)) == N.PDD_OK
        return r.value, c.value

    assert shape("C2", 1) == (16, 64) and shape("C2", 0) == (32, 64)
    assert shape("C4", 1) == (16, 64) and shape("C4", 0) == (16, 128)
    assert shape("C5", 1) == (32, 64) and shape("C5", 0) == (16, 128)
    assert shape("C5", 1, n=513) == (16, 64) and shape("C5", 0, n=513) == (32, 64)
    r, c = C.c_int32(0), C.c_int32(0)
    assert lib.pdd_choose_tile_shape(2, 0.0, 1.0, 1, C.byref(r), C.byref(c)) == N.PDD_E_INVALID
