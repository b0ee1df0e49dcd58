"""Does the in-tile sweep behave like Gauss-Seidel?  Single-tile problems: GPU rounds (k_inner
sweeps each) vs the oracle's fast-sweeping count (4 orientations).  Dev tool."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O, pdd_inputs as I
from paper_1502_01629_b200 import Solver

def fastsweep(inst, tol):
    n = inst.n
    J, Ii = np.meshgrid(np.arange(n), np.arange(n), indexing='ij')
    b = (J * n + Ii)
    ords = [b.reshape(-1), b[:, ::-1].reshape(-1), b[::-1, :].reshape(-1), b[::-1, ::-1].reshape(-1)]
    V = O.init_v0(inst); s = 0
    while True:
        r = O.gauss_seidel(inst, ords[s % 4], V0=V, tol=0, max_sweeps=1); V = r["V"]; s += 1
        if r["residual"] < tol or s > 3000: return s, V

for cfg, n in [("C5", 31), ("C4", 31), ("C2", 31), ("C5", 129), ("C5", 257), ("C5", 513)]:
    inst = I.make_config(cfg, n=n)
    fs, Vf = fastsweep(inst, 1e-7)
    J = O.jacobi(inst, tol=1e-7)
    out = [cfg, n, "oracle jacobi", J["sweeps"], "fastsweep", fs]
    for kern in (0, 3):
        s = Solver(inst, precision=32)
        s.build_static(*inst.static_blocks)
        st = s.solve("static", tol=1e-7, k_inner=4, kernel=kern)
        out += [f"k{kern}: rounds", st["rounds"], "sweeps_eq", round(st["node_updates"] / inst.free_count(), 1),
                "err", float(np.abs(s.get_values() - Vf).max())]
        s.close()
    print(*out, flush=True)
