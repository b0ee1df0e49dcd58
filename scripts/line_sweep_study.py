"""Convergence study (fp64, oracle operator): point Gauss-Seidel in 4 orientations vs line
sweeps (a whole row updated from the values before the row: Jacobi along the line, Gauss-Seidel
across lines), rows only or alternating rows/columns.  Development aid for the tensor-core
design study in DESIGN.md; not part of the product."""
import argparse, time
import numpy as np
import oracle as O
import pdd_inputs as I

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="C5"); ap.add_argument("--n", type=int, default=257)
ap.add_argument("--tol", type=float, default=1e-9); ap.add_argument("--max", type=int, default=3000)
a = ap.parse_args()
inst = I.make_config(a.cfg, n=a.n)
n = inst.n
free = (np.asarray(inst.kind).reshape(n, n) == 0)
ref = O.jacobi(inst, tol=1e-13 * (1 - inst.beta), max_sweeps=10**6)["V"]

def run(kind):
    V = O.init_v0(inst).copy()
    t0 = time.time()
    for s in range(1, a.max + 1):
        old = V.copy()
        o = s % 4
        if kind == "point":
            ys = range(n) if o in (0, 1) else range(n - 1, -1, -1)
            xs = np.arange(n) if o in (0, 2) else np.arange(n - 1, -1, -1)
            idx = np.concatenate([y * n + xs for y in ys])
            V = O.gauss_seidel(inst, idx, V0=V, tol=0.0, max_sweeps=1)["V"]
        else:
            cols = kind == "rowcol" and (s // 2) % 2 == 1
            lines = range(n) if s % 2 == 0 else range(n - 1, -1, -1)
            for l in lines:
                idx = (np.arange(n) * n + l) if cols else (l * n + np.arange(n))
                out, _ = O.apply_at(inst, V, idx)
                V[idx] = np.where(free.reshape(-1)[idx], out, V[idx])
        r = np.abs(V - old).max()
        if r < a.tol:
            break
    return s, np.abs(V - ref).max(), time.time() - t0

for k in ("point", "rows", "rowcol"):
    print(k, run(k), flush=True)
