"""GPU analogue of the paper's Tables 1 and 2: PDD (patchy pipeline,
including the pre-computation, as the paper's PDD times do) vs DD (static four squares) on the
eikonal-diffusion and Zermelo exit problems, fine grids 100^2 .. 800^2 cells, eps swept across
the upwind diffusion ball threshold.  Reports wall time on the stream, sweep-equivalents (node
updates / free nodes: the GPU analogue of the paper's iteration count) and the regime flag from
pdd_regime_analyse.  fp64, tol 1e-9.  Output: one JSON line per cell (stdout)."""
import argparse, json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import pdd_inputs as I
from paper_1502_01629_b200 import Solver, regime_analyse

T1 = [1e-9, 1e-8, 1e-7, 1e-6, 1e-5, 1e-4, 6.25e-4, 1.25e-3, 2.5e-3, 5e-3, 1e-2]
T2 = [1e-9, 1e-8, 1e-7, 1e-6, 1e-5, 0.0025 / 120, 0.005 / 120, 0.01 / 120, 0.02 / 120, 1e-3, 5e-3]
ap = argparse.ArgumentParser()
ap.add_argument("--cells", default="100,200,400,800")
ap.add_argument("--problems", default="eikonal,zermelo")
ap.add_argument("--precision", type=int, default=64)
ap.add_argument("--tol", type=float, default=1e-9)
a = ap.parse_args()
for problem in a.problems.split(","):
    for cells in map(int, a.cells.split(",")):
        for eps in (T1 if problem == "eikonal" else T2):
            inst = I.paper_instance(problem, cells, eps)
            fmin, fmax = I.PAPER_FMINMAX[problem]
            reg = regime_analyse(fmin, fmax, math.sqrt(2 * eps), inst.dx)
            s = Solver(inst, precision=a.precision)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            cs = s.coarse_solve(inst.tol_coarse)
            s.synthesize()
            s.build_patches(inst.n_patches)
            sp = s.solve("patchy", tol=a.tol, max_rounds=10 ** 6)
            e1.record(); torch.cuda.synchronize()
            t_pdd = e0.elapsed_time(e1) * 1e-3
            s.build_static(*inst.static_blocks)
            sd = s.solve("static", tol=a.tol, max_rounds=10 ** 6)
            s.close()
            free = inst.free_count()
            print(json.dumps(dict(problem=problem, cells=cells, dx=inst.dx, eps=eps,
                                  hyperbolic=reg["hyperbolic"], h_over_dx=inst.h / inst.dx,
                                  pdd_s=round(t_pdd, 5), pdd_sweq=round(sp["node_updates"] / free, 2),
                                  pdd_rounds=sp["rounds"], coarse_sweeps=cs["sweeps"],
                                  dd_s=round(sd["seconds_total"], 5),
                                  dd_sweq=round(sd["node_updates"] / free, 2), dd_rounds=sd["rounds"],
                                  kernel=sp["kernel_used"])), flush=True)
