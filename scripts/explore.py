"""Ad-hoc exploration of solve parameters on one config (GPU).  Not part of the product."""
import argparse, json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import pdd_inputs as I
from paper_1502_01629_b200 import Solver, _native
if os.environ.get("PDD_LIB"):          # A/B builds (scripts/ab*.sh); the product path loads the in-tree lib
    _native.use_library(os.environ["PDD_LIB"])

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="C5"); ap.add_argument("--n", type=int, default=None)
ap.add_argument("--paper", default=None, help="problem:cells:eps (paper_instance)")
ap.add_argument("--general", default=None, help="cost:sigma:n:eps:n_coarse (general_instance)")
ap.add_argument("--prec", type=int, default=32); ap.add_argument("--k", default="0")
ap.add_argument("--modes", default="patchy,static"); ap.add_argument("--tol", type=float, default=1e-6)
ap.add_argument("--kernel", type=int, default=0); ap.add_argument("--delta", default="0")
ap.add_argument("--max_rounds", type=int, default=200000); ap.add_argument("--schedule", default="rounds"); ap.add_argument("--policy", type=int, default=0); ap.add_argument("--qt", type=int, default=0); ap.add_argument("--cols", type=int, default=0)
a = ap.parse_args()
t = time.time()
if a.paper:
    pb, ce, ep = a.paper.split(":")
    inst = I.paper_instance(pb, int(ce), float(ep))
elif a.general:
    co, sg, nn, ep, nc = a.general.split(":")
    inst = I.general_instance(int(nn), cost=int(co), sigma=int(sg), eps=float(ep), n_coarse=int(nc))
else:
    inst = I.make_config(a.cfg, n=a.n)
print("gen", time.time() - t, flush=True)
t = time.time(); s = Solver(inst, precision=a.prec); torch.cuda.synchronize(); print("create", time.time() - t, flush=True)
cs = s.coarse_solve(inst.tol_coarse); print("coarse", cs, flush=True)
if a.cols: s.set_tile_cols(a.cols)
t = time.time(); s.synthesize(); s.build_patches(inst.n_patches); print("synth+patches", time.time() - t, flush=True)
for mode in a.modes.split(","):
    if mode == "static": s.build_static(*inst.static_blocks)
    else: s.build_patches(inst.n_patches)
    for k in map(int, a.k.split(",")):
        for d in map(float, a.delta.split(",")):
            t = time.time()
            st = s.solve(mode, tol=a.tol, k_inner=k, kernel=a.kernel, delta=d, max_rounds=a.max_rounds, schedule=a.schedule, bucket_policy=a.policy, queue_target=a.qt, raise_on_noconverge=False)
            wall = time.time() - t
            nu = st["node_updates"]
            print(json.dumps(dict(mode=mode, k=k, delta=d, wall=round(wall, 3), rounds=st["rounds"], conv=st["converged"],
                  nu=nu, sweeps_equiv=round(nu / inst.free_count(), 1), t_total=round(st["seconds_total"], 3),
                  t_sweep=round(st["seconds_sweep"], 3), t_verify=round(st["seconds_verify"], 4),
                  kern_nups=f"{nu / max(st['seconds_sweep'],1e-9):.3e}", res=st["final_residual"], kernel=st["kernel_used"],
                  tiles=st["tiles_processed"], ntiles=st["n_tiles"])), flush=True)
            L = _native.lib()
            if hasattr(L, "pdd_dev_phases"):      # PDD_TIMING builds: cycles per visit phase
                import ctypes
                ph = (ctypes.c_ulonglong * 8)()
                L.pdd_dev_phases(ph)
                tot = float(sum(ph)) or 1.0
                names = ["fetch/idle", "stage-load", "convert", "sweep", "reduce", "writeback", "queue-ops", "admit"]
                print("phases: " + ", ".join(f"{nm} {100 * v / tot:.1f}%" for nm, v in zip(names, ph)) +
                      f"  (total {tot:.3e} CTA-cycles)", flush=True)
