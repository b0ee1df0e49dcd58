"""Run the C5 patchy pipeline for a bounded number of fine-solve rounds (for ncu captures of the
steady-state sweep kernel).  Not part of the product."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import pdd_inputs as I
from paper_1502_01629_b200 import Solver
ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="C5"); ap.add_argument("--n", type=int, default=None)
ap.add_argument("--rounds", type=int, default=40); ap.add_argument("--prec", type=int, default=32)
ap.add_argument("--mode", default="patchy"); ap.add_argument("--k", type=int, default=4)
a = ap.parse_args()
inst = I.make_config(a.cfg, n=a.n)
s = Solver(inst, precision=a.prec)
s.coarse_solve(inst.tol_coarse); s.synthesize(); s.build_patches(inst.n_patches)
if a.mode == "static": s.build_static(*inst.static_blocks)
st = s.solve(a.mode, tol=1e-6, k_inner=a.k, max_rounds=a.rounds, raise_on_noconverge=False)
torch.cuda.synchronize()
print({k: st[k] for k in ("rounds", "node_updates", "seconds_sweep", "tiles_processed")})
