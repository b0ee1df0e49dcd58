"""Node-updates done by one device-driven round of the C5 solve (for the ncu traffic per
node-update): runs the same solve as scripts/profile_sweep.py capped at R and at R+1 rounds."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pdd_inputs as I
from paper_1502_01629_b200 import Solver
ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="C5"); ap.add_argument("--mode", default="patchy")
ap.add_argument("--k", type=int, default=1); ap.add_argument("--round", type=int, default=151)
a = ap.parse_args()
inst = I.make_config(a.cfg)
out = []
for R in (a.round - 1, a.round):
    s = Solver(inst, precision=32)
    s.coarse_solve(inst.tol_coarse); s.synthesize(); s.build_patches(inst.n_patches)
    if a.mode == "static":
        s.build_static(*inst.static_blocks)
    st = s.solve(a.mode, tol=1e-6, k_inner=a.k, max_rounds=R, raise_on_noconverge=False, trace=True)   # one round per batch: exact cap
    out.append(st["node_updates"]); s.close()
print(json.dumps({"cfg": a.cfg, "mode": a.mode, "k": a.k, "round": a.round,
                  "node_updates_in_round": out[1] - out[0]}))
