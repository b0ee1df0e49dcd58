"""A/B of the canonical fp64 pre-computation kernels (coarse sweep, synthesis) on one config:
device time of pdd_coarse_solve and pdd_synthesize, a SHA-256 of u_c and a* (variants must be
bit-identical).  PDD_LIB selects the build."""
import argparse, hashlib, json, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
import torch
import pdd_inputs as I
from paper_1502_01629_b200 import Solver, _native
if os.environ.get("PDD_LIB"):
    _native.use_library(os.environ["PDD_LIB"])
ap = argparse.ArgumentParser(); ap.add_argument("--cfg", default="C5"); ap.add_argument("--n", type=int, default=None)
a = ap.parse_args()
inst = I.make_config(a.cfg, n=a.n)
s = Solver(inst, precision=32)
def dev_ms(fn, reps=3):
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(); r = fn(); e1.record(); torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return out, r
tc, cs = dev_ms(lambda: s.coarse_solve(inst.tol_coarse))
ts, _ = dev_ms(lambda: s.synthesize())
h = hashlib.sha256(s.get_coarse_values().tobytes()).hexdigest()[:16]
ha = hashlib.sha256(s.get_controls().tobytes()).hexdigest()[:16]
print(json.dumps(dict(lib=os.environ.get("PDD_LIB", "product"), cfg=a.cfg, coarse_ms=[round(x, 2) for x in tc],
                      coarse_stats_s=cs["seconds"], sweeps=cs["sweeps"], synth_ms=[round(x, 2) for x in ts], uc_sha=h, astar_sha=ha)))
