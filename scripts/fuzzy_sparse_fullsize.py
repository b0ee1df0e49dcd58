"""Sparse fuzzy patches at full size (C5: 8193^2, 256 patches, K = 4): run once, report the sweep
count, time, overlap degree and decomposition quality, then the patchy solve on those patches."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import pdd_inputs as I
from paper_1502_01629_b200 import Solver

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4
eps_P = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-2
inst = I.make_config(cfg)
s = Solver(inst, precision=32)
s.coarse_solve(inst.tol_coarse); s.synthesize()
t = time.time()
st = s.build_fuzzy_patches_sparse(inst.n_patches, K=K, eps_P=eps_P, tau_P=0.3)
wall = time.time() - t
lab = s.get_labels()
free = inst.kind == I.KIND_FREE
own = lab[free]
out = dict(config=cfg, n=inst.n, patches=inst.n_patches, K=K, eps_P=eps_P, sweeps=st["sweeps"],
           seconds=st["seconds"], wall=wall, converged=st["converged"], overlap_nodes=st["overlap_nodes"],
           longest_list=st["max_list"], orphan_fraction=float((own == inst.n_patches).mean()),
           patches_used=int(np.unique(own[own < inst.n_patches]).size),
           scratch_gb=(20 * K * inst.n * inst.n + 512) / 1e9)
sol = s.solve("patchy", tol=inst.tol)
out.update(solve_converged=sol["converged"], solve_seconds=sol["seconds_total"],
           patches_active=sol["patches_active"], patches_converged=sol["patches_converged"])
s.build_patches(inst.n_patches)
lab2 = s.get_labels()
out["owner_agreement_with_successor_labels"] = float((lab2[free] == own).mean())
print(json.dumps(out))
