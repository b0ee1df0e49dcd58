"""Where does the end-to-end (host-buffer) step spend its time?  Dev tool."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import pdd_inputs as I
from paper_1502_01629_b200 import Solver
inst = I.make_config("C5")
views = Solver.make_views(inst, pin_host=True)
hostV = torch.empty(inst.n * inst.n, dtype=torch.float32).pin_memory()
for it in range(3):
    torch.cuda.synchronize(); t = [time.perf_counter()]
    s = Solver(inst, precision=32, views=views); torch.cuda.synchronize(); t.append(time.perf_counter())
    s.coarse_solve(inst.tol_coarse); t.append(time.perf_counter())
    s.synthesize(); t.append(time.perf_counter())
    s.build_patches(inst.n_patches); t.append(time.perf_counter())
    st = s.solve("patchy", tol=inst.tol, k_inner=4); t.append(time.perf_counter())
    s.get_values_into(hostV, on_device=False, as_fp64=False); t.append(time.perf_counter())
    s.close(); torch.cuda.synchronize(); t.append(time.perf_counter())
    names = ["create", "coarse", "synth", "patches", "solve", "get_values", "close"]
    print(" ".join(f"{n}={1e3*(b-a):.1f}ms" for n, a, b in zip(names, t, t[1:])), f"solve_dev={st['seconds_total']*1e3:.1f}ms", flush=True)
