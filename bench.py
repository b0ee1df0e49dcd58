"""bench.py -- the hot path of arXiv 1502.01629 on B200, BASELINE.json metric
"SL sweep node-updates/s, time-to-converge patchy vs static (1 B200)".

A step = one pass of the whole hot path on config C5
(8193^2 Zermelo navigation, 64 controls, 4 Markov branches, fp32 arithmetic): coarse solve on
513^2 -> prolongation -> synthesis -> patch labels (256 patches) -> patchy fine solve until the
full-grid Jacobi residual is < 1e-7 (verified; at 1e-7 the fp32 V is within 1e-6 max|V| of the
certified fp64 fixed point).  Inputs are resident in HBM when the timed
region starts (the problem arrays are uploaded once by pdd_create); V (fp64, 537 MB) and the
other per-node arrays are larger than L2, so no flush is needed between steps.

value      = free-node updates performed by the sweep kernel in the K timed steps, all ranks,
             / max-over-ranks device time of the K steps (CUDA events, barrier + sync on both
             sides).
e2e        = same metric through the C ABI with HOST buffers: every step creates the context
             from pinned host arrays (H2D inside the timed region), runs the pipeline and copies
             V back to pinned host memory (D2H).
roofline   = the sweep kernel (k_sweep_queue, the persistent work-queue launch): algorithmic fp32
             flop per node-update F = N_A * (15 * 2p + 10) (4480 at C5; the
             bilinear reconstructions alone, N_A 2p x 4 FMA = 2048, are reported as
             frac_bilinear_only) times the updates of the timed region / the summed duration of
             the sweep launches (CUDA events on the launching stream); peak = the FP32 FFMA rate
             MEASURED on the box by libpdd's micro-benchmark (pdd_measure_alu_peaks; the derived
             148 SMs x 128 lanes x 2 flop x 1965 MHz = 74.4 TFLOP/s is reported beside it);
             "bound": "alu"; traffic = DRAM bytes per node-update of the committed ncu capture
             (profiles/sweep_traffic.json) x the node-updates per launch.
accuracy_run = the same pipeline in fp64 arithmetic (BASELINE config C5: "fp32 with an fp64
             accuracy run") and max |V32 - V64| / max|V|, computed on the device.
oracle_time_to_converge = MEASURED plain-Jacobi oracle solves (C1, C2 by default); C5's figure in
             time_to_converge is extrapolated and named so.
cpu_baseline = the fp64 oracle (oracle/, plain C + OpenMP on all host cores) applying the same
             operator T to a bounded sample of the same grid (a band of rows of C5), in
             node-updates/s.

--impl reference : the oracle as the reference arm (this tier has no reference code): each step
             is a bounded sample (one oracle Jacobi application to a band of C5 rows).
--gpus N (torchrun): "replicas only": every rank solves its own copy; value sums
             the ranks' updates over the max-over-ranks time; scaling "weak".
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SL sweep node-updates/s, time-to-converge patchy vs static (1 B200)"
UNIT = "node-updates/s"
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12      # 74.4
FP64_PEAK_TFLOPS = FP32_PEAK_TFLOPS / 2.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--n", type=int, default=None, help="override grid size (not for the headline)")
    ap.add_argument("--precision", type=int, default=32)
    ap.add_argument("--k-inner", type=int, default=None,
                    help="sweeps per tile visit (default: the API's per-mode default, 1 patchy / 4 static)")
    ap.add_argument("--tol", type=float, default=1e-7)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-static", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-others", action="store_true",
                    help="skip the time-to-converge report of the other BASELINE configs")
    ap.add_argument("--no-accuracy-run", action="store_true",
                    help="skip the fp64 accuracy run of the same pipeline (BASELINE config C5: fp32 with an fp64 accuracy run)")
    ap.add_argument("--oracle-ttc", default="C1,C2",
                    help="configs whose oracle (plain fp64 Jacobi, host cores) time-to-converge is MEASURED "
                         "(cfg or cfg@n, comma separated; C3@1025 takes minutes; '' = none)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- distributed
def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce(val, op, world):
    if world == 1:
        return val
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(val)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return float(t.item())


def aggregate(node_updates, seconds, world):
    """Replicas-only aggregation: value = all ranks' node-updates / the slowest rank's device
    time (max over ranks; never a wall clock)."""
    import torch.distributed as dist
    if world == 1:
        return node_updates, seconds, node_updates / seconds
    t_max = allreduce(seconds, dist.ReduceOp.MAX, world)
    nu = allreduce(node_updates, dist.ReduceOp.SUM, world)
    return nu, t_max, nu / t_max


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- oracle legs
def oracle_sample(inst, seconds: float):
    """Time the oracle's operator T (fp64, all host cores) on a band of rows of ``inst``,
    sized to take about ``seconds``.  Returns (node-updates/s, description, threads)."""
    import numpy as np
    import oracle as O
    n = inst.n
    V = O.init_v0(inst)
    rows0 = max(8, min(n, 64))
    idx = np.arange(n * (n // 2), n * (n // 2) + rows0 * n, dtype=np.int64)
    t = time.perf_counter()
    O.apply_at(inst, V, idx)
    dt = max(time.perf_counter() - t, 1e-6)
    rate = idx.size / dt
    rows = int(min(n, max(rows0, seconds * rate / n)))
    j0 = max(0, n // 2 - rows // 2)
    idx = np.arange(j0 * n, (j0 + rows) * n, dtype=np.int64)
    t = time.perf_counter()
    O.apply_at(inst, V, idx)
    dt = time.perf_counter() - t
    desc = (f"one fp64 application of the scheme's operator T (oracle, {O.num_threads()} threads) "
            f"to {rows} full rows ({idx.size} nodes) of the {inst.name} grid ({n}^2), "
            f"{dt:.1f} s")
    return idx.size / dt, desc, O.num_threads(), dt


def workload_config(inst, args, world):
    """The workload both arms are quoted on (BASELINE.json configs[4] by default)."""
    return {"workload": f"{inst.name}: patchy pipeline (coarse {inst.coarse.n}^2 solve,"
                        f" synthesis, {inst.n_patches} patch labels, fine solve to "
                        f"tol {args.tol:g}) on {inst.n}^2",
            "grid": inst.n, "controls": inst.n_controls, "branches": 2 * inst.p,
            "patches": inst.n_patches,
            "k_inner": args.k_inner if args.k_inner is not None else {"patchy": "auto (1)", "static": "auto (4)"},
            "schedule": "work queue (persistent sweep CTAs, key-order admission), then full-grid verification",
            "path3_tile": {"patchy": "16x64" if ((inst.n + 63) // 64) * ((inst.n + 31) // 32) <= 16384 else "32x64",
                           "static": "16x128" if 128 * inst.dx <= 0.125 + 1e-12 else "32x64"},
            "l2": "inputs larger than L2 (V fp64 %d MB)" % (inst.n * inst.n * 8 >> 20),
            "parallelism": f"replicas x{world}" if world > 1 else "single GPU"}


def run_reference(args, world, rank):
    import pdd_inputs as I
    import oracle as O
    if rank != 0:
        return
    inst = I.make_config(args.config, n=args.n)
    per = max(2.0, min(args.cpu_seconds, 60.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        oracle_sample(inst, per / 4)
    vals, times, desc = [], [], ""
    for _ in range(args.steps):
        v, desc, thr, dt = oracle_sample(inst, per)
        vals.append(v)
        times.append(dt)
    value = sum(vals) / len(vals)
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        # the same workload as our arm; each step is a bounded sample of it (cpu_baseline.sample):
        # the oracle's node-update rate on the fine grid of that config
        "config": workload_config(inst, args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": thr, "kind": "oracle",
                         "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


def oracle_time_to_converge(spec: str):
    """Measured wall time of the oracle's plain Jacobi value iteration to the config's tolerance
    (fp64, all host cores): the CPU side of the paper's time-to-converge comparison."""
    import pdd_inputs as I
    import oracle as O
    out = {}
    for item in [x for x in spec.split(",") if x]:
        cfg, _, nn = item.partition("@")
        inst = I.make_config(cfg, n=int(nn) if nn else None)
        t = time.perf_counter()
        r = O.jacobi(inst, tol=inst.tol, max_sweeps=10**6)
        dt = time.perf_counter() - t
        out[item] = {"grid": inst.n, "tol": inst.tol, "sweeps": int(r["sweeps"]), "seconds": dt,
                     "threads": O.num_threads(), "kind": "measured",
                     "node_updates_per_s": inst.free_count() * int(r["sweeps"]) / dt}
    return out


def decomposition_quality(s, inst):
    """Orphan fraction and non-empty patch count of the patch labels held by the solver."""
    import numpy as np
    import pdd_inputs as I
    lab = s.get_labels()
    own = lab[inst.kind == I.KIND_FREE]
    return {"patches": int(inst.n_patches), "orphan_fraction": float((own == inst.n_patches).mean()),
            "patches_nonempty": int(np.unique(own[(own >= 0) & (own < inst.n_patches)]).size)}


# ----------------------------------------------------------------------------- our arm
def pipeline_step(s, inst, args, mode="patchy"):
    """One pass of the hot path on a resident context; returns the fine-solve stats."""
    if mode == "patchy":
        s.coarse_solve(inst.tol_coarse)
        s.synthesize()
        s.build_patches(inst.n_patches)
    else:
        s.build_static(*inst.static_blocks)
    return s.solve(mode, tol=args.tol, k_inner=args.k_inner)


def main():
    args = parse()
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        barrier(world)
        return
    import numpy as np
    import torch
    import torch.distributed as dist
    import pdd_inputs as I
    from paper_1502_01629_b200 import Solver, measure_alu_peaks

    torch.cuda.set_device(local)
    inst = I.make_config(args.config, n=args.n)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    s = Solver(inst, precision=args.precision, device=str(dev))

    for _ in range(args.warmup):
        pipeline_step(s, inst, args)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier(world)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = s.kernel_launches()
    ev0.record(stream)
    nu, t_sweep, t_verify, rounds, t_solve, sweep_launches = 0, 0.0, 0.0, 0, 0.0, 0
    for _ in range(args.steps):
        st = pipeline_step(s, inst, args)
        assert st["converged"] == 1
        nu += st["node_updates"]
        t_sweep += st["seconds_sweep"]
        t_verify += st["seconds_verify"]
        t_solve += st["seconds_total"]
        rounds += st["rounds"]
        sweep_launches += st["rounds"] - st["verify_passes"]
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    launches = s.kernel_launches() - l0
    clk = clocks.stop()
    t_local = ev0.elapsed_time(ev1) * 1e-3
    nu_all, t_max, value = aggregate(nu, t_local, world)
    last = st
    decomp = decomposition_quality(s, inst) if rank == 0 else None
    # roofline denominators measured on this box (FFMA and LDS.128 micro-benchmarks of libpdd)
    alu = measure_alu_peaks(5)

    # fp64 accuracy run (BASELINE.json C5: "fp32 with an fp64 accuracy run"): the same pipeline in
    # fp64 arithmetic on a second context, compared with the fp32 V on the device
    accuracy = None
    if not args.no_accuracy_run and rank == 0 and args.precision == 32:
        N = inst.n * inst.n
        V32 = torch.empty(N, dtype=torch.float64, device=dev)
        s.get_values_into(V32, on_device=True)
        s64 = Solver(inst, precision=64, device=str(dev))
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        st64 = pipeline_step(s64, inst, args)
        a1.record(stream)
        torch.cuda.synchronize()
        V64 = torch.empty(N, dtype=torch.float64, device=dev)
        s64.get_values_into(V64, on_device=True)
        vmax = float(V64.abs().max().item())
        accuracy = {"fp64_pipeline_s": a0.elapsed_time(a1) * 1e-3, "fp64_solve_s": st64["seconds_total"],
                    "fp64_converged": st64["converged"], "fp64_final_residual": st64["final_residual"],
                    "fp64_apost_bound": st64["apost_bound"], "fp64_kernel": st64["kernel_used"],
                    "fp64_kernel_node_updates_per_s": st64["node_updates"] / max(st64["seconds_sweep"], 1e-12),
                    "fp64_sweep_equivalents": st64["node_updates"] / inst.free_count(),
                    "max_abs_fp32_minus_fp64": float((V32 - V64).abs().max().item()),
                    "max_abs_V": vmax,
                    "rel_to_max_V": float((V32 - V64).abs().max().item()) / vmax,
                    "bar": "north_star: fp32 within 5e-5 max|V| (the fp64 V is within apost_bound of the fixed point)"}
        s64.close()
        del s64, V32, V64

    # static decomposition on the same kernels (time-to-converge comparison)
    static = None
    if not args.no_static:
        sst = pipeline_step(s, inst, args, mode="static")
        static = {"time_to_converge_s": sst["seconds_total"], "rounds": sst["rounds"],
                  "node_updates": sst["node_updates"],
                  "sweep_equivalents": sst["node_updates"] / inst.free_count(),
                  "kernel_node_updates_per_s": sst["node_updates"] / max(sst["seconds_sweep"], 1e-12),
                  "converged": sst["converged"], "final_residual": sst["final_residual"]}

    # end to end through the C ABI with host buffers
    e2e = None
    if not args.no_e2e:
        views = Solver.make_views(inst, pin_host=True)
        hostV = torch.empty(inst.n * inst.n, dtype=torch.float64 if args.precision == 64 else torch.float32).pin_memory()
        h2d = sum(int(a.nbytes) for v in views if v is not None for a in v._keep
                  if hasattr(a, "nbytes") and not hasattr(a, "pin_memory"))
        del s
        torch.cuda.synchronize()
        barrier(world)
        # device-timed (CUDA events on the stream; host gaps between the calls are inside the
        # interval because the events complete in stream order)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e_nu = 0
        for _ in range(max(1, min(args.steps, 2))):
            se = Solver(inst, precision=args.precision, device=str(dev), views=views, stream=stream)
            st_e = pipeline_step(se, inst, args)
            se.get_values_into(hostV, on_device=False, as_fp64=(args.precision == 64))
            e_nu += st_e["node_updates"]
            se.close()
            del se
        e1.record(stream)
        torch.cuda.synchronize()
        e_nu, t_e, _ = aggregate(e_nu, e0.elapsed_time(e1) * 1e-3, world)
        e2e = {"value": e_nu / t_e, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": int(hostV.numel() * hostV.element_size())}

    # F = N_A (15 * 2p + 10) algorithmic flop per node-update (per branch: 2 FADD
    # offset, 2 FADD frac, 3 lerps = 3 FADD + 3 FFMA, 1 accumulate, 1 Lambda0 op; per control: 2
    # FFMA base offset, numerator and denominator FFMA, div, min); the conservative count of the
    # bilinear reconstructions alone (N_A 2p x 4 FMA) is reported beside it
    nbr = 2 * inst.p if inst.p > 0 else 1
    flop_per_update = inst.n_controls * (15 * nbr + 10)
    flop_bilinear = inst.n_controls * nbr * 4 * 2
    achieved = flop_per_update * nu / max(t_sweep, 1e-12) / 1e12
    peak32 = alu["fp32_tflops"] if alu["fp32_tflops"] > 0 else FP32_PEAK_TFLOPS
    peak64 = alu["fp64_tflops"] if alu.get("fp64_tflops", 0) > 0 else peak32 / 2.0
    peak = peak32 if args.precision == 32 else peak64
    roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": None,
            "flop_basis": "SURVEY.md 8(d): F = N_A (15 * 2p + 10) per node-update",
            "flop_per_node_update_bilinear_only": flop_bilinear,
            "frac_bilinear_only": flop_bilinear * nu / max(t_sweep, 1e-12) / 1e12 / peak,
            "kernel": {1: "k_sweep path 1 (general stencil)",
                       2: "k_sweep path 2 (row-table stencil, one node per warp step)",
                       3: "k_sweep_queue path 3 (row-table stencil, in-tile Gauss-Seidel, 4 nodes per "
                          "step; persistent CTAs on the tile work queue)",
                       4: "k_sweep_queue path 4 (lean general stencil)"}
                      .get(last["kernel_used"], "k_sweep"),
            "flop_per_node_update": flop_per_update,
            "kernel_node_updates_per_s": nu / max(t_sweep, 1e-12),
            "kernel_seconds_share_of_step": t_sweep / max(t_local, 1e-12),
            "peak_basis": ("measured on this GPU: FFMA micro-benchmark of libpdd (pdd_measure_alu_peaks, best "
                           "of 5; fp64: its DFMA twin); derived figure 148 SM x 128 lanes x 2 x 1.965 GHz = "
                           "%.1f TFLOP/s" % FP32_PEAK_TFLOPS),
            "peak_derived": FP32_PEAK_TFLOPS if args.precision == 32 else FP64_PEAK_TFLOPS,
            "frac_of_derived_peak": achieved / (FP32_PEAK_TFLOPS if args.precision == 32 else FP64_PEAK_TFLOPS),
            "smem_peak_tbs_measured": alu["smem_tbs"], "fp64_peak_tflops_measured": alu.get("fp64_tflops"),
            "step": {"patchy_fine_solve_s": t_solve / args.steps, "patchy_pipeline_s": t_max / args.steps,
                     "static_solve_s": static["time_to_converge_s"] if static else None,
                     "static_over_patchy_pipeline": (static["time_to_converge_s"] / (t_max / args.steps)) if static else None},
            "sweep_launches_per_step": sweep_launches / args.steps}
    if accuracy:
        accuracy["fp64_kernel_alu_frac"] = accuracy["fp64_kernel_node_updates_per_s"] * flop_per_update / 1e12 / peak64
        accuracy["fp64_peak_tflops_measured"] = peak64
    if static:
        # the same kernel in the static solve's full rounds (16 x 128 path-3 tiles at C4/C5,
        # runtime.cu p3_use_wide; the patchy step above runs 32 x 64 tiles)
        static["kernel_alu_frac"] = static["kernel_node_updates_per_s"] * flop_per_update / 1e12 / peak
    prof = os.path.join(ROOT, "profiles", "sweep_traffic.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            per_launch_updates = nu / max(1, sweep_launches)
            roof["traffic"] = pj["dram_bytes_per_node_update"] * per_launch_updates
            roof["algorithmic_bytes_per_launch"] = pj.get("algorithmic_bytes_per_node_update", 18.4) * per_launch_updates
            if "ncu_pipes" in pj:
                roof["ncu"] = pj["ncu_pipes"]
            roof["traffic_basis"] = ("dram bytes per node-update from ncu --set full (%s) x the "
                                     "average node-updates per sweep launch of this run; "
                                     "algorithmic bytes per node-update ~18.4 at one sweep per visit "
                                     "(tile + halo fp64 read, fp64 write, kinds)" % pj["source"])
        except Exception:
            pass

    # the other BASELINE configs at full size (time-to-converge only; not the headline): patchy
    # pipeline (coarse solve .. verified fine solve) and static solve on the same kernels
    others = None
    if not args.no_others and rank == 0 and args.n is None:
        others = {}
        for cfg in ("C1", "C2", "C3", "C4"):
            if cfg == args.config:
                continue
            ci = I.make_config(cfg)
            prec = 64 if cfg == "C1" else args.precision
            so = Solver(ci, precision=prec, device=str(dev))
            rec = {"grid": ci.n, "precision": prec, "tol": ci.tol}
            flop_o = ci.n_controls * (15 * (2 * ci.p if ci.p > 0 else 1) + 10)
            peak_o = peak32 if prec == 32 else peak64
            for mode in (("static",) if ci.coarse is None else ("patchy", "static")):
                pipeline_step(so, ci, args, mode=mode)                       # warm-up
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                if mode == "patchy":
                    so.coarse_solve(ci.tol_coarse)
                    so.synthesize()
                    so.build_patches(ci.n_patches)
                else:
                    so.build_static(*ci.static_blocks)
                sto = so.solve(mode, tol=ci.tol)
                e1.record(stream)
                torch.cuda.synchronize()
                rec[mode] = {"pipeline_s": e0.elapsed_time(e1) * 1e-3,
                             "solve_s": sto["seconds_total"],
                             "sweep_equivalents": sto["node_updates"] / ci.free_count(),
                             "kernel_node_updates_per_s": sto["node_updates"] / max(sto["seconds_sweep"], 1e-12),
                             "kernel": sto["kernel_used"], "converged": sto["converged"]}
                rec[mode]["kernel_alu_frac"] = rec[mode]["kernel_node_updates_per_s"] * flop_o / 1e12 / peak_o
                if mode == "patchy":
                    rec["decomposition"] = decomposition_quality(so, ci)
            so.close()
            del so
            others[cfg] = rec

    cpu = None
    ottc = None
    if not args.no_cpu and rank == 0 and world == 1:
        v, desc, thr, _ = oracle_sample(inst, args.cpu_seconds)
        cpu = {"value": v, "unit": UNIT, "cores": thr, "kind": "oracle", "sample": desc}
        ottc = oracle_time_to_converge(args.oracle_ttc)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if args.precision == 32 else "f64", "data": "synthetic",
            "config": workload_config(inst, args, world),
            "time_to_converge": {"patchy_s": t_solve / args.steps,
                                 "patchy_pipeline_s": t_max / args.steps,
                                 "static_s": static["time_to_converge_s"] if static else None,
                                 "rounds_patchy": rounds // args.steps,
                                 "sweep_equivalents_patchy": nu / args.steps / inst.free_count()},
            "static": static,
            "decomposition": decomp,
            "accuracy_run": accuracy,
            "other_configs": others,
            "oracle_time_to_converge": ottc,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
        }
        # SURVEY.md 8(d) metric 2, work-normalised speed: free nodes x the oracle's Jacobi sweep count
        # (C5: ~0.71 n sweeps, extrapolated from the measured 513^2 / 1025^2 oracle runs) / GPU time
        out["time_to_converge"]["effective_node_updates_per_s_vs_jacobi"] = (
            inst.free_count() * 0.71 * inst.n / (t_max / args.steps))
        if cpu:
            # EXTRAPOLATED (not measured): plain-Jacobi oracle sweeps ~ 0.71 n (
            # the measured oracle solves of the smaller configs are in oracle_time_to_converge)
            out["time_to_converge"]["oracle_jacobi_extrapolated_s"] = (
                inst.free_count() * 0.71 * inst.n / cpu["value"])
        print(json.dumps(out), flush=True)
    barrier(world)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
