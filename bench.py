#!/usr/bin/env python
"""DDM hot-path benchmark (BASELINE.json metric: DDM iterations/s and
Munknown-iters/s at 1 GPU; achieved HBM GB/s vs peak).

Workload: BASELINE config 4 (2048^2, 16x16 subdomains, overlap 8, PML 24,
20 random layers, complex fp64) -- the north star's target configuration.
A "step" is one DDM iteration (DdmEngine::sweep, proj/src/ddm.cpp:174-214) of the
preconditioner M = precondition(r, K) used inside FGMRES(30) (cli.cpp:210-228);
the timed region is ONE precondition call of exactly --steps sweeps on a dense
seeded residual vector already resident in HBM (what FGMRES feeds it after its
first iteration). Factor data (~1 GB) and per-subdomain vectors (~0.8 GB) exceed
the 126 MB L2, so no flush is needed between steps.

value      = DDM iterations/s over all ranks (replicas, weak scaling)
e2e        = the full FGMRES(30)+DDM(K=32) solve to 1e-6 through the public C-ABI
             with HOST buffers (b in, x out), DDM iterations/s = iters*K / wall
roofline   = the batched supernodal solve stage: algorithmic bytes
             (B_fac + B_vec) / its CUDA-event duration
cpu_baseline = the unmodified reference (oracle/_ref) on this host's cores,
             bounded sample of the same workload

--impl reference times the reference CPU implementation alone (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1807_04180_b200.problems import config  # noqa: E402
from paper_1807_04180_b200.roofline import step_bytes  # noqa: E402

METRIC = "ddm_iterations_per_s"
UNIT = "iter/s"


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) < 9:
                continue
            for k, nm in enumerate(names):
                if r[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": sorted(reasons), "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")
    return world, rank, local


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def solve_traffic(cfg: int):
    """Solve-stage DRAM bytes per solve from the committed ncu step summary of this
    config (profiles/r02_step_summary_cfg<N>.json, tools/ncu_step.py)."""
    path = os.path.join(ROOT, "profiles", f"r02_final_step_summary_cfg{cfg}.json")
    if not os.path.exists(path):
        path = os.path.join(ROOT, "profiles", f"r02_step_summary_cfg{cfg}.json")
    try:
        with open(path) as f:
            return json.load(f)["solve_dram_bytes"]
    except (OSError, KeyError, ValueError):
        return None


def dense_residual(prob, seed: int = 1234) -> np.ndarray:
    """Seeded dense complex vector, zero on the global ring (an FGMRES Krylov
    vector after the first iteration is dense)."""
    rng = np.random.default_rng(seed)
    r = (rng.standard_normal(prob.n_global) + 1j * rng.standard_normal(prob.n_global))
    r = r.reshape(prob.gny, prob.gnx)
    r[0, :] = r[-1, :] = 0
    r[:, 0] = r[:, -1] = 0
    r = r.ravel()
    return r / np.linalg.norm(r)


def reference_sample(prob, steps: int, warmup: int, threads: int, min_s: float = 0.0):
    """Time the unmodified reference (or, if it was not built, the C port)
    precondition(r, K) on host cores: K = steps, raised (one re-run) until the timed
    call takes at least min_s seconds of CPU work. Returns (iter/s, kind, threads,
    seconds, K)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    r = dense_residual(prob)
    eng = None
    if pyoracle.ref_available():
        try:
            eng = pyoracle.RefEngine(prob, threads=threads)
            kind = "reference"
        except ValueError:  # config 3: the reference has no lens medium -> the C port
            eng = None
    if eng is None:
        eng = pyoracle.OracleEngine(prob)
        kind = "port"
        threads = 1
    if warmup > 0:
        eng.precondition(r, warmup)
    t0 = time.perf_counter()
    eng.precondition(r, steps)
    dt = time.perf_counter() - t0
    if dt < min_s:
        steps = int(min(512, max(steps + 1, np.ceil(steps * min_s / max(dt, 1e-3)))))
        t0 = time.perf_counter()
        eng.precondition(r, steps)
        dt = time.perf_counter() - t0
    eng.close()
    return steps / dt, kind, threads, dt, steps


def run_reference(args, world, rank):
    if rank != 0:
        return
    if args.config == 5:
        print(json.dumps({"impl": "reference", "unavailable": "the reference has no 3-D code "
                          "(SPEC.md:12); the 3-D restatement's single-threaded factorization of "
                          "config 5's 57^3 windows does not finish in minutes"}), flush=True)
        return
    prob = config(args.config)
    threads = os.cpu_count() or 1
    # bounded sample: the reference needs ~0.6 s per config-4 sweep on 16 cores; the
    # same warm-up count as the GPU arm
    steps = args.steps
    warm = args.warmup
    val, kind, thr, dt, steps = reference_sample(prob, steps, warm, threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
        "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": 1e3 * dt / steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": prob.name, "grid": f"{prob.mx}x{prob.my}",
                   "subdomains": f"{prob.n1}x{prob.n2}", "n_global": prob.n_global,
                   "parallelism": "host threads (reference WorkerPool)"},
        "munknown_iters_per_s": val * prob.n_global / 1e6,
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": thr, "kind": kind,
                         "sample": f"precondition(r, K={steps}) on {prob.name}, dense seeded r"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def dense_residual3(prob, seed: int = 1234) -> np.ndarray:
    """dense_residual for a 3-D problem: zero on the global boundary shell."""
    rng = np.random.default_rng(seed)
    gx, gy, gz = prob.gdims
    r = rng.standard_normal((gz, gy, gx)) + 1j * rng.standard_normal((gz, gy, gx))
    r[0], r[-1] = 0, 0
    r[:, 0], r[:, -1] = 0, 0
    r[:, :, 0], r[:, :, -1] = 0, 0
    r = r.ravel()
    return r / np.linalg.norm(r)


def run_ours3(args, world, rank, local):
    """Config 5 (3-D, include/hddm3.h): the same measurements as run_ours."""
    import torch
    from paper_1807_04180_b200.engine import DdmStats, FgmresOptions
    from paper_1807_04180_b200.engine3 import DdmEngine3
    from paper_1807_04180_b200.roofline import step_bytes3

    prob = config(5)
    torch.cuda.set_device(local)
    eng = DdmEngine3(prob, device=local)
    ci = eng.class_info()
    r = torch.from_numpy(dense_residual3(prob)).to(f"cuda:{local}")
    z = torch.empty_like(r)
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device=f"cuda:{local}")
    eng.precondition(r, max(args.warmup, 1), DdmStats(), out=z)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    eng.set_timing(True)
    barrier(world)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    st = DdmStats()
    e0.record(stream)
    eng.precondition(r, args.steps, st, out=z)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ms = e0.elapsed_time(e1)
    clocks = sampler.stop()
    launches = eng.launch_count()
    max_local_rel, corrections = eng.refine_stats()
    solve_ms_per = eng.time_solve(max(5, args.steps))
    ms_max = allreduce_max(ms, world)
    value = world * args.steps / (ms_max / 1e3)
    peak, peak_kind = measured_peaks()
    nnz = [c["factor_nnz"] for c in ci]
    B = step_bytes3(prob, nnz)
    achieved = B["B_solve"] / (solve_ms_per / 1e3) / 1e9
    step_achieved = B["B_step"] / (ms / args.steps / 1e3) / 1e9
    e2e = None
    if not args.skip_e2e:
        f_host = prob.source_f()
        nbytes = 16 * prob.n_global
        eng.fgmres(f_host, FgmresOptions(prob.tol, 1, prob.restart), prob.k_steps)
        K = prob.k_steps
        t0 = time.perf_counter()
        x, res = eng.fgmres(f_host, FgmresOptions(prob.tol, prob.max_iters, prob.restart), K)
        wall = time.perf_counter() - t0
        total_steps = res.iters * K
        e2e = {"value": world * total_steps / wall, "unit": UNIT,
               "h2d_bytes_per_step": nbytes / max(total_steps, 1),
               "d2h_bytes_per_step": nbytes / max(total_steps, 1),
               "what": f"FGMRES({prob.restart})+DDM(K={K}) to {prob.tol} from host b to host x",
               "gmres_iters": res.iters, "ddm_steps": total_steps,
               "true_relres": res.true_relres, "wall_s": wall}
    fp = eng.footprint()
    if rank == 0:
        gx, gy, gz = prob.gdims
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": prob.name, "grid": f"{prob.mx}x{prob.my}x{prob.mz}",
                       "subdomains": f"{prob.n1}x{prob.n2}x{prob.n3}", "n_global": prob.n_global,
                       "classes": len(ci), "parallelism": f"replicas x{world}",
                       "l2": f"factors {16 * sum(nnz) / 1e9:.1f} GB vs 126 MB L2: no flush",
                       "step": "one DDM sweep of precondition(r, K=steps), dense r"},
            "munknown_iters_per_s": value * prob.n_global / 1e6,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None,
                         "kernel": "batched dense supernodal solve stage (fwd+bwd, all classes)",
                         "bytes_per_launch": B["B_solve"], "ms_per_launch": solve_ms_per,
                         "peak_kind": peak_kind},
            "step_roofline": {"achieved_gbs": step_achieved, "bytes_per_step": B["B_step"],
                              "frac": step_achieved / peak},
            "factor": {"ms": eng.factor_ms(), "classes": len(ci),
                       "stored_values_per_class": fp["stored_values_per_class"],
                       "ref_nnz_per_class": fp["ref_nnz_per_class"],
                       "factor_bytes": 16 * fp["stored_values_per_class"] * len(ci),
                       "device_bytes_in_use": fp["device_bytes_in_use"], "hbm_bytes": 180e9},
            "solve_launches_per_step": eng.solve_launches(),
            "refine": {"max_first_pass_relres": max_local_rel, "solves_corrected": corrections},
            "cpu_baseline": None,
            "e2e": e2e, "clocks": clocks, "gpu_launches": launches,
            "solves": st.solves, "skipped": st.skipped,
        }
        print(json.dumps(line), flush=True)
    eng.close()


def run_ours(args, world, rank, local):
    import torch
    from paper_1807_04180_b200.engine import DdmEngine, DdmStats, FgmresOptions

    if args.config == 5:
        return run_ours3(args, world, rank, local)
    prob = config(args.config)
    torch.cuda.set_device(local)
    eng = DdmEngine(prob, device=local)
    ci = eng.class_info()
    r_host = dense_residual(prob)
    r = torch.from_numpy(r_host).to(f"cuda:{local}")
    z = torch.empty_like(r)
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device=f"cuda:{local}")
    # warm-up
    eng.precondition(r, max(args.warmup, 1), DdmStats(), out=z)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    eng.set_timing(True)  # resets the launch counter
    barrier(world)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    st = DdmStats()
    e0.record(stream)
    eng.precondition(r, args.steps, st, out=z)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ms = e0.elapsed_time(e1)
    clocks = sampler.stop()
    launches = eng.launch_count()
    max_local_rel, corrections = eng.refine_stats()
    eng.set_timing(False)
    # dominant kernel group: the batched solve stage, timed on the engine stream
    # (CUDA graph of its kernels, right-hand sides of the last timed sweep)
    solve_ms_per = eng.time_solve(max(5, args.steps))
    # the other step stages, each timed alone on the last sweep's state (CUDA events)
    stage_ms = {k: eng.time_kernel(k, 20) for k in ("transfer", "check", "accumulate")}
    ms_max = allreduce_max(ms, world)
    value = world * args.steps / (ms_max / 1e3)

    peak, peak_kind = measured_peaks()
    nnz = [c["factor_nnz"] for c in ci]
    B = step_bytes(prob, nnz, None)
    all_active = st.solves == prob.nsub * args.steps
    achieved = B["B_solve"] / (solve_ms_per / 1e3) / 1e9 if solve_ms_per > 0 else None
    # steps >= 2 read only the forward factor blocks of patch-holding subtrees
    # (RHS nonzero on the transfer patches only); SURVEY 8(d) counts the blocks read
    nw = prob.window[0] * prob.window[1]
    stage_bytes = {"transfer": B["B_xfer"], "accumulate": B["B_acc"],
                   "check": 16.0 * prob.nsub * nw}
    stage_roof = {k: {"ms": stage_ms[k], "bytes": stage_bytes[k],
                      "achieved_gbs": stage_bytes[k] / (stage_ms[k] / 1e3) / 1e9,
                      "frac": stage_bytes[k] / (stage_ms[k] / 1e3) / 1e9 / peak}
                  for k in stage_ms}
    stage_roof["note"] = ("algorithmic bytes (SURVEY 8(d)): transfer B_xfer = 16(|patch|+|w|) per "
                          "executed transfer, accumulate B_acc = 48|region| per subdomain, check "
                          "= the solutions read once (16 n_w per subdomain; its reads of B on the "
                          "transfer patches not counted: a lower bound)")
    fwd_full, fwd_sparse = eng.fwd_entries()
    saved = 16.0 * len(ci) * (fwd_full - fwd_sparse) * (args.steps - 1) / args.steps
    B_step_read = B["B_step"] - saved
    step_achieved = B_step_read / (ms / args.steps / 1e3) / 1e9

    # e2e: full FGMRES solve through the C-ABI with host buffers
    e2e = None
    if not args.skip_e2e:
        f_host = prob.source_f()
        nbytes = 16 * prob.n_global
        # untimed warm-up of the same call: the Krylov workspace (2m+1 global vectors) is
        # allocated and the solve graphs instantiated on first use, not per solve
        if prob.mode == "standalone":
            eng.solve_iterative(f_host, prob.tol, 1, DdmStats())
        else:
            eng.fgmres(f_host, FgmresOptions(prob.tol, 1, prob.restart), prob.k_steps)
        if prob.mode == "standalone":  # config 1: solve_iterative, cli.cpp:173-179
            t0 = time.perf_counter()
            sst = DdmStats()
            eng.solve_iterative(f_host, prob.tol, prob.steps, sst)
            wall = time.perf_counter() - t0
            total_steps = sst.steps
            what = f"solve_iterative({prob.steps} standalone DDM iterations) from host f to host u"
            extra = {"ddm_steps": total_steps, "relres": sst.relres}
        else:
            K = prob.k_steps
            t0 = time.perf_counter()
            x, res = eng.fgmres(f_host, FgmresOptions(prob.tol, prob.max_iters, prob.restart), K)
            wall = time.perf_counter() - t0
            total_steps = res.iters * K
            what = f"FGMRES({prob.restart})+DDM(K={K}) to {prob.tol} from host b to host x"
            extra = {"gmres_iters": res.iters, "ddm_steps": total_steps,
                     "true_relres": res.true_relres}
        e2e_val = world * total_steps / wall if wall > 0 else None
        e2e = {"value": e2e_val, "unit": UNIT,
               "h2d_bytes_per_step": nbytes / max(total_steps, 1),
               "d2h_bytes_per_step": nbytes / max(total_steps, 1),
               "what": what, **extra, "wall_s": wall}

    cpu = None
    if rank == 0 and not args.skip_cpu:
        try:
            # the reference on every host core (the headline baseline) and on one core
            # (SURVEY 8(d)); thread scaling is capped by its per-class mutex
            # bounded samples of about args.cpu_seconds of CPU work each (K raised
            # until the timed call takes that long)
            cval, kind, thr, dt, k = reference_sample(prob, args.cpu_steps, 0,
                                                      os.cpu_count() or 1, args.cpu_seconds)
            cpu = {"value": cval, "unit": UNIT, "cores": thr, "kind": kind,
                   "sample": f"precondition(r, K={k}) on {prob.name}, dense "
                             f"seeded r, {dt:.1f} s"}
            if thr > 1:
                cval1, _, thr1, dt1, k1 = reference_sample(prob, 1, 0, 1, args.cpu_seconds)
                cpu["single_thread"] = {"value": cval1, "unit": UNIT, "cores": thr1,
                                        "sample": f"precondition(r, K={k1}), {dt1:.1f} s"}
        except Exception as exc:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "unavailable",
                   "sample": f"{type(exc).__name__}: {exc}"}

    fp = eng.footprint()
    factor_info = {"ms": eng.factor_ms(), "classes": len(ci),
                   "stored_values_per_class": fp["stored_values_per_class"],
                   "factor_bytes": 16 * fp["stored_values_per_class"] * len(ci),
                   "device_bytes_in_use": fp["device_bytes_in_use"],
                   "hbm_bytes": 180e9}
    fac_b = 16.0 * sum(nnz)
    vec_b = 16.0 * 6 * prob.nsub * prob.window[0] * prob.window[1]
    l2_note = (f"factors {fac_b / 1e6:.0f} MB + per-subdomain vectors {vec_b / 1e6:.0f} MB vs "
               f"126 MB L2: " + ("inputs larger than L2, no flush" if fac_b > 126e6 else
                                 "factors fit in L2 (warm-cache number, supplementary config)"))
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": prob.name, "grid": f"{prob.mx}x{prob.my}",
                       "subdomains": f"{prob.n1}x{prob.n2}", "n_global": prob.n_global,
                       "classes": len(ci), "parallelism": f"replicas x{world}",
                       "l2": l2_note,
                       "step": "one DDM sweep of precondition(r, K=steps), dense r"},
            "munknown_iters_per_s": value * prob.n_global / 1e6,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None,
                         "traffic": solve_traffic(args.config),
                         "traffic_note": "DRAM bytes of the solve-stage kernels of one step, "
                                         f"profiles/r02[_final]_step_summary_cfg{args.config}.json "
                                         "(ncu launch list, cache flushed per launch: an upper bound)",
                         "kernel": "batched supernodal solve stage (fwd+bwd, all classes)",
                         "bytes_per_launch": B["B_solve"], "ms_per_launch": solve_ms_per,
                         "peak_kind": peak_kind},
            "step_roofline": {"achieved_gbs": step_achieved, "bytes_per_step": B_step_read,
                              "bytes_per_step_full": B["B_step"],
                              "fwd_entries": {"full": fwd_full, "sparse_rhs": fwd_sparse},
                              "frac": step_achieved / peak, "all_active": all_active},
            "stage_rooflines": stage_roof,
            "factor": factor_info,
            "solve_launches_per_step": eng.solve_launches(),
            "refine": {"max_first_pass_relres": max_local_rel,
                       "solves_corrected": corrections},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks,
            "gpu_launches": launches,
            "solves": st.solves, "skipped": st.skipped,
        }
        print(json.dumps(line), flush=True)
    eng.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=32)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
