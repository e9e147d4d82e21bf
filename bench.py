#!/usr/bin/env python3
"""Benchmark: ACR factor+solve DOF/s (fp64) on B200, per BASELINE.json.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

One step = acr_factor (H-matrix lift + all cyclic-reduction levels + apex) followed
by the solve of the configuration's right-hand sides, on a seeded synthetic
system of BASELINE.json configs[C-1] (default C = 2, "configs[1]").

value  : DOF/s = N * nrhs / t_step with the system and RHS already resident in HBM
         (acrgpu_factor_resident + acrgpu_solve_device), CUDA events on the library
         stream, max over ranks.
e2e    : same metric through the reference-facing API with HOST buffers
         (acr_factor(System) + AcrFactorization.solve(numpy)), H2D of the COO system and
         RHS and D2H of the solution inside the timed region.
roofline / cpu_baseline / clocks / gpu_launches: see DESIGN.md §6.

--impl reference: the reference's CPU path (the C++ oracle restatement; the reference
itself cannot be built here -- no Eigen), all host threads, on a bounded sample of the
same workload, extrapolated to the full configuration by its nominal FLOP count.

Multi-GPU (--gpus N > 1 under torchrun): the plane partition of execute_parallel_factor
(parallel.cpp:96-297) -- one system, rank w owns plan_schedule(n, N)'s planes, per-level
NCCL point-to-point exchange inside libacrgpu (strong scaling: value = DOF / max-over-ranks
step time).  --replicas instead runs N independent copies (weak scaling).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

# libacrgpu uses 16 streams (4 lanes x 4); must be set before the CUDA context exists
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ACR factor+solve DOF/sec (fp64) at 1/2/4/8 B200 vs roofline; relative residual"
FP64_PEAK_TFLOPS = 37.14   # measured mma.sync.m8n8k4.f64 (DMMA) on this pool, profiles/r01_fp64_peak.txt
FP64_DFMA_TFLOPS = 34.16   # measured DFMA (same file)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, help="BASELINE.json config index (1-5)")
    ap.add_argument("--n", type=int, default=None, help="override plane count (testing only)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--exact-dense-products", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--seed", type=int, default=2024)
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent copies instead of the partition")
    ap.add_argument("--cpu-sample-n", type=int, default=16, help="plane count of the CPU baseline's sample")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return

        def reader():
            for line in self.proc.stdout:
                self.rows.append([x.strip() for x in line.split(",")])

        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                smax.append(float(r[1]))
                for nm, v in zip(names, r[4:8]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def config_system(args):
    """The step's system.  Replicas (--replicas, N > 1) each factor their own seeded copy;
    every other mode -- in particular the plane partition, where the ranks factor ONE
    system together -- builds the identical system on every rank."""
    from paper_1701_00182_b200 import problems as P
    ws, rank, _ = dist_env()
    seed = args.seed + 1000 * rank if (args.replicas and ws > 1) else args.seed
    return P.config_system(args.config, n=args.n, seed=seed)


def workload_name(args, sysm):
    from paper_1701_00182_b200 import problems as P
    c = P.CONFIGS[args.config]
    return f"C{args.config} {c['kind']} n={sysm.n} N={sysm.total_dim} leaf={c['leaf']} eps={c['eps']:g} nrhs={sysm.rhs.shape[0]}"


# ----------------------------------------------------------------------------- CPU arm
CPU_CALIBRATION = os.path.join(ROOT, "profiles", "r02_cpu_c2_p16.json")


def cpu_sample(args, sysm_full, flops_full=None, threads=None):
    """The reference path's CPU cost (the oracle: C++ restatement of it, -O3, all host threads,
    plane-parallel like parallel.cpp:383-405) on a bounded sample -- the same operator and
    tolerance at n = --cpu-sample-n planes (a 1-2 s factorization) -- extrapolated to the full
    configuration by nominal FLOPs.  When a full-size CPU run of this configuration was measured
    on a GPU box host (tools/cpu_baseline.py -> profiles/r02_cpu_c2_p16.json: C2, 16 threads,
    543.7 s measured vs 1770.9 s extrapolated from the n=16 sample), the extrapolation is
    scaled by that measured/extrapolated ratio and the record says so."""
    from oracle import oracle as O
    from paper_1701_00182_b200 import problems as P
    c = P.CONFIGS[args.config]
    threads = threads or os.cpu_count() or 1
    n_full = sysm_full.n
    n_s = min(n_full, args.cpu_sample_n)
    samp = P.config_system(args.config, n=n_s, seed=args.seed, nrhs=sysm_full.rhs.shape[0])
    O.flops_reset()
    t0 = time.perf_counter()
    f = O.Factorization(samp, eps=c["eps"], leaf_size=c["leaf"], threads=threads)
    u = f.solve()
    dt = time.perf_counter() - t0
    fl = O.flops_read()
    flops_s = sum(fl[k] for k in ("gemm", "geqrf", "orgqr", "svd", "lu"))
    res = samp.relative_residual(u)
    dof_s = samp.total_dim * samp.rhs.shape[0]
    out = {"sample": f"oracle factor+solve of C{args.config} operator at n={n_s} (N={samp.total_dim}), "
                     f"{dt:.2f} s, {flops_s:.3e} nominal flops, residual {res:.3e}",
           "cores": threads, "kind": "port", "t_sample_s": dt, "flops_sample": flops_s,
           "sample_dof_per_s": dof_s / dt}
    if n_s == n_full:
        out["value"] = dof_s / dt
        out["unit"] = "DOF/s"
    elif flops_full:
        t_full = dt * flops_full / flops_s
        out["sample"] += f"; extrapolated to n={n_full} by nominal flops ({flops_full:.3e}) -> {t_full:.1f} s"
        out["extrapolated"] = True
        try:
            cal = json.load(open(CPU_CALIBRATION))
            if cal["config"] == args.config and cal["full"]["n"] == n_full and cal["sample"]["n"] == n_s:
                ratio = cal["calibration_measured_over_extrapolated"]
                t_full *= ratio
                out["calibration"] = {
                    "source": os.path.relpath(CPU_CALIBRATION, ROOT), "ratio_measured_over_extrapolated": ratio,
                    "measured_full_s": cal["measured_full_s"], "measured_threads": cal["threads"],
                    "measured_cpu": cal["cpu"], "measured_dof_per_s": cal["full"]["dof_per_s"]}
                out["sample"] += f", calibrated x{ratio:.3f} by the measured full-size run -> {t_full:.1f} s"
        except Exception:
            pass
        out["value"] = sysm_full.total_dim * sysm_full.rhs.shape[0] / t_full
        out["unit"] = "DOF/s"
    return out


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from paper_1701_00182_b200 import problems as P
    sysm = P.config_system(args.config, n=args.n, seed=args.seed)
    # the full-size nominal FLOP count comes from the flop model of the oracle run at
    # the sample size scaled by the GPU-measured ratio when available; otherwise the
    # sample's own DOF/s is reported (labelled).
    flops_full = None
    fpath = os.path.join(ROOT, "profiles", "nominal_flops.json")
    if os.path.exists(fpath):
        try:
            flops_full = json.load(open(fpath)).get(f"C{args.config}:n={sysm.n}")
        except Exception:
            flops_full = None
    vals, samp_s = [], []
    cb = None
    for i in range(args.warmup + args.steps):
        cb = cpu_sample(args, sysm, flops_full)
        if i >= args.warmup:
            vals.append(cb.get("value", cb["sample_dof_per_s"]))
            samp_s.append(cb["t_sample_s"])
    v = statistics.median(vals)
    line = {"metric": METRIC, "value": v, "unit": "DOF/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * sysm.total_dim * sysm.rhs.shape[0] / v, "higher_is_better": True,
            "ms_per_step_is_extrapolated": bool(cb.get("extrapolated")),
            "sample_ms_per_step": 1000.0 * statistics.median(samp_s),
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(args, sysm)}, "impl": "reference",
            "cpu_baseline": {**cb, "value": v},
            "e2e": {"value": v, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm
def parse_profile(text):
    """Rows of acrgpu_profile_report (kernel ms launches ctas nominal_flops), slowest first."""
    rows = []
    for line in text.strip().splitlines():
        if line.startswith("#"):
            continue
        p = line.split()
        if len(p) >= 5:
            rows.append({"kernel": p[0], "ms": float(p[1]), "launches": int(p[2]), "ctas": int(p[3]),
                         "flops": float(p[4]), "executed_flops": float(p[5]) if len(p) > 5 else float(p[4])})
    rows.sort(key=lambda r: -r["ms"])
    return rows


def run_ours(args):
    ws, rank, local = dist_env()
    import numpy as np
    import torch
    if not torch.cuda.is_available():
        print(json.dumps({"metric": METRIC, "error": "no CUDA device"}))
        return 1
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1701_00182_b200 import acr, problems as P
    c = P.CONFIGS[args.config]
    sysm = config_system(args)
    nrhs = sysm.rhs.shape[0]
    cfg = acr.AcrConfig(eps=c["eps"], leaf_size=c["leaf"], exact_dense_products=args.exact_dense_products)
    ctx = acr.Context(local)
    dsys = acr.DeviceSystem(sysm, ctx)
    f_dev = torch.from_numpy(np.ascontiguousarray(sysm.rhs)).to(f"cuda:{local}")
    u_dev = torch.empty_like(f_dev)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    comm = None
    if ws > 1 and not args.replicas:
        uid = [acr.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = acr.Comm.nccl(uid[0], ws, rank)
    partitioned = comm is not None

    def step():
        if partitioned:
            u_dev.zero_()  # planes owned by other ranks
            fact = acr.acr_factor_partitioned(dsys, comm, cfg)
        else:
            fact = acr.acr_factor(dsys, cfg)
        fact.solve_device(f_dev.data_ptr(), u_dev.data_ptr(), nrhs)
        return fact

    # Warm-up.  The last warm-up step times EVERY launch (CUDA events on the launching
    # streams) to find the dominant kernel and the per-kernel table; the timed steps then
    # record events around that kernel's launches only, so the roofline figure is measured
    # inside the timed region without two event records on each of the other launches.
    fact = None
    acr.profile_select(None)
    for i in range(args.warmup):
        if i == args.warmup - 1:
            acr.profile_report(reset=True)
            acr.profile_select("*")
        fact = step()
        del fact
        fact = None
    torch.cuda.synchronize()
    warm_rows = parse_profile(acr.profile_report(reset=True))
    dom_name = warm_rows[0]["kernel"] if warm_rows else None
    acr.profile_select(dom_name)
    sampler = ClockSampler(local)
    barrier()
    sampler.start()
    t_fac, t_sol, launches, flops = [], [], 0, 0.0
    start = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    wall = []
    for _ in range(args.steps):
        barrier()
        w0 = time.perf_counter()
        start.record()
        fact = step()
        end.record()
        end.synchronize()
        wall.append(time.perf_counter() - w0)
        tm = fact.timing()
        t_fac.append(tm["factor_ms"])
        t_sol.append(tm["solve_ms"])
        launches += tm["factor_launches"] + tm["solve_launches"]
        flops = tm["flops_nominal"]
        if _ < args.steps - 1:
            del fact
    barrier()
    clocks = sampler.stop()
    prof = acr.profile_report(reset=True)
    acr.profile_select(None)
    # device time per step from the library's own stream events (factor + solve)
    step_ms = [a + b for a, b in zip(t_fac, t_sol)]
    ms = max(step_ms) if step_ms else float("nan")
    ms_mean = sum(step_ms) / len(step_ms)
    if dist is not None:
        t = torch.tensor([ms_mean], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_mean = float(t.item())
    dof = sysm.total_dim * nrhs
    value = (1 if partitioned else ws) * dof / (ms_mean / 1000.0)
    # accuracy of the last factorization (a partition's ranks each hold their own planes)
    if partitioned:
        dist.all_reduce(u_dev, op=dist.ReduceOp.SUM)
    u = u_dev.cpu().numpy()
    res = sysm.relative_residual(u)
    st = fact.inverse_rank_stats()
    lv = fact.level_info()
    fb = fact.factor_bytes()
    tm = fact.timing()
    avg_rank, largest = st.average_rank, st.largest_rank
    if partitioned:
        t = torch.tensor([st.average_rank * st.lowrank_leaf_count, st.lowrank_leaf_count, fb], device=f"cuda:{local}",
                         dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        avg_rank = float(t[0] / t[1]) if float(t[1]) > 0 else 0.0
        fb = int(t[2].item())
        t = torch.tensor([st.largest_rank], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        largest = int(t.item())
    del fact
    # the plane partition's contract (test_parallel.cpp:75-89): the gathered solution is
    # bitwise the single-GPU one -- rank 0 recomputes it alone after the timed steps
    single_check = None
    if partitioned:
        if rank == 0:
            f1 = acr.acr_factor(dsys, cfg)
            u1 = torch.empty_like(f_dev)
            f1.solve_device(f_dev.data_ptr(), u1.data_ptr(), nrhs)
            single_check = bool(np.array_equal(u1.cpu().numpy(), u))
            del f1
        dist.barrier()

    # roofline of the dominant kernel: its launches in the timed steps (events on its stream)
    rows = parse_profile(prof)
    dom = next((r for r in rows if r["kernel"] == dom_name), None)
    tot_ms = sum(r["ms"] for r in warm_rows) or 1.0
    roof = None
    if dom:
        avg_ms = dom["ms"] / max(1, dom["launches"])
        fl_launch = dom["flops"] / max(1, dom["launches"])
        ach = fl_launch / (avg_ms / 1000.0) / 1e12 if avg_ms > 0 else 0.0
        ach_exec = dom["executed_flops"] / max(1, dom["launches"]) / (avg_ms / 1000.0) / 1e12 if avg_ms > 0 else 0.0
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tpath):
            try:
                traffic = json.load(open(tpath)).get(dom["kernel"])
            except Exception:
                traffic = None
        roof = {"bound": "fp64", "kernel": dom["kernel"], "achieved": ach, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": ach / FP64_PEAK_TFLOPS, "traffic": traffic,
                "achieved_executed": ach_exec, "frac_executed": ach_exec / FP64_PEAK_TFLOPS,
                "share_of_step": (next(r["ms"] for r in warm_rows if r["kernel"] == dom_name) / tot_ms),
                "share_source": "per-kernel event times of the last warm-up step (every launch timed)",
                "peak_source": "measured FP64 DMMA mma.sync.m8n8k4 (profiles/r01_fp64_peak.txt); "
                               "MEASURED_PEAKS.json carries no FP64 figure",
                "whole_factor_achieved_tflops": flops / (sum(t_fac) / len(t_fac) / 1000.0) / 1e12 if t_fac else None,
                "kernels": warm_rows[:10]}

    # solve against the HBM roofline (k_mv_t + k_mv_resolve + k_mv_slab of the profiled warm-up step):
    # every stored entry of every applied H-matrix is read once and takes part in 2*nrhs flops
    # (k_mv_resolve, > 4 right-hand sides only: leaf records and packed x of the bulk-copy slab kernel)
    solve_roof = None
    mv = [r for r in warm_rows if r["kernel"] in ("k_mv_t", "k_mv_resolve", "k_mv_slab")]
    if mv:
        peak_gbs = None
        try:
            peak_gbs = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
        except Exception:
            peak_gbs = 6442.2
        mv_ms = sum(r["ms"] for r in mv)
        mv_bytes = 8.0 * sum(r["flops"] for r in mv) / (2.0 * nrhs)
        ach = mv_bytes / (mv_ms / 1e3) / 1e9 if mv_ms > 0 else 0.0
        solve_roof = {"bound": "hbm", "kernels": sorted(r["kernel"] for r in mv), "achieved": ach, "peak": peak_gbs,
                      "unit": "GB/s", "frac": ach / peak_gbs, "bytes_per_solve": mv_bytes, "kernel_ms": mv_ms,
                      "peak_source": "MEASURED_PEAKS.json hbm_gbs"}

    # end-to-end through the public API with host buffers (pinned)
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        hsys = P.System(sysm.n, sysm.dim, pin(sysm.coords), pin(sysm.blk_off), pin(sysm.rows), pin(sysm.cols),
                        pin(sysm.vals), pin(sysm.rhs), sysm.name)
        h2d = sum(a.nbytes for a in (hsys.coords, hsys.blk_off, hsys.rows, hsys.cols, hsys.vals, hsys.rhs))
        d2h = hsys.rhs.nbytes
        ts = []
        for _ in range(max(1, min(args.steps, 2))):
            barrier()
            t0 = time.perf_counter()
            fe = acr.acr_factor_partitioned(hsys, comm, cfg, ctx=ctx) if partitioned else acr.acr_factor(hsys, cfg, ctx=ctx)
            ue = fe.solve(hsys.rhs)
            ts.append(time.perf_counter() - t0)
            del fe
        t_e2e = max(ts)
        if dist is not None:
            t = torch.tensor([t_e2e], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_e2e = float(t.item())
        e2e = {"value": (1 if partitioned else ws) * dof / t_e2e, "unit": "DOF/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "seconds_per_step": t_e2e}
        acr.profile_report(reset=True)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_sample(args, sysm, flops_full=flops)
            fpath = os.path.join(ROOT, "profiles", "nominal_flops.json")
            try:
                d = json.load(open(fpath)) if os.path.exists(fpath) else {}
                d[f"C{args.config}:n={sysm.n}"] = flops
                json.dump(d, open(fpath, "w"), indent=1)
            except Exception:
                pass
        except Exception as ex:  # pragma: no cover
            cpu = {"error": str(ex)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_mean, "higher_is_better": True,
                "scaling": "strong" if partitioned else "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload_name(args, sysm),
                           "parallelism": f"plane-partition p{ws} (NCCL p2p)" if partitioned
                           else ("replicas" if ws > 1 else "single"),
                           "l2": "working set (GB of H-matrix factors) far exceeds the 126 MB L2; no flush needed",
                           "exact_dense_products": bool(args.exact_dense_products)},
                "relative_residual": res, "largest_rank": largest, "average_rank": avg_rank,
                "partition_bitwise_equals_single_gpu": single_check,
                "factor_bytes": fb, "factor_ms": sum(t_fac) / len(t_fac), "solve_ms": sum(t_sol) / len(t_sol),
                "ms_per_step_max": ms, "wall_s_per_step": max(wall),
                "factor_dof_per_s": dof / nrhs / (sum(t_fac) / len(t_fac) / 1000.0),
                "solve_dof_per_s": dof / (sum(t_sol) / len(t_sol) / 1000.0),
                "nominal_flops_per_step": flops, "gpu_launches": launches // max(1, args.steps),
                "levels": [{"level": l.level, "planes": l.plane_count, "largest_rank": l.largest_rank,
                            "average_rank": round(l.average_rank, 3)} for l in lv],
                "roofline": roof, "solve_roofline": solve_roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        if comm is not None:
            comm.close()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
