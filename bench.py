#!/usr/bin/env python
"""Benchmark of the MDOT-PNCG hot path on B200 (driver contract, one JSON line).

Workload (BASELINE.json metric "time-to-eps (marginal L1 1e-6) and marginal
evals/s; HBM GB/s vs peak"): configs[3], the north_star's headline case --
n = 16384, X, Y ~ U[0,1]^2, C = d^2/max fp32 (1 GiB, materialised), Dirichlet(1)
marginals, FIXED gamma schedule to gamma_bar = 4096 (T = 16, the paper's rule
gamma_t = gbar / max(1, floor(gbar/256))), stop at marginal L1
<= 1e-6.  One "step" = one complete mdot_solve (MD loop + PNCG projections +
rounding + cost) with inputs resident in HBM.

value       = marginal evaluations / s over the timed steps (every O(n^2) pass
              of the solve counts; the same unit as the oracle's cpu_baseline)
ms_per_step = time-to-eps (ms), device-timed with CUDA events, max over ranks
roofline    = the fused marginal kernel K1 (k_eval_tma): algorithmic bytes
              4 n^2 (C read once) per launch / mean launch time (CUDA events
              around K1 on the library's stream, sampled on the first slot of
              every device-control graph in the timed region), vs the
              measured HBM copy bandwidth in MEASURED_PEAKS.json; traffic =
              dram read+write bytes per launch from profiles/k1_traffic.json
e2e         = the same metric through the C ABI with HOST buffers (pinned C,
              r, c in; U, V out), copies inside the timed region
cpu_baseline= the fp64 oracle (oracle/), as it stands, on a bounded sample of
              the same workload on this host's cores

--impl reference runs the oracle (this tier's reference arm) on the same
config, metric and unit, each step a bounded sample.
Multi-GPU (torchrun): rows of C sharded over ranks (mdot_solve_sharded); per
evaluation the column totals and row scalars are exchanged inside the
persistent kernel with peer-memory stores and system-scope flags
(mdot_comm_enable_peer; NCCL allreduce in CUDA-graph slots if peer access is
unavailable or MDOT_NO_PEER is set); strong scaling (n fixed).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-to-eps (marginal L1 1e-6) and marginal evals/s; HBM GB/s vs peak at 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--gamma-bar", type=float, default=4096.0)
    ap.add_argument("--T", type=int, default=0)
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--projector", default="pncg", choices=["pncg", "sinkhorn"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--instance", type=int, default=0)
    ap.add_argument("--eps-md", type=float, default=0.0,
                    help="tolerance of the intermediate MD steps (0 = eps at every step, the paper's protocol)")
    ap.add_argument("--sharded-selftest", action="store_true",
                    help="run the multi-GPU code path on one rank (1-rank NCCL communicator; tests only)")
    ap.add_argument("--no-config5", action="store_true",
                    help="skip the config-5 block (n=65536, d=16, on-the-fly cost; north_star scaling target)")
    ap.add_argument("--c5-evals", type=int, default=48,
                    help="config-5 step = the first K O(n^2) evaluations of the config-5 solve (fixed budget)")
    ap.add_argument("--c5-recipe", default="dot", choices=["dot", "diff"],
                    help="on-the-fly cost recipe of the config-5 block: dot form (Z22b, d + 7 FP32 ops per pair) "
                         "or difference form (Z22, 2d + 5)")
    ap.add_argument("--c5-dense-ab", type=int, default=1,
                    help="also time the full config-5 solve with the screen off (dense K2 only)")
    ap.add_argument("--c5-full", type=int, default=1,
                    help="also time one complete config-5 solve to L1 1e-5 (time-to-eps; ~10 s on one B200)")
    ap.add_argument("--adaptive-gamma-leg", type=float, default=256.0,
                    help="also time the solve with MDOT_SCHED_ADAPTIVE starting at this gamma_1 (Z29), reported "
                         "under 'adaptive_gamma'; 0 disables")
    ap.add_argument("--adaptive-leg", type=float, default=1e-3,
                    help="also time the solve with this eps_md (SURVEY 8(f) rank 1), reported under "
                         "'adaptive_eps'; 0 disables")
    ap.add_argument("--two-d", type=int, default=1,
                    help="at N >= 4 (even) also time one config-4 solve on a 2 x N/2 grid of blocks "
                         "(mdot_solve_sharded_2d, NCCL team communicators, device control); 0 disables")
    return ap.parse_args()


def run_two_d(a, rank, world, local_rank, dev, M, dist, barrier, headline):
    """2-D (row x column) sharded config-4 solve (mdot_solve_sharded_2d,
    SURVEY 8(f) rank 4): Gr = 2 row blocks x Gc = N / 2 column blocks, row and
    column teams as NCCL communicators (uniqueId broadcast over torch
    subgroups), the line search under device control.  One warm-up + one timed
    solve, device time as the max over ranks."""
    import numpy as np
    import torch
    Gr = 2 if world >= 4 else 1        # 1 x 1 under --sharded-selftest (1-rank NCCL teams)
    Gc = world // Gr
    ai, bi = rank // Gc, rank % Gc

    def team(members):
        grp = dist.new_group(members)
        if rank not in members:
            return None
        uid = M.mdot_get_unique_id() if rank == members[0] else bytes(128)
        t = torch.frombuffer(bytearray(uid), dtype=torch.uint8).to(dev)
        dist.broadcast(t, members[0], group=grp)
        return M.mdot_comm_create(bytes(t.cpu().numpy()), len(members), members.index(rank), local_rank)

    rc = cc = None
    for x in range(Gr):
        cm = team([x * Gc + y for y in range(Gc)])
        rc = cm if x == ai else rc
    for y in range(Gc):
        cm = team([x * Gc + y for x in range(Gr)])
        cc = cm if y == bi else cc
    inst = instance(a)
    n = inst.n
    rows = np.array_split(np.arange(n), Gr)[ai]
    cols = np.array_split(np.arange(n), Gc)[bi]
    r0, nr, c0, nc = int(rows[0]), len(rows), int(cols[0]), len(cols)
    Cb = torch.from_numpy(np.ascontiguousarray(inst.C[r0:r0 + nr, c0:c0 + nc])).to(dev)
    del inst.C
    r = torch.from_numpy(inst.r).to(dev)
    c = torch.from_numpy(inst.c).to(dev)
    U = torch.empty(nr, dtype=torch.float64, device=dev)
    V = torch.empty(nc, dtype=torch.float64, device=dev)
    sched = M.schedule(M.MDOT_SCHED_FIXED, a.gamma_bar, T=a.T)
    opts = M.options(eps=a.eps, eps_md=a.eps_md)

    def solve():
        return M.mdot_solve_sharded_2d(rc, cc, r0, nr, c0, nc, Cb, r, c, n=n, schedule=sched, options=opts,
                                       u_local_out=U, v_local_out=V)
    solve()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = solve()
    e1.record()
    barrier()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    M.mdot_comm_destroy(rc)
    M.mdot_comm_destroy(cc)
    return {
        "grid": f"{Gr}x{Gc}", "api": "mdot_solve_sharded_2d", "control_path": res["control_path"],
        "time_to_eps_s": ms / 1000.0, "evals_per_s": res["evaluations"] / (ms / 1000.0),
        "evaluations_per_solve": res["evaluations"], "status_name": res["status_name"],
        "cost_unrounded": res["cost_unrounded"], "l1_final": res["l1_final"],
        "cost_rel_diff_vs_1d": abs(res["cost_unrounded"] - headline) / abs(headline),
        "exchange_bytes_per_eval_per_rank": 8 * (nr + nc) + 4 * 16 * 8,
        "exchange_bytes_per_eval_per_rank_1d": 8 * (n + 16),
        "note": "row sums over the row team, column sums over the column team (NCCL, captured in the graph "
                "slots); DESIGN.md section 8 '2-D sharding'"}


def workload_name(a):
    return (f"cfg4-dense-n{a.n}-dirichlet1-gbar{int(a.gamma_bar)}-T{a.T or 'paper'}-"
            f"L1eps{a.eps:g}-{a.projector}" + (f"-epsmd{a.eps_md:g}" if a.eps_md else ""))


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback (B200_PROFILING.md)"


def profile_traffic(name="k1_traffic.json"):
    """dram bytes per launch of K1 (K2: k2_traffic.json) from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", name)
    if os.path.exists(p):
        try:
            return json.load(open(p)).get("bytes_per_launch")
        except Exception:
            return None
    return None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return

        def rd():
            for line in self.proc.stdout:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 7:
                    self.samples.append(parts)
        self.thread = threading.Thread(target=rd, daemon=True)
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
        sm = []
        mx = None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in self.samples:
            try:
                sm.append(float(s[0]))
                mx = float(s[1])
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if s[3 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------
def instance(a):
    import synthetic as S
    return S.config4(a.instance, n=a.n)


def cpu_baseline(a, inst, seconds):
    """The oracle as it stands on this host: MDOT with PNCG from the same
    instance and schedule, stopped after a bounded number of O(n^2)
    evaluations (the metric's unit), timed wall clock."""
    import oracle as O
    prob = O.OracleProblem(inst)
    sched = O.schedule_fixed(a.gamma_bar, T=a.T)
    proj = O.PNCG if a.projector == "pncg" else O.SINKHORN
    # one evaluation to size the sample
    t0 = time.perf_counter()
    U, V, res, _ = O.mdot(prob, sched[:1], O.make_options(eps=a.eps, projector=proj, max_evals=1))
    t1 = time.perf_counter() - t0
    k = max(1, int(seconds / max(t1, 1e-3)))
    t0 = time.perf_counter()
    U, V, res, _ = O.mdot(prob, sched, O.make_options(eps=a.eps, projector=proj, max_evals=k))
    dt = time.perf_counter() - t0
    # the rounding pass at the end is included in dt; count its 3 passes as evaluations
    evals = res["evaluations"] + 3
    cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    return {"value": evals / dt, "unit": "evals/s", "cores": cores, "kind": "oracle",
            "sample": f"oracle MDOT-PNCG on the same n={a.n} instance, first {res['evaluations']} "
                      f"O(n^2) evaluations of the solve (+3 rounding passes), {dt:.1f} s wall",
            "seconds": dt}


def run_reference(a, rank, world):
    if rank != 0:
        return
    inst = instance(a)
    steps = []
    for s in range(a.warmup + a.steps):
        cb = cpu_baseline(a, inst, a.cpu_seconds)
        if s >= a.warmup:
            steps.append(cb)
    v = statistics.mean(x["value"] for x in steps)
    ms = statistics.mean(x["seconds"] for x in steps) * 1000.0
    line = {"metric": METRIC, "value": v, "unit": "evals/s", "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(a), "n": a.n, "gamma_bar": a.gamma_bar,
                       "eps": a.eps, "sample": "bounded oracle sample per step"},
            "impl": "reference",
            "cpu_baseline": {k: steps[-1][k] for k in ("kind", "cores", "sample")} | {"value": v, "unit": "evals/s"},
            "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def run_ours(a, rank, world, local_rank):
    # --sharded-selftest: the multi-GPU code path (process group, NCCL
    # communicator, fused peer exchange, sharded solve, e2e leg) on ONE rank,
    # with a 1-rank NCCL communicator forced onto the sharded path
    sharded = world > 1 or a.sharded_selftest
    if a.sharded_selftest:
        os.environ["MDOT_SHARDED_SELFTEST"] = "1"
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
    import numpy as np
    import torch

    import paper_2307_08507_b200 as M

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if sharded:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    inst = instance(a)
    n = inst.n
    sched = M.schedule(M.MDOT_SCHED_FIXED, a.gamma_bar, T=a.T)
    proj = M.MDOT_PROJ_PNCG if a.projector == "pncg" else M.MDOT_PROJ_SINKHORN
    opts = M.options(eps=a.eps, projector=proj, time_kernels=1, eps_md=a.eps_md)
    r = torch.from_numpy(inst.r).to(dev)
    c = torch.from_numpy(inst.c).to(dev)
    comm = None
    exchange = None
    if sharded:
        rows = np.array_split(np.arange(n), world)[rank]
        row0, nloc = int(rows[0]), len(rows)
        C = torch.from_numpy(np.ascontiguousarray(inst.C[row0:row0 + nloc])).to(dev)
        uid = M.mdot_get_unique_id() if rank == 0 else bytes(128)
        t = torch.frombuffer(bytearray(uid), dtype=torch.uint8).to(dev)
        dist.broadcast(t, 0)
        comm = M.mdot_comm_create(bytes(t.cpu().numpy()), world, rank, local_rank)
        # fused peer exchange (column totals pushed over NVLink inside the
        # persistent kernel); every rank gets the same status, NCCL otherwise
        exchange = "nccl allreduce in CUDA-graph slots"
        if not os.environ.get("MDOT_NO_PEER") and M.mdot_comm_enable_peer(comm, n, check=False) == 0:
            exchange = "fused peer exchange in the persistent kernel (self-validating records over NVLink)"
        U = torch.empty(nloc, dtype=torch.float64, device=dev)
    else:
        C = torch.from_numpy(inst.C).to(dev)
        U = torch.empty(n, dtype=torch.float64, device=dev)
        row0, nloc = 0, n
    V = torch.empty(n, dtype=torch.float64, device=dev)
    del inst.C  # keep host memory bounded; e2e re-creates it pinned

    def solve():
        if comm is not None:
            return M.mdot_solve_sharded(comm, row0, nloc, C, r, c, n=n, schedule=sched, options=opts,
                                        u_local_out=U, v_out=V)
        if a.projector == "sinkhorn":
            return M.mdot_sinkhorn(C, r, c, schedule=sched, options=opts, u_out=U, v_out=V)
        return M.mdot_solve(C, r, c, schedule=sched, options=opts, u_out=U, v_out=V)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for w_i in range(a.warmup):
        try:
            res = solve()
        except M.MdotError:
            if comm is None or exchange is None or not exchange.startswith("fused") or w_i > 0:
                raise
            # the fused peer exchange failed on this box (e.g. a flag timeout):
            # drop it on every rank and keep the NCCL path
            M.mdot_comm_enable_peer(comm, 0, check=False)
            exchange = "nccl allreduce in CUDA-graph slots (fused peer exchange failed)"
            res = solve()
    barrier()
    clk = ClockSampler(local_rank)
    clk.start()
    st = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    results = []
    barrier()
    e0.record(st)
    for _ in range(a.steps):
        results.append(solve())
    e1.record(st)
    barrier()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    evals = sum(x["evaluations"] for x in results)
    kern_ms = sum(x["kernel_ms"] for x in results)
    kern_n = sum(x["kernel_launches"] for x in results)
    launches = sum(x.get("all_launches", 0) for x in results)
    nsamp = sum(x.get("stage_samples", 0) for x in results)
    path = results[-1].get("control_path", 1)
    stages = None
    if nsamp:
        names = (["ctrl+prep", "k1", "finalize", "combine"] if path == 2 else ["ctrl", "prep", "k1", "finalize"])
        stages = {nm: 1000.0 * sum(x["stage_ms"][q] for x in results) / nsamp for q, nm in enumerate(names)}
    control = {0: "host loop", 1: "CUDA-graph slots (device controller)",
               2: "persistent cooperative kernel (device controller)"}.get(path, str(path))
    timing = ("K1 phase of the persistent kernel, measured on the device with %globaltimer between its grid "
              "barriers (CTA 0), every evaluation of the timed region (a phase of one launch cannot be "
              "bracketed by CUDA events)" if path == 2 else
              "CUDA events around K1 on the library stream, first slot of every device-control graph "
              "(sampled), timed region only")
    value = evals / (ms / 1000.0)
    ms_step = ms / a.steps
    hbm, peak_kind = measured_peaks()
    bytes_per_launch = 4.0 * nloc * n
    mean_launch_s = (kern_ms / kern_n) / 1000.0 if kern_n else float("nan")
    achieved = bytes_per_launch / mean_launch_s / 1e9 if kern_n else None
    if dist is not None and achieved is not None:
        t = torch.tensor([achieved], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        achieved = float(t.item())
        hbm = hbm * world
    traffic = profile_traffic()
    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32+f64",
        "data": "synthetic (seeded config 4 instance, no dataset)",
        "config": {"workload": workload_name(a), "n": n, "gamma_bar": a.gamma_bar,
                   "T": int(results[-1]["md_steps"]), "eps": a.eps, "stop": "marginal L1",
                   "projector": a.projector, "parallelism": f"rows sharded x{world}" if sharded else "1 GPU",
                   "exchange": exchange,
                   "l2": "C (4 n^2 B) is larger than L2 (126 MB): no flush needed",
                   "instance_seed": 4000 + a.instance},
        "time_to_eps_s": ms_step / 1000.0,
        "evaluations_per_solve": evals / a.steps,
        "solve": {k: results[-1][k] for k in ("cost_rounded", "cost_unrounded", "l1_final", "iterations",
                                              "evaluations", "ls_evaluations", "fallbacks", "md_steps",
                                              "status_name")},
        "roofline": {"kernel": "k_eval_tma (K1: fused row+column marginal evaluation)", "bound": "hbm",
                     "achieved": achieved, "peak": hbm,
                     "unit": "GB/s", "frac": (achieved / hbm) if achieved else None,
                     "traffic": traffic, "peak_source": peak_kind,
                     "bytes_per_launch": bytes_per_launch, "launches_timed": kern_n,
                     "timing": timing,
                     "mean_launch_us": mean_launch_s * 1e6,
                     "kernel_evals_per_s": (1.0 / mean_launch_s) if kern_n else None,
                     "kernel_share_of_step": (mean_launch_s * evals / (ms / 1000.0)) if kern_n else None,
                     # the algorithmic-bytes fraction counts the L2-resident quarter of C and
                     # the stages prefetched outside the K1 window as if read in it; these two bracket it
                     "frac_dram_in_window": (traffic * (nloc / n) / mean_launch_s / 1e9 / (hbm / (world if dist else 1)))
                     if (kern_n and traffic) else None,
                     "frac_whole_slot": (bytes_per_launch * evals / (ms / 1000.0) / 1e9 / (hbm / (world if dist else 1)))
                     if evals else None},
        "clocks": clocks,
        "gpu_launches": launches,
        "control": control,
        "slot_stage_us": stages,
    }
    # adaptive gamma (Z29): the step sizes chosen on the fly from
    # each projection's cost, the paper's eps at every step; same final plan by
    # Lemma 2.  Reported beside the paper-protocol headline.
    if a.adaptive_gamma_leg > 0 and not a.eps_md and a.projector == "pncg":
        sched_a = M.schedule(M.MDOT_SCHED_ADAPTIVE, a.gamma_bar, step_max=a.adaptive_gamma_leg)
        oa = M.options(eps=a.eps, projector=proj)

        def solve_a():
            if comm is not None:
                return M.mdot_solve_sharded(comm, row0, nloc, C, r, c, n=n, schedule=sched_a, options=oa,
                                            u_local_out=U, v_out=V)
            return M.mdot_solve(C, r, c, schedule=sched_a, options=oa, u_out=U, v_out=V)
        solve_a()
        barrier()
        rg = []
        e0.record(st)
        for _ in range(a.steps):
            rg.append(solve_a())
        e1.record(st)
        barrier()
        ms_g = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([ms_g], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_g = float(t.item())
        ev_g = sum(x["evaluations"] for x in rg)
        line["adaptive_gamma"] = {
            "gamma_1": a.adaptive_gamma_leg, "realised_gammas": rg[-1]["gammas"],
            "time_to_eps_s": ms_g / a.steps / 1000.0, "evals_per_s": ev_g / (ms_g / 1000.0),
            "evaluations_per_solve": ev_g / a.steps, "speedup_vs_headline": ms_step / (ms_g / a.steps),
            "cost_unrounded": rg[-1]["cost_unrounded"], "l1_final": rg[-1]["l1_final"],
            "cost_rel_diff_vs_headline": abs(rg[-1]["cost_unrounded"] - results[-1]["cost_unrounded"])
            / abs(results[-1]["cost_unrounded"]),
            "status_name": rg[-1]["status_name"],
            "note": "MDOT_SCHED_ADAPTIVE (DESIGN.md Z29): gamma doubles while the gbar gained per evaluation does "
                    "not fall; eps at every MD step as in the paper; Lemma 2 (PAPER.md:152-155) fixes the final plan"}
    # adaptive eps: the same solve with loose intermediate
    # MD steps; same final eps, same device timing.  Reported beside the
    # paper-protocol headline, not instead of it.
    if a.adaptive_leg > 0 and not a.eps_md:
        oa = M.options(eps=a.eps, projector=proj, eps_md=a.adaptive_leg)
        sv = opts
        opts = oa
        solve()
        barrier()
        ra = []
        e0.record(st)
        for _ in range(a.steps):
            ra.append(solve())
        e1.record(st)
        barrier()
        opts = sv
        ms_a = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([ms_a], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_a = float(t.item())
        ev_a = sum(x["evaluations"] for x in ra)
        line["adaptive_eps"] = {
            "eps_md": a.adaptive_leg, "time_to_eps_s": ms_a / a.steps / 1000.0,
            "evals_per_s": ev_a / (ms_a / 1000.0), "evaluations_per_solve": ev_a / a.steps,
            "speedup_vs_headline": ms_step / (ms_a / a.steps),
            "cost_unrounded": ra[-1]["cost_unrounded"], "l1_final": ra[-1]["l1_final"],
            "cost_rel_diff_vs_headline": abs(ra[-1]["cost_unrounded"] - results[-1]["cost_unrounded"])
            / abs(results[-1]["cost_unrounded"]),
            "status_name": ra[-1]["status_name"],
            "note": "intermediate MD steps stop at eps_md, the last at eps; Lemma 2 (PAPER.md:152-155) makes "
                    "the final plan independent of the intermediate accuracy"}
    if not a.no_config5:
        line["config5"] = run_config5(a, rank, world, dev, M, dist, comm, barrier)
    if a.two_d and ((world >= 4 and world % 2 == 0) or a.sharded_selftest):
        line["two_d"] = run_two_d(a, rank, world, local_rank, dev, M, dist, barrier, results[-1]["cost_unrounded"])
    # end-to-end through the C ABI with host buffers (rank 0, 1 GPU)
    if not sharded and not a.no_e2e:
        import synthetic as S
        inst2 = S.config4(a.instance, n=n)
        Ch = torch.from_numpy(inst2.C).pin_memory()
        del inst2.C
        rh = torch.from_numpy(inst2.r)
        ch = torch.from_numpy(inst2.c)
        Uh = torch.empty(n, dtype=torch.float64).pin_memory()
        Vh = torch.empty(n, dtype=torch.float64).pin_memory()
        o2 = M.options(eps=a.eps, projector=proj, eps_md=a.eps_md)
        M.mdot_solve(Ch, rh, ch, schedule=sched, options=o2, u_out=Uh, v_out=Vh)   # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev = 0
        for _ in range(a.steps):
            rr = M.mdot_solve(Ch, rh, ch, schedule=sched, options=o2, u_out=Uh, v_out=Vh)
            ev += rr["evaluations"]
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        line["e2e"] = {"value": ev / dt, "unit": "evals/s", "h2d_bytes_per_step": 4 * n * n + 16 * n,
                       "d2h_bytes_per_step": 16 * n, "ms_per_step": 1000.0 * dt / a.steps,
                       "timing": "host wall clock around the synchronous C-ABI call"}
        del Ch
    elif sharded and not a.no_e2e:
        # every rank: its row slab of C from pinned host memory through
        # mdot_solve_sharded (MDOT_MEM_HOST), U_local / V back to the host;
        # whole-job evaluations over the max of the ranks' wall clocks
        import synthetic as S
        inst2 = S.config4(a.instance, n=n)
        Ch = torch.from_numpy(np.ascontiguousarray(inst2.C[row0:row0 + nloc])).pin_memory()
        del inst2.C
        rh = torch.from_numpy(inst2.r)
        ch = torch.from_numpy(inst2.c)
        Uh = torch.empty(nloc, dtype=torch.float64).pin_memory()
        Vh = torch.empty(n, dtype=torch.float64).pin_memory()
        o2 = M.options(eps=a.eps, projector=proj, eps_md=a.eps_md)

        def solve_host():
            return M.mdot_solve_sharded(comm, row0, nloc, C_local=Ch, r=rh, c=ch, n=n, schedule=sched, options=o2,
                                        u_local_out=Uh, v_out=Vh)
        solve_host()   # warm
        barrier()
        t0 = time.perf_counter()
        ev = 0
        for _ in range(a.steps):
            ev += solve_host()["evaluations"]
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        line["e2e"] = {"value": ev / dt, "unit": "evals/s", "h2d_bytes_per_step": 4 * nloc * n + 16 * n,
                       "d2h_bytes_per_step": 8 * (nloc + n), "ms_per_step": 1000.0 * dt / a.steps,
                       "timing": "host wall clock around the synchronous C-ABI call, max over ranks; bytes per rank"}
        del Ch
    if rank == 0 and not a.no_cpu_baseline:
        import synthetic as S
        inst3 = S.config4(a.instance, n=n)
        line["cpu_baseline"] = {k: v for k, v in cpu_baseline(a, inst3, a.cpu_seconds).items()
                                if k != "seconds"}
    if comm is not None:
        M.mdot_comm_destroy(comm)
    if rank == 0:
        emit(line)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def run_config5(a, rank, world, dev, M, dist, comm, barrier):
    """BASELINE configs[4] -- the north_star scaling target (n = 65536, X, Y ~
    U[0,1]^16, C_ij = ||x_i - y_j||^2 / 16 computed in-kernel (K2, Z22),
    Dirichlet(1), FIXED gbar 4096 (T = 16), L1 1e-5), rows of X sharded over
    the ranks with one NCCL allreduce of [column totals | row scalars] per
    evaluation.  A step is the first --c5-evals O(n^2)
    evaluations of the solve (fixed budget, so the driver's 20 steps fit);
    the complete solve is timed once more for time-to-eps.  Roofline: K2 is
    bound by the FP32 pipe (d + 7 = 23 FMA-pipe ops per pair for the dot form,
    2d + 5 = 37 for the difference form; K2), peak = 148 SMs x 128
    FP32 lanes x 1.965 GHz / ops (unit counts measured, profiles/r02_mufu_ffma2_rate.txt);
    the MUFU floor (1 ex2 per pair, 16 per SM per clock) is reported beside it."""
    import numpy as np
    import torch

    import synthetic as S
    inst = S.config5(0)
    n, d = inst.n, inst.X.shape[1]
    rows = np.array_split(np.arange(n), world)[rank]
    row0, nloc = int(rows[0]), len(rows)
    X = torch.from_numpy(np.ascontiguousarray(inst.X[row0:row0 + nloc])).to(dev)
    Y = torch.from_numpy(inst.Y).to(dev)
    r = torch.from_numpy(inst.r).to(dev)
    c = torch.from_numpy(inst.c).to(dev)
    U = torch.empty(nloc, dtype=torch.float64, device=dev)
    V = torch.empty(n, dtype=torch.float64, device=dev)
    gb, eps = 4096.0, 1e-5
    sched = M.schedule(M.MDOT_SCHED_FIXED, gb)

    def solve(max_evals):
        o = M.options(eps=eps, time_kernels=1, max_evals=max_evals)
        if comm is not None:
            return M.mdot_solve_sharded(comm, row0, nloc, X_local=X, Y=Y, scale=inst.scale, r=r, c=c, n=n,
                                        schedule=sched, options=o, u_local_out=U, v_out=V, check=False,
                                        recipe=a.c5_recipe)
        return M.mdot_solve(X=X, Y=Y, scale=inst.scale, r=r, c=c, schedule=sched, options=o, u_out=U, v_out=V,
                            check=False, recipe=a.c5_recipe)

    def maxr(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    K = a.c5_evals
    solve(K)
    barrier()
    st = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    res = []
    barrier()
    e0.record(st)
    for _ in range(a.steps):
        res.append(solve(K))
    e1.record(st)
    barrier()
    ms = maxr(e0.elapsed_time(e1))
    ev = sum(x["evaluations"] for x in res)
    kms = sum(x["kernel_ms"] for x in res)
    kn = sum(x["kernel_launches"] for x in res)
    pairs_per_eval = float(n) * n
    launch_s = kms / kn / 1000.0 if kn else float("nan")
    achieved = float(nloc) * n / launch_s if kn else None
    if dist is not None and achieved is not None:
        t = torch.tensor([achieved], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        achieved = float(t.item())
    ops = (d + 7) if a.c5_recipe == "dot" else (2 * d + 5)   # FMA-pipe ops per pair (power-of-two scale folded)
    fp32_peak = world * 148 * 128 * 1.965e9 / ops
    mufu_peak = world * 148 * 16 * 1.965e9
    out = {
        "workload": f"cfg5-otf-n{n}-d{d}-dirichlet1-gbar4096-T16-L1eps1e-05-{a.c5_recipe}",
        "cost_recipe": ("dot form (Z22b): max(fmaf(-2, x.y, |x|^2 + |y|^2), 0) / 16" if a.c5_recipe == "dot"
                        else "difference form (Z22): fmaf chain of (x - y)^2, / 16"),
        "step": f"first {K} O(n^2) evaluations of the solve (fixed budget per step)",
        "parallelism": f"rows of X sharded x{world}" if world > 1 else "1 GPU",
        "exchange": "NCCL allreduce of [column totals | row scalars] per evaluation in CUDA-graph slots"
                    if world > 1 else None,
        "steps": a.steps, "ms_per_step": ms / a.steps,
        "evals_per_s": ev / (ms / 1000.0), "pairs_per_s": ev * pairs_per_eval / (ms / 1000.0),
        "roofline": {"kernel": "k_eval_otf<16> (K2: on-the-fly cost, fused marginals)", "bound": "alu",
                     "achieved": achieved / 1e9 if achieved else None, "unit": "Gpairs/s",
                     "peak": fp32_peak / 1e9, "frac": (achieved / fp32_peak) if achieved else None,
                     "peak_source": f"FP32 pipe: 148 SMs x 128 lanes x 1.965 GHz / ({ops} ops per pair)",
                     "mufu_floor_frac": (achieved / mufu_peak) if achieved else None,
                     "mean_launch_ms": launch_s * 1e3, "launches_timed": kn,
                     "traffic": profile_traffic("k2_traffic.json") if a.c5_recipe == "dot" else None,
                     "traffic_note": "DRAM bytes per K2 launch (ncu --set full, profiles/k2_traffic.json): X, Y "
                                     "are L2-resident; the bytes are mostly the fp64 row / column partials"},
        "status_name": res[-1]["status_name"],
    }
    if a.c5_full:
        def full_solve():
            solve(0)   # warm the full path once (graph capture, L2)
            barrier()
            e0.record(st)
            f = solve(0)
            e1.record(st)
            barrier()
            return f, maxr(e0.elapsed_time(e1)), M.mdot_last_screen_stats()
        if a.c5_dense_ab and world == 1:
            # the same solve with every evaluation on the dense K2 (K2s off): the screen's gain, measured
            os.environ["MDOT_SCREEN"] = "0"
            fd, ms_dense, _ = full_solve()
            os.environ.pop("MDOT_SCREEN", None)
            out["time_to_eps_dense_k2_s"] = ms_dense / 1000.0
            out["dense_k2_solve"] = {k: fd[k] for k in ("evaluations", "cost_unrounded", "l1_final", "status_name")}
        full, ms_full, sst = full_solve()
        out["time_to_eps_s"] = ms_full / 1000.0
        out["full_solve"] = {k: full[k] for k in ("evaluations", "iterations", "md_steps", "l1_final",
                                                   "cost_unrounded", "cost_rounded", "status_name")}
        out["full_solve"]["evals_per_s"] = full["evaluations"] / (ms_full / 1000.0)
        if sst["evals"] > 0:
            # K2s (csrc/screen.cu): the tensor-core screen of the later MD steps.  Floor: the
            # tf32 MMA work, 2 x 24 flops per pair (K = 24) at the tf32 dense peak (the measured
            # bf16 burst peak x 1.1 / 2.25, the guide's nominal ratio); the dense-equivalent pair
            # rate is the rate at which the screened kernel resolves all n^2 pairs.
            pp = os.path.join(ROOT, "MEASURED_PEAKS.json")
            pk = json.load(open(pp)) if os.path.exists(pp) else {"bf16_tflops": 2250.0}
            tf32 = (float(pk.get("bf16_tflops", 2250.0)) * 1.1 / 2.25) * 1e12
            k2s_s = sst["ms"] / sst["timed"] / 1000.0 if sst["timed"] else None
            floor_s = 2.0 * 24.0 * float(n) * n / tf32
            out["screen"] = {
                "kernel": "k_eval_screen<16> (K2s: tcgen05 kind::tf32 screen + exact recipe on the survivors)",
                "screened_evaluations": sst["evals"], "kept_fraction": sst["kept_frac"],
                "mean_launch_ms": k2s_s * 1e3 if k2s_s else None, "launches_timed": sst["timed"],
                "dense_equivalent_pairs_per_s": (float(n) * n / k2s_s) if k2s_s else None,
                "vs_dense_k2_fp32_floor": ((float(n) * n / k2s_s) / fp32_peak) if k2s_s else None,
                "roofline": {"bound": "tensor", "unit": "ms", "floor_ms": floor_s * 1e3,
                             "frac": (floor_s / k2s_s) if k2s_s else None,
                             "peak_source": f"tf32 dense = measured bf16 {pk.get('bf16_tflops')} TF/s x 1.1/2.25; "
                                            "2 x 24 flops per pair (K = 24)"},
                "note": "bound: keep (i, j) iff log2 P_ij >= min(row, column total) - 48 (rigorous, "
                        "DESIGN.md Z30); the first MD step and projections keeping > 0.8 % run the dense K2",
            }
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        # the oracle's pair rate on this host: exact fp64 log-marginals of 32
        # sampled rows of the same instance at the same potentials (O(n d) each)
        import oracle as O
        prob = O.OracleProblem(inst, recipe=a.c5_recipe)
        rows_s = np.arange(0, n, n // 32)[:32]
        A0, B0 = np.log(inst.r), np.log(inst.c)
        t0 = time.perf_counter()
        O.log_marginal_subset(prob, A0, B0, gb, rows=rows_s)
        dt = time.perf_counter() - t0
        cores = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
        out["cpu_baseline"] = {"value": len(rows_s) * n / dt, "unit": "pairs/s", "cores": cores, "kind": "oracle",
                               "sample": f"oracle log-sum-exp of {len(rows_s)} rows x {n} columns (2 passes), "
                                         f"{dt:.2f} s wall"}
    return out


_JSON_FD = None


def emit(line):
    """The JSON line goes to the real stdout; everything else libraries write
    to fd 1 (e.g. the NCCL version banner torch prints when a communicator
    comes up) was redirected to stderr by main()."""
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)


def main():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    run_ours(a, rank, world, local_rank)


if __name__ == "__main__":
    main()
