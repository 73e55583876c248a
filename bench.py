"""Benchmark: factor+solve DoF/s of the multifrontal path (BASELINE.json metric).

One step = one numeric factorization (every tree level, one Foata class per
level launch sequence) + one solve of the workload's right-hand sides, on
device-resident inputs.  Symbolic planning is excluded from the timed region,
as in the reference's own timing window (cli.py:153-161).

  python bench.py [--config cfg5] [--gpus N] [--steps K] [--warmup W]
  python bench.py --impl reference ...   (the reference's arithmetic on the host cores:
                                          oracle/cpu_baseline.py, no product import)

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "cfg1": dict(shape=(1024,), degree=1, nrhs=1,
                 label="1D FEM linear elements, 1024 elements, single RHS"),
    "cfg2": dict(shape=(64, 64), degree=2, nrhs=1,
                 label="2D FEM quadratic elements on 64x64 mesh, nested dissection"),
    "cfg3": dict(shape=(1024, 1024), degree=1, nrhs=64,
                 label="2D FEM Q1 1024x1024 mesh, 64 RHS"),
    "cfg3p2": dict(shape=(1024, 1024), degree=2, nrhs=64,
                   label="2D FEM Q2 1024x1024 mesh, 64 RHS"),
    "cfg4": dict(shape=(64, 64, 64), degree=1, nrhs=1, label="3D FEM Q1 64^3 mesh"),
    "cfg5": dict(shape=(4096, 4096), degree=1, nrhs=1,
                 label="2D FEM Q1 4096x4096 mesh (largest 2D config)"),
}
DEFAULT_CONFIG = "cfg5"
FP64_PEAK_TFLOPS = 35.47  # measured cuBLAS DGEMM on this pool: profiles/r01_dgemm_cublas_peak.log


def measured_traffic(config, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (tools/ncu_traffic.py -> profiles/traffic_<config>.json), else None."""
    try:
        d = json.loads((ROOT / "profiles" / f"traffic_{config}.json").read_text())
        return d["kernels"][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


def measured_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def build_problem(cfg):
    import paper_2306_08994_b200 as tf
    mesh = tf.TensorMesh(cfg["shape"], cfg["degree"])
    fronts = tf.generate_fronts(mesh)
    tree = tf.build_elimination_tree(tf.sort_fronts(fronts), n_dof=mesh.n_dof)
    system = tf.assemble_system(mesh, "one")
    plan = tf.symbolic_eliminate(tree, system)
    return tf, mesh, fronts, system, plan


# ---------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, gpu_index=0):
        self.samples, self._stop, self.gpu = [], threading.Event(), gpu_index

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=10)

    def summary(self):
        sm = [float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------- CPU baseline
def cpu_baseline(args) -> dict:
    """The reference arm's measurement (below) run once in a fresh interpreter
    (no torch / CUDA state is forked), on rank 0 at N=1."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--config", args.config,
           "--steps", "1", "--warmup", "0"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1800, cwd=str(ROOT),
                         env={k: v for k, v in os.environ.items()
                              if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")})
    if out.returncode != 0:
        return {"error": out.stderr[-500:]}
    return json.loads(out.stdout.strip().splitlines()[-1])["cpu_baseline"]


# ------------------------------------------------------------------ reference
def run_reference(args, cfg):
    """The reference's arithmetic on the host cores (oracle/cpu_baseline.py).

    Imports nothing from the product package.  ms_per_step is the measured
    wall time of one step (one factor+solve of the sample per core); value is
    the workload's DoF/s (measured when the sample is the workload, cfg1 /
    cfg2; else extrapolated by the workload's exact reference task count)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import cpu_baseline as cb
    sshape = cb.sample_shape(cfg["shape"], cfg["degree"])
    # the reference solves one column per call (engine.py:471-472): the sample solves
    # min(nrhs, 4) columns and the solve time scales to the workload's nrhs
    sample = cb.Sample(sshape, cfg["degree"], nrhs=min(cfg["nrhs"], 4))
    procs, rss = cb.choose_procs(sample)
    for _ in range(args.warmup):
        cb.run_step(sample, procs)
    walls, per = [], []
    t_start = time.perf_counter()
    for _ in range(args.steps):
        w, p, _ = cb.run_step(sample, procs)
        walls.append(w)
        per.extend(p)
    t_total = time.perf_counter() - t_start
    wall = float(np.mean(walls))
    base = cb.describe(cfg["shape"], cfg["degree"], cfg["nrhs"], sample, procs, wall, per)
    base["max_rss_bytes_per_process"] = int(rss)
    v = base["value"]
    line = {"metric": "factor+solve DoF/s", "value": v, "unit": "DoF/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": args.config, "label": cfg["label"],
                       "n_dof": int(np.prod([x * cfg["degree"] + 1 for x in cfg["shape"]])),
                       "nrhs": cfg["nrhs"], "sample_shape": list(sshape),
                       "value_basis": base["value_basis"]},
            "timed_seconds_total": t_total,
            "cpu_baseline": base,
            "e2e": {"value": v, "unit": "DoF/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ scaling model
NVLINK_GBS = 450.0  # effective one-direction NVLink 5 P2P bandwidth assumed per transfer


def modelled_scaling(dp, level_ms, solve_ms, worlds=(2, 4, 8)):
    """Strong-scaling model of the subtree-sharded path from
    the MEASURED one-GPU per-level times: a level with n_L fronts on P GPUs takes
    level_ms x (most fronts any rank owns) / n_L (independent fronts split
    evenly; the top log2 P levels keep whole fronts on single GPUs), plus the
    root-ward packed Schur complements of every cross-rank tree edge at
    NVLINK_GBS.  The solve scales like the factorization's level profile.  A
    model, not a measurement: this pool has one GPU per box."""
    from paper_2306_08994_b200.distributed import ShardPlan
    sizes = [dl.n_fronts for dl in dp.levels]
    t1 = float(sum(level_ms)) + solve_ms
    out = {}
    for P in worlds:
        sp = ShardPlan(sizes, P)
        t = 0.0
        for L, ls in enumerate(sp.levels):
            most = max(f1 - f0 for f0, f1 in ls.ranges)
            t += level_ms[L] * most / max(sizes[L], 1)
            if L > 0:
                for c, q, p_ in sp.upward(L):
                    t += 8.0 * dp.levels[L - 1].upd_stride / (NVLINK_GBS * 1e6)
        ts = solve_ms * (t / max(sum(level_ms), 1e-9))
        out[str(P)] = {"ms_per_step": t + ts, "speedup": t1 / (t + ts),
                       "efficiency": t1 / (P * (t + ts)), "split_level": sp.split}
    return out


# ---------------------------------------------------------------------- ours
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    tf, mesh, fronts, system, plan = build_problem(cfg)
    if args.small_max_m is not None:
        from paper_2306_08994_b200.device import set_small_front_limit
        set_small_front_limit(args.small_max_m)
    state = tf.init_state(system, plan)
    dp = tf.compile_execution(plan, None, state)
    nrhs = cfg["nrhs"]
    n = mesh.n_dof
    stats = plan.level_stats()
    dev = torch.device("cuda", local)
    rng = np.random.default_rng(0)
    b_host = torch.from_numpy(rng.standard_normal((n, nrhs))).pin_memory()
    b = b_host.to(dev)
    x = torch.empty_like(b)
    thr = state.zero_threshold
    lib = dp.lib
    stream = torch.cuda.current_stream(dev)
    sp = C.c_void_p(stream.cuda_stream)
    nl = len(dp.levels)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nl + 1)]
           for _ in range(args.steps)]
    level_ms = np.zeros(nl)

    sharded = None
    if world > 1:
        from paper_2306_08994_b200.distributed import ShardedFactorization, TorchComm
        sharded = ShardedFactorization(dp, world, TorchComm(), ranks=[rank])
        # a collective on every rank before the first (partial) P2P batch, so
        # the NCCL communicator exists on all ranks
        dist.barrier()

    def step(ev=None):
        record = ev is not None
        if record:
            ev[0].record(stream)
        if sharded is not None:
            hook = (lambda L: ev[L + 1].record(stream)) if record else None
            if sharded.factor(thr, stream, level_hook=hook) != -1:
                raise RuntimeError("zero pivot in benchmark system")
            sharded.solve_into(b, x, stream)
            return
        # one Foata class per level (tf_level_factor); the bottom levels as one
        # subtree launch (tf_subtree_factor)
        dp.factor(thr, stream, level_hook=(lambda L: ev[L + 1].record(stream)) if record else None)
        dp.solve_into(b, x, stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if sharded is None and dp.zero_pivot_position() != -1:
        raise RuntimeError("zero pivot in benchmark system")
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    from paper_2306_08994_b200 import _lib as tflib
    graph = None
    if sharded is None and not args.no_graph:
        # the whole factor + solve as one CUDA graph (DevicePlan.capture)
        # forward sweeps of the lower levels overlapped with the top levels'
        # latency-bound factorization (DevicePlan.factor_solve)
        graph = dp.capture(thr, b, x, warmup=False, overlap=not args.no_overlap)
        for _ in range(2):
            graph.replay()
        torch.cuda.synchronize()
        if dp.zero_pivot_position() != -1:
            raise RuntimeError("zero pivot in benchmark system (graph)")
    with ClockSampler(local) as clk:
        t0.record(stream)
        for i in range(args.steps):
            if graph is not None:
                graph.replay()
            else:
                step()
        t1.record(stream)
        torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / args.steps
    # diagnostic pass (not the headline): the same steps launched eagerly with
    # per-level events and per-kernel-class events inside the library
    lib.tf_timing_enable(1)
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d0.record(stream)
    for i in range(args.steps):
        step(evs[i])
    d1.record(stream)
    torch.cuda.synchronize()
    lib.tf_timing_enable(0)
    eager_ms = d0.elapsed_time(d1) / args.steps
    ktime = tflib.kernel_timing(lib)
    for ev in evs:
        for L in range(nl):
            level_ms[L] += ev[L].elapsed_time(ev[L + 1])
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    level_ms /= args.steps
    # per-level profile with the top slices off (the slices' levels finish
    # together in the pass above): the per-level times the scaling model and
    # the level report use
    level_ms_seq = level_ms
    if sharded is None and dp._split_plan() is not None:
        saved, dp.split_top = dp.split_top, 1
        level_ms_seq = np.zeros(nl)
        for i in range(args.steps):
            step(evs[i])
        torch.cuda.synchronize()
        for ev in evs:
            for L in range(nl):
                level_ms_seq[L] += ev[L].elapsed_time(ev[L + 1])
        level_ms_seq /= args.steps
        dp.split_top = saved
    # correctness guard on the measured system: relative residual of A x = b
    res = system.matvec(x[:, 0].cpu().numpy()) - b_host[:, 0].numpy()
    rel_res = float(np.abs(res).max() / np.abs(b_host[:, 0].numpy()).max())

    # ---- end-to-end through the public API with host buffers
    x_host = torch.empty((n, nrhs), dtype=torch.float64).pin_memory()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    elem_host = torch.from_numpy(np.ascontiguousarray(fronts.values).ravel()).pin_memory()
    copy_stream = torch.cuda.Stream(dev)
    b_dev = torch.empty((n, nrhs), dtype=torch.float64, device=dev)

    def e2e_step():
        dp.elem.copy_(elem_host, non_blocking=True)               # H2D: element matrices
        with torch.cuda.stream(copy_stream):                      # H2D: right-hand sides,
            b_dev.copy_(b_host, non_blocking=True)                # overlapping the factorization
        if sharded is not None:                                   # sharded path (N > 1)
            if sharded.factor(thr, stream) != -1:
                raise RuntimeError("zero pivot")
            stream.wait_stream(copy_stream)
            xd = torch.empty_like(b_dev)
            sharded.solve_into(b_dev, xd, stream)
        else:
            fac = tf.run_sequential(plan, state)                  # public API (checks pivots)
            stream.wait_stream(copy_stream)
            xd = tf.solve(fac, b_dev)
        x_host.copy_(xd, non_blocking=True)                       # D2H: solution
        torch.cuda.synchronize()

    for _ in range(max(1, args.warmup)):
        e2e_step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    h2d = b_host.numel() * 8 + elem_host.numel() * 8
    d2h = x_host.numel() * 8

    # ---- roofline of the dominant kernel (largest device time in the timed region)
    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    large = [dl.large for dl in dp.levels]
    schur_flops = panel_flops = small_bytes = asm_bytes = 0.0
    for L, (dl, st) in enumerate(zip(dp.levels, stats)):
        if large[L]:
            m_ = dl.tables.front_m().astype(float)
            k_ = dl.tables.front_k().astype(float)
            sf = float(((m_ - k_) * (m_ - k_ + 1) * k_).sum())
            schur_flops += sf
            panel_flops += st["ldl_flops"] - sf
            # the Schur epilogue writes S (fused assembly): the assembly kernel
            # reads the children and writes the panel
            asm_bytes += st["bytes"] - 8.0 * st["upd_entries"]
        else:
            small_bytes += st["bytes"]
    # solve sweeps (per direction): algorithmic bytes of each level
    solve_small = solve_large = 0.0
    for L, (dl, st) in enumerate(zip(dp.levels, stats)):
        # factor entries read once per sweep + each pivot's RHS row
        # read and written once (the update blocks passed between levels are
        # layout traffic, not algorithmic work)
        b_ = 8.0 * st["fac_entries"] + 16.0 * nrhs * float(st["pivots"])
        if large[L]:
            solve_large += b_
        else:
            solve_small += b_
    work = {  # algorithmic work per step of each kernel class
        "large_update_kernel<1> (schur)": ("tensor", schur_flops),
        "factor_small_kernel": ("hbm", small_bytes),
        "large_assemble_kernel": ("hbm", asm_bytes),
        "solve_fwd_small": ("hbm", solve_small),
        "solve_bwd_small": ("hbm", solve_small),
        "solve_fwd_wave": ("hbm", solve_large),
        "solve_bwd_wave": ("hbm", solve_large),
    }
    name = max(ktime, key=lambda k: ktime[k][0])
    tot_ms = sum(v[0] for v in ktime.values())
    k_ms, k_n = ktime[name]
    bound, w = work.get(name, ("tensor", None))
    if w is None:  # a class without a separate work model: fall back to the panel flops
        w = panel_flops
    t_launch = k_ms / k_n / 1e3
    per_launch = w * args.steps / k_n
    if bound == "hbm":
        roof = {"bound": "hbm", "achieved": per_launch / t_launch / 1e9, "peak": hbm,
                "unit": "GB/s"}
    else:
        roof = {"bound": "tensor", "achieved": per_launch / t_launch / 1e12,
                "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s"}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = measured_traffic(args.config, name)
    roof["kernel"] = name
    roof["launches_per_step"] = k_n / args.steps
    roof["share_of_kernel_time"] = k_ms / max(tot_ms, 1e-9)
    roof["time_basis"] = ("CUDA events around every launch of the class on its stream, "
                          "union of the launch intervals (concurrent launches counted once)")
    roof["peak_source"] = ("MEASURED_PEAKS.json hbm_gbs" if roof["bound"] == "hbm" else
                           "measured cuBLAS DGEMM 35.47 TF/s (profiles/r01_dgemm_cublas_peak.log)")
    kernel_ms = {k: round(v[0] / args.steps, 4) for k, v in
                 sorted(ktime.items(), key=lambda kv: -kv[1][0])}

    launches = dp.launches_per_factor() + dp.launches_per_solve(nrhs)
    total_ldl = sum(s["ldl_flops"] for s in stats)
    total_bytes = sum(s["bytes"] for s in stats)
    line = {
        "metric": "factor+solve DoF/s", "value": n / (ms / 1e3), "unit": "DoF/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong",  # same system for every N
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": args.config, "label": cfg["label"], "n_dof": n, "nrhs": nrhs,
                   "levels": nl, "factor_ms": float(level_ms.sum()),
                   "solve_ms": float(eager_ms - level_ms.sum()),
                   "launch": "one CUDA graph per step" if graph is not None else "eager",
                   "schedule": ("factor, then solve" if args.no_overlap else
                                f"forward sweeps of the levels below the top "
                                f"{dp.fwd_overlap_top} overlapped with their factorization"),
                   "eager_ms_per_step": eager_ms,
                   "top_slices": (None if world > 1 or dp._split_plan() is None else
                                  {"levels": [dp._split_plan()[0], dp._split_plan()[1] - 1],
                                   "slices": dp.split_top,
                                   "note": "factored concurrently in the timed schedule; "
                                           "level_ms is a per-level pass with the slices "
                                           "off"}),
                   "ldl_gflop": total_ldl / 1e9, "alg_bytes_gb": total_bytes / 1e9,
                   "l2": "working set >> 126 MB L2 (no flush needed)", "rel_residual": rel_res,
                   "parallelism": (f"subtree-sharded over {world} GPUs (NCCL P2P of root-ward "
                                   f"Schur complements)" if world > 1 else "1 GPU")},
        "e2e": {"value": n / (e2e_ms / 1e3), "unit": "DoF/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms},
        "gpu_launches": launches * args.steps,
        "clocks": clk.summary(),
        "roofline": roof,
        "level_ms": [round(float(t), 4) for t in level_ms_seq],
        "modelled_scaling": (modelled_scaling(dp, level_ms_seq, eager_ms - float(level_ms.sum()))
                             if world == 1 else None),
        "kernel_ms_per_step": kernel_ms,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-overlap", action="store_true",
                    help="factor, then solve (no forward sweeps during the top levels)")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch every kernel from the host each step instead of a CUDA graph")
    ap.add_argument("--small-max-m", type=int, default=None,
                    help="tuning: largest front order kept on the shared-memory kernels")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
