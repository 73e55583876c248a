"""TEST INFRASTRUCTURE ONLY — the reference arm / CPU baseline of bench.py.

Times the reference's arithmetic on the host cores: the C port of
factorize_nested_loops + solve (oracle/tf_oracle.c, bitwise equal to the
reference, engine.py:500-552 and 468-493) on a bounded sample of the
workload.  Imports nothing from the product package: the problem comes
from oracle/mesh_nd.py and the work model from oracle/workmodel.py.

* The sample is the workload itself when it is small (cfg1, cfg2), else the
  same element type and dimension on a mesh halved per axis until one
  factor+solve is <= SAMPLE_LU_BUDGET reference task-flops (about 1-3 s per core).
* One step forks one process per usable core; each factors + solves its own
  copy of the sample (the reference's cell-level order is sequential per
  system, so independent systems are how its arithmetic uses many cores).
  Step time = wall time of the whole step.
* `value` (DoF/s of the WORKLOAD) = n_dof(workload) x aggregate measured
  task-flop rate / task-flops(workload): the sample's measured rate applied
  to the workload's exact task count, assuming the workload's tasks would
  spread perfectly over all cores (generous to the CPU).  When the sample is
  the workload, the value is measured directly.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import platform
import resource
import time

import numpy as np

from . import workmodel
from .mesh_nd import element_matrix, tensor_mesh
from .tfo import OracleFactors, load

SAMPLE_LU_BUDGET = 3.0e8


def cpu_info() -> dict:
    model = platform.processor() or "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count() or 1
    return {"cpu_model": model, "nproc": usable, "logical_cpus": os.cpu_count()}


def sample_shape(ns, p):
    ns = tuple(int(x) for x in ns)
    s = ns
    while workmodel.workload(s, p)["lu_task_flops"] > SAMPLE_LU_BUDGET and min(s) > 1:
        s = tuple(max(1, x // 2) for x in s)
    return s


class Sample:
    def __init__(self, ns, p, nrhs: int = 1):
        load()
        self.ns, self.p, self.nrhs = tuple(ns), p, int(nrhs)
        self.n_dof, elems, _ = tensor_mesh(self.ns, p)
        self.dofs = np.asarray(elems, dtype=np.int32)
        self.emat = element_matrix(self.ns, p)
        self.work = workmodel.workload(self.ns, p)
        self.rhs = np.random.default_rng(0).standard_normal((self.n_dof, self.nrhs))

    def run_once(self) -> tuple[float, float]:
        """(factor seconds, solve seconds); the reference solves one column at a time."""
        t0 = time.perf_counter()
        o = OracleFactors(self.n_dof, self.dofs, self.emat)
        t1 = time.perf_counter()
        for j in range(self.nrhs):
            o.solve(self.rhs[:, j])
        t2 = time.perf_counter()
        del o
        return t1 - t0, t2 - t1


def _child(sample: Sample, q):
    tf_, ts_ = sample.run_once()
    q.put((tf_, ts_, resource.getrusage(resource.RUSAGE_SELF).ru_maxrss * 1024))


def run_step(sample: Sample, procs: int):
    """Fork `procs` independent factor+solve runs: (wall seconds, [(t_factor, t_solve)], max rss)."""
    ctx = mp.get_context("fork")
    q = ctx.Queue()
    t0 = time.perf_counter()
    ps = [ctx.Process(target=_child, args=(sample, q)) for _ in range(procs)]
    for p in ps:
        p.start()
    res = [q.get() for _ in ps]
    for p in ps:
        p.join()
    wall = time.perf_counter() - t0
    return wall, [(r[0], r[1]) for r in res], max(r[2] for r in res)


def choose_procs(sample: Sample) -> tuple[int, int]:
    """(processes, max rss of one run) bounded by usable cores and available memory."""
    _, _, rss = run_step(sample, 1)
    cores = cpu_info()["nproc"]
    avail = None
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable"):
                avail = int(line.split()[1]) * 1024
    except OSError:
        pass
    n = cores
    if avail:
        n = max(1, min(n, int(0.6 * avail / max(rss, 1))))
    return n, rss


def describe(work_ns, p, nrhs: int, sample: Sample, procs: int, wall: float, per: list) -> dict:
    """Workload DoF/s from a measured step.  Factor time scales with the
    reference task count, solve time with factor entries x right-hand sides."""
    w = workmodel.workload(work_ns, p)
    same = tuple(work_ns) == sample.ns and nrhs == sample.nrhs
    tf_ = np.array([a for a, _ in per])
    ts_ = np.array([b for _, b in per])
    f_frac = float(tf_.mean() / (tf_.mean() + ts_.mean()))
    r_f = w["lu_task_flops"] / sample.work["lu_task_flops"]
    r_s = (w["factor_entries"] * nrhs) / (sample.work["factor_entries"] * sample.nrhs)
    t_work = wall * (f_frac * r_f + (1 - f_frac) * r_s) / procs      # all cores
    t_one = float(tf_.min()) * r_f + float(ts_.min()) * r_s           # one core
    info = cpu_info()
    return {
        "value": w["n_dof"] / t_work, "unit": "DoF/s", "cores": procs, "kind": "port",
        "value_basis": "measured" if same and procs == 1 else
                       ("measured (aggregate of independent copies)" if same else "extrapolated"),
        "sample": (f"{'x'.join(map(str, sample.ns))} Q{p} ({sample.n_dof} DoF, "
                   f"{sample.work['lu_task_flops']:.3e} reference task-flops, {sample.nrhs} RHS) "
                   f"factor+solve with the reference's cell-level arithmetic "
                   f"(oracle/tf_oracle.c), {procs} independent copies in parallel, one per core"
                   + ("" if same else
                      f"; workload: factor time x {r_f:.4g} (task-flop ratio), solve time x "
                      f"{r_s:.4g} (factor entries x RHS ratio)")),
        "sample_seconds_per_step": wall,
        "sample_dof_per_s_measured": procs * sample.n_dof / wall,
        "single_core_value": w["n_dof"] / t_one,
        "factor_fraction": f_frac,
        "workload_task_flops": w["lu_task_flops"],
        "cpu_model": info["cpu_model"], "nproc": info["nproc"],
    }
