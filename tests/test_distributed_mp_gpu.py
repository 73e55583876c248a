"""The multi-process sharded path with the REAL kernels: two processes, one GPU.

Each process is one rank of a world-2 torch.distributed group (gloo; the
device buffers are staged through host memory by HostStagedComm, so the two
ranks never wait on each other's kernels) and factors only the fronts it
owns with the production level kernels (tf_level_factor on slice views),
exchanging root-ward Schur complements and solve blocks point to point.
Checks, per rank:
* factors (after gather_all) bitwise equal to the one-GPU factorization;
* the sharded solve (forward/backward block exchanges + all-gather of owned
  rows) matches the reference golden solution;
* the public API run_concurrent(schedule, graph, state, workers=2) returns a
  complete FactorResult whose solve matches too.
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _written_equal(dp, ref, got):
    import torch
    for L, dl in enumerate(dp.levels):
        lt = dl.tables
        for f in range(dl.n_fronts):
            row = lt.pat[lt.pattern_of[f]]
            m, k, kp = int(row[0]), int(row[1]), int(row[9])
            if k == 0:
                continue
            a = ref[L][f * dl.fac_stride: f * dl.fac_stride + m * kp + kp]
            b = got[L][f * dl.fac_stride: f * dl.fac_stride + m * kp + kp]
            mask = torch.tril(torch.ones(m, kp, dtype=torch.bool, device=a.device))
            mask[:, k:] = False
            if not (torch.equal(a[:m * kp].view(m, kp)[mask], b[:m * kp].view(m, kp)[mask]) and
                    torch.equal(a[m * kp:m * kp + k], b[m * kp:m * kp + k])):
                return (L, f)
    return None


def _worker(rank, world, port, name, q):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    import paper_2306_08994_b200 as tf
    from paper_2306_08994_b200.distributed import HostStagedComm, ShardedFactorization
    from conftest import golden, mesh_of
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        g = golden(name)
        mesh = mesh_of(g)
        system = tf.assemble_system(mesh, "one")
        tree = tf.build_elimination_tree(tf.sort_fronts(tf.generate_fronts(mesh)))
        plan = tf.symbolic_eliminate(tree, system)
        # one-GPU reference factorization in this process
        single = tf.run_sequential(plan, tf.init_state(system, plan))
        ref = [t.clone() for t in single.device_plan.factors]
        # sharded: this rank's fronts only
        state = tf.init_state(system, plan)
        dp = tf.compile_execution(plan, None, state)
        sf = ShardedFactorization(dp, world, HostStagedComm(), ranks=[rank])
        out["zero_pivot"] = sf.factor(state.zero_threshold)
        torch.cuda.synchronize()
        b = torch.from_numpy(np.stack([g["rhs"], g["rhs"] * 2.0], 1)).cuda()
        x = torch.empty_like(b)
        sf.solve_into(b, x)
        xs = x[:, 0].cpu().numpy()
        out["solve_err"] = float(np.abs(xs - g["x"]).max() / np.abs(g["x"]).max())
        out["col2"] = float(np.abs(x[:, 1].cpu().numpy() - 2.0 * xs).max())
        sf.gather_all()
        out["mismatch"] = _written_equal(dp, ref, dp.factors)
        # public API: run_concurrent over the group
        graph = tf.build_task_graph(tree, system) if plan.native.keep_lists else plan
        st2 = tf.init_state(system, plan)
        res = tf.run_concurrent(None, graph, st2, workers=world)
        x2 = tf.solve(res, g["rhs"])
        out["api_err"] = float(np.abs(x2 - g["x"]).max() / np.abs(g["x"]).max())
    except Exception as exc:  # report, do not hang the peer
        import traceback
        out["error"] = traceback.format_exc()
    finally:
        q.put((rank, out))
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["2d_64x64_p2", "2d_16x16_p2", "3d_4x4x4_p1", "1d_n1000_p1"])
def test_two_processes_one_gpu_real_kernels(name, cuda_ok):
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        o = res[r]
        assert "error" not in o, o.get("error")
        assert o["zero_pivot"] == -1
        assert o["mismatch"] is None, o["mismatch"]
        assert o["solve_err"] <= 1e-10 and o["api_err"] <= 1e-10, o
        assert o["col2"] <= 1e-12
