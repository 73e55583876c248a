"""Per-level timing of the GPU factorization + solve (CUDA events), for profiling runs."""
import argparse, ctypes as C, json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2306_08994_b200 as tf
from paper_2306_08994_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="1024,1024")
ap.add_argument("--degree", type=int, default=1)
ap.add_argument("--nrhs", type=int, default=1)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--small-max-m", type=int, default=None)
a = ap.parse_args()
if a.small_max_m is not None:
    from paper_2306_08994_b200.device import set_small_front_limit
    set_small_front_limit(a.small_max_m)
shape = tuple(int(x) for x in a.shape.split(","))
t0 = time.time()
mesh = tf.TensorMesh(shape, a.degree)
fronts = tf.generate_fronts(mesh)
tree = tf.build_elimination_tree(tf.sort_fronts(fronts), n_dof=mesh.n_dof)
system = tf.assemble_system(mesh, "one")
plan = tf.symbolic_eliminate(tree, system)
state = tf.init_state(system, plan)
dp = tf.compile_execution(plan, None, state)
print(f"plan {time.time()-t0:.1f}s n_dof={mesh.n_dof}", flush=True)
stats = plan.level_stats()
lib = dp.lib
def run_levels():
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(dp.levels) + 1)]
    dp.err.fill_(-1)
    prev = None
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    ev[0].record()
    for L, dl in enumerate(dp.levels):
        out = dp.upd[L & 1]
        rc = lib.tf_level_factor(C.byref(dl.view), None if prev is None else C.c_void_p(prev.data_ptr()),
                                 C.c_void_p(dp.elem.data_ptr()), C.c_void_p(dp.factors[L].data_ptr()),
                                 C.c_void_p(out.data_ptr()), C.c_double(state.zero_threshold),
                                 C.c_void_p(dp.err.data_ptr()), None, 0, sp)
        assert rc == 0
        prev = out
        ev[L + 1].record()
    torch.cuda.synchronize()
    return [ev[i].elapsed_time(ev[i + 1]) for i in range(len(dp.levels))]
for r in range(a.reps):
    times = run_levels()
assert dp.zero_pivot_position() == -1
# per-level kernel-class breakdown (events around every launch)
lib.tf_timing_enable(1)
_lib.kernel_timing(lib)
cls_rows = []
dp.err.fill_(-1)
prev = None
sp0 = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for L, dl in enumerate(dp.levels):
    out = dp.upd[L & 1]
    assert lib.tf_level_factor(C.byref(dl.view), None if prev is None else C.c_void_p(prev.data_ptr()),
                               C.c_void_p(dp.elem.data_ptr()), C.c_void_p(dp.factors[L].data_ptr()),
                               C.c_void_p(out.data_ptr()), C.c_double(state.zero_threshold),
                               C.c_void_p(dp.err.data_ptr()), None, 0, sp0) == 0
    prev = out
    torch.cuda.synchronize()
    cls_rows.append(_lib.kernel_timing(lib))
lib.tf_timing_enable(0)
tot = sum(times)
print(f"factor total {tot:.3f} ms")
for L, (t, s) in enumerate(zip(times, stats)):
    gfs = s["ldl_flops"] / t / 1e6 if t > 0 else 0
    gbs = s["bytes"] / t / 1e6 if t > 0 else 0
    print(f"L{L:2d} fronts={s['fronts']:9d} m={s['max_m']:5d} k={s['max_k']:5d} t={t:8.3f}ms "
          f"{gfs/1e3:7.2f} TF/s {gbs:8.1f} GB/s")
    print("      " + "  ".join(f"{k.split(' ')[0].replace('large_', '')[:14]}{k.split(' ')[-1] if '(' in k else ''}"
                              f"={v[0]:.3f}/{v[1]}" for k, v in cls_rows[L].items()))
b = torch.randn(mesh.n_dof, a.nrhs, dtype=torch.float64, device="cuda")
x = torch.empty_like(b)
for r in range(a.reps):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); dp.solve_into(b, x); e1.record(); torch.cuda.synchronize()
ts = e0.elapsed_time(e1)
print(f"solve nrhs={a.nrhs} {ts:.3f} ms")
r = torch.from_numpy(system.matvec(x.cpu().numpy())).cuda() - b
print("rel residual", (r.abs().max() / b.abs().max()).item())
print(json.dumps({"factor_ms": tot, "solve_ms": ts, "dof_per_s": mesh.n_dof / (tot + ts) * 1e3}))

# ---- per-level solve timing (forward then backward), CUDA events between launches
def solve_levels(nrhs):
    bb = torch.randn(mesh.n_dof, nrhs, dtype=torch.float64, device="cuda")
    xx = torch.empty_like(bb)
    dp.solve_into(bb, xx)  # allocate blocks
    torch.cuda.synchronize()
    nl = len(dp.levels)
    evf = [torch.cuda.Event(enable_timing=True) for _ in range(nl + 1)]
    evb = [torch.cuda.Event(enable_timing=True) for _ in range(nl + 1)]
    sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda t: None if t is None else C.c_void_p(t.data_ptr())
    blk, y = dp._blk, dp._y
    lib.tf_permute_rows(P(dp.pivot_order), dp.n_pivots, P(bb), P(y), nrhs, 0, sp)
    prev = None
    evf[0].record()
    for L, dl in enumerate(dp.levels):
        cur = blk[L & 1]
        ch = dp.levels[L - 1] if L > 0 else None
        assert lib.tf_level_solve_fwd(C.byref(dl.view), C.byref(ch.view) if ch else None,
                                      P(dp.factors[L]), P(prev), ch.max_m if ch else 0, P(cur),
                                      dl.max_m, P(y), nrhs, P(dp._ws), dp._ws_bytes, sp) == 0
        prev = cur
        evf[L + 1].record()
    prev = None
    evb[nl].record()
    for L in range(nl - 1, -1, -1):
        dl = dp.levels[L]
        cur = blk[L & 1]
        pa = dp.levels[L + 1] if L + 1 < nl else None
        assert lib.tf_level_solve_bwd(C.byref(dl.view), C.byref(pa.view) if pa else None,
                                      P(dp.factors[L]), P(prev), pa.max_m if pa else 0, P(cur),
                                      dl.max_m, P(y), nrhs, P(dp._ws), dp._ws_bytes, sp) == 0
        prev = cur
        evb[L].record()
    torch.cuda.synchronize()
    fw = [evf[L].elapsed_time(evf[L + 1]) for L in range(nl)]
    bw = [evb[L + 1].elapsed_time(evb[L]) for L in range(nl)]
    print(f"solve nrhs={nrhs} fwd {sum(fw):.3f} ms bwd {sum(bw):.3f} ms")
    for L in range(nl):
        print(f"  L{L:2d} fwd {fw[L]:8.3f} bwd {bw[L]:8.3f} ms")

solve_levels(a.nrhs)
