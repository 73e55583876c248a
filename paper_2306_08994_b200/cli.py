"""Command-line harness mirroring `tracefront` (cli.py:64-356): plan, factorize,
solve, verify, bench.  Same flags and exit codes (0 ok, 1 usage, 2 numerical,
3 verification failure); `--mesh NxN[xN]` selects a 2D/3D tensor mesh and
`--nrhs` solves several right-hand sides at once.

    python -m paper_2306_08994_b200.cli solve --elements 1024 --degree 1
    python -m paper_2306_08994_b200.cli bench --mesh 1024x1024 --degree 1 --nrhs 64
"""

from __future__ import annotations

import argparse
import csv
import sys
import time
from pathlib import Path
from typing import Optional

import numpy as np

from . import fileio

EXIT_OK, EXIT_USAGE, EXIT_NUMERICAL, EXIT_VERIFY = 0, 1, 2, 3
DEFAULT_ORACLE_CAP = 2000


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        self.print_usage(sys.stderr)
        print(f"{self.prog}: error: {message}", file=sys.stderr)
        sys.exit(EXIT_USAGE)


def build_parser() -> _Parser:
    from .fem import RHS_FUNCTIONS
    parser = _Parser(prog="tracefront-b200", description=__doc__)
    sub = parser.add_subparsers(dest="command", required=True)

    def common(p):
        g = p.add_mutually_exclusive_group(required=True)
        g.add_argument("--elements", type=int, help="1D element count")
        g.add_argument("--mesh", type=str, help="tensor mesh, e.g. 64x64 or 32x32x32")
        p.add_argument("--degree", type=int, default=1)
        p.add_argument("--rhs", default="one", choices=sorted(RHS_FUNCTIONS))
        p.add_argument("--workers", type=int, default=1)
        p.add_argument("--nrhs", type=int, default=1)
        p.add_argument("--out", type=Path, default=Path("."))

    common(sub.add_parser("generate", help="export matrix.mtx, rhs.txt, manifest.json"))
    common(sub.add_parser("plan", help="tree / level-schedule statistics"))
    common(sub.add_parser("factorize", help="factorize and export the pivot order"))
    common(sub.add_parser("solve", help="factorize and solve, export the solution"))
    pv = sub.add_parser("verify", help="check against a dense CPU solve")
    common(pv)
    pv.add_argument("--oracle-cap", type=int, default=DEFAULT_ORACLE_CAP)
    pv.add_argument("--tolerance", type=float, default=None)
    pb = sub.add_parser("bench", help="timing, CSV output")
    common(pb)
    pb.add_argument("--repeats", type=int, default=5)
    return parser


def _mesh(args, parser):
    from . import Mesh, TensorMesh
    if args.degree not in (1, 2, 3):
        parser.error(f"--degree must be 1, 2, or 3, got {args.degree}")
    if args.workers < 1 or args.nrhs < 1:
        parser.error("--workers and --nrhs must be >= 1")
    if args.elements is not None:
        if args.elements < 1:
            parser.error(f"--elements must be >= 1, got {args.elements}")
        return Mesh(args.elements, args.degree)
    try:
        shape = tuple(int(t) for t in args.mesh.lower().split("x"))
    except ValueError:
        parser.error(f"bad --mesh {args.mesh!r}")
    if not 1 <= len(shape) <= 3 or min(shape) < 1:
        parser.error(f"bad --mesh {args.mesh!r}")
    return TensorMesh(shape, args.degree)


def _pipeline(mesh, rhs_name):
    import paper_2306_08994_b200 as tf
    system = tf.assemble_system(mesh, rhs_name)
    tree = tf.build_elimination_tree(tf.sort_fronts(tf.generate_fronts(mesh)), n_dof=mesh.n_dof)
    plan = tf.symbolic_eliminate(tree, system)
    return tf, system, tree, plan


def _rhs(system, nrhs):
    b = np.asarray(system.rhs, dtype=float)
    if nrhs == 1:
        return b
    extra = np.random.default_rng(0).standard_normal((len(b), nrhs - 1))
    return np.concatenate([b[:, None], extra], axis=1)


def cmd_generate(args, parser) -> int:
    """matrix.mtx, rhs.txt, manifest.json (cli.py:164-183)."""
    import json
    mesh = _mesh(args, parser)
    from .fem import assemble_system
    system = assemble_system(mesh, args.rhs)
    args.out.mkdir(parents=True, exist_ok=True)
    fileio.write_matrix_market_symmetric(args.out / "matrix.mtx", system)
    fileio.write_vector(args.out / "rhs.txt", system.rhs)
    manifest = {"n_elements": int(getattr(mesh, "n_elements", 0)), "degree": mesh.degree,
                "n_dof": mesh.n_dof, "rhs": args.rhs}
    if hasattr(mesh, "domain_start"):
        manifest["domain"] = [mesh.domain_start, mesh.domain_end]
    if hasattr(mesh, "shape"):
        manifest["shape"] = list(mesh.shape)
    (args.out / "manifest.json").write_text(json.dumps(manifest, sort_keys=True, indent=2) + "\n")
    print(f"wrote matrix.mtx rhs.txt manifest.json to {args.out} (n_dof={mesh.n_dof})")
    return EXIT_OK


def cmd_plan(args, parser) -> int:
    mesh = _mesh(args, parser)
    tf, system, tree, plan = _pipeline(mesh, args.rhs)
    ls = plan.level_stats()
    print(f"n_dof={mesh.n_dof}")
    print(f"tree_depth={tree.n_levels}")
    if plan.native.keep_lists:
        # the reference's atomic trace (cli.py:184-196), streamed natively
        sched = tf.compute_atomic_fnf(plan)
        for kind in tf.TaskKind:
            print(f"tasks_{kind.name.lower()}={sched.kind_counts[kind]}")
        print(f"tasks_total={sched.n_tasks}")
    else:
        sched = tf.compute_fnf(plan)
    st = tf.schedule_stats(sched)
    print(f"foata_classes={st.n_classes}")
    print(f"max_class_width={st.max_width}")
    print(f"level_classes={tree.n_levels}")
    print(f"pivots={plan.native.n_pivots}")
    print(f"max_front={plan.native.max_m}")
    print(f"ldl_flops={sum(s['ldl_flops'] for s in ls):.6e}")
    print(f"lu_task_flops={sum(s['lu_flops'] for s in ls):.6e}")
    return EXIT_OK


def _factorize(tf, plan, system):
    import torch
    state = tf.init_state(system, plan)
    tf.compile_execution(plan, None, state)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    factors = tf.run_sequential(plan, state)
    torch.cuda.synchronize()
    return factors, time.perf_counter() - t0


def cmd_factorize_solve(args, parser) -> int:
    mesh = _mesh(args, parser)
    tf, system, tree, plan = _pipeline(mesh, args.rhs)
    factors, wall = _factorize(tf, plan, system)
    args.out.mkdir(parents=True, exist_ok=True)
    if args.command == "factorize":  # cli.py:207-218 exports
        lower, upper = fileio.factor_exports(factors)
        fileio.write_matrix_market_general(args.out / "L.mtx", mesh.n_dof, mesh.n_dof, lower)
        fileio.write_matrix_market_general(args.out / "U.mtx", mesh.n_dof, mesh.n_dof, upper)
        fileio.write_vector(args.out / "pivot_order.txt", factors.pivot_order)
    else:
        b = _rhs(system, args.nrhs)
        x = tf.solve(factors, b)
        if x.ndim == 1:
            fileio.write_vector(args.out / "solution.txt", x)
        else:
            np.savetxt(args.out / "solution.txt", x, fmt="%.17g")
        r = system.matvec(x) - b
        scale = np.linalg.norm(b)
        print(f"residual={np.linalg.norm(r) / (scale if scale > 0 else 1.0):.3e}")
    print(f"mode=gpu n_dof={mesh.n_dof} p={args.degree} workers={args.workers} "
          f"wall_seconds={wall:.6f}")
    return EXIT_OK


def cmd_verify(args, parser) -> int:
    mesh = _mesh(args, parser)
    if mesh.n_dof > args.oracle_cap:
        parser.error(f"n_dof={mesh.n_dof} exceeds the oracle cap {args.oracle_cap}; "
                     "raise --oracle-cap to verify larger systems")
    tol_res = 1e-10 if args.tolerance is None else args.tolerance
    tol_fac = 1e-12 if args.tolerance is None else args.tolerance
    tf, system, tree, plan = _pipeline(mesh, args.rhs)
    factors, _ = _factorize(tf, plan, system)
    dense = system.to_dense()
    lower, upper = factors.permuted_dense_factors()
    perm = factors.permutation()
    fdev = np.linalg.norm(lower @ upper - dense[np.ix_(perm, perm)]) / np.linalg.norm(dense)
    b = _rhs(system, 1)
    x = tf.solve(factors, b)
    xo = np.linalg.solve(dense, b)  # independent dense check (verification only)
    sdev = np.linalg.norm(x - xo) / max(np.linalg.norm(xo), 1e-300)
    res = np.linalg.norm(dense @ x - b) / max(np.linalg.norm(b), 1e-300)
    print(f"factor_deviation={fdev:.3e} (tolerance {tol_fac:.1e})")
    print(f"solution_deviation={sdev:.3e} (tolerance {tol_res:.1e})")
    print(f"residual={res:.3e} (tolerance {tol_res:.1e})")
    ok = fdev <= tol_fac and sdev <= tol_res and res <= tol_res
    print("verify: PASS" if ok else "verify: FAIL")
    return EXIT_OK if ok else EXIT_VERIFY


def cmd_bench(args, parser) -> int:
    import torch
    mesh = _mesh(args, parser)
    tf, system, tree, plan = _pipeline(mesh, args.rhs)
    state = tf.init_state(system, plan)
    dp = tf.compile_execution(plan, None, state)
    b = torch.from_numpy(np.ascontiguousarray(_rhs(system, args.nrhs))).cuda()
    x = torch.empty_like(b)
    walls = []
    for i in range(args.repeats + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dp.factor(state.zero_threshold)
        dp.solve_into(b, x)
        e1.record()
        torch.cuda.synchronize()
        if i:
            walls.append(e0.elapsed_time(e1) / 1e3)
    if dp.zero_pivot_position() != -1:
        raise SystemExit(EXIT_NUMERICAL)
    wall = float(np.mean(walls))
    out = args.out if args.out.suffix == ".csv" else args.out / "bench.csv"
    out.parent.mkdir(parents=True, exist_ok=True)
    ls = plan.level_stats()
    with open(out, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["n_dof", "p", "workers", "mode", "wall_seconds", "tasks_total",
                    "foata_classes", "nrhs", "dof_per_s"])
        w.writerow([mesh.n_dof, args.degree, args.workers, "gpu", f"{wall:.6f}",
                    f"{sum(s['lu_flops'] for s in ls):.0f}", tree.n_levels, args.nrhs,
                    f"{mesh.n_dof / wall:.6e}"])
    print(f"bench n_dof={mesh.n_dof} p={args.degree} workers={args.workers} mode=gpu "
          f"wall_seconds={wall:.6f} dof_per_s={mesh.n_dof / wall:.3e}")
    return EXIT_OK


def main(argv: Optional[list[str]] = None) -> int:
    from .errors import TracefrontError, ZeroPivotError
    parser = build_parser()
    args = parser.parse_args(argv)
    cmds = {"generate": cmd_generate, "plan": cmd_plan, "factorize": cmd_factorize_solve, "solve": cmd_factorize_solve,
            "verify": cmd_verify, "bench": cmd_bench}
    try:
        return cmds[args.command](args, parser)
    except ZeroPivotError as exc:
        print(f"numerical error: {exc}", file=sys.stderr)
        return EXIT_NUMERICAL
    except TracefrontError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_USAGE


if __name__ == "__main__":
    sys.exit(main())
