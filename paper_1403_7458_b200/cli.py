"""Command-line drop-in for the reference's ``spamm`` CLI on the GPU path
(reference cli.py:114-176, 336-384).

    python -m paper_1403_7458_b200 multiply A.mtx B.mtx --tau 1e-8 --out C.mtx --stats s.json
    python -m paper_1403_7458_b200 sp2 F.mtx --n-occ 150 --tau 1e-7 --out P.mtx --report r.json
    python -m paper_1403_7458_b200 sweep tau --f F.mtx --n-occ 150 --taus 1e-6,1e-8 --out e.csv
    python -m paper_1403_7458_b200 rerun C.mtx.manifest.json

Same subcommand names, flags, defaults, output files (MatrixMarket with 17
significant digits, the reference's stats / report JSON schemas, CSV columns)
and exit codes (0 on success, including a flagged non-convergence, which is
reported data; 2 on argument or input errors) as the reference.  Every
command writes ``<out>.manifest.json``; ``rerun`` replays it.  ``--mode``,
``--workers`` and ``--deterministic`` are accepted and validated as in the
reference; the device path is deterministic for any setting.  Extra flags:
``--leaf-kernel {auto,ozaki,dmma,exact}`` (exact = the reference's rounding, bitwise)
and, for ``sp2``, ``--criterion {trace,fro}`` / ``--fro-tol`` (BASELINE's
||X^2 - X||_F stopping rule).  The reference's ``gen``, ``sweep size`` and
``sweep pe`` (input generators and the decomposition simulator) are outside
the hot path.
"""

from __future__ import annotations

import argparse
import csv
import sys

from . import __version__, io

__all__ = ["main", "build_parser"]


# ----------------------------------------------------------------- helpers

def _floats(text: str) -> list:
    return [float(x) for x in text.split(",") if x]


def _tree(path, args):
    from .quadtree import build_from_dense
    return build_from_dense(io.read_matrix_market(path), args.block_size, args.chunk_size)


def _manifest(out_path, args, command: str, inputs: list, outputs: list, seeds=None) -> None:
    params = {k: v for k, v in vars(args).items() if k not in ("func", "argv")}
    io.write_manifest(f"{out_path}.manifest.json",
                      io.build_manifest(command, params, seeds or {}, inputs, outputs,
                                        argv=args.argv))


def _exec_kwargs(args) -> dict:
    return dict(mode=args.mode, workers=args.workers, kernel=args.leaf_kernel)


# ---------------------------------------------------------------- commands

def cmd_multiply(args) -> int:
    from .kernel import multiply
    from .quadtree import to_dense
    a, b = _tree(args.a, args), _tree(args.b, args)
    c, stats = multiply(a, b, args.tau, deterministic=args.deterministic,
                        **_exec_kwargs(args))
    io.write_matrix_market(args.out, to_dense(c), fmt=args.format)
    written = [args.out]
    if args.stats:
        io.write_json(args.stats, stats.to_json_dict())
        written.append(args.stats)
    _manifest(args.out, args, "multiply", [args.a, args.b], written)
    print(f"wrote {args.out}: leaf_products={stats.leaf_products} "
          f"flops~{stats.flop_estimate}")
    return 0


def cmd_sp2(args) -> int:
    from .quadtree import to_dense
    from .sp2 import idempotency_error, sp2_solve
    f = _tree(args.f, args)
    p, state = sp2_solve(f, args.n_occ, args.tau, max_iter=args.max_iter,
                         idem_tol=args.idem_tol, criterion=args.criterion,
                         fro_tol=args.fro_tol, **_exec_kwargs(args))
    io.write_matrix_market(args.out, to_dense(p), fmt=args.format)
    written = [args.out]
    if args.report:
        idem = idempotency_error(p, **_exec_kwargs(args))
        io.write_json(args.report, state.to_report_dict(idem_error=idem))
        written.append(args.report)
    _manifest(args.out, args, "sp2", [args.f], written)
    flag = "converged" if state.converged else "NOT CONVERGED"
    print(f"wrote {args.out}: {flag} after {state.iteration} iterations, "
          f"trace={state.trace_history[-1]:.6f}")
    return 0


def cmd_sweep_tau(args) -> int:
    """Energy error vs tolerance (cli.py:152-176; the paper's Fig. 2 study)."""
    from .kernel import convolution_census
    from .sp2 import energy_error, idempotency_error, sp2_solve
    f = _tree(args.f, args)
    kw = _exec_kwargs(args)
    p_ref, ref_state = sp2_solve(f, args.n_occ, 0.0, max_iter=args.max_iter, **kw)
    rows = []
    for tau in args.taus:
        p_tau, state = sp2_solve(f, args.n_occ, tau, max_iter=args.max_iter, **kw)
        err = energy_error(f, p_ref, p_tau, **kw)
        rows.append({
            "tau": tau,
            "energy_error": err,
            "abs_energy_error": abs(err),
            "idempotency_error": idempotency_error(p_tau, **kw),
            "iterations": state.iteration,
            "converged": state.converged,
            "leaf_products": convolution_census(p_tau, p_tau, tau).leaf_products,
        })
    with open(args.out, "w", newline="") as handle:
        w = csv.DictWriter(handle, fieldnames=list(rows[0].keys()))
        w.writeheader()
        w.writerows(rows)
    _manifest(args.out, args, "sweep tau", [args.f], [args.out])
    print(f"wrote {args.out}: {len(rows)} tolerance points "
          f"(reference solve: {ref_state.iteration} iterations)")
    return 0


def cmd_rerun(args) -> int:
    argv = io.read_manifest(args.manifest)["argv"]
    print(f"replaying: spamm {' '.join(argv)}")
    return main(argv)


# ------------------------------------------------------------------ parser

def _tree_flags(p) -> None:
    p.add_argument("--block-size", type=int, default=16,
                   help="dense leaf block edge (power of two)")
    p.add_argument("--chunk-size", type=int, default=None,
                   help="distribution chunk edge (power of two, default n_padded/8)")


def _exec_flags(p) -> None:
    from .kernel import WORKERS_ENV_VAR
    p.add_argument("--mode", choices=["serial", "tasked"], default="serial")
    p.add_argument("--workers", type=int, default=None,
                   help=f"tasked-mode worker count (default ${WORKERS_ENV_VAR} or cpu count)")
    p.add_argument("--deterministic", action=argparse.BooleanOptionalAction, default=True,
                   help="fix the accumulation order (the device path always does)")
    p.add_argument("--leaf-kernel", choices=["auto", "ozaki", "dmma", "exact"], default="auto",
                   help="auto: INT8-digit tensor-core products for block size 64 (ozaki), "
                        "FP64 tensor cores (dmma) otherwise (rel. Frobenius <= 1e-12); "
                        "exact: bitwise the reference's rounding")


def _format_flag(p) -> None:
    p.add_argument("--format", choices=list(io.MM_FORMATS), default="auto")


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="spamm", description="Occluded quadtree multiply and SP2 projection on B200")
    parser.add_argument("--version", action="version", version=__version__)
    sub = parser.add_subparsers(dest="command", required=True)

    mul = sub.add_parser("multiply", help="occluded product of two matrices")
    mul.add_argument("a")
    mul.add_argument("b")
    mul.add_argument("--tau", type=float, default=0.0)
    _tree_flags(mul)
    _exec_flags(mul)
    _format_flag(mul)
    mul.add_argument("--out", required=True)
    mul.add_argument("--stats", default=None, help="write occlusion stats JSON")
    mul.set_defaults(func=cmd_multiply)

    sp2 = sub.add_parser("sp2", help="spectral projection solve")
    sp2.add_argument("f")
    sp2.add_argument("--n-occ", type=int, required=True)
    sp2.add_argument("--tau", type=float, default=0.0)
    sp2.add_argument("--max-iter", type=int, default=100)
    sp2.add_argument("--idem-tol", type=float, default=1e-9)
    sp2.add_argument("--criterion", choices=["trace", "fro"], default="trace")
    sp2.add_argument("--fro-tol", type=float, default=1e-6)
    _tree_flags(sp2)
    _exec_flags(sp2)
    _format_flag(sp2)
    sp2.add_argument("--out", required=True)
    sp2.add_argument("--report", default=None, help="write solve report JSON")
    sp2.set_defaults(func=cmd_sp2)

    sweep = sub.add_parser("sweep", help="experiment sweeps to CSV")
    kinds = sweep.add_subparsers(dest="sweep_kind", required=True)
    tau = kinds.add_parser("tau", help="energy error vs tolerance")
    tau.add_argument("--f", required=True)
    tau.add_argument("--n-occ", type=int, required=True)
    tau.add_argument("--taus", type=_floats, default=[1e-6, 1e-8, 1e-10])
    tau.add_argument("--max-iter", type=int, default=100)
    _tree_flags(tau)
    _exec_flags(tau)
    tau.add_argument("--out", required=True)
    tau.set_defaults(func=cmd_sweep_tau)

    rerun = sub.add_parser("rerun", help="replay a recorded manifest")
    rerun.add_argument("manifest")
    rerun.set_defaults(func=cmd_rerun)
    return parser


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    args = build_parser().parse_args(argv)
    args.argv = argv
    try:
        return args.func(args)
    except (ValueError, FileNotFoundError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
