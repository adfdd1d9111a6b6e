"""`online` command on the GPU plan -- drop-in for `subapsnap online`
(reference cli.py:637-666, parser cli.py:694-698, exit codes cli.py:30-32).

    python -m paper_2510_04825_b200.cli online <config> --artifacts DIR [--out DIR] [--workers N]

Reads the reference's experiment config and offline artifacts exactly as the
reference does (basis.npz, selector_<strategy>.json, plan_<strategy>.npz in
the reference formats) and writes the same results.csv (method, p,
relative_residual, output_error, wall_time_s), but the online phase runs on
libsas: precompute_online/load_plan build the device plan, solve_batch is one
batched GPU solve, OnlineSolution.lift is the GPU lift (sas_lift).  The
verification residual ||A(p) x - b(p)|| / max(||b(p)||, 1e-300) uses the
system's own matrix and right-hand side, outside the timed region, as the
reference does.

The experiment vocabulary (config parsing, problem builders, test sweeps,
CSV formatting) is the reference's own: it is imported from the reference
package (the baseline/_ref install, else /root/reference when present) --
this module only swaps the online engine.
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def _reference():
    for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (p / "subapsnap" / "__init__.py").exists():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            import subapsnap.cli
            import subapsnap.errors
            import subapsnap.snapshot
            import subapsnap.subsample
            import subapsnap.systems
            return subapsnap
    raise ImportError("the reference package (subapsnap) is needed for its config and problem vocabulary; "
                      "install it into baseline/_ref (see DESIGN.md)")


def run_online(cfg, artifacts_dir, outdir, workers: int = 1, device: int = 0) -> dict:
    """cli.run_online (cli.py:637-666) with the GPU online phase."""
    from . import online
    ref = _reference()
    rcli, rsys_mod, ConfigError = ref.cli, ref.systems, ref.errors.ConfigError
    artifacts_dir = Path(artifacts_dir)
    outdir = Path(outdir)
    outdir.mkdir(parents=True, exist_ok=True)
    system = rsys_mod.build_problem(cfg.problem)
    basis_path = artifacts_dir / "basis.npz"
    if not basis_path.exists():
        raise ConfigError(f"missing offline artifact {basis_path}")
    basis = ref.snapshot.load_snapshot(basis_path)
    params = rcli.test_parameters(system, cfg)
    rows = []
    for strat in rcli._strategies(cfg.methods):
        sel_path = artifacts_dir / f"selector_{strat}.json"
        plan_path = artifacts_dir / f"plan_{strat}.npz"
        if not sel_path.exists() or not plan_path.exists():
            raise ConfigError(f"missing offline artifacts for {strat!r} in {artifacts_dir}")
        sel = ref.subsample.load_selector(sel_path)
        plan = online.load_plan(plan_path, system, basis, sel, device=device)
        batch = online.solve_batch(plan, params, workers=workers)
        xs = online.lift_batch(plan, np.stack([row.solution.coefficients for row in batch]))
        for row, p, x in zip(batch, params, xs):
            b = system.full_rhs(p)
            bn = max(np.linalg.norm(b), 1e-300)
            res = np.linalg.norm(system.matrix(p) @ x - b)
            rows.append((f"subapsnap-{strat}", rcli.format_param(p), rcli._fmt(res / bn), "",
                         rcli._fmt(row.wall_time)))
    results_path = outdir / "results.csv"
    rcli._write_csv(results_path, rcli.RESULT_HEADER, rows)
    return {"results": results_path}


def _build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2510_04825_b200.cli",
                                     description="SubApSnap online phase on B200 (drop-in for `subapsnap online`)")
    sub = parser.add_subparsers(dest="command", required=True)
    p_on = sub.add_parser("online", help="run the online phase from artifacts")
    p_on.add_argument("config")
    p_on.add_argument("--artifacts", required=True)
    p_on.add_argument("--out", default="out")
    p_on.add_argument("--workers", type=int, default=1)
    p_on.add_argument("--device", type=int, default=0)
    return parser


def main(argv=None) -> int:
    from . import errors as own
    args = _build_parser().parse_args(argv)
    ref = _reference()
    rcli, errors = ref.cli, ref.errors
    try:
        cfg = rcli.load_config(rcli.resolve_config(args.config))
        paths = run_online(cfg, args.artifacts, args.out, workers=args.workers, device=args.device)
    except (errors.ConfigError, own.ConfigError) as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return rcli.EXIT_CONFIG
    except (errors.SubapsnapError, own.SubapsnapError) as exc:
        print(f"numerical failure: {exc}", file=sys.stderr)
        return rcli.EXIT_NUMERICAL
    for key, path in sorted(paths.items()):
        print(f"{key}: {path}")
    return rcli.EXIT_OK


if __name__ == "__main__":
    raise SystemExit(main())
