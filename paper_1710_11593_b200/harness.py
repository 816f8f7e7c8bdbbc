"""Convergence tables on the GPU path, in the reference harness's output format.

Restates `run_convergence` / `exponent_ladder` / `emit_csv` / `emit_markdown`
(reference proj/src/harness.cpp:135-164, 184-236, 296-316) for the schemes on
this path (Example 2 = transport, Scheme 2; Example 3 = wave, Scheme 3;
Example 4 = diffusion, Scheme 4, harness.cpp:58-86): manufactured solutions at h = 2^-e (tau = 2^-e, or a fixed
tau = 2^-P), the final-time L2 error (`l2_error`, schemes.cpp:525-542), the
rate between consecutive ladder levels, and the CSV header/columns the
reference emits (`%.17g` doubles).  The forcing is generated on the device
(`ft_assemble_rhs_modes`); iterations are 0 (direct D&C, no Krylov).

    python -m paper_1710_11593_b200.harness --example 4 --gamma 0.5 --levels 3..8
"""
from __future__ import annotations

import argparse
import io
import math
import sys
from dataclasses import dataclass
from typing import Iterable, List, Optional

import numpy as np

from . import Plan, SchemeId, SolveMethod
from . import workloads as W

SCHEME_NAME = {SchemeId.Hyperbolic: "hyperbolic", SchemeId.DiffusionWave: "wave",
               SchemeId.Diffusion: "diffusion"}  # schemes.cpp:24-32
HEADER = "mesh_exp,h,tau,l2_error,rate,iterations,wall_seconds,method,gamma,scheme"  # harness.cpp:297


@dataclass
class ConvergenceRow:
    mesh_exp: int
    h: float
    tau: float
    l2_error: float
    rate: Optional[float]
    iterations: int
    wall_seconds: float
    method: str
    gamma: float
    scheme: str


def exponent_ladder(lo: int, hi: int, fixed_time_exp: Optional[int] = None):
    """harness.cpp:135-152: (exponent, time_steps, space_cells) per level."""
    if lo < 1 or hi < lo:
        raise ValueError("exponent_ladder: need 1 <= from <= to")
    return [(e, 1 << (fixed_time_exp if fixed_time_exp is not None else e), 1 << e) for e in range(lo, hi + 1)]


def _example(eid: int, gamma: float, time_steps: int, cells: int) -> W.Workload:
    w = W.example(eid, gamma, 1)
    s = w.specs[0]
    s.time_steps, s.space_cells = time_steps, cells
    return w


def run_example(eid: int, gamma: float, exp: int, time_steps: int, cells: int,
                method: SolveMethod = SolveMethod.Fast) -> ConvergenceRow:
    """harness.cpp:176-194 on the GPU: solve the manufactured problem, L2 error at t = T."""
    import torch

    if eid not in (2, 3, 4):
        raise ValueError("example id must be 2 (transport), 3 (wave) or 4 (diffusion) on this path")
    w = _example(eid, gamma, time_steps, cells)
    plan = Plan(w.specs)
    rhs = torch.empty(plan.shape, dtype=torch.float64, device="cuda")
    plan.assemble_rhs_modes(rhs, w.a, w.k, w.p, w.trig, w.u0amp, w.phiamp)
    u = torch.empty_like(rhs)
    _, rep = (plan.solve_fast if method == SolveMethod.Fast else plan.solve_direct)(rhs, u)
    s = w.specs[0]
    err = W.l2_final(w, u.cpu().numpy())
    return ConvergenceRow(exp, s.h(), s.tau(), err, None, rep.iterations, rep.seconds, rep.method, gamma,
                          SCHEME_NAME[s.scheme])


def run_convergence(eid: int, gammas: Iterable[float], ladder, methods=(SolveMethod.Fast,)) -> List[ConvergenceRow]:
    """harness.cpp:196-236: rows ordered gamma, method, mesh; rates within each run."""
    rows: List[ConvergenceRow] = []
    for g in gammas:
        for m in methods:
            run = [run_example(eid, g, e, n, c, m) for e, n, c in ladder]
            for i in range(1, len(run)):
                run[i].rate = math.log2(run[i - 1].l2_error / run[i].l2_error)
            rows += run
    return rows


def _g(v: float) -> str:
    return "%.17g" % v


def emit_csv(rows: List[ConvergenceRow], out=None) -> str:
    """harness.cpp:296-304 (same header, column order and %.17g formatting)."""
    buf = io.StringIO()
    buf.write(HEADER + "\n")
    for r in rows:
        buf.write(",".join([str(r.mesh_exp), _g(r.h), _g(r.tau), _g(r.l2_error), "" if r.rate is None else _g(r.rate),
                            str(r.iterations), _g(r.wall_seconds), r.method, _g(r.gamma), r.scheme]) + "\n")
    text = buf.getvalue()
    if out is not None:
        out.write(text)
    return text


def emit_markdown(rows: List[ConvergenceRow], out=None) -> str:
    """harness.cpp:306-316 (table form)."""
    lines = ["| mesh | h | tau | L2 error | rate | iters | seconds | method | gamma | scheme |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        lines.append(f"| 2^-{r.mesh_exp} | {r.h:.6g} | {r.tau:.6g} | {r.l2_error:.6e} | "
                     f"{'' if r.rate is None else f'{r.rate:.4f}'} | {r.iterations} | {r.wall_seconds:.4g} | "
                     f"{r.method} | {r.gamma:g} | {r.scheme} |")
    text = "\n".join(lines) + "\n"
    if out is not None:
        out.write(text)
    return text


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--example", type=int, required=True, choices=(2, 3, 4))
    ap.add_argument("--gamma", type=float, nargs="+", required=True)
    ap.add_argument("--levels", default="3..8", help="exponent range A..B (mesh 2^-A .. 2^-B)")
    ap.add_argument("--fixed-tau-exp", type=int, default=None)
    ap.add_argument("--method", nargs="+", default=["fast"], choices=("fast", "direct"))
    ap.add_argument("--format", default="csv", choices=("csv", "markdown"))
    a = ap.parse_args(argv)
    lo, hi = (int(v) for v in a.levels.split(".."))
    methods = [SolveMethod.Fast if m == "fast" else SolveMethod.Direct for m in a.method]
    rows = run_convergence(a.example, a.gamma, exponent_ladder(lo, hi, a.fixed_tau_exp), methods)
    (emit_csv if a.format == "csv" else emit_markdown)(rows, sys.stdout)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
