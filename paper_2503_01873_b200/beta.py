"""Host-side beta solver: the optimal-accuracy condition for the shift fraction
(beta_solver.hpp / beta_solver.cpp:11-54).  Scalar FP64 arithmetic with exactly
two binary16 roundings; the CLI's ``solve-beta`` and the choice of beta* = 0.984497
 come from here.  Checked against the oracle's restatement and the
paper's Appendix A tables in tests/test_host_surface.py."""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


class SolverDivergenceError(RuntimeError):
    """beta_solver.hpp:14-16."""


def _f16(x: float) -> float:
    return float(np.float16(x))  # one RNE rounding from double


@dataclass
class InvarianceReport:
    beta: float = 0.0
    n: int = 0
    a: float = 0.0           # fl16(1 - beta/n) + b
    b: float = 0.0           # fl16(beta/n)
    inva_ideal: float = 0.0  # beta/(1-beta)
    inva_actual: float = 0.0
    rel_err: float = 0.0


def invariance_parameter(beta: float, n: int) -> InvarianceReport:
    """beta_solver.cpp:11-30."""
    if not (beta > 0.0) or not (beta < 1.0):
        raise ValueError("invariance: beta must lie in (0, 1)")
    if n == 0:
        raise ValueError("invariance: n must be >= 1")
    nd = float(n)
    r = InvarianceReport(beta=beta, n=n)
    r.b = _f16(beta / nd)
    r.a = _f16(1.0 - beta / nd) + r.b
    denom = r.a - r.b * nd
    if denom == 0.0:
        raise ZeroDivisionError("invariance: a - b*n == 0, factor is singular")
    r.inva_actual = r.b * nd / (r.a * denom) + (1.0 - r.a) / r.a
    r.inva_ideal = beta / (1.0 - beta)
    r.rel_err = abs(r.inva_ideal - r.inva_actual) / abs(r.inva_ideal)
    return r


@dataclass
class BetaSolution:
    beta_star: float = 0.0
    iterations: int = 0
    report: InvarianceReport = field(default_factory=InvarianceReport)


def optimal_beta(beta0: float, n: int = 128, tol: float = 1e-8) -> BetaSolution:
    """beta_solver.cpp:32-52: beta <- f/(1 + f), f = inva_actual(beta), until the
    relative change is <= tol; SolverDivergenceError after 10000 iterations."""
    if not (tol > 0.0):
        raise ValueError("optimal_beta: tol must be > 0")
    beta = beta0
    for it in range(1, 10001):
        f = invariance_parameter(beta, n).inva_actual
        nxt = f / (1.0 + f)
        err = abs(nxt - beta) / abs(beta)
        beta = nxt
        if err <= tol:
            return BetaSolution(beta, it, invariance_parameter(beta, n))
    raise SolverDivergenceError("optimal_beta: no convergence after 10000 iterations")
