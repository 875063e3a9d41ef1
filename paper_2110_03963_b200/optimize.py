"""Variational optimisation on top of the batched evolution.

The paper's workflow minimises the objective f(theta) = <psi(theta)|Q|psi(theta)> with a
gradient-based optimiser ("BFGS ... L-BFGS-B"; the gradient by finite differences
computed in parallel, "forward or central differences"). Here one objective +
gradient evaluation is ONE `qva_evolve_batch` call over the 2*len(theta) + 1 parameter sets
[theta, theta + h e_1, theta - h e_1, ...] (reading R12: central differences, h = 1e-6), so the
parameter sets run as extra coordinates of the same GPU passes and, on several ranks, shard
over the ranks with one all-reduce of the values (COMM-grad-f analogue). The optimiser itself
(scipy.optimize) is host logic; no arithmetic of the state evolution runs here.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np


def central_difference_sets(theta, h: float = 1e-6) -> np.ndarray:
    """[B = 2*len(theta) + 1][len(theta)]: theta, then theta +/- h e_k for k = 1..len(theta)
    (batch order of reading R12)."""
    theta = np.asarray(theta, np.float64)
    k = theta.size
    out = np.repeat(theta[None, :], 2 * k + 1, axis=0)
    for j in range(k):
        out[1 + 2 * j, j] += h
        out[2 + 2 * j, j] -= h
    return out


def objective_and_gradient(plan, theta, h: float = 1e-6, ansatz: str = "qaoa"):
    """(f(theta), central-difference gradient) from one batched evolution.
    ansatz "ex": theta is the ex-QAOA vector (|theta| = (1 + |Sigma|) D) and the
    sets go through evolve_ex_batch."""
    theta = np.asarray(theta, np.float64)
    sets = central_difference_sets(theta, h)
    f = np.asarray(plan.evolve_ex_batch(sets) if ansatz == "ex" else plan.evolve_batch(sets), np.float64)
    g = (f[1::2] - f[2::2]) / (2.0 * h)
    return float(f[0]), g


@dataclass
class OptimizeResult:
    theta: np.ndarray
    fun: float
    nit: int
    nfev: int                       # objective+gradient evaluations (one batched evolution each)
    success: bool
    message: str
    history: List[float] = field(default_factory=list)


def minimize(plan, theta0, method: str = "L-BFGS-B", h: float = 1e-6, maxiter: int = 200,
             gtol: float = 1e-7, bounds=None, callback: Optional[Callable] = None,
             ansatz: str = "qaoa") -> OptimizeResult:
    """Minimise <Q> over theta = [gamma_1, beta_1, ..., gamma_p, beta_p] (reading R7) with a
    quasi-Newton method (BFGS / L-BFGS-B as in PAPER.md:341) and batched central-difference
    gradients. `plan` needs qualities (and the mixer data) set; create it with
    max_batch >= 2 * len(theta0) + 1 so that a gradient is one launch sequence.  ansatz "ex":
    ex-QAOA parameters (per layer one angle per edge term, then t_i)."""
    from scipy.optimize import minimize as sp_minimize

    history: List[float] = []

    def fg(th):
        f, g = objective_and_gradient(plan, th, h, ansatz)
        history.append(f)
        return f, g

    opts = {"maxiter": maxiter, "gtol": gtol}
    res = sp_minimize(fg, np.asarray(theta0, np.float64), jac=True, method=method, bounds=bounds,
                      callback=callback, options=opts)
    return OptimizeResult(theta=np.asarray(res.x), fun=float(res.fun), nit=int(getattr(res, "nit", 0)),
                          nfev=len(history), success=bool(res.success), message=str(res.message),
                          history=history)
