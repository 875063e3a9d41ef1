"""Optimiser loop on top of the batched evolution.

CPU tests drive paper_2110_03963_b200.optimize with a stand-in plan whose evolve_batch is the
CPU oracle (host logic only); the GPU test runs the real plan.  Pin: for the ring C_n (n >= 8)
the p = 1 QAOA optimum cuts 3/4 of the edges (2-regular graphs: <C>/|E| = 3/4), i.e.
min f = -3n/4 with q = -cut."""
import math

import numpy as np
import pytest

import oracle as O
from paper_2110_03963_b200.optimize import central_difference_sets, minimize, objective_and_gradient


class _OraclePlan:
    def __init__(self, n, q, u=None, v=None):
        self.n, self.q, self.u, self.v = n, q, u, v

    def evolve_batch(self, thetas):
        return np.array([O.expectation(O.evolve_x(self.n, self.q, th), self.q) for th in thetas])

    def evolve_ex_batch(self, thetas):
        return np.array([O.expectation(O.evolve_ex(self.n, self.u, self.v, None, th), self.q) for th in thetas])


def _ring(n):
    return np.arange(n), (np.arange(n) + 1) % n


def test_central_difference_sets_order():
    th = np.array([0.1, 0.2, 0.3, 0.4])
    S = central_difference_sets(th, 1e-3)
    assert S.shape == (9, 4)
    assert np.all(S[0] == th)
    for k in range(4):
        d = np.zeros(4)
        d[k] = 1e-3
        assert np.allclose(S[1 + 2 * k], th + d) and np.allclose(S[2 + 2 * k], th - d)


def test_gradient_matches_analytic_ring():
    """The batched central difference (one evolve_batch of 2k+1 sets) equals an independent
    larger-step difference of the oracle objective (the analytic ring derivative is pinned on the
    oracle itself by P13 in test_oracle_pins.py)."""
    n = 8
    u, v = _ring(n)
    q = O.maxcut_q(n, u, v)
    plan = _OraclePlan(n, q)
    th = np.array([0.4, 0.3])
    f, g = objective_and_gradient(plan, th, 1e-6)
    # independent second-order finite difference with a larger step on the oracle objective
    def F(t):
        return plan.evolve_batch([t])[0]
    e = 1e-4
    g2 = np.array([(F(th + np.array([e, 0])) - F(th - np.array([e, 0]))) / (2 * e),
                   (F(th + np.array([0, e])) - F(th - np.array([0, e]))) / (2 * e)])
    assert abs(f - F(th)) < 1e-14
    assert np.allclose(g, g2, atol=1e-6)


@pytest.mark.parametrize("method", ["L-BFGS-B", "BFGS"])
def test_minimize_ring_reaches_three_quarters(method):
    n = 8
    u, v = _ring(n)
    q = O.maxcut_q(n, u, v)
    res = minimize(_OraclePlan(n, q), [0.5, 0.4], method=method, maxiter=100)
    assert res.fun <= -0.75 * n + 1e-7, res
    assert res.history[0] > res.fun


def test_minimize_ex_qaoa_ring():
    """ex-QAOA contains QAOA (equal angles, R25), so its p = 1 optimum on the
    ring is at least as good: <= -3n/4."""
    n = 8
    u, v = _ring(n)
    q = O.maxcut_q(n, u, v)
    th0 = np.r_[np.full(n, 0.5), 0.4]
    res = minimize(_OraclePlan(n, q, u, v), th0, maxiter=100, ansatz="ex")
    assert res.fun <= -0.75 * n + 1e-7, res


@pytest.mark.gpu
def test_minimize_ex_on_gpu_plan():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2110_03963_b200 as Q
    n = 14
    u, v = _ring(n)
    with Q.Plan(1 << n, "x", n_qubits=n) as P:
        P.set_qualities_maxcut(u, v)
        res = minimize(P, np.r_[np.full(n, 0.5), 0.4], maxiter=100, ansatz="ex")
    assert res.fun <= -0.75 * n + 1e-7, res


@pytest.mark.gpu
def test_minimize_on_gpu_plan():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2110_03963_b200 as Q
    n = 16
    u, v = _ring(n)
    with Q.Plan(1 << n, "x", n_qubits=n, max_batch=5) as P:
        P.set_qualities_maxcut(u, v)
        res = minimize(P, [0.5, 0.4], maxiter=100)
    assert res.fun <= -0.75 * n + 1e-7, res
