"""Seeded synthetic workloads for the five BASELINE.json configs (cfg1..cfg5).

This module is shared by the oracle side (tests, golden scripts, bench.py's
cpu_baseline leg) and the CUDA side (tests, bench.py, smoke).  It holds NONE
of the method's arithmetic: it only draws graphs, weights, angles and
(for cfg3) the quality vector itself, which the config defines as iid N(0,1).
Qualities of the max-cut configs are *not* computed here: each side derives
q_x = -cut_w(x) from the edge list on its own (oracle: plain C loop;
CUDA path: on-device generator).

Recipe:
  numpy SeedSequence(seed).spawn(4) -> streams (graph, weights, angles, q).
  cfg1 seed 1: random 3-regular graph on 10 vertices, unit weights, p=2.
  cfg2 seed 2: G(20, 0.5), weights U(0,1), p=5, 21 central-difference sets, h=1e-6.
  cfg3 seed 3: N = 10! states, q ~ N(0,1), complete-graph Laplacian spectrum, p=4.
  cfg4 seed 4: random 3-regular graph on 30 vertices, unit weights, p=3.
  cfg5 seed 5: random 4-regular graph on 34 vertices, weights U(0,1), p=2
               (weak-scaling family n = 30..34 uses the same recipe).
Angles gamma, beta ~ U(0, pi) (BASELINE.json configs); theta layout
[g1, b1, g2, b2, ...] (reading R7).
The paper's own benchmarks are synthetic too (PAPER.md:1003 Fig. strong caption:
random q and theta); no public dataset is involved.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "Workload", "random_regular_graph", "erdos_renyi_graph", "make_config",
    "fd_batch_thetas", "CONFIG_NAMES",
]

CONFIG_NAMES = ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5")


@dataclass
class Workload:
    name: str
    mixer: str                      # "x" | "circulant"
    dim: int                        # N
    n_qubits: int                   # log2 N for the X mixer, -1 otherwise
    p: int                          # layers
    theta: np.ndarray               # [2p] fp64, [g1,b1,...]
    edges_u: Optional[np.ndarray] = None   # int32 [m]
    edges_v: Optional[np.ndarray] = None   # int32 [m]
    weights: Optional[np.ndarray] = None   # fp64 [m] or None for unit weights
    q: Optional[np.ndarray] = None          # fp64 [N] when the config defines q directly
    lam0: Optional[float] = None            # circulant spectrum (complete graph family)
    lam_rest: Optional[float] = None
    batch_thetas: Optional[np.ndarray] = None  # [B][2p]
    fd_h: Optional[float] = None
    seed: int = 0
    meta: dict = field(default_factory=dict)


def random_regular_graph(n: int, d: int, rng: np.random.Generator, max_tries: int = 10000):
    """Pairing (configuration) model with rejection: uniform random simple d-regular graph.

    Returns (u, v) int32 arrays with u < v, sorted lexicographically."""
    if (n * d) % 2:
        raise ValueError("n*d must be even")
    for _ in range(max_tries):
        stubs = np.repeat(np.arange(n), d)
        rng.shuffle(stubs)
        pairs = stubs.reshape(-1, 2)
        a = np.minimum(pairs[:, 0], pairs[:, 1])
        b = np.maximum(pairs[:, 0], pairs[:, 1])
        if np.any(a == b):
            continue
        key = a * n + b
        if len(np.unique(key)) != len(key):
            continue
        order = np.lexsort((b, a))
        return a[order].astype(np.int32), b[order].astype(np.int32)
    raise RuntimeError("pairing model failed to produce a simple graph")


def erdos_renyi_graph(n: int, p_edge: float, rng: np.random.Generator):
    """G(n, p): for u < v in lexicographic order keep the edge iff U < p_edge."""
    us, vs = [], []
    draws = rng.random(n * (n - 1) // 2)
    k = 0
    for u in range(n):
        for v in range(u + 1, n):
            if draws[k] < p_edge:
                us.append(u)
                vs.append(v)
            k += 1
    return np.asarray(us, np.int32), np.asarray(vs, np.int32)


def fd_batch_thetas(theta: np.ndarray, h: float) -> np.ndarray:
    """Central-difference parameter sets [theta, theta+h e_1, theta-h e_1, ...] (R12)."""
    P = len(theta)
    out = np.empty((2 * P + 1, P), np.float64)
    out[0] = theta
    for k in range(P):
        out[1 + 2 * k] = theta
        out[1 + 2 * k, k] += h
        out[2 + 2 * k] = theta
        out[2 + 2 * k, k] -= h
    return out


def _angles(rng: np.random.Generator, p: int) -> np.ndarray:
    return rng.uniform(0.0, math.pi, size=2 * p).astype(np.float64)


def make_config(name: str, n_override: Optional[int] = None, p_override: Optional[int] = None) -> Workload:
    """Build one of cfg1..cfg5.  n_override re-draws the same family at another size
    (used for the weak-scaling series and for small parity cases)."""
    seeds = {"cfg1": 1, "cfg2": 2, "cfg3": 3, "cfg4": 4, "cfg5": 5}
    if name not in seeds:
        raise KeyError(name)
    seed = seeds[name]
    s_graph, s_w, s_ang, s_q = np.random.SeedSequence(seed).spawn(4)
    g_rng, w_rng, a_rng, q_rng = (np.random.default_rng(s) for s in (s_graph, s_w, s_ang, s_q))

    if name == "cfg1":
        n = n_override or 10
        p = p_override or 2
        u, v = random_regular_graph(n, 3, g_rng)
        return Workload(name, "x", 1 << n, n, p, _angles(a_rng, p), u, v, None, seed=seed)
    if name == "cfg2":
        n = n_override or 20
        p = p_override or 5
        u, v = erdos_renyi_graph(n, 0.5, g_rng)
        w = w_rng.uniform(0.0, 1.0, size=len(u)).astype(np.float64)
        theta = _angles(a_rng, p)
        h = 1e-6
        return Workload(name, "x", 1 << n, n, p, theta, u, v, w,
                        batch_thetas=fd_batch_thetas(theta, h), fd_h=h, seed=seed)
    if name == "cfg3":
        N = n_override or math.factorial(10)
        p = p_override or 4
        q = q_rng.standard_normal(N).astype(np.float64)
        return Workload(name, "circulant", N, -1, p, _angles(a_rng, p), q=q,
                        lam0=0.0, lam_rest=float(N), seed=seed)
    if name == "cfg4":
        n = n_override or 30
        p = p_override or 3
        u, v = random_regular_graph(n, 3, g_rng)
        return Workload(name, "x", 1 << n, n, p, _angles(a_rng, p), u, v, None, seed=seed)
    # cfg5
    n = n_override or 34
    p = p_override or 2
    u, v = random_regular_graph(n, 4, g_rng)
    w = w_rng.uniform(0.0, 1.0, size=len(u)).astype(np.float64)
    return Workload(name, "x", 1 << n, n, p, _angles(a_rng, p), u, v, w, seed=seed)
