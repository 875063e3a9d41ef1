"""Times ex-QAOA (qva_evolve_ex) against plain QAOA (qva_evolve) on the cfg4 graph (n = 30, p = 3)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2110_03963_b200 as Q  # noqa: E402
from qva_inputs import make_config  # noqa: E402

wl = make_config("cfg4")
m = len(wl.edges_u)
p = wl.p
rng = np.random.default_rng(5)
with Q.Plan(wl.dim, "x", n_qubits=wl.n_qubits) as P:
    P.set_qualities_maxcut(wl.edges_u, wl.edges_v)
    for name, fn, th in [("qaoa", P.evolve, [wl.theta] * 6),
                         ("ex-qaoa same theta", P.evolve_ex, [rng.uniform(0, np.pi, (m + 1) * p)] * 6),
                         ("ex-qaoa new theta", P.evolve_ex, [rng.uniform(0, np.pi, (m + 1) * p) for _ in range(6)])]:
        ts = []
        for t in th:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn(t)
            f = P.expectation()
            ts.append((time.perf_counter() - t0) * 1e3)
        print(f"{name:20s} ms per evaluation (median of last 4): {np.median(ts[2:]):.2f}  f={f:.6f}")
