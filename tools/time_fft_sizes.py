"""QWOA evolution times (p=2) at several N: codelet sizes and runtime-planned (generic) ones."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2110_03963_b200 as Q
for N in [3628800, 40320 * 90, 1000003, 5040 * 5040, 2 ** 22 * 3]:
    q = np.random.default_rng(1).standard_normal(N)
    with Q.Plan(N, "circulant") as P:
        P.set_qualities(q)
        P.set_circulant_eigenvalues_const(0.0, float(N))
        ts = []
        for i in range(5):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            P.evolve([0.3, 0.7, 1.1, 0.4]); f = P.expectation()
            ts.append(time.perf_counter() - t0)
        print(f"N={N} shape={Q.qva_circulant_plan_shape(N)['M1']}x{Q.qva_circulant_plan_shape(N)['M2']}: {np.median(ts[2:])*1e3:.3f} ms", flush=True)
