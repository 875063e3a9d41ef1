"""cfg2 (batch of 21 weighted n=20 evolutions): stored fp64 q vs generated q (factorised phase)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2110_03963_b200 as Q
from qva_inputs import make_config
wl = make_config("cfg2")
for always in (False, True, False, True):
    with Q.Plan(wl.dim, "x", n_qubits=wl.n_qubits, max_batch=21, qgen_f64_always=always) as P:
        P.set_qualities_maxcut(wl.edges_u, wl.edges_v, wl.weights)
        for _ in range(3):
            f = P.evolve_batch(wl.batch_thetas)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(10):
            f = P.evolve_batch(wl.batch_thetas)
        torch.cuda.synchronize()
        print("generated" if always else "stored   ", "%.3f ms" % ((time.perf_counter() - t0) * 100), f[0])
