"""n = 33 (128 GiB state) QAOA evaluation time on one GPU (cfg5 family, weighted, p = 2)."""
import sys, time
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2110_03963_b200 as Q
from qva_inputs import make_config
wl = make_config("cfg5", n_override=33)
with Q.Plan(wl.dim, "x", n_qubits=33) as P:
    P.set_qualities_maxcut(wl.edges_u, wl.edges_v, wl.weights)
    for i in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        P.evolve(wl.theta); f = P.expectation()
        dt = time.perf_counter() - t0
        print(f"n=33 p=2 evolve+<Q>: {dt*1e3:.1f} ms  ({wl.dim*2/dt/1e9:.2f} G amp-layers/s)  f={f:.12f}", flush=True)
