"""Virtual-shard X-mixer evolution time with the exchange fused into the pass store (default) or
run as a transpose pass (QVA_FUSE_EXCHANGE=0)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2110_03963_b200 as Q
from qva_inputs import make_config
for n, G in [(26, 2), (26, 8), (28, 4)]:
    wl = make_config("cfg4", n_override=n)
    with Q.Plan(1 << n, "x", n_qubits=n, virtual_shards=G) as P:
        P.set_qualities_maxcut(wl.edges_u, wl.edges_v)
        for i in range(5):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            P.evolve(wl.theta); f = P.expectation()
            dt = time.perf_counter() - t0
        print(f"n={n} G={G} p={wl.p}: {dt*1e3:.2f} ms  f={f:.12f}", flush=True)
